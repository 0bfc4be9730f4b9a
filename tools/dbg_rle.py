"""Debug: decode one RLE cascade on the GPU without raising, report error bits and the first rows that differ
from the oracle (usage: dbg_rle.py [column] [cascade] [sf] [rows_per_chunk])."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import oracle  # noqa: E402
from paper_2602_08190_b200 import cdm, encoder  # noqa: E402
from paper_2602_08190_b200.inputs import TPCH  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "l_orderkey"
spec = sys.argv[2] if len(sys.argv) > 2 else "RLE|[Delta|RLE|[BitPack,BitPack],BitPack]"
sf = float(sys.argv[3]) if len(sys.argv) > 3 else 0.02
rpc = int(sys.argv[4]) if len(sys.argv) > 4 else 50_001
col = TPCH(sf).column(name)
casc = cdm.Cascade(spec, col.dtype, col.width)
chunks = encoder.encode_chunks(spec, col, rpc)
eng = cdm.Engine(0, n_slots=int(os.environ.get('SLOTS', '4')))
decs = []
for ch in chunks:
    out, offs = cdm.output_buffers(ch)
    out.fill_(0xAB)
    decs.append(cdm.Decode(casc, cdm.pinned(ch), out, offs, dev_chunk=torch.from_numpy(ch).cuda()))
MODE = os.environ.get("MODE", "batch")
if MODE == "engine":
    for d in decs:
        d.dev_chunk = None
    class _B:
        def launch(self):
            if os.environ.get("ONE"):
                self.t = [eng.submit(d) for d in decs]
            else:
                self.t = eng.submit_batch(decs)
        def results(self, raise_on_error=False):
            return [eng.wait(t, raise_on_error=False) for t in self.t]
    b = _B()
else:
    b = cdm.Batch(eng, decs)
reps = int(os.environ.get("REPS", "1"))
for rep in range(reps):
    for d in decs:
        d.dev_out.fill_(0xAB)
    b.launch()
    res = b.results(raise_on_error=False)
    if rep < reps - 1:
        nbad = 0
        for ch, d in zip(chunks, decs):
            exp, _ = oracle.decode_chunk(ch)
            nbad += int((d.dev_out.cpu().numpy()[: exp.size] != exp).sum())
        print("rep", rep, "bad bytes", nbad, [r["error_bits"] for r in res])
for i, (ch, d, r) in enumerate(zip(chunks, decs, res)):
    exp, _ = oracle.decode_chunk(ch)
    got = d.dev_out.cpu().numpy()[: exp.size]
    bad = np.nonzero(got != exp)[0]
    print(f"chunk {i}: {r} mismatching bytes {bad.size}", "first" if bad.size else "", bad[:8] // 8 if bad.size else "")
if len(sys.argv) > 5:
    ci = int(sys.argv[5])
    exp, _ = oracle.decode_chunk(chunks[ci])
    e = exp.view(np.int64)
    g = decs[ci].dev_out.cpu().numpy()[: exp.size].view(np.int64)
    bad = np.nonzero(g != e)[0]
    if bad.size == 0:
        sys.exit(0)
    lo = max(0, bad[0] - 6)
    for k in range(lo, lo + 40):
        print(k, e[k], g[k], "" if e[k] == g[k] else "<<")
