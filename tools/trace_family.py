"""Timeline of the RLE family (CDM_TRACE) on one config-2 batch: per kernel the start/end distribution and
per-phase medians, all relative to the first rle_sums CTA of the last launch."""
import collections
import os
import sys
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
path = os.path.join(ROOT, "gpurun_out", "trace.csv")
os.environ["CDM_TRACE"] = path
if os.path.exists(path):
    os.remove(path)
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2602_08190_b200 import cdm  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "config2"
cols = bench.build_workload(0, wl)
eng = cdm.Engine(0)
decs = []
for name, spec, dtype, width, chunks, _ in cols:
    if "RLE" not in spec:
        continue
    casc = cdm.Cascade(spec, dtype, width)
    for ch in chunks:
        out, offs = cdm.output_buffers(ch)
        decs.append(cdm.Decode(casc, ch, out, offs, dev_chunk=torch.from_numpy(ch).cuda()))
b = cdm.Batch(eng, decs)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    flush.zero_()
    torch.cuda.synchronize()
    b.launch()
    b.results()
rows = [l.strip().split(",") for l in open(path)]
by = collections.defaultdict(list)
for r in rows:
    by[r[0] + (r[1] if r[0] == "rle" else "")].append([int(x) for x in r[2:]])
# columns: tile, s0, s1, s2, s3, s4, smid, s5, s6
arr = {k: np.array(v[-len(v) // 3:], dtype=np.float64) for k, v in by.items()}
t0 = min(a[:, 1][a[:, 1] > 0].min() for a in arr.values())
for k in ["sums", "rscan"] + sorted(k for k in arr if k.startswith("rle")):
    if k not in arr:
        continue
    a = arr[k]
    rel = lambda c: (a[:, c] - t0) / 1e3
    st, en = rel(1), rel(5)
    print(f"{k:6s} n={len(a):5d} start p0 {st.min():6.1f} p50 {np.median(st):6.1f} p100 {st.max():6.1f} | "
          f"end p50 {np.median(en):6.1f} p100 {en.max():6.1f} us | median dur {np.median(en - st):5.2f}")
    names = {7: "s5", 2: "s1", 3: "s2", 4: "s3"}
    for c, nm in names.items():
        ok = a[:, c] > 0
        if ok.any() and c < a.shape[1]:
            print(f"        {nm} - start median {np.median((rel(c) - st)[ok]):5.2f} us")
