"""Per-tile timeline of the look-back kernels (CDM_TRACE): run config 2's batch a few times, summarise."""
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

cols = bench.build_workload(0)
eng = cdm.Engine(0)
decs = []
for name, spec, dtype, width, chunks, _ in cols:
    casc = cdm.Cascade(spec, dtype, width)
    for ch in chunks:
        out, offs = cdm.output_buffers(ch)
        decs.append(cdm.Decode(casc, ch, out, offs, dev_chunk=torch.from_numpy(ch).cuda()))
b = cdm.Batch(eng, decs)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
import time
for _ in range(3):
    flush.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b.launch()
    b.results()
    print("step wall ms %.3f" % ((time.perf_counter() - t0) * 1e3))
rows = [l.strip().split(",") for l in open(path)]
import collections
by = collections.defaultdict(list)
for r in rows:
    by[(r[0], r[1])].append([int(x) for x in r[2:]])
for key, recs in by.items():
    a = np.array(recs[-len(recs) // 3:], dtype=np.float64)  # last launch
    t0 = a[:, 1].min()
    st = (a[:, 1:6] - t0) / 1e3
    print(f"{key}: tiles={len(a)} span={st[:, 4].max():.1f}us")
    print("   median phase durations (us): unpack %.2f scan %.2f lookback %.2f expand %.2f" % tuple(
        np.median(np.diff(st, axis=1), axis=0)))
    print("   start times  p0 %.1f p50 %.1f p100 %.1f | end p50 %.1f p100 %.1f" % (
        st[:, 0].min(), np.median(st[:, 0]), st[:, 0].max(), np.median(st[:, 4]), st[:, 4].max()))
    t5 = (a[:, 7] - t0) / 1e3
    print("   stamp5 (descriptor/window) - start: median %.2fus" % np.median(t5 - st[:, 0]))
    if a.shape[1] > 8:
        t6 = (a[:, 8] - t0) / 1e3
        ok = a[:, 8] > 0
        if ok.any():
            print("   stamp6 - start: median %.2fus" % np.median((t6 - st[:, 0])[ok]))
    lb = st[:, 3] - st[:, 2]
    for q in (0, 10, 50, 90, 99, 100):
        print(f"   lookback p{q}: {np.percentile(lb, q):.2f}us", end="")
    print()
    order = np.argsort(a[:, 0])
    print("   tiles by id: lookback(us) every 64th:", " ".join(f"{lb[i]:.1f}" for i in order[::64]))
