"""GPU timeline of the e2e path (pinned host -> cdm_submit_batch -> cdm_wait) under torch.profiler.

usage: python tools/e2e_timeline.py [workload]   -> prints the last step's copies/kernels relative to its start
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2602_08190_b200 import cdm  # noqa: E402

workload = sys.argv[1] if len(sys.argv) > 1 else "config2"
cols = bench.build_workload(0, workload)
eng = cdm.Engine(0, n_slots=4, slot_bytes=64 << 20, order_policy=1)
sizes = [int(c.size) for (_, _, _, _, chs, _) in cols for c in chs]
pinned_all = torch.empty(sum(sizes), dtype=torch.uint8).pin_memory()
pin_np = pinned_all.numpy()
decs = []
pos = 0
for name, spec, dtype, width, chunks, _ in cols:
    casc = cdm.Cascade(spec, dtype, width)
    for ch in chunks:
        out, offs = cdm.output_buffers(ch)
        pin_np[pos:pos + ch.size] = ch
        decs.append(cdm.Decode(casc, pinned_all[pos:pos + ch.size], out, offs))
        pos += ch.size
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


mode = sys.argv[2] if len(sys.argv) > 2 else "pipeline"
pipe = cdm.Pipeline(eng, decs) if mode == "pipeline" else None
stream = torch.cuda.Stream()


def step():
    flush.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if pipe is not None:
        pipe.launch(stream)
        t1 = time.perf_counter()
        pipe.results()
    else:
        ts = eng.submit_batch(decs)
        t1 = time.perf_counter()
        for t in ts:
            eng.wait(t)
    return (t1 - t0) * 1e6, (time.perf_counter() - t0) * 1e6


for _ in range(5):
    step()
from torch.profiler import profile, ProfilerActivity  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    walls = [step() for _ in range(3)]
path = os.path.join(ROOT, "gpurun_out", f"e2e_trace_{workload}.json")
prof.export_chrome_trace(path)
print("walls (submit_us, total_us):", [(round(a), round(b)) for a, b in walls])
ev = json.load(open(path))["traceEvents"]
gpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
api = [e for e in ev if e.get("ph") == "X" and e.get("cat") == "cuda_runtime"]
# last step = events after the last flush memset/fill kernel
fills = [e for e in gpu if "fill" in e["name"].lower() or e.get("cat") == "gpu_memset"]
t_last = max(e["ts"] + e["dur"] for e in fills) if fills else min(e["ts"] for e in gpu)
last = sorted([e for e in gpu if e["ts"] >= t_last], key=lambda e: e["ts"])
print(f"last step: {len(last)} GPU activities; t=0 at end of flush")
for e in last:
    nm = e["name"]
    nm = nm.split("(")[0][-40:] if e.get("cat") == "kernel" else nm[:40]
    extra = e.get("args", {})
    by = extra.get("bytes", "")
    print(f"  {e['ts'] - t_last:9.1f} +{e['dur']:8.1f}us  s{extra.get('stream', '?'):<3} {nm} {by}")
api_last = sorted([e for e in api if e["ts"] >= t_last - 50], key=lambda e: e["ts"])
from collections import Counter  # noqa: E402
c = Counter()
d = Counter()
for e in api_last:
    c[e["name"]] += 1
    d[e["name"]] += e["dur"]
print("host API calls in the last step (count, total us):")
for k, v in c.most_common():
    print(f"  {k:40s} {v:4d} {d[k]:9.1f}")
