"""Micro-experiment: latency from an H2D memcpy node to a dependent kernel node on another branch of a
CUDA graph (torch capture), under CUPTI.  usage: python tools/graph_lag.py"""
import json
import os
import sys

import torch
from torch.profiler import profile, ProfilerActivity

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
h = [torch.empty(n, dtype=torch.uint8).pin_memory() for n in (3 << 20, 2 << 20, 1 << 20)]
d = [torch.empty(n, dtype=torch.uint8, device="cuda") for n in (3 << 20, 2 << 20, 1 << 20)]
work = [torch.zeros(4 << 20, device="cuda") for _ in range(3)]
origin, cs = torch.cuda.Stream(), torch.cuda.Stream()
lanes = [torch.cuda.Stream() for _ in range(3)]
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=origin):
    ev0 = torch.cuda.Event()
    ev0.record(origin)
    cs.wait_event(ev0)
    for l in lanes:
        l.wait_event(ev0)
    done = []
    for i in range(3):
        with torch.cuda.stream(cs):
            d[i].copy_(h[i], non_blocking=True)
            e = torch.cuda.Event()
            e.record(cs)
            done.append(e)
    for i, l in enumerate(lanes):
        if i == 2:  # lane 2 first runs an unrelated kernel
            with torch.cuda.stream(l):
                work[2].mul_(1.0001)
        l.wait_event(done[i])
        with torch.cuda.stream(l):
            work[i].add_(1.0)
    for l in lanes + [cs]:
        e = torch.cuda.Event()
        e.record(l)
        origin.wait_event(e)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        g.replay()
        torch.cuda.synchronize()
path = os.path.join(ROOT, "gpurun_out", "graph_lag.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
gpu = sorted([e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy")], key=lambda e: e["ts"])
t0 = gpu[-1]["ts"] - 400
for e in gpu:
    if e["ts"] >= gpu[len(gpu) * 2 // 3]["ts"]:
        print(f"{e['ts'] - t0:8.1f} - {e['ts'] + e['dur'] - t0:8.1f} s{e['args'].get('stream')} {e['name'][:50]}")
