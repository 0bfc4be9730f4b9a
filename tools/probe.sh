#!/bin/bash
# One-shot box probe: GPU count, topology, host cores/RAM, pinned H2D bandwidth.
mkdir -p gpurun_out/probe
nvidia-smi -L > gpurun_out/probe/smi_L.txt 2>&1
nvidia-smi topo -m > gpurun_out/probe/topo.txt 2>&1
lscpu > gpurun_out/probe/lscpu.txt 2>&1
free -g > gpurun_out/probe/free.txt 2>&1
nvidia-smi -q -d CLOCK,POWER > gpurun_out/probe/clocks.txt 2>&1
python - > gpurun_out/probe/h2d.txt 2>&1 <<'PY'
import torch, time
print(torch.cuda.get_device_properties(0))
p = torch.cuda.get_device_properties(0)
print("sms", p.multi_processor_count, "l2", getattr(p, "L2_cache_size", None))
for mb in (8, 64, 256):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    best = 1e9
    for i in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(); d.copy_(h, non_blocking=True); e1.record()
        e1.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(f"h2d {mb} MB: {n/best/1e6:.1f} GB/s")
# store / copy peaks
n = 1 << 30
a = torch.empty(n, dtype=torch.uint8, device="cuda"); b = torch.empty_like(a)
for name, fn in (("fill", lambda: a.fill_(7)), ("copy", lambda: b.copy_(a))):
    best = 1e9
    for i in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
    mult = 1 if name == "fill" else 2
    print(f"{name}: {mult*n/best/1e6:.1f} GB/s")
PY
