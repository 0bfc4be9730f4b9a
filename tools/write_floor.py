"""Floor for a step that writes N MB after the bench's L2 flush: a torch fill of N MB (one kernel), timed
with CUDA events, after (a) the 256 MiB flush write only and (b) the flush write + a 256 MiB read."""
import sys
import torch

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
for mb in [int(x) for x in (sys.argv[1:] or ["48", "96", "144"])]:
    buf = torch.empty(mb << 20, dtype=torch.uint8, device="cuda")
    for mode in ("dirty", "clean"):
        tot = 0.0
        for k in range(30):
            flush.zero_()
            if mode == "clean":
                clean.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            buf.fill_(7)
            e1.record()
            torch.cuda.synchronize()
            if k >= 5:
                tot += e0.elapsed_time(e1)
        us = tot / 25 * 1e3
        print(f"{mb:4d} MB write after {mode:5s} L2: {us:7.1f} us  {mb * 1.048576 / us * 1e3 / 1e3:6.2f} TB/s")
