"""Device time per step of a config-2 batch restricted to some columns (graph mode, L2 flushed), to see how
the kernel families overlap.  usage: fam_time.py [workload] [colfilter ...]"""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2602_08190_b200 import cdm  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "config2"
cols = bench.build_workload(0, wl)
eng = cdm.Engine(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(64 << 20, dtype=torch.float32, device="cuda")  # 256 MiB read after the flush write
CLEAN = os.environ.get("CLEAN") == "1"
stream = torch.cuda.Stream()
for filt in (sys.argv[2:] or ["all"]):
    decs = []
    for name, spec, dtype, width, chunks, _ in cols:
        if filt != "all" and filt not in name:
            continue
        casc = cdm.Cascade(spec, dtype, width)
        for ch in chunks:
            out, offs = cdm.output_buffers(ch)
            decs.append(cdm.Decode(casc, ch, out, offs, dev_chunk=torch.from_numpy(ch).cuda()))
    b = cdm.Batch(eng, decs)
    b.set_graph(os.environ.get("GRAPH", "1") == "1")
    b.set_timing(os.environ.get("TIMING", "1") == "1")
    for _ in range(5):
        b.launch(stream)
        b.collect_timing()
    b.results(stream)
    b.set_timing(os.environ.get("TIMING", "1") == "1")
    tot = 0.0
    n = 50
    for _ in range(n):
        with torch.cuda.stream(stream):
            flush.zero_()
            if CLEAN:
                clean.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            b.launch(stream)
            e1.record(stream)
        b.collect_timing()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    km = b.kernel_ms()
    print(f"{filt:12s} step {1e3 * tot / n:7.1f} us  families " +
          " ".join(f"{k}={1e3 * v[0] / n:.1f}us" for k, v in km.items() if v[1]))
    b.close()
