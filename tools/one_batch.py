"""Run config 2's device batch a few times (for ncu / compute-sanitizer)."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2602_08190_b200 import cdm  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
workload = sys.argv[2] if len(sys.argv) > 2 else "config2"
if len(sys.argv) > 3:  # override the l_comment LZ4 sub-chunk size
    bench.WORKLOADS[workload]["cols"] = [(n, s.replace("LZ4(sub=16384)", f"LZ4(sub={sys.argv[3]})")) for n, s in bench.WORKLOADS[workload]["cols"]]
cols = bench.build_workload(0, workload)
eng = cdm.Engine(0)
decs = []
for name, spec, dtype, width, chunks, _ in cols:
    casc = cdm.Cascade(spec, dtype, width)
    for ch in chunks:
        out, offs = cdm.output_buffers(ch)
        decs.append(cdm.Decode(casc, ch, out, offs, dev_chunk=torch.from_numpy(ch).cuda()))
b = cdm.Batch(eng, decs)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(reps):
    flush.zero_()
    b.launch()
    b.results()
print("ok")
