"""Per kernel: DRAM bytes (read + write) from an ncu --set full report -> profiles/ncu_traffic.json.
usage: python tools/ncu_traffic.py gpurun_out/prof_X.ncu-rep [out.json] [--key WORKLOAD:LABEL]
  without --key: per-step sums keyed by kernel name (fp_kernel, rle_sums_kernel, rle_kernel(level0), ...);
  with --key: the DRAM bytes PER LAUNCH (mean over the captured launches) are merged into out.json under
  WORKLOAD:LABEL, the key bench.py looks up for roofline.traffic (e.g. config4:lz4_thread_kernel)."""
import csv
import io
import json
import subprocess
import sys

args = [a for a in sys.argv[1:] if not a.startswith("--key")]
key = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--key=")), None)
rep = args[0]
out = args[1] if len(args) > 1 else "profiles/ncu_traffic.json"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
k, rd, wr, dur = (h.index(x) for x in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                       "gpu__time_duration.sum"))
units = rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
fam = {"fp_kernel": "fp", "fpc_kernel": "fp", "scan_kernel": "scan", "scan_sums_kernel": "scan",
       "scan_kernel_rts": "scan", "scan_kernel_lb": "scan", "rle_sums_kernel": "rle", "rle_kernel": "rle",
       "rle_big_kernel": "rle", "lz4_kernel": "lz4", "lz4_thread_kernel": "lz4", "lz4_group_kernel": "lz4",
       "ans_warp_kernel": "ans", "ans_kernel": "ans", "sd_expand_kernel": "strdict"}
acc = {}
detail = []
for r in rows[2:]:
    full = r[k]
    name = full.split("::")[-1].split("(")[0].split("<")[0]
    if name not in fam:
        continue
    # rle_kernel<TRACE, LIN>: the LIN variant is the level-0 (value lineage) launch in these workloads
    f = "rle_kernel(level0)" if name == "rle_kernel" and ", 1>" in full else name
    b = float(r[rd].replace(",", "")) * scale[units[rd]] + float(r[wr].replace(",", "")) * scale[units[wr]]
    acc[f] = acc.get(f, 0) + b
    detail.append({"kernel": f, "dram_bytes": b, "us": float(r[dur].replace(",", ""))})
if key:
    prev = json.load(open(out)) if __import__("os").path.exists(out) else {}
    n = len(detail)
    per = sum(d["dram_bytes"] for d in detail) / max(n, 1)
    prev[key] = int(per)
    prev.setdefault("_keyed", {})[key] = {"launches_captured": n, "dram_bytes_per_launch": int(per),
                                          "us_per_launch": sum(d["us"] for d in detail) / max(n, 1),
                                          "report": rep}
    json.dump(prev, open(out, "w"), indent=1)
    print(json.dumps(prev[key]))
    sys.exit(0)
res = {f: int(v) for f, v in acc.items()}
res["_detail"] = detail
res["_how"] = ("ncu --set full (cache control on: caches flushed before each replayed kernel), one config-2 device "
               "batch, CDM_SERIAL=1; per kernel, the sum over its launches of dram__bytes_read.sum + "
               "dram__bytes_write.sum")
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
