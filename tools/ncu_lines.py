"""Per-source-line instruction / stall-sample shares of one kernel in an ncu report.
usage: ncu_lines.py REPORT KERNEL_REGEX [launch_skip] [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--launch-skip", skip,
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
f_ = None
agg, aggs, srcl = collections.Counter(), collections.Counter(), {}
for x in csv.reader(io.StringIO(out)):
    if len(x) >= 2 and x[0] == "File Path":
        f_ = x[1].split("/")[-1]
        continue
    if len(x) < 9 or x[0] in ("Line No", "Function Name") or x[2] != "-":
        continue
    try:
        ie, sm = float(x[7].replace(",", "")), float(x[4].replace(",", ""))
    except ValueError:
        continue
    key = (f_, int(x[0]))
    agg[key] += ie
    aggs[key] += sm
    srcl[key] = x[1]
tot, ts = sum(agg.values()) or 1, sum(aggs.values()) or 1
print(f"warp instructions {tot:.0f}, stall samples {ts:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{k[0]}:{k[1]} {100 * v / tot:5.1f}% inst {100 * aggs[k] / ts:5.1f}% samp  {srcl[k].strip()[:90]}")
