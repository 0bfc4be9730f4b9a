#!/bin/bash
# rle family A/B: bench family times with PDL on/off + trace + cold launch list
mkdir -p gpurun_out
TAG=${1:-ab}
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_${TAG}.log
for pdl in 1 0; do
  CDM_PDL=$pdl timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_${TAG}_pdl$pdl.json 2>/dev/null
  python - <<PY
import json; d=json.load(open("gpurun_out/bench_${TAG}_pdl$pdl.json"))
print("pdl=$pdl value", d["value"], "ms", d["ms_per_step"], "fam", d["roofline"]["families_ms_per_step"], "e2e", d["e2e"]["value"])
PY
done
CDM_SERIAL=1 timeout 300 python tools/trace_rle.py > gpurun_out/trace_${TAG}.txt 2>&1; grep -A2 "('rle'\|('sums'" gpurun_out/trace_${TAG}.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_${TAG}.csv python tools/one_batch.py 3 config2 > /dev/null 2>&1
python - <<PY
import csv, collections
rows=[r for r in csv.DictReader(l for l in open("gpurun_out/launches_${TAG}.csv") if l.startswith('"'))]
t=collections.defaultdict(list)
for r in rows:
    if r["Metric Name"]=="gpu__time_duration.sum": t[r["Kernel Name"].split("(")[0][-40:]].append(float(r["Metric Value"]))
for k,v in t.items(): print("%-42s n=%d last=%s" % (k, len(v), v[-3:]))
PY
