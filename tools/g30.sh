mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "scan or varchar or tpch_columns or delta or empty" > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_sel.log
timeout 600 python tools/microbench.py SCAN > gpurun_out/mb_scan.txt 2>&1; grep "^|" gpurun_out/mb_scan.txt | tail -7
python -c "
import json
for l in open('gpurun_out/mb_scan.txt'):
    if l.startswith('{'):
        d=json.loads(l); print(d['case'], {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})"
