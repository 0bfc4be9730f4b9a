mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_boundary.py -q -x -p no:cacheprovider > gpurun_out/pytest_b.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_b.log
timeout 1200 python bench.py --workload config5 --steps 2 --warmup 1 --ingest 0 --no-cpu-baseline > gpurun_out/c5i.log 2> gpurun_out/c5i.err; echo "c5 ingest rc=$?"; python -c "
import json; d=json.loads([l for l in open('gpurun_out/c5i.log') if l.startswith('{')][-1]); print(d['value'], d['ms_per_step'], d['e2e']['bar_cr_x_0.8_x_pcie'], d['parity']['mismatches'], d['config']['ingest_devices'])"
ncu --set full --import-source on -k regex:scan --launch-count 2 -o gpurun_out/scan_c3 -f python tools/microbench.py SCAN --filter "l_comment" --steps 1 > gpurun_out/ncu_scan.log 2>&1; tail -1 gpurun_out/ncu_scan.log
