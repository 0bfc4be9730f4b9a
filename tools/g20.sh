mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "strdict or o_comment or all_families or full_size" > gpurun_out/pytest_sd.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_sd.log
for v in 0 1; do CDM_SD_EXPAND=$v timeout 900 python bench.py --workload strdict --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/sd_$v.log 2>&1; echo "variant $v rc=$?"; python -c "
import json; d=json.loads([l for l in open('gpurun_out/sd_$v.log') if l.startswith('{')][-1]); print(d['device_resident']['value'], json.dumps(d['roofline']['families']))"; done
