mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "rle or orderkey or dstride or giant or gp_ or config2 or all_families" > gpurun_out/pytest_rle.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_rle.log
timeout 600 python tools/microbench.py E3 E2L > gpurun_out/mb_e3.txt 2>&1; grep "^|" gpurun_out/mb_e3.txt | tail -18
timeout 600 python bench.py --workload config2 --steps 20 --warmup 3 > gpurun_out/c2.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/c2.log') if l.startswith('{')][-1]); print(d['device_resident']['value'], d['device_resident']['ms_per_step'], json.dumps(d['roofline']['families']))"
