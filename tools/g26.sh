mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "full_size" > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_full.log
for w in 32 128; do CDM_C5_WINDOW=$w timeout 1200 python bench.py --workload config5 --steps 3 --warmup 1 > gpurun_out/c5_$w.log 2> gpurun_out/c5_$w.err; echo "c5 W=$w rc=$?"; python -c "
import json; d=json.loads([l for l in open('gpurun_out/c5_$w.log') if l.startswith('{')][-1]); print(d['value'], d['ms_per_step'], d['e2e']['bar_cr_x_0.8_x_pcie'], d['parity']['mismatches'])"; done
