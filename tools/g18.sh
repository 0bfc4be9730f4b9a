mkdir -p gpurun_out
timeout 1200 python bench.py --workload config5 --steps 3 --warmup 1 > gpurun_out/c5.log 2> gpurun_out/c5.err; echo "c5 rc=$?"; python -c "
import json; d=json.loads([l for l in open('gpurun_out/c5.log') if l.startswith('{')][-1]); print(d['value'], d['ms_per_step'], d['e2e']['bar_cr_x_0.8_x_pcie'], d['parity'])"
timeout 1500 python tools/tune.py --sf 10 > gpurun_out/tune.txt 2>&1; echo "tune rc=$?"; tail -8 gpurun_out/tune.txt
