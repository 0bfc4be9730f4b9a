mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload config4sd --no-cpu-baseline > gpurun_out/c4sd.log 2> gpurun_out/c4sd.err; echo "c4sd rc=$?"; python -c "
import json; d=json.loads([l for l in open('gpurun_out/c4sd.log') if l.startswith('{')][-1]); print(d['value'], d['e2e']['value'], d['e2e']['bar_cr_x_0.8_x_pcie'], d['config']['compression_ratio'], d['device_resident']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['parity'])"
