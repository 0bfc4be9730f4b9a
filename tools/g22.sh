mkdir -p gpurun_out
timeout 600 python tools/microbench.py E3 > gpurun_out/mb_e3.txt 2>&1; grep "^|" gpurun_out/mb_e3.txt | tail -8
timeout 600 python bench.py --workload config2 --steps 20 --warmup 3 > gpurun_out/c2.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/c2.log') if l.startswith('{')][-1]); print(d['device_resident']['value'], d['device_resident']['ms_per_step'], json.dumps(d['roofline']['families']))"
timeout 600 python tools/microbench.py NP --filter "one sub-chunk" > gpurun_out/mb_one.txt 2>&1; grep "^|" gpurun_out/mb_one.txt | tail -3
