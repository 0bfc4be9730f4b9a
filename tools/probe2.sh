set -x
mkdir -p gpurun_out/probe2
{ nproc; free -g; cat /proc/meminfo | head -5; ulimit -l; numactl -H; lscpu | head -30; nvidia-smi topo -m; cat /sys/fs/cgroup/memory.max; cat /sys/fs/cgroup/cpu.max; } > gpurun_out/probe2/host.txt 2>&1
python - > gpurun_out/probe2/pin.txt 2>&1 <<'PY'
import torch, time
t=time.time()
bufs=[]
for i in range(6):
    b=torch.empty(4<<30, dtype=torch.uint8).pin_memory(); bufs.append(b)
    print("pinned", 4*(i+1), "GB", time.time()-t, flush=True)
PY
python -m pytest tests -m gpu -x -q > gpurun_out/probe2/pytest.log 2>&1
tail -3 gpurun_out/probe2/pytest.log
