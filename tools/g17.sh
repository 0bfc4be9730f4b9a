mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --workload config5 --steps 3 --warmup 1 > gpurun_out/c5.log 2> gpurun_out/c5.err; echo "c5 rc=$?"; tail -c 2500 gpurun_out/c5.log; tail -3 gpurun_out/c5.err
