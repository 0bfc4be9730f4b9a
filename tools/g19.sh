mkdir -p gpurun_out
ncu --set full -k regex:lz4_thread --launch-count 1 -o gpurun_out/c4_lz4 -f python tools/one_batch.py 1 config4 > gpurun_out/ncu_c4lz4.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_c4lz4.log
python tools/ncu_traffic.py gpurun_out/c4_lz4.ncu-rep profiles/ncu_traffic.json --key=config4:lz4_thread_kernel
