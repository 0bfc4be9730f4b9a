mkdir -p gpurun_out
ncu --set full --import-source on -k regex:lz4_thread --launch-count 1 -o gpurun_out/lz4_thread2 -f python tools/microbench.py NP --filter "sub=16384" --steps 1 > gpurun_out/ncu_lz4.log 2>&1; tail -1 gpurun_out/ncu_lz4.log
ncu --set full --import-source on -k regex:scan_kernel_rts --launch-count 1 -o gpurun_out/scan_rts3 -f python tools/microbench.py SCAN --filter "walk w=8" --steps 1 > gpurun_out/ncu_scan.log 2>&1; tail -1 gpurun_out/ncu_scan.log
