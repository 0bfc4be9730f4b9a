mkdir -p gpurun_out
timeout 600 python tools/microbench.py NP --filter "lz4" > gpurun_out/mb_np.txt 2>&1; grep "^|" gpurun_out/mb_np.txt | tail -6
CDM_LZ4_L2HINT=1 timeout 600 python tools/microbench.py NP --filter "lz4 sub" > gpurun_out/mb_np_hint.txt 2>&1; grep "^|" gpurun_out/mb_np_hint.txt | tail -3
