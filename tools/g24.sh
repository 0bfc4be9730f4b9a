mkdir -p gpurun_out
CDM_LZ4_PIPE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "lz4 or varchar or empty or l_comment" > gpurun_out/pytest_lz4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_lz4.log
CDM_LZ4_PIPE=1 timeout 600 python tools/microbench.py NP --filter "lz4" > gpurun_out/mb_np_pipe.txt 2>&1; grep "^|" gpurun_out/mb_np_pipe.txt | tail -6
