mkdir -p gpurun_out
ncu --set full --import-source on -k regex:scan --launch-skip 0 --launch-count 4 -o gpurun_out/scan_rts -f python tools/microbench.py SCAN --filter "config1 sorted" --steps 1 > gpurun_out/ncu_scan.log 2>&1; tail -3 gpurun_out/ncu_scan.log
ncu --set full --import-source on -k regex:lz4_thread --launch-skip 0 --launch-count 1 -o gpurun_out/lz4_thread -f env CDM_LZ4_G=1 python tools/microbench.py NP --filter "sub=16384" --steps 1 > gpurun_out/ncu_lz4.log 2>&1; tail -3 gpurun_out/ncu_lz4.log
timeout 600 python tools/microbench.py CHR > gpurun_out/mb_chr.txt 2>&1; grep "^|" gpurun_out/mb_chr.txt | tail -6
