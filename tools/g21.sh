mkdir -p gpurun_out
ncu --set full --import-source on -k regex:"sd_" --launch-count 3 -o gpurun_out/sd_p -f python tools/one_batch.py 1 strdict > gpurun_out/ncu_sd.log 2>&1; tail -1 gpurun_out/ncu_sd.log
CDM_SD_EXPAND=1 ncu --set full --import-source on -k regex:"sd_" --launch-count 3 -o gpurun_out/sd_1 -f python tools/one_batch.py 1 strdict > gpurun_out/ncu_sd1.log 2>&1; tail -1 gpurun_out/ncu_sd1.log
