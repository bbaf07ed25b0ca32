bash tools/round_cfg4.sh
bash tools/sweep_libs.sh release ct48 ck3 rs8 fs8 release > gpurun_out/sweep_libs.log 2>&1
