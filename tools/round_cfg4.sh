# cfg4 evidence on one GPU: the full-width certificate test, one rank's strip
# (16384 x 131072, u64) timed, and a --set full capture of k_pass1<u64> on a
# 4096 x 131072 tile row of the same recipe
set -x
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -k "full_width" > gpurun_out/cfg4_test.txt 2>&1; echo rc=$? >> gpurun_out/cfg4_test.txt
timeout 900 python tools/cfg4_strip.py > gpurun_out/cfg4_strip.json 2> gpurun_out/cfg4_strip.err
CMD="python tools/cfg4_strip.py 4096 131072 1"
ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 3 -c 1 -o gpurun_out/full_cfg4_pass1 $CMD > gpurun_out/ncu_cfg4.log 2>&1
ncu -i gpurun_out/full_cfg4_pass1.ncu-rep --page details --csv > gpurun_out/full_cfg4_pass1_details.csv 2>&1
ncu -i gpurun_out/full_cfg4_pass1.ncu-rep --page raw --csv > gpurun_out/full_cfg4_pass1_raw.csv 2>&1
rm -f gpurun_out/full_cfg4_pass1.ncu-rep
echo done
