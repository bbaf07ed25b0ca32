# bench line + ncu launch list + one --set full capture of each hot kernel (cfg3)
set -x
python bench.py > gpurun_out/bench.log 2>&1
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-ooc"
$CMD > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k k_pass1 -s 3 -c 1 -o gpurun_out/full_pass1 $CMD > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k k_d8v -s 3 -c 1 -o gpurun_out/full_d8 $CMD > gpurun_out/ncu_full_d8.log 2>&1
ncu --set full --clock-control none --import-source on -k k_finalize -s 3 -c 1 -o gpurun_out/full_fin $CMD > gpurun_out/ncu_full_fin.log 2>&1
ncu --set full --clock-control none --import-source on -k k_walk -s 3 -c 1 -o gpurun_out/full_walk $CMD > gpurun_out/ncu_full_walk.log 2>&1
echo done
