# bench line + ncu launch list + one --set full capture of each hot kernel (cfg3);
# the captures are exported on the box (details + source pages as CSV) and the
# .ncu-rep files removed, so gpurun_out stays under its copy-back limit
set -x
python bench.py > gpurun_out/bench.log 2>&1
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-ooc"
$CMD > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
for k in k_pass1 k_d8v k_finalize; do
  ncu --set full --clock-control none --import-source on -k $k -s 3 -c 1 -o gpurun_out/full_$k $CMD > gpurun_out/ncu_full_$k.log 2>&1
  ncu -i gpurun_out/full_$k.ncu-rep --page details --csv > gpurun_out/full_${k}_details.csv 2>&1
  ncu -i gpurun_out/full_$k.ncu-rep --page raw --csv > gpurun_out/full_${k}_raw.csv 2>&1
  ncu -i gpurun_out/full_$k.ncu-rep --page source --print-source cuda,sass --csv > gpurun_out/full_${k}_source.csv 2>&1
  gzip -f gpurun_out/full_${k}_source.csv
  rm -f gpurun_out/full_$k.ncu-rep
done
echo done
