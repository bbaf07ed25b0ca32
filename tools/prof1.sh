set -x
CMD="python bench.py --rows 8192 --steps 1 --warmup 3 --no-cpu --no-ooc"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 3 -c 1 -o gpurun_out/p1 $CMD > gpurun_out/ncu_p1.log 2>&1
echo done $?
