# ncu --set full of one k_pass2 launch (EVICT) on an 8192^2 cfg3 variant
CMD="python bench.py --rows 8192 --steps 1 --warmup 3 --no-cpu --no-ooc"
export FA_EVICT=1
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pass2 -s 3 -c 1 -o gpurun_out/p2 $CMD > gpurun_out/ncu_p2.log 2>&1
echo done $?
