# ncu --set full of one launch of kernel $K (regex) in the cfg3 bench step
K=${K:-k_retain}
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-ooc"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_$K $CMD > gpurun_out/ncu_$K.log 2>&1
echo done $?
