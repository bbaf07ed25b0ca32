# per-kernel launch list of one bench step (cold-cache, serialised; shares only)
ARGS=${ARGS:-"--steps 1 --warmup 3 --no-cpu --no-ooc"}
python bench.py $ARGS > gpurun_out/launch_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1
echo done $?
