# quick GPU iteration: parity subset, cfg3 bench line (device path only), one
# --set full capture of $K on the 8192^2 cfg3 variant (NCU=1)
set -x
timeout 900 python -m pytest tests -q -m gpu -x -k "${TESTS:-parity or options or loopback_dem or serpentine}" > gpurun_out/it_tests.log 2>&1
echo tests_rc=$? >> gpurun_out/it_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-ooc --no-cpu > gpurun_out/it_bench.log 2>&1
if [ "${NCU:-0}" = "1" ]; then
  CMD="python bench.py --rows 8192 --steps 1 --warmup 3 --no-cpu --no-ooc"
  ncu --set full --clock-control none --import-source on -k regex:${K:-k_pass1v} -s 3 -c 1 -o gpurun_out/${OUT:-it} $CMD > gpurun_out/it_ncu.log 2>&1
fi
echo done
