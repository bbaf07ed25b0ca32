# compute-sanitizer over tools/sanitize_cases.py: memcheck, racecheck (shared
# memory hazards), synccheck, initcheck; logs in gpurun_out/san_*.log
CS=/usr/local/cuda/bin/compute-sanitizer
python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1
for tool in memcheck synccheck racecheck initcheck; do
  timeout 1500 $CS --tool $tool --target-processes all --print-limit 50 python tools/sanitize_cases.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_rc.log
done
