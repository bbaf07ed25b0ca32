# The checked build (device-side bounds / invariant assertions, FA_CHECKED)
# over the sanitizer case set and the GPU test suite -- this pool's substitute
# for compute-sanitizer, which is closed here.  Logs: gpurun_out/check_*.log
python tools/build_variant.py checked FA_CHECKED=1 > /dev/null
export FA_LIB=paper_1608_04431_b200/libfa_checked.so
python tools/sanitize_cases.py > gpurun_out/check_cases.log 2>&1; echo "cases rc=$?" >> gpurun_out/check_cases.log
timeout 1500 python -m pytest tests -q -m "gpu and not slow" -k "not fullsize" > gpurun_out/check_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/check_tests.log
