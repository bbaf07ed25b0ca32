nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/box.txt
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/gputest.txt 2>&1; echo rc=$? >> gpurun_out/gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/gputest.txt 2>&1
timeout 1500 bash tools/round_profile.sh
