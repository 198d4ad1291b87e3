set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_sim_gpu.py tests/test_dropin_gpu.py -x -q -rA > gpurun_out/pytest_prune.txt 2>&1; tail -3 gpurun_out/pytest_prune.txt
grep -E "PASSED|FAILED" gpurun_out/pytest_prune.txt | grep -i "dropin\|experiment" | head
