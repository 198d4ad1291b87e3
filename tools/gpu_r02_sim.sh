# Round 2: the refactored simulator -- GPU tests, then config-4 phase timings.
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sim_gpu.py tests/test_shard_gpu.py -x -q > gpurun_out/pytest_sim.txt 2>&1
timeout 600 python tools/c4_phases.py > gpurun_out/c4_phases_new.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1
