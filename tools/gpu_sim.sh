set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sim_gpu.py -x -q > gpurun_out/pytest_sim.txt 2>&1
timeout 900 python tools/c4_phases.py > gpurun_out/c4phase.txt 2>&1
