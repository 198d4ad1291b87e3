# Round-2 baseline on a fresh box: GPU tests, sim phases, and a source-level ncu capture of the
# miso simulation (1024 config-4 seeds) for tools/ncu_lines.py.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1
timeout 600 python tools/c4_phases.py > gpurun_out/c4_phases.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/sim_miso_r02a -f python tools/sim_one_policy.py miso 1024 > gpurun_out/ncu_sim.log 2>&1
