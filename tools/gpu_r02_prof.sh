set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_shard_gpu.py -x -q > gpurun_out/pytest_shard.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/sim_miso_r02b -f python tools/sim_one_policy.py miso 1024 > gpurun_out/ncu_sim.log 2>&1
