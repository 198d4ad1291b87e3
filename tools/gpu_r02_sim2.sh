set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sim_gpu.py tests/test_shard_gpu.py tests/test_dropin_gpu.py tests/test_predict_gpu.py -x -q > gpurun_out/pytest_sim.txt 2>&1
timeout 600 python tools/c4_phases.py > gpurun_out/c4_phases_new.txt 2>&1
MISO_B200_SIM_DRAWS=0 timeout 600 python tools/c4_phases.py > gpurun_out/c4_phases_nodraws.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/sim_miso_r02c -f python tools/sim_one_policy.py miso 1024 > gpurun_out/ncu_sim.log 2>&1
