# miso at one full wave (3552 seeds = 24 resident blocks x 148 SMs) vs 1024 seeds: what saturates?
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/sim_miso_wave -f python tools/sim_one_policy.py miso 3552 > gpurun_out/ncu_sim2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/sim_miso_1024 -f python tools/sim_one_policy.py miso 1024 >> gpurun_out/ncu_sim2.log 2>&1
