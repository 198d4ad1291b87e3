set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/sim_miso_cur -f python tools/sim_one_policy.py miso 1024 > gpurun_out/ncu_sim5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/sim_pruned_cur -f python tools/sim_pruned_once.py 1024 >> gpurun_out/ncu_sim5.log 2>&1
