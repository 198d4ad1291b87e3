set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/sim_miso_new -f python tools/sim_one_policy.py miso 1024 > gpurun_out/ncu_sim3.log 2>&1
