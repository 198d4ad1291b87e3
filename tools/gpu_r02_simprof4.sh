set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/sim_static_new -f python tools/sim_static_once.py 256 1 > gpurun_out/ncu_sim4.log 2>&1
