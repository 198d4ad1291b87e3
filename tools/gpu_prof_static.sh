mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/sim_static -f python tools/sim_static_once.py 256 0 > gpurun_out/ncu_static.log 2>&1
