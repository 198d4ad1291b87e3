mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/sim_full -f python bench.py --config c4 --steps 1 --warmup 0 --seeds 148 --no-cpu-baseline > gpurun_out/ncu_sim.log 2>&1
