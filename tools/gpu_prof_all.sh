# ncu --set full captures of the simulator (miso, 1024 seeds; best-static candidates, 256 traces)
# and the predictor (config 3), for profiles/.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/sim_miso -f python tools/sim_one_policy.py miso 1024 > gpurun_out/ncu_sim.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/sim_static -f python tools/sim_static_once.py 256 1 >> gpurun_out/ncu_sim.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:predict_batch -s 2 -c 1 -o gpurun_out/predict -f python bench.py --config c3 --steps 2 --warmup 2 --no-cpu-baseline >> gpurun_out/ncu_sim.log 2>&1
