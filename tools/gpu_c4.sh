set -x
mkdir -p gpurun_out
timeout 900 python bench.py --config c4 --steps 3 --warmup 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --config c3 --steps 5 --warmup 2 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/sim_full -f python bench.py --config c4 --steps 1 --warmup 0 --seeds 256 --no-cpu-baseline > gpurun_out/ncu_sim.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:predict_batch -s 2 -c 1 -o gpurun_out/pred_full -f python bench.py --config c3 --steps 1 --warmup 2 > gpurun_out/ncu_pred.log 2>&1
