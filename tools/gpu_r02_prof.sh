# Round 2 evidence: config-4 phase timings, ncu --set full of the simulator (miso 1024 seeds;
# best-static candidates of 256 traces), of one search launch, and the default bench's launch list.
set -x
mkdir -p gpurun_out
timeout 600 python tools/c4_phases.py > gpurun_out/c4_phases.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/sim_miso -f python tools/sim_one_policy.py miso 1024 > gpurun_out/ncu_sim.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/sim_static -f python tools/sim_static_once.py 256 1 >> gpurun_out/ncu_sim.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:optimize_ -s 3 -c 1 -o gpurun_out/search_full -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
