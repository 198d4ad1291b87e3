# Current captures for profiles/: simulate_kernel<miso> (1024 config-4 seeds), the pruned
# best-static search (1024 traces), the full best-static candidates of 256 traces.
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/sim_miso -f python tools/sim_one_policy.py miso 1024 > gpurun_out/ncu_sim.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/sim_pruned -f python tools/sim_pruned_once.py 1024 >> gpurun_out/ncu_sim.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/sim_static -f python tools/sim_static_once.py 256 1 >> gpurun_out/ncu_sim.log 2>&1
