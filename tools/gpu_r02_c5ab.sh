# Config 5 trials: full vs pruned static search at 8192 seeds (same box), with phase times.
set -x
mkdir -p gpurun_out
MISO_C4_PRUNED_STATIC=0 timeout 900 python bench.py --config c5 --no-cpu-baseline > gpurun_out/c5_full.json 2> gpurun_out/c5_full.err
MISO_C4_PRUNED_STATIC=1 timeout 900 python bench.py --config c5 --no-cpu-baseline > gpurun_out/c5_pruned.json 2> gpurun_out/c5_pruned.err
timeout 900 python tools/c5_phases.py > gpurun_out/c5_phases.txt 2>&1
