# Simulator changes vs the round-2 head build (alt_head.so): simulator GPU tests on the working
# library, then config-4 trials/s alternating the two builds on one box, and the pruning stats.
set -x
mkdir -p gpurun_out
L=$PWD/paper_2207_11428_b200/_lib
timeout 900 python -m pytest tests/test_sim_gpu.py tests/test_dropin_gpu.py -q -x > gpurun_out/pytest_sim.txt 2>&1
J4() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline'].get('miso_ms'))"; }
for i in 1 2; do
  for V in alt_head libmiso_b200; do
    echo "$V c4 $(MISO_B200_LIB=$L/$V.so timeout 600 python bench.py --config c4 --no-cpu-baseline 2>/dev/null | J4)" >> gpurun_out/ab5.txt
  done
done
timeout 600 python tools/prune_eff.py 1024 > gpurun_out/prune_eff3.json 2>&1
