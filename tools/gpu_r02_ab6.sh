# Working library vs the previous commit's build (alt_prev.so) and the round-2 head (alt_head.so):
# simulator GPU tests, per-set times, config-4 trials/s alternating on one box.
set -x
mkdir -p gpurun_out
L=$PWD/paper_2207_11428_b200/_lib
timeout 900 python -m pytest tests/test_sim_gpu.py tests/test_dropin_gpu.py -q -x > gpurun_out/pytest_sim.txt 2>&1
J4() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline'].get('miso_ms'))"; }
for V in alt_prev libmiso_b200; do
  echo "$V $(MISO_B200_LIB=$L/$V.so timeout 600 python tools/c4_sets.py 2>/dev/null | tail -1)" >> gpurun_out/ab6_sets.txt
done
for i in 1 2; do
  for V in ${AB_LIBS:-alt_prev libmiso_b200}; do
    echo "$V c4 $(MISO_B200_LIB=$L/$V.so timeout 600 python bench.py --config c4 --no-cpu-baseline 2>/dev/null | J4)" >> gpurun_out/ab6.txt
  done
done
