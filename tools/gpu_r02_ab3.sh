# Occupancy of the nopart/optsta simulator kernels (MISO_SIM_MIN_BLOCKS 32 / 24 / 16) with the
# L1 carveout: config 4 and config-5 trials, alternating, same box; then the config-4 timeline.
set -x
mkdir -p gpurun_out
L=$PWD/paper_2207_11428_b200/_lib
J4() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline'].get('miso_ms'))"; }
J5() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['trials'])"; }
for i in 1 2; do
  for V in work alt_mb24 alt_mb16; do
    if [ $V = work ]; then LIB=$L/libmiso_b200.so; else LIB=$L/$V.so; fi
    echo "$V c4 $(MISO_B200_LIB=$LIB timeout 600 python bench.py --config c4 --no-cpu-baseline 2>/dev/null | J4)" >> gpurun_out/ab3.txt
    echo "$V c5 $(MISO_B200_LIB=$LIB timeout 900 python bench.py --config c5 --no-cpu-baseline --steps 5 2>/dev/null | J5)" >> gpurun_out/ab3.txt
  done
done
timeout 900 python tools/c4_timeline.py > gpurun_out/c4_timeline2.json 2> gpurun_out/c4_timeline2.err
