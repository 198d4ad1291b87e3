# Job records as two aligned 128-byte lines, event-path fields first (alt_jobline.so): parity
# tests against the alternate library, then config 4 / config-5 trials A/B on one box.
set -x
mkdir -p gpurun_out
L=$PWD/paper_2207_11428_b200/_lib
MISO_B200_LIB=$L/alt_jobline.so timeout 900 python -m pytest tests/test_sim_gpu.py tests/test_shard_gpu.py -q -x > gpurun_out/pytest_jobline.txt 2>&1
J4() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline'].get('miso_ms'))"; }
J5() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['trials']['value'])"; }
for i in 1 2; do
  for V in libmiso_b200 alt_jobline; do
    echo "$V c4 $(MISO_B200_LIB=$L/$V.so timeout 600 python bench.py --config c4 --no-cpu-baseline 2>/dev/null | J4)" >> gpurun_out/ab4.txt
    echo "$V c5 $(MISO_B200_LIB=$L/$V.so timeout 900 python bench.py --config c5 --no-cpu-baseline --steps 5 2>/dev/null | J5)" >> gpurun_out/ab4.txt
  done
done
