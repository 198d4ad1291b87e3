# Alternate library builds (AB_LIBS, default: alt_prev = HEAD, libmiso_b200 = working tree) on one
# box: simulator GPU tests on the working library, per-set times, config-4 and config-5 trials/s.
set -x
mkdir -p gpurun_out
L=$PWD/paper_2207_11428_b200/_lib
LIBS=${AB_LIBS:-alt_prev libmiso_b200}
rm -f gpurun_out/ab7*.txt
timeout 900 python -m pytest tests/test_sim_gpu.py tests/test_dropin_gpu.py -q -x > gpurun_out/pytest_sim.txt 2>&1
J4() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline'].get('miso_ms'))"; }
J5() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['trials']['value'])"; }
for V in $LIBS; do
  echo "$V $(MISO_B200_LIB=$L/$V.so timeout 600 python tools/c4_sets.py 2>/dev/null | tail -1)" >> gpurun_out/ab7_sets.txt
done
for i in 1 2; do
  for V in $LIBS; do
    echo "$V c4 $(MISO_B200_LIB=$L/$V.so timeout 600 python bench.py --config c4 --no-cpu-baseline 2>/dev/null | J4)" >> gpurun_out/ab7.txt
    echo "$V c5 $(MISO_B200_LIB=$L/$V.so timeout 900 python bench.py --config c5 --no-cpu-baseline --steps 3 2>/dev/null | J5)" >> gpurun_out/ab7.txt
  done
done
