# Simulator prefetch change: parity tests, then A/B against the HEAD build on one box.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sim_gpu.py -q -x > gpurun_out/pytest_sim.txt 2>&1
bash tools/gpu_ab_lib.sh alt_head.so > gpurun_out/ab1.txt 2>&1
for i in 1 2; do
  MISO_B200_LIB=$PWD/paper_2207_11428_b200/_lib/alt_head.so timeout 600 python bench.py --config c4 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('HEAD c4', d['value'], d['roofline']['miso_ms'])" >> gpurun_out/ab1.txt
  timeout 600 python bench.py --config c4 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('WORK c4', d['value'], d['roofline']['miso_ms'])" >> gpurun_out/ab1.txt
done
