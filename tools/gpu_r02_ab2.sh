# Single-writer Ctx updates (CTX_SET) + L1 carveout for the simulator; all-thread empty-barrier
# arrivals for the search ring (alt_allarrive.so): parity tests, racecheck of both, perf A/B.
set -x
mkdir -p gpurun_out
L=$PWD/paper_2207_11428_b200/_lib
timeout 900 python -m pytest tests/test_sim_gpu.py tests/test_search_gpu.py tests/test_shard_gpu.py -q -x > gpurun_out/pytest_ab2.txt 2>&1
timeout 1200 compute-sanitizer --tool racecheck python tools/sanitize_run.py > gpurun_out/race_work.txt 2>&1
MISO_B200_LIB=$L/alt_allarrive.so timeout 1200 compute-sanitizer --tool racecheck python tools/sanitize_run.py > gpurun_out/race_allarrive.txt 2>&1
J() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline'].get('miso_ms', d['roofline'].get('frac')))"; }
for i in 1 2; do
  echo "HEAD c4 $(MISO_B200_LIB=$L/alt_head.so timeout 600 python bench.py --config c4 --no-cpu-baseline 2>/dev/null | J)" >> gpurun_out/ab2.txt
  echo "WORK c4 $(timeout 600 python bench.py --config c4 --no-cpu-baseline 2>/dev/null | J)" >> gpurun_out/ab2.txt
  echo "WORK-carve-1 c4 $(MISO_B200_SIM_CARVEOUT=-1 timeout 600 python bench.py --config c4 --no-cpu-baseline 2>/dev/null | J)" >> gpurun_out/ab2.txt
  echo "WORK c2 $(timeout 600 python bench.py --no-secondary --no-cpu-baseline 2>/dev/null | J)" >> gpurun_out/ab2.txt
  echo "ALLARRIVE c2 $(MISO_B200_LIB=$L/alt_allarrive.so timeout 600 python bench.py --no-secondary --no-cpu-baseline 2>/dev/null | J)" >> gpurun_out/ab2.txt
done
