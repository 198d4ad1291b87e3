# Config-1 latency path: predictor GPU tests (incl. the resident decide server), the latency
# probe (tools/decide_probe.cu) and the c1 bench.
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_predict_gpu.py -x -q > gpurun_out/pytest_c1.txt 2>&1
tail -3 gpurun_out/pytest_c1.txt
for i in 1 2; do timeout 60 ./tools/decide_probe.bin 3000 400; done > gpurun_out/probe.txt 2>&1
cat gpurun_out/probe.txt
timeout 300 python bench.py --config c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
cat gpurun_out/bench_c1.json; tail -5 gpurun_out/bench_c1.err
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/sanitize_racecheck.txt 2>&1
echo "racecheck rc=$?"; tail -2 gpurun_out/sanitize_racecheck.txt
