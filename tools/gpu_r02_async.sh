# Asynchronous STP: GPU tests, sync/async identity, synccheck/racecheck of the shipped ring and
# racecheck of the atomic-ring build, config-4/5 A/B against the pre-async build (alt_prev).
set -x
mkdir -p gpurun_out
L=$PWD/paper_2207_11428_b200/_lib
timeout 900 python -m pytest tests/test_sim_gpu.py tests/test_dropin_gpu.py -q -x > gpurun_out/pytest_sim.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/sanitize_synccheck.txt 2>&1
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/sanitize_racecheck.txt 2>&1
MISO_B200_LIB=$L/alt_atomicring.so timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/sanitize_racecheck_atomicring.txt 2>&1
rm -f gpurun_out/ab7*.txt
AB_LIBS="alt_prev libmiso_b200" bash tools/gpu_r02_ab7.sh
