# A/B the search-kernel configurations (MISO_B200_PIPE_CFG) and check cfg 3 parity.
set -x
mkdir -p gpurun_out
python tools/tune_search.py ${CFGS:-0 3 4} > gpurun_out/tune.txt 2>&1
MISO_B200_PIPE_CFG=${TESTCFG:-3} timeout 900 python -m pytest tests/test_search_gpu.py -x -q > gpurun_out/pytest_cfg.txt 2>&1
