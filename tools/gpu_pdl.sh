mkdir -p gpurun_out
python tools/search_scaling.py > gpurun_out/scaling_contig.json 2>&1
MISO_B200_PIPE_CFG=4 python tools/search_scaling.py > gpurun_out/scaling_rr.json 2>&1
python tools/search_scaling.py > gpurun_out/scaling_contig2.json 2>&1
timeout 900 python -m pytest tests/test_search_gpu.py -x -q > gpurun_out/pytest_contig.txt 2>&1
