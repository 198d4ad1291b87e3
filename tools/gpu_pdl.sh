mkdir -p gpurun_out
python tools/search_scaling.py > gpurun_out/scaling_dyn.json 2>&1
MISO_B200_STATIC_TILES=1 python tools/search_scaling.py > gpurun_out/scaling_static.json 2>&1
timeout 900 python -m pytest tests/test_search_gpu.py -x -q > gpurun_out/pytest_dyn.txt 2>&1
