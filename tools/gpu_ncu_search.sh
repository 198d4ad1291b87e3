# ncu --set full of one search launch under MISO_B200_PIPE_CFG=$CFG (bench's 1M batch).
set -x
mkdir -p gpurun_out
CFG=${CFG:-0}
MISO_B200_PIPE_CFG=$CFG timeout 600 ncu --set full --clock-control none --import-source on -k regex:optimize_ -s 3 -c 1 -o gpurun_out/search_cfg$CFG -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_cfg$CFG.log 2>&1
