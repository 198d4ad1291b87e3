# ncu --set full capture of the search kernel (bench's 1M batch) + launch list.
set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:optimize_ -s 3 -c 1 -o gpurun_out/search_full -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1
