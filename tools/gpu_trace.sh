mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 --fmad=false -I include -DMISO_B200_TRACE=1 tools/trace_search.cu -o /tmp/trace > gpurun_out/trace_build.txt 2>&1
timeout 120 /tmp/trace > gpurun_out/trace.txt 2>&1
