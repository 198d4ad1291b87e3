mkdir -p gpurun_out
for c in 32768 65536 131072 262144 524288; do
  MISO_B200_E2E_CHUNK=$c python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_chunk_$c.json 2>&1
done
