mkdir -p gpurun_out
for pad in 0 28000 56000 75000 110000; do
  echo "pad $pad" >> gpurun_out/simpad.txt
  MISO_SIM_SMEM_PAD=$pad timeout 300 python tools/sim_static_once.py 1024 >> gpurun_out/simpad.txt 2>&1
  MISO_SIM_SMEM_PAD=$pad timeout 300 python tools/sim_static_once.py 1024 >> gpurun_out/simpad.txt 2>&1
done
