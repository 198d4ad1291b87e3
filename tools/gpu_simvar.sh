for mb in 4 6 8; do
  MISO_B200_LIB=$PWD/paper_2207_11428_b200/_lib/libmiso_b200_mb$mb.so timeout 600 python tools/c4_phases.py > gpurun_out/c4phase_mb$mb.txt 2>&1
done
