# A/B the working tree's library against _lib/alt_head.so (HEAD) on one box: c4 phases, alternating.
for i in 1 2 3; do
  echo "HEAD"; MISO_B200_LIB=$PWD/paper_2207_11428_b200/_lib/alt_head.so timeout 600 python tools/c4_phases.py 2>&1 | tail -1
  echo "WORK"; timeout 600 python tools/c4_phases.py 2>&1 | tail -1
done
