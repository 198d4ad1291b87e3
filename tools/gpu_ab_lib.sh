# A/B library builds on one box: c4 phases for each _lib/alt_*.so given on the command line
# (and the working tree's library), alternating.
for i in 1 2; do
  for L in "$@"; do
    echo "$L"; MISO_B200_LIB=$PWD/paper_2207_11428_b200/_lib/$L timeout 600 python tools/c4_phases.py 2>&1 | tail -1
  done
  echo "WORK"; timeout 600 python tools/c4_phases.py 2>&1 | tail -1
done
