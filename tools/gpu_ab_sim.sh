# A/B sim-kernel builds: current lib vs $ALTS (space-separated .so paths) on the same box.
mkdir -p gpurun_out
cp paper_2207_11428_b200/_lib/libmiso_b200.so /tmp/cur.so
echo "cur" >> gpurun_out/ab_sim.txt; python tools/sim_static_once.py 1024 >> gpurun_out/ab_sim.txt 2>&1
for a in $ALTS; do
  cp "$a" paper_2207_11428_b200/_lib/libmiso_b200.so
  echo "$a" >> gpurun_out/ab_sim.txt; python tools/sim_static_once.py 1024 >> gpurun_out/ab_sim.txt 2>&1
done
cp /tmp/cur.so paper_2207_11428_b200/_lib/libmiso_b200.so
