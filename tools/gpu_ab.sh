# A/B the current library against an alternative build ($ALT, a .so path) on the same box.
mkdir -p gpurun_out
cp paper_2207_11428_b200/_lib/libmiso_b200.so /tmp/cur.so
python tools/search_scaling.py > gpurun_out/ab_cur.json 2>&1
cp "$ALT" paper_2207_11428_b200/_lib/libmiso_b200.so
python tools/search_scaling.py > gpurun_out/ab_alt.json 2>&1
cp /tmp/cur.so paper_2207_11428_b200/_lib/libmiso_b200.so
python tools/search_scaling.py > gpurun_out/ab_cur2.json 2>&1
