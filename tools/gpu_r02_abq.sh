# Search queue depth A/B: alt_prev (<= 32 batches per launch) vs the working library (<= 64),
# the default headline (50 queued 1M-instance steps), alternating on one box.
mkdir -p gpurun_out
L=$PWD/paper_2207_11428_b200/_lib
rm -f gpurun_out/abq.txt
JQ() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print(d['value'], r['frac'], r['steps_per_launch'], r['one_launch_per_step']['frac'], r['two_streams']['frac'])"; }
for i in 1 2 3; do
  for V in ${AB_LIBS:-alt_prev libmiso_b200}; do
    echo "$V $(MISO_B200_LIB=$L/$V.so timeout 600 python bench.py --no-secondary --no-cpu-baseline 2>/dev/null | JQ)" >> gpurun_out/abq.txt
  done
done
