# Config 5 trials with the pruned vs the full best-static search (after the per-partition prune bound)
set -x
mkdir -p gpurun_out
J5() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['trials']['value'], d['trials'].get('static_search'))"; }
for i in 1 2; do
  for P in 0 1; do
    echo "pruned=$P c5 $(MISO_C4_PRUNED_STATIC=$P timeout 900 python bench.py --config c5 --no-cpu-baseline --steps 5 2>/dev/null | J5)" >> gpurun_out/c5prune.txt
  done
done
