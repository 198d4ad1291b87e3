# Config-4 schedules: probes (full metrics) then the pruned rest; the static search in chunks.
set -x
mkdir -p gpurun_out
timeout 900 python tools/c4_timeline.py probes > gpurun_out/c4_tl_probes.json 2> gpurun_out/c4_tl_probes.err
timeout 900 python tools/c4_timeline.py chunks > gpurun_out/c4_tl_chunks.json 2> gpurun_out/c4_tl_chunks.err
