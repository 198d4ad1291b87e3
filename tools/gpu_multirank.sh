# Multi-rank bench logic on a single-GPU box: 2 ranks share GPU 0, collectives over gloo.
mkdir -p gpurun_out
export MISO_B200_DIST_BACKEND=gloo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/mr_c2.json 2> gpurun_out/mr_c2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --impl reference --steps 2 --warmup 1 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --config c5 --c5-chunks 8 --c5-seeds 256 --steps 3 --warmup 2 > gpurun_out/mr_c5.json 2> gpurun_out/mr_c5.err
