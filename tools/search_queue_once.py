"""One warm-up and one measured miso_b200_optimize_batches launch of Q config-2 steps (1M
mixes each, two input copies alternating, own outputs per step) -- for ncu captures of the
queued search launch (bench.py's headline schedule). usage: search_queue_once.py [Q]"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2207_11428_b200 as miso  # noqa: E402

Q = int(sys.argv[1]) if len(sys.argv) > 1 else 32
sp, off, m = bench.gen_mixes(1000, bench.N_PER_GPU)
ins = [(torch.from_numpy(sp).cuda(), torch.from_numpy(off.view("int32")).cuda()) for _ in range(2)]
n = len(m)
q = [ins[i % 2] + (torch.empty(n, dtype=torch.uint8, device="cuda"),
                   torch.empty(n, dtype=torch.float64, device="cuda")) for i in range(Q)]
ctx = miso.Context(0)
for _ in range(2):
    ctx.optimize_batches(q)
torch.cuda.synchronize()
print("queued launch of", Q, "steps done")
