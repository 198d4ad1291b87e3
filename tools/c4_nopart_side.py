import sys, os, json, time
sys.path.insert(0,'.')
import numpy as np, torch
import bench, paper_2207_11428_b200 as miso
runner = bench.TrialRunner(0)
tr = miso.generate_traces_device(runner.ctx[0], np.arange(1024, dtype=np.uint64), 1000, lambda_s=10.0)
(s_alt,) = runner.part.streams(0, 1)   # a second stream on the miso partition
orig = runner.part_st
def t():
    runner(tr); ts=[]
    for _ in range(3):
        torch.cuda.synchronize(); t0=time.perf_counter(); runner(tr); torch.cuda.synchronize(); ts.append(time.perf_counter()-t0)
    return round(sorted(ts)[1]*1e3,1)
out={}
for i in range(2):
    runner.part_st = orig; os.environ["MISO_C4_STAGGER"]="1"; out.setdefault("shipped",[]).append(t())
    runner.part_st = (s_alt, orig[1], orig[2]); os.environ["MISO_C4_STAGGER"]="0"; out.setdefault("nopart_on_miso_side",[]).append(t())
    runner.part_st = (s_alt, orig[1], orig[2]); os.environ["MISO_C4_STAGGER"]="1"; out.setdefault("nopart_on_miso_side_static_after",[]).append(t())
print(json.dumps(out))
