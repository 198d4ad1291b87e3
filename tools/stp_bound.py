import sys, json, time
sys.path.insert(0,'.')
import numpy as np, torch
import paper_2207_11428_b200 as miso
ctx=miso.Context(0)
tr=miso.generate_traces_device(ctx, np.arange(1024,dtype=np.uint64),1000,lambda_s=10.0)
opts=miso.SimOptions(policy="miso",cluster_size=100,predictor="noisy")
def t(jct):
    s=torch.cuda.current_stream()
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record(s)
    miso.simulate_batch(ctx,tr,opts,jct_only=jct)
    b.record(s); torch.cuda.synchronize(); return round(a.elapsed_time(b),1)
out={}
for j in (False,True,False,True):
    t(j); out.setdefault(str(j),[]).append(t(j))
print(json.dumps(out))
