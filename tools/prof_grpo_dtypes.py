import sys; sys.path.insert(0,'.')
import ctypes, torch
import numpy as np
from paper_2509_18883_b200 import objective as O, _lib as L
dev=torch.device('cuda',0)
V,R=131072,65536
g=np.random.default_rng(0)
b=O.GRPOBatch.pack(g.integers(0,V,R), g.normal(-12,.3,R), g.normal(-12,.3,R), [0,R//2,R],[1.,-1.],[1,1],2,R,device=dev)
for dt in (torch.bfloat16, torch.float32):
    lg=torch.empty((R,V),dtype=dt,device=dev)
    L.call("rlk_synth_normal", L.ptr(lg), L.dtype_code(dt), lg.numel(), 0, 7, 2.0, None, L.stream_handle())
    for _ in range(2): O.grpo_forward_backward(lg,b)
    torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): O.grpo_forward_backward(lg,b)
    e1.record(); torch.cuda.synchronize()
    ms=e0.elapsed_time(e1)/5
    by=R*V*(4 if dt==torch.bfloat16 else 8)
    print(dt, ms, by/ms/1e6, "GB/s")
    del lg; torch.cuda.empty_cache()
