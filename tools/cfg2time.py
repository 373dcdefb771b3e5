import sys, time
sys.path.insert(0, '.')
import torch
from bench import Workload, cfg_id
w = Workload(cfg_id('cfg2'), 10)
for _ in range(5):
    w.reset(); w.launch()
torch.cuda.synchronize()
ts=[]
for _ in range(20):
    w.reset()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); w.launch(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
ts.sort(); print('cfg2 ms median', ts[len(ts)//2], 'min', ts[0])
