import time, sys, numpy as np, torch
sys.path.insert(0,'/root/repo')
import paper_2502_00356_b200 as bg
from paper_2502_00356_b200 import besselk
print('raw', torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()), 'cur', torch.cuda.current_stream().cuda_stream)
s=torch.cuda.Stream()
with torch.cuda.stream(s):
    print('in ctx raw', torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()), 'cur', torch.cuda.current_stream().cuda_stream)
n=1<<26
rng=np.random.default_rng(1)
x=140*(1-rng.random(n)); nu=20*(1-rng.random(n))
def run(tag):
    tt=[]
    for k in range(7):
        torch.cuda.synchronize(); t=time.perf_counter(); bg.bessel_k_batch(x,nu); torch.cuda.synchronize(); tt.append(time.perf_counter()-t)
    print(tag, ['%.1f'%(1e3*v) for v in tt])
run('new')
old=besselk._stream_handle
besselk._stream_handle=lambda: torch.cuda.current_stream().cuda_stream
run('old')
besselk._stream_handle=old
run('new again')
