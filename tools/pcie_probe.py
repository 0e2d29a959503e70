"""PCIe ceiling of the end-to-end (host-buffer) leg: pinned host -> device and
device -> host copies of c2's 109 MB, alone and both directions at once on
two streams.  python tools/pcie_probe.py"""
import torch, time
n=109<<20
h=torch.empty(n,dtype=torch.uint8).pin_memory(); d=torch.empty(n,dtype=torch.uint8,device='cuda')
h2=torch.empty(n,dtype=torch.uint8).pin_memory(); d2=torch.empty(n,dtype=torch.uint8,device='cuda')
s1=torch.cuda.Stream(); s2=torch.cuda.Stream()
def t(fn,reps=10):
    fn(); torch.cuda.synchronize(); t0=time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter()-t0)/reps
a=t(lambda: d.copy_(h,non_blocking=True)); print('H2D GB/s',n/a/1e9)
b=t(lambda: h2.copy_(d2,non_blocking=True)); print('D2H GB/s',n/b/1e9)
def both():
    with torch.cuda.stream(s1): d.copy_(h,non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2,non_blocking=True)
c=t(both); print('both: per-direction GB/s',n/c/1e9,'total',2*n/c/1e9)
