"""How much data survives in L2 between two passes?  Times a re-read of a
buffer of S MB right after touching it (read or write), L2 flushed before."""
import torch


def t(fn, reps=5):
    ms = []
    for _ in range(reps):
        fn[0]()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn[1]()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return sorted(ms)[len(ms) // 2]


flush = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
for mb in (16, 32, 48, 64, 80, 96, 104, 112, 120, 128, 160):
    x = torch.empty(mb << 20, dtype=torch.uint8, device="cuda")
    x.fill_(1)
    y = torch.empty(mb << 18, dtype=torch.int32, device="cuda")
    cold = t((lambda: flush.fill_(0), lambda: x.view(torch.int32).sum()))
    warm_r = t((lambda: (flush.fill_(0), x.view(torch.int32).sum()), lambda: x.view(torch.int32).sum()))
    warm_w = t((lambda: (flush.fill_(0), x.fill_(2)), lambda: x.view(torch.int32).sum()))
    print(f"{mb:4d} MB  cold {cold*1e3:7.1f}us ({mb/1024/cold*1e3:6.0f} GB/s)  after-read {warm_r*1e3:7.1f}us "
          f"({mb/1024/warm_r*1e3:6.0f} GB/s)  after-write {warm_w*1e3:7.1f}us ({mb/1024/warm_w*1e3:6.0f} GB/s)",
          flush=True)
    del x, y
