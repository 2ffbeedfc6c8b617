import sys, time
sys.path.insert(0, '.')
import bench
with bench.ClockSampler(0) as c:
    import torch
    x = torch.randn(8192, 8192, device='cuda')
    for _ in range(20): y = x @ x
    torch.cuda.synchronize()
print(c.summary())
