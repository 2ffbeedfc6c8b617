import runpy, sys, numpy as np
sys.argv = ["trace_rare.py"] + sys.argv[1:]
g = runpy.run_path("tools/trace_rare.py")
buf, work = g["buf"], g["work"]
wb = work & (buf[:, 15] > 0) & (buf[:, 18] > 0) & (buf[:, 11] > 0) & (buf[:, 12] > 0)
names = ["valid mask", "select 1", "list", "exact+place", "spawn select"]
cols = [11, 15, 16, 17, 18, 12]
for k in range(1, len(cols)):
    dt = (buf[wb, cols[k]].astype(np.int64) - buf[wb, cols[k - 1]].astype(np.int64)) / 1e3
    print(f"rank {names[k-1]:12s}: median {np.median(dt):.2f} max {dt.max():.2f} us")
