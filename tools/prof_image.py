"""Image-observation kernel driver (timing / ncu).

python tools/prof_image.py [n_images] [view] [reps]
Renders `reps` launches of n images from random valid observations; prints
ms per launch and achieved GB/s.  Under ncu: `-k regex:image_kernel -c 1`.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2312_12044_b200.render import image_observations  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
v = int(sys.argv[2]) if len(sys.argv) > 2 else 5
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
g = torch.Generator(device="cuda").manual_seed(0)
tile = torch.randint(0, 15, (n, v, v), device="cuda", generator=g, dtype=torch.int32)
color = torch.randint(0, 14, (n, v, v), device="cuda", generator=g, dtype=torch.int32)
obs = torch.stack([tile, color], -1).to(torch.uint8)
out = torch.empty((n, 224, 224, 3), dtype=torch.uint8, device="cuda")
image_observations(obs, out=out)
ts = []
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    image_observations(obs, out=out, check=False)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
by = n * (224 * 224 * 3 + 2 * v * v)
print(f"n={n} v={v}: ms", " ".join(f"{t:.3f}" for t in ts), "| GB/s", " ".join(f"{by / t / 1e6:.0f}" for t in ts))
