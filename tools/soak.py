"""Soak test: many steps of a large batch through the pipelined step (PDL
overlap, per-chunk release), a slice checked against the oracle every step,
the whole batch against a second engine path (fused rollout) at the end.

python tools/soak.py [steps] [n] [env] [config]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from helpers import benchmark_file, oracle_from_table  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2312_12044_b200 import VecEnv, key_from_seed, load_benchmark, make, policy_keys, random_actions  # noqa

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 16
env_name = sys.argv[3] if len(sys.argv) > 3 else "XLand-MiniGrid-R4-13x13"
config = sys.argv[4] if len(sys.argv) > 4 else ("medium" if env_name.startswith("XLand") else None)
_, params = make(env_name)
if config:
    bm = load_benchmark(benchmark_file(config))
    table = bm.task_table()
else:
    from paper_2312_12044_b200.ruleset import TaskTable
    bm = None
    table = TaskTable(np.zeros((1, 4), np.uint32), 0, 0, 0)
vec = VecEnv(params, n, bm, reuse_outputs=True)
root, pol = key_from_seed(123), key_from_seed(456)
vec.reset(root)
w, off = 256, n // 3
ids = (np.arange(off, off + w) % table.num_tasks).astype(np.int64) if config else np.zeros(w, np.int64)
ora = oracle_from_table(params, table, ids)
k0, k1 = O.split_batch((root.hi, root.lo), w, offset=off)
ora.reset_with_keys(k0, k1)
keys = [O.fold_in((pol.hi, pol.lo), off + i) for i in range(w)]
pk0 = np.array([k[0] for k in keys], np.uint64)
pk1 = np.array([k[1] for k in keys], np.uint64)
pk = policy_keys(pol, n, device=vec.device)
t0 = time.time()
chunk = 1024
bad = 0
for c0 in range(0, steps, chunk):
    k = min(chunk, steps - c0)
    acts = random_actions(pk, c0, k)
    ah = O.random_actions(pk0, pk1, c0, k)
    for t in range(k):
        ts = vec.step(acts[t])
        o, r, d, s = ora.step(ah[t])
        sl = slice(off, off + w)
        if not (np.array_equal(ts.step_types[sl].cpu().numpy(), s)
                and np.array_equal(ts.observations[sl].cpu().numpy(), o)
                and np.array_equal(ts.rewards[sl].cpu().numpy(), r.astype(np.float32))):
            bad += 1
            print("MISMATCH at step", c0 + t, flush=True)
            break
    vec.check()
    if bad:
        break
    assert np.array_equal(vec.grids[off:off + w].cpu().numpy(), ora.grids), f"grids at {c0 + k}"
    print(f"steps {c0 + k}: ok ({time.time() - t0:.0f} s)", flush=True)
roll = VecEnv(params, n, bm)
roll.reset(root)
roll.rollout(steps, policy_keys=pk, record=())
same = torch.equal(roll.grids, vec.grids) and torch.equal(roll.state_words(), vec.state_words()) and torch.equal(roll.rng, vec.rng)
print(f"soak {env_name} n={n} steps={steps}: slice vs oracle {'ok' if not bad else 'FAILED'}; "
      f"full batch vs fused rollout {'identical' if same else 'DIFFERENT'}")
sys.exit(0 if (not bad and same) else 1)
