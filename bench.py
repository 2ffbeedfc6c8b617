"""Benchmark: env-steps/s of the batched XLand-MiniGrid step on B200.

Contract (one JSON line on rank 0):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c3]
With --gpus N > 1 and no WORLD_SIZE in the environment, bench.py re-launches
itself under torch.distributed.run with N ranks (one GPU each, NCCL; ranks
sharing a GPU fall back to gloo and are only a code-path check).  Each rank
owns a contiguous global env range (parallel.shard_range, weak scaling, no
per-step communication); one all-reduce of the episode statistics runs after
the timed window, and the reported time is the max over ranks of the
device-timed window.

Workload (default "c3", BASELINE.json configs[2]): XLand-MiniGrid-R4-13x13
with the "1m-style" medium table (data/medium-1048576.xmgb, M = 2^20 rows,
reference generator, seed 42; env i runs row i mod M), 2^20 envs per GPU,
random policy (Philox word t of fold_in(key_from_seed(1), i) mod 6),
auto-reset on.  A step is one VecEnv.step over the whole batch (validate +
the step kernels, + a reset-ahead batch every 16th step).  Inputs (state
0.4 GB/GPU + actions) exceed the 126 MB L2.  The timed window always
contains the synchronized budget auto-reset burst (t = 507): when K < 507 it
is placed to straddle it.  Extra windows: a burst-free steady state and one
whole trial from reset (BASELINE.md §3's T = budget + 1).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

WORKLOADS = {
    # name: (env id, benchmark config or None, envs per GPU, BASELINE.json config text)
    "c1": ("MiniGrid-Empty-8x8", None, 1024, "MiniGrid-Empty-8x8 random-policy rollout, 1024 envs"),
    "c2": ("XLand-MiniGrid-R1-9x9", "trivial", 1 << 16, "XLand-MiniGrid-R1-9x9 trivial-style, 2^16 envs"),
    "c3": ("XLand-MiniGrid-R4-13x13", "medium", 1 << 20,
           "XLand-MiniGrid-R4-13x13 medium-1m-style, 2^20 envs/GPU"),
    "c4": ("XLand-MiniGrid-R9-25x25", "high", 1 << 19, "XLand-MiniGrid-R9-25x25 high-1m-style, 2^19 envs/GPU"),
    "doorkey": ("MiniGrid-DoorKey-8x8", None, 1 << 20, "MiniGrid-DoorKey-8x8, 2^20 envs/GPU"),
}
# ruleset table rows per config: C2 trivial 2^16, C3 / C4 "1m-style" 2^20
TABLE_ROWS = {"trivial": 1 << 16, "medium": 1 << 20, "high": 1 << 20}
METRIC = "env-steps/sec (random policy, auto-reset)"


def algorithmic_bytes(h: int, w: int, rules: int, v: int) -> int:
    """SURVEY.md §8(d), read-once-grid model: grid + agent in/out + goal + rule
    slots + action + obs + reward + discount + step type, bytes per env-step."""
    return h * w + 6 + 6 + 4 + 4 * rules + 1 + 2 * v * v + 4 + 4 + 1


def window_bytes(h: int, w: int, rules: int, v: int) -> int:
    """Window-aware model: the same terms with the grid read replaced by the
    bytes a step must read, the flat span of the view window ((v-1) rows of
    the grid plus v cells, ref vecenv.py:481-500), capped at the grid.  The
    physical roofline model for grids much wider than the view (C4: 105 of
    625 bytes)."""
    return min(h * w, (v - 1) * w + v) + 6 + 6 + 4 + 4 * rules + 1 + 2 * v * v + 4 + 4 + 1


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region (NVML:
    one sample on entry, every ~1 ms from a thread, one on exit; nvidia-smi as
    fallback when NVML is unavailable)."""

    def __init__(self, index: int, period_s: float = 0.001):
        self.index = index
        self.period = period_s
        self.sm: list[float] = []
        self.max_sm: float | None = None
        self.reasons: set[str] = set()
        self.errors: list[str] = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nvml = None
        self._h = None

    def _sample(self):
        N, h = self._nvml, self._h
        try:
            self.sm.append(float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)))
            get = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons
            bits = get(h)
            for attr, name in (("HwSlowdown", "hw_slowdown"), ("HwThermalSlowdown", "hw_thermal_slowdown"),
                               ("SwThermalSlowdown", "sw_thermal_slowdown"), ("SwPowerCap", "sw_power_cap"),
                               ("HwPowerBrakeSlowdown", "hw_power_brake_slowdown")):
                k = getattr(N, "nvmlClocksEventReason" + attr, None) or getattr(N, "nvmlClocksThrottleReason" + attr)
                if bits & k:
                    self.reasons.add(name)
        except Exception as exc:  # keep going; report it
            if len(self.errors) < 3:
                self.errors.append(f"{type(exc).__name__}: {exc}")

    def _smi(self):
        try:
            out = subprocess.run(["nvidia-smi", f"--id={self.index}", "--query-gpu=clocks.sm,clocks.max.sm",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
            a, b = (float(x) for x in out.stdout.strip().split(","))
            self.sm.append(a)
            self.max_sm = b
        except Exception as exc:
            if len(self.errors) < 3:
                self.errors.append(f"nvidia-smi: {type(exc).__name__}: {exc}")

    def _run(self):
        while not self._stop.is_set():
            self._sample() if self._nvml else self._smi()
            self._stop.wait(self.period if self._nvml else 0.05)

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self._h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = float(N.nvmlDeviceGetMaxClockInfo(self._h, N.NVML_CLOCK_SM))
            self._nvml = N
            self._sample()
        except Exception as exc:
            self.errors.append(f"nvml init: {type(exc).__name__}: {exc}")
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)
        if self._nvml:
            self._sample()

    def summary(self) -> dict:
        out = {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max_sm,
               "reasons": sorted(self.reasons) if self.sm else ["unsampled"], "samples": len(self.sm)}
        if self.errors:
            out["errors"] = self.errors
        return out


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def table_path(config):
    """The workload's ruleset table: the specified size when it is present,
    else the largest table of the config (named in the JSON line).
    XMG_BENCH_ROWS=<M> picks another size (development comparisons)."""
    from helpers import benchmark_file
    try:
        return benchmark_file(config, int(os.environ.get("XMG_BENCH_ROWS", 0)) or TABLE_ROWS.get(config))
    except FileNotFoundError:
        import glob
        paths = glob.glob(os.path.join(ROOT, "data", f"{config}-*.xmgb"))
        return max(paths, key=lambda p: int(os.path.basename(p)[len(config) + 1:-5]))


_BM_CACHE: dict = {}


def make_workload(name: str, device, n: int, offset: int, **kw):
    from paper_2312_12044_b200 import VecEnv, load_benchmark, make
    env_id, config, _, _ = WORKLOADS[name]
    _, params = make(env_id)
    bm = None
    if config:
        path = table_path(config)
        if path not in _BM_CACHE:
            _BM_CACHE[path] = load_benchmark(path)
        bm = _BM_CACHE[path]
    kw.setdefault("reuse_outputs", True)
    vec = VecEnv(params, n, bm, device=device, global_offset=offset, **kw)
    return params, bm, vec


def window_plan(budget: int, K: int, W: int) -> tuple[int, int]:
    """(untimed steps before the timed window, window start): W warm-up steps,
    then as many untimed steps as put the synchronized budget reset
    (t = budget - 1, the step that ends the first trials) in the middle of a
    K-step window."""
    pre = max(0, (budget - 1) - K // 2 - W) if K < budget else 0
    return pre, W + pre


def cpu_port(name: str, n: int, threads: int):
    """The oracle port (oracle/xmg_oracle.c, OpenMP over `threads`) on the
    workload's first `n` envs, reset, with the random policy's per-env keys."""
    from helpers import oracle_from_table
    from oracle import oracle as O
    from paper_2312_12044_b200 import load_benchmark, make
    from paper_2312_12044_b200.ruleset import TaskTable
    env_id, config, _, _ = WORKLOADS[name]
    _, params = make(env_id)
    if config:
        table = load_benchmark(table_path(config)).task_table()
    else:
        table = TaskTable(np.zeros((1, 4), np.uint32), 0, 0, 0)
    ids = (np.arange(n) % table.num_tasks).astype(np.int64)
    ora = oracle_from_table(params, table, ids, threads)
    ora.reset(O.key_from_seed(0))
    pk = O.philox(np.stack([np.arange(n, dtype=np.uint64), np.zeros(n, np.uint64), np.full(n, 3, np.uint64),
                            np.zeros(n, np.uint64)], axis=1),
                  np.tile(np.array(O.key_from_seed(1), np.uint64), (n, 1)))
    return params, ora, np.ascontiguousarray(pk[:, 0]), np.ascontiguousarray(pk[:, 1])


def port_window(name: str, n: int, start: int, k: int, threads: int) -> dict:
    """The port on the same envs, actions and phase as the GPU's timed window:
    advanced `start` steps untimed, then k steps timed (wall clock)."""
    _, ora, pk0, pk1 = cpu_port(name, n, threads)
    done = 0
    while done < start:
        m = min(64, start - done)
        ora.rollout_random(pk0, pk1, done, m, compute_obs=True)
        done += m
    t0 = time.perf_counter()
    ora.rollout_random(pk0, pk1, start, k, compute_obs=True)
    el = time.perf_counter() - t0
    return {"value": n * k / el, "envs": n, "steps": k, "seconds": el, "start": start}


# ---- the real reference (rulegrid.VecEnv, pure Python + NumPy), installed
# unmodified into baseline/_ref; its process-pool slicing as in
# ref harness.py:169-181 (contiguous slices of one global split_batch,
# reset_with_keys per slice), timed with the wall clock like _time_slice
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _rulegrid_job(job):
    """One worker's slice [lo, hi) of the sample: reset, `start` untimed steps,
    then k timed steps.  Returns the timed wall seconds."""
    env_id, table, lo, hi, start, k = job
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    from rulegrid import VecEnv as RVecEnv
    from rulegrid.benchio import load_benchmark as rload
    from rulegrid.registry import make as rmake
    from rulegrid.rng import draw_block_array, key_from_seed as rkey, philox4_array, split_batch as rsplit
    _, params = rmake(env_id)
    rulesets = None
    if table:
        bm = rload(table)
        m = bm.num_rulesets()
        rulesets = [bm.get_ruleset(i % m) for i in range(lo, hi)]
    vec = RVecEnv(params, hi - lo, rulesets)
    k0, k1 = rsplit(rkey(0), hi)
    vec.reset_with_keys(k0[lo:hi], k1[lo:hi])
    root = rkey(1)
    w = philox4_array(np.arange(lo, hi, dtype=np.uint64), 0, 3, 0, root[0], root[1])  # fold_in(root, i)
    pk0, pk1 = w[0], w[1]

    def actions(t):
        return (draw_block_array(pk0, pk1, t // 4)[t % 4] % np.uint64(6)).astype(np.int64)
    for t in range(start):
        vec.step(actions(t))
    acts = [actions(t) for t in range(start, start + k)]
    t0 = time.perf_counter()
    for a in acts:
        vec.step(a)
    return time.perf_counter() - t0


def rulegrid_window(name: str, per_worker: int, workers: int, start: int, k: int) -> dict | None:
    """rulegrid.VecEnv on `workers` processes x `per_worker` envs (global env
    indices 0 .. workers*per_worker - 1, the same keys, tasks and actions as
    the GPU run), the same phase, k timed steps; env-steps/s over the slowest
    worker (ref harness.py:179-181)."""
    if not os.path.isdir(os.path.join(REF_DIR, "rulegrid")):
        return None
    from concurrent.futures import ProcessPoolExecutor
    env_id, config, _, _ = WORKLOADS[name]
    table = None
    if config:  # the sample's rows (< 2^16) are the same in every size of the config's table
        from helpers import benchmark_file
        table = benchmark_file(config)
    n = per_worker * workers
    jobs = [(env_id, table, w * per_worker, (w + 1) * per_worker, start, k) for w in range(workers)]
    t0 = time.perf_counter()
    if workers == 1:
        secs = [_rulegrid_job(jobs[0])]
    else:
        import multiprocessing as mp
        with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("fork")) as pool:
            secs = list(pool.map(_rulegrid_job, jobs))
    return {"value": n * k / max(secs), "envs": n, "workers": workers, "steps": k, "start": start,
            "seconds": max(secs), "wall_s": time.perf_counter() - t0}


def run_reference(args):
    """The reference arm.  Headline: the oracle port (a C restatement of
    rulegrid.VecEnv, OpenMP over all host threads) on the SAME workload as our
    arm (all envs of the shard, same keys, tasks, actions) and the same K-step
    window (the W warm-up and placement steps run untimed first).  Beside it,
    the reference itself (rulegrid from baseline/_ref) on a sample of the same
    envs and window, with 1 worker and one worker per host core (ref
    harness.py:184-218); the port / reference factor is reported."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    env_id, config, n_gpu, desc = WORKLOADS[args.workload]
    if args.envs:
        n_gpu = args.envs
    from paper_2312_12044_b200 import make
    _, params = make(env_id)
    threads = os.cpu_count() or 1
    K, W = max(args.steps, 1), max(args.warmup, 0)
    _, start = window_plan(params.step_budget, K, W)
    r = port_window(args.workload, n_gpu, start, K, threads)
    value = r["value"]
    sample = (f"all {n_gpu} envs of the workload (same keys, tasks and random-policy actions as the GPU arm), "
              f"steps [{start}, {start + K}) timed after {start} untimed steps ({r['seconds']:.2f} s)")
    rg = None
    if not args.no_rulegrid:
        kr = min(K, args.rulegrid_steps)
        pw = args.rulegrid_envs
        one = rulegrid_window(args.workload, pw, 1, start, kr)
        many = rulegrid_window(args.workload, pw, threads, start, kr) if one and threads > 1 else None
        if one:
            rg = {"impl": "rulegrid.VecEnv (baseline/_ref, unmodified reference)", "per_worker_envs": pw,
                  "steps": kr, "window": f"[{start}, {start + kr})", "workers_1": one, f"workers_{threads}": many,
                  "port_over_reference_1core": None,
                  "note": "process pool of contiguous slices of one global split_batch, reset_with_keys per "
                          "slice (ref harness.py:169-181); wall clock of the timed steps, slowest worker"}
            p1 = port_window(args.workload, min(n_gpu, 1 << 14), start, kr, 1)
            rg["port_1core"] = p1
            rg["port_over_reference_1core"] = p1["value"] / one["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "env-steps/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": 1e3 * r["seconds"] / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": desc, "env": env_id, "rulesets": os.path.relpath(table_path(config), ROOT)
                   if config else None, "envs_per_gpu": n_gpu, "timed_window": f"steps [{start}, {start + K})"},
        "cpu_baseline": {"value": value, "unit": "env-steps/s", "cores": threads, "kind": "port",
                         "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "rulegrid": rg,
        "note": "reference arm = the C port of rulegrid.VecEnv (oracle/xmg_oracle.c) on all host threads, on "
                "exactly the GPU arm's workload and window; `rulegrid` times the reference itself on a sample",
    }
    print(json.dumps(line), flush=True)


def load_traffic(kernel_key: str):
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as fh:
            return json.load(fh).get(kernel_key)
    except Exception:
        return None


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2312_12044_b200 import key_from_seed, policy_keys, random_actions
    from paper_2312_12044_b200.parallel import all_reduce_max, all_reduce_stats, shard_range
    rank, world, local = dist_env()
    # one rank per GPU over NCCL; ranks sharing a GPU (more ranks than
    # devices: only a code-path check, the numbers mean nothing) use gloo with
    # CPU-side collectives, since NCCL refuses two ranks on one device
    ndev = max(torch.cuda.device_count(), 1)
    shared = world > ndev
    dev = torch.device("cuda", (local % ndev) if world > 1 else 0)
    torch.cuda.set_device(dev)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            # the communicator's init lines stay visible on stderr (rank count, devices)
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)

    def coll(t: torch.Tensor) -> torch.Tensor:  # tensor placement the backend reduces
        return t.cpu() if shared else t

    def max_over_ranks(x: float) -> float:
        return float(all_reduce_max(coll(torch.tensor([x], dtype=torch.float64, device=dev))).item())

    env_id, config, n, desc = WORKLOADS[args.workload]
    if args.envs:
        n = args.envs
    offset, n = shard_range(n * world, rank, world)  # weak scaling: n envs per GPU
    params, bm, vec = make_workload(args.workload, dev, n, offset, graph=args.graph)
    budget = params.step_budget
    K, W = args.steps, args.warmup
    pre, start = window_plan(budget, K, W)
    total = start + K
    stream = torch.cuda.current_stream(dev)

    pkeys = policy_keys(key_from_seed(1), n, offset=offset, device=dev)
    actions = random_actions(pkeys, 0, max(total, budget + 2, 100 + min(K, 200)))

    def advance(v, t1, validate=True):
        v.reset(key_from_seed(0))
        for t in range(t1):
            v.step(actions[t], validate=validate)

    def timed(v, t0, k, validate=True):
        """Device ms of steps [t0, t0 + k) on `v` (already at t0), max over ranks."""
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        e0.record(stream)
        for t in range(t0, t0 + k):
            v.step(actions[t], validate=validate)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return max_over_ranks(e0.elapsed_time(e1))

    stats = vec.enable_stats()
    advance(vec, start)
    torch.cuda.synchronize(dev)

    # ---- timed window: K public-API steps, device-resident inputs
    l0 = vec.launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(dev.index if dev.index is not None else 0) as clocks:
        ev0.record(stream)
        for t in range(start, total):
            vec.step(actions[t])
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches = vec.launches - l0
    vec.check()
    ms_max = max_over_ranks(ev0.elapsed_time(ev1))
    value = n * world * K / (ms_max / 1e3)

    # ---- episode statistics: the single collective (NCCL all-reduce, ~24 B)
    tot = all_reduce_stats(coll(vec.episode_stats())).cpu().numpy()
    del stats

    # ---- extra windows on the same envs and actions: a burst-free steady
    # state, and one whole trial from reset (T = budget + 1)
    windows = None
    if not args.no_windows:
        ks = min(K, 200)
        advance(vec, 100)
        st_ms = timed(vec, 100, ks)
        vec.reset(key_from_seed(0))
        tr_ms = timed(vec, 0, budget + 1)
        windows = {"steady": {"steps": f"[100, {100 + ks})", "value": n * world * ks / (st_ms / 1e3),
                              "ms_per_step": st_ms / ks},
                   "trial": {"steps": f"[0, {budget + 1})", "value": n * world * (budget + 1) / (tr_ms / 1e3),
                             "ms_per_step": tr_ms / (budget + 1),
                             "note": "one whole trial from reset incl. its budget reset (BASELINE.md §3)"}}

    # ---- the dominant kernel alone (roofline): the library's profiling hook
    # records CUDA events around step_main and step_rare of each xmg_step on
    # the launching stream (serialising them), on a fresh env driven to the
    # same phase with the same actions; validate off so only the step kernels
    # run.  Separate from the timed window above.
    from paper_2312_12044_b200 import _lib as xlib
    L = xlib.lib()
    advance(vec, start, validate=False)
    torch.cuda.synchronize(dev)
    L.xmg_profile(1)
    for t in range(start, total):
        vec.step(actions[t], validate=False)
    L.xmg_profile(0)
    import ctypes as C
    m_ms, r_ms, nst = C.c_double(), C.c_double(), C.c_int64()
    L.xmg_profile_read(C.byref(m_ms), C.byref(r_ms), C.byref(nst))
    if nst.value:
        main_ms = m_ms.value / nst.value
        rare_ms = r_ms.value / nst.value
    else:  # graph mode: the one fused kernel per step is the whole step
        main_ms, rare_ms = ms_max / K, 0.0
    rules = vec.table.rule_width if params.scenario == "xland" else 0
    h, w, v = params.height, params.width, params.view_size
    bpe = algorithmic_bytes(h, w, rules, v)
    bpw = window_bytes(h, w, rules, v)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = bpw * n / (main_ms / 1e3) / 1e9
    step_gbs = bpw * n * world / (ms_max / K / 1e3) / 1e9 / world
    traffic = load_traffic(f"{args.workload}:step_main:dram_bytes_per_launch")
    if traffic is not None and n != WORKLOADS[args.workload][2]:
        traffic = traffic * n / WORKLOADS[args.workload][2]
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic,
                "kernel": "step_main (streaming one-thread-per-env pass; step_rare drains the queued PUT_DOWN "
                          "events / rebuilds and overlaps the next step_main)",
                "kernel_ms": main_ms, "rare_kernel_ms": rare_ms, "pipelined_step_ms": ms_max / K,
                "bytes_per_env_step": bpw, "bytes_per_launch": bpw * n,
                "bytes_model": "window-aware: SURVEY.md 8(d) terms with the grid read = the view window's flat span "
                               "min(H*W, (v-1)*W + v); bytes per env per launch",
                "step_achieved": step_gbs, "step_frac": step_gbs / peak,
                "step_note": "the whole pipelined step of the timed window (all kernels, incl. the budget-reset "
                             "burst and the reset-ahead batches): bytes_per_env_step x envs / ms_per_step",
                "survey_model": {"bytes_per_env_step": bpe, "achieved": bpe * n / (main_ms / 1e3) / 1e9,
                                 "frac": bpe * n / (main_ms / 1e3) / 1e9 / peak,
                                 "step_frac": bpe * n / (ms_max / K / 1e3) / 1e9 / peak,
                                 "model": "SURVEY.md 8(d) read-once-grid: H*W + 12 + 4 + 4R + 1 + 2v^2 + 9"},
                "timing": "xmg_profile events around each kernel, K steps at the timed window's phase",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)" if peaks
                               else "fallback 6650 GB/s (B200_PROFILING.md)",
                "traffic_note": "ncu dram__bytes_read.sum + dram__bytes_write.sum of one step_main launch "
                                "(profiles/ncu_summary.json, this round's capture)"}
    if traffic is not None:
        roofline["dram_achieved"] = traffic / (main_ms / 1e3) / 1e9
        roofline["dram_frac"] = roofline["dram_achieved"] / peak

    # ---- e2e through the public API with HOST buffers (pinned), per step:
    # H2D of the step's actions, the step, D2H of the whole VecTimeStep.  At
    # the timed window's phase (the env is advanced to it untimed).  The D2H
    # copies run on their own stream (double-buffered pinned slots), so step
    # t+1 computes while the record of step t crosses PCIe.
    e2e = None
    if not args.no_e2e:
        if not vec.graph:
            vec.reuse_outputs = False
            vec._outs = None
        we = min(W, start)  # the last W steps before the window run through this loop untimed (warm-up)
        advance(vec, start - we)
        copy_stream = torch.cuda.Stream(dev)
        ke = min(K, args.e2e_steps)
        host_actions = actions[start - we: start + ke].cpu().pin_memory()
        slots = [(torch.empty((n, v, v, 2), dtype=torch.uint8).pin_memory(),
                  torch.empty(n, dtype=torch.float32).pin_memory(), torch.empty(n, dtype=torch.float32).pin_memory(),
                  torch.empty(n, dtype=torch.int8).pin_memory()) for _ in range(2)]
        done_ev = [torch.cuda.Event(), torch.cuda.Event()]
        dev_act = torch.empty(n, dtype=torch.uint8, device=dev)
        checksum = 0.0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for t in range(we + ke):
            if t == we:  # warm-up done: the timed region starts with the window
                torch.cuda.synchronize(dev)
                if world > 1:
                    dist.barrier()
                e0.record(stream)
            sl = t & 1
            if t >= 2:  # the host consumes step t-2's record before reusing its buffers
                done_ev[sl].synchronize()
                checksum += float(slots[sl][1][0])
            dev_act.copy_(host_actions[t], non_blocking=True)
            ts = vec.step(dev_act)
            stepped = torch.cuda.Event()
            stepped.record(stream)
            copy_stream.wait_event(stepped)
            with torch.cuda.stream(copy_stream):
                for dst, src in zip(slots[sl], (ts.observations, ts.rewards, ts.discounts, ts.step_types)):
                    dst.copy_(src, non_blocking=True)
                    src.record_stream(copy_stream)
                done_ev[sl].record(copy_stream)
            if vec.graph:  # graph mode writes fixed record buffers: the copy precedes the next step
                stream.wait_event(done_ev[sl])
        stream.wait_stream(copy_stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ems = max_over_ranks(e0.elapsed_time(e1))
        e2e = {"value": n * world * ke / (ems / 1e3), "unit": "env-steps/s",
               "h2d_bytes_per_step": n, "d2h_bytes_per_step": n * (2 * v * v + 4 + 4 + 1), "steps": ke,
               "window": f"steps [{start}, {start + ke}) after {we} untimed warm-up steps of the same loop",
               "api": "VecEnv.step with pinned host actions in, full VecTimeStep out (double-buffered pinned "
                      "slots, D2H on a copy stream overlapping the next step), at the timed window's phase"}
        vec.reuse_outputs = True
        vec._outs = None

    # ---- the same K steps through VecEnv.steps (one host call per block of
    # 64 steps; records written to a reused (64, n) trajectory buffer)
    block = None
    if not args.no_block and (n * 2 * v ** 2) % 16 == 0:
        from paper_2312_12044_b200.vecenv import Trajectory
        bk = int(max(1, min(64, 8e9 // (n * (2 * v ** 2 + 9)))))  # record buffer <= 8 GB

        def part(tr, k):  # the first k records of the reused buffer (no allocation in the window)
            return tr if k == bk else Trajectory(tr.observations[:k], tr.rewards[:k], tr.discounts[:k],
                                                 tr.step_types[:k])
        traj = Trajectory(torch.empty((bk, n, v, v, 2), dtype=torch.uint8, device=dev),
                          torch.empty((bk, n), dtype=torch.float32, device=dev),
                          torch.empty((bk, n), dtype=torch.float32, device=dev),
                          torch.empty((bk, n), dtype=torch.int8, device=dev))
        vec.reset(key_from_seed(0))
        t = 0
        while t < start:
            k = min(bk, start - t)
            vec.steps(actions[t:t + k], validate=False, out=part(traj, k))
            t += k
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        while t < total:
            k = min(bk, total - t)
            vec.steps(actions[t:t + k], validate=False, out=part(traj, k))
            t += k
        b1.record(stream)
        torch.cuda.synchronize(dev)
        bms = max_over_ranks(b0.elapsed_time(b1))
        fused_block = vec.aligned_fused_choice()
        block = {"value": n * world * K / (bms / 1e3), "unit": "env-steps/s", "ms_per_step": bms / K,
                 "block_steps": bk, "kernel": "xmg_rollout (fused)" if fused_block else "xmg_steps (per-call kernels)",
                 "note": "VecEnv.steps: the same K steps and actions as the timed window, block_steps per host call "
                         "(its default kernel choice: the fused kernel where it keeps >= 12 warps/SM, else K x the "
                         "per-call kernels), bit-identical to step() (tests/test_rollout_gpu.py)"}
        del traj

    # ---- fused rollout: the same K steps (same actions,
    # same phase) as xmg_rollout launches of `chunk` steps each, state on chip
    # within a launch; per env-step only the trajectory record leaves the SM.
    fused = None
    if not args.no_fused:
        chunk = int(max(1, min(args.fused_chunk, 8e9 // (n * (2 * v ** 2 + 9)))))
        traj = None
        modes = {}
        for mode, rec in (("records", ("observations", "rewards", "discounts", "step_types")), ("stats_only", ())):
            vec.reset(key_from_seed(0))
            if start:
                vec.rollout(start, policy_keys=pkeys, t0=0, record=())
            traj = vec.rollout(chunk, policy_keys=pkeys, t0=start, record=rec) if rec else None  # allocate
            if traj is not None:
                from paper_2312_12044_b200.vecenv import Trajectory as _T

                def rpart(k, tr=traj):  # the first k records of the reused buffer
                    return tr if k == chunk else _T(tr.observations[:k], tr.rewards[:k], tr.discounts[:k],
                                                    tr.step_types[:k])
            vec.reset(key_from_seed(0))
            if start:
                vec.rollout(start, policy_keys=pkeys, t0=0, record=())
            torch.cuda.synchronize(dev)
            if world > 1:
                dist.barrier()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            l1 = vec.launches
            f0.record(stream)
            t = start
            while t < total:
                k = min(chunk, total - t)
                if rec:
                    vec.rollout(k, policy_keys=pkeys, t0=t, record=rec, out=rpart(k))
                else:
                    vec.rollout(k, policy_keys=pkeys, t0=t, record=())
                t += k
            f1.record(stream)
            torch.cuda.synchronize(dev)
            fms = max_over_ranks(f0.elapsed_time(f1))
            bpe_f = (2 * v * v + 9) if rec else 0
            ach = bpe_f * n * K / (fms / 1e3) / 1e9
            modes[mode] = {"value": n * world * K / (fms / 1e3), "ms_per_step": fms / K, "launches": vec.launches - l1,
                           "record_bytes_per_env_step": bpe_f,
                           "achieved_gbs": ach, "frac_of_hbm_peak": ach / peak if bpe_f else None}
        del traj
        fused = {"unit": "env-steps/s", "chunk_steps": chunk, **modes,
                 "kernel": "xmg_rollout (fused)" if vec.aligned_fused_choice() else
                           "xmg_steps (per-call kernels, random_actions per block: VecEnv.rollout's choice here)",
                 "note": "VecEnv.rollout: xmg_rollout (one kernel per chunk of steps, state resident in shared memory "
                         "/ registers, random policy evaluated in-kernel) where it keeps >= 12 warps per SM, else "
                         "the per-call kernels; bit-identical to K VecEnv.step calls "
                         "(tests/test_rollout_gpu.py); same K steps and phase as the timed window; records = "
                         "obs + reward + discount + step type per env-step written to HBM"}

    # ---- 224x224 image observations of one step's
    # records: xmg_image_obs, HBM-write bound (150528 B out per image)
    image = None
    if not args.no_image:
        from paper_2312_12044_b200.render import image_observations
        ni = min(n, 1 << 14)
        obs_src = vec._alloc_out(True)[0][:ni]
        img_out = torch.empty((ni, 224, 224, 3), dtype=torch.uint8, device=dev)
        for _ in range(2):
            image_observations(obs_src, out=img_out, check=False)
        reps = 10
        i0, i1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        i0.record(stream)
        for _ in range(reps):
            image_observations(obs_src, out=img_out, check=False)
        i1.record(stream)
        torch.cuda.synchronize(dev)
        ims = i0.elapsed_time(i1) / reps
        ib = ni * (224 * 224 * 3 + 2 * v * v)
        image = {"images_per_s": ni / (ims / 1e3), "images": ni, "ms_per_launch": ims,
                 "bytes_per_image": 224 * 224 * 3 + 2 * v * v, "achieved_gbs": ib / (ims / 1e3) / 1e9,
                 "frac_of_hbm_peak": ib / (ims / 1e3) / 1e9 / peak,
                 "note": "xmg_image_obs on one step's observations (ref render.py:225-243), output 2.4 GB > L2"}
        del img_out

    # ---- CPU baseline: the port on the same envs and window (rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        r = port_window(args.workload, n, start, K, threads)
        cpu = {"value": r["value"], "unit": "env-steps/s", "cores": threads, "kind": "port",
               "sample": f"all {n} envs of the workload, steps [{start}, {total}) after {start} untimed steps "
                         f"({r['seconds']:.2f} s timed; OpenMP over all host threads)",
               "cpu_model": cpu_model()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "env-steps/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic",
            "config": {"workload": desc, "env": env_id,
                       "rulesets": os.path.relpath(table_path(config), ROOT) if config else None,
                       "table_rows": bm.num_rulesets() if bm is not None else None,
                       "envs_per_gpu": n, "global_envs": n * world,
                       "parallelism": f"env-shard x{world}" + (" (ranks sharing a GPU: code-path check only)"
                                                                 if shared else ""),
                       "timed_window": f"steps [{start}, {total}) incl. budget reset burst at t={budget}",
                       "reset_ahead": bool(vec.reset_ahead),
                       "step_path": "graph: xmg_step_fused (one kernel per step) replayed from a CUDA graph"
                                    if vec.graph else "xmg_step: validate + step_main + step_rare (PDL-overlapped)",
                       "l2": "inputs larger than L2" if n * params.height * params.width > 126e6
                             else "state resident in L2 (small workload)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "windows": windows, "steps_block": block, "fused_rollout": fused, "image_obs": image,
            "clocks": clocks.summary(),
            "episode_stats": {"return_sum": float(tot[0]), "trials": float(tot[1]), "length_sum": float(tot[2])},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def relaunch(args) -> int:
    """--gpus N > 1 without a torchrun environment: start N ranks of this
    script under torch.distributed.run (rendezvous on 127.0.0.1)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1024)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--envs", type=int, default=0, help="override envs per GPU")
    ap.add_argument("--e2e-steps", type=int, default=256)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fused", action="store_true")
    ap.add_argument("--no-image", action="store_true")
    ap.add_argument("--no-block", action="store_true")
    ap.add_argument("--fused-chunk", type=int, default=32)
    ap.add_argument("--no-windows", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="VecEnv(graph=True): one fused kernel per step replayed from a CUDA graph (small batches)")
    ap.add_argument("--no-rulegrid", action="store_true")
    ap.add_argument("--rulegrid-envs", type=int, default=2048, help="envs per rulegrid worker")
    ap.add_argument("--rulegrid-steps", type=int, default=20)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
