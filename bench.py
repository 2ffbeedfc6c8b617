"""Benchmark: env-steps/s of the batched XLand-MiniGrid step on B200.

Contract (one JSON line on rank 0):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c3]
Under torchrun (N > 1) each rank owns a contiguous global env range (weak
scaling, no per-step communication); one NCCL all-reduce of the episode
statistics runs after the timed window, and the reported time is the max over
ranks of the device-timed window.

Workload (default "c3", BASELINE.json configs[2]): XLand-MiniGrid-R4-13x13
with medium-style rulesets (data/medium-65536.xmgb, reference generator,
seed 42; env i runs row i mod M), 2^20 envs per GPU, random policy (Philox
word t of fold_in(key_from_seed(1), i) mod 6), auto-reset on.  A step is one
VecEnv.step over the whole batch (validate + fused step kernel).  Inputs
(state 0.22 GB/GPU + actions) exceed the 126 MB L2.  The timed window always
contains the synchronized budget auto-reset burst (t = 507): when K < 507 it
is placed to straddle it, which weights resets MORE than steady state.
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
    "c3": ("XLand-MiniGrid-R4-13x13", "medium", 1 << 20, "XLand-MiniGrid-R4-13x13 medium-style, 2^20 envs/GPU"),
    "c4": ("XLand-MiniGrid-R9-25x25", "high", 1 << 19, "XLand-MiniGrid-R9-25x25 high-style, 2^19 envs/GPU"),
    "doorkey": ("MiniGrid-DoorKey-8x8", None, 1 << 20, "MiniGrid-DoorKey-8x8, 2^20 envs/GPU"),
}
METRIC = "env-steps/sec (random policy, auto-reset)"


def algorithmic_bytes(h: int, w: int, rules: int, v: int) -> int:
    """grid + agent in/out + goal + rule slots + action + obs
    + reward + discount + step type, bytes per env-step."""
    return h * w + 6 + 6 + 4 + 4 * rules + 1 + 2 * v * v + 4 + 4 + 1


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


def _allreduce(dist, t, op):
    dist.all_reduce(t, op=op)
    return t


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


def make_workload(name: str, device, n: int, offset: int):
    from helpers import benchmark_file
    from paper_2312_12044_b200 import VecEnv, load_benchmark, make
    env_id, config, _, _ = WORKLOADS[name]
    _, params = make(env_id)
    bm = load_benchmark(benchmark_file(config)) if config else None
    vec = VecEnv(params, n, bm, device=device, global_offset=offset, reuse_outputs=True)
    return params, bm, vec


def cpu_sample(name: str, n_sample: int, threads: int):
    """The oracle port (oracle/xmg_oracle.c, OpenMP over `threads`) on the
    workload restricted to its first `n_sample` envs, reset, with the random
    policy's per-env keys."""
    from helpers import benchmark_file, oracle_from_table
    from oracle import oracle as O
    from paper_2312_12044_b200 import make
    from paper_2312_12044_b200.ruleset import TaskTable, load_benchmark
    env_id, config, _, _ = WORKLOADS[name]
    _, params = make(env_id)
    if config:
        table = load_benchmark(benchmark_file(config)).task_table()
    else:
        table = TaskTable(np.zeros((1, 4), np.uint32), 0, 0, 0)
    ids = (np.arange(n_sample) % table.num_tasks).astype(np.int64)
    ora = oracle_from_table(params, table, ids, threads)
    ora.reset(O.key_from_seed(0))
    keys = [O.fold_in(O.key_from_seed(1), i) for i in range(n_sample)]
    pk0 = np.array([k[0] for k in keys], np.uint64)
    pk1 = np.array([k[1] for k in keys], np.uint64)
    return ora, pk0, pk1


def cpu_reference(name: str, n_sample: int, steps: int, threads: int, budget_s: float = 20.0,
                  min_s: float = 0.0) -> dict:
    """The oracle port on host cores: the sample stepping until `steps` steps
    or `budget_s` seconds (and for at least `min_s` seconds).  Returns
    env-steps/s."""
    ora, pk0, pk1 = cpu_sample(name, n_sample, threads)
    done, t0 = 0, time.perf_counter()
    chunk = 16
    while (done < steps or time.perf_counter() - t0 < min_s) and time.perf_counter() - t0 < budget_s:
        k = chunk if done >= steps else min(chunk, steps - done)
        ora.rollout_random(pk0, pk1, done, k, compute_obs=True)
        done += k
    el = time.perf_counter() - t0
    return {"value": n_sample * done / el, "steps": done, "envs": n_sample, "seconds": el}


def run_reference(args):
    """The reference arm: the oracle port on all host threads, W untimed then
    K timed steps, each step one bounded sample of the workload (n_sample
    envs advanced m env-steps, m sized so the K steps take ~12 s)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    env_id, config, n_gpu, desc = WORKLOADS[args.workload]
    threads = os.cpu_count() or 1
    n_sample = min(n_gpu, 1 << 16)
    ora, pk0, pk1 = cpu_sample(args.workload, n_sample, threads)
    # calibrate (after a first untimed pass: thread start-up, first touch):
    # seconds per env-step pass over the sample, from >= 0.5 s of passes
    ora.rollout_random(pk0, pk1, 0, 16, compute_obs=True)
    done, t0 = 16, time.perf_counter()
    while time.perf_counter() - t0 < 0.5:
        ora.rollout_random(pk0, pk1, done, 16, compute_obs=True)
        done += 16
    per = (time.perf_counter() - t0) / (done - 16)
    # longer passes run faster per env-step (each env's state stays in cache
    # across the pass): re-measure at the pass length the steps will use
    # (capped at ~1 s)
    m = max(16, min(int(12.0 / max(args.steps, 1) / max(per, 1e-9)), int(1.0 / max(per, 1e-9))))
    t0 = time.perf_counter()
    ora.rollout_random(pk0, pk1, done, m, compute_obs=True)
    per = (time.perf_counter() - t0) / m
    done += m
    k_steps, w_steps = max(args.steps, 1), max(args.warmup, 0)
    m = max(1, int(round(12.0 / k_steps / max(per, 1e-9))))
    for _ in range(w_steps):
        ora.rollout_random(pk0, pk1, done, m, compute_obs=True)
        done += m
    t0 = time.perf_counter()
    for _ in range(k_steps):
        ora.rollout_random(pk0, pk1, done, m, compute_obs=True)
        done += m
    el = time.perf_counter() - t0
    value = n_sample * m * k_steps / el
    sample = (f"each step: {n_sample} envs x {m} env-steps of the {desc} workload "
              f"({k_steps} steps in {el:.1f} s after {w_steps} warm-up steps)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "env-steps/s", "n_gpus": args.gpus,
        "steps": k_steps, "warmup": w_steps, "ms_per_step": 1e3 * el / k_steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": desc, "env": env_id, "rulesets": config, "envs_per_gpu": n_gpu,
                   "sample_envs": n_sample, "env_steps_per_step": m},
        "cpu_baseline": {"value": value, "unit": "env-steps/s", "cores": threads, "kind": "port",
                         "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference arm = CPU oracle port of rulegrid.VecEnv (oracle/xmg_oracle.c, OpenMP over host "
                "threads); the Python reference cannot travel to the GPU box",
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
    rank, world, local = dist_env()
    # one rank per GPU over NCCL; ranks sharing a GPU (more ranks than
    # devices: only a code-path check, the numbers mean nothing) use gloo with
    # CPU-side collectives, since NCCL refuses two ranks on one device
    ndev = max(torch.cuda.device_count(), 1)
    shared = world > ndev
    dev = torch.device("cuda", (local % ndev) if world > 1 else 0)
    if world > 1:
        torch.cuda.set_device(dev)
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def coll(t: torch.Tensor) -> torch.Tensor:  # tensor placement the backend reduces
        return t.cpu() if shared else t
    torch.cuda.set_device(dev)
    env_id, config, n, desc = WORKLOADS[args.workload]
    if args.envs:
        n = args.envs
    offset = rank * n
    params, bm, vec = make_workload(args.workload, dev, n, offset)
    budget = params.step_budget
    K, W = args.steps, args.warmup
    pre = max(0, (budget - 1) - K // 2 - W) if K < budget else 0
    total = W + pre + K
    stream = torch.cuda.current_stream(dev)

    vec.reset(key_from_seed(0))
    pkeys = policy_keys(key_from_seed(1), n, offset=offset, device=dev)
    actions = random_actions(pkeys, 0, total)
    stats = vec.enable_stats()
    for t in range(W + pre):
        vec.step(actions[t])
    torch.cuda.synchronize(dev)

    # ---- timed window: K public-API steps, device-resident inputs
    l0 = vec.launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(dev.index if dev.index is not None else 0) as clocks:
        ev0.record(stream)
        for t in range(W + pre, total):
            vec.step(actions[t])
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches = vec.launches - l0
    ms = ev0.elapsed_time(ev1)
    vec.check()
    t_max = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        t_max = _allreduce(dist, coll(t_max), dist.ReduceOp.MAX)
    ms_max = float(t_max.item())
    value = n * world * K / (ms_max / 1e3)

    # ---- episode statistics: the single collective (NCCL all-reduce, ~24 B)
    tot = vec.episode_stats()
    if world > 1:
        tot = _allreduce(dist, coll(tot), dist.ReduceOp.SUM)
    tot = tot.cpu().numpy()

    # ---- the dominant kernel alone (roofline): the library's profiling hook
    # records CUDA events around step_main and step_rare of each xmg_step on
    # the launching stream (serialising them), on a fresh env driven to the
    # same phase with the same actions; validate off so only the two step
    # kernels run.  Separate from the timed window above.
    from paper_2312_12044_b200 import _lib as xlib
    L = xlib.lib()
    params2, _, vec2 = make_workload(args.workload, dev, n, offset)
    vec2.reset(key_from_seed(0))
    for t in range(W + pre):
        vec2.step(actions[t], validate=False)
    torch.cuda.synchronize(dev)
    L.xmg_profile(1)
    for t in range(W + pre, total):
        vec2.step(actions[t], validate=False)
    L.xmg_profile(0)
    import ctypes as C
    m_ms, r_ms, nst = C.c_double(), C.c_double(), C.c_int64()
    L.xmg_profile_read(C.byref(m_ms), C.byref(r_ms), C.byref(nst))
    main_ms = m_ms.value / max(nst.value, 1)
    rare_ms = r_ms.value / max(nst.value, 1)
    del vec2
    rules = vec.table.rule_width if params.scenario == "xland" else 0
    bpe = algorithmic_bytes(params.height, params.width, rules, params.view_size)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = bpe * n / (main_ms / 1e3) / 1e9
    traffic = load_traffic(f"{args.workload}:step_main:dram_bytes_per_launch")
    if traffic is not None and n != WORKLOADS[args.workload][2]:
        traffic = traffic * n / WORKLOADS[args.workload][2]
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic,
                "kernel": "step_main (streaming one-thread-per-env pass; step_rare drains the queued PUT_DOWN "
                          "events / resets and overlaps the next step_main)",
                "kernel_ms": main_ms, "rare_kernel_ms": rare_ms, "pipelined_step_ms": ms_max / K,
                "bytes_per_env_step": bpe, "bytes_per_launch": bpe * n,
                "bytes_model": "SURVEY.md 8(d): H*W + 12 + 4 + 4R + 1 + 2v^2 + 9 (read-once-grid model), per env",
                "timing": "xmg_profile events around each kernel, K steps at the timed window's phase",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)" if peaks
                               else "fallback 6650 GB/s (B200_PROFILING.md)",
                "traffic_note": "ncu dram__bytes_read.sum + dram__bytes_write.sum of one step_main launch "
                                "(profiles/ncu_summary.json)"}
    if traffic is not None:
        # the DRAM bytes step_main actually moves over its measured launch
        # time: where the window reads less than the read-once-grid model
        # (25x25 grids), `frac` is an effective bandwidth and this is the
        # physical one
        roofline["dram_achieved"] = traffic / (main_ms / 1e3) / 1e9
        roofline["dram_frac"] = roofline["dram_achieved"] / peak

    # ---- e2e through the public API with HOST buffers (pinned), per step:
    # H2D of the step's actions, the step, D2H of the whole VecTimeStep.  The
    # D2H copies run on their own stream (fresh output tensors every step,
    # held for the copy with record_stream), so step t+1 computes while the
    # record of step t crosses PCIe.
    e2e = None
    if not args.no_e2e:
        params3, bm3, _ = make_workload(args.workload, dev, 1, offset)
        from paper_2312_12044_b200 import VecEnv as _VecEnv
        vec3 = _VecEnv(params3, n, bm3, device=dev, global_offset=offset, reuse_outputs=False)
        vec3.reset(key_from_seed(0))
        copy_stream = torch.cuda.Stream(dev)
        ke = min(K, args.e2e_steps)
        host_actions = actions[W + pre: W + pre + ke].cpu().pin_memory()
        v = params3.view_size
        slots = [(torch.empty((n, v, v, 2), dtype=torch.uint8).pin_memory(),
                  torch.empty(n, dtype=torch.float32).pin_memory(), torch.empty(n, dtype=torch.float32).pin_memory(),
                  torch.empty(n, dtype=torch.int8).pin_memory()) for _ in range(2)]
        done_ev = [torch.cuda.Event(), torch.cuda.Event()]
        dev_act = torch.empty(n, dtype=torch.uint8, device=dev)
        checksum = 0.0
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for t in range(ke):
            s = t & 1
            if t >= 2:  # the host consumes step t-2's record before reusing its buffers
                done_ev[s].synchronize()
                checksum += float(slots[s][1][0])
            dev_act.copy_(host_actions[t], non_blocking=True)
            ts = vec3.step(dev_act)
            stepped = torch.cuda.Event()
            stepped.record(stream)
            copy_stream.wait_event(stepped)
            with torch.cuda.stream(copy_stream):
                for dst, src in zip(slots[s], (ts.observations, ts.rewards, ts.discounts, ts.step_types)):
                    dst.copy_(src, non_blocking=True)
                    src.record_stream(copy_stream)
                done_ev[s].record(copy_stream)
        stream.wait_stream(copy_stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ems = e0.elapsed_time(e1)
        te = torch.tensor([ems], dtype=torch.float64, device=dev)
        if world > 1:
            te = _allreduce(dist, coll(te), dist.ReduceOp.MAX)
        e2e = {"value": n * world * ke / (float(te.item()) / 1e3), "unit": "env-steps/s",
               "h2d_bytes_per_step": n, "d2h_bytes_per_step": n * (2 * v * v + 4 + 4 + 1), "steps": ke,
               "api": "VecEnv.step with pinned host actions in, full VecTimeStep out (double-buffered pinned "
                      "slots, D2H on a copy stream overlapping the next step)"}
        del vec3

    # ---- the same K steps through VecEnv.steps (one host call and one fused
    # kernel per block of 64 steps, no per-step host round trip; records
    # written to a reused (64, n) trajectory buffer)
    block = None
    if not args.no_block and (n * 2 * params.view_size ** 2) % 16 == 0:
        params5, _, vec5 = make_workload(args.workload, dev, n, offset)
        vec5.reset(key_from_seed(0))
        rec_bytes = n * (2 * params.view_size ** 2 + 9)
        bk = int(max(1, min(64, 8e9 // rec_bytes)))  # record buffer <= 8 GB
        t = 0
        while t < W + pre:
            k = min(bk, W + pre - t)
            vec5.steps(actions[t:t + k], validate=False)
            t += k
        buf = vec5.steps(actions[t:t + 1], validate=False)  # allocate a 1-step record, reused below
        from paper_2312_12044_b200.vecenv import Trajectory
        v = params5.view_size
        traj = Trajectory(torch.empty((bk, n, v, v, 2), dtype=torch.uint8, device=dev),
                          torch.empty((bk, n), dtype=torch.float32, device=dev),
                          torch.empty((bk, n), dtype=torch.float32, device=dev),
                          torch.empty((bk, n), dtype=torch.int8, device=dev))
        del buf
        vec5.reset(key_from_seed(0))
        t = 0
        while t < W + pre:
            k = min(bk, W + pre - t)
            vec5.steps(actions[t:t + k], validate=False, out=traj if k == bk else None)
            t += k
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        while t < total:
            k = min(bk, total - t)
            vec5.steps(actions[t:t + k], validate=False, out=traj if k == bk else None)
            t += k
        b1.record(stream)
        torch.cuda.synchronize(dev)
        bms = b0.elapsed_time(b1)
        tb = torch.tensor([bms], dtype=torch.float64, device=dev)
        if world > 1:
            tb = _allreduce(dist, coll(tb), dist.ReduceOp.MAX)
        bms = float(tb.item())
        fused_block = vec5.aligned_fused_choice()
        block = {"value": n * world * K / (bms / 1e3), "unit": "env-steps/s", "ms_per_step": bms / K,
                 "block_steps": bk, "kernel": "xmg_rollout (fused)" if fused_block else "xmg_steps (per-call kernels)",
                 "note": "VecEnv.steps: the same K steps and actions as the timed window, block_steps per host call "
                         "(its default kernel choice: the fused kernel, xmg_rollout with the given actions, where it "
                         "keeps >= 12 warps/SM, else K x the per-call kernels), bit-identical to step() "
                         "(tests/test_rollout_gpu.py)"}
        del traj, vec5

    # ---- fused rollout: the same K steps (same actions,
    # same phase) as xmg_rollout launches of `chunk` steps each, state on chip
    # within a launch; per env-step only the trajectory record leaves the SM.
    fused = None
    if not args.no_fused:
        params4, _, vec4 = make_workload(args.workload, dev, n, offset)
        vec4.reset(key_from_seed(0))
        vec4.enable_stats()
        chunk = int(max(1, min(args.fused_chunk, 8e9 // (n * (2 * params.view_size ** 2 + 9)))))
        if W + pre:
            vec4.rollout(W + pre, policy_keys=pkeys, t0=0, record=())
        v = params4.view_size
        traj = None
        modes = {}
        for mode, rec in (("records", ("observations", "rewards", "discounts", "step_types")), ("stats_only", ())):
            vec4.reset(key_from_seed(0))
            if W + pre:
                vec4.rollout(W + pre, policy_keys=pkeys, t0=0, record=())
            traj = vec4.rollout(chunk, policy_keys=pkeys, t0=W + pre, record=rec) if rec else None  # warm / allocate
            vec4.reset(key_from_seed(0))
            if W + pre:
                vec4.rollout(W + pre, policy_keys=pkeys, t0=0, record=())
            torch.cuda.synchronize(dev)
            if world > 1:
                dist.barrier()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            l0 = vec4.launches
            f0.record(stream)
            t = W + pre
            while t < total:
                k = min(chunk, total - t)
                if rec:
                    vec4.rollout(k, policy_keys=pkeys, t0=t, record=rec, out=traj if k == chunk else None)
                else:
                    vec4.rollout(k, policy_keys=pkeys, t0=t, record=())
                t += k
            f1.record(stream)
            torch.cuda.synchronize(dev)
            fms = f0.elapsed_time(f1)
            tf = torch.tensor([fms], dtype=torch.float64, device=dev)
            if world > 1:
                tf = _allreduce(dist, coll(tf), dist.ReduceOp.MAX)
            fms = float(tf.item())
            bpe_f = (2 * v * v + 9) if rec else 0
            ach = bpe_f * n * K / (fms / 1e3) / 1e9
            modes[mode] = {"value": n * world * K / (fms / 1e3), "ms_per_step": fms / K, "launches": vec4.launches - l0,
                           "record_bytes_per_env_step": bpe_f,
                           "achieved_gbs": ach, "frac_of_hbm_peak": ach / peak if bpe_f else None}
        del traj, vec4
        fused = {"unit": "env-steps/s", "chunk_steps": chunk, **modes,
                 "note": "xmg_rollout (one kernel per chunk of steps, state resident in shared memory / registers, "
                         "random policy evaluated in-kernel), bit-identical to K VecEnv.step calls "
                         "(tests/test_rollout_gpu.py); same K steps and phase as the timed window; records = "
                         "obs + reward + discount + step type per env-step written to HBM"}

    # ---- 224x224 image observations of the last step's
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
        vv = params.view_size
        ib = ni * (224 * 224 * 3 + 2 * vv * vv)
        image = {"images_per_s": ni / (ims / 1e3), "images": ni, "ms_per_launch": ims,
                 "bytes_per_image": 224 * 224 * 3 + 2 * vv * vv, "achieved_gbs": ib / (ims / 1e3) / 1e9,
                 "frac_of_hbm_peak": ib / (ims / 1e3) / 1e9 / peak,
                 "note": "xmg_image_obs on the timed window's last observations (ref render.py:225-243), "
                         "output 2.4 GB > L2"}
        del img_out

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        r = cpu_reference(args.workload, min(n, 1 << 14), 1 << 20, os.cpu_count() or 1, budget_s=12.0)
        r1 = cpu_reference(args.workload, 1 << 12, 1 << 20, 1, budget_s=3.0)  # one core, for scale
        cpu = {"value": r["value"], "unit": "env-steps/s", "cores": os.cpu_count() or 1, "kind": "port",
               "sample": f"{r['envs']} envs x {r['steps']} steps of the same workload on the host "
                         f"({r['seconds']:.1f} s, OpenMP over all host threads)",
               "cpu_model": cpu_model(), "one_core_value": r1["value"]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "env-steps/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic",
            "config": {"workload": desc, "env": env_id, "rulesets": f"data/{config}-65536.xmgb" if config else None,
                       "envs_per_gpu": n, "global_envs": n * world,
                       "parallelism": f"env-shard x{world}" + (" (ranks sharing a GPU: code-path check only)"
                                                                 if shared else ""),
                       "timed_window": f"steps [{W + pre}, {total}) incl. budget reset burst at t={budget}",
                       "l2": "inputs larger than L2" if n * params.height * params.width > 126e6
                             else "state resident in L2 (small workload)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "steps_block": block, "fused_rollout": fused, "image_obs": image,
            "clocks": clocks.summary(),
            "episode_stats": {"return_sum": float(tot[0]), "trials": float(tot[1]), "length_sum": float(tot[2])},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


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
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
