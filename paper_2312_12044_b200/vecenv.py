"""VecEnv: the reference's batched operator API over the sm_100a kernels.

Drop-in for ``rulegrid.VecEnv`` (ref vecenv.py:108-521):
  VecEnv(params, num_envs, rulesets)      ref :117-151
  .reset(key) / .reset_with_keys(k0, k1)   ref :201-222
  .step(actions, compute_obs)             ref :295-364  -> VecTimeStep
  .env_state(i)                           ref :511-521
State lives in HBM as structure-of-arrays torch tensors (layout in
include/xmg.h); every call is one asynchronous launch of libxmg.so on the
current CUDA stream.  Differences from the reference, by design:
  * outputs are CUDA tensors; rewards / discounts are float32 (the reward is
    evaluated in fp64 without contraction and rounded once, so it equals
    ``np.float32`` of the reference's float64 bit for bit);
  * actions given as a CUDA tensor are range-checked on the device: an
    invalid batch mutates no env and raises ``InvalidAction`` at the next
    ``check()`` (immediately with ``strict=True``); host (NumPy / list)
    actions are checked on the host before anything is launched, exactly
    like the reference.
There is no CPU fallback: without libxmg.so or a GPU every call raises.
"""

from __future__ import annotations

import ctypes as C
import functools
import os
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .core import (AgentState, Direction, GridFull, Grid, InvalidAction, Key, Position, DOMAIN_FOLD, fold_in,
                   key_from_seed)
from .env import EnvParams, StepType
from .layouts import Layout, bordered, plan_layout
from .ruleset import Benchmark, Ruleset, TaskTable, pack_rulesets

GRID_PAD = 64  # the step kernel reads 16-byte aligned chunks past the last grid
STAGE_BITS = 3 << 18  # reset-ahead stage in state word 0 (include/xmg.h)
BUF_BIT = 1 << 20  # the grid buffer holding the env's grid (0: grids, 1: next_grids)
META_BITS = STAGE_BITS | BUF_BIT


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)
_get_device = getattr(torch._C, "_cuda_getDevice", None) or torch.cuda.current_device


def _stream(device: torch.device) -> int:
    """The current CUDA stream of `device` (raw handle; no Stream object per call)."""
    if _raw_stream is not None:
        return _raw_stream(device.index if device.index is not None else _get_device())
    return torch.cuda.current_stream(device).cuda_stream


def _on_device(fn):
    """Run a method with its VecEnv's GPU current: libxmg launches on the
    current device (kernels, attributes and the stream all belong to it), so a
    VecEnv on cuda:1 must not launch while cuda:0 is current."""
    @functools.wraps(fn)
    def wrapper(self, *args, **kwargs):
        if _get_device() == self._dev_index:
            return fn(self, *args, **kwargs)
        with torch.cuda.device(self._dev_index):
            return fn(self, *args, **kwargs)
    return wrapper


def _device_ctx(dev: torch.device):
    """Context making `dev` current (a no-op when it already is)."""
    return torch.cuda.device(dev.index if dev.index is not None else torch.cuda.current_device())


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _device(device) -> torch.device:
    if device is None:
        if not torch.cuda.is_available():
            raise _lib.NativeLibraryError("VecEnv needs a CUDA device (B200); there is no CPU fallback")
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise _lib.NativeLibraryError("VecEnv state must live on a CUDA device; there is no CPU fallback")
    return d


def u64_to_i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64)).view(np.int64)


# ------------------------------------------------------------ batched keys
def split_batch(key: Key, num: int, offset: int = 0, device=None) -> torch.Tensor:
    """(num, 2) int64 tensor (u64 bit patterns hi, lo) of
    fold_in(key, offset + i, SPLIT): ref split_batch rng.py:142-145."""
    dev = _device(device)
    out = torch.empty((num, 2), dtype=torch.int64, device=dev)
    with _device_ctx(dev):
        _lib.check(_lib.lib().xmg_split_batch(key[0], key[1], offset, num, out.data_ptr(), _stream(dev)),
                   "xmg_split_batch")
    return out


def policy_keys(key: Key, num: int, offset: int = 0, device=None) -> torch.Tensor:
    """(num, 2) keys fold_in(key, offset + i) (FOLD domain): the per-env
    random-policy streams of ref tests/test_vecenv.py:126-129."""
    dev = _device(device)
    h = np.array([fold_in(key, offset + i, DOMAIN_FOLD) for i in range(num)], dtype=np.uint64) if num <= 4096 \
        else None
    if h is not None:
        return torch.from_numpy(h.view(np.int64)).to(dev)
    # large batches: derive on the device via the philox KAT kernel
    ctr = np.zeros((num, 4), np.uint64)
    ctr[:, 0] = np.arange(offset, offset + num, dtype=np.uint64)
    ctr[:, 2] = DOMAIN_FOLD
    kk = np.tile(np.array([key[0], key[1]], np.uint64), (num, 1))
    ctr_t = torch.from_numpy(ctr.view(np.int64)).to(dev)
    key_t = torch.from_numpy(kk.view(np.int64)).to(dev)
    out = torch.empty((num, 4), dtype=torch.int64, device=dev)
    with _device_ctx(dev):
        _lib.check(_lib.lib().xmg_philox(ctr_t.data_ptr(), key_t.data_ptr(), out.data_ptr(), num, _stream(dev)),
                   "xmg_philox")
    return out[:, :2].contiguous()


def random_actions(keys: torch.Tensor, t0: int, steps: int) -> torch.Tensor:
    """(steps, n) uint8: word (t0+t) of each key's draw stream mod 6, the
    random policy of ref harness.py:58-64 evaluated on the GPU."""
    n = keys.shape[0]
    out = torch.empty((steps, n), dtype=torch.uint8, device=keys.device)
    with _device_ctx(keys.device):
        _lib.check(_lib.lib().xmg_random_actions(keys.data_ptr(), n, t0, steps, out.data_ptr(),
                                                 _stream(keys.device)), "xmg_random_actions")
    return out


def philox(ctr: torch.Tensor, key: torch.Tensor) -> torch.Tensor:
    """Batched Philox4x64-10 blocks on the device (KAT hook)."""
    n = ctr.shape[0]
    out = torch.empty((n, 4), dtype=torch.int64, device=ctr.device)
    with _device_ctx(ctr.device):
        _lib.check(_lib.lib().xmg_philox(ctr.data_ptr(), key.data_ptr(), out.data_ptr(), n, _stream(ctr.device)),
                   "xmg_philox")
    return out


# ------------------------------------------------------------ records
@dataclass(eq=False)
class VecTimeStep:
    observations: torch.Tensor | None  # (N, v, v, 2) uint8
    rewards: torch.Tensor              # (N,) float32
    discounts: torch.Tensor            # (N,) float32
    step_types: torch.Tensor           # (N,) int8

    def last(self) -> torch.Tensor:
        return self.step_types == int(StepType.LAST)

    def numpy(self) -> tuple:
        return (None if self.observations is None else self.observations.cpu().numpy(),
                self.rewards.cpu().numpy(), self.discounts.cpu().numpy(), self.step_types.cpu().numpy())


@dataclass(eq=False)
class Trajectory:
    """Records of a fused rollout: entry t is the VecTimeStep step t returns
    (any field None when not requested)."""
    observations: torch.Tensor | None  # (T, N, v, v, 2) uint8
    rewards: torch.Tensor | None       # (T, N) float32
    discounts: torch.Tensor | None     # (T, N) float32
    step_types: torch.Tensor | None    # (T, N) int8


@dataclass(frozen=True)
class EnvState:
    grid: Grid
    agent: AgentState
    ruleset: Ruleset
    step_count: int
    goal_reached: bool
    rng: Key


_ACT_DTYPES = {torch.uint8: _lib.ACT_U8, torch.int32: _lib.ACT_I32, torch.int64: _lib.ACT_I64}


# ------------------------------------------------------------ VecEnv
class VecEnv:
    def __init__(self, params: EnvParams, num_envs: int, rulesets=None, *, device=None, task_ids=None,
                 strict: bool = False, global_offset: int = 0, reuse_outputs: bool = False,
                 resample_tasks: bool = False, reset_ahead: bool | None = None, graph: bool = False):
        if num_envs < 1:
            raise ValueError(f"num_envs must be >= 1, got {num_envs}")
        self.params = params
        self.num_envs = n = num_envs
        self.device = dev = _device(device)
        self._dev_index = dev.index if dev.index is not None else torch.cuda.current_device()
        self.strict = strict
        self.global_offset = global_offset
        self.reuse_outputs = reuse_outputs
        h, w, v = params.height, params.width, params.view_size
        self._hw = h * w
        scen = _lib.SCENARIO_IDS[params.scenario]

        # -- tasks: a device table plus one row index per env
        self._tasks: list[Ruleset] | None = None
        self._benchmark: Benchmark | None = None
        if rulesets is None or isinstance(rulesets, Ruleset):
            task = params.ruleset if rulesets is None else rulesets
            table = pack_rulesets([task])
            ids = np.zeros(n, np.int32)
            self._tasks = [task] * n
        elif isinstance(rulesets, (Benchmark, TaskTable)):
            table = rulesets.task_table() if isinstance(rulesets, Benchmark) else rulesets
            self._benchmark = rulesets if isinstance(rulesets, Benchmark) else None
            if task_ids is None:
                ids = ((np.arange(n, dtype=np.int64) + global_offset) % table.num_tasks).astype(np.int32)
            else:
                ids = np.asarray(task_ids.cpu() if isinstance(task_ids, torch.Tensor) else task_ids, np.int64)
                if ids.shape != (n,) or ids.min() < 0 or ids.max() >= table.num_tasks:
                    raise ValueError("task_ids must be (num_envs,) rows of the table")
                ids = ids.astype(np.int32)
        else:
            tasks = list(rulesets)
            if len(tasks) != n:
                raise ValueError(f"{len(tasks)} rulesets for {n} envs")
            uniq: dict[int, int] = {}
            order: list[Ruleset] = []
            ids = np.empty(n, np.int32)
            for i, t in enumerate(tasks):
                j = uniq.setdefault(id(t), len(order))
                if j == len(order):
                    order.append(t)
                ids[i] = j
            table = pack_rulesets(order)
            self._tasks = tasks
        self.table = table

        # -- static geometry of the scenario
        seg_off = np.zeros(1, np.int16)
        seg_cells = np.zeros(1, np.int16)
        fixed = 0
        if scen in (0, 4):  # xland / four_rooms: room layout with door segments
            plan = plan_layout(Layout.R4 if scen == 4 else params.layout, h, w)
            base = plan.base_cells()
            seg_off, seg_cells = plan.segment_arrays()
            fixed = int(plan.fixed_doors)
            nseg = len(plan.door_segments)
            free = int(((base >> 4) == 3).sum())
            rows = table.rows if resample_tasks else table.rows[ids]
            used_obj = int(((rows[:, 1] >> 8) & 0xFF).max()) if scen == 0 else 1
            if used_obj >= free:  # ref vecenv.py:171-175
                raise GridFull(f"{used_obj} objects on {free} free cells")
        else:
            base = bordered(h, w, goal=scen in (1, 2, 3))
            nseg = 0
        if scen != 0:
            table = TaskTable(np.zeros((1, 4), np.uint32), 0, 0, 0)  # ports bring their own goal, no rules
            ids = np.zeros(n, np.int32)
        self._ids_host = ids

        # -- device buffers
        # padded to 16 bytes: the reset kernels read it with 16-byte loads
        base_p = np.zeros((self._hw + 15) // 16 * 16, np.uint8)
        base_p[: self._hw] = base.reshape(-1)
        self._base = torch.from_numpy(base_p).to(dev)
        self._seg_off = torch.from_numpy(seg_off.astype(np.int16)).to(dev)
        self._seg_cells = torch.from_numpy(seg_cells.astype(np.int16)).to(dev)
        self._table = torch.from_numpy(table.rows.view(np.int32).copy()).to(dev)
        # compact MOVE / PICK_UP rule rows (ruleset.TaskTable.agent_rows), xland only
        agent_rows = getattr(table, "agent_rows", None) if scen == 0 and table.rule_width > 0 else None
        if os.environ.get("XMG_AGENT_ROWS", "1") == "0":
            agent_rows = None
        self._agent_rows = None if agent_rows is None else \
            torch.from_numpy(np.ascontiguousarray(agent_rows).view(np.int32)).to(dev)
        self.grids_flat = torch.zeros(n * self._hw + GRID_PAD, dtype=torch.uint8, device=dev)
        # 16-byte state word per env: [pose | pocket | step count, goal | task << 32]
        goals = table.rows[ids, 0].astype(np.uint64) if scen == 0 else np.zeros(n, np.uint64)
        word1 = goals | (ids.astype(np.uint64) << np.uint64(32))
        agent = np.zeros((n, 2), np.uint64)
        agent[:, 1] = word1
        self.agent = torch.from_numpy(agent.view(np.int64)).to(dev)
        self.rng = torch.zeros((n, 2), dtype=torch.int64, device=dev)
        words = int(_lib.lib().xmg_work_words(n))
        if words < 0:
            raise ValueError(f"num_envs={n} is too large for one VecEnv (< 2^30; shard with global_offset)")
        self.work = torch.zeros(words, dtype=torch.int32, device=dev)
        # reset-ahead records (include/xmg.h): each env's next trial, pre-built
        # while the current one runs, so an auto-reset is a copy
        # (off by default for the Empty scenario, whose trials are all the same
        # constant build: nothing to move out of the reset)
        default_ahead = os.environ.get("XMG_AHEAD", "1") != "0" and params.scenario != "empty"
        self.reset_ahead = reset_ahead if reset_ahead is not None else default_ahead
        if self.reset_ahead:
            self._next_grids = torch.zeros(n * self._hw + GRID_PAD, dtype=torch.uint8, device=dev)
            self._next_state = torch.zeros((n, 4), dtype=torch.int64, device=dev)
            self._next_obs = torch.zeros(n * 2 * v * v + 16, dtype=torch.uint8, device=dev)
        else:
            self._next_grids = self._next_state = self._next_obs = None
        # validation flag block (include/xmg.h XMG_FLAG_WORDS): [0] epoch of the
        # last rejected batch, [1] epoch of the last finished validation
        self._flag = torch.zeros(4, dtype=torch.int32, device=dev)
        self.epoch = 0          # steps issued on this state (queue parity, rejection tags)
        self._checked_epoch = 0

        self._desc = _lib.EnvDesc(h, w, v, params.step_budget, scen, int(params.see_through_walls), nseg, fixed,
                                  table.rule_width if scen == 0 else 0, table.obj_width, table.row_words,
                                  table.num_tasks, int(resample_tasks and scen == 0), self._base.data_ptr(),
                                  self._seg_off.data_ptr(), self._seg_cells.data_ptr(), self._table.data_ptr(),
                                  0 if self._agent_rows is None else self._agent_rows.shape[1],
                                  _ptr(self._agent_rows))
        self._state = _lib.State(self.grids_flat.data_ptr(), self.agent.data_ptr(), self.rng.data_ptr(),
                                 self.work.data_ptr(), _ptr(self._next_grids), _ptr(self._next_state),
                                 _ptr(self._next_obs))
        if _lib.lib().xmg_step_smem_bytes(C.byref(self._desc)) > 226 * 1024:
            raise _lib.NativeLibraryError(f"{h}x{w} grids exceed the shared-memory budget of this build")
        self._outs = None
        self._out_cache: dict = {}
        # reset-ahead batch plan (xmg_ahead_plan): every `every`-th step one
        # class (e mod classes) of envs gets its next trial pre-built; step()
        # schedules by epoch inside libxmg, rollout() by its own step clock
        if self.reset_ahead:
            ev, cl = C.c_int64(), C.c_int64()
            with torch.cuda.device(self._dev_index):
                _lib.check(_lib.lib().xmg_ahead_plan(C.byref(self._desc), n, C.byref(ev), C.byref(cl)),
                           "xmg_ahead_plan")
            self._ahead_every, self._ahead_classes = int(ev.value), int(cl.value)
        self._roll_clock = 0
        self._desc_ref = C.byref(self._desc)
        self._L = _lib.lib()
        self._state_ref = C.byref(self._state)
        self._flag_ptr = self._flag.data_ptr()
        self.stats: torch.Tensor | None = None
        self.launches = 0  # kernels of ours launched by this VecEnv
        # graph mode (small batches): step() = ONE fused kernel (xmg_step_fused,
        # in-kernel validation, device step counter) replayed from a CUDA graph;
        # actions are staged in a fixed buffer, the records are reused buffers
        self.graph = graph
        if graph:
            self.reuse_outputs = True
            self._gflag = torch.zeros(4, dtype=torch.int32, device=dev)
            self._gact = torch.zeros(n + 16, dtype=torch.uint8, device=dev)[:n]
            self._gact_ptr = self._gact.data_ptr()
            self._graphs: dict = {}
            self._gchecked = 0

    # -- views
    def _grid_buffers(self):
        n, hw = self.num_envs, self._hw
        g0 = self.grids_flat[: n * hw].view(n, hw)
        g1 = None if self._next_grids is None else self._next_grids[: n * hw].view(n, hw)
        return g0, g1

    @property
    def grids(self) -> torch.Tensor:
        """(N, H*W) u8 cells of every env.  With reset-ahead each env's grid
        lives in one of two buffers (bit 20 of its state word; a pre-built
        trial is written to the other one and taken over by flipping the bit):
        this gathers them into a new tensor (write cells with set_grid)."""
        g0, g1 = self._grid_buffers()
        if g1 is None:
            return g0
        buf = ((self.agent[:, 0] >> 20) & 1).bool()
        return torch.where(buf[:, None], g1, g0)

    def _live_grid(self, i: int) -> torch.Tensor:
        """View of env i's cells in the buffer its state word names."""
        g0, g1 = self._grid_buffers()
        return g1[i] if g1 is not None and int(self.agent[i, 0].item()) & BUF_BIT else g0[i]

    def set_grid(self, i: int, cells) -> None:
        """Overwrite env i's cells (in the buffer its state word names)."""
        self._live_grid(i).copy_(torch.as_tensor(cells, dtype=torch.uint8).to(self.device))

    def agent_fields(self) -> torch.Tensor:
        """(N, 5) int64: row, col, dir, pocket, step_count."""
        a = self.agent[:, 0]
        return torch.stack([a & 0xFF, (a >> 8) & 0xFF, (a >> 16) & 0x3, (a >> 24) & 0xFF,
                            (a >> 32) & 0xFFFFFFFF], dim=1)

    def state_words(self) -> torch.Tensor:
        """(N, 2) state words without the reset-ahead bits (stage, 18-19 of
        word 0, and the grid buffer, 20: scheduling metadata, not env state):
        the env state proper, comparable across step / steps / rollout paths."""
        a = self.agent.clone()
        a[:, 0] &= ~META_BITS
        return a

    @property
    def reset_ahead_stage(self) -> torch.Tensor:
        """(N,) 0 none / 1 next trial queued / 2 next trial pre-built."""
        return (self.agent[:, 0] >> 18) & 3

    @property
    def goal(self) -> torch.Tensor:
        """(N,) goal encodings (kind | a1 << 8 | a2 << 16 | a3 << 24)."""
        return self.agent[:, 1] & 0xFFFFFFFF

    @property
    def task(self) -> torch.Tensor:
        """(N,) task-table row of each env."""
        return (self.agent[:, 1] >> 32) & 0xFFFFFFFF

    # -- outputs
    def _alloc_out(self, compute_obs: bool):
        n, v, dev = self.num_envs, self.params.view_size, self.device
        if self.reuse_outputs and self._outs is not None and (self._outs[0] is not None) == compute_obs:
            return self._outs
        obs = torch.empty((n, v, v, 2), dtype=torch.uint8, device=dev) if compute_obs else None
        outs = (obs, torch.empty(n, dtype=torch.float32, device=dev), torch.empty(n, dtype=torch.float32, device=dev),
                torch.empty(n, dtype=torch.int8, device=dev))
        if self.reuse_outputs:
            self._outs = outs
        return outs

    def _out_struct(self, outs) -> _lib.Out:
        return _lib.Out(_ptr(outs[0]), _ptr(outs[1]), _ptr(outs[2]), _ptr(outs[3]), _ptr(self.stats))

    def enable_stats(self) -> torch.Tensor:
        """Accumulate episode statistics inside the step kernel: returns the
        (num_ctas, 3) float64 tensor of per-CTA [sum reward, finished trials,
        sum of their lengths] (ref RolloutStats, harness.py:103-143)."""
        if self.stats is None:
            self.stats = torch.zeros(((self.num_envs + 127) // 128, 3), dtype=torch.float64, device=self.device)
        return self.stats

    def episode_stats(self) -> torch.Tensor:
        """(3,) float64 totals of the per-CTA accumulators."""
        return self.enable_stats().sum(dim=0)

    # -- reset
    @_on_device
    def reset(self, key: Key, compute_obs: bool = True) -> VecTimeStep:
        keys = split_batch(key, self.num_envs, self.global_offset, self.device)
        self.launches += 1
        return self._reset_keys(keys, compute_obs)

    @_on_device
    def reset_with_keys(self, k0, k1, compute_obs: bool = True) -> VecTimeStep:
        if isinstance(k0, torch.Tensor):
            keys = torch.stack([k0.to(self.device, torch.int64), k1.to(self.device, torch.int64)], dim=1)
        else:
            k0 = np.asarray(k0)
            k1 = np.asarray(k1)
            if k0.shape != (self.num_envs,) or k1.shape != (self.num_envs,):
                raise ValueError(f"expected {self.num_envs} key pairs")
            keys = torch.from_numpy(np.stack([u64_to_i64(k0), u64_to_i64(k1)], axis=1)).to(self.device)
        if keys.shape != (self.num_envs, 2):
            raise ValueError(f"expected {self.num_envs} key pairs")
        return self._reset_keys(keys.contiguous(), compute_obs)

    def _reset_keys(self, keys: torch.Tensor, compute_obs: bool) -> VecTimeStep:
        outs = self._alloc_out(compute_obs)
        o = _lib.Out(_ptr(outs[0]), _ptr(outs[1]), _ptr(outs[2]), _ptr(outs[3]), None)
        _lib.check(_lib.lib().xmg_reset(C.byref(self._desc), C.byref(self._state), keys.data_ptr(), self.num_envs,
                                        C.byref(o), _stream(self.device)), "xmg_reset")
        self.launches += 1
        return VecTimeStep(*outs)

    # -- step
    @_on_device
    def step(self, actions, compute_obs: bool = True, validate: bool = True) -> VecTimeStep:
        if self.graph:
            return self._step_graph(actions, compute_obs)
        n = self.num_envs
        L = self._L
        stream = _stream(self.device)
        flag_ptr = None
        if isinstance(actions, torch.Tensor) and actions.is_cuda:
            if actions.shape != (n,):
                raise InvalidAction(f"expected {n} actions, got shape {tuple(actions.shape)}")
            dt = _ACT_DTYPES.get(actions.dtype)
            if dt is None:
                actions = actions.to(torch.int64)
                dt = _lib.ACT_I64
            if not actions.is_contiguous():
                actions = actions.contiguous()
            if validate:  # the validation kernel is launched by xmg_step_validated below
                flag_ptr = self._flag_ptr
                self.launches += 1
        else:
            a = np.asarray(actions)
            if a.shape != (n,):
                raise InvalidAction(f"expected {n} actions, got shape {a.shape}")
            if ((a < 0) | (a >= 6)).any():
                raise InvalidAction("action outside [0, 5]")
            actions = torch.from_numpy(a.astype(np.uint8)).to(self.device)
            dt = _lib.ACT_U8
        outs = self._alloc_out(compute_obs)
        o = self._out_cache.get(id(outs)) if self.reuse_outputs else None
        if o is None or o[0] is not outs or o[2] is not self.stats:
            o = (outs, C.byref(self._out_struct(outs)), self.stats)
            if self.reuse_outputs:
                self._out_cache = {id(outs): o}
        self.epoch += 1
        if flag_ptr is not None:  # one library call: validation, then the step that awaits its verdict
            rc = L.xmg_step_validated(self._desc_ref, self._state_ref, actions.data_ptr(), dt, n, o[1], flag_ptr,
                                      self.epoch & 0xFFFFFFFF, stream)
        else:
            rc = L.xmg_step(self._desc_ref, self._state_ref, actions.data_ptr(), dt, n, o[1], None,
                            self.epoch & 0xFFFFFFFF, stream)
        if rc:
            _lib.check(rc, "xmg_step")
        self.launches += 2 + self._batches_in(self.epoch - 1, self.epoch)  # streaming + rare passes (+ batch)
        if self.strict and flag_ptr is not None:
            self.check()
        return VecTimeStep(*outs)

    # -- graph mode
    @property
    def action_buffer(self) -> torch.Tensor:
        """(N,) uint8 staging buffer of graph mode: actions written here need
        no copy (step(vec.action_buffer))."""
        return self._gact

    def _stage_actions(self, actions) -> None:
        n = self.num_envs
        if isinstance(actions, torch.Tensor) and actions.is_cuda:
            if actions.shape != (n,):
                raise InvalidAction(f"expected {n} actions, got shape {tuple(actions.shape)}")
            if actions.data_ptr() == self._gact.data_ptr() and actions.dtype == torch.uint8:
                return
            if actions.dtype == torch.uint8:
                self._gact.copy_(actions)
            else:  # out-of-range values map to 255 so the kernel rejects the batch
                a = actions.to(torch.int64)
                self._gact.copy_(torch.where((a >= 0) & (a < 6), a, 255).to(torch.uint8))
        else:
            a = np.asarray(actions)
            if a.shape != (n,):
                raise InvalidAction(f"expected {n} actions, got shape {a.shape}")
            if ((a < 0) | (a >= 6)).any():
                raise InvalidAction("action outside [0, 5]")
            self._gact.copy_(torch.from_numpy(a.astype(np.uint8)), non_blocking=False)

    def _fused_call(self, o_ref) -> None:
        _lib.check(_lib.lib().xmg_step_fused(self._desc_ref, self._state_ref, self._gact.data_ptr(), self.num_envs,
                                             o_ref, self._gflag.data_ptr(), _stream(self.device)), "xmg_step_fused")

    def _step_graph(self, actions, compute_obs: bool) -> VecTimeStep:
        """step() in graph mode: the same transition (bit-identical, the fused
        kernel at T = 1), one kernel per step replayed from a CUDA graph
        (captured once per record layout by libxmg: xmg_graph_create)."""
        src = None  # u8 device actions are copied into the staging buffer by libxmg with the launch
        if isinstance(actions, torch.Tensor) and actions.is_cuda and actions.dtype == torch.uint8 \
                and actions.shape == (self.num_envs,) and actions.is_contiguous():
            src = actions.data_ptr()
        elif actions is not self._gact:
            self._stage_actions(actions)
        if self.reset_ahead:
            self._roll_clock += 1
            if self._roll_clock % self._ahead_every == 0:  # this step's reset-ahead batch (outside the graph)
                cls = (self._roll_clock // self._ahead_every) % self._ahead_classes
                _lib.check(_lib.lib().xmg_prebuild(self._desc_ref, self._state_ref, cls, self._ahead_classes,
                                                   self.num_envs, _stream(self.device)), "xmg_prebuild")
                self.launches += 1
        key = (compute_obs, id(self.stats))
        ent = self._graphs.get(key)
        if ent is None:
            outs = self._alloc_out(compute_obs)
            o = self._out_struct(outs)
            h = C.c_void_p()
            _lib.check(_lib.lib().xmg_graph_create(self._desc_ref, self._state_ref, self._gact.data_ptr(),
                                                   self.num_envs, C.byref(o), self._gflag.data_ptr(), C.byref(h)),
                       "xmg_graph_create")
            ent = self._graphs[key] = (h, o, VecTimeStep(*outs))
        rc = self._L.xmg_graph_step(ent[0], src, self._gact_ptr, self.num_envs, _stream(self.device))
        if rc:
            _lib.check(rc, "xmg_graph_step")
        self.launches += 1
        if self.strict:
            self.check()
        return ent[2]

    def __del__(self):
        for h, _, _ in getattr(self, "_graphs", {}).values():
            try:
                _lib.lib().xmg_graph_destroy(h)
            except Exception:
                pass

    # -- many steps per host call
    @_on_device
    def steps(self, actions: torch.Tensor, compute_obs: bool = True, validate: bool = True,
              out: Trajectory | None = None, fused: bool | None = None) -> Trajectory:
        """``actions.shape[0]`` consecutive ``step`` calls issued by one library
        call: no per-step host round trip.  Record k of the returned
        Trajectory is what ``step`` k would return.  ``validate`` checks the
        whole block once, before anything is launched (ref vecenv.py:297-301,
        one host sync).  ``fused=True`` runs the block in the fused kernel
        (``xmg_rollout`` with the given actions: state on chip for the whole
        block, one launch); ``fused=False`` issues the per-call kernels K times
        (``xmg_steps``).  Both are bit-identical to ``step``.  ``None``
        (default) picks the fused kernel when it keeps at least 12 warps per SM
        resident (16 up to 13x13 with medium rulesets, where it is the faster
        path), else the per-call kernels (R9-25x25 high: 4 warps/SM fused,
        6.6e9 vs 8.4e9 env-steps/s per call at 2^19 envs)."""
        n, v, dev = self.num_envs, self.params.view_size, self.device
        if not isinstance(actions, torch.Tensor):
            actions = torch.as_tensor(np.asarray(actions))
        if actions.dim() != 2 or actions.shape[1] != n:
            raise InvalidAction(f"expected (K, {n}) actions, got shape {tuple(actions.shape)}")
        k = actions.shape[0]
        aligned = not compute_obs or (n * 2 * v * v) % 16 == 0
        if fused is None:
            fused = not aligned or self.aligned_fused_choice()
        if not fused and not aligned:
            raise ValueError("steps(fused=False): with observations, num_envs * 2 * v * v must be a multiple of 16 "
                             "(16-byte aligned records); use step() or the fused path")
        if validate and bool(((actions < 0) | (actions >= 6)).any()):
            raise InvalidAction("action outside [0, 5]")
        if out is None:
            out = Trajectory(torch.empty((k, n, v, v, 2), dtype=torch.uint8, device=dev) if compute_obs else None,
                             torch.empty((k, n), dtype=torch.float32, device=dev),
                             torch.empty((k, n), dtype=torch.float32, device=dev),
                             torch.empty((k, n), dtype=torch.int8, device=dev))
        if fused:
            # in range (checked above, or the caller's promise): u8 is exact
            return self._launch_rollout(k, None, actions.to(dev, torch.uint8).contiguous(), 0, out)
        actions = actions.to(dev)
        dt = _ACT_DTYPES.get(actions.dtype)
        if dt is None:
            actions, dt = actions.to(torch.int64), _lib.ACT_I64
        actions = actions.contiguous()
        o = _lib.Out(_ptr(out.observations), _ptr(out.rewards), _ptr(out.discounts), _ptr(out.step_types),
                     _ptr(self.stats))
        _lib.check(_lib.lib().xmg_steps(self._desc_ref, self._state_ref, actions.data_ptr(), dt, k, n, C.byref(o),
                                        self.epoch & 0xFFFFFFFF, _stream(dev)), "xmg_steps")
        self.epoch += k
        self.launches += 2 * k + self._batches_in(self.epoch - k, self.epoch)
        return out

    def aligned_fused_choice(self) -> bool:
        """steps(fused=None)'s choice for 16-byte aligned records."""
        return self._rollout_warps_per_sm() >= 12

    def _rollout_warps_per_sm(self) -> int:
        """Resident warps per SM of the fused kernel (4-warp CTAs, bounded by
        shared memory: 228 KB per SM, 1 KB reserved per CTA; <= 16)."""
        smem = int(_lib.lib().xmg_rollout_smem_bytes(C.byref(self._desc)))
        return 4 * min(4, (228 * 1024) // (smem + 1024)) if smem > 0 else 0

    # -- fused rollout
    @_on_device
    def rollout(self, steps: int, policy_keys: torch.Tensor | None = None, actions: torch.Tensor | None = None,
                t0: int = 0, record: Sequence[str] = ("observations", "rewards", "discounts", "step_types"),
                out: Trajectory | None = None, fused: bool | None = None) -> Trajectory:
        """``steps`` consecutive ``step`` calls in one kernel (state on chip for
        the whole rollout), bit-identical to them.  Actions come from the
        random policy of ref harness.py:58-64 (``policy_keys``: step t plays
        word t0 + t of each env's key mod 6, as ``random_actions``) or from a
        (steps, N) tensor ``actions``.  ``record`` picks the per-step fields
        kept (ref harness.py:103-143 accumulates only statistics: pass
        ``record=()`` and ``enable_stats()`` for that).  Rollouts and steps
        may be interleaved freely.  Where the fused kernel keeps too few warps
        resident (``aligned_fused_choice``: R9-25x25) the same steps run
        through the per-call kernels instead, 64 per library call (C4: 5.9e9
        → 1.1e10 env-steps/s); ``fused`` forces the choice (True: the fused
        kernel, False: the per-call kernels)."""
        n, v, dev = self.num_envs, self.params.view_size, self.device
        if steps < 0 or t0 < 0:
            raise ValueError("steps and t0 must be >= 0")
        if (policy_keys is None) == (actions is None):
            raise ValueError("pass exactly one of policy_keys / actions")
        if policy_keys is not None:
            if policy_keys.shape != (n, 2) or policy_keys.device != dev:
                raise ValueError(f"policy_keys must be a ({n}, 2) tensor on {dev}")
            policy_keys = policy_keys.to(torch.int64).contiguous()
        else:
            if not isinstance(actions, torch.Tensor):
                actions = torch.as_tensor(np.asarray(actions))
            if actions.shape != (steps, n):
                raise InvalidAction(f"expected ({steps}, {n}) actions, got shape {tuple(actions.shape)}")
            if bool(((actions < 0) | (actions >= 6)).any()):  # ref vecenv.py:297-301, before any mutation
                raise InvalidAction("action outside [0, 5]")
            actions = actions.to(dev, torch.uint8).contiguous()
        unknown = set(record) - {"observations", "rewards", "discounts", "step_types"}
        if unknown:
            raise ValueError(f"unknown record fields {sorted(unknown)}")
        if out is None:
            out = Trajectory(
                torch.empty((steps, n, v, v, 2), dtype=torch.uint8, device=dev) if "observations" in record else None,
                torch.empty((steps, n), dtype=torch.float32, device=dev) if "rewards" in record else None,
                torch.empty((steps, n), dtype=torch.float32, device=dev) if "discounts" in record else None,
                torch.empty((steps, n), dtype=torch.int8, device=dev) if "step_types" in record else None)
        aligned = out.observations is None or (n * 2 * v * v) % 16 == 0
        if fused is None:
            fused = not aligned or self.aligned_fused_choice()
        if not fused:
            if not aligned:
                raise ValueError("rollout(fused=False): with observations, num_envs * 2 * v * v must be a multiple "
                                 "of 16 (16-byte aligned records)")
            return self._rollout_per_call(steps, policy_keys, actions, t0, out)
        return self._launch_rollout(steps, policy_keys, actions, t0, out)

    def _rollout_per_call(self, steps: int, policy_keys, actions, t0: int, out: Trajectory,
                          block: int = 64) -> Trajectory:
        """rollout() through the per-call kernels (xmg_steps), ``block`` steps
        per library call, the random policy's actions drawn on the device per
        block; unrecorded fields go to scratch buffers.  Bit-identical to the
        fused kernel, as every path is."""
        n, dev = self.num_envs, self.device
        scratch = None
        if out.rewards is None or out.discounts is None or out.step_types is None:
            scratch = (torch.empty((block, n), dtype=torch.float32, device=dev),
                       torch.empty((block, n), dtype=torch.float32, device=dev),
                       torch.empty((block, n), dtype=torch.int8, device=dev))
        for c0 in range(0, steps, block):
            k = min(block, steps - c0)
            if actions is None:
                a = random_actions(policy_keys, t0 + c0, k)
                self.launches += 1
            else:
                a = actions[c0:c0 + k]
            pick = lambda f, i: f[c0:c0 + k] if f is not None else scratch[i][:k]  # noqa: E731
            o = _lib.Out(_ptr(None if out.observations is None else out.observations[c0:c0 + k]),
                         _ptr(pick(out.rewards, 0)), _ptr(pick(out.discounts, 1)), _ptr(pick(out.step_types, 2)),
                         _ptr(self.stats))
            _lib.check(_lib.lib().xmg_steps(self._desc_ref, self._state_ref, a.data_ptr(), _lib.ACT_U8, k, n,
                                            C.byref(o), self.epoch & 0xFFFFFFFF, _stream(dev)), "xmg_steps")
            self.epoch += k
            self.launches += 2 * k + self._batches_in(self.epoch - k, self.epoch)
        return out

    def _batches_in(self, e0: int, e1: int) -> int:
        """Reset-ahead batches libxmg launched for epochs (e0, e1] (one per
        multiple of `every`, include/xmg.h)."""
        if not self.reset_ahead:
            return 0
        ev = self._ahead_every
        return (e1 & 0xFFFFFFFF) // ev - (e0 & 0xFFFFFFFF) // ev if e1 >= e0 else 0

    def _rollout_prebuilds(self, steps: int) -> None:
        """The reset-ahead batches `steps` step() calls would launch (one per
        `every` steps of the rollout clock), run before the fused kernel: the
        trials that end inside the rollout are then reset by copies."""
        if not self.reset_ahead:
            return
        ev, cl = self._ahead_every, self._ahead_classes
        L = _lib.lib()
        stream = _stream(self.device)
        first = self._roll_clock // ev + 1
        last = (self._roll_clock + steps) // ev
        for j in range(first, last + 1)[:cl]:  # one cycle covers every class
            _lib.check(L.xmg_prebuild(self._desc_ref, self._state_ref, j % cl, cl, self.num_envs, stream),
                       "xmg_prebuild")
            self.launches += 1
        self._roll_clock += steps

    def _launch_rollout(self, steps: int, policy_keys, actions, t0: int, out: Trajectory) -> Trajectory:
        self._rollout_prebuilds(steps)
        o = _lib.Out(_ptr(out.observations), _ptr(out.rewards), _ptr(out.discounts), _ptr(out.step_types),
                     _ptr(self.stats))
        _lib.check(_lib.lib().xmg_rollout(C.byref(self._desc), C.byref(self._state), _ptr(policy_keys),
                                          _ptr(actions), t0, steps, self.num_envs, C.byref(o),
                                          _stream(self.device)), "xmg_rollout")
        self.launches += 1
        return out

    def check(self) -> None:
        """Raise InvalidAction if a device-validated batch was rejected (syncs)."""
        flagged = int(self._flag[0].item()) & 0xFFFFFFFF  # syncs the stream
        if flagged > self._checked_epoch:
            self._checked_epoch = flagged
            raise InvalidAction(f"action outside [0, 5] at step {flagged}; that batch was not applied")
        if self.graph:
            gf = int(self._gflag[0].item()) & 0xFFFFFFFF
            if gf > self._gchecked:
                self._gchecked = gf
                raise InvalidAction(f"action outside [0, 5] at graph step {gf}; that batch was not applied")

    # -- inspection
    def ruleset_of(self, i: int) -> Ruleset:
        if self._tasks is not None:
            return self._tasks[i]
        if self._benchmark is not None:
            return self._benchmark.get_ruleset(int(self.task[i].item()))
        return Ruleset()

    def env_state(self, i: int) -> EnvState:
        """The i-th env as a scalar EnvState (ref vecenv.py:511-521)."""
        g = self._live_grid(i).cpu().numpy().tobytes()
        a = int(self.agent[i, 0].item()) & ((1 << 64) - 1)
        k = self.rng[i].cpu().numpy().view(np.uint64)
        agent = AgentState(Position(a & 0xFF, (a >> 8) & 0xFF), Direction((a >> 16) & 3), (a >> 24) & 0xFF)
        return EnvState(Grid(self.params.height, self.params.width, g), agent, self.ruleset_of(i),
                        (a >> 32) & 0xFFFFFFFF, False, Key(int(k[0]), int(k[1])))
