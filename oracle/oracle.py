"""ctypes wrapper of the CPU oracle (oracle/xmg_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg as the *checker*.  The
product package (paper_2312_12044_b200) never imports this module.

``OracleVecEnv`` mirrors the reference's ``rulegrid.VecEnv``
(/root/reference/pkg/src/rulegrid/vecenv.py:108-521): SoA state, per-env
left-packed tasks, ``reset_with_keys`` / ``step`` with auto-reset and a
float64 reward, so oracle results compare 1:1 with the reference fixtures.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libxmg_oracle.so")

SCENARIOS = {"xland": 0, "empty": 1, "empty_random": 2, "door_key": 3, "four_rooms": 4,
             "unlock": 5, "unlock_pickup": 6}

_lock = threading.Lock()
_lib = None


def build() -> str:
    """Compile the oracle with its Makefile (gcc); returns the .so path."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


class _Params(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("height", "width", "view_size", "budget", "scenario", "layout",
                                          "see_through_walls", "rule_width", "obj_width")]


class _State(C.Structure):
    _fields_ = [("grids", C.c_void_p), ("agent_r", C.c_void_p), ("agent_c", C.c_void_p),
                ("agent_dir", C.c_void_p), ("pocket", C.c_void_p), ("step_count", C.c_void_p),
                ("rng", C.c_void_p), ("goals", C.c_void_p), ("rules", C.c_void_p),
                ("rule_count", C.c_void_p), ("objs", C.c_void_p), ("obj_count", C.c_void_p)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                build()
            L = C.CDLL(LIB_PATH)
            vp, i64, i32, u64 = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64
            L.xmgo_reset.argtypes = [C.POINTER(_Params), C.POINTER(_State), vp, vp, i64, vp, i32]
            L.xmgo_step.argtypes = [C.POINTER(_Params), C.POINTER(_State), vp, i64, vp, vp, vp, vp, i32]
            L.xmgo_rollout_random.argtypes = [C.POINTER(_Params), C.POINTER(_State), vp, vp, i64, i64, i64, i32,
                                              vp, vp, vp, i32]
            L.xmgo_observe.argtypes = [C.POINTER(_Params), C.POINTER(_State), i64, vp]
            L.xmgo_philox.argtypes = [vp, vp, vp, i64]
            L.xmgo_key_from_seed.argtypes = [u64, u64, vp]
            L.xmgo_fold_in.argtypes = [u64, u64, u64, i32, vp]
            L.xmgo_split_batch.argtypes = [u64, u64, i64, i64, vp, vp]
            L.xmgo_random_actions.argtypes = [vp, vp, i64, i64, i64, vp]
            for f in ("xmgo_reset", "xmgo_step", "xmgo_rollout_random"):
                getattr(L, f).restype = i32
            _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data


# ---------------------------------------------------------------- keys
def philox(ctr: np.ndarray, key: np.ndarray) -> np.ndarray:
    ctr = np.ascontiguousarray(ctr, np.uint64).reshape(-1, 4)
    key = np.ascontiguousarray(key, np.uint64).reshape(-1, 2)
    out = np.empty_like(ctr)
    lib().xmgo_philox(_p(ctr), _p(key), _p(out), len(ctr))
    return out


def key_from_seed(seed: int) -> tuple[int, int]:
    out = np.empty(2, np.uint64)
    lib().xmgo_key_from_seed(seed & (2**64 - 1), (seed >> 64) & (2**64 - 1), _p(out))
    return int(out[0]), int(out[1])


def fold_in(key, data: int, domain: int = 3) -> tuple[int, int]:
    out = np.empty(2, np.uint64)
    lib().xmgo_fold_in(key[0], key[1], data, domain, _p(out))
    return int(out[0]), int(out[1])


def split_batch(key, n: int, offset: int = 0):
    k0 = np.empty(n, np.uint64)
    k1 = np.empty(n, np.uint64)
    lib().xmgo_split_batch(key[0], key[1], offset, n, _p(k0), _p(k1))
    return k0, k1


def random_actions(k0: np.ndarray, k1: np.ndarray, t0: int, steps: int) -> np.ndarray:
    k0 = np.ascontiguousarray(k0, np.uint64)
    k1 = np.ascontiguousarray(k1, np.uint64)
    out = np.empty((steps, len(k0)), np.uint8)
    lib().xmgo_random_actions(_p(k0), _p(k1), len(k0), t0, steps, _p(out))
    return out


# --------------------------------------------------------------- env
class OracleVecEnv:
    """CPU restatement of rulegrid.VecEnv over explicit task arrays.

    goals (n,4) u8; rules (n,R,4) u8 left-packed with rule_count (n,);
    objs (n,O) u8 left-packed with obj_count (n,).
    """

    def __init__(self, height, width, view_size, budget, scenario, layout, see_through_walls,
                 goals, rules, rule_count, objs, obj_count, threads: int = 1):
        n = len(goals)
        self.n = n
        self.threads = threads
        self.h, self.w, self.v = height, width, view_size
        rules = np.ascontiguousarray(rules, np.uint8).reshape(n, -1, 4)
        objs = np.ascontiguousarray(objs, np.uint8).reshape(n, -1)
        sc = SCENARIOS[scenario] if isinstance(scenario, str) else int(scenario)
        self.params = _Params(height, width, view_size, budget, sc, int(layout), int(see_through_walls),
                              rules.shape[1], objs.shape[1])
        hw = height * width
        self.grids = np.zeros((n, hw), np.uint8)
        self.agent_r = np.zeros(n, np.int32)
        self.agent_c = np.zeros(n, np.int32)
        self.agent_dir = np.zeros(n, np.int32)
        self.pocket = np.zeros(n, np.int32)
        self.step_count = np.zeros(n, np.int64)
        self.rng = np.zeros((n, 2), np.uint64)
        self.goals = np.ascontiguousarray(goals, np.uint8).copy()
        self.rules = rules.copy()
        self.rule_count = np.ascontiguousarray(rule_count, np.int32).copy()
        self.objs = objs.copy()
        self.obj_count = np.ascontiguousarray(obj_count, np.int32).copy()
        self.state = _State(*(_p(a) for a in (self.grids, self.agent_r, self.agent_c, self.agent_dir,
                                              self.pocket, self.step_count, self.rng, self.goals,
                                              self.rules, self.rule_count, self.objs, self.obj_count)))

    @classmethod
    def from_fixture(cls, fx, threads: int = 1):
        h, w, v, budget, sc, layout, see = (int(x) for x in fx["meta"])
        return cls(h, w, v, budget, sc, layout, see, fx["goals"], fx["rules"], fx["rule_count"],
                   fx["objs"], fx["obj_count"], threads)

    def _obs_buf(self):
        return np.empty((self.n, self.v, self.v, 2), np.uint8)

    def reset_with_keys(self, k0, k1, compute_obs: bool = True):
        k0 = np.ascontiguousarray(k0, np.uint64)
        k1 = np.ascontiguousarray(k1, np.uint64)
        obs = self._obs_buf() if compute_obs else None
        rc = lib().xmgo_reset(C.byref(self.params), C.byref(self.state), _p(k0), _p(k1), self.n,
                              _p(obs) if obs is not None else None, self.threads)
        if rc:
            raise RuntimeError(f"oracle reset failed ({rc})")
        return obs

    def reset(self, key, compute_obs: bool = True):
        return self.reset_with_keys(*split_batch(key, self.n), compute_obs)

    def step(self, actions, compute_obs: bool = True):
        a = np.ascontiguousarray(actions, np.int64)
        if a.shape != (self.n,):
            raise ValueError(f"expected {self.n} actions")
        obs = self._obs_buf() if compute_obs else None
        rew = np.empty(self.n, np.float64)
        disc = np.empty(self.n, np.float64)
        st = np.empty(self.n, np.int8)
        rc = lib().xmgo_step(C.byref(self.params), C.byref(self.state), _p(a), self.n,
                             _p(obs) if obs is not None else None, _p(rew), _p(disc), _p(st), self.threads)
        if rc == -2:
            raise ValueError("action outside [0, 6)")
        if rc:
            raise RuntimeError(f"oracle step failed ({rc})")
        return obs, rew, disc, st

    def rollout_random(self, pk0, pk1, t0: int, steps: int, compute_obs: bool = True):
        pk0 = np.ascontiguousarray(pk0, np.uint64)
        pk1 = np.ascontiguousarray(pk1, np.uint64)
        obs = self._obs_buf()
        ret = np.zeros(self.n, np.float64)
        trials = np.zeros(self.n, np.int64)
        rc = lib().xmgo_rollout_random(C.byref(self.params), C.byref(self.state), _p(pk0), _p(pk1), self.n,
                                       t0, steps, int(compute_obs), _p(obs), _p(ret), _p(trials), self.threads)
        if rc:
            raise RuntimeError(f"oracle rollout failed ({rc})")
        return ret, trials

    def observe(self):
        obs = self._obs_buf()
        lib().xmgo_observe(C.byref(self.params), C.byref(self.state), self.n, _p(obs))
        return obs

    def agent(self) -> np.ndarray:
        return np.stack([self.agent_r, self.agent_c, self.agent_dir, self.pocket], axis=1)


# ------------------------------------------------------------ observation images
IMAGE_SIDE = 224  # ref render.py:21


def sprite(tile: int, color: int, px: int) -> np.ndarray:
    """(px, px, 3) u8 sprite, ref render.py:158-169 (xmg_render_oracle.c)."""
    L = lib()
    out = np.empty((px, px, 3), np.uint8)
    if L.xmgo_sprite(C.c_int32(tile), C.c_int32(color), C.c_int32(px), C.c_void_p(_p(out))) != 0:
        raise ValueError(f"no sprite for tile {tile} color {color} at {px}px")
    return out


def image_observations(obs: np.ndarray) -> np.ndarray:
    """(n, 224, 224, 3) images of (n, v, v, 2) observations, ref render.py:225-243."""
    obs = np.ascontiguousarray(obs, dtype=np.uint8)
    n, v = obs.shape[0], obs.shape[1]
    out = np.empty((n, IMAGE_SIDE, IMAGE_SIDE, 3), np.uint8)
    L = lib()
    L.xmgo_image_observations.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p]
    if L.xmgo_image_observations(_p(obs), n, v, _p(out)) != 0:
        raise ValueError("observation outside the renderer's range")
    return out
