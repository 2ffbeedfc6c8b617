"""Loader for libxmg.so, the sm_100a C-ABI library (include/xmg.h).

The product path has no CPU fallback: if the library is missing or was not
built for this machine, every entry point raises instead of computing
anything on the host.  ``build()`` compiles it in-tree with nvcc so the
shared object travels with the repository snapshot to the GPU box.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB_PATH = os.environ.get("XMG_LIB") or os.path.join(PKG, "libxmg.so")
SOURCES = [os.path.join(PKG, "csrc", "xmg_step.cu")]
DEPENDS = [os.path.join(PKG, "csrc", f) for f in ("xmg_common.cuh", "xmg_build.cuh", "xmg_main.cuh", "xmg_rare.cuh",
                                                  "xmg_rollout.cuh", "xmg_render.cuh")]
HEADER = os.path.join(ROOT, "include", "xmg.h")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xptxas", "-v", "-shared", "-Xcompiler", "-fPIC"]

ABI_VERSION = 3

# scenario ids of include/xmg.h (ref scenarios.py:177-185)
SCENARIO_IDS = {"xland": 0, "empty": 1, "empty_random": 2, "door_key": 3, "four_rooms": 4,
                "unlock": 5, "unlock_pickup": 6}
ACT_U8, ACT_I32, ACT_I64 = 0, 1, 2

EXPORTS = ("xmg_abi_version", "xmg_last_error", "xmg_philox", "xmg_split_batch", "xmg_random_actions",
           "xmg_key_from_seed", "xmg_fold_in", "xmg_philox_host", "xmg_reset", "xmg_validate_actions",
           "xmg_step", "xmg_step_smem_bytes", "xmg_work_words", "xmg_profile", "xmg_profile_read", "xmg_rollout",
           "xmg_rollout_smem_bytes", "xmg_sprites", "xmg_image_obs", "xmg_steps", "xmg_image_atlas_bytes",
           "xmg_image_atlas", "xmg_image_obs_aligned", "xmg_ahead_plan", "xmg_prebuild",
           "xmg_step_fused", "xmg_graph_create", "xmg_graph_launch", "xmg_graph_destroy", "xmg_step_validated",
           "xmg_graph_step")


class NativeLibraryError(RuntimeError):
    """libxmg.so is missing, stale, or a CUDA call failed."""


class EnvDesc(C.Structure):
    _fields_ = [("height", C.c_int32), ("width", C.c_int32), ("view_size", C.c_int32), ("budget", C.c_int32),
                ("scenario", C.c_int32), ("see_through_walls", C.c_int32), ("num_segments", C.c_int32),
                ("fixed_doors", C.c_int32), ("rule_width", C.c_int32), ("obj_width", C.c_int32),
                ("row_words", C.c_int32), ("num_tasks", C.c_int32), ("resample_tasks", C.c_int32),
                ("base_cells", C.c_void_p),
                ("seg_off", C.c_void_p), ("seg_cells", C.c_void_p), ("task_rows", C.c_void_p),
                ("agent_row_words", C.c_int32), ("agent_rows", C.c_void_p)]


class State(C.Structure):
    _fields_ = [("grids", C.c_void_p), ("agent", C.c_void_p), ("rng", C.c_void_p), ("work", C.c_void_p),
                ("next_grids", C.c_void_p), ("next_state", C.c_void_p), ("next_obs", C.c_void_p)]


class Out(C.Structure):
    _fields_ = [("obs", C.c_void_p), ("reward", C.c_void_p), ("discount", C.c_void_p),
                ("step_type", C.c_void_p), ("stats", C.c_void_p)]


_lock = threading.Lock()
_lib = None


def build(verbose: bool = False, out: str | None = None, defines: tuple[str, ...] = ()) -> str:
    """Compile libxmg.so for sm_100a in-tree (nvcc); returns its path."""
    out = out or os.path.join(PKG, "libxmg.so")
    cmd = ["nvcc", *NVCC_FLAGS, *(f"-D{d}" for d in defines), "-o", out, *SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise NativeLibraryError(f"nvcc failed:\n{res.stderr}")
    if verbose:
        print(res.stderr)
    return out


def _bind(L):
    vp, i64, i32, u64 = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64
    sig = {
        "xmg_abi_version": ([], i32),
        "xmg_last_error": ([], C.c_char_p),
        "xmg_philox": ([vp, vp, vp, i64, vp], i32),
        "xmg_split_batch": ([u64, u64, i64, i64, vp, vp], i32),
        "xmg_random_actions": ([vp, i64, i64, i64, vp, vp], i32),
        "xmg_key_from_seed": ([u64, u64, vp], None),
        "xmg_fold_in": ([u64, u64, u64, u64, i32, vp], None),
        "xmg_philox_host": ([vp, u64, u64, vp], None),
        "xmg_reset": ([C.POINTER(EnvDesc), C.POINTER(State), vp, i64, C.POINTER(Out), vp], i32),
        "xmg_validate_actions": ([vp, i32, i64, C.c_uint32, vp, vp], i32),
        "xmg_step": ([C.POINTER(EnvDesc), C.POINTER(State), vp, i32, i64, C.POINTER(Out), vp, C.c_uint32, vp], i32),
        "xmg_step_validated": ([C.POINTER(EnvDesc), C.POINTER(State), vp, i32, i64, C.POINTER(Out), vp, C.c_uint32,
                                vp], i32),
        "xmg_step_smem_bytes": ([C.POINTER(EnvDesc)], i64),
        "xmg_work_words": ([i64], i64),
        "xmg_profile": ([i32], i32),
        "xmg_profile_read": ([vp, vp, vp], i32),
        "xmg_rollout": ([C.POINTER(EnvDesc), C.POINTER(State), vp, vp, i64, i64, i64, C.POINTER(Out), vp], i32),
        "xmg_rollout_smem_bytes": ([C.POINTER(EnvDesc)], i64),
        "xmg_sprites": ([i32, vp, vp], i32),
        "xmg_steps": ([C.POINTER(EnvDesc), C.POINTER(State), vp, i32, i64, i64, C.POINTER(Out), C.c_uint32, vp], i32),
        "xmg_image_obs": ([vp, i64, i32, vp, vp, vp], i32),
        "xmg_image_atlas_bytes": ([i32], i64),
        "xmg_image_atlas": ([i32, vp, vp, vp], i32),
        "xmg_image_obs_aligned": ([vp, i64, i32, vp, vp, vp], i32),
        "xmg_ahead_plan": ([C.POINTER(EnvDesc), i64, vp, vp], i32),
        "xmg_prebuild": ([C.POINTER(EnvDesc), C.POINTER(State), i64, i64, i64, vp], i32),
        "xmg_step_fused": ([C.POINTER(EnvDesc), C.POINTER(State), vp, i64, C.POINTER(Out), vp, vp], i32),
        "xmg_graph_create": ([C.POINTER(EnvDesc), C.POINTER(State), vp, i64, C.POINTER(Out), vp,
                              C.POINTER(C.c_void_p)], i32),
        "xmg_graph_launch": ([vp, vp], i32),
        "xmg_graph_step": ([vp, vp, vp, i64, vp], i32),
        "xmg_graph_destroy": ([vp], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    return L


def lib():
    """The loaded library; raises NativeLibraryError when it is unavailable."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryError(
                    f"{LIB_PATH} is missing; run __graft_entry__.build() (nvcc, sm_100a). "
                    "There is no CPU fallback for the batched step.")
            L = _bind(C.CDLL(LIB_PATH))
            v = L.xmg_abi_version()
            if v != ABI_VERSION:
                raise NativeLibraryError(f"libxmg ABI {v} != expected {ABI_VERSION}; rebuild")
            _lib = L
    return _lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().xmg_last_error().decode(errors="replace")
        raise NativeLibraryError(f"{what} failed: {msg}")
