"""C-ABI library checks that need no GPU: libxmg.so loads, exports every
entry point include/xmg.h declares, reports its ABI version, validates
descriptions before touching CUDA, and its host key helpers agree with the
oracle (and so with the reference, see test_oracle_golden.py)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from paper_2312_12044_b200 import _lib, fold_in, key_from_seed, random_words, split
from paper_2312_12044_b200.core import philox_block

from .conftest import ROOT

HEADER = os.path.join(ROOT, "include", "xmg.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(xmg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = C.CDLL(_lib.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 12
    for name in names:
        assert hasattr(L, name), f"{name} declared in include/xmg.h but not exported"
    assert set(names) == set(_lib.EXPORTS)


def test_abi_version_and_error_channel():
    L = _lib.lib()
    assert L.xmg_abi_version() == _lib.ABI_VERSION
    # a bad description is rejected on the host, before any CUDA call
    d = _lib.EnvDesc(9, 9, 4, 243, 0, 1, 0, 0, 0, 0, 4, 1, 0, 1, 1, 1, 1, 0, None)
    st = _lib.State(1, 1, 1, 1)
    out = _lib.Out(None, 1, 1, 1, None)
    rc = L.xmg_step(C.byref(d), C.byref(st), 1, 0, 8, C.byref(out), None, 1, None)
    assert rc < 0
    assert b"view_size" in L.xmg_last_error()
    d.view_size, d.height = 5, 300
    assert L.xmg_reset(C.byref(d), C.byref(st), 1, 8, C.byref(out), None) < 0
    assert b"grid size" in L.xmg_last_error()
    assert L.xmg_work_words(1 << 20) > (1 << 21)
    assert L.xmg_work_words(1 << 30) == -1 and L.xmg_work_words(-1) == -1


def test_host_key_helpers_match_oracle():
    for seed in (0, 1, 20240601, 2**70 + 5):
        k = key_from_seed(seed)
        assert tuple(k) == O.key_from_seed(seed)
        assert tuple(fold_in(k, 77)) == O.fold_in(tuple(k), 77, 3)
        assert [tuple(x) for x in split(k, 3)] == [O.fold_in(tuple(k), i, 2) for i in range(3)]
    k = key_from_seed(9)
    words = random_words(k, 11)
    ref = O.philox(np.array([[b, 0, 1, 0] for b in range(3)], np.uint64), np.array([[k.hi, k.lo]] * 3, np.uint64))
    assert words == [int(x) for x in ref.reshape(-1)[:11]]
    assert philox_block((1, 2, 3, 4), k) == tuple(int(x) for x in O.philox(np.array([[1, 2, 3, 4]], np.uint64),
                                                                          np.array([[k.hi, k.lo]], np.uint64))[0])


def test_vecenv_refuses_cpu_device():
    from paper_2312_12044_b200 import EnvParams, NativeLibraryError, VecEnv
    with pytest.raises(NativeLibraryError):
        VecEnv(EnvParams(), 4, device="cpu")


def test_fold_in_takes_the_full_128_bit_counter():
    """ref rng.py:107-110 folds in (data & 2^64-1, data >> 64 & 2^64-1):
    negative and >= 2^64 data must match the reference (values from
    rulegrid.rng.fold_in(key_from_seed(7), data), computed with the
    reference in the build container)."""
    k = key_from_seed(7)
    assert tuple(k) == (5153160078105390988, 9456252307694779705)
    want = {-1: (7204942696657869296, 9289732693193205544),
            2 ** 64 + 5: (12675942302801154926, 15253322680772628831),
            2 ** 70 - 3: (14688658413190397962, 14771808042739616059),
            12345: (3444096608153625987, 1418527488995923867)}
    for data, key in want.items():
        assert tuple(fold_in(k, data)) == key, data
