"""Rulesets, benchmark files and the on-device task table.

* ``Ruleset`` mirrors ref ruleset.py:20-59 (goal + rules + initial objects;
  ``active_rules`` / ``active_objects`` drop all-zero slots).
* ``.xmgb`` I/O follows the normative layout of ref docs/format.md and
  ref benchio.py:25-148 (little-endian header ``<4sHHIHHQH``, optional
  whole-body deflate, rows of 4 + 4*max_rules + max_objects bytes).  The body
  is kept as one (M, row) uint8 matrix: a 2^20-task file is never turned into
  Python objects on the hot path.
* ``TaskTable`` is the device form the step kernel reads (include/xmg.h):
  u32 rows [goal, rule_count | obj_count << 8, MOVE-gated slot mask,
  PICK_UP-gated slot mask, R left-packed rules, ceil(O/4) words of
  left-packed objects], built with vectorised NumPy.
* ``Benchmark.sample_ruleset`` = ``rulesets[randint(key, M)]``
  (ref benchio.py:57-58) and ``sample_indices`` is its batched twin for
  ``fold_in(root, i)`` keys, evaluated on the GPU.
"""

from __future__ import annotations

import math
import os
import struct
import threading
import zlib
from dataclasses import dataclass
from functools import cached_property
from pathlib import Path
from typing import Sequence

import numpy as np

from .core import FormatError, InvalidEncoding, InvalidProportion, Key, UnknownBenchmark, random_words, randint

HEADER_WORDS = 4  # task-table row header: goal, counts, MOVE mask, PICK_UP mask
MAX_RULES = 18
MAX_INIT_OBJECTS = 18
EMPTY_RULE = (0, 0, 0, 0)
EMPTY_GOAL = (0, 0, 0, 0)


@dataclass(frozen=True)
class Ruleset:
    goal: tuple[int, int, int, int] = EMPTY_GOAL
    rules: tuple[tuple[int, int, int, int], ...] = ()
    init_objects: tuple[int, ...] = ()

    @cached_property
    def active_rules(self) -> tuple[tuple[int, int, int, int], ...]:
        return tuple(tuple(r) for r in self.rules if tuple(r) != EMPTY_RULE)

    @cached_property
    def active_objects(self) -> tuple[int, ...]:
        return tuple(o for o in self.init_objects if o)

    def padded(self, max_rules: int = MAX_RULES, max_objects: int = MAX_INIT_OBJECTS) -> "Ruleset":
        ar, ao = self.active_rules, self.active_objects
        if len(ar) > max_rules or len(ao) > max_objects:
            raise InvalidEncoding("ruleset exceeds padded widths")
        return Ruleset(self.goal, ar + (EMPTY_RULE,) * (max_rules - len(ar)), ao + (0,) * (max_objects - len(ao)))

    def validate(self) -> "Ruleset":
        """Reject malformed encodings (ref ruleset.py:61-69 -> rules.py:126-144,
        goals.py:101-127): kinds in range, empty slots all zero, entity codes
        with tile <= 14 and color <= 13, unused arguments zero."""
        def code(c, what):
            if not (0 <= c <= 255 and c >> 4 <= 14 and c & 15 <= 13):
                raise InvalidEncoding(f"{what}: code {c} is not an entity")

        def four(enc, what):
            if len(enc) != 4 or any(not 0 <= v <= 255 for v in enc):
                raise InvalidEncoding(f"{what} encoding must be four bytes, got {enc!r}")
            return tuple(int(v) for v in enc)

        kind, a1, a2, a3 = four(self.goal, "goal")
        if kind == 0:
            if (a1, a2, a3) != (0, 0, 0):
                raise InvalidEncoding("empty goal must be all zeros")
        elif kind > 14:
            raise InvalidEncoding(f"unknown goal id {kind}")
        elif kind == 5:  # AGENT_ON_POSITION: (row, col)
            if a3 != 0:
                raise InvalidEncoding("agent-on-position goal carries (row, col) only")
        elif kind == 6:  # TILE_ON_POSITION
            code(a1, "goal tile argument")
        else:
            code(a1, "goal argument a")
            if kind in (4, 7, 8, 9, 10):  # tile-near pair goals
                code(a2, "goal argument b")
                if a3 != 0:
                    raise InvalidEncoding("pair goal carries two entity arguments only")
            elif (a2, a3) != (0, 0):
                raise InvalidEncoding(f"goal id {kind} takes a single argument")
        for r in self.rules:
            kind, a, b, out = four(r, "rule")
            if kind == 0:
                if (a, b, out) != (0, 0, 0):
                    raise InvalidEncoding("empty rule must be all zeros")
                continue
            if kind > 11:
                raise InvalidEncoding(f"unknown rule id {kind}")
            code(a, "rule input a")
            code(out, "rule output")
            if 3 <= kind <= 7:  # tile-near pair rules
                code(b, "rule input b")
            elif b != 0:
                raise InvalidEncoding(f"rule id {kind} takes a single input, in_b must be 0")
        for o in self.init_objects:
            if o:
                code(int(o), "initial object")
        return self

    def to_row(self, max_rules: int = MAX_RULES, max_objects: int = MAX_INIT_OBJECTS) -> np.ndarray:
        p = self.padded(max_rules, max_objects)
        return np.array([*p.goal, *(b for r in p.rules for b in r), *p.init_objects], np.uint8)


EMPTY_RULESET = Ruleset()


# ------------------------------------------------------------- task table
@dataclass
class TaskTable:
    """Host-side packed table; ``to_device`` uploads it once."""

    rows: np.ndarray          # (M, row_words) uint32
    rule_width: int           # R
    obj_width: int            # O
    max_objects_used: int     # max active objects over rows (GridFull check)
    # (M, agent_row_words) uint32 or None: per task only the rules a MOVE /
    # PICK_UP can fire (AGENT_HOLD and the AGENT_NEAR family), in stored order:
    # word 0 = count | MOVE slot mask << 8 | PICK_UP slot mask << 20 (masks
    # over these compact slots), then the rule words as in `rows`; rows padded
    # to 16 bytes.  step_main fetches it instead of the whole row (C3: 32 B
    # instead of 64 B per MOVE / PICK_UP action).  None when a task has more
    # than AGENT_ROW_MAX such rules.
    agent_rows: np.ndarray | None = None

    @property
    def num_tasks(self) -> int:
        return self.rows.shape[0]

    @property
    def row_words(self) -> int:
        return self.rows.shape[1]

    @property
    def goals(self) -> np.ndarray:
        return self.rows[:, 0]

    @property
    def agent_row_words(self) -> int:
        return 0 if self.agent_rows is None else self.agent_rows.shape[1]

    def to_device(self, device):
        import torch
        return torch.from_numpy(self.rows.view(np.int32)).to(device)

    def agent_rows_to_device(self, device):
        import torch
        return None if self.agent_rows is None else torch.from_numpy(self.agent_rows.view(np.int32)).to(device)


def _left_pack(active: np.ndarray, values: np.ndarray) -> np.ndarray:
    """Stable partition of active slots to the front, per row."""
    order = np.argsort(~active, axis=1, kind="stable")
    return np.take_along_axis(values, order[..., None] if values.ndim == 3 else order, axis=1)


def pack_raw_rows(raw: np.ndarray, max_rules: int, max_objects: int) -> TaskTable:
    """(M, 4+4*max_rules+max_objects) benchmark rows -> TaskTable."""
    m = raw.shape[0]
    goal = raw[:, :4]
    rules = raw[:, 4:4 + 4 * max_rules].reshape(m, max_rules, 4)
    objs = raw[:, 4 + 4 * max_rules:4 + 4 * max_rules + max_objects]
    ra = rules.any(axis=2)
    oa = objs != 0
    rc = ra.sum(axis=1)
    oc = oa.sum(axis=1)
    R = int(rc.max(initial=0))
    O = int(oc.max(initial=0))
    rules = _left_pack(ra, rules)[:, :R]
    objs = _left_pack(oa, objs)[:, :O]
    ow = (O + 3) // 4
    # rows padded to 16 bytes so the kernel fetches them with 128-bit loads
    words = np.zeros((m, (HEADER_WORDS + R + ow + 3) // 4 * 4), np.uint32)
    words[:, 0] = np.ascontiguousarray(goal).view(np.uint32)[:, 0]
    words[:, 1] = rc.astype(np.uint32) | (oc.astype(np.uint32) << 8)
    if R:
        kinds = rules[..., 0].astype(np.int64)
        slot_bits = (np.uint64(1) << np.arange(min(R, 32), dtype=np.uint64))
        agent_near = (kinds == 2) | ((kinds >= 8) & (kinds <= 11))
        # slots gated on MOVE / PICK_UP (ref rules.py:60-72); 0xFFFFFFFF when R > 32
        if R <= 32:
            words[:, 2] = (agent_near[:, :R].astype(np.uint64) * slot_bits).sum(axis=1).astype(np.uint32)
            words[:, 3] = ((agent_near | (kinds == 1))[:, :R].astype(np.uint64) * slot_bits).sum(axis=1) \
                .astype(np.uint32)
        else:
            words[:, 2] = words[:, 3] = 0xFFFFFFFF
        # AGENT_NEAR-family rules take no second input (in_b is 0, ref
        # rules.py:140-143): the table stores there the neighbour slots the
        # kind tries (NEAR_OFFSETS up, left, right, down = bits 0..3), so the
        # step kernel needs no per-kind decoding
        rules = rules.copy()
        allow = np.where(kinds == 2, 0xF, np.where((kinds >= 8) & (kinds <= 11),
                                                   (0x2841 >> (4 * np.clip(kinds - 8, 0, 3))) & 0xF, 0))
        rules[..., 2] = np.where(agent_near, allow, rules[..., 2]).astype(np.uint8)
        words[:, HEADER_WORDS:HEADER_WORDS + R] = np.ascontiguousarray(rules).view(np.uint32)[..., 0]
        agent_rows = _pack_agent_rows(words[:, HEADER_WORDS:HEADER_WORDS + R], kinds)
    else:
        agent_rows = None
    if O:
        ob = np.zeros((m, 4 * ow), np.uint8)
        ob[:, :O] = objs
        words[:, HEADER_WORDS + R:HEADER_WORDS + R + ow] = ob.view(np.uint32)
    return TaskTable(words, R, O, O, agent_rows)


AGENT_ROW_MAX = 12  # compact agent rules per task (12-bit slot masks)


def _pack_agent_rows(rule_words: np.ndarray, kinds: np.ndarray) -> np.ndarray | None:
    """TaskTable.agent_rows from the packed rule words (M, R) and their kinds."""
    near = (kinds == 2) | ((kinds >= 8) & (kinds <= 11))   # gated on MOVE and PICK_UP
    fam = near | (kinds == 1)                              # + AGENT_HOLD: PICK_UP only
    count = fam.sum(axis=1)
    a = int(count.max(initial=0))
    if a > AGENT_ROW_MAX:
        return None
    m = rule_words.shape[0]
    out = np.zeros((m, (1 + a + 3) // 4 * 4), np.uint32)
    if a:
        compact = _left_pack(fam, rule_words)[:, :a]
        near_c = _left_pack(fam, near)[:, :a]
        live = np.arange(a)[None, :] < count[:, None]
        bits = np.uint64(1) << np.arange(a, dtype=np.uint64)
        move = ((near_c & live).astype(np.uint64) * bits).sum(axis=1)
        pick = (live.astype(np.uint64) * bits).sum(axis=1)
        out[:, 1:1 + a] = np.where(live, compact, 0)
        out[:, 0] = (count.astype(np.uint64) | (move << np.uint64(8)) | (pick << np.uint64(20))).astype(np.uint32)
    return out


def pack_rulesets(rulesets: Sequence[Ruleset]) -> TaskTable:
    mr = max([len(r.active_rules) for r in rulesets] + [0])
    mo = max([len(r.active_objects) for r in rulesets] + [0])
    raw = np.stack([r.to_row(max(mr, 1), max(mo, 1)) for r in rulesets])
    return pack_raw_rows(raw, max(mr, 1), max(mo, 1))


# --------------------------------------------------------------- benchmark
MAGIC = b"XMGB"
VERSION = 1
_FLAG_DEFLATE = 1
_HEADER = struct.Struct("<4sHHIHHQH")


class Benchmark:
    """An ordered collection of equally padded rulesets (ref benchio.py:36-72),
    stored as a byte matrix (num_rulesets, row_size)."""

    def __init__(self, raw: np.ndarray, max_rules: int = MAX_RULES, max_objects: int = MAX_INIT_OBJECTS,
                 config_name: str = "", seed: int = 0):
        raw = np.ascontiguousarray(raw, np.uint8)
        if raw.ndim != 2 or raw.shape[1] != 4 + 4 * max_rules + max_objects:
            raise ValueError("benchmark rows do not match the padded widths")
        self.raw = raw
        self.max_rules = max_rules
        self.max_objects = max_objects
        self.config_name = config_name
        self.seed = seed
        self._table: TaskTable | None = None

    @classmethod
    def from_rulesets(cls, rulesets: Sequence[Ruleset], config_name: str = "", seed: int = 0) -> "Benchmark":
        widths = {(len(r.rules), len(r.init_objects)) for r in rulesets}
        if len(widths) > 1:
            raise ValueError(f"rulesets have mixed padded widths: {sorted(widths)}")
        mr, mo = widths.pop() if widths else (MAX_RULES, MAX_INIT_OBJECTS)
        raw = np.stack([np.array([*r.goal, *(b for x in r.rules for b in x), *r.init_objects], np.uint8)
                        for r in rulesets])
        return cls(raw, mr, mo, config_name, seed)

    def num_rulesets(self) -> int:
        return self.raw.shape[0]

    def __len__(self) -> int:
        return self.raw.shape[0]

    def get_ruleset(self, i: int) -> Ruleset:
        if not 0 <= i < len(self):
            raise IndexError(f"ruleset id {i} outside [0, {len(self)})")
        row = self.raw[i]
        mr = self.max_rules
        return Ruleset(tuple(int(x) for x in row[:4]),
                       tuple(tuple(int(x) for x in row[4 + 4 * s:8 + 4 * s]) for s in range(mr)),
                       tuple(int(x) for x in row[4 + 4 * mr:]))

    def sample_ruleset(self, key: Key) -> Ruleset:
        return self.get_ruleset(randint(key, len(self)))

    def shuffle(self, key: Key) -> "Benchmark":
        words = np.array(random_words(key, len(self)), dtype=np.uint64)
        order = np.argsort(words, kind="stable")
        return Benchmark(self.raw[order], self.max_rules, self.max_objects, self.config_name, self.seed)

    def split(self, prop: float) -> tuple["Benchmark", "Benchmark"]:
        if not 0.0 < prop < 1.0:
            raise InvalidProportion(f"proportion {prop} outside (0, 1)")
        cut = math.floor(prop * len(self))
        mk = lambda r: Benchmark(r, self.max_rules, self.max_objects, self.config_name, self.seed)  # noqa: E731
        return mk(self.raw[:cut]), mk(self.raw[cut:])

    def task_table(self) -> TaskTable:
        if self._table is None:
            self._table = pack_raw_rows(self.raw, self.max_rules, self.max_objects)
        return self._table


def save_benchmark(path, benchmark: Benchmark, compress: bool = True) -> None:
    if len(benchmark) == 0:
        raise ValueError("refusing to save an empty benchmark")
    payload = benchmark.raw.tobytes()
    flags = 0
    if compress:
        flags |= _FLAG_DEFLATE
        payload = zlib.compress(payload)
    name = benchmark.config_name.encode("utf-8")
    header = _HEADER.pack(MAGIC, VERSION, flags, len(benchmark), benchmark.max_rules, benchmark.max_objects,
                          benchmark.seed, len(name))
    with open(path, "wb") as fh:
        fh.write(header + name + payload)


def load_benchmark(path) -> Benchmark:
    raw = Path(path).read_bytes()
    if len(raw) < _HEADER.size:
        raise FormatError(f"{path}: truncated header ({len(raw)} bytes)")
    magic, version, flags, count, max_rules, max_objects, seed, name_len = _HEADER.unpack_from(raw)
    if magic != MAGIC:
        raise FormatError(f"{path}: bad magic {magic!r}")
    if version != VERSION:
        raise FormatError(f"{path}: unsupported version {version} (expected {VERSION})")
    name_end = _HEADER.size + name_len
    if len(raw) < name_end:
        raise FormatError(f"{path}: truncated metadata")
    name = raw[_HEADER.size:name_end].decode("utf-8")
    body = raw[name_end:]
    if flags & _FLAG_DEFLATE:
        try:
            body = zlib.decompress(body)
        except zlib.error as exc:
            raise FormatError(f"{path}: corrupt compressed body ({exc})") from exc
    row = 4 + 4 * max_rules + max_objects
    if len(body) != count * row:
        raise FormatError(f"{path}: body is {len(body)} bytes, expected {count}x{row}")
    mat = np.frombuffer(body, np.uint8).reshape(count, row)
    return Benchmark(mat, max_rules, max_objects, name, seed)


# -------------------------------------------------------- named benchmarks
REGISTERED_BENCHMARKS = ("high", "medium", "small", "trivial")
_CACHE: dict[str, tuple[int, Benchmark]] = {}
_CACHE_LOCK = threading.Lock()


def data_dir() -> Path:
    override = os.environ.get("XMINIGRID_DATA")
    return Path(override) if override else Path.home() / ".xland_minigrid"


def benchmark_path(name: str) -> Path:
    return data_dir() / f"{name}.xmgb"


def registered_benchmarks() -> tuple[str, ...]:
    return REGISTERED_BENCHMARKS


def load_named(name: str) -> Benchmark:
    """ref benchio.py:190-206: named files under $XMINIGRID_DATA, cached per
    (name, format version)."""
    if name not in REGISTERED_BENCHMARKS:
        raise UnknownBenchmark(f"unknown benchmark {name!r}; registered: {', '.join(REGISTERED_BENCHMARKS)}")
    with _CACHE_LOCK:
        hit = _CACHE.get(name)
        if hit is not None and hit[0] == VERSION:
            return hit[1]
        bm = load_benchmark(benchmark_path(name))
        _CACHE[name] = (VERSION, bm)
        return bm


def clear_cache() -> None:
    with _CACHE_LOCK:
        _CACHE.clear()
