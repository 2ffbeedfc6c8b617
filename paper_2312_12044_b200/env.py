"""Environment parameters, action / step-type enums and the registry.

``EnvParams`` and ``make`` keep the reference's names and defaults
(ref env.py:35-73, ref registry.py:9-51): 30 registered ids, view 5,
budget 3*H*W, see-through walls.  ``make`` returns ``(Environment, params)``;
the batched engine is :class:`paper_2312_12044_b200.vecenv.VecEnv`.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import IntEnum

from .core import UnknownEnvironment
from .layouts import Layout
from .ruleset import EMPTY_RULESET, Ruleset

SCENARIO_NAMES = ("xland", "empty", "empty_random", "door_key", "four_rooms", "unlock", "unlock_pickup")


class Action(IntEnum):
    MOVE_FORWARD = 0
    TURN_LEFT = 1
    TURN_RIGHT = 2
    PICK_UP = 3
    PUT_DOWN = 4
    TOGGLE = 5


class StepType(IntEnum):
    FIRST = 0
    MID = 1
    LAST = 2


@dataclass(frozen=True)
class EnvParams:
    layout: Layout = Layout.R1
    height: int = 9
    width: int = 9
    view_size: int = 5
    max_steps: int | None = None  # None: 3*H*W
    see_through_walls: bool = True
    ruleset: Ruleset = field(default=EMPTY_RULESET)
    scenario: str = "xland"

    def __post_init__(self) -> None:
        if self.view_size < 3 or self.view_size % 2 == 0:
            raise ValueError(f"view_size must be odd and >= 3, got {self.view_size}")
        if self.scenario not in SCENARIO_NAMES:
            raise ValueError(f"unknown scenario {self.scenario!r}")

    def replace(self, **changes) -> "EnvParams":
        """Immutable update, ``env_params.replace(ruleset=...)`` as in the
        paper's JAX API (dataclasses.replace)."""
        from dataclasses import replace
        return replace(self, **changes)

    @property
    def step_budget(self) -> int:
        return self.max_steps if self.max_steps is not None else 3 * self.height * self.width


class Environment:
    """Factory handle returned by :func:`make` (ref env.py:104-117).

    The batched engine is ``VecEnv``; ``Environment.vec`` builds one.
    """

    num_actions = len(Action)

    def observation_shape(self, params: EnvParams) -> tuple[int, int, int]:
        return (params.view_size, params.view_size, 2)

    def vec(self, params: EnvParams, num_envs: int, rulesets=None, **kw):
        from .vecenv import VecEnv
        return VecEnv(params, num_envs, rulesets, **kw)


_XLAND_SIZES = {Layout.R1: (9, 13, 17), Layout.R2: (9, 13, 17), Layout.R4: (9, 13, 17),
                Layout.R6: (13, 17, 19), Layout.R9: (16, 19, 25)}
_PORT_SIZES = (5, 6, 8, 16)


def _registry() -> dict[str, EnvParams]:
    envs: dict[str, EnvParams] = {}
    for layout, sizes in _XLAND_SIZES.items():
        for s in sizes:
            envs[f"XLand-MiniGrid-R{int(layout)}-{s}x{s}"] = EnvParams(layout=layout, height=s, width=s)
    for s in _PORT_SIZES:
        envs[f"MiniGrid-Empty-{s}x{s}"] = EnvParams(height=s, width=s, scenario="empty")
        envs[f"MiniGrid-EmptyRandom-{s}x{s}"] = EnvParams(height=s, width=s, scenario="empty_random")
        envs[f"MiniGrid-DoorKey-{s}x{s}"] = EnvParams(height=s, width=s, scenario="door_key")
    envs["MiniGrid-FourRooms"] = EnvParams(layout=Layout.R4, height=19, width=19, scenario="four_rooms")
    envs["MiniGrid-Unlock"] = EnvParams(height=6, width=11, scenario="unlock")
    envs["MiniGrid-UnlockPickUp"] = EnvParams(height=6, width=11, scenario="unlock_pickup")
    return envs


REGISTRY = _registry()


def registered_environments() -> list[str]:
    return sorted(REGISTRY)


def make(name: str) -> tuple[Environment, EnvParams]:
    try:
        params = REGISTRY[name]
    except KeyError:
        raise UnknownEnvironment(f"no environment named {name!r}; see registered_environments()") from None
    return Environment(), params
