"""Scheme enum, tiling config and fault specs (reference tiled.py:42-146).

``TilingConfig`` keeps the reference's meaning on B200: ``thread_n`` (Nt) is the
checksum column-group width and ``thread_m`` (Mt) the number of rows folded into
one thread-tile verdict; ``tb_m`` / ``tb_n`` only define the zero-padded extents
the verdict grid covers (tiled.py:423-431).  The CTA tile of the sm_100a kernel
is a separate, internal choice.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass
from typing import Union

import numpy as np

from .shapes import GemmShape


class Scheme(enum.Enum):
    UNPROTECTED = "unprotected"
    GLOBAL_ABFT = "global-abft"
    THREAD_ONE_SIDED = "thread-one-sided"
    THREAD_TWO_SIDED = "thread-two-sided"
    THREAD_REPLICATION_FULL = "thread-replication-full"
    THREAD_REPLICATION_SINGLE_ACC = "thread-replication-single-acc"


THREAD_LEVEL_SCHEMES = (
    Scheme.THREAD_ONE_SIDED,
    Scheme.THREAD_TWO_SIDED,
    Scheme.THREAD_REPLICATION_FULL,
    Scheme.THREAD_REPLICATION_SINGLE_ACC,
)
PROTECTED_SCHEMES = (Scheme.GLOBAL_ABFT,) + THREAD_LEVEL_SCHEMES

# C-ABI scheme codes (include/abft_b200.h), same order as the enum
SCHEME_CODE = {s: i for i, s in enumerate(Scheme)}


def scheme_from_name(name: str) -> Scheme:
    for s in Scheme:
        if s.value == name:
            return s
    raise ValueError(f"unknown scheme {name!r}; expected one of {[s.value for s in Scheme]}")


@dataclass(frozen=True)
class TilingConfig:
    tb_m: int = 128
    tb_n: int = 128
    warp_m: int = 64
    warp_n: int = 64
    thread_m: int = 16
    thread_n: int = 8
    k_step: int = 2

    def __post_init__(self):
        for f in ("tb_m", "tb_n", "warp_m", "warp_n", "thread_m", "thread_n", "k_step"):
            if getattr(self, f) < 1:
                raise ValueError(f"TilingConfig.{f} must be >= 1")
        if self.tb_m % self.warp_m or self.tb_n % self.warp_n:
            raise ValueError("threadblock tile must be divisible by the warp tile")
        if self.warp_m % self.thread_m or self.warp_n % self.thread_n:
            raise ValueError("warp tile must be divisible by the thread tile")
        if self.thread_m % 2:
            raise ValueError("thread_m must be even (each MMA consumes two rows)")


@dataclass(frozen=True)
class OutputFault:
    """delta added to output element (row, col) after accumulation."""

    row: int
    col: int
    delta: float

    def __post_init__(self):
        if self.delta == 0:
            raise ValueError("fault delta must be nonzero")


@dataclass(frozen=True)
class ThreadMmaFault:
    """A corrupted MMA of one thread's K walk; lands on cell local_index of its Mt x Nt tile."""

    thread_row: int
    thread_col: int
    step: int
    local_index: int
    delta: float

    def __post_init__(self):
        if self.delta == 0:
            raise ValueError("fault delta must be nonzero")


FaultSpec = Union[OutputFault, ThreadMmaFault]


def random_output_fault(rng: np.random.Generator, shape: GemmShape, delta: float) -> OutputFault:
    return OutputFault(row=int(rng.integers(shape.m)), col=int(rng.integers(shape.n)), delta=delta)


def random_thread_mma_fault(rng: np.random.Generator, shape: GemmShape, tiling: TilingConfig,
                            delta: float) -> ThreadMmaFault:
    """Uniform over real (non-padding) output cells and K steps (tiled.py:131-146)."""
    row, col = int(rng.integers(shape.m)), int(rng.integers(shape.n))
    return ThreadMmaFault(
        thread_row=row // tiling.thread_m,
        thread_col=col // tiling.thread_n,
        step=int(rng.integers(-(-shape.k // tiling.k_step))),
        local_index=(row % tiling.thread_m) * tiling.thread_n + col % tiling.thread_n,
        delta=delta,
    )


def validate_faults(faults, shape: GemmShape, tiling: TilingConfig) -> None:
    """Range checks of tiled.py:360-383 (ValueError, padding cells rejected)."""
    steps = -(-shape.k // tiling.k_step)
    mt, nt = tiling.thread_m, tiling.thread_n
    for f in faults:
        if isinstance(f, OutputFault):
            if not (0 <= f.row < shape.m and 0 <= f.col < shape.n):
                raise ValueError(f"output fault at ({f.row}, {f.col}) is outside the {shape.m}x{shape.n} output")
        elif isinstance(f, ThreadMmaFault):
            if not (0 <= f.local_index < mt * nt):
                raise ValueError(f"local output index {f.local_index} outside {mt}x{nt} tile")
            if not (0 <= f.step < steps):
                raise ValueError(f"step {f.step} outside {steps} K steps")
            r, c = fault_cell(f, tiling)[:2]
            if not (0 <= r < shape.m and 0 <= c < shape.n):
                raise ValueError(f"thread-mma fault maps to padding cell ({r}, {c}) of {shape.m}x{shape.n} output")
        else:
            raise ValueError(f"unsupported fault type {type(f).__name__}")


def fault_cell(f: FaultSpec, tiling: TilingConfig) -> tuple:
    """(row, col, delta) of the output element a fault corrupts (tiled.py:386-397)."""
    if isinstance(f, OutputFault):
        return f.row, f.col, f.delta
    return (f.thread_row * tiling.thread_m + f.local_index // tiling.thread_n,
            f.thread_col * tiling.thread_n + f.local_index % tiling.thread_n, f.delta)
