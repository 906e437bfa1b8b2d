"""Seeded fault-injection campaigns on the B200 path (the reference's campaign semantics).

"The same deterministic injected faults" of the north star are defined by the
reference harness (campaign.py:198-259): trial t of scheme index s draws its GEMM
extents, operands, fault magnitude, fault site and fault position from
``SeedSequence([seed, s, kind, t])`` (kind 0 injected, 1 fault-free control).  This
module keeps that generator bit for bit and swaps only the executor: every trial runs
the sm_100a protected GEMM through ``tiled.execute``.  A trial is *detected* when the
report flags, *masked* when it does not and |delta| <= tau of the verdict responsible
for the faulted cell (campaign.py:213-224), *missed* otherwise.

The reference's process pool (campaign.py:281-310) is host plumbing and is not
reproduced: trials run back to back on the one GPU of this process.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from .schemes import OutputFault, Scheme, TilingConfig, random_output_fault, random_thread_mma_fault
from .shapes import DType, DTypeTag, GemmShape

# campaign.py:45 — small tiling that still exercises the whole thread hierarchy
CAMPAIGN_TILING = TilingConfig(tb_m=32, tb_n=32, warp_m=16, warp_n=16, thread_m=8, thread_n=8, k_step=2)
SITE_OUTPUT, SITE_THREAD_MMA, SITE_MIXED = "output-element", "thread-mma", "mixed"


@dataclass(frozen=True)
class DeltaDistribution:
    """campaign.py:52-65: nonzero uniform integers, or sign * log-uniform magnitude."""

    kind: str
    low: float
    high: float

    def sample(self, rng: np.random.Generator):
        negative = bool(rng.integers(2))
        if self.kind == "int-uniform":
            mag = int(rng.integers(int(self.low), int(self.high) + 1))
            return -mag if negative else mag
        mag = float(np.exp(rng.uniform(np.log(self.low), np.log(self.high))))
        return -mag if negative else mag


INT_DELTAS = DeltaDistribution("int-uniform", 1, 100)
FP_DELTAS = DeltaDistribution("log-uniform", 1e-2, 1e2)


@dataclass(frozen=True)
class CampaignConfig:
    trials: int
    seed: int
    gemm_min: int
    gemm_max: int
    schemes: tuple
    dtype: DType
    delta: DeltaDistribution
    control_trials: int
    site: str = SITE_MIXED
    tiling: TilingConfig = CAMPAIGN_TILING


@dataclass
class SchemeStats:
    injected_trials: int = 0
    detected: int = 0
    masked_by_tolerance: int = 0
    missed: int = 0
    control_trials: int = 0
    false_positives: int = 0
    outcomes: list = field(default_factory=list)     # per injected trial: "detected" | "masked" | "missed"

    @property
    def detection_rate(self) -> float:
        return self.detected / self.injected_trials if self.injected_trials else 0.0

    @property
    def false_positive_rate(self) -> float:
        return self.false_positives / self.control_trials if self.control_trials else 0.0


def trial_rng(seed: int, scheme_index: int, kind: int, trial: int) -> np.random.Generator:
    """campaign.py:198-199."""
    return np.random.default_rng(np.random.SeedSequence([seed, scheme_index, kind, trial]))


def random_matrices(rng: np.random.Generator, shape: GemmShape, dtype: DType):
    """campaign.py:202-210: ints in [-8, 8] (exact) or U(-1, 1) in the storage type."""
    if dtype.is_exact:
        return (rng.integers(-8, 9, size=(shape.m, shape.k), dtype=np.int64),
                rng.integers(-8, 9, size=(shape.k, shape.n), dtype=np.int64))
    t = np.float16 if dtype.tag is DTypeTag.BINARY16 else np.float32
    return (rng.uniform(-1.0, 1.0, size=(shape.m, shape.k)).astype(t),
            rng.uniform(-1.0, 1.0, size=(shape.k, shape.n)).astype(t))


def _shape(rng, cfg: CampaignConfig) -> GemmShape:
    return GemmShape(m=int(rng.integers(cfg.gemm_min, cfg.gemm_max + 1)),
                     n=int(rng.integers(cfg.gemm_min, cfg.gemm_max + 1)),
                     k=int(rng.integers(cfg.gemm_min, cfg.gemm_max + 1)))


def responsible_tolerance(report, fault, tiling: TilingConfig) -> float:
    """campaign.py:213-224: tau of the verdict covering the faulted cell."""
    if report.scheme is Scheme.GLOBAL_ABFT:
        return report.verdicts[0].tolerance_used
    if isinstance(fault, OutputFault):
        coords = (fault.row // tiling.thread_m, fault.col // tiling.thread_n)
    else:
        coords = (fault.thread_row, fault.thread_col)
    for v in report.verdicts:
        if (v.thread_row, v.thread_col) == coords:
            return v.tolerance_used
    return 0.0


def trial_spec(cfg: CampaignConfig, scheme_index: int, trial: int):
    """The seeded draws of one injected trial (campaign.py:229-243): shape, A, B, delta, fault."""
    rng = trial_rng(cfg.seed, scheme_index, 0, trial)
    shape = _shape(rng, cfg)
    a, b = random_matrices(rng, shape, cfg.dtype)
    delta = cfg.delta.sample(rng)
    site = cfg.site
    if site == SITE_MIXED:
        site = SITE_OUTPUT if rng.integers(2) else SITE_THREAD_MMA
    fault = (random_output_fault(rng, shape, delta) if site == SITE_OUTPUT
             else random_thread_mma_fault(rng, shape, cfg.tiling, delta))
    return shape, a, b, delta, fault


def injected_trial(cfg: CampaignConfig, scheme: Scheme, scheme_index: int, trial: int):
    """One injected trial (campaign.py:227-247) -> (outcome, delta, responsible tau)."""
    from .tiled import execute
    shape, a, b, delta, fault = trial_spec(cfg, scheme_index, trial)
    report = execute(a, b, cfg.tiling, scheme, faults=[fault], dtype=cfg.dtype)
    tau = responsible_tolerance(report, fault, cfg.tiling)
    if report.detected:
        return "detected", delta, tau
    return ("masked" if abs(delta) <= tau else "missed"), delta, tau


def control_trial(cfg: CampaignConfig, scheme: Scheme, scheme_index: int, trial: int) -> bool:
    """One fault-free trial (campaign.py:250-259) -> flagged (a false positive)."""
    from .tiled import execute
    rng = trial_rng(cfg.seed, scheme_index, 1, trial)
    shape = _shape(rng, cfg)
    a, b = random_matrices(rng, shape, cfg.dtype)
    return execute(a, b, cfg.tiling, scheme, dtype=cfg.dtype).detected


def run_campaign(cfg: CampaignConfig, trial_range: Sequence[int] | None = None) -> dict:
    """All schemes' injected and control trials; returns {scheme: SchemeStats}."""
    out = {}
    for si, scheme in enumerate(cfg.schemes):
        st = SchemeStats()
        rng_trials = trial_range if trial_range is not None else range(cfg.trials)
        for t in rng_trials:
            outcome, _, _ = injected_trial(cfg, scheme, si, t)
            st.injected_trials += 1
            st.outcomes.append(outcome)
            if outcome == "detected":
                st.detected += 1
            elif outcome == "masked":
                st.masked_by_tolerance += 1
            else:
                st.missed += 1
        for t in range(cfg.control_trials if trial_range is None else len(rng_trials)):
            st.control_trials += 1
            st.false_positives += int(control_trial(cfg, scheme, si, t))
        out[scheme] = st
    return out
