"""A B200 ``DeviceProfile`` fitted to measured per-layer timings.

The reference selector (cost.select, cost.py:174-238) predicts each layer's unprotected,
global and thread-level time from a four-number device model (cost.py:77-128: tensor rate,
scalar ALU rate, memory bandwidth, verification launch latency).  Its defaults describe the
paper's T4.  ``fit_device_profile`` searches a log grid of those four numbers around the
measured B200 peaks for the profile whose *model-only* choices (no measured rows) agree with
the choices the measured timings make on the most layers; ties go to the profile whose
choices cost the least measured protected time.  Host-only: no GPU, no kernels.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass
from typing import Sequence

from .cost import SELECTABLE_SCHEMES, scheme_time
from .schemes import Scheme, TilingConfig
from .shapes import DeviceProfile, DType, GemmShape


@dataclass(frozen=True)
class LayerTiming:
    """One layer's shape and measured seconds per scheme (unprotected, global, one-sided)."""

    shape: GemmShape
    t_unprotected: float
    t_global: float
    t_thread: float

    def measured(self, scheme: Scheme) -> float:
        return {Scheme.UNPROTECTED: self.t_unprotected, Scheme.GLOBAL_ABFT: self.t_global,
                Scheme.THREAD_ONE_SIDED: self.t_thread}[scheme]

    def best_measured(self) -> Scheme:
        # cost.select's rule on measured rows: lowest overhead, ties -> global (SELECTABLE order)
        return min(SELECTABLE_SCHEMES, key=lambda s: (self.measured(s), SELECTABLE_SCHEMES.index(s)))


@dataclass(frozen=True)
class FitResult:
    device: DeviceProfile
    agreement: float            # fraction of layers whose model choice equals the measured choice
    model_plan_time: float      # sum of measured times of the model-chosen schemes
    measured_plan_time: float   # sum of measured times of the measured-optimal schemes
    unprotected_time: float
    n_layers: int


def model_choice(shape: GemmShape, dtype: DType, device: DeviceProfile, tiling: TilingConfig) -> Scheme:
    t = {s: scheme_time(shape, dtype, device, s, tiling) for s in SELECTABLE_SCHEMES}
    return min(SELECTABLE_SCHEMES, key=lambda s: (t[s], SELECTABLE_SCHEMES.index(s)))


def evaluate(rows: Sequence[LayerTiming], dtype: DType, device: DeviceProfile,
             tiling: TilingConfig = TilingConfig()) -> FitResult:
    agree, t_model, t_best, t_un = 0, 0.0, 0.0, 0.0
    for r in rows:
        c = model_choice(r.shape, dtype, device, tiling)
        b = r.best_measured()
        agree += int(c == b)
        t_model += r.measured(c)
        t_best += r.measured(b)
        t_un += r.t_unprotected
    return FitResult(device=device, agreement=agree / max(1, len(rows)), model_plan_time=t_model,
                     measured_plan_time=t_best, unprotected_time=t_un, n_layers=len(rows))


def fit_device_profile(rows: Sequence[LayerTiming], dtype: DType, peaks: DeviceProfile,
                       scales=(1 / 16, 1 / 8, 1 / 4, 1 / 2, 1.0, 2.0),
                       latencies=(0.0, 0.25e-6, 0.5e-6, 1e-6, 2e-6, 5e-6),
                       tiling: TilingConfig = TilingConfig()) -> FitResult:
    """Grid search (scales of the measured peaks x verification latencies); best agreement wins,
    then the least measured protected time of the model's plan."""
    best = None
    for ts, as_, bs, lat in itertools.product(scales, scales, scales, latencies):
        dev = DeviceProfile(name=f"{peaks.name}-fitted", tensor_throughput=peaks.tensor_throughput * ts,
                            alu_throughput=peaks.alu_throughput * as_, memory_bandwidth=peaks.memory_bandwidth * bs,
                            verification_launch_latency=lat)
        res = evaluate(rows, dtype, dev, tiling)
        if best is None or (res.agreement, -res.model_plan_time) > (best.agreement, -best.model_plan_time):
            best = res
    return best
