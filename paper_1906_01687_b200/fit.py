"""fit_gcp_adam — the reference's epoch-based stochastic fit
(src/optimizer.cpp:68-158, include/gcp/optimizer.hpp:42-93) driven natively
by gcpb_fit_gcp_adam: the epoch loop runs on the device (one CUDA graph per
epoch of `epoch_iters` iterations), with the reference's init, fixed-sample
loss estimate, accept/rollback and learning-rate decay."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _capi
from ._capi import lib
from .gcp import Engine, LossFunction, SamplerKind, _check


@dataclass
class FitConfig:
    """FitConfig (include/gcp/optimizer.hpp:42-65); defaults as the reference."""
    rank: int = 2
    sampler: SamplerKind = field(default_factory=lambda: SamplerKind.uniform(1))
    learning_rate: float = 0.01
    beta1: float = 0.9
    beta2: float = 0.999
    epsilon: float = 1e-8
    epoch_iters: int = 1000
    max_bad_epochs: int = 1
    decay: float = 0.1
    lower_bound: Optional[float] = None   # None: the loss's default bound
    no_lower_bound: bool = False          # force no bound (reference: explicit nullopt via loss)
    estimator_samples: int = 100000
    estimator_kind: Optional[int] = None  # None: stratified if sparse, uniform if dense
    max_epochs: int = 100
    seed: int = 0
    keep_factors: bool = False            # start from the engine's current factors
    draw_stream: str = "philox"           # "reference": RefStream, the reference's own draws


@dataclass
class FitTraceRecord:
    epoch: int
    loss_estimate: float
    learning_rate: float
    seconds: float
    accepted: bool


@dataclass
class FitResult:
    model: List[np.ndarray]
    trace: List[FitTraceRecord]
    final_loss_estimate: float


def fit_gcp_adam(engine: Engine, loss: LossFunction, cfg: FitConfig) -> FitResult:
    if cfg.rank != engine.rank:
        raise ValueError("FitConfig.rank must match the engine rank")
    c = _capi.gcpb_fit_config()
    c.sampler = cfg.sampler.c()
    c.learning_rate = cfg.learning_rate
    c.beta1, c.beta2, c.epsilon = cfg.beta1, cfg.beta2, cfg.epsilon
    c.epoch_iters = cfg.epoch_iters
    c.max_bad_epochs = cfg.max_bad_epochs
    c.decay = cfg.decay
    if cfg.no_lower_bound:
        c.lower_bound_mode = 2
    elif cfg.lower_bound is not None:
        c.lower_bound_mode, c.lower_bound = 1, float(cfg.lower_bound)
    else:
        c.lower_bound_mode = 0
    c.estimator_samples = cfg.estimator_samples
    c.estimator_kind = -1 if cfg.estimator_kind is None else int(cfg.estimator_kind)
    c.max_epochs = cfg.max_epochs
    c.seed = cfg.seed
    c.keep_factors = 1 if cfg.keep_factors else 0
    c.draw_stream = 1 if cfg.draw_stream == "reference" else 0
    cap = cfg.max_epochs + 1
    trace = (_capi.gcpb_trace_record * cap)()
    n = C.c_int64()
    final = C.c_double()
    ls = loss.c()
    _check(lib.gcpb_fit_gcp_adam(engine.handle, C.byref(ls), C.byref(c), trace, cap, C.byref(n),
                                 C.byref(final)), engine.handle)
    recs = [FitTraceRecord(int(t.epoch), t.loss_estimate, t.learning_rate, t.seconds,
                           bool(t.accepted)) for t in trace[:min(n.value, cap)]]
    return FitResult(engine.factors(), recs, final.value)
