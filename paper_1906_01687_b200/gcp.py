"""Host-side mirror of the reference API for the stochastic GCP hot path.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/gcp/*.hpp); every computation on the hot path
goes through the C-ABI (include/gcpb.h) into the sm_100a engine.  Exceptions
mirror the reference's: std::invalid_argument -> InvalidArgument(ValueError),
std::domain_error -> DomainError(ValueError), std::out_of_range ->
OutOfRange(IndexError), std::logic_error -> LogicError, std::runtime_error ->
GcpRuntimeError.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _capi
from ._capi import lib


# ---------------------------------------------------------------------------
# Errors (status codes of include/gcpb.h)
# ---------------------------------------------------------------------------
class GcpError(Exception):
    pass


class InvalidArgument(GcpError, ValueError):
    pass


class DomainError(GcpError, ValueError):
    pass


class OutOfRange(GcpError, IndexError):
    pass


class LogicError(GcpError, RuntimeError):
    pass


class GcpRuntimeError(GcpError, RuntimeError):
    pass


_ERR = {_capi.ERR_RUNTIME: GcpRuntimeError, _capi.ERR_USAGE: InvalidArgument,
        _capi.ERR_DOMAIN: DomainError, _capi.ERR_RANGE: OutOfRange, _capi.ERR_LOGIC: LogicError}


def _check(rc: int, ctx=None) -> None:
    if rc != _capi.OK:
        msg = lib.gcpb_last_error(ctx)
        raise _ERR.get(rc, GcpRuntimeError)(msg.decode() if msg else f"gcpb error {rc}")


def _i64(a):
    return a.ctypes.data_as(_capi.i64p)


def _f64(a):
    return a.ctypes.data_as(_capi.f64p)


def _i32(a):
    return a.ctypes.data_as(_capi.i32p)


# ---------------------------------------------------------------------------
# LossFunction (include/gcp/loss.hpp:8-57, src/loss.cpp)
# ---------------------------------------------------------------------------
GAUSSIAN, POISSON, BERNOULLI_ODDS, GAMMA, BETA_HALF, HUBER = range(6)
_LOSS_NAMES = {GAUSSIAN: "gaussian", POISSON: "poisson", BERNOULLI_ODDS: "bernoulli-odds",
               GAMMA: "gamma", BETA_HALF: "beta-half", HUBER: "huber"}


@dataclass(frozen=True)
class LossFunction:
    kind: int
    delta: float = 0.0

    kEps = 1e-10

    @staticmethod
    def gaussian():
        return LossFunction(GAUSSIAN)

    @staticmethod
    def poisson():
        return LossFunction(POISSON)

    @staticmethod
    def bernoulli_odds():
        return LossFunction(BERNOULLI_ODDS)

    @staticmethod
    def gamma():
        return LossFunction(GAMMA)

    @staticmethod
    def beta_half():
        return LossFunction(BETA_HALF)

    @staticmethod
    def huber(delta: float):
        if not delta > 0.0:  # loss.cpp:17-18
            raise InvalidArgument("huber: delta must be > 0")
        return LossFunction(HUBER, float(delta))

    @staticmethod
    def parse(token: str) -> "LossFunction":  # loss.cpp:21-40
        simple = {"gaussian": GAUSSIAN, "poisson": POISSON, "bernoulli-odds": BERNOULLI_ODDS,
                  "gamma": GAMMA, "beta-half": BETA_HALF}
        if token in simple:
            return LossFunction(simple[token])
        if token.startswith("huber:"):
            arg = token[6:]
            try:
                delta = float(arg)
            except ValueError:
                raise InvalidArgument(f"huber: bad delta '{arg}'") from None
            return LossFunction.huber(delta)
        raise InvalidArgument(f"unknown loss '{token}'")

    @property
    def name(self) -> str:
        return f"huber:{self.delta:f}" if self.kind == HUBER else _LOSS_NAMES[self.kind]

    def c(self) -> _capi.gcpb_loss:
        return _capi.gcpb_loss(self.kind, self.delta)

    def value(self, x: float, m: float) -> float:
        self.check_domain(x)
        loss = self.c()
        return lib.gcpb_loss_value(C.byref(loss), float(x), float(m))

    def deriv(self, x: float, m: float) -> float:
        self.check_domain(x)
        loss = self.c()
        return lib.gcpb_loss_deriv(C.byref(loss), float(x), float(m))

    def check_domain(self, x: float) -> None:  # loss.cpp:42-62
        if self.kind in (POISSON, GAMMA, BETA_HALF) and not x >= 0.0:
            raise DomainError(f"{self.name} loss: data value {x} out of domain (x >= 0 required)")
        if self.kind == BERNOULLI_ODDS and x not in (0.0, 1.0):
            raise DomainError(f"{self.name} loss: data value {x} out of domain (x in {{0,1}} required)")

    def default_lower_bound(self) -> Optional[float]:  # loss.cpp:112-124
        return 0.0 if self.kind in (POISSON, BERNOULLI_ODDS, GAMMA, BETA_HALF) else None


# ---------------------------------------------------------------------------
# SamplerKind / RejectionStats (include/gcp/samplers.hpp:31-57)
# ---------------------------------------------------------------------------
UNIFORM, STRATIFIED, SEMI_STRATIFIED = _capi.UNIFORM, _capi.STRATIFIED, _capi.SEMI_STRATIFIED


@dataclass
class SamplerKind:
    strategy: int = UNIFORM
    num_samples: int = 0
    nonzero_samples: int = 0
    zero_samples: int = 0
    oversample: float = 1.1

    @staticmethod
    def uniform(s: int) -> "SamplerKind":
        k = SamplerKind(UNIFORM, num_samples=int(s))
        k.validate()
        return k

    @staticmethod
    def stratified(p: int, q: int, rho: float = 1.1) -> "SamplerKind":
        k = SamplerKind(STRATIFIED, nonzero_samples=int(p), zero_samples=int(q), oversample=rho)
        k.validate()
        return k

    @staticmethod
    def semi_stratified(p: int, q: int) -> "SamplerKind":
        k = SamplerKind(SEMI_STRATIFIED, nonzero_samples=int(p), zero_samples=int(q))
        k.validate()
        return k

    @staticmethod
    def from_token(token: str, total_samples: int) -> "SamplerKind":  # samplers.cpp:37-45
        if token == "uniform":
            return SamplerKind.uniform(total_samples)
        if token == "stratified":
            return SamplerKind.stratified(total_samples // 2, total_samples - total_samples // 2)
        if token == "semi-stratified":
            return SamplerKind.semi_stratified(total_samples // 2,
                                               total_samples - total_samples // 2)
        raise InvalidArgument(f"unknown sampler '{token}' (expected uniform, stratified, or "
                              "semi-stratified)")

    def token(self) -> str:
        return {UNIFORM: "uniform", STRATIFIED: "stratified",
                SEMI_STRATIFIED: "semi-stratified"}[self.strategy]

    def validate(self) -> None:  # samplers.cpp:56-67
        if self.strategy == UNIFORM:
            if self.num_samples < 1:
                raise InvalidArgument("uniform sampler: s must be >= 1")
            return
        if self.nonzero_samples < 0 or self.zero_samples < 0 or \
                self.nonzero_samples + self.zero_samples < 1:
            raise InvalidArgument("sampler: need p, q >= 0 and p + q >= 1")
        if self.strategy == STRATIFIED and not self.oversample > 1.0:
            raise InvalidArgument("stratified sampler: oversample rate must be > 1")

    def total(self) -> int:
        return self.num_samples if self.strategy == UNIFORM else \
            self.nonzero_samples + self.zero_samples

    def c(self) -> _capi.gcpb_sampler:
        return _capi.gcpb_sampler(self.strategy, self.num_samples, self.nonzero_samples,
                                  self.zero_samples, self.oversample)


@dataclass
class RejectionStats:
    tested: int = 0
    accepted: int = 0
    rejected: int = 0


# ---------------------------------------------------------------------------
# The device engine (one GCP problem on one GPU)
# ---------------------------------------------------------------------------
class RngStream:
    """The reference's splittable counter stream (rng.hpp:15-47) as a state
    the device generators consume and advance."""

    def __init__(self, seed: int = 0):
        self._s = _capi.gcpb_rng()
        _check(lib.gcpb_rng_seed(seed, C.byref(self._s)))

    def split(self, label: int) -> "RngStream":
        child = RngStream.__new__(RngStream)
        child._s = _capi.gcpb_rng()
        _check(lib.gcpb_rng_split(C.byref(self._s), label, C.byref(child._s)))
        return child

    @property
    def key(self) -> int:
        return int(self._s.key)

    @property
    def counter(self) -> int:
        return int(self._s.counter)


@dataclass
class BinaryProblemSpec:
    """BinaryProblemSpec (synthetic.hpp:22-31); shape and rank come from the Engine."""
    delta: float = 0.15
    p_high: float = 0.9
    p_low: float = 0.0025


class Engine:
    """Owns a gcpb context: factors, gradient, Adam moments, tensor, estimator.

    dims: tensor extents (n_1..n_d); rank: r; dtype "f32" (B200 fast path) or
    "f64" (the reference's arithmetic type).
    """

    def __init__(self, dims: Sequence[int], rank: int, dtype: str = "f32", device: int = 0):
        self.dims = tuple(int(n) for n in dims)
        self.d = len(self.dims)
        self.rank = int(rank)
        self.dtype = dtype
        dt = {"f32": _capi.F32, "f64": _capi.F64}.get(dtype)
        if dt is None:
            raise InvalidArgument("dtype must be 'f32' or 'f64'")
        arr = np.asarray(self.dims, dtype=np.int64)
        h = _capi.ctx_p()
        _check(lib.gcpb_create(device, dt, self.d, _i64(arr), self.rank, C.byref(h)))
        self._h = h
        self.total = math.prod(self.dims)

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.gcpb_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _ck(self, rc: int) -> None:
        _check(rc, self._h)

    @property
    def handle(self):
        return self._h

    # ---- tensor ------------------------------------------------------------
    def set_sparse(self, coords, values) -> None:
        coords = np.ascontiguousarray(coords, dtype=np.int64).reshape(-1, self.d)
        values = np.ascontiguousarray(values, dtype=np.float64)
        if len(values) != len(coords):
            raise InvalidArgument("sparse tensor: index/value count mismatch")
        self._ck(lib.gcpb_set_sparse(self._h, len(values), _i64(coords), _f64(values)))

    def set_sparse_device(self, keys_ptr: int, values_ptr: int, nnz: int, value_dtype: str) -> None:
        vd = _capi.F32 if value_dtype == "f32" else _capi.F64
        self._ck(lib.gcpb_set_sparse_device(self._h, int(nnz), C.c_void_p(keys_ptr),
                                            C.c_void_p(values_ptr), vd))

    @property
    def nnz(self) -> int:
        return int(lib.gcpb_nnz(self._h))

    def get_sparse(self):
        n = self.nnz
        coords = np.zeros((n, self.d), dtype=np.int64)
        vals = np.zeros(n, dtype=np.float64)
        self._ck(lib.gcpb_get_sparse(self._h, _i64(coords), _f64(vals)))
        return coords, vals

    def set_dense(self, values, storage: str = "f64") -> None:
        st = {"u8": _capi.STORE_U8, "f32": _capi.STORE_F32, "f64": _capi.STORE_F64,
              "bit": _capi.STORE_BIT}[storage]
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        if v.size != self.total:
            raise InvalidArgument("dense tensor: value count mismatch")
        self._ck(lib.gcpb_set_dense(self._h, _f64(v), st))

    def generate_dense_bernoulli(self, true_factors: Sequence[np.ndarray], seed: int,
                                 storage: str = "bit") -> None:
        R = true_factors[0].shape[1]
        flat = np.ascontiguousarray(np.concatenate([np.asarray(f, np.float64).reshape(-1)
                                                    for f in true_factors]))
        st = {"u8": _capi.STORE_U8, "bit": _capi.STORE_BIT}[storage]
        self._ck(lib.gcpb_generate_dense_bernoulli(self._h, R, _f64(flat), seed, st))

    def tensor_norm(self) -> float:
        out = C.c_double()
        self._ck(lib.gcpb_tensor_norm(self._h, C.byref(out)))
        return out.value

    def value_at(self, idx) -> np.ndarray:
        idx = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1, self.d)
        out = np.zeros(len(idx), dtype=np.float64)
        self._ck(lib.gcpb_value_at(self._h, len(idx), _i64(idx), _f64(out)))
        return out

    # ---- factors / gradient / moments --------------------------------------
    def _mode_sizes(self):
        return [n * self.rank for n in self.dims]

    def _split(self, flat):
        out, at = [], 0
        for n in self.dims:
            out.append(flat[at:at + n * self.rank].reshape(n, self.rank))
            at += n * self.rank
        return out

    def _flat(self, mats):
        if len(mats) != self.d:
            raise InvalidArgument("expected one matrix per mode")
        for k, m in enumerate(mats):
            if np.shape(m) != (self.dims[k], self.rank):
                raise InvalidArgument(f"mode {k}: expected shape {(self.dims[k], self.rank)}")
        return np.ascontiguousarray(np.concatenate([np.asarray(m, np.float64).reshape(-1)
                                                    for m in mats]))

    def set_factors(self, mats) -> None:
        self._ck(lib.gcpb_set_factors(self._h, -1, _f64(self._flat(mats))))

    def set_factor(self, mode: int, mat) -> None:
        """One mode's factor matrix (n_k x r, row-major)."""
        m = np.ascontiguousarray(np.asarray(mat, np.float64).reshape(-1))
        if m.size != self.dims[mode] * self.rank:
            raise InvalidArgument(f"mode {mode}: expected shape {(self.dims[mode], self.rank)}")
        self._ck(lib.gcpb_set_factors(self._h, mode, _f64(m)))

    def factor(self, mode: int) -> np.ndarray:
        out = np.zeros((self.dims[mode], self.rank))
        self._ck(lib.gcpb_get_factors(self._h, mode, _f64(out)))
        return out

    def grad_mode(self, mode: int) -> np.ndarray:
        out = np.zeros((self.dims[mode], self.rank))
        self._ck(lib.gcpb_get_grad(self._h, mode, _f64(out)))
        return out

    def factors(self):
        flat = np.zeros(sum(self._mode_sizes()), dtype=np.float64)
        self._ck(lib.gcpb_get_factors(self._h, -1, _f64(flat)))
        return self._split(flat)

    def grad(self):
        flat = np.zeros(sum(self._mode_sizes()), dtype=np.float64)
        self._ck(lib.gcpb_get_grad(self._h, -1, _f64(flat)))
        return self._split(flat)

    def grad_flat(self) -> np.ndarray:
        flat = np.zeros(sum(self._mode_sizes()), dtype=np.float64)
        self._ck(lib.gcpb_get_grad(self._h, -1, _f64(flat)))
        return flat

    def set_grad(self, mats) -> None:
        self._ck(lib.gcpb_set_grad(self._h, -1, _f64(self._flat(mats))))

    def moment(self, which: int):
        flat = np.zeros(sum(self._mode_sizes()), dtype=np.float64)
        self._ck(lib.gcpb_get_moment(self._h, which, -1, _f64(flat)))
        return self._split(flat)

    def set_moment(self, which: int, mats) -> None:
        self._ck(lib.gcpb_set_moment(self._h, which, -1, _f64(self._flat(mats))))

    # ---- hot path ------------------------------------------------------------
    def stoch_grad(self, sampler: SamplerKind, loss: LossFunction, seed: int, it: int,
                   want_stats: bool = True) -> Optional[RejectionStats]:
        sk, ls = sampler.c(), loss.c()
        st = _capi.gcpb_stats()
        self._ck(lib.gcpb_stoch_grad(self._h, C.byref(sk), C.byref(ls), seed, it,
                                     C.byref(st) if want_stats else None))
        return RejectionStats(st.tested, st.accepted, st.rejected) if want_stats else None

    def draw_samples(self, sampler: SamplerKind, loss: LossFunction, seed: int, it: int):
        n = sampler.total()
        idx = np.zeros((max(n, 1), self.d), dtype=np.int64)
        x, w, m, y = (np.zeros(max(n, 1)) for _ in range(4))
        flag = np.zeros(max(n, 1), dtype=np.int32)
        nout = C.c_int64()
        st = _capi.gcpb_stats()
        sk, ls = sampler.c(), loss.c()
        self._ck(lib.gcpb_draw_samples(self._h, C.byref(sk), C.byref(ls), seed, it, n, _i64(idx),
                                       _f64(x), _f64(w), _i32(flag), _f64(m), _f64(y),
                                       C.byref(nout), C.byref(st)))
        k = nout.value
        return dict(idx=idx[:k], x=x[:k], w=w[:k], flag=flag[:k], m=m[:k], y=y[:k],
                    stats=RejectionStats(st.tested, st.accepted, st.rejected))

    def eval_deriv(self, idx, x, w, loss: LossFunction, flags=None):
        idx = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1, self.d)
        n = len(idx)
        x = np.ascontiguousarray(x, dtype=np.float64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        fl = None if flags is None else np.ascontiguousarray(flags, dtype=np.int32)
        m = np.zeros(n)
        y = np.zeros(n)
        ls = loss.c()
        self._ck(lib.gcpb_eval_deriv(self._h, n, _i64(idx), _f64(x), _f64(w),
                                     _i32(fl) if fl is not None else None, C.byref(ls),
                                     _f64(m), _f64(y)))
        return m, y

    def mttkrp_samples(self, idx, y) -> None:
        idx = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1, self.d)
        y = np.ascontiguousarray(y, dtype=np.float64)
        self._ck(lib.gcpb_mttkrp_samples(self._h, len(idx), _i64(idx), _f64(y)))

    # ---- optimizer -------------------------------------------------------------
    def adam_step(self, learning_rate: float, beta1=0.9, beta2=0.999, epsilon=1e-8,
                  lower_bound: Optional[float] = None) -> None:
        a = _capi.gcpb_adam(learning_rate, beta1, beta2, epsilon,
                            0 if lower_bound is None else 1,
                            0.0 if lower_bound is None else float(lower_bound))
        self._ck(lib.gcpb_adam_step(self._h, C.byref(a)))

    @staticmethod
    def _adam(learning_rate, beta1=0.9, beta2=0.999, epsilon=1e-8, lower_bound=None):
        return _capi.gcpb_adam(learning_rate, beta1, beta2, epsilon,
                               0 if lower_bound is None else 1,
                               0.0 if lower_bound is None else float(lower_bound))

    def step(self, sampler: SamplerKind, loss: LossFunction, seed: int, it: int,
             learning_rate: float, beta1=0.9, beta2=0.999, epsilon=1e-8,
             lower_bound: Optional[float] = None) -> None:
        """One epoch-loop iteration (optimizer.cpp:116-119) on the device."""
        sk, ls = sampler.c(), loss.c()
        a = self._adam(learning_rate, beta1, beta2, epsilon, lower_bound)
        self._ck(lib.gcpb_step(self._h, C.byref(sk), C.byref(ls), seed, it, C.byref(a)))

    def step_host(self, sampler: SamplerKind, loss: LossFunction, seed: int, it: int,
                  learning_rate: float, model_in: Optional[np.ndarray], model_out: Optional[np.ndarray],
                  beta1=0.9, beta2=0.999, epsilon=1e-8, lower_bound: Optional[float] = None) -> None:
        """One iteration on a host-resident model (flattened factors in/out)."""
        sk, ls = sampler.c(), loss.c()
        a = self._adam(learning_rate, beta1, beta2, epsilon, lower_bound)
        self._ck(lib.gcpb_step_host(self._h, C.byref(sk), C.byref(ls), seed, it, C.byref(a),
                                    _f64(model_in) if model_in is not None else None,
                                    _f64(model_out) if model_out is not None else None))

    def run_steps(self, sampler: SamplerKind, loss: LossFunction, seed: int, it0: int, n: int,
                  learning_rate: float, beta1=0.9, beta2=0.999, epsilon=1e-8,
                  lower_bound: Optional[float] = None) -> None:
        """n iterations it0..it0+n-1 replayed as one CUDA graph (asynchronous)."""
        sk, ls = sampler.c(), loss.c()
        a = self._adam(learning_rate, beta1, beta2, epsilon, lower_bound)
        self._ck(lib.gcpb_run_steps(self._h, C.byref(sk), C.byref(ls), seed, it0, n, C.byref(a)))

    @property
    def steps_path(self) -> str:
        """Engine of the last run_steps: "graph" or "small" (cluster kernel)."""
        return {0: "graph", 1: "small"}.get(int(lib.gcpb_steps_path(self._h)), "unknown")

    def run_steps_launches(self) -> int:
        """Kernels the last run_steps launched (step-graph kernel nodes)."""
        n = C.c_int64()
        self._ck(lib.gcpb_run_steps_launches(self._h, C.byref(n)))
        return int(n.value)

    def last_transfer_bytes(self) -> tuple:
        """(h2d, d2h) model bytes the last step_host moved over the bus (fp32
        engines narrow large page-locked fp64 models on the host)."""
        a, b = C.c_int64(), C.c_int64()
        self._ck(lib.gcpb_last_transfer_bytes(self._h, C.byref(a), C.byref(b)))
        return int(a.value), int(b.value)

    @property
    def hot_rows(self) -> tuple:
        """(hot rows selected, copies per hot row used by the last scatter)."""
        rows, copies = C.c_int(), C.c_int()
        self._ck(lib.gcpb_hot_rows(self._h, C.byref(rows), C.byref(copies)))
        return rows.value, copies.value

    @property
    def interleaved(self) -> tuple:
        """(interleaved factor/gradient table enabled, last scatter used it)."""
        en, last = C.c_int(), C.c_int()
        self._ck(lib.gcpb_interleaved(self._h, C.byref(en), C.byref(last)))
        return bool(en.value), bool(last.value)

    def adam_reset(self) -> None:
        self._ck(lib.gcpb_adam_reset(self._h))

    @property
    def iterations(self) -> int:
        self.synchronize()
        v = C.c_int64()
        self._ck(lib.gcpb_get_iterations(self._h, C.byref(v)))
        return v.value

    @iterations.setter
    def iterations(self, t: int) -> None:
        self._ck(lib.gcpb_set_iterations(self._h, int(t)))

    # ---- estimator ---------------------------------------------------------------
    def estimator_set(self, idx, x, w) -> None:
        idx = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1, self.d)
        x = np.ascontiguousarray(x, dtype=np.float64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        self._ck(lib.gcpb_estimator_set(self._h, len(idx), _i64(idx), _f64(x), _f64(w)))

    def estimator_draw(self, kind: int, count: int, seed: int, rho: float = 1.1) -> None:
        self._ck(lib.gcpb_estimator_draw(self._h, kind, count, rho, seed))

    def estimator_get(self):
        n = int(lib.gcpb_estimator_size(self._h))
        idx = np.zeros((max(n, 1), self.d), dtype=np.int64)
        x = np.zeros(max(n, 1))
        w = np.zeros(max(n, 1))
        self._ck(lib.gcpb_estimator_get(self._h, _i64(idx), _f64(x), _f64(w)))
        return idx[:n], x[:n], w[:n]

    def estimate(self, loss: LossFunction) -> float:
        out = C.c_double()
        ls = loss.c()
        self._ck(lib.gcpb_estimate(self._h, C.byref(ls), C.byref(out)))
        return out.value

    # ---- snapshots / multi-GPU -------------------------------------------------------
    def gradient_full(self, loss: LossFunction) -> None:
        """Exact gradient over every entry (kernels.cpp:170-198) -> grad()."""
        ls = loss.c()
        self._ck(lib.gcpb_gradient_full(self._h, C.byref(ls)))

    def gradient_poisson_implicit(self, loss: LossFunction) -> None:
        """Exact Poisson gradient touching only nonzeros (kernels.cpp:200-235)."""
        ls = loss.c()
        self._ck(lib.gcpb_gradient_poisson_implicit(self._h, C.byref(ls)))

    def gradient_moments(self, sampler: SamplerKind, loss: LossFunction, trials: int,
                         seed: int) -> tuple[np.ndarray, np.ndarray]:
        """Per-coordinate mean and sample variance of `trials` stochastic gradients."""
        sk, ls = sampler.c(), loss.c()
        n = sum(self._mode_sizes())
        mean, var = np.zeros(n), np.zeros(n)
        self._ck(lib.gcpb_gradient_moments(self._h, C.byref(sk), C.byref(ls), trials, seed,
                                           _f64(mean), _f64(var)))
        return mean, var

    def bias_variance(self, sampler: SamplerKind, loss: LossFunction, trials: int, seed: int,
                      exact: Optional[np.ndarray] = None) -> tuple[float, float]:
        """empirical_bias_variance (samplers.cpp:134-168) on the device."""
        sk, ls = sampler.c(), loss.c()
        b, v = C.c_double(), C.c_double()
        ex = None if exact is None else np.ascontiguousarray(exact, dtype=np.float64)
        self._ck(lib.gcpb_bias_variance(self._h, C.byref(sk), C.byref(ls), trials, seed,
                                        _f64(ex) if ex is not None else None, C.byref(b),
                                        C.byref(v)))
        return b.value, v.value

    # ---- synthetic problems (synthetic.cpp) --------------------------------
    def gen_gamma_problem(self, rng: "RngStream", storage: str = "f64") -> list:
        """gen_gamma_problem (synthetic.cpp:26-41) on the device: dense
        exponential data around a random-uniform truth; returns the truth
        factors (fp64) and advances ``rng`` like the reference."""
        st = {"f32": _capi.STORE_F32, "f64": _capi.STORE_F64}[storage]
        truth = np.zeros(sum(self._mode_sizes()))
        self._ck(lib.gcpb_gen_gamma_problem(self._h, C.byref(rng._s), st, _f64(truth)))
        return self._split_modes(truth)

    def gen_binary_problem(self, spec: "BinaryProblemSpec", rng: "RngStream") -> list:
        """gen_binary_problem (synthetic.cpp:58-146) on the device: sparse
        binary tensor + truth factors; advances ``rng`` like the reference."""
        sp = _capi.gcpb_binary_spec(spec.delta, spec.p_high, spec.p_low)
        truth = np.zeros(sum(self._mode_sizes()))
        self._ck(lib.gcpb_gen_binary_problem(self._h, C.byref(sp), C.byref(rng._s), _f64(truth)))
        return self._split_modes(truth)

    def _split_modes(self, flat: np.ndarray) -> list:
        out, at = [], 0
        for n in self.dims:
            out.append(flat[at:at + n * self.rank].reshape(n, self.rank).copy())
            at += n * self.rank
        return out

    def set_draw_stream(self, kind: str = "philox", counter: int = 0) -> None:
        """'philox' (default) or 'reference' (RefStream: the reference's
        RngStream sequence; stoch_grad's seed is then the stream key)."""
        k = {"philox": 0, "reference": 1}[kind]
        self._ck(lib.gcpb_set_draw_stream(self._h, k, counter))

    @property
    def draw_counter(self) -> int:
        v = C.c_uint64()
        self._ck(lib.gcpb_get_draw_counter(self._h, C.byref(v)))
        return v.value

    def kernel_timing(self, enable: bool) -> None:
        self._ck(lib.gcpb_kernel_timing(self._h, 1 if enable else 0))

    def kernel_time(self) -> tuple[float, int]:
        """(summed ms, launches) of the fused kernel since kernel_timing(True)."""
        t, n = C.c_double(), C.c_int64()
        self._ck(lib.gcpb_kernel_time(self._h, C.byref(t), C.byref(n)))
        return t.value, n.value

    def synchronize(self) -> None:
        self._ck(lib.gcpb_synchronize(self._h))

    def snapshot_save(self) -> None:
        self._ck(lib.gcpb_snapshot_save(self._h))

    def snapshot_restore(self) -> None:
        self._ck(lib.gcpb_snapshot_restore(self._h))

    def set_stream(self, stream_ptr: Optional[int]) -> None:
        self._ck(lib.gcpb_set_stream(self._h, C.c_void_p(stream_ptr) if stream_ptr else None))

    def set_shard(self, rank: int, nranks: int) -> None:
        self._ck(lib.gcpb_set_shard(self._h, rank, nranks))

    def peer_handle(self) -> bytes:
        """This rank's table, exportable to the other ranks (gcpb_peer_handle)."""
        buf = C.create_string_buffer(_capi.PEER_HANDLE_BYTES)
        self._ck(lib.gcpb_peer_handle(self._h, buf))
        return buf.raw

    def peer_open(self, handles: Sequence[bytes]) -> None:
        """Map every rank's table (rank order) for the fused reduce-scatter +
        Adam + all-gather kernel (gcpb_peer_open)."""
        blob = b"".join(bytes(h) for h in handles)
        self._ck(lib.gcpb_peer_open(self._h, blob, len(handles)))

    def peer_close(self) -> None:
        """Back to the NCCL all-reduce + replicated Adam exchange (gcpb_peer_close)."""
        self._ck(lib.gcpb_peer_close(self._h))

    def comm_init(self, unique_id: bytes, rank: int, nranks: int) -> None:
        self._ck(lib.gcpb_comm_init(self._h, unique_id, rank, nranks))

    def allreduce_grad(self) -> None:
        self._ck(lib.gcpb_allreduce_grad(self._h))

    def comm_init_host(self, rank: int, nranks: int,
                       allgather: Callable[[int], Sequence[int]],
                       allreduce: Callable[[np.ndarray], None]) -> None:
        """Host-callback communicator: allgather(value) -> list of nranks ints;
        allreduce(array) sums the float64 array across ranks in place."""
        def _ag(user, send, recv):
            try:
                vals = allgather(int(send))
                for i, v in enumerate(vals):
                    recv[i] = int(v)
                return 0
            except Exception:  # surfaced as GCPB_ERR_RUNTIME
                return 1

        def _ar(user, buf, n):
            try:
                arr = np.ctypeslib.as_array(buf, shape=(n,))
                allreduce(arr)
                return 0
            except Exception:
                return 1

        self._comm_cbs = (_capi.ALLGATHER_FN(_ag), _capi.ALLREDUCE_FN(_ar))
        self._ck(lib.gcpb_comm_init_host(self._h, rank, nranks, self._comm_cbs[0],
                                         self._comm_cbs[1], None))


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib.gcpb_nccl_unique_id(buf))
    return buf.raw


# ---------------------------------------------------------------------------
# Host-only helpers
# ---------------------------------------------------------------------------
def philox_bounded(seed: int, tag: int, it: int, t: int, slot: int, n: int) -> int:
    return int(lib.gcpb_philox_bounded(seed, tag, it, t, slot, n))


def zero_batch_size(total: float, zeta: float, rho: float, shortfall: int) -> int:
    return int(lib.gcpb_zero_batch_size(total, zeta, rho, shortfall))


def shard_range(n: int, rank: int, nranks: int) -> tuple[int, int]:
    b, e = C.c_int64(), C.c_int64()
    lib.gcpb_shard_range(n, rank, nranks, C.byref(b), C.byref(e))
    return b.value, e.value


def stratified_keep(accepted_per_rank: Sequence[int], rank: int, need: int) -> tuple[int, int]:
    arr = np.ascontiguousarray(accepted_per_rank, dtype=np.int64)
    off, keep = C.c_int64(), C.c_int64()
    lib.gcpb_stratified_keep(_i64(arr), len(arr), rank, need, C.byref(off), C.byref(keep))
    return off.value, keep.value


TAG_GRAD_UNIFORM, TAG_GRAD_NZ_PICK, TAG_GRAD_ZERO_CAND, TAG_GRAD_SEMI_Q = 1, 2, 3, 4
TAG_EST_UNIFORM, TAG_EST_NZ_PICK, TAG_EST_ZERO_CAND = 5, 6, 7
