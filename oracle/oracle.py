"""ctypes access to the oracles — TEST INFRASTRUCTURE ONLY.

* ``Oracle``  : oracle/liboracle.so, the C restatement (gcp_oracle.c) incl. the
                host replica of the product's Philox stream.
* ``Reference``: oracle/_ref/libgcpref.so, the UNMODIFIED reference library
                (/root/reference/proj/src/*.cpp) compiled here, via ref_capi.cpp.
                Absent on the GPU box unless the prebuilt .so travelled with
                the snapshot; callers must skip when ``reference()`` is None.

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
legs may import this module.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path
from typing import Optional

import numpy as np

HERE = Path(__file__).resolve().parent
LIBORACLE = HERE / "liboracle.so"
LIBREF = HERE / "_ref" / "libgcpref.so"

i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
i32p = C.POINTER(C.c_int32)
u64p = C.POINTER(C.c_uint64)


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _i64(a):
    return _p(a, i64p)


def _f64(a):
    return _p(a, f64p)


def _u64(a):
    return _p(a, u64p)


# ---------------------------------------------------------------------------
# C restatement
# ---------------------------------------------------------------------------
class or_rng(C.Structure):
    _fields_ = [("key", C.c_uint64), ("counter", C.c_uint64)]


class or_src(C.Structure):
    _fields_ = [("mode", C.c_int), ("script", u64p), ("len", C.c_int64), ("at", C.c_int64),
                ("seed", C.c_uint64), ("iter", C.c_uint64), ("tag_uniform", C.c_uint32),
                ("tag_pick", C.c_uint32), ("tag_zero", C.c_uint32), ("strategy", C.c_int),
                ("p", C.c_int64), ("d", C.c_int), ("rng", or_rng), ("exhausted", C.c_int)]


class or_tensor(C.Structure):
    _fields_ = [("d", C.c_int), ("dims", i64p), ("is_sparse", C.c_int), ("nnz", C.c_int64),
                ("coords", i64p), ("values", f64p), ("keys", u64p), ("dense", f64p)]


class or_sampler(C.Structure):
    _fields_ = [("strategy", C.c_int), ("s", C.c_int64), ("p", C.c_int64), ("q", C.c_int64),
                ("rho", C.c_double)]


class Tensor:
    """Normalised tensor for the oracle (keeps numpy buffers alive)."""

    def __init__(self, dims, coords=None, values=None, dense=None):
        self.dims = np.ascontiguousarray(dims, dtype=np.int64)
        self.d = len(self.dims)
        self.is_sparse = dense is None
        if self.is_sparse:
            o = oracle()
            coords = np.ascontiguousarray(coords, dtype=np.int64).reshape(-1, self.d)
            values = np.ascontiguousarray(values, dtype=np.float64)
            n = len(values)
            self.coords = np.zeros((max(n, 1), self.d), dtype=np.int64)
            self.values = np.zeros(max(n, 1))
            self.keys = np.zeros(max(n, 1), dtype=np.uint64)
            nnz = o.lib.or_sparse_normalize(self.d, _i64(self.dims), n, _i64(coords),
                                            _f64(values), _i64(self.coords), _f64(self.values),
                                            _u64(self.keys))
            if nnz == -4:
                raise IndexError("index out of range")
            if nnz < 0:
                raise ValueError("unsupported shape")
            self.nnz = int(nnz)
            self.coords = self.coords[:self.nnz].copy()
            self.values = self.values[:self.nnz].copy()
            self.keys = self.keys[:self.nnz].copy()
            self.dense = None
        else:
            self.dense = np.ascontiguousarray(dense, dtype=np.float64).reshape(-1)
            self.nnz = 0
            self.coords = self.values = self.keys = None

    def c(self) -> or_tensor:
        t = or_tensor()
        t.d = self.d
        t.dims = _i64(self.dims)
        t.is_sparse = 1 if self.is_sparse else 0
        t.nnz = self.nnz
        if self.is_sparse:
            t.coords = _i64(self.coords if self.nnz else np.zeros((1, self.d), np.int64))
            t.values = _f64(self.values if self.nnz else np.zeros(1))
            t.keys = _u64(self.keys if self.nnz else np.zeros(1, np.uint64))
        else:
            t.dense = _f64(self.dense)
        self._keep = t
        return t

    @property
    def total(self) -> int:
        return int(np.prod(self.dims.astype(object)))


class Oracle:
    def __init__(self, path: Path = LIBORACLE):
        if not path.exists():
            raise ImportError(f"{path} missing: run `make -C oracle liboracle`")
        L = self.lib = C.CDLL(str(path))
        L.or_mix64.restype = C.c_uint64
        L.or_mix64.argtypes = [C.c_uint64]
        L.or_rng_init.argtypes = [C.POINTER(or_rng), C.c_uint64]
        L.or_rng_split_label.argtypes = [C.POINTER(or_rng), C.c_char_p, C.POINTER(or_rng)]
        L.or_rng_split_u64.argtypes = [C.POINTER(or_rng), C.c_uint64, C.POINTER(or_rng)]
        L.or_rng_next_u64.restype = C.c_uint64
        L.or_rng_next_u64.argtypes = [C.POINTER(or_rng)]
        L.or_rng_next_double.restype = C.c_double
        L.or_rng_next_double.argtypes = [C.POINTER(or_rng)]
        L.or_rng_next_below.restype = C.c_uint64
        L.or_rng_next_below.argtypes = [C.POINTER(or_rng), C.c_uint64]
        L.or_draw_bounded.restype = C.c_uint64
        L.or_draw_bounded.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_int,
                                      C.c_uint64]
        L.or_loss_value.restype = C.c_double
        L.or_loss_value.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double]
        L.or_loss_deriv.restype = C.c_double
        L.or_loss_deriv.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double]
        L.or_entry.restype = C.c_double
        L.or_entry.argtypes = [C.c_int, i64p, C.c_int64, f64p, i64p]
        L.or_mttkrp_sampled_all.argtypes = [C.c_int, i64p, C.c_int64, f64p, C.c_int64, i64p, f64p,
                                            f64p]
        L.or_adam_step.argtypes = [C.c_int, i64p, C.c_int64, f64p, f64p, f64p, i64p, C.c_double,
                                   f64p, C.c_double, C.c_double, C.c_double, C.c_int, C.c_double]
        L.or_sparse_normalize.restype = C.c_int64
        L.or_sparse_normalize.argtypes = [C.c_int, i64p, C.c_int64, i64p, f64p, i64p, f64p, u64p]
        L.or_draw_gradient_samples.restype = C.c_int
        L.or_draw_gradient_samples.argtypes = [C.POINTER(or_tensor), C.c_int64, f64p, C.c_int,
                                               C.c_double, C.POINTER(or_sampler),
                                               C.POINTER(or_src), C.c_int64, i64p, f64p, f64p,
                                               i32p, f64p, i64p, i64p]
        L.or_estimator_draw.restype = C.c_int
        L.or_estimator_draw.argtypes = [C.POINTER(or_tensor), C.c_int, C.c_int64, C.c_double,
                                        C.POINTER(or_src), C.c_int64, i64p, f64p, f64p, i64p]
        L.or_estimate.restype = C.c_double
        L.or_estimate.argtypes = [C.c_int, i64p, C.c_int64, f64p, C.c_int, C.c_double, C.c_int64,
                                  i64p, f64p, f64p]
        L.or_zero_batch_size.restype = C.c_int64
        L.or_zero_batch_size.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int64]

    # -- rng
    def rng_stream(self, seed: int):
        r = or_rng()
        self.lib.or_rng_init(C.byref(r), seed)
        return r

    def split(self, r: or_rng, label) -> or_rng:
        out = or_rng()
        if isinstance(label, str):
            self.lib.or_rng_split_label(C.byref(r), label.encode(), C.byref(out))
        else:
            self.lib.or_rng_split_u64(C.byref(r), label, C.byref(out))
        return out

    def draw_bounded(self, seed, tag, it, t, k, n) -> int:
        return int(self.lib.or_draw_bounded(seed, tag, it, t, k, n))

    # -- model / kernels
    @staticmethod
    def flat(factors) -> np.ndarray:
        return np.ascontiguousarray(np.concatenate([np.asarray(f, np.float64).reshape(-1)
                                                    for f in factors]))

    def mttkrp(self, dims, r, factors, idx, y) -> np.ndarray:
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        idx = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1, len(dims))
        y = np.ascontiguousarray(y, dtype=np.float64)
        out = np.zeros(int(np.sum(dims)) * r)
        self.lib.or_mttkrp_sampled_all(len(dims), _i64(dims), r, _f64(self.flat(factors)),
                                       len(idx), _i64(idx), _f64(y), _f64(out))
        return out

    def entries(self, dims, r, factors, idx) -> np.ndarray:
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        idx = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1, len(dims))
        F = self.flat(factors)
        return np.array([self.lib.or_entry(len(dims), _i64(dims), r, _f64(F), _i64(idx[e:e + 1]))
                         for e in range(len(idx))])

    def adam(self, dims, r, factors, first, second, iterations, lr, grads, beta1=0.9,
             beta2=0.999, eps=1e-8, lb=None):
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        A = self.flat(factors).copy()
        B = np.ascontiguousarray(first, dtype=np.float64).copy()
        Cm = np.ascontiguousarray(second, dtype=np.float64).copy()
        it = C.c_int64(iterations)
        g = np.ascontiguousarray(grads, dtype=np.float64)
        self.lib.or_adam_step(len(dims), _i64(dims), r, _f64(A), _f64(B), _f64(Cm), C.byref(it),
                              lr, _f64(g), beta1, beta2, eps, 0 if lb is None else 1,
                              0.0 if lb is None else lb)
        return A, B, Cm, it.value

    def estimate(self, dims, r, factors, loss_kind, delta, idx, x, w) -> float:
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        idx = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1, len(dims))
        return float(self.lib.or_estimate(len(dims), _i64(dims), r, _f64(self.flat(factors)),
                                          loss_kind, delta, len(idx), _i64(idx),
                                          _f64(np.ascontiguousarray(x, np.float64)),
                                          _f64(np.ascontiguousarray(w, np.float64))))

    # -- samplers
    def source(self, mode, script=None, seed=0, it=0, estimator=False, rng_seed=None):
        s = or_src()
        s.mode = mode
        if script is not None:
            arr = np.ascontiguousarray(script, dtype=np.uint64)
            s.script = _u64(arr)
            s.len = len(arr)
            s._arr = arr
        s.seed = seed
        s.iter = it
        if estimator:
            s.tag_uniform, s.tag_pick, s.tag_zero = 5, 6, 7
        else:
            s.tag_uniform, s.tag_pick, s.tag_zero = 1, 2, 3
        if mode == 2:
            self.lib.or_rng_init(C.byref(s.rng), rng_seed if rng_seed is not None else seed)
        return s

    def draw_gradient_samples(self, tensor: Tensor, r, factors, loss_kind, delta, strategy, s=0,
                              p=0, q=0, rho=1.1, src: Optional[or_src] = None, cap=None):
        cap = cap or max(1, (s if strategy == 0 else p + q))
        d = tensor.d
        idx = np.zeros((cap, d), dtype=np.int64)
        x, w, y = np.zeros(cap), np.zeros(cap), np.zeros(cap)
        flag = np.zeros(cap, dtype=np.int32)
        n = C.c_int64()
        stats = np.zeros(3, dtype=np.int64)
        ks = or_sampler(strategy, s, p, q, rho)
        tc = tensor.c()
        # The semi-stratified unrestricted draws use their own Philox tag.
        if strategy == 2 and src.mode == 1:
            src.tag_zero = 4 if src.tag_uniform == 1 else src.tag_zero
        rc = self.lib.or_draw_gradient_samples(C.byref(tc), r, _f64(self.flat(factors)), loss_kind,
                                               delta, C.byref(ks), C.byref(src), cap, _i64(idx),
                                               _f64(x), _f64(w), flag.ctypes.data_as(i32p),
                                               _f64(y), C.byref(n), _i64(stats))
        k = n.value
        return rc, dict(idx=idx[:k], x=x[:k], w=w[:k], flag=flag[:k], y=y[:k],
                        stats=tuple(int(v) for v in stats), consumed=src.at)

    def estimator_draw(self, tensor: Tensor, kind, count, rho, src):
        cap = max(count, 1)
        idx = np.zeros((cap, tensor.d), dtype=np.int64)
        x, w = np.zeros(cap), np.zeros(cap)
        n = C.c_int64()
        tc = tensor.c()
        rc = self.lib.or_estimator_draw(C.byref(tc), kind, count, rho, C.byref(src), cap,
                                        _i64(idx), _f64(x), _f64(w), C.byref(n))
        k = n.value
        return rc, idx[:k], x[:k], w[:k]


# ---------------------------------------------------------------------------
# The reference itself
# ---------------------------------------------------------------------------
class RefError(Exception):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Reference:
    def __init__(self, path: Path = LIBREF):
        L = self.lib = C.CDLL(str(path))
        L.ref_last_error.restype = C.c_char_p
        vp = C.c_void_p
        L.ref_rng_new.restype = vp
        L.ref_rng_new.argtypes = [C.c_uint64]
        L.ref_rng_free.argtypes = [vp]
        L.ref_rng_split_label.restype = vp
        L.ref_rng_split_label.argtypes = [vp, C.c_char_p]
        L.ref_rng_split_u64.restype = vp
        L.ref_rng_split_u64.argtypes = [vp, C.c_uint64]
        L.ref_rng_next_u64.restype = C.c_uint64
        L.ref_rng_next_u64.argtypes = [vp]
        L.ref_rng_next_double.restype = C.c_double
        L.ref_rng_next_double.argtypes = [vp]
        L.ref_rng_next_below.argtypes = [vp, C.c_uint64, u64p]
        L.ref_loss_value.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, f64p]
        L.ref_loss_deriv.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, f64p]
        L.ref_sparse_new.argtypes = [C.c_int, i64p, C.c_int64, i64p, f64p, C.POINTER(vp)]
        L.ref_dense_new.argtypes = [C.c_int, i64p, f64p, C.POINTER(vp)]
        L.ref_tensor_free.argtypes = [vp]
        L.ref_sparse_nnz.restype = C.c_int64
        L.ref_sparse_nnz.argtypes = [vp]
        L.ref_sparse_export.argtypes = [vp, i64p, f64p]
        L.ref_tensor_norm.restype = C.c_double
        L.ref_tensor_norm.argtypes = [vp]
        L.ref_model_entry.argtypes = [C.c_int, i64p, C.c_int64, f64p, C.c_int64, i64p, f64p]
        L.ref_draw_gradient_samples_scripted.argtypes = [
            vp, C.c_int, i64p, C.c_int64, f64p, C.c_int, C.c_double, C.c_int, C.c_int64,
            C.c_int64, C.c_int64, C.c_double, u64p, C.c_int64, C.c_int64, i64p, f64p, i64p, i64p,
            i64p]
        L.ref_draw_gradient_samples_seeded.argtypes = [
            vp, C.c_int, i64p, C.c_int64, f64p, C.c_int, C.c_double, C.c_int, C.c_int64,
            C.c_int64, C.c_int64, C.c_double, C.c_uint64, C.c_int64, i64p, f64p, i64p]
        L.ref_weighted_derivs.argtypes = [C.c_int, i64p, C.c_int64, f64p, C.c_int, C.c_double,
                                          C.c_int64, i64p, f64p, f64p, C.c_int, f64p]
        L.ref_mttkrp_sampled_all.argtypes = [C.c_int, i64p, C.c_int64, f64p, C.c_int64, i64p,
                                             f64p, C.c_int, f64p]
        L.ref_gradient_full.argtypes = [vp, C.c_int, i64p, C.c_int64, f64p, C.c_int, C.c_double,
                                        f64p]
        L.ref_gen_gamma.argtypes = [C.c_int, i64p, C.c_int64, C.c_uint64, C.POINTER(vp), f64p,
                                    u64p]
        L.ref_gen_binary.argtypes = [C.c_int, i64p, C.c_int64, C.c_double, C.c_double, C.c_double,
                                     C.c_uint64, C.POINTER(vp), f64p, u64p]
        L.ref_variance_ordering.argtypes = [f64p, f64p]
        L.ref_write_model.argtypes = [C.c_int, i64p, C.c_int64, f64p, C.c_char_p]
        L.ref_read_model.argtypes = [C.c_char_p, C.POINTER(C.c_int), i64p, i64p, f64p, C.c_int64]
        L.ref_write_trace.argtypes = [C.c_char_p, C.c_int64, i64p, f64p, f64p, f64p,
                                      C.POINTER(C.c_int)]
        L.ref_acceptance_instance.argtypes = [C.c_int, C.POINTER(vp), f64p]
        L.ref_similarity.argtypes = [C.c_int, i64p, C.c_int64, f64p, C.c_int64, f64p, f64p]
        L.ref_read_tns.argtypes = [C.c_char_p, C.POINTER(vp), C.POINTER(C.c_int), i64p]
        L.ref_write_tns.argtypes = [vp, C.c_char_p]
        L.ref_read_dense.argtypes = [C.c_char_p, C.POINTER(vp), C.POINTER(C.c_int), i64p]
        L.ref_write_dense.argtypes = [vp, C.c_char_p]
        L.ref_dense_export.argtypes = [vp, f64p]
        L.ref_gradient_poisson_implicit.argtypes = [vp, C.c_int, i64p, C.c_int64, f64p, f64p]
        L.ref_empirical_bias_variance.argtypes = [vp, C.c_int, i64p, C.c_int64, f64p, C.c_int,
                                                  C.c_double, C.c_int, C.c_int64, C.c_int64,
                                                  C.c_int64, C.c_double, C.c_int64, C.c_uint64,
                                                  f64p, f64p]
        L.ref_adam_step.argtypes = [C.c_int, i64p, C.c_int64, f64p, f64p, f64p, i64p, C.c_double,
                                    f64p, C.c_double, C.c_double, C.c_double, C.c_int, C.c_double]
        L.ref_estimator_scripted.argtypes = [vp, C.c_int, C.c_int64, C.c_double, u64p, C.c_int64,
                                             C.c_int, i64p, C.c_int64, f64p, C.c_int, C.c_double,
                                             C.c_int64, i64p, f64p, f64p, i64p, f64p]
        L.ref_estimate_given.argtypes = [C.c_int, i64p, C.c_int64, f64p, C.c_int, C.c_double,
                                         C.c_int64, i64p, f64p, f64p, f64p]
        L.ref_fit_gcp_adam.argtypes = [vp, C.c_int, C.c_double, C.c_int64, C.c_int, C.c_int64,
                                       C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_double,
                                       C.c_double, C.c_double, C.c_int64, C.c_int64, C.c_double,
                                       C.c_int, C.c_double, C.c_int64, C.c_int, C.c_int64,
                                       C.c_uint64, C.c_int, C.c_int64, f64p, i64p, f64p, f64p]
        L.ref_tensor_value_at.argtypes = [vp, i64p, C.POINTER(C.c_double)]
        L.ref_bench_model_new.argtypes = [C.c_int, i64p, C.c_int64, f64p, C.POINTER(vp)]
        L.ref_bench_model_free.argtypes = [vp]
        L.ref_bench_step_given.argtypes = [vp, C.c_int, C.c_double, C.c_int64, i64p, f64p,
                                           C.c_double, C.c_int, C.c_double, C.c_int, C.c_double,
                                           C.c_int, f64p]
        L.ref_bench_step_semi_given.argtypes = [vp, C.c_int, C.c_double, C.c_int64, i64p, f64p,
                                                C.c_int64, i64p, C.c_int64, C.c_double, C.c_int,
                                                C.c_double, C.c_int, C.c_double, C.c_int, f64p]
        L.ref_bench_step_sampler.argtypes = [vp, vp, C.c_int, C.c_double, C.c_int, C.c_int64,
                                             C.c_int64, C.c_int64, C.c_double, C.c_uint64,
                                             C.c_int, C.c_double, C.c_int, C.c_double, C.c_int,
                                             f64p, i64p]

    def _ck(self, rc):
        if rc != 0:
            raise RefError(rc, self.lib.ref_last_error().decode())

    # -- tensors
    def sparse(self, dims, coords, values):
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        coords = np.ascontiguousarray(coords, dtype=np.int64).reshape(-1, len(dims))
        values = np.ascontiguousarray(values, dtype=np.float64)
        h = C.c_void_p()
        self._ck(self.lib.ref_sparse_new(len(dims), _i64(dims), len(values), _i64(coords),
                                         _f64(values), C.byref(h)))
        return RefTensor(self, h, dims)

    def dense(self, dims, values):
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        values = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        h = C.c_void_p()
        self._ck(self.lib.ref_dense_new(len(dims), _i64(dims), _f64(values), C.byref(h)))
        return RefTensor(self, h, dims)

    def gen_gamma(self, dims, r, seed):
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        h, nxt = C.c_void_p(), C.c_uint64()
        truth = np.zeros(int(dims.sum()) * r)
        self._ck(self.lib.ref_gen_gamma(len(dims), _i64(dims), r, seed, C.byref(h), _f64(truth),
                                        C.byref(nxt)))
        return RefTensor(self, h, dims), truth, nxt.value

    def gen_binary(self, dims, r, delta, p_high, p_low, seed):
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        h, nxt = C.c_void_p(), C.c_uint64()
        truth = np.zeros(int(dims.sum()) * r)
        self._ck(self.lib.ref_gen_binary(len(dims), _i64(dims), r, delta, p_high, p_low, seed,
                                         C.byref(h), _f64(truth), C.byref(nxt)))
        return RefTensor(self, h, dims), truth, nxt.value

    def variance_ordering(self):
        """acceptance.cpp criterion 5: (model factors flat, [var_uni, var_strat, var_semi])."""
        model = np.zeros((40 + 30 + 20) * 3)
        var = np.zeros(3)
        self._ck(self.lib.ref_variance_ordering(_f64(model), _f64(var)))
        return model, var

    def acceptance_instance(self, criterion):
        """(RefTensor, model flat) of acceptance criterion 4 or 10."""
        dims = {4: (6, 5, 4), 10: (10, 8, 6)}[criterion]
        h = C.c_void_p()
        model = np.zeros(sum(dims) * 2)
        self._ck(self.lib.ref_acceptance_instance(criterion, C.byref(h), _f64(model)))
        return RefTensor(self, h, np.array(dims, dtype=np.int64)), model

    def similarity(self, dims, est, r_est, truth, r_true):
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        out = C.c_double()
        self._ck(self.lib.ref_similarity(len(dims), _i64(dims), r_est, _f64(Oracle.flat(est)),
                                         r_true, _f64(Oracle.flat(truth)), C.byref(out)))
        return out.value

    def write_model(self, factors, path):
        dims = np.array([len(f) for f in factors], dtype=np.int64)
        self._ck(self.lib.ref_write_model(len(dims), _i64(dims), factors[0].shape[1],
                                          _f64(Oracle.flat(factors)), str(path).encode()))

    def read_model(self, path, cap=1 << 22):
        d, r = C.c_int(), C.c_int64()
        dims = np.zeros(16, dtype=np.int64)
        flat = np.zeros(cap)
        self._ck(self.lib.ref_read_model(str(path).encode(), C.byref(d), _i64(dims), C.byref(r),
                                         _f64(flat), cap))
        out, at = [], 0
        for n in dims[:d.value]:
            out.append(flat[at:at + n * r.value].reshape(n, r.value).copy())
            at += n * r.value
        return out

    def write_trace(self, path, epoch, loss, lr, secs, accepted):
        n = len(epoch)
        acc = (C.c_int * max(n, 1))(*[int(a) for a in accepted])
        self._ck(self.lib.ref_write_trace(str(path).encode(), n,
                                          _i64(np.asarray(epoch, dtype=np.int64)),
                                          _f64(np.asarray(loss, dtype=np.float64)),
                                          _f64(np.asarray(lr, dtype=np.float64)),
                                          _f64(np.asarray(secs, dtype=np.float64)), acc))

    def read_tns(self, path):
        h, d, dims = C.c_void_p(), C.c_int(), np.zeros(16, dtype=np.int64)
        self._ck(self.lib.ref_read_tns(str(path).encode(), C.byref(h), C.byref(d), _i64(dims)))
        return RefTensor(self, h, dims[:d.value].copy())

    def read_dense(self, path):
        h, d, dims = C.c_void_p(), C.c_int(), np.zeros(16, dtype=np.int64)
        self._ck(self.lib.ref_read_dense(str(path).encode(), C.byref(h), C.byref(d), _i64(dims)))
        return RefTensor(self, h, dims[:d.value].copy())

    # -- rng
    def rng(self, seed):
        return RefRng(self, self.lib.ref_rng_new(seed))

    # -- loss
    def loss_value(self, kind, delta, x, m):
        out = C.c_double()
        self._ck(self.lib.ref_loss_value(kind, delta, x, m, C.byref(out)))
        return out.value

    def loss_deriv(self, kind, delta, x, m):
        out = C.c_double()
        self._ck(self.lib.ref_loss_deriv(kind, delta, x, m, C.byref(out)))
        return out.value

    # -- kernels
    def entries(self, dims, r, factors, idx):
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        idx = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1, len(dims))
        out = np.zeros(len(idx))
        self._ck(self.lib.ref_model_entry(len(dims), _i64(dims), r, _f64(Oracle.flat(factors)),
                                          len(idx), _i64(idx), _f64(out)))
        return out

    def weighted_derivs(self, dims, r, factors, loss_kind, delta, idx, x, w, subtract_zero=False):
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        idx = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1, len(dims))
        out = np.zeros(len(idx))
        self._ck(self.lib.ref_weighted_derivs(
            len(dims), _i64(dims), r, _f64(Oracle.flat(factors)), loss_kind, delta, len(idx),
            _i64(idx), _f64(np.ascontiguousarray(x, np.float64)),
            _f64(np.ascontiguousarray(w, np.float64)), 1 if subtract_zero else 0, _f64(out)))
        return out

    def mttkrp(self, dims, r, factors, idx, y, threads=1):
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        idx = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1, len(dims))
        y = np.ascontiguousarray(y, dtype=np.float64)
        out = np.zeros(int(np.sum(dims)) * r)
        self._ck(self.lib.ref_mttkrp_sampled_all(len(dims), _i64(dims), r,
                                                 _f64(Oracle.flat(factors)), len(idx), _i64(idx),
                                                 _f64(y), threads, _f64(out)))
        return out

    def adam(self, dims, r, factors, first, second, iterations, lr, grads, beta1=0.9,
             beta2=0.999, eps=1e-8, lb=None):
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        A = Oracle.flat(factors).copy()
        B = np.ascontiguousarray(first, dtype=np.float64).copy()
        Cm = np.ascontiguousarray(second, dtype=np.float64).copy()
        it = C.c_int64(iterations)
        self._ck(self.lib.ref_adam_step(len(dims), _i64(dims), r, _f64(A), _f64(B), _f64(Cm),
                                        C.byref(it), lr,
                                        _f64(np.ascontiguousarray(grads, np.float64)), beta1,
                                        beta2, eps, 0 if lb is None else 1,
                                        0.0 if lb is None else lb))
        return A, B, Cm, it.value

    def estimate_given(self, dims, r, factors, loss_kind, delta, idx, x, w):
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        idx = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1, len(dims))
        out = C.c_double()
        self._ck(self.lib.ref_estimate_given(len(dims), _i64(dims), r, _f64(Oracle.flat(factors)),
                                             loss_kind, delta, len(idx), _i64(idx),
                                             _f64(np.ascontiguousarray(x, np.float64)),
                                             _f64(np.ascontiguousarray(w, np.float64)),
                                             C.byref(out)))
        return out.value


class RefRng:
    def __init__(self, ref: Reference, h):
        self.ref, self.h = ref, h

    def __del__(self):
        try:
            self.ref.lib.ref_rng_free(self.h)
        except Exception:
            pass

    def split(self, label):
        if isinstance(label, str):
            return RefRng(self.ref, self.ref.lib.ref_rng_split_label(self.h, label.encode()))
        return RefRng(self.ref, self.ref.lib.ref_rng_split_u64(self.h, label))

    def next_u64(self):
        return int(self.ref.lib.ref_rng_next_u64(self.h))

    def next_double(self):
        return float(self.ref.lib.ref_rng_next_double(self.h))

    def next_below(self, n):
        out = C.c_uint64()
        self.ref._ck(self.ref.lib.ref_rng_next_below(self.h, n, C.byref(out)))
        return out.value


class RefTensor:
    def __init__(self, ref: Reference, h, dims):
        self.ref, self.h, self.dims = ref, h, dims

    def __del__(self):
        try:
            self.ref.lib.ref_tensor_free(self.h)
        except Exception:
            pass

    @property
    def nnz(self):
        return int(self.ref.lib.ref_sparse_nnz(self.h))

    def export(self):
        n = self.nnz
        coords = np.zeros((max(n, 1), len(self.dims)), dtype=np.int64)
        vals = np.zeros(max(n, 1))
        self.ref._ck(self.ref.lib.ref_sparse_export(self.h, _i64(coords), _f64(vals)))
        return coords[:n], vals[:n]

    def norm(self):
        return float(self.ref.lib.ref_tensor_norm(self.h))

    def value_at(self, idx):
        """TensorView::value_at (tensor.hpp:95-97): lookup / dense read."""
        ix = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1)
        out = C.c_double()
        self.ref._ck(self.ref.lib.ref_tensor_value_at(self.h, _i64(ix), C.byref(out)))
        return out.value

    def write_tns(self, path):
        self.ref._ck(self.ref.lib.ref_write_tns(self.h, str(path).encode()))

    def write_dense(self, path):
        self.ref._ck(self.ref.lib.ref_write_dense(self.h, str(path).encode()))

    def dense_values(self):
        out = np.zeros(int(np.prod(self.dims)))
        self.ref._ck(self.ref.lib.ref_dense_export(self.h, _f64(out)))
        return out

    def draw_scripted(self, r, factors, loss_kind, delta, strategy, s, p, q, rho, script,
                      cap=None):
        d = len(self.dims)
        cap = cap or max(1, s if strategy == 0 else p + q)
        idx = np.zeros((cap, d), dtype=np.int64)
        y = np.zeros(cap)
        n = C.c_int64()
        consumed = C.c_int64()
        stats = np.zeros(3, dtype=np.int64)
        sc = np.ascontiguousarray(script, dtype=np.uint64)
        self.ref._ck(self.ref.lib.ref_draw_gradient_samples_scripted(
            self.h, d, _i64(self.dims), r, _f64(Oracle.flat(factors)), loss_kind, delta,
            strategy, s, p, q, rho, _u64(sc), len(sc), cap, _i64(idx), _f64(y), C.byref(n),
            C.byref(consumed), _i64(stats)))
        k = n.value
        return dict(idx=idx[:k], y=y[:k], consumed=consumed.value,
                    stats=tuple(int(v) for v in stats))

    def draw_seeded(self, r, factors, loss_kind, delta, strategy, s, p, q, rho, seed, cap=None):
        d = len(self.dims)
        cap = cap or max(1, s if strategy == 0 else p + q)
        idx = np.zeros((cap, d), dtype=np.int64)
        y = np.zeros(cap)
        n = C.c_int64()
        self.ref._ck(self.ref.lib.ref_draw_gradient_samples_seeded(
            self.h, d, _i64(self.dims), r, _f64(Oracle.flat(factors)), loss_kind, delta,
            strategy, s, p, q, rho, seed, cap, _i64(idx), _f64(y), C.byref(n)))
        k = n.value
        return idx[:k], y[:k]

    def estimator_scripted(self, kind, count, rho, script, r, factors, loss_kind, delta):
        d = len(self.dims)
        cap = max(count, 1)
        idx = np.zeros((cap, d), dtype=np.int64)
        x, w = np.zeros(cap), np.zeros(cap)
        n = C.c_int64()
        est = C.c_double()
        sc = np.ascontiguousarray(script, dtype=np.uint64)
        self.ref._ck(self.ref.lib.ref_estimator_scripted(
            self.h, kind, count, rho, _u64(sc), len(sc), d, _i64(self.dims), r,
            _f64(Oracle.flat(factors)), loss_kind, delta, cap, _i64(idx), _f64(x), _f64(w),
            C.byref(n), C.byref(est)))
        k = n.value
        return idx[:k], x[:k], w[:k], est.value

    def gradient_poisson_implicit(self, r, factors):
        out = np.zeros(int(np.sum(self.dims)) * r)
        self.ref._ck(self.ref.lib.ref_gradient_poisson_implicit(
            self.h, len(self.dims), _i64(self.dims), r, _f64(Oracle.flat(factors)), _f64(out)))
        return out

    def bias_variance(self, r, factors, loss_kind, delta, strategy, s, p, q, rho, trials, seed):
        b, v = C.c_double(), C.c_double()
        self.ref._ck(self.ref.lib.ref_empirical_bias_variance(
            self.h, len(self.dims), _i64(self.dims), r, _f64(Oracle.flat(factors)), loss_kind,
            delta, strategy, s, p, q, rho, trials, seed, C.byref(b), C.byref(v)))
        return b.value, v.value

    def gradient_full(self, r, factors, loss_kind, delta):
        out = np.zeros(int(np.sum(self.dims)) * r)
        self.ref._ck(self.ref.lib.ref_gradient_full(self.h, len(self.dims), _i64(self.dims), r,
                                                     _f64(Oracle.flat(factors)), loss_kind, delta,
                                                     _f64(out)))
        return out


_ORACLE: Optional[Oracle] = None
_REF: Optional[Reference] = None


def oracle() -> Oracle:
    global _ORACLE
    if _ORACLE is None:
        _ORACLE = Oracle()
    return _ORACLE


def reference() -> Optional[Reference]:
    """The compiled reference, or None when oracle/_ref was not built/shipped."""
    global _REF
    if _REF is None and LIBREF.exists():
        _REF = Reference()
    return _REF


def rel_error(got, want) -> float:
    """tests/oracles.hpp:174-182: ||got - want||_2 / ||want||_2 (or ||got|| if want = 0)."""
    got = np.asarray(got, dtype=np.float64).reshape(-1)
    want = np.asarray(want, dtype=np.float64).reshape(-1)
    denom = np.linalg.norm(want)
    if denom == 0.0:
        return float(np.linalg.norm(got))
    return float(np.linalg.norm(got - want) / denom)


def philox_script(o: Oracle, strategy, dims, seed, it, s=0, p=0, eta=0, n_cand=0, q=0,
                  estimator=False):
    """The reference-order draw script the product's Philox stream produces:
    uniform: for t<s, k<d; stratified: p picks then n_cand candidates x d;
    semi: p picks then q draws x d.  Feed to ScriptedRng (script[at++] % n)."""
    d = len(dims)
    tu, tp, tz = (5, 6, 7) if estimator else (1, 2, 3)
    out = []
    if strategy == 0:
        for t in range(s):
            for k in range(d):
                out.append(o.draw_bounded(seed, tu, it, t, k, int(dims[k])))
        return np.array(out, dtype=np.uint64)
    for t in range(p):
        out.append(o.draw_bounded(seed, tp, it, t, 0, eta))
    tag = tz if strategy == 1 else 4
    count = n_cand if strategy == 1 else q
    for t in range(count):
        for k in range(d):
            out.append(o.draw_bounded(seed, tag, it, t, k, int(dims[k])))
    return np.array(out, dtype=np.uint64)
