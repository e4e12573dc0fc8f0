"""Tensor files (include/gcp/io.hpp; src/io.cpp), parsed by the engine
library's native reader (csrc/gcpb_io.cpp).

* ``read_tns`` / ``write_tns`` — the reference's coordinate text format
  (1-based indices, optional ``#shape:`` header, ``#`` comments).
* ``read_coo`` / ``write_coo`` — this framework's binary coordinate format
  (GCPBCOO1), the fast path for large tensors.
* ``read_dense`` / ``write_dense`` — raw little-endian f64 with a ``.shape``
  sidecar (io.cpp:195-250).

Readers return entries in file order; ``Engine.set_sparse`` normalises them
(sums duplicates, drops zeros, sorts by linear key) exactly like the
reference's SparseTensor constructor.  Errors raise the same classes as the
reference (runtime errors -> ``GcpRuntimeError`` carrying ``path:line:``).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _capi
from ._capi import lib
from .gcp import Engine, _check


@dataclass
class CooTensor:
    """A coordinate list: dims, coords (nnz x d, 0-based) and values."""
    dims: tuple
    coords: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return len(self.values)

    @property
    def ndims(self) -> int:
        return len(self.dims)

    def to_engine(self, rank: int, dtype: str = "f64", device: int = 0) -> Engine:
        e = Engine(self.dims, rank, dtype=dtype, device=device)
        e.set_sparse(self.coords, self.values)
        return e


def _take(c: _capi.gcpb_coo) -> CooTensor:
    try:
        d, nnz = int(c.d), int(c.nnz)
        dims = tuple(int(c.dims[k]) for k in range(d))
        if nnz:
            coords = np.ctypeslib.as_array(c.coords, shape=(nnz, d)).copy()
            values = np.ctypeslib.as_array(c.values, shape=(nnz,)).copy()
        else:
            coords = np.zeros((0, d), dtype=np.int64)
            values = np.zeros(0)
        return CooTensor(dims, coords, values)
    finally:
        lib.gcpb_coo_free(C.byref(c))


def _pack(t: CooTensor):
    coords = np.ascontiguousarray(t.coords, dtype=np.int64).reshape(-1, len(t.dims))
    values = np.ascontiguousarray(t.values, dtype=np.float64)
    c = _capi.gcpb_coo()
    c.d = len(t.dims)
    for k, n in enumerate(t.dims):
        c.dims[k] = int(n)
    c.nnz = len(values)
    c.coords = coords.ctypes.data_as(_capi.i64p)
    c.values = values.ctypes.data_as(_capi.f64p)
    return c, (coords, values)


def read_tns(path: str | os.PathLike, threads: int = 0) -> CooTensor:
    """read_tns (io.cpp:75-139), parsed in parallel."""
    c = _capi.gcpb_coo()
    _check(lib.gcpb_tns_read(os.fsencode(path), threads, C.byref(c)))
    return _take(c)


def write_tns(t: CooTensor, path: str | os.PathLike) -> None:
    """write_tns (io.cpp:141-151): header, 1-based entries, %.17g values."""
    c, keep = _pack(t)
    _check(lib.gcpb_tns_write(os.fsencode(path), C.byref(c)))


def read_coo(path: str | os.PathLike, threads: int = 0) -> CooTensor:
    c = _capi.gcpb_coo()
    _check(lib.gcpb_coo_read(os.fsencode(path), threads, C.byref(c)))
    return _take(c)


def write_coo(t: CooTensor, path: str | os.PathLike) -> None:
    c, keep = _pack(t)
    _check(lib.gcpb_coo_write(os.fsencode(path), C.byref(c)))


def read_dense(path: str | os.PathLike):
    """read_dense (io.cpp:195-226) -> (dims, values in first-mode-fastest order)."""
    d = C.c_int32()
    dims = np.zeros(16, dtype=np.int64)
    _check(lib.gcpb_dense_shape(os.fsencode(path), C.byref(d), dims.ctypes.data_as(_capi.i64p)))
    dims = tuple(int(n) for n in dims[:d.value])
    n = int(np.prod(np.array(dims, dtype=object)))
    vals = np.zeros(n)
    _check(lib.gcpb_dense_read(os.fsencode(path), n, vals.ctypes.data_as(_capi.f64p)))
    return dims, vals


def write_dense(dims: Sequence[int], values, path: str | os.PathLike) -> None:
    dims_a = np.ascontiguousarray(dims, dtype=np.int64)
    vals = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
    _check(lib.gcpb_dense_write(os.fsencode(path), len(dims_a), dims_a.ctypes.data_as(_capi.i64p),
                                vals.ctypes.data_as(_capi.f64p)))


def read_model(path: str | os.PathLike):
    """read_model (io.cpp:153-177) -> list of n_k x r factor matrices."""
    d = C.c_int32()
    dims = np.zeros(16, dtype=np.int64)
    r = C.c_int64()
    _check(lib.gcpb_model_read_header(os.fsencode(path), C.byref(d), dims.ctypes.data_as(_capi.i64p),
                                      C.byref(r)))
    dims = [int(n) for n in dims[:d.value]]
    flat = np.zeros(sum(dims) * r.value)
    _check(lib.gcpb_model_read(os.fsencode(path), flat.ctypes.data_as(_capi.f64p)))
    out, at = [], 0
    for n in dims:
        out.append(flat[at:at + n * r.value].reshape(n, r.value).copy())
        at += n * r.value
    return out


def write_model(factors, path: str | os.PathLike) -> None:
    """write_model (io.cpp:179-193): %.17g values, bit-exact round trip."""
    factors = [np.ascontiguousarray(f, dtype=np.float64) for f in factors]
    dims = np.array([f.shape[0] for f in factors], dtype=np.int64)
    r = factors[0].shape[1]
    flat = np.concatenate([f.reshape(-1) for f in factors])
    _check(lib.gcpb_model_write(os.fsencode(path), len(dims), dims.ctypes.data_as(_capi.i64p), r,
                                flat.ctypes.data_as(_capi.f64p)))


def write_trace_csv(trace, path: str | os.PathLike) -> None:
    """write_trace_csv (io.cpp:252-260) from FitResult.trace records."""
    arr = (_capi.gcpb_trace_record * max(len(trace), 1))()
    for i, t in enumerate(trace):
        arr[i].epoch, arr[i].loss_estimate = int(t.epoch), float(t.loss_estimate)
        arr[i].learning_rate, arr[i].seconds = float(t.learning_rate), float(t.seconds)
        arr[i].accepted = 1 if t.accepted else 0
    _check(lib.gcpb_trace_write_csv(os.fsencode(path), arr, len(trace)))


def engine_from_file(path: str | os.PathLike, rank: int, dtype: str = "f64", device: int = 0,
                     storage: Optional[str] = None) -> Engine:
    """Load a .tns / GCPBCOO1 / dense file straight into a device engine."""
    p = os.fspath(path)
    if os.path.exists(p + ".shape"):
        dims, vals = read_dense(p)
        e = Engine(dims, rank, dtype=dtype, device=device)
        e.set_dense(vals, storage or dtype)
        return e
    with open(p, "rb") as f:
        magic = f.read(8)
    t = read_coo(p) if magic == b"GCPBCOO1" else read_tns(p)
    return t.to_engine(rank, dtype, device)
