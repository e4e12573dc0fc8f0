"""paper_1906_01687_b200 — B200-native stochastic GCP gradient engine.

The hot path of arXiv 1906.01687 (sample tensor entries -> evaluate the
Kruskal model -> loss derivative -> d-mode sparse MTTKRP -> Adam) as
hand-written sm_100a CUDA behind the C-ABI in include/gcpb.h.  This package
holds the in-tree engine library (libgcpb.so), its ctypes binding and the
host-side mirror of the reference API.

Public names are loaded lazily so that ``python -m paper_1906_01687_b200.build``
works before the engine library exists; touching any of them without the
library raises ImportError (there is no CPU fallback).
"""
__version__ = "0.1.0"

_PUBLIC = {
    "BERNOULLI_ODDS", "BETA_HALF", "GAMMA", "GAUSSIAN", "HUBER", "POISSON", "SEMI_STRATIFIED",
    "STRATIFIED", "UNIFORM", "DomainError", "Engine", "GcpError", "GcpRuntimeError",
    "InvalidArgument", "LogicError", "LossFunction", "OutOfRange", "RejectionStats",
    "SamplerKind", "nccl_unique_id", "philox_bounded", "shard_range", "stratified_keep",
    "zero_batch_size", "RngStream", "BinaryProblemSpec", "FitConfig", "FitResult", "fit_gcp_adam",
}


def __getattr__(name):
    if name in _PUBLIC:
        if name in ("FitConfig", "FitResult", "fit_gcp_adam"):
            from . import fit as _m
        else:
            from . import gcp as _m
        return getattr(_m, name)
    raise AttributeError(name)
