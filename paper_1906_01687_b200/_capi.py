"""ctypes binding of the C-ABI in include/gcpb.h (libgcpb.so, built in-tree).

There is no fallback: if the engine library is missing, importing this module
raises — build it with ``python -m paper_1906_01687_b200.build``.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_LIB_PATH = Path(os.environ.get("GCPB_LIB", Path(__file__).resolve().parent / "libgcpb.so"))

if not _LIB_PATH.exists():
    raise ImportError(
        f"gcpb engine library not found at {_LIB_PATH}; build it with "
        "`python -m paper_1906_01687_b200.build` (there is no CPU fallback)")



def _preload_torch_nccl() -> None:
    """libgcpb.so links libnccl.so.2; so does torch, which bundles a newer copy
    and needs its symbols.  The first copy loaded serves the whole process, so
    when torch's is installed it is loaded first here — importing this package
    before torch must not leave torch with the system's older library."""
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
        if spec and spec.submodule_search_locations:
            for d in spec.submodule_search_locations:
                p = Path(d) / "lib" / "libnccl.so.2"
                if p.exists():
                    C.CDLL(str(p), mode=C.RTLD_GLOBAL)
                    return
    except (ImportError, OSError, ValueError):
        pass


_preload_torch_nccl()
lib = C.CDLL(str(_LIB_PATH))

# status codes (gcpb.h)
OK, ERR_RUNTIME, ERR_USAGE, ERR_DOMAIN, ERR_RANGE, ERR_LOGIC = 0, 1, 2, 3, 4, 5
PEER_HANDLE_BYTES = 256  # GCPB_PEER_HANDLE_BYTES (include/gcpb.h)
F32, F64 = 0, 1
STORE_U8, STORE_F32, STORE_F64, STORE_BIT = 0, 1, 2, 3
UNIFORM, STRATIFIED, SEMI_STRATIFIED = 0, 1, 2
EST_UNIFORM, EST_STRATIFIED = 0, 1


class gcpb_loss(C.Structure):
    _fields_ = [("kind", C.c_int32), ("delta", C.c_double)]


class gcpb_sampler(C.Structure):
    _fields_ = [("strategy", C.c_int32), ("num_samples", C.c_int64),
                ("nonzero_samples", C.c_int64), ("zero_samples", C.c_int64),
                ("oversample", C.c_double)]


class gcpb_stats(C.Structure):
    _fields_ = [("tested", C.c_int64), ("accepted", C.c_int64), ("rejected", C.c_int64)]


class gcpb_adam(C.Structure):
    _fields_ = [("learning_rate", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("epsilon", C.c_double), ("has_lower_bound", C.c_int32),
                ("lower_bound", C.c_double)]


class gcpb_fit_config(C.Structure):
    _fields_ = [("sampler", gcpb_sampler), ("learning_rate", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("epsilon", C.c_double), ("epoch_iters", C.c_int64),
                ("max_bad_epochs", C.c_int64), ("decay", C.c_double),
                ("lower_bound_mode", C.c_int32), ("lower_bound", C.c_double),
                ("estimator_samples", C.c_int64), ("estimator_kind", C.c_int32),
                ("max_epochs", C.c_int64), ("seed", C.c_uint64), ("keep_factors", C.c_int32),
                ("draw_stream", C.c_int32)]


class gcpb_trace_record(C.Structure):
    _fields_ = [("epoch", C.c_int64), ("loss_estimate", C.c_double),
                ("learning_rate", C.c_double), ("seconds", C.c_double), ("accepted", C.c_int32)]


class gcpb_rng(C.Structure):
    _fields_ = [("key", C.c_uint64), ("counter", C.c_uint64), ("has_cached_normal", C.c_int32),
                ("cached_normal", C.c_double)]


class gcpb_binary_spec(C.Structure):
    _fields_ = [("delta", C.c_double), ("p_high", C.c_double), ("p_low", C.c_double)]


class gcpb_coo(C.Structure):
    _fields_ = [("d", C.c_int32), ("dims", C.c_int64 * 16), ("nnz", C.c_int64),
                ("coords", C.POINTER(C.c_int64)), ("values", C.POINTER(C.c_double))]


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.POINTER(C.c_int64))
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int64)

ctx_p = C.c_void_p
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
i32p = C.POINTER(C.c_int32)
u64p = C.POINTER(C.c_uint64)

# (name, restype, argtypes) for every entry point of include/gcpb.h
SIGNATURES = [
    ("gcpb_create", C.c_int, [C.c_int, C.c_int, C.c_int, i64p, C.c_int64, C.POINTER(ctx_p)]),
    ("gcpb_destroy", None, [ctx_p]),
    ("gcpb_last_error", C.c_char_p, [ctx_p]),
    ("gcpb_version", C.c_char_p, []),
    ("gcpb_set_stream", C.c_int, [ctx_p, C.c_void_p]),
    ("gcpb_get_stream", C.c_void_p, [ctx_p]),
    ("gcpb_set_sparse", C.c_int, [ctx_p, C.c_int64, i64p, f64p]),
    ("gcpb_set_sparse_device", C.c_int, [ctx_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int]),
    ("gcpb_nnz", C.c_int64, [ctx_p]),
    ("gcpb_get_sparse", C.c_int, [ctx_p, i64p, f64p]),
    ("gcpb_set_dense", C.c_int, [ctx_p, f64p, C.c_int]),
    ("gcpb_set_dense_device", C.c_int, [ctx_p, C.c_void_p, C.c_int]),
    ("gcpb_generate_dense_bernoulli", C.c_int, [ctx_p, C.c_int64, f64p, C.c_uint64, C.c_int]),
    ("gcpb_tensor_norm", C.c_int, [ctx_p, f64p]),
    ("gcpb_value_at", C.c_int, [ctx_p, C.c_int64, i64p, f64p]),
    ("gcpb_set_factors", C.c_int, [ctx_p, C.c_int, f64p]),
    ("gcpb_get_factors", C.c_int, [ctx_p, C.c_int, f64p]),
    ("gcpb_get_grad", C.c_int, [ctx_p, C.c_int, f64p]),
    ("gcpb_set_grad", C.c_int, [ctx_p, C.c_int, f64p]),
    ("gcpb_get_moment", C.c_int, [ctx_p, C.c_int, C.c_int, f64p]),
    ("gcpb_set_moment", C.c_int, [ctx_p, C.c_int, C.c_int, f64p]),
    ("gcpb_stoch_grad", C.c_int, [ctx_p, C.POINTER(gcpb_sampler), C.POINTER(gcpb_loss),
                                  C.c_uint64, C.c_uint64, C.POINTER(gcpb_stats)]),
    ("gcpb_draw_samples", C.c_int, [ctx_p, C.POINTER(gcpb_sampler), C.POINTER(gcpb_loss),
                                    C.c_uint64, C.c_uint64, C.c_int64, i64p, f64p, f64p, i32p,
                                    f64p, f64p, i64p, C.POINTER(gcpb_stats)]),
    ("gcpb_eval_deriv", C.c_int, [ctx_p, C.c_int64, i64p, f64p, f64p, i32p,
                                  C.POINTER(gcpb_loss), f64p, f64p]),
    ("gcpb_mttkrp_samples", C.c_int, [ctx_p, C.c_int64, i64p, f64p]),
    ("gcpb_adam_step", C.c_int, [ctx_p, C.POINTER(gcpb_adam)]),
    ("gcpb_adam_reset", C.c_int, [ctx_p]),
    ("gcpb_get_iterations", C.c_int, [ctx_p, i64p]),
    ("gcpb_set_iterations", C.c_int, [ctx_p, C.c_int64]),
    ("gcpb_step", C.c_int, [ctx_p, C.POINTER(gcpb_sampler), C.POINTER(gcpb_loss), C.c_uint64,
                            C.c_uint64, C.POINTER(gcpb_adam)]),
    ("gcpb_step_host", C.c_int, [ctx_p, C.POINTER(gcpb_sampler), C.POINTER(gcpb_loss), C.c_uint64,
                                 C.c_uint64, C.POINTER(gcpb_adam), f64p, f64p]),
    ("gcpb_run_steps", C.c_int, [ctx_p, C.POINTER(gcpb_sampler), C.POINTER(gcpb_loss),
                                 C.c_uint64, C.c_uint64, C.c_int64, C.POINTER(gcpb_adam)]),
    ("gcpb_synchronize", C.c_int, [ctx_p]),
    ("gcpb_steps_path", C.c_int, [ctx_p]),
    ("gcpb_run_steps_launches", C.c_int, [ctx_p, C.POINTER(C.c_int64)]),
    ("gcpb_last_transfer_bytes", C.c_int, [ctx_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("gcpb_debug_guard_failures", C.c_int64, [C.POINTER(C.c_int64)]),
    ("gcpb_debug_check_failures", C.c_int64, [C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("gcpb_hot_rows", C.c_int, [ctx_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("gcpb_interleaved", C.c_int, [ctx_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("gcpb_gradient_full", C.c_int, [ctx_p, C.POINTER(gcpb_loss)]),
    ("gcpb_gradient_poisson_implicit", C.c_int, [ctx_p, C.POINTER(gcpb_loss)]),
    ("gcpb_gradient_moments", C.c_int, [ctx_p, C.POINTER(gcpb_sampler), C.POINTER(gcpb_loss),
                                        C.c_int64, C.c_uint64, f64p, f64p]),
    ("gcpb_bias_variance", C.c_int, [ctx_p, C.POINTER(gcpb_sampler), C.POINTER(gcpb_loss),
                                     C.c_int64, C.c_uint64, f64p, f64p, f64p]),
    ("gcpb_set_draw_stream", C.c_int, [ctx_p, C.c_int, C.c_uint64]),
    ("gcpb_get_draw_counter", C.c_int, [ctx_p, u64p]),
    ("gcpb_kernel_timing", C.c_int, [ctx_p, C.c_int]),
    ("gcpb_kernel_time", C.c_int, [ctx_p, f64p, i64p]),
    ("gcpb_fit_gcp_adam", C.c_int, [ctx_p, C.POINTER(gcpb_loss), C.POINTER(gcpb_fit_config),
                                    C.POINTER(gcpb_trace_record), C.c_int64, i64p, f64p]),
    ("gcpb_estimator_set", C.c_int, [ctx_p, C.c_int64, i64p, f64p, f64p]),
    ("gcpb_estimator_draw", C.c_int, [ctx_p, C.c_int, C.c_int64, C.c_double, C.c_uint64]),
    ("gcpb_estimator_size", C.c_int64, [ctx_p]),
    ("gcpb_estimator_get", C.c_int, [ctx_p, i64p, f64p, f64p]),
    ("gcpb_estimate", C.c_int, [ctx_p, C.POINTER(gcpb_loss), f64p]),
    ("gcpb_snapshot_save", C.c_int, [ctx_p]),
    ("gcpb_snapshot_restore", C.c_int, [ctx_p]),
    ("gcpb_nccl_unique_id", C.c_int, [C.c_char_p]),
    ("gcpb_comm_init", C.c_int, [ctx_p, C.c_char_p, C.c_int, C.c_int]),
    ("gcpb_set_shard", C.c_int, [ctx_p, C.c_int, C.c_int]),
    ("gcpb_peer_handle", C.c_int, [ctx_p, C.c_void_p]),
    ("gcpb_peer_open", C.c_int, [ctx_p, C.c_char_p, C.c_int]),
    ("gcpb_peer_close", C.c_int, [ctx_p]),
    ("gcpb_allreduce_grad", C.c_int, [ctx_p]),
    ("gcpb_comm_init_host", C.c_int, [ctx_p, C.c_int, C.c_int, ALLGATHER_FN, ALLREDUCE_FN,
                                      C.c_void_p]),
    ("gcpb_rng_seed", C.c_int, [C.c_uint64, C.POINTER(gcpb_rng)]),
    ("gcpb_rng_split", C.c_int, [C.POINTER(gcpb_rng), C.c_uint64, C.POINTER(gcpb_rng)]),
    ("gcpb_gen_gamma_problem", C.c_int, [ctx_p, C.POINTER(gcpb_rng), C.c_int, f64p]),
    ("gcpb_gen_binary_problem", C.c_int, [ctx_p, C.POINTER(gcpb_binary_spec),
                                          C.POINTER(gcpb_rng), f64p]),
    ("gcpb_tns_read", C.c_int, [C.c_char_p, C.c_int, C.POINTER(gcpb_coo)]),
    ("gcpb_tns_write", C.c_int, [C.c_char_p, C.POINTER(gcpb_coo)]),
    ("gcpb_coo_write", C.c_int, [C.c_char_p, C.POINTER(gcpb_coo)]),
    ("gcpb_coo_read", C.c_int, [C.c_char_p, C.c_int, C.POINTER(gcpb_coo)]),
    ("gcpb_coo_free", None, [C.POINTER(gcpb_coo)]),
    ("gcpb_dense_shape", C.c_int, [C.c_char_p, i32p, i64p]),
    ("gcpb_dense_read", C.c_int, [C.c_char_p, C.c_int64, f64p]),
    ("gcpb_dense_write", C.c_int, [C.c_char_p, C.c_int, i64p, f64p]),
    ("gcpb_model_read_header", C.c_int, [C.c_char_p, i32p, i64p, i64p]),
    ("gcpb_model_read", C.c_int, [C.c_char_p, f64p]),
    ("gcpb_model_write", C.c_int, [C.c_char_p, C.c_int, i64p, C.c_int64, f64p]),
    ("gcpb_trace_write_csv", C.c_int, [C.c_char_p, C.POINTER(gcpb_trace_record), C.c_int64]),
    ("gcpb_philox_bounded", C.c_uint64, [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_int,
                                         C.c_uint64]),
    ("gcpb_zero_batch_size", C.c_int64, [C.c_double, C.c_double, C.c_double, C.c_int64]),
    ("gcpb_shard_range", None, [C.c_int64, C.c_int, C.c_int, i64p, i64p]),
    ("gcpb_stratified_keep", None, [i64p, C.c_int, C.c_int, C.c_int64, i64p, i64p]),
    ("gcpb_loss_deriv", C.c_double, [C.POINTER(gcpb_loss), C.c_double, C.c_double]),
    ("gcpb_loss_value", C.c_double, [C.POINTER(gcpb_loss), C.c_double, C.c_double]),
]

for _name, _res, _args in SIGNATURES:
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = [s[0] for s in SIGNATURES]
