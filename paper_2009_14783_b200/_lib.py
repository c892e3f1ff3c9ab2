"""ctypes binding of the C ABI in include/hetpar_b200.h.

The shared library is built in-tree by tools/build_native.py (called from
__graft_entry__.build()).  There is no fallback: if the library is missing the
import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhetpar_b200.so")
if os.environ.get("HP_LIB_VARIANT"):  # A/B builds (tools/build_native.py HP_VARIANT)
    LIB_PATH = os.path.join(_HERE, f"libhetpar_b200_{os.environ['HP_LIB_VARIANT']}.so")

HP_OK, HP_ESHAPE, HP_ECONFIG, HP_EINDEX, HP_EIO, HP_ECOMM, HP_ENUMERIC, HP_ECUDA = range(8)
HP_ARCH_MASKED_TOKEN_MODEL = 3
HP_ARCH_BERT_ENCODER = 16
HP_ARCH_SEQ2SEQ = 17
HP_OPT_SGD, HP_OPT_ADAM, HP_OPT_ADAMW = 0, 1, 2
HP_POLICY_SENTENCES, HP_POLICY_TOKENS = 1, 2
HP_COMPUTE_F32, HP_COMPUTE_BF16 = 0, 1


# Reference error taxonomy (include/hetpar/common.hpp:14-34).
class BaseError(RuntimeError):
    pass


class ShapeError(BaseError):
    pass


class ConfigError(BaseError):
    pass


class IndexError_(BaseError):
    pass


class IoError(BaseError):
    pass


class CommError(BaseError):
    pass


class NumericError(BaseError):
    pass


class CudaError(BaseError):
    pass


_ERRORS = {HP_ESHAPE: ShapeError, HP_ECONFIG: ConfigError, HP_EINDEX: IndexError_,
           HP_EIO: IoError, HP_ECOMM: CommError, HP_ENUMERIC: NumericError,
           HP_ECUDA: CudaError}


class MlmGenDesc(C.Structure):
    _fields_ = [("n", C.c_uint64), ("vocab", C.c_int64), ("docs", C.c_uint64),
                ("sentences_per_doc", C.c_uint64), ("min_words", C.c_uint64),
                ("max_words", C.c_uint64), ("p_select", C.c_double), ("p_mask", C.c_double),
                ("p_random", C.c_double), ("seed", C.c_uint64), ("max_seq_tokens", C.c_uint64)]


class PairGenDesc(C.Structure):
    _fields_ = [("n", C.c_uint64), ("vocab", C.c_int64), ("min_len", C.c_uint64),
                ("max_len", C.c_uint64), ("seed", C.c_uint64)]


class ModelDesc(C.Structure):
    _fields_ = [("arch", C.c_int), ("d_model", C.c_uint64), ("heads", C.c_uint64),
                ("vocab", C.c_uint64), ("max_seq", C.c_uint64), ("layers", C.c_uint64),
                ("d_ff", C.c_uint64), ("with_nsp", C.c_int), ("label_smooth_eps", C.c_double)]


class OptimDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("weight_decay", C.c_double)]


class ExecDesc(C.Structure):
    _fields_ = [("compute", C.c_int), ("policy", C.c_int), ("device", C.c_int),
                ("bucket_mb", C.c_double), ("max_tokens", C.c_uint64), ("max_batch", C.c_uint64),
                ("max_masks", C.c_uint64), ("update_freq", C.c_uint64)]


class BatchDesc(C.Structure):
    _fields_ = [("n_inst", C.c_uint64), ("tok_off", C.c_void_p), ("tokens", C.c_void_p),
                ("segments", C.c_void_p), ("mask_off", C.c_void_p), ("mask_pos", C.c_void_p),
                ("mask_orig", C.c_void_p), ("label", C.c_void_p)]


class LoadedDesc(C.Structure):
    _fields_ = [("batch_index", C.c_uint64), ("dummy", C.c_int), ("batch", BatchDesc)]


class CkptDesc(C.Structure):
    _fields_ = [("epoch", C.c_uint64), ("step", C.c_uint64), ("seed", C.c_uint64),
                ("policy", C.c_int), ("world_size", C.c_uint64), ("update_freq", C.c_uint64),
                ("sched_kind", C.c_int), ("peak_lr", C.c_double), ("sched_d_model", C.c_uint64),
                ("warmup_steps", C.c_uint64), ("total_steps", C.c_uint64), ("opt_kind", C.c_int),
                ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("opt_t", C.c_uint64), ("weight_decay", C.c_double)]


class RoundOut(C.Structure):
    _fields_ = [("updated", C.c_int), ("step", C.c_uint64), ("loss", C.c_double),
                ("weight", C.c_double), ("local_loss_sum", C.c_double),
                ("local_weight", C.c_double)]


P = C.c_void_p
U64 = C.c_uint64
I64 = C.c_int64
I = C.c_int
D = C.c_double

# name -> argtypes (every entry point returns hp_status)
_SIGS = {
    "hp_splitmix64": [U64, U64, P],
    "hp_shuffle_iota": [U64, U64, P],
    "hp_build_epoch_batches": [P, U64, U64, U64, U64, U64, P, P, P],
    "hp_partition_for_rank": [U64, U64, U64, P, P, P],
    "hp_mlm_generate_size": [P, P, P],
    "hp_mlm_generate": [P, P, P, P, P, P, P, P],
    "hp_pairs_generate_size": [P, P],
    "hp_pairs_generate": [P, P, P, P],
    "hp_param_count": [P, P, P],
    "hp_param_info": [P, U64, C.c_char_p, U64, P, P, P, P],
    "hp_init_parameters": [P, U64, P],
    "hp_bucket_plan": [P, D, P, P, P],
    "hp_comm_unique_id": [P],
    "hp_comm_create": [I, I, I, P, P],
    "hp_comm_destroy": [P],
    "hp_engine_create": [P, P, P, P, P],
    "hp_engine_destroy": [P],
    "hp_engine_set_params": [P, P, U64, I],
    "hp_engine_get_params": [P, P, U64, I],
    "hp_engine_broadcast_params": [P, I],
    "hp_engine_get_adam": [P, P, P, P],
    "hp_engine_set_adam": [P, P, P, U64],
    "hp_comm_create_tcp": [C.c_char_p, C.c_uint16, I, I, I, I, P],
    "hp_pg_broadcast": [P, P, U64, U64, P, U64, P],
    "hp_pg_all_reduce_sum": [P, P, U64, P],
    "hp_pg_gather_scalars": [P, C.c_double, P],
    "hp_pg_barrier": [P],
    "hp_comm_allreduce_bench": [P, U64, D, I, I, P],
    "hp_shards_open": [C.c_char_p, P],
    "hp_shards_info": [P, P, P],
    "hp_shards_token_lengths": [P, P, U64],
    "hp_shards_close": [P],
    "hp_mlm_write_shards": [C.c_char_p, U64, U64, P, P, P, P, P, P, P],
    "hp_loader_create": [P, P, P, U64, P, P, U64, U64, P],
    "hp_loader_next": [P, P, P],
    "hp_loader_destroy": [P],
    "hp_checkpoint_write": [C.c_char_p, P, P, P, P, P],
    "hp_checkpoint_read": [C.c_char_p, P, P, P, P, P, U64],
    "hp_engine_save_checkpoint": [P, C.c_char_p, P],
    "hp_engine_load_checkpoint": [P, C.c_char_p, P],
    "hp_resume_position": [P, U64, U64, U64, U64, U64, U64, U64, P, P],
    "hp_engine_set_capture": [P, I],
    "hp_engine_get_local_grads": [P, P, U64],
    "hp_engine_stage_batch": [P, P],
    "hp_engine_round_async": [P, I, D],
    "hp_engine_round_sync": [P, P],
    "hp_engine_round": [P, I, D, P],
    "hp_engine_params_digest": [P, P],
    "hp_engine_kernel_launches": [P, P],
    "hp_engine_timers": [P, I],
    "hp_engine_timer_read": [P, I, C.c_char_p, U64, P, P, P, P],
    "hp_engine_class_replay": [P, I, I, P, P, P],
    "hp_engine_step_count": [P, P],
    "hp_engine_set_step": [P, U64],
    "hp_engine_pending_rounds": [P, P],
    "hp_engine_mark": [P, I],
    "hp_engine_elapsed": [P, I, I, P],
    "hp_engine_synchronize": [P],
    "hp_engine_io_bytes": [P, P, P],
    "hp_engine_set_grad_comm": [P, I],
    "hp_engine_set_digest_check": [P, U64, I],
    "hp_engine_forward": [P, P, P],
    "hp_kern_dot_f32": [P, P, U64, P, P],
    "hp_kern_sum_f32": [P, U64, P, P],
    "hp_kern_maxv_f32": [P, U64, P, P],
    "hp_kern_add_f32": [P, P, P, U64, P],
    "hp_kern_scale_f32": [P, C.c_float, P, U64, P],
    "hp_kern_axpy_f32": [C.c_float, P, P, U64, P],
    "hp_kern_relu_f32": [P, P, U64, P],
    "hp_kern_relu_bwd_f32": [P, P, P, U64, P],
    "hp_kern_sgd_update_f32": [P, P, U64, C.c_float, P],
    "hp_kern_adam_update_f32": [P, P, P, P, U64, C.c_float, C.c_float, C.c_float, C.c_float, C.c_float, C.c_float, P],
    "hp_kern_dot_f64": [P, P, U64, P, P],
    "hp_kern_sum_f64": [P, U64, P, P],
    "hp_kern_maxv_f64": [P, U64, P, P],
    "hp_kern_add_f64": [P, P, P, U64, P],
    "hp_kern_scale_f64": [P, D, P, U64, P],
    "hp_kern_axpy_f64": [D, P, P, U64, P],
    "hp_kern_relu_f64": [P, P, U64, P],
    "hp_kern_relu_bwd_f64": [P, P, P, U64, P],
    "hp_kern_sgd_update_f64": [P, P, U64, D, P],
    "hp_kern_adam_update_f64": [P, P, P, P, U64, D, D, D, D, D, D, P],
    "hp_debug_gemm": [I, I, I, I, P, I64, I, P, I64, I, I64, I64, P, I64, I, I64, I64, P, I, P, P,
                      I64, I, I, I],
    "hp_debug_sync": [],
    "hp_debug_set_stream": [P],
    "hp_debug_gemm_trace": [P],
    "hp_debug_gemm_generic": [I],
    "hp_debug_attention": [I, P, I, I, I, I, P, P, P, P, P, I],
    "hp_debug_layernorm": [I, I, I, P, P, P, P, P, P, P, P, P, P, P, I],
    "hp_debug_attention2": [I, P, P, I, I, I, I, I, I, I, P, I64, I, P, I64, I, P, I64, I, P, P,
                            P, P, I64, I, P, I64, I, P, I64, I, I, I],
    "hp_debug_adam": [P, P, P, P, U64, C.c_float, C.c_float, C.c_float, C.c_float, C.c_float,
                      C.c_float, I, C.c_float],
}

EXPORTED = sorted(_SIGS) + ["hp_last_error", "hp_version"]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, args in _SIGS.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = C.c_int
    lib.hp_last_error.restype = C.c_char_p
    lib.hp_last_error.argtypes = []
    lib.hp_version.restype = C.c_char_p
    lib.hp_version.argtypes = []
    return lib


lib = _load()


def check(status: int) -> None:
    if status != HP_OK:
        msg = lib.hp_last_error().decode(errors="replace")
        raise _ERRORS.get(status, BaseError)(msg)


def call(name: str, *args) -> None:
    check(getattr(lib, name)(*args))
