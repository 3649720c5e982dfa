"""ctypes binding of the C-ABI library (include/kvrerank_b200.h).

The product path has no CPU fallback: if the shared library is missing or a
CUDA device is absent, the first call raises.  Loading (``lib()``) works
without a GPU so the symbol table can be checked on CPU-only hosts.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import ConfigError, KvRerankError, ShapeError

LIB_PATH = os.environ.get("KRR_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                    "_kvrerank_b200.so")

F32, F16, BF16 = 0, 1, 2
DTYPE_CODES = {"f32": F32, "f16": F16, "bf16": BF16}
EPI_STORE, EPI_GELU, EPI_RESIDUAL, EPI_QKV_ROPE, EPI_GLU_GELU, EPI_GLU_SILU = 0, 1, 2, 3, 4, 5
MLP_GELU, MLP_GEGLU, MLP_SWIGLU = 0, 1, 2
GEMM_AUTO, GEMM_TCGEN05, GEMM_SIMT = 0, 1, 2
ATTN_AUTO, ATTN_MMA, ATTN_SIMT, ATTN_TCGEN05 = 0, 1, 2, 3
ATTN_TC = ATTN_MMA

# every symbol include/kvrerank_b200.h declares
EXPORTS = (
    "krr_last_error", "krr_version", "krr_launch_count", "krr_workspace_bytes", "krr_forward",
    "krr_profile_enable", "krr_profile_read", "krr_init_uniform", "krr_embed", "krr_rmsnorm",
    "krr_gemm", "krr_attention", "krr_attention_quant", "krr_attention_occupancy", "krr_score_head", "krr_segmented_topk", "krr_dequant_kv",
    "krr_quant_pages", "krr_dequant_pages",
)

vp = C.c_void_p
i32, i64, u64 = C.c_int32, C.c_int64, C.c_uint64


class QKV(C.Structure):
    _fields_ = [("heads", i32), ("kv_heads", i32), ("head_dim", i32), ("seq_len", i32),
                ("pos0", i32), ("layer", i32), ("kv_len", i32), ("rope_cos", vp),
                ("rope_sin", vp), ("q_out", vp), ("kv_seq", vp), ("positions", vp)]


class Model(C.Structure):
    _fields_ = [("layers", i32), ("model_dim", i32), ("heads", i32), ("kv_heads", i32),
                ("head_dim", i32), ("vocab_size", i32), ("max_position", i32),
                ("act_dtype", i32), ("gemm_backend", i32), ("attn_backend", i32),
                ("token_embedding", vp), ("rope_cos", vp), ("rope_sin", vp),
                ("final_gain", vp), ("score_head", vp), ("attn_gain", vp), ("mlp_gain", vp),
                ("wqkv", vp), ("wo", vp), ("w_up", vp), ("w_down", vp),
                ("ffn_dim", i32), ("mlp_kind", i32), ("embed_scale", C.c_float)]


class Batch(C.Structure):
    _fields_ = [("n_seqs", i32), ("seq_len", i32), ("pos0", i32), ("prefix_len", i32),
                ("cur_kv_layers", i32), ("tokens", vp), ("tok_valid", vp), ("prefix_valid_len", vp),
                ("prefix_kv", vp), ("cur_kv", vp), ("last_index", vp), ("scores", vp),
                ("prefix_pool", vp), ("prefix_pool_bytes", i64), ("cur_pool", vp),
                ("cur_pool_bytes", i64), ("x_in", vp), ("x_out", vp), ("positions", vp),
                ("prefix_bits", i32), ("prefix_scales", vp)]


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise KvRerankError(
                f"CUDA extension {LIB_PATH} is missing; build it with "
                "`python -m paper_2504_02921_b200.build_ext` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.krr_last_error.restype = C.c_char_p
        L.krr_version.restype = C.c_char_p
        L.krr_launch_count.restype = u64
        L.krr_workspace_bytes.argtypes = [C.POINTER(Model), i64, C.POINTER(C.c_size_t)]
        L.krr_forward.argtypes = [C.POINTER(Model), C.POINTER(Batch), vp, C.c_size_t, vp]
        L.krr_profile_enable.argtypes = [C.c_int]
        L.krr_profile_read.argtypes = [C.POINTER(C.c_double), C.POINTER(u64),
                                       C.POINTER(C.c_double)]
        L.krr_init_uniform.argtypes = [u64, C.c_double, i64, i64, C.c_int, C.c_int, vp, i64, vp]
        L.krr_embed.argtypes = [vp, vp, i64, i32, vp, vp]
        L.krr_rmsnorm.argtypes = [vp, vp, i64, i32, C.c_int, vp, vp]
        L.krr_gemm.argtypes = [C.c_int, C.c_int, vp, vp, i64, i32, i32, C.c_int, vp,
                               C.POINTER(QKV), vp]
        L.krr_attention.argtypes = [C.c_int, C.c_int, vp, i32, i32, i32, i32, i32, i32, i32,
                                    i32, vp, vp, vp, vp, vp, vp, i64, vp, i64, vp]
        L.krr_attention_quant.argtypes = [C.c_int, C.c_int, vp, i32, i32, i32, i32, i32, i32,
                                          i32, i32, vp, vp, vp, vp, vp, vp, i64, vp, i64, i32,
                                          vp, vp]
        L.krr_attention_occupancy.argtypes = [C.c_int, i32, C.POINTER(i32)]
        L.krr_score_head.argtypes = [vp, i32, i32, i32, vp, vp, vp, vp, vp]
        L.krr_segmented_topk.argtypes = [vp, vp, i32, i32, i32, vp, vp, vp]
        L.krr_dequant_kv.argtypes = [vp, vp, i32, i32, i32, i32, C.c_int, vp, vp]
        L.krr_quant_pages.argtypes = [vp, C.c_int, i32, i32, i32, i32, i32, vp, vp, vp]
        L.krr_dequant_pages.argtypes = [vp, vp, i32, i32, i32, i32, i32, C.c_int, vp, vp]
        _LIB = L
    return _LIB


def check(rc: int) -> None:
    """Map a KRR_E* status to the reference's exception classes (errors.py)."""
    if rc == 0:
        return
    msg = lib().krr_last_error().decode("utf-8", "replace")
    if rc == 1:
        raise ConfigError(msg)
    if rc == 2:
        raise ShapeError(msg)
    if rc == 4:
        raise ConfigError(f"unsupported: {msg}")
    raise KvRerankError(f"CUDA failure: {msg}")


def launch_count() -> int:
    return int(lib().krr_launch_count())


def profile_enable(on: bool) -> None:
    check(lib().krr_profile_enable(1 if on else 0))


def profile_read():
    ms = (C.c_double * 3)()
    n = (u64 * 3)()
    fl = C.c_double()
    check(lib().krr_profile_read(ms, n, C.byref(fl)))
    return {"gemm_ms": ms[0], "attn_ms": ms[1], "misc_ms": ms[2],
            "gemm_launches": int(n[0]), "attn_launches": int(n[1]), "misc_launches": int(n[2]),
            "gemm_flops": fl.value}
