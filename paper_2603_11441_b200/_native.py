"""ctypes binding of libdart_b200.so (include/dart_b200.h).

The product path has no CPU fallback: if the shared library is missing, or no CUDA
device is present, every forward raises.  `load()` is the single place the library
is opened; it is built in-tree by `__graft_entry__.build()` (csrc/Makefile).
"""

from __future__ import annotations

import ctypes
import os

# DART_LIB_PATH: A/B microbenchmarks of another build (the product path loads the in-tree library)
LIB_PATH = os.environ.get("DART_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libdart_b200.so")
MAX_BLOCKS = 256

DART_OK = 0
DART_ERR_INVALID = 1
DART_ERR_CUDA = 2
FLAG_IMAGE_RANGE = 1
FLAG_NONFINITE = 2

# Every symbol include/dart_b200.h declares (checked by tests/test_native_abi.py).
EXPORTS = (
    "dart_model_create",
    "dart_model_destroy",
    "dart_model_fork",
    "dart_model_set_precision",
    "dart_model_get_precision",
    "dart_expected_weight_count",
    "dart_backbone",
    "dart_backbone_embed",
    "dart_backbone_blocks",
    "dart_backbone_fpn",
    "dart_encdec",
    "dart_encdec_prefix",
    "dart_encdec_from_prefix",
    "dart_postprocess",
    "dart_model_get_desc",
    "dart_nccl_available",
    "dart_nccl_unique_id",
    "dart_nccl_comm_create",
    "dart_nccl_comm_destroy",
    "dart_nccl_comm_check",
    "dart_nccl_comm_abort",
    "dart_nccl_comm_size",
    "dart_nccl_comm_rank",
    "dart_nccl_all_gather",
    "dart_nccl_all_reduce_max_i32",
    "dart_class_sharded",
    "dart_model_set_mask_head",
    "dart_mask_head",
    "dart_gemm",
    "dart_gemm_plan",
    "dart_gemm_resid_ln",
    "dart_gemm_force_plan",
    "dart_gemm_trace",
    "dart_layernorm",
    "dart_mlp_fused",
    "dart_mlp_fused_ln",
    "dart_gemm_force_splitk",
    "dart_set_pdl",
    "dart_set_ln_fold",
    "dart_attention_kv_split",
    "dart_set_chain",
    "dart_gemm_force_precision",
    "dart_attention_force_safe",
    "dart_attention_trace",
    "dart_attention_variant",
    "dart_attention",
    "dart_attention_qkv",
    "dart_launch_count",
    "dart_reset_launch_count",
    "dart_last_error",
    "dart_version",
)


class NativeError(RuntimeError):
    """A CUDA-side failure reported by the C ABI (DART_ERR_CUDA)."""


class ModelDesc(ctypes.Structure):
    _fields_ = [
        ("image_size", ctypes.c_int32),
        ("patch_size", ctypes.c_int32),
        ("embed_dim", ctypes.c_int32),
        ("num_blocks", ctypes.c_int32),
        ("window_size", ctypes.c_int32),
        ("num_heads", ctypes.c_int32),
        ("fpn_dims", ctypes.c_int32 * 3),
        ("text_tokens", ctypes.c_int32),
        ("text_dim", ctypes.c_int32),
        ("num_queries", ctypes.c_int32),
        ("num_encoder_layers", ctypes.c_int32),
        ("num_decoder_layers", ctypes.c_int32),
        ("block_global", ctypes.c_int32 * MAX_BLOCKS),
        ("attn_enabled", ctypes.c_int32 * MAX_BLOCKS),
        ("mlp_enabled", ctypes.c_int32 * MAX_BLOCKS),
    ]


_lib = None

P = ctypes.c_void_p
I32 = ctypes.c_int32
F64 = ctypes.c_double


class _Unbound:
    """A symbol an older A/B build does not export: its binding is skipped."""

    def __setattr__(self, key, value):
        pass


class _Tolerant:
    """DART_LIB_PATH builds only: tolerate symbols added after that build."""

    def __init__(self, lib):
        object.__setattr__(self, "_lib", lib)

    def __getattr__(self, name):
        try:
            return getattr(self._lib, name)
        except AttributeError:
            return _Unbound()


def load() -> ctypes.CDLL:
    """Open the in-tree library once; raise if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the DART B200 path)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    if os.environ.get("DART_LIB_PATH"):
        lib = _Tolerant(lib)
    lib.dart_model_create.argtypes = [ctypes.POINTER(ModelDesc), ctypes.POINTER(ctypes.c_void_p), I32,
                                      ctypes.POINTER(ctypes.c_void_p)]
    lib.dart_model_create.restype = ctypes.c_int
    lib.dart_model_destroy.argtypes = [P]
    lib.dart_model_destroy.restype = None
    lib.dart_model_fork.argtypes = [P, ctypes.POINTER(ctypes.c_void_p)]
    lib.dart_model_fork.restype = ctypes.c_int
    lib.dart_model_set_precision.argtypes = [P, I32]
    lib.dart_model_set_precision.restype = ctypes.c_int
    lib.dart_model_get_precision.argtypes = [P]
    lib.dart_model_get_precision.restype = I32
    lib.dart_expected_weight_count.argtypes = [ctypes.POINTER(ModelDesc)]
    lib.dart_expected_weight_count.restype = I32
    lib.dart_backbone.argtypes = [P, P, I32, P, P, P, P, P]
    lib.dart_backbone.restype = ctypes.c_int
    lib.dart_backbone_embed.argtypes = [P, P, I32, P, P, P]
    lib.dart_backbone_embed.restype = ctypes.c_int
    lib.dart_backbone_blocks.argtypes = [P, P, I32, I32, I32, P, P, P]
    lib.dart_backbone_blocks.restype = ctypes.c_int
    lib.dart_backbone_fpn.argtypes = [P, P, I32, P, P, P, P, P]
    lib.dart_backbone_fpn.restype = ctypes.c_int
    lib.dart_encdec.argtypes = [P, P, I32, P, I32, P, P, P, P, P]
    lib.dart_encdec.restype = ctypes.c_int
    lib.dart_encdec_prefix.argtypes = [P, P, I32, P, P]
    lib.dart_encdec_prefix.restype = ctypes.c_int
    lib.dart_encdec_from_prefix.argtypes = [P, P, I32, P, I32, P, P, P, P, P]
    lib.dart_encdec_from_prefix.restype = ctypes.c_int
    lib.dart_postprocess.argtypes = [P, P, P, P, I32, I32, F64, F64, F64, I32, P, P, P, P, P, P, P]
    lib.dart_postprocess.restype = ctypes.c_int
    lib.dart_model_get_desc.argtypes = [P]
    lib.dart_model_get_desc.restype = ctypes.POINTER(ModelDesc)
    lib.dart_nccl_available.argtypes = []
    lib.dart_nccl_available.restype = ctypes.c_int
    lib.dart_nccl_unique_id.argtypes = [P]
    lib.dart_nccl_unique_id.restype = ctypes.c_int
    lib.dart_nccl_comm_create.argtypes = [P, I32, I32, ctypes.POINTER(ctypes.c_void_p)]
    lib.dart_nccl_comm_create.restype = ctypes.c_int
    lib.dart_nccl_comm_destroy.argtypes = [P]
    lib.dart_nccl_comm_destroy.restype = None
    lib.dart_nccl_comm_check.argtypes = [P]
    lib.dart_nccl_comm_check.restype = ctypes.c_int
    lib.dart_nccl_comm_abort.argtypes = [P]
    lib.dart_nccl_comm_abort.restype = ctypes.c_int
    lib.dart_nccl_comm_size.argtypes = [P]
    lib.dart_nccl_comm_size.restype = I32
    lib.dart_nccl_comm_rank.argtypes = [P]
    lib.dart_nccl_comm_rank.restype = I32
    lib.dart_nccl_all_gather.argtypes = [P, P, P, ctypes.c_int64, P]
    lib.dart_nccl_all_gather.restype = ctypes.c_int
    lib.dart_nccl_all_reduce_max_i32.argtypes = [P, P, ctypes.c_int64, P]
    lib.dart_nccl_all_reduce_max_i32.restype = ctypes.c_int
    lib.dart_class_sharded.argtypes = [P, P, P, I32, P, I32, P, P, P, P, P]
    lib.dart_class_sharded.restype = ctypes.c_int
    lib.dart_model_set_mask_head.argtypes = [P, P, P, P, P]
    lib.dart_model_set_mask_head.restype = ctypes.c_int
    lib.dart_mask_head.argtypes = [P, P, I32, I32, P, P, P]
    lib.dart_mask_head.restype = ctypes.c_int
    lib.dart_gemm.argtypes = [P, P, P, P, P, I32, I32, I32, I32, P, P, I32, I32, I32, P]
    lib.dart_gemm.restype = ctypes.c_int
    lib.dart_gemm_resid_ln.argtypes = [P, P, P, P, P, P, P, I32, I32, P]
    lib.dart_gemm_resid_ln.restype = ctypes.c_int
    lib.dart_gemm_plan.argtypes = [I32, I32, I32, ctypes.POINTER(I32), ctypes.POINTER(I32)]
    lib.dart_gemm_plan.restype = None
    lib.dart_gemm_force_plan.argtypes = [I32, I32]
    lib.dart_gemm_force_plan.restype = None
    lib.dart_gemm_trace.argtypes = [P]
    lib.dart_gemm_trace.restype = ctypes.c_int
    lib.dart_layernorm.argtypes = [P, P, P, P, I32, I32, I32, P]
    lib.dart_layernorm.restype = ctypes.c_int
    lib.dart_mlp_fused.argtypes = [P, P, P, P, P, P, I32, P]
    lib.dart_mlp_fused.restype = ctypes.c_int
    lib.dart_mlp_fused_ln.argtypes = [P, P, P, P, P, P, P, P, P, I32, P]
    lib.dart_mlp_fused_ln.restype = ctypes.c_int
    lib.dart_gemm_force_splitk.argtypes = [I32]
    lib.dart_gemm_force_splitk.restype = None
    lib.dart_set_pdl.argtypes = [I32]
    lib.dart_set_pdl.restype = None
    lib.dart_set_ln_fold.argtypes = [I32]
    lib.dart_set_ln_fold.restype = None
    lib.dart_attention_kv_split.argtypes = [I32]
    lib.dart_attention_kv_split.restype = None
    lib.dart_set_chain.argtypes = [I32]
    lib.dart_set_chain.restype = None
    lib.dart_gemm_force_precision.argtypes = [I32]
    lib.dart_gemm_force_precision.restype = None
    lib.dart_attention.argtypes = [P, P, P, P, I32, I32, I32, I32, I32, I32, I32, I32, ctypes.c_int64,
                                   ctypes.c_int64, ctypes.c_int64, I32, I32, P]
    lib.dart_attention.restype = ctypes.c_int
    lib.dart_attention_qkv.argtypes = [P, P, I32, I32, I32, I32, P, P]
    lib.dart_attention_qkv.restype = ctypes.c_int
    lib.dart_attention_force_safe.argtypes = [I32]
    lib.dart_attention_force_safe.restype = None
    lib.dart_attention_trace.argtypes = [P]
    lib.dart_attention_trace.restype = None
    lib.dart_attention_variant.argtypes = [I32]
    lib.dart_attention_variant.restype = None
    lib.dart_launch_count.argtypes = [P]
    lib.dart_launch_count.restype = ctypes.c_int64
    lib.dart_reset_launch_count.argtypes = [P]
    lib.dart_reset_launch_count.restype = None
    lib.dart_last_error.argtypes = []
    lib.dart_last_error.restype = ctypes.c_char_p
    lib.dart_version.argtypes = []
    lib.dart_version.restype = ctypes.c_char_p
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if rc == DART_OK:
        return
    msg = load().dart_last_error().decode(errors="replace")
    if rc == DART_ERR_INVALID:
        raise ValueError(msg)
    raise NativeError(msg)
