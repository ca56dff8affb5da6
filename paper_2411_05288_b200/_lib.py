"""ctypes binding of the C ABI in include/vpipe_b200.h (libvpipe_b200.so).

The shared library is built in-tree (paper_2411_05288_b200/lib/) by
`build.build()`; there is no fallback: importing the product path on a box
without the library raises immediately.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_void_p

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
# VPIPE_LIB: an alternative build of the same library (developer A/B of
# compile-time kernel variants, tools/build_variant.sh)
LIB_PATH = os.environ.get("VPIPE_LIB") or os.path.join(LIB_DIR, "libvpipe_b200.so")

VP_OK, VP_EINVAL, VP_ECUDA, VP_ENCCL, VP_EINTERNAL = 0, 1, 2, 3, 4


class vp_shard_t(ctypes.Structure):
    _fields_ = [("W", c_void_p), ("ldw", c_int64), ("row_begin", c_int64), ("row_end", c_int64), ("index", c_int32)]


class vp_batch_t(ctypes.Structure):
    _fields_ = [("X", c_void_p), ("ldx", c_int64), ("labels", c_void_p), ("n_tok", c_int64), ("h", c_int64)]


class vp_stats_t(ctypes.Structure):
    _fields_ = [("m", c_void_p), ("sum", c_void_p)]


# name -> (restype, argtypes); every symbol declared in include/vpipe_b200.h
SIGNATURES = {
    "vp_abi_version": (c_int, []),
    "vp_last_error": (c_char_p, []),
    "vp_ctx_create": (c_int, [c_int, POINTER(c_void_p)]),
    "vp_ctx_destroy": (c_int, [c_void_p]),
    "vp_ctx_set_stream": (c_int, [c_void_p, c_void_p]),
    "vp_ctx_get_stream": (c_void_p, [c_void_p]),
    "vp_ctx_sync": (c_int, [c_void_p]),
    "vp_ctx_reserve": (c_int, [c_void_p, c_int64, c_int64, c_int]),
    "vp_ctx_set_option": (c_int, [c_void_p, c_char_p, c_int64]),
    "vp_ctx_launch_count": (c_int64, [c_void_p]),
    "vp_ctx_fused_c1_count": (c_int64, [c_void_p]),
    "vp_ctx_peer_input_count": (c_int64, [c_void_p]),
    "vp_workspace_query": (c_int, [c_int64, c_int64, c_int64, c_int, POINTER(c_int64), POINTER(c_int64),
                                   POINTER(c_int64)]),
    "vp_debug_occupy_sms": (c_int, [c_void_p, c_void_p, c_int, c_int64]),
    "vp_ctx_set_logit_shift": (c_int, [c_void_p, c_void_p]),
    "vp_shard_logits": (c_int, [c_void_p, POINTER(vp_batch_t), POINTER(vp_shard_t), c_void_p, c_int64]),
    "vp_shard_label_rows": (c_int, [c_void_p, POINTER(vp_batch_t), POINTER(vp_shard_t), c_void_p, c_int64]),
    "vp_ctx_gemm_timing": (c_int, [c_void_p, c_int, POINTER(ctypes.c_double), POINTER(c_int64)]),
    "vp_comm_unique_id": (c_int, [c_void_p]),
    "vp_comm_loopback_id": (c_int, [c_void_p]),
    "vp_ctx_comm_init": (c_int, [c_void_p, c_int, c_int, c_void_p]),
    "vp_comm_init_all": (c_int, [POINTER(c_void_p), c_int]),
    "vp_ctx_comm_backend": (c_char_p, [c_void_p]),
    "vp_ctx_comm_info": (c_int, [c_void_p, POINTER(c_int), POINTER(c_int)]),
    "vp_state_create": (c_int, [c_void_p, c_int64, c_int64, c_int64, POINTER(c_void_p)]),
    "vp_state_destroy": (c_int, [c_void_p]),
    "vp_state_local_stats": (c_int, [c_void_p, POINTER(c_void_p), POINTER(c_void_p)]),
    "vp_state_grad_terms": (c_int, [c_void_p, POINTER(c_void_p), POINTER(c_int64)]),
    "vp_state_copy_local_stats": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "vp_state_copy_grad_terms": (c_int, [c_void_p, c_void_p, c_void_p, c_int64]),
    "vp_alg1_pass_S": (c_int, [c_void_p, POINTER(vp_batch_t), POINTER(vp_shard_t), c_void_p]),
    "vp_alg2_pass_S": (c_int, [c_void_p, POINTER(vp_batch_t), POINTER(vp_shard_t), c_void_p]),
    "vp_merge_max_sum": (c_int, [c_void_p, POINTER(c_void_p), c_int, c_double, vp_stats_t]),
    "vp_merge_stats_raw": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int64, c_int64, c_double, vp_stats_t]),
    "vp_alg1_pass_T": (c_int, [c_void_p, c_void_p, vp_stats_t, POINTER(vp_batch_t), POINTER(vp_shard_t),
                               c_void_p, c_int64, c_void_p, c_int64]),
    "vp_reduce_grad_x": (c_int, [c_void_p, POINTER(c_void_p), c_int, c_int64, c_int64, c_int64, c_void_p, c_int64]),
    "vp_alg2_barrier_C1": (c_int, [c_void_p, POINTER(c_void_p), POINTER(vp_shard_t), c_int, POINTER(vp_batch_t),
                                   c_double, vp_stats_t, c_void_p, c_int64]),
    "vp_alg2_pass_T": (c_int, [c_void_p, c_void_p, vp_stats_t, POINTER(vp_batch_t), POINTER(vp_shard_t),
                               c_void_p, c_int64]),
    "vp_output_loss": (c_int, [c_void_p, POINTER(c_void_p), POINTER(vp_shard_t), c_int, vp_stats_t,
                               POINTER(vp_batch_t), c_void_p]),
    "vp_shard_softmax": (c_int, [c_void_p, c_void_p, vp_stats_t, c_void_p, c_int64]),
    "vp_naive_partitioned_output": (c_int, [c_void_p, POINTER(vp_batch_t), POINTER(vp_shard_t), POINTER(c_void_p),
                                            c_int, vp_stats_t, c_void_p, c_void_p, c_int64, POINTER(c_void_p),
                                            c_int64]),
    "vp_run_alg1": (c_int, [c_void_p, POINTER(vp_batch_t), POINTER(vp_shard_t), POINTER(c_void_p), c_int, c_double,
                            vp_stats_t, c_void_p, c_void_p, c_int64, POINTER(c_void_p), c_int64]),
    "vp_run_alg2": (c_int, [c_void_p, POINTER(vp_batch_t), POINTER(vp_shard_t), POINTER(c_void_p), c_int, c_double,
                            vp_stats_t, c_void_p, c_void_p, c_int64, POINTER(c_void_p), c_int64]),
    "vp_run_alg2_chunked": (c_int, [c_void_p, POINTER(vp_batch_t), POINTER(vp_shard_t), POINTER(c_void_p), c_int,
                                    c_int64, c_double, vp_stats_t, c_void_p, c_void_p, c_int64, POINTER(c_void_p),
                                    c_int64]),
    "vp_input_forward": (c_int, [c_void_p, c_void_p, c_int64, c_int64, POINTER(vp_shard_t), c_void_p, c_int64,
                                 c_int]),
    "vp_input_forward_gathered": (c_int, [c_void_p, c_void_p, c_int64, c_int64, POINTER(vp_shard_t), c_void_p,
                                          c_int64]),
    "vp_input_grad_broadcast": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int64, c_int64, c_int]),
    "vp_input_backward_gathered": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_void_p, c_int64, c_int64, c_void_p,
                                           c_void_p, c_int64, c_int, c_int]),
    "vp_input_backward": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_void_p, c_int64, c_int64,
                                  POINTER(vp_shard_t), c_void_p, c_int64, c_int]),
    "vp_allreduce_sum": (c_int, [c_void_p, c_void_p, c_int64, c_int]),
    "vp_program_parse": (c_int, [c_char_p, POINTER(c_void_p)]),
    "vp_program_destroy": (c_int, [c_void_p]),
    "vp_program_info": (c_int, [c_void_p, POINTER(c_int), POINTER(c_int), POINTER(c_int)]),
    "vp_program_validate": (c_int, [c_void_p, c_char_p, c_int64, POINTER(c_int)]),
    "vp_program_run": (c_int, [c_void_p, c_void_p, POINTER(vp_batch_t), POINTER(vp_shard_t), c_int,
                               POINTER(c_void_p), POINTER(vp_stats_t), POINTER(c_void_p), POINTER(c_void_p), c_int64,
                               POINTER(c_void_p), c_int64]),
    "vp_ctx_capture_begin": (c_int, [c_void_p]),
    "vp_ctx_capture_end": (c_int, [c_void_p, POINTER(c_void_p)]),
    "vp_graph_launch": (c_int, [c_void_p, c_void_p]),
    "vp_graph_destroy": (c_int, [c_void_p]),
}


class VpError(RuntimeError):
    """Non-EINVAL failure (CUDA, NCCL, internal)."""


_LIB = None


def load() -> ctypes.CDLL:
    """Load libvpipe_b200.so (once).  Raises if it has not been built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the product path)")
    # libvpipe_b200.so needs libnccl.so.2.  torch bundles a newer NCCL under
    # the same soname; whichever loads first wins process-wide, and torch
    # needs its own, so let torch load it first (ours is ABI-compatible).
    try:
        import torch  # noqa: F401
    except ImportError:
        pass
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        if os.environ.get("VPIPE_LIB") and not hasattr(lib, name):
            continue  # an older developer build under A/B lacks a newer entry point
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def check(rc: int) -> None:
    """Map a vp_* return code to the reference's exception types."""
    if rc == VP_OK:
        return
    msg = (load().vp_last_error() or b"").decode()
    if rc == VP_EINVAL:
        raise ValueError(msg)  # std::invalid_argument in the reference
    raise VpError(f"vp error {rc}: {msg}")
