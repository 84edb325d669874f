"""Loader for the in-tree C-ABI library ``libcard_b200.so``.

The product path has no CPU fallback: if the library (or a GPU) is
missing, every device entry point raises ``DeviceError`` loudly.  The
signatures below are exactly the declarations of include/card_b200.h.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_uint8, c_uint64, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcard_b200.so")

_lib = None


class CacheState(ctypes.Structure):
    _fields_ = [(n, c_int32) for n in (
        "n_nodes", "root", "n_frontier", "epoch", "dead", "status", "vstatus", "stamp",
        "top_layer", "last_width", "compacted", "moved", "K", "k", "max_depth", "eos",
        "capacity", "hash_mask", "fresh", "new_root", "q_hit", "q_len", "chain_len", "alive_below",
        "n_precompact", "r0", "r1", "r2", "r3", "r4", "r5", "r6")]


# name -> (restype, argtypes)
_P = c_void_p
SIGNATURES = {
    "card_abi_version": (c_int, []),
    "card_strerror": (ctypes.c_char_p, [c_int]),
    "card_last_cuda_error": (ctypes.c_char_p, []),
    "card_kgram_dist": (c_int, [c_uint64, c_uint64, c_double, _P, c_int, c_int, c_int, c_int, c_double, c_double, _P,
                                _P]),
    "card_rows_topk": (c_int, [_P, c_int, c_int, c_int, _P, _P, _P, _P, _P]),
    "card_log_cr": (c_int, [_P, _P, c_int, _P]),
    "card_exp_cr": (c_int, [_P, _P, c_int, _P]),
    "card_cache_create": (c_int, [c_int, c_int, c_int, c_int, c_int, c_int, POINTER(c_void_p)]),
    "card_cache_destroy": (c_int, [_P]),
    "card_cache_reset": (c_int, [_P, _P, c_int, _P]),
    "card_cache_clear": (c_int, [_P, c_int, _P]),
    "card_cache_expand": (c_int, [_P, _P, c_int, c_int, _P]),
    "card_cache_expand_topk": (c_int, [_P, _P, _P, _P, c_int, c_int, _P, _P]),
    "card_cache_pool": (c_int, [_P, _P, c_int, c_int, _P, _P, _P, _P, _P]),
    "card_cache_query": (c_int, [_P, c_int, _P]),
    "card_cache_query_if": (c_int, [_P, c_int, _P, _P]),
    "card_mailbox_create": (c_int, [c_int, c_int, POINTER(c_void_p)]),
    "card_mailbox_destroy": (c_int, [_P]),
    "card_mailbox_reset": (c_int, [_P]),
    "card_mailbox_skip_flag": (c_int, [_P, POINTER(c_void_p)]),
    "card_mailbox_query_view": (c_int, [_P, POINTER(c_void_p), POINTER(c_void_p)]),
    "card_mailbox_poll_commit": (c_int, [_P, _P, _P]),
    "card_mailbox_publish_query": (c_int, [_P, _P, c_int, _P]),
    "card_mailbox_wait_query": (c_int, [_P, _P]),
    "card_mailbox_publish_commit": (c_int, [_P, _P, _P]),
    "card_target_rows_view": (c_int, [_P, _P, _P, _P, _P, c_int, c_int, _P, c_int, _P, _P]),
    "card_cache_query_buffers": (c_int, [_P, POINTER(c_void_p), POINTER(c_void_p), POINTER(c_void_p)]),
    "card_cache_correct": (c_int, [_P, _P, _P, _P, _P, _P]),
    "card_cache_advance_root": (c_int, [_P, _P, _P, _P, _P]),
    "card_cache_count_alive": (c_int, [_P, _P]),
    "card_cache_clear_status": (c_int, [_P, _P]),
    "card_cache_read_state": (c_int, [_P, POINTER(CacheState), _P]),
    "card_cache_snapshot": (c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "card_cache_device_ptrs": (c_int, [_P] + [POINTER(c_void_p)] * 8),
    # model plug-in
    "card_linear_create": (c_int, [_P, c_int, c_int, c_int, _P, c_int, c_int, _P, c_int, _P, POINTER(c_void_p)]),
    "card_linear_run": (c_int, [_P, _P, _P]),
    "card_linear_info": (c_int, [_P, _P]),
    "card_linear_trace": (c_int, [_P, _P]),
    "card_linear_fuse_norm": (c_int, [_P, _P, c_int, c_int, ctypes.c_float, c_int, _P]),
    "card_linear_fuse_resid": (c_int, [_P, _P, c_int, _P]),
    "card_linear_fuse_rope": (c_int, [_P, _P, _P, _P, _P, c_int, c_int, c_int, _P, _P, _P]),
    "card_linear_fuse_kgram": (c_int, [_P, _P, c_int, c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_float,
                                       ctypes.c_float]),
    "card_linear_fuse_topk": (c_int, [_P, c_int, ctypes.c_float]),
    "card_lmhead_topk_merge": (c_int, [_P, _P, c_int, c_int, c_int, c_int, _P, _P, _P, _P]),
    "card_linear_destroy": (c_int, [_P]),
    "card_pfwd_create": (c_int, [c_int, c_int, c_int, c_int, c_int, c_int, c_int, _P, _P, _P, _P, _P, _P, c_int, _P,
                                 _P, _P, c_int, _P, _P, _P, _P, ctypes.c_float, POINTER(c_void_p)]),
    "card_pfwd_run": (c_int, [_P, _P, c_int, c_int, _P]),
    "card_pfwd_info": (c_int, [_P, _P]),
    "card_pfwd_bind": (c_int, [_P, _P, _P]),
    "card_pfwd_set_qsw": (c_int, [_P, _P, c_int]),
    "card_pfwd_set_grid": (c_int, [_P, c_int]),
    "card_green_create": (c_int, [c_int, c_int, POINTER(c_void_p)]),
    "card_green_stream": (c_int, [_P, c_int, POINTER(c_void_p), POINTER(c_int)]),
    "card_green_destroy": (c_int, [_P]),
    "card_pfwd_trace": (c_int, [_P, _P]),
    "card_pfwd_tune": (c_int, [_P, c_int, c_int]),
    "card_pfwd_destroy": (c_int, [_P]),
    "card_embed": (c_int, [_P, _P, c_int, _P, c_int, c_int, _P, _P, _P, c_int, _P]),
    "card_gather_rows": (c_int, [_P, _P, c_int, c_int, _P, _P, c_int, _P, _P, c_int, _P]),
    "card_resid_add": (c_int, [_P, c_int, c_int, _P, _P, _P, _P, c_int, _P]),
    "card_rmsnorm": (c_int, [_P, _P, c_int, ctypes.c_float, _P, c_int, _P, _P, c_int, _P]),
    "card_rope_kv": (c_int, [_P, _P, c_int, _P, _P, _P, _P, c_int, c_int, c_int, _P, _P, _P, c_int, _P]),
    "card_attention_work_floats": (c_int, [c_int, c_int, c_int, c_int]),
    "card_attention_trace": (c_int, [_P]),
    "card_attention": (c_int, [_P, _P, c_int, _P, _P, _P, _P, c_int, _P, _P, c_int, c_int, c_int, c_int, c_int, _P,
                               _P, c_int, _P]),
    "card_attention_paged": (c_int, [_P, _P, c_int, _P, _P, _P, c_int, _P, _P, _P, c_int, c_int, c_int, c_int, _P,
                                     _P]),
    "card_attention_batch": (c_int, [_P, _P, c_int, _P, c_int, _P, _P, _P, c_int, _P, _P, _P, c_int, c_int, c_int,
                                     c_int, c_int, c_int, _P, _P]),
    "card_attention_tree": (c_int, [_P, c_int, _P, c_int, _P, _P, _P, c_int, _P, _P, _P, c_int, c_int, c_int, c_int,
                                    _P, _P]),
    "card_lmhead_work_floats": (c_int, [c_int, c_int]),
    "card_topk_logits": (c_int, [_P, _P, c_int, c_int, c_int, c_double, _P, _P, _P, _P, _P, c_int, c_int, c_uint64,
                                 c_uint64, ctypes.c_float, ctypes.c_float, _P]),
    "card_argmax_logits": (c_int, [_P, _P, c_int, c_int, _P, _P, _P, c_int, c_int, c_uint64, c_uint64, ctypes.c_float,
                                   ctypes.c_float, _P]),
    "card_softmax64": (c_int, [_P, _P, c_int, c_int, c_double, _P, _P]),
    "card_logit_bias": (c_int, [_P, _P, c_int, c_int, _P, c_int, c_int, c_uint64, c_uint64, ctypes.c_float,
                                ctypes.c_float, _P]),
    # engine
    "card_engine_state_bytes": (c_int, []),
    "card_draft_rows": (c_int, [_P, _P, _P, _P, c_int, c_int, c_int, _P, c_int, _P, _P]),
    "card_target_rows": (c_int, [_P, _P, _P, _P, c_int, c_int, _P, c_int, _P, _P]),
    "card_draft_rows_at": (c_int, [_P, _P, _P, _P, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, _P, c_int,
                                   _P, _P]),
    "card_target_rows_at": (c_int, [_P, _P, _P, _P, c_int, c_int, c_int, c_int, c_int, _P, c_int, _P, _P]),
    "card_eos_fix": (c_int, [_P, c_int, _P, c_int, c_int, c_int, _P, _P]),
    "card_record_width": (c_int, [_P, _P, _P, _P]),
    "card_verify_argmax": (c_int, [_P, _P, _P, _P]),
    "card_verify_probs": (c_int, [_P, _P, _P, c_int, _P, _P, _P]),
    "card_commit": (c_int, [_P, _P, _P]),
    "card_verify_result": (c_int, [_P, _P, _P]),
    "card_draft_promote": (c_int, [_P, _P, _P, _P, c_int, c_int, c_int, c_int, c_int, _P, _P]),
    "card_kv_compact": (c_int, [_P, _P, _P, _P, c_int, c_int, c_int, c_int, _P, c_int, _P]),
    "card_cycle_end": (c_int, [_P, _P, _P]),
    "card_engine_handoff": (c_int, [_P, _P, _P]),
    "card_enable_peer_access": (c_int, [c_int, c_int]),
}


class EngineState(ctypes.Structure):
    """Host mirror of card_engine_state (csrc/card_engine.cu)."""
    _fields_ = [(n, c_int32) for n in (
        "C", "Pd", "out_len", "done", "max_new", "eos", "stop", "n_widths", "hit", "L", "n_acc", "corr",
        "rec_acc", "rec_lnew", "cursor", "n_uni", "base_len", "C_prev", "order", "sampling",
        "rec_n_widths", "rec_hit", "rec_L", "rec_n_acc", "rec_corr", "rec_done", "n_commit", "anchor_origin")] + [
        ("widths", c_int32 * 64), ("rec_widths", c_int32 * 64), ("acc", c_int32 * 64),
        ("committed_now", c_int32 * 72), ("rec_depth", c_int32), ("rec_alive", c_int32), ("kv_keep", c_int32), ("kv_drop", c_int32),
        ("consumed", c_int32), ("cursor_prev", c_int32), ("spare", c_int32 * 2)]


# kernels launched per C-ABI call (for the bench's gpu_launches count)
LAUNCHES = {
    "card_kgram_dist": 1, "card_rows_topk": 1, "card_log_cr": 1, "card_exp_cr": 1,
    "card_cache_reset": 2, "card_cache_clear": 3, "card_cache_expand": 2, "card_cache_expand_topk": 1, "card_cache_pool": 2,
    "card_cache_query": 1, "card_cache_correct": 1, "card_cache_advance_root": 1, "card_cache_count_alive": 1,
    "card_cache_clear_status": 1, "card_embed": 1, "card_resid_add": 1, "card_rmsnorm": 1, "card_rope_kv": 1, "card_attention": lambda a: 1 if (a[10] == 0 and a[17] == 0 and a[13] in (64, 128) and a[4] and _attn_fits(a)) else 3,
    "card_topk_logits": 2, "card_lmhead_topk_merge": 1, "card_argmax_logits": 2, "card_softmax64": 1, "card_logit_bias": 1,
    "card_draft_rows": 1, "card_target_rows": 1, "card_draft_rows_at": 1, "card_target_rows_at": 1, "card_eos_fix": 1, "card_record_width": 1,
    "card_attention_paged": 1, "card_verify_argmax": 1, "card_verify_probs": 1, "card_commit": 1, "card_verify_result": 1, "card_draft_promote": 2,
    "card_kv_compact": 2, "card_cycle_end": 1, "card_engine_handoff": 1, "card_pfwd_run": 1, "card_attention_tree": 1,
    "card_attention_batch": 1, "card_gather_rows": 1, "card_cache_query_if": 1, "card_mailbox_poll_commit": 1,
    "card_mailbox_publish_query": 1, "card_mailbox_wait_query": 1, "card_mailbox_publish_commit": 1,
    "card_target_rows_view": 1,
}
launch_count = [0]


def _attn_fits(a) -> bool:
    """Mirror of attn_tc_fits / attn_fused_fits (card_attn_tc.cu, card_attn.cu):
    the one-launch kernels gather at most 1024 extra slots per query tile."""
    m_max, nh, nkv, extra_max, hd = a[2], a[11], a[12], a[7], a[13]
    G = nh // nkv
    rows_tc = 128 // G + 2
    if m_max * G >= 256 and hd in (64, 128) and rows_tc <= 136 and rows_tc * extra_max <= 1024:
        return True
    qt = 128 if m_max * G >= 512 else 64
    rows = qt // G + 2
    return rows <= 136 and rows * extra_max <= 1024


class _Counted:
    """Proxy over the CDLL that tallies kernel launches per call."""

    def __init__(self, handle):
        self._h = handle

    def __getattr__(self, name):
        fn = getattr(self._h, name)
        n = LAUNCHES.get(name)
        if not n:
            return fn

        def call(*args):
            launch_count[0] += n(args) if callable(n) else n
            return fn(*args)

        return call


def lib():
    """Load (once) and return the ctypes handle; raises DeviceError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    from .errors import DeviceError

    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (no CPU fallback exists)")
    handle = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    if handle.card_engine_state_bytes() != ctypes.sizeof(EngineState):
        raise DeviceError("EngineState layout does not match the library")
    _lib = _Counted(handle)
    return _lib


def raw():
    """The underlying CDLL (symbol introspection)."""
    lib()
    return _lib._h


def exported_symbols() -> list[str]:
    return list(SIGNATURES)
