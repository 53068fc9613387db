"""ctypes loader for libsocket_b200.so -- argument marshalling only.

The library is built in-tree by `paper_2602_06283_b200.build` (or
`__graft_entry__.build()`).  There is no fallback: if the shared library is
missing or fails to load, importing the ops raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SOCKET_LIB_VARIANT") or os.path.join(HERE, "libsocket_b200.so")   # variant: experiments only (tools/variant_build.py)

SOCKET_OK, SOCKET_EINVAL, SOCKET_EUNSUPPORTED, SOCKET_ECUDA, SOCKET_EWORKSPACE = range(5)
GROUP_KV_SHARED, GROUP_PER_QHEAD = 0, 1
OP_HASH, OP_TABLES, OP_SCORE, OP_TOPK, OP_SPARSE_DECODE, OP_DENSE_DECODE, OP_RESOLVE, OP_DECODE_STEP = range(8)
FLAG_CHAINED_STEP = 1
FLAG_ONE_LAUNCH = 2
MAX_SHARDS = 64
TOPK_STATE_WORDS = 8
TOPK_MSG_WORDS = 8 + 2048

# every symbol include/socket_b200.h declares (tests check the export table)
EXPORTS = (
    "socket_code_slots", "socket_codes_bytes", "socket_workspace_bytes", "socket_hash_keys",
    "socket_pack_codes", "socket_unpack_codes", "socket_query_tables", "socket_score",
    "socket_topk", "socket_sparse_decode", "socket_lse_combine", "socket_dense_decode",
    "socket_topk_digest", "socket_topk_bracket", "socket_topk_window", "socket_topk_resolve",
    "socket_topk_emit", "socket_last_error", "socket_version", "socket_build_lut",
    "socket_score_lut", "socket_decode_step", "socket_sample_decode",
    "socket_decode_step_launches",
)


class SocketCfg(ctypes.Structure):
    _fields_ = [
        ("B", ctypes.c_int32), ("H_q", ctypes.c_int32), ("H_kv", ctypes.c_int32),
        ("d", ctypes.c_int32), ("N_max", ctypes.c_int32), ("L", ctypes.c_int32),
        ("P", ctypes.c_int32), ("tau", ctypes.c_float), ("sm_scale", ctypes.c_float),
        ("group_mode", ctypes.c_int32), ("scoring", ctypes.c_int32), ("flags", ctypes.c_int32),
        ("index_base", ctypes.c_int64),
    ]


class SocketError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"socket status {status}: {msg}")
        self.status = status


_lib = None


def lib():
    """Load (once) and return the ctypes handle; raises if the library is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2602_06283_b200.build` "
                          "(the CUDA library is required; there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    i32 = ctypes.c_int32
    cfgp = ctypes.POINTER(SocketCfg)
    sig = {
        "socket_code_slots": (i32, [i32]),
        "socket_codes_bytes": (ctypes.c_size_t, [cfgp]),
        "socket_workspace_bytes": (ctypes.c_size_t, [cfgp, i32, i32]),
        "socket_hash_keys": (i32, [cfgp, P, P, i32, i32, P, P, P, P]),
        "socket_pack_codes": (i32, [cfgp, P, P, P]),
        "socket_unpack_codes": (i32, [cfgp, P, P, P]),
        "socket_query_tables": (i32, [cfgp, P, P, P, P]),
        "socket_score": (i32, [cfgp, P, P, P, P, P, P, P, P, ctypes.c_size_t, P]),
        "socket_topk": (i32, [cfgp, P, P, i32, i32, i32, P, P, P, P, ctypes.c_size_t, P]),
        "socket_sparse_decode": (i32, [cfgp, P, P, P, P, P, i32, P, P, P, P, ctypes.c_size_t, P]),
        "socket_lse_combine": (i32, [cfgp, P, i32, P, P, P]),
        "socket_dense_decode": (i32, [cfgp, P, P, P, P, P, P, P, ctypes.c_size_t, P]),
        "socket_topk_digest": (i32, [cfgp, P, P, i32, i32, i32, i32, i32, P, P, ctypes.c_size_t, P]),
        "socket_topk_bracket": (i32, [cfgp, P, i32, i32, i32, P, P]),
        "socket_topk_window": (i32, [cfgp, P, P, i32, i32, P, P, P, ctypes.c_size_t, P]),
        "socket_topk_resolve": (i32, [cfgp, P, i32, i32, P, P]),
        "socket_topk_emit": (i32, [cfgp, P, P, i32, i32, i32, P, P, P, P, P, ctypes.c_size_t, P]),
        "socket_build_lut": (i32, [cfgp, P, P, P, ctypes.c_size_t, P]),
        "socket_score_lut": (i32, [cfgp, P, P, P, P, P, P, P]),
        "socket_decode_step": (i32, [cfgp, P, P, P, P, P, P, P, P, i32, P, P, i32, i32, i32, P, P,
                                     P, P, P, P, ctypes.c_size_t, P]),
        "socket_sample_decode": (i32, [cfgp, P, P, P, P, P, i32, P, P, P]),
        "socket_decode_step_launches": (i32, [cfgp]),
        "socket_last_error": (ctypes.c_char_p, []),
        "socket_version": (i32, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(status: int):
    if status != SOCKET_OK:
        raise SocketError(status, lib().socket_last_error().decode())
