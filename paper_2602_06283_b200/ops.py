"""Thin torch-facing wrappers over the C ABI (include/socket_b200.h).

Marshalling only: each function validates tensor dtypes/shapes/devices,
allocates outputs and workspaces with torch (PyTorch = device memory and
streams), and calls the library on the current CUDA stream.  Every step of
the SOCKET path runs in the library's sm_100a kernels.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import SocketCfg, check, lib

KV_SHARED = _lib.GROUP_KV_SHARED
PER_QHEAD = _lib.GROUP_PER_QHEAD


@dataclass(frozen=True)
class Config:
    """Mirror of socket_cfg (see include/socket_b200.h)."""
    B: int
    H_q: int
    H_kv: int
    N_max: int
    L: int = 60            # Table 6 default
    P: int = 8
    tau: float = 0.5
    sm_scale: float | None = None   # default 1/sqrt(d) (reading R-2)
    group_mode: int = KV_SHARED
    d: int = 128
    scoring: int = 0       # SOCKET_SCORING_SOFT (Eq. 4); 1 = hard LSH collision counts (Eq. 3)
    flags: int = 0         # SOCKET_FLAG_* (1 = chained decode step; 2 = one-launch step whenever it applies)
    index_base: int = 0    # global position of local key 0 (sequence shards)

    def c(self) -> SocketCfg:
        s = self.sm_scale if self.sm_scale is not None else 1.0 / math.sqrt(self.d)
        return SocketCfg(self.B, self.H_q, self.H_kv, self.d, self.N_max, self.L, self.P,
                         float(self.tau), float(s), int(self.group_mode), int(self.scoring),
                         int(self.flags), int(self.index_base))

    @property
    def H_sel(self) -> int:
        return self.H_q if self.group_mode == PER_QHEAD else self.H_kv

    @property
    def code_slots(self) -> int:
        return int(lib().socket_code_slots(self.L))

    @property
    def scale(self) -> float:
        return self.sm_scale if self.sm_scale is not None else 1.0 / math.sqrt(self.d)


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(t):
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _need(t, dtype, shape, name):
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{name}: must be a contiguous CUDA tensor")


def _need_uva(t, dtype, shape, name):
    """Like _need, but a pinned (UVA-mapped) host tensor is accepted too: the
    decode step may read its inputs / write its output in host memory."""
    if t.is_cuda:
        return _need(t, dtype, shape, name)
    if t.dtype != dtype or tuple(t.shape) != tuple(shape) or not t.is_contiguous() or not t.is_pinned():
        raise ValueError(f"{name}: expected a contiguous {dtype} {tuple(shape)} CUDA or pinned host tensor")


def workspace_bytes(cfg: Config, op: int, k: int = 1) -> int:
    c = cfg.c()
    return int(lib().socket_workspace_bytes(ctypes.byref(c), op, k))


def workspace(cfg: Config, op: int, k: int, device) -> torch.Tensor:
    """Zero-filled: the decode step's row-spread control words must start at zero
    (include/socket_b200.h, socket_decode_step)."""
    n = max(16, workspace_bytes(cfg, op, k))
    return torch.zeros(n, dtype=torch.uint8, device=device)


def codes_bytes(cfg: Config) -> int:
    c = cfg.c()
    return int(lib().socket_codes_bytes(ctypes.byref(c)))


def alloc_codes(cfg: Config, device) -> torch.Tensor:
    return torch.zeros(codes_bytes(cfg), dtype=torch.uint8, device=device)


# ---------------------------------------------------------------------------
def hash_keys(cfg: Config, K, W, codes, V=None, vnorm=None, n_begin: int = 0, n_count=None):
    """Alg. 1 on rows [n_begin, n_begin+n_count) of every (b, kv head)."""
    n_count = cfg.N_max - n_begin if n_count is None else n_count
    _need(K, torch.bfloat16, (cfg.B, cfg.H_kv, cfg.N_max, cfg.d), "K")
    _need(W, torch.bfloat16, (cfg.L, cfg.P, cfg.d), "W")
    _need(codes, torch.uint8, (codes_bytes(cfg),), "codes")
    if V is not None:
        _need(V, torch.bfloat16, K.shape, "V")
        _need(vnorm, torch.float32, (cfg.B, cfg.H_kv, cfg.N_max), "vnorm")
    c = cfg.c()
    check(lib().socket_hash_keys(ctypes.byref(c), _p(K), _p(V), n_begin, n_count, _p(W),
                                 _p(codes), _p(vnorm), _stream(K)))
    return codes


def plain_code_dtype(cfg: Config):
    """Element type of plain [B][H_kv][L][N_max] codes: uint8 for P <= 8, 16-bit
    (int16 holding the uint16 bit pattern) for P > 8."""
    return torch.uint8 if cfg.P <= 8 else torch.int16


def pack_codes(cfg: Config, plain):
    _need(plain, plain_code_dtype(cfg), (cfg.B, cfg.H_kv, cfg.L, cfg.N_max), "plain codes")
    codes = alloc_codes(cfg, plain.device)
    c = cfg.c()
    check(lib().socket_pack_codes(ctypes.byref(c), _p(plain), _p(codes), _stream(plain)))
    return codes


def unpack_codes(cfg: Config, codes):
    _need(codes, torch.uint8, (codes_bytes(cfg),), "codes")
    plain = torch.zeros((cfg.B, cfg.H_kv, cfg.L, cfg.N_max), dtype=plain_code_dtype(cfg),
                        device=codes.device)
    c = cfg.c()
    check(lib().socket_unpack_codes(ctypes.byref(c), _p(codes), _p(plain), _stream(codes)))
    return plain


def query_tables(cfg: Config, q, W):
    """Alg. 2 tables [B][H_sel][L][2^P] (group-summed in KV_SHARED mode)."""
    _need(q, torch.bfloat16, (cfg.B, cfg.H_q, cfg.d), "q")
    _need(W, torch.bfloat16, (cfg.L, cfg.P, cfg.d), "W")
    t = torch.empty((cfg.B, cfg.H_sel, cfg.L, 1 << cfg.P), dtype=torch.float32, device=q.device)
    c = cfg.c()
    check(lib().socket_query_tables(ctypes.byref(c), _p(q), _p(W), _p(t), _stream(q)))
    return t


def _need_index(cfg: Config, codes, vnorm, seq_lens, mask=None):
    _need(codes, torch.uint8, (codes_bytes(cfg),), "codes")
    _need(vnorm, torch.float32, (cfg.B, cfg.H_kv, cfg.N_max), "vnorm")
    _need(seq_lens, torch.int32, (cfg.B,), "seq_lens")
    if mask is not None:
        _need(mask, torch.uint8, (cfg.B, cfg.N_max), "mask")


def _need_ws(ws, cfg: Config, op: int, k: int, name="ws"):
    if not ws.is_cuda or ws.dtype != torch.uint8 or ws.numel() < workspace_bytes(cfg, op, k):
        raise ValueError(f"{name}: expected a CUDA uint8 buffer of >= {workspace_bytes(cfg, op, k)} bytes")


def _need_kv(cfg: Config, K, V):
    _need(K, torch.bfloat16, (cfg.B, cfg.H_kv, cfg.N_max, cfg.d), "K")
    _need(V, torch.bfloat16, (cfg.B, cfg.H_kv, cfg.N_max, cfg.d), "V")


def score(cfg: Config, q, W, codes, vnorm, seq_lens, mask=None, out=None, ws=None):
    """Eq. 4 + Alg. 4 scores [B][H_sel][N_max] (fp32, -inf for invalid keys)."""
    _need(q, torch.bfloat16, (cfg.B, cfg.H_q, cfg.d), "q")
    _need(W, torch.bfloat16, (cfg.L, cfg.P, cfg.d), "W")
    _need_index(cfg, codes, vnorm, seq_lens, mask)
    if out is None:
        out = torch.empty((cfg.B, cfg.H_sel, cfg.N_max), dtype=torch.float32, device=q.device)
    _need(out, torch.float32, (cfg.B, cfg.H_sel, cfg.N_max), "scores")
    if ws is None:
        ws = workspace(cfg, _lib.OP_SCORE, 1, q.device)
    _need_ws(ws, cfg, _lib.OP_SCORE, 1)
    c = cfg.c()
    check(lib().socket_score(ctypes.byref(c), _p(q), _p(W), _p(codes), _p(vnorm), _p(seq_lens),
                             _p(mask), _p(out), _p(ws), ws.numel(), _stream(q)))
    return out


def build_lut(cfg: Config, q, W, lut=None):
    """Alg. 2 tables as the score kernel's shared-memory image (opaque buffer)."""
    _need(q, torch.bfloat16, (cfg.B, cfg.H_q, cfg.d), "q")
    _need(W, torch.bfloat16, (cfg.L, cfg.P, cfg.d), "W")
    if lut is None:
        lut = workspace(cfg, _lib.OP_SCORE, 1, q.device)
    _need_ws(lut, cfg, _lib.OP_SCORE, 1, "lut")
    c = cfg.c()
    check(lib().socket_build_lut(ctypes.byref(c), _p(q), _p(W), _p(lut), lut.numel(), _stream(q)))
    return lut


def score_lut(cfg: Config, lut, codes, vnorm, seq_lens, mask=None, out=None):
    """Eq. 4 + Alg. 4 scores from a LUT built by build_lut."""
    _need_ws(lut, cfg, _lib.OP_SCORE, 1, "lut")
    _need_index(cfg, codes, vnorm, seq_lens, mask)
    if out is None:
        out = torch.empty((cfg.B, cfg.H_sel, cfg.N_max), dtype=torch.float32, device=lut.device)
    _need(out, torch.float32, (cfg.B, cfg.H_sel, cfg.N_max), "scores")
    c = cfg.c()
    check(lib().socket_score_lut(ctypes.byref(c), _p(lut), _p(codes), _p(vnorm), _p(seq_lens),
                                 _p(mask), _p(out), _stream(lut)))
    return out


def decode_step(cfg: Config, q, K, V, W, codes, vnorm, seq_lens, k: int, append: bool = True,
                sink: int = 0, window: int = 0, mask=None, scores=None, idx=None, cnt=None,
                out=None, lse=None, ws=None, k_new=None, v_new=None):
    """One fused decode step (append-hash of key seq_lens[b]-1, tables, scores,
    top-k, sparse decode) -- socket_decode_step.  With k_new / v_new
    ([B][H_kv][d] bf16) the step also stores the new token's rows into K / V."""
    _need_uva(q, torch.bfloat16, (cfg.B, cfg.H_q, cfg.d), "q")
    if k_new is not None:
        _need_uva(k_new, torch.bfloat16, (cfg.B, cfg.H_kv, cfg.d), "k_new")
        _need_uva(v_new, torch.bfloat16, (cfg.B, cfg.H_kv, cfg.d), "v_new")
    _need_kv(cfg, K, V)
    _need(W, torch.bfloat16, (cfg.L, cfg.P, cfg.d), "W")
    _need_index(cfg, codes, vnorm, seq_lens, mask)
    dev = K.device
    if scores is None:
        scores = torch.empty((cfg.B, cfg.H_sel, cfg.N_max), dtype=torch.float32, device=dev)
    if idx is None:
        idx = torch.empty((cfg.B, cfg.H_sel, k), dtype=torch.int32, device=dev)
    if cnt is None:
        cnt = torch.empty((cfg.B, cfg.H_sel), dtype=torch.int32, device=dev)
    if out is None:
        out = torch.empty((cfg.B, cfg.H_q, cfg.d), dtype=torch.bfloat16, device=dev)
    if lse is None:
        lse = torch.empty((cfg.B, cfg.H_q), dtype=torch.float32, device=dev)
    if ws is None:
        ws = workspace(cfg, _lib.OP_DECODE_STEP, k, dev)
    _need(scores, torch.float32, (cfg.B, cfg.H_sel, cfg.N_max), "scores")
    _need(idx, torch.int32, (cfg.B, cfg.H_sel, k), "idx")
    _need(cnt, torch.int32, (cfg.B, cfg.H_sel), "cnt")
    _need_uva(out, torch.bfloat16, (cfg.B, cfg.H_q, cfg.d), "out")
    _need(lse, torch.float32, (cfg.B, cfg.H_q), "lse")
    _need_ws(ws, cfg, _lib.OP_DECODE_STEP, k)
    c = cfg.c()
    check(lib().socket_decode_step(ctypes.byref(c), _p(q), _p(K), _p(V), _p(W), _p(codes), _p(vnorm),
                                   _p(seq_lens), _p(mask), int(bool(append)), _p(k_new), _p(v_new),
                                   k, sink, window,
                                   _p(scores), _p(idx), _p(cnt), _p(out), _p(lse), _p(ws),
                                   ws.numel(), _stream(K)))
    return out, lse


def decode_step_launches(cfg: Config) -> int:
    """Kernel launches of one socket_decode_step for cfg (1 = the one-launch cluster kernel)."""
    c = cfg.c()
    return int(lib().socket_decode_step_launches(ctypes.byref(c)))


def topk(cfg: Config, scores, seq_lens, k: int, sink: int = 0, window: int = 0,
         idx=None, cnt=None, sel_scores=None, want_scores: bool = False, ws=None):
    """Alg. 3 l.244 TopK: idx [B][H_sel][k] ascending (-1 past cnt), cnt [B][H_sel].
    Rows longer than 655360 keys keep their key slices in `ws`."""
    _need(scores, torch.float32, (cfg.B, cfg.H_sel, cfg.N_max), "scores")
    _need(seq_lens, torch.int32, (cfg.B,), "seq_lens")
    dev = scores.device
    if idx is None:
        idx = torch.empty((cfg.B, cfg.H_sel, k), dtype=torch.int32, device=dev)
    if cnt is None:
        cnt = torch.empty((cfg.B, cfg.H_sel), dtype=torch.int32, device=dev)
    if want_scores and sel_scores is None:
        sel_scores = torch.empty((cfg.B, cfg.H_sel, k), dtype=torch.float32, device=dev)
    _need(idx, torch.int32, (cfg.B, cfg.H_sel, k), "idx")
    _need(cnt, torch.int32, (cfg.B, cfg.H_sel), "cnt")
    if sel_scores is not None:
        _need(sel_scores, torch.float32, (cfg.B, cfg.H_sel, k), "sel_scores")
    if ws is None and workspace_bytes(cfg, _lib.OP_TOPK, k) > 0:
        ws = workspace(cfg, _lib.OP_TOPK, k, dev)
    c = cfg.c()
    check(lib().socket_topk(ctypes.byref(c), _p(scores), _p(seq_lens), k, sink, window, _p(idx),
                            _p(cnt), _p(sel_scores), _p(ws), 0 if ws is None else ws.numel(),
                            _stream(scores)))
    return (idx, cnt, sel_scores) if want_scores else (idx, cnt)


# ---------------------------------------------------------------------------
# sequence-shard exact top-k (include/socket_b200.h)
# ---------------------------------------------------------------------------
def topk_digest(cfg: Config, scores, seq_lens, k: int, shards: int, Q: int = 64, sink: int = 0,
                window: int = 0, digest=None, ws=None):
    """This shard's digest [B][H_sel][Q][2] (int32 view of u32 (edge key, #keys >= edge))."""
    _need(scores, torch.float32, (cfg.B, cfg.H_sel, cfg.N_max), "scores")
    _need(seq_lens, torch.int32, (cfg.B,), "seq_lens")
    if digest is None:
        digest = torch.empty((cfg.B, cfg.H_sel, Q, 2), dtype=torch.int32, device=scores.device)
    _need(digest, torch.int32, (cfg.B, cfg.H_sel, Q, 2), "digest")
    if ws is None and workspace_bytes(cfg, _lib.OP_TOPK, k) > 0:
        ws = workspace(cfg, _lib.OP_TOPK, k, scores.device)
    c = cfg.c()
    check(lib().socket_topk_digest(ctypes.byref(c), _p(scores), _p(seq_lens), k, sink, window, shards,
                                   Q, _p(digest), _p(ws), 0 if ws is None else ws.numel(),
                                   _stream(scores)))
    return digest


def topk_bracket(cfg: Config, all_digests, k: int, state=None):
    """Initial per-row state [B][H_sel][8] from the G gathered digests [G][B][H_sel][Q][2]."""
    G, Q = int(all_digests.shape[0]), int(all_digests.shape[3])
    _need(all_digests, torch.int32, (G, cfg.B, cfg.H_sel, Q, 2), "all_digests")
    if state is None:
        state = torch.empty((cfg.B, cfg.H_sel, _lib.TOPK_STATE_WORDS), dtype=torch.int32,
                            device=all_digests.device)
    _need(state, torch.int32, (cfg.B, cfg.H_sel, _lib.TOPK_STATE_WORDS), "state")
    c = cfg.c()
    check(lib().socket_topk_bracket(ctypes.byref(c), _p(all_digests), G, Q, k, _p(state),
                                    _stream(all_digests)))
    return state


def topk_window(cfg: Config, scores, seq_lens, state, sink: int = 0, window: int = 0, msg=None,
                ws=None):
    """This shard's window message [B][H_sel][8 + 2048] for the state's brackets."""
    _need(scores, torch.float32, (cfg.B, cfg.H_sel, cfg.N_max), "scores")
    _need(seq_lens, torch.int32, (cfg.B,), "seq_lens")
    _need(state, torch.int32, (cfg.B, cfg.H_sel, _lib.TOPK_STATE_WORDS), "state")
    if msg is None:
        msg = torch.empty((cfg.B, cfg.H_sel, _lib.TOPK_MSG_WORDS), dtype=torch.int32, device=scores.device)
    _need(msg, torch.int32, (cfg.B, cfg.H_sel, _lib.TOPK_MSG_WORDS), "msg")
    if ws is None and workspace_bytes(cfg, _lib.OP_TOPK, 1) > 0:
        ws = workspace(cfg, _lib.OP_TOPK, 1, scores.device)
    c = cfg.c()
    check(lib().socket_topk_window(ctypes.byref(c), _p(scores), _p(seq_lens), sink, window, _p(state),
                                   _p(msg), _p(ws), 0 if ws is None else ws.numel(), _stream(scores)))
    return msg


def topk_resolve(cfg: Config, all_msgs, rank: int, state):
    """Resolve (or narrow) every row's threshold from the G gathered messages."""
    G = int(all_msgs.shape[0])
    _need(all_msgs, torch.int32, (G, cfg.B, cfg.H_sel, _lib.TOPK_MSG_WORDS), "all_msgs")
    _need(state, torch.int32, (cfg.B, cfg.H_sel, _lib.TOPK_STATE_WORDS), "state")
    c = cfg.c()
    check(lib().socket_topk_resolve(ctypes.byref(c), _p(all_msgs), G, rank, _p(state),
                                    _stream(all_msgs)))
    return state


def topk_emit(cfg: Config, scores, seq_lens, k: int, state, sink: int = 0, window: int = 0,
              idx=None, cnt=None, sel_scores=None, ws=None):
    """This shard's share of the global selection (local indices ascending, cnt)."""
    _need(scores, torch.float32, (cfg.B, cfg.H_sel, cfg.N_max), "scores")
    _need(seq_lens, torch.int32, (cfg.B,), "seq_lens")
    _need(state, torch.int32, (cfg.B, cfg.H_sel, _lib.TOPK_STATE_WORDS), "state")
    dev = scores.device
    if idx is None:
        idx = torch.empty((cfg.B, cfg.H_sel, k), dtype=torch.int32, device=dev)
    if cnt is None:
        cnt = torch.empty((cfg.B, cfg.H_sel), dtype=torch.int32, device=dev)
    _need(idx, torch.int32, (cfg.B, cfg.H_sel, k), "idx")
    _need(cnt, torch.int32, (cfg.B, cfg.H_sel), "cnt")
    if ws is None and workspace_bytes(cfg, _lib.OP_TOPK, k) > 0:
        ws = workspace(cfg, _lib.OP_TOPK, k, dev)
    c = cfg.c()
    check(lib().socket_topk_emit(ctypes.byref(c), _p(scores), _p(seq_lens), k, sink, window, _p(state),
                                 _p(idx), _p(cnt), _p(sel_scores), _p(ws),
                                 0 if ws is None else ws.numel(), _stream(scores)))
    return idx, cnt


def sparse_decode(cfg: Config, q, K, V, idx, cnt, k: int, out=None, lse=None, partial=None,
                  ws=None, want_out: bool = True):
    """Eq. 2 exact attention over the selected rows; out bf16 [B][H_q][d], lse fp32."""
    _need(q, torch.bfloat16, (cfg.B, cfg.H_q, cfg.d), "q")
    _need_kv(cfg, K, V)
    _need(idx, torch.int32, (cfg.B, cfg.H_sel, k), "idx")
    _need(cnt, torch.int32, (cfg.B, cfg.H_sel), "cnt")
    if partial is not None:
        _need(partial, torch.float32, (cfg.B, cfg.H_q, cfg.d + 2), "partial")
    dev = q.device
    if want_out and out is None:
        out = torch.empty((cfg.B, cfg.H_q, cfg.d), dtype=torch.bfloat16, device=dev)
        lse = torch.empty((cfg.B, cfg.H_q), dtype=torch.float32, device=dev) if lse is None else lse
    if ws is None:
        ws = workspace(cfg, _lib.OP_SPARSE_DECODE, k, dev)
    _need_ws(ws, cfg, _lib.OP_SPARSE_DECODE, k)
    if out is not None:
        _need(out, torch.bfloat16, (cfg.B, cfg.H_q, cfg.d), "out")
    if lse is not None:
        _need(lse, torch.float32, (cfg.B, cfg.H_q), "lse")
    c = cfg.c()
    check(lib().socket_sparse_decode(ctypes.byref(c), _p(q), _p(K), _p(V), _p(idx), _p(cnt), k,
                                     _p(out), _p(lse), _p(partial), _p(ws), ws.numel(), _stream(q)))
    return out, lse


def sample_decode(cfg: Config, scores, vnorm, V, seq_lens, uniforms, samples=None, out=None,
                  want_samples: bool = True):
    """Eq. 6 value-aware sampling estimator (PER_QHEAD rows): M = uniforms.shape[-1]
    draws by inverse CDF of p_j = s_j / sum s; out bf16 [B][H_q][d], samples
    int32 [B][H_q][M] (J_m in the order of the uniforms)."""
    _need(scores, torch.float32, (cfg.B, cfg.H_q, cfg.N_max), "scores")
    M = int(uniforms.shape[-1])
    _need(uniforms, torch.float32, (cfg.B, cfg.H_q, M), "uniforms")
    _need(vnorm, torch.float32, (cfg.B, cfg.H_kv, cfg.N_max), "vnorm")
    _need(V, torch.bfloat16, (cfg.B, cfg.H_kv, cfg.N_max, cfg.d), "V")
    _need(seq_lens, torch.int32, (cfg.B,), "seq_lens")
    dev = scores.device
    if out is None:
        out = torch.empty((cfg.B, cfg.H_q, cfg.d), dtype=torch.bfloat16, device=dev)
    if want_samples and samples is None:
        samples = torch.empty((cfg.B, cfg.H_q, M), dtype=torch.int32, device=dev)
    _need(out, torch.bfloat16, (cfg.B, cfg.H_q, cfg.d), "out")
    if samples is not None:
        _need(samples, torch.int32, (cfg.B, cfg.H_q, M), "samples")
    c = cfg.c()
    check(lib().socket_sample_decode(ctypes.byref(c), _p(scores), _p(vnorm), _p(V), _p(seq_lens),
                                     _p(uniforms), M, _p(samples), _p(out), _stream(scores)))
    return out, samples


def dense_decode(cfg: Config, q, K, V, seq_lens, out=None, lse=None, ws=None):
    """Eq. 1 dense flash-decode over j < seq_lens[b] (the k = n baseline)."""
    _need(q, torch.bfloat16, (cfg.B, cfg.H_q, cfg.d), "q")
    _need_kv(cfg, K, V)
    _need(seq_lens, torch.int32, (cfg.B,), "seq_lens")
    dev = q.device
    if out is None:
        out = torch.empty((cfg.B, cfg.H_q, cfg.d), dtype=torch.bfloat16, device=dev)
    if lse is None:
        lse = torch.empty((cfg.B, cfg.H_q), dtype=torch.float32, device=dev)
    if ws is None:
        ws = workspace(cfg, _lib.OP_DENSE_DECODE, 1, dev)
    _need_ws(ws, cfg, _lib.OP_DENSE_DECODE, 1)
    _need(out, torch.bfloat16, (cfg.B, cfg.H_q, cfg.d), "out")
    _need(lse, torch.float32, (cfg.B, cfg.H_q), "lse")
    c = cfg.c()
    check(lib().socket_dense_decode(ctypes.byref(c), _p(q), _p(K), _p(V), _p(seq_lens), _p(out),
                                    _p(lse), _p(ws), ws.numel(), _stream(q)))
    return out, lse


def lse_combine(cfg: Config, partials, out=None, lse=None):
    """Merge G partial states [G][B][H_q][d+2] -> out bf16, lse."""
    G = partials.shape[0]
    _need(partials, torch.float32, (G, cfg.B, cfg.H_q, cfg.d + 2), "partials")
    dev = partials.device
    if out is None:
        out = torch.empty((cfg.B, cfg.H_q, cfg.d), dtype=torch.bfloat16, device=dev)
    if lse is None:
        lse = torch.empty((cfg.B, cfg.H_q), dtype=torch.float32, device=dev)
    _need(out, torch.bfloat16, (cfg.B, cfg.H_q, cfg.d), "out")
    _need(lse, torch.float32, (cfg.B, cfg.H_q), "lse")
    c = cfg.c()
    check(lib().socket_lse_combine(ctypes.byref(c), _p(partials), G, _p(out), _p(lse),
                                   _stream(partials)))
    return out, lse
