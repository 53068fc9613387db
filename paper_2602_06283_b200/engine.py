"""SocketDecoder: the decode-time hot path of SOCKET on one GPU.

Owns the SOCKET index (codes, value norms) and every per-step buffer, so one
decode step is a fixed sequence of library launches on one stream, capturable
in a CUDA graph:

    socket_decode_step:
    1. prologue launch: Alg. 1 on the newest key (append) || Alg. 2 tables (LUT)
    2. score (Eq. 4 / Alg. 4)        -- PDL-chained
    3. top-k (Alg. 3 l.244)          -- PDL-chained
    4. sparse decode + LSE combine   -- PDL-chained (Eq. 2)

The KV cache (K, V) belongs to the caller (the model writes the new token's
K/V row before the step); PyTorch provides memory, streams and graphs.
"""
from __future__ import annotations

import torch

from . import _lib
from . import ops
from .ops import Config


class SocketDecoder:
    def __init__(self, cfg: Config, W: torch.Tensor, K: torch.Tensor, V: torch.Tensor, k: int,
                 sink: int = 0, window: int = 0):
        self.cfg, self.W, self.K, self.V = cfg, W, K, V
        self.k, self.sink, self.window = int(k), int(sink), int(window)
        dev = K.device
        self.device = dev
        self.codes = ops.alloc_codes(cfg, dev)
        self.vnorm = torch.zeros((cfg.B, cfg.H_kv, cfg.N_max), dtype=torch.float32, device=dev)
        self.scores = torch.empty((cfg.B, cfg.H_sel, cfg.N_max), dtype=torch.float32, device=dev)
        self.idx = torch.empty((cfg.B, cfg.H_sel, self.k), dtype=torch.int32, device=dev)
        self.cnt = torch.empty((cfg.B, cfg.H_sel), dtype=torch.int32, device=dev)
        self.out = torch.empty((cfg.B, cfg.H_q, cfg.d), dtype=torch.bfloat16, device=dev)
        self.lse = torch.empty((cfg.B, cfg.H_q), dtype=torch.float32, device=dev)
        self.fused = cfg.code_slots <= 64 and cfg.P <= 8
        self.ws_step = ops.workspace(cfg, _lib.OP_DECODE_STEP, self.k, dev) if self.fused else None
        self.ws_score = ops.workspace(cfg, _lib.OP_SCORE, 1, dev)
        self.ws_dec = ops.workspace(cfg, _lib.OP_SPARSE_DECODE, self.k, dev)
        self.graph = None

    # --- prefill: Alg. 1 over the whole cache ---------------------------------
    def prefill(self, n_tokens: int | None = None):
        n = self.cfg.N_max if n_tokens is None else n_tokens
        ops.hash_keys(self.cfg, self.K, self.W, self.codes, V=self.V, vnorm=self.vnorm,
                      n_begin=0, n_count=n)

    # --- one decode step --------------------------------------------------------
    def step(self, q: torch.Tensor, seq_lens: torch.Tensor, append: bool = False, mask=None):
        """One decode step.  append=True first hashes the newest key of every
        sequence (position seq_lens[b] - 1; the caller has written its K/V row).
        Uses the fused socket_decode_step (one library call, 4 launches)."""
        if not self.fused:
            return self.step_unfused(q, seq_lens, append, mask)
        ops.decode_step(self.cfg, q, self.K, self.V, self.W, self.codes, self.vnorm, seq_lens,
                        self.k, append=append, sink=self.sink, window=self.window, mask=mask,
                        scores=self.scores, idx=self.idx, cnt=self.cnt, out=self.out, lse=self.lse,
                        ws=self.ws_step)
        return self.out, self.lse

    def step_unfused(self, q, seq_lens, append: bool = False, mask=None):
        """Same step as separate library calls (one per stage); used for stage
        timing and as the path for L > 64.  Append requires equal seq_lens."""
        cfg = self.cfg
        if append:
            n = int(seq_lens.max().item())
            if int(seq_lens.min().item()) != n:
                raise ValueError("step_unfused(append=True) needs equal seq_lens; use step()")
            ops.hash_keys(cfg, self.K, self.W, self.codes, V=self.V, vnorm=self.vnorm,
                          n_begin=n - 1, n_count=1)
        ops.score(cfg, q, self.W, self.codes, self.vnorm, seq_lens, mask=mask, out=self.scores,
                  ws=self.ws_score)
        ops.topk(cfg, self.scores, seq_lens, self.k, self.sink, self.window, idx=self.idx,
                 cnt=self.cnt)
        ops.sparse_decode(cfg, q, self.K, self.V, self.idx, self.cnt, self.k, out=self.out,
                          lse=self.lse, ws=self.ws_dec)
        return self.out, self.lse

    # --- CUDA graph of one step ---------------------------------------------------
    def capture(self, q: torch.Tensor, seq_lens: torch.Tensor, append: bool = False):
        """Capture step(q) into a CUDA graph (q, seq_lens are the static inputs)."""
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self.step(q, seq_lens, append)              # warm-up outside the graph
        torch.cuda.current_stream(self.device).wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step(q, seq_lens, append)
        self.graph = g
        return g

    def replay(self):
        self.graph.replay()
        return self.out, self.lse
