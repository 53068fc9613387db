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
        self.fused = cfg.code_slots <= 64
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
    def step(self, q: torch.Tensor, seq_lens: torch.Tensor, append: bool = False, mask=None,
             k_new=None, v_new=None, out=None):
        """One decode step.  append=True first hashes the newest key of every
        sequence (position seq_lens[b] - 1): its K/V rows are either already in
        the cache, or passed as k_new / v_new ([B][H_kv][d]) and stored by the
        step itself.  Uses socket_decode_step (one library call)."""
        if not self.fused:
            if k_new is not None:
                n = seq_lens.long() - 1
                bi = torch.arange(self.cfg.B, device=self.device)
                self.K[bi, :, n] = k_new
                self.V[bi, :, n] = v_new
            return self.step_unfused(q, seq_lens, append, mask)
        o = self.out if out is None else out
        ops.decode_step(self.cfg, q, self.K, self.V, self.W, self.codes, self.vnorm, seq_lens,
                        self.k, append=append, sink=self.sink, window=self.window, mask=mask,
                        scores=self.scores, idx=self.idx, cnt=self.cnt, out=o, lse=self.lse,
                        ws=self.ws_step, k_new=k_new, v_new=v_new)
        return o, self.lse

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

    # --- host I/O: pinned host inputs -> step -> pinned host output -------------
    def bind_host(self, seq_lens: torch.Tensor):
        """Allocate pinned host I/O buffers for host_step(): q [B][H_q][d] and the
        new token's K and V rows [B][H_kv][d] packed in one pinned input buffer,
        and a pinned output [B][H_q][d].  host_step() replays the decode step as
        a CUDA graph that reads the inputs from the pinned, UVA-mapped buffer
        (staged by one copy kernel on the chained path), stores the new rows into
        the cache at seq_lens[b] - 1, hashes them, and writes the output straight
        into the pinned output -- no DMA copy either way.
        (Memcpy nodes from pinned host memory inside the graph cost ~50 us of
        launch latency per replay on this driver, so the copies stay outside.)
        Binding does not modify the cache: its warm-up step runs without the
        append.  Returns the pinned views (q_in, k_in, v_in, out)."""
        cfg, dev = self.cfg, self.device
        nq = cfg.B * cfg.H_q * cfg.d
        nk = cfg.B * cfg.H_kv * cfg.d
        self._in_h = torch.empty(nq + 2 * nk, dtype=torch.bfloat16).pin_memory()
        self._in_d = torch.empty(nq + 2 * nk, dtype=torch.bfloat16, device=dev)
        out_h = torch.empty((cfg.B, cfg.H_q, cfg.d), dtype=torch.bfloat16).pin_memory()
        views = lambda t: (t[:nq].view(cfg.B, cfg.H_q, cfg.d), t[nq:nq + nk].view(cfg.B, cfg.H_kv, cfg.d),
                           t[nq + nk:].view(cfg.B, cfg.H_kv, cfg.d))
        q_d, k_d, v_d = views(self._in_d)
        self._in_h.zero_()
        self._in_d.zero_()

        direct = self.fused      # socket_decode_step writes `out` straight into the
                                 # pinned (UVA-mapped) host buffer: no D2H copy
        # and it takes q and the new rows from the mapped host buffer: the
        # one-launch kernel (small batch) reads each input once in place, the
        # chained path stages them with one copy kernel (no DMA copy outside the graph)
        self._host_inputs_direct = direct
        src_q, src_k, src_v = views(self._in_h) if self._host_inputs_direct else (q_d, k_d, v_d)

        def body():
            self.step(src_q, seq_lens, append=True, k_new=src_k, v_new=src_v,
                      out=out_h if direct else None)

        # warm-up outside the graph WITHOUT the append: it exercises the same
        # launches but leaves the cache, codes and norms of key seq_lens[b] - 1
        # untouched (the pinned k/v inputs are still zeros here)
        s = torch.cuda.Stream(dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            self.step(src_q, seq_lens, append=False, out=out_h if direct else None)
        torch.cuda.current_stream(dev).wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            body()
        self.graph_host = g
        self._host_direct = direct
        self._host = (*views(self._in_h), out_h)
        return self._host

    def host_step(self):
        """One step from the pinned inputs of bind_host() to its pinned output
        (asynchronous on the current stream)."""
        if not self._host_inputs_direct:
            self._in_d.copy_(self._in_h, non_blocking=True)
        self.graph_host.replay()
        if not self._host_direct:
            self._host[3].copy_(self.out, non_blocking=True)
        return self._host[3]
