"""Multi-GPU shard layer for the SOCKET decode step.

One process per GPU, torch.distributed for the plumbing (NCCL over NVLink /
NVSwitch on GPUs, gloo for the CPU tests).  Two layouts:

KV-head sharding (BASELINE configs[2], 128K context): rank g owns KV heads
  [g H_kv/G, (g+1) H_kv/G) and their query heads, with all their tokens.  The
  per-head computation is independent, so the decode step needs NO
  collective; outputs stay head-sharded (tensor-parallel style).

Sequence sharding (BASELINE configs[3], 1M tokens): rank s owns global token
  positions [s N_s, (s+1) N_s) of every head (cfg.index_base = s N_s; every
  call takes the sequences' TOTAL lengths).  One step is
    1. local scores (socket_score) and the shard's digest (socket_topk_digest):
       Q exact (edge, #keys >= edge) pairs per row;             all-gather
    2. socket_topk_bracket: every rank derives the same bracket [T_lo, T_hi)
       around the global threshold key T;
    3. socket_topk_window: #keys >= T_hi and the bracket's keys (or their
       histogram) per row;                                       all-gather
       socket_topk_resolve: T exact (or a narrower bracket; <= 3 rounds);
    4. socket_topk_emit: the shard's share of the exact global top-k (keys > T
       and its quota of ties at T in global index order);
    5. local sparse flash-decode over the share -> partial (m, l, o);
                                                                 all-gather
       socket_lse_combine.
  Messages per GPU and round at configs[3] (8 rows): digest 4 KB, window
  66 KB, partials 16.6 KB -- instead of the 6.7 MB of a bulk candidate
  exchange.  Sink / local-window forcing works on global
  positions.

`ops` is the local-compute provider: the CUDA library (paper_2602_06283_b200.ops)
in the product; the CPU tests inject a host model with the same call
signatures to check this orchestration under gloo.  The transport is a
torch.distributed process group, or `VirtualShards` -- G shards held by one
process (one GPU), whose all-gathers are stacks; it runs the identical kernel
sequence and serves tests and the single-GPU bench of the layout.
"""
from __future__ import annotations

from dataclasses import replace

import torch
import torch.distributed as dist

from . import _lib
from .ops import Config

MAX_WINDOW_ROUNDS = 3     # 2048-bin histograms take any 32-bit bracket to one key value


def _gather(t: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather `t` from every rank, stacked in rank order: [G, *t.shape]."""
    G = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((G,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
        return out
    parts = [torch.empty_like(t) for _ in range(G)]
    dist.all_gather(parts, t.contiguous(), group=group)
    return torch.stack(parts)


# ---------------------------------------------------------------------------
# KV-head sharding
# ---------------------------------------------------------------------------
def kv_head_range(H_kv: int, world: int, rank: int):
    if H_kv % world:
        raise ValueError(f"H_kv={H_kv} not divisible by world size {world}")
    n = H_kv // world
    return rank * n, (rank + 1) * n


def kv_head_shard_config(cfg: Config, world: int, rank: int) -> Config:
    """Config of rank's KV-head shard (same B, N, L, P, tau; fewer heads)."""
    g0, g1 = kv_head_range(cfg.H_kv, world, rank)
    G = cfg.H_q // cfg.H_kv
    return replace(cfg, H_kv=g1 - g0, H_q=(g1 - g0) * G)


def kv_head_shard(cfg: Config, world: int, rank: int, q, K, V):
    """Slice q [B,H_q,d] and K/V [B,H_kv,N,d] to rank's heads (contiguous copies)."""
    g0, g1 = kv_head_range(cfg.H_kv, world, rank)
    G = cfg.H_q // cfg.H_kv
    return (q[:, g0 * G:g1 * G].contiguous(), K[:, g0:g1].contiguous(), V[:, g0:g1].contiguous())


# ---------------------------------------------------------------------------
# sequence sharding
# ---------------------------------------------------------------------------
def seq_shard_config(cfg: Config, world: int, rank: int) -> Config:
    """Config of rank's sequence shard: cfg.N_max / world tokens per shard at
    global positions [rank N_s, (rank+1) N_s)."""
    if cfg.N_max % world or (cfg.N_max // world) % 32:
        raise ValueError(f"N_max={cfg.N_max} must split into {world} shards of a multiple of 32 tokens")
    Ns = cfg.N_max // world
    return replace(cfg, N_max=Ns, index_base=rank * Ns)


class SeqShard:
    """One sequence shard's buffers and local calls (rank `rank` of `world`).

    cfg: the SHARD config (N_max = tokens per shard, index_base = first global
    position).  K, V, codes, vnorm hold this shard's keys."""

    def __init__(self, cfg: Config, W, K, V, k: int, rank: int, world: int, ops=None,
                 sink: int = 0, window: int = 0, Q: int = 64):
        if ops is None:
            from . import ops as gpu_ops
            ops = gpu_ops
        self.ops, self.cfg, self.W, self.K, self.V = ops, cfg, W, K, V
        self.k, self.rank, self.world = int(k), int(rank), int(world)
        self.sink, self.window, self.Q = int(sink), int(window), int(Q)
        dev = K.device
        self.codes = ops.alloc_codes(cfg, dev)
        self.vnorm = torch.zeros((cfg.B, cfg.H_kv, cfg.N_max), dtype=torch.float32, device=dev)
        self.scores = torch.empty((cfg.B, cfg.H_sel, cfg.N_max), dtype=torch.float32, device=dev)
        self.idx = torch.empty((cfg.B, cfg.H_sel, self.k), dtype=torch.int32, device=dev)
        self.cnt = torch.empty((cfg.B, cfg.H_sel), dtype=torch.int32, device=dev)
        self.part = torch.empty((cfg.B, cfg.H_q, cfg.d + 2), dtype=torch.float32, device=dev)
        self.state = None
        # window message buffer, zero-filled once: the kernel writes only the
        # header and the wc entries the resolve reads; the tail is all-gathered too
        self.msg = torch.zeros((cfg.B, cfg.H_sel, _lib.TOPK_MSG_WORDS), dtype=torch.int32, device=dev)

    def prefill(self, n_tokens=None):
        n = self.cfg.N_max if n_tokens is None else n_tokens
        self.ops.hash_keys(self.cfg, self.K, self.W, self.codes, V=self.V, vnorm=self.vnorm,
                           n_begin=0, n_count=n)

    # protocol phases (each returns what the transport all-gathers next)
    def digest(self, q, seq_lens):
        self.ops.score(self.cfg, q, self.W, self.codes, self.vnorm, seq_lens, out=self.scores)
        return self.ops.topk_digest(self.cfg, self.scores, seq_lens, self.k, self.world, self.Q,
                                    sink=self.sink, window=self.window)

    def bracket(self, all_digests):
        self.state = self.ops.topk_bracket(self.cfg, all_digests, self.k, state=self.state)

    def window_msg(self, seq_lens):
        return self.ops.topk_window(self.cfg, self.scores, seq_lens, self.state, sink=self.sink,
                                    window=self.window, msg=self.msg)

    def resolve(self, all_msgs):
        self.ops.topk_resolve(self.cfg, all_msgs, self.rank, self.state)

    def resolved(self) -> bool:
        return bool((self.state[..., 3] != 0).all().item())

    def attend(self, q, seq_lens):
        self.ops.topk_emit(self.cfg, self.scores, seq_lens, self.k, self.state, sink=self.sink,
                           window=self.window, idx=self.idx, cnt=self.cnt)
        self.ops.sparse_decode(self.cfg, q, self.K, self.V, self.idx, self.cnt, self.k,
                               partial=self.part, want_out=False)
        return self.part

    def combine(self, all_parts):
        return self.ops.lse_combine(self.cfg, all_parts)


def _run_protocol(shards, gather, q, seq_lens, rounds=None):
    """Drive the protocol over the shards this process holds (one per rank, or
    all G virtual shards); `gather(list_of_local_tensors)` returns the
    [G, ...] all-gather.  rounds=None: stop as soon as every row is resolved
    (reads one flag per round); an int: exactly that many window rounds
    (MAX_WINDOW_ROUNDS is always exact; capturable)."""
    all_d = gather([s.digest(q, seq_lens) for s in shards])
    for s in shards:
        s.bracket(all_d)
    n_rounds = MAX_WINDOW_ROUNDS if rounds is None else int(rounds)
    for _ in range(n_rounds):
        all_m = gather([s.window_msg(seq_lens) for s in shards])
        for s in shards:
            s.resolve(all_m)
        if rounds is None and all(s.resolved() for s in shards):
            break
    all_p = gather([s.attend(q, seq_lens) for s in shards])
    return [s.combine(all_p) for s in shards]


class SeqShardDecoder:
    """Sequence-sharded SOCKET decode step over a torch.distributed group
    (one shard per rank; exact global top-k + LSE combine).

    cfg: the SHARD config (seq_shard_config: N_max = tokens per shard,
    index_base = rank * N_max).  K, V are this rank's shard; step() takes the
    sequences' TOTAL lengths."""

    def __init__(self, cfg: Config, W, K, V, k: int, group=None, ops=None, sink: int = 0,
                 window: int = 0, Q: int = 64):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if cfg.index_base != self.rank * cfg.N_max:
            raise ValueError("cfg.index_base must be rank * N_max (use seq_shard_config)")
        self.shard = SeqShard(cfg, W, K, V, k, self.rank, self.world, ops=ops, sink=sink,
                              window=window, Q=Q)
        self.graph = None

    @property
    def idx(self):
        return self.shard.idx

    @property
    def cnt(self):
        return self.shard.cnt

    def prefill(self, n_tokens=None):
        self.shard.prefill(n_tokens)

    def step(self, q, seq_lens, rounds=None):
        """Returns (out [B,H_q,d] bf16, lse [B,H_q]) replicated on every rank;
        self.idx / self.cnt hold this rank's share (shard-local indices)."""
        gather = lambda ts: _gather(ts[0], self.group)
        return _run_protocol([self.shard], gather, q, seq_lens, rounds)[0]

    def capture(self, q, seq_lens):
        """Capture one step (fixed MAX_WINDOW_ROUNDS rounds, always exact) in a
        CUDA graph, NCCL collectives included."""
        s = torch.cuda.Stream(q.device)
        s.wait_stream(torch.cuda.current_stream(q.device))
        with torch.cuda.stream(s):
            self.step(q, seq_lens, rounds=MAX_WINDOW_ROUNDS)
        torch.cuda.current_stream(q.device).wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.out, self.lse = self.step(q, seq_lens, rounds=MAX_WINDOW_ROUNDS)
        self.graph = g
        return g

    def replay(self):
        self.graph.replay()
        return self.out, self.lse


class VirtualShards:
    """G sequence shards held by ONE process (one device): the same kernels and
    message flow as SeqShardDecoder, with each all-gather a stack of the G
    shards' buffers.  Used for the exactness tests at full configs[3] size on
    one GPU and for the layout's single-GPU bench.

    cfg: the FULL config (N_max = total tokens); K, V the full cache
    [B][H_kv][N_max][d]; shards are views of contiguous copies."""

    def __init__(self, cfg: Config, W, K, V, k: int, G: int, ops=None, sink: int = 0,
                 window: int = 0, Q: int = 64):
        self.G = int(G)
        self.shards = []
        for r in range(self.G):
            sc = seq_shard_config(cfg, self.G, r)
            sl = slice(r * sc.N_max, (r + 1) * sc.N_max)
            self.shards.append(SeqShard(sc, W, K[:, :, sl].contiguous(), V[:, :, sl].contiguous(), k, r,
                                        self.G, ops=ops, sink=sink, window=window, Q=Q))
        self.graph = None

    def prefill(self):
        for s in self.shards:
            s.prefill()

    def step(self, q, seq_lens, rounds=None):
        """Returns (out, lse) of shard 0 (every shard holds the same combine)
        and the global selection as a list over shards of (idx, cnt)."""
        res = _run_protocol(self.shards, lambda ts: torch.stack(ts), q, seq_lens, rounds)
        return res[0]

    def global_selection(self, b: int, r: int):
        """Global indices of row (b, r) over all shards (ascending)."""
        out = []
        for s in self.shards:
            n = int(s.cnt[b, r])
            out += (s.idx[b, r, :n].long() + s.cfg.index_base).tolist()
        return out
