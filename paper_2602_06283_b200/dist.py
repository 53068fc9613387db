"""Multi-GPU shard layer for the SOCKET decode step.

One process per GPU, torch.distributed for the plumbing (NCCL over NVLink /
NVSwitch on GPUs, gloo for the CPU tests).  Two layouts:

KV-head sharding (BASELINE configs[2], 128K context): rank g owns KV heads
  [g H_kv/G, (g+1) H_kv/G) and their query heads, with all their tokens.  The
  per-head computation is independent, so the decode step needs NO
  collective; outputs stay head-sharded (tensor-parallel style).

Sequence sharding (BASELINE configs[3], 1M tokens): rank g owns tokens
  [g N_s, (g+1) N_s) of every head.  One step is
    1. local scores (socket_score) and local top-k with candidate scores
       (socket_topk, sel_scores) -- the shard's part of the global top-k is
       contained in its local top-k;
    2. all-gather of the candidate (score, local index) lists, rank order;
    3. socket_topk_resolve: the exact global top-k under (score desc, global
       index asc) over the G*k candidates; each rank keeps its own share;
    4. local sparse flash-decode over the share -> partial (m, l, o);
    5. all-gather of the partials and socket_lse_combine.
  Sink / local-window forcing is not supported in this layout (they refer to
  global positions); use sink = window = 0.

`ops` is the local-compute provider: the CUDA library (paper_2602_06283_b200.ops)
in the product; the CPU tests inject an oracle-backed provider with the same
call signatures to check this orchestration under gloo.
"""
from __future__ import annotations

from dataclasses import replace

import torch
import torch.distributed as dist

from .ops import Config


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
class SeqShardDecoder:
    """Sequence-sharded SOCKET decode step (exact global top-k + LSE combine).

    cfg: the SHARD config (N_max = tokens per shard).  K, V, codes, vnorm are
    this rank's shard; seq_lens are the shard-local valid lengths.
    """

    def __init__(self, cfg: Config, W, K, V, k: int, group=None, ops=None):
        if ops is None:
            from . import ops as gpu_ops
            ops = gpu_ops
        self.ops, self.cfg, self.W, self.K, self.V = ops, cfg, W, K, V
        self.k, self.group = int(k), group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.codes = ops.alloc_codes(cfg, K.device)
        self.vnorm = torch.zeros((cfg.B, cfg.H_kv, cfg.N_max), dtype=torch.float32, device=K.device)

    def prefill(self, n_tokens=None):
        n = self.cfg.N_max if n_tokens is None else n_tokens
        self.ops.hash_keys(self.cfg, self.K, self.W, self.codes, V=self.V, vnorm=self.vnorm,
                           n_begin=0, n_count=n)

    def step(self, q, seq_lens):
        """Returns (out [B,H_q,d] bf16, lse [B,H_q], local idx [B,H_sel,k], cnt) --
        the output is replicated on every rank; idx/cnt are this rank's share
        (shard-local indices)."""
        ops, cfg, k = self.ops, self.cfg, self.k
        scores = ops.score(cfg, q, self.W, self.codes, self.vnorm, seq_lens)
        c_idx, _, c_scores = ops.topk(cfg, scores, seq_lens, k, want_scores=True)
        all_scores = _gather(c_scores, self.group)          # [G, B, H_sel, k]
        all_idx = _gather(c_idx, self.group)
        idx, cnt = ops.topk_resolve(cfg, all_scores, all_idx, self.rank, k)
        part = torch.empty((cfg.B, cfg.H_q, cfg.d + 2), dtype=torch.float32, device=q.device)
        ops.sparse_decode(cfg, q, self.K, self.V, idx, cnt, k, partial=part, want_out=False)
        parts = _gather(part, self.group)                    # [G, B, H_q, d+2]
        out, lse = ops.lse_combine(cfg, parts)
        return out, lse, idx, cnt
