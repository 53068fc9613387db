"""The shard layer (paper_2602_06283_b200/dist.py) on the GPU with NCCL, in a
one-process world (only one GPU is available to this build): the sequence-
sharded step with G = 1 runs the whole exchange path -- scores, digest, NCCL
all-gather, bracket, window message, NCCL all-gather, resolve, emit, partial-
state decode, NCCL all-gather of the partials, socket_lse_combine -- eagerly
and as one CUDA graph (collectives captured), and must give the single-device
selection and output.  The multi-rank logic is covered with gloo in
tests/test_dist_gloo.py and with G virtual shards in tests/test_gpu_shard.py."""
import os
import socket

import pytest
import torch
import torch.distributed as dist

from helpers import bits_to_dev

pytestmark = pytest.mark.gpu

ops = pytest.importorskip("paper_2602_06283_b200.ops")
from paper_2602_06283_b200 import Config, SocketDecoder  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sequence_shard_path_on_gpu_nccl_world_of_one():
    import datagen
    from paper_2602_06283_b200.dist import SeqShardDecoder, seq_shard_config
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        B, H_q, H_kv, N, L, k = 2, 8, 2, 4096, 60, 400
        c = datagen.make_case(B, H_q, H_kv, N, 128, seed=71, seq_lens=[4096, 3000])
        W = bits_to_dev(datagen.make_projections(72, L, 8, 128))
        q, K, V = bits_to_dev(c["q"]), bits_to_dev(c["K"]), bits_to_dev(c["V"])
        lens = torch.from_numpy(c["seq_lens"]).cuda()
        cfg = Config(B=B, H_q=H_q, H_kv=H_kv, N_max=N, L=L, P=8)
        sd = SeqShardDecoder(seq_shard_config(cfg, 1, 0), W, K, V, k)
        sd.prefill()
        out, lse = [t.clone() for t in sd.step(q, lens)]
        ref = SocketDecoder(cfg, W, K.clone(), V.clone(), k=k)
        ref.prefill()
        ref.step_unfused(q, lens, append=False)
        torch.cuda.synchronize()
        assert torch.equal(sd.idx, ref.idx) and torch.equal(sd.cnt, ref.cnt)
        assert (out.float() - ref.out.float()).abs().max().item() <= 2e-3
        assert (lse - ref.lse).abs().max().item() <= 1e-3
        # the same step captured in a CUDA graph (fixed 3 window rounds, NCCL inside)
        sd.capture(q, lens)
        sd.idx.fill_(-7)
        og, lg = sd.replay()
        torch.cuda.synchronize()
        assert torch.equal(sd.idx, ref.idx) and torch.equal(og, out) and torch.equal(lg, lse)
    finally:
        dist.destroy_process_group()
