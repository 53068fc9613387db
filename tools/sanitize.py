"""Small-shape workload touching every kernel of libsocket_b200 once, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python tools/sanitize.py

Covers: the tcgen05 prefill hash and the CUDA-core hash, code pack/unpack,
query tables (plain + LUT), the byte-code and wide-code score kernels, top-k
(cluster select, sink/window, ties), the sequence-shard protocol (digest,
bracket, window, resolve, emit), sparse / dense decode, the LSE combine, the
sampling decode, and socket_decode_step on both the one-launch row-spread
kernel (incl. all-tied keys, forced-only selection, 4 CTAs per row) and the
PDL-chained kernels (device and pinned-host inputs).
"""
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2602_06283_b200 import Config, SocketDecoder, ops  # noqa: E402
from paper_2602_06283_b200.dist import VirtualShards  # noqa: E402


def bits(x):
    return torch.from_numpy(x.view("int16")).cuda().view(torch.bfloat16)


def main():
    dev = "cuda"
    B, Hq, Hkv, N, L, k = 2, 8, 2, 2048, 60, 200
    c = datagen.make_case(B, Hq, Hkv, N, 128, seed=1, seq_lens=[2048, 1500])
    q, K, V = bits(c["q"]), bits(c["K"]), bits(c["V"])
    W = bits(datagen.make_projections(2, L, 8, 128))
    lens = torch.from_numpy(c["seq_lens"]).to(dev)
    cfg = Config(B=B, H_q=Hq, H_kv=Hkv, N_max=N, L=L, P=8)
    # prefill (tcgen05) + CUDA-core append range, pack / unpack
    codes = ops.alloc_codes(cfg, dev)
    vnorm = torch.zeros((B, Hkv, N), dtype=torch.float32, device=dev)
    ops.hash_keys(cfg, K, W, codes, V=V, vnorm=vnorm)
    ops.hash_keys(cfg, K, W, codes, n_begin=N - 5, n_count=5)
    plain = ops.unpack_codes(cfg, codes)
    ops.pack_codes(cfg, plain)
    ops.query_tables(cfg, q, W)
    sc = ops.score(cfg, q, W, codes, vnorm, lens)
    idx, cnt = ops.topk(cfg, sc, lens, k, sink=3, window=7)
    ops.sparse_decode(cfg, q, K, V, idx, cnt, k)
    ops.dense_decode(cfg, q, K, V, lens)
    part = torch.zeros((B, Hq, 130), dtype=torch.float32, device=dev)
    ops.sparse_decode(cfg, q, K, V, idx, cnt, k, partial=part, want_out=False)
    ops.lse_combine(cfg, torch.stack([part, part]))
    # ties
    tied = torch.floor(sc * 4) / 4
    ops.topk(cfg, tied, lens, k)
    # sampling (PER_QHEAD)
    cq = dataclasses.replace(cfg, group_mode=1)
    sq = ops.score(cq, q, W, codes, vnorm, lens)
    u = torch.rand((B, Hq, 64), device=dev)
    ops.sample_decode(cq, sq, vnorm, V, lens, u)
    # wide codes (P = 10 and P = 12)
    for P in (10, 12):
        cw = dataclasses.replace(cfg, P=P)
        Ww = bits(datagen.make_projections(3, L, P, 128))
        cwc = ops.alloc_codes(cw, dev)
        ops.hash_keys(cw, K, Ww, cwc, V=V, vnorm=vnorm)
        ops.score(cw, q, Ww, cwc, vnorm, lens)
    # decode step: one launch and chained, device and pinned-host inputs
    for flags in (0, 1):
        cs = dataclasses.replace(cfg, flags=flags)
        dec = SocketDecoder(cs, W, K.clone(), V.clone(), k=k, sink=2, window=4)
        dec.prefill()
        dec.step(q, lens, append=True)
        kn = torch.randn((B, Hkv, 128), device=dev).to(torch.bfloat16)
        dec.step(q.cpu().pin_memory(), lens, append=True, k_new=kn.cpu().pin_memory(),
                 v_new=kn.cpu().pin_memory())
    # one-launch row-spread kernel: every key tied (refinement levels, one-value bin),
    # forced-only selection, and 32 rows (4 CTAs per row, SOCKET_FLAG_ONE_LAUNCH)
    Vt = V[:, :, :1].expand_as(V).contiguous()
    dec = SocketDecoder(cfg, torch.zeros_like(W), K.clone(), Vt, k=k)
    dec.prefill()
    dec.step(q, lens, append=True)
    dec = SocketDecoder(cfg, W, K.clone(), V.clone(), k=8, sink=4, window=4)
    dec.prefill()
    dec.step(q, lens, append=True)
    c4 = datagen.make_case(4, 32, 8, 1024, 128, seed=5, seq_lens=[1024, 77, 1000, 512])
    c4cfg = Config(B=4, H_q=32, H_kv=8, N_max=1024, L=L, P=8, flags=2)
    dec = SocketDecoder(c4cfg, W, bits(c4["K"]), bits(c4["V"]), k=100, sink=3, window=5)
    dec.prefill()
    dec.step(bits(c4["q"]), torch.from_numpy(c4["seq_lens"]).to(dev), append=True)
    # sequence-shard protocol on 4 virtual shards (ties)
    vs = VirtualShards(cfg, W, K, V, k, 4, sink=1, window=2)
    vs.prefill()
    vs.step(q, lens, rounds=3)
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
