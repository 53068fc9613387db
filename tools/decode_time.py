"""Time socket_sparse_decode alone on the bench workload's selection (L2
flushed, CUDA events; the product library, or SOCKET_LIB_VARIANT).

    python tools/decode_time.py [--batch 16] [--ctx 32768] [--sparsity 10]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2602_06283_b200 import Config, SocketDecoder, ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--ctx", type=int, default=32768)
ap.add_argument("--sparsity", type=float, default=10)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
B, N = a.batch, a.ctx
k = int(round(N / a.sparsity))
cfg = Config(B=B, H_q=32, H_kv=8, N_max=N, L=60, P=8)
q, K, V = datagen.torch_make_cache(B, 32, 8, N, 128, seed=1)
W = torch.from_numpy(datagen.make_projections(4242, 60, 8, 128).view("int16")).cuda().view(torch.bfloat16)
lens = torch.full((B,), N, dtype=torch.int32, device="cuda")
dec = SocketDecoder(cfg, W, K, V, k=k)
dec.prefill()
sc = ops.score(cfg, q, W, dec.codes, dec.vnorm, lens)
idx, cnt = ops.topk(cfg, sc, lens, k)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ws = ops.workspace(cfg, 4, k, q.device)
out = torch.empty_like(q)
lse = torch.empty((B, 32), dtype=torch.float32, device="cuda")
ops.sparse_decode(cfg, q, K, V, idx, cnt, k, out=out, lse=lse, ws=ws)
ref = out.clone()
tot = 0.0
for _ in range(a.reps):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ops.sparse_decode(cfg, q, K, V, idx, cnt, k, out=out, lse=lse, ws=ws)
    e1.record()
    e1.synchronize()
    tot += e0.elapsed_time(e1)
ab = B * 8 * k * (2 * 128 * 2 + 4) + B * 32 * 128 * 4
us = tot / a.reps * 1e3
print(f"{os.environ.get('SOCKET_LIB_VARIANT', 'product')}: B={B} N={N} k={k} decode {us:.2f} us "
      f"{ab / (us * 1e-6) / 1e12:.2f} TB/s same={bool(torch.equal(ref, out))}")
