"""Eq. 6 sampling decode timing on the bench cache (PER_QHEAD rows, M = k)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2602_06283_b200 import Config, PER_QHEAD, SocketDecoder, ops  # noqa: E402

B, N = int(sys.argv[1]) if len(sys.argv) > 1 else 16, 32768
k = 3277
q, K, V = datagen.torch_make_cache(B, 32, 8, N, 128, seed=1)
W = torch.from_numpy(datagen.make_projections(4242, 60, 8, 128).view("int16")).cuda().view(torch.bfloat16)
cfg = Config(B=B, H_q=32, H_kv=8, N_max=N, L=60, P=8, group_mode=PER_QHEAD)
lens = torch.full((B,), N, dtype=torch.int32, device="cuda")
dec = SocketDecoder(cfg, W, K, V, k=k)
dec.prefill()
sc = ops.score(cfg, q, W, dec.codes, dec.vnorm, lens)
u = torch.rand((B, 32, k), device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for M in (k, 256, 8192):
    uu = torch.rand((B, 32, M), device="cuda")
    for _ in range(3):
        ops.sample_decode(cfg, sc, dec.vnorm, V, lens, uu)
    tot = 0
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ops.sample_decode(cfg, sc, dec.vnorm, V, lens, uu)
        e1.record()
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    print(f"B={B} rows={B * 32} M={M}: {tot / 10 * 1e3:.1f} us")
_, J = ops.sample_decode(cfg, sc, dec.vnorm, V, lens, u)
J = J.view(B * 32, k)
d = [int(torch.unique(J[r]).numel()) for r in range(0, B * 32, 37)]
print(f"distinct J per row (M={k}): mean {sum(d) / len(d):.0f}", flush=True)
