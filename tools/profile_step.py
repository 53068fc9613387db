"""Run prefill + a few eager SOCKET decode steps of the bench workload (for ncu).

    python tools/profile_step.py [--batch 16] [--ctx 32768] [--sparsity 10] [--tables 60] [--steps 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2602_06283_b200 import Config, KV_SHARED, PER_QHEAD, SocketDecoder  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--ctx", type=int, default=32768)
ap.add_argument("--sparsity", type=float, default=10.0)
ap.add_argument("--tables", type=int, default=60)
ap.add_argument("--bits", type=int, default=8)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--mode", default="kv_shared")
ap.add_argument("--dense", action="store_true")
ap.add_argument("--unfused", action="store_true", help="also run the stage-by-stage step")
ap.add_argument("--hard", action="store_true", help="hard-LSH tables (Eq. 3)")
ap.add_argument("--chained", action="store_true", help="never the one-launch kernel (SOCKET_FLAG_CHAINED_STEP)")
a = ap.parse_args()
B, N, L = a.batch, a.ctx, a.tables
k = int(round(N / a.sparsity))
cfg = Config(B=B, H_q=32, H_kv=8, N_max=N, L=L, P=a.bits, tau=0.5,
             group_mode=KV_SHARED if a.mode == "kv_shared" else PER_QHEAD, scoring=int(a.hard),
             flags=int(a.chained))
q, K, V = datagen.torch_make_cache(B, 32, 8, N, 128, seed=1)
W = torch.from_numpy(datagen.make_projections(4242, L, a.bits, 128).view("int16")).cuda().view(torch.bfloat16)
lens = torch.full((B,), N, dtype=torch.int32, device="cuda")
dec = SocketDecoder(cfg, W, K, V, k=k)
dec.prefill()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(a.steps):
    flush.zero_()
    dec.step(q, lens, append=True)
    if a.unfused:
        dec.step_unfused(q, lens, append=False)
    if a.dense:
        from paper_2602_06283_b200 import ops
        ops.dense_decode(cfg, q, K, V, lens)
torch.cuda.synchronize()
print("done")
