"""Wide-code (L = 60, P = 10 by default) score kernel timing on the bench cache (B = 16, 32K).
    python tools/wide_time.py [B] [P] [mode: kv_shared | per_qhead]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2602_06283_b200 import Config, SocketDecoder, _lib, ops  # noqa: E402

B, N = int(sys.argv[1]) if len(sys.argv) > 1 else 16, 32768
P = int(sys.argv[2]) if len(sys.argv) > 2 else 10
mode = ops.PER_QHEAD if len(sys.argv) > 3 and sys.argv[3] == "per_qhead" else ops.KV_SHARED
q, K, V = datagen.torch_make_cache(B, 32, 8, N, 128, seed=1)
cfg = Config(B=B, H_q=32, H_kv=8, N_max=N, L=60, P=P, group_mode=mode)
W = torch.from_numpy(datagen.make_projections(4343, 60, P, 128).view("int16")).cuda().view(torch.bfloat16)
lens = torch.full((B,), N, dtype=torch.int32, device="cuda")
dec = SocketDecoder(cfg, W, K, V, k=3277)
dec.prefill()
lut = ops.workspace(cfg, _lib.OP_SCORE, 1, "cuda")
ops.build_lut(cfg, q, W, lut)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    ops.score_lut(cfg, lut, dec.codes, dec.vnorm, lens, out=dec.scores)
tot = 0.0
for _ in range(20):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ops.score_lut(cfg, lut, dec.codes, dec.vnorm, lens, out=dec.scores)
    e1.record()
    e1.synchronize()
    tot += e0.elapsed_time(e1)
ms = tot / 20
# stored bytes read / written: packed codes (Lp P / 8 per key), norm, score (per selection row)
sb = B * 8 * N * (ops.codes_bytes(cfg) // (B * 8 * N) + 4) + B * cfg.H_sel * N * 4
print(f"wide score B={B} P={P} {'per_qhead' if mode == ops.PER_QHEAD else 'kv_shared'}: "
      f"{ms * 1e3:.1f} us  {sb / (ms * 1e-3) / 1e9:.0f} GB/s (stored bytes)")
