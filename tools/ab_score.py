"""A/B of the score-kernel variants inside the graph-replayed bench step.

    python tools/ab_score.py        (env knobs: SOCKET_SCORE_V1, SOCKET_SCORE_TMA)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2602_06283_b200 import Config, SocketDecoder, ops  # noqa: E402

B, N = 16, 32768
q, K, V = datagen.torch_make_cache(B, 32, 8, N, 128, seed=1)
W = torch.from_numpy(datagen.make_projections(4242, 60, 8, 128).view("int16")).cuda().view(torch.bfloat16)
lens = torch.full((B,), N, dtype=torch.int32, device="cuda")
cfg = Config(B=B, H_q=32, H_kv=8, N_max=N)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn, n=30):
    for _ in range(5):
        flush.zero_()
        fn()
    torch.cuda.synchronize()
    tot = 0
    for _ in range(n):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / n * 1e3


variants = {"v1 cp.async ring": {"SOCKET_SCORE_V1": "1"}, "tma ring": {"SOCKET_SCORE_TMA": "1"}, "register": {}}
res = {k: [] for k in variants}
dec = SocketDecoder(cfg, W, K, V, k=3277)
dec.prefill()
lut = ops.build_lut(cfg, q, W)
for rep in range(3):
    for name, env in variants.items():
        for k2 in ("SOCKET_SCORE_V1", "SOCKET_SCORE_TMA"):
            os.environ.pop(k2, None)
        os.environ.update(env)
        d2 = SocketDecoder(cfg, W, K, V, k=3277)
        d2.codes, d2.vnorm = dec.codes, dec.vnorm
        d2.capture(q, lens, append=True)
        step = timeit(d2.replay)
        sc = timeit(lambda: ops.score_lut(cfg, lut, dec.codes, dec.vnorm, lens, out=dec.scores))
        res[name].append((round(step, 1), round(sc, 1)))
        del d2
for k, v in res.items():
    print(f"{k:18s} step/score us: {v}")
