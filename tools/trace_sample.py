"""Phase timing of the Eq. 6 sampling kernel (SM_STAMP in csrc/sample.cu).
    python tools/trace_sample.py [--batch 16] [--M 3277]"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from trace_topk import build_trace  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--M", type=int, default=3277)
    a = ap.parse_args()
    libpath = build_trace()
    from paper_2602_06283_b200 import _lib
    _lib.LIB_PATH = libpath
    L = _lib.lib()
    import datagen
    from paper_2602_06283_b200 import Config, PER_QHEAD, SocketDecoder, ops
    B, N = a.batch, 32768
    q, K, V = datagen.torch_make_cache(B, 32, 8, N, 128, seed=1)
    W = torch.from_numpy(datagen.make_projections(4242, 60, 8, 128).view("int16")).cuda().view(torch.bfloat16)
    cfg = Config(B=B, H_q=32, H_kv=8, N_max=N, group_mode=PER_QHEAD)
    lens = torch.full((B,), N, dtype=torch.int32, device="cuda")
    dec = SocketDecoder(cfg, W, K, V, k=3277)
    dec.prefill()
    sc = ops.score(cfg, q, W, dec.codes, dec.vnorm, lens)
    u = torch.rand((B, 32, a.M), device="cuda")
    for _ in range(3):
        ops.sample_decode(cfg, sc, dec.vnorm, V, lens, u)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (1024 * 8))()
    assert L.socket_debug_sample_trace(buf, 1024 * 8) == 0
    t = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 8).astype(np.int64)
    t = t[t[:, 0] != 0]
    names = ["sort", "segment sums + scan", "targets + walk", "gather + reduce"]
    print(f"rows {len(t)}: total cycles median {np.median(t[:, 4] - t[:, 0]):.0f}")
    for i, nm in enumerate(names):
        d = t[:, i + 1] - t[:, i]
        print(f"   {nm:22s} median {np.median(d):8.0f} max {np.max(d):8.0f}")


if __name__ == "__main__":
    main()
