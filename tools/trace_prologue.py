"""Phase timing of the decode-step prologue (tables || append CTAs) from
in-kernel stamps (PRO_STAMP in csrc/step_dev.cuh).

    python tools/trace_prologue.py [--batch 16] [--ctx 32768]

Builds the -DSK_TRACE library (build/trace/; the product library is untouched),
runs socket_decode_step on the bench workload and prints, for table CTAs and
append CTAs separately, the median / max cycles of each phase, and the spread
of CTA start times (globaltimer, ns) -- i.e. whether the grid ran as one wave.
"""
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

TAB = ["entry", "staging", "projection", "sigma", "half tables", "LUT write"]
APP = ["entry", "staging", "projection", "(none)", "(none)", "code+norm"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--ctx", type=int, default=32768)
    a = ap.parse_args()
    libpath = build_trace()
    from paper_2602_06283_b200 import _lib
    _lib.LIB_PATH = libpath
    L = _lib.lib()
    import datagen
    from paper_2602_06283_b200 import Config, SocketDecoder
    B, N = a.batch, a.ctx
    q, K, V = datagen.torch_make_cache(B, 32, 8, N, 128, seed=1)
    W = torch.from_numpy(datagen.make_projections(4242, 60, 8, 128).view("int16")).cuda().view(torch.bfloat16)
    cfg = Config(B=B, H_q=32, H_kv=8, N_max=N, L=60, P=8, tau=0.5)
    lens = torch.full((B,), N, dtype=torch.int32, device="cuda")
    dec = SocketDecoder(cfg, W, K, V, k=N // 10)
    dec.prefill()
    for _ in range(3):
        dec.step(q, lens, append=True)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (8192 * 12))()
    assert L.socket_debug_prologue_trace(buf, 8192 * 12) == 0
    t = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 12).astype(np.int64)
    n_tab = (B * 32 + 15) // 16 * 8
    for name, rows, ph in (("tables", t[:n_tab], TAB), ("append", t[n_tab:], APP)):
        rows = rows[rows[:, 0] != 0]
        if not len(rows):
            continue
        st = rows[:, 0] - t[t[:, 0] != 0, 0].min()
        print(f"{name}: {len(rows)} CTAs, start spread (ns) median {np.median(st):.0f} max {st.max():.0f}; "
              f"CTAs per SM max {np.bincount(rows[:, 11]).max()}")
        tot = rows[:, 6] - rows[:, 1]
        print(f"   total cycles median {np.median(tot):.0f} max {tot.max():.0f}")
        for i in range(1, 6):
            ok = (rows[:, i + 1] != 0) & (rows[:, i] != 0)
            d = rows[ok, i + 1] - rows[ok, i]
            if d.size and ph[i] != "(none)":
                print(f"   {ph[i]:12s} median {np.median(d):8.0f}  max {np.max(d):8.0f} cycles")


if __name__ == "__main__":
    main()
