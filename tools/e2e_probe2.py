import sys, os, torch
sys.path.insert(0, os.getcwd())
import datagen
from paper_2602_06283_b200 import Config, SocketDecoder, ops
B, N = 16, 32768
q, K, V = datagen.torch_make_cache(B, 32, 8, N, 128, seed=1)
W = torch.from_numpy(datagen.make_projections(4242, 60, 8, 128).view("int16")).cuda().view(torch.bfloat16)
lens = torch.full((B,), N, dtype=torch.int32, device="cuda")
cfg = Config(B=B, H_q=32, H_kv=8, N_max=N)
dec = SocketDecoder(cfg, W, K, V, k=3277); dec.prefill()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
kd = K[:, :, N - 1].contiguous(); vd = V[:, :, N - 1].contiguous()
def timeit(fn, n=20, fl=True):
    for _ in range(5):
        if fl: flush.zero_()
        fn()
    torch.cuda.synchronize(); tot = 0
    for _ in range(n):
        if fl: flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize(); tot += e0.elapsed_time(e1)
    return tot / n * 1e3
def graph(fn):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s): fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g): fn()
    return g
g0 = graph(lambda: dec.step(q, lens, append=True))
g1 = graph(lambda: dec.step(q, lens, append=True, k_new=kd, v_new=vd))
g2 = graph(lambda: (K[:, :, N - 1].copy_(kd), V[:, :, N - 1].copy_(vd), dec.step(q, lens, append=True)))
for name, g in (("plain", g0), ("k_new", g1), ("copy+plain", g2)):
    print(name, "flush", round(timeit(g.replay), 1), "noflush", round(timeit(g.replay, fl=False), 1))
print("eager plain", round(timeit(lambda: dec.step(q, lens, append=True)), 1))
print("eager k_new", round(timeit(lambda: dec.step(q, lens, append=True, k_new=kd, v_new=vd)), 1))
