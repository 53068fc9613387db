import sys, os, torch, time
sys.path.insert(0, os.getcwd())
import datagen
from paper_2602_06283_b200 import Config, SocketDecoder
B, N = int(sys.argv[1]), 32768
q, K, V = datagen.torch_make_cache(B, 32, 8, N, 128, seed=1)
W = torch.from_numpy(datagen.make_projections(4242, 60, 8, 128).view("int16")).cuda().view(torch.bfloat16)
lens = torch.full((B,), N, dtype=torch.int32, device="cuda")
cfg = Config(B=B, H_q=32, H_kv=8, N_max=N)
dec = SocketDecoder(cfg, W, K, V, k=3277); dec.prefill()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def timeit(fn, n=20):
    for _ in range(5): flush.zero_(); fn()
    torch.cuda.synchronize(); tot = 0
    for _ in range(n):
        flush.zero_(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize(); tot += e0.elapsed_time(e1)
    return tot / n * 1e3
dec.capture(q, lens, append=True)
print("device graph", timeit(dec.replay))
qh, kh, vh, oh = dec.bind_host(lens)
print("host graph packed", timeit(dec.host_step))
# raw copies only
hb = torch.empty(328 * 1024 // 2, dtype=torch.bfloat16).pin_memory(); db = torch.empty_like(hb, device="cuda")
ob = torch.empty(64 * 1024, dtype=torch.bfloat16).pin_memory(); dob = torch.empty_like(ob, device="cuda")
print("H2D 328KB + D2H 128KB", timeit(lambda: (db.copy_(hb, non_blocking=True), ob.copy_(dob, non_blocking=True))))
# isolate: device-side step with k_new/v_new (no copies)
kd = K[:, :, N - 1].contiguous(); vd = V[:, :, N - 1].contiguous()
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    dec.step(q, lens, append=True, k_new=kd, v_new=vd)
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    dec.step(q, lens, append=True, k_new=kd, v_new=vd)
print("device graph + k_new", timeit(g.replay))
# H2D + step (no D2H)
g2 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g2):
    db.copy_(hb, non_blocking=True)
    dec.step(q, lens, append=True, k_new=kd, v_new=vd)
print("H2D + step", timeit(g2.replay))
g3 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g3):
    dec.step(q, lens, append=True, k_new=kd, v_new=vd)
    ob.copy_(dob, non_blocking=True)
print("step + D2H", timeit(g3.replay))
