"""Benchmark of the SOCKET decode hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--layout kv_head|seq|replicas] [--batch B] [--ctx N]
                    [--sparsity S] [--tables L] [--bits P]

A step is one SOCKET decode step of one attention layer over the whole batch:
  append-hash of the new key (Alg. 1) -> query tables (Alg. 2) -> soft-collision
  scores (Eq. 4 / Alg. 4) -> top-k (Alg. 3) -> sparse flash-decode + split LSE
  combine (Eq. 2)
on a Llama-3.1-8B-shaped cache (32 q / 8 KV heads, d = 128), L = 60, P = 8,
tau = 0.5, KV-shared selection.  Layouts (BASELINE.json configs, DESIGN.md
"Multi-GPU"), one process per GPU under torchrun:
  kv_head  (default) configs[1] workload (32K, batch 16, 10x) -- configs[2] with
           --ctx 131072 --batch 8: rank g owns KV heads [g 8/N, (g+1) 8/N) and
           their query heads; no collective; tokens/s = B / max-rank step time
           (strong scaling: the workload is fixed).
  seq      configs[3]: 1M-token context (batch 1, 10x), sequence-sharded: rank s
           owns 2^20/N tokens; the exact global top-k exchange (digest + window
           rounds) and the partial-state all-gather run over NCCL inside the
           CUDA graph of the step (strong scaling).
  replicas every rank runs the full configs[1] workload on its own batch (weak
           scaling; labelled extra).
L2 is flushed (256 MB memset) before every timed step.

--impl reference times the CPU oracle (oracle/, float64 numpy) on the same
workload: full steps when they fit the run, else a labelled sample of (b, kv
head) units.  Prints exactly one JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sparse-decode tokens/s at 32K/128K ctx vs dense; score+attn HBM GB/s vs peak"

# dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernels
# at the default workload, from the committed ncu --set full capture
# (profiles/<round>/traffic.json); None = not captured for this configuration.
TRAFFIC = {}
for _r in ("r2", "r1"):
    try:
        _t = json.load(open(os.path.join(ROOT, "profiles", _r, "traffic.json")))
        TRAFFIC = {k: v for k, v in _t.items() if isinstance(v, (int, float))}
        break
    except Exception:
        pass

PAPER_CONTEXT = ("paper (P:701, A100/H200, GPT-FAST, Llama-2-7b single layer, batch 1, 33x sparsity): "
                 "1.12x over FlashAttention at 36K, 1.26x at 72K, up to 1.5x at 145K on H200; "
                 "1.19x / 1.3x / 1.52x at 18K / 36K / 72K on A100 -- other hardware, context only")

LAYOUT_DEFAULTS = {"kv_head": (16, 32768, 10.0), "replicas": (16, 32768, 10.0), "seq": (1, 1 << 20, 10.0)}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layout", default="kv_head", choices=["kv_head", "seq", "replicas"])
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--ctx", type=int, default=None)
    ap.add_argument("--sparsity", type=float, default=None)
    ap.add_argument("--tables", type=int, default=60)
    ap.add_argument("--bits", type=int, default=8)
    ap.add_argument("--tau", type=float, default=0.5)
    ap.add_argument("--mode", default="kv_shared", choices=["kv_shared", "per_qhead"])
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-rows", action="store_true", help="skip the NEXT-row measurements")
    ap.add_argument("--no-b1", action="store_true", help="skip the batch-1 context x sparsity rows")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    a = ap.parse_args()
    b, c, s = LAYOUT_DEFAULTS[a.layout]
    a.batch = b if a.batch is None else a.batch
    a.ctx = c if a.ctx is None else a.ctx
    a.sparsity = s if a.sparsity is None else a.sparsity
    return a


def workload(a):
    k = int(round(a.ctx / a.sparsity))
    base = {"kv_head": "BASELINE configs[1]" if a.ctx <= 65536 else "BASELINE configs[2]",
            "replicas": "BASELINE configs[1] (replicas)", "seq": "BASELINE configs[3]"}[a.layout]
    return {
        "workload": f"llama3.1-8b-shaped decode attention (32q/8kv, d=128), ctx {a.ctx}, "
                    f"batch {a.batch}, {a.sparsity:g}x sparsity (k={k}), L={a.tables}, P={a.bits}, "
                    f"tau={a.tau}, {a.mode} selection; {base}",
        "layout": a.layout, "batch": a.batch, "ctx": a.ctx, "k": k, "L": a.tables, "P": a.bits,
        "tau": a.tau, "H_q": 32, "H_kv": 8, "d": 128, "selection": a.mode,
        "l2": "flushed (256 MB memset) before every timed step",
    }, k


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.t.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace('.', '').isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace('.', '').isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) > 8:
                for n, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], "measured (MEASURED_PEAKS.json copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# CPU oracle (reference arm / cpu_baseline)
# ---------------------------------------------------------------------------
class OracleStep:
    """One decode step of the workload on the CPU oracle, as (b, kv-head) units:
    append-hash of the newest key, tables, scores, top-k and the attention of
    the unit's query heads (oracle.decode_step on that unit).  The index (Alg. 1
    over the cache) is prefill, built once untimed."""

    def __init__(self, a, k):
        import datagen
        import oracle as O
        self.O, self.a, self.k = O, a, k
        N, L, P = a.ctx, a.tables, a.bits
        c = datagen.make_case(1, 4, 1, N, 128, seed=123)
        self.c = c
        self.Wb = datagen.make_projections(4242, L, P, 128)
        self.codes, _ = O.hash_keys(O.widen(c["K"]), O.widen(self.Wb))   # prefill, untimed
        self.mode = O.GROUP_KV_SHARED if a.mode == "kv_shared" else O.GROUP_PER_QHEAD
        self.units_per_step = a.batch * 8

    def unit(self):
        O, c, N = self.O, self.c, self.a.ctx
        kn, _ = O.hash_keys(O.widen(c["K"][0, 0, N - 1:N]), O.widen(self.Wb))
        self.codes[0, 0][:, N - 1:N] = kn
        rows = [(0, 0)] if self.mode == O.GROUP_KV_SHARED else [(0, h) for h in range(4)]
        O.decode_step(c["q"], c["K"], c["V"], self.Wb, c["seq_lens"], tau=self.a.tau, k=self.k,
                      sm_scale=1 / math.sqrt(128), group_mode=self.mode, codes=self.codes, rows=rows)

    def run(self, units):
        """Time `units` units; returns (wall s, cores actually used = cpu s / wall s)."""
        c0, t0 = time.process_time(), time.perf_counter()
        for _ in range(units):
            self.unit()
        wall = time.perf_counter() - t0
        return wall, (time.process_time() - c0) / max(wall, 1e-9)


def oracle_baseline(a, k, steps, warmup, budget_s):
    """Reference timing: full steps when steps x (one step) fits budget_s, else
    each step is a sample of units (labelled, extrapolated)."""
    st = OracleStep(a, k)
    w1, _ = st.run(1)                                   # warm-up + estimate
    est_step = w1 * st.units_per_step
    full = est_step * steps <= budget_s
    per = st.units_per_step if full else max(1, int(budget_s / max(steps, 1) / max(w1, 1e-6)))
    per = min(per, st.units_per_step)
    for _ in range(max(0, warmup - 1)):
        st.run(1)
    walls, cores = [], []
    for _ in range(steps):
        w, c = st.run(per)
        walls.append(w)
        cores.append(c)
    t_step = statistics.mean(walls) * st.units_per_step / per
    sample = (f"{'full steps' if full else 'sampled steps'}: {steps} timed step(s) of {per} of the "
              f"{st.units_per_step} (b, kv-head) units each (numpy float64"
              f"{'' if full else '; step time extrapolated x' + format(st.units_per_step / per, '.1f')}); "
              f"warm-up {warmup} x 1 unit; CPU {cpu_model()}, os.cpu_count() = {os.cpu_count()}")
    return {"value": a.batch / t_step, "unit": "tokens/s", "cores": round(statistics.mean(cores), 2),
            "kind": "oracle", "sample": sample, "ms_per_step": t_step * 1e3,
            "extrapolated": not full, "units_timed_per_step": per, "units_per_step": st.units_per_step,
            "cpu_model": cpu_model()}


def run_reference(a):
    """Reference arm of this tier: the CPU oracle, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg, k = workload(a)
    cb = oracle_baseline(a, k, a.steps, a.warmup, budget_s=150.0)
    line = {"metric": METRIC, "value": cb["value"], "unit": "tokens/s", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": cb["ms_per_step"],
            "higher_is_better": True, "scaling": "strong" if a.layout != "replicas" else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg, "impl": "reference",
            "cpu_baseline": {k2: cb[k2] for k2 in ("value", "unit", "cores", "kind", "sample")},
            "extrapolated": cb["extrapolated"], "units_timed_per_step": cb["units_timed_per_step"],
            "e2e": {"value": cb["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    emit_line(line)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def algorithmic_bytes(B, N, L, P, k, H_q=32, H_kv=8, H_sel=8):
    """Per-step algorithmic bytes by stage."""
    cb = L * ((P + 7) // 8)
    return {
        "score": B * H_kv * N * (cb + 4) + B * H_sel * N * 4,      # codes + norms read, scores written
        "topk": B * H_sel * N * 4 + B * H_sel * k * 4,              # scores read, idx written
        "sparse_decode": B * H_sel * k * (2 * 128 * 2 + 4)      # gathered K/V rows + idx
        + B * H_q * 128 * 2 * 2,                                    # q in, out written
    }


def _time(fn, flush, stream, warmup, steps):
    import torch
    for _ in range(warmup):
        flush.zero_()
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / steps


class Ctx:
    """Process-group plumbing of one bench process."""

    def __init__(self, need_pg):
        import torch
        import torch.distributed as dist
        self.dist = dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        self.pg = False
        if self.world > 1 or need_pg:
            if self.world == 1:
                os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
                os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
                os.environ.setdefault("RANK", "0")
                os.environ.setdefault("WORLD_SIZE", "1")
            dist.init_process_group("nccl", device_id=self.dev)
            self.pg = True

    def barrier(self):
        import torch
        if self.pg:
            self.dist.barrier()
        torch.cuda.synchronize()

    def max(self, x):
        import torch
        if not self.pg:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.item()

    def gather_float(self, x):
        import torch
        if not self.pg:
            return [x]
        t = torch.tensor([x], dtype=torch.float64, device=self.dev)
        out = [torch.zeros_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t)
        return [o.item() for o in out]

    def close(self):
        if self.pg:
            self.dist.destroy_process_group()


def timed_replay(ctx, replay, flush, stream, a):
    """The headline timing: W untimed steps, then K steps each bracketed by CUDA
    events on the launching stream with the L2 flushed before, barrier +
    synchronize on both sides, nvidia-smi clocks sampled during the region."""
    import torch
    for _ in range(a.warmup):
        flush.zero_()
        replay()
    ctx.barrier()
    clocks = Clocks(ctx.local)
    clocks.start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(a.steps)]
    for e0, e1 in evs:
        flush.zero_()
        e0.record(stream)
        replay()
        e1.record(stream)
    ctx.barrier()
    clk = clocks.stop()
    step_ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / a.steps
    return step_ms, clk


def run_ours(a):
    import torch
    ctx = Ctx(need_pg=a.layout == "seq")
    try:
        line = run_seq(a, ctx) if a.layout == "seq" else run_heads(a, ctx)
        if ctx.rank == 0:
            emit_line(line)
    finally:
        torch.cuda.synchronize()
        ctx.close()


def _common_line(a, ctx, cfgd, value, step_ms, clk, launches):
    return {
        "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": ctx.world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(step_ms, 5),
        "higher_is_better": True, "scaling": "weak" if a.layout == "replicas" else "strong",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded N(0,1) bf16 q/K/V and projections)", "config": cfgd,
        "gpu_launches": launches, "clocks": clk, "paper_context": PAPER_CONTEXT,
        "projection_32_layers": {
            "tokens_per_s": round(value / 32, 1),
            "note": "projection, not measured: 32 attention layers of Llama-3.1-8B at this step time "
                    "(attention only; no MLP, no weights)"},
    }


def run_heads(a, ctx):
    """kv_head (default) and replicas layouts."""
    import torch

    import datagen
    from paper_2602_06283_b200 import Config, KV_SHARED, PER_QHEAD, SocketDecoder, ops
    from paper_2602_06283_b200 import _lib
    from paper_2602_06283_b200.dist import kv_head_shard_config

    cfgd, k = workload(a)
    B, N, L, P = a.batch, a.ctx, a.tables, a.bits
    dev = ctx.dev
    mode = KV_SHARED if a.mode == "kv_shared" else PER_QHEAD
    full = Config(B=B, H_q=32, H_kv=8, N_max=N, L=L, P=P, tau=a.tau, group_mode=mode)
    if a.layout == "kv_head":
        cfg = kv_head_shard_config(full, ctx.world, ctx.rank)
        par = (f"kv-head shard x{ctx.world}: {cfg.H_kv} KV heads / {cfg.H_q} q heads per rank, "
               f"no collective")
    else:
        cfg = full
        par = f"batch replicas x{ctx.world} (every rank the full workload; labelled extra)"
    q, K, V = datagen.torch_make_cache(B, cfg.H_q, cfg.H_kv, N, 128, seed=1000 + ctx.rank, device=dev)
    W = torch.from_numpy(datagen.make_projections(4242, L, P, 128).view("int16")).to(dev).view(torch.bfloat16)
    lens = torch.full((B,), N, dtype=torch.int32, device=dev)
    dec = SocketDecoder(cfg, W, K, V, k=k)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dec.prefill()
    torch.cuda.synchronize()
    prefill_s = time.perf_counter() - t0
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    # prefill key hashing (Alg. 1) on the tensor cores: codes only (the GEMM)
    pre_ms = _time(lambda: ops.hash_keys(cfg, K, W, dec.codes, n_begin=0, n_count=N), flush, stream, 2, 5)
    pre_flops = 2.0 * B * cfg.H_kv * N * 128 * L * P
    try:
        bf16_peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
    except Exception:
        bf16_peak = 1654.9
    prefill = {"kernel": "hash_keys_tc2_kernel (tcgen05)", "ms": round(pre_ms, 4),
               "TFLOP/s": round(pre_flops / (pre_ms * 1e-3) / 1e12, 1),
               "frac_of_bf16_peak": round(pre_flops / (pre_ms * 1e-3) / 1e12 / bf16_peak, 4),
               "keys": B * cfg.H_kv * N, "flops": pre_flops}

    # ---- (1) graph-replayed step: headline ---------------------------------------
    dec.capture(q, lens, append=True)
    step_ms, clk = timed_replay(ctx, dec.replay, flush, stream, a)
    step_ms_rank = step_ms
    step_ms = ctx.max(step_ms)
    launches_per_step = ops.decode_step_launches(cfg)

    # ---- (2) per-kernel timing (each stage's call R times back to back) -----------
    stage_names = ["append_hash", "tables", "score", "topk", "sparse_decode"]
    lut = ops.workspace(cfg, _lib.OP_SCORE, 1, dev)
    ops.build_lut(cfg, q, W, lut)
    calls = {
        "append_hash": lambda: ops.hash_keys(cfg, K, W, dec.codes, V=V, vnorm=dec.vnorm,
                                             n_begin=N - 1, n_count=1),
        "tables": lambda: ops.build_lut(cfg, q, W, lut),
        "score": lambda: ops.score_lut(cfg, lut, dec.codes, dec.vnorm, lens, out=dec.scores),
        "topk": lambda: ops.topk(cfg, dec.scores, lens, k, idx=dec.idx, cnt=dec.cnt),
        "sparse_decode": lambda: ops.sparse_decode(cfg, q, K, V, dec.idx, dec.cnt, k, out=dec.out,
                                                   lse=dec.lse, ws=dec.ws_dec),
    }
    R = 10
    stage_ms = {}
    for s_ in stage_names:
        fn = calls[s_]
        for _ in range(a.warmup):
            fn()
        tot = 0.0
        reps = max(1, a.steps // 5)
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(R):
                fn()
            e1.record(stream)
            e1.synchronize()
            tot += e0.elapsed_time(e1) / R
        stage_ms[s_] = tot / reps
    eager_ms = sum(stage_ms.values())
    ab = algorithmic_bytes(B, N, L, P, k, H_q=cfg.H_q, H_kv=cfg.H_kv, H_sel=cfg.H_sel)
    hbm, peak_src = peaks()
    stages = {}
    for s_ in ("score", "topk", "sparse_decode"):
        gbs = ab[s_] / (stage_ms[s_] * 1e-3) / 1e9
        stages[s_] = {"ms": round(stage_ms[s_], 5), "alg_bytes": ab[s_], "GB/s": round(gbs, 1),
                      "frac": round(gbs / hbm, 4), "share": round(stage_ms[s_] / eager_ms, 4)}
    for s_ in ("append_hash", "tables"):
        stages[s_] = {"ms": round(stage_ms[s_], 5), "share": round(stage_ms[s_] / eager_ms, 4)}
    dom = max(("score", "sparse_decode"), key=lambda s_: stage_ms[s_])
    kern = {"score": "score_reg_kernel", "sparse_decode": "decode_mma_kernel"}[dom]
    roof = {"bound": "hbm", "kernel": kern, "achieved": stages[dom]["GB/s"], "peak": hbm,
            "unit": "GB/s", "frac": stages[dom]["frac"],
            "traffic": TRAFFIC.get(kern) if (a.layout == "replicas" or ctx.world == 1) and
            (B, N, a.sparsity) == (16, 32768, 10.0) else None,
            "peak_source": peak_src,
            "algorithmic": f"{dom}: {ab[dom]} B per launch (DESIGN.md section 4 per-unit bytes x units)"}
    step_bytes = ab["score"] + ab["topk"] + ab["sparse_decode"]
    per_rank_frac = ctx.gather_float(step_bytes / (step_ms_rank * 1e-3) / 1e9 / hbm)

    # ---- (3) dense comparators on the same cache ---------------------------------
    dense = {} if a.no_dense else dense_baselines(a, cfg, q, K, V, lens, flush, stream)

    # ---- (3b) batch-1 rows (the paper's protocol) and SURVEY 8(f) rows -----
    b1 = {} if (a.no_b1 or ctx.world > 1 or a.layout != "kv_head") else b1_rows(a, flush, stream, dev)
    rows = {}
    if not a.no_rows and ctx.world == 1:
        rows = next_rows(a, cfg, dec, q, K, V, W, lens, k, flush, stream, dev, hbm)

    # ---- (4) end to end through the public API with host buffers -----------------
    e2e = end_to_end(a, cfg, dec, q, K, V, lens, N, flush, stream, dev)
    e2e_ms = ctx.max(e2e["ms"])

    if ctx.rank != 0:
        return None
    value = B / (step_ms * 1e-3) * (ctx.world if a.layout == "replicas" else 1)
    cpu = oracle_baseline(a, k, 1, 1, budget_s=a.cpu_seconds) if ctx.world == 1 else None
    cfgd.update({"prefill_hash_s": round(prefill_s, 3), "parallelism": par})
    line = _common_line(a, ctx, cfgd, value, step_ms, clk, launches_per_step * a.steps)
    line.update({
        "roofline": roof, "stages": stages, "eager_ms_per_step": round(eager_ms, 5),
        "step_hbm": {"alg_bytes_per_rank": step_bytes,
                     "frac_per_rank": [round(x, 4) for x in per_rank_frac]},
        "prefill": prefill,
        "e2e": {"value": round(B / (e2e_ms * 1e-3) * (ctx.world if a.layout == "replicas" else 1), 1),
                "unit": "tokens/s", "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"]},
    })
    if dense:
        best = min(dense.items(), key=lambda kv: kv[1]["ms"])
        line["dense"] = {"best": best[0], "ms_per_step": best[1]["ms"], "all": dense,
                         "speedup_sparse_vs_dense": round(best[1]["ms"] / step_ms, 3),
                         "note": "rank 0's shard" if ctx.world > 1 else "same cache"}
    if b1:
        line["batch1"] = b1
    if rows:
        line["next_rows"] = rows
    if cpu:
        line["cpu_baseline"] = {k2: cpu[k2] for k2 in ("value", "unit", "cores", "kind", "sample")}
    return line


def run_seq(a, ctx):
    """configs[3]: sequence-sharded 1M-token context, exact global top-k over NCCL."""
    import torch

    import datagen
    from paper_2602_06283_b200 import Config, ops
    from paper_2602_06283_b200 import _lib
    from paper_2602_06283_b200.dist import MAX_WINDOW_ROUNDS, SeqShardDecoder, seq_shard_config, _gather

    cfgd, k = workload(a)
    B, N, L, P = a.batch, a.ctx, a.tables, a.bits
    dev = ctx.dev
    full = Config(B=B, H_q=32, H_kv=8, N_max=N, L=L, P=P, tau=a.tau)
    cfg = seq_shard_config(full, ctx.world, ctx.rank)
    Ns = cfg.N_max
    g = torch.Generator(device=dev).manual_seed(2000)
    q = torch.randn((B, 32, 128), generator=g, device=dev).to(torch.bfloat16)     # same q on every rank
    _, K, V = datagen.torch_make_cache(B, 32, 8, Ns, 128, seed=3000 + ctx.rank, device=dev)
    W = torch.from_numpy(datagen.make_projections(4242, L, P, 128).view("int16")).to(dev).view(torch.bfloat16)
    lens = torch.full((B,), N, dtype=torch.int32, device=dev)                      # total lengths
    sd = SeqShardDecoder(cfg, W, K, V, k)
    sd.prefill()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sd.capture(q, lens)
    step_ms, clk = timed_replay(ctx, sd.replay, flush, stream, a)
    step_ms_rank = step_ms
    step_ms = ctx.max(step_ms)

    # per-kernel times of this rank's step (eager, back to back)
    sh = sd.shard
    hbm, peak_src = peaks()
    dig = ops.topk_digest(cfg, sh.scores, lens, k, ctx.world, sh.Q)
    msg = ops.topk_window(cfg, sh.scores, lens, sh.state)
    calls = {
        "score": lambda: ops.score(cfg, q, W, sh.codes, sh.vnorm, lens, out=sh.scores),
        "digest": lambda: ops.topk_digest(cfg, sh.scores, lens, k, ctx.world, sh.Q, digest=dig),
        "window": lambda: ops.topk_window(cfg, sh.scores, lens, sh.state, msg=msg),
        "emit": lambda: ops.topk_emit(cfg, sh.scores, lens, k, sh.state, idx=sh.idx, cnt=sh.cnt),
        "sparse_decode": lambda: ops.sparse_decode(cfg, q, K, V, sh.idx, sh.cnt, k, partial=sh.part,
                                                   want_out=False),
    }
    stage_ms = {n_: _time(f, flush, stream, 2, max(3, a.steps // 4)) for n_, f in calls.items()}
    k_loc = int(sh.cnt.sum().item()) // max(1, cfg.B * cfg.H_sel)      # this rank's share per row
    ab = algorithmic_bytes(B, Ns, L, P, max(1, k_loc), H_sel=cfg.H_sel)
    stages = {}
    for s_, key in (("score", "score"), ("sparse_decode", "sparse_decode")):
        gbs = ab[key] / (stage_ms[s_] * 1e-3) / 1e9
        stages[s_] = {"ms": round(stage_ms[s_], 5), "alg_bytes": ab[key], "GB/s": round(gbs, 1),
                      "frac": round(gbs / hbm, 4)}
    for s_ in ("digest", "window", "emit"):
        stages[s_] = {"ms": round(stage_ms[s_], 5)}
    roof = {"bound": "hbm", "kernel": "score_reg_kernel", "achieved": stages["score"]["GB/s"], "peak": hbm,
            "unit": "GB/s", "frac": stages["score"]["frac"], "traffic": None, "peak_source": peak_src,
            "algorithmic": f"score: {ab['score']} B per launch per rank ({Ns} keys x 8 kv heads x (L + 4) "
                           f"+ 4 B score per key)"}
    # the step's collectives alone: digest, window rounds, partials (NCCL all-gathers)
    bufs = [torch.zeros((B, 8, sh.Q, 2), dtype=torch.int32, device=dev)] + \
           [torch.zeros((B, 8, _lib.TOPK_MSG_WORDS), dtype=torch.int32, device=dev)] * MAX_WINDOW_ROUNDS + \
           [torch.zeros((B, 32, 130), dtype=torch.float32, device=dev)]
    sent = sum(t.numel() * t.element_size() for t in bufs)
    coll_ms = _time(lambda: [_gather(t) for t in bufs], flush, stream, 2, max(3, a.steps // 4))
    per_rank = ctx.gather_float((ab["score"] + ab["sparse_decode"]) / (step_ms_rank * 1e-3) / 1e9 / hbm)

    # end to end: q from pinned host memory, out back to pinned host memory
    q_h = q.cpu().pin_memory()
    out_h = torch.empty((B, 32, 128), dtype=torch.bfloat16).pin_memory()

    def host_step():
        q.copy_(q_h, non_blocking=True)
        sd.replay()
        out_h.copy_(sd.out, non_blocking=True)
    e2e_ms = ctx.max(_time(host_step, flush, stream, a.warmup, a.steps))

    dense = {}
    if ctx.world == 1 and not a.no_dense:
        qq = q.view(B, 32, 1, 128)
        f = lambda: torch.nn.functional.scaled_dot_product_attention(qq, K, V, scale=cfg.scale, enable_gqa=True)
        dense["torch_sdpa"] = {"ms": round(_time(f, flush, stream, a.warmup, a.steps), 5)}
        ws = ops.workspace(full, _lib.OP_DENSE_DECODE, 1, dev)
        dense["ours_dense_split_kv"] = {"ms": round(_time(lambda: ops.dense_decode(full, q, K, V, lens, ws=ws),
                                                          flush, stream, a.warmup, a.steps), 5)}
    if ctx.rank != 0:
        return None
    value = B / (step_ms * 1e-3)
    cpu = None
    if ctx.world == 1:
        cpu = oracle_seq_baseline(a, k)
    cfgd.update({"parallelism": f"sequence shard x{ctx.world}: {Ns} tokens per rank, exact global top-k "
                                f"(digest + {MAX_WINDOW_ROUNDS} window rounds) + partial all-gather over NCCL, "
                                f"captured in the step's CUDA graph"})
    # launches per step: score (2: tables + score), digest, bracket, 3 x (window, resolve), emit, decode (+ combine)
    launches = 2 + 1 + 1 + 2 * MAX_WINDOW_ROUNDS + 1 + 1 + 1
    line = _common_line(a, ctx, cfgd, value, step_ms, clk, launches * a.steps)
    line.update({
        "roofline": roof, "stages": stages,
        "collectives": {"all_gathers_per_step": 2 + MAX_WINDOW_ROUNDS, "bytes_sent_per_rank": sent,
                        "bytes_received_per_rank": sent * ctx.world, "ms_alone": round(coll_ms, 5),
                        "share_of_step": round(coll_ms / step_ms, 4)},
        "step_hbm": {"frac_per_rank": [round(x, 4) for x in per_rank]},
        "e2e": {"value": round(B / (e2e_ms * 1e-3), 1), "unit": "tokens/s",
                "h2d_bytes_per_step": q_h.numel() * 2, "d2h_bytes_per_step": out_h.numel() * 2},
    })
    if dense:
        best = min(dense.items(), key=lambda kv: kv[1]["ms"])
        line["dense"] = {"best": best[0], "ms_per_step": best[1]["ms"], "all": dense,
                         "speedup_sparse_vs_dense": round(best[1]["ms"] / step_ms, 3)}
    if cpu:
        line["cpu_baseline"] = cpu
    return line


def oracle_seq_baseline(a, k):
    """cpu_baseline of the seq layout: one (b, kv head) unit of a 1M-token row
    costs the oracle seconds (scores of 2^20 keys, a 2^20-key sort), so the
    sample is a shorter 131072-key row (one shard's worth), scaled by keys."""
    import copy
    b = copy.copy(a)
    b.ctx, b.batch = 131072, 1
    r = oracle_baseline(b, int(round(b.ctx / a.sparsity)), 1, 1, budget_s=a.cpu_seconds)
    scale = a.ctx / b.ctx
    return {"value": r["value"] / scale, "unit": "tokens/s", "cores": r["cores"], "kind": "oracle",
            "sample": r["sample"] + f"; sampled on a {b.ctx}-key row and scaled x{scale:g} to {a.ctx} keys"}


def b1_rows(a, flush, stream, dev):
    """Batch 1 at 32K / 64K / 128K x 5 / 10 / 33x sparsity (the paper's protocol:
    single layer, batch 1): our graph-replayed step vs the best
    dense decode on the same cache."""
    import torch

    import datagen
    from paper_2602_06283_b200 import Config, SocketDecoder, ops
    out = {}
    W = torch.from_numpy(datagen.make_projections(4242, a.tables, a.bits, 128).view("int16")).to(dev).view(torch.bfloat16)
    for N in (32768, 65536, 131072):
        q, K, V = datagen.torch_make_cache(1, 32, 8, N, 128, seed=7, device=dev)
        lens = torch.full((1,), N, dtype=torch.int32, device=dev)
        cfg = Config(B=1, H_q=32, H_kv=8, N_max=N, L=a.tables, P=a.bits, tau=a.tau)
        dense = dense_baselines(a, cfg, q, K, V, lens, flush, stream)
        best = min(dense.items(), key=lambda kv: kv[1]["ms"])
        row = {"dense_best": best[0], "dense_ms": best[1]["ms"]}
        for sp in (5, 10, 33):
            k = int(round(N / sp))
            dec = SocketDecoder(cfg, W, K, V, k=k)
            dec.prefill()
            dec.capture(q, lens, append=True)
            ms = _time(dec.replay, flush, stream, a.warmup, a.steps)
            row[f"{sp}x"] = {"ms": round(ms, 5), "tokens_per_s": round(1 / (ms * 1e-3), 1),
                             "speedup_vs_dense": round(best[1]["ms"] / ms, 3),
                             "launches": ops.decode_step_launches(cfg)}
            del dec
        out[f"{N // 1024}K"] = row
        del q, K, V
        torch.cuda.empty_cache()
    return out


def next_rows(a, cfg, dec, q, K, V, W, lens, k, flush, stream, dev, hbm):
    """SURVEY 8(f) rows on the bench cache, each timed like the headline (L2
    flushed before every step, CUDA events on the launching stream):
      hard_lsh  (f3): the step with Eq. 3 hard-LSH tables (scoring = 1);
      wide_codes(f2): the RULER setting L = 60, P = 10 (600 bits/token),
                      graph-replayed step; its score kernel's HBM rate;
      sampling  (f4): Eq. 6 sampling decode over PER_QHEAD rows, M = k draws."""
    import dataclasses

    import torch

    import datagen
    from paper_2602_06283_b200 import PER_QHEAD, SocketDecoder, ops
    from paper_2602_06283_b200 import _lib
    B, N = cfg.B, cfg.N_max
    out = {}
    # f3 -------------------------------------------------------------------------
    cfg_h = dataclasses.replace(cfg, scoring=1)
    dh = SocketDecoder(cfg_h, W, K, V, k=k)
    dh.codes, dh.vnorm = dec.codes, dec.vnorm            # same index, hard tables
    dh.capture(q, lens, append=True)
    ms = _time(dh.replay, flush, stream, a.warmup, a.steps)
    out["hard_lsh"] = {"ms_per_step": round(ms, 5), "tokens_per_s": round(B / (ms * 1e-3), 1),
                       "config": "same workload, scoring = hard (Eq. 3 collision counts x ||v||)"}
    del dh
    # f2 -------------------------------------------------------------------------
    Lw, Pw = 60, 10
    cfg_w = dataclasses.replace(cfg, L=Lw, P=Pw)
    Ww = torch.from_numpy(datagen.make_projections(4343, Lw, Pw, 128).view("int16")).to(dev).view(torch.bfloat16)
    dw = SocketDecoder(cfg_w, Ww, K, V, k=k)
    dw.prefill()
    dw.capture(q, lens, append=True)
    ms = _time(dw.replay, flush, stream, a.warmup, a.steps)
    lut = ops.workspace(cfg_w, _lib.OP_SCORE, 1, dev)
    ops.build_lut(cfg_w, q, Ww, lut)
    sms = _time(lambda: ops.score_lut(cfg_w, lut, dw.codes, dw.vnorm, lens, out=dw.scores),
                flush, stream, a.warmup, a.steps)
    code_bytes = ops.codes_bytes(cfg_w) // (B * cfg.H_kv * N)     # stored bytes per key
    sb = B * cfg.H_kv * N * (code_bytes + 4) + B * cfg_w.H_sel * N * 4
    out["wide_codes"] = {"ms_per_step": round(ms, 5), "tokens_per_s": round(B / (ms * 1e-3), 1),
                         "score_ms": round(sms, 5), "score_GB/s": round(sb / (sms * 1e-3) / 1e9, 1),
                         "score_frac": round(sb / (sms * 1e-3) / 1e9 / hbm, 4),
                         "stored_code_bits_per_token": code_bytes * 8,
                         "config": "L=60, P=10 (600 bits/token), graph-replayed step"}
    del dw, lut
    torch.cuda.empty_cache()
    # f4 -------------------------------------------------------------------------
    cfg_s = dataclasses.replace(cfg, group_mode=PER_QHEAD)
    sc = ops.score(cfg_s, q, W, dec.codes, dec.vnorm, lens)
    g = torch.Generator(device=dev).manual_seed(99)
    u = torch.rand((B, cfg.H_q, k), generator=g, device=dev)
    smp = torch.empty((B, cfg.H_q, k), dtype=torch.int32, device=dev)
    o = torch.empty((B, cfg.H_q, 128), dtype=torch.bfloat16, device=dev)
    ms = _time(lambda: ops.sample_decode(cfg_s, sc, dec.vnorm, V, lens, u, samples=smp, out=o),
               flush, stream, a.warmup, a.steps)
    ab = B * cfg.H_q * (N * 8 + k * (4 + 4 + 256 + 4) + 256)
    out["sampling"] = {"ms": round(ms, 5), "GB/s": round(ab / (ms * 1e-3) / 1e9, 1),
                       "frac": round(ab / (ms * 1e-3) / 1e9 / hbm, 4), "M": k,
                       "config": "Eq. 6 over PER_QHEAD rows (B x 32), M = k draws; "
                                 "bytes = scores + norms per row + per draw (u, J, v row, norm)"}
    del sc
    return out


def dense_baselines(a, cfg, q, K, V, lens, flush, stream):
    import torch
    from paper_2602_06283_b200 import ops
    res = {}
    ws = ops.workspace(cfg, 5, 1, q.device)
    out = torch.empty_like(q)
    lse = torch.empty((cfg.B, cfg.H_q), dtype=torch.float32, device=q.device)
    res["ours_dense_split_kv"] = {"ms": round(_time(lambda: ops.dense_decode(cfg, q, K, V, lens, out, lse, ws),
                                                   flush, stream, a.warmup, a.steps), 5)}
    try:
        qq = q.view(cfg.B, cfg.H_q, 1, 128)
        f = lambda: torch.nn.functional.scaled_dot_product_attention(qq, K, V, scale=cfg.scale, enable_gqa=True)
        res["torch_sdpa"] = {"ms": round(_time(f, flush, stream, a.warmup, a.steps), 5)}
    except Exception as e:  # noqa: BLE001
        res["torch_sdpa"] = {"error": str(e)[:120], "ms": float("inf")}
    try:
        from flash_attn import flash_attn_with_kvcache
        Kn = K.transpose(1, 2).contiguous()     # [B, N, H_kv, d] layout flash_attn expects
        Vn = V.transpose(1, 2).contiguous()
        qn = q.view(cfg.B, 1, cfg.H_q, 128)
        f = lambda: flash_attn_with_kvcache(qn, Kn, Vn, cache_seqlens=lens, softmax_scale=cfg.scale)
        res["flash_attn_2"] = {"ms": round(_time(f, flush, stream, a.warmup, a.steps), 5)}
        del Kn, Vn
    except Exception as e:  # noqa: BLE001
        res["flash_attn_2"] = {"error": str(e)[:160], "ms": float("inf")}
    try:
        import flashinfer
        wsb = torch.empty(256 << 20, dtype=torch.uint8, device=q.device)
        page = 16
        npg = cfg.N_max // page
        # paged view of the same cache, HND layout: [pages, 2, H_kv, page, d]
        kv = torch.stack([K.view(cfg.B, cfg.H_kv, npg, page, 128).permute(0, 2, 1, 3, 4),
                          V.view(cfg.B, cfg.H_kv, npg, page, 128).permute(0, 2, 1, 3, 4)], dim=2)
        kv = kv.reshape(cfg.B * npg, 2, cfg.H_kv, page, 128).contiguous()
        w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(wsb, "HND")
        indptr = torch.arange(0, cfg.B + 1, dtype=torch.int32, device=q.device) * npg
        indices = torch.arange(cfg.B * npg, dtype=torch.int32, device=q.device)
        last = torch.full((cfg.B,), page, dtype=torch.int32, device=q.device)
        w.plan(indptr, indices, last, cfg.H_q, cfg.H_kv, 128, page, q_data_type=torch.bfloat16,
               kv_data_type=torch.bfloat16, sm_scale=cfg.scale)
        f = lambda: w.run(q, kv)
        res["flashinfer"] = {"ms": round(_time(f, flush, stream, a.warmup, a.steps), 5)}
        del kv
    except Exception as e:  # noqa: BLE001
        res["flashinfer"] = {"error": str(e)[:160], "ms": float("inf")}
    return res


def end_to_end(a, cfg, dec, q, K, V, lens, N, flush, stream, dev):
    """Public API with host buffers (SocketDecoder.bind_host / host_step): q and
    the new token's K/V rows from pinned memory, the step (which stores the new
    rows into the cache and hashes them) and the output into pinned memory, all
    inside the timed region, replayed as one CUDA graph."""
    k_row, v_row = K[:, :, N - 1].cpu(), V[:, :, N - 1].cpu()
    q_h, k_h, v_h, out_h = dec.bind_host(lens)
    q_h.copy_(q.cpu())
    k_h.copy_(k_row)
    v_h.copy_(v_row)
    ms = _time(dec.host_step, flush, stream, a.warmup, a.steps)
    h2d = q_h.numel() * 2 + k_h.numel() * 2 + v_h.numel() * 2
    return {"ms": ms, "h2d": h2d, "d2h": out_h.numel() * 2}


_JSON_OUT = None


def emit_line(line):
    """The one JSON line on stdout (every other print, including the C
    libraries' -- e.g. NCCL's version banner -- goes to stderr, see main)."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    # stdout carries exactly one JSON line: keep a private handle on it and send
    # file descriptor 1 (Python prints and native libraries alike) to stderr
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
