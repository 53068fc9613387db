"""Benchmark of the SOCKET decode hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--batch B] [--ctx N] [--sparsity S] [--tables L]

A step is one SOCKET decode step of one attention layer over the whole batch
(BASELINE.json configs[1]: Llama-3.1-8B-shaped 32 q / 8 KV heads, d = 128,
32K context; default batch 16, 10x sparsity, L = 60, P = 8, tau = 0.5,
KV-shared selection):
  append-hash of the new key (Alg. 1, n_count = 1) -> query tables (Alg. 2) ->
  soft-collision scores (Eq. 4 / Alg. 4) -> top-k (Alg. 3) -> sparse
  flash-decode + split LSE combine (Eq. 2).
tokens/s = B * n_gpus / t_step.  Multi-GPU (torchrun): every rank runs its own
batch shard (weak scaling, no collective on the data path); the step time is
the max over ranks.  L2 is flushed (256 MB memset) before every timed step.

--impl reference times the CPU oracle (oracle/, float64 numpy) on the same
workload, as a bounded sample: it is the reference arm of this
tier.  Prints exactly one JSON line on rank 0.
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
# (profiles/r1/ncu_summary.md); None = not captured for this configuration.
TRAFFIC = {}
try:
    _t = json.load(open(os.path.join(ROOT, "profiles", "r1", "traffic.json")))
    TRAFFIC = {k: v for k, v in _t.items() if isinstance(v, (int, float))}
except Exception:
    pass


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--sparsity", type=float, default=10.0)
    ap.add_argument("--tables", type=int, default=60)
    ap.add_argument("--bits", type=int, default=8)
    ap.add_argument("--tau", type=float, default=0.5)
    ap.add_argument("--mode", default="kv_shared", choices=["kv_shared", "per_qhead"])
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-rows", action="store_true", help="skip the NEXT-row measurements")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


def workload(a):
    k = int(round(a.ctx / a.sparsity))
    return {
        "workload": f"llama3.1-8b-shaped decode attention (32q/8kv, d=128), ctx {a.ctx}, "
                    f"batch {a.batch}, {a.sparsity:g}x sparsity (k={k}), L={a.tables}, P={a.bits}, "
                    f"tau={a.tau}, {a.mode} selection; BASELINE configs[1]",
        "batch": a.batch, "ctx": a.ctx, "k": k, "L": a.tables, "P": a.bits, "tau": a.tau,
        "H_q": 32, "H_kv": 8, "d": 128, "selection": a.mode,
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


# ---------------------------------------------------------------------------
# CPU oracle (reference arm / cpu_baseline): one (b, kv-head) unit at a time
# ---------------------------------------------------------------------------
def oracle_units(a, k, seconds, units=None, skip=0):
    import numpy as np

    import datagen
    import oracle as O

    N, L, P = a.ctx, a.tables, a.bits
    c = datagen.make_case(1, 4, 1, N, 128, seed=123)
    Wb = datagen.make_projections(4242, L, P, 128)
    codes, _ = O.hash_keys(O.widen(c["K"]), O.widen(Wb))   # prefill: not part of a step
    mode = O.GROUP_KV_SHARED if a.mode == "kv_shared" else O.GROUP_PER_QHEAD
    def one_unit():
        # one decode step of one (b, kv-head) unit: append-hash of the newest key,
        # tables, scores, top-k, attention of the group's 4 query heads
        kn, _ = O.hash_keys(O.widen(c["K"][0, 0, N - 1:N]), O.widen(Wb))
        codes[0, 0][:, N - 1:N] = kn
        rows = [(0, 0)] if mode == O.GROUP_KV_SHARED else [(0, h) for h in range(4)]
        O.decode_step(c["q"], c["K"], c["V"], Wb, c["seq_lens"], tau=a.tau, k=k,
                      sm_scale=1 / math.sqrt(128), group_mode=mode, codes=codes, rows=rows)

    if units is not None:                  # fixed number of samples, first `skip` untimed
        for _ in range(skip):
            one_unit()
        t0 = time.perf_counter()
        for _ in range(units - skip):
            one_unit()
        el = time.perf_counter() - t0
        units = units - skip
    else:                                  # time-bounded sample
        t0 = time.perf_counter()
        units = 0
        while True:
            one_unit()
            units += 1
            el = time.perf_counter() - t0
            if el >= seconds:
                break
    per_unit = el / units
    step_units = a.batch * 8                    # (b, kv-head) units of one full step
    t_step = per_unit * step_units
    try:
        import numpy
        threads = int(os.environ.get("OMP_NUM_THREADS", 0)) or os.cpu_count()
    except Exception:
        threads = os.cpu_count()
    return {"value": a.batch / t_step, "unit": "tokens/s", "cores": threads, "kind": "oracle",
            "sample": f"{units} (b, kv-head) units of the step ({el:.1f} s; numpy float64, "
                      f"BLAS threads up to {threads}); step = {step_units} units, extrapolated",
            "s_per_unit": per_unit, "ms_per_step": t_step * 1e3}


def run_reference(a):
    """Reference arm of this tier: the CPU oracle.  Each of the W + K steps is a
    bounded sample -- one (b, kv-head) unit of the decode step -- timed on the
    host; the K timed units are extrapolated to the full step (B * 8 units)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg, k = workload(a)
    cb = oracle_units(a, k, 0.0, units=a.warmup + a.steps, skip=a.warmup)
    line = {"metric": METRIC, "value": cb["value"], "unit": "tokens/s", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": cb["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": cfg, "impl": "reference",
            "cpu_baseline": {k2: cb[k2] for k2 in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


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


def run_ours(a):
    import torch
    import torch.distributed as dist

    import datagen
    from paper_2602_06283_b200 import Config, KV_SHARED, PER_QHEAD, SocketDecoder, ops
    from paper_2602_06283_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfgd, k = workload(a)
    B, N, L, P = a.batch, a.ctx, a.tables, a.bits
    mode = KV_SHARED if a.mode == "kv_shared" else PER_QHEAD
    cfg = Config(B=B, H_q=32, H_kv=8, N_max=N, L=L, P=P, tau=a.tau, group_mode=mode)
    q, K, V = datagen.torch_make_cache(B, 32, 8, N, 128, seed=1000 + rank, device=dev)
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
    # prefill key hashing (Alg. 1) on the tensor cores: codes only (the projection
    # GEMM), timed with events; algorithmic flops = 2 * keys * d * L * P
    def prefill_codes():
        ops.hash_keys(cfg, K, W, dec.codes, n_begin=0, n_count=N)
    pre_ms = _time(prefill_codes, flush, stream, 2, 5)
    pre_flops = 2.0 * B * 8 * N * 128 * L * P
    bf16_peak = 1654.9
    try:
        bf16_peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
    except Exception:
        pass
    prefill = {"kernel": "hash_keys_tc (tcgen05)", "ms": round(pre_ms, 4),
               "TFLOP/s": round(pre_flops / (pre_ms * 1e-3) / 1e12, 1),
               "frac_of_bf16_peak": round(pre_flops / (pre_ms * 1e-3) / 1e12 / bf16_peak, 4),
               "keys": B * 8 * N, "flops": pre_flops,
               "hbm_GB/s": round(B * 8 * N * (256 + L * ((P + 7) // 8)) / (pre_ms * 1e-3) / 1e9, 1)}

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    # ---- (1) graph-replayed step: headline ---------------------------------------
    dec.capture(q, lens, append=True)
    for _ in range(a.warmup):
        flush.zero_()
        dec.replay()
    barrier()
    clocks = Clocks(local)
    clocks.start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(a.steps)]
    for e0, e1 in evs:
        flush.zero_()
        e0.record(stream)
        dec.replay()
        e1.record(stream)
    barrier()
    clk = clocks.stop()
    step_ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / a.steps
    step_ms = max_over_ranks(step_ms)
    # 1 (one-launch cluster kernel, small batch) or 4 (prologue, score, top-k, decode)
    launches_per_step = ops.decode_step_launches(cfg)

    # ---- (2) per-kernel timing: each stage's call launched R times back to back
    # between two events on its stream (L2 flushed before each burst), so a
    # kernel's average duration excludes host launch gaps.  The headline above
    # uses the fused call; these give each kernel's share and roofline.
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
    ab = algorithmic_bytes(B, N, L, P, k, H_sel=cfg.H_sel)
    hbm, peak_src = peaks()
    stages = {}
    for s_, key in (("score", "score"), ("topk", "topk"), ("sparse_decode", "sparse_decode")):
        gbs = ab[key] / (stage_ms[s_] * 1e-3) / 1e9
        stages[s_] = {"ms": round(stage_ms[s_], 5), "alg_bytes": ab[key], "GB/s": round(gbs, 1),
                      "frac": round(gbs / hbm, 4), "share": round(stage_ms[s_] / eager_ms, 4)}
    for s_ in ("append_hash", "tables"):
        stages[s_] = {"ms": round(stage_ms[s_], 5), "share": round(stage_ms[s_] / eager_ms, 4)}
    dom = max(("score", "sparse_decode"), key=lambda s_: stage_ms[s_])
    kern = {"score": "score_reg_kernel", "sparse_decode": "decode_mma_kernel"}[dom]
    roof = {"bound": "hbm", "kernel": kern, "achieved": stages[dom]["GB/s"], "peak": hbm,
            "unit": "GB/s", "frac": stages[dom]["frac"], "traffic": TRAFFIC.get(kern),
            "peak_source": peak_src}

    # ---- (3) dense comparators on the same cache ---------------------------------
    dense = {}
    if not a.no_dense:
        dense = dense_baselines(a, cfg, q, K, V, lens, flush, stream)

    # ---- (3b) the SURVEY section 8(f) rows on the same cache ------------------------
    rows = {}
    if not a.no_rows and world == 1:
        rows = next_rows(a, cfg, dec, q, K, V, W, lens, k, flush, stream, dev, hbm)

    # ---- (4) end to end through the public API with host buffers -----------------
    e2e = end_to_end(a, cfg, dec, q, K, V, lens, N, flush, stream, dev)
    e2e_ms = max_over_ranks(e2e["ms"])

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    value = B * world / (step_ms * 1e-3)
    cpu = oracle_units(a, k, a.cpu_seconds) if world == 1 else None
    cfgd.update({"prefill_hash_s": round(prefill_s, 3), "parallelism": f"batch-shard x{world} (replicas)"})
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(step_ms, 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded N(0,1) bf16 q/K/V and projections)", "config": cfgd,
        "roofline": roof, "stages": stages, "eager_ms_per_step": round(eager_ms, 5),
        "gpu_launches": launches_per_step * a.steps, "clocks": clk, "prefill": prefill,
        "e2e": {"value": round(B * world / (e2e_ms * 1e-3), 1), "unit": "tokens/s",
                "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"]},
    }
    if dense:
        best = min(dense.items(), key=lambda kv: kv[1]["ms"])
        line["dense"] = {"best": best[0], "tokens_per_s": round(B * world / (best[1]["ms"] * 1e-3), 1),
                         "ms_per_step": best[1]["ms"], "all": dense,
                         "speedup_sparse_vs_dense": round(best[1]["ms"] / step_ms, 3)}
    if rows:
        line["next_rows"] = rows
    if cpu:
        line["cpu_baseline"] = {k2: cpu[k2] for k2 in ("value", "unit", "cores", "kind", "sample")}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def next_rows(a, cfg, dec, q, K, V, W, lens, k, flush, stream, dev, hbm):
    """SURVEY 8(f) rows on the bench cache, each timed like the headline (L2
    flushed before every step, CUDA events on the launching stream):
      hard_lsh  (f3): the fused step with Eq. 3 hard-LSH tables (scoring = 1);
      wide_codes(f2): the RULER setting L = 60, P = 10 (600 bits/token, uint16
                      codes), graph-replayed step; its score kernel's HBM rate;
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
    sb = B * cfg.H_kv * N * (Lw * 2 + 4) + B * cfg_w.H_sel * N * 4
    out["wide_codes"] = {"ms_per_step": round(ms, 5), "tokens_per_s": round(B / (ms * 1e-3), 1),
                         "score_ms": round(sms, 5), "score_GB/s": round(sb / (sms * 1e-3) / 1e9, 1),
                         "score_frac": round(sb / (sms * 1e-3) / 1e9 / hbm, 4),
                         "config": "L=60, P=10 (uint16 codes, 600 bits/token), graph-replayed step"}
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
    """Public API with host buffers (SocketDecoder.bind_host / host_step): one
    H2D copy of q and the new token's K/V rows from pinned memory, the step
    (which stores the new rows into the cache and hashes them) and the D2H copy
    of the output, all inside the timed region, replayed as one CUDA graph."""
    k_row, v_row = K[:, :, N - 1].cpu(), V[:, :, N - 1].cpu()   # before bind_host's warm-up step
    q_h, k_h, v_h, out_h = dec.bind_host(lens)
    q_h.copy_(q.cpu())
    k_h.copy_(k_row)
    v_h.copy_(v_row)
    ms = _time(dec.host_step, flush, stream, a.warmup, a.steps)
    h2d = q_h.numel() * 2 + k_h.numel() * 2 + v_h.numel() * 2
    return {"ms": ms, "h2d": h2d, "d2h": out_h.numel() * 2}


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
