#!/usr/bin/env python
"""Benchmark of the coarse-grid Dirac operator apply (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload M1..M5] [--prec fp32|fp16] [--pgrid P0,P1,P2,P3] [--transport peer|nccl]

BASELINE.json's metric is "coarse-Dslash GFLOPS and HBM GB/s (% of B200 roofline) at 1/2/4/8
GPUs"; the configuration it is quoted on at 1/2/4/8 GPUs is configs[4] = M5, a 16^3 x 32
coarse lattice, Nvec = 24, fp16 storage (the Iso64 64^3 x 128 fine lattice blocked 4^4,
PAPER.md:325 Table 2), which fits one B200 (10.9 GB of links).  So the headline workload is M5
at every N: STRONG scaling, the global lattice fixed and split along T over the N ranks
(--pgrid 1,1,2,4 gives BASELINE's T4 x Z2 variant at N = 8).  A "step" is one apply y = D v of
the whole lattice: on every rank, all SURVEY §8(a) rows (decode, link streaming, neighbour
gather, dot products, reductions, store; for N > 1 the halo pack + transfer, the arrival wait
and the halo-term kernel).  Steps are chained (v -> y -> v ...) like a coarse-grid solver.

Every other BASELINE config (M1 per call and as a D^n chain, M2 and M3 in fp32 and fp16, M4,
M5) is measured on one GPU under "configs" (hot and cold, clocks per window; N = 1 only).

Rank 0 prints ONE JSON line.  Inputs are synthetic (device generator, links x
2^-4), resident in HBM; M5's links (10.9 GB; 1.36 GB per rank at N = 8) are far larger than
the 126 MB L2, so no flush is needed between steps.  Timing: CUDA events on the launching
stream, barrier + synchronize on both sides, max over ranks; the timed region is cut into
segments of <= 400 applies and v is regenerated (untimed, between the segments' events) so
the iterate stays finite (|D| ~ 1.09 with links x 2^-4).  `e2e`: the same metric through the
public API with pinned host buffers (H2D of v, apply, D2H of y, every step, pipelined on three
streams).  `cpu_baseline` / --impl reference: the float64 oracle (oracle/) on this host's
cores, on a bounded periodic sub-lattice of the same Nvec (per-site work is identical).
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs as concrete synthetic workloads
WORKLOADS = {
    "M1": {"dims": (2, 2, 2, 2), "nvec": 24, "prec": "fp32", "cfg": 0,
           "name": "coarse lattice 2^4, Nvec=24 (48 dof/site), fp32"},
    "M2": {"dims": (4, 4, 4, 4), "nvec": 24, "prec": "fp32", "cfg": 1,
           "name": "coarse lattice 4^4, Nvec=24, fp32/fp16"},
    "M3": {"dims": (8, 8, 8, 8), "nvec": 24, "prec": "fp32", "cfg": 2,
           "name": "coarse lattice 8^4, Nvec=24 (48^3x96 fine lattice blocked 6^3x12)"},
    "M4": {"dims": (6, 6, 6, 12), "nvec": 32, "prec": "fp32", "cfg": 3,
           "name": "coarse lattice 6^3x12, Nvec=32, second MG level"},
    "M5": {"dims": (16, 16, 16, 32), "nvec": 24, "prec": "fp16", "cfg": 4,
           "name": "coarse lattice 16^3x32, Nvec=24, fp16 storage (Iso64 64^3x128 blocked 4^4)"},
}
HEADLINE = "M5"
_RESULT_FD = 1


def emit(obj):
    """Write the result line to the process's real stdout (see main())."""
    os.write(_RESULT_FD, (json.dumps(obj) + "\n").encode())
SEG = 400   # applies per timed segment (keeps the chained iterate finite)


def _perfmodel():
    """The byte / flop model (perfmodel.py), loaded by path: no product library is mapped."""
    spec = importlib.util.spec_from_file_location("cd_perfmodel", os.path.join(ROOT, "perfmodel.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


# ------------------------------------------------------------------ clocks (nvidia-smi during timing)
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # nvidia-smi needs ~0.1-0.3 s to start: it runs for the whole bench, every row is stamped
    # with the host clock when it arrives, and a summary covers the rows inside one window
    # (window() marks); a window shorter than 3 samples adds the rows just before it (the same
    # workload's settle phase) and says so.

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.device), "-lms", "20"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append([time.perf_counter()] + parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=5)

    def summary(self, t0, t1, settle=0.5):
        rows = [r[1:] for r in self.rows if t0 <= r[0] <= t1 + 0.02]
        window = "timed region"
        if len(rows) < 3:
            rows = [r[1:] for r in self.rows if t0 - settle <= r[0] <= t1 + 0.02]
            window = "settle phase + timed region (same workload)"
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "window": window}


# ------------------------------------------------------------------ oracle timing (CPU baseline)
SAMPLE_LADDER = [(2, 2, 2, 2), (4, 2, 2, 2), (4, 4, 2, 2), (4, 4, 4, 2), (4, 4, 4, 4), (8, 4, 4, 4), (8, 8, 4, 4),
                 (8, 8, 8, 2), (8, 8, 8, 4), (8, 8, 8, 8)]


def _oracle():
    import oracle
    import synth
    return oracle, synth


def _oracle_rate(oracle, synth, nvec, dims, budget_s, threads):
    """float64 oracle applies on a periodic sub-lattice for ~budget_s: (GFLOPS, reps, seconds)."""
    pm = _perfmodel()
    oracle.set_threads(threads)
    N = 2 * nvec
    L = synth.links(dims, N, scale_log2=-4)
    v = synth.vector(dims, N)
    oracle.apply(dims, L, v)   # warm-up
    reps, t0 = 0, time.perf_counter()
    while True:
        v = oracle.apply(dims, L, v)
        reps += 1
        el = time.perf_counter() - t0
        if (el >= budget_s and reps >= 2) or reps >= 100000:
            break
    V = dims[0] * dims[1] * dims[2] * dims[3]
    return pm.flops_per_site(nvec) * V * reps / el / 1e9, reps, el


def cpu_baseline(nvec, budget_s=12.0):
    """The oracle as it stands on this host: all cores (8^4 sample) and 1 thread (4^4 sample)."""
    oracle, synth = _oracle()
    cores = len(os.sched_getaffinity(0))
    pm = _perfmodel()
    dims = (8, 8, 8, 8)
    g, reps, el = _oracle_rate(oracle, synth, nvec, dims, budget_s * 0.75, cores)
    g1, reps1, el1 = _oracle_rate(oracle, synth, nvec, (4, 4, 4, 4), budget_s * 0.25, 1)
    oracle.set_threads(cores)
    V = 4096
    return {"value": round(g, 3), "unit": "GFLOPS", "cores": cores, "kind": "oracle",
            "sample": f"{reps} chained float64 oracle applies of a periodic 8^4 lattice ({V} sites, Nvec={nvec}; "
                      f"per-site work identical to the workload's), {el:.1f} s on {cores} threads",
            "gbs_fp64": round(pm.metric_bytes_per_site(nvec, 'fp64') * V * reps / el / 1e9, 3),
            "one_thread": {"value": round(g1, 3), "unit": "GFLOPS", "cores": 1,
                           "sample": f"{reps1} applies of a periodic 4^4 lattice, {el1:.1f} s on 1 thread"}}


# ------------------------------------------------------------------ distributed plumbing
def dist_setup():
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("CD_BENCH_BACKEND", "gloo" if "--same-gpu" in sys.argv else "nccl")
        dist.init_process_group(backend)
    return world, rank, local


def dist_max(x: float, world: int, device=None) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    if dist.get_backend() != "nccl":
        device = None   # gloo: host tensor
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def measured_peak():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: 1 Gi bf16 copy, read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(key, variant):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel from the
    committed ncu --set full capture (profiles/ncu_traffic.json) -- only if that capture is of
    the variant this run chose -- else None."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))[key]
        return t[variant]["bytes"] if variant in t else None
    except Exception:
        return None


def _events_us(torch, fn, reps, stream=None):
    s = stream or torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # a ~100 us spin kernel ahead of the start event keeps the stream busy while the host
    # submits fn, so host launch latency does not show up as device idle time in the window
    with torch.cuda.stream(s):
        torch.cuda._sleep(200000)
    e0.record(s)
    fn(reps)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


# ------------------------------------------------------------------ per-config measurements (N = 1)
def _rate(pm, nvec, prec, V, us, peak):
    gbs = pm.metric_bytes_per_site(nvec, prec) * V / us / 1e3
    return {"us": round(us, 3), "GFLOPS": round(pm.flops_per_site(nvec) * V / us / 1e3, 1), "GBs": round(gbs, 1),
            "pct_of_8tbs": round(100 * gbs / 8000, 2), "frac_measured_peak": round(gbs / peak, 4)}


def measure_config(cd, torch, pm, sampler, key, prec, peak):
    """Hot time of one coarse_dslash_apply for a BASELINE config: K chained
    applies (v -> y -> v), captured in one CUDA graph for the L2-resident sizes (so launch gaps
    count, PDL edges kept), replayed R times, t = median / K.  Returns (record, state); the cold
    time is measured later by measure_cold(state) -- after every hot measurement, because an L2
    flush leaves later L2-resident replays slower for the rest of the process
    (profiles/m2_factors.py: 4^4 fp32 graph 5.42 -> 6.79 us per apply after one 256 MB flush)."""
    w = WORKLOADS[key]
    dims, nvec = w["dims"], w["nvec"]
    V = dims[0] * dims[1] * dims[2] * dims[3]
    ctx = cd.Context(dims, nvec)
    L = ctx.links_generate(prec, kind="general", scale_log2=-4)
    a, b = ctx.field(prec), ctx.field(prec)
    a.generate()
    L.apply(b, a)   # autotune (excluded)
    torch.cuda.synchronize()
    small = V <= 256
    K = {16: 400, 256: 200}.get(V, 20)
    R = 20 if small else 5
    s = torch.cuda.Stream()
    t0 = time.perf_counter()
    hot = []
    with torch.cuda.stream(s):
        if small:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                x, y = a, b
                for _ in range(K):
                    L.apply(y, x, s)
                    x, y = y, x
            for _ in range(R):
                a.generate(stream=s)
                hot.append(_events_us(torch, lambda n: g.replay(), 1, s) / K)
        else:
            def chained(n):
                x, y = a, b
                for _ in range(n):
                    L.apply(y, x, s)
                    x, y = y, x
            for _ in range(R):
                a.generate(stream=s)
                hot.append(_events_us(torch, chained, K, s))
    t1 = time.perf_counter()
    variant = ctx.variants(prec)[ctx.chosen_variant(prec)]
    rec = {"workload": w["name"], "baseline_config": w["cfg"], "dims": list(dims), "nvec": nvec, "prec": prec,
           "sites": V, "op": "coarse_dslash_apply", "variant": variant,
           "hot": dict(_rate(pm, nvec, prec, V, statistics.median(hot), peak),
                       protocol=(f"CUDA graph of {K} chained applies, median of {R} replays / {K}" if small else
                                 f"{K} chained applies, median of {R} windows"),
                       regime="L2-resident (effective rate under the BASELINE byte formula)" if small
                       else "HBM streaming (inputs > L2)"),
           "clocks": sampler.summary(t0, t1),
           "ncu_traffic": ncu_traffic(f"{key}_{prec}", variant)}
    return rec, (ctx, L, a, b, s, small, nvec, prec, V)


def measure_cold(cd, torch, pm, sampler, rec, state, peak):
    """cold: K applies, each behind an L2 flush (256 MB written = 2 x L2), minus K flushes alone,
    both as CUDA graphs (a single few-microsecond apply is below the event timer's resolution)."""
    ctx, L, a, b, s, small, nvec, prec, V = state
    flush = 256 << 20
    ctx.flush_l2(flush)   # allocates the flush buffer outside capture
    torch.cuda.synchronize()
    KC = 40 if small else 10
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        gf, gfa = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(gf, stream=s):
            for _ in range(KC):
                ctx.flush_l2(flush, stream=s)
        with torch.cuda.graph(gfa, stream=s):
            for _ in range(KC):
                ctx.flush_l2(flush, stream=s)
                L.apply(b, a, s)
        tf, tfa = [], []
        for _ in range(5):
            tf.append(_events_us(torch, lambda n: gf.replay(), 1, s))
            tfa.append(_events_us(torch, lambda n: gfa.replay(), 1, s))
    cold_us = (statistics.median(tfa) - statistics.median(tf)) / KC
    rec["cold"] = dict(_rate(pm, nvec, prec, V, cold_us, peak),
                       protocol=f"graph of {KC} x (256 MB L2 flush + apply) minus graph of {KC} flushes, / {KC}")
    rec["clocks_cold"] = sampler.summary(t0, time.perf_counter())
    return rec


def measure_chain(cd, torch, pm, sampler):
    """M1 as a D^n chain in ONE persistent kernel (coarse_dslash_apply_chain): links stay on chip
    for all n applies, so this is an effective rate on the BASELINE byte formula, not the
    per-call target (that is configs.M1_fp32.hot)."""
    ctx = cd.Context((2, 2, 2, 2), 24)
    L = ctx.links_generate("fp32", scale_log2=-4)
    a, b = ctx.field("fp32"), ctx.field("fp32")
    a.generate()
    L.apply_chain(a, b, 8)
    torch.cuda.synchronize()
    t0 = time.perf_counter()

    def chain_us(n):
        ts = []
        for _ in range(3):
            a.generate()
            torch.cuda.synchronize()
            ts.append(_events_us(torch, lambda k: L.apply_chain(a, b, k), n))
        return statistics.median(ts)
    us, us200 = chain_us(800), chain_us(200)
    t1 = time.perf_counter()
    assert all(map(lambda z: z == z, a.export().ravel()[:64]))
    marg = (us * 800 - us200 * 200) / 600
    r = _rate(pm, 24, "fp32", 16, us, measured_peak()[0])
    return {"workload": WORKLOADS["M1"]["name"], "op": "coarse_dslash_apply_chain (800 applies per launch)",
            "variant": ctx.chosen_chain_variant("fp32"), "effective": r,
            "us_marginal": round(marg, 3), "pct_of_8tbs_marginal": round(100 * pm.metric_bytes_per_site(24, "fp32") * 16
                                                                           / marg / 1e3 / 8000, 2),
            "note": "links resident on chip for all applies: an effective rate, NOT the per-call apply",
            "clocks": sampler.summary(t0, t1)}


def measure_overlap(cd, torch, pm, sampler):
    """Overlap of the halo exchange with the interior, on one GPU: M5 with T routed through the
    halo path (CD_OPT_HALO_SELF_MASK: the T faces are packed, exchanged with this rank itself
    and added by the halo-term kernel, exactly the multi-rank code path) for the peer and NCCL
    transports, against the same apply with no split and the exchange alone.  The three
    configurations are timed in interleaved rounds (the power-capped clock drifts over seconds)."""
    w = WORKLOADS["M5"]
    dims, nvec, prec = w["dims"], w["nvec"], w["prec"]
    t0 = time.perf_counter()
    runs = {}
    for tr in ("none", "peer", "nccl"):
        ctx = cd.Context(dims, nvec)
        if tr != "none":
            ctx.set_option(cd.CD_OPT_HALO_SELF_MASK, 8)
            if tr == "peer":
                ctx.peer_connect([ctx.peer_handle()])
            ctx.set_transport(tr)
        L = ctx.links_generate(prec, scale_log2=-4)
        a, b = ctx.field(prec), ctx.field(prec)
        a.generate()
        L.apply(b, a)   # tunes
        if tr != "none":
            ctx.halo_exchange(a, copy_out=False)
        torch.cuda.synchronize()
        runs[tr] = (ctx, L, a, b)
    t_ap = {k: [] for k in runs}
    t_x = {k: [] for k in runs if k != "none"}
    for _ in range(5):
        for tr, (ctx, L, a, b) in runs.items():
            a.generate()
            t_ap[tr].append(_events_us(torch, lambda k: [L.apply(b, a) if i % 2 == 0 else L.apply(a, b)
                                                          for i in range(k)], 16))
            if tr != "none":
                t_x[tr].append(_events_us(torch, lambda k: [ctx.halo_exchange(a, copy_out=False) for _ in range(k)], 40))
    plain = statistics.median(t_ap["none"])
    pl = cd.cd_halo_plan_create(dims, nvec, (1, 1, 1, 1), 0, prec, 8)
    out = {"workload": w["name"], "split": "T through the halo path, self exchange (1 GPU)",
           "us_no_split": round(plain, 2), "halo_bytes": int(pl.total_bytes),
           "face_sites": 2 * dims[0] * dims[1] * dims[2]}
    for tr in ("peer", "nccl"):
        ctx = runs[tr][0]
        sp, x = statistics.median(t_ap[tr]), statistics.median(t_x[tr])
        out[tr] = {"us_split_apply": round(sp, 2), "us_exchange_only": round(x, 2), "exposed_us": round(sp - plain, 2),
                   "variant": ctx.variants(prec)[ctx.chosen_variant(prec)]}
    out["note"] = ("exposed = split apply - unsplit apply: the halo-term kernel over the face sites (one more read "
                   "of their remote-hop matrices and a y read-modify-write) plus any exchange time not hidden "
                   "behind the interior; exchange only = coarse_halo_exchange (pack + transfer + arrival wait) "
                   "run alone; medians of 5 interleaved rounds")
    out["clocks"] = sampler.summary(t0, time.perf_counter())
    del runs
    return out


def extras(cd, torch, pm, sampler):
    """NEXT-row kernels at 8^4, Nvec 24 (informational)."""
    out = {}
    peak_bw = measured_peak()[0]
    try:
        peak_tf = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"])
    except Exception:
        peak_tf = 2250.0
    nvec, V = 24, 4096
    # 128 right-hand sides on the tcgen05 tensor cores (fp16 storage)
    t0 = time.perf_counter()
    ctx = cd.Context((8, 8, 8, 8), nvec)
    L = ctx.links_generate("fp16", scale_log2=-4)
    a, b = ctx.field("fp16", nrhs=128), ctx.field("fp16", nrhs=128)
    a.generate()
    L.apply_mrhs(b, a)
    torch.cuda.synchronize()
    us = _events_us(torch, lambda n: [L.apply_mrhs(b, a) for _ in range(n)], 10)
    tf = pm.flops_per_site(nvec) * V * 128 / us / 1e6
    N = 2 * nvec
    comp = V * 9 * (4 * N * N + 16) + 2 * V * (128 * 4 * N + 16)   # links once + every block read and written
    out["8^4_fp16_mrhs128"] = {"us_per_apply": round(us, 1), "us_per_rhs": round(us / 128, 3),
                               "TFLOPS": round(tf, 1), "tensor_frac": round(tf / peak_tf, 3),
                               "tensor_peak_source": "MEASURED_PEAKS.json bf16_tflops (fp16 dense = bf16 dense)",
                               "compulsory_bytes": comp, "hbm_GBs": round(comp / us / 1e3, 1),
                               "hbm_frac": round(comp / us / 1e3 / peak_bw, 3),
                               "limiter": "per-hop barrier hand-offs of the single-thread roles (DESIGN.md §6)",
                               "clocks": sampler.summary(t0, time.perf_counter())}
    del L, a, b, ctx
    # hermiticity-compressed links (5 matrices / site) and the even-odd Schur operator, fp32
    t0 = time.perf_counter()
    ctx = cd.Context((8, 8, 8, 8), nvec)
    L = ctx.links_generate("fp32", kind="hermitian", scale_log2=-4)
    C, _ = L.compress_hermitian(check=False)
    a, b = ctx.field("fp32"), ctx.field("fp32")
    a.generate()
    C.apply(b, a)
    torch.cuda.synchronize()
    us = _events_us(torch, lambda n: [C.apply(b, a) for _ in range(n)], 200)
    gb = (5 * 48 * 48 + 10 * 48) * 8 * V / us / 1e3
    out["8^4_fp32_compressed"] = {"us_per_apply": round(us, 2), "GBs_5matrix": round(gb, 1),
                                  "hbm_frac": round(gb / peak_bw, 3), "clocks": sampler.summary(t0, time.perf_counter())}
    del C
    t0 = time.perf_counter()
    E = L.prepare_eo()
    xe, ye = ctx.field("fp32", parity=0), ctx.field("fp32", parity=0)
    xe.import_(torch.randn(V // 2, 48, dtype=torch.complex64))
    E.apply_eo(ye, xe)
    torch.cuda.synchronize()
    us = _events_us(torch, lambda n: [E.apply_eo(ye, xe) for _ in range(n)], 200)
    gb = (V // 2) * (17 * 48 * 48 + 19 * 48) * 8 / us / 1e3
    out["8^4_fp32_even_odd_schur"] = {"us_per_apply": round(us, 2), "GBs": round(gb, 1),
                                      "hbm_frac": round(gb / peak_bw, 3),
                                      "clocks": sampler.summary(t0, time.perf_counter())}
    del E, L, a, b, xe, ye, ctx
    # prolongator / restrictor: Wilson 32^4 fine grid -> 8^4 coarse, 4^4 aggregates, Nvec 24
    t0 = time.perf_counter()
    ctx = cd.Context((8, 8, 8, 8), nvec)
    Vf = V * 256
    T = ctx.transfer((4, 4, 4, 4), 4, 3, torch.randn(Vf, 4, 3, nvec, dtype=torch.complex64, device="cuda"))
    f = T.fine_field()
    c = ctx.field("fp32")
    c.generate()
    T.prolong(f, c)
    T.restrict(c, f)
    torch.cuda.synchronize()
    nbytes = Vf * 12 * nvec * 8 + Vf * 12 * 8 + V * 48 * 8
    us_p = _events_us(torch, lambda n: [T.prolong(f, c) for _ in range(n)], 20)
    us_r = _events_us(torch, lambda n: [T.restrict(c, f) for _ in range(n)], 20)
    out["transfer_32^4_to_8^4"] = {"us_prolong": round(us_p, 1), "us_restrict": round(us_r, 1),
                                   "hbm_frac_prolong": round(nbytes / us_p / 1e3 / peak_bw, 3),
                                   "hbm_frac_restrict": round(nbytes / us_r / 1e3 / peak_bw, 3),
                                   "clocks": sampler.summary(t0, time.perf_counter())}
    del T, f, c, ctx
    return out


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    world, rank, local = dist_setup()
    if args.same_gpu:   # functional check of the multi-rank path on a one-GPU box (timings time-sliced)
        local = 0
    torch.cuda.set_device(local)
    import paper_1612_07873_b200 as cd
    pm = _perfmodel()

    w = WORKLOADS[args.workload]
    gdims, nvec = w["dims"], w["nvec"]
    prec = args.prec or w["prec"]
    N = 2 * nvec
    if args.pgrid:
        pgrid = tuple(int(x) for x in args.pgrid.split(","))
    else:
        pgrid = (1, 1, 1, world)
    assert pgrid[0] * pgrid[1] * pgrid[2] * pgrid[3] == world, "--pgrid must multiply to the number of ranks"
    nccl_id = None
    if world > 1 and args.transport == "nccl":
        import torch.distributed as dist
        obj = [cd.cd_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    ctx = cd.Context(gdims, nvec, pgrid, device=local, nranks=world, rank=rank, nccl_id=nccl_id)
    fallback = None
    if world > 1:
        if args.transport == "peer":
            # every rank must agree on the transport: if any rank cannot open its neighbours' CUDA-IPC
            # windows (a container without IPC between processes, GPUs without peer access), all
            # fall back to NCCL rather than leave the scaling run without a line
            import torch.distributed as dist
            try:
                ctx.connect_peers()
                ok = 1
            except Exception as e:   # noqa: BLE001 -- reported in the JSON line
                ok, fallback = 0, f"peer connect failed on rank {rank}: {e}"[:300]
            flag = torch.tensor([ok], device="cpu" if dist.get_backend() == "gloo" else f"cuda:{local}")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag.item()) == 0:
                obj = [cd.cd_get_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(obj, src=0)
                del ctx
                ctx = cd.Context(gdims, nvec, pgrid, device=local, nranks=world, rank=rank, nccl_id=obj[0])
                args.transport = "nccl"
                fallback = fallback or "peer connect failed on another rank"
        ctx.set_transport(args.transport)
    ld = ctx.local_dims
    V_local = ctx.V
    V_glob = V_local * world
    stream = torch.cuda.current_stream()
    links = ctx.links_generate(prec, kind="general", seed=0x1612, scale_log2=-4)
    a, b = ctx.field(prec), ctx.field(prec)
    a.generate(seed=0x7873, tag=2)
    torch.cuda.synchronize()

    def steps(n):
        x, y = a, b
        for _ in range(n):
            links.apply(y, x, stream)
            x, y = y, x

    # warm-up (the first call autotunes; excluded, as the paper excludes its tuning solve)
    steps(max(args.warmup, 3))
    torch.cuda.synchronize()
    if world > 1:
        # every rank runs rank 0's tuned variant: per-rank tuning on noisy timings could otherwise pick
        # kernels with different split protocols (fused one-launch ring vs pack + halo-term kernels)
        import torch.distributed as dist
        obj = [ctx.chosen_variant(prec)]
        dist.broadcast_object_list(obj, src=0)
        ctx.set_option(cd.CD_OPT_VARIANT, int(obj[0]))
        steps(2)
        torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    # settle clocks under load (~0.5 s) before the timed region.  Every apply is collective when
    # N > 1, so all ranks must run the SAME number: rank 0's per-step time sets the count (a
    # time-based loop per rank let the ranks' apply counts diverge and the last applies wait
    # forever for a neighbour that had already stopped)
    if world > 1:
        import torch.distributed as dist
        t_s = time.perf_counter()
        steps(4)
        torch.cuda.synchronize()
        obj = [(time.perf_counter() - t_s) / 4]
        dist.broadcast_object_list(obj, src=0)
        for _ in range(max(1, min(2000, int(0.5 / max(8 * float(obj[0]), 1e-6))))):
            steps(8)
            torch.cuda.synchronize()
    else:
        t_end = time.perf_counter() + 0.5
        while time.perf_counter() < t_end:
            steps(8)
            torch.cuda.synchronize()
    a.generate(seed=0x7873, tag=2)
    barrier(world)
    torch.cuda.synchronize()
    t_mark0 = time.perf_counter()
    n0 = cd.cd_launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range((args.steps + SEG - 1) // SEG)]
    done = 0
    for i, (e0, e1) in enumerate(ev):
        k = min(SEG, args.steps - done)
        if i:
            a.generate(seed=0x7873, tag=2, stream=stream)   # untimed: between the segments' events
        e0.record(stream)
        steps(k)
        e1.record(stream)
        done += k
    torch.cuda.synchronize()
    t_mark1 = time.perf_counter()
    launches = cd.cd_launch_count() - n0 - (len(ev) - 1)   # minus the untimed regenerations
    ms_local = sum(e0.elapsed_time(e1) for e0, e1 in ev) / args.steps
    last = a if args.steps % 2 == 0 else b
    import numpy as np
    finite = bool(np.isfinite(last.export(dtype=np.complex64)).all())
    barrier(world)
    ms = dist_max(ms_local, world, device=f"cuda:{local}")
    clocks = sampler.summary(t_mark0, t_mark1)

    flops = pm.flops_per_site(nvec) * V_glob
    gflops = flops / (ms * 1e-3) / 1e9
    gbs_local = pm.metric_bytes_per_site(nvec, prec) * V_local / (ms * 1e-3) / 1e9
    peak, peak_src = measured_peak()

    # ---- multi-rank: exchange alone (comm-only) and the local operator alone, to show overlap
    comm = None
    if world > 1:
        def exch(n):
            for _ in range(n):
                ctx.halo_exchange(a, stream, copy_out=False)
        exch(3)
        barrier(world)
        us_comm = dist_max(_events_us(torch, exch, 50), world, device=f"cuda:{local}")
        solo = cd.Context(ld, nvec, device=local)      # same local volume, no halo
        Ls = solo.links_generate(prec, kind="general", scale_log2=-4)
        sa, sb = solo.field(prec), solo.field(prec)
        sa.generate()
        Ls.apply(sb, sa)
        torch.cuda.synchronize()
        us_solo = dist_max(_events_us(torch, lambda n: [Ls.apply(sb, sa, stream) if i % 2 == 0 else
                                                         Ls.apply(sa, sb, stream) for i in range(n)], 20),
                           world, device=f"cuda:{local}")
        pl = cd.cd_halo_plan_create(gdims, nvec, pgrid, rank, prec)
        hidden = (us_solo + us_comm - ms * 1e3) / us_comm if us_comm > 0 else None
        comm = {"transport": args.transport, "halo_bytes_per_rank": int(pl.total_bytes),
                "us_exchange_only": round(us_comm, 2), "us_local_operator_no_halo": round(us_solo, 2),
                "us_step": round(ms * 1e3, 2),
                "overlap_hidden_frac": None if hidden is None else round(max(-1.0, min(1.0, hidden)), 3),
                "note": "exchange only = coarse_halo_exchange (pack + transfer + arrival wait, no stencil); "
                        "hidden frac = (local + exchange - step) / exchange"}
        del Ls, sa, sb, solo

    # ---- e2e through the public API with pinned host buffers (h2d of v, d2h of y, every step).
    # Pipeline: step i's H2D (copy stream), apply (compute stream) and D2H (copy-back stream) are
    # ordered by events; NS buffer slots in groups of G let the copies of neighbouring groups
    # overlap the applies.  Every step still moves its full input and result over PCIe inside
    # the timed region (first H2D after the start event, last D2H before the end event).
    cdt = torch.complex64
    NS, G = 4, 2
    hv = [torch.empty((V_local, N), dtype=cdt).pin_memory() for _ in range(NS)]
    hy = [torch.empty((V_local, N), dtype=cdt).pin_memory() for _ in range(NS)]
    a.generate(seed=0x7873, tag=2)
    a.export(hv[0], stream=stream)
    for h in hv[1:]:
        h.copy_(hv[0])
    fa = [a] + [ctx.field(prec) for _ in range(NS - 1)]
    fb = [b] + [ctx.field(prec) for _ in range(NS - 1)]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    ngrp = NS // G
    evs = {k: [torch.cuda.Event() for _ in range(ngrp)] for k in ("in", "done", "out")}
    k_e2e = max(args.steps, 40)

    def e2e_steps(n, f0=None):
        if f0 is not None:
            s_in.wait_event(f0)
        for g0 in range(0, n, G):
            grp = range(g0, min(n, g0 + G))
            q = (g0 // G) % ngrp
            if g0 >= NS:
                s_in.wait_event(evs["done"][q])
            for i in grp:
                fa[i % NS].import_(hv[i % NS], s_in)
            evs["in"][q].record(s_in)
            stream.wait_event(evs["in"][q])
            if g0 >= NS:
                stream.wait_event(evs["out"][q])
            for i in grp:
                links.apply(fb[i % NS], fa[i % NS], stream)
            evs["done"][q].record(stream)
            s_out.wait_event(evs["done"][q])
            for i in grp:
                fb[i % NS].export(hy[i % NS], stream=s_out, sync=False)
            evs["out"][q].record(s_out)
        stream.wait_stream(s_in)
        stream.wait_stream(s_out)

    e2e_steps(4)
    barrier(world)
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    e2e_steps(k_e2e, f0)
    f1.record(stream)
    torch.cuda.synchronize()
    ms_e2e = dist_max(f0.elapsed_time(f1) / k_e2e, world, device=f"cuda:{local}")
    e2e_val = flops / (ms_e2e * 1e-3) / 1e9
    # the same steps strictly serialised on one stream (no copy / compute overlap), for reference
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    for _ in range(10):
        a.import_(hv[0], stream)
        links.apply(b, a, stream)
        b.export(hy[0], stream=stream, sync=False)
    g1.record(stream)
    torch.cuda.synchronize()
    ms_serial = dist_max(g0.elapsed_time(g1) / 10, world, device=f"cuda:{local}")
    del fa[1:], fb[1:], hv, hy

    # ---- every BASELINE config on one GPU (N = 1 only), in a fresh process: the headline's
    # allocations and power state do not leak into the small latency-bound configs (or back)
    configs = None
    also = None
    sampler.stop()
    if world == 1 and not args.no_extras:
        variant_name = ctx.variants(prec)[ctx.chosen_variant(prec)]
        del links, a, b, fa, fb
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        r = subprocess.run([sys.executable, os.path.abspath(__file__), "--configs-only"], capture_output=True,
                           text=True, timeout=900)
        lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        if r.returncode == 0 and lines:
            sub = json.loads(lines[-1])
            configs, also = sub["configs"], sub["also"]
        else:
            configs = {"error": f"configs subprocess rc={r.returncode}: {r.stderr[-500:]}"}

    # ---- cpu baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(nvec, budget_s=args.cpu_budget)

    if rank == 0:
        variant = ctx.variants(prec)[ctx.chosen_variant(prec)]
        key = f"{args.workload}_{prec}" + (f"_{'x'.join(map(str, ld))}" if world > 1 else "")
        out = {
            "metric": "coarse-Dslash GFLOPS and HBM GB/s (% of B200 roofline) at 1/2/4/8 GPUs",
            "value": round(gflops, 2),
            "unit": "GFLOPS",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms, 6),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32" if prec == "fp32" else "f16-storage/f32-accumulate",
            "data": "synthetic (device splitmix64 generator, links x 2^-4; DESIGN.md §3)",
            "config": {"workload": w["name"], "baseline_config": w["cfg"], "global_dims": list(gdims),
                       "proc_grid": list(pgrid), "local_dims": list(ld), "nvec": nvec, "storage": prec,
                       "op": "apply (D v), chained v->y->v", "variant": variant,
                       "transport": args.transport if world > 1 else None,
                       **({"transport_fallback": fallback} if fallback else {}),
                       "l2": "inputs larger than L2: links %.1f MB per GPU vs 126 MB L2" %
                             (V_local * 9 * (N * N * (8 if prec == 'fp32' else 4)) / 1e6),
                       "parallelism": f"proc grid {'x'.join(map(str, pgrid))} (T{'xZ' if pgrid[2] > 1 else ''} split)"
                       if world > 1 else "single GPU"},
            "gbs": round(gbs_local * world, 1),
            "gbs_per_gpu": round(gbs_local, 1),
            "pct_of_8tbs_per_gpu": round(100 * gbs_local / 8000.0, 2),
            "roofline": {"bound": "hbm", "achieved": round(gbs_local, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(gbs_local / peak, 4), "traffic": ncu_traffic(key, variant),
                         "kernel": variant, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": pm.metric_bytes_per_site(nvec, prec) * V_local,
                         "timing": "events around the chained applies on the launching stream; at N = 1 a step is "
                                   "exactly one launch of this kernel" if world == 1 else
                                   "per-rank step time, max over ranks (ring + peer transport: one fused launch per "
                                   "step; otherwise pack, interior, arrival wait and halo-term kernels)"},
            "e2e": {"value": round(e2e_val, 2), "unit": "GFLOPS", "ms_per_step": round(ms_e2e, 5),
                    "h2d_bytes_per_step": V_local * N * 8, "d2h_bytes_per_step": V_local * N * 8,
                    "steps": k_e2e, "ms_per_step_serialised": round(ms_serial, 5),
                    "pipeline": "H2D / apply / D2H on three streams, 4 buffer slots, groups of 2 steps"},
            "gpu_launches": int(launches),
            "iterate_finite": finite,
            "clocks": clocks,
            "comm": comm,
            "configs": configs,
            "cpu_baseline": cpu,
            "also": also,
        }
        emit(out)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------------ reference arm (the oracle)
def run_reference(args):
    world, rank = env_int("WORLD_SIZE", 1), env_int("RANK", 0)
    if rank != 0:
        return
    pm = _perfmodel()
    w = WORKLOADS[args.workload]
    nvec = w["nvec"]
    oracle, synth = _oracle()
    cores = len(os.sched_getaffinity(0))
    oracle.set_threads(cores)
    N = 2 * nvec
    # per-site oracle time, then the largest ladder sample whose steps fit the budget
    d0 = (4, 4, 4, 4)
    L0, v0 = synth.links(d0, N, scale_log2=-4), synth.vector(d0, N)
    oracle.apply(d0, L0, v0)
    t0 = time.perf_counter()
    oracle.apply(d0, L0, v0)
    t_site = (time.perf_counter() - t0) / 256
    dims = SAMPLE_LADDER[0]
    for d in SAMPLE_LADDER:
        if d[0] * d[1] * d[2] * d[3] * t_site * (args.steps + args.warmup) <= args.ref_budget:
            dims = d
    V = dims[0] * dims[1] * dims[2] * dims[3]
    L = synth.links(dims, N, scale_log2=-4)
    v = synth.vector(dims, N)
    for _ in range(args.warmup):
        v = oracle.apply(dims, L, v)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v = oracle.apply(dims, L, v)
    el = time.perf_counter() - t0
    ms = el / args.steps * 1e3
    gflops = pm.flops_per_site(nvec) * V / (ms * 1e-3) / 1e9
    sample = f"each step: one float64 oracle apply on a periodic {'x'.join(map(str, dims))} sub-lattice " \
             f"({V} of the workload's sites per step, Nvec={nvec}, same per-site work), {cores} threads"
    out = {
        "impl": "reference",
        "metric": "coarse-Dslash GFLOPS and HBM GB/s (% of B200 roofline) at 1/2/4/8 GPUs",
        "value": round(gflops, 3), "unit": "GFLOPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (synth/ splitmix64 generator, links x 2^-4)",
        "config": {"workload": w["name"], "baseline_config": w["cfg"], "nvec": nvec, "sample_dims": list(dims)},
        "cpu_baseline": {"value": round(gflops, 3), "unit": "GFLOPS", "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(gflops, 3), "unit": "GFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(out)


def run_configs_only():
    """Every BASELINE config + the NEXT-row kernels on one GPU (bench.py's "configs" / "also")."""
    import torch
    torch.cuda.set_device(0)
    import paper_1612_07873_b200 as cd
    pm = _perfmodel()
    peak = measured_peak()[0]
    sampler = ClockSampler(0)
    sampler.start()
    time.sleep(1.0)   # idle: the latency-bound 2^4 chain first, at an unthrottled clock (reported)
    configs = {"M1_fp32_chain": measure_chain(cd, torch, pm, sampler)}
    states = {}
    for key, prec_k in (("M1", "fp32"), ("M2", "fp32"), ("M2", "fp16"), ("M3", "fp32"), ("M3", "fp16"),
                        ("M4", "fp32"), ("M4", "fp16")):
        configs[f"{key}_{prec_k}"], states[f"{key}_{prec_k}"] = measure_config(cd, torch, pm, sampler, key, prec_k, peak)
    for name, st in states.items():   # every cold (flushed) measurement after all the hot ones
        measure_cold(cd, torch, pm, sampler, configs[name], st, peak)
    del states
    configs["M5_fp16_self_halo_overlap"] = measure_overlap(cd, torch, pm, sampler)
    also = extras(cd, torch, pm, sampler)
    sampler.stop()
    emit({"configs": configs, "also": also})


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=HEADLINE)
    ap.add_argument("--prec", choices=["fp32", "fp16"], default=None, help="override the workload's storage")
    ap.add_argument("--pgrid", default=None, help="process grid P0,P1,P2,P3 (default 1,1,1,N: T split)")
    ap.add_argument("--transport", choices=["peer", "nccl", "auto"], default="peer")
    ap.add_argument("--same-gpu", action="store_true",
                    help="all ranks on cuda:0 (functional check of the N > 1 path on a one-GPU box; peer transport)")
    ap.add_argument("--configs-only", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-extras", action="store_true", help="skip the per-config and NEXT-row measurements")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--ref-budget", type=float, default=90.0)
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    # exactly ONE line on stdout: anything the libraries print there (e.g. NCCL's version banner
    # when a communicator is created) is sent to stderr; the JSON line goes to the real stdout
    sys.stdout.flush()
    real_out = os.dup(1)
    os.dup2(2, 1)
    global _RESULT_FD
    _RESULT_FD = real_out
    if args.configs_only:
        run_configs_only()
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
