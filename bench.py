#!/usr/bin/env python
"""Benchmark of the coarse-grid Dirac operator apply (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--prec fp32|fp16]

A "step" is one apply y = D v of the whole local lattice (all hot-path rows of SURVEY §8(a):
decode, link streaming, neighbour gather, dot products, reductions, store; for N > 1 also the
halo pack, NCCL exchange and halo-term kernel).  Steps are chained (v -> y -> v ...), as in a
coarse-grid solver.  N = 1 workload: the 8^4, Nvec = 24 lattice the north_star target is quoted
on (BASELINE.json configs[2]).  N > 1: weak scaling, every rank holds an 8^4 block of a
8 x 8 x 8 x (8N) lattice split along T, with the NCCL halo exchange.

Rank 0 prints ONE JSON line.  Inputs are synthetic (device generator, links
scaled by 2^-4), resident in HBM; the link field (680 MB) is larger than L2 (126 MB), so no L2
flush is needed between steps.  Timing: CUDA events on the launching stream, barrier +
synchronize on both sides, max over ranks.  `e2e` is the same metric through the public API
with host buffers: pinned-host -> device import of v, apply, device -> pinned-host export of y,
every step.  `cpu_baseline` / --impl reference: the float64 oracle (oracle/) timed on this
host's cores on a bounded periodic sub-lattice of the same Nvec (per-site work is identical).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = {
    "dims": (8, 8, 8, 8),
    "nvec": 24,
    "name": "coarse lattice 8^4, Nvec=24 (48^3x96 fine lattice blocked 6^3x12)",
}


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
    # nvidia-smi needs ~0.1-0.3 s to start: it is started before the settle phase, every row is
    # stamped with the host clock when it arrives, and the summary keeps the rows that arrived
    # inside the timed window (mark(), unmark()); if fewer than 3 did, the settle-phase rows
    # (the same workload, already under load) are added and the summary says so.

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

    def mark(self):
        self.t0 = time.perf_counter()

    def unmark(self):
        self.t1 = time.perf_counter()

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=5)

    def summary(self):
        t0, t1 = getattr(self, "t0", None), getattr(self, "t1", None)
        rows = [r[1:] for r in self.rows if t0 is None or t1 is None or t0 <= r[0] <= t1 + 0.02]
        window = "timed region"
        if len(rows) < 3 and t1 is not None:
            rows = [r[1:] for r in self.rows if r[0] <= t1 + 0.02]
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


def _oracle_setup(nvec):
    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    import oracle
    import synth
    return oracle, synth, int(os.environ["OMP_NUM_THREADS"])


def oracle_time_per_site(nvec, dims=(4, 4, 4, 4)):
    oracle, synth, cores = _oracle_setup(nvec)
    N = 2 * nvec
    L = synth.links(dims, N, scale_log2=-4)
    v = synth.vector(dims, N)
    oracle.apply(dims, L, v)
    t0 = time.perf_counter()
    oracle.apply(dims, L, v)
    return (time.perf_counter() - t0) / (dims[0] * dims[1] * dims[2] * dims[3])


def cpu_baseline(nvec, budget_s=15.0, dims=(8, 8, 8, 8)):
    """float64 oracle apply on a periodic sub-lattice, repeated for ~budget_s seconds."""
    from paper_1612_07873_b200 import perfmodel  # model only; no library call
    oracle, synth, cores = _oracle_setup(nvec)
    N = 2 * nvec
    L = synth.links(dims, N, scale_log2=-4)
    v = synth.vector(dims, N)
    oracle.apply(dims, L, v)   # warm-up
    reps, t0 = 0, time.perf_counter()
    while True:
        v = oracle.apply(dims, L, v)
        reps += 1
        el = time.perf_counter() - t0
        if (el >= budget_s and reps >= 3) or reps >= 100000:
            break
    V = dims[0] * dims[1] * dims[2] * dims[3]
    gflops = perfmodel.flops_per_site(nvec) * V * reps / el / 1e9
    return {"value": round(gflops, 3), "unit": "GFLOPS", "cores": cores, "kind": "oracle",
            "sample": f"{reps} chained float64 oracle applies of a periodic {'x'.join(map(str, dims))} lattice "
                      f"({V} sites, Nvec={nvec}), {el:.1f} s on {cores} threads",
            "gbs_fp64": round(perfmodel.metric_bytes_per_site(nvec, 'fp64') * V * reps / el / 1e9, 3)}


# ------------------------------------------------------------------ distributed plumbing
def dist_setup():
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if os.environ.get("CD_BENCH_BACKEND", "nccl") == "nccl" else "gloo"
        dist.init_process_group(backend)
    return world, rank, local


def dist_max(x: float, world: int, device=None) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
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


def ncu_traffic(prec, variant):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel from the
    committed ncu --set full capture (profiles/ncu_traffic.json) -- only if that capture is of
    the variant this run chose -- else None."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))[f"8^4_nvec24_{prec}"]
        return t[variant]["bytes"] if variant in t else None
    except Exception:
        return None


def _events_us(torch, fn, reps):
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # a ~100 us spin kernel ahead of the start event keeps the stream busy while the host
    # submits fn, so host launch latency does not show up as device idle time in the window
    torch.cuda._sleep(200000)
    e0.record(s)
    fn(reps)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def extras(cd, perfmodel, torch, other_prec="fp16"):
    """Secondary measurements (each a few hundred ms), reported under "also"."""
    out = {}
    peak_bw = measured_peak()[0]
    try:
        peak_tf = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"])
    except Exception:
        peak_tf = 2250.0   # nominal dense fp16 (fallback)
    nvec = WORKLOAD["nvec"]
    # 2^4 coarsest grid (BASELINE.json configs[0] shape): n chained applies in one kernel.
    # Measured first, after a short idle: this latency-bound kernel's time scales with the SM
    # clock, which the power-capped HBM runs before it leave depressed for a while.
    time.sleep(0.5)
    ctx = cd.Context((2, 2, 2, 2), nvec)
    L = ctx.links_generate("fp32", scale_log2=-4)
    a, b = ctx.field("fp32"), ctx.field("fp32")
    a.generate()
    L.apply_chain(a, b, 8)
    torch.cuda.synchronize()
    # 800 applies per launch: with links x 2^-4 the iterate grows ~1.09x per apply (1e30 after
    # 800, finite in fp32); v is regenerated (untimed) before every timed launch
    def chain_us(n):
        ts = []
        for _ in range(3):
            a.generate()
            torch.cuda.synchronize()
            ts.append(_events_us(torch, lambda k: L.apply_chain(a, b, k), n))
        return statistics.median(ts)

    us = chain_us(800)
    us200 = chain_us(200)
    # marginal cost of one more apply inside a chain (the per-launch cost -- kernel launch, the
    # links' one-time load, the first apply from global memory -- drops out of the slope)
    us_marg = (us * 800 - us200 * 200) / 600
    gbs = perfmodel.metric_bytes_per_site(nvec, "fp32") * 16 / us / 1e3
    vid = ctx.chosen_chain_variant("fp32")
    gbs_marg = perfmodel.metric_bytes_per_site(nvec, "fp32") * 16 / us_marg / 1e3
    out["2^4_fp32_chain"] = {"us_per_apply": round(us, 3), "GBs_effective": round(gbs, 1),
                             "pct_of_8tbs": round(100 * gbs / 8000, 1), "variant": vid,
                             "applies_per_launch": 800,
                             "us_per_apply_marginal": round(us_marg, 3),
                             "pct_of_8tbs_marginal": round(100 * gbs_marg / 8000, 1),
                             "note": "coarse_dslash_apply_chain (one persistent kernel, on-chip resident; "
                                     "variant 4000: cluster push chain, 3001+: LL-register chain)"}
    del L, a, b, ctx
    # the 8^4 workload with the other storage precision
    ctx = cd.Context(WORKLOAD["dims"], nvec)
    L = ctx.links_generate(other_prec, scale_log2=-4)
    a, b = ctx.field(other_prec), ctx.field(other_prec)
    a.generate()

    def chained(n):
        x, y = a, b
        for _ in range(n):
            L.apply(y, x)
            x, y = y, x
    chained(20)
    torch.cuda.synchronize()
    us = _events_us(torch, chained, 500)
    V = 4096
    gbs = perfmodel.metric_bytes_per_site(nvec, other_prec) * V / us / 1e3
    out[f"8^4_{other_prec}"] = {"us_per_apply": round(us, 2), "GFLOPS": round(perfmodel.flops_per_site(nvec) * V / us / 1e3, 1),
                                "GBs": round(gbs, 1), "pct_of_8tbs": round(100 * gbs / 8000, 1),
                                "variant": ctx.variants(other_prec)[ctx.chosen_variant(other_prec)]}
    del L, a, b, ctx
    # 128 right-hand sides on the tcgen05 tensor cores (fp16 storage), 8^4
    ctx = cd.Context(WORKLOAD["dims"], nvec)
    L = ctx.links_generate("fp16", scale_log2=-4)
    a, b = ctx.field("fp16", nrhs=128), ctx.field("fp16", nrhs=128)
    a.generate()
    L.apply_mrhs(b, a)
    torch.cuda.synchronize()
    us = _events_us(torch, lambda n: [L.apply_mrhs(b, a) for _ in range(n)], 10)
    tf = perfmodel.flops_per_site(nvec) * V * 128 / us / 1e6
    out["8^4_fp16_mrhs128"] = {"us_per_apply": round(us, 1), "us_per_rhs": round(us / 128, 3),
                               "TFLOPS": round(tf, 1), "tensor_frac": round(tf / peak_tf, 3),
                               "tensor_peak_source": "MEASURED_PEAKS.json bf16_tflops (fp16 dense = bf16 dense)",
                               "note": "coarse_dslash_apply_mrhs, tcgen05.mma kind::f16, fp32 accumulators in TMEM"}
    del L, a, b, ctx
    # hermiticity-compressed links (5 matrices / site) and the even-odd Schur operator, fp32, 8^4
    ctx = cd.Context(WORKLOAD["dims"], nvec)
    L = ctx.links_generate("fp32", kind="hermitian", scale_log2=-4)
    C, _ = L.compress_hermitian(check=False)
    a, b = ctx.field("fp32"), ctx.field("fp32")
    a.generate()
    C.apply(b, a)
    torch.cuda.synchronize()
    us = _events_us(torch, lambda n: [C.apply(b, a) for _ in range(n)], 200)
    gb = (5 * 48 * 48 + 10 * 48) * 8 * V / us / 1e3
    out["8^4_fp32_compressed"] = {"us_per_apply": round(us, 2), "GBs_5matrix": round(gb, 1),
                                  "hbm_frac": round(gb / peak_bw, 3),
                                  "note": "coarse_links_compress_hermitian: X + 4 forward links per site"}
    del C
    E = L.prepare_eo()
    xe, ye = ctx.field("fp32", parity=0), ctx.field("fp32", parity=0)
    xe.import_(torch.randn(V // 2, 48, dtype=torch.complex64))
    E.apply_eo(ye, xe)
    torch.cuda.synchronize()
    us = _events_us(torch, lambda n: [E.apply_eo(ye, xe) for _ in range(n)], 200)
    gb = (V // 2) * (17 * 48 * 48 + 19 * 48) * 8 / us / 1e3
    out["8^4_fp32_even_odd_schur"] = {"us_per_apply": round(us, 2), "GBs": round(gb, 1),
                                      "hbm_frac": round(gb / peak_bw, 3),
                                      "note": "coarse_dslash_apply_eo: M_ee = X_e - D_eo X_o^-1 D_oe (two kernels)"}
    del E, L, a, b, xe, ye, ctx
    # prolongator / restrictor: Wilson 32^4 fine grid -> 8^4 coarse, 4^4 aggregates, Nvec 24
    ctx = cd.Context(WORKLOAD["dims"], nvec)
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
    out["transfer_32^4_to_8^4"] = {"us_prolong": round(us_p, 1), "GBs_prolong": round(nbytes / us_p / 1e3, 1),
                                   "us_restrict": round(us_r, 1), "GBs_restrict": round(nbytes / us_r / 1e3, 1),
                                   "hbm_frac_prolong": round(nbytes / us_p / 1e3 / peak_bw, 3),
                                   "hbm_frac_restrict": round(nbytes / us_r / 1e3 / peak_bw, 3),
                                   "note": "coarse_prolong / coarse_restrict, fp32 basis 2.4 GB"}
    del T, f, c, ctx
    return out


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    import paper_1612_07873_b200 as cd
    from paper_1612_07873_b200 import perfmodel

    L0, L1, L2, L3 = WORKLOAD["dims"]
    nvec = WORKLOAD["nvec"]
    gdims = (L0, L1, L2, L3 * world)
    pgrid = (1, 1, 1, world)
    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        obj = [cd.cd_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    ctx = cd.Context(gdims, nvec, pgrid, device=local, nranks=world, rank=rank, nccl_id=nccl_id)
    prec = args.prec
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
    sampler = ClockSampler(local)
    sampler.start()
    t_end = time.perf_counter() + 0.5       # settle clocks under load before the timed region
    while time.perf_counter() < t_end:
        steps(50)
        torch.cuda.synchronize()
    a.generate(seed=0x7873, tag=2)
    barrier(world)
    torch.cuda.synchronize()
    sampler.mark()
    n0 = cd.cd_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    steps(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    sampler.unmark()
    sampler.stop()
    launches = cd.cd_launch_count() - n0
    ms_local = e0.elapsed_time(e1) / args.steps
    barrier(world)
    ms = dist_max(ms_local, world, device=f"cuda:{local}")
    clocks = sampler.summary()

    V_local = L0 * L1 * L2 * L3
    V_glob = V_local * world
    flops = perfmodel.flops_per_site(nvec) * V_glob
    gflops = flops / (ms * 1e-3) / 1e9
    gbs_local = perfmodel.metric_bytes_per_site(nvec, prec) * V_local / (ms * 1e-3) / 1e9
    peak, peak_src = measured_peak()

    # ---- e2e through the public API with pinned host buffers (h2d of v, d2h of y, every step).
    # Serving-style pipeline: step i's H2D (copy stream), apply (compute stream) and D2H (copy-back
    # stream) are ordered by events; two buffer slots let step i+1's H2D and step i-1's D2H overlap
    # step i's apply.  Every step still moves its full input and result over PCIe inside the timed
    # region (first H2D after the start event, last D2H before the end event).
    N = 2 * nvec
    cdt = torch.complex64
    # NS buffer slots, steps issued in groups of G: the H2D copies of a group land while the
    # previous group computes, so the compute stream waits on the copy stream once per group and
    # the applies inside a group stay back to back (programmatic dependent launch between them;
    # an event wait between two kernels would drain the first before the second starts).
    NS, G = 8, 4
    hv = [torch.empty((V_local, N), dtype=cdt).pin_memory() for _ in range(NS)]
    hy = [torch.empty((V_local, N), dtype=cdt).pin_memory() for _ in range(NS)]
    a.export(hv[0], stream=stream)
    for h in hv[1:]:
        h.copy_(hv[0])
    fa = [a] + [ctx.field(prec) for _ in range(NS - 1)]
    fb = [b] + [ctx.field(prec) for _ in range(NS - 1)]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    ngrp = NS // G
    ev = {k: [torch.cuda.Event() for _ in range(ngrp)] for k in ("in", "done", "out")}
    k_e2e = max(10, min(args.steps, 500))

    def e2e_steps(n, f0=None):
        if f0 is not None:
            s_in.wait_event(f0)
        for g0 in range(0, n, G):
            grp = range(g0, min(n, g0 + G))
            q = (g0 // G) % ngrp                     # event set of this group (slots q*G .. q*G+G-1)
            if g0 >= NS:
                s_in.wait_event(ev["done"][q])       # the applies of group g-ngrp finished reading fa[]
            for i in grp:
                fa[i % NS].import_(hv[i % NS], s_in)
            ev["in"][q].record(s_in)
            stream.wait_event(ev["in"][q])
            if g0 >= NS:
                stream.wait_event(ev["out"][q])      # the D2H of group g-ngrp finished with fb[]
            for i in grp:
                links.apply(fb[i % NS], fa[i % NS], stream)
            ev["done"][q].record(stream)
            s_out.wait_event(ev["done"][q])
            for i in grp:
                fb[i % NS].export(hy[i % NS], stream=s_out, sync=False)
            ev["out"][q].record(s_out)
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
    # the same steps strictly serialised on one stream (no overlap), for reference
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    for _ in range(k_e2e):
        a.import_(hv[0], stream)
        links.apply(b, a, stream)
        b.export(hy[0], stream=stream, sync=False)
    g1.record(stream)
    torch.cuda.synchronize()
    ms_serial = dist_max(g0.elapsed_time(g1) / k_e2e, world, device=f"cuda:{local}")
    del fa[1:], fb[1:]

    # ---- informational extras on one GPU (not the headline): fp16 storage, the 2^4 coarsest
    # grid as chained applies in one kernel, 128 right-hand sides on the tcgen05 tensor cores
    also = None
    if world == 1 and not args.no_extras:
        also = extras(cd, perfmodel, torch, other_prec="fp16" if prec == "fp32" else "fp32")

    # ---- cpu baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(nvec, budget_s=args.cpu_budget)

    if rank == 0:
        variant = ctx.variants(prec)[ctx.chosen_variant(prec)]
        traffic = ncu_traffic(prec, variant)
        out = {
            "metric": "coarse-Dslash GFLOPS and HBM GB/s (% of B200 roofline)",
            "value": round(gflops, 2),
            "unit": "GFLOPS",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms, 6),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32" if prec == "fp32" else "f16-storage/f32-accumulate",
            "data": "synthetic (device splitmix64 generator, links x 2^-4; DESIGN.md §3)",
            "config": {"workload": WORKLOAD["name"] if world == 1 else
                       f"coarse lattice 8x8x8x{8 * world} (8^4 per GPU, T-partitioned), Nvec=24",
                       "global_dims": list(gdims), "proc_grid": list(pgrid), "nvec": nvec, "storage": prec,
                       "op": "apply (D v), chained v->y->v", "variant": variant,
                       "l2": "inputs larger than L2: links %.1f MB per GPU vs 126 MB L2" %
                             (V_local * 9 * (N * N * (8 if prec == 'fp32' else 4)) / 1e6),
                       "parallelism": f"T-split x{world}" if world > 1 else "single GPU"},
            "gbs": round(gbs_local * world, 1),
            "gbs_per_gpu": round(gbs_local, 1),
            "pct_of_8tbs_per_gpu": round(100 * gbs_local / 8000.0, 2),
            "roofline": {"bound": "hbm", "achieved": round(gbs_local, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(gbs_local / peak, 4), "traffic": traffic,
                         "kernel": variant, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": perfmodel.metric_bytes_per_site(nvec, prec) * V_local},
            "e2e": {"value": round(e2e_val, 2), "unit": "GFLOPS", "ms_per_step": round(ms_e2e, 5),
                    "h2d_bytes_per_step": V_local * N * 8, "d2h_bytes_per_step": V_local * N * 8,
                    "pipeline": "H2D / apply / D2H on three streams, 8 buffer slots, groups of 4 steps",
                    "ms_per_step_serialised": round(ms_serial, 5)},
            "gpu_launches": int(launches),
            "clocks": clocks,
            "cpu_baseline": cpu,
            "also": also,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------------ reference arm (the oracle)
def run_reference(args):
    world, rank = env_int("WORLD_SIZE", 1), env_int("RANK", 0)
    if rank != 0:
        return
    from paper_1612_07873_b200 import perfmodel  # model only
    nvec = WORKLOAD["nvec"]
    oracle, synth, cores = _oracle_setup(nvec)
    N = 2 * nvec
    budget = args.ref_budget
    t_site = oracle_time_per_site(nvec)
    dims = SAMPLE_LADDER[0]
    for d in SAMPLE_LADDER:
        V = d[0] * d[1] * d[2] * d[3]
        if V * t_site * (args.steps + args.warmup) <= budget:
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
    gflops = perfmodel.flops_per_site(nvec) * V / (ms * 1e-3) / 1e9
    sample = f"each step: one float64 oracle apply on a periodic {'x'.join(map(str, dims))} sub-lattice " \
             f"({V} of the workload's sites per step, Nvec={nvec}, same per-site work)"
    out = {
        "impl": "reference",
        "metric": "coarse-Dslash GFLOPS and HBM GB/s (% of B200 roofline)",
        "value": round(gflops, 3), "unit": "GFLOPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (synth/ splitmix64 generator, links x 2^-4)",
        "config": {"workload": WORKLOAD["name"], "nvec": nvec, "sample_dims": list(dims)},
        "cpu_baseline": {"value": round(gflops, 3), "unit": "GFLOPS", "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(gflops, 3), "unit": "GFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--prec", choices=["fp32", "fp16"], default="fp32")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-extras", action="store_true", help="skip the informational 'also' measurements")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--ref-budget", type=float, default=90.0)
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
