#!/usr/bin/env python
"""TRPL+K bench (BASELINE.json metric: matvecs/s & time to p eigenpairs, fp64, HBM GB/s vs peak).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]

A "step" is one full trplk_solve (time to the p smallest eigenpairs) of the BASELINE config.
Default: C5 = configs[4] (512^3 7-pt Laplacian + diag(d), n = 1.34e8) -- BASELINE's metric names
no config, so the bench runs the largest single-GPU configuration (the one north_star's HBM and
scaling targets are stated on); --config C1..C4 runs the others.  Inputs are resident in HBM
(the context is created before the timed region); the inputs are far larger than the 126 MB L2
at C3-C5 and a 256 MiB buffer is written between timed steps in any case.
`value` = A-matvecs of the solve / solve time (whole job; max over ranks).
`e2e` = the same metric through the public API with HOST CSR buffers (pinned): create
(validation scan, H2D of the CSR, DIA/SELL conversion) + solve + D2H of eigenvectors +
destroy, after untimed create/solve/destroy rounds.
`roofline` = the inner-step kernel with the largest share of the step: live CUDA events around
the three kernel groups of the middle inner step of every cycle of every timed solve
(trplk_profile; the event nodes serialise that step's kernels, so the timed solves carry their
cost), algorithmic bytes of DESIGN.md / event time, against MEASURED_PEAKS.json hbm_gbs; the
kernel named is the instantiation the library launched (trplk_profile_kernels) and `traffic` its
ncu DRAM bytes per launch (profiles/traffic_<cfg>.json).  `cpu_baseline` = the oracle
(oracle/, plain C + OpenMP) on the host cores, rank 0 at N=1 only: the full solve where it takes
seconds (C1, C2), else a bounded sample of oracle inner steps at the config's full size (see
oracle_sample).

--impl reference: this tier has no reference implementation; the reference arm is the oracle
timed as it stands on the host cores, each step one bounded sample of the same workload.
For N>1 run under torchrun: one rank per GPU, z-slab row partition, NCCL.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "matvecs/s & time to p eigenpairs (fp64), HBM GB/s vs peak, at 1/2/4/8 B200"
UNIT = "matvecs/s"
PROFILES = os.path.join(ROOT, "profiles")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "host"],
                    help="N>1 exchanges: nccl (production) or host (host-staged through a gloo group; "
                         "lets several ranks share one GPU -- tests of the multi-process path only)")
    ap.add_argument("--precond", default="jacobi", choices=["jacobi", "none", "shifted", "ic0"],
                    help="none: M = I (with --k-plus 0: the thick-restart Lanczos baseline, eq 2.1); "
                         "shifted: Jacobi of A - rho_i B per cycle (P:171); ic0: IC(0) of A - sigma B")
    ap.add_argument("--k-plus", type=int, default=None, help="override the config's k_plus (l)")
    ap.add_argument("--block", type=int, default=1,
                    help="block TRPL+K (options.block, NEXT-3): b vectors per SpMM in the inner loop")
    ap.add_argument("--profile-last-only", action="store_true",
                    help="kernel-profile events on the last timed step only (default: every timed step)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="oracle sample budget")
    ap.add_argument("--method", default="trplk", choices=["trplk", "pl1"],
                    help="pl1: PL+1 (Algorithm 2, NEXT-1) for the lowest eigenpair, one GPU")
    ap.add_argument("--pl1-m", type=int, default=4, help="PL+1 Krylov block size m")
    return ap.parse_args()


def ncu_name(demangled):
    """'void trplk::k_step1_pipe<16, true>(trplk::SdotsArgs)' -> 'k_step1_pipe<16, 1>' (ncu's form)."""
    x = demangled.replace("void ", "").replace("trplk::", "").split("(")[0].strip()
    return x.replace("true", "1").replace("false", "0")


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = max(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


def plane_of(P):
    return 1 if P.grid["dim"] == 1 else P.grid["N"] ** 2


FULL_SOLVE_CFGS = ("C1", "C2")  # oracle full solve in seconds; C3/C4 take 20-30 min, C5 hours


def static_config(name, P, n, world, precond="Jacobi", comm="nccl", block=1):
    """The `config` object of both arms (identical keys and values)."""
    return {"workload": f"{name}: {P.desc}; p={P.p}, max_basis={P.q}, k_plus={P.l}, tol={P.tol}, "
                        f"{precond} preconditioner, seed 12" + (f", block TRPL+K b={block}" if block > 1 else ""),
            "n": n, "step": "one full trplk_solve (time to p eigenpairs)",
            "l2": "inputs larger than L2 at C3-C5; a 256 MiB buffer is written between timed steps",
            "parallelism": f"z-slab row partition x{world}" + (" (host-staged gloo exchanges)" if comm == "host" else "")}


class OracleSample:
    """The oracle as it stands (oracle/, plain C + OpenMP) on a bounded sample of the workload.

    C1, C2: the full oracle solve (seconds).  C3-C5 (a full oracle solve takes 20 min to hours):
    orc_inner_steps -- the code orc_trplk_solve runs for one inner step of eq 3.1 (z = A g, the
    T column U^T z, w = M (z - rho g), CGS2 of w against the basis, g_next = w / beta) -- on the
    config's full-size matrix with a basis of the cycle-average width k = p^ + (m+1)/2 (unit
    vectors: orthonormal; every page written before timing so the reads are real DRAM reads).
    One inner step = one A-matvec; the +K, Rayleigh-Ritz, rotation and residual work of a cycle
    (about 10-15 % of its bytes in DESIGN.md's model) is not in the sample, so the sample's
    matvecs/s is an upper bound of the oracle's full-solve rate."""

    def __init__(self, name, P=None):
        import numpy as np
        import oracle
        from paper_1711_10128_b200 import inputs
        oracle.build()
        self.name = name
        self.P = P if P is not None else inputs.make(name)
        self.cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
        self.full = name in FULL_SOLVE_CFGS
        if not self.full:
            P = self.P
            n = P.A.n
            m = P.q - P.p - P.l
            self.k0 = P.p + (m + 1) // 2
            self.U = np.empty((n, self.k0 + 1), order="F")
            self.U[:] = 0.0
            for c in range(self.k0):
                self.U[(c * 7919) % n, c] = 1.0
            self.work = np.empty(4 * n)
            self.work[:] = 0.0
            self.M = oracle.jacobi_diag(P.A, P.B, P.sigma)
            self.T = np.zeros((self.k0 + 1, self.k0 + 1), order="F")

    def step(self):
        """One sample; returns (A-matvecs, seconds)."""
        import oracle
        P = self.P
        if self.full:
            t0 = time.perf_counter()
            r = oracle.solve(P.A, P.B, P.p, P.q, P.l, P.tol, P.sigma, want_vectors=False)
            return r["a_matvecs"], time.perf_counter() - t0
        t0 = time.perf_counter()
        done, _ = oracle.inner_steps(P.A, P.B, self.M, 1.0, self.U, self.k0, 1, self.T, self.work)
        return done, time.perf_counter() - t0

    def describe(self, steps):
        P = self.P
        if self.full:
            return f"full oracle solve of {self.name}"
        return (f"{steps} oracle inner step(s) of eq 3.1 (orc_inner_steps: SpMV, T column, Jacobi, CGS2) at "
                f"full {self.name} size (n={P.A.n}) with basis width k={self.k0} (cycle average); "
                f"+K/RR/rotation/residual work not sampled (upper bound of the full-solve rate)")


def cpu_baseline(name, budget_s, P=None):
    """rank 0 at N=1: the oracle sample repeated until ~budget_s seconds of host work."""
    smp = OracleSample(name, P)
    mv = 0
    dt = 0.0
    steps = 0
    while True:
        a, t = smp.step()
        mv += a
        dt += t
        steps += 1
        if dt >= budget_s:
            break
    return {"value": mv / dt, "unit": UNIT, "cores": smp.cores, "kind": "oracle", "sample": smp.describe(steps),
            "seconds": dt}


def run_reference(args):
    """Reference arm = the oracle (this tier has no reference implementation), each step one
    OracleSample of the same workload as our arm."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    smp = OracleSample(args.config)
    P = smp.P
    mvs, times = [], []
    for i in range(args.warmup + args.steps):
        a, t = smp.step()
        if i >= args.warmup:
            mvs.append(a)
            times.append(t)
    v = sum(mvs) / sum(times)
    out = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded generator, BASELINE configs; paper matrices unavailable)",
           "config": static_config(args.config, P, P.A.n, args.gpus),
           "cpu_baseline": {"kind": "oracle", "cores": smp.cores, "sample": smp.describe(1) + " per step",
                            "value": v, "unit": UNIT},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


def run_pl1(args):
    """PL+1 (Algorithm 2) on one GPU: a step = one trplk_pl1_solve to tol (time to the lowest
    eigenpair).  value = A-matvecs / device solve time; roofline = the solve's algorithmic bytes
    (every launch of the iteration, DESIGN.md byte model) / solve time; e2e = create from pinned
    host CSR + solve + D2H of x + destroy; cpu_baseline = the oracle's orc_pl1_solve."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import torch
    from paper_1711_10128_b200 import build
    build.build()
    from paper_1711_10128_b200 import inputs, trplk
    P = inputs.make(args.config)
    m, tol = args.pl1_m, P.tol
    ctx = trplk.trplk_create(P.A, P.B, P.sigma)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(args.warmup):
        trplk.trplk_pl1_solve(ctx, m, tol)
    clocks = Clocks(int(os.environ.get("LOCAL_RANK", "0")))
    times, sts = [], []
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        rho, res, x, st, log = trplk.trplk_pl1_solve(ctx, m, tol)
        torch.cuda.synchronize()
        assert st["status"] == "OK", st
        times.append(st["solve_seconds"] * 1e3)
        sts.append(st)
    ck = clocks.stop()
    ms = statistics.mean(times)
    mv = sts[-1]["a_matvecs"]
    peak, peak_src = peaks()
    ach = sts[-1]["model_bytes"] / (ms * 1e-3) / 1e9
    # e2e: pinned host CSR -> create -> PL+1 -> x to pinned host -> destroy
    pin = [torch.from_numpy(a).pin_memory() for M in (P.A, P.B) if M is not None for a in (M.rowptr, M.col, M.val)]

    class _H:
        def __init__(self, rp, c, v):
            self.rowptr, self.col, self.val, self.n, self.row_begin = rp.numpy(), c.numpy(), v.numpy(), P.A.n, 0

    HA = _H(*pin[0:3])
    HB = _H(*pin[3:6]) if P.B is not None else None
    xh = torch.empty(P.A.n, dtype=torch.float64).pin_memory()
    et = []
    stream = torch.cuda.current_stream()
    for it in range(1 + max(1, min(args.steps, 3))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        c2 = trplk.trplk_create(HA, HB, P.sigma)
        trplk.trplk_pl1_solve(c2, m, tol, x_out=xh)
        c2.close()
        e1.record(stream)
        torch.cuda.synchronize()
        if it:
            et.append(e0.elapsed_time(e1))
    cpu = None
    if not args.no_cpu_baseline:
        import oracle
        oracle.build()
        t0 = time.perf_counter()
        o = oracle.pl1_solve(P.A, P.B, m=m, tol=tol, sigma=P.sigma)
        dt = time.perf_counter() - t0
        cpu = {"value": o["a_matvecs"] / dt, "unit": UNIT, "cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)),
               "kind": "oracle", "sample": f"full oracle PL+1 solve of {args.config} (m={m}, {o['cycles']} iterations)"}
    out = {"metric": "PL+1 A-matvecs/s to the lowest eigenpair (fp64)", "value": round(mv / (ms * 1e-3), 2),
           "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded generator, BASELINE configs; paper matrices unavailable)",
           "config": {"workload": f"{args.config}: {P.desc}; PL+1 m={m}, tol={tol}, Jacobi, seed 12",
                      "n": P.A.n, "iterations": sts[-1]["cycles"], "a_matvecs_per_solve": mv,
                      "rho": rho, "l2": "flushed (256 MiB write) between timed steps"},
           "roofline": {"bound": "hbm", "kernel": "whole PL+1 iteration (all launches, model bytes)",
                        "achieved": round(ach, 1), "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
                        "traffic": None, "peak_source": peak_src},
           "cpu_baseline": cpu,
           "e2e": {"value": mv / (statistics.mean(et) * 1e-3), "unit": UNIT,
                   "h2d_bytes_per_step": sum(t.numel() * t.element_size() for t in pin),
                   "d2h_bytes_per_step": P.A.n * 8, "ms_per_step": statistics.mean(et)},
           "gpu_launches": sts[-1]["kernel_launches"], "clocks": ck}
    ctx.close()
    print(json.dumps(out))
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.method == "pl1":
        return run_pl1(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % torch.cuda.device_count())
    group = None
    if world > 1:
        if args.comm == "host":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
    red_dev = "cpu" if args.comm == "host" else "cuda"  # max over ranks
    from paper_1711_10128_b200 import build
    build.build()
    from paper_1711_10128_b200 import inputs, trplk

    dim, N = inputs.CONFIGS[args.config][0], inputs.CONFIGS[args.config][1]
    n = N if dim == 1 else N ** 3
    plane = 1 if dim == 1 else N * N
    rb, re = inputs.slab_rows(n, world, rank, plane)
    P = inputs.make(args.config, row_begin=rb, row_end=re)
    if args.k_plus is not None:
        P.l = args.k_plus
    prec = {"jacobi": 0, "none": 1, "shifted": 2, "ic0": 3}[args.precond]
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    ctx = trplk.trplk_create(P.A, P.B, P.sigma, n_global=n, row_begin=rb, row_end=re, group=group,
                             comm=args.comm)
    evecs = torch.empty((P.p, ctx.n_local), dtype=torch.float64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def solve(**kw):
        return trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol, evecs_out=evecs, precond=prec, block=args.block, **kw)

    for w in range(args.warmup):
        # the last warm-up solve runs with the profile on too, so the timed region finds the
        # profiled cycle graphs already instantiated
        trplk.trplk_profile(ctx, w == args.warmup - 1)
        ev, _, rs, st = solve()
        assert st["status"] == "OK", st
    trplk.trplk_profile(ctx, False)
    clocks = Clocks(local)
    times, stats = [], []
    for it in range(args.steps):
        # the live kernel profile (CUDA event nodes around the middle inner step of every cycle)
        # serialises that step's kernels.  HBM-sized problems (n >= 2^21: C3-C5; cost below
        # 0.3 %): on every timed step.  The latency-bound ones (C1, C2), whose kernels otherwise
        # overlap inside the cycle graph (C2: 65.0 ms with it on every step against 60.4 ms,
        # profiles/r02_variants.md): on the last timed step only, as with --profile-last-only
        last_only = args.profile_last_only or n < (1 << 21)
        if it == (args.steps - 1 if last_only else 0):
            trplk.trplk_profile(ctx, True)
        flush.fill_(1.0)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ev, _, rs, st = solve()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        times.append(e0.elapsed_time(e1))
        stats.append(st)
    ck = clocks.stop()
    prof = trplk.trplk_profile_read(ctx)
    kern_names = trplk.trplk_profile_kernels(ctx)
    phases = trplk.trplk_profile_phases(ctx)
    trplk.trplk_profile(ctx, False)
    t_sum = torch.tensor([sum(times)], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t_sum, op=dist.ReduceOp.MAX)
    ms_per_step = t_sum.item() / args.steps
    mv = stats[-1]["a_matvecs"]
    assert all(s["a_matvecs"] == mv for s in stats)
    value = mv / (ms_per_step / 1e3)

    # roofline: inner-step kernel group with the largest share (live CUDA events, per launch)
    groups = ["K1 (SpMV + Jacobi + T-column / h1 dots)", "K2 (CGS pass 2: update + dots)",
              "K3 (CGS final update + normalisation)"]
    if kern_names and "k_fin_step1" in kern_names[0]:  # fused step: [K3 of step j + K1 of step j+1, K2, -]
        groups = ["K3+K1 (CGS final update of step j + SpMV/Jacobi/T-column/h1 dots of step j+1)",
                  "K2 (CGS pass 2: update + dots)", "-"]
    peak, peak_src = peaks()
    cnt = max(prof["count"], 1)
    per_ms = prof["ms"] / cnt
    per_b = prof["bytes"] / cnt
    kd = int(np.argmax(per_ms))
    kname = ncu_name(kern_names[kd]) if kd < len(kern_names) else ""
    # `achieved` counts ALGORITHMIC bytes: SURVEY 8(d)'s per-kernel figures, matrix as CSR
    # (bytes(A) = 12 nnz + 4 (n + 1); K1 = bytes(A) [+ bytes(B)] + 8n(k+2), K2 / K3 = 8n(k+2)
    # [+ the B products]), whatever format the kernel reads.  The library's own figures (per_b)
    # count the device format actually read (DIA values 8 ndiag n, DIA-C presence bits, SELL)
    # and are reported beside it as `device_format`.  The one-launch paths (C1's single-CTA
    # inner loop, the grid-wide loop, the fused step) keep the library's figures.
    alg_b = per_b.copy()
    std3 = len(kern_names) >= 3 and all(not any(t in x for t in ("k_inner_small", "k_inner_grid", "k_fin_step1"))
                                        for x in kern_names) and per_b[2] > 0
    if std3:
        info = trplk.trplk_info(ctx)
        csr = lambda M: 0.0 if M is None else 12.0 * len(M.val) + 4.0 * len(M.rowptr)  # noqa: E731
        vec = per_b[2]  # 8n(k+2) averaged over the profiled steps
        alg_b[0] = csr(P.A) + csr(P.B) + vec
        alg_b[1] = per_b[1] + 2.0 * (csr(P.B) - float(info["sell_bytes_b"])) if P.B is not None else per_b[1]
    achieved = alg_b[kd] / (per_ms[kd] * 1e-3) / 1e9
    step_gbs = alg_b.sum() / (per_ms.sum() * 1e-3) / 1e9
    dev_gbs = per_b[kd] / (per_ms[kd] * 1e-3) / 1e9
    dev_step_gbs = per_b.sum() / (per_ms.sum() * 1e-3) / 1e9
    # ncu DRAM bytes per launch of the same kernel instantiation (profiles/traffic_<cfg>.json,
    # tools/make_traffic.py, cold cache)
    traffic = None
    tfile = os.path.join(PROFILES, f"traffic_{args.config}.json")
    if os.path.exists(tfile) and kname:
        traffic = json.load(open(tfile)).get(kname)
    roof = {"bound": "hbm", "kernel": f"{groups[kd]}: {kname}", "achieved": round(achieved, 1), "peak": peak,
            "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
            "traffic_source": f"profiles/traffic_{args.config}.json[{kname!r}]" if traffic else None,
            "peak_source": peak_src, "kernels": [ncu_name(x) for x in kern_names],
            "bytes_per_launch": alg_b[kd], "ms_per_launch": per_ms[kd],
            "bytes_model": ("SURVEY 8(d) algorithmic bytes (matrix as CSR: 12 nnz + 4(n+1))" if std3
                            else "library figures (device format)"),
            "inner_step": {"achieved": round(step_gbs, 1), "frac": round(step_gbs / peak, 4),
                           "bytes": alg_b.sum(), "ms": per_ms.sum(),
                           "share_ms": [round(x / per_ms.sum(), 3) for x in per_ms]},
            "device_format": {"bytes_per_launch": per_b[kd], "achieved": round(dev_gbs, 1),
                              "frac": round(dev_gbs / peak, 4),
                              "inner_step": {"bytes": per_b.sum(), "achieved": round(dev_step_gbs, 1),
                                             "frac": round(dev_step_gbs / peak, 4)}},
            "cycle_phases_ms": {nm: round(v / max(phases["count"], 1), 4) for nm, v in zip(phases["phases"], phases["ms"])},
            "cycle_phase_share": {nm: round(v / max(phases["ms"].sum(), 1e-30), 4)
                                  for nm, v in zip(phases["phases"], phases["ms"])},
            "solve_model_gbs": round(stats[-1]["model_bytes"] / (ms_per_step * 1e-3) / 1e9, 1),
            "samples": prof["count"]}

    # e2e through the public API with host buffers (pinned), every step
    e2e = None
    if not args.no_e2e:
        pin = []
        for M in (P.A, P.B):
            if M is None:
                continue
            pin += [torch.from_numpy(M.rowptr).pin_memory(), torch.from_numpy(M.col).pin_memory(),
                    torch.from_numpy(M.val).pin_memory()]
        host_evecs = torch.empty((P.p, ctx.n_local), dtype=torch.float64).pin_memory()

        class _HostCSR:
            def __init__(self, rp, c, v, n_):
                self.rowptr, self.col, self.val, self.n, self.row_begin = rp.numpy(), c.numpy(), v.numpy(), n_, rb

        HA = _HostCSR(*pin[0:3], n)
        HB = _HostCSR(*pin[3:6], n) if P.B is not None else None
        h2d = sum(t.numel() * t.element_size() for t in pin)
        d2h = host_evecs.numel() * 8 + 2 * P.p * 8
        et = []
        big = n > 50_000_000  # C5: each e2e round is a full create + 20 s solve
        ne_warm = 1 if big else max(1, min(args.warmup, 3))
        for it in range(ne_warm + (max(1, min(args.steps, 2)) if big else max(1, min(args.steps, 5)))):
            flush.fill_(1.0)
            barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            c2 = trplk.trplk_create(HA, HB, P.sigma, n_global=n, row_begin=rb, row_end=re, group=group,
                                    comm=args.comm)
            ev2, _, rs2, st2 = trplk.trplk_solve(c2, P.p, P.q, P.l, P.tol, evecs_out=host_evecs, precond=prec,
                                                 block=args.block)
            c2.close()
            e1.record(stream)
            torch.cuda.synchronize()
            if it >= ne_warm:  # untimed warm-up: first-touch allocator growth, lazy module loads
                et.append(e0.elapsed_time(e1))
        te = torch.tensor([statistics.mean(et)], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": st2["a_matvecs"] / (te.item() / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": te.item()}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if not args.no_e2e:
            del pin, HA, HB, host_evecs  # release the pinned host copies before the oracle sample
        cb = cpu_baseline(args.config, args.cpu_seconds, P)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}

    if rank == 0:
        out = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (seeded generator, BASELINE configs; paper matrices unavailable)",
               "config": static_config(args.config, P, n, world,
                                       {0: "Jacobi", 1: "no (M = I)", 2: "per-cycle shifted Jacobi", 3: "IC(0)"}[prec],
                                       args.comm, args.block),
               "solve": {"a_matvecs_per_solve": mv, "cycles": stats[-1]["cycles"],
                         "time_to_p_eigenpairs_ms": round(ms_per_step, 4),
                         "status": stats[-1]["status"]},
               "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": int(sum(s["kernel_launches"] for s in stats)), "clocks": ck,
               "eigenvalues": [float(x) for x in ev], "max_residual": float(np.max(rs))}
        print(json.dumps(out))
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
