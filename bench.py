#!/usr/bin/env python
"""bench.py -- PSP-GMRES implicit-Euler time steps on B200 through libpspgmres (C ABI).

One "step" = one pass of the whole hot path: the restarted PSP-GMRES
solve of (I - dt L) u^{n+1} = u^n (Alg.1) with probe recording, then the MREP fit
(Alg.2), the R21 gate and the banded factorisation for the next step.  Workload: BASELINE
configs[3] (C4, 3-D variable-kappa diffusion 512^3, d = 3, GMRES(30), tol 1e-8, m_max = 32).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--size 512]

metric/unit: BASELINE.json's metric, measured as unknown-iterations/s = sum over ranks of
n * (inner iterations) / (max over ranks of the device time of the K timed steps).
The --impl reference arm times the CPU oracle (oracle/) on a bounded sample of the same
workload on the host cores (rank 0 only).  See DESIGN.md section 8.
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
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "PSP-GMRES unknown-iterations/s and MREP rows/s at 1/2/4/8 GPUs, % HBM peak"
UNIT = "unknown-iterations/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size", type=int, default=512, help="grid points per axis (512 = C4)")
    ap.add_argument("--ortho", default="1reduce", choices=["1reduce", "literal"])
    ap.add_argument("--fused", type=int, default=1,
                    help="1: ring-resident Krylov basis, steps fused_kmin..fused_kmax as one fused pass; 0: split passes")
    ap.add_argument("--fused-kmin", type=int, default=None)
    ap.add_argument("--fused-kmax", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-size", type=int, default=128)
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent replicas instead of one z-slab-sharded problem")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 MREP / banded-solve kernel sweep point")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "host"],
                    help="multi-rank collectives: NCCL (one GPU a rank), or the library's host transport over "
                         "torch.distributed gloo (the sharded path with several ranks on one GPU: testing)")
    ap.add_argument("--c5-log2n", type=int, default=26)
    ap.add_argument("--no-sweep", action="store_true",
                    help="skip the C5 sweep (m x d grid) and the C1 / C2 / PSP-CG config lines")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if self.p is None:
            return out
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return out
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        out.update(sm_mhz=statistics.median(sm) if sm else None, sm_max_mhz=max(mx) if mx else None,
                   reasons=reasons, samples=len(rows))
        return out


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"host_cpu": model, "nproc": os.cpu_count()}


def cpu_baseline(size, budget_s=20.0):
    """The oracle as it stands (single-threaded C, literal Alg.1) on a bounded sample of C4."""
    import numpy as np

    import oracle
    from paper_1308_5626_b200 import inputs
    prob = inputs.c4(n=size, steps=1)
    b = prob.u0
    eps = prob.tol * float(np.linalg.norm(b))
    iters = 0
    t0 = time.perf_counter()
    x0 = b.copy()
    cycles = 0
    while time.perf_counter() - t0 < budget_s:
        r = oracle.pspgmres(prob.op, b, x0, eps, prob.restart, 1)
        iters += r["report"]["iterations"]
        cycles += 1
        x0 = r["x"]
        if r["report"]["converged"]:
            break
    t = time.perf_counter() - t0
    n = prob.op.rows
    return {"value": n * iters / t, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"C4 recipe at {size}^3 (n={n}), first time step, {cycles} GMRES(30) cycle(s) "
                      f"= {iters} iterations in {t:.1f} s, literal MGS, 1 host thread", **host_info()}


def c5_point(log2n, m, d, peak):
    """One C5 sweep point (BASELINE configs[4]): MREP fit, banded factor and two-sweep solve on
    device-generated probes (inputs.c5_torch recipe), each timed with CUDA events."""
    import torch

    from paper_1308_5626_b200 import inputs, pspgmres as P
    n = 1 << log2n
    g = inputs.c5_torch(n, m, d, seed=0)
    scratch = P.raw_scratch(n, d)
    s = torch.cuda.current_stream()

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    fit = {}

    def do_fit():
        fit.update(P.psp_mrep_fit_raw(g["px"], g["py"], d, scratch=scratch, want_kind=False))
    t_fit = timed(do_fit, 3)
    bands = fit["bands"]
    lu_box = {}

    def do_factor():
        lu_box["st"], lu_box["lu"] = P.psp_banded_factor_raw(bands, d, scratch=scratch)
    t_fac = timed(do_factor, 1)
    z = torch.empty_like(g["v"])
    t_sol = timed(lambda: P.psp_banded_solve_raw(lu_box["lu"], d, g["v"], scratch=scratch, out=z), 10)
    b_fit, b_sol, b_fac = 16 * m + 8 * (2 * d + 1), 8 * (2 * d + 5), 16 * (2 * d + 1)

    def rl(b, t):
        ach = b * n / (t / 1e3) / 1e9
        return {"ms": t, "rows_per_s": n / (t / 1e3), "bytes_per_row": b, "achieved_GBps": ach,
                "frac": ach / peak}
    out = {"workload": f"C5 (BASELINE configs[4]) n=2^{log2n}, m={m}, d={d}", "gate_accepted": fit["gate_accepted"],
           "mrep_fit": rl(b_fit, t_fit), "banded_factor": rl(b_fac, t_fac), "banded_solve": rl(b_sol, t_sol)}
    del g, scratch, bands, lu_box, z
    torch.cuda.empty_cache()
    return out


def c5_sweep(log2n, peak, ms=(16, 32, 64, 128), ds=(1, 2, 3, 4)):
    """BASELINE configs[4] as a grid: MREP fit rows/s and its fraction of the measured copy peak
    for every m x d (n = 2^log2n; m = 128 at 2^(log2n-1): the P_x / P_y pair of 2^26 x 128 columns
    would take 128 GiB), the banded factor and solve per d (independent of m)."""
    import torch

    from paper_1308_5626_b200 import inputs, pspgmres as P
    s = torch.cuda.current_stream()

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    out = {"mrep_fit": [], "banded_factor": [], "banded_solve": []}
    for m in ms:
        l2 = log2n - (1 if m >= 128 else 0)
        n = 1 << l2
        for d in ds:
            g = inputs.c5_torch(n, m, d, seed=0)
            scratch = P.raw_scratch(n, d)
            box = {}
            t = timed(lambda: box.update(P.psp_mrep_fit_raw(g["px"], g["py"], d, scratch=scratch, want_kind=False)), 2)
            b = 16 * m + 8 * (2 * d + 1)
            ach = b * n / (t / 1e3) / 1e9
            out["mrep_fit"].append({"n": n, "m": m, "d": d, "ms": t, "rows_per_s": n / (t / 1e3), "bytes_per_row": b,
                                    "achieved_GBps": ach, "frac": ach / peak, "gate_accepted": box["gate_accepted"]})
            if m == 32:
                lu_box = {}

                def do_factor():
                    lu_box["st"], lu_box["lu"] = P.psp_banded_factor_raw(box["bands"], d, scratch=scratch)
                tf = timed(do_factor, 1)
                z = torch.empty_like(g["v"])
                ts = timed(lambda: P.psp_banded_solve_raw(lu_box["lu"], d, g["v"], scratch=scratch, out=z), 5)
                bf, bs = 16 * (2 * d + 1), 8 * (2 * d + 5)
                for key, tt, bb in (("banded_factor", tf, bf), ("banded_solve", ts, bs)):
                    a2 = bb * n / (tt / 1e3) / 1e9
                    out[key].append({"n": n, "d": d, "ms": tt, "rows_per_s": n / (tt / 1e3), "bytes_per_row": bb,
                                     "achieved_GBps": a2, "frac": a2 / peak})
                del lu_box, z
            del g, scratch, box
            torch.cuda.empty_cache()
    return out


def config_lines():
    """The other BASELINE configs as step timings through the same C ABI (CUDA events around
    psp_step): C1 (1-D, n = 1024, 5 steps) and C2 (2-D 512^2, d = 1, 20 steps) on the
    device-resident solve (f2), C3 (2-D 2048^2 advection-diffusion, the first 2 of its 10 steps,
    default options: fused passes) and C4 with PSP-CG (f4, 3 steps after one warm-up)."""
    import torch

    from paper_1308_5626_b200 import inputs, pspgmres as P
    res = {}
    for key, mk, steps, warm, kw in (("C1_resident", lambda: inputs.c1(), 5, 0, dict(resident=2)),
                                     ("C2_resident", lambda: inputs.c2(d=1), 20, 0, dict(resident=2)),
                                     ("C3", lambda: inputs.c3(steps=2), 2, 0, {}),
                                     ("C4_psp_cg", lambda: inputs.c4(steps=4), 3, 1, dict(method=P.PSP_METHOD_CG))):
        prob = mk()
        opts = P.default_opts(max_cycles=prob.max_cycles, m_max=prob.m_max, **kw)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol, opts=opts, stream=st)
            u = torch.as_tensor(prob.u0).cuda()
        for _ in range(warm):
            ctx.psp_step(u, u)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        reps = [ctx.psp_step(u, u) for _ in range(steps)]
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        n = prob.op.rows
        its = [r["iterations"] for r in reps]
        res[key] = {"n": n, "steps": steps, "ms_per_step": ms / steps, "iterations_per_step": its,
                    "unknown_iterations_per_s": n * sum(its) / (ms / 1e3),
                    "converged": all(r["converged"] for r in reps),
                    "gate_accepted_per_step": [r["mrep_gate_accepted"] for r in reps]}
        ctx.close()
        del ctx, u, prob
        torch.cuda.empty_cache()
    return res


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    import numpy as np

    import oracle
    from paper_1308_5626_b200 import inputs
    size = args.cpu_sample_size
    prob = inputs.c4(n=size, steps=1)
    b = prob.u0
    eps = prob.tol * float(np.linalg.norm(b))
    n = prob.op.rows

    def one_step():   # bounded sample of one time step: its first GMRES(30) cycle
        t0 = time.perf_counter()
        r = oracle.pspgmres(prob.op, b, b, eps, prob.restart, 1)
        return r["report"]["iterations"], time.perf_counter() - t0

    for _ in range(args.warmup):
        one_step()
    tot_it, tot_t = 0, 0.0
    for _ in range(args.steps):
        it, t = one_step()
        tot_it += it
        tot_t += t
    value = n * tot_it / tot_t
    sample = f"C4 recipe at {size}^3 (n={n}), one GMRES(30) cycle of the first time step per step"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": "C4 (BASELINE configs[3]) sample", "grid": [size] * 3,
                                            "d": 3, "restart": 30, "tol": 1e-8},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                             **host_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch

    from paper_1308_5626_b200 import inputs, pspgmres as P

    assert torch.cuda.is_available(), "bench.py needs a GPU (libpspgmres has no CPU path)"
    host_tr = args.transport == "host"
    torch.cuda.set_device(local % torch.cuda.device_count() if host_tr else local)
    red_dev = "cpu" if host_tr else "cuda"              # device of the bench's own reductions
    dist = None
    if world > 1:
        import torch.distributed as dist
        if host_tr:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    # ---- workload: C4 512^3.  N > 1: one problem, z-slab sharded over the ranks (SURVEY 8(e):
    #      halo planes by NCCL send/recv, all-reduced Arnoldi scalars); --replicas: one
    #      independent replica per rank ----
    t_gen = time.perf_counter()
    prob = inputs.c4(n=args.size, steps=args.warmup + args.steps)
    t_gen = time.perf_counter() - t_gen
    n = prob.op.rows
    sharded = world > 1 and not args.replicas
    comm = None
    transport = None
    if sharded:
        if host_tr:
            transport = P.TorchDistTransport()                # (kept alive with the communicator)
            comm = P.psp_comm_host_create(transport, world, rank)
        else:
            uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
            if rank == 0:
                uid.copy_(torch.frombuffer(bytearray(P.psp_comm_unique_id()), dtype=torch.uint8))
            dist.broadcast(uid, 0)
            comm = P.psp_comm_init(bytes(uid.cpu().numpy().tobytes()), world, rank)
        # every collective of the hot path once over the communicator, checked (fail loudly)
        st = P.psp_comm_selftest(comm, torch.cuda.current_stream())
        if st != P.PSP_OK:
            raise RuntimeError(f"communicator self-test failed on rank {rank}: status {st}")
    ortho = P.PSP_MGS_1REDUCE if args.ortho == "1reduce" else P.PSP_MGS_LITERAL
    fk = {}
    if args.fused_kmin is not None:
        fk["fused_kmin"] = args.fused_kmin
    if args.fused_kmax is not None:
        fk["fused_kmax"] = args.fused_kmax
    # timing 1 (the reports' solve / MREP / factor times) in the headline region; the per-launch
    # event pairs (timing 2) only in the instrumented region after it (psp_set_timing)
    opts = P.default_opts(max_cycles=prob.max_cycles, m_max=prob.m_max, ortho=ortho, timing=1, fused=args.fused, **fk)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        if sharded:
            ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol, opts=opts, stream=stream,
                            comm=comm, nranks=world, rank=rank)
            u = torch.as_tensor(prob.u0[ctx.row0:ctx.row0 + ctx.n]).cuda()
        else:
            ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol, opts=opts, stream=stream)
            u = torch.as_tensor(prob.u0).cuda()
    n_local = ctx.n
    prob.u0 = None
    prob.op.field = None
    stream.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()

    # ---- warm-up (untimed) ----
    for _ in range(args.warmup):
        ctx.psp_step(u, u)
    ctx.psp_kernel_stats(reset=True)
    l0 = ctx.psp_launch_count()

    # ---- timed region: K steps, device time via CUDA events on the solver stream ----
    clocks = Clocks(torch.cuda.current_device())
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0.record(stream)
    reps = []
    for _ in range(args.steps):
        reps.append(ctx.psp_step(u, u))
    ev1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    barrier()
    t_ms = ev0.elapsed_time(ev1)
    launches = ctx.psp_launch_count() - l0
    iters = sum(r["iterations"] for r in reps)

    # ---- instrumented region: K more steps with an event pair around every launch (the kernel
    # table and the roofline's per-launch times; its own device time is reported beside) ----
    ctx.psp_set_timing(2)
    ctx.psp_kernel_stats(reset=True)
    ev2 = torch.cuda.Event(enable_timing=True)
    ev3 = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    ev2.record(stream)
    reps_i = [ctx.psp_step(u, u) for _ in range(args.steps)]
    ev3.record(stream)
    torch.cuda.synchronize()
    barrier()
    t_instr_ms = ev2.elapsed_time(ev3)
    kstats = ctx.psp_kernel_stats(reset=True)
    ctx.psp_set_timing(1)
    iters_instr = sum(r["iterations"] for r in reps_i)
    if dist is not None:
        tt = torch.tensor([t_ms], dtype=torch.float64, device=red_dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
        # sharded: every rank iterates the same global problem (n unknowns); replicas: sum
        it = torch.tensor([float(n * iters)], dtype=torch.float64, device=red_dev)
        dist.all_reduce(it, op=dist.ReduceOp.MAX if sharded else dist.ReduceOp.SUM)
        total_unknown_iters = float(it.item())
    else:
        total_unknown_iters = float(n * iters)
    value = total_unknown_iters / (t_ms / 1e3)

    # ---- roofline of the dominant kernel class (largest share of the timed device time) ----
    peak, peak_src = peaks()
    dom = max((k for k in kstats if kstats[k]["launches"] > 0), key=lambda k: kstats[k]["ms"])
    ds = kstats[dom]
    avg_ms = ds["ms"] / ds["launches"]
    avg_bytes = ds["bytes"] / ds["launches"]
    achieved = avg_bytes / (avg_ms / 1e3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        if dom in tj and tj[dom].get("size") == args.size:
            traffic = tj[dom]["traffic_over_algorithmic"] * avg_bytes
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": avg_bytes, "avg_launch_ms": avg_ms,
                "share_of_step": ds["ms"] / t_instr_ms,
                "measured_in": "the instrumented region (K steps after the headline region, timing 2)"}
    kernel_table = {k: {"ms": v["ms"], "launches": v["launches"],
                        "GBps": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 else None,
                        "share": v["ms"] / t_instr_ms} for k, v in kstats.items() if v["launches"]}

    # ---- e2e: same metric through the C ABI with host buffers, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        host = torch.empty(n_local, dtype=torch.float64).pin_memory()
        host.copy_(u.cpu())
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        it_e2e = 0
        with torch.cuda.stream(stream):
            for _ in range(args.steps):
                u.copy_(host, non_blocking=True)             # H2D of the step's input u^n
                r = ctx.psp_step(u, u)
                host.copy_(u, non_blocking=True)             # D2H of the step's result u^{n+1}
                it_e2e += r["iterations"]
        e1.record(stream)
        torch.cuda.synchronize()
        te = e0.elapsed_time(e1)
        tot = float(n * it_e2e)
        if dist is not None:
            tt = torch.tensor([te], dtype=torch.float64, device=red_dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
            it = torch.tensor([tot], dtype=torch.float64, device=red_dev)
            dist.all_reduce(it, op=dist.ReduceOp.MAX if sharded else dist.ReduceOp.SUM)
            tot = float(it.item())
        e2e = {"value": tot / (te / 1e3), "unit": UNIT, "h2d_bytes_per_step": 8 * n_local,
               "d2h_bytes_per_step": 8 * n_local}
        ctx.psp_kernel_stats(reset=True)

    line = None
    if rank == 0:
        mrep_ms = kstats.get("mrep_fit", {}).get("ms", 0.0)
        solve_ms = sum(r["t_solve_ms"] for r in reps) if reps and reps[0]["t_solve_ms"] else None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C4: 3-D variable-kappa diffusion {args.size}^3 (BASELINE configs[3]), "
                                   "one implicit-Euler PSP-GMRES time step (solve + MREP fit + gate + factor)",
                       "grid": [args.size] * 3, "n": n, "d": prob.d, "restart": prob.restart, "tol": prob.tol,
                       "m_max": prob.m_max,
                       "ortho": args.ortho + (f"-ring(fused k={opts.fused_kmin}..{opts.fused_kmax})" if args.fused else "-split"),
                       "dt": prob.op.dt,
                       "l2": "inputs larger than L2 (each vector 8n bytes >> 126 MB); no flush needed",
                       "parallelism": (f"z-slab x{world} ({'host transport over gloo' if host_tr else 'NCCL'} halo + all-reduce)" if sharded else
                                       ("replicas" if world > 1 else "single"))},
            "iterations_per_step": [r["iterations"] for r in reps],
            "cycles_per_step": [r["cycles"] for r in reps],
            "precond_identity_per_step": [r["precond_identity"] for r in reps],
            "gate_accepted_per_step": [r["mrep_gate_accepted"] for r in reps],
            "converged": all(r["converged"] for r in reps),
            "true_resid_over_eps": max(r["final_resid_true"] / r["eps"] for r in reps),
            "mrep_rows_per_s": (n * args.steps / (mrep_ms / 1e3)) if mrep_ms else None,
            # SURVEY 8(d)'s reading: t_solve only (the MREP fit, gate and factor timed apart);
            # `value` above keeps them inside the step
            "solve_only": ({"value": n * sum(r["iterations"] for r in reps) / (solve_ms / 1e3),
                            "unit": UNIT, "ms_per_step": solve_ms / args.steps,
                            "definition": "n x sum(iterations) / sum(t_solve), CUDA events (opts.timing)"}
                           if solve_ms else None),
            # the steady-state time per Arnoldi iteration (t_solve / iterations of
            # each timed step, its median over the steps)
            "ms_per_iteration": ({"median": statistics.median([r["t_solve_ms"] / r["iterations"] for r in reps
                                                                if r["iterations"]]),
                                  "per_step": [r["t_solve_ms"] / r["iterations"] for r in reps if r["iterations"]]}
                                 if solve_ms else None),
            "kernels": kernel_table,
            # the kernel table and the roofline come from this second region of K steps (event
            # pairs around every launch); `value` / ms_per_step from the headline region without them
            "instrumented_region": {"ms_per_step": t_instr_ms / args.steps,
                                    "iterations_per_step": [r["iterations"] for r in reps_i],
                                    "unknown_it_per_s": n * iters_instr / (t_instr_ms / 1e3)},
            "roofline": roofline,
            "gpu_launches": int(launches),
            "clocks": clk,
            "e2e": e2e,
            "input_generation_s": t_gen,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args.cpu_sample_size)
    ctx.close()
    if comm is not None:
        P.psp_comm_destroy(comm)
    del ctx, u
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    if line is not None and world == 1 and not args.no_c5:
        # the north star's per-kernel targets (matvec from the C4 step above; MREP fit and the
        # banded solve on a C5 point, where the gate accepts N)
        try:
            c5 = c5_point(args.c5_log2n, 32, 3, peak)
        except Exception as e:  # noqa: BLE001 -- the C4 line stands; say what failed
            c5 = {"error": f"{type(e).__name__}: {e}"[:300]}
            line["c5"] = c5
            print(json.dumps(line), flush=True)
            if dist is not None:
                dist.destroy_process_group()
            return 0
        line["c5"] = c5
        if not args.no_sweep:
            try:
                line["c5_sweep"] = c5_sweep(args.c5_log2n, peak)
            except Exception as e:  # noqa: BLE001
                line["c5_sweep"] = {"error": f"{type(e).__name__}: {e}"[:300]}
            try:
                line["configs"] = config_lines()
            except Exception as e:  # noqa: BLE001
                line["configs"] = {"error": f"{type(e).__name__}: {e}"[:300]}
        mv = kstats.get("matvec", {})
        line["kernel_rooflines"] = {
            "matvec": {"achieved_GBps": kernel_table.get("matvec", {}).get("GBps"), "peak": peak,
                       "frac": (kernel_table.get("matvec", {}).get("GBps") or 0.0) / peak,
                       "bytes_per_row": 24, "workload": "C4 step (ring mode: x and kappa read, A x written)"} if mv else None,
            "mrep_fit": {"achieved_GBps": c5["mrep_fit"]["achieved_GBps"], "peak": peak,
                         "frac": c5["mrep_fit"]["frac"], "workload": c5["workload"]},
            "banded_solve": {"achieved_GBps": c5["banded_solve"]["achieved_GBps"], "peak": peak,
                             "frac": c5["banded_solve"]["frac"], "workload": c5["workload"]}}
    if line is not None:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
