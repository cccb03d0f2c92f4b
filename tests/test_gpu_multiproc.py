"""The multi-rank path across PROCESSES: world_size-2 (and 3) torch.distributed jobs (gloo) on one
B200, each rank a separate process driving psp_step through the library with the process-level
host transport (psp_comm_host_create over pspgmres.TorchDistTransport).  Host-mediated: every
collective synchronises the rank's stream and moves data through pinned host buffers, so no
kernel waits on another process.  The sharded result must match the single-rank solve (T4 floor,
T5) and the oracle (both solve the same implicit-Euler steps to tol)."""
import os
import socket
import tempfile

import numpy as np
import pytest

from paper_1308_5626_b200 import inputs

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(name):
    if name == "C4s":
        return inputs.Problem("C4s", inputs.OperatorSpec(3, "cell_diff", (20, 18, 16), 2e-4,
                                                         field=np.exp(np.random.default_rng(5).standard_normal(20 * 18 * 16))),
                              np.random.default_rng(6).uniform(-1, 1, 20 * 18 * 16), 30, 1e-8, 3, 2, 32, 1000)
    return inputs.c1(steps=3)


def _worker(rank, world, port, name, steps, outdir):
    import torch
    import torch.distributed as dist

    from paper_1308_5626_b200 import pspgmres as P
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    prob = _problem(name)
    tr = P.TorchDistTransport()
    comm = P.psp_comm_host_create(tr, world, rank)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        opts = P.default_opts(max_cycles=prob.max_cycles, m_max=prob.m_max)
        ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol, opts=opts, stream=s,
                        comm=comm, nranks=world, rank=rank)
        u = torch.as_tensor(prob.u0[ctx.row0:ctx.row0 + ctx.n]).cuda()
        reps = [ctx.psp_step(u, u) for _ in range(steps)]
        s.synchronize()
    np.savez(os.path.join(outdir, f"r{rank}.npz"), u=u.cpu().numpy(), row0=ctx.row0,
             iters=[r["iterations"] for r in reps], cycles=[r["cycles"] for r in reps],
             gate=[r["mrep_gate_accepted"] for r in reps], ident=[r["precond_identity"] for r in reps],
             h0=reps[0]["resid_history"], b0=reps[0]["beta_history"], tr=[r["final_resid_true"] / r["eps"] for r in reps])
    ctx.close()
    P.psp_comm_destroy(comm)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world,steps", [("C4s", 2, 2), ("C4s", 3, 2), ("C1", 2, 3)])
def test_multiprocess_step_matches_single_rank(orc, name, world, steps):
    import torch
    import torch.multiprocessing as mp

    from paper_1308_5626_b200 import pspgmres as P
    assert torch.cuda.is_available()
    prob = _problem(name)
    with tempfile.TemporaryDirectory() as td:
        ctx = mp.get_context("spawn")
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, world, port, name, steps, td)) for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=600)
            assert p.exitcode == 0
        parts = [dict(np.load(os.path.join(td, f"r{r}.npz"))) for r in range(world)]
    u = np.concatenate([p["u"] for p in parts])
    for p in parts[1:]:                                   # every rank reports the same thing
        assert list(p["iters"]) == list(parts[0]["iters"]) and list(p["gate"]) == list(parts[0]["gate"])
    # the single-rank solve of the same steps (host-driven, as the sharded path)
    opts = P.default_opts(max_cycles=prob.max_cycles, m_max=prob.m_max, resident=0)
    c1 = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol, opts=opts)
    us = torch.as_tensor(prob.u0).cuda()
    reps = [c1.psp_step(us, us) for _ in range(steps)]
    c1.close()
    p0 = parts[0]
    for s in range(steps):
        assert abs(int(p0["iters"][s]) - reps[s]["iterations"]) <= 1
        assert int(p0["ident"][s]) == reps[s]["precond_identity"]
        assert bool(p0["gate"][s]) == bool(reps[s]["mrep_gate_accepted"])
        assert p0["tr"][s] <= 1.05
    h0, hs = p0["h0"], reps[0]["resid_history"]
    first = min(len(h0), len(hs), prob.restart)
    beta = reps[0]["beta_history"][0]
    assert np.all(np.abs(h0[:first] - hs[:first]) <= 1e-8 * hs[:first] + 1e-11 * beta)   # T4, first cycle
    r = orc.time_steps(prob.op, prob.u0, steps, prob.restart, prob.max_cycles, prob.tol, prob.d, prob.m_max)
    assert abs(int(p0["iters"][0]) - r["reports"][0]["solve"]["iterations"]) <= 1
    if name == "C1":
        kappa = 1 + 4 * 1e-3 * 1025.0 ** 2
        assert np.linalg.norm(u - r["u"]) <= kappa * 2 * prob.tol * np.linalg.norm(r["u"]) * steps
    else:
        h = 1.0 / 21
        normA = 1 + 12 * prob.op.dt * prob.op.field.max() / h ** 2
        assert np.linalg.norm(u - r["u"]) <= 2 * steps * prob.tol * normA * np.linalg.norm(prob.u0)
