"""Debug aid: the C1 time steps on 1 rank vs nranks loopback ranks, step by step."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_1308_5626_b200 import inputs, pspgmres as P  # noqa: E402
from test_gpu_multirank import multi_steps, single_steps, run_ranks  # noqa: E402

nranks = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prob = inputs.c1(steps=3)
m = multi_steps(torch, P, prob, nranks, 3)
s = single_steps(torch, P, prob, 3)
for i, (rm, rs) in enumerate(zip(m["reps"], s["reps"])):
    print("step", i, "iters multi/single", rm["iterations"], rs["iterations"], "ident", rm["precond_identity"],
          rs["precond_identity"], "gate", rm["mrep_gate_accepted"], rs["mrep_gate_accepted"],
          "ridge", rm["mrep_rows_ridge"] if "mrep_rows_ridge" in rm else None)
    print("   resid multi", rm["resid_history"][:8])
    print("   resid single", rs["resid_history"][:8])
db = np.abs(m["bands"] - s["bands"])
print("bands max diff", db.max(), "at", np.unravel_index(db.argmax(), db.shape), "n", m["bands"].shape)
for p in m["parts"]:
    print("rank row0", p["row0"], "iters", [r["iterations"] for r in p["reps"]])
cols = np.where(db.max(axis=0) > 1e-6)[0]
print("bad columns", cols[:40], len(cols))
# precond solve with the single-rank bands on multi ranks
bands = s["bands"]
v = np.random.default_rng(1).standard_normal(bands.shape[1])
ctx1 = P.Context(prob.op, d=prob.d, restart=4, tol=1e-8)
assert ctx1.psp_set_bands(torch.as_tensor(bands).cuda())
z1 = torch.empty(bands.shape[1], dtype=torch.float64, device="cuda")
ctx1.psp_precond_apply(torch.as_tensor(v).cuda(), z1)
z1 = z1.cpu().numpy()


def fn(rank, comm):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        ctx = P.Context(prob.op, d=prob.d, restart=4, tol=1e-8, stream=st, comm=comm, nranks=nranks, rank=rank)
        bl = torch.as_tensor(np.ascontiguousarray(bands[:, ctx.row0:ctx.row0 + ctx.n])).cuda()
        acc = ctx.psp_set_bands(bl)
        vl = torch.as_tensor(v[ctx.row0:ctx.row0 + ctx.n]).cuda()
        zl = torch.empty_like(vl)
        ctx.psp_precond_apply(vl, zl)
        st.synchronize()
        return acc, zl.cpu().numpy()


res = run_ranks(P, nranks, fn)
z = np.concatenate([r[1] for r in res])
print("accepted", [r[0] for r in res], "precond rel diff", np.linalg.norm(z - z1) / np.linalg.norm(z1))
dz = np.abs(z - z1)
print("worst rows", np.argsort(dz)[-10:], dz.max())
