"""Host logic of the multi-rank path (no GPU): the slab decomposition of psp_partition, checked
directly and from a world_size-2 torch.distributed (gloo) job, the way bench.py / a user's
torchrun job would call it -- each rank computes its own slab and the slabs must tile the grid."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1308_5626_b200 import pspgmres as P


@pytest.mark.parametrize("n_axes", [(1024,), (64, 48), (16, 12, 10), (512, 512, 512), (7, 5, 3)])
@pytest.mark.parametrize("nranks", [1, 2, 3, 8])
def test_partition_tiles_grid(n_axes, nranks):
    ax = len(n_axes) - 1
    if n_axes[ax] < nranks:
        pytest.skip("fewer planes than ranks")
    plane = 1
    for a in range(ax):
        plane *= n_axes[a]
    total = 1
    for v in n_axes:
        total *= v
    nxt = 0
    lens = []
    for r in range(nranks):
        row0, nrows, s0, sl = P.psp_partition(n_axes, nranks, r)
        assert row0 == nxt and nrows == sl * plane and row0 == s0 * plane
        nxt += nrows
        lens.append(sl)
    assert nxt == total
    assert max(lens) - min(lens) <= 1                      # balanced to one plane


def test_partition_rejects_too_many_ranks():
    with pytest.raises(P.PspError):
        P.psp_partition((8, 8, 3), 4, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_axes, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    row0, nrows, _, _ = P.psp_partition(n_axes, world, rank)
    mine = torch.tensor([row0, nrows], dtype=torch.int64)
    allr = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allr, mine)
    # the global ||x||^2 of a multi-rank reduction = the all-reduce of the slab partial sums
    x = torch.arange(row0, row0 + nrows, dtype=torch.float64)
    part = torch.tensor([float((x * x).sum())], dtype=torch.float64)
    dist.all_reduce(part)
    if rank == 0:
        out_q.put(([tuple(t.tolist()) for t in allr], float(part.item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_axes", [(40, 36, 33), (1024,)])
def test_partition_gloo_world2(n_axes):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_axes, q)) for r in range(2)]
    for p in procs:
        p.start()
    slabs, sq = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    total = 1
    for v in n_axes:
        total *= v
    assert slabs[0][0] == 0 and slabs[0][0] + slabs[0][1] == slabs[1][0]
    assert slabs[1][0] + slabs[1][1] == total
    ref = float(sum(float(i) * float(i) for i in range(total)))
    assert sq == pytest.approx(ref, rel=1e-15)
