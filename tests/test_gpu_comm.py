"""The communicator backends' collectives (all-reduce sum / max / min, all-gather, the slab
neighbours' send/recv) through psp_comm_selftest, on one B200: a real one-rank NCCL
communicator (the dlopen'ed NCCL bindings of comm.cu), the in-process loopback group at 2 and 3
ranks (one host thread and stream per rank) and the process-level host transport in a
world-size-2 gloo job.  NCCL refuses two ranks on one device, so its multi-rank data plane is
exercised only by a multi-GPU job (bench.py --gpus N runs the same self-test first)."""
import os
import socket
import tempfile
import threading

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "the -m gpu tests need a B200"
    from paper_1308_5626_b200 import pspgmres
    pspgmres.lib()
    return pspgmres


def test_nccl_one_rank_selftest(P):
    import torch
    uid = P.psp_comm_unique_id()
    h = P.psp_comm_init(uid, 1, 0)
    s = torch.cuda.Stream()
    assert P.psp_comm_selftest(h, s) == P.PSP_OK
    P.psp_comm_destroy(h)


def test_one_rank_without_nccl_selftest(P):
    h = P._vp()
    assert P.lib().psp_comm_init(None, 1, 0, P.C.byref(h)) == P.PSP_OK
    assert P.psp_comm_selftest(h) == P.PSP_OK
    P.psp_comm_destroy(h)


@pytest.mark.parametrize("nranks", [2, 3])
def test_loopback_selftest(P, nranks):
    import torch
    hs = P.psp_comm_loopback_create(nranks)
    out = [None] * nranks

    def run(r):
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        out[r] = P.psp_comm_selftest(hs[r], s)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    assert out == [P.PSP_OK] * nranks
    for h in hs:
        P.psp_comm_destroy(h)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _host_worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist

    from paper_1308_5626_b200 import pspgmres as P
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    tr = P.TorchDistTransport()
    comm = P.psp_comm_host_create(tr, world, rank)
    st = P.psp_comm_selftest(comm, torch.cuda.Stream())
    with open(os.path.join(outdir, f"r{rank}.txt"), "w") as f:
        f.write(str(st))
    P.psp_comm_destroy(comm)
    dist.barrier()
    dist.destroy_process_group()


def test_host_transport_selftest_two_processes(P):
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as td:
        ctx = mp.get_context("spawn")
        port = _free_port()
        procs = [ctx.Process(target=_host_worker, args=(r, 2, port, td)) for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=300)
            assert p.exitcode == 0
        for r in range(2):
            assert open(os.path.join(td, f"r{r}.txt")).read() == str(P.PSP_OK)
