"""The process-level host transport of psp_comm_host_create (include/pspgmres.h) as the library
calls it, from a world_size-2 torch.distributed (gloo) job on CPU: the ctypes callbacks of
pspgmres.TorchDistTransport are invoked through their C function pointers on host buffers, with the
library's conventions (in-place all-reduce sum / max / min; send_lo -> rank-1 whose send_hi lands in
recv_lo; NULL pointers and zero counts at the ends; allgather in rank order).  No GPU needed; the
GPU test tests/test_gpu_multiproc.py drives psp_step through the same transport."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1308_5626_b200 import pspgmres as P


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = P.TorchDistTransport()
    st = t.struct
    res = {}
    for op in (0, 1, 2):
        buf = np.array([1.0 + rank, -2.0 * rank, 3.5], dtype=np.float64)
        assert st.allreduce(None, _dp(buf), 3, op) == 0
        res[f"allreduce{op}"] = buf.tolist()
    # halos (n_lo = n_hi = 2, the same count both ways): rank r sends [10r, 10r+1] down and
    # [10r+5, 10r+6] up
    send_lo = np.array([10.0 * rank, 10.0 * rank + 1])
    send_hi = np.array([10.0 * rank + 5, 10.0 * rank + 6])
    recv_lo = np.full(2, -1.0)        # rank-1's send_hi
    recv_hi = np.full(2, -1.0)        # rank+1's send_lo
    lo, hi = rank > 0, rank < world - 1
    null = C.POINTER(C.c_double)()
    assert st.sendrecv(None, _dp(send_lo) if lo else null, _dp(recv_lo) if lo else null, 2 if lo else 0,
                       _dp(send_hi) if hi else null, _dp(recv_hi) if hi else null, 2 if hi else 0) == 0
    res["recv_lo"], res["recv_hi"] = recv_lo.tolist(), recv_hi.tolist()
    send = np.array([rank + 0.25, rank + 0.5])
    recv = np.zeros(2 * world)
    assert st.allgather(None, _dp(send), _dp(recv), 2) == 0
    res["allgather"] = recv.tolist()
    out_q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_torch_dist_transport_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        g = got[r]
        assert g["allreduce0"] == [sum(1.0 + q for q in range(world)), sum(-2.0 * q for q in range(world)), 3.5 * world]
        assert g["allreduce1"] == [float(world), 0.0, 3.5]
        assert g["allreduce2"] == [1.0, -2.0 * (world - 1), 3.5]
        assert g["allgather"] == [v for q in range(world) for v in (q + 0.25, q + 0.5)]
        if r > 0:
            assert g["recv_lo"] == [10.0 * (r - 1) + 5, 10.0 * (r - 1) + 6]
        else:
            assert g["recv_lo"] == [-1.0, -1.0]
        if r < world - 1:
            assert g["recv_hi"] == [10.0 * (r + 1), 10.0 * (r + 1) + 1]
        else:
            assert g["recv_hi"] == [-1.0, -1.0]
