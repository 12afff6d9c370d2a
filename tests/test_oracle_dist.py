"""World-size-2 (and 4) gloo tests of the row-partitioned decomposition (oracle.dist, north_star
row partition; TSQR reading R-A26). Each rank holds a contiguous row block; the gathered Q and the
replicated R / x must equal the single-process oracle (exact arithmetic -> rounding level)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as W


class TorchComm:
    def __init__(self):
        self.rank, self.size = dist.get_rank(), dist.get_world_size()

    def allreduce_sum(self, x):
        t = torch.from_numpy(np.array(x, dtype=np.float64, copy=True))
        dist.all_reduce(t)
        return t.numpy()

    def allgather(self, x):
        t = torch.from_numpy(np.array(x, dtype=np.float64, copy=True))
        out = [torch.empty_like(t) for _ in range(self.size)]
        dist.all_gather(out, t)
        return [o.numpy() for o in out]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, m, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.dist import dist_pcgls, dist_rgs
    a = W.gaussian(m, n, seed=77).astype(np.float64)
    b, _ = W.consistent_rhs(a.astype(np.float32), seed=78)
    rows = np.array_split(np.arange(m), world)[rank]
    comm = TorchComm()
    q_loc, r = dist_rgs(a[rows], comm, br=64)
    x, info = dist_pcgls(a[rows], b[rows], r, comm, tol=1e-12, maxit=50)
    q.put((rank, rows[0], q_loc, r, x, info.iterations))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_dist_rgs_gloo_matches_single_process(world):
    from oracle.cgls import pcgls
    from oracle.qr import rgs
    m, n = 512, 96
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    a = W.gaussian(m, n, seed=77).astype(np.float64)
    b, _ = W.consistent_rhs(a.astype(np.float32), seed=78)
    q0, r0 = rgs(a, panel="caqr", br=64)
    x0, _ = pcgls(a, b, r0, tol=1e-12, maxit=50)
    qd = np.vstack([t[2] for t in res])
    for t in res:
        assert np.array_equal(t[3], res[0][3])          # R replicated bitwise on all ranks
        assert np.array_equal(t[4], res[0][4])          # x replicated bitwise
    assert np.linalg.norm(res[0][3] - r0) / np.linalg.norm(r0) < 1e-13
    assert np.max(np.abs(qd - q0)) < 1e-12
    assert np.linalg.norm(res[0][4] - x0) / np.linalg.norm(x0) < 1e-12


def test_dist_selfcomm_equals_rgs():
    from oracle.dist import SelfComm, dist_rgs
    from oracle.qr import rgs
    a = W.gaussian(300, 70, seed=3).astype(np.float64)
    q, r = dist_rgs(a, SelfComm(), br=64)
    q0, r0 = rgs(a, panel="caqr", br=64)
    assert np.array_equal(q, q0) and np.array_equal(r, r0)
