"""World-size-2 multi-process checks of the N > 1 host path on CPU (gloo backend, no GPU).

The data path has no collective (units are independent); what crosses ranks is
(a) the cost-balanced shard plan each rank derives on its own, which must partition Λ, (b) the
threshold rule's MAX all-reduce of the per-rank maxima (P:1179 threshold, reading R15), and
(c) the bench's max-over-ranks timing and sum of retained entries, and (d) the consumer's exchange: the
sharded FISTA's all-reduce of the gradient Θ_Lᵀr = Σ_r Θ_rᵀ r_r.  The per-rank maxima here come
from the oracle (the GPU computes them in the real run) — the exchange is what is tested.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import operator as op
        from paper_2005_09870_b200 import pcwd as P
        from synth import configs as C
        p = C.micro(16, 2, 4, 3, 2, 2, 31, retain="threshold", tau_rel=1e-4)
        spec = P.Spec(p.d, p.n, p.J, p.h, p.u, p.v, dtype="f64", retain="threshold", tau_rel=1e-4,
                      rank=rank, world=world)
        r0, r1 = P.plan_shard(spec)
        T = op.theta_dense(p)
        local = float(np.abs(T[r0:r1]).max()) if r1 > r0 else 0.0
        M = P.allreduce_max(local)
        nnz_local = int(np.count_nonzero(np.abs(T[r0:r1]) >= 1e-4 * M))
        nnz_all = P.allreduce_sum(nnz_local)
        t_all = P.allreduce_max(float(rank + 1))          # bench: max over ranks of the step time
        out[rank] = (r0, r1, M, nnz_all, t_all, float(np.abs(T).max()),
                     int(np.count_nonzero(np.abs(T) >= 1e-4 * np.abs(T).max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_world2_shards_and_threshold_exchange(world):
    from paper_2005_09870_b200 import _build
    _build.build()
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    res = [out[r] for r in range(world)]
    assert res[0][0] == 0 and res[-1][1] == 256
    for a, b in zip(res, res[1:]):
        assert a[1] == b[0]
    for r in res:
        assert r[2] == r[5]               # all-reduced max = global max of Θ
        assert r[3] == r[6]               # summed shard counts = global retained count
        assert r[4] == float(world)       # max over ranks


def _worker_shards(rank, world, port, out):
    """C-b offsets, C-c shard gather and C-d transposed-apply reduction over the shards of an oracle Θ (the GPU
    computes the shards in the real run; here the exchanges are what is tested)."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        from oracle import operator as op
        from paper_2005_09870_b200 import pcwd as P
        from synth import configs as C
        p = C.micro(16, 2, 4, 3, 2, 2, 32, retain="threshold", tau_rel=1e-3)
        T = op.theta_dense(p)
        M = float(np.abs(T).max())
        spec = P.Spec(p.d, p.n, p.J, p.h, p.u, p.v, dtype="f64", retain="threshold", tau_rel=1e-3,
                      rank=rank, world=world)
        r0, r1 = P.plan_shard(spec)
        keep = np.abs(T[r0:r1]) >= 1e-3 * M
        rp = np.concatenate([[0], np.cumsum(keep.sum(axis=1))]).astype(np.int64)
        col = np.nonzero(keep)[1].astype(np.int32)
        val = T[r0:r1][keep]
        offs = P.global_row_offsets(len(col))
        g = P.gather_csr(torch.from_numpy(rp), torch.from_numpy(col), torch.from_numpy(val), r0, p.N)
        # Θᵀ x as the sum of the shards' partials Θ_rᵀ x[r0:r1]
        x = np.random.default_rng(0).standard_normal(p.N)
        part = np.zeros(p.N)
        dense = np.zeros((r1 - r0, p.N))
        dense[keep] = val
        part += dense.T @ x[r0:r1]
        y = torch.from_numpy(part)
        dist.all_reduce(y, op=dist.ReduceOp.SUM)
        steps = P.allreduce_max_vec(np.array([rank + 1.0, 5.0 - rank]))
        out[rank] = (offs, None if g is None else tuple(t.numpy() for t in g), y.numpy(), steps, len(col), r0)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_offsets_gather_apply():
    from oracle import operator as op
    from synth import configs as C
    from paper_2005_09870_b200 import _build
    _build.build()
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_shards, args=(world, port, out), nprocs=world, join=True)
    res = [out[r] for r in range(world)]
    p = C.micro(16, 2, 4, 3, 2, 2, 32, retain="threshold", tau_rel=1e-3)
    T = op.theta_dense(p)
    keep = np.abs(T) >= 1e-3 * np.abs(T).max()
    nnz = [r[4] for r in res]
    assert res[0][0] == res[1][0] == [0, nnz[0], nnz[0] + nnz[1]]          # C-b: identical on every rank
    rp, col, val = res[0][1]                                                # C-c: the whole Θ on rank 0
    assert res[1][1] is None
    assert np.array_equal(rp, np.concatenate([[0], np.cumsum(keep.sum(axis=1))]))
    assert np.array_equal(col, np.nonzero(keep)[1]) and np.array_equal(val, T[keep])
    x = np.random.default_rng(0).standard_normal(p.N)
    dense = np.where(keep, T, 0.0)
    for r in res:                                                           # C-d: Σ_r Θ_rᵀ x_r = Θᵀ x
        assert np.allclose(r[2], dense.T @ x, rtol=1e-13, atol=1e-13)
        assert list(r[3]) == [2.0, 5.0]                                     # per-step max over ranks


class _ShardStub:
    """Stands in for a sharded handle on CPU: fista_sharded calls the reduce it is given on this rank's partial
    gradient (and Jacobi column sums), as pcwd_fista_sharded does, and returns what the reduce left."""
    def __init__(self, rank):
        self.rank = rank

    def fista_sharded(self, z0, w, iters, reduce, precond=False, tau=0.0, stream=0):
        import torch
        g = torch.full_like(z0, float(self.rank + 1))
        calls = 0
        for _ in range(iters):
            reduce(0, g)
            calls += 1
            g /= 2.0                          # keep values exact: 3 → 1.5 + 1.5 …
        d = torch.arange(z0.numel(), dtype=torch.float64) * (self.rank + 1)
        if precond:
            reduce(1, d)
        return g, d


def _worker_fista(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        from paper_2005_09870_b200 import pcwd as P
        z0 = torch.zeros(8, dtype=torch.float64)
        g, d = P.fista_distributed(_ShardStub(rank), z0, z0, 1, precond=True)
        out[rank] = (g.numpy(), d.numpy())
    finally:
        dist.destroy_process_group()


def test_gloo_world2_fista_distributed_reduces_over_ranks():
    """fista_distributed's exchange: the gradient (which 0) and the Jacobi column sums (which 1) are summed over
    the ranks in place (gloo, world 2) — the host side of the sharded FISTA."""
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_fista, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        g, d = out[r]
        assert np.array_equal(g, np.full(8, 1.5)) and np.array_equal(d, np.arange(8) * 3.0)
