"""CPU tests of the multi-GPU host logic: the row partition and the
exchange/combine order of the distributed SRHT (world_size 2 over gloo).

The numpy model below is what csrc/rhqr_dist.cu does per column: every rank
runs the in-tile FWHT on its own tiles and the rank-local subtree over them,
the (ell)-vectors are all-gathered, and the top log2(P) tree levels are
combined in rank order (lower rank = left operand)."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sketchqr_oracle as O
from paper_2405_10923_b200.dist import local_rows, omega_span


def test_partition_covers_rows_once():
    for N, m, P in ((1 << 16, 32, 2), (1 << 16, 32, 8), (50_000, 100, 4), (1 << 20, 128, 8)):
        n_pad = 1 << (N - m - 1).bit_length()
        rows = [local_rows(N, m, n_pad, P, p) for p in range(P)]
        allr = np.concatenate(rows)
        assert np.array_equal(np.sort(allr), np.arange(N))
        assert np.array_equal(rows[0][:m], np.arange(m))
        span = omega_span(n_pad, P)
        for p in range(1, P):
            if len(rows[p]):
                assert rows[p][0] == m + p * span  # whole tiles, aligned


def test_partition_rejects_tiny_problems():
    with pytest.raises(ValueError):
        omega_span(1 << 12, 2)  # fp64 tile is 4096 coordinates
    with pytest.raises(ValueError):
        omega_span(1 << 20, 3)


def _local_partials(op, x, TB, p, P):
    """rank p's subtree values for every sampled output (no normalisation)."""
    span = op.n_pad // P
    v = np.zeros(op.n_pad)
    v[: op.n] = x * op.scale
    v[: op.n] *= op.signs[: op.n]
    mine = v[p * span:(p + 1) * span].reshape(span // TB, TB).copy()
    h = 1
    while h < TB:
        t = mine.reshape(mine.shape[0], TB // (2 * h), 2, h)
        a, b = t[:, :, 0].copy(), t[:, :, 1].copy()
        t[:, :, 0] = a + b
        t[:, :, 1] = a - b
        h <<= 1
    r_lo, r_hi = op.indices % TB, op.indices // TB
    leaves = mine[:, r_lo]
    lvl = 0
    while leaves.shape[0] > 1:
        a, b = leaves[0::2], leaves[1::2]
        leaves = np.where(((r_hi >> lvl) & 1).astype(bool)[None, :], a - b, a + b)
        lvl += 1
    return leaves[0], lvl


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        op = O.SRHT(256, (1 << 15) - 64, 9)
        x = np.random.default_rng(3).standard_normal(op.n)
        TB = 4096
        part, lvl = _local_partials(op, x, TB, rank, world)
        out = [torch.zeros(op.ell, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(out, torch.from_numpy(part))
        vals = [o.numpy() for o in out]
        r_hi = op.indices // TB
        w = 1
        while w < world:
            neg = ((r_hi >> lvl) & 1).astype(bool)
            for s in range(0, world, 2 * w):
                vals[s] = np.where(neg, vals[s] - vals[s + w], vals[s] + vals[s + w])
            w <<= 1
            lvl += 1
        y = vals[0] * (op.n_pad ** -0.5)
        q.put((rank, bool(np.array_equal(y, op.apply(x)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_distributed_srht_exchange_is_bitwise(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def test_four_rank_model_bitwise():
    """Same model, 4 ranks emulated in-process (exchange = list)."""
    op = O.SRHT(128, (1 << 16) - 32, 4)
    x = np.random.default_rng(1).standard_normal(op.n)
    TB, P = 4096, 4
    parts = [_local_partials(op, x, TB, p, P) for p in range(P)]
    vals = [p[0] for p in parts]
    lvl = parts[0][1]
    r_hi = op.indices // TB
    w = 1
    while w < P:
        neg = ((r_hi >> lvl) & 1).astype(bool)
        for s in range(0, P, 2 * w):
            vals[s] = np.where(neg, vals[s] - vals[s + w], vals[s] + vals[s + w])
        w <<= 1
        lvl += 1
    assert np.array_equal(vals[0] * (op.n_pad ** -0.5), op.apply(x))


# ---------------------------------------------------------------- row-partitioned Arnoldi (host logic)
def _cd_matrix(k):
    import scipy.sparse
    from paper_2405_10923_b200.workloads import convection_diffusion_csr
    ip, ix, dv = convection_diffusion_csr(k)
    return scipy.sparse.csr_matrix((dv, ix, ip), shape=(k * k, k * k))


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_krylov_partition_and_remapped_spmv(P):
    from paper_2405_10923_b200.dist import gather_layout, krylov_partition, local_operator_host
    import scipy.sparse
    k, m = 192, 20
    A = _cd_matrix(k)
    n = k * k
    n_pad = 1 << (n - m - 2).bit_length()
    row0s, rows, seg = krylov_partition(n, m, n_pad, P)
    assert row0s[0] == 0 and sum(rows) == n
    for p in range(1, P):
        if rows[p]:
            assert row0s[p] == row0s[p - 1] + rows[p - 1]  # contiguous ranges, in rank order
    x = np.random.default_rng(P).standard_normal(n)
    xg = gather_layout(x, m, n_pad, P)
    y = A @ x
    for p in range(P):
        ip, ix, dv, r0, nr, sg = local_operator_host(A, m, n_pad, P, p)
        B = scipy.sparse.csr_matrix((dv, ix, ip), shape=(nr, P * sg))
        assert np.array_equal(B @ xg, y[r0:r0 + nr])  # same CSR row order -> bitwise


def _gmres_worker(rank, world, port, out):
    """world_size-2 gloo model of the per-step exchange of the row-partitioned
    Arnoldi: all-gather of the local q rows into the [rank][seg] layout, local
    CSR rows times the gathered vector."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2405_10923_b200.dist import krylov_partition, local_operator_host
    import scipy.sparse
    k, m = 128, 12
    A = _cd_matrix(k)
    n = k * k
    n_pad = 1 << (n - m - 2).bit_length()
    row0s, rows, seg = krylov_partition(n, m, n_pad, world)
    x = np.random.default_rng(0).standard_normal(n)
    mine = np.zeros(seg)
    mine[:rows[rank]] = x[row0s[rank]:row0s[rank] + rows[rank]]
    parts = [torch.zeros(seg, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(mine))
    xg = torch.cat(parts).numpy()
    ip, ix, dv, r0, nr, sg = local_operator_host(A, m, n_pad, world, rank)
    yl = scipy.sparse.csr_matrix((dv, ix, ip), shape=(nr, world * sg)) @ xg
    out[rank] = bool(np.array_equal(yl, (A @ x)[r0:r0 + nr]))
    dist.destroy_process_group()


def test_gmres_exchange_gloo_world2():
    mgr = mp.Manager()
    out = mgr.dict()
    port = 29600 + os.getpid() % 300
    mp.spawn(_gmres_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] and out[1]


def _halo_worker(rank, world, port, out):
    """world_size-2 gloo model of the halo exchange: every rank
    publishes its halo ranges once (all_gather_object, as the facade does),
    then per step sends only the ranges its peers reference and receives
    only its own (point-to-point, as the NCCL group in dist_halo_exchange);
    the local CSR rows times that partially filled gathered vector equal the
    global SpMV rows bitwise, and the exchanged volume is one grid row per
    neighbour, not the whole vector."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2405_10923_b200.dist import halo_ranges, krylov_partition, local_operator_host
    import scipy.sparse
    k, m = 128, 12
    A = _cd_matrix(k)
    n = k * k
    n_pad = 1 << (n - m - 2).bit_length()
    row0s, rows, seg = krylov_partition(n, m, n_pad, world)
    ip, ix, dv, r0, nr, sg = local_operator_host(A, m, n_pad, world, rank)
    mine = halo_ranges(ix, seg, world, rank)
    table = [None] * world
    dist.all_gather_object(table, mine.tolist())
    table = np.asarray(table, dtype=np.int64)
    x = np.random.default_rng(0).standard_normal(n)
    q = x[row0s[rank]:row0s[rank] + rows[rank]].copy()
    G = np.zeros(world * seg)
    G[rank * seg:rank * seg + rows[rank]] = q
    reqs, moved = [], 0
    for p in range(world):
        if p == rank:
            continue
        slo, shi = table[p, rank]
        if shi > slo:
            reqs.append(dist.isend(torch.from_numpy(q[slo:shi].copy()), p))
        rlo, rhi = table[rank, p]
        if rhi > rlo:
            buf = torch.zeros(rhi - rlo, dtype=torch.float64)
            dist.recv(buf, p)
            G[p * seg + rlo:p * seg + rhi] = buf.numpy()
            moved += rhi - rlo
    for r in reqs:
        r.wait()
    yl = scipy.sparse.csr_matrix((dv, ix, ip), shape=(nr, world * sg)) @ G
    out[rank] = (bool(np.array_equal(yl, (A @ x)[r0:r0 + nr])), int(moved))
    dist.destroy_process_group()


def test_halo_exchange_gloo_world2():
    mgr = mp.Manager()
    out = mgr.dict()
    port = 29300 + os.getpid() % 300
    mp.spawn(_halo_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0][0] and out[1][0]
    assert out[0][1] <= 128 and out[1][1] <= 128  # one grid row (k = 128) per neighbour


def test_halo_ranges_stencil():
    from paper_2405_10923_b200.dist import halo_ranges, krylov_partition, local_operator_host
    k, m, world = 96, 10, 4
    A = _cd_matrix(k)
    n = k * k
    n_pad = 1 << (n - m - 2).bit_length()
    _, rows, seg = krylov_partition(n, m, n_pad, world)
    for r in range(world):
        ip, ix, dv, r0, nr, sg = local_operator_host(A, m, n_pad, world, r)
        h = halo_ranges(ix, seg, world, r)
        for p in range(world):
            size = h[p, 1] - h[p, 0]
            if abs(p - r) == 1 and nr and rows[p]:
                assert 0 < size <= k  # one grid row with each (non-empty) neighbour
            else:
                assert size == 0
