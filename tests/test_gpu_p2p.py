"""In-kernel peer-memory exchange (sqb_p2p_*) of the row-partitioned sweep:
each rank's per-column partials are stored straight into its peers' mailboxes
and published with release flags the step kernel acquires (no collective
launch).  With virtual ranks on one B200 the factors are bitwise the
single-GPU ones, as with the copy / NCCL exchange; world 1 runs the real IPC
set-up path."""

import os

import numpy as np
import pytest

from paper_2405_10923_b200 import workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available()
    import paper_2405_10923_b200 as P
    return P


@pytest.mark.parametrize("nranks", [1, 2, 4, 8])
def test_p2p_virtual_rhqr_left_bitwise(P, nranks):
    from paper_2405_10923_b200 import dist
    N, m = (1 << 16) + 77, 24
    W = np.random.default_rng(nranks + 40).standard_normal((N, m))
    om = P.SRHTSketch(96, N - m, 17)
    F1 = P.rhqr_left(W, om)
    Fv = dist.rhqr_left_virtual(W, om, nranks, exchange="p2p")
    for k in ("R", "S", "T", "U", "sigmas", "rhos", "betas"):
        assert np.array_equal(getattr(Fv, k), getattr(F1, k)), k
    # the mailboxes are released: the copy exchange still works afterwards
    Fc = dist.rhqr_left_virtual(W, om, nranks)
    assert np.array_equal(Fc.R, F1.R)


@pytest.mark.parametrize("nranks,m", [(2, 48), (8, 64)])
def test_p2p_virtual_rec_rhqr_bitwise(P, nranks, m):
    from paper_2405_10923_b200 import dist
    N = (1 << 16) + 77
    W = workloads.gen_cmatrix(N, m)
    om = P.SRHTSketch(4 * m, N - m, 19)
    F1 = P.rec_rhqr(W, om)
    Fv = dist.rec_rhqr_virtual(W, om, nranks, exchange="p2p")
    for k in ("R", "S", "T", "sigmas", "rhos", "betas"):
        assert np.array_equal(getattr(Fv, k), getattr(F1, k)), k


def test_p2p_world1_ipc_path(P, monkeypatch):
    """sqb_p2p_mailbox / sqb_p2p_open through torch.distributed (world 1),
    then the row-partitioned factorizations over the mailboxes; repeated
    calls reuse the monotone exchange sequence numbers.  The bitwise twin of
    the partitioned sweep is the single-GPU launch chain (SQB_PERSIST=0)."""
    monkeypatch.setenv("SQB_PERSIST", "0")
    import torch.distributed as dist
    from paper_2405_10923_b200 import dist as D
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(29900 + os.getpid() % 90))
    created = False
    if not dist.is_initialized():
        dist.init_process_group("gloo", rank=0, world_size=1)
        created = True
    try:
        # small: fused exchange (the step kernel folds the rank-local subtree,
        # stores it into the mailboxes and waits); large: the same with the
        # cross-pass overlap of the column passes (per-block flags)
        for N, m, ell in (((1 << 14) + 5, 16, 64), ((1 << 20) + 4096 + 40, 40, 96)):
            W = np.random.default_rng(0).standard_normal((N, m))
            om = P.SRHTSketch(ell, N - m, 3)
            D.init_p2p(m, om.ell)
            F1 = P.rhqr_left(W, om)
            for _ in range(3):
                Fd = D.rhqr_left_distributed(W, om, m)
                for k in ("R", "S", "T", "U"):
                    assert np.array_equal(getattr(Fd, k), getattr(F1, k)), (k, N)
            D.close_p2p()
    finally:
        if created:
            dist.destroy_process_group()


def test_p2p_silent_peer_times_out_instead_of_hanging(P, monkeypatch):
    """Failure detection of the in-kernel exchange: rank 0 of a 2-rank
    partition whose peer never publishes its flag (an all-zero IPC handle
    stands for it) must fail with an error naming rank 1 after the wait
    limit, and the context must be usable again afterwards."""
    monkeypatch.setenv("SQB_PERSIST", "0")
    import ctypes as C
    import torch.distributed as dist
    from paper_2405_10923_b200 import _lib, dist as D
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(29900 + os.getpid() % 90))
    created = False
    if not dist.is_initialized():
        dist.init_process_group("gloo", rank=0, world_size=1)
        created = True
    N, m, ell = (1 << 14) + 5, 16, 64
    W = np.random.default_rng(0).standard_normal((N, m))
    om = P.SRHTSketch(ell, N - m, 3)
    ctx = _lib.context()
    try:
        h = C.create_string_buffer(64)
        ctx.check(_lib.lib().sqb_p2p_mailbox(ctx.h, 2, D.p2p_slot_count(m, ell), h), "sqb_p2p_mailbox")
        table = C.create_string_buffer(h.raw + bytes(64), 128)
        ctx.check(_lib.lib().sqb_p2p_open(ctx.h, 0, table), "sqb_p2p_open")
        D.set_p2p_timeout(50)
        rows0 = D.local_rows(N, m, om.n_pad, 2, 0, "double")
        with pytest.raises(_lib.SketchQRError, match="timed out waiting for rank 1"):
            D.rhqr_left_distributed(W[rows0], om, m)
    finally:
        D.close_p2p()
        if created:
            dist.destroy_process_group()
    F = P.rhqr_left(W, om)  # the status word was consumed: the next call runs
    assert np.isfinite(F.R).all()


def test_row_partition_fuzz_is_bitwise_the_single_gpu_run(P, monkeypatch, capsys):
    """A short seeded run of scripts/fuzz_dist.py: random shapes (ragged last
    ranks, ranks that own only padding, n_pad / P down to one tile), formats,
    scalings and exchanges on 1-8 virtual ranks; every factor bitwise the
    single-GPU launch chain, every failure the same exception."""
    import importlib.util
    import sys
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts", "fuzz_dist.py")
    spec = importlib.util.spec_from_file_location("fuzz_dist", path)
    mod = importlib.util.module_from_spec(spec)
    monkeypatch.setenv("SQB_PERSIST", "0")
    spec.loader.exec_module(mod)
    rc = mod.main(["--seconds", "12", "--seed", "7"])
    out = capsys.readouterr().out
    assert rc == 0, out
    assert "0 disagreements" in out
    sys.modules.pop("fuzz_dist", None)
