"""CPU check of the GPU SRHT decomposition: in-tile FWHT over
TB = 2^t coordinates with stages h = 1..TB/2, gather of the ell sampled rows
r_lo = idx mod TB from every tile, then a binary tree over tiles in level
order whose level-t sign is bit t of r_hi = idx div TB (lower tile = left
operand), then one multiply by fl(n_pad^-1/2).  This is what
csrc/srht.cuh does; here it is replayed in numpy and compared bitwise with
the oracle (which restates sketching.py:21-43, 149-155)."""

import numpy as np
import pytest

from oracle import sketchqr_oracle as O


def tiled_srht(op, x, TB, dt=np.float64, ranks=1):
    dt = np.dtype(dt)
    n_pad = op.n_pad
    TB = min(TB, n_pad)
    v = np.zeros(n_pad, dtype=dt)
    v[: op.n] = x.astype(dt) * dt.type(op.scale)
    v[: op.n] *= op.signs[: op.n].astype(dt)
    tiles = v.reshape(n_pad // TB, TB).copy()
    h = 1
    while h < TB:  # in-tile stages in order
        t = tiles.reshape(tiles.shape[0], TB // (2 * h), 2, h)
        a, b = t[:, :, 0].copy(), t[:, :, 1].copy()
        t[:, :, 0] = a + b
        t[:, :, 1] = a - b
        h <<= 1
    r_lo = op.indices % TB
    r_hi = op.indices // TB
    leaves = tiles[:, r_lo]  # (n_tiles, ell)
    level = 0
    while leaves.shape[0] > 1:
        a, b = leaves[0::2], leaves[1::2]
        neg = ((r_hi >> level) & 1).astype(bool)
        leaves = np.where(neg[None, :], a - b, a + b)
        level += 1
    return (leaves[0] * dt.type(n_pad ** -0.5)).astype(np.float64)


@pytest.mark.parametrize("ell,n,seed", [(8, 12, 3), (64, 1000, 5), (128, 16352, 7),
                                         (256, 65536 - 128, 11), (400, 8191, 13)])
@pytest.mark.parametrize("TB", [2, 64, 1024, 4096])
def test_tile_tree_bitwise(ell, n, seed, TB):
    op = O.SRHT(ell, n, seed)
    x = np.random.default_rng(seed).standard_normal(n)
    assert np.array_equal(tiled_srht(op, x, TB), op.apply(x))


@pytest.mark.parametrize("tag", ["single", "half", "bf16"])
def test_tile_tree_low_precision_bitwise(tag):
    op = O.SRHT(64, 4080, 31)
    x = O.round_to(np.random.default_rng(1).standard_normal(4080), tag)
    dt = O.TAG_DTYPE[tag]
    assert np.array_equal(tiled_srht(op, x, 256, dt), op.apply(x, dt))
