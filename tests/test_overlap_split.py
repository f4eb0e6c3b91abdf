"""Host logic of the multi-rank overlap (CPU): ``march.split_columns_by_sends``
cuts march columns along z into the planes whose cells another rank needs
(marched first, then exchanged on a side stream) and the rest (marched while
the messages fly).  The pieces must partition every column, and every source
cell of every send tag must lie in a boundary piece -- also in the strong-
scaled C2 layout at 8 ranks, where every box touches another rank."""

from types import SimpleNamespace

import numpy as np
import pytest

from paper_1604_03570_b200 import _native
from paper_1604_03570_b200.box import Box
from paper_1604_03570_b200.boxarray import BoxArray, DistributionMapping, Geometry
from paper_1604_03570_b200.fillplan import build_fill_plan_units
from paper_1604_03570_b200.halo import exchange_lists
from paper_1604_03570_b200.march import _even_chunks, split_columns_by_sends


def fake_rank(n, mgs, ranks, me, ng=1, rows=16):
    dom = Box((0, 0, 0), (n - 1,) * 3)
    ba = BoxArray.chop(dom, mgs)
    geom = Geometry(dom, (True, True, True), (1.0 / n,) * 3)
    dm = DistributionMapping(ba, ranks)
    owners = [dm[g] for g in range(len(ba))]
    local = [u for u in range(len(ba)) if owners[u] == me]
    plan = build_fill_plan_units(list(ba), geom, ng, grids=list(ba))
    _, sends, _ = exchange_lists(owners, plan.tags, me)
    send_src = {}
    for ids in sends.values():
        for t in ids:
            send_src.setdefault(plan.tags[t][2], []).append(plan.tags[t][3])
    mf = SimpleNamespace(layout=SimpleNamespace(nghost=ng), local_units=local,
                         units=[SimpleNamespace(valid=b) for b in ba])
    cols = []
    for s, u in enumerate(local):
        nx, ny, nz = ba[u].extents
        for y0, sz in _even_chunks(ny, rows):
            cols.append((s, 16, ng + y0, ng, nx, sz, nz, 0))
    arr = np.zeros(len(cols), dtype=_native.BLOCK_DTYPE)
    for k, name in enumerate(_native.BLOCK_DTYPE.names):
        arr[name] = np.array(cols)[:, k]
    return mf, arr, send_src, ba


def planes(mf, pieces):
    """{(slot, y0, global z)} covered by column pieces."""
    out = []
    for c in pieces:
        v = mf.units[mf.local_units[int(c["slot"])]].valid
        for k in range(int(c["nz"])):
            out.append((int(c["slot"]), int(c["y0"]), v.lo[2] + int(c["z0"]) - mf.layout.nghost + k))
    return out


@pytest.mark.parametrize("n,mgs,ranks,me", [(256, 64, 8, 3), (256, 64, 2, 1), (64, 16, 3, 0), (128, 32, 4, 2)])
def test_split_partitions_columns_and_covers_sends(n, mgs, ranks, me):
    mf, cols, send_src, ba = fake_rank(n, mgs, ranks, me)
    bnd, inner = split_columns_by_sends(mf, cols, send_src)
    pb, pi = planes(mf, bnd), planes(mf, inner)
    assert len(set(pb)) == len(pb) and len(set(pi)) == len(pi) and not set(pb) & set(pi)
    assert sorted(pb + pi) == sorted(planes(mf, cols))
    # every source cell of a send tag sits in a boundary piece (its column's rows, its plane)
    L = mf.layout
    bset = set(pb)
    for u, boxes in send_src.items():
        s = mf.local_units.index(u)
        v = ba[u]
        for b in boxes:
            for c in cols[cols["slot"] == s]:
                ylo = v.lo[1] + int(c["y0"]) - L.nghost
                if b.hi[1] < ylo or b.lo[1] > ylo + int(c["ny"]) - 1:
                    continue
                for z in range(b.lo[2], b.hi[2] + 1):
                    assert (s, int(c["y0"]), z) in bset
    # interior work remains for the overlap (C2 strong at 8 ranks: all 8 boxes touch other ranks)
    assert len(pi) > len(pb) // 2


def test_c2_eight_ranks_boundary_share():
    """C2 strong-scaled to 8 ranks: a rank holds 8 boxes (two y-rows of one
    z-layer); the boundary launch covers the z-face planes of every column plus
    the columns along the remote y faces -- about a quarter of the planes."""
    mf, cols, send_src, _ = fake_rank(256, 64, 8, 5)
    bnd, inner = split_columns_by_sends(mf, cols, send_src)
    nb, ni = int(bnd["nz"].sum()), int(inner["nz"].sum())
    assert nb + ni == 8 * 4 * 64
    assert 0.15 < nb / (nb + ni) < 0.35
