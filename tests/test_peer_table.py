"""Host logic of the peer (NVLink) halo path (CPU): ``peer.peer_face_table``
encodes every y/z face whose neighbour lives on another rank as
TM_NBR_PEER(p, s) -- slot s of the p-th peer rank -- and refuses layouts whose
x faces cross ranks.  Checked against a brute-force periodic-image lookup on
the strong-scaled C2 layout (8 ranks: every box has remote y and z faces) and
on a weak-scaled slab layout (remote z faces only)."""

from types import SimpleNamespace

import numpy as np
import pytest

from paper_1604_03570_b200 import _native
from paper_1604_03570_b200.box import Box
from paper_1604_03570_b200.boxarray import BoxArray, DistributionMapping, Geometry
from paper_1604_03570_b200.peer import peer_face_table


def fake_rank(n, mgs, ranks, me, ng=1):
    dom = Box((0, 0, 0), tuple(x - 1 for x in n))
    ba = BoxArray.chop(dom, mgs)
    geom = Geometry(dom, (True, True, True), tuple(1.0 / x for x in n))
    dm = DistributionMapping(ba, ranks)
    owners = tuple(dm[g] for g in range(len(ba)))
    local = [u for u in range(len(ba)) if owners[u] == me]
    e = ba[0].extents
    layout = SimpleNamespace(nghost=ng, xoff=16, ny=e[1] + 2 * ng, nz=e[2] + 2 * ng)
    mf = SimpleNamespace(layout=layout, nghost=ng, local_units=local, unit_owner=owners,
                         units=[SimpleNamespace(valid=b) for b in ba], slot_of={u: s for s, u in enumerate(local)})
    return mf, geom, ba


def decode(v):
    q = -3 - int(v)
    return q >> 24, q & 0xFFFFFF


@pytest.mark.parametrize("n,mgs,ranks", [((256,) * 3, 64, 8), ((128, 128, 256), 32, 4), ((128,) * 3, 32, 2)])
def test_peer_faces_match_periodic_images(n, mgs, ranks):
    for me in range(ranks):
        mf, geom, ba = fake_rank(n, mgs, ranks, me)
        table, peers = peer_face_table(mf, geom)
        assert me not in peers and len(peers) <= _native.MAX_PEERS
        slots = {r: [u for u in range(len(ba)) if mf.unit_owner[u] == r] for r in range(ranks)}
        for s, u in enumerate(mf.local_units):
            v = ba[u]
            for k in range(6):
                d, side = divmod(k, 2)
                lo = list(v.lo)
                lo[d] = (lo[d] + (-v.extents[d] if side == 0 else v.extents[d])) % n[d]
                nb = next(i for i, b in enumerate(ba) if tuple(b.lo) == tuple(lo))
                r = mf.unit_owner[nb]
                if r == me:
                    assert table[s, k] == mf.slot_of[nb]
                else:
                    assert k >= 2 and table[s, k] <= -3
                    p, ps = decode(table[s, k])
                    assert peers[p] == r and slots[r][ps] == nb


def test_c2_strong_eight_ranks_has_remote_y_and_z():
    mf, geom, _ = fake_rank((256,) * 3, 64, 8, 3)
    table, peers = peer_face_table(mf, geom)
    assert (table[:, 2:4] <= -3).any() and (table[:, 4:6] <= -3).all()
    assert sorted(peers) == [1, 2, 5]  # the other half of the z-layer (both y faces), the two z layers


def test_remote_x_face_is_refused():
    # 27 boxes over 2 ranks: the split falls inside an x row
    mf, geom, _ = fake_rank((48, 48, 48), 16, 2, 0)
    with pytest.raises(ValueError, match="x-face"):
        peer_face_table(mf, geom)


def test_nbr_peer_code_range():
    assert _native.nbr_peer(0, 0) == -3
    assert decode(_native.nbr_peer(7, (1 << 24) - 1)) == (7, (1 << 24) - 1)
    with pytest.raises(ValueError):
        _native.nbr_peer(8, 0)
    assert np.int32(_native.nbr_peer(7, (1 << 24) - 1)) < 0
