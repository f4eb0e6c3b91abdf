"""A few steps of rank 0's peer-halo march in the emulated C2 strong-scaled layout at 8 ranks
(8 boxes per rank, remote y and z faces read from the other ranks' storage) -- the launches
profiled in profiles/r02/ncu_peer_march_c2x8.txt.  PYTHONPATH=. python tools/peer_ncu.py"""

import torch


def main():
    import paper_1604_03570_b200 as tm
    from paper_1604_03570_b200.boxarray import DistributionMapping
    from paper_1604_03570_b200.peer import PeerFused

    w = tm.CONFIGS["C2"]
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    dm = DistributionMapping(ba, 8)
    glob = torch.rand((1,) + tuple(w.domain.extents[::-1]), dtype=torch.float64, device="cuda")
    pairs = []
    for r in range(8):
        a = tm.MultiFab(ba, 1, 1, dm=dm, rank=r)
        a.from_global(glob)
        pairs.append((a, a.clone_empty()))
    fields = {r: (p[0].ptr, p[1].ptr) for r, p in enumerate(pairs)}
    a, b = pairs[0]
    pf = PeerFused(a, b, geom, fields)
    pf.prime(a)
    params = tm.HeatParams.stable(1.0, geom.dx)
    for k in range(4):
        pf.step(b, a, params) if k % 2 == 0 else pf.step(a, b, params, reverse=True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
