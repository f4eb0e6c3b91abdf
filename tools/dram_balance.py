"""Launches for the DRAM channel-balance check (run under ncu, see profiles/r02/dram_balance.txt):
two fused C2 steps (the bench kernel) and a plain 268 MB device copy of the same size."""

import torch


def main():
    import paper_1604_03570_b200 as tm
    from paper_1604_03570_b200.runner import HeatRunner

    w = tm.CONFIGS["C2"]
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    mf = tm.MultiFab(tm.BoxArray.chop(w.domain, w.max_grid_size), 1, 1)
    mf.data.copy_(torch.rand_like(mf.data))
    r = HeatRunner(mf, geom, tm.HeatParams.stable(1.0, geom.dx), use_graph=False)
    r.advance(3)
    src = torch.rand(1 << 25, dtype=torch.float64, device="cuda")  # 268 MB
    dst = torch.empty_like(src)
    for _ in range(2):
        dst.copy_(src)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
