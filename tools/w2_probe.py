"""One Kernel W2 launch in each halo mode on the C2-shaped wide4 problem
(256^3, 64^3 boxes, nghost 4), for ncu: python tools/w2_probe.py [reps]"""

import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1604_03570_b200 as tm  # noqa: E402
from paper_1604_03570_b200.wide4 import _launch  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    w = dataclasses.replace(tm.CONFIGS["C2"].scaled(256, 64, 2), nghost=4)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    a = tm.MultiFab(tm.BoxArray.chop(w.domain, w.max_grid_size), 1, 4)
    a.from_global(tm.make_init(w))
    b = a.clone_empty()
    dt = tm.wide4_stable_dt(1.0, geom.dx)
    co = tm.derive_coeffs8()
    tm.fill_boundary(a, geom)
    r = tm.Wide4Runner(a, geom, 1.0, dt, co, use_graph=False)
    for _ in range(reps):
        _launch(b, a, geom, 1.0, dt, co)   # W2 GHOST
        r._step(r.a, r.b)                  # W2 NBR
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
