"""Copy roofline at stencil-sized working sets: torch copy_ of N fp64 (read N*8 + write N*8 bytes)."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from tools.sweep_shapes import graph_time  # noqa: E402

for mb in (134, 268, 536, 1074, 4295):
    n = mb * 1000 * 1000 // 8
    a = torch.rand(n, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    ms = graph_time(lambda: torch.mul(a, 1.0, out=b), 10)
    print(f"copy {mb} MB: {ms * 1e3:.1f} us  {2 * n * 8 / ms / 1e6:.0f} GB/s (read+write)")
    del a, b

# strided rows like the MultiFab layout: 64 used doubles of every 96-double pitch
for pitch in (96, 80, 64):
    rows = 134 * 1000 * 1000 // 8 // 64
    a = torch.rand(rows, pitch, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    av, bv = a[:, 16:80] if pitch > 64 else a, b[:, 16:80] if pitch > 64 else b
    if pitch == 80:
        av, bv = a[:, 8:72], b[:, 8:72]
    ms = graph_time(lambda: torch.mul(av, 1.0, out=bv), 10)
    print(f"strided copy pitch={pitch}: 134 MB used in {ms * 1e3:.1f} us  {2 * rows * 64 * 8 / ms / 1e6:.0f} GB/s")
    del a, b
