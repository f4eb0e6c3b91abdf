"""Plotfile-lite I/O from the device.

Reference: ``write_plotfile`` / ``read_plotfile`` (level.py:326-359) and the
FAB dump ``FArrayBox.write`` / ``read`` (fab.py:86-97): a text ``HEADER``
plus one binary file per unit, ``unit_NNNNN.fab`` = 7 little-endian int64
(allocation box lo, hi, ncomp) followed by the raw float64 payload of the
grown box, x fastest, component slowest.  The files written here are
byte-identical to the reference's for the same MultiFab contents.

Device side: the padded slots are packed into one dense staging buffer by
copy-kernel launches (one per distinct unit shape), so only payload bytes
cross PCIe, in one device-to-host copy.  Multi-rank: every rank writes the
fab files of the units it owns; rank 0 writes the HEADER (all units).
"""

from __future__ import annotations

import os

import numpy as np

from . import _native
from .boxarray import Geometry
from .fab import FArrayBox


def pack_units(mf) -> dict:
    """Grown-box payload of every local unit, gathered on the device into one
    dense buffer and copied to the host once: ``{unit: flat float64 array}``."""
    import torch

    L = mf.layout
    groups: dict = {}
    for u in mf.local_units:
        groups.setdefault(mf.units[u].fab.abox.extents, []).append(u)
    offsets, total = {}, 0
    for ext, units in groups.items():
        n = ext[0] * ext[1] * ext[2] * mf.ncomp
        for u in units:
            offsets[u] = total
            total += n
    stage = torch.empty(max(total, 1), dtype=torch.float64, device=mf.device)
    for ext, units in groups.items():
        tags = np.zeros(len(units), dtype=_native.COPY_TAG_DTYPE)
        for t, u in enumerate(units):
            src = mf.slot_of[u] * L.slot + (L.xoff - mf.nghost)
            tags[t] = (offsets[u], src, ext[0], ext[1], ext[2], 0)
        side = (ext[0], ext[0] * ext[1], ext[0] * ext[1] * ext[2])
        _native.CopyPlan(tags, mf.ncomp).run(stage.data_ptr(), side, mf.ptr, L.side(), mf.stream())
    host = stage.cpu().numpy()
    out = {}
    for u in mf.local_units:
        e = mf.units[u].fab.abox.extents
        out[u] = host[offsets[u]:offsets[u] + e[0] * e[1] * e[2] * mf.ncomp]
    return out


def header_text(mf, geom: Geometry) -> str:
    lines = [
        f"domain {geom.domain}",
        f"periodic {int(geom.periodic[0])} {int(geom.periodic[1])} {int(geom.periodic[2])}",
        f"dx {geom.dx[0]!r} {geom.dx[1]!r} {geom.dx[2]!r}",
        f"ncomp {mf.ncomp}",
        f"nghost {mf.nghost}",
        f"layout {mf.layout_kind}",
        f"nunits {len(mf.units)}",
    ]
    for u in mf.units:
        lines.append(f"unit grid={u.grid} valid={u.valid}")
    return "\n".join(lines) + "\n"


def write_plotfile(mf, geom: Geometry, path: str) -> None:
    """Text HEADER plus one binary fab dump per unit (level.py:326-345)."""
    os.makedirs(path, exist_ok=True)
    if mf.rank == 0:
        with open(os.path.join(path, "HEADER"), "w") as fh:
            fh.write(header_text(mf, geom))
    for u, flat in pack_units(mf).items():
        with open(os.path.join(path, f"unit_{u:05d}.fab"), "wb") as fh:
            FArrayBox(mf.units[u].fab.abox, mf.ncomp, _flat=flat).write(fh)


def read_plotfile(path: str) -> tuple:
    """(header text, [FArrayBox per unit in unit order]) (level.py:348-359)."""
    with open(os.path.join(path, "HEADER")) as fh:
        header = fh.read()
    fabs = []
    n = 0
    while True:
        p = os.path.join(path, f"unit_{n:05d}.fab")
        if not os.path.exists(p):
            break
        with open(p, "rb") as fh:
            fabs.append(FArrayBox.read(fh))
        n += 1
    return header, fabs
