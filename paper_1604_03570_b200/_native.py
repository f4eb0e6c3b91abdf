"""ctypes binding of ``libtilemesh_b200.so`` (the C ABI in
``include/tilemesh_b200.h``).

The library is the only compute path: there is no CPU fallback.  Loading
fails loudly when the shared object is missing (run
``__graft_entry__.build()``), and every compute call checks the returned
status and raises with the library's message.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TILEMESH_LIB") or os.path.join(HERE, "libtilemesh_b200.so")

TM_OK = 0
TM_ERR_INVALID = 1
TM_ERR_CUDA = 2
ABI_VERSION = 4

# halo_mode of tm_heat_march (include/tilemesh_b200.h)
HALO_GHOSTS, HALO_PACKED, HALO_FUSED_SCATTER, HALO_FUSED_NBR, HALO_GHOSTS_XH, HALO_FUSED_NBR_GHOSTS = 0, 1, 2, 3, 4, 5
# peer halos (include/tilemesh_b200.h): neighbour-table code of slot s on peer p of a peer set
MAX_PEERS, PEER_SETS, MAX_RANKS = 8, 4, 64


def nbr_peer(p: int, s: int) -> int:
    """TM_NBR_PEER(p, s)."""
    if not (0 <= p < MAX_PEERS and 0 <= s < (1 << 24)):
        raise ValueError(f"peer face ({p}, {s}) out of range")
    return -3 - ((p << 24) + s)


class tm_layout(ctypes.Structure):
    _fields_ = [("nslots", ctypes.c_int64), ("ncomp", ctypes.c_int32), ("nghost", ctypes.c_int32),
                ("pitch", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("xoff", ctypes.c_int32)]


class tm_side(ctypes.Structure):
    _fields_ = [("sy", ctypes.c_int64), ("sz", ctypes.c_int64), ("sc", ctypes.c_int64)]


# numpy images of the C structs (arrays of them are passed by pointer)
COPY_TAG_DTYPE = np.dtype([("dst_off", "<i8"), ("src_off", "<i8"), ("ex", "<i4"), ("ey", "<i4"),
                           ("ez", "<i4"), ("reserved", "<i4")])
BLOCK_DTYPE = np.dtype([("slot", "<i4"), ("x0", "<i4"), ("y0", "<i4"), ("z0", "<i4"), ("nx", "<i4"),
                        ("ny", "<i4"), ("nz", "<i4"), ("parity", "<i4")])
assert COPY_TAG_DTYPE.itemsize == 32 and BLOCK_DTYPE.itemsize == 32

EXPORTS = [
    "tm_last_error", "tm_abi_version", "tm_device_check",
    "tm_copy_plan_create", "tm_copy_plan_destroy", "tm_copy_plan_elements", "tm_copy_run", "tm_xh_to_ghosts",
    "tm_sweep_plan_create", "tm_sweep_plan_destroy", "tm_heat_sweep", "tm_gsrb_color",
    "tm_residual_maxnorm", "tm_reduce_sum", "tm_reduce_minmax",
    "tm_march_plan_create", "tm_march_plan_destroy", "tm_march_plan_reset_halos", "tm_heat_march", "tm_heat_march_fill",
    "tm_gsrb_march", "tm_wide4_march",
    "tm_wide4_march_fused", "tm_wide4_march_nbr", "tm_wide4_march_fill",
    "tm_gsrb_split", "tm_gsrb_merge", "tm_gsrb_split_pass", "tm_face_flux", "tm_divergence_update",
    "tm_comm_nccl_version", "tm_comm_unique_id", "tm_comm_create", "tm_comm_destroy",
    "tm_exchange_create", "tm_exchange_destroy", "tm_halo_exchange",
    "tm_ipc_export", "tm_ipc_open", "tm_ipc_close", "tm_march_plan_set_peers", "tm_heat_march_peer",
    "tm_peer_barrier",
]

_lib = None


class TilemeshError(RuntimeError):
    pass


def load():
    """Load and type the library (no GPU needed just to load)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise TilemeshError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                            "g.build()'` (nvcc, sm_100a); there is no CPU fallback")
    try:  # torch loads its libnccl.so.2 at import: tm_comm.cu then reuses it (one NCCL per process)
        import torch  # noqa: F401
    except ImportError:  # pragma: no cover
        pass
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    P = ctypes.POINTER
    L.tm_last_error.restype = ctypes.c_char_p
    L.tm_last_error.argtypes = []
    L.tm_abi_version.restype = ctypes.c_int
    L.tm_device_check.argtypes = [ctypes.c_int]
    L.tm_copy_plan_create.argtypes = [vp, i64, i32, P(vp)]
    L.tm_copy_plan_destroy.argtypes = [vp]
    L.tm_copy_plan_elements.argtypes = [vp]
    L.tm_copy_plan_elements.restype = i64
    L.tm_copy_run.argtypes = [vp, vp, P(tm_side), vp, P(tm_side), vp]
    L.tm_xh_to_ghosts.argtypes = [P(tm_layout), vp, vp, i32, vp]
    L.tm_sweep_plan_create.argtypes = [vp, i64, P(vp)]
    L.tm_sweep_plan_destroy.argtypes = [vp]
    L.tm_heat_sweep.argtypes = [vp, P(tm_layout), vp, vp, i32, i32, f64, f64, f64, f64, vp]
    L.tm_gsrb_color.argtypes = [vp, P(tm_layout), vp, P(tm_layout), vp, i32, f64, vp]
    L.tm_residual_maxnorm.argtypes = [vp, P(tm_layout), vp, P(tm_layout), vp, f64, vp, vp]
    L.tm_reduce_sum.argtypes = [vp, P(tm_layout), vp, i32, vp, vp, vp]
    L.tm_reduce_minmax.argtypes = [vp, P(tm_layout), vp, i32, vp, vp]
    L.tm_march_plan_create.argtypes = [vp, i64, i32, P(vp)]
    L.tm_march_plan_destroy.argtypes = [vp]
    L.tm_march_plan_reset_halos.argtypes = [vp]
    L.tm_heat_march.argtypes = [vp, P(tm_layout), vp, vp, i32, f64, f64, f64, f64, i32, vp, vp, vp, i32, vp]
    L.tm_heat_march_fill.argtypes = [vp, P(tm_layout), vp, vp, i32, f64, f64, f64, f64, vp, vp, vp, vp, i64, vp]
    L.tm_gsrb_march.argtypes = [vp, P(tm_layout), vp, P(tm_layout), vp, i32, f64, vp, vp, vp]
    L.tm_wide4_march.argtypes = [vp, P(tm_layout), vp, vp, i32, vp, f64, f64, f64, f64, vp]
    L.tm_wide4_march_fused.argtypes = [vp, P(tm_layout), vp, vp, i32, vp, f64, f64, f64, f64, vp, vp, vp]
    L.tm_wide4_march_nbr.argtypes = [vp, P(tm_layout), vp, vp, i32, vp, f64, f64, f64, f64, vp, vp, vp]
    L.tm_wide4_march_fill.argtypes = [vp, P(tm_layout), vp, vp, i32, vp, f64, f64, f64, f64, vp, vp, vp, i64, vp]
    L.tm_gsrb_split.argtypes = [P(tm_layout), vp, i32, i32, i32, vp, vp, vp, P(tm_layout), vp, vp, vp, vp]
    L.tm_gsrb_merge.argtypes = [P(tm_layout), vp, i32, i32, i32, vp, vp, vp, vp]
    L.tm_gsrb_split_pass.argtypes = [vp, i32, i32, i32, i32, i32, f64, vp, vp, vp, vp, vp]
    L.tm_face_flux.argtypes = [vp, i64, i64, i32, i32, i32, i32, f64, vp, i64, i64, vp]
    L.tm_divergence_update.argtypes = [vp, vp, i64, i64, vp, i64, i64, vp, i64, i64, vp, i64, i64, i32, i32, i32,
                                       f64, f64, f64, f64, vp]
    L.tm_comm_nccl_version.argtypes = [P(i32)]
    L.tm_comm_unique_id.argtypes = [ctypes.c_char_p]
    L.tm_comm_create.argtypes = [ctypes.c_char_p, i32, i32, P(vp)]
    L.tm_comm_destroy.argtypes = [vp]
    L.tm_exchange_create.argtypes = [vp, i32, vp, vp, vp, vp, vp, P(vp)]
    L.tm_exchange_destroy.argtypes = [vp]
    L.tm_halo_exchange.argtypes = [vp, vp, vp, vp]
    L.tm_ipc_export.argtypes = [vp, ctypes.c_char_p, P(i64)]
    L.tm_ipc_open.argtypes = [ctypes.c_char_p, i64, P(vp)]
    L.tm_ipc_close.argtypes = [vp, i64]
    L.tm_march_plan_set_peers.argtypes = [vp, i32, P(tm_layout), i32, P(vp), P(i64)]
    L.tm_heat_march_peer.argtypes = [vp, P(tm_layout), vp, vp, i32, f64, f64, f64, f64, vp, vp, vp, i32, i32, vp]
    L.tm_peer_barrier.argtypes = [vp, vp, vp, i32, i32, vp, vp, i64, vp]
    for name in EXPORTS:
        if name not in ("tm_last_error", "tm_abi_version", "tm_copy_plan_elements"):
            getattr(L, name).restype = ctypes.c_int
    if L.tm_abi_version() != ABI_VERSION:
        raise TilemeshError("libtilemesh_b200.so ABI version mismatch; rebuild it")
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    if rc != TM_OK:
        msg = load().tm_last_error().decode(errors="replace")
        if rc == TM_ERR_INVALID:
            raise ValueError(f"{what}: {msg}")
        raise TilemeshError(f"{what} failed ({rc}): {msg}")


def stream_handle(device=None) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream


class CopyPlan:
    """Library-owned device tag table (``tm_copy_plan``)."""

    def __init__(self, tags: np.ndarray, ncomp: int):
        L = load()
        tags = np.ascontiguousarray(tags, dtype=COPY_TAG_DTYPE)
        h = ctypes.c_void_p()
        check(L.tm_copy_plan_create(tags.ctypes.data if len(tags) else None, len(tags), ncomp, ctypes.byref(h)),
              "tm_copy_plan_create")
        self.handle = h
        self.ntags = len(tags)
        self.elements = int(L.tm_copy_plan_elements(h))

    def run(self, dst_ptr: int, dst_side: tuple, src_ptr: int, src_side: tuple, stream: int) -> None:
        ds = tm_side(*dst_side)
        ss = tm_side(*src_side)
        check(load().tm_copy_run(self.handle, dst_ptr, ctypes.byref(ds), src_ptr, ctypes.byref(ss), stream),
              "tm_copy_run")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib is not None:
            _lib.tm_copy_plan_destroy(h)
            self.handle = None


class SweepPlan:
    """Library-owned device block table (``tm_sweep_plan``)."""

    def __init__(self, blocks: np.ndarray):
        L = load()
        blocks = np.ascontiguousarray(blocks, dtype=BLOCK_DTYPE)
        h = ctypes.c_void_p()
        check(L.tm_sweep_plan_create(blocks.ctypes.data if len(blocks) else None, len(blocks), ctypes.byref(h)),
              "tm_sweep_plan_create")
        self.handle = h
        self.nblocks = len(blocks)
        self.blocks = blocks

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib is not None:
            _lib.tm_sweep_plan_destroy(h)
            self.handle = None


class MarchPlan:
    """Library-owned column/segment tables of the persistent sweep (``tm_march_plan``)."""

    def __init__(self, columns: np.ndarray, nctas: int):
        L = load()
        columns = np.ascontiguousarray(columns, dtype=BLOCK_DTYPE)
        h = ctypes.c_void_p()
        check(L.tm_march_plan_create(columns.ctypes.data if len(columns) else None, len(columns), nctas,
                                     ctypes.byref(h)), "tm_march_plan_create")
        self.handle = h
        self.ncolumns = len(columns)
        self.nctas = nctas
        self.columns = columns

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib is not None:
            _lib.tm_march_plan_destroy(h)
            self.handle = None
