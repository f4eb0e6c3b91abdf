// Column/segment tables of the persistent march kernels (tm_march.cu heat and
// GSRB, tm_wide4.cu): library-internal, shared by the translation units.
#pragma once

#include "tm_common.cuh"

namespace tmk {

struct Segment {
    int32_t col;     // column index
    int32_t k0, k1;  // local planes [k0, k1) of the column
    int32_t reserved;
};

}  // namespace tmk

struct tm_march_plan {
    int64_t ncols = 0, nsegs = 0;
    int32_t nctas = 0;
    tm_block *d_cols = nullptr;
    tmk::Segment *d_segs = nullptr;
    int32_t *d_seg_begin = nullptr;
    int max_nx = 0, max_ny = 0;
    bool even = true;
    bool uniform_ny = true;  // every column has max_ny rows
    bool uniform_nx = true;  // every column has max_nx cells per row
    bool ny_mult4 = true;    // every column's row count is a multiple of 4 (Kernel W2 row groups)
    int32_t x0_common = -1;  // the x0 every column starts at, or -1
    int32_t last_halo_mode = -1;          // mode of the last fused tm_heat_march (tm_march_plan_reset_halos)
    const void *last_xh_new = nullptr;    // and the packed x halo it wrote
    // peer sets (tm_march_plan_set_peers): per set, 2 TMA maps per peer (column rows, one row)
    // over another rank's storage, in device memory; -1 = set not encoded
    CUtensorMap *d_peer_maps = nullptr;  // [TM_PEER_SETS][TM_MAX_PEERS][2]
    int32_t peer_n[TM_PEER_SETS] = {-1, -1, -1, -1};
    int32_t peer_box_x = 0, peer_box_y = 0;  // the column box the maps were encoded for
};
