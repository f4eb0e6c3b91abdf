// Kernel B's unit of work (tm_copy.cu), shared with the march kernel's fill warp
// (tm_march.cu, tm_heat_march_fill): a tag cut into warp tasks of whole rows.
#pragma once

#include "tm_common.cuh"

namespace tmc {

constexpr int kCopyThreads = 256;
constexpr int kWarps = kCopyThreads / 32;
constexpr uint32_t kShortRow = 8;        // rows up to this width: one row per lane
constexpr int64_t kLongTaskCells = 256;  // target cells per task for long rows

// A run of nrows consecutive y rows of one (z, component) slice of a tag:
// every row of a task starts one side-row stride after the previous.
struct Task {
    int64_t src_off, dst_off;  // the tag's
    int32_t ex, ey, ez;        // the tag's
    int32_t y0, z;
    uint16_t c, nrows;
};

struct SideDev {
    int64_t sy, sz, sc;
};

// offset of cell (0, y, z, c) of a tag on one side; sy == 0: packed per tag
__device__ __forceinline__ int64_t cell_offset(const SideDev &s, int64_t y, int64_t z, int64_t c, int64_t ex,
                                               int64_t ey, int64_t ez) {
    if (s.sy == 0) return ex * (y + ey * (z + ez * c));
    return s.sy * y + s.sz * z + s.sc * c;
}

// One warp copies one task (all lanes call it with the same task).
__device__ __forceinline__ void copy_task(const Task &tk, double *__restrict__ dst, const SideDev &ds,
                                          const double *__restrict__ src, const SideDev &ss, int lane) {
    const int64_t ex = tk.ex, ey = tk.ey, ez = tk.ez;
    const int64_t sy = ss.sy == 0 ? ex : ss.sy, dy = ds.sy == 0 ? ex : ds.sy;  // row strides
    const double *s0 = src + tk.src_off + cell_offset(ss, tk.y0, tk.z, tk.c, ex, ey, ez);
    double *d0 = dst + tk.dst_off + cell_offset(ds, tk.y0, tk.z, tk.c, ex, ey, ez);
    if (ex <= kShortRow) {
        // Short rows (x-face ghosts): lanes split a row (4 x 16 B, or 8 x 8 B when a
        // row is odd-sized or unaligned) so one instruction touches 8 (4) rows, not 32;
        // all of the task's loads are issued before its stores.
        const bool vec = ((ex | ((uintptr_t)s0 >> 3) | ((uintptr_t)d0 >> 3) | sy | dy) & 1) == 0;
        if (vec) {
            const int sub = lane & 3, rr = lane >> 2;
            double2 v[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int row = 8 * i + rr;
                if (row < tk.nrows && 2 * sub < ex)
                    v[i] = __ldg(reinterpret_cast<const double2 *>(s0 + sy * row) + sub);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int row = 8 * i + rr;
                if (row < tk.nrows && 2 * sub < ex) reinterpret_cast<double2 *>(d0 + dy * row)[sub] = v[i];
            }
        } else {
            const int sub = lane & 7, rr = lane >> 3;
            double v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int row = 4 * i + rr;
                if (row < tk.nrows && sub < ex) v[i] = __ldg(s0 + sy * row + sub);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int row = 4 * i + rr;
                if (row < tk.nrows && sub < ex) d0[dy * row + sub] = v[i];
            }
        }
    } else {
        // Long rows (y/z faces, gathers): a task is <= 256 cells (or one row); lanes
        // take 16-B pairs (8-B cells when odd-sized/unaligned) in row-major order, all
        // loads of a pass before its stores.
        const bool vec = ((ex | ((uintptr_t)s0 >> 3) | ((uintptr_t)d0 >> 3) | sy | dy) & 1) == 0;
        const uint32_t w = vec ? (uint32_t)(ex / 2) : (uint32_t)ex;  // units per row
        const uint32_t n = (uint32_t)tk.nrows * w;
        for (uint32_t base = 0; base < n; base += 128) {
            if (vec) {
                double2 v[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t q = base + lane + 32 * i;
                    if (q < n) {
                        const uint32_t r = q / w, x = q - r * w;
                        v[i] = __ldg(reinterpret_cast<const double2 *>(s0 + sy * r) + x);
                    }
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t q = base + lane + 32 * i;
                    if (q < n) {
                        const uint32_t r = q / w, x = q - r * w;
                        reinterpret_cast<double2 *>(d0 + dy * r)[x] = v[i];
                    }
                }
            } else {
                double v[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t q = base + lane + 32 * i;
                    if (q < n) {
                        const uint32_t r = q / w, x = q - r * w;
                        v[i] = __ldg(s0 + sy * r + x);
                    }
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t q = base + lane + 32 * i;
                    if (q < n) {
                        const uint32_t r = q / w, x = q - r * w;
                        d0[dy * r + x] = v[i];
                    }
                }
            }
        }
    }
}

}  // namespace tmc

struct tm_copy_plan {
    int32_t ncomp = 1;
    int64_t ntags = 0;
    int64_t ntasks = 0;
    int64_t elements = 0;
    tmc::Task *d_tasks = nullptr;
    int grid = 0;
};
