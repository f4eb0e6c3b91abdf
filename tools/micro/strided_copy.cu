// Copy bandwidth vs row layout: 64 used doubles per row at pitch P (the
// MultiFab i-row layout), read+write, one warp per row, 4 rows in flight per
// warp.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o strided_copy strided_copy.cu
#include <cstdio>
#include <cuda_runtime.h>

template <bool ALIGNED>
__global__ void copy_rows(const double *__restrict__ a, double *__restrict__ b, long rows, int pitch, int off) {
    const int lane = threadIdx.x & 31;
    const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
    const long nwarps = (gridDim.x * (long)blockDim.x) >> 5;
    for (long r0 = warp * 4; r0 < rows; r0 += nwarps * 4) {
        double2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long r = r0 + u;
            if (r < rows) {
                const double *p = a + r * pitch + off + 2 * lane;
                if (ALIGNED) v[u] = *reinterpret_cast<const double2 *>(p);
                else v[u] = make_double2(p[0], p[1]);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long r = r0 + u;
            if (r < rows) {
                double *p = b + r * pitch + off + 2 * lane;
                if (ALIGNED) *reinterpret_cast<double2 *>(p) = v[u];
                else { p[0] = v[u].x; p[1] = v[u].y; }
            }
        }
    }
}

int main() {
    const long rows = 134L * 1000 * 1000 / 8 / 64;
    const int pitches[] = {64, 66, 68, 72, 80, 96, 128};
    const int offs[] = {0, 1, 2, 4, 8, 16, 32};
    for (int t = 0; t < 7; ++t) {
        const int P = pitches[t], off = offs[t];
        double *a, *b;
        cudaMalloc(&a, rows * P * 8);
        cudaMalloc(&b, rows * P * 8);
        cudaMemset(a, 0, rows * P * 8);
        const bool al = off % 2 == 0;
        for (int bpsm = 4; bpsm <= 16; bpsm *= 2) {
            const int grid = 148 * bpsm;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            for (int w = 0; w < 3; ++w)
                al ? copy_rows<true><<<grid, 256>>>(a, b, rows, P, off) : copy_rows<false><<<grid, 256>>>(a, b, rows, P, off);
            cudaEventRecord(e0);
            const int n = 20;
            for (int w = 0; w < n; ++w)
                al ? copy_rows<true><<<grid, 256>>>(a, b, rows, P, off) : copy_rows<false><<<grid, 256>>>(a, b, rows, P, off);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            ms /= n;
            printf("pitch %3d off %2d ctas/SM %2d: %.1f us  %.0f GB/s of used bytes (r+w)\n", P, off, bpsm, ms * 1e3,
                   2.0 * rows * 64 * 8 / (ms * 1e-3) / 1e9);
        }
        cudaFree(a);
        cudaFree(b);
    }
    return 0;
}
