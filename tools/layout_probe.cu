// Standalone probe: copy 64-double rows stored at pitch P (P = 64, 80, 96, 128) with a
// plain vectorised kernel; does the padding between rows cost DRAM bandwidth?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o layout_probe tools/layout_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void copy_rows(const double2 *__restrict__ src, double2 *__restrict__ dst, long rows, int pitch2) {
    // one warp per row: 32 lanes x double2 = 64 doubles
    long row = (long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    for (; row < rows; row += (long)gridDim.x * (blockDim.x / 32)) {
        double2 v = src[row * pitch2 + lane];
        dst[row * pitch2 + lane] = v;
    }
}

int main() {
    const long rows = 134000000L / 8 / 64;
    for (int pitch : {64, 72, 80, 96, 128}) {
        double2 *a, *b;
        cudaMalloc(&a, rows * pitch * 8);
        cudaMalloc(&b, rows * pitch * 8);
        cudaMemset(a, 0, rows * pitch * 8);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int w = 0; w < 3; ++w) copy_rows<<<148 * 8, 256>>>(a, b, rows, pitch / 2);
        cudaEventRecord(e0);
        for (int r = 0; r < 20; ++r) copy_rows<<<148 * 8, 256>>>(a, b, rows, pitch / 2);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 20;
        printf("pitch %3d: %.1f us, %.0f GB/s of used bytes (r+w)\n", pitch, ms * 1e3, 2.0 * rows * 512 / (ms * 1e-3) / 1e9);
        cudaFree(a);
        cudaFree(b);
    }
    return 0;
}
