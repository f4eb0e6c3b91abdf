// Micro-benchmark: 1-D bulk-copy (cp.async.bulk global->shared) throughput per SM.
// One thread per CTA streams a contiguous region through a ring of D stages of
// S bytes (no consumer work).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 bulk_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void bulk_kernel(const char *src, size_t per_cta, int S, int D) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + (size_t)S * D);
    if (threadIdx.x != 0) return;
    for (int i = 0; i < D; ++i)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + i)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    const char *p = src + per_cta * blockIdx.x;
    const int64_t nst = per_cta / S;
    for (int64_t s = 0; s < nst; ++s) {
        const int slot = (int)(s % D);
        if (s >= D) {
            const uint32_t par = (uint32_t)((s / D - 1) & 1);
            asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W%=;\n}\n" ::"r"(smem_u32(bar + slot)), "r"(par) : "memory");
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar + slot)), "r"(S) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(smem + (size_t)slot * S)), "l"(p + s * S), "r"(S), "r"(smem_u32(bar + slot)) : "memory");
    }
    for (int64_t s = nst > D ? nst - D : 0; s < nst; ++s) {
        const int slot = (int)(s % D);
        const uint32_t par = (uint32_t)((s / D) & 1);
        asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W%=;\n}\n" ::"r"(smem_u32(bar + slot)), "r"(par) : "memory");
    }
}

int main() {
    const size_t per_cta = 3u << 20;
    char *src;
    cudaMalloc(&src, per_cta * 148);
    cudaMemset(src, 1, per_cta * 148);
    cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int sizes[] = {512, 4096, 12288, 24576};
    int depths[] = {2, 4, 6, 8};
    int ctas[] = {64, 148};
    for (int c : ctas)
        for (int S : sizes)
            for (int D : depths) {
                if ((size_t)S * D > 190 * 1024) continue;
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                bulk_kernel<<<c, 32, (size_t)S * D + 8 * D>>>(src, per_cta, S, D);
                cudaEventRecord(a);
                for (int r = 0; r < 5; ++r) bulk_kernel<<<c, 32, (size_t)S * D + 8 * D>>>(src, per_cta, S, D);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                ms /= 5;
                printf("ctas %3d S %6d D %d: %.3f ms  %.1f GB/s per CTA  %.0f GB/s total  (%s)\n", c, S, D, ms,
                       per_cta / (ms * 1e-3) / 1e9, per_cta * c / (ms * 1e-3) / 1e9,
                       cudaGetErrorString(cudaGetLastError()));
            }
    return 0;
}
