// Per-launch cost of the peer barrier's ingredients on one GPU (loopback), 200 launches per
// CUDA graph, PDL on every launch.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bp barrier_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

template <int V>
__global__ void k(uint64_t *inbox, uint64_t *epoch) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (V == 0) return;
    __shared__ uint64_t t;
    if (threadIdx.x == 0) { t = *epoch + 1; *epoch = t; }
    __syncwarp();
    if (threadIdx.x != 0) return;
    if (V >= 2) asm volatile("fence.acq_rel.sys;" ::: "memory");
    if (V >= 3) {
        if (V == 5) asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(inbox) : "memory");
        else asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(inbox) : "memory");
    }
    if (V >= 4) {
        uint64_t v;
        do {
            if (V == 5) asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(inbox) : "memory");
            else asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(inbox) : "memory");
        } while (v < t);
    }
}

template <int V>
float run(uint64_t *inbox, uint64_t *epoch, cudaStream_t s) {
    cudaMemset(inbox, 0, 8);
    cudaMemset(epoch, 0, 8);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 200; ++i) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(1);
        cfg.blockDim = dim3(32);
        cfg.stream = s;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        a[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = a;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k<V>, inbox, epoch);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1e3f / 2000.f;
}

int main() {
    uint64_t *inbox, *epoch;
    cudaMalloc(&inbox, 8);
    cudaMalloc(&epoch, 8);
    cudaStream_t s;
    cudaStreamCreate(&s);
    printf("empty PDL kernel        %.3f us\n", run<0>(inbox, epoch, s));
    printf("+ epoch rw              %.3f us\n", run<1>(inbox, epoch, s));
    printf("+ fence.acq_rel.sys     %.3f us\n", run<2>(inbox, epoch, s));
    printf("+ red.release.sys       %.3f us\n", run<3>(inbox, epoch, s));
    printf("+ ld.acquire.sys spin   %.3f us\n", run<4>(inbox, epoch, s));
    printf("gpu-scope red + spin    %.3f us\n", run<5>(inbox, epoch, s));
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
