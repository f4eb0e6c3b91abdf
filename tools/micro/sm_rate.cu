// Is the spread of CTA finish times in a persistent streaming kernel a property of the SM a
// CTA lands on?  296 CTAs (2 per SM) each copy an equal contiguous share of a 268-MB
// read + write stream (the C2 step's traffic) with 16-B accesses; every CTA records its SM id
// and its start / end globaltimer.  Repeated launches, fresh and back to back: per-SM mean
// duration and the correlation of the per-SM durations between launches.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sm_rate sm_rate.cu && /tmp/sm_rate
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
#include <vector>

struct Rec {
    uint32_t smid;
    uint64_t t0, t1;
};

__global__ void __launch_bounds__(288, 2) stream_copy(const double2 *__restrict__ src, double2 *__restrict__ dst,
                                                      int64_t per_cta, Rec *rec) {
    uint64_t t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    const int64_t base = (int64_t)blockIdx.x * per_cta;
    for (int64_t i = threadIdx.x; i < per_cta; i += 4 * blockDim.x) {
        double2 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (i + j * blockDim.x < per_cta) v[j] = src[base + i + j * blockDim.x];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (i + j * blockDim.x < per_cta) dst[base + i + j * blockDim.x] = v[j];
    }
    __syncthreads();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) {
        uint32_t s;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
        rec[blockIdx.x] = Rec{s, t0, t1};
    }
}

// The same stream with dynamic shares: CTAs claim chunks of `chunk` 16-B elements through one
// atomic counter, the next claim issued before the current chunk is copied.
__global__ void __launch_bounds__(288, 2) stream_copy_dyn(const double2 *__restrict__ src, double2 *__restrict__ dst,
                                                          int64_t n16, int chunk, unsigned *counter, Rec *rec) {
    __shared__ unsigned claim[2];
    uint64_t t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (threadIdx.x == 0) claim[0] = atomicAdd(counter, 1u);
    __syncthreads();
    const unsigned nchunks = (unsigned)((n16 + chunk - 1) / chunk);
    for (int it = 0;; ++it) {
        const unsigned c = claim[it & 1];
        if (c >= nchunks) break;
        if (threadIdx.x == 0) claim[(it + 1) & 1] = atomicAdd(counter, 1u);
        const int64_t base = (int64_t)c * chunk;
        const int64_t len = min((int64_t)chunk, n16 - base);
        for (int64_t i = threadIdx.x; i < len; i += 4 * blockDim.x) {
            double2 v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (i + j * blockDim.x < len) v[j] = src[base + i + j * blockDim.x];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (i + j * blockDim.x < len) dst[base + i + j * blockDim.x] = v[j];
        }
        __syncthreads();
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) {
        uint32_t s;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
        rec[blockIdx.x] = Rec{s, t0, t1};
    }
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int nctas = 2 * nsm, launches = 12;
    const int64_t n16 = (int64_t)134217728 / 16;  // 134 MB read + 134 MB written
    const int64_t per_cta = n16 / nctas;
    double2 *src, *dst;
    Rec *rec;
    cudaMalloc(&src, n16 * 16);
    cudaMalloc(&dst, n16 * 16);
    cudaMalloc(&rec, sizeof(Rec) * nctas * launches);
    cudaMemset(src, 1, n16 * 16);
    cudaMemset(dst, 0, n16 * 16);
    for (int w = 0; w < 3; ++w) stream_copy<<<nctas, 288>>>(src, dst, per_cta, rec);
    cudaDeviceSynchronize();
    for (int l = 0; l < launches; ++l) {
        stream_copy<<<nctas, 288>>>(l % 2 ? dst : src, l % 2 ? src : dst, per_cta, rec + (int64_t)l * nctas);
        if (l < launches / 2) cudaDeviceSynchronize();  // first half: isolated launches; second half: back to back
    }
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("CUDA error\n"); return 1; }
    std::vector<Rec> h(nctas * launches);
    cudaMemcpy(h.data(), rec, sizeof(Rec) * h.size(), cudaMemcpyDeviceToHost);
    std::vector<std::vector<double>> per_sm(launches, std::vector<double>(nsm, 0.0));
    for (int l = 0; l < launches; ++l) {
        uint64_t first = ~0ull, last = 0, dmin = ~0ull, dmax = 0;
        std::vector<int> cnt(nsm, 0);
        for (int c = 0; c < nctas; ++c) {
            const Rec &r = h[(size_t)l * nctas + c];
            first = std::min(first, r.t0);
            last = std::max(last, r.t1);
            dmin = std::min(dmin, r.t1 - r.t0);
            dmax = std::max(dmax, r.t1 - r.t0);
            if (r.smid < (uint32_t)nsm) { per_sm[l][r.smid] += (double)(r.t1 - r.t0); ++cnt[r.smid]; }
        }
        int two = 0;
        for (int s = 0; s < nsm; ++s) { if (cnt[s]) per_sm[l][s] /= cnt[s]; two += cnt[s] == 2; }
        uint64_t end_min = ~0ull;
        for (int c = 0; c < nctas; ++c) end_min = std::min(end_min, h[(size_t)l * nctas + c].t1);
        printf("launch %2d: span %.1f us, CTA duration min %.1f max %.1f us, first CTA done %.1f us before the last, "
               "%d of %d SMs hold exactly 2 CTAs\n", l, (last - first) / 1e3, dmin / 1e3, dmax / 1e3,
               (last - end_min) / 1e3, two, nsm);
    }
    // dynamic shares, several chunk sizes (16-B elements): span between the first start and the last end
    {
        unsigned *counter;
        cudaMalloc(&counter, sizeof(unsigned));
        const int chunks[] = {288 * 4, 288 * 8, 288 * 16, 288 * 32, 288 * 64};
        for (int chunk : chunks) {
            double span = 0, spread = 0;
            const int reps = 8;
            for (int l = 0; l < reps + 2; ++l) {
                cudaMemset(counter, 0, sizeof(unsigned));
                stream_copy_dyn<<<nctas, 288>>>(l % 2 ? dst : src, l % 2 ? src : dst, n16, chunk, counter, rec);
                cudaDeviceSynchronize();
                if (l < 2) continue;
                cudaMemcpy(h.data(), rec, sizeof(Rec) * nctas, cudaMemcpyDeviceToHost);
                uint64_t first = ~0ull, last = 0, end_min = ~0ull;
                for (int c = 0; c < nctas; ++c) {
                    first = std::min(first, h[c].t0);
                    last = std::max(last, h[c].t1);
                    end_min = std::min(end_min, h[c].t1);
                }
                span += (last - first) / 1e3 / reps;
                spread += (last - end_min) / 1e3 / reps;
            }
            printf("dynamic shares, chunk %6d B: span %.1f us, first CTA done %.1f us before the last\n", chunk * 16,
                   span, spread);
        }
    }
    // correlation of per-SM mean durations between launch 0 and the others
    auto corr = [&](const std::vector<double> &a, const std::vector<double> &b) {
        double ma = 0, mb = 0;
        for (int s = 0; s < nsm; ++s) { ma += a[s]; mb += b[s]; }
        ma /= nsm; mb /= nsm;
        double sab = 0, saa = 0, sbb = 0;
        for (int s = 0; s < nsm; ++s) { sab += (a[s] - ma) * (b[s] - mb); saa += (a[s] - ma) * (a[s] - ma); sbb += (b[s] - mb) * (b[s] - mb); }
        return sab / std::sqrt(saa * sbb);
    };
    printf("correlation of per-SM durations with launch 0:");
    for (int l = 1; l < launches; ++l) printf(" %.2f", corr(per_sm[0], per_sm[l]));
    printf("\n");
    // per-SM mean over all launches, sorted: is there a systematic fast / slow group?
    std::vector<std::pair<double, int>> mean(nsm);
    for (int s = 0; s < nsm; ++s) {
        double m = 0;
        for (int l = 0; l < launches; ++l) m += per_sm[l][s];
        mean[s] = {m / launches / 1e3, s};
    }
    std::sort(mean.begin(), mean.end());
    printf("per-SM mean CTA duration (us), sorted:\n");
    for (int s = 0; s < nsm; ++s) printf("%s sm%-3d %.1f", s % 8 ? " |" : "\n ", mean[s].second, mean[s].first);
    printf("\n");
    return 0;
}
