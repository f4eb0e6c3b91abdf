// Device reductions over a MultiFab, one sweep block per unit (grid).
//
// tm_reduce_sum reproduces the reference's checksum bit for bit
// (level.py:183-190 + compiled.py:20-29): per grid, a strictly serial
// x-fastest accumulation starting from 0.0; then the grid partials added
// serially in grid order.  One warp per grid loads 32 consecutive cells of
// a row (coalesced) and lane 0 consumes them in order through shuffles, so
// the dependency chain is exactly the reference's.
//
// tm_reduce_minmax is order-independent (reference reduce_max/min :175-181)
// and uses atomics on an order-preserving integer image of the doubles.
#include <string>

#include "tm_common.cuh"

struct tm_sweep_plan;  // defined in tm_stencil.cu; only its block table is used here
extern "C" int tm_internal_plan_blocks(const tm_sweep_plan *p, const tm_block **d_blocks, int64_t *n);

namespace {

// The chain of dependent adds is the reference's and cannot be shortened; what
// must not sit on it is memory or shuffle latency.  Two warps per grid: warp 1
// gathers the next batch of kBatch cells (flat x-fastest, then y, z order)
// into a shared-memory double buffer while lane 0 of warp 0 adds the current
// batch serially, reading ahead with 16-byte shared loads.
constexpr int kBatch = 1024;

__global__ void __launch_bounds__(64) serial_sum_kernel(const tm_block *__restrict__ blocks, const double *__restrict__ base,
                                                        tm_layout L, int comp, double *__restrict__ partial) {
    __shared__ __align__(16) double buf[2][kBatch];
    const tm_block b = blocks[blockIdx.x];
    const tmk::Strides st = tmk::strides_of(L);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double *p0 = base + (int64_t)b.slot * st.slot + (int64_t)comp * st.comp +
                       (int64_t)b.z0 * st.plane + (int64_t)b.y0 * st.row + b.x0;
    const int64_t n = (int64_t)b.nx * b.ny * b.nz;
    const int64_t nbatch = (n + kBatch - 1) / kBatch;
    auto gather = [&](int64_t bi) {  // warp 1 only
        double *dst = buf[bi & 1];
        for (int t0 = 0; t0 < kBatch / 32; t0 += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t idx = bi * kBatch + (t0 + u) * 32 + lane;
                v[u] = 0.0;
                if (idx < n) {
                    const int64_t r = idx / b.nx;
                    const int64_t k = r / b.ny;
                    v[u] = __ldg(p0 + k * st.plane + (r - k * b.ny) * st.row + (idx - r * b.nx));
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) dst[(t0 + u) * 32 + lane] = v[u];
        }
    };
    if (warp == 1) gather(0);
    __syncthreads();
    double total = 0.0;
    for (int64_t bi = 0; bi < nbatch; ++bi) {
        if (warp == 1) {
            if (bi + 1 < nbatch) gather(bi + 1);
        } else if (lane == 0) {
            const uint32_t src = tmk::smem_u32(buf[bi & 1]);
            const int64_t left = n - bi * kBatch;
            const int cnt = left < kBatch ? (int)left : kBatch;
            if (cnt == kBatch) {
                for (int t = 0; t < kBatch; t += 32) {
                    double v[32];
#pragma unroll
                    for (int u = 0; u < 32; u += 2) tmk::lds_f64x2(src + 8u * (t + u), v[u], v[u + 1]);
#pragma unroll
                    for (int u = 0; u < 32; ++u) total = __dadd_rn(total, v[u]);
                }
            } else {
                for (int t = 0; t < cnt; ++t) total = __dadd_rn(total, tmk::lds_f64(src + 8u * t));
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = total;
}

__global__ void ordered_sum_kernel(const double *__restrict__ partial, int64_t n, double *__restrict__ out) {
    double total = 0.0;
    for (int64_t b = 0; b < n; ++b) total = __dadd_rn(total, partial[b]);
    out[0] = total;
}

__device__ __forceinline__ unsigned long long order_key(double v) {
    unsigned long long u = (unsigned long long)__double_as_longlong(v);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_key(unsigned long long k) {
    unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)u);
}

__global__ void minmax_init_kernel(unsigned long long *keys) {
    keys[0] = 0ull;    // running max key
    keys[1] = ~0ull;   // running min key
}

__global__ void __launch_bounds__(256) minmax_kernel(const tm_block *__restrict__ blocks, const double *__restrict__ base,
                                                     tm_layout L, int comp, unsigned long long *keys) {
    const tm_block b = blocks[blockIdx.x];
    const tmk::Strides st = tmk::strides_of(L);
    const double *p0 = base + (int64_t)b.slot * st.slot + (int64_t)comp * st.comp;
    unsigned long long kmax = 0ull, kmin = ~0ull;
    const int64_t rows = (int64_t)b.ny * b.nz;
    for (int64_t r = threadIdx.x / 32; r < rows; r += blockDim.x / 32) {
        const int j = (int)(r % b.ny), k = (int)(r / b.ny);
        const double *row = p0 + (int64_t)(b.z0 + k) * st.plane + (int64_t)(b.y0 + j) * st.row + b.x0;
        for (int x = threadIdx.x % 32; x < b.nx; x += 32) {
            const unsigned long long key = order_key(__ldg(row + x));
            kmax = key > kmax ? key : kmax;
            kmin = key < kmin ? key : kmin;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, kmax, o);
        const unsigned long long c = __shfl_xor_sync(0xffffffffu, kmin, o);
        kmax = a > kmax ? a : kmax;
        kmin = c < kmin ? c : kmin;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&keys[0], kmax);
        atomicMin(&keys[1], kmin);
    }
}

__global__ void minmax_final_kernel(unsigned long long *keys) {
    double *out = reinterpret_cast<double *>(keys);
    const double mx = from_key(keys[0]);
    const double mn = from_key(keys[1]);
    out[0] = mx;
    out[1] = mn;
}

int check_args(const tm_sweep_plan *plan, const tm_layout *L, const double *base, int comp, const char *who,
               const tm_block **blocks, int64_t *n) {
    using namespace tmk;
    int rc = check_layout(L, who);
    if (rc) return rc;
    if (!plan || !base) return fail(TM_ERR_INVALID, std::string(who) + ": null argument");
    if (comp < 0 || comp >= L->ncomp) return fail(TM_ERR_INVALID, std::string(who) + ": component out of range");
    tm_internal_plan_blocks(plan, blocks, n);
    if (*n == 0) return fail(TM_ERR_INVALID, std::string(who) + ": reduction over an empty BoxArray");
    return TM_OK;
}

}  // namespace

extern "C" {

int tm_reduce_sum(tm_sweep_plan *plan, const tm_layout *layout, const double *base, int32_t comp, double *d_partial,
                  double *d_total, void *stream) {
    using namespace tmk;
    const tm_block *blocks;
    int64_t n;
    int rc = check_args(plan, layout, base, comp, "tm_reduce_sum", &blocks, &n);
    if (rc) return rc;
    if (!d_partial || !d_total) return fail(TM_ERR_INVALID, "tm_reduce_sum: null output");
    serial_sum_kernel<<<(unsigned)n, 64, 0, as_stream(stream)>>>(blocks, base, *layout, comp, d_partial);
    ordered_sum_kernel<<<1, 1, 0, as_stream(stream)>>>(d_partial, n, d_total);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "tm_reduce_sum launch");
    return TM_OK;
}

int tm_reduce_minmax(tm_sweep_plan *plan, const tm_layout *layout, const double *base, int32_t comp, double *d_out,
                     void *stream) {
    using namespace tmk;
    const tm_block *blocks;
    int64_t n;
    int rc = check_args(plan, layout, base, comp, "tm_reduce_minmax", &blocks, &n);
    if (rc) return rc;
    if (!d_out) return fail(TM_ERR_INVALID, "tm_reduce_minmax: null output");
    auto *keys = reinterpret_cast<unsigned long long *>(d_out);
    cudaStream_t s = as_stream(stream);
    minmax_init_kernel<<<1, 1, 0, s>>>(keys);
    minmax_kernel<<<(unsigned)n, 256, 0, s>>>(blocks, base, *layout, comp, keys);
    minmax_final_kernel<<<1, 1, 0, s>>>(keys);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "tm_reduce_minmax launch");
    return TM_OK;
}

}  // extern "C"
