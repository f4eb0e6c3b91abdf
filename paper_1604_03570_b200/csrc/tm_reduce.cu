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

__global__ void __launch_bounds__(32) serial_sum_kernel(const tm_block *__restrict__ blocks, const double *__restrict__ base,
                                                        tm_layout L, int comp, double *__restrict__ partial) {
    const tm_block b = blocks[blockIdx.x];
    const tmk::Strides st = tmk::strides_of(L);
    const int lane = threadIdx.x;
    const double *p0 = base + (int64_t)b.slot * st.slot + (int64_t)comp * st.comp;
    double total = 0.0;
    for (int k = 0; k < b.nz; ++k)
        for (int j = 0; j < b.ny; ++j) {
            const double *row = p0 + (int64_t)(b.z0 + k) * st.plane + (int64_t)(b.y0 + j) * st.row + b.x0;
            int x = 0;
            for (; x + 32 <= b.nx; x += 32) {  // full chunks: shuffles unrolled, only the adds chain
                const double v = __ldg(row + x + lane);
#pragma unroll
                for (int l = 0; l < 32; ++l) total = __dadd_rn(total, __shfl_sync(0xffffffffu, v, l));
            }
            if (x < b.nx) {
                const int n = b.nx - x;
                const double v = lane < n ? __ldg(row + x + lane) : 0.0;
                for (int l = 0; l < n; ++l) total = __dadd_rn(total, __shfl_sync(0xffffffffu, v, l));
            }
        }
    if (lane == 0) partial[blockIdx.x] = total;
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
    serial_sum_kernel<<<(unsigned)n, 32, 0, as_stream(stream)>>>(blocks, base, *layout, comp, d_partial);
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
