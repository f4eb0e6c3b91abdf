// Device reductions over a MultiFab, one sweep block per unit (grid).
//
// tm_reduce_sum reproduces the reference's checksum bit for bit
// (level.py:183-190 + compiled.py:20-29): per grid, a strictly serial
// x-fastest accumulation starting from 0.0; then the grid partials added
// serially in grid order.  The per-grid chain is evaluated warp-parallel in
// exact integer arithmetic wherever that provably gives the same roundings
// (see fast_chain below), serially elsewhere.
//
// tm_reduce_minmax is order-independent (reference reduce_max/min :175-181)
// and uses atomics on an order-preserving integer image of the doubles.
#include <cmath>
#include <cstdint>
#include <string>

#include "tm_common.cuh"

struct tm_sweep_plan;  // defined in tm_stencil.cu; only its block table is used here
extern "C" int tm_internal_plan_blocks(const tm_sweep_plan *p, const tm_block **d_blocks, int64_t *n);
extern "C" int64_t tm_internal_plan_max_cells(const tm_sweep_plan *p);

namespace {

// The reference's chain of dependent adds (T <- fl(T + v), in order) is
// reproduced exactly without walking it one add at a time.  While the running
// sum T stays positive in one binade [2^e, 2^(e+1)) -- more precisely while
// every exact T + v falls in it -- each step rounds to the grid q = 2^(e-52):
// T_(i+1) = T_i + q * round(v_i / q), ties to even.  In units of q the chain
// is integer addition: K_(i+1) = K_i + R_i with R_i = floor(w_i) + (frac(w_i)
// > 1/2), w_i = v_i / q (exact: power-of-2 scaling), and "T_i + v_i in the
// binade" is 2^52 <= K_i + floor(w_i) <= 2^53 - 1.  So a warp takes 8
// consecutive values per lane, forms the R_i and their in-lane prefix with
// 64-bit integers, scans the lane totals, and checks the binade condition per
// lane; the first lane that fails (binade change, exact tie, NaN/Inf, sum
// near 0 or out of the safe exponent range) is added serially with __dadd_rn
// and the warp retries the rest of the chunk from the new T.  Negative T
// uses the mirror image (fl(-x) = -fl(x)).  The result is the serial sum bit
// for bit; the serial adds left are the few per binade change.
//
// One CTA per grid: a producer warp streams the grid's cells in the
// reference order (x fastest, then y, z) into a shared-memory ring --
// several rows per 1-D bulk copy when rows are 16-byte aligned with x extents
// a multiple of 8, else by coalesced loads -- and four consumer warps take
// the stages in turn (fast_sum_kernel).
constexpr int kFsStage = 3072;  // doubles per ring stage (a span's row padding included)
constexpr int kFsVals = 2048;   // values per stage at most
constexpr int kFsStages = 6;
constexpr size_t kFsSmem = (size_t)kFsStages * kFsStage * sizeof(double) + 2 * kFsStages * sizeof(uint64_t);

__device__ __forceinline__ void bulk_row_load(uint32_t dst, const double *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

__device__ __forceinline__ void mbar_expect_tx_u32(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

// Add the `n` (<= 8) values at shared address `a` (16-B aligned) to T in
// order, serially: loads first, then the dependent adds.
__device__ __forceinline__ double serial8(double T, uint32_t a, int n) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; u += 2) tmk::lds_f64x2(a + 8u * u, v[u], v[u + 1]);
#pragma unroll
    for (int u = 0; u < 8; ++u)
        if (u < n) T = __dadd_rn(T, v[u]);
    return T;
}

constexpr int64_t kKLo = 1ll << 52, kKHi = (1ll << 53) - 1;

// One value in units of q: w = v / q (exact; `scale` = +-1/q carries T's
// sign).  R = round-to-nearest(w) (ties are flagged: their direction depends
// on the running sum's parity), F = floor(w).  1.5 * 2^52 added to |w| <
// 2^51 leaves round(w) in the low mantissa bits, read as an integer
// difference of bit patterns.
__device__ __forceinline__ void units_of_q(double v, double scale, int64_t &F, int64_t &R, bool &bad) {
    constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
    const double w = __dmul_rn(v, scale);
    const bool ok = fabs(w) < 2251799813685248.0;  // 2^51; false for NaN
    const double t = __dadd_rn(ok ? w : 0.0, kMagic);
    const double d = __dsub_rn(w, __dsub_rn(t, kMagic));  // w - round(w), exact
    R = (int64_t)(__double_as_longlong(t) - __double_as_longlong(kMagic));
    F = R - (d < 0.0 ? 1 : 0);
    bad |= !ok || fabs(d) == 0.5;
}

// Lane summary of up to 8 values: in-lane sum of R, min / max of (prefix + F)
// (the binade test), any value the fast path cannot take.  When no F is
// negative the prefixes only grow and (prefix + F) is nondecreasing, so its
// extremes are the first and last values -- no per-value min / max.
struct LaneSum {
    int64_t P, lo, hi;
    bool bad;
};
// The common case, 8 values: branch-free.  F is needed only for the first
// and last value unless some value is negative.
__device__ __forceinline__ LaneSum lane_summary8(const double (&v)[8], double scale, bool neg) {
    constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
    const double sc = neg ? -scale : scale;
    LaneSum r{0, 0, 0, false};
    int64_t R[8];
    double d[8];
    bool bad = false, down = false;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const double w = __dmul_rn(v[u], sc);
        const double t = __dadd_rn(w, kMagic);
        d[u] = __dsub_rn(w, __dsub_rn(t, kMagic));
        R[u] = (int64_t)(__double_as_longlong(t) - __double_as_longlong(kMagic));
        bad |= !(fabs(w) < 2251799813685248.0) || fabs(d[u]) == 0.5;  // 2^51 (catches NaN); ties
        down |= w < 0.0;
        r.P += R[u];
    }
    r.bad = bad;
    if (!down) {
        r.lo = R[0] - (d[0] < 0.0 ? 1 : 0);
        r.hi = r.P - R[7] + R[7] - (d[7] < 0.0 ? 1 : 0);
    } else {
        int64_t P = 0;
        r.lo = INT64_MAX;
        r.hi = INT64_MIN;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t F = R[u] - (d[u] < 0.0 ? 1 : 0);
            r.lo = min(r.lo, P + F);
            r.hi = max(r.hi, P + F);
            P += R[u];
        }
    }
    return r;
}

__device__ __forceinline__ LaneSum lane_summary(const double (&v)[8], int myn, bool mine, double scale, bool neg) {
    LaneSum r{0, 0, 0, false};
    if (!mine) return r;
    if (myn == 8) return lane_summary8(v, scale, neg);
    const double sc = neg ? -scale : scale;
    int64_t F[8], R[8];
    bool down = false;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        F[u] = R[u] = 0;
        if (u < myn) {
            units_of_q(v[u], sc, F[u], R[u], r.bad);
            down |= F[u] < 0;
        }
    }
    if (!down) {
        int64_t last = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (u < myn) {
                last = r.P + F[u];
                r.P += R[u];
            }
        r.lo = F[0];
        r.hi = last;
    } else {
        r.lo = INT64_MAX;
        r.hi = INT64_MIN;
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (u < myn) {
                r.lo = min(r.lo, r.P + F[u]);
                r.hi = max(r.hi, r.P + F[u]);
                r.P += R[u];
            }
    }
    return r;
}

__device__ __forceinline__ int64_t warp_incl_scan(int64_t x, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += t;
    }
    return x;
}

// Is T in the fast path's range?  Sets the binade scaling and |T| / q.
__device__ __forceinline__ bool fast_range(double T, double &scale, double &q, bool &neg, int64_t &K) {
    const uint64_t tb = (uint64_t)__double_as_longlong(T);
    const int ex = (int)((tb >> 52) & 0x7ff);
    if (ex <= 63 || ex >= 2000) return false;  // need 2^-960 < |T| < 2^977: the scalings are exact
    neg = tb >> 63;
    scale = __longlong_as_double((long long)(2098 - ex) << 52);  // 2^(52-e)
    q = __longlong_as_double((long long)(ex - 52) << 52);        // 2^(e-52)
    K = (int64_t)((tb & ((1ull << 52) - 1)) | (1ull << 52));
    return true;
}
__device__ __forceinline__ double from_units(int64_t K, double q, bool neg) {
    const double mag = __dmul_rn((double)K, q);  // exact: 2^52 <= K <= 2^53, q a power of 2
    return neg ? -mag : mag;
}

// One chunk (lane L: values c0 + 8L ..), lanes below `from` already in T;
// retries the fast path from each lane it had to add serially, and gives
// up to serial adds after three attempts.  Warp-uniform.
template <class At>
__device__ __forceinline__ double chunk_slow(double T, const double (&v)[8], int myn, int c0, int from, int cnt,
                                             int lane, const At &at) {
    int tries = 0;
    while (from < 32) {
        if (tries++ == 3) {
            for (; from < 32; ++from) {
                const int s0 = c0 + from * 8;
                T = serial8(T, at(s0), max(0, min(8, cnt - s0)));
            }
            break;
        }
        const bool mine = lane >= from && myn > 0;
        double scale, q;
        bool neg;
        int64_t K;
        if ((uint64_t)__double_as_longlong(T) == 0) {  // T = +0 stays +0 through +-0 values
            bool nz = false;
#pragma unroll
            for (int u = 0; u < 8; ++u) nz |= u < myn && ((uint64_t)__double_as_longlong(v[u]) << 1) != 0;
            const unsigned m = __ballot_sync(0xffffffffu, mine && nz);
            if (!m) break;
            from = __ffs(m) - 1;
        } else if (fast_range(T, scale, q, neg, K)) {
            const LaneSum ls = lane_summary(v, myn, mine, scale, neg);
            const int64_t inc = warp_incl_scan(ls.P, lane), off = inc - ls.P;
            const bool fail = mine && (ls.bad || K + off + ls.lo < kKLo || K + off + ls.hi > kKHi);
            const unsigned m = __ballot_sync(0xffffffffu, fail);
            const int upto = m ? __ffs(m) - 1 : 31;
            K += m ? __shfl_sync(0xffffffffu, off, upto) : __shfl_sync(0xffffffffu, inc, 31);
            T = from_units(K, q, neg);
            if (!m) break;
            from = upto;
        }
        const int s0 = c0 + from * 8;  // lane `from`'s values, serially
        T = serial8(T, at(s0), max(0, min(8, cnt - s0)));
        ++from;
    }
    return T;
}

// Consume `cnt` values (the reference order) at shared address `a` into T.
// Value g sits at a + 8 g, or -- `rstride` != 0: rows of `nx` values at a
// stride of `rstride` (nx % 8 == 0, so no 8-value group straddles rows) --
// at a + 8 ((g / nx) rstride + g % nx).  Four chunks of 256 are summarised
// at once in the units of T's binade at their start (independent work: the
// FP64 latencies overlap) and then checked in order; the units stay valid
// across the chunks, since the check itself bounds every partial sum to the
// binade.  Warp-uniform: every lane returns the same T.
constexpr int kFsGroup = 4;
__device__ __forceinline__ double fast_chain(double T, uint32_t a, int g0, int cnt, int lane, int nx, int rstride) {
    auto at = [&](int g) -> uint32_t {
        if (g >= cnt) return a;  // past the stage's values: never read, but keep it a valid address
        if (!rstride) return a + 8u * (uint32_t)g;
        const int r = g / nx;
        return a + 8u * (uint32_t)(r * rstride + (g - r * nx));
    };
    for (int c0 = g0; c0 < cnt; c0 += kFsGroup * 256) {
        double v[kFsGroup][8];
        int myn[kFsGroup];
#pragma unroll
        for (int j = 0; j < kFsGroup; ++j) {
            const int my0 = c0 + j * 256 + lane * 8;
            myn[j] = max(0, min(8, cnt - my0));
            const uint32_t mya = at(my0);
            if (myn[j] == 8) {
#pragma unroll
                for (int u = 0; u < 8; u += 2) tmk::lds_f64x2(mya + 8u * u, v[j][u], v[j][u + 1]);
            } else {
#pragma unroll
                for (int u = 0; u < 8; ++u) v[j][u] = u < myn[j] ? tmk::lds_f64(mya + 8u * u) : 0.0;
            }
        }
        int jfail = 0, from = 0;  // where the slow path takes over
        double scale, q;
        bool neg;
        int64_t K;
        if (fast_range(T, scale, q, neg, K)) {
            LaneSum ls[kFsGroup];
            int64_t inc[kFsGroup];
#pragma unroll
            for (int j = 0; j < kFsGroup; ++j) ls[j] = lane_summary(v[j], myn[j], myn[j] > 0, scale, neg);
#pragma unroll
            for (int j = 0; j < kFsGroup; ++j) inc[j] = warp_incl_scan(ls[j].P, lane);
            jfail = kFsGroup;
#pragma unroll
            for (int j = 0; j < kFsGroup; ++j) {
                if (jfail == kFsGroup) {
                    const int64_t off = inc[j] - ls[j].P;
                    const bool fail = myn[j] > 0 && (ls[j].bad || K + off + ls[j].lo < kKLo || K + off + ls[j].hi > kKHi);
                    const unsigned m = __ballot_sync(0xffffffffu, fail);
                    if (!m) {
                        K += __shfl_sync(0xffffffffu, inc[j], 31);
                    } else {
                        from = __ffs(m) - 1;
                        K += __shfl_sync(0xffffffffu, off, from);
                        jfail = j;
                    }
                }
            }
            T = from_units(K, q, neg);
            if (jfail == kFsGroup) continue;
            const int s0 = c0 + jfail * 256 + from * 8;  // the failing lane's values, serially
            T = serial8(T, at(s0), max(0, min(8, cnt - s0)));
            ++from;
        }
#pragma unroll
        for (int j = 0; j < kFsGroup; ++j)
            if (j >= jfail) T = chunk_slow(T, v[j], myn[j], c0 + j * 256, j == jfail ? from : 0, cnt, lane, at);
    }
    return T;
}

// Shared-address form of a stage's value g (see fast_chain).
__device__ __forceinline__ uint32_t stage_at(uint32_t a, int g, int nx, int rstride) {
    if (!rstride) return a + 8u * (uint32_t)g;
    const int r = g / nx;
    return a + 8u * (uint32_t)(r * rstride + (g - r * nx));
}

constexpr int kFsWarps = 4;  // consumer warps; warp kFsWarps is the producer
constexpr int kFsChunks = kFsVals / 256;

// Consumer warp w owns stages w, w + W, w + 2W, ...  In each round the W
// warps summarise their stages at once, all in the units of the binade of T
// at the start of the round (speculation: the binade rarely changes), then
// pass T down the warps in stage order: each checks its summaries against
// the incoming T and either adds them (a few ballots) or, where the check
// fails or T left the speculated binade, finishes its stage with fast_chain.
__global__ void __launch_bounds__((kFsWarps + 1) * 32, 1)
    fast_sum_kernel(const tm_block *__restrict__ blocks, const double *__restrict__ base, tm_layout L, int comp,
                    double *__restrict__ partial) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *ring = reinterpret_cast<double *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + (size_t)kFsStages * kFsStage * sizeof(double));
    __shared__ double hand[kFsWarps];
    const tm_block b = blocks[blockIdx.x];
    const tmk::Strides st = tmk::strides_of(L);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double *p0 = base + (int64_t)b.slot * st.slot + (int64_t)comp * st.comp + (int64_t)b.z0 * st.plane +
                       (int64_t)b.y0 * st.row + b.x0;
    const int64_t n = (int64_t)b.ny * b.nz * b.nx;
    // span mode (x extent a multiple of 8, 16-B aligned rows): a stage is up to
    // rps consecutive rows of one z plane fetched as ONE bulk copy of the
    // contiguous span (row padding included, skipped by the consumer); else
    // flat stages of kFsVals values gathered by loads
    const bool span = ((reinterpret_cast<uintptr_t>(p0) & 15) == 0) && (b.nx & 7) == 0 && (st.row & 1) == 0 &&
                      st.row <= kFsStage && b.nx <= kFsVals;
    int rps = 0;  // rows per stage: fit the ring stage, prefer whole 1024-value groups
    if (span) {
        const int rmax = (int)min(min((int64_t)((kFsStage - b.nx) / st.row + 1), (int64_t)b.ny),
                                  (int64_t)(kFsVals / b.nx));
        rps = rmax;
        for (int r = rmax; r >= 1; --r)
            if ((r * b.nx) % (kFsGroup * 256) == 0) {
                rps = r;
                break;
            }
    }
    const int spp = span ? (b.ny + rps - 1) / rps : 0;  // stages per plane
    const int64_t nstage = span ? (int64_t)b.nz * spp : (n + kFsVals - 1) / kFsVals;
    const uint32_t sring = tmk::smem_u32(ring), sfull = tmk::smem_u32(bars), sempty = sfull + 8u * kFsStages;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kFsStages; ++i) {
            tmk::mbar_init(bars + i, span ? 1 : 32);
            tmk::mbar_init(bars + kFsStages + i, 1);
        }
        tmk::fence_mbar_init();
    }
    __syncthreads();
    if (warp == kFsWarps) {  // producer
        int pj = 0;              // span: first row of the next stage in plane pk
        int64_t pk = 0;
        int gx = lane % b.nx;    // loads: this lane's next cell (flat index lane + 32 t)
        int64_t gj = (lane / b.nx) % b.ny, gk = lane / b.nx / b.ny;
        for (int64_t s = 0; s < nstage; ++s) {
            const int slot = (int)(s % kFsStages);
            if (s >= kFsStages) tmk::mbar_wait_u32(sempty + 8u * slot, (uint32_t)((s / kFsStages - 1) & 1));
            const uint32_t dst = sring + (uint32_t)(slot * kFsStage * 8);
            if (span) {
                const int rows = min(rps, b.ny - pj);
                if (lane == 0) {
                    const uint32_t bytes = (uint32_t)(((int64_t)(rows - 1) * st.row + b.nx) * 8);
                    mbar_expect_tx_u32(sfull + 8u * slot, bytes);
                    bulk_row_load(dst, p0 + pk * st.plane + (int64_t)pj * st.row, bytes, sfull + 8u * slot);
                }
                pj += rows;
                if (pj == b.ny) pj = 0, ++pk;
            } else {
                const int cnt = (int)min((int64_t)kFsVals, n - s * kFsVals);
                for (int t = lane; t < cnt; t += 32) {  // (gx, gj, gk): this lane's next cell
                    tmk::sts_f64(dst + 8u * t, __ldg(p0 + gk * st.plane + gj * st.row + gx));
                    gx += 32;
                    while (gx >= b.nx) {
                        gx -= b.nx;
                        if (++gj == b.ny) gj = 0, ++gk;
                    }
                }
                tmk::mbar_arrive_u32(sfull + 8u * slot);
            }
        }
        // stay resident until the consumers have drained every copy this warp issued
        for (int64_t s = max((int64_t)0, nstage - kFsStages); s < nstage; ++s)
            tmk::mbar_wait_u32(sempty + 8u * (uint32_t)(s % kFsStages), (uint32_t)((s / kFsStages) & 1));
        return;
    }
    const int rstride = span ? (int)st.row : 0;
    double Tbase = 0.0;  // T at the start of the round (every consumer warp)
    const int64_t nround = (nstage + kFsWarps - 1) / kFsWarps;
    for (int64_t r = 0; r < nround; ++r) {
        const int64_t s = r * kFsWarps + warp;
        const bool active = s < nstage;
        const int slot = (int)(s % kFsStages);
        const uint32_t a = sring + (uint32_t)(slot * kFsStage * 8);
        int cnt = 0;
        if (active) {
            if (span) {
                const int i = (int)(s % spp);
                cnt = min(rps, b.ny - i * rps) * b.nx;
            } else {
                cnt = (int)min((int64_t)kFsVals, n - s * kFsVals);
            }
            tmk::mbar_wait_u32(sfull + 8u * slot, (uint32_t)((s / kFsStages) & 1));
        }
        // speculative summaries of every chunk of the stage in Tbase's binade
        double scale, q;
        bool neg;
        int64_t Kb;
        const bool spec = active && fast_range(Tbase, scale, q, neg, Kb);
        LaneSum ls[kFsChunks];
        int64_t inc[kFsChunks];
#pragma unroll
        for (int j = 0; j < kFsChunks; ++j) {
            const int my0 = j * 256 + lane * 8;
            const int myn = spec ? max(0, min(8, cnt - my0)) : 0;
            double v[8];
            const uint32_t mya = myn > 0 ? stage_at(a, my0, b.nx, rstride) : a;
            if (myn == 8) {
#pragma unroll
                for (int u = 0; u < 8; u += 2) tmk::lds_f64x2(mya + 8u * u, v[u], v[u + 1]);
            } else {
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = u < myn ? tmk::lds_f64(mya + 8u * u) : 0.0;
            }
            ls[j] = lane_summary(v, myn, myn > 0, scale, neg);
        }
#pragma unroll
        for (int j = 0; j < kFsChunks; ++j) inc[j] = warp_incl_scan(ls[j].P, lane);
        // the whole stage folded into one test: total, and min / max over every value of
        // (prefix + floor) relative to the stage start -- so the ordered hand-off below is
        // one comparison per warp unless the stage needs the chunk-by-chunk path
        int64_t stot = 0, slo = INT64_MAX, shi = INT64_MIN;
        bool sbad = false;
        if (spec) {
#pragma unroll
            for (int j = 0; j < kFsChunks; ++j) {
                if (j * 256 + lane * 8 < cnt) {
                    const int64_t base_l = stot + inc[j] - ls[j].P;
                    slo = min(slo, base_l + ls[j].lo);
                    shi = max(shi, base_l + ls[j].hi);
                    sbad |= ls[j].bad;
                }
                stot += __shfl_sync(0xffffffffu, inc[j], 31);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                slo = min(slo, (int64_t)__shfl_xor_sync(0xffffffffu, slo, o));
                shi = max(shi, (int64_t)__shfl_xor_sync(0xffffffffu, shi, o));
            }
            sbad = __any_sync(0xffffffffu, sbad);
        }
        // T = +0 (a zero field's start): does the stage hold only +-0?  Then T stays +0.
        bool zeros = false;
        if (active && __double_as_longlong(Tbase) == 0) {
            bool nz = false;
            for (int g = lane; g < cnt; g += 32)
                nz |= ((uint64_t)__double_as_longlong(tmk::lds_f64(stage_at(a, g, b.nx, rstride))) << 1) != 0;
            zeros = !__any_sync(0xffffffffu, nz);
        }
        // T from the previous stage's owner
        double T;
        if (warp == 0) {
            T = Tbase;
        } else {
            tmk::named_barrier_sync(warp, 64);
            T = hand[warp - 1];
        }
        if (active && zeros && __double_as_longlong(T) == 0) {
            __syncwarp();
            if (lane == 0) tmk::mbar_arrive_u32(sempty + 8u * slot);
        } else if (active) {
            int jf = 0, from = 0;  // where fast_chain must take over (jf == kFsChunks: nowhere)
            double sc2, q2;
            bool neg2;
            int64_t K;
            const bool same = spec && fast_range(T, sc2, q2, neg2, K) && sc2 == scale && neg2 == neg;
            if (same && !sbad && K + slo >= kKLo && K + shi <= kKHi) {
                jf = kFsChunks;  // the common case: the whole stage at once
                K += stot;
                T = from_units(K, q, neg);
            } else if (same) {
                jf = kFsChunks;
#pragma unroll
                for (int j = 0; j < kFsChunks; ++j) {
                    if (jf == kFsChunks && j * 256 < cnt) {
                        const int64_t off = inc[j] - ls[j].P;
                        const bool fail = j * 256 + lane * 8 < cnt &&
                                          (ls[j].bad || K + off + ls[j].lo < kKLo || K + off + ls[j].hi > kKHi);
                        const unsigned m = __ballot_sync(0xffffffffu, fail);
                        if (!m) {
                            K += __shfl_sync(0xffffffffu, inc[j], 31);
                        } else {
                            from = __ffs(m) - 1;
                            K += __shfl_sync(0xffffffffu, off, from);
                            jf = j;
                        }
                    }
                }
                T = from_units(K, q, neg);
            }
            if (jf < kFsChunks) {
                auto at = [&](int g) -> uint32_t { return g >= cnt ? a : stage_at(a, g, b.nx, rstride); };
                int g0 = jf * 256;
                if (from > 0 || jf > 0) {  // finish chunk jf from lane `from` (that lane serially first)
                    const int s0 = g0 + from * 8;
                    T = serial8(T, at(s0), max(0, min(8, cnt - s0)));
                    double v[8];
                    const int my0 = g0 + lane * 8;
                    const int myn = max(0, min(8, cnt - my0));
                    const uint32_t mya = at(my0);
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = u < myn ? tmk::lds_f64(mya + 8u * u) : 0.0;
                    T = chunk_slow(T, v, myn, g0, from + 1, cnt, lane, at);
                    g0 += 256;
                }
                T = fast_chain(T, a, g0, cnt, lane, b.nx, rstride);
            }
            __syncwarp();
            if (lane == 0) tmk::mbar_arrive_u32(sempty + 8u * slot);
        }
        if (lane == 0) hand[warp] = T;
        if (warp + 1 < kFsWarps) tmk::named_barrier_arrive(warp + 1, 64);
        tmk::named_barrier_sync(kFsWarps, kFsWarps * 32);  // round done: every warp sees the last T
        Tbase = hand[kFsWarps - 1];  // (rewritten next round only after every warp passed its hand-off)
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = Tbase;
}

// Small grids (many of them): the plain serial chain, many light CTAs per SM.
// What must not sit on the chain is memory or shuffle latency.  Two warps per grid: warp 1
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
    // Many small grids: the light serial kernel packs 32 CTAs per SM; few large
    // grids: the warp-parallel kernel (one heavy CTA per grid).  Estimated times,
    // ~9 ns per serial add vs ~2 ns per value + 5 us per CTA.
    int sms = 148;
    {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const double cells = (double)tm_internal_plan_max_cells(plan);
    const double t_serial = std::ceil((double)n / (sms * 32.0)) * cells * 9e-9;
    const double t_fast = std::ceil((double)n / sms) * (cells * 2e-9 + 5e-6);
    if (t_serial < t_fast) {
        serial_sum_kernel<<<(unsigned)n, 64, 0, as_stream(stream)>>>(blocks, base, *layout, comp, d_partial);
        ordered_sum_kernel<<<1, 1, 0, as_stream(stream)>>>(d_partial, n, d_total);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "tm_reduce_sum launch");
        return TM_OK;
    }
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(fast_sum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFsSmem);
        if (e != cudaSuccess) return cuda_fail(e, "tm_reduce_sum smem attribute");
        attr = true;
    }
    fast_sum_kernel<<<(unsigned)n, (kFsWarps + 1) * 32, kFsSmem, as_stream(stream)>>>(blocks, base, *layout, comp, d_partial);
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
