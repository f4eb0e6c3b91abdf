/* A C host of the drop-in boundary (include/tilemesh_b200.h), no Python:
 * FillBoundary of one periodic box as 26 copy tags (tm_copy_run), three heat
 * steps (tm_heat_sweep) and the checksum (tm_reduce_sum), each checked bit for
 * bit against a plain C restatement of the reference arithmetic
 * (compiled.py:32-99 flux form, level.py:183-190 serial sum).
 * Build: gcc -std=c11 -O2 -ffp-contract=off -I include -I $CUDA/include heat_host.c
 *        -L paper_1604_03570_b200 -ltilemesh_b200 -L $CUDA/lib64 -lcudart */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "tilemesh_b200.h"

enum { NX = 16, NY = 12, NZ = 10, NG = 1, XOFF = 16, PITCH = 48, SY = NY + 2 * NG, SZ = NZ + 2 * NG };

static int64_t off(int i, int j, int k) { /* valid-relative (i, j, k) -> storage offset */
    return ((int64_t)(k + NG) * SY + (j + NG)) * PITCH + (i + XOFF);
}

#define CHECK(x)                                                                              \
    do {                                                                                      \
        int rc_ = (x);                                                                        \
        if (rc_ != TM_OK) {                                                                   \
            fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, tm_last_error());                \
            return 1;                                                                         \
        }                                                                                     \
    } while (0)

static void host_step(double *un, const double *uo, double dxi, double dtD) {
    /* periodic wrap instead of ghosts; reference operation order, no FMA */
#define U(i, j, k) uo[off(((i) + NX) % NX, ((j) + NY) % NY, ((k) + NZ) % NZ)]
    for (int k = 0; k < NZ; ++k)
        for (int j = 0; j < NY; ++j)
            for (int i = 0; i < NX; ++i) {
                double fx0 = (U(i, j, k) - U(i - 1, j, k)) * dxi, fx1 = (U(i + 1, j, k) - U(i, j, k)) * dxi;
                double fy0 = (U(i, j, k) - U(i, j - 1, k)) * dxi, fy1 = (U(i, j + 1, k) - U(i, j, k)) * dxi;
                double fz0 = (U(i, j, k) - U(i, j, k - 1)) * dxi, fz1 = (U(i, j, k + 1) - U(i, j, k)) * dxi;
                double ax = (fx1 - fx0) * dxi, ay = (fy1 - fy0) * dxi, az = (fz1 - fz0) * dxi;
                double s = ax + ay;
                s = s + az;
                un[off(i, j, k)] = U(i, j, k) + dtD * s;
            }
#undef U
}

int main(void) {
    const size_t n = (size_t)SZ * SY * PITCH;
    const tm_layout L = {1, 1, NG, PITCH, SY, SZ, XOFF};
    const tm_side side = {PITCH, (int64_t)PITCH * SY, (int64_t)PITCH * SY * SZ};
    CHECK(tm_device_check(0));

    /* FillBoundary of one periodic box: 26 tags, ghost slab <- valid slab one period away */
    tm_copy_tag tags[26];
    int nt = 0;
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                if (!dx && !dy && !dz) continue;
                int lo[3], ex[3], d[3] = {dx, dy, dz}, N[3] = {NX, NY, NZ};
                for (int a = 0; a < 3; ++a) {
                    lo[a] = d[a] < 0 ? -NG : d[a] > 0 ? N[a] : 0;
                    ex[a] = d[a] ? NG : N[a];
                }
                tags[nt].dst_off = off(lo[0], lo[1], lo[2]);
                tags[nt].src_off = off(lo[0] - dx * NX, lo[1] - dy * NY, lo[2] - dz * NZ);
                tags[nt].ex = ex[0];
                tags[nt].ey = ex[1];
                tags[nt].ez = ex[2];
                tags[nt].reserved = 0;
                ++nt;
            }
    tm_copy_plan *fill;
    CHECK(tm_copy_plan_create(tags, nt, 1, &fill));
    const tm_block blk = {0, XOFF, NG, NG, NX, NY, NZ, 0};
    tm_sweep_plan *sweep;
    CHECK(tm_sweep_plan_create(&blk, 1, &sweep));

    double *h = malloc(n * sizeof(double)), *ref = malloc(n * sizeof(double)), *tmp = malloc(n * sizeof(double));
    unsigned s = 12345u;
    for (size_t q = 0; q < n; ++q) h[q] = 0.0;
    for (int k = 0; k < NZ; ++k)
        for (int j = 0; j < NY; ++j)
            for (int i = 0; i < NX; ++i) {
                s = s * 1664525u + 1013904223u;
                h[off(i, j, k)] = (double)(s >> 8) / 16777216.0;
            }
    memcpy(ref, h, n * sizeof(double));
    double *d0, *d1, *dpart, *dtot;
    if (cudaMalloc((void **)&d0, n * sizeof(double)) || cudaMalloc((void **)&d1, n * sizeof(double)) ||
        cudaMalloc((void **)&dpart, sizeof(double)) || cudaMalloc((void **)&dtot, 2 * sizeof(double)))
        return 2;
    cudaMemcpy(d0, h, n * sizeof(double), cudaMemcpyHostToDevice);
    cudaMemcpy(d1, h, n * sizeof(double), cudaMemcpyHostToDevice);

    const double dx = 1.0 / NX, dxi = 1.0 / (dx * dx), dtD = 0.9 * dx * dx / 6.0;
    for (int step = 0; step < 3; ++step) {
        CHECK(tm_copy_run(fill, d0, &side, d0, &side, NULL));
        CHECK(tm_heat_sweep(sweep, &L, d0, d1, 0, 1, dxi, dxi, dxi, dtD, NULL));
        double *t = d0;
        d0 = d1;
        d1 = t;
        host_step(tmp, ref, dxi, dtD);
        for (int k = 0; k < NZ; ++k)
            for (int j = 0; j < NY; ++j)
                for (int i = 0; i < NX; ++i) ref[off(i, j, k)] = tmp[off(i, j, k)];
    }
    cudaMemcpy(h, d0, n * sizeof(double), cudaMemcpyDeviceToHost);
    long bad = 0;
    double want = 0.0;
    for (int k = 0; k < NZ; ++k)
        for (int j = 0; j < NY; ++j)
            for (int i = 0; i < NX; ++i) {
                if (memcmp(&h[off(i, j, k)], &ref[off(i, j, k)], sizeof(double))) ++bad;
                want = want + ref[off(i, j, k)];
            }
    CHECK(tm_reduce_sum(sweep, &L, d0, 0, dpart, dtot, NULL));
    double got;
    cudaMemcpy(&got, dtot, sizeof(double), cudaMemcpyDeviceToHost);
    if (bad || memcmp(&got, &want, sizeof(double))) {
        fprintf(stderr, "c-abi mismatch: %ld cells differ, checksum %.17g vs %.17g\n", bad, got, want);
        return 1;
    }
    printf("c-abi ok: %d tags, 3 steps bit-exact, checksum %.17g\n", nt, got);
    tm_copy_plan_destroy(fill);
    tm_sweep_plan_destroy(sweep);
    return 0;
}
