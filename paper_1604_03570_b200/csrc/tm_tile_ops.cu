// The reference's per-tile heat operations on device FABs:
//   heat_flux               kernels.py:86-120   (compiled.flux_x/y/z, compiled.py:32-63)
//   heat_divergence_update  kernels.py:122-144  (compiled.divergence, compiled.py:66-81)
// They are not on the bench path (heat_step / the column march fuse them), but a
// caller that builds its own update from fluxes -- as the reference's tests do --
// gets them on the device, bit-identical (reference operation order, no FMA).
// Arrays are strided 3-D views with x contiguous (FAB views of a MultiFab slot,
// or the caller's flux buffers); one thread per face / cell, x fastest.
#include <algorithm>
#include <string>

#include "tm_common.cuh"

namespace {

struct View3 {
    int64_t sy, sz;  // element strides of y and z (x is contiguous)
};

__global__ void face_flux_kernel(const double *__restrict__ u, View3 su, int dir, int32_t nx, int32_t ny,
                                 int32_t nz, double dxi, double *__restrict__ out, View3 so) {
    const int64_t n = (int64_t)nx * ny * nz;
    const int64_t back = dir == 0 ? 1 : (dir == 1 ? su.sy : su.sz);  // the low cell of a face
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t % nx, j = (t / nx) % ny, k = t / ((int64_t)nx * ny);
        const double *hi = u + i + j * su.sy + k * su.sz;  // face f reads cells f - e_dir and f
        out[i + j * so.sy + k * so.sz] = tmk::rn_mul(tmk::rn_sub(hi[0], hi[-back]), dxi);
    }
}

__global__ void divergence_kernel(double *__restrict__ unew, const double *__restrict__ uold, View3 su,
                                  const double *__restrict__ fx, View3 sx, const double *__restrict__ fy, View3 sy,
                                  const double *__restrict__ fz, View3 sz, int32_t nx, int32_t ny, int32_t nz,
                                  double dxi0, double dxi1, double dxi2, double dtD) {
    using namespace tmk;
    const int64_t n = (int64_t)nx * ny * nz;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t % nx, j = (t / nx) % ny, k = t / ((int64_t)nx * ny);
        const double *px = fx + i + j * sx.sy + k * sx.sz;
        const double *py = fy + i + j * sy.sy + k * sy.sz;
        const double *pz = fz + i + j * sz.sy + k * sz.sz;
        const double ax = rn_mul(rn_sub(px[1], px[0]), dxi0);
        const double ay = rn_mul(rn_sub(py[sy.sy], py[0]), dxi1);
        const double az = rn_mul(rn_sub(pz[sz.sz], pz[0]), dxi2);
        const int64_t o = i + j * su.sy + k * su.sz;
        unew[o] = rn_add(uold[o], rn_mul(dtD, rn_add(rn_add(ax, ay), az)));
    }
}

int grid_for(int64_t n) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t blocks = (n + 255) / 256;
    return (int)std::min<int64_t>(std::max<int64_t>(blocks, 1), (int64_t)sms * 16);
}

}  // namespace

extern "C" {

int tm_face_flux(const double *u, int64_t u_sy, int64_t u_sz, int32_t direction, int32_t nx, int32_t ny,
                 int32_t nz, double dxi, double *out, int64_t out_sy, int64_t out_sz, void *stream) {
    using namespace tmk;
    if (!u || !out || direction < 0 || direction > 2 || nx < 0 || ny < 0 || nz < 0)
        return fail(TM_ERR_INVALID, "tm_face_flux: bad arguments");
    const int64_t n = (int64_t)nx * ny * nz;
    if (n == 0) return TM_OK;
    face_flux_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(u, View3{u_sy, u_sz}, direction, nx, ny, nz, dxi,
                                                                 out, View3{out_sy, out_sz});
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "face_flux_kernel launch");
    return TM_OK;
}

int tm_divergence_update(double *unew, const double *uold, int64_t u_sy, int64_t u_sz, const double *fx,
                         int64_t fx_sy, int64_t fx_sz, const double *fy, int64_t fy_sy, int64_t fy_sz,
                         const double *fz, int64_t fz_sy, int64_t fz_sz, int32_t nx, int32_t ny, int32_t nz,
                         double dxi0, double dxi1, double dxi2, double dtD, void *stream) {
    using namespace tmk;
    if (!unew || !uold || !fx || !fy || !fz || nx < 0 || ny < 0 || nz < 0)
        return fail(TM_ERR_INVALID, "tm_divergence_update: bad arguments");
    const int64_t n = (int64_t)nx * ny * nz;
    if (n == 0) return TM_OK;
    divergence_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(
        unew, uold, View3{u_sy, u_sz}, fx, View3{fx_sy, fx_sz}, fy, View3{fy_sy, fy_sz}, fz, View3{fz_sy, fz_sz}, nx, ny,
        nz, dxi0, dxi1, dxi2, dtD);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "divergence_kernel launch");
    return TM_OK;
}

}  // extern "C"
