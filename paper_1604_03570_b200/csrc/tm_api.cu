// C-ABI plumbing: thread-local error string, layout validation, device
// check, and tensor-map encoding through the runtime's driver entry point.
#include <cudaTypedefs.h>

#include <mutex>
#include <string>

#include "tm_common.cuh"

namespace tmk {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int fail(int code, const std::string &msg) {
    set_error(msg);
    return code;
}

int cuda_fail(cudaError_t e, const char *what) {
    return fail(TM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorName(e) + ": " + cudaGetErrorString(e));
}

int check_layout(const tm_layout *L, const char *who) {
    if (!L) return fail(TM_ERR_INVALID, std::string(who) + ": null layout");
    if (L->nslots < 0 || L->ncomp < 1 || L->nghost < 0 || L->pitch < 1 || L->ny < 1 || L->nz < 1 ||
        L->xoff < L->nghost)
        return fail(TM_ERR_INVALID, std::string(who) + ": malformed layout");
    if (L->pitch % 16 != 0 || L->xoff % 16 != 0)
        return fail(TM_ERR_INVALID, std::string(who) + ": pitch and xoff must be multiples of 16 doubles");
    return TM_OK;
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

int encode_plane_map(CUtensorMap *map, const tm_layout &L, const double *base, int box_x, int box_y) {
    Strides s = strides_of(L);
    return encode_plane_map_strided(map, base, L.pitch, L.ny, L.nz, L.nslots * L.ncomp, s.plane, s.comp, box_x, box_y);
}

int encode_plane_map_strided(CUtensorMap *map, const double *base, int64_t pitch, int64_t ny, int64_t nz, int64_t nw,
                             int64_t plane_stride, int64_t w_stride, int box_x, int box_y) {
    std::call_once(g_encode_once, [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    });
    if (!g_encode) return fail(TM_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    if (box_x < 2 || box_x > 256 || (box_x & 1) || box_y < 1 || box_y > 256)
        return fail(TM_ERR_INVALID, "TMA plane box out of range");
    if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) return fail(TM_ERR_INVALID, "storage not 16-B aligned");
    cuuint64_t dims[4] = {(cuuint64_t)pitch, (cuuint64_t)ny, (cuuint64_t)nz, (cuuint64_t)nw};
    cuuint64_t gstr[3] = {(cuuint64_t)(pitch * 8), (cuuint64_t)(plane_stride * 8), (cuuint64_t)(w_stride * 8)};
    cuuint32_t box[4] = {(cuuint32_t)box_x, (cuuint32_t)box_y, 1, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double *>(base), dims, gstr, box,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(TM_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return TM_OK;
}

}  // namespace tmk

extern "C" {

const char *tm_last_error(void) { return tmk::g_last_error.c_str(); }

int tm_abi_version(void) { return TM_ABI_VERSION; }

int tm_device_check(int device) {
    cudaDeviceProp p;
    cudaError_t e = cudaGetDeviceProperties(&p, device);
    if (e != cudaSuccess) return tmk::cuda_fail(e, "cudaGetDeviceProperties");
    if (p.major != 10 || p.minor != 0)
        return tmk::fail(TM_ERR_CUDA, "libtilemesh_b200 is built for sm_100a; device is sm_" +
                                         std::to_string(p.major) + std::to_string(p.minor));
    return TM_OK;
}

}  // extern "C"
