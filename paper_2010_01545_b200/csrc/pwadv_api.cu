// pwadv_api.cu — the extern "C" boundary of libpwadv.so (include/pwadv.h).
//
// Argument checks mirror the reference's error behaviour so the Python shim can
// raise the same exceptions (GridError/ValueError before any compute,
// grid.py:52-58, kernel.py:178-179, schedules.py:65-68); here they come back
// as negative codes with a message in pwadv_last_error().
#include <algorithm>
#include <condition_variable>
#include <cstdarg>
#include <deque>
#include <functional>
#include <thread>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include <immintrin.h>

#include "pwadv_internal.h"

namespace pwadv {

static thread_local char g_err[512] = "";
static thread_local uint64_t g_launches = 0;

int set_error(int code, const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int set_cuda_error(const char *what, cudaError_t e)
{
    return set_error(PWADV_E_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

void count_launch() { ++g_launches; }

static constexpr int kMaxDevices = 64;
static DeviceInfo g_devs[kMaxDevices];
static std::once_flag g_dev_once[kMaxDevices];

const DeviceInfo *device_info()
{
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
    std::call_once(g_dev_once[dev], [dev]() {
        DeviceInfo d;
        d.device = dev;
        d.sms = 148;
        d.smem_optin = 227 * 1024;
        cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        g_devs[dev] = d;
    });
    return &g_devs[dev];
}

static int check_dims(int64_t nx, int64_t ny, int64_t nz)
{
    if (nx < 1 || ny < 1)
        return set_error(PWADV_E_DIMS, "horizontal extents must be >= 1, got %lldx%lld",
                         (long long)nx, (long long)ny);
    if (nz < 2)
        return set_error(PWADV_E_DIMS, "nz must be >= 2 (column stencil starts at k=2), got %lld",
                         (long long)nz);
    return PWADV_OK;
}

static int check_ptrs(std::initializer_list<const void *> ps)
{
    for (const void *p : ps) {
        if (!p) return set_error(PWADV_E_NULL, "null pointer argument");
        if ((uintptr_t)p & 7) return set_error(PWADV_E_ALIGN, "pointer %p is not 8-byte aligned", p);
    }
    return PWADV_OK;
}

static int run_box(const double *u, const double *v, const double *w, double *o0, double *o1,
                   double *o2, int64_t nx, int64_t ny, int64_t nz, double tcx, double tcy,
                   const double *tzc1, const double *tzc2, double dt, bool step, int64_t x0,
                   int64_t x1, int64_t y0, int64_t y1, const pwadv_opts *opts, void *stream,
                   const pwadv_peers *peers = nullptr, bool pull = false)
{
    int rc = check_dims(nx, ny, nz);
    if (rc) return rc;
    rc = check_ptrs({u, v, w, o0, o1, o2, tzc1, tzc2});
    if (rc) return rc;
    if (x0 < 1 || x1 > nx + 1 || x0 > x1 || y0 < 1 || y1 > ny + 1 || y0 > y1)
        return set_error(PWADV_E_RANGE, "box [%lld,%lld)x[%lld,%lld) outside interior %lldx%lld",
                         (long long)x0, (long long)x1, (long long)y0, (long long)y1,
                         (long long)nx, (long long)ny);
    BoxLaunch L;
    L.u = u;
    L.v = v;
    L.w = w;
    L.o0 = o0;
    L.o1 = o1;
    L.o2 = o2;
    L.tzc1 = tzc1;
    L.tzc2 = tzc2;
    L.nx = nx;
    L.ny = ny;
    L.nz = nz;
    L.tcx = tcx;
    L.tcy = tcy;
    L.dt = dt;
    L.x0 = x0;
    L.x1 = x1;
    L.y0 = y0;
    L.y1 = y1;
    L.step = step;
    L.flags = opts ? opts->flags : 0u;
    L.tile_j = opts ? opts->tile_j : 0;
    L.stages = opts ? opts->stages : 0;
    L.grid = opts ? opts->grid : 0;
    L.max_threads = opts ? opts->max_threads : 0;
    L.chunks = opts ? opts->chunks : 0;
    L.trace = opts ? opts->trace : nullptr;
    L.peers = peers;
    L.pull = pull;
    if (L.tile_j < 0 || L.stages < 0 || L.grid < 0 || L.max_threads < 0 || L.chunks < 0)
        return set_error(PWADV_E_ARG, "negative tuning value");
    return launch_box(L, (cudaStream_t)stream);
}

}  // namespace pwadv

using namespace pwadv;

namespace {
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev)
    {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard()
    {
        if (prev >= 0) cudaSetDevice(prev);
    }
};
}  // namespace

extern "C" {

int pwadv_abi_version(void) { return PWADV_ABI_VERSION; }

#ifndef PWADV_SOURCE_ID
#define PWADV_SOURCE_ID "unknown"
#endif
const char *pwadv_source_id(void) { return PWADV_SOURCE_ID; }
const char *pwadv_last_error(void) { return g_err; }
uint64_t pwadv_launch_count(void) { return g_launches; }
void pwadv_reset_launch_count(void) { g_launches = 0; }

int pwadv_advect_f64(const double *u, const double *v, const double *w, double *su, double *sv,
                     double *sw, int64_t nx, int64_t ny, int64_t nz, double tcx, double tcy,
                     const double *tzc1, const double *tzc2, const pwadv_opts *opts, void *stream)
{
    return run_box(u, v, w, su, sv, sw, nx, ny, nz, tcx, tcy, tzc1, tzc2, 0.0, false, 1, nx + 1,
                   1, ny + 1, opts, stream);
}

int pwadv_advect_box_f64(const double *u, const double *v, const double *w, double *su,
                         double *sv, double *sw, int64_t nx, int64_t ny, int64_t nz, double tcx,
                         double tcy, const double *tzc1, const double *tzc2, int64_t x_begin,
                         int64_t x_end, int64_t y_begin, int64_t y_end, const pwadv_opts *opts,
                         void *stream)
{
    return run_box(u, v, w, su, sv, sw, nx, ny, nz, tcx, tcy, tzc1, tzc2, 0.0, false, x_begin,
                   x_end, y_begin, y_end, opts, stream);
}

int pwadv_step_box_f64(const double *u, const double *v, const double *w, double *u_new,
                       double *v_new, double *w_new, int64_t nx, int64_t ny, int64_t nz,
                       double tcx, double tcy, const double *tzc1, const double *tzc2, double dt,
                       int64_t x_begin, int64_t x_end, int64_t y_begin, int64_t y_end,
                       const pwadv_opts *opts, void *stream)
{
    if (u == u_new || v == v_new || w == w_new)
        return set_error(PWADV_E_ARG, "fused step needs distinct (ping-pong) output buffers");
    return run_box(u, v, w, u_new, v_new, w_new, nx, ny, nz, tcx, tcy, tzc1, tzc2, dt, true,
                   x_begin, x_end, y_begin, y_end, opts, stream);
}

// peer table of the fused push / pull entry points: complete, aligned to
// `align` bytes, extents consistent with an x-y decomposition
static int check_peers(const pwadv_peers *peers, int64_t nx, int64_t ny, uintptr_t align)
{
    if (!peers) return set_error(PWADV_E_NULL, "null peers");
    for (int d = 0; d < 8; ++d) {
        if (!peers->u[d] || !peers->v[d] || !peers->w[d])
            return set_error(PWADV_E_NULL, "peer %d buffers missing", d);
        if (((uintptr_t)peers->u[d] | (uintptr_t)peers->v[d] | (uintptr_t)peers->w[d]) & (align - 1))
            return set_error(PWADV_E_ALIGN, "peer %d buffers not %d-byte aligned", d, (int)align);
        if (peers->nx[d] < 1 || peers->ny[d] < 1)
            return set_error(PWADV_E_DIMS, "peer %d extents invalid", d);
    }
    // x neighbours share my y extent, y neighbours my x extent
    if (peers->ny[PWADV_NB_XM] != ny || peers->ny[PWADV_NB_XP] != ny ||
        peers->nx[PWADV_NB_YM] != nx || peers->nx[PWADV_NB_YP] != nx)
        return set_error(PWADV_E_RANGE, "peer extents inconsistent with an x-y decomposition");
    return PWADV_OK;
}

int pwadv_step_push_f64(const double *u, const double *v, const double *w, double *u_new,
                        double *v_new, double *w_new, int64_t nx, int64_t ny, int64_t nz,
                        double tcx, double tcy, const double *tzc1, const double *tzc2, double dt,
                        const pwadv_peers *peers, const pwadv_opts *opts, void *stream)
{
    int rc = check_peers(peers, nx, ny, 8);
    if (rc) return rc;
    if (u == u_new || v == v_new || w == w_new)
        return set_error(PWADV_E_ARG, "fused step needs distinct (ping-pong) output buffers");
    return run_box(u, v, w, u_new, v_new, w_new, nx, ny, nz, tcx, tcy, tzc1, tzc2, dt, true, 1,
                   nx + 1, 1, ny + 1, opts, stream, peers);
}

int pwadv_advect_pull_f64(const double *u, const double *v, const double *w, double *su,
                          double *sv, double *sw, int64_t nx, int64_t ny, int64_t nz, double tcx,
                          double tcy, const double *tzc1, const double *tzc2,
                          const pwadv_peers *src, const pwadv_opts *opts, void *stream)
{
    int rc = check_peers(src, nx, ny, 16);
    if (rc) return rc;
    return run_box(u, v, w, su, sv, sw, nx, ny, nz, tcx, tcy, tzc1, tzc2, 0.0, false, 1, nx + 1, 1,
                   ny + 1, opts, stream, src, true);
}

int pwadv_step_pull_f64(const double *u, const double *v, const double *w, double *u_new,
                        double *v_new, double *w_new, int64_t nx, int64_t ny, int64_t nz,
                        double tcx, double tcy, const double *tzc1, const double *tzc2, double dt,
                        const pwadv_peers *src, const pwadv_opts *opts, void *stream)
{
    int rc = check_peers(src, nx, ny, 16);
    if (rc) return rc;
    if (u == u_new || v == v_new || w == w_new)
        return set_error(PWADV_E_ARG, "fused step needs distinct (ping-pong) output buffers");
    return run_box(u, v, w, u_new, v_new, w_new, nx, ny, nz, tcx, tcy, tzc1, tzc2, dt, true, 1,
                   nx + 1, 1, ny + 1, opts, stream, src, true);
}

int pwadv_pull_halos_f64(double *u, double *v, double *w, int64_t nx, int64_t ny, int64_t nz,
                         const pwadv_peers *src, void *stream)
{
    int rc = check_dims(nx, ny, nz);
    if (rc) return rc;
    if ((rc = check_ptrs({u, v, w}))) return rc;
    if ((rc = check_peers(src, nx, ny, 8))) return rc;
    // the corner neighbours sit on my x neighbours' rows and my y neighbours' columns
    if (src->nx[PWADV_NB_XMYM] != src->nx[PWADV_NB_XM] || src->nx[PWADV_NB_XMYP] != src->nx[PWADV_NB_XM] ||
        src->nx[PWADV_NB_XPYM] != src->nx[PWADV_NB_XP] || src->nx[PWADV_NB_XPYP] != src->nx[PWADV_NB_XP] ||
        src->ny[PWADV_NB_XMYM] != src->ny[PWADV_NB_YM] || src->ny[PWADV_NB_XPYM] != src->ny[PWADV_NB_YM] ||
        src->ny[PWADV_NB_XMYP] != src->ny[PWADV_NB_YP] || src->ny[PWADV_NB_XPYP] != src->ny[PWADV_NB_YP])
        return set_error(PWADV_E_RANGE, "corner peer extents inconsistent with an x-y decomposition");
    return launch_pull_halos3(u, v, w, nx, ny, nz, src, (cudaStream_t)stream);
}

// Base address of the allocation containing `ptr`, through the driver's
// cuMemGetAddressRange (fetched with cudaGetDriverEntryPoint: no libcuda link).
static int allocation_base(const void *ptr, uintptr_t *base)
{
    typedef int (*range_fn)(unsigned long long *, size_t *, unsigned long long);
    static range_fn fn = nullptr;
    if (!fn) {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q);
        if (e != cudaSuccess || !f) return set_cuda_error("cudaGetDriverEntryPoint", e);
        fn = (range_fn)f;
    }
    unsigned long long b = 0;
    size_t sz = 0;
    if (fn(&b, &sz, (unsigned long long)(uintptr_t)ptr) != 0)
        return set_error(PWADV_E_ARG, "pointer %p is not device memory", ptr);
    *base = (uintptr_t)b;
    return PWADV_OK;
}

int pwadv_ipc_export(const void *dev_ptr, unsigned char handle[64], uint64_t *offset)
{
    if (!dev_ptr || !handle || !offset) return set_error(PWADV_E_NULL, "null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) <= 64, "IPC handle size");
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void *>(dev_ptr));
    if (e != cudaSuccess) return set_cuda_error("cudaIpcGetMemHandle", e);
    uintptr_t base = 0;
    int rc = allocation_base(dev_ptr, &base);
    if (rc) return rc;
    memset(handle, 0, 64);
    memcpy(handle, &h, sizeof(h));
    *offset = (uint64_t)((uintptr_t)dev_ptr - base);  // the handle names the whole allocation
    return PWADV_OK;
}

int pwadv_ipc_open(const unsigned char handle[64], uint64_t offset, void **dev_ptr)
{
    if (!handle || !dev_ptr) return set_error(PWADV_E_NULL, "null argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void *base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return set_cuda_error("cudaIpcOpenMemHandle", e);
    *dev_ptr = (void *)((char *)base + offset);
    return PWADV_OK;
}

int pwadv_ipc_close(void *dev_ptr, uint64_t offset)
{
    if (!dev_ptr) return set_error(PWADV_E_NULL, "null argument");
    cudaError_t e = cudaIpcCloseMemHandle((void *)((char *)dev_ptr - offset));
    if (e != cudaSuccess) return set_cuda_error("cudaIpcCloseMemHandle", e);
    return PWADV_OK;
}

int pwadv_describe_plan(int64_t nx, int64_t ny, int64_t nz, int64_t x0, int64_t x1, int64_t y0,
                        int64_t y1, const pwadv_opts *opts, int device, pwadv_plan_info *out)
{
    int rc = check_dims(nx, ny, nz);
    if (rc) return rc;
    if (!out) return set_error(PWADV_E_NULL, "null out");
    DeviceGuard g(device);
    const DeviceInfo *dev = device_info();
    if (!dev) return set_error(PWADV_E_CUDA, "no CUDA device");
    BoxLaunch L{};
    // nominal 256-byte aligned pointers: the plan only depends on alignment
    L.u = L.v = L.w = reinterpret_cast<const double *>(256);
    L.o0 = L.o1 = L.o2 = reinterpret_cast<double *>(256);
    L.nx = nx;
    L.ny = ny;
    L.nz = nz;
    L.x0 = x0;
    L.x1 = x1;
    L.y0 = y0;
    L.y1 = y1;
    L.flags = opts ? opts->flags : 0u;
    L.tile_j = opts ? opts->tile_j : 0;
    L.stages = opts ? opts->stages : 0;
    L.grid = opts ? opts->grid : 0;
    L.max_threads = opts ? opts->max_threads : 0;
    L.chunks = opts ? opts->chunks : 0;
    XmarchPlan p{};
    *out = pwadv_plan_info{};
    if (plan_xmarch(L, *dev, &p)) {
        out->kernel = p.ct ? 5 : (p.elem ? 4 : 1);
        out->tile_j = p.tj;
        out->threads_per_column = p.kp;
        out->stages = p.stages;
        out->threads = p.threads;
        out->grid = p.grid;
        out->smem_bytes = (int64_t)p.smem;
        out->strips = p.nstrips;
        out->chunks = p.nchunks;
        out->long_strips = (int32_t)p.nlong;
        out->spare_ctas = p.spare;
        out->main_chunk_planes = (int32_t)p.mlen;
    } else if (!(L.flags & (PWADV_FLAG_SIMPLE | PWADV_FLAG_RIM))) {
        out->kernel = 3;  // the general march (launch_box)
        out->threads = 128;
    } else {
        out->kernel = 2;
        out->threads = 256;
    }
    return PWADV_OK;
}

int pwadv_compute_block_f64(const double *const *roles, double *su, double *sv, double *sw,
                            int64_t ncols, int64_t nz, double tcx, double tcy,
                            const double *tzc1, const double *tzc2, uint32_t flags, void *stream)
{
    if (!roles) return set_error(PWADV_E_NULL, "null role table");
    if (ncols < 0) return set_error(PWADV_E_DIMS, "ncols %lld < 0", (long long)ncols);
    if (nz < 2) return set_error(PWADV_E_DIMS, "nz %lld < 2", (long long)nz);
    for (int m = 0; m < 17; ++m) {
        int rc = check_ptrs({roles[m]});
        if (rc) return rc;
    }
    int rc = check_ptrs({su, sv, sw, tzc1, tzc2});
    if (rc) return rc;
    return pwadv::launch_compute_block(roles, su, sv, sw, ncols, nz, tcx, tcy, tzc1, tzc2,
                                       (flags & PWADV_FLAG_FMA) != 0, (cudaStream_t)stream);
}

int pwadv_formula_f64(int32_t which, const double *const *args, const int64_t *strides, int64_t n,
                      int32_t top, double *out, uint32_t flags, void *stream)
{
    if (which < 0 || which > 2) return set_error(PWADV_E_ARG, "formula %d (0 su, 1 sv, 2 sw)", which);
    if (!args || !strides) return set_error(PWADV_E_NULL, "null argument table");
    if (n < 0) return set_error(PWADV_E_DIMS, "n %lld < 0", (long long)n);
    for (int m = 0; m < 19; ++m) {
        int rc = check_ptrs({args[m]});
        if (rc) return rc;
        if (strides[m] != 0 && strides[m] != 1)
            return set_error(PWADV_E_ARG, "argument %d stride %lld (0 or 1)", m, (long long)strides[m]);
    }
    int rc = check_ptrs({out});
    if (rc) return rc;
    return pwadv::launch_formula(which, args, strides, n, top, out, (flags & PWADV_FLAG_FMA) != 0,
                                 (cudaStream_t)stream);
}

int pwadv_wrap_halos_f64(double *f, int64_t nx, int64_t ny, int64_t nz, void *stream)
{
    int rc = check_dims(nx, ny, nz);
    if (rc) return rc;
    if ((rc = check_ptrs({f}))) return rc;
    return launch_wrap3(f, nullptr, nullptr, 1, nx, ny, nz, (cudaStream_t)stream);
}

int pwadv_wrap_halos3_f64(double *u, double *v, double *w, int64_t nx, int64_t ny, int64_t nz,
                          void *stream)
{
    int rc = check_dims(nx, ny, nz);
    if (rc) return rc;
    if ((rc = check_ptrs({u, v, w}))) return rc;
    return launch_wrap3(u, v, w, 3, nx, ny, nz, (cudaStream_t)stream);
}

int pwadv_wrap_axis3_f64(double *u, double *v, double *w, int64_t nx, int64_t ny, int64_t nz,
                         int32_t axis, void *stream)
{
    int rc = check_dims(nx, ny, nz);
    if (rc) return rc;
    if ((rc = check_ptrs({u, v, w}))) return rc;
    if (axis != 0 && axis != 1) return set_error(PWADV_E_ARG, "axis must be 0 or 1");
    return launch_wrap_axis3(u, v, w, nx, ny, nz, axis, (cudaStream_t)stream);
}

int pwadv_fill_f64(double *u, double *v, double *w, int64_t nx, int64_t ny, int64_t nz,
                   int32_t mode, uint64_t seed, double a, double b, double c, void *stream)
{
    int rc = check_dims(nx, ny, nz);
    if (rc) return rc;
    if ((rc = check_ptrs({u, v, w}))) return rc;
    if (mode < 0 || mode > 2) return set_error(PWADV_E_ARG, "unknown generator mode %d", mode);
    return launch_fill(u, v, w, nx, ny, nz, mode, seed, a, b, c, (cudaStream_t)stream);
}

int pwadv_fill_box_f64(double *u, double *v, double *w, int64_t nx, int64_t ny, int64_t nz,
                       int64_t gnx, int64_t gny, int64_t x_off, int64_t y_off, int32_t mode,
                       uint64_t seed, double a, double b, double c, void *stream)
{
    int rc = check_dims(nx, ny, nz);
    if (rc) return rc;
    if ((rc = check_ptrs({u, v, w}))) return rc;
    if (mode < 0 || mode > 2) return set_error(PWADV_E_ARG, "unknown generator mode %d", mode);
    if (x_off < 0 || y_off < 0 || x_off + nx > gnx || y_off + ny > gny)
        return set_error(PWADV_E_RANGE, "block [%lld,+%lld)x[%lld,+%lld) outside global %lldx%lld",
                         (long long)x_off, (long long)nx, (long long)y_off, (long long)ny,
                         (long long)gnx, (long long)gny);
    return launch_fill_box(u, v, w, nx, ny, nz, gnx, gny, x_off, y_off, mode, seed, a, b, c,
                           (cudaStream_t)stream);
}

static int face(const double *u, const double *v, const double *w, double *buf, int64_t nx,
                int64_t ny, int64_t nz, int axis, int64_t index, bool pack, void *stream)
{
    int rc = check_dims(nx, ny, nz);
    if (rc) return rc;
    if ((rc = check_ptrs({u, v, w, buf}))) return rc;
    const int64_t lim = axis == 0 ? nx + 1 : ny + 1;
    if (index < 0 || index > lim)
        return set_error(PWADV_E_RANGE, "face index %lld outside 0..%lld", (long long)index,
                         (long long)lim);
    return launch_face3(const_cast<double *>(u), const_cast<double *>(v), const_cast<double *>(w),
                        buf, nx, ny, nz, axis, index, pack, (cudaStream_t)stream);
}

int pwadv_pack_yface3_f64(const double *u, const double *v, const double *w, double *buf,
                          int64_t nx, int64_t ny, int64_t nz, int64_t j, void *stream)
{
    return face(u, v, w, buf, nx, ny, nz, 1, j, true, stream);
}

int pwadv_unpack_yface3_f64(double *u, double *v, double *w, const double *buf, int64_t nx,
                            int64_t ny, int64_t nz, int64_t j, void *stream)
{
    return face(u, v, w, const_cast<double *>(buf), nx, ny, nz, 1, j, false, stream);
}

int pwadv_pack_xface3_f64(const double *u, const double *v, const double *w, double *buf,
                          int64_t nx, int64_t ny, int64_t nz, int64_t i, void *stream)
{
    return face(u, v, w, buf, nx, ny, nz, 0, i, true, stream);
}

int pwadv_unpack_xface3_f64(double *u, double *v, double *w, const double *buf, int64_t nx,
                            int64_t ny, int64_t nz, int64_t i, void *stream)
{
    return face(u, v, w, const_cast<double *>(buf), nx, ny, nz, 0, i, false, stream);
}

int pwadv_pack_faces3_f64(const double *u, const double *v, const double *w, double *buf_lo,
                          double *buf_hi, int64_t nx, int64_t ny, int64_t nz, int32_t axis,
                          void *stream)
{
    int rc = check_dims(nx, ny, nz);
    if (rc) return rc;
    if ((rc = check_ptrs({u, v, w, buf_lo, buf_hi}))) return rc;
    if (axis != 0 && axis != 1) return set_error(PWADV_E_ARG, "axis must be 0 or 1");
    const int64_t n = axis == 0 ? nx : ny;
    return launch_faces3(const_cast<double *>(u), const_cast<double *>(v), const_cast<double *>(w),
                         buf_lo, buf_hi, nx, ny, nz, axis, 1, n, true, (cudaStream_t)stream);
}

int pwadv_unpack_faces3_f64(double *u, double *v, double *w, const double *buf_lo,
                            const double *buf_hi, int64_t nx, int64_t ny, int64_t nz, int32_t axis,
                            void *stream)
{
    int rc = check_dims(nx, ny, nz);
    if (rc) return rc;
    if ((rc = check_ptrs({u, v, w, buf_lo, buf_hi}))) return rc;
    if (axis != 0 && axis != 1) return set_error(PWADV_E_ARG, "axis must be 0 or 1");
    const int64_t n = axis == 0 ? nx : ny;
    return launch_faces3(u, v, w, const_cast<double *>(buf_lo), const_cast<double *>(buf_hi), nx, ny,
                         nz, axis, 0, n + 1, false, (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------
// Automatic X-slab chunk count for the host-buffer path (measured on B200,
// tools/e2e_sweep.py, tools/pcie.py): a single synchronous call needs ~16
// chunks for its H2D / K1 / D2H pipeline to fill; a stream of submissions
// already overlaps one grid's H2D with the previous grid's D2H, so there the
// copies only need to stay large (~64 MiB per field and chunk).
static int32_t auto_chunks(int64_t nx, int64_t plane_doubles, bool streamed)
{
    const double field_bytes = (double)(nx + 2) * (double)plane_doubles * sizeof(double);
    int64_t n;
    if (streamed) n = (int64_t)(field_bytes / (64.0 * 1024 * 1024) + 0.5);
    else n = field_bytes < 32.0 * 1024 * 1024 ? 1 : 16;
    if (n < 1) n = 1;
    if (n > 16) n = 16;
    if (n > nx) n = nx;
    return (int32_t)n;
}

// host-buffer context: pipelined H2D / K1 / D2H over X-slab chunks

namespace pwadv {

// Host copy with non-temporal (streaming) stores: the destination lines are
// written without being read first (no read-for-ownership), a third less
// DRAM traffic than memcpy's cached stores for a staging buffer that is
// read next by the DMA engine, not by the CPU.
__attribute__((target("avx2"))) static void stream_copy_avx2(void *dst, const void *src, size_t n)
{
    char *d = (char *)dst;
    const char *s = (const char *)src;
    const size_t head = (64 - ((uintptr_t)d & 63)) & 63;
    if (n < head + 256) {
        memcpy(d, s, n);
        return;
    }
    memcpy(d, s, head);
    d += head;
    s += head;
    n -= head;
    const size_t body = n & ~(size_t)127;
    for (size_t o = 0; o < body; o += 128) {
        const __m256i a0 = _mm256_loadu_si256((const __m256i *)(s + o));
        const __m256i a1 = _mm256_loadu_si256((const __m256i *)(s + o + 32));
        const __m256i a2 = _mm256_loadu_si256((const __m256i *)(s + o + 64));
        const __m256i a3 = _mm256_loadu_si256((const __m256i *)(s + o + 96));
        _mm256_stream_si256((__m256i *)(d + o), a0);
        _mm256_stream_si256((__m256i *)(d + o + 32), a1);
        _mm256_stream_si256((__m256i *)(d + o + 64), a2);
        _mm256_stream_si256((__m256i *)(d + o + 96), a3);
    }
    _mm_sfence();
    memcpy(d + body, s + body, n - body);
}

static void host_copy(void *dst, const void *src, size_t n)
{
    static const bool avx2 = __builtin_cpu_supports("avx2");
    if (avx2) stream_copy_avx2(dst, src, n);
    else memcpy(dst, src, n);
}

// Small persistent host thread pool: one memcpy split across the workers
// (pageable <-> pinned staging for host buffers that are not page-locked).
class CopyPool {
  public:
    explicit CopyPool(int n) : stop_(false), pending_(0)
    {
        for (int i = 0; i < n; ++i) workers_.emplace_back([this] { run(); });
    }
    ~CopyPool()
    {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto &t : workers_) t.join();
    }
    struct Copy {
        void *dst;
        const void *src;
        size_t bytes;
    };
    // All copies of a batch split into ~1 MiB pieces spread over the workers
    // and the calling thread; returns when every piece is done.
    void memcpy_batch(const Copy *cps, int n)
    {
        constexpr size_t kPiece = size_t(1) << 20;
        std::vector<Copy> pieces;
        for (int i = 0; i < n; ++i)
            for (size_t off = 0; off < cps[i].bytes; off += kPiece)
                pieces.push_back({(char *)cps[i].dst + off, (const char *)cps[i].src + off,
                                  std::min(kPiece, cps[i].bytes - off)});
        if (pieces.empty()) return;
        const size_t nt = workers_.size() + 1;
        const size_t per = (pieces.size() + nt - 1) / nt;
        auto job = [pieces, per](size_t t) {
            for (size_t k = t * per; k < std::min(pieces.size(), (t + 1) * per); ++k)
                host_copy(pieces[k].dst, pieces[k].src, pieces[k].bytes);
        };
        const size_t used = (pieces.size() + per - 1) / per;
        {
            std::lock_guard<std::mutex> lk(mu_);
            for (size_t t = 1; t < used; ++t) {
                tasks_.push_back([job, t] { job(t); });
                ++pending_;
            }
        }
        cv_.notify_all();
        job(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [this] { return pending_ == 0; });
    }

  private:
    void run()
    {
        for (;;) {
            std::function<void()> job;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [this] { return stop_ || !tasks_.empty(); });
                if (stop_ && tasks_.empty()) return;
                job = std::move(tasks_.front());
                tasks_.pop_front();
            }
            job();
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (--pending_ == 0) done_.notify_all();
            }
        }
    }
    std::vector<std::thread> workers_;
    std::deque<std::function<void()>> tasks_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    bool stop_;
    int pending_;
};

}  // namespace pwadv

struct pwadv_ctx {
    int device;
    int64_t nx, ny, nz;
    double *d_in[3];
    double *d_out[3];
    double *d_tz;
    cudaStream_t s_h2d, s_cmp, s_d2h;
    std::vector<cudaEvent_t> ev_in, ev_cmp;
    uint64_t last_h2d, last_d2h;
    // pageable-host staging (created on first use)
    pwadv::CopyPool *pool;
    double *pin_in[2], *pin_out[2];
    int64_t pin_planes;  // planes per field a staging buffer holds
    cudaEvent_t ev_h2d[2], ev_d2h[2];
    // asynchronous submissions alternate between two device buffer sets
    double *set2_in[3], *set2_out[3], *set2_tz;  // set 1 (lazily allocated)
    cudaEvent_t ev_in_free[2], ev_out_free[2];   // set s's inputs / outputs no longer in use
    bool set_used[2];
    uint64_t submits;
};


int pwadv_ctx_create(pwadv_ctx **out, int device, int64_t nx, int64_t ny, int64_t nz)
{
    if (!out) return set_error(PWADV_E_NULL, "null ctx out pointer");
    *out = nullptr;
    int rc = check_dims(nx, ny, nz);
    if (rc) return rc;
    DeviceGuard g(device);
    pwadv_ctx *c = new pwadv_ctx();
    c->device = device;
    c->nx = nx;
    c->ny = ny;
    c->nz = nz;
    const size_t n = (size_t)(nx + 2) * (ny + 2) * nz;
    cudaError_t e = cudaSuccess;
    for (int m = 0; m < 3 && e == cudaSuccess; ++m) e = cudaMalloc(&c->d_in[m], n * sizeof(double));
    for (int m = 0; m < 3 && e == cudaSuccess; ++m) e = cudaMalloc(&c->d_out[m], n * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&c->d_tz, 2 * (size_t)nz * sizeof(double));
    for (int m = 0; m < 3 && e == cudaSuccess; ++m) e = cudaMemset(c->d_out[m], 0, n * sizeof(double));
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->s_cmp, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        pwadv_ctx_destroy(c);
        return set_cuda_error("pwadv_ctx_create", e);
    }
    *out = c;
    return PWADV_OK;
}

int pwadv_ctx_destroy(pwadv_ctx *c)
{
    if (!c) return PWADV_OK;
    DeviceGuard g(c->device);
    for (int m = 0; m < 3; ++m) {
        if (c->d_in[m]) cudaFree(c->d_in[m]);
        if (c->d_out[m]) cudaFree(c->d_out[m]);
    }
    if (c->d_tz) cudaFree(c->d_tz);
    for (int b = 0; b < 2; ++b) {
        if (c->pin_in[b]) cudaFreeHost(c->pin_in[b]);
        if (c->pin_out[b]) cudaFreeHost(c->pin_out[b]);
        if (c->ev_h2d[b]) cudaEventDestroy(c->ev_h2d[b]);
        if (c->ev_d2h[b]) cudaEventDestroy(c->ev_d2h[b]);
    }
    delete c->pool;
    for (int m = 0; m < 3; ++m) {
        if (c->set2_in[m]) cudaFree(c->set2_in[m]);
        if (c->set2_out[m]) cudaFree(c->set2_out[m]);
    }
    if (c->set2_tz) cudaFree(c->set2_tz);
    for (int b = 0; b < 2; ++b) {
        if (c->ev_in_free[b]) cudaEventDestroy(c->ev_in_free[b]);
        if (c->ev_out_free[b]) cudaEventDestroy(c->ev_out_free[b]);
    }
    if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
    if (c->s_cmp) cudaStreamDestroy(c->s_cmp);
    if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
    for (auto ev : c->ev_in) cudaEventDestroy(ev);
    for (auto ev : c->ev_cmp) cudaEventDestroy(ev);
    delete c;
    return PWADV_OK;
}

int pwadv_ctx_last_bytes(const pwadv_ctx *c, uint64_t *h2d, uint64_t *d2h)
{
    if (!c || !h2d || !d2h) return set_error(PWADV_E_NULL, "null argument");
    *h2d = c->last_h2d;
    *d2h = c->last_d2h;
    return PWADV_OK;
}

static bool is_pinned(const void *p)
{
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return attr.type == cudaMemoryTypeHost;
}

// Host buffers that are not page-locked: stream them through double-buffered
// pinned staging. Per chunk the host threads copy the inputs into staging
// while the previous chunk's H2D, K1 and D2H run, then copy the previous
// chunk's outputs out of staging.
// Inputs or outputs in pageable memory: the pageable side goes through two
// page-locked staging buffers filled / drained by the host copy pool while
// the DMA engines work on the other buffer; a page-locked side is copied
// directly (in_direct / out_direct).
static int advect_host_staged(pwadv_ctx *c, const double *const hin[3], double *const hout[3],
                              double tcx, double tcy, const pwadv_opts *o, uint64_t *h2d,
                              uint64_t *d2h, bool in_direct, bool out_direct)
{
    const int64_t nx = c->nx, ny = c->ny, nz = c->nz;
    const size_t plane = (size_t)(ny + 2) * nz;
    const size_t pb = plane * sizeof(double);
    cudaError_t e;
    if (!c->pool) {
#ifndef PWADV_STAGING_MB
#define PWADV_STAGING_MB 48
#endif
        const int64_t target = (int64_t)((size_t)PWADV_STAGING_MB << 20) / (int64_t)(3 * pb);  // per buffer
        c->pin_planes = std::max<int64_t>(3, std::min<int64_t>(target, nx + 2));
        for (int b = 0; b < 2; ++b) {
            e = cudaHostAlloc(&c->pin_in[b], 3 * c->pin_planes * pb, cudaHostAllocDefault);
            if (e == cudaSuccess) e = cudaHostAlloc(&c->pin_out[b], 3 * c->pin_planes * pb, cudaHostAllocDefault);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_h2d[b], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_d2h[b], cudaEventDisableTiming);
            if (e != cudaSuccess) return set_cuda_error("staging buffers", e);
        }
        const unsigned hc = std::thread::hardware_concurrency();
        c->pool = new pwadv::CopyPool((int)std::min(15u, hc > 1 ? hc - 1 : 1u));
    }
    const int64_t P = c->pin_planes;
    // output chunk of at most P-2 planes so its input range (+1 plane each side) fits
    const int64_t per = std::max<int64_t>(1, P - 2);
    const int chunks = (int)((nx + per - 1) / per);
    while ((int)c->ev_cmp.size() < chunks) {
        cudaEvent_t a;
        cudaEventCreateWithFlags(&a, cudaEventDisableTiming);
        c->ev_cmp.push_back(a);
    }
    int64_t copied = 0;
    int64_t prev_o0 = 0, prev_o1 = 0;
    auto drain = [&](int ch, int64_t o0, int64_t o1) -> int {
        if (out_direct) return PWADV_OK;
        const int b = ch & 1;
        cudaError_t err = cudaEventSynchronize(c->ev_d2h[b]);
        if (err != cudaSuccess) return set_cuda_error("D2H wait", err);
        pwadv::CopyPool::Copy cps[3];
        for (int m = 0; m < 3; ++m)
            cps[m] = {hout[m] + o0 * plane, c->pin_out[b] + m * P * plane, (size_t)(o1 - o0) * pb};
        c->pool->memcpy_batch(cps, 3);
        return PWADV_OK;
    };
    for (int ch = 0; ch < chunks; ++ch) {
        const int b = ch & 1;
        const int64_t x0 = 1 + (int64_t)ch * per;
        const int64_t x1 = std::min<int64_t>(nx + 1, x0 + per);
        const int64_t need = (ch == chunks - 1) ? nx + 2 : x1 + 1;
        if (ch >= 2 && !in_direct) {
            e = cudaEventSynchronize(c->ev_h2d[b]);  // staging b no longer read by its H2D
            if (e != cudaSuccess) return set_cuda_error("H2D wait", e);
        }
        const int64_t n_in = need - copied;
        if (!in_direct) {
            pwadv::CopyPool::Copy cps[3];
            for (int m = 0; m < 3; ++m)
                cps[m] = {c->pin_in[b] + m * P * plane, hin[m] + copied * plane, (size_t)n_in * pb};
            c->pool->memcpy_batch(cps, 3);
        }
        for (int m = 0; m < 3; ++m) {
            const double *src = in_direct ? hin[m] + copied * plane : c->pin_in[b] + m * P * plane;
            e = cudaMemcpyAsync(c->d_in[m] + copied * plane, src, n_in * pb, cudaMemcpyHostToDevice,
                                c->s_h2d);
            if (e != cudaSuccess) return set_cuda_error("H2D", e);
        }
        *h2d += 3 * (uint64_t)n_in * pb;
        copied = need;
        cudaEventRecord(c->ev_h2d[b], c->s_h2d);
        cudaStreamWaitEvent(c->s_cmp, c->ev_h2d[b], 0);
        int rc = pwadv_advect_box_f64(c->d_in[0], c->d_in[1], c->d_in[2], c->d_out[0], c->d_out[1],
                                      c->d_out[2], nx, ny, nz, tcx, tcy, c->d_tz, c->d_tz + nz, x0, x1,
                                      1, ny + 1, o, c->s_cmp);
        if (rc) return rc;
        cudaEventRecord(c->ev_cmp[ch], c->s_cmp);
        cudaStreamWaitEvent(c->s_d2h, c->ev_cmp[ch], 0);
        const int64_t o0 = (ch == 0) ? 0 : x0;
        const int64_t o1 = (ch == chunks - 1) ? nx + 2 : x1;
        for (int m = 0; m < 3; ++m) {
            double *dst = out_direct ? hout[m] + o0 * plane : c->pin_out[b] + m * P * plane;
            e = cudaMemcpyAsync(dst, c->d_out[m] + o0 * plane, (o1 - o0) * pb, cudaMemcpyDeviceToHost,
                                c->s_d2h);
            if (e != cudaSuccess) return set_cuda_error("D2H", e);
        }
        *d2h += 3 * (uint64_t)(o1 - o0) * pb;
        cudaEventRecord(c->ev_d2h[b], c->s_d2h);
        if (ch >= 1 && (rc = drain(ch - 1, prev_o0, prev_o1))) return rc;
        prev_o0 = o0;
        prev_o1 = o1;
    }
    int rc = drain(chunks - 1, prev_o0, prev_o1);
    if (rc == PWADV_OK && out_direct) {
        e = cudaStreamSynchronize(c->s_d2h);
        if (e != cudaSuccess) return set_cuda_error("D2H wait", e);
    }
    return rc;
}

// Page-locked host buffers: H2D, K1 and D2H of X-slab chunks on three streams
// into buffer set `set`; returns once everything is enqueued. Waits (on the
// device) until the set's previous use has released its inputs / outputs.
// Interior plane where chunk `ch` of `chunks` starts (1-based). Uniform: a
// short last chunk to shorten the drain measured no faster (tools/e2e_sweep.py).
static int64_t chunk_edge(int64_t nx, int chunks, int ch)
{
    return 1 + nx * (ch < chunks ? ch : chunks) / chunks;
}

static int enqueue_pinned(pwadv_ctx *c, int set, const double *const hin[3], double *const hout[3],
                          double tcx, double tcy, int chunks, const pwadv_opts *o, uint64_t *h2d,
                          uint64_t *d2h)
{
    const int64_t nx = c->nx, ny = c->ny, nz = c->nz;
    const size_t plane = (size_t)(ny + 2) * nz;
    const size_t pb = plane * sizeof(double);
    double *din[3], *dout[3];
    for (int m = 0; m < 3; ++m) {
        din[m] = set ? c->set2_in[m] : c->d_in[m];
        dout[m] = set ? c->set2_out[m] : c->d_out[m];
    }
    const double *tz = set ? c->set2_tz : c->d_tz;
    while ((int)c->ev_in.size() < chunks) {
        cudaEvent_t a, b;
        cudaEventCreateWithFlags(&a, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&b, cudaEventDisableTiming);
        c->ev_in.push_back(a);
        c->ev_cmp.push_back(b);
    }
    if (!c->ev_in_free[set]) {
        cudaEventCreateWithFlags(&c->ev_in_free[set], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&c->ev_out_free[set], cudaEventDisableTiming);
    }
    if (c->set_used[set]) {
        cudaStreamWaitEvent(c->s_h2d, c->ev_in_free[set], 0);   // kernels done reading inputs
        cudaStreamWaitEvent(c->s_cmp, c->ev_out_free[set], 0);  // D2H done reading outputs
    }
    cudaError_t e;
    int64_t copied = 0;  // input planes [0, copied) are on the device
    for (int ch = 0; ch < chunks; ++ch) {
        const int64_t x0 = chunk_edge(nx, chunks, ch), x1 = chunk_edge(nx, chunks, ch + 1);
        const int64_t need = (ch == chunks - 1) ? nx + 2 : x1 + 1;  // planes up to x1 inclusive
        if (need > copied) {
            for (int m = 0; m < 3; ++m) {
                e = cudaMemcpyAsync(din[m] + copied * plane, hin[m] + copied * plane,
                                    (need - copied) * pb, cudaMemcpyHostToDevice, c->s_h2d);
                if (e != cudaSuccess) return set_cuda_error("H2D", e);
            }
            *h2d += 3 * (uint64_t)(need - copied) * pb;
            copied = need;
        }
        cudaEventRecord(c->ev_in[ch], c->s_h2d);
        cudaStreamWaitEvent(c->s_cmp, c->ev_in[ch], 0);
        int rc = pwadv_advect_box_f64(din[0], din[1], din[2], dout[0], dout[1], dout[2], nx, ny, nz,
                                      tcx, tcy, tz, tz + nz, x0, x1, 1, ny + 1, o, c->s_cmp);
        if (rc) return rc;
        cudaEventRecord(c->ev_cmp[ch], c->s_cmp);
        cudaStreamWaitEvent(c->s_d2h, c->ev_cmp[ch], 0);
        // output planes of this chunk; the first/last chunk also returns the
        // all-zero halo planes 0 / nx+1 so host outputs match zeros_sources
        const int64_t o0 = (ch == 0) ? 0 : x0;
        const int64_t o1 = (ch == chunks - 1) ? nx + 2 : x1;
        for (int m = 0; m < 3; ++m) {
            e = cudaMemcpyAsync(hout[m] + o0 * plane, dout[m] + o0 * plane, (o1 - o0) * pb,
                                cudaMemcpyDeviceToHost, c->s_d2h);
            if (e != cudaSuccess) return set_cuda_error("D2H", e);
        }
        *d2h += 3 * (uint64_t)(o1 - o0) * pb;
    }
    cudaEventRecord(c->ev_in_free[set], c->s_cmp);
    cudaEventRecord(c->ev_out_free[set], c->s_d2h);
    c->set_used[set] = true;
    return PWADV_OK;
}

int pwadv_ctx_advect_host(pwadv_ctx *c, const double *u, const double *v, const double *w,
                          double *su, double *sv, double *sw, double tcx, double tcy,
                          const double *tzc1, const double *tzc2, int32_t chunks,
                          const pwadv_opts *opts)
{
    if (!c) return set_error(PWADV_E_NULL, "null ctx");
    if (!u || !v || !w || !su || !sv || !sw || !tzc1 || !tzc2)
        return set_error(PWADV_E_NULL, "null pointer argument");
    DeviceGuard g(c->device);
    const int64_t nx = c->nx, nz = c->nz;
    if (chunks < 1) chunks = auto_chunks(nx, (c->ny + 2) * nz, false);
    if (chunks > nx) chunks = (int32_t)nx;
    const double *hin[3] = {u, v, w};
    double *hout[3] = {su, sv, sw};
    uint64_t h2d = 0, d2h = 0;
    cudaError_t e;
    if (c->set_used[0]) cudaStreamWaitEvent(c->s_h2d, c->ev_in_free[0], 0);
    e = cudaMemcpyAsync(c->d_tz, tzc1, nz * sizeof(double), cudaMemcpyHostToDevice, c->s_h2d);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(c->d_tz + nz, tzc2, nz * sizeof(double), cudaMemcpyHostToDevice,
                            c->s_h2d);
    if (e != cudaSuccess) return set_cuda_error("coefficient upload", e);
    h2d += 2 * nz * sizeof(double);
    pwadv_opts o = opts ? *opts : pwadv_opts{0u, 0, 0, 0, 0, 0, nullptr};
    bool in_pinned = true, out_pinned = true;
    for (int m = 0; m < 3; ++m) {
        in_pinned = in_pinned && is_pinned(hin[m]);
        out_pinned = out_pinned && is_pinned(hout[m]);
    }
    if (!(in_pinned && out_pinned)) {
        if (c->set_used[0]) {  // an earlier asynchronous submission may still use set 0
            cudaStreamWaitEvent(c->s_h2d, c->ev_in_free[0], 0);
            cudaStreamWaitEvent(c->s_cmp, c->ev_out_free[0], 0);
        }
        uint64_t sh2d = 0, sd2h = 0;
        int rc = advect_host_staged(c, hin, hout, tcx, tcy, &o, &sh2d, &sd2h, in_pinned, out_pinned);
        if (rc) return rc;
        c->last_h2d = h2d + sh2d;
        c->last_d2h = sd2h;
        return PWADV_OK;
    }
    int rc = enqueue_pinned(c, 0, hin, hout, tcx, tcy, chunks, &o, &h2d, &d2h);
    if (rc) return rc;
    e = cudaStreamSynchronize(c->s_d2h);
    if (e != cudaSuccess) return set_cuda_error("ctx_advect_host sync", e);
    c->last_h2d = h2d;
    c->last_d2h = d2h;
    return PWADV_OK;
}

int pwadv_ctx_submit_host(pwadv_ctx *c, const double *u, const double *v, const double *w,
                          double *su, double *sv, double *sw, double tcx, double tcy,
                          const double *tzc1, const double *tzc2, int32_t chunks,
                          const pwadv_opts *opts)
{
    if (!c) return set_error(PWADV_E_NULL, "null ctx");
    if (!u || !v || !w || !su || !sv || !sw || !tzc1 || !tzc2)
        return set_error(PWADV_E_NULL, "null pointer argument");
    DeviceGuard g(c->device);
    const double *hin[3] = {u, v, w};
    double *hout[3] = {su, sv, sw};
    for (int m = 0; m < 3; ++m)
        if (!is_pinned(hin[m]) || !is_pinned(hout[m]))
            return set_error(PWADV_E_ARG, "asynchronous submission needs page-locked host buffers");
    const int64_t nx = c->nx, ny = c->ny, nz = c->nz;
    cudaError_t e = cudaSuccess;
    if (!c->set2_in[0]) {
        const size_t n = (size_t)(nx + 2) * (ny + 2) * nz;
        for (int m = 0; m < 3 && e == cudaSuccess; ++m) e = cudaMalloc(&c->set2_in[m], n * sizeof(double));
        for (int m = 0; m < 3 && e == cudaSuccess; ++m) e = cudaMalloc(&c->set2_out[m], n * sizeof(double));
        if (e == cudaSuccess) e = cudaMalloc(&c->set2_tz, 2 * (size_t)nz * sizeof(double));
        for (int m = 0; m < 3 && e == cudaSuccess; ++m) e = cudaMemset(c->set2_out[m], 0, n * sizeof(double));
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) return set_cuda_error("second buffer set", e);
    }
    if (chunks < 1) chunks = auto_chunks(nx, (c->ny + 2) * nz, true);
    if (chunks > nx) chunks = (int32_t)nx;
    const int set = (int)(c->submits & 1);
    ++c->submits;
    pwadv_opts o = opts ? *opts : pwadv_opts{0u, 0, 0, 0, 0, 0, nullptr};
    uint64_t h2d = 0, d2h = 0;
    double *tz = set ? c->set2_tz : c->d_tz;
    if (c->set_used[set]) cudaStreamWaitEvent(c->s_h2d, c->ev_in_free[set], 0);
    e = cudaMemcpyAsync(tz, tzc1, nz * sizeof(double), cudaMemcpyHostToDevice, c->s_h2d);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(tz + nz, tzc2, nz * sizeof(double), cudaMemcpyHostToDevice, c->s_h2d);
    if (e != cudaSuccess) return set_cuda_error("coefficient upload", e);
    h2d += 2 * nz * sizeof(double);
    int rc = enqueue_pinned(c, set, hin, hout, tcx, tcy, chunks, &o, &h2d, &d2h);
    if (rc) return rc;
    c->last_h2d = h2d;
    c->last_d2h = d2h;
    return PWADV_OK;
}

int pwadv_ctx_sync(pwadv_ctx *c)
{
    if (!c) return set_error(PWADV_E_NULL, "null ctx");
    DeviceGuard g(c->device);
    cudaError_t e = cudaStreamSynchronize(c->s_d2h);
    if (e != cudaSuccess) return set_cuda_error("ctx_sync", e);
    return PWADV_OK;
}

}  // extern "C"
