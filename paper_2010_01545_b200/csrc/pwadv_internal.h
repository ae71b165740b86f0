// pwadv_internal.h — shared declarations between the libpwadv translation units.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/pwadv.h"

namespace pwadv {

struct DeviceInfo {
    int device;
    int sms;
    int smem_optin;
};

// One K1/K4 launch over an interior box.
struct BoxLaunch {
    const double *u, *v, *w;
    double *o0, *o1, *o2;
    const double *tzc1, *tzc2;
    int64_t nx, ny, nz;
    double tcx, tcy, dt;
    int64_t x0, x1, y0, y1;
    bool step;
    uint32_t flags;
    int tile_j, stages, grid, max_threads, chunks;
    void *trace;
    const pwadv_peers *peers;  // fused step: push boundary values into these halos; with
                               // pull: the neighbours' current buffers to load halos from
    bool pull = false;
};

struct XmarchPlan {
    int maxt, tj, kp, stages, threads, grid, nchunks;
    size_t smem;
    int64_t nstrips;
    int64_t rounds;  // units per CTA (the kernel's unit table holds kMaxUnitsPerCta)
    int64_t nlong;   // strips run as whole-X units (full rounds)
    int elem;        // 1: unaligned tile runs (UA kernels: odd nz, 8-byte alignment)
    int rot, nface, nchf;  // halo pull: strip rotation and the y-face strips' chunking
    int spare;             // spare-tail plan: CTAs running the strips' tail chunks (0 = off)
    int64_t mlen;          //   planes per main chunk (nchunks main chunks per strip)
    int ct = 0;            // 1: column-tile X-march (k_advect_ctile): tj x kt tiles
    int kt = 0;            //   levels per slab
    int nslab = 1;         //   slabs per column (nstrips counts y-strips x slabs)
};

// cached attributes of the current device (lazily filled, thread-safe)
const DeviceInfo *device_info();

int set_error(int code, const char *fmt, ...);
int set_cuda_error(const char *what, cudaError_t e);
void count_launch();

bool plan_xmarch(const BoxLaunch &L, const DeviceInfo &dev, XmarchPlan *p);
int launch_compute_block(const double *const roles[17], double *su, double *sv, double *sw,
                         int64_t ncols, int64_t nz, double tcx, double tcy, const double *tzc1,
                         const double *tzc2, bool fma, cudaStream_t s);
int launch_formula(int which, const double *const args[19], const int64_t strides[19], int64_t n,
                   int top, double *out, bool fma, cudaStream_t s);
int launch_box(const BoxLaunch &L, cudaStream_t stream);

// auxiliary kernels (pwadv_aux.cu)
int launch_wrap3(double *u, double *v, double *w, int nf, int64_t nx, int64_t ny, int64_t nz,
                 cudaStream_t s);
int launch_pull_halos3(double *u, double *v, double *w, int64_t nx, int64_t ny, int64_t nz,
                       const pwadv_peers *src, cudaStream_t s);
int launch_wrap_axis3(double *u, double *v, double *w, int64_t nx, int64_t ny, int64_t nz,
                      int axis, cudaStream_t s);
int launch_fill(double *u, double *v, double *w, int64_t nx, int64_t ny, int64_t nz, int mode,
                uint64_t seed, double a, double b, double c, cudaStream_t s);
int launch_fill_box(double *u, double *v, double *w, int64_t nx, int64_t ny, int64_t nz,
                    int64_t gnx, int64_t gny, int64_t x_off, int64_t y_off, int mode, uint64_t seed,
                    double a, double b, double c, cudaStream_t s);
int launch_faces3(double *u, double *v, double *w, double *buf_a, double *buf_b, int64_t nx,
                  int64_t ny, int64_t nz, int axis, int64_t ia, int64_t ib, bool pack, cudaStream_t s);
int launch_face3(double *u, double *v, double *w, double *buf, int64_t nx, int64_t ny,
                 int64_t nz, int axis, int64_t index, bool pack, cudaStream_t s);

}  // namespace pwadv
