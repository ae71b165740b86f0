// pwadv_aux.cu — K2 periodic halo wrap, K5 device field generator, halo-face
// pack/unpack for the multi-GPU exchange.
//
// K2 reproduces wrap_halos (pkg/src/pwadvect/grid.py:203-208): X halos first,
// then Y halos over all i including the X halos, so corners are doubly
// periodic (docs/model-notes.md §1). Because every halo cell is a copy of an
// interior cell, the result equals "each halo cell (i, j) takes interior cell
// (wrap(i), wrap(j))", which needs no ordering and runs as one launch.
//
// K5 reproduces lcg_doubles + fill_fields (grid.py:164-239) bit-for-bit: the
// Knuth MMIX LCG is pure uint64 arithmetic with an O(log n) skip-ahead, so
// every thread can start at its own stream offset.
#include "pwadv_device.cuh"
#include "pwadv_internal.h"

namespace pwadv {

static constexpr uint64_t kLcgMult = 6364136223846793005ULL;
static constexpr uint64_t kLcgInc = 1442695040888963407ULL;

// ---------------------------------------------------------------------------
// K2

__device__ __forceinline__ int64_t halo_col(int64_t h, int64_t nx, int64_t ny, int64_t *i)
{
    // enumerates halo columns: i=0 plane, i=nx+1 plane (all j), then j=0 and
    // j=ny+1 for interior i
    const int64_t ny2 = ny + 2;
    if (h < ny2) {
        *i = 0;
        return h;
    }
    h -= ny2;
    if (h < ny2) {
        *i = nx + 1;
        return h;
    }
    h -= ny2;
    if (h < nx) {
        *i = 1 + h;
        return 0;
    }
    *i = 1 + (h - nx);
    return ny + 1;
}

__global__ void k_wrap3(double *f0, double *f1, double *f2, int nf, int64_t nx, int64_t ny,
                        int64_t nz)
{
    const int64_t ncols = 2 * (ny + 2) + 2 * nx;
    const int64_t total = ncols * nz;
    double *fs[3] = {f0, f1, f2};
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = idx % nz, h = idx / nz;
        int64_t i;
        const int64_t j = halo_col(h, nx, ny, &i);
        const int64_t si = i == 0 ? nx : (i == nx + 1 ? 1 : i);
        const int64_t sj = j == 0 ? ny : (j == ny + 1 ? 1 : j);
        const int64_t dst = (i * (ny + 2) + j) * nz + k;
        const int64_t src = (si * (ny + 2) + sj) * nz + k;
        for (int m = 0; m < nf; ++m) fs[m][dst] = fs[m][src];
    }
}

// K2p — the halo wrap of one block of an x-y decomposition, gathered from
// the neighbours' buffers (peer loads over NVLink for another GPU's block):
// every halo cell (i, j) of this block takes the neighbour's interior cell
// that a two-phase periodic exchange (wrap_halos, grid.py:203-208: the X pass,
// then the Y pass over the X halos) would have delivered — x-halo planes from
// XM's last / XP's first interior plane, y-halo columns from YM's last / YP's
// first interior column, the four corner columns from the diagonal
// neighbours. Along an undivided axis the neighbour is this block itself and
// the copy is the plain wrap. Only this block's halos are written, only
// interiors are read: concurrent gathers of neighbouring blocks never touch
// the same cell.
struct PeerSrc {
    const double *f[3][8];
    int64_t nx[8], ny[8];
};

__global__ void k_pull_halos3(double *f0, double *f1, double *f2, int64_t nx, int64_t ny,
                              int64_t nz, const __grid_constant__ PeerSrc p)
{
    const int64_t ncols = 2 * (ny + 2) + 2 * nx;
    const int64_t total = ncols * nz;
    double *fs[3] = {f0, f1, f2};
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = idx % nz, h = idx / nz;
        int64_t i;
        const int64_t j = halo_col(h, nx, ny, &i);
        const int xs = i == 0 ? -1 : (i == nx + 1 ? 1 : 0);
        const int ys = j == 0 ? -1 : (j == ny + 1 ? 1 : 0);
        int d;
        if (xs < 0) d = ys < 0 ? PWADV_NB_XMYM : (ys > 0 ? PWADV_NB_XMYP : PWADV_NB_XM);
        else if (xs > 0) d = ys < 0 ? PWADV_NB_XPYM : (ys > 0 ? PWADV_NB_XPYP : PWADV_NB_XP);
        else d = ys < 0 ? PWADV_NB_YM : PWADV_NB_YP;
        const int64_t si = xs < 0 ? p.nx[d] : (xs > 0 ? 1 : i);
        const int64_t sj = ys < 0 ? p.ny[d] : (ys > 0 ? 1 : j);
        const int64_t dst = (i * (ny + 2) + j) * nz + k;
        const int64_t src = (si * (p.ny[d] + 2) + sj) * nz + k;
        for (int m = 0; m < 3; ++m) fs[m][dst] = p.f[m][d][src];
    }
}

// One axis of the periodic wrap (an undivided axis of a decomposition).
// axis 0: planes 0 <- nx, nx+1 <- 1 (all j); axis 1: columns 0 <- ny,
// ny+1 <- 1 for all i in 0..nx+1.
__global__ void k_wrap_axis3(double *f0, double *f1, double *f2, int64_t nx, int64_t ny,
                             int64_t nz, int axis)
{
    const int64_t ny2 = ny + 2;
    const int64_t per = axis == 0 ? ny2 * nz : (nx + 2) * nz;  // elements per face
    const int64_t total = 2 * per;
    double *fs[3] = {f0, f1, f2};
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int side = idx >= per;
        const int64_t e = idx - side * per;
        int64_t dst, src;
        if (axis == 0) {
            dst = (side ? (nx + 1) : 0) * ny2 * nz + e;
            src = (side ? 1 : nx) * ny2 * nz + e;
        } else {
            const int64_t i = e / nz, k = e % nz;
            dst = (i * ny2 + (side ? ny + 1 : 0)) * nz + k;
            src = (i * ny2 + (side ? 1 : ny)) * nz + k;
        }
        for (int m = 0; m < 3; ++m)
            if (fs[m]) fs[m][dst] = fs[m][src];
    }
}

// Face pack/unpack. axis 0: plane `index` (all j, k) <-> buf[m][(ny+2)*nz];
// axis 1: column j=`index` for all i in 0..nx+1 <-> buf[m][(nx+2)*nz].
__global__ void k_face3(double *f0, double *f1, double *f2, double *buf, int64_t nx,
                        int64_t ny, int64_t nz, int axis, int64_t index, int pack)
{
    const int64_t ny2 = ny + 2;
    const int64_t per = axis == 0 ? ny2 * nz : (nx + 2) * nz;
    const int64_t total = 3 * per;
    double *fs[3] = {f0, f1, f2};
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int m = (int)(idx / per);
        const int64_t e = idx - m * per;
        int64_t off;
        if (axis == 0) {
            off = index * ny2 * nz + e;
        } else {
            const int64_t i = e / nz, k = e % nz;
            off = (i * ny2 + index) * nz + k;
        }
        if (pack)
            buf[idx] = fs[m][off];
        else
            fs[m][off] = buf[idx];
    }
}

// Both faces of an axis in one launch: buffer a <-> index ia, buffer b <-> index ib.
__global__ void k_faces3(double *f0, double *f1, double *f2, double *buf_a, double *buf_b,
                         int64_t nx, int64_t ny, int64_t nz, int axis, int64_t ia, int64_t ib,
                         int pack)
{
    const int64_t ny2 = ny + 2;
    const int64_t per = axis == 0 ? ny2 * nz : (nx + 2) * nz;
    const int64_t total = 6 * per;
    double *fs[3] = {f0, f1, f2};
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const bool second = idx >= 3 * per;
        const int64_t r = second ? idx - 3 * per : idx;
        const int m = (int)(r / per);
        const int64_t e = r - m * per;
        const int64_t index = second ? ib : ia;
        int64_t off;
        if (axis == 0) {
            off = index * ny2 * nz + e;
        } else {
            const int64_t i = e / nz, k = e % nz;
            off = (i * ny2 + index) * nz + k;
        }
        double *buf = second ? buf_b : buf_a;
        if (pack)
            buf[r] = fs[m][off];
        else
            fs[m][off] = buf[r];
    }
}

// ---------------------------------------------------------------------------
// K5

__device__ __forceinline__ uint64_t lcg_skip(uint64_t seed, uint64_t steps)
{
    uint64_t a_s = 1, c_s = 0, a_step = kLcgMult, c_step = kLcgInc;
    while (steps) {
        if (steps & 1) {
            a_s *= a_step;
            c_s = c_s * a_step + c_step;
        }
        c_step = c_step * a_step + c_step;
        a_step *= a_step;
        steps >>= 1;
    }
    return a_s * seed + c_s;
}

static constexpr int kFillRun = 8;  // consecutive stream values per thread

// Fill the interior columns of a local (nx, ny) block whose interior column
// (i, j) is global column (x_off + i, y_off + j) of a (gnx, gny) grid: the
// stream index of a value is that of the global grid, so every block of a
// decomposition holds exactly its part of the global fields.
__global__ void k_fill_lcg(double *u, double *v, double *w, int64_t nx, int64_t ny, int64_t nz,
                           int64_t gnx, int64_t gny, int64_t x_off, int64_t y_off, uint64_t seed,
                           int baseline)
{
    const int64_t cells = gnx * gny * nz;
    const int64_t runs_per_col = (nz + kFillRun - 1) / kFillRun;
    const int64_t total = 3 * nx * ny * runs_per_col;
    double *fs[3] = {u, v, w};
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx % runs_per_col;
        const int64_t col = idx / runs_per_col;  // over 3*nx*ny
        const int m = (int)(col / (nx * ny));
        const int64_t q = col - m * nx * ny;      // interior column, C order over (i, j)
        const int64_t i = 1 + q / ny, j = 1 + q % ny;
        const int64_t kb = r * kFillRun;
        const int64_t gq = (x_off + i - 1) * gny + (y_off + j - 1);  // global interior column
        const int64_t n0 = m * cells + gq * nz + kb;  // stream index of the first value
        uint64_t s = lcg_skip(seed, (uint64_t)n0);
        double *dst = fs[m] + (i * (ny + 2) + j) * nz;
        for (int t = 0; t < kFillRun; ++t) {
            const int64_t k = kb + t;
            if (k >= nz) break;
            s = s * kLcgMult + kLcgInc;
            double d = __dmul_rn((double)(s >> 11), 0x1.0p-53);
            if (baseline) {
                d = __dsub_rn(__dmul_rn(d, 20.0), 10.0);
                if (m == 2 && (k == 0 || k == nz - 1)) d = 0.0;
            }
            dst[k] = d;
        }
    }
}

__global__ void k_fill_uniform(double *u, double *v, double *w, int64_t n, double a, double b,
                               double c)
{
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        u[idx] = a;
        v[idx] = b;
        w[idx] = c;
    }
}

// ---------------------------------------------------------------------------
// launchers

static unsigned grid_for(int64_t total, int threads)
{
    const DeviceInfo *dev = device_info();
    int64_t blocks = (total + threads - 1) / threads;
    const int64_t cap = (int64_t)(dev ? dev->sms : 148) * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (unsigned)blocks;
}

static int check_launch(const char *what)
{
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(what, e);
    return PWADV_OK;
}

int launch_wrap3(double *u, double *v, double *w, int nf, int64_t nx, int64_t ny, int64_t nz,
                 cudaStream_t s)
{
    const int64_t total = (2 * (ny + 2) + 2 * nx) * nz;
    k_wrap3<<<grid_for(total, 256), 256, 0, s>>>(u, v, w, nf, nx, ny, nz);
    return check_launch("wrap_halos");
}

int launch_pull_halos3(double *u, double *v, double *w, int64_t nx, int64_t ny, int64_t nz,
                       const pwadv_peers *src, cudaStream_t s)
{
    PeerSrc p;
    for (int d = 0; d < 8; ++d) {
        p.f[0][d] = src->u[d];
        p.f[1][d] = src->v[d];
        p.f[2][d] = src->w[d];
        p.nx[d] = src->nx[d];
        p.ny[d] = src->ny[d];
    }
    const int64_t total = (2 * (ny + 2) + 2 * nx) * nz;
    k_pull_halos3<<<grid_for(total, 256), 256, 0, s>>>(u, v, w, nx, ny, nz, p);
    return check_launch("pull_halos");
}

int launch_wrap_axis3(double *u, double *v, double *w, int64_t nx, int64_t ny, int64_t nz,
                      int axis, cudaStream_t s)
{
    const int64_t per = axis == 0 ? (ny + 2) * nz : (nx + 2) * nz;
    k_wrap_axis3<<<grid_for(2 * per, 256), 256, 0, s>>>(u, v, w, nx, ny, nz, axis);
    return check_launch("wrap_axis");
}

int launch_face3(double *u, double *v, double *w, double *buf, int64_t nx, int64_t ny,
                 int64_t nz, int axis, int64_t index, bool pack, cudaStream_t s)
{
    const int64_t per = axis == 0 ? (ny + 2) * nz : (nx + 2) * nz;
    k_face3<<<grid_for(3 * per, 256), 256, 0, s>>>(u, v, w, buf, nx, ny, nz, axis, index,
                                                   pack ? 1 : 0);
    return check_launch(pack ? "pack_face" : "unpack_face");
}

int launch_faces3(double *u, double *v, double *w, double *buf_a, double *buf_b, int64_t nx,
                  int64_t ny, int64_t nz, int axis, int64_t ia, int64_t ib, bool pack, cudaStream_t s)
{
    const int64_t per = axis == 0 ? (ny + 2) * nz : (nx + 2) * nz;
    k_faces3<<<grid_for(6 * per, 256), 256, 0, s>>>(u, v, w, buf_a, buf_b, nx, ny, nz, axis, ia, ib,
                                                    pack ? 1 : 0);
    return check_launch(pack ? "pack_faces" : "unpack_faces");
}

int launch_fill(double *u, double *v, double *w, int64_t nx, int64_t ny, int64_t nz, int mode,
                uint64_t seed, double a, double b, double c, cudaStream_t s)
{
    int rc = launch_fill_box(u, v, w, nx, ny, nz, nx, ny, 0, 0, mode, seed, a, b, c, s);
    if (rc || mode == 2) return rc;
    return launch_wrap3(u, v, w, 3, nx, ny, nz, s);
}

int launch_fill_box(double *u, double *v, double *w, int64_t nx, int64_t ny, int64_t nz,
                    int64_t gnx, int64_t gny, int64_t x_off, int64_t y_off, int mode, uint64_t seed,
                    double a, double b, double c, cudaStream_t s)
{
    if (mode == 2) {
        const int64_t n = (nx + 2) * (ny + 2) * nz;
        k_fill_uniform<<<grid_for(n, 256), 256, 0, s>>>(u, v, w, n, a, b, c);
        return check_launch("fill_uniform");
    }
    const int64_t runs = (nz + kFillRun - 1) / kFillRun;
    const int64_t total = 3 * nx * ny * runs;
    k_fill_lcg<<<grid_for(total, 256), 256, 0, s>>>(u, v, w, nx, ny, nz, gnx, gny, x_off, y_off, seed,
                                                    mode == 1);
    return check_launch("fill_lcg");
}

}  // namespace pwadv
