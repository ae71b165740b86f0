// pwadv_xmarch.cuh — device code of K1 (PW advection) and K4 (fused forward step)
// for sm_100a, shared by the kernel instantiation units (pwadv_k_*.cu) and
// the host launcher (pwadv_advect.cu).
//
// Replaces the reference hot path run_reference -> compute_block ->
// su/sv/sw_formula (pkg/src/pwadvect/kernel.py:73-185). Three kernels:
//
//  * k_advect_xmarch — the production kernel. A CTA owns a strip of TJ
//    y-columns (all nz levels) and marches through X (the GPU analogue of the
//    reference's x_reordered schedule, schedules.py:160-191, and the paper's
//    Listing 3 shift buffers). Each i-plane tile of u, v, w — (TJ+2) columns
//    x nz levels, one contiguous run per field in the k-fastest layout — is
//    brought into a shared-memory ring by 1-D bulk async copies (TMA engine,
//    cp.async.bulk + mbarrier complete_tx), several planes ahead of the
//    compute. Threads own a (column, k-pair); the x-1/x/x+1 window lives in
//    registers (each value is read from shared memory once and rolled), the
//    k-1/k+1 neighbours come from the neighbouring lanes by warp shuffles,
//    the j+-1 neighbours from the shared plane. su, sv and sw are produced in
//    the same pass, so each input byte crosses HBM about once and each output
//    byte once (48 B per point). fp64 CUDA cores only: this is
//    not a contraction, no tensor cores. 512 threads: three compute
//    warpgroups and a producer warpgroup (one thread issues every refill when
//    the stage's empty mbarrier completes; setmaxnreg moves its registers to
//    the compute warps). For nz = 64 / 128 the tile layout is a template
//    constant (immediate-offset shared loads). The x-direction operand sums
//    are carried from plane to plane and three z-sums are shared by the
//    k-pair: 57 fp64 operations per point for the reference's 63, same bits.
//    Work distribution: whole strips for every full round of a persistent
//    grid of one CTA per SM, the leftover strips in X chunks (see unit_at and
//    plan_xmarch); a CTA moving to its next unit just continues its plane
//    sequence (the ring never drains). Variants: UA (odd nz, 8-byte-aligned
//    fields: tile runs copied from the 16-byte boundary below them, scalar
//    shared loads), PULL (the multi-GPU halo exchange fused in: halo cells
//    copied from the neighbours' buffers), STEP (K4, the forward update
//    fused into the epilogue, optionally pushing boundary values into the
//    neighbours' halos).
//
//  * k_advect_march (K1m) — a register-window X-march without the plane
//    ring, for what the X-march does not take (nz > 768, inputs whose
//    16-byte phases differ).
//
//  * k_advect_simple — one thread per output point, direct global loads: the
//    one-cell rims of the overlapped multi-GPU evaluation, and an
//    independent cross-check.
//
// Both are bit-exact with the reference by construction (pwadv_device.cuh).
#pragma once
#include "pwadv_device.cuh"
#include "pwadv_internal.h"

#include <cuda.h>

#include <type_traits>

namespace pwadv {

struct BoxArgs {
    const double *__restrict__ u;
    const double *__restrict__ v;
    const double *__restrict__ w;
    double *o0;  // su, or u_new for the fused step
    double *o1;
    double *o2;
    const double *__restrict__ tzc1;
    const double *__restrict__ tzc2;
    int64_t nx, ny, nz;
    double tcx, tcy, dt;
    int64_t x0, x1, y0, y1;  // interior box, 1-based, half-open
    unsigned long long *trace;  // profiling only: per-plane issue/arrival timestamps (CTA 0)
    int push;                   // fused step only: also store boundary values into peers' halos
    int pull;                   // X-march: load halo cells from the peers' current buffers
    int rim;                    // simple kernel: only the one-cell rim of the box (x0/x1-1/y0/y1-1)
    pwadv_peers peers;          // (include/pwadv.h) push: the neighbours' new buffers; pull:
                                // their current u, v, w; and their extents
};

// Fused halo push (K4 + exchange in one kernel): an interior boundary value of
// this block is also stored into every neighbour halo cell that mirrors it —
// x/y faces and the four corners — in the neighbour's NEW buffers (peer
// memory: the same GPU, or another GPU's memory mapped over NVLink by CUDA
// IPC). After all ranks' kernels finish (one barrier per step) every block's
// halos equal the periodic wrap of the global field, exactly as the two-phase
// exchange and wrap_halos (grid.py:203-208) leave them.
template <int N>
__device__ __forceinline__ void push_to(const pwadv_peers &p, int d, int64_t pi, int64_t pj, int64_t nz,
                                        int64_t k, const double *a, const double *b, const double *c)
{
    const int64_t off = (pi * (p.ny[d] + 2) + pj) * nz + k;
    if constexpr (N == 2) {
        store2(p.u[d] + off, a[0], a[1]);
        store2(p.v[d] + off, b[0], b[1]);
        store2(p.w[d] + off, c[0], c[1]);
    } else {
        p.u[d][off] = a[0];
        p.v[d][off] = b[0];
        p.w[d][off] = c[0];
    }
}

template <int N>
__device__ __forceinline__ void push_boundary(const BoxArgs &A, int64_t i, int64_t j, int64_t k,
                                              const double *a, const double *b, const double *c)
{
    const bool xm = i == 1, xp = i == A.nx, ym = j == 1, yp = j == A.ny;
    if (!(xm || xp || ym || yp)) return;
    const pwadv_peers &p = A.peers;
    const int64_t nz = A.nz;
    if (xm) push_to<N>(p, PWADV_NB_XM, p.nx[PWADV_NB_XM] + 1, j, nz, k, a, b, c);
    if (xp) push_to<N>(p, PWADV_NB_XP, 0, j, nz, k, a, b, c);
    if (ym) push_to<N>(p, PWADV_NB_YM, i, p.ny[PWADV_NB_YM] + 1, nz, k, a, b, c);
    if (yp) push_to<N>(p, PWADV_NB_YP, i, 0, nz, k, a, b, c);
    if (xm && ym) push_to<N>(p, PWADV_NB_XMYM, p.nx[PWADV_NB_XMYM] + 1, p.ny[PWADV_NB_XMYM] + 1, nz, k, a, b, c);
    if (xm && yp) push_to<N>(p, PWADV_NB_XMYP, p.nx[PWADV_NB_XMYP] + 1, 0, nz, k, a, b, c);
    if (xp && ym) push_to<N>(p, PWADV_NB_XPYM, 0, p.ny[PWADV_NB_XPYM] + 1, nz, k, a, b, c);
    if (xp && yp) push_to<N>(p, PWADV_NB_XPYP, 0, 0, nz, k, a, b, c);
}

// The boundary path of the fused step, out of line: only the few threads on a
// block face take it, and keeping it out of the march keeps the march's
// registers (the kernel parameters are __grid_constant__, so no copy is made).
static __device__ __noinline__ void push_pair(const BoxArgs *A, int64_t i, int64_t j, int64_t k0, double a0,
                                       double a1, double b0, double b1, double c0, double c1)
{
    const double pa[2] = {a0, a1}, pb[2] = {b0, b1}, pc[2] = {c0, c1};
    push_boundary<2>(*A, i, j, k0, pa, pb, pc);
}

// As push_pair for the X-march's UA form: 8-byte stores, and for odd nz the
// pair's second level may be past the column.
static __device__ __noinline__ void push_pair_ua(const BoxArgs *A, int64_t i, int64_t j, int64_t k0,
                                          double a0, double a1, double b0, double b1, double c0,
                                          double c1)
{
    push_boundary<1>(*A, i, j, k0, &a0, &b0, &c0);
    if (k0 + 1 < A->nz) push_boundary<1>(*A, i, j, k0 + 1, &a1, &b1, &c1);
}

struct TileCfg {
    int tj;           // columns per strip
    int kp;           // threads per column (= (nz+1)/2)
    int stages;       // ring depth
    int nchunks;      // X chunks per strip; work unit = (chunk, strip)
    int debug;        // ablation bits (PWADV_FLAG_DEBUG_*): 1 = no PW arithmetic, 4 = no stores
    int l2hint;       // 1: load each unit's first two planes with L2 evict_last
    int64_t nstrips;  // ceil((y1-y0)/tj)
    int64_t nlong;    // strips 0..nlong-1 are whole-X units (full rounds); the rest are chunked
    int rot;          // strips are rotated by this much (halo pull: the two y-face strips,
                      // whose tiles take six copies per plane, fall in the chunked tail)
    int nface;        // halo pull: the last nface strips of the tail (the y-face strips)
    int nchf;         //   are cut into nchf chunks instead of nchunks (shorter units)
    // spare-tail plan (spare > 0; plan_xmarch): every strip is cut into nchunks
    // main chunks of mlen planes, run by CTAs 0 .. nstrips*nchunks-1 in one
    // round, and one tail chunk (the rest of X), run by the `spare` remaining
    // CTAs, several in sequence — so a grid whose strips do not divide the SM
    // count still keeps every SM busy for about the same time
    int spare;
    int64_t mlen;
    int nslab;  // column-tile kernel (k_advect_ctile): k-slabs per column; strips of the
                // unit numbering are (y-strip, slab) pairs, slab fastest. 1 otherwise
};

// work units of a launch (unit_at's numbering)
__host__ __device__ __forceinline__ int64_t units_of(const TileCfg &t, int64_t G)
{
    if (t.spare > 0) return G * ((t.nstrips + t.spare - 1) / t.spare);  // rounds x grid, with holes
    return t.nlong + (t.nstrips - t.nlong - t.nface) * t.nchunks + (int64_t)t.nface * t.nchf;
}

// Work units (unit_at) are dealt round-robin to the CTAs: CTA b runs units
// b, b+G, b+2G, ... All CTAs start a round together and march at the same
// rate, so CTAs on adjacent strips stand on the same X planes at the same
// time and each strip's two halo columns (the neighbours' edge columns) are
// served from L2 instead of HBM.
struct Unit {
    int64_t strip, ib, ie;  // outputs i in [ib, ie) of this strip
};

// Units 0..nlong-1 are whole strips (the full rounds: every CTA marches the
// whole X range, all CTAs in step); the remaining strips are cut into
// nchunks X chunks so the last rounds keep the grid busy.
__device__ __forceinline__ Unit unit_at(const BoxArgs &a, const TileCfg &t, int64_t u)
{
    const int64_t nxr = a.x1 - a.x0;
    Unit w;
    if (t.spare > 0) {
        // spare-tail plan: unit u = round r of CTA b. Round 0 of CTAs
        // 0 .. M-1 are the main chunks (CTA b: strip b % nstrips, chunk
        // b / nstrips — all concurrent, so neighbouring strips stand on the
        // same planes and share their halo columns through L2); the tail
        // chunks go to the spare CTAs M .. G-1, strip r*spare + (b-M) in
        // round r (adjacent strips' tails again run concurrently). Units
        // outside these are empty (ib == ie) and skipped.
        const int64_t G = gridDim.x, M = t.nstrips * t.nchunks;
        const int64_t r = u / G, b = u - r * G;
        w.ib = w.ie = a.x0;
        w.strip = 0;
        if (b < M) {
            if (r == 0) {
                w.strip = b % t.nstrips;
                w.ib = a.x0 + (b / t.nstrips) * t.mlen;
                w.ie = w.ib + t.mlen;
            }
        } else {
            const int64_t s = r * t.spare + (b - M);
            if (s < t.nstrips) {
                w.strip = s;
                w.ib = a.x0 + t.nchunks * t.mlen;
                w.ie = a.x1;
            }
        }
        return w;
    }
    if (u < t.nlong) {
        w.strip = u + t.rot < t.nstrips ? u + t.rot : u + t.rot - t.nstrips;
        w.ib = a.x0;
        w.ie = a.x1;
        return w;
    }
    const int64_t treg = t.nstrips - t.nlong - t.nface;  // tail strips with nchunks chunks
    const int64_t v = u - t.nlong;
    int64_t chunk, idx, nch;
    if (v < treg * t.nchunks) {
        chunk = v / treg;
        idx = v - chunk * treg;
        nch = t.nchunks;
    } else {  // the y-face strips of a pull plan, in shorter chunks
        const int64_t r = v - treg * t.nchunks;
        chunk = r / t.nface;
        idx = treg + (r - chunk * t.nface);
        nch = t.nchf;
    }
    w.strip = t.nlong + idx + t.rot;
    if (w.strip >= t.nstrips) w.strip -= t.nstrips;
    w.ib = a.x0 + (nxr * chunk) / nch;
    w.ie = a.x0 + (nxr * (chunk + 1)) / nch;
    return w;
}

// ---------------------------------------------------------------------------
// march kernel (K1m): the general X-march for shapes the plane ring does not
// take (nz > 768, inputs with different 16-byte phases). A 32 x 4 thread block
// owns a tile of 32 levels x 4 columns and marches through an X chunk with
// the x-1/x/x+1 window of its own (j, k) in registers; j +- 1 operands are
// read-only-cache loads (the neighbouring columns' own operands, mostly L1
// hits), k +- 1 come from the neighbouring lanes by shuffles (lane 0 / 31
// load across the tile edge), and the x-shifted diagonal operands are
// carried from the previous plane. 10 loads per point instead of K1s's 27.

template <bool FMA, bool STEP>
__global__ void __launch_bounds__(128) k_advect_march(BoxArgs a, int64_t nchunks)
{
    const int64_t nz = a.nz, ny2 = a.ny + 2;
    const int64_t nbx = a.x1 - a.x0;
    const int64_t ktiles = (nz + 31) / 32;
    const int64_t tile = blockIdx.x;
    const int64_t kt = tile % ktiles, jt = tile / ktiles;
    const int lane = threadIdx.x;
    const int64_t k = kt * 32 + lane;
    const int64_t j = a.y0 + jt * 4 + threadIdx.y;
    const int64_t chunk = blockIdx.y;
    const int64_t ib = a.x0 + nbx * chunk / nchunks, ie = a.x0 + nbx * (chunk + 1) / nchunks;
    const bool kin = k < nz;
    const bool active = kin && j < a.y1;
    // loads of an inactive lane read a valid cell (its column clamped into the
    // box, level clamped into the column); its results are never stored
    const int64_t jj = j < a.y1 ? j : a.y1 - 1;
    const int64_t kk = kin ? k : nz - 1;
    const int64_t sI = ny2 * nz, sJ = nz;
    const bool top = (k == nz - 1);
    const bool lo_edge = lane == 0 && k > 0;            // k-1 lives in the previous tile
    const bool hi_edge = lane == 31 && k + 1 < nz;      // k+1 lives in the next tile
    const double tcx = a.tcx, tcy = a.tcy, dt = a.dt;
    const double c1 = __ldg(a.tzc1 + kk), c2 = __ldg(a.tzc2 + kk);
    const unsigned full = 0xffffffffu;
    if (ib >= ie) return;

    auto at = [&](const double *f, int64_t i, int64_t jx, int64_t kx) -> double {
        return __ldg(f + (i * ny2 + jx) * nz + kx);
    };
    auto up = [&](double x, const double *f, int64_t i, int64_t jx) -> double {  // value at k-1
        double m = __shfl_up_sync(full, x, 1);
        if (lo_edge) m = at(f, i, jx, k - 1);
        return m;
    };
    auto down = [&](double x, const double *f, int64_t i, int64_t jx) -> double {  // value at k+1
        double q = __shfl_down_sync(full, x, 1);
        if (hi_edge) q = at(f, i, jx, k + 1);
        return q;
    };

    // plane ib-1 (x-1 window) and plane ib
    double u_m = at(a.u, ib - 1, jj, kk), v_m = at(a.v, ib - 1, jj, kk), w_m = at(a.w, ib - 1, jj, kk);
    double u_xm1_jp1 = at(a.u, ib - 1, jj + 1, kk);
    double u_xm1_km1 = up(u_m, a.u, ib - 1, jj);
    double u_c = at(a.u, ib, jj, kk), v_c = at(a.v, ib, jj, kk), w_c = at(a.w, ib, jj, kk);
#ifndef PWADV_MARCH_L2_AHEAD
#define PWADV_MARCH_L2_AHEAD 2
#endif
    for (int64_t i = ib; i < ie; ++i) {
        // planes i+1+AHEAD into L2 ahead of their loads (no registers held;
        // a one-plane-ahead register prefetch measured slower: occupancy)
        if (PWADV_MARCH_L2_AHEAD > 0 && i + 1 + PWADV_MARCH_L2_AHEAD <= ie) {
            const int64_t o = ((i + 1 + PWADV_MARCH_L2_AHEAD) * ny2 + jj) * nz + kk;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a.u + o));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a.v + o));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a.w + o));
        }
        const double u_p = at(a.u, i + 1, jj, kk), v_p = at(a.v, i + 1, jj, kk);
        const double w_p = at(a.w, i + 1, jj, kk);
        const double v_p_jm1 = at(a.v, i + 1, jj - 1, kk);
        // current plane i: j +- 1
        const double u_jm1 = at(a.u, i, jj - 1, kk), u_jp1 = at(a.u, i, jj + 1, kk);
        const double v_jm1 = at(a.v, i, jj - 1, kk), v_jp1 = at(a.v, i, jj + 1, kk);
        const double w_jm1 = at(a.w, i, jj - 1, kk), w_jp1 = at(a.w, i, jj + 1, kk);
        // k +- 1 from the neighbouring lanes
        const double u_km1 = up(u_c, a.u, i, jj), u_kp1 = down(u_c, a.u, i, jj);
        const double v_km1 = up(v_c, a.v, i, jj), v_kp1 = down(v_c, a.v, i, jj);
        const double w_km1 = up(w_c, a.w, i, jj), w_kp1 = down(w_c, a.w, i, jj);
        const double w_p_km1 = up(w_p, a.w, i + 1, jj);
        const double w_jp1_km1 = up(w_jp1, a.w, i, jj + 1);
        const double v_jm1_km1 = up(v_jm1, a.v, i, jj - 1);

        double r0 = 0.0, r1 = 0.0, r2 = 0.0;
        if (k > 0) {
            // operand wiring kernel.py:117-128 (the top level never reads k+1)
            r0 = su_formula<FMA>(tcx, tcy, c1, c2, u_c, u_m, u_p, u_jm1, u_jp1, u_km1, u_kp1,
                                 v_jm1, v_p_jm1, v_c, v_p, w_km1, w_p_km1, w_c, w_p, top);
            r1 = sv_formula<FMA>(tcx, tcy, c1, c2, v_c, v_m, v_p, v_jm1, v_jp1, v_km1, v_kp1,
                                 u_m, u_xm1_jp1, u_c, u_jp1, w_km1, w_jp1_km1, w_c, w_jp1, top);
            r2 = sw_formula<FMA>(tcx, tcy, c1, c2, w_c, w_m, w_p, w_jm1, w_jp1, w_km1, w_kp1,
                                 u_xm1_km1, u_m, u_km1, u_c, v_jm1_km1, v_jm1, v_km1, v_c, top);
        }
        if constexpr (STEP) {
            r0 = fwd_update(u_c, dt, r0);
            r1 = fwd_update(v_c, dt, r1);
            r2 = fwd_update(w_c, dt, r2);
        }
        if (active) {
            const int64_t o = (i * ny2 + j) * nz + k;
            a.o0[o] = r0;
            a.o1[o] = r1;
            a.o2[o] = r2;
        }
        // roll the window; diagonal operands of the next plane
        u_xm1_jp1 = u_jp1;
        u_xm1_km1 = u_km1;
        u_m = u_c;
        v_m = v_c;
        w_m = w_c;
        u_c = u_p;
        v_c = v_p;
        w_c = w_p;
    }
    (void)sI;
    (void)sJ;
}

// ---------------------------------------------------------------------------
// simple kernel

template <bool FMA, bool STEP>
__global__ void __launch_bounds__(256) k_advect_simple(BoxArgs a)
{
    const int64_t nz = a.nz, ny2 = a.ny + 2;
    const int64_t nbx = a.x1 - a.x0, nby = a.y1 - a.y0;
    // rim mode (nbx, nby >= 3): columns of the planes x0 and x1-1, then of the
    // rows y0 and y1-1 between them — the part of a block that needs halos
    const int64_t ncols = a.rim ? 2 * nby + 2 * (nbx - 2) : nbx * nby;
    const int64_t total = ncols * nz;
    const int64_t sI = ny2 * nz, sJ = nz;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = idx % nz;
        const int64_t col = idx / nz;
        int64_t i, j;
        if (!a.rim) {
            i = a.x0 + col / nby;
            j = a.y0 + col % nby;
        } else if (col < 2 * nby) {
            i = col < nby ? a.x0 : a.x1 - 1;
            j = a.y0 + (col < nby ? col : col - nby);
        } else {
            const int64_t r = col - 2 * nby;
            i = a.x0 + 1 + (r < nbx - 2 ? r : r - (nbx - 2));
            j = r < nbx - 2 ? a.y0 : a.y1 - 1;
        }
        const int64_t o = (i * ny2 + j) * nz + k;
        double r0 = 0.0, r1 = 0.0, r2 = 0.0;
        if (k > 0) {
            const bool top = (k == nz - 1);
            const double *U = a.u + o, *V = a.v + o, *W = a.w + o;
            const double c1 = __ldg(a.tzc1 + k), c2 = __ldg(a.tzc2 + k);
            // operand wiring: kernel.py:117-128 (f, dx, dy, dk)
            const double u_c = __ldg(U), u_xm1 = __ldg(U - sI), u_xp1 = __ldg(U + sI);
            const double u_jm1 = __ldg(U - sJ), u_jp1 = __ldg(U + sJ);
            const double u_km1 = __ldg(U - 1), u_kp1 = top ? 0.0 : __ldg(U + 1);
            const double u_xm1_jp1 = __ldg(U - sI + sJ), u_xm1_km1 = __ldg(U - sI - 1);
            const double v_c = __ldg(V), v_xm1 = __ldg(V - sI), v_xp1 = __ldg(V + sI);
            const double v_jm1 = __ldg(V - sJ), v_jp1 = __ldg(V + sJ);
            const double v_km1 = __ldg(V - 1), v_kp1 = top ? 0.0 : __ldg(V + 1);
            const double v_jm1_xp1 = __ldg(V + sI - sJ), v_jm1_km1 = __ldg(V - sJ - 1);
            const double w_c = __ldg(W), w_xm1 = __ldg(W - sI), w_xp1 = __ldg(W + sI);
            const double w_jm1 = __ldg(W - sJ), w_jp1 = __ldg(W + sJ);
            const double w_km1 = __ldg(W - 1), w_kp1 = top ? 0.0 : __ldg(W + 1);
            const double w_km1_xp1 = __ldg(W + sI - 1), w_km1_jp1 = __ldg(W + sJ - 1);
            r0 = su_formula<FMA>(a.tcx, a.tcy, c1, c2, u_c, u_xm1, u_xp1, u_jm1, u_jp1, u_km1,
                                 u_kp1, v_jm1, v_jm1_xp1, v_c, v_xp1, w_km1, w_km1_xp1, w_c,
                                 w_xp1, top);
            r1 = sv_formula<FMA>(a.tcx, a.tcy, c1, c2, v_c, v_xm1, v_xp1, v_jm1, v_jp1, v_km1,
                                 v_kp1, u_xm1, u_xm1_jp1, u_c, u_jp1, w_km1, w_km1_jp1, w_c,
                                 w_jp1, top);
            r2 = sw_formula<FMA>(a.tcx, a.tcy, c1, c2, w_c, w_xm1, w_xp1, w_jm1, w_jp1, w_km1,
                                 w_kp1, u_xm1_km1, u_xm1, u_km1, u_c, v_jm1_km1, v_jm1, v_km1,
                                 v_c, top);
        }
        if constexpr (STEP) {
            r0 = fwd_update(__ldg(a.u + o), a.dt, r0);
            r1 = fwd_update(__ldg(a.v + o), a.dt, r1);
            r2 = fwd_update(__ldg(a.w + o), a.dt, r2);
        }
        a.o0[o] = r0;
        a.o1[o] = r1;
        a.o2[o] = r2;
        if constexpr (STEP) {
            if (a.push) push_boundary<1>(a, i, j, k, &r0, &r1, &r2);
        }
    }
}

// ---------------------------------------------------------------------------
// X-march kernel

// value at k0-1 of the thread's pair: the previous lane's k1, or (across a
// warp boundary inside a column, FIX only) straight from the shared plane.
// When columns straddle warps (FIX, e.g. nz = 128) the neighbour is read from
// the staged plane instead (measured faster there than shuffles + fix-ups).
#ifndef PWADV_PRODUCER_SLEEP_NS
#define PWADV_PRODUCER_SLEEP_NS 0
#endif
#ifndef PWADV_NBR_SMEM
#define PWADV_NBR_SMEM 0
#endif
template <bool FIX>
__device__ __forceinline__ double nbr_m(double2 p, const double *colp, int k0, bool fix)
{
    if constexpr (PWADV_NBR_SMEM || FIX) return colp[k0 > 0 ? k0 - 1 : 0];
    double m = __shfl_up_sync(0xffffffffu, p.y, 1);
    if constexpr (FIX) {
        if (fix) m = colp[k0 - 1];
    }
    return m;
}

// value at k0+2: the next lane's k0, or from the shared plane.
template <bool FIX>
__device__ __forceinline__ double nbr_q(double2 p, const double *colp, int k0, bool fix, int nz)
{
    if constexpr (PWADV_NBR_SMEM || FIX) return colp[k0 + 2 < nz ? k0 + 2 : nz - 1];
    double q = __shfl_down_sync(0xffffffffu, p.x, 1);
    if constexpr (FIX) {
        if (fix) q = colp[k0 + 2];
    }
    return q;
}

// Per-CTA ring bookkeeping in shared memory. Planes are numbered by a CTA-
// local sequence number q (the order the CTA consumes them); plane q lives in
// stage q % S. Unit k of this CTA (global unit blockIdx.x + k*gridDim.x)
// streams planes first[k] .. first[k+1]-1 = its chunk plus one plane each side.
constexpr int kMaxUnitsPerCta = 64;

struct RingState {
    int total;                        // planes this CTA streams
    int nunits;                       // units of this CTA
    int first[kMaxUnitsPerCta + 1];   // first sequence number of each unit
    uint32_t bytes[kMaxUnitsPerCta];  // bytes per field per plane of each unit
    int64_t src[kMaxUnitsPerCta];     // element offset of the unit's first plane tile
    int32_t ui0[kMaxUnitsPerCta];     // halo pull: plane index of the unit's first plane (ib - 1)
    int32_t uj0[kMaxUnitsPerCta];     //   first interior column of its strip
    int32_t utj[kMaxUnitsPerCta];     //   columns of its strip
    int32_t dsto[kMaxUnitsPerCta];    //   where the local run lands in a slot (doubles)
    int64_t clo[kMaxUnitsPerCta];     //   y-face units: YM / YP halo column of the unit's first
    int64_t chi[kMaxUnitsPerCta];     //   plane in the neighbour's field (elements), or -1
    int l2hint;                       // TileCfg::l2hint
    int released[16];                 // per stage: warps done with its current plane
};

__device__ __forceinline__ unsigned long long gtime()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Halo pull (K1 with the exchange fused in, pwadv_advect_pull_f64): the halo
// cells of plane q's tile are copied from the neighbours' current buffers
// instead of this block's halos — an x-halo plane (i = 0 / nx+1) from the x
// neighbour's last / first interior plane, the y-halo columns (j = 0 / ny+1)
// of an interior plane from the y neighbour's last / first interior column,
// and the two corner columns the stencil reads, u(0, ny+1) and v(nx+1, 0),
// from the diagonal neighbours (wrap_halos' semantics, grid.py:203-208: the
// X pass then the Y pass over the X halos). Peer buffers are read over NVLink
// by the same bulk copies; cells the stencil never reads (the other corner
// cells) are left unfilled. At most three pieces per field and plane, and
// only for halo planes and y-face strips: all other tiles are one local run.
__device__ __forceinline__ void copy_cols(double *dst, const double *u, const double *v,
                                          const double *w, int64_t off, int CS, uint32_t bytes,
                                          uint64_t *bar)
{
    bulk_g2s(dst, u + off, bytes, bar);
    bulk_g2s(dst + CS, v + off, bytes, bar);
    bulk_g2s(dst + 2 * CS, w + off, bytes, bar);
}

// x-halo plane i (0 or nx+1) of unit k.
__device__ __forceinline__ void issue_plane_pull(const RingState *rs, const BoxArgs &a, int k,
                                                 int64_t i, int st, int CS, double *ring,
                                                 uint64_t *full)
{
    const int64_t jlo = rs->uj0[k] - 1, jhi = rs->uj0[k] + rs->utj[k];  // tile columns [jlo, jhi]
    const int64_t nz = a.nz, ny = a.ny, ny2 = a.ny + 2;
    const uint32_t cb = (uint32_t)(nz * sizeof(double));  // bytes per column
    const pwadv_peers &p = a.peers;
    const int64_t c0 = jlo > 1 ? jlo : 1, c1 = jhi < ny ? jhi : ny;  // interior columns of the tile
    const bool lo = jlo == 0, hi = jhi == ny + 1;
    double *dst = ring + (size_t)st * 3 * CS;
    uint64_t *bar = &full[st];
    (void)c1;
    if (i == 0) {  // x-lo halo plane: the XM neighbour's last plane; u(0, ny+1) from XMYP
        const uint32_t b = (uint32_t)(c1 - jlo + 1) * cb;
        mbar_arrive_expect_tx(bar, 3 * b + (hi ? cb : 0));
        const int d = PWADV_NB_XM;
        copy_cols(dst, p.u[d], p.v[d], p.w[d], (p.nx[d] * ny2 + jlo) * nz, CS, b, bar);
        if (hi) {
            const int e = PWADV_NB_XMYP;
            bulk_g2s(dst + (jhi - jlo) * nz, p.u[e] + (p.nx[e] * (p.ny[e] + 2) + 1) * nz, cb, bar);
        }
    } else {  // x-hi halo plane: XP's first plane; v(nx+1, 0) from XPYM
        const uint32_t b = (uint32_t)(jhi - c0 + 1) * cb;
        mbar_arrive_expect_tx(bar, 3 * b + (lo ? cb : 0));
        const int d = PWADV_NB_XP;
        copy_cols(dst + (c0 - jlo) * nz, p.u[d], p.v[d], p.w[d], (ny2 + c0) * nz, CS, b, bar);
        if (lo) {
            const int e = PWADV_NB_XPYM;
            bulk_g2s(dst + CS, p.v[e] + ((p.ny[e] + 2) + p.ny[e]) * nz, cb, bar);
        }
    }
}

// Issue the bulk copies of plane q (3 fields, one contiguous run each) into
// stage st, completing on full[st]. A table lookup and one multiply-add: the
// warp that issues must not fall behind the others (it gates the next refill).
template <bool TRACE = true, bool PULL = false>
__device__ __forceinline__ void issue_plane(const RingState *rs, const BoxArgs &a, int q, int st,
                                            int CS, double *ring, uint64_t *full)
{
    if (TRACE && a.trace && blockIdx.x == 0 && q < 4096) a.trace[2 * q] = gtime();
    int k = 0;
    while (rs->first[k + 1] <= q) ++k;
    double *dst = ring + (size_t)st * 3 * CS;
    if constexpr (PULL) dst += rs->dsto[k] > 0 ? rs->dsto[k] : 0;  // y-face unit: trimmed run
    const uint32_t bytes = rs->bytes[k];
    const int64_t off = rs->src[k] + (int64_t)(q - rs->first[k]) * ((a.ny + 2) * a.nz);
    mbar_arrive_expect_tx(&full[st], 3 * bytes);
    // the first two planes of a unit are read again, much later, by the unit
    // of the previous X chunk (as its last two planes): keep them in L2
    if (rs->l2hint && q - rs->first[k] < 2) {
        const uint64_t pol = policy_evict_last();
        bulk_g2s_hint(dst, a.u + off, bytes, &full[st], pol);
        bulk_g2s_hint(dst + CS, a.v + off, bytes, &full[st], pol);
        bulk_g2s_hint(dst + 2 * CS, a.w + off, bytes, &full[st], pol);
        return;
    }
    bulk_g2s(dst, a.u + off, bytes, &full[st]);
    bulk_g2s(dst + CS, a.v + off, bytes, &full[st]);
    bulk_g2s(dst + 2 * CS, a.w + off, bytes, &full[st]);
}

// Unaligned tile runs (UA kernels: odd nz, 8-byte-aligned fields). A plane
// tile of a field is still one contiguous run, but its start need not be
// 16-byte aligned: the copy starts at the 16-byte boundary below it (d = 0 or
// 1 element early; u, v and w share d, plan_xmarch checks) and is rounded up
// to 16 bytes, so the tile sits at offset d of the stage slot and the compute
// warps read it with scalar loads. Only a run that ends at the very end of a
// field can have its rounded copy overrun the array by one element; then the
// copy stops 16 bytes short and the producer moves the last element itself
// (before arming the barrier, whose arrive releases the store).
__device__ __forceinline__ void issue_plane_ua(const RingState *rs, const BoxArgs &a, int q, int st,
                                               int CS, double *ring, uint64_t *full)
{
    int k = 0;
    while (rs->first[k + 1] <= q) ++k;
    const int64_t off = rs->src[k] + (int64_t)(q - rs->first[k]) * ((a.ny + 2) * a.nz);
    const int64_t d = (int64_t)(((uintptr_t)(a.u + off) >> 3) & 1);
    const int64_t run = rs->bytes[k] / sizeof(double);  // elements of the tile run
    uint32_t n = (uint32_t)(((d + run) * 8 + 15) & ~(int64_t)15);
    double *dst = ring + (size_t)st * 3 * CS;
    const int64_t total = (a.nx + 2) * (a.ny + 2) * a.nz;  // elements per field
    if (off - d + n / 8 > total) {  // overrun of one element at the end of the fields
        n -= 16;
        const int64_t last = off - d + n / 8;  // == total - 1, the run's last element
        dst[n / 8] = a.u[last];
        dst[CS + n / 8] = a.v[last];
        dst[2 * CS + n / 8] = a.w[last];
    }
    mbar_arrive_expect_tx(&full[st], 3 * n);
    bulk_g2s(dst, a.u + off - d, n, &full[st]);
    bulk_g2s(dst + CS, a.v + off - d, n, &full[st]);
    bulk_g2s(dst + 2 * CS, a.w + off - d, n, &full[st]);
}

// X-march kernel. Register slots U0[3], V0[3], ... hold plane p in slot p % 3
// (relative to the unit start), so the x-1/x/x+1 window rotates by renaming —
// the step body is instantiated for the three rotations and unrolled, with no
// register moves.
//
// Ring protocol. MAXT == 512 (default): each compute warp, once it has read
// everything it needs from plane q, arrives on empty[q % S]; the producer
// thread waits for the stage's 12 arrivals and issues plane q+S into it.
// Other thread budgets (no producer warp): each warp bumps released[q % S]
// and the warp that completes the count issues the refill. Either way refills
// happen in sequence order and planes q+1 .. q+S-1 are resident or in flight
// when q is released.
// resident CTAs per SM for a thread budget (each CTA keeps <= 168 registers)
__host__ __device__ constexpr int ctas_per_sm(int maxt) { return maxt <= 128 ? 3 : (maxt <= 192 ? 2 : 1); }

// NZC > 0 (warp-specialised kernel only): nz, TJ and the tile layout are
// compile-time constants, so every staged operand is one LDS at an immediate
// offset from a per-plane base register (the BASELINE nz = 64 / 128 cases).
// UA: unaligned tile runs (issue_plane_ua) — each staged plane sits at offset
// d in its slot, scalar shared loads and output stores (odd nz or 8-byte-
// aligned fields; warp-specialised kernel only).
template <bool FMA, bool STEP, int MAXT, bool FIX, int NZC = 0, bool UA = false, bool PULL = false>
__global__ void __launch_bounds__(MAXT, ctas_per_sm(MAXT))
    k_advect_xmarch(const __grid_constant__ BoxArgs a, const __grid_constant__ TileCfg t)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    static_assert(NZC == 0 || MAXT == 512, "compile-time layout: WS only");
    static_assert(!UA || (MAXT == 512 && NZC == 0), "unaligned runs: warp-specialised, run-time layout");
    static_assert(!PULL || (MAXT == 512 && !UA), "halo pull: warp-specialised, aligned runs");
    // programmatic dependent launch (launch_box): let the next grid be
    // scheduled as our CTAs retire, and wait until the previous grid on the
    // stream has completed and its writes are visible (they may be our
    // inputs) before any global access. The unit table and the ring barriers
    // (shared memory and kernel parameters only) are set up BEFORE the wait,
    // while the previous grid drains; tid 0 waits before the first bulk copy,
    // every other thread after the CTA barrier that publishes the table.
    // No-ops for an ordinary launch.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int S = t.stages;
    const int TJ = NZC ? 384 / (NZC / 2) : t.tj;
    const int KP = NZC ? NZC / 2 : t.kp;
    const int nz = NZC ? NZC : (int)a.nz;
    // doubles per field slot of a stage (UA: room for the offset d and the
    // 16-byte rounding of the copy, kept even so every slot is 16-byte aligned)
    const int CS = UA ? (((TJ + 2) * nz + 3) & ~1) : (TJ + 2) * nz;
    double *ring = reinterpret_cast<double *>(smem_raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem_raw + (size_t)S * 3 * CS * sizeof(double));
    uint64_t *empty = full + S;  // warp-specialised variant only
    RingState *rs = reinterpret_cast<RingState *>(full + 2 * S);
    // MAXT == 512: warp-specialised — warpgroups 0-2 compute, warpgroup 3 is
    // the producer (one thread issuing refills as soon as a stage's last
    // consumer warp arrives on its empty barrier; setmaxnreg moves the
    // producer's registers to the consumers)
    constexpr bool WS = (MAXT == 512);
    constexpr int kComputeWarps = WS ? 12 : MAXT / 32;

    const int tid = threadIdx.x, lane = tid & 31;
    const int nwarps = WS ? kComputeWarps : (int)(blockDim.x >> 5);
    const bool in_tile = tid < TJ * KP;
    const int c = in_tile ? tid / KP : TJ - 1;
    const int kp = in_tile ? tid - (tid / KP) * KP : 0;
    const int k0 = 2 * kp, k1 = k0 + 1;
    const bool fixM = FIX && (lane == 0) && kp > 0;
    const bool fixQ = FIX && (lane == 31) && kp < KP - 1;
    const bool top_b = (k1 == nz - 1);
    const bool top_a = UA && (k0 == nz - 1);  // odd nz: the top is a pair's first level
    const bool lvl0 = (k0 == 0);
    const int k1c = UA ? (k1 < nz ? k1 : nz - 1) : k1;  // odd nz: k1 = nz is past the column

    const double tcx = a.tcx, tcy = a.tcy, dt = a.dt;

    const int64_t ny2 = a.ny + 2;
    const int64_t G = gridDim.x;
    const int64_t nunits = units_of(t, G);
    if ((int64_t)blockIdx.x >= nunits) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        return;
    }

    if (tid == 0) {
        int q = 0, k = 0;
        for (int64_t u = blockIdx.x; u < nunits && k < kMaxUnitsPerCta; u += G) {
            const Unit w = unit_at(a, t, u);
            if (w.ie <= w.ib) continue;  // a hole of the spare-tail plan
            const int64_t j0 = a.y0 + w.strip * TJ;
            const int64_t tjs = (a.y1 - j0) < TJ ? (a.y1 - j0) : TJ;
            rs->first[k] = q;
            rs->bytes[k] = (uint32_t)((tjs + 2) * nz * sizeof(double));
            rs->src[k] = ((w.ib - 1) * ny2 + (j0 - 1)) * nz;
            rs->ui0[k] = (int32_t)(w.ib - 1);
            rs->uj0[k] = (int32_t)j0;
            rs->utj[k] = (int32_t)tjs;
            rs->dsto[k] = -1;  // not a y-face unit
            if constexpr (PULL) {  // y-face unit: its local run skips the halo columns
                const bool lo = j0 == 1, hi = j0 + tjs == a.ny + 1;
                const pwadv_peers &pp = a.peers;
                rs->clo[k] = lo ? ((w.ib - 1) * (pp.ny[PWADV_NB_YM] + 2) + pp.ny[PWADV_NB_YM]) * nz : -1;
                rs->chi[k] = hi ? ((w.ib - 1) * (pp.ny[PWADV_NB_YP] + 2) + 1) * nz : -1;
                if (lo || hi) {
                    rs->src[k] += lo ? nz : 0;
                    rs->bytes[k] -= (uint32_t)(((lo ? 1 : 0) + (hi ? 1 : 0)) * nz * sizeof(double));
                    rs->dsto[k] = lo ? nz : 0;
                }
            }
            q += (int)(w.ie - w.ib + 2);
            ++k;
        }
        rs->first[k] = q;
        rs->total = q;
        rs->nunits = k;
        rs->l2hint = t.l2hint;
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kComputeWarps);
            rs->released[s] = 0;
        }
        fence_mbar_init();
        asm volatile("griddepcontrol.wait;" ::: "memory");  // inputs final from here on
        const int n0 = PULL ? 0 : (q < S ? q : S);  // pull: the producer warp issues all
        for (int n = 0; n < n0; ++n) {
            if constexpr (UA) issue_plane_ua(rs, a, n, n, CS, ring, full);
            else issue_plane<NZC == 0>(rs, a, n, n, CS, ring, full);
        }
    }
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const double c1a = __ldg(a.tzc1 + k0), c1b = __ldg(a.tzc1 + k1c);
    const double c2a = __ldg(a.tzc2 + k0), c2b = __ldg(a.tzc2 + k1c);
    const int total = rs->total;
    const int my_units = rs->nunits;
    if constexpr (WS) {
        if (tid >= 32 * kComputeWarps) {  // producer warpgroup
            if constexpr (UA || PULL) {  // 4 x 32 x 32 + 12 x 32 x 160 = 64 K registers
                asm volatile("setmaxnreg.dec.sync.aligned.u32 32;\n" ::: "memory");
            } else {
                asm volatile("setmaxnreg.dec.sync.aligned.u32 24;\n" ::: "memory");
            }
            if constexpr (PULL) {
                // the producer thread: x-halo planes from the x / diagonal
                // neighbours, else the local run (trimmed on y-face units) plus
                // the y-halo columns from YM / YP, with per-unit offsets
                // precomputed in the unit table (this loop must keep pace
                // with the consumers).
                if (tid == 32 * kComputeWarps) {
                    const pwadv_peers &pp = a.peers;
                    const int64_t slo = (pp.ny[PWADV_NB_YM] + 2) * a.nz, shi = (pp.ny[PWADV_NB_YP] + 2) * a.nz;
                    const uint32_t cb = (uint32_t)(nz * sizeof(double));
                    int k = 0;
                    for (int q = 0; q < total; ++q) {
                        while (rs->first[k + 1] <= q) ++k;
                        const int st = q % S;
                        if (q >= S) mbar_wait(&empty[st], (uint32_t)(((q / S) - 1) & 1));
                        fence_proxy_async();
                        const int rel = q - rs->first[k];
                        const int64_t i = rs->ui0[k] + rel;
                        if (i == 0 || i == a.nx + 1) {
                            issue_plane_pull(rs, a, k, i, st, CS, ring, full);
                            continue;
                        }
                        // the local run (trimmed on y-face units) and, on those,
                        // the y-halo columns from YM / YP
                        double *dst = ring + (size_t)st * 3 * CS;
                        const int64_t lo = rs->clo[k], hi = rs->chi[k];
                        const uint32_t bytes = rs->bytes[k];
                        const int64_t off = rs->src[k] + (int64_t)rel * ((a.ny + 2) * a.nz);
                        mbar_arrive_expect_tx(&full[st], 3 * (bytes + (lo >= 0 ? cb : 0) + (hi >= 0 ? cb : 0)));
                        copy_cols(dst + (rs->dsto[k] > 0 ? rs->dsto[k] : 0), a.u, a.v, a.w, off, CS, bytes,
                                  &full[st]);
                        if (lo >= 0) {
                            const int d = PWADV_NB_YM;
                            copy_cols(dst, pp.u[d], pp.v[d], pp.w[d], lo + rel * slo, CS, cb, &full[st]);
                        }
                        if (hi >= 0) {
                            const int d = PWADV_NB_YP;
                            copy_cols(dst + (rs->utj[k] + 1) * nz, pp.u[d], pp.v[d], pp.w[d], hi + rel * shi,
                                      CS, cb, &full[st]);
                        }
                    }
                }
                return;
            }
            if (tid == 32 * kComputeWarps) {
                for (int q = (total < S ? total : S); q < total; ++q) {
                    const int st = q % S;
#if PWADV_PRODUCER_SLEEP_NS > 0
                    mbar_wait_sleep(&empty[st], (uint32_t)(((q / S) - 1) & 1), PWADV_PRODUCER_SLEEP_NS);
#else
                    mbar_wait(&empty[st], (uint32_t)(((q / S) - 1) & 1));
#endif
                    fence_proxy_async();
                    if constexpr (UA) issue_plane_ua(rs, a, q, st, CS, ring, full);
                    else issue_plane<NZC == 0, PULL>(rs, a, q, st, CS, ring, full);
                }
            }
            return;
        }
        asm volatile("setmaxnreg.inc.sync.aligned.u32 160;\n" ::: "memory");
    }

    // consumer ring position: sequence number, stage and parity of the
    // plane to wait for next
    int cseq = 0, cst = 0;
    uint32_t cph = 0;
    const int toff = (c + 1) * nz + k0;  // this thread's pair in a field tile-plane

    auto release = [&](int seq, int st) {
        __syncwarp();
        if constexpr (WS) {
            if (lane == 0) mbar_arrive(&empty[st]);
            return;
        }
        if (lane == 0) {
            __threadfence_block();  // this warp's reads of the stage happen before the refill
            const int done = atomicAdd(&rs->released[st], 1);
            if (done == nwarps - 1) {
                rs->released[st] = 0;
                if (seq + S < total) {
                    fence_proxy_async();
                    issue_plane<NZC == 0>(rs, a, seq + S, st, CS, ring, full);
                }
            }
        }
    };
    auto wait_next = [&]() -> const double * {
        mbar_wait(&full[cst], cph);
        if constexpr (NZC == 0) {  // plane-arrival stamps (tools/trace.py): generic kernel only
            if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && cseq < 4096)
                a.trace[2 * cseq + 1] = gtime();
        }
        return ring + (size_t)cst * 3 * CS;
    };
    auto advance = [&]() {
        ++cseq;
        if (++cst == S) {
            cst = 0;
            cph ^= 1u;
        }
    };
    auto P = [&](const double *pl, int f, int dy) -> double2 {
        const double *x = pl + f * CS + dy * nz + toff;
        if constexpr (UA) return make_double2(x[0], x[1]);  // 8-byte aligned only
        return *reinterpret_cast<const double2 *>(x);
    };
    auto colp = [&](const double *pl, int f, int dy) -> const double * {
        return pl + f * CS + (c + 1 + dy) * nz;
    };
    // UA: offset d of a staged plane in its slot (plane stride parity toggles
    // it from plane to plane; the unit's first plane fixes it)
    const int psodd = UA ? (int)(((a.ny + 2) * a.nz) & 1) : 0;
    const int inpar = UA ? (int)(((uintptr_t)a.u >> 3) & 1) : 0;

    double2 U0[3], V0[3], W0[3], VM[3];
    double W0M[3];
    // x-direction operand sums carried from plane i-1 to plane i (the x+1 sum
    // of one step is the x-1 sum of the next; IEEE addition is commutative):
    // su  u(i-1)+u(i)                       (kernel.py:73-84, x-term)
    // sv  u(i-1,j)+u(i-1,j+1)               (kernel.py:87-98, x-term)
    // sw  u(i-1,k-1)+u(i-1,k)               (kernel.py:101-112, x-term)
    double sxu_a, sxu_b, txu_a, txu_b, rxu_a, rxu_b;

    for (int k = 0; k < my_units; ++k) {
        // the unit's geometry from the table tid 0 built (planes ib-1 .. ie)
        const int64_t ib = (int64_t)rs->ui0[k] + 1;
        const int64_t ie = ib + (rs->first[k + 1] - rs->first[k]) - 2;
        const int64_t j0 = rs->uj0[k];
        const int64_t tjs = rs->utj[k];
        const bool active = in_tile && c < tjs;
        // fused step with the halo push: a thread on the y = 1 or y = ny face
        // stores its pair into one neighbour's halo column every plane — a
        // fixed target, resolved here once per unit (the x faces, corners and
        // the ny == 1 case take the general out-of-line path below)
        int ydir = -1;
        int64_t ypj = 0, ystr = 0;
        if constexpr (STEP) {
            if (a.push && active && a.ny > 1) {
                if (j0 + c == 1) {
                    ydir = PWADV_NB_YM;
                    ypj = a.peers.ny[PWADV_NB_YM] + 1;
                } else if (j0 + c == a.ny) {
                    ydir = PWADV_NB_YP;
                }
                if (ydir >= 0) ystr = a.peers.ny[ydir] + 2;
            }
        }

        // UA: offset of the unit's first plane in its slot
        int dC = UA ? (inpar ^ (int)((((ib - 1) * ny2 + (j0 - 1)) * (int64_t)nz) & 1)) : 0;
        // plane ib-1 -> slot 2 (the x-1 window of the first step)
        {
            const double *pl = wait_next() + dC;
            U0[2] = P(pl, 0, 0);
            const double2 u1 = P(pl, 0, 1);
            V0[2] = P(pl, 1, 0);
            W0[2] = P(pl, 2, 0);
            const double u0M = nbr_m<FIX>(U0[2], colp(pl, 0, 0), k0, fixM);
            release(cseq, cst);
            advance();
            txu_a = __dadd_rn(U0[2].x, u1.x);
            txu_b = __dadd_rn(U0[2].y, u1.y);
            rxu_a = __dadd_rn(u0M, U0[2].x);
            rxu_b = __dadd_rn(U0[2].x, U0[2].y);
        }
        // plane ib -> slot 0 (items read from the leading plane)
        int pst = cst;  // stage of the current x plane, released one step later
        dC ^= psodd;
        {
            const double *pl = wait_next() + dC;
            U0[0] = P(pl, 0, 0);
            V0[0] = P(pl, 1, 0);
            W0[0] = P(pl, 2, 0);
            VM[0] = P(pl, 1, -1);
            W0M[0] = nbr_m<FIX>(W0[0], colp(pl, 2, 0), k0, fixM);
            advance();
            sxu_a = __dadd_rn(U0[0].x, U0[2].x);
            sxu_b = __dadd_rn(U0[0].y, U0[2].y);
        }

        double *o0 = a.o0 + (ib * ny2 + (j0 + c)) * (int64_t)nz + k0;
        double *o1 = a.o1 + (ib * ny2 + (j0 + c)) * (int64_t)nz + k0;
        double *o2 = a.o2 + (ib * ny2 + (j0 + c)) * (int64_t)nz + k0;
        const int64_t ostep = ny2 * nz;

        int64_t ci = ib;  // the output plane of the current step
        auto body = [&](auto R) {
            constexpr int r = decltype(R)::value;
            constexpr int rm = (r + 2) % 3, rp = (r + 1) % 3;
            const int lst = cst;
            const int dL = dC ^ psodd;
            const double *L = wait_next() + dL;                      // plane i+1
            const double *C = ring + (size_t)pst * 3 * CS + dC;      // plane i
            U0[rp] = P(L, 0, 0);
            V0[rp] = P(L, 1, 0);
            W0[rp] = P(L, 2, 0);
            VM[rp] = P(L, 1, -1);
            W0M[rp] = nbr_m<FIX>(W0[rp], colp(L, 2, 0), k0, fixM);
            const double2 u1c = P(C, 0, 1);
            const double2 umc = P(C, 0, -1), v1c = P(C, 1, 1), w1c = P(C, 2, 1), wmc = P(C, 2, -1);
            const double w1cM = nbr_m<FIX>(w1c, colp(C, 2, 1), k0, fixM);
            const double u0cM = nbr_m<FIX>(U0[r], colp(C, 0, 0), k0, fixM);
            const double u0cQ = nbr_q<FIX>(U0[r], colp(C, 0, 0), k0, fixQ, nz);
            const double v0cM = nbr_m<FIX>(V0[r], colp(C, 1, 0), k0, fixM);
            const double v0cQ = nbr_q<FIX>(V0[r], colp(C, 1, 0), k0, fixQ, nz);
            const double w0cQ = nbr_q<FIX>(W0[r], colp(C, 2, 0), k0, fixQ, nz);
            const double vmcM = nbr_m<FIX>(VM[r], colp(C, 1, -1), k0, fixM);
            release(cseq - 1, pst);  // plane i fully consumed by this warp

            const double2 u0m = U0[rm], u0c = U0[r], u0p = U0[rp];
            const double2 v0m = V0[rm], v0c = V0[r], v0p = V0[rp];
            const double2 w0m = W0[rm], w0c = W0[r], w0p = W0[rp];
            const double2 vmc = VM[r], vmp = VM[rp];
            const double w0cM = W0M[r], w0pM = W0M[rp];

            // sums shared with the next plane (x-carry) or within the k-pair
            const double nsxu_a = __dadd_rn(u0c.x, u0p.x), nsxu_b = __dadd_rn(u0c.y, u0p.y);
            const double ntxu_a = __dadd_rn(u0c.x, u1c.x), ntxu_b = __dadd_rn(u0c.y, u1c.y);
            const double nrxu_a = __dadd_rn(u0cM, u0c.x), nrxu_b = __dadd_rn(u0c.x, u0c.y);
            const double szu = __dadd_rn(w0c.x, w0p.x);  // su: B(k0) = A(k1)
            const double szv = __dadd_rn(w0c.x, w1c.x);  // sv: B(k0) = A(k1)
            const double szw = __dadd_rn(w0c.x, w0c.y);  // sw: B(k0) = A(k1) (commuted)

            double su_a, sv_a, sw_a, su_b, sv_b, sw_b;
            if (NZC == 0 && (t.debug & 1)) {  // ablation (generic kernel): no PW arithmetic
                su_a = sv_a = sw_a = su_b = sv_b = sw_b =
                    (u0c.x + u0p.x) + (umc.x + u1c.x) + (v1c.x + w1c.x) + (wmc.x + vmp.x) +
                    (v0m.x + w0m.y) + (vmc.y + v0p.y) + (w0cM + w0pM) + (u0cQ + v0cQ) +
                    (w0cQ + vmcM) + (v0cM + w1cM) + (u0cM + w0p.x);
            } else {
                // level k0 (the top only for odd nz, UA; level 0 is identically zero).
                // pw_sums(x1, x2+x3, x4, x5+x6, y1, .., z1, z2+z3, z4, z5+z6)
                // with the operand wiring of kernel.py:117-128
                su_a = pw_sums<FMA>(tcx, tcy, c1a, c2a, u0m.x, sxu_a, u0p.x, nsxu_a,
                                    umc.x, __dadd_rn(vmc.x, vmp.x), u1c.x, __dadd_rn(v0c.x, v0p.x),
                                    u0cM, __dadd_rn(w0cM, w0pM), u0c.y, szu, top_a);
                sv_a = pw_sums<FMA>(tcx, tcy, c1a, c2a, v0m.x, txu_a, v0p.x, ntxu_a,
                                    vmc.x, __dadd_rn(v0c.x, vmc.x), v1c.x, __dadd_rn(v0c.x, v1c.x),
                                    v0cM, __dadd_rn(w0cM, w1cM), v0c.y, szv, top_a);
                sw_a = pw_sums<FMA>(tcx, tcy, c1a, c2a, w0m.x, rxu_a, w0p.x, nrxu_a,
                                    wmc.x, __dadd_rn(vmcM, vmc.x), w1c.x, __dadd_rn(v0cM, v0c.x),
                                    w0cM, __dadd_rn(w0c.x, w0cM), w0c.y, szw, top_a);
                // level k1 (the top when k1 == nz-1)
                su_b = pw_sums<FMA>(tcx, tcy, c1b, c2b, u0m.y, sxu_b, u0p.y, nsxu_b,
                                    umc.y, __dadd_rn(vmc.y, vmp.y), u1c.y, __dadd_rn(v0c.y, v0p.y),
                                    u0c.x, szu, u0cQ, __dadd_rn(w0c.y, w0p.y), top_b);
                sv_b = pw_sums<FMA>(tcx, tcy, c1b, c2b, v0m.y, txu_b, v0p.y, ntxu_b,
                                    vmc.y, __dadd_rn(v0c.y, vmc.y), v1c.y, __dadd_rn(v0c.y, v1c.y),
                                    v0c.x, szv, v0cQ, __dadd_rn(w0c.y, w1c.y), top_b);
                sw_b = pw_sums<FMA>(tcx, tcy, c1b, c2b, w0m.y, rxu_b, w0p.y, nrxu_b,
                                    wmc.y, __dadd_rn(vmc.x, vmc.y), w1c.y, __dadd_rn(v0c.x, v0c.y),
                                    w0c.x, szw, w0cQ, __dadd_rn(w0c.y, w0cQ), top_b);
            }
            sxu_a = nsxu_a;
            sxu_b = nsxu_b;
            txu_a = ntxu_a;
            txu_b = ntxu_b;
            rxu_a = nrxu_a;
            rxu_b = nrxu_b;
            if (lvl0) {
                su_a = 0.0;
                sv_a = 0.0;
                sw_a = 0.0;
            }
            if constexpr (STEP) {
                su_a = fwd_update(u0c.x, dt, su_a);
                su_b = fwd_update(u0c.y, dt, su_b);
                sv_a = fwd_update(v0c.x, dt, sv_a);
                sv_b = fwd_update(v0c.y, dt, sv_b);
                sw_a = fwd_update(w0c.x, dt, sw_a);
                sw_b = fwd_update(w0c.y, dt, sw_b);
            }
            if (active && !(NZC == 0 && (t.debug & 4))) {
                if constexpr (UA) {  // 8-byte-aligned pairs; odd nz: k1 may be past the column
                    __stcs(o0, su_a);
                    __stcs(o1, sv_a);
                    __stcs(o2, sw_a);
                    if (!top_a) {
                        __stcs(o0 + 1, su_b);
                        __stcs(o1 + 1, sv_b);
                        __stcs(o2 + 1, sw_b);
                    }
                } else {
                    store2(o0, su_a, su_b);
                    store2(o1, sv_a, sv_b);
                    store2(o2, sw_a, sw_b);
                }
            }
            if constexpr (STEP) {
                if (a.push && active) {
                    if (ci == 1 || ci == a.nx || a.ny == 1) {
                        if (ci == 1 || ci == a.nx || j0 + c == 1 || j0 + c == a.ny) {
                            if constexpr (UA)
                                push_pair_ua(&a, ci, j0 + c, k0, su_a, su_b, sv_a, sv_b, sw_a, sw_b);
                            else
                                push_pair(&a, ci, j0 + c, k0, su_a, su_b, sv_a, sv_b, sw_a, sw_b);
                        }
                    } else if (ydir >= 0) {
                        const int64_t off = (ci * ystr + ypj) * (int64_t)nz + k0;
                        if constexpr (UA) {
                            a.peers.u[ydir][off] = su_a;
                            a.peers.v[ydir][off] = sv_a;
                            a.peers.w[ydir][off] = sw_a;
                            if (!top_a) {
                                a.peers.u[ydir][off + 1] = su_b;
                                a.peers.v[ydir][off + 1] = sv_b;
                                a.peers.w[ydir][off + 1] = sw_b;
                            }
                        } else {
                            store2(a.peers.u[ydir] + off, su_a, su_b);
                            store2(a.peers.v[ydir] + off, sv_a, sv_b);
                            store2(a.peers.w[ydir] + off, sw_a, sw_b);
                        }
                    }
                }
            }
            ++ci;
            o0 += ostep;
            o1 += ostep;
            o2 += ostep;
            pst = lst;
            dC = dL;
            advance();
        };

        using R0 = std::integral_constant<int, 0>;
        using R1 = std::integral_constant<int, 1>;
        using R2 = std::integral_constant<int, 2>;
        const int nsteps = (int)(ie - ib);
        int n = 0;
        for (; n + 3 <= nsteps; n += 3) {
            body(R0{});
            body(R1{});
            body(R2{});
        }
        if (n < nsteps) {
            body(R0{});
            if (n + 1 < nsteps) body(R1{});
        }
        release(cseq - 1, pst);  // plane ie was only read as the x+1 plane
    }
}

}  // namespace pwadv

#include "pwadv_ctile.cuh"
