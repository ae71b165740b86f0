// pwadv_advect.cu — K1 (PW advection) and K4 (fused forward step) for sm_100a.
//
// Replaces the reference hot path run_reference -> compute_block ->
// su/sv/sw_formula (pkg/src/pwadvect/kernel.py:73-185). Two kernels:
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
//    not a contraction, no tensor cores.
//    Work distribution: the (strip, plane) space is split evenly over a
//    persistent grid of one CTA per SM; a CTA crossing a strip boundary just
//    continues its plane sequence (the ring never drains).
//
//  * k_advect_simple — one thread per output point, direct global loads. Used
//    for shapes the X-march does not cover (odd nz, misaligned pointers, very
//    tall columns), for thin rim boxes, and as an independent check.
//
// Both are bit-exact with the reference by construction (pwadv_device.cuh).
#include "pwadv_device.cuh"
#include "pwadv_internal.h"

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
};

struct TileCfg {
    int tj;           // columns per strip
    int kp;           // threads per column (= nz/2)
    int stages;       // ring depth
    int streaming;    // st.global.cs for outputs
    int64_t nstrips;  // ceil((y1-y0)/tj)
};

// ---------------------------------------------------------------------------
// simple kernel

template <bool FMA, bool STEP>
__global__ void __launch_bounds__(256) k_advect_simple(BoxArgs a)
{
    const int64_t nz = a.nz, ny2 = a.ny + 2;
    const int64_t nbx = a.x1 - a.x0, nby = a.y1 - a.y0;
    const int64_t total = nbx * nby * nz;
    const int64_t sI = ny2 * nz, sJ = nz;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = idx % nz;
        const int64_t col = idx / nz;
        const int64_t i = a.x0 + col / nby;
        const int64_t j = a.y0 + col % nby;
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
    }
}

// ---------------------------------------------------------------------------
// X-march kernel

// value at k0-1 of the thread's pair: the previous lane's k1, or (across a
// warp boundary inside a column) straight from the shared plane.
__device__ __forceinline__ double nbr_m(double2 p, const double *colp, int k0, bool fix)
{
    double m = __shfl_up_sync(0xffffffffu, p.y, 1);
    if (fix) m = colp[k0 - 1];
    return m;
}

// value at k0+2: the next lane's k0, or from the shared plane.
__device__ __forceinline__ double nbr_q(double2 p, const double *colp, int k0, bool fix)
{
    double q = __shfl_down_sync(0xffffffffu, p.x, 1);
    if (fix) q = colp[k0 + 2];
    return q;
}

template <bool FMA, bool STEP, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) k_advect_xmarch(BoxArgs a, TileCfg t)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int S = t.stages, TJ = t.tj, KP = t.kp;
    const int nz = (int)a.nz;
    const int CS = (TJ + 2) * nz;  // doubles per field per tile-plane
    double *ring = reinterpret_cast<double *>(smem_raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem_raw + (size_t)S * 3 * CS * sizeof(double));
    uint64_t *empty = full + S;

    const int tid = threadIdx.x, lane = tid & 31;
    const int nwarps = blockDim.x >> 5;
    const bool in_tile = tid < TJ * KP;
    const int c = in_tile ? tid / KP : TJ - 1;
    const int kp = in_tile ? tid - (tid / KP) * KP : 0;
    const int k0 = 2 * kp, k1 = k0 + 1;
    const bool fixM = (lane == 0) && kp > 0;
    const bool fixQ = (lane == 31) && kp < KP - 1;
    const bool top_b = (k1 == nz - 1);
    const bool lvl0 = (k0 == 0);

    const double tcx = a.tcx, tcy = a.tcy, dt = a.dt;
    const double c1a = __ldg(a.tzc1 + k0), c1b = __ldg(a.tzc1 + k1);
    const double c2a = __ldg(a.tzc2 + k0), c2b = __ldg(a.tzc2 + k1);

    const int64_t ny2 = a.ny + 2;
    const int64_t nxr = a.x1 - a.x0;
    const int64_t W = t.nstrips * nxr;
    const int64_t wb = (W * (int64_t)blockIdx.x) / gridDim.x;
    const int64_t we = (W * (int64_t)(blockIdx.x + 1)) / gridDim.x;
    if (wb >= we) return;
    const int64_t sb0 = wb / nxr, sb1 = (we - 1) / nxr;
    const int total = (int)((we - wb) + 2 * (sb1 - sb0 + 1));  // planes this CTA streams

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], nwarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    // ---- producer state (thread 0 only) --------------------------------
    int pseq = 0;
    int64_t p_strip = sb0, p_plane = 0, p_end = 0;
    auto seg_ib = [&](int64_t s) { return a.x0 + (wb - s * nxr > 0 ? wb - s * nxr : 0); };
    auto seg_ie = [&](int64_t s) { return a.x0 + (we - s * nxr < nxr ? we - s * nxr : nxr); };
    if (tid == 0) {
        p_plane = seg_ib(sb0) - 1;
        p_end = seg_ie(sb0);
    }
    auto issue = [&]() {
        const int st = (int)(pseq % S);
        if (pseq >= S) mbar_wait(&empty[st], (uint32_t)(((pseq / S) - 1) & 1));
        const int64_t j0 = a.y0 + p_strip * TJ;
        const int64_t tjs = (a.y1 - j0) < TJ ? (a.y1 - j0) : TJ;
        const uint32_t bytes = (uint32_t)((tjs + 2) * nz * sizeof(double));
        mbar_arrive_expect_tx(&full[st], 3 * bytes);
        const int64_t off = (p_plane * ny2 + (j0 - 1)) * nz;
        double *dst = ring + (size_t)st * 3 * CS;
        bulk_g2s(dst, a.u + off, bytes, &full[st]);
        bulk_g2s(dst + CS, a.v + off, bytes, &full[st]);
        bulk_g2s(dst + 2 * CS, a.w + off, bytes, &full[st]);
        ++pseq;
        if (++p_plane > p_end) {
            ++p_strip;
            if (p_strip <= sb1) {
                p_plane = seg_ib(p_strip) - 1;
                p_end = seg_ie(p_strip);
            }
        }
    };
    if (tid == 0) {
        const int n0 = total < S ? total : S;
        for (int n = 0; n < n0; ++n) issue();
    }
    // warp 0 releases planes in sequence order; after each release thread 0
    // refills the stage released one step earlier (keeps S-3 planes in flight
    // beyond the next one without stalling on the slowest warp).
    auto release = [&](int seq) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[seq % S]);
        if (tid == 0) {
            while (pseq < total && pseq <= seq - 1 + S) issue();
        }
    };
    auto wait_full = [&](int seq) -> const double * {
        const int st = (int)(seq % S);
        mbar_wait(&full[st], (uint32_t)((seq / S) & 1));
        return ring + (size_t)st * 3 * CS;
    };
    // pair (k0, k0+1) of field f, column offset dy, in a staged plane
    auto P = [&](const double *pl, int f, int dy) -> double2 {
        return *reinterpret_cast<const double2 *>(pl + f * CS + (c + 1 + dy) * nz + k0);
    };
    auto colp = [&](const double *pl, int f, int dy) -> const double * {
        return pl + f * CS + (c + 1 + dy) * nz;
    };

    int cseq = 0;
    for (int64_t s = sb0; s <= sb1; ++s) {
        const int64_t ib = seg_ib(s), ie = seg_ie(s);
        const int64_t j0 = a.y0 + s * TJ;
        const int64_t tjs = (a.y1 - j0) < TJ ? (a.y1 - j0) : TJ;
        const bool active = in_tile && c < tjs;

        // plane ib-1: the x-1 window
        const double *pl = wait_full(cseq);
        double2 u0m = P(pl, 0, 0), u1m = P(pl, 0, 1), v0m = P(pl, 1, 0), w0m = P(pl, 2, 0);
        double u0mM = nbr_m(u0m, colp(pl, 0, 0), k0, fixM);
        release(cseq);
        ++cseq;
        // plane ib: the x window (leading items)
        pl = wait_full(cseq);
        double2 u0c = P(pl, 0, 0), v0c = P(pl, 1, 0), w0c = P(pl, 2, 0), vmc = P(pl, 1, -1);
        double w0cM = nbr_m(w0c, colp(pl, 2, 0), k0, fixM);
        ++cseq;

        int64_t obase = (ib * ny2 + (j0 + c)) * (int64_t)nz + k0;
        const int64_t ostep = ny2 * nz;
        const int nsteps = (int)(ie - ib);
        for (int n = 0; n < nsteps; ++n, obase += ostep) {
            const double *L = wait_full(cseq);                       // plane i+1
            const double *C = ring + (size_t)((cseq - 1) % S) * 3 * CS;  // plane i
            const double2 u0p = P(L, 0, 0), v0p = P(L, 1, 0), w0p = P(L, 2, 0), vmp = P(L, 1, -1);
            const double w0pM = nbr_m(w0p, colp(L, 2, 0), k0, fixM);
            const double2 u1c = P(C, 0, 1), umc = P(C, 0, -1), v1c = P(C, 1, 1);
            const double2 w1c = P(C, 2, 1), wmc = P(C, 2, -1);
            const double w1cM = nbr_m(w1c, colp(C, 2, 1), k0, fixM);
            const double u0cM = nbr_m(u0c, colp(C, 0, 0), k0, fixM);
            const double u0cQ = nbr_q(u0c, colp(C, 0, 0), k0, fixQ);
            const double v0cM = nbr_m(v0c, colp(C, 1, 0), k0, fixM);
            const double v0cQ = nbr_q(v0c, colp(C, 1, 0), k0, fixQ);
            const double w0cQ = nbr_q(w0c, colp(C, 2, 0), k0, fixQ);
            const double vmcM = nbr_m(vmc, colp(C, 1, -1), k0, fixM);
            release(cseq - 1);  // plane i fully consumed by this warp

            // level k0 (never the top; level 0 is identically zero)
            double su_a = su_formula<FMA>(tcx, tcy, c1a, c2a, u0c.x, u0m.x, u0p.x, umc.x, u1c.x,
                                          u0cM, u0c.y, vmc.x, vmp.x, v0c.x, v0p.x, w0cM, w0pM,
                                          w0c.x, w0p.x, false);
            double sv_a = sv_formula<FMA>(tcx, tcy, c1a, c2a, v0c.x, v0m.x, v0p.x, vmc.x, v1c.x,
                                          v0cM, v0c.y, u0m.x, u1m.x, u0c.x, u1c.x, w0cM, w1cM,
                                          w0c.x, w1c.x, false);
            double sw_a = sw_formula<FMA>(tcx, tcy, c1a, c2a, w0c.x, w0m.x, w0p.x, wmc.x, w1c.x,
                                          w0cM, w0c.y, u0mM, u0m.x, u0cM, u0c.x, vmcM, vmc.x,
                                          v0cM, v0c.x, false);
            // level k1 (the top when k1 == nz-1)
            double su_b = su_formula<FMA>(tcx, tcy, c1b, c2b, u0c.y, u0m.y, u0p.y, umc.y, u1c.y,
                                          u0c.x, u0cQ, vmc.y, vmp.y, v0c.y, v0p.y, w0c.x, w0p.x,
                                          w0c.y, w0p.y, top_b);
            double sv_b = sv_formula<FMA>(tcx, tcy, c1b, c2b, v0c.y, v0m.y, v0p.y, vmc.y, v1c.y,
                                          v0c.x, v0cQ, u0m.y, u1m.y, u0c.y, u1c.y, w0c.x, w1c.x,
                                          w0c.y, w1c.y, top_b);
            double sw_b = sw_formula<FMA>(tcx, tcy, c1b, c2b, w0c.y, w0m.y, w0p.y, wmc.y, w1c.y,
                                          w0c.x, w0cQ, u0m.x, u0m.y, u0c.x, u0c.y, vmc.x, vmc.y,
                                          v0c.x, v0c.y, top_b);
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
            if (active) {
                store2(a.o0 + obase, su_a, su_b, t.streaming);
                store2(a.o1 + obase, sv_a, sv_b, t.streaming);
                store2(a.o2 + obase, sw_a, sw_b, t.streaming);
            }
            // roll the x window
            u0m = u0c;
            u0mM = u0cM;
            u0c = u0p;
            u1m = u1c;
            v0m = v0c;
            v0c = v0p;
            w0m = w0c;
            w0c = w0p;
            w0cM = w0pM;
            vmc = vmp;
            ++cseq;
        }
        release(cseq - 1);  // plane ie was only read as the x+1 plane
    }
}

// ---------------------------------------------------------------------------
// host-side planning and launch

static int round_up(int x, int m) { return (x + m - 1) / m * m; }

int launch_box(const BoxLaunch &L, cudaStream_t stream)
{
    BoxArgs a;
    a.u = L.u;
    a.v = L.v;
    a.w = L.w;
    a.o0 = L.o0;
    a.o1 = L.o1;
    a.o2 = L.o2;
    a.tzc1 = L.tzc1;
    a.tzc2 = L.tzc2;
    a.nx = L.nx;
    a.ny = L.ny;
    a.nz = L.nz;
    a.tcx = L.tcx;
    a.tcy = L.tcy;
    a.dt = L.dt;
    a.x0 = L.x0;
    a.x1 = L.x1;
    a.y0 = L.y0;
    a.y1 = L.y1;
    const bool fma = (L.flags & PWADV_FLAG_FMA) != 0;
    const int64_t nbx = L.x1 - L.x0, nby = L.y1 - L.y0;
    if (nbx <= 0 || nby <= 0) return PWADV_OK;

    const DeviceInfo *dev = device_info();
    if (!dev) return PWADV_E_CUDA;

    XmarchPlan plan;
    const bool tiled = plan_xmarch(L, *dev, &plan);
    if (tiled) {
        TileCfg t;
        t.tj = plan.tj;
        t.kp = plan.kp;
        t.stages = plan.stages;
        t.streaming = (L.flags & PWADV_FLAG_NO_STREAMING) ? 0 : 1;
        t.nstrips = plan.nstrips;
        void (*kern)(BoxArgs, TileCfg) = nullptr;
#define PWADV_PICK(MT)                                                                      \
    if (plan.maxt == MT) {                                                                  \
        if (L.step)                                                                         \
            kern = fma ? k_advect_xmarch<true, true, MT> : k_advect_xmarch<false, true, MT>; \
        else                                                                                \
            kern = fma ? k_advect_xmarch<true, false, MT> : k_advect_xmarch<false, false, MT>; \
    }
        PWADV_PICK(512)
        PWADV_PICK(384)
        PWADV_PICK(256)
#undef PWADV_PICK
        if (!kern) return set_error(PWADV_E_ARG, "unsupported thread budget %d", plan.maxt);
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)plan.smem);
        if (e != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute", e);
        kern<<<plan.grid, plan.threads, plan.smem, stream>>>(a, t);
    } else {
        const int64_t total = nbx * nby * L.nz;
        int64_t blocks = (total + 255) / 256;
        const int64_t cap = (int64_t)dev->sms * 8;
        if (blocks > cap) blocks = cap;
        if (blocks < 1) blocks = 1;
        if (L.step) {
            if (fma)
                k_advect_simple<true, true><<<(unsigned)blocks, 256, 0, stream>>>(a);
            else
                k_advect_simple<false, true><<<(unsigned)blocks, 256, 0, stream>>>(a);
        } else {
            if (fma)
                k_advect_simple<true, false><<<(unsigned)blocks, 256, 0, stream>>>(a);
            else
                k_advect_simple<false, false><<<(unsigned)blocks, 256, 0, stream>>>(a);
        }
    }
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error("advect launch", e);
    return PWADV_OK;
}

bool plan_xmarch(const BoxLaunch &L, const DeviceInfo &dev, XmarchPlan *p)
{
    if (L.flags & PWADV_FLAG_SIMPLE) return false;
    const int64_t nz = L.nz;
    if (nz % 2 != 0 || nz > 1024) return false;
    // 16-byte alignment for the bulk copies and the paired loads/stores
    const uintptr_t al = (uintptr_t)L.u | (uintptr_t)L.v | (uintptr_t)L.w | (uintptr_t)L.o0 |
                         (uintptr_t)L.o1 | (uintptr_t)L.o2;
    if (al & 15) return false;
    const int kp = (int)(nz / 2);
    const int64_t nby = L.y1 - L.y0, nbx = L.x1 - L.x0;
    // thread budget per CTA (register file / CTA): 384 by default, which
    // leaves ~168 registers per thread for the rolled x-window
    int maxt = L.max_threads > 0 ? L.max_threads : 384;
    if (maxt != 512 && maxt != 384 && maxt != 256) return false;
    if (kp > maxt) return false;
    int tj = L.tile_j > 0 ? L.tile_j : maxt / kp;
    if (tj > maxt / kp) tj = maxt / kp;
    if (tj < 1) return false;
    if (tj > nby) tj = (int)nby;
    const size_t bar_bytes = 2 * 16 * sizeof(uint64_t);
    const size_t smem_cap = (size_t)dev.smem_optin - bar_bytes - 1024;
    int stages = 0;
    for (;;) {
        const size_t stage_bytes = (size_t)3 * (tj + 2) * nz * sizeof(double);
        int smax = (int)(smem_cap / stage_bytes);
        if (smax > 8) smax = 8;
        stages = L.stages > 0 ? (L.stages < smax ? L.stages : smax) : smax;
        if (stages >= 3) break;
        if (tj == 1) return false;
        tj = tj / 2;
    }
    p->maxt = maxt;
    p->tj = tj;
    p->kp = kp;
    p->stages = stages;
    p->threads = round_up(tj * kp, 32);
    p->smem = (size_t)stages * 3 * (tj + 2) * nz * sizeof(double) + 2 * stages * sizeof(uint64_t);
    p->nstrips = (nby + tj - 1) / tj;
    const int64_t work = p->nstrips * nbx;
    int64_t grid = L.grid > 0 ? L.grid : (int64_t)dev.sms;  // one resident CTA per SM
    const int64_t min_planes = 4;
    int64_t cap = (work + min_planes - 1) / min_planes;
    if (L.grid <= 0 && grid > cap) grid = cap;
    if (grid > work) grid = work;
    if (grid < 1) grid = 1;
    p->grid = (int)grid;
    return true;
}

}  // namespace pwadv
