// pwadv_ctile.cuh — K1c: the X-march with column tiles (k-slabs), included at
// the end of pwadv_xmarch.cuh (it shares BoxArgs, TileCfg, unit_at, RingState
// and the ring protocol with k_advect_xmarch); instantiated in pwadv_k_ct*.cu.
//
// k_advect_xmarch stages a whole column height per plane tile, so deep
// columns shrink its strip (TJ = 384 / (nz/2): nz = 512 leaves one column per
// CTA and three staged columns per computed one) and nz > 768 does not fit
// the ring at all (it ran on K1m, ~60% of HBM). Here a work unit is (X chunk,
// y-strip, k-slab): the CTA's tile is TJ columns x KT levels, KT a compile-
// time 32 / 48 / 64 / 96 / 128 (TJ = 768 / KT), and each plane tile of a field is ONE
// 3-D tensor-map TMA box (cp.async.bulk.tensor, SASS UTMALDG) of KT + 4
// levels x TJ + 2 columns x 1 plane starting at level kb - 2 — the hardware
// walks the TJ + 2 column runs and zero-fills levels outside [0, nz) and
// columns past ny + 1. (One 1-D bulk copy per staged column was measured
// first: ~100 cycles per request per SM capped it at 40-60% of HBM.) The box
// lands densely, a slot of CW = KT + 4 doubles per column, so thread kp's
// pair (kb + 2kp, kb + 2kp + 1) sits at slot index s0 = 2 + 2kp — 16-byte
// aligned; k +- 1 operands come from the neighbouring lanes by shuffles and,
// at the slab edges, from the slot's halo levels. Slabs per column =
// ceil(nz / KT); a partial last slab's extra threads compute on the zero
// fill and store nothing. Arithmetic, operand wiring and the x-carried sums
// are k_advect_xmarch's (bit-exact with kernel.py:73-185).
//
// Odd nz (ODD): the column stride nz * 8 is not a 16-byte multiple, so the
// field is mapped as rows of column pairs instead (see k_advect_ctile).
//
// Requirements (plan_ctile): 16-byte-aligned fields, no halo pull / push.

#include <cuda.h>

#ifndef PWADV_CT_REALIGN_LDS
#define PWADV_CT_REALIGN_LDS 1  // odd columns (odd nz): two 8-byte shared loads (default; 0 = the
                                // 16-byte load + shuffle: 5-15% slower, profiles/r02_ct_odd_nz.jsonl)
#endif
#ifndef PWADV_CT_SHIFTED
#define PWADV_CT_SHIFTED 1  // odd nz, fixed column parity: odd columns' pairs at odd levels (A/B switch)
#endif
#ifndef PWADV_CT_DBG
#define PWADV_CT_DBG 0  // debug builds only (tools/build_variant.py): 1 = odd nz loads one half, 2 = no stores
#endif

namespace pwadv {

template <int KT, bool ODD>
struct CtLayout {
    static constexpr int KP = KT / 2;       // threads per column slab
    static constexpr int TJ = 384 / KP;     // columns per strip
    static constexpr int CW = KT + 4;       // doubles per staged column (slot)
    static constexpr int NC = TJ + 2;       // staged columns per field
    // odd nz: column-pair rows, even and odd global columns in two halves
    static constexpr int NP = TJ / 2 + 2;   // pair rows per box (covers NC columns at any phase)
    static constexpr int HALF = (NP * CW + 15) / 16 * 16;  // second half's offset (128-byte aligned:
                                                           // a tensor copy's destination must be)
    static constexpr int BOX = ODD ? 2 * NP * CW : NC * CW;  // doubles a field's plane tile delivers
    static constexpr int SPAN = ODD ? HALF + NP * CW : NC * CW;
    static constexpr int CS = (SPAN + 15) / 16 * 16;  // doubles per field slot (128-byte multiple)
    static_assert(KT % 2 == 0 && 384 % KP == 0 && NC <= 64 && TJ % 2 == 0, "column-tile layout");
};

// the three fields' tensor maps: even nz dims {nz, ny+2, nx+2}, box {KT+4,
// TJ+2, 1}; odd nz (column-pair rows) dims {2 nz, (nx+2)(ny+2)/2}, box {KT+4, NP}
struct CtMaps {
    CUtensorMap u, v, w;
};

__device__ __forceinline__ void tma_load_3d(void *dst_smem, const CUtensorMap *map, int c0, int c1,
                                            int c2, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(dst_smem)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2),
        "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void *dst_smem, const CUtensorMap *map, int c0, int c1,
                                            uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];"
        ::"r"(smem_u32(dst_smem)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1),
        "r"(smem_u32(bar))
        : "memory");
}

// ODD (odd nz): a field is viewed as rows of column PAIRS — global columns
// g = i*(ny+2) + j, row g/2 holding columns 2r and 2r+1, 2 nz levels, a
// 16-byte-multiple row stride — and a plane tile is two boxes per field of NP
// pair rows from row G0/2 (G0 = the tile's first global column), landing in
// two halves of the slot: the even columns' levels [kb-2, kb+KT+2) (inner
// start kb - 2) and the odd columns' levels [kb-3, kb+KT+1) (inner start
// nz + kb - 3: a box row must start on a 16-byte boundary, so an odd column's
// staged copy sits one level higher in its slot). A tile column's half and row
// follow from the parity of G0, which flips from plane to plane when ny+2 is
// odd, so the consumers select their column offsets per plane. Two pairings
// (run_unit's QV): when ny+2 is even a column's parity is fixed over a unit
// and an odd column's pairs start at odd levels (kb - 1 + 2kp) — its own pairs
// and all stores are on the 16-byte grid, only the neighbouring columns' pairs
// are off it (slot shift -1 / +1), read with two 8-byte loads; when ny+2 is odd
// every pair starts at an even level (kb + 2kp) and an odd column's own pairs
// are off the grid (8-byte loads, scalar stores). Either choice is warp-
// uniform (one column parity owns a warp: KT 64 / 128, plan_ctile). The top
// level nz - 1 is the first or second level of its pair, level 0 may be a
// shifted pair's second level (the first, level -1, is not stored). Levels a
// box reads past its column (the other column of the pair, or the zero fill)
// feed only operands of levels that are not stored, the zeroed level 0, or the
// top formula's unread k+1.
template <bool FMA, bool STEP, int KT, bool ODD>
__global__ void __launch_bounds__(512, 1)
    k_advect_ctile(const __grid_constant__ BoxArgs a, const __grid_constant__ TileCfg t,
                   const __grid_constant__ CtMaps maps)
{
    using Lay = CtLayout<KT, ODD>;
    constexpr int KP = Lay::KP, TJ = Lay::TJ, CW = Lay::CW, CS = Lay::CS, HALF = Lay::HALF;
    constexpr int kComputeWarps = 12;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int S = t.stages;
    double *ring = reinterpret_cast<double *>(smem_raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem_raw + (size_t)S * 3 * CS * sizeof(double));
    uint64_t *empty = full + S;
    RingState *rs = reinterpret_cast<RingState *>(full + 2 * S);

    const int tid = threadIdx.x, lane = tid & 31;
    const int c = tid / KP;             // interior column of the strip (compute threads)
    const int kp = tid - c * KP;
    const int tc = c + 1;               // its staged column
    const int s0 = 2 + 2 * kp;          // slot index of the pair
    const bool fixM = (kp == 0) || (lane == 0);        // k0-1 from the slot, not a shuffle
    const bool fixQ = (kp == KP - 1) || (lane == 31);  // k0+2 likewise
    const int64_t nz = a.nz, ny2 = a.ny + 2;
    const double tcx = a.tcx, tcy = a.tcy, dt = a.dt;
    const int64_t nslab = t.nslab;      // k-slabs per column

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
            if (w.ie <= w.ib) continue;
            const int64_t sy = w.strip / nslab, sl = w.strip - sy * nslab;
            const int64_t j0 = a.y0 + sy * TJ;
            const int64_t tjs = (a.y1 - j0) < TJ ? (a.y1 - j0) : TJ;
            rs->first[k] = q;
            rs->ui0[k] = (int32_t)(w.ib - 1);
            rs->uj0[k] = (int32_t)j0;
            rs->utj[k] = (int32_t)tjs;
            rs->dsto[k] = (int32_t)(sl * KT);  // the slab's nominal first level
            q += (int)(w.ie - w.ib + 2);
            ++k;
        }
        rs->first[k] = q;
        rs->total = q;
        rs->nunits = k;
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kComputeWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");  // inputs final from here on
    const int total = rs->total;
    const int my_units = rs->nunits;

    if (tid >= 32 * kComputeWarps) {  // producer warpgroup: warp 12 issues, 13-15 idle
        asm volatile("setmaxnreg.dec.sync.aligned.u32 32;\n" ::: "memory");
        if (tid == 32 * kComputeWarps) {  // one thread: three (odd nz: six) boxes per plane
#if PWADV_CT_DBG & 1
            constexpr uint32_t kBox = (uint32_t)((ODD ? Lay::BOX / 2 : Lay::BOX) * sizeof(double));
#else
            constexpr uint32_t kBox = (uint32_t)(Lay::BOX * sizeof(double));
#endif
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.u)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.v)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.w)) : "memory");
            int k = 0;
            for (int q = 0; q < total; ++q) {
                while (rs->first[k + 1] <= q) ++k;
                const int st = q % S;
                if (q >= S) mbar_wait(&empty[st], (uint32_t)(((q / S) - 1) & 1));
                fence_proxy_async();
                const int i = rs->ui0[k] + (q - rs->first[k]);
                const int jl = rs->uj0[k] - 1, kl = rs->dsto[k] - 2;
                double *dst = ring + (size_t)st * 3 * CS;
                mbar_arrive_expect_tx(&full[st], 3 * kBox);
                if constexpr (ODD) {
                    const int r0 = (int)(((int64_t)i * ny2 + jl) >> 1);
                    const int ko = (int)nz + kl - 1;  // even: 16-byte-aligned box rows
                    tma_load_2d(dst, &maps.u, kl, r0, &full[st]);
                    tma_load_2d(dst + CS, &maps.v, kl, r0, &full[st]);
                    tma_load_2d(dst + 2 * CS, &maps.w, kl, r0, &full[st]);
#if PWADV_CT_DBG & 1
                    (void)ko;
#else
                    tma_load_2d(dst + HALF, &maps.u, ko, r0, &full[st]);
                    tma_load_2d(dst + CS + HALF, &maps.v, ko, r0, &full[st]);
                    tma_load_2d(dst + 2 * CS + HALF, &maps.w, ko, r0, &full[st]);
#endif
                } else {
                    tma_load_3d(dst, &maps.u, kl, jl, i, &full[st]);
                    tma_load_3d(dst + CS, &maps.v, kl, jl, i, &full[st]);
                    tma_load_3d(dst + 2 * CS, &maps.w, kl, jl, i, &full[st]);
                }
            }
        }
        return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 160;\n" ::: "memory");

    int cseq = 0, cst = 0;
    uint32_t cph = 0;
    // column offsets (doubles) of the thread's column and its j -+ 1
    // neighbours in a staged plane whose first global column has parity pg
    auto coff = [&](int pg, int dy) -> int {
        if constexpr (ODD) {
            const int x = pg + tc + dy;
            return (x & 1) * HALF + (x >> 1) * CW;
        } else {
            (void)pg;
            return (tc + dy) * CW;
        }
    };
    const int e_m = coff(0, -1), e_z = coff(0, 0), e_p = coff(0, 1);
    const int o_m = coff(1, -1), o_z = coff(1, 0), o_p = coff(1, 1);
    const int podd = ODD ? (int)(ny2 & 1) : 0;  // G0's parity flips from plane to plane
    auto release = [&](int st) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    };
    auto wait_next = [&]() -> const double * {
        mbar_wait(&full[cst], cph);
        return ring + (size_t)cst * 3 * CS;
    };
    auto advance = [&]() {
        ++cseq;
        if (++cst == S) {
            cst = 0;
            cph ^= 1u;
        }
    };
    // pl: a staged plane advanced to the column's slot; f: field; sh: where
    // the pair sits relative to slot index s0 (odd nz only, warp-uniform):
    // 0 = on the 16-byte grid, +-1 = one level up / down (an odd column's
    // copy sits one level higher in its slot) — read with two 8-byte loads
    auto P = [&](const double *pl, int f, int sh) -> double2 {
        if (ODD && sh) {
#if PWADV_CT_REALIGN_LDS
            return make_double2(pl[f * CS + s0 + sh], pl[f * CS + s0 + sh + 1]);
#else
            const double2 x = *reinterpret_cast<const double2 *>(pl + f * CS + s0 + sh - 1);
            double d = __shfl_down_sync(0xffffffffu, x.x, 1);
            if (fixQ) d = pl[f * CS + s0 + sh + 1];
            return make_double2(x.y, d);
#endif
        }
        return *reinterpret_cast<const double2 *>(pl + f * CS + s0);
    };
    // k0-1 / k0+2 of the pair: the neighbouring lane's value, or the slot's
    auto M = [&](double2 p, const double *pl, int f, int sh) -> double {
        double m = __shfl_up_sync(0xffffffffu, p.y, 1);
        if (fixM) m = pl[f * CS + s0 - 1 + sh];
        return m;
    };
    auto Q = [&](double2 p, const double *pl, int f, int sh) -> double {
        double v = __shfl_down_sync(0xffffffffu, p.x, 1);
        if (fixQ) v = pl[f * CS + s0 + 2 + sh];
        return v;
    };

    double2 U0[3], V0[3], W0[3], VM[3];
    double W0M[3];
    double sxu_a, sxu_b, txu_a, txu_b, rxu_a, rxu_b;

    for (int k = 0; k < my_units; ++k) {
        const int64_t ib = (int64_t)rs->ui0[k] + 1;
        const int64_t ie = ib + (rs->first[k + 1] - rs->first[k]) - 2;
        const int64_t j0 = rs->uj0[k];
        const bool active = c < rs->utj[k];
        // parity of the first global column of plane ib-1's tile
        int pg = ODD ? (int)((((ib - 1) * ny2) + (j0 - 1)) & 1) : 0;

        // the unit's steps, specialised on the parity of the thread's global
        // column (odd nz): QV 0 / 1 when it is the same on every plane of the
        // unit (ny+2 even; warp-uniform), 2 when it alternates from plane to
        // plane, -1 for even nz — so the realignment and store choices of the
        // common cases are compile-time
        auto run_unit = [&](auto QVC) {
            constexpr int QV = decltype(QVC)::value;
            // odd nz, column parity fixed over the unit: an odd column's pairs
            // start at odd levels (kb - 1 + 2kp), on the 16-byte grid in its
            // slot and in global memory; only the neighbouring columns' pairs
            // are off it (slot shift -1 / +1). Otherwise every pair starts at
            // an even level and an odd column's own pairs are off the grid.
            constexpr bool SS = PWADV_CT_SHIFTED && ODD && (QV == 0 || QV == 1);
            const int pflip = QV == 2 ? podd : 0;
            // this thread's levels in this slab (even nz: a pair is in or out
            // whole, the top is a pair's second level; odd nz: either)
            const int64_t k0 = (int64_t)rs->dsto[k] + 2 * kp - (SS && QV == 1 ? 1 : 0);
            const bool va = (!SS || k0 >= 0) && k0 < nz, vb = k0 + 1 < nz;
            const bool top_a = ODD && k0 == nz - 1, top_b = k0 + 1 == nz - 1;
            const bool z_a = k0 == 0, z_b = SS && k0 == -1;
            const int64_t kia = k0 < 0 ? 0 : (k0 < nz ? k0 : nz - 1);  // coefficient levels (clamped)
            const int64_t kib = k0 + 1 < nz ? k0 + 1 : nz - 1;
            const double c1a = __ldg(a.tzc1 + kia), c1b = __ldg(a.tzc1 + kib);
            const double c2a = __ldg(a.tzc2 + kia), c2b = __ldg(a.tzc2 + kib);
            // slot shifts of the thread's own column and of its neighbours
            auto sh_own = [&](int q) -> int { return SS ? 0 : q; };
            auto sh_nbr = [&](int q) -> int { return SS ? (QV == 1 ? -1 : 1) : (ODD ? q ^ 1 : 0); };
            auto qof = [&](int pgx) -> int {
                if constexpr (QV < 0) {
                    (void)pgx;
                    return 0;
                } else if constexpr (QV < 2) {
                    (void)pgx;
                    return QV;
                } else {
                    return (pgx + tc) & 1;
                }
            };
            {  // plane ib-1 -> slot 2
                const double *pl = wait_next();
                const double *pz = pl + (pg ? o_z : e_z), *pp = pl + (pg ? o_p : e_p);
                const int qz = sh_own(qof(pg)), qn = sh_nbr(qof(pg));  // slot shifts: own / neighbours
                U0[2] = P(pz, 0, qz);
                const double2 u1 = P(pp, 0, qn);
                V0[2] = P(pz, 1, qz);
                W0[2] = P(pz, 2, qz);
                const double u0M = M(U0[2], pz, 0, qz);
                release(cst);
                advance();
                txu_a = __dadd_rn(U0[2].x, u1.x);
                txu_b = __dadd_rn(U0[2].y, u1.y);
                rxu_a = __dadd_rn(u0M, U0[2].x);
                rxu_b = __dadd_rn(U0[2].x, U0[2].y);
            }
            int pst = cst;
            pg ^= pflip;
            {  // plane ib -> slot 0
                const double *pl = wait_next();
                const double *pz = pl + (pg ? o_z : e_z), *pm = pl + (pg ? o_m : e_m);
                const int qz = sh_own(qof(pg)), qn = sh_nbr(qof(pg));
                U0[0] = P(pz, 0, qz);
                V0[0] = P(pz, 1, qz);
                W0[0] = P(pz, 2, qz);
                VM[0] = P(pm, 1, qn);
                W0M[0] = M(W0[0], pz, 2, qz);
                advance();
                sxu_a = __dadd_rn(U0[0].x, U0[2].x);
                sxu_b = __dadd_rn(U0[0].y, U0[2].y);
            }

            const int64_t obase = (ib * ny2 + (j0 + c)) * nz + k0;
            double *o0 = a.o0 + obase;
            double *o1 = a.o1 + obase;
            double *o2 = a.o2 + obase;
            const int64_t ostep = ny2 * nz;

            auto body = [&](auto R) {
                constexpr int r = decltype(R)::value;
                constexpr int rm = (r + 2) % 3, rp = (r + 1) % 3;
                const int lst = cst;
                const double *L = wait_next();                       // plane i+1
                const double *C = ring + (size_t)pst * 3 * CS;      // plane i
                const int pgl = pg ^ pflip;
                const double *Lz = L + (pgl ? o_z : e_z), *Lm = L + (pgl ? o_m : e_m);
                const double *Cz = C + (pg ? o_z : e_z), *Cm = C + (pg ? o_m : e_m);
                const double *Cp = C + (pg ? o_p : e_p);
                const int lq = sh_own(qof(pgl)), lqn = sh_nbr(qof(pgl));  // plane i+1
                const int cq = sh_own(qof(pg)), cqn = sh_nbr(qof(pg));    // plane i
                U0[rp] = P(Lz, 0, lq);
                V0[rp] = P(Lz, 1, lq);
                W0[rp] = P(Lz, 2, lq);
                VM[rp] = P(Lm, 1, lqn);
                W0M[rp] = M(W0[rp], Lz, 2, lq);
                const double2 u1c = P(Cp, 0, cqn);
                const double2 umc = P(Cm, 0, cqn), v1c = P(Cp, 1, cqn), w1c = P(Cp, 2, cqn), wmc = P(Cm, 2, cqn);
                const double w1cM = M(w1c, Cp, 2, cqn);
                const double u0cM = M(U0[r], Cz, 0, cq);
                const double u0cQ = Q(U0[r], Cz, 0, cq);
                const double v0cM = M(V0[r], Cz, 1, cq);
                const double v0cQ = Q(V0[r], Cz, 1, cq);
                const double w0cQ = Q(W0[r], Cz, 2, cq);
                const double vmcM = M(VM[r], Cm, 1, cqn);
                release(pst);  // plane i fully consumed by this warp

                const double2 u0m = U0[rm], u0c = U0[r], u0p = U0[rp];
                const double2 v0m = V0[rm], v0c = V0[r], v0p = V0[rp];
                const double2 w0m = W0[rm], w0c = W0[r], w0p = W0[rp];
                const double2 vmc = VM[r], vmp = VM[rp];
                const double w0cM = W0M[r], w0pM = W0M[rp];

                const double nsxu_a = __dadd_rn(u0c.x, u0p.x), nsxu_b = __dadd_rn(u0c.y, u0p.y);
                const double ntxu_a = __dadd_rn(u0c.x, u1c.x), ntxu_b = __dadd_rn(u0c.y, u1c.y);
                const double nrxu_a = __dadd_rn(u0cM, u0c.x), nrxu_b = __dadd_rn(u0c.x, u0c.y);
                const double szu = __dadd_rn(w0c.x, w0p.x);
                const double szv = __dadd_rn(w0c.x, w1c.x);
                const double szw = __dadd_rn(w0c.x, w0c.y);

                // the operand wiring of kernel.py:117-128, as k_advect_xmarch
                double su_a = pw_sums<FMA>(tcx, tcy, c1a, c2a, u0m.x, sxu_a, u0p.x, nsxu_a,
                                           umc.x, __dadd_rn(vmc.x, vmp.x), u1c.x, __dadd_rn(v0c.x, v0p.x),
                                           u0cM, __dadd_rn(w0cM, w0pM), u0c.y, szu, top_a);
                double sv_a = pw_sums<FMA>(tcx, tcy, c1a, c2a, v0m.x, txu_a, v0p.x, ntxu_a,
                                           vmc.x, __dadd_rn(v0c.x, vmc.x), v1c.x, __dadd_rn(v0c.x, v1c.x),
                                           v0cM, __dadd_rn(w0cM, w1cM), v0c.y, szv, top_a);
                double sw_a = pw_sums<FMA>(tcx, tcy, c1a, c2a, w0m.x, rxu_a, w0p.x, nrxu_a,
                                           wmc.x, __dadd_rn(vmcM, vmc.x), w1c.x, __dadd_rn(v0cM, v0c.x),
                                           w0cM, __dadd_rn(w0c.x, w0cM), w0c.y, szw, top_a);
                double su_b = pw_sums<FMA>(tcx, tcy, c1b, c2b, u0m.y, sxu_b, u0p.y, nsxu_b,
                                           umc.y, __dadd_rn(vmc.y, vmp.y), u1c.y, __dadd_rn(v0c.y, v0p.y),
                                           u0c.x, szu, u0cQ, __dadd_rn(w0c.y, w0p.y), top_b);
                double sv_b = pw_sums<FMA>(tcx, tcy, c1b, c2b, v0m.y, txu_b, v0p.y, ntxu_b,
                                           vmc.y, __dadd_rn(v0c.y, vmc.y), v1c.y, __dadd_rn(v0c.y, v1c.y),
                                           v0c.x, szv, v0cQ, __dadd_rn(w0c.y, w1c.y), top_b);
                double sw_b = pw_sums<FMA>(tcx, tcy, c1b, c2b, w0m.y, rxu_b, w0p.y, nrxu_b,
                                           wmc.y, __dadd_rn(vmc.x, vmc.y), w1c.y, __dadd_rn(v0c.x, v0c.y),
                                           w0c.x, szw, w0cQ, __dadd_rn(w0c.y, w0cQ), top_b);
                sxu_a = nsxu_a;
                sxu_b = nsxu_b;
                txu_a = ntxu_a;
                txu_b = ntxu_b;
                rxu_a = nrxu_a;
                rxu_b = nrxu_b;
                if (z_a) su_a = sv_a = sw_a = 0.0;
                if (z_b) su_b = sv_b = sw_b = 0.0;
                if constexpr (STEP) {
                    su_a = fwd_update(u0c.x, dt, su_a);
                    su_b = fwd_update(u0c.y, dt, su_b);
                    sv_a = fwd_update(v0c.x, dt, sv_a);
                    sv_b = fwd_update(v0c.y, dt, sv_b);
                    sw_a = fwd_update(w0c.x, dt, sw_a);
                    sw_b = fwd_update(w0c.y, dt, sw_b);
                }
                if (active && (va || (SS && vb)) && !(PWADV_CT_DBG & 2)) {
                    if (!ODD || (va && vb && (SS || qof(pg) == 0))) {  // on the 16-byte grid
                        store2(o0, su_a, su_b);
                        store2(o1, sv_a, sv_b);
                        store2(o2, sw_a, sw_b);
                    } else if (va) {  // odd nz: an odd global column (unshifted), or the top
                        __stcs(o0, su_a);
                        __stcs(o1, sv_a);
                        __stcs(o2, sw_a);
                        if (vb) {
                            __stcs(o0 + 1, su_b);
                            __stcs(o1 + 1, sv_b);
                            __stcs(o2 + 1, sw_b);
                        }
                    } else {  // shifted odd column: level 0 is its first pair's second level
                        __stcs(o0 + 1, su_b);
                        __stcs(o1 + 1, sv_b);
                        __stcs(o2 + 1, sw_b);
                    }
                }
                o0 += ostep;
                o1 += ostep;
                o2 += ostep;
                pst = lst;
                pg = pgl;
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
            release(pst);  // plane ie was only read as the x+1 plane
        };
        if constexpr (!ODD) {
            run_unit(std::integral_constant<int, -1>{});
        } else if (podd) {
            run_unit(std::integral_constant<int, 2>{});
        } else if ((pg + tc) & 1) {
            run_unit(std::integral_constant<int, 1>{});
        } else {
            run_unit(std::integral_constant<int, 0>{});
        }
    }
}

}  // namespace pwadv
