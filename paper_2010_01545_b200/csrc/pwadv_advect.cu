// pwadv_advect.cu — host side of K1 / K4 / K1c: work planning (plan_xmarch,
// plan_ctile, plan_work), the launcher launch_box, and the small K1m / K1s
// launches. The kernels themselves are in pwadv_xmarch.cuh / pwadv_ctile.cuh
// (design notes there) and are instantiated in pwadv_k_*.cu (pwadv_kernels.h).
//
// Replaces the reference hot path run_reference -> compute_block ->
// su/sv/sw_formula (pkg/src/pwadvect/kernel.py:73-185).
#include "pwadv_kernels.h"

#include <cudaTypedefs.h>

#include <algorithm>
#include <climits>
#include <mutex>
#include <vector>

namespace pwadv {

// ---------------------------------------------------------------------------
// host-side planning and launch

static int round_up(int x, int m) { return (x + m - 1) / m * m; }

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device)
// and size: it costs a driver call per launch otherwise (host overhead that
// shows at small per-GPU blocks).
static cudaError_t ensure_smem_attr(const void *kern, int device, int bytes)
{
    struct Entry {
        const void *kern;
        int device, bytes;
    };
    static std::mutex mu;
    static std::vector<Entry> done;
    {
        std::lock_guard<std::mutex> lk(mu);
        for (const Entry &x : done)
            if (x.kern == kern && x.device == device && x.bytes >= bytes) return cudaSuccess;
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) {
        std::lock_guard<std::mutex> lk(mu);
        for (Entry &x : done)
            if (x.kern == kern && x.device == device) {
                if (bytes > x.bytes) x.bytes = bytes;
                return e;
            }
        done.push_back({kern, device, bytes});
    }
    return e;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// libcuda link): resolved once.
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// a field (nx+2, ny+2, nz): even nz as a 3-D tensor {nz, ny+2, nx+2}, box
// {kt+4, tj+2, 1}; odd nz as a 2-D tensor of column-pair rows {2 nz,
// (nx+2)(ny+2)/2}, box {kt+4, tj/2+2} (k_advect_ctile, ODD)
static int encode_field_map(CUtensorMap *m, const double *f, const BoxLaunch &L, int kt, int tj)
{
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    if (!enc) return set_error(PWADV_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    const bool odd = L.nz % 2 != 0;
    const cuuint64_t dims3[3] = {(cuuint64_t)L.nz, (cuuint64_t)(L.ny + 2), (cuuint64_t)(L.nx + 2)};
    const cuuint64_t dims2[2] = {(cuuint64_t)(2 * L.nz), (cuuint64_t)((L.nx + 2) * (L.ny + 2) / 2)};
    const cuuint64_t strides3[2] = {(cuuint64_t)L.nz * sizeof(double),
                                    (cuuint64_t)((L.ny + 2) * L.nz) * sizeof(double)};
    const cuuint64_t strides2[1] = {(cuuint64_t)(2 * L.nz) * sizeof(double)};
    const cuuint32_t box3[3] = {(cuuint32_t)(kt + 4), (cuuint32_t)(tj + 2), 1};
    const cuuint32_t box2[2] = {(cuuint32_t)(kt + 4), (cuuint32_t)(tj / 2 + 2)};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, odd ? 2 : 3, const_cast<double *>(f),
                           odd ? dims2 : dims3, odd ? strides2 : strides3, odd ? box2 : box3, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(PWADV_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return PWADV_OK;
}

// K1c / K4c launch (plan.ct): the fields' tensor maps are kernel parameters
static int launch_ctile(const BoxLaunch &L, const BoxArgs &a, const TileCfg &t, const XmarchPlan &plan,
                        bool fma, cudaStream_t stream)
{
    // the maps depend only on (fields, shape, slab height): a small per-thread
    // cache keeps the encodes off the launch path of repeated launches
    // (time steps, ping-pong buffers, graph capture)
    struct MapEntry {
        const double *u, *v, *w;
        int64_t nx, ny, nz;
        int kt;
        CtMaps maps;
    };
    thread_local MapEntry cache[4];
    thread_local int cache_next = 0;
    CtMaps maps;
    bool hit = false;
    for (const MapEntry &e : cache) {
        if (e.u == L.u && e.v == L.v && e.w == L.w && e.nx == L.nx && e.ny == L.ny && e.nz == L.nz &&
            e.kt == plan.kt && e.u) {
            maps = e.maps;
            hit = true;
            break;
        }
    }
    if (!hit) {
        int rc = encode_field_map(&maps.u, L.u, L, plan.kt, plan.tj);
        if (rc == PWADV_OK) rc = encode_field_map(&maps.v, L.v, L, plan.kt, plan.tj);
        if (rc == PWADV_OK) rc = encode_field_map(&maps.w, L.w, L, plan.kt, plan.tj);
        if (rc != PWADV_OK) return rc;
        cache[cache_next] = MapEntry{L.u, L.v, L.w, L.nx, L.ny, L.nz, plan.kt, maps};
        cache_next = (cache_next + 1) % 4;
    }
    CtileKern kern = kern_ctile(plan.kt, L.nz % 2 != 0, L.step, fma);
    if (!kern) return set_error(PWADV_E_ARG, "unsupported slab height %d", plan.kt);
    const DeviceInfo *dev = device_info();
    cudaError_t e = ensure_smem_attr((const void *)kern, dev->device, (int)plan.smem);
    if (e != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute", e);
    if (L.flags & PWADV_FLAG_NO_PDL) {
        kern<<<plan.grid, plan.threads, plan.smem, stream>>>(a, t, maps);
    } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)plan.grid);
        cfg.blockDim = dim3((unsigned)plan.threads);
        cfg.dynamicSmemBytes = plan.smem;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, kern, a, t, maps);
        if (e != cudaSuccess) return set_cuda_error("advect launch", e);
    }
    count_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error("advect launch", e);
    return PWADV_OK;
}

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
    a.trace = reinterpret_cast<unsigned long long *>(L.trace);
    a.push = (L.peers != nullptr && !L.pull) ? 1 : 0;
    a.pull = L.pull ? 1 : 0;
    a.rim = (L.flags & PWADV_FLAG_RIM) && (L.x1 - L.x0) >= 3 && (L.y1 - L.y0) >= 3 ? 1 : 0;
    if (L.peers) a.peers = *L.peers;
    else a.peers = pwadv_peers{};
    const bool fma = (L.flags & PWADV_FLAG_FMA) != 0;
    const int64_t nbx = L.x1 - L.x0, nby = L.y1 - L.y0;
    if (nbx <= 0 || nby <= 0) return PWADV_OK;

    const DeviceInfo *dev = device_info();
    if (!dev) return PWADV_E_CUDA;

    XmarchPlan plan;
    const bool tiled = plan_xmarch(L, *dev, &plan);
    if (L.pull && (!tiled || plan.elem || plan.maxt != 512))
        return set_error(PWADV_E_ARG, "halo pull needs the aligned X-march (even nz <= 768, "
                                      "16-byte-aligned fields, 512-thread plan)");
    if (tiled && plan.rounds > kMaxUnitsPerCta) {
        // more strips than one launch's unit tables hold (very long y): split
        // the box along y at a strip boundary and launch the halves in order
        const int64_t half = (nby / 2 + plan.tj - 1) / plan.tj * plan.tj;
        if (half >= nby) {  // one strip already (column tiles of extreme depth): the march kernel
            BoxLaunch m = L;
            m.flags |= PWADV_FLAG_MARCH;
            return launch_box(m, stream);
        }
        BoxLaunch lo = L, hi = L;
        lo.y1 = L.y0 + half;
        hi.y0 = L.y0 + half;
        const int rc = launch_box(lo, stream);
        return rc != PWADV_OK ? rc : launch_box(hi, stream);
    }
    if (tiled) {
        TileCfg t;
        t.nslab = plan.ct ? plan.nslab : 1;
        t.tj = plan.tj;
        t.kp = plan.kp;
        t.stages = plan.stages;
        t.nchunks = plan.nchunks;
        t.debug = (int)((L.flags >> 8) & 5u);
        t.l2hint = (L.flags & PWADV_FLAG_L2_UNIT_HEAD) ? 1 : 0;
        t.nstrips = plan.nstrips;
        t.nlong = plan.nlong;
        t.rot = plan.rot;
        t.nface = plan.nface;
        t.nchf = plan.nchf;
        t.spare = plan.spare;
        t.mlen = plan.mlen;
        if (plan.ct) return launch_ctile(L, a, t, plan, fma, stream);
        XmarchKern kern = nullptr;
        const bool fix = (32 % plan.kp) != 0;  // a column straddles a warp boundary
        // compile-time tile layout (NZC) at the default tile for the depths
        // that have one (pwadv_k_nzc*.cu: 16 .. 128)
        const int nzc = (!plan.elem && plan.maxt == 512 && plan.tj == 384 / plan.kp && has_nzc((int)L.nz) &&
                         !(L.flags & (PWADV_FLAG_GENERIC | PWADV_FLAG_DEBUG_NO_COMPUTE |
                                      PWADV_FLAG_DEBUG_NO_STORE)))
                            ? (int)L.nz : 0;
        if (L.pull)  // the pull has compile-time layouts at 64 / 128 only
            kern = kern_xmarch_pull(nzc == 64 || nzc == 128 ? nzc : 0, fix, L.step, fma);
        else if (plan.elem)
            kern = kern_xmarch_ua(fix, L.step, fma);
        else if (nzc)
            kern = kern_xmarch_nzc(nzc, L.step, fma);  // nullptr for a DFMA build off 64 / 128
        if (!kern) kern = kern_xmarch_generic(plan.maxt, fix, L.step, fma);
        if (!kern) return set_error(PWADV_E_ARG, "unsupported thread budget %d", plan.maxt);
        cudaError_t e = ensure_smem_attr((const void *)kern, dev->device, (int)plan.smem);
        if (e != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute", e);
        if (L.flags & PWADV_FLAG_NO_PDL) {
            kern<<<plan.grid, plan.threads, plan.smem, stream>>>(a, t);
        } else {
            // back-to-back launches overlap the next grid's launch with this
            // grid's tail (the kernel waits on griddepcontrol before reading)
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)plan.grid);
            cfg.blockDim = dim3((unsigned)plan.threads);
            cfg.dynamicSmemBytes = plan.smem;
            cfg.stream = stream;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            e = cudaLaunchKernelEx(&cfg, kern, a, t);
            if (e != cudaSuccess) return set_cuda_error("advect launch", e);
        }
    } else if (!a.rim && !a.push && !(L.flags & PWADV_FLAG_SIMPLE)) {
        // K1m: the general march (nz > 768, inputs with different 16-byte phases)
        const int64_t tiles = ((L.nz + 31) / 32) * ((nby + 3) / 4);
        int64_t nch = ((int64_t)dev->sms * 16 + tiles - 1) / tiles;
        const int64_t nch_max = nbx / 8 > 1 ? nbx / 8 : 1;
        if (nch > nch_max) nch = nch_max;
        if (nch > 65535) nch = 65535;
        if (tiles > 0x7fffffff) return set_error(PWADV_E_DIMS, "box too large for the march kernel");
        const dim3 grid((unsigned)tiles, (unsigned)nch), block(32, 4);
        if (L.step) {
            if (fma)
                k_advect_march<true, true><<<grid, block, 0, stream>>>(a, nch);
            else
                k_advect_march<false, true><<<grid, block, 0, stream>>>(a, nch);
        } else {
            if (fma)
                k_advect_march<true, false><<<grid, block, 0, stream>>>(a, nch);
            else
                k_advect_march<false, false><<<grid, block, 0, stream>>>(a, nch);
        }
    } else {
        const int64_t total = (a.rim ? 2 * nby + 2 * (nbx - 2) : nbx * nby) * L.nz;
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

// doubles per field slot of a ring stage (k_advect_xmarch's CS)
static size_t slot_doubles(int64_t tj, int64_t nz, bool ua)
{
    const int64_t run = (tj + 2) * nz;
    return (size_t)(ua ? ((run + 3) & ~(int64_t)1) : run);
}

// Work units for p->nstrips strips (y-strips, or y-strip x k-slab pairs of the
// column-tile kernel) of nbx planes: full rounds of whole strips, the rest in
// X chunks, optionally the spare-tail plan (plan_xmarch's notes below).
static void plan_work(const BoxLaunch &L, const DeviceInfo &dev, int per_sm, XmarchPlan *p)
{
    const int64_t nbx = L.x1 - L.x0;
    // Work units dealt round-robin to one wave of CTAs. Whole strips fill
    // as many full rounds as there are (long units keep all CTAs marching in
    // step: at 4096x4096x128, 36 short units per CTA instead of 5 long ones
    // drifted apart and ran 39% slower at the same DRAM bytes); the strips
    // left over are cut into X chunks chosen by a cost model fitted on B200
    // (tools/sweep.py --rounds, profiles/README.md): a round of n concurrent
    // units takes (planes per unit + 1) x max(n, A) plane-times, A = g0/1.15
    // being the CTAs that already saturate HBM (fewer stream at their own
    // latency-bound rate) and +1 the plane pair a unit re-reads. E.g. 3 chunks
    // at 512x512x64 (one round of 129 CTAs), 5 at 1024^2; at 2048^2 one full
    // round plus 23 strips in 32 chunks. opts.chunks > 0 forces uniform
    // chunking of every strip.
    const int64_t g0 = L.grid > 0 ? L.grid : (int64_t)dev.sms * per_sm;  // one wave of resident CTAs
    const int64_t sat = (g0 * 100 + 114) / 115;
    const int64_t full_rounds = L.chunks > 0 ? 0 : p->nstrips / g0;
    p->nlong = full_rounds * g0;
    const int64_t tail = p->nstrips - p->nlong;
    int64_t best_nch = 1;
    double best_cost = -1.0;
    const int64_t nch_max = nbx < 4096 ? nbx : 4096;
    for (int64_t nch = L.chunks > 0 ? (L.chunks < nch_max ? L.chunks : nch_max) : 1;
         tail > 0 && nch <= nch_max; ++nch) {
        const int64_t units = tail * nch;
        const int64_t rounds = full_rounds + (units + g0 - 1) / g0;
        if (rounds > kMaxUnitsPerCta) break;
        const int64_t full = units / g0, last = units % g0;
        const double active = (double)(full * g0) + (last ? (double)(last > sat ? last : sat) : 0.0);
        const double cost = ((double)((nbx + nch - 1) / nch) + 1.0) * active;
        if (best_cost < 0.0 || cost < best_cost * (1.0 - 1e-9)) {
            best_cost = cost;
            best_nch = nch;
        }
        if (L.chunks > 0) break;
    }
    p->nchunks = (int)best_nch;
    int64_t units = p->nlong + tail * best_nch;
    int64_t grid = units < g0 ? units : g0;
    if (grid < 1) grid = 1;
    p->grid = (int)grid;
    p->rounds = (units + grid - 1) / grid;
    // Halo pull: the two y-face strips copy six runs per plane instead of
    // three and set the pace of whatever round they are in. Rotate the strips
    // by one so they are the last two of the chunked tail, and cut them into
    // shorter chunks using the tail round's free CTA slots (no extra round).
    p->rot = 0;
    p->nface = 0;
    p->nchf = 0;
#ifndef PWADV_PULL_ROT
#define PWADV_PULL_ROT 1
#endif
    if (L.pull && PWADV_PULL_ROT && p->nstrips > 1 && tail > 0) {
        p->rot = 1;
        p->nface = (int)(tail < 2 ? tail : 2);
        const int64_t spare = L.grid > 0 || L.chunks > 0 ? 0 : p->rounds * g0 - units;
        int64_t nchf = best_nch + spare / p->nface;
        if (nchf > nbx) nchf = nbx;
        if (nchf < best_nch) nchf = best_nch;
        p->nchf = (int)nchf;
        units += (int64_t)p->nface * (nchf - best_nch);
        grid = units < g0 ? units : g0;
        if (grid < 1) grid = 1;
        p->grid = (int)grid;
        p->rounds = (units + grid - 1) / grid;
    }
    // Spare-tail plan. A single-round plan whose units do not fill the SMs
    // is rebalanced: each strip gets m main chunks of L planes (one per CTA,
    // all concurrent) and one tail chunk of nbx - m*L planes; the G - n*m
    // spare CTAs run the n tail chunks, ceil(n / spare) each in sequence. L
    // balances a main CTA's L + 2 planes against a spare CTA's tail planes
    // (512x256x64, the C2 block per GPU at 2x4: 22 strips x 6 chunks = 132
    // CTAs of 86 planes -> m = 6, L = 79, 16 spare CTAs: 81 planes per CTA).
    // Measured in bursts of back-to-back launches (tools/sweep.py
    // --burst-sleep, profiles/README.md) it pays only for SHORT units: +1% at
    // 512x256x64, +2% at 256x256x64; with units of 150+ planes the classic
    // plan's ~129 CTAs already saturate HBM and the tail CTAs' extra plane
    // pairs and out-of-step halo columns cost more than the idle SMs (C1
    // 512x512x64: 131.9 classic vs 130.1 spare, 768^2: 135.0 vs 131.5,
    // 1024x512: 136.3 vs 132.0 Gpts/s). PWADV_FLAG_SPARE_TAIL forces it.
    p->spare = 0;
    p->mlen = 0;
    if (!L.pull && L.chunks <= 0 && L.grid <= 0 && full_rounds == 0 && per_sm == 1 &&
        !(L.flags & PWADV_FLAG_NO_SPARE_TAIL) && p->rounds == 1 && !p->nface) {
        const int64_t n = p->nstrips;
        int64_t best_m = 0, best_l = 0, best_sp = 0, best_planes = 0;
        for (int64_t m = 1; n * m < g0; ++m) {
            const int64_t sp = std::min<int64_t>(g0 - n * m, n);
            const int64_t rt = (n + sp - 1) / sp;
            if (rt > kMaxUnitsPerCta) continue;
            // L + 2 = rt * (nbx - m*L + 2)  ->  L = (rt*(nbx+2) - 2) / (1 + m*rt)
            const int64_t l0 = (rt * (nbx + 2) - 2) / (1 + m * rt);
            for (int64_t l = l0; l <= l0 + 1; ++l) {
                if (l < 1 || m * l >= nbx) continue;
                const int64_t planes = std::max<int64_t>(l + 2, rt * (nbx - m * l + 2));
                if (best_m == 0 || planes < best_planes) {
                    best_m = m;
                    best_l = l;
                    best_sp = sp;
                    best_planes = planes;
                }
            }
        }
        const int64_t cur = (nbx + p->nchunks - 1) / p->nchunks + 2;  // planes per CTA now
        const bool pays = cur <= 130 && best_planes * 100 <= cur * 95;
        if (best_m > 0 && ((L.flags & PWADV_FLAG_SPARE_TAIL) || pays)) {
            p->spare = (int)best_sp;
            p->mlen = best_l;
            p->nchunks = (int)best_m;
            p->grid = (int)(n * best_m + best_sp);
            p->rounds = (n + best_sp - 1) / best_sp;
        }
    }
}

// Slab height of the column-tile plan: the least (slab levels x preference).
// Measured at equal slab fill KT 128 ~ 96 >= 64 ~ 48 (within 1-2%) > 32 (5-8%:
// two columns per warp): nz 1024 -> 128, 1030 -> 96 (11 slabs, 2.5% idle
// levels), 190 -> 96, 140 -> 48, 160 -> 32 (tools/shape_sweep.py,
// profiles/r02_ct_slab_heights.jsonl).
static double ct_pref(int kt)
{
    switch (kt) {
    case 128: return 1.0;
    case 96: return 1.0;
    case 64: return 1.01;
    case 48: return 1.01;
    default: return 1.07;  // 32: two columns per warp
    }
}

static int ctile_kt(int64_t nz)
{
    int kt = 128;
    double best = 0.0;
    for (int c : {128, 96, 64, 48, 32}) {
        if (nz % 2 && (c / 2) % 32) continue;  // odd nz: one column parity per warp
        const double pref = ct_pref(c);
        const double cost = (double)((nz + c - 1) / c * c) * pref;
        if (best == 0.0 || cost < best) {
            best = cost;
            kt = c;
        }
    }
    return kt;
}

// Whole-column X-march vs column tiles, from a fit to the measured rates
// (profiles/README.md, round 2): relative rate = busy-thread fraction x a
// strip-width factor (whole columns: 1.0 at TJ >= 6, 0.97 / 0.95 / 0.93 /
// 0.9 / 0.8 at TJ = 5 / 4 / 3 / 2 / 1, x 0.92 off the compile-time layouts;
// column tiles 0.98 / slab preference). E.g. nz 64, 128: whole columns (1.0
// vs 0.98); 80, 96, 100, 130-150: whole (idle slab levels); 110-126, 160,
// 192, 256 and deeper: tiles.
static bool ctile_pays(int64_t nz, int64_t ny)
{
    // odd nz. With ny+2 even a unit's column parities are fixed and odd
    // columns take shifted pairs (every thread's own loads and all stores on
    // the 16-byte grid): 107-121 Gpts/s against the UA form's 102-112 at nz
    // 63-255, 119-122 vs 87 at 511 — taken whenever its slabs are >= 90% busy
    // (nz 63, 127, 191 yes; 33, 95 no: a half-empty slab). With ny+2 odd the
    // parity alternates per plane (unshifted pairs, odd columns scalar): 89 vs
    // the UA form's 107 at nz 63, ahead once the UA strips narrow (nz >= 255)
    // and against K1m above 767.
    if (nz % 2 != 0) {
        if (nz >= 255) return true;
        if ((ny + 2) % 2 != 0) return false;
        const int kt = ctile_kt(nz);
        return (double)nz >= 0.9 * (double)((nz + 1 + kt - 1) / kt * kt);
    }
    const int kt = ctile_kt(nz);
    const double pref = ct_pref(kt);
    const double ct = 0.98 * (double)nz / (double)((nz + kt - 1) / kt * kt) / pref;
    const int64_t kp = nz / 2;
    if (kp > 384) return true;  // no whole-column plan
    const int64_t tj = 384 / kp;
    static const double width[6] = {0.0, 0.8, 0.9, 0.93, 0.95, 0.97};
    // the whole-column tile has a compile-time layout only at the depths of
    // has_nzc (16-128 in steps of 8, and 100); elsewhere its run-time layout
    // costs ~8% at equal occupancy
    // (nz 110 / 120: 117 / 122 Gpts/s against K1c's 128 / 131 with the same
    // busy fraction; profiles/r02_monc_depths.jsonl)
    // (with a compile-time layout the narrow strips cost nothing measurable
    // down to TJ = 4: nz 192 at 133.6 Gpts/s, 152 at 128-131 — the width
    // factors are the run-time layout's)
    const double whole = (double)(tj * kp) / 384.0 *
                         (has_nzc((int)nz) ? 1.0 : (tj >= 6 ? 1.0 : width[tj]) * 0.92);
    return ct > whole;
}

// Column-tile plan (k_advect_ctile). Applies to 16-byte-aligned fields,
// without the fused halo pull / push, at the 512-thread budget. Slab height KT from opts.tile_j (768 / tile_j) or the default below.
static bool plan_ctile(const BoxLaunch &L, const DeviceInfo &dev, XmarchPlan *p)
{
    const int64_t nz = L.nz;
    const uintptr_t al = (uintptr_t)L.u | (uintptr_t)L.v | (uintptr_t)L.w | (uintptr_t)L.o0 |
                         (uintptr_t)L.o1 | (uintptr_t)L.o2;
    if ((al & 15) || L.peers || L.pull ||
        (L.max_threads > 0 && L.max_threads != 512) ||
        (L.flags & (PWADV_FLAG_DEBUG_NO_COMPUTE | PWADV_FLAG_DEBUG_NO_STORE | PWADV_FLAG_UNALIGNED |
                    PWADV_FLAG_GENERIC)))
        return false;
    // TMA coordinates are 32-bit: planes and columns (even nz), column-pair
    // rows (odd nz)
    if (L.nx + 2 > INT32_MAX || L.ny + 2 > INT32_MAX || nz > INT32_MAX / 2 ||
        (nz % 2 && (L.nx + 2) * (L.ny + 2) / 2 > INT32_MAX))
        return false;
    int kt = ctile_kt(nz);
    if (L.tile_j > 0) {
        if (L.tile_j != 6 && L.tile_j != 8 && L.tile_j != 12 && L.tile_j != 16 && L.tile_j != 24)
            return false;
        kt = 768 / L.tile_j;
    }
    // odd nz: one column parity per warp (KT 64 / 128) for the warp-uniform
    // choice of odd columns' slot shifts
    if (nz % 2 && (kt / 2) % 32) {
        if (L.tile_j > 0) return false;
        kt = 64;
    }
    const int tj = 768 / kt;
    const int64_t nby = L.y1 - L.y0;
    // odd nz: an odd column's pairs may start one level low (k_advect_ctile's
    // shifted pairs), so the slabs cover nz + 1 levels
    const int64_t nslab = (nz + (nz & 1) + kt - 1) / kt;
    // CtLayout::CS: even nz (tj+2) column slots, odd nz two halves of tj/2+2
    const int half = ((tj / 2 + 2) * (kt + 4) + 15) / 16 * 16;
    const int box = nz % 2 ? half + (tj / 2 + 2) * (kt + 4) : (tj + 2) * (kt + 4);
    const size_t stage_bytes = (size_t)3 * ((box + 15) / 16 * 16) * sizeof(double);
    const size_t bar_bytes = 2 * 16 * sizeof(uint64_t) + sizeof(RingState);
    const size_t smem_cap = (size_t)dev.smem_optin - bar_bytes - 1024;
    int smax = (int)(smem_cap / stage_bytes);
    if (smax > 16) smax = 16;
    const int stages = L.stages > 0 ? (L.stages < smax ? L.stages : smax) : (smax < 5 ? smax : 5);
    if (stages < 3) return false;
    *p = XmarchPlan{};
    p->ct = 1;
    p->kt = kt;
    p->nslab = (int)nslab;
    p->maxt = 512;
    p->tj = tj;
    p->kp = kt / 2;
    p->stages = stages;
    p->threads = 512;
    p->smem = (size_t)stages * stage_bytes + 2 * stages * sizeof(uint64_t) + sizeof(RingState);
    p->nstrips = (nby + tj - 1) / tj * nslab;
    plan_work(L, dev, 1, p);
    return true;
}

bool plan_xmarch(const BoxLaunch &L, const DeviceInfo &dev, XmarchPlan *p)
{
    if (L.flags & (PWADV_FLAG_SIMPLE | PWADV_FLAG_RIM | PWADV_FLAG_MARCH)) return false;
    // the column-tile X-march: forced, or the default where it is expected to
    // be faster (ctile_pays: deep columns, whose whole-column strips shrink to
    // 1-5 columns — measured 122-133 Gpts/s at nz 160-2048 against 106-124
    // for the whole-column X-march and ~80 for K1m above 768)
    if (!(L.flags & PWADV_FLAG_NO_CTILE) && ((L.flags & PWADV_FLAG_CTILE) || (L.tile_j <= 0 && ctile_pays(L.nz, L.ny))) &&
        plan_ctile(L, dev, p))
        return true;
    const int64_t nz = L.nz;
    // 16-byte alignment and even nz for 16-byte-aligned tile runs and the
    // paired loads/stores; otherwise UA (unaligned runs: the copies start up to
    // one element early, scalar shared loads and stores, also into the peers'
    // halos) — warp-specialised only, u, v, w with the same 16-byte phase
    uintptr_t al = (uintptr_t)L.u | (uintptr_t)L.v | (uintptr_t)L.w | (uintptr_t)L.o0 |
                   (uintptr_t)L.o1 | (uintptr_t)L.o2;
    // fused push: the aligned form stores boundary pairs into the peers'
    // halos with 16-byte stores too — 8-byte-aligned peers take the UA form
    // (scalar stores); pwadv_step_push_f64 requires 8-byte-aligned peers
    if (L.peers && !L.pull)
        for (int d = 0; d < 8; ++d)
            al |= (uintptr_t)L.peers->u[d] | (uintptr_t)L.peers->v[d] | (uintptr_t)L.peers->w[d];
    const bool ua = (nz % 2 != 0) || (al & 15) || (L.flags & PWADV_FLAG_UNALIGNED);
    const uintptr_t inpar = ((uintptr_t)L.u ^ (uintptr_t)L.v) | ((uintptr_t)L.u ^ (uintptr_t)L.w);
    if (ua && ((al & 7) || (inpar & 8) || (L.max_threads > 0 && L.max_threads != 512) ||
               (L.flags & (PWADV_FLAG_DEBUG_NO_COMPUTE | PWADV_FLAG_DEBUG_NO_STORE))))
        return false;
    if (nz > 1024) return false;
    p->elem = ua ? 1 : 0;
    const int kp = (int)((nz + 1) / 2);
    const int64_t nby = L.y1 - L.y0;
    // thread budget per CTA (register file / CTA): 384 by default, which
    // leaves ~168 registers per thread for the rolled x-window
    // default: warp-specialised 512 threads (3 compute warpgroups of 160
    // registers + a producer warpgroup); measured 125 Gpts/s at C1/C3 vs 110
    // for the 384-thread kernel whose warps issue the refills themselves
    int maxt = L.max_threads > 0 ? L.max_threads : 512;
    if (maxt != 512 && maxt != 384 && maxt != 256 && maxt != 192 && maxt != 128) return false;
    const int tile_threads = maxt == 512 ? 384 : maxt;  // 512: 3 compute + 1 producer warpgroup
    const int per_sm = ctas_per_sm(maxt);
    if (kp > maxt) return false;
    int tj = L.tile_j > 0 ? L.tile_j : tile_threads / kp;
    if (tj > tile_threads / kp) tj = tile_threads / kp;
    if (tj < 1) return false;
    if (tj > nby) tj = (int)nby;
    const size_t bar_bytes = 2 * 16 * sizeof(uint64_t) + sizeof(RingState);
    // shared memory per CTA: the SM's 228 KB split between resident CTAs
    size_t smem_cap = (size_t)dev.smem_optin - bar_bytes - 1024;
    if (per_sm > 1) smem_cap = (size_t)(228 * 1024) / per_sm - bar_bytes - 1024 - 1024;
    int stages = 0;
    for (;;) {
        const size_t stage_bytes = (size_t)3 * slot_doubles(tj, nz, ua) * sizeof(double);
        int smax = (int)(smem_cap / stage_bytes);
        if (smax > 16) smax = 16;  // RingState::released
        // default ring depth 5 (tools/sweep.py; see the note at the end)
        stages = L.stages > 0 ? (L.stages < smax ? L.stages : smax) : (smax < 5 ? smax : 5);
        if (stages >= 3) break;
        if (tj == 1) return false;
        tj = tj / 2;
    }
    p->maxt = maxt;
    p->tj = tj;
    p->kp = kp;
    p->stages = stages;
    p->threads = maxt == 512 ? 512 : round_up(tj * kp, 32);
    p->smem = (size_t)stages * 3 * slot_doubles(tj, nz, ua) * sizeof(double) + 2 * stages * sizeof(uint64_t) +
              sizeof(RingState);
    p->nstrips = (nby + tj - 1) / tj;
    plan_work(L, dev, per_sm, p);
    // Ring depth: 5 stages (the default above) for every plan. Measured as
    // the bench runs it — bursts of back-to-back launches at full clocks
    // (tools/sweep.py --burst-sleep 0.3 --prewarm-ms 30, profiles/README.md):
    // C1 131 / C2 131.8 / C3 133.8 / C4 block 134.8 Gpts/s with 5 stages
    // against 118-126 with 6 and 128 with 4. (Round 1 chose 6 for single-
    // round plans from sustained, power-capped runs.)
    return true;
}

}  // namespace pwadv
