// pwadv_device.cuh — device-side arithmetic and sm_100a async-copy primitives.
//
// The PW formulas follow the reference's exact association
// (pkg/src/pwadvect/kernel.py:73-112, docs/model-notes.md §2, SURVEY.md
// Appendix B). Every operation uses an explicit round-to-nearest intrinsic
// (__dadd_rn/__dsub_rn/__dmul_rn), which nvcc never contracts into DFMA, so
// the default build is bit-exact with the reference regardless of --fmad.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pwadv {

// s = ((tcx*(x1*(x2+x3) - x4*(x5+x6))) + (tcy*(y1*(y2+y3) - y4*(y5+y6))))
//     + ((c1*z1)*(z2+z3) - (c2*z4)*(z5+z6))          [mid level]
//     + ((c1*z1)*(z2+z3))                              [top level, k = nz-1]
// su/sv/sw are this expression with the operand wiring of kernel.py:117-128.
// The same expression from precomputed operand sums sx1 = x2+x3, sx2 = x5+x6,
// sy1, sy2, sz1, sz2 (a sum may be shared between neighbouring points: IEEE
// addition is commutative, so x+y computed once serves as both x+y and y+x).
template <bool FMA>
__device__ __forceinline__ double pw_sums(double tcx, double tcy, double c1, double c2,
                                          double x1, double sx1, double x4, double sx2,
                                          double y1, double sy1, double y4, double sy2,
                                          double z1, double sz1, double z4, double sz2, bool top)
{
    if constexpr (!FMA) {
        double X = __dmul_rn(tcx, __dsub_rn(__dmul_rn(x1, sx1), __dmul_rn(x4, sx2)));
        double Y = __dmul_rn(tcy, __dsub_rn(__dmul_rn(y1, sy1), __dmul_rn(y4, sy2)));
        double s = __dadd_rn(X, Y);
        double A = __dmul_rn(__dmul_rn(c1, z1), sz1);
        if (top) return __dadd_rn(s, A);
        double B = __dmul_rn(__dmul_rn(c2, z4), sz2);
        return __dadd_rn(s, __dsub_rn(A, B));
    } else {
        double xd = __fma_rn(x1, sx1, -__dmul_rn(x4, sx2));
        double yd = __fma_rn(y1, sy1, -__dmul_rn(y4, sy2));
        double s = __fma_rn(tcx, xd, __dmul_rn(tcy, yd));
        double c1z = __dmul_rn(c1, z1);
        if (top) return __dadd_rn(s, __dmul_rn(c1z, sz1));
        double B = __dmul_rn(__dmul_rn(c2, z4), sz2);
        return __dadd_rn(s, __fma_rn(c1z, sz1, -B));
    }
}

template <bool FMA>
__device__ __forceinline__ double pw_expr(double tcx, double tcy, double c1, double c2,
                                          double x1, double x2, double x3, double x4,
                                          double x5, double x6, double y1, double y2,
                                          double y3, double y4, double y5, double y6,
                                          double z1, double z2, double z3, double z4,
                                          double z5, double z6, bool top)
{
    return pw_sums<FMA>(tcx, tcy, c1, c2, x1, __dadd_rn(x2, x3), x4, __dadd_rn(x5, x6),
                        y1, __dadd_rn(y2, y3), y4, __dadd_rn(y5, y6),
                        z1, __dadd_rn(z2, z3), z4, __dadd_rn(z5, z6), top);
}

// su_formula (kernel.py:73-84): argument order as the reference.
template <bool FMA>
__device__ __forceinline__ double su_formula(double tcx, double tcy, double c1, double c2,
                                             double u_c, double u_xm1, double u_xp1,
                                             double u_jm1, double u_jp1, double u_km1,
                                             double u_kp1, double v_jm1, double v_jm1_xp1,
                                             double v_c, double v_xp1, double w_km1,
                                             double w_km1_xp1, double w_c, double w_xp1,
                                             bool top)
{
    return pw_expr<FMA>(tcx, tcy, c1, c2,
                        u_xm1, u_c, u_xm1, u_xp1, u_c, u_xp1,
                        u_jm1, v_jm1, v_jm1_xp1, u_jp1, v_c, v_xp1,
                        u_km1, w_km1, w_km1_xp1, u_kp1, w_c, w_xp1, top);
}

// sv_formula (kernel.py:87-98).
template <bool FMA>
__device__ __forceinline__ double sv_formula(double tcx, double tcy, double c1, double c2,
                                             double v_c, double v_xm1, double v_xp1,
                                             double v_jm1, double v_jp1, double v_km1,
                                             double v_kp1, double u_xm1, double u_xm1_jp1,
                                             double u_c, double u_jp1, double w_km1,
                                             double w_km1_jp1, double w_c, double w_jp1,
                                             bool top)
{
    return pw_expr<FMA>(tcx, tcy, c1, c2,
                        v_xm1, u_xm1, u_xm1_jp1, v_xp1, u_c, u_jp1,
                        v_jm1, v_c, v_jm1, v_jp1, v_c, v_jp1,
                        v_km1, w_km1, w_km1_jp1, v_kp1, w_c, w_jp1, top);
}

// sw_formula (kernel.py:101-112).
template <bool FMA>
__device__ __forceinline__ double sw_formula(double tcx, double tcy, double c1, double c2,
                                             double w_c, double w_xm1, double w_xp1,
                                             double w_jm1, double w_jp1, double w_km1,
                                             double w_kp1, double u_xm1_km1, double u_xm1,
                                             double u_km1, double u_c, double v_jm1_km1,
                                             double v_jm1, double v_km1, double v_c,
                                             bool top)
{
    return pw_expr<FMA>(tcx, tcy, c1, c2,
                        w_xm1, u_xm1_km1, u_xm1, w_xp1, u_km1, u_c,
                        w_jm1, v_jm1_km1, v_jm1, w_jp1, v_km1, v_c,
                        w_km1, w_c, w_km1, w_kp1, w_c, w_kp1, top);
}

// forward update f + dt*s (mul then add; the composed oracle's numpy order)
__device__ __forceinline__ double fwd_update(double f, double dt, double s)
{
    return __dadd_rn(f, __dmul_rn(dt, s));
}

// ---------------------------------------------------------------------------
// mbarrier + 1-D bulk async copy (TMA engine, SASS UBLKCP) helpers

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
                 ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// `count` arrivals at once (on behalf of threads with nothing to deliver)
__device__ __forceinline__ void mbar_arrive_cnt(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(count)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra.uni WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// As mbar_wait, with a suspend-time hint: the waiting thread may sleep up to
// `ns` nanoseconds per try instead of re-polling (the producer's wait).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity, uint32_t ns)
{
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra.uni WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(ns)
        : "memory");
}

// Global -> shared bulk copy completing on an mbarrier (bytes % 16 == 0,
// both addresses 16-byte aligned).
__device__ __forceinline__ void bulk_g2s(void *dst_smem, const void *src_gmem, uint32_t bytes,
                                         uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst_smem)), "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// As bulk_g2s with an L2 eviction-priority policy (createpolicy result).
__device__ __forceinline__ void bulk_g2s_hint(void *dst_smem, const void *src_gmem, uint32_t bytes,
                                              uint64_t *bar, uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(dst_smem)), "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// outputs are written once and not re-read by this kernel: evict-first stores
__device__ __forceinline__ void store2(double *p, double a, double b)
{
    __stcs(reinterpret_cast<double2 *>(p), make_double2(a, b));
}

// 8-byte global -> shared asynchronous copy (LDGSTS; any 8-byte alignment)
__device__ __forceinline__ void cp_async8(void *dst_smem, const void *src_gmem)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst_smem)), "l"(src_gmem)
                 : "memory");
}

// 16-byte global -> shared asynchronous copy (LDGSTS.128, L2 only)
__device__ __forceinline__ void cp_async16(void *dst_smem, const void *src_gmem)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst_smem)), "l"(src_gmem)
                 : "memory");
}

// arrive on `bar` once this thread's earlier cp.async copies have landed; the
// barrier's expected count includes this arrival (.noinc)
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t *bar)
{
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

}  // namespace pwadv
