// pwadv_kernels.h — the kernel instantiations of K1 / K4 / K1c, compiled in
// separate translation units (pwadv_k_*.cu, built in parallel by build.py)
// and handed to the host launcher (pwadv_advect.cu) as function pointers.
#pragma once
#include "pwadv_xmarch.cuh"

namespace pwadv {

using XmarchKern = void (*)(BoxArgs, TileCfg);
using CtileKern = void (*)(BoxArgs, TileCfg, CtMaps);

// whole-column X-march with a compile-time tile layout for depth nz (NZC), or
// nullptr where none is built (the depths of has_nzc; DFMA builds: 64 / 128)
XmarchKern kern_xmarch_nzc(int nz, bool step, bool fma);
bool has_nzc(int nz);
// the same with the fused halo pull: nzc 64 / 128 or 0 (run-time layout)
XmarchKern kern_xmarch_pull(int nzc, bool fix, bool step, bool fma);
// run-time layout, warp-specialised (maxt 512) or the plain budgets 384..128
XmarchKern kern_xmarch_generic(int maxt, bool fix, bool step, bool fma);
// unaligned-run (UA) form
XmarchKern kern_xmarch_ua(bool fix, bool step, bool fma);
// column tiles: slab height kt, odd nz (column-pair rows)
CtileKern kern_ctile(int kt, bool odd, bool step, bool fma);

// per-unit parts of kern_xmarch_nzc (pwadv_k_nzc*.cu)
XmarchKern kern_nzc_part0(int nz, bool step, bool fma);
XmarchKern kern_nzc_part1(int nz, bool step, bool fma);
XmarchKern kern_nzc_part2(int nz, bool step, bool fma);
XmarchKern kern_nzc_part3(int nz, bool step, bool fma);
CtileKern kern_ctile_even(int kt, bool step, bool fma);
CtileKern kern_ctile_odd(int kt, bool step, bool fma);
XmarchKern kern_generic_small(int maxt, bool fix, bool step, bool fma);

}  // namespace pwadv

// one (step, fma) quadruple of a kernel template instantiation
#define PWADV_SF(T, ...)                                                              \
    (step ? (fma ? &T<true, true, __VA_ARGS__> : &T<false, true, __VA_ARGS__>)        \
          : (fma ? &T<true, false, __VA_ARGS__> : &T<false, false, __VA_ARGS__>))
// the non-DFMA (bit-exact) pair only
#define PWADV_S(T, ...) (fma ? nullptr : (step ? &T<false, true, __VA_ARGS__> : &T<false, false, __VA_ARGS__>))
