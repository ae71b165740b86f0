// pwadv_k_nzc0.cu — kernel instantiations (see pwadv_kernels.h).
#include "pwadv_kernels.h"

namespace pwadv {

// compile-time-layout whole-column X-march (K1 / K4), depths 16, 24, 32 and the
// BASELINE depths 64 / 128 (those also as DFMA builds); kern_xmarch_nzc and
// has_nzc dispatch over the three parts
XmarchKern kern_nzc_part0(int nz, bool step, bool fma)
{
    switch (nz) {
    case 64: return PWADV_SF(k_advect_xmarch, 512, false, 64);
    case 128: return PWADV_SF(k_advect_xmarch, 512, true, 128);
    case 16: return PWADV_S(k_advect_xmarch, 512, false, 16);
    case 24: return PWADV_S(k_advect_xmarch, 512, true, 24);
    case 32: return PWADV_S(k_advect_xmarch, 512, false, 32);
    default: return nullptr;
    }
}

bool has_nzc(int nz)
{
    switch (nz) {
    case 16:
    case 24:
    case 32:
    case 40:
    case 48:
    case 56:
    case 64:
    case 72:
    case 80:
    case 88:
    case 96:
    case 100:
    case 104:
    case 112:
    case 120:
    case 128:
    case 136:
    case 144:
    case 152:
    case 160:
    case 168:
    case 176:
    case 184:
    case 192:
        return true;
    default:
        return false;
    }
}

XmarchKern kern_xmarch_nzc(int nz, bool step, bool fma)
{
    if (XmarchKern k = kern_nzc_part0(nz, step, fma)) return k;
    if (XmarchKern k = kern_nzc_part1(nz, step, fma)) return k;
    if (XmarchKern k = kern_nzc_part2(nz, step, fma)) return k;
    return kern_nzc_part3(nz, step, fma);
}

}  // namespace pwadv
