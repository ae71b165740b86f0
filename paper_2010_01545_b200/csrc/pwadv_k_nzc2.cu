// pwadv_k_nzc2.cu — kernel instantiations (see pwadv_kernels.h).
#include "pwadv_kernels.h"

namespace pwadv {

// compile-time-layout whole-column X-march (K1 / K4), depths 80, 88, 96, 100, 104, 112, 120
XmarchKern kern_nzc_part2(int nz, bool step, bool fma)
{
    switch (nz) {
    case 80: return PWADV_S(k_advect_xmarch, 512, true, 80);
    case 88: return PWADV_S(k_advect_xmarch, 512, true, 88);
    case 96: return PWADV_S(k_advect_xmarch, 512, true, 96);
    case 100: return PWADV_S(k_advect_xmarch, 512, true, 100);
    case 104: return PWADV_S(k_advect_xmarch, 512, true, 104);
    case 112: return PWADV_S(k_advect_xmarch, 512, true, 112);
    case 120: return PWADV_S(k_advect_xmarch, 512, true, 120);
    default: return nullptr;
    }
}

}  // namespace pwadv
