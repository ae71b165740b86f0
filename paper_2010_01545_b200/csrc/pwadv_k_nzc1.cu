// pwadv_k_nzc1.cu — kernel instantiations (see pwadv_kernels.h).
#include "pwadv_kernels.h"

namespace pwadv {

// compile-time-layout whole-column X-march (K1 / K4), depths 40, 48, 56, 72
XmarchKern kern_nzc_part1(int nz, bool step, bool fma)
{
    switch (nz) {
    case 40: return PWADV_S(k_advect_xmarch, 512, true, 40);
    case 48: return PWADV_S(k_advect_xmarch, 512, true, 48);
    case 56: return PWADV_S(k_advect_xmarch, 512, true, 56);
    case 72: return PWADV_S(k_advect_xmarch, 512, true, 72);
    default: return nullptr;
    }
}

}  // namespace pwadv
