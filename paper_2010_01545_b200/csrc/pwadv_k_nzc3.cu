// pwadv_k_nzc3.cu — kernel instantiations (see pwadv_kernels.h).
#include "pwadv_kernels.h"

namespace pwadv {

// compile-time-layout whole-column X-march (K1 / K4), depths 136, 144, 152, 160, 168, 176, 184, 192
XmarchKern kern_nzc_part3(int nz, bool step, bool fma)
{
    switch (nz) {
    case 136: return PWADV_S(k_advect_xmarch, 512, true, 136);
    case 144: return PWADV_S(k_advect_xmarch, 512, true, 144);
    case 152: return PWADV_S(k_advect_xmarch, 512, true, 152);
    case 160: return PWADV_S(k_advect_xmarch, 512, true, 160);
    case 168: return PWADV_S(k_advect_xmarch, 512, true, 168);
    case 176: return PWADV_S(k_advect_xmarch, 512, true, 176);
    case 184: return PWADV_S(k_advect_xmarch, 512, true, 184);
    case 192: return PWADV_S(k_advect_xmarch, 512, true, 192);
    default: return nullptr;
    }
}

}  // namespace pwadv
