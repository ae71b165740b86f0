// pwadv_k_pull.cu — kernel instantiations (see pwadv_kernels.h).
#include "pwadv_kernels.h"

namespace pwadv {

// K1 / K4 with the fused halo pull (own instantiations: the producer's extra
// work stays out of the other kernels); compile-time layouts at 64 / 128
XmarchKern kern_xmarch_pull(int nzc, bool fix, bool step, bool fma)
{
    if (nzc == 64) return PWADV_SF(k_advect_xmarch, 512, false, 64, false, true);
    if (nzc == 128) return PWADV_SF(k_advect_xmarch, 512, true, 128, false, true);
    return fix ? PWADV_SF(k_advect_xmarch, 512, true, 0, false, true)
               : PWADV_SF(k_advect_xmarch, 512, false, 0, false, true);
}

}  // namespace pwadv
