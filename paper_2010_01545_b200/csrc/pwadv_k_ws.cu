// pwadv_k_ws.cu — kernel instantiations (see pwadv_kernels.h).
#include "pwadv_kernels.h"

namespace pwadv {

// run-time-layout warp-specialised X-march (K1 / K4) and its unaligned-run
// (UA) form
XmarchKern kern_xmarch_generic(int maxt, bool fix, bool step, bool fma)
{
    if (maxt == 512)
        return fix ? PWADV_SF(k_advect_xmarch, 512, true) : PWADV_SF(k_advect_xmarch, 512, false);
    return kern_generic_small(maxt, fix, step, fma);
}

XmarchKern kern_xmarch_ua(bool fix, bool step, bool fma)
{
    return fix ? PWADV_SF(k_advect_xmarch, 512, true, 0, true)
               : PWADV_SF(k_advect_xmarch, 512, false, 0, true);
}

}  // namespace pwadv
