// pwadv_k_small.cu — kernel instantiations (see pwadv_kernels.h).
#include "pwadv_kernels.h"

namespace pwadv {

// the X-march at the plain (not warp-specialised) thread budgets 384..128
// (PWADV opts.max_threads; experiments and the tiling tests)
XmarchKern kern_generic_small(int maxt, bool fix, bool step, bool fma)
{
    switch (maxt) {
    case 384: return fix ? PWADV_SF(k_advect_xmarch, 384, true) : PWADV_SF(k_advect_xmarch, 384, false);
    case 256: return fix ? PWADV_SF(k_advect_xmarch, 256, true) : PWADV_SF(k_advect_xmarch, 256, false);
    case 192: return fix ? PWADV_SF(k_advect_xmarch, 192, true) : PWADV_SF(k_advect_xmarch, 192, false);
    case 128: return fix ? PWADV_SF(k_advect_xmarch, 128, true) : PWADV_SF(k_advect_xmarch, 128, false);
    default: return nullptr;
    }
}

}  // namespace pwadv
