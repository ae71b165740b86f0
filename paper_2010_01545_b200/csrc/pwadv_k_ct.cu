// pwadv_k_ct.cu — kernel instantiations (see pwadv_kernels.h).
#include "pwadv_kernels.h"

namespace pwadv {

// column-tile X-march K1c (k_advect_ctile), even nz: slab heights 32..128
CtileKern kern_ctile_even(int kt, bool step, bool fma)
{
    switch (kt) {
    case 32: return PWADV_SF(k_advect_ctile, 32, false);
    case 48: return PWADV_SF(k_advect_ctile, 48, false);
    case 64: return PWADV_SF(k_advect_ctile, 64, false);
    case 96: return PWADV_SF(k_advect_ctile, 96, false);
    case 128: return PWADV_SF(k_advect_ctile, 128, false);
    default: return nullptr;
    }
}

CtileKern kern_ctile(int kt, bool odd, bool step, bool fma)
{
    return odd ? kern_ctile_odd(kt, step, fma) : kern_ctile_even(kt, step, fma);
}

}  // namespace pwadv
