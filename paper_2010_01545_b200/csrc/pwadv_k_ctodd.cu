// pwadv_k_ctodd.cu — kernel instantiations (see pwadv_kernels.h).
#include "pwadv_kernels.h"

namespace pwadv {

// column-tile X-march K1c, odd nz (column-pair rows): slab heights 64 / 128
CtileKern kern_ctile_odd(int kt, bool step, bool fma)
{
    switch (kt) {
    case 64: return PWADV_SF(k_advect_ctile, 64, true);
    case 128: return PWADV_SF(k_advect_ctile, 128, true);
    default: return nullptr;
    }
}

}  // namespace pwadv
