// kernels_presence.cu -- instantiations of the presence-bitmap ARA kernel.
#include "presence_kernel.cuh"
#include "variants.cuh"

namespace ara {

static const Variant kTable[] = {
    // first per row width = default (B200 sweeps)
    ARA_PRES_FX(1, 1, 32), ARA_PRES(1, 1, 1, 24), ARA_PRES(1, 1, 1, 16),
    ARA_PRES_FX(2, 1, 32), ARA_PRES(2, 1, 1, 24), ARA_PRES(2, 1, 1, 16),
    ARA_PRES_FX(4, 1, 32), ARA_PRES(4, 1, 1, 24), ARA_PRES(4, 1, 1, 16),
    ARA_PRES_FX(8, 1, 32), ARA_PRES(8, 1, 1, 24), ARA_PRES(8, 1, 1, 16),
    ARA_PRES_FX(8, 2, 32), ARA_PRES(8, 2, 1, 24), ARA_PRES(8, 2, 1, 16), ARA_PRES(8, 2, 2, 24), ARA_PRES(8, 2, 1, 28),
};

const Variant* presence_variants_narrow(int* n) {
  *n = (int)(sizeof(kTable) / sizeof(kTable[0]));
  return kTable;
}

}  // namespace ara
