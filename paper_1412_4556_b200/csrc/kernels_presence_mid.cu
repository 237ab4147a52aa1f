// kernels_presence_mid.cu -- instantiations of the presence-bitmap ARA kernel.
#include "presence_kernel.cuh"
#include "variants.cuh"

namespace ara {

static const Variant kTable[] = {
    // first per row width = default: one lane per row with sparse records (G = 1); then full-row batches
    ARA_PRES_FX(8, 3, 32), ARA_PRES(8, 3, 2, 16), ARA_PRES(8, 3, 4, 16), ARA_PRES(8, 3, 2, 24),
    ARA_PRES_FX(8, 4, 32), ARA_PRES(8, 4, 2, 16), ARA_PRES(8, 4, 4, 16), ARA_PRES(8, 4, 2, 24),
    ARA_PRES_FX(8, 5, 32), ARA_PRES(8, 5, 16, 16), ARA_PRES(8, 5, 8, 16), ARA_PRES(8, 5, 16, 24),
    ARA_PRES_FX(8, 6, 32), ARA_PRES(8, 6, 16, 16), ARA_PRES(8, 6, 8, 16), ARA_PRES(8, 6, 16, 24),
    ARA_PRES_FX(8, 7, 32), ARA_PRES(8, 7, 16, 16), ARA_PRES(8, 7, 8, 16), ARA_PRES(8, 7, 16, 24),
    ARA_PRES_FX(8, 8, 32), ARA_PRES(8, 8, 16, 16), ARA_PRES(8, 8, 8, 16), ARA_PRES(8, 8, 16, 24),
    ARA_PRES_FX(8, 9, 32), ARA_PRES(8, 9, 16, 16), ARA_PRES(8, 9, 8, 16), ARA_PRES(8, 9, 16, 24),
};

const Variant* presence_variants_mid(int* n) {
  *n = (int)(sizeof(kTable) / sizeof(kTable[0]));
  return kTable;
}

}  // namespace ara
