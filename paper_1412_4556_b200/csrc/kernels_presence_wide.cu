// kernels_presence_wide.cu -- instantiations of the presence-bitmap ARA kernel.
#include "presence_kernel.cuh"
#include "variants.cuh"

namespace ara {

static const Variant kTable[] = {
    // first per row width = default: one lane per row with sparse records (G = 1); then full-row batches
    ARA_PRES_FX(8, 10, 32), ARA_PRES(8, 10, 16, 16), ARA_PRES(8, 10, 8, 16), ARA_PRES(8, 10, 16, 24),
    ARA_PRES_FX(8, 11, 32), ARA_PRES(8, 11, 16, 16), ARA_PRES(8, 11, 8, 16), ARA_PRES(8, 11, 16, 24),
    ARA_PRES_FX(8, 12, 32), ARA_PRES(8, 12, 16, 16), ARA_PRES(8, 12, 8, 16), ARA_PRES(8, 12, 16, 24),
    ARA_PRES_FX(8, 13, 32), ARA_PRES(8, 13, 16, 16), ARA_PRES(8, 13, 8, 16), ARA_PRES(8, 13, 16, 24),
    ARA_PRES_FX(8, 14, 32), ARA_PRES(8, 14, 16, 16), ARA_PRES(8, 14, 8, 16), ARA_PRES(8, 14, 16, 24),
    ARA_PRES_FX(8, 15, 32), ARA_PRES(8, 15, 16, 16), ARA_PRES(8, 15, 8, 16), ARA_PRES(8, 15, 16, 24),
    ARA_PRES_FX(8, 16, 32), ARA_PRES(8, 16, 16, 16), ARA_PRES(8, 16, 8, 16), ARA_PRES(8, 16, 16, 24),
};

const Variant* presence_variants_wide(int* n) {
  *n = (int)(sizeof(kTable) / sizeof(kTable[0]));
  return kTable;
}

}  // namespace ara
