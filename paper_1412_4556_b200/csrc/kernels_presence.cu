// kernels_presence.cu -- instantiations of the presence-bitmap ARA kernel.
#include "presence_kernel.cuh"
#include "variants.cuh"

namespace ara {

#define ARA_PRES(V_, NV_, G_, NW_) \
  {KIND_PRESENCE, (uint32_t)((V_) * (NV_)), V_, NV_, G_, 0, NW_, ara_presence_kernel<V_, NV_, G_, NW_>, \
   "ara_presence_kernel<V=" #V_ ",NV=" #NV_ ",G=" #G_ ",NW=" #NW_ ">"}


static const Variant kTable[] = {
    // ---- presence-bitmap kernels (default path); first per row width = default (B200 sweeps)
    ARA_PRES(1, 1, 1, 32), ARA_PRES(1, 1, 1, 24), ARA_PRES(1, 1, 1, 16),
    ARA_PRES(2, 1, 1, 32), ARA_PRES(2, 1, 1, 24), ARA_PRES(2, 1, 1, 16),
    ARA_PRES(4, 1, 1, 32), ARA_PRES(4, 1, 1, 24), ARA_PRES(4, 1, 1, 16),
    ARA_PRES(8, 1, 1, 32), ARA_PRES(8, 1, 1, 24), ARA_PRES(8, 1, 1, 16),
    ARA_PRES(8, 2, 1, 32), ARA_PRES(8, 2, 1, 24), ARA_PRES(8, 2, 1, 16), ARA_PRES(8, 2, 2, 24), ARA_PRES(8, 2, 1, 28),
    ARA_PRES(8, 3, 2, 16), ARA_PRES(8, 3, 4, 16), ARA_PRES(8, 3, 2, 24),
    ARA_PRES(8, 4, 2, 16), ARA_PRES(8, 4, 4, 16), ARA_PRES(8, 4, 2, 24),
    ARA_PRES(8, 5, 16, 16), ARA_PRES(8, 5, 8, 16), ARA_PRES(8, 5, 16, 24),
    ARA_PRES(8, 6, 16, 16), ARA_PRES(8, 6, 8, 16), ARA_PRES(8, 6, 16, 24),
    ARA_PRES(8, 7, 16, 16), ARA_PRES(8, 7, 8, 16), ARA_PRES(8, 7, 16, 24),
    ARA_PRES(8, 8, 16, 16), ARA_PRES(8, 8, 8, 16), ARA_PRES(8, 8, 16, 24),
    ARA_PRES(8, 9, 16, 16), ARA_PRES(8, 9, 8, 16), ARA_PRES(8, 9, 16, 24),
    ARA_PRES(8, 10, 16, 16), ARA_PRES(8, 10, 8, 16), ARA_PRES(8, 10, 16, 24),
    ARA_PRES(8, 11, 16, 16), ARA_PRES(8, 11, 8, 16), ARA_PRES(8, 11, 16, 24),
    ARA_PRES(8, 12, 16, 16), ARA_PRES(8, 12, 8, 16), ARA_PRES(8, 12, 16, 24),
    ARA_PRES(8, 13, 16, 16), ARA_PRES(8, 13, 8, 16), ARA_PRES(8, 13, 16, 24),
    ARA_PRES(8, 14, 16, 16), ARA_PRES(8, 14, 8, 16), ARA_PRES(8, 14, 16, 24),
    ARA_PRES(8, 15, 16, 16), ARA_PRES(8, 15, 8, 16), ARA_PRES(8, 15, 16, 24),
    ARA_PRES(8, 16, 16, 16), ARA_PRES(8, 16, 8, 16), ARA_PRES(8, 16, 16, 24),
};

const Variant* presence_variants(int* n) {
  *n = (int)(sizeof(kTable) / sizeof(kTable[0]));
  return kTable;
}

}  // namespace ara
