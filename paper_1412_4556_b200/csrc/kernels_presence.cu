// kernels_presence.cu -- instantiations of the presence-bitmap ARA kernel.
#include "presence_kernel.cuh"
#include "variants.cuh"

namespace ara {

#define ARA_PRES(V_, NV_, G_, NW_) \
  {KIND_PRESENCE, (uint32_t)((V_) * (NV_)), V_, NV_, G_, 0, NW_, ara_presence_kernel<V_, NV_, G_, NW_, false>, \
   "ara_presence_kernel<V=" #V_ ",NV=" #NV_ ",G=" #G_ ",NW=" #NW_ ">", ara_presence_kernel<V_, NV_, G_, NW_, true>}
// default one-lane-per-row variant, also instantiated with the exact filter stage (FX) and with the
// precombined occurrence-net table (PC)
#define ARA_PRES_FX(V_, NV_, NW_) \
  {KIND_PRESENCE, (uint32_t)((V_) * (NV_)), V_, NV_, 1, 0, NW_, ara_presence_kernel<V_, NV_, 1, NW_, false>, \
   "ara_presence_kernel<V=" #V_ ",NV=" #NV_ ",G=1,NW=" #NW_ ">", ara_presence_kernel<V_, NV_, 1, NW_, true>, \
   ara_presence_kernel<V_, NV_, 1, NW_, false, true>, ara_presence_kernel<V_, NV_, 1, NW_, true, true>, \
   ara_presence_kernel<V_, NV_, 1, NW_, false, false, true>, ara_presence_kernel<V_, NV_, 1, NW_, true, false, true>}


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
