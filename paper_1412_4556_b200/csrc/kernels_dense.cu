// kernels_dense.cu -- instantiations of the dense direct-access ARA kernel.
#include "ara_kernel.cuh"
#include "variants.cuh"

namespace ara {

#define ARA_DENSE(V_, NV_, G_, U_) \
  {KIND_DENSE, (uint32_t)((V_) * (NV_)), V_, NV_, G_, U_, 0, ara_layer_kernel<V_, NV_, G_, U_>, \
   "ara_layer_kernel<V=" #V_ ",NV=" #NV_ ",G=" #G_ ",U=" #U_ ">", ara_layer_kernel<V_, NV_, G_, U_>}

static const Variant kTable[] = {
    // ---- dense kernels: every occurrence gathers its row (the plain direct-access path)
    ARA_DENSE(1, 1, 1, 8),  ARA_DENSE(1, 1, 1, 16),
    ARA_DENSE(2, 1, 1, 8),  ARA_DENSE(2, 1, 1, 16),
    ARA_DENSE(4, 1, 1, 8),  ARA_DENSE(4, 1, 1, 16),
    ARA_DENSE(8, 1, 1, 4),  ARA_DENSE(8, 1, 1, 8),
    ARA_DENSE(8, 2, 2, 4),  ARA_DENSE(8, 2, 2, 8),  ARA_DENSE(8, 2, 1, 4), ARA_DENSE(8, 2, 2, 16), ARA_DENSE(8, 2, 1, 8),
    ARA_DENSE(8, 3, 4, 8),  ARA_DENSE(8, 3, 2, 4),
    ARA_DENSE(8, 4, 4, 8),  ARA_DENSE(8, 4, 2, 4),
    ARA_DENSE(8, 5, 8, 8),  ARA_DENSE(8, 5, 4, 4),
    ARA_DENSE(8, 6, 8, 8),  ARA_DENSE(8, 6, 4, 4),
    ARA_DENSE(8, 7, 8, 8),  ARA_DENSE(8, 7, 4, 4),
    ARA_DENSE(8, 8, 8, 8),  ARA_DENSE(8, 8, 4, 4),
    ARA_DENSE(8, 9, 8, 4),  ARA_DENSE(8, 9, 16, 8),
    ARA_DENSE(8, 10, 8, 4), ARA_DENSE(8, 10, 16, 8),
    ARA_DENSE(8, 11, 8, 4), ARA_DENSE(8, 11, 16, 8),
    ARA_DENSE(8, 12, 8, 4), ARA_DENSE(8, 12, 16, 8),
    ARA_DENSE(8, 13, 8, 4), ARA_DENSE(8, 13, 16, 8),
    ARA_DENSE(8, 14, 8, 4), ARA_DENSE(8, 14, 16, 8),
    ARA_DENSE(8, 15, 8, 4), ARA_DENSE(8, 15, 16, 8),
    ARA_DENSE(8, 16, 8, 4), ARA_DENSE(8, 16, 16, 8),
};

const Variant* dense_variants(int* n) {
  *n = (int)(sizeof(kTable) / sizeof(kTable[0]));
  return kTable;
}

}  // namespace ara
