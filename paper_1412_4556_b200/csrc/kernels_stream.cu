// kernels_stream.cu -- instantiations of the fixed-length-trial ARA kernels (options beside the default
// presence kernel): the per-lane-queue kernel (lane_kernel.cuh), the warp-ring kernel (stream_kernel.cuh)
// and the candidate-mask kernel (mask_kernel.cuh).
#include "lane_kernel.cuh"
#include "mask_kernel.cuh"
#include "stream_kernel.cuh"
#include "variants.cuh"

namespace ara {

#define ARA_LANE(NW_) \
  {NW_, ara_lane_kernel<NW_, false>, ara_lane_kernel<NW_, true>, "ara_lane_kernel<NW=" #NW_ ">", 0, 0}
#define ARA_LANE_XS(NW_) \
  {NW_, ara_lane_kernel<NW_, false, true>, ara_lane_kernel<NW_, true, true>, "ara_lane_kernel<NW=" #NW_ ",XS>", 0, 1}
#define ARA_LANE_XS2(NW_) \
  {NW_, ara_lane_kernel<NW_, false, true, 2>, ara_lane_kernel<NW_, true, true, 2>, "ara_lane_kernel<NW=" #NW_ ",XS2>", 0, 1}
#define ARA_MASK(NW_) \
  {NW_, ara_mask_kernel<NW_, false>, ara_mask_kernel<NW_, true>, "ara_mask_kernel<NW=" #NW_ ">", 2, 0}
#define ARA_MASK_PF(NW_, D_)                                                                  \
  {NW_, ara_mask_kernel<NW_, false, 8, D_>, ara_mask_kernel<NW_, true, 8, D_>,                      \
   "ara_mask_kernel<NW=" #NW_ ",PFD=" #D_ ">", 2, 0}
#define ARA_RING(NW_) \
  {NW_, ara_stream_kernel<NW_, false>, ara_stream_kernel<NW_, true>, "ara_stream_kernel<NW=" #NW_ ">", 1, 0}

// ARA_OPT_STREAM = index + 1; the first XS entry is the automatic choice for layers whose folded bitmap
// nominates far more candidates than it holds rows (ARA_OPT_FILTER auto)
static const StreamVariant kStream[] = {ARA_LANE(32),    ARA_LANE(24),     ARA_LANE(16),    ARA_RING(32),
                                        ARA_LANE_XS(24), ARA_LANE_XS2(24), ARA_LANE_XS(32), ARA_LANE_XS(16),
                                        ARA_MASK(32),    ARA_MASK_PF(32, 4)};

const StreamVariant* stream_variants(int* n) {
  *n = (int)(sizeof(kStream) / sizeof(kStream[0]));
  return kStream;
}

}  // namespace ara
