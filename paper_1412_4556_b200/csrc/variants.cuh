// variants.cuh -- registry of compiled ARA kernel instantiations (one translation unit per kernel kind,
// so the template sets compile in parallel).
#pragma once
#include <stdint.h>

#include "ara_kernel.cuh"

namespace ara {

typedef void (*KernelFn)(LayerParams);

enum KernelKind { KIND_PRESENCE = 0, KIND_DENSE = 1 };

struct Variant {
  int kind;
  uint32_t jpad;
  int V, NV, G, U, NW;  // U: dense rows per group; NW: presence warps per block (fixed block size)
  KernelFn fn;
  const char* name;
  KernelFn fn_olt;  // the same kernel also producing the occurrence loss table (presence kernels; dense: fn)
  KernelFn fn_fx = nullptr;      // presence, one lane per row: with the exact filter stage (FX), or nullptr
  KernelFn fn_fx_olt = nullptr;  // the same with the occurrence loss table
  KernelFn fn_pc = nullptr;      // presence, one lane per row: precombined o[e] table, or nullptr
  KernelFn fn_pc_olt = nullptr;
};

// Defined in kernels_presence.cu / kernels_dense.cu.  First entry per row width is the default.
const Variant* presence_variants_narrow(int* n);  // rows of <= 16 columns
const Variant* presence_variants_mid(int* n);     // 17..72 columns
const Variant* presence_variants_wide(int* n);    // 73..128 columns
const Variant* dense_variants(int* n);

// Fixed-length-trial kernel (stream_kernel.cuh): one instantiation serves every row width.
struct StreamVariant {
  int NW;
  KernelFn fn, fn_olt;
  const char* name;
  int ring;  // 0: per-lane queues (lane_kernel.cuh), 1: warp hit ring (stream_kernel.cuh), 2: candidate masks
             // (mask_kernel.cuh, trials of <= 1024 occurrences)
  int xs;    // 1: exact scan filter (lane_kernel.cuh XS)
};
const StreamVariant* stream_variants(int* n);  // kernels_stream.cu; first = default

// Variant-table entries of the presence kernel (presence_kernel.cuh; used by the kernels_presence*.cu
// instantiation tables).  ARA_PRES: one (V, NV, G, NW) shape with and without the occurrence loss table.
// ARA_PRES_FX: the default one-lane-per-row shape of a row width, also instantiated with the exact filter
// stage (FX) and the precombined occurrence-net table (PC).
#define ARA_PRES(V_, NV_, G_, NW_) \
  {KIND_PRESENCE, (uint32_t)((V_) * (NV_)), V_, NV_, G_, 0, NW_, ara_presence_kernel<V_, NV_, G_, NW_, false>, \
   "ara_presence_kernel<V=" #V_ ",NV=" #NV_ ",G=" #G_ ",NW=" #NW_ ">", ara_presence_kernel<V_, NV_, G_, NW_, true>}
#define ARA_PRES_FX(V_, NV_, NW_) \
  {KIND_PRESENCE, (uint32_t)((V_) * (NV_)), V_, NV_, 1, 0, NW_, ara_presence_kernel<V_, NV_, 1, NW_, false>, \
   "ara_presence_kernel<V=" #V_ ",NV=" #NV_ ",G=1,NW=" #NW_ ">", ara_presence_kernel<V_, NV_, 1, NW_, true>, \
   ara_presence_kernel<V_, NV_, 1, NW_, false, true>, ara_presence_kernel<V_, NV_, 1, NW_, true, true>, \
   ara_presence_kernel<V_, NV_, 1, NW_, false, false, true>, ara_presence_kernel<V_, NV_, 1, NW_, true, false, true>}

}  // namespace ara
