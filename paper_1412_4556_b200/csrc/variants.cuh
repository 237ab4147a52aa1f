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
};

// Defined in kernels_presence.cu / kernels_dense.cu.  First entry per row width is the default.
const Variant* presence_variants(int* n);
const Variant* dense_variants(int* n);

}  // namespace ara
