// study.cuh -- parameters of the Section IV.B data-structure study kernels (kernels_study.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

namespace ara {

enum StudyLayout { STUDY_INTERLEAVED = 0, STUDY_INDEPENDENT = 1, STUDY_SORTED = 2, STUDY_HASH = 3, STUDY_INDEX = 4 };

struct StudyParams {
  const float* table;        // interleaved (C+1) x jpad
  const float* indep;        // J x (C+1)
  const uint32_t* sorted_ids;
  const float* sorted_loss;
  const uint32_t* sorted_off;  // J+1 offsets into sorted_ids / sorted_loss (device)
  const uint2* hash;           // STUDY_HASH: per ELT an open-addressing table of (event id, loss bits)
  const uint32_t* hash_off;    // J+1 offsets (in slots); each ELT's capacity is a power of two
  const uint32_t* hash_bits;   // J: log2 of each ELT's capacity
  const uint32_t* row_index;   // STUDY_INDEX: event -> compact row (0 = no loss in any ELT), (C+1) entries
  const float* compact;        // compact rows (jpad floats each), row 0 all zero
  const uint32_t* ids;
  const uint64_t* offsets;
  uint64_t num_trials;
  uint64_t rows;  // C + 1
  uint32_t K, C, J, jpad;
  double* ylt;
  double r2, l2, r3, l3;
  double r1[128], l1[128];
};

void* study_kernel_fn(int layout);
void study_transpose(float* indep, const float* table, uint32_t jpad, uint32_t J, uint64_t rows, int sms,
                     cudaStream_t s);

}  // namespace ara
