/* ara_synth.h -- device side of the seeded input generator "ARA-GEN-1" (test/bench infrastructure).
 *
 * Not part of the ARA method and not part of the product ABI (include/ara.h).  It exists so that a
 * 4-32 GB Year Event Table can be produced directly in HBM instead of being generated on the host
 * and copied.  The recipe is the integer-only counter generator documented in
 * paper_1412_4556_b200/synth/__init__.py; the device and host versions are tested
 * bit-for-bit against each other (tests/test_synth.py, tests/test_gpu_synth.py).
 *
 * The shapes it produces follow the paper's YET: trials of event ids drawn from a catalogue of C
 * events (Section III "YET"); timestamps are not produced (they never enter
 * Algorithm 1).
 */
#ifndef ARA_SYNTH_H
#define ARA_SYNTH_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Write ids of global occurrences q0 .. q0+count-1 into out[0 .. count):
 *     out[i] = 1 + uni(draw(seed, 1<<32, q0+i), catalog_size)
 * out        device pointer, count*4 bytes, caller-owned.
 * stream     cudaStream_t (NULL = legacy default stream).  Asynchronous.
 * Returns 0 on success, 1 on invalid arguments (catalog_size == 0, out == NULL with count > 0),
 * 6 on a CUDA launch error (message via ara_synth_last_error()). */
__attribute__((visibility("default"))) int ara_synth_yet_ids(uint32_t* out, uint64_t seed, uint64_t q0, uint64_t count, uint32_t catalog_size,
                      void* stream);

__attribute__((visibility("default"))) const char* ara_synth_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
