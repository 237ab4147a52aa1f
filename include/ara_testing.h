/* ara_testing.h -- TEST-ONLY exports of libara_testing.so (test hooks stay out of the
 * product ABI of include/ara.h).  The library reads a context created by libara.so (same process, same
 * build: it shares the internal context layout, csrc/ctx.cuh); it performs no analysis.
 * Seeded input generation for tests lives in libara_synth.so (include/ara_synth.h). */
#ifndef ARA_TESTING_H
#define ARA_TESTING_H

#include "ara.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Copy row `event` (0 <= event <= C; row 0 is the all-zero row) of layer `layer`'s event-major
 * direct-access table T[e][0..jpad) -- PAPER.md:209-213's interleaved ELT representation, fp32 -- to
 * HOST out[jpad] (jpad = the layer's row stride in floats, ara_layer_info).  Synchronous.
 * Errors: ARA_E_ARG (NULL ctx/out, layer out of range), ARA_E_RANGE (event > C), ARA_E_CUDA. */
ARA_API ara_status ara_table_row(ara_ctx* ctx, uint32_t layer, uint32_t event, float* out);

/* Message of this library's last error on the calling thread. */
ARA_API const char* ara_testing_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* ARA_TESTING_H */
