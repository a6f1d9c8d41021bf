/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the clairvoyant plan build.
 *
 * A plain-C restatement of the reference (clairsim) hot path, written from the
 * reference's published behaviour, each function citing the file:line it follows
 * (paths relative to /root/reference/proj).  Parity of this restatement is pinned by
 * tests/test_oracle.py against (a) the reference's own golden vectors
 * (tests/test_rng.cpp:12-22, fixtures/perm_seed42_*.txt) re-hosted in tests/golden/ and
 * (b) the reference itself compiled untouched into oracle/_ref/ (oracle/Makefile).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this.
 */
#ifndef CLAIRPLAN_ORACLE_H
#define CLAIRPLAN_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

uint64_t orc_mix64(uint64_t z);
uint64_t orc_derive_key(uint64_t seed, uint64_t tag);
/* bounded draw at stream state (key, *pos): advances *pos like CounterRng::bounded */
uint64_t orc_bounded(uint64_t key, uint64_t* pos, uint64_t n);
int orc_epoch_permutation(uint64_t seed, uint32_t epoch, uint32_t F, uint32_t* out);
int orc_epoch_permutation_norej(uint64_t seed, uint32_t epoch, uint32_t F, uint32_t* out);
void orc_batch_slice(uint64_t batch_size, uint32_t workers, uint32_t worker, uint64_t* begin,
                     uint64_t* end);
int orc_generate_sizes(uint64_t F, double mean, double sigma, int has_total, double total,
                       uint64_t seed, int sigma_relative, double* out);

typedef struct orc_plan orc_plan;
/* full plan from the seed; returns NULL on invalid partition (message via orc_last_error) */
orc_plan* orc_plan_build(uint64_t seed, uint32_t F, uint32_t N, uint32_t B, uint32_t E,
                         int drop_last, uint32_t J, const double* caps, const double* sizes);
/* nopfs_assign_caches on explicit streams + dense counts (N x F) */
orc_plan* orc_assign_from_streams(uint32_t N, uint32_t F, const uint32_t* entries,
                                  const uint64_t* offsets, const uint32_t* counts, uint32_t J,
                                  const double* caps, const double* sizes);
uint64_t orc_plan_stream(const orc_plan* p, uint32_t w, const uint32_t** data);
uint64_t orc_plan_class_list(const orc_plan* p, uint32_t w, uint32_t j, const uint32_t** data);
uint64_t orc_plan_holders(const orc_plan* p, const uint64_t** offsets, const uint32_t** holders);
void orc_plan_free(orc_plan* p);
const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
