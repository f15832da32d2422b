/* oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle of the PAAM analysis (and, in des.cpp, of the PAAM
 * arbitration simulation).  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  It shares no code with the CUDA product path; it includes
 * only gen/paam_gen.h (the shared seeded input generator, which holds none of the method).
 *
 * The declarations below are the oracle's own; the flat batch has the same field meanings as
 * paam_batch in include/paam.h, but is declared independently here.
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_UNSCHED UINT64_MAX
#define OR_UNB UINT64_MAX

/* per-set status, same numbering as documented in DESIGN.md "Validation" */
enum { OR_OK = 0, OR_ERANGE = 1, OR_EDANGLING = 2, OR_EACCEL = 3, OR_ESHAPE = 4, OR_EDUPPRIO = 5,
       OR_EDEADLINE = 6, OR_ECORE = 7 };
#define OR_FLAG_BLOCKING_SOUND 0x1u
#define OR_FLAG_WFD_UNITS 0x2u

typedef struct {
  uint32_t n_sets;
  int32_t mem;
  uint32_t n_chains, n_cbs, n_segs, n_execs, n_accels, n_bins;
  const uint32_t *set_chain_off, *set_exec_off, *set_accel_off;
  const uint64_t *chain_T, *chain_D;
  const uint32_t *chain_prio;
  const uint8_t *chain_class;
  const uint32_t *chain_cb_off;
  const uint16_t *cb_exec;
  const uint32_t *cb_seg_off;
  const uint8_t *seg_kind;
  const uint64_t *seg_wcet;
  const uint8_t *seg_accel, *seg_unit;
  const uint8_t *exec_core;
  const uint32_t *exec_prio;
  const uint8_t *exec_wait;
  const uint8_t *accel_buckets, *accel_units, *accel_server_core;
  const uint64_t *accel_eps, *accel_kappa;
  const uint32_t *set_bin;
  uint64_t comm_cost;
  uint32_t flags;
  uint32_t _pad;
} or_batch;

/* Per-set detail for unit tests (first set of a batch). Arrays sized generously. */
#define OR_DMAX 256
typedef struct {
  int32_t status;
  uint32_t n_sub, n_aseg;
  /* per sub-chain, in the order chains appear, then by position in the chain */
  int32_t sub_chain[OR_DMAX], sub_exec[OR_DMAX];
  uint64_t sub_B[OR_DMAX], sub_E[OR_DMAX], sub_S[OR_DMAX], sub_C[OR_DMAX], sub_Hstar[OR_DMAX],
      sub_R[OR_DMAX], sub_iters[OR_DMAX];
  /* per ACCEL segment, in global segment order of the set */
  int32_t aseg_sub[OR_DMAX], aseg_bucket[OR_DMAX];
  uint64_t aseg_Astar[OR_DMAX], aseg_LPB[OR_DMAX], aseg_H[OR_DMAX];
  /* work counters: mu-term evaluations, literal (one per interfering segment) and regrouped
   * (one per interfering chain and unit), over Lemma 2, Lemma 3 and the hp/hpp sums */
  uint64_t mu_literal, mu_regrouped, iterations;
} or_detail;

int32_t oracle_analyze_batch(const or_batch* b, uint64_t* out_wcrt, uint8_t* out_sched,
                             int32_t* out_status, int64_t* out_bins, int nthreads);
int32_t oracle_analyze_detail(const or_batch* b, uint32_t set_index, or_detail* out);

/* Generate (gen/paam_gen.h) and analyse sets [first, first+n) without materialising the batch.
 * params points at a pg_params; counters (may be NULL) receives {mu_literal, mu_regrouped,
 * iterations} summed over the sets. */
int32_t oracle_generate_analyze(const void* params, uint64_t seed, uint64_t first, uint32_t n,
                                uint64_t comm_cost, uint32_t flags, uint64_t* out_wcrt_or_null,
                                uint32_t wcrt_stride, uint8_t* out_sched, int64_t* out_bins,
                                uint64_t* counters, int nthreads);

/* Discrete-event simulation (des.cpp, DESIGN.md App. A): per chain max / count of observed end-to-end
 * responses, misc[3] = {deadline misses (D16), BE drops (D14), peak backlog = the most live
 * instances the chain ever had at once (D14: CRITICAL chains queue every release)}; per set an order-independent
 * FNV-1a-64 digest of the event records; violations of `bound` counted for CRITICAL chains of sets
 * whose every CRITICAL chain has bound <= D (the analysis' schedulable sets).  phases_or_null: explicit release phases per chain (brute force), else pg_phase(). */
int32_t oracle_simulate_batch(const or_batch* b, uint64_t horizon, uint64_t seed, uint64_t first_index,
                              uint32_t sim_flags /* 1 = FIFO_DIRECT */, const uint64_t* phases_or_null, uint64_t* out_resp, uint64_t* out_count,
                              uint64_t* out_misc, uint64_t* out_digest, const uint64_t* bound,
                              int64_t* out_violations, int nthreads);

#ifdef __cplusplus
}
#endif
