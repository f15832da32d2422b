/* paam_gen.h -- seeded, integer-only, counter-based synthetic chain-set generator.
 *
 * INPUT GENERATION ONLY.  This module is the one piece of code that both the
 * CPU oracle (oracle/, compiled by g++) and the CUDA product path
 * (paper_2404_06452_b200/csrc/generate.cu, compiled by nvcc) include.  It holds
 * none of the analysed method's arithmetic: no buckets, no interference sets,
 * no fixed points -- only the workload recipe of SURVEY.md §8(d), which follows
 * the paper's analytical study (PAPER.md:680-686 / :931-937: "fixed chain length
 * of 4 callbacks per chain", "random periodicity", "1:1 Accelerator:CPU
 * utilization ratio ... equally distributed amongst all the callbacks") and
 * SPEC.md:368-397 (log-uniform periods, one accelerator segment per callback
 * placed between two CPU halves, random unique priorities, worst-fit executor
 * placement).
 *
 * Every draw is a pure function of (seed, set index, purpose, draw index), so a
 * set can be generated independently on any thread of any rank, and the host and
 * the device produce identical bytes.
 */
#pragma once
#include <stdint.h>
#include "exp2_table.h"

#ifdef __CUDACC__
#define PG_FN static __host__ __device__ __forceinline__
#ifdef __CUDA_ARCH__
#define PG_TABLE(i) __ldg(PG_EXP2_Q30_DEV + (i))
#else
#define PG_TABLE(i) PG_EXP2_Q30[i]
#endif
#else
#define PG_FN static inline
#define PG_TABLE(i) PG_EXP2_Q30[i]
#endif

#define PG_MAX_CHAINS 32
#define PG_MAX_CBS_PER_CHAIN 8
#define PG_MAX_CBS 64
#define PG_MAX_EXEC 32
#define PG_MAX_ACCEL 4

/* Layout-identical to paam_gen_params in include/paam.h (checked by tests). */
typedef struct {
  uint32_t m_lo, m_hi, cbs_per_chain, n_bins;
  uint32_t u_lo_q20, u_step_q20;           /* U_total of bin b = u_lo + b*u_step, units 2^-20 */
  uint32_t ratio_acc, ratio_cpu;           /* accelerator : CPU utilisation split */
  uint32_t period_min_us, period_span_q12; /* T = Tmin * 2^(x/4096), x uniform in [0, span] */
  uint32_t exec_mode, n_cores, n_exec;     /* 0: executor per chain on n_cores; 1: n_exec shared */
  uint32_t n_accel;
  uint32_t buckets[PG_MAX_ACCEL], units[PG_MAX_ACCEL];
  uint64_t eps[PG_MAX_ACCEL], kappa[PG_MAX_ACCEL];
  uint32_t be_frac_q16, spin_frac_q16, cpu_only_frac_q16, xexec_frac_q16, rm_priorities;
  uint32_t _pad;
} pg_params;

/* One generated set, set-local indices, fixed capacity. */
typedef struct {
  uint32_t m, K, n_cb, n_exec, n_accel, n_seg, bin;
  uint64_t T[PG_MAX_CHAINS], D[PG_MAX_CHAINS];
  uint32_t prio[PG_MAX_CHAINS];
  uint8_t cls[PG_MAX_CHAINS];
  uint8_t chain_ncb[PG_MAX_CHAINS];        /* callbacks of chain c are [c*K, c*K + ncb) */
  uint16_t cb_exec[PG_MAX_CBS];
  uint8_t cb_nseg[PG_MAX_CBS];             /* 1 (CPU only) or 3 (CPU, ACCEL, CPU) */
  uint8_t cb_accel[PG_MAX_CBS], cb_unit[PG_MAX_CBS];
  uint64_t cb_wcet[PG_MAX_CBS][3];
  uint8_t exec_core[PG_MAX_EXEC], exec_wait[PG_MAX_EXEC];
  uint32_t exec_prio[PG_MAX_EXEC];
  uint8_t acc_buckets[PG_MAX_ACCEL], acc_units[PG_MAX_ACCEL], acc_server_core[PG_MAX_ACCEL];
  uint64_t acc_eps[PG_MAX_ACCEL], acc_kappa[PG_MAX_ACCEL];
} pg_set;

enum { PG_D_M = 1, PG_D_CUT, PG_D_PERIOD, PG_D_CPUONLY, PG_D_ACC, PG_D_UNIT, PG_D_PERM,
       PG_D_SPIN, PG_D_XEXEC, PG_D_PHASE };

/* Release phase of chain c of set `index` for a simulation seeded with `seed` (DESIGN.md App. A D2):
 * 0 when seed == 0 (synchronous critical instant), else uniform in [0, T).  Input generation: the
 * simulator draws no random numbers itself; both sides take the phases from here. */

PG_FN uint64_t pg_mix(uint64_t z) { /* SplitMix64 finaliser */
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
PG_FN uint64_t pg_key(uint64_t seed, uint64_t set_index) { return pg_mix(seed ^ pg_mix(set_index)); }
PG_FN uint64_t pg_draw(uint64_t key, uint32_t purpose, uint32_t idx) {
  return pg_mix(key + pg_mix(((uint64_t)purpose << 32) | idx));
}
/* uniform in [0, n) */
PG_FN uint32_t pg_bounded(uint64_t r, uint32_t n) { return (uint32_t)(((r >> 32) * (uint64_t)n) >> 32); }
/* Bernoulli with probability q16 / 65536 */
PG_FN int pg_coin(uint64_t r, uint32_t q16) { return (uint32_t)(r >> 48) < q16; }

PG_FN uint64_t pg_phase(uint64_t seed, uint64_t index, uint32_t c, uint64_t T) {
  if (seed == 0 || T == 0) return 0;
  const uint64_t r = pg_draw(pg_key(seed, index), PG_D_PHASE, c);
#ifdef __CUDA_ARCH__
  return __umul64hi(r, T);
#else
  return (uint64_t)(((unsigned __int128)r * T) >> 64);
#endif
}

/* Returns 0 on success, nonzero if the parameters exceed the generator's caps. */
PG_FN int pg_check_params(const pg_params* p) {
  if (p->m_lo < 1 || p->m_hi < p->m_lo || p->m_hi > PG_MAX_CHAINS) return 1;
  if (p->cbs_per_chain < 1 || p->cbs_per_chain > PG_MAX_CBS_PER_CHAIN) return 1;
  if (p->m_hi * p->cbs_per_chain > PG_MAX_CBS) return 1;
  if (p->ratio_acc + p->ratio_cpu == 0) return 1;
  if (p->period_min_us < 1 || p->period_min_us > (1u << 21) || p->period_span_q12 > 10u * 4096u) return 1;
  if (p->n_accel < 1 || p->n_accel > PG_MAX_ACCEL) return 1;
  for (uint32_t a = 0; a < p->n_accel; a++)
    if (p->buckets[a] < 1 || p->buckets[a] > 32 || p->units[a] < 1 || p->units[a] > 8) return 1;
  if (p->exec_mode == 0 && (p->n_cores < 1 || p->n_cores > 32)) return 1;
  if ((uint64_t)p->u_lo_q20 + (uint64_t)(p->n_bins ? p->n_bins - 1 : 0) * p->u_step_q20 >= (1ull << 31)) return 1;
  if (p->exec_mode == 1 && (p->n_exec < 2 || p->n_exec > PG_MAX_EXEC)) return 1;
  if (p->exec_mode > 1) return 1;
  return 0;
}

/* Generate set `index` of the stream `seed`.  Follows SURVEY.md §8(d). */
PG_FN void pg_generate_set(const pg_params* p, uint64_t seed, uint64_t index, pg_set* s) {
  const uint64_t key = pg_key(seed, index);
  const uint32_t K = p->cbs_per_chain;
  s->K = K;
  s->bin = p->n_bins ? (uint32_t)(index % p->n_bins) : 0u;
  const uint64_t U = (uint64_t)p->u_lo_q20 + (uint64_t)s->bin * p->u_step_q20; /* Q20 */
  const uint32_t m = p->m_lo + pg_bounded(pg_draw(key, PG_D_M, 0), p->m_hi - p->m_lo + 1);
  s->m = m;

  /* Per-chain utilisation: m-1 sorted uniform cut points of [0, U] (integer UUniFast analogue). */
  uint64_t cut[PG_MAX_CHAINS];
  for (uint32_t j = 0; j + 1 < m; j++) {
    cut[j] = pg_bounded(pg_draw(key, PG_D_CUT, j), (uint32_t)U + 1u);
  }
  for (uint32_t j = 1; j + 1 < m; j++) { /* insertion sort */
    uint64_t v = cut[j]; int32_t i = (int32_t)j - 1;
    while (i >= 0 && cut[i] > v) { cut[i + 1] = cut[i]; i--; }
    cut[i + 1] = v;
  }
  uint64_t share[PG_MAX_CHAINS];
  uint64_t prev = 0;
  for (uint32_t c = 0; c < m; c++) {
    uint64_t hi = (c + 1 < m) ? cut[c] : U;
    share[c] = hi - prev;
    prev = hi;
  }

  /* Log-uniform periods rounded to 1 us; implicit deadlines D = T. */
  for (uint32_t c = 0; c < m; c++) {
    uint32_t x = pg_bounded(pg_draw(key, PG_D_PERIOD, c), p->period_span_q12 + 1);
    uint32_t oct = x >> 12, frac = x & 4095u;
    uint64_t t_us = (((uint64_t)p->period_min_us * PG_TABLE(frac)) << oct) >> 30;
    if (t_us < 1) t_us = 1;
    s->T[c] = t_us * 1000ull;
    s->D[c] = s->T[c];
  }

  /* WCETs: chain budget C = u*T split evenly over K callbacks (remainder to the first),
   * each callback = CPU floor(E/2), ACCEL A, CPU ceil(E/2) with A = budget*a/(a+b). */
  uint32_t ncb = 0;
  uint64_t chain_cpu[PG_MAX_CHAINS];
  for (uint32_t c = 0; c < m; c++) {
    const uint64_t C = (share[c] * s->T[c]) >> 20;
    const uint64_t base = C / K, rem = C % K;
    s->chain_ncb[c] = (uint8_t)K;
    chain_cpu[c] = 0;
    for (uint32_t j = 0; j < K; j++) {
      const uint32_t cb = c * K + j;
      const uint64_t budget = base + (j < rem ? 1 : 0);
      s->cb_accel[cb] = 0; s->cb_unit[cb] = 0;
      if (p->cpu_only_frac_q16 && pg_coin(pg_draw(key, PG_D_CPUONLY, cb), p->cpu_only_frac_q16)) {
        s->cb_nseg[cb] = 1;
        s->cb_wcet[cb][0] = budget ? budget : 1;
        s->cb_wcet[cb][1] = 0; s->cb_wcet[cb][2] = 0;
        chain_cpu[c] += s->cb_wcet[cb][0];
      } else {
        uint64_t A = budget * p->ratio_acc / (p->ratio_acc + p->ratio_cpu);
        uint64_t E = budget - A;
        uint64_t e1 = E / 2, e2 = E - E / 2;
        s->cb_nseg[cb] = 3;
        s->cb_wcet[cb][0] = e1 ? e1 : 1;
        s->cb_wcet[cb][1] = A ? A : 1;
        s->cb_wcet[cb][2] = e2 ? e2 : 1;
        const uint32_t a = pg_bounded(pg_draw(key, PG_D_ACC, cb), p->n_accel);
        s->cb_accel[cb] = (uint8_t)a;
        s->cb_unit[cb] = (uint8_t)pg_bounded(pg_draw(key, PG_D_UNIT, cb), p->units[a]);
        chain_cpu[c] += s->cb_wcet[cb][0] + s->cb_wcet[cb][2];
      }
      ncb++;
    }
  }
  s->n_cb = ncb;

  /* Unique priorities (larger = higher): CAPA-random permutation, or rate-monotonic. */
  if (p->rm_priorities) {
    for (uint32_t c = 0; c < m; c++) {
      uint32_t rank = 0; /* chains strictly before c in (T asc, index asc) */
      for (uint32_t d = 0; d < m; d++)
        if (s->T[d] < s->T[c] || (s->T[d] == s->T[c] && d < c)) rank++;
      s->prio[c] = m - rank;
    }
  } else {
    for (uint32_t c = 0; c < m; c++) s->prio[c] = c + 1;
    for (uint32_t j = m - 1; j >= 1; j--) {
      uint32_t k = pg_bounded(pg_draw(key, PG_D_PERM, j), j + 1);
      uint32_t t = s->prio[j]; s->prio[j] = s->prio[k]; s->prio[k] = t;
    }
  }
  const uint32_t n_be = (uint32_t)(((uint64_t)m * p->be_frac_q16) >> 16);
  for (uint32_t c = 0; c < m; c++) s->cls[c] = (s->prio[c] <= n_be) ? 1 : 0;

  /* CPU utilisation (Q20) per chain, for worst-fit placement; order = util desc, index asc. */
  uint64_t util[PG_MAX_CHAINS];
  uint8_t order[PG_MAX_CHAINS];
  for (uint32_t c = 0; c < m; c++) { util[c] = (chain_cpu[c] << 20) / s->T[c]; order[c] = (uint8_t)c; }
  for (uint32_t j = 1; j < m; j++) {
    uint8_t v = order[j]; int32_t i = (int32_t)j - 1;
    while (i >= 0 && util[order[i]] < util[v]) { order[i + 1] = order[i]; i--; }
    order[i + 1] = v;
  }

  uint32_t n_client_cores;
  if (p->exec_mode == 0) {
    /* One executor per chain, worst-fit onto n_cores client cores; process priority = chain priority. */
    uint64_t load[32];
    for (uint32_t k = 0; k < p->n_cores; k++) load[k] = 0;
    s->n_exec = m;
    for (uint32_t j = 0; j < m; j++) {
      const uint32_t c = order[j];
      uint32_t best = 0;
      for (uint32_t k = 1; k < p->n_cores; k++) if (load[k] < load[best]) best = k;
      load[best] += util[c];
      s->exec_core[c] = (uint8_t)best;
      s->exec_prio[c] = s->prio[c];
      for (uint32_t i = 0; i < s->chain_ncb[c]; i++) s->cb_exec[c * K + i] = (uint16_t)c;
    }
    n_client_cores = p->n_cores;
  } else {
    /* n_exec single-threaded executors, each on its own core ("4xST");
     * chains placed worst-fit; a fraction are split across two executors. */
    uint64_t load[PG_MAX_EXEC];
    const uint32_t X = p->n_exec;
    for (uint32_t x = 0; x < X; x++) load[x] = 0;
    s->n_exec = X;
    for (uint32_t j = 0; j < m; j++) {
      const uint32_t c = order[j];
      uint32_t best = 0;
      for (uint32_t x = 1; x < X; x++) if (load[x] < load[best]) best = x;
      const int split = p->xexec_frac_q16 && K >= 2 && pg_coin(pg_draw(key, PG_D_XEXEC, c), p->xexec_frac_q16);
      if (!split) {
        load[best] += util[c];
        for (uint32_t i = 0; i < K; i++) s->cb_exec[c * K + i] = (uint16_t)best;
      } else {
        uint32_t second = (best == 0) ? 1 : 0;
        for (uint32_t x = 0; x < X; x++) if (x != best && load[x] < load[second]) second = x;
        const uint32_t h = (K + 1) / 2;
        for (uint32_t i = 0; i < K; i++) s->cb_exec[c * K + i] = (uint16_t)(i < h ? best : second);
        load[best] += util[c] / 2;
        load[second] += util[c] - util[c] / 2;
      }
    }
    for (uint32_t x = 0; x < X; x++) { s->exec_core[x] = (uint8_t)x; s->exec_prio[x] = x + 1; }
    n_client_cores = X;
  }
  for (uint32_t x = 0; x < s->n_exec; x++)
    s->exec_wait[x] = (uint8_t)(p->spin_frac_q16 && pg_coin(pg_draw(key, PG_D_SPIN, x), p->spin_frac_q16));

  s->n_accel = p->n_accel;
  for (uint32_t a = 0; a < p->n_accel; a++) {
    s->acc_buckets[a] = (uint8_t)p->buckets[a];
    s->acc_units[a] = (uint8_t)p->units[a];
    s->acc_server_core[a] = (uint8_t)(n_client_cores + a);
    s->acc_eps[a] = p->eps[a];
    s->acc_kappa[a] = p->kappa[a];
  }
  uint32_t nseg = 0;
  for (uint32_t cb = 0; cb < ncb; cb++) nseg += s->cb_nseg[cb];
  s->n_seg = nseg;
}

/* The sizes pg_generate_set produces for set `index` -- {chains, callbacks, segments, executors,
 * accelerators} -- from the same draws (m, and the CPU-only coin of every callback), without
 * generating the rest of the set.  Checked against pg_generate_set by tests/test_generator.py. */
PG_FN void pg_set_sizes(const pg_params* p, uint64_t seed, uint64_t index, uint32_t out[5]) {
  const uint64_t key = pg_key(seed, index);
  const uint32_t K = p->cbs_per_chain;
  const uint32_t m = p->m_lo + pg_bounded(pg_draw(key, PG_D_M, 0), p->m_hi - p->m_lo + 1);
  uint32_t nseg = 0;
  for (uint32_t cb = 0; cb < m * K; cb++)
    nseg += (p->cpu_only_frac_q16 && pg_coin(pg_draw(key, PG_D_CPUONLY, cb), p->cpu_only_frac_q16)) ? 1u : 3u;
  out[0] = m;
  out[1] = m * K;
  out[2] = nseg;
  out[3] = p->exec_mode == 0 ? m : p->n_exec;
  out[4] = p->n_accel;
}

/* Flat CSR raw-batch arrays (same meaning as paam_batch in include/paam.h). */
typedef struct {
  uint32_t *set_chain_off, *set_exec_off, *set_accel_off;      /* [n+1] */
  uint64_t *chain_T, *chain_D; uint32_t *chain_prio; uint8_t *chain_class;
  uint32_t *chain_cb_off;                                       /* [n_chains+1] */
  uint16_t *cb_exec; uint32_t *cb_seg_off;                      /* [n_cbs+1] */
  uint8_t *seg_kind; uint64_t *seg_wcet; uint8_t *seg_accel, *seg_unit;
  uint8_t *exec_core; uint32_t *exec_prio; uint8_t *exec_wait;
  uint8_t *accel_buckets, *accel_units, *accel_server_core;
  uint64_t *accel_eps, *accel_kappa;
  uint32_t *set_bin;
} pg_arrays;

/* Write set `i` of a batch at the given global bases (chain, callback, segment, exec, accel).
 * The caller owns the final sentinel entries of the offset arrays. */
PG_FN void pg_write_set(const pg_set* s, uint32_t i, uint32_t ch0, uint32_t cb0, uint32_t sg0,
                        uint32_t ex0, uint32_t ac0, const pg_arrays* o) {
  o->set_chain_off[i] = ch0;
  o->set_exec_off[i] = ex0;
  o->set_accel_off[i] = ac0;
  if (o->set_bin) o->set_bin[i] = s->bin;
  uint32_t cb = cb0, sg = sg0;
  for (uint32_t c = 0; c < s->m; c++) {
    o->chain_T[ch0 + c] = s->T[c];
    o->chain_D[ch0 + c] = s->D[c];
    o->chain_prio[ch0 + c] = s->prio[c];
    o->chain_class[ch0 + c] = s->cls[c];
    o->chain_cb_off[ch0 + c] = cb;
    for (uint32_t j = 0; j < s->chain_ncb[c]; j++) {
      const uint32_t lc = c * s->K + j;
      o->cb_exec[cb] = s->cb_exec[lc];
      o->cb_seg_off[cb] = sg;
      for (uint32_t k = 0; k < s->cb_nseg[lc]; k++) {
        const int acc = (s->cb_nseg[lc] == 3 && k == 1);
        o->seg_kind[sg] = (uint8_t)acc;
        o->seg_wcet[sg] = s->cb_wcet[lc][k];
        o->seg_accel[sg] = acc ? s->cb_accel[lc] : 0;
        o->seg_unit[sg] = acc ? s->cb_unit[lc] : 0;
        sg++;
      }
      cb++;
    }
  }
  for (uint32_t x = 0; x < s->n_exec; x++) {
    o->exec_core[ex0 + x] = s->exec_core[x];
    o->exec_prio[ex0 + x] = s->exec_prio[x];
    o->exec_wait[ex0 + x] = s->exec_wait[x];
  }
  for (uint32_t a = 0; a < s->n_accel; a++) {
    o->accel_buckets[ac0 + a] = s->acc_buckets[a];
    o->accel_units[ac0 + a] = s->acc_units[a];
    o->accel_server_core[ac0 + a] = s->acc_server_core[a];
    o->accel_eps[ac0 + a] = s->acc_eps[a];
    o->accel_kappa[ac0 + a] = s->acc_kappa[a];
  }
}
