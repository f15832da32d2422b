/* paam_gen_host.c -- host build of the shared seeded input generator (gen/paam_gen.h).
 * Input generation only: used by tests and bench.py to materialise raw batches in host memory
 * (for the oracle and for the end-to-end path from host buffers). */
#include <stdlib.h>
#include "paam_gen.h"

/* Totals of sets [first, first+n): out[0..4] = chains, callbacks, segments, executors, accelerators. */
int pg_batch_totals(const pg_params* p, uint64_t seed, uint64_t first, uint32_t n, uint64_t* out) {
  if (!p || !out || pg_check_params(p)) return -1;
  for (int k = 0; k < 5; k++) out[k] = 0;
  for (uint32_t i = 0; i < n; i++) {
    uint32_t z[5];
    pg_set_sizes(p, seed, first + i, z);
    for (int k = 0; k < 5; k++) out[k] += z[k];
  }
  return 0;
}

/* Number of sets in [first, first+n) whose pg_set_sizes differ from pg_generate_set's (tests: 0). */
int64_t pg_sizes_mismatch(const pg_params* p, uint64_t seed, uint64_t first, uint32_t n) {
  if (!p || pg_check_params(p)) return -1;
  pg_set* s = (pg_set*)malloc(sizeof(pg_set));
  if (!s) return -2;
  int64_t bad = 0;
  for (uint32_t i = 0; i < n; i++) {
    uint32_t z[5];
    pg_generate_set(p, seed, first + i, s);
    pg_set_sizes(p, seed, first + i, z);
    bad += (z[0] != s->m || z[1] != s->n_cb || z[2] != s->n_seg || z[3] != s->n_exec || z[4] != s->n_accel);
  }
  free(s);
  return bad;
}

/* Fill caller-allocated arrays (sizes from pg_batch_totals), including the offset sentinels. */
int pg_batch_fill(const pg_params* p, uint64_t seed, uint64_t first, uint32_t n, const pg_arrays* o) {
  if (!p || !o || pg_check_params(p)) return -1;
  pg_set* s = (pg_set*)malloc(sizeof(pg_set));
  if (!s) return -2;
  uint32_t ch = 0, cb = 0, sg = 0, ex = 0, ac = 0;
  for (uint32_t i = 0; i < n; i++) {
    pg_generate_set(p, seed, first + i, s);
    pg_write_set(s, i, ch, cb, sg, ex, ac, o);
    ch += s->m; cb += s->n_cb; sg += s->n_seg; ex += s->n_exec; ac += s->n_accel;
  }
  o->set_chain_off[n] = ch;
  o->set_exec_off[n] = ex;
  o->set_accel_off[n] = ac;
  o->chain_cb_off[ch] = cb;
  o->cb_seg_off[cb] = sg;
  free(s);
  return 0;
}

uint32_t pg_params_size(void) { return (uint32_t)sizeof(pg_params); }
uint32_t pg_arrays_size(void) { return (uint32_t)sizeof(pg_arrays); }
