/* paam_gen_host.c -- host build of the shared seeded input generator (gen/paam_gen.h).
 * Input generation only: used by tests and bench.py to materialise raw batches in host memory
 * (for the oracle and for the end-to-end path from host buffers). */
#include <stdlib.h>
#include "paam_gen.h"

/* Totals of sets [first, first+n): out[0..4] = chains, callbacks, segments, executors, accelerators. */
int pg_batch_totals(const pg_params* p, uint64_t seed, uint64_t first, uint32_t n, uint64_t* out) {
  if (!p || !out || pg_check_params(p)) return -1;
  pg_set* s = (pg_set*)malloc(sizeof(pg_set));
  if (!s) return -2;
  for (int k = 0; k < 5; k++) out[k] = 0;
  for (uint32_t i = 0; i < n; i++) {
    pg_generate_set(p, seed, first + i, s);
    out[0] += s->m; out[1] += s->n_cb; out[2] += s->n_seg; out[3] += s->n_exec; out[4] += s->n_accel;
  }
  free(s);
  return 0;
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
