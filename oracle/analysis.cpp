// analysis.cpp -- TEST INFRASTRUCTURE ONLY (see oracle.h).
//
// The PAAM worst-case response-time analysis written out literally from the paper, one function per
// definition, in the paper's notation.  No blocking, no regrouping, no incremental tricks: every
// interfering accelerator segment is visited one by one, every fixed point is iterated exactly as the
// paper states it (start value, recurrence, stop on convergence), u64 nanoseconds throughout.
//
// Citations: P:<line> = /root/reference/PAPER.md, S:<line> = SPEC.md; A<k> = reading k in DESIGN.md
// (same numbering as SURVEY.md §8(c)).
#include "oracle.h"

#include <algorithm>
#include <cassert>
#include <cstring>
#include <thread>
#include <vector>

#include "../gen/paam_gen.h"

#include "model.h"

using namespace oracle_model;

namespace {

// ------------------------------------------------------------------------------------------------
// Lemma 1 / Eq.2: mu(t) = ceil(t / T) + 1.
u64 mu(u64 t, u64 T) { return (t + T - 1) / T + 1; }

// Sums and products saturate at SAT = 2^62, far above every cutoff (< 2^31, A14): a saturated value
// is "above the deadline" either way, so no finite result and no verdict can change.
const u64 SAT = 1ull << 62;
u64 sadd(u64 a, u64 b) { return (a >= SAT || b >= SAT || a + b >= SAT) ? SAT : a + b; }
u64 smul(u64 a, u64 b) {
  if (a == 0 || b == 0) return 0;
  return (a >= SAT / b) ? SAT : a * b;
}

struct ASeg { int chain, sub, cb, accel, unit; u64 Astar; u64 eps; };
struct Sub { int chain; int exec; std::vector<int> cbs; std::vector<int> asegs; };

struct Analysis {
  const System& s;
  std::vector<Sub> subs;
  std::vector<ASeg> asegs;
  std::vector<std::vector<int>> bucket;  // bucket[chain][accel], -1 if the chain does not use it
  std::vector<u64> LPB, H;               // per accelerator segment
  std::vector<int> state;                // per sub-chain: 0 todo, 1 in progress, 2 done
  std::vector<u64> R, Hstar, S, C, B, E, iters;
  u64 mu_literal = 0, mu_regrouped = 0, n_iter = 0;

  explicit Analysis(const System& sys) : s(sys) {}

  u64 cutoff(int chain) const { return std::min(s.chains[chain].D, s.chains[chain].T); }  // A4, A12
  u32 prio(int chain) const { return s.chains[chain].prio; }
  static u64 cpu(const Cb& cb) {  // E_i: WCET of the CPU segments of a callback
    u64 e = 0;
    for (const Seg& g : cb.segs) if (g.kind == 0) e += g.wcet;
    return e;
  }

  void derive() {
    const int m = (int)s.chains.size();
    // Sub-chains: maximal runs of consecutive callbacks on one executor.
    for (int c = 0; c < m; c++) {
      const Chain& ch = s.chains[c];
      for (int j = 0; j < (int)ch.cbs.size(); j++) {
        if (j == 0 || ch.cbs[j].exec != ch.cbs[j - 1].exec) subs.push_back(Sub{c, ch.cbs[j].exec, {}, {}});
        subs.back().cbs.push_back(j);
      }
    }
    // Accelerator segments with A* = A + 2 kappa_eff (kappa_eff = 0 when n = 1, A6).
    for (int si = 0; si < (int)subs.size(); si++) {
      const Chain& ch = s.chains[subs[si].chain];
      for (int j : subs[si].cbs)
        for (const Seg& g : ch.cbs[j].segs)
          if (g.kind == 1) {
            const Accel& a = s.accels[g.accel];
            const u64 keff = a.buckets > 1 ? a.kappa : 0;
            subs[si].asegs.push_back((int)asegs.size());
            asegs.push_back(ASeg{subs[si].chain, si, j, g.accel, g.unit, g.wcet + 2 * keff, a.eps});
          }
    }
    // Buckets (A5): see bucket_map in model.h.
    bucket = bucket_map(s);
    // LP blocking per segment (first max term of Eq.3/Eq.4): the largest A* of a segment of a
    // lower-priority chain on the same accelerator unit and in the same bucket (R2-R3).
    LPB.assign(asegs.size(), 0);
    for (size_t i = 0; i < asegs.size(); i++) {
      const ASeg& si = asegs[i];
      for (const ASeg& q : asegs)
        if (q.accel == si.accel && q.unit == si.unit && prio(q.chain) < prio(si.chain) &&
            bucket[q.chain][q.accel] == bucket[si.chain][si.accel])
          LPB[i] = std::max(LPB[i], q.Astar);
    }
  }

  // hps(s): segments of higher-priority chains on the same accelerator unit.
  bool in_hps(const ASeg& q, const ASeg& si) const {
    return q.accel == si.accel && q.unit == si.unit && prio(q.chain) > prio(si.chain);
  }

  // Lemma 2 / Eq.3: H = A* + LPB + sum_{q in hps} mu(H, T_q) A*_q, starting from the
  // first two terms; UNB once an iterate exceeds the chain's cutoff (A4).
  void lemma2_all() {
    H.assign(asegs.size(), 0);
    for (size_t i = 0; i < asegs.size(); i++) {
      const ASeg& si = asegs[i];
      const u64 first_two = si.Astar + LPB[i];
      u64 h = first_two;
      for (;;) {
        if (h > cutoff(si.chain)) { h = OR_UNB; break; }
        u64 g = first_two;
        std::vector<int> seen_chains;
        for (const ASeg& q : asegs)
          if (in_hps(q, si)) {
            g = sadd(g, smul(mu(h, s.chains[q.chain].T), q.Astar));
            mu_literal++;
            if (std::find(seen_chains.begin(), seen_chains.end(), q.chain) == seen_chains.end()) {
              seen_chains.push_back(q.chain);
              mu_regrouped++;
            }
          }
        n_iter++;
        if (g == h) break;
        h = g;
      }
      H[i] = h;
    }
  }

  // Lemma 3 / Eq.4 (union form A1): C_c(R) = sum_{s in c}(A*_s + LPB_s)
  //   + sum_{q in U_{s in c} hps(s)} mu(R, T_q) A*_q, each interfering segment once.
  u64 lemma3(int sub, u64 R) {
    const Sub& c = subs[sub];
    u64 v = 0;
    for (int i : c.asegs) v += asegs[i].Astar + LPB[i];
    std::vector<int> seen_chains;
    for (size_t q = 0; q < asegs.size(); q++) {
      bool in_union = false;
      for (int i : c.asegs) in_union |= in_hps(asegs[q], asegs[i]);
      if (in_union) {
        v = sadd(v, smul(mu(R, s.chains[asegs[q].chain].T), asegs[q].Astar));
        mu_literal++;
        if (std::find(seen_chains.begin(), seen_chains.end(), asegs[q].chain) == seen_chains.end()) {
          seen_chains.push_back(asegs[q].chain);
          mu_regrouped++;
        }
      }
    }
    return v;
  }

  // Per-segment bound summed over the sub-chain: UNB if any term is UNB.
  u64 per_segment_sum(int sub) const {
    u64 v = 0;
    for (int i : subs[sub].asegs) {
      if (H[i] == OR_UNB) return OR_UNB;
      v += H[i];
    }
    return v;
  }
  u64 eps_sum(int sub) const {  // delta_c * eps, per accelerator (A11)
    u64 v = 0;
    for (int i : subs[sub].asegs) v += asegs[i].eps;
    return v;
  }
  // Eq.1 with the double bound: H*_c(R) = min(S_c, C_c(R)) + sum eps; min(UNB, x) = x.
  u64 hstar(int sub, u64 R) {
    const u64 Sc = per_segment_sum(sub);
    const u64 Cc = lemma3(sub, R);
    return sadd(std::min(Sc, Cc), eps_sum(sub));  // OR_UNB == UINT64_MAX > SAT: min() absorbs it
  }
  u64 exec_sum(int sub) const {  // calligraphic E_c = sum of E_i over the sub-chain
    u64 v = 0;
    for (int j : subs[sub].cbs) v += cpu(s.chains[subs[sub].chain].cbs[j]);
    return v;
  }
  // hp(c): sub-chains on the same executor with higher chain priority.
  bool in_hp(int h, int c) const { return h != c && subs[h].exec == subs[c].exec && prio(subs[h].chain) > prio(subs[c].chain); }
  // hpp(c): sub-chains of executors on the same core with higher process priority.
  bool in_hpp(int h, int c) const {
    const Exec& xh = s.execs[subs[h].exec];
    const Exec& xc = s.execs[subs[c].exec];
    return subs[h].exec != subs[c].exec && xh.core == xc.core && xh.prio > xc.prio;
  }
  // lp(c): sub-chains on the same executor with lower chain priority.
  bool in_lp(int l, int c) const { return l != c && subs[l].exec == subs[c].exec && prio(subs[l].chain) < prio(subs[c].chain); }

  // B_c = max_{Gamma_l in lp(c)} max_{tau_j in Gamma_l} E_j, or with
  // PAAM_FLAG_BLOCKING_SOUND the LP callback's accelerator handling as well (A10).
  // Returns OR_UNSCHED when the sound variant needs an unbounded Lemma-2 value.
  u64 blocking(int c) const {
    u64 B = 0;
    for (int l = 0; l < (int)subs.size(); l++) {
      if (!in_lp(l, c)) continue;
      const Chain& ch = s.chains[subs[l].chain];
      for (int j : subs[l].cbs) {
        u64 v = cpu(ch.cbs[j]);
        if (s.flags & OR_FLAG_BLOCKING_SOUND) {
          for (int i : subs[l].asegs)
            if (asegs[i].cb == j) {
              if (H[i] == OR_UNB) return OR_UNSCHED;
              v += H[i] + asegs[i].eps;
            }
        }
        B = std::max(B, v);
      }
    }
    return B;
  }

  // Theorem 1 / Eq.5, memoised recursion over the (acyclic) dependencies on hp and
  // hpp sub-chains; H*_h is taken at h's own converged R_h (A7, A8).
  void solve(int c) {
    if (state[c] == 2) return;
    assert(state[c] == 0);  // hp / hpp dependencies are acyclic
    state[c] = 1;
    bool poisoned = false;
    for (int h = 0; h < (int)subs.size(); h++) {
      const bool spin = s.execs[subs[h].exec].wait == 1;
      if (in_hp(h, c) || (in_hpp(h, c) && spin)) {
        solve(h);
        if (R[h] == OR_UNSCHED) poisoned = true;  // A8
      }
    }
    const u64 cut = cutoff(subs[c].chain);
    B[c] = blocking(c);
    E[c] = exec_sum(c);
    S[c] = per_segment_sum(c);
    u64 r = OR_UNSCHED;
    if (!poisoned && B[c] != OR_UNSCHED) {
      // "The recurrence starts with the first three terms".
      u64 Rk = sadd(sadd(B[c], E[c]), hstar(c, 0));
      for (;;) {
        iters[c]++;
        n_iter++;
        if (Rk > cut) { Rk = OR_UNSCHED; break; }
        u64 F = sadd(sadd(B[c], E[c]), hstar(c, Rk));
        for (int h = 0; h < (int)subs.size(); h++) {
          const u64 Th = s.chains[subs[h].chain].T;
          if (in_hp(h, c)) {
            F = sadd(F, smul(mu(Rk, Th), sadd(exec_sum(h), Hstar[h])));
            mu_literal++; mu_regrouped++;
          } else if (in_hpp(h, c)) {
            const bool spin = s.execs[subs[h].exec].wait == 1;
            const u64 sp = spin ? Hstar[h] : eps_sum(h);  // spin(Gamma_h)
            F = sadd(F, smul(mu(Rk, Th), sadd(exec_sum(h), sp)));
            mu_literal++; mu_regrouped++;
          }
        }
        if (F == Rk) break;
        Rk = F;
      }
      r = Rk;
    }
    R[c] = r;
    if (r != OR_UNSCHED) {
      const u64 ml = mu_literal, mr = mu_regrouped;  // not counted: the last iterate already did it
      C[c] = lemma3(c, r);
      Hstar[c] = hstar(c, r);
      mu_literal = ml; mu_regrouped = mr;
    } else {
      C[c] = OR_UNB;
      Hstar[c] = OR_UNB;
    }
    state[c] = 2;
  }

  void run() {
    derive();
    lemma2_all();
    const size_t n = subs.size();
    state.assign(n, 0);
    R.assign(n, 0); Hstar.assign(n, 0); S.assign(n, 0); C.assign(n, 0); B.assign(n, 0); E.assign(n, 0);
    iters.assign(n, 0);
    for (int c = 0; c < (int)n; c++) solve(c);
  }

  // End-to-end (A9): R* = sum of sub-chain R_c + comm per executor crossing.
  u64 end_to_end(int chain) const {
    u64 v = 0;
    int k = 0;
    for (size_t c = 0; c < subs.size(); c++)
      if (subs[c].chain == chain) {
        if (R[c] == OR_UNSCHED) return OR_UNSCHED;
        v += R[c];
        k++;
      }
    return v + s.comm * (u64)(k - 1);
  }
};

// Analyse one set: status, per-chain R*, verdict (every critical chain meets D).
struct SetResult { int status; std::vector<u64> wcrt; int sched; u64 mu_literal, mu_regrouped, iters; };

SetResult analyze_system(const System& s) {
  SetResult out;
  out.status = validate(s);
  out.wcrt.assign(s.chains.size(), OR_UNSCHED);
  out.sched = 0;
  out.mu_literal = out.mu_regrouped = out.iters = 0;
  if (out.status != OR_OK) return out;
  System sw = s;
  if (s.flags & OR_FLAG_WFD_UNITS) apply_wfd(sw);  // units by WFD
  Analysis an(sw);
  an.run();
  int sched = 1;
  for (int c = 0; c < (int)s.chains.size(); c++) {
    out.wcrt[c] = an.end_to_end(c);
    if (s.chains[c].cls == 0 && (out.wcrt[c] == OR_UNSCHED || out.wcrt[c] > s.chains[c].D)) sched = 0;
  }
  out.sched = sched;
  out.mu_literal = an.mu_literal;
  out.mu_regrouped = an.mu_regrouped;
  out.iters = an.n_iter;
  return out;
}

template <class F>
void parallel_for(uint32_t n, int nthreads, F f) {
  if (nthreads <= 1 || n < 64) {
    for (uint32_t i = 0; i < n; i++) f(i, 0);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; t++) {
    th.emplace_back([=, &f]() {
      const uint64_t lo = (uint64_t)n * t / nthreads, hi = (uint64_t)n * (t + 1) / nthreads;
      for (uint64_t i = lo; i < hi; i++) f((uint32_t)i, t);
    });
  }
  for (auto& x : th) x.join();
}

}  // namespace

extern "C" int32_t oracle_analyze_batch(const or_batch* b, uint64_t* out_wcrt, uint8_t* out_sched,
                                        int32_t* out_status, int64_t* out_bins, int nthreads) {
  if (!b) return -1;
  const uint32_t n = b->n_sets;
  std::vector<int64_t> bins_local((size_t)(nthreads > 0 ? nthreads : 1) * b->n_bins * 2, 0);
  parallel_for(n, nthreads, [&](uint32_t i, int t) {
    System s = read_set(b, i);
    // a utilisation bin outside [0, n_bins) is a size-range error of the set (reading V):
    // the set is rejected and counted in no bin
    const bool bad_bin = b->set_bin && b->n_bins && b->set_bin[i] >= b->n_bins;
    SetResult r = analyze_system(s);
    if (bad_bin) {
      r.status = OR_ERANGE;
      r.sched = 0;
      r.wcrt.assign(s.chains.size(), OR_UNSCHED);
    }
    if (out_wcrt)
      for (size_t c = 0; c < r.wcrt.size(); c++) out_wcrt[b->set_chain_off[i] + c] = r.wcrt[c];
    if (out_sched) out_sched[i] = (uint8_t)r.sched;
    if (out_status) out_status[i] = r.status;
    if (b->set_bin && b->n_bins && !bad_bin) {
      const uint32_t bin = b->set_bin[i];
      bins_local[((size_t)t * b->n_bins + bin) * 2] += 1;
      bins_local[((size_t)t * b->n_bins + bin) * 2 + 1] += r.sched;
    }
  });
  if (out_bins && b->set_bin)
    for (size_t t = 0; t < bins_local.size() / (2 * (size_t)(b->n_bins ? b->n_bins : 1)); t++)
      for (uint32_t k = 0; k < 2 * b->n_bins; k++) out_bins[k] += bins_local[t * 2 * b->n_bins + k];
  return 0;
}

extern "C" int32_t oracle_analyze_detail(const or_batch* b, uint32_t set_index, or_detail* out) {
  if (!b || !out || set_index >= b->n_sets) return -1;
  std::memset(out, 0, sizeof(*out));
  System s = read_set(b, set_index);
  out->status = validate(s);
  if (out->status != OR_OK) return 0;
  if (s.flags & OR_FLAG_WFD_UNITS) apply_wfd(s);
  Analysis an(s);
  an.run();
  if (an.subs.size() > OR_DMAX || an.asegs.size() > OR_DMAX) return -2;
  out->n_sub = (uint32_t)an.subs.size();
  out->n_aseg = (uint32_t)an.asegs.size();
  for (size_t c = 0; c < an.subs.size(); c++) {
    out->sub_chain[c] = an.subs[c].chain;
    out->sub_exec[c] = an.subs[c].exec;
    out->sub_B[c] = an.B[c]; out->sub_E[c] = an.E[c]; out->sub_S[c] = an.S[c]; out->sub_C[c] = an.C[c];
    out->sub_Hstar[c] = an.Hstar[c]; out->sub_R[c] = an.R[c]; out->sub_iters[c] = an.iters[c];
  }
  for (size_t i = 0; i < an.asegs.size(); i++) {
    out->aseg_sub[i] = an.asegs[i].sub;
    out->aseg_bucket[i] = an.bucket[an.asegs[i].chain][an.asegs[i].accel];
    out->aseg_Astar[i] = an.asegs[i].Astar;
    out->aseg_LPB[i] = an.LPB[i];
    out->aseg_H[i] = an.H[i];
  }
  out->mu_literal = an.mu_literal;
  out->mu_regrouped = an.mu_regrouped;
  out->iterations = an.n_iter;
  return 0;
}

extern "C" int32_t oracle_generate_analyze(const void* params, uint64_t seed, uint64_t first, uint32_t n,
                                           uint64_t comm_cost, uint32_t flags, uint64_t* out_wcrt,
                                           uint32_t wcrt_stride, uint8_t* out_sched, int64_t* out_bins,
                                           uint64_t* counters, int nthreads) {
  const pg_params* p = (const pg_params*)params;
  if (!p || pg_check_params(p)) return -1;
  const int T = nthreads > 0 ? nthreads : 1;
  std::vector<int64_t> bins_local((size_t)T * (p->n_bins ? p->n_bins : 1) * 2, 0);
  std::vector<uint64_t> cnt((size_t)T * 3, 0);
  parallel_for(n, T, [&](uint32_t i, int t) {
    pg_set g;
    pg_generate_set(p, seed, first + i, &g);
    System s = from_generated(g, comm_cost, flags);
    SetResult r = analyze_system(s);
    if (out_wcrt)
      for (size_t c = 0; c < r.wcrt.size() && c < wcrt_stride; c++) out_wcrt[(uint64_t)i * wcrt_stride + c] = r.wcrt[c];
    if (out_sched) out_sched[i] = (uint8_t)r.sched;
    if (p->n_bins) {
      bins_local[((size_t)t * p->n_bins + g.bin) * 2] += 1;
      bins_local[((size_t)t * p->n_bins + g.bin) * 2 + 1] += r.sched;
    }
    cnt[t * 3 + 0] += r.mu_literal;
    cnt[t * 3 + 1] += r.mu_regrouped;
    cnt[t * 3 + 2] += r.iters;
  });
  if (out_bins && p->n_bins)
    for (int t = 0; t < T; t++)
      for (uint32_t k = 0; k < 2 * p->n_bins; k++) out_bins[k] += bins_local[(size_t)t * 2 * p->n_bins + k];
  if (counters) {
    counters[0] = counters[1] = counters[2] = 0;
    for (int t = 0; t < T; t++)
      for (int k = 0; k < 3; k++) counters[k] += cnt[t * 3 + k];
  }
  return 0;
}

// Lemma 1 / Eq.2 exposed for the worked-example pins.
extern "C" uint64_t oracle_mu(uint64_t t, uint64_t T) { return mu(t, T); }
