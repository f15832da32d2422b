// model.h -- TEST INFRASTRUCTURE ONLY (see oracle.h).  The oracle's own system-model types
// (P:101-142), readers from the flat batch / the shared generator, validation and the bucket map.
#pragma once
#include <algorithm>
#include <cstdint>
#include <vector>

#include "../gen/paam_gen.h"
#include "oracle.h"

typedef uint64_t u64;
typedef uint32_t u32;

namespace oracle_model {

// ------------------------------------------------------------------------------------------------
// System model: callbacks are alternating CPU / accelerator segments, chains are
// sequences of callbacks with period, deadline and a unique priority, executors are single-threaded
// processes on a core with a process priority, accelerators are PAAM servers with n buckets.
struct Seg { int kind; u64 wcet; int accel; int unit; };          // kind 0 CPU, 1 ACCEL
struct Cb { int exec; std::vector<Seg> segs; };
struct Chain { u64 T, D; u32 prio; int cls; std::vector<Cb> cbs; };  // cls 0 CRITICAL, 1 BE
struct Exec { int core; u32 prio; int wait; };                      // wait 0 SUSPEND, 1 SPIN
struct Accel { int buckets, units, server_core; u64 eps, kappa; };
struct System { std::vector<Chain> chains; std::vector<Exec> execs; std::vector<Accel> accels;
                u64 comm; u32 flags; };

// Every input time must be < 2^48 ns (about 78 hours; A14 as revised in round 2: the boundary is u64,
// S:26-31).  Below 2^48 every sum of the analysis (at most 192 terms) stays below 2^56 and every product
// saturates at 2^62 (analysis.cpp), so the arithmetic is exact up to the saturation, which lies far
// above every cutoff.
const u64 LIMT = 1ull << 48;

inline System read_set(const or_batch* b, u32 i) {
  System s;
  s.comm = b->comm_cost;
  s.flags = b->flags;
  for (u32 g = b->set_chain_off[i]; g < b->set_chain_off[i + 1]; g++) {
    Chain c;
    c.T = b->chain_T[g]; c.D = b->chain_D[g]; c.prio = b->chain_prio[g]; c.cls = b->chain_class[g];
    for (u32 j = b->chain_cb_off[g]; j < b->chain_cb_off[g + 1]; j++) {
      Cb cb;
      cb.exec = b->cb_exec[j];
      for (u32 k = b->cb_seg_off[j]; k < b->cb_seg_off[j + 1]; k++)
        cb.segs.push_back(Seg{b->seg_kind[k], b->seg_wcet[k], b->seg_accel[k], b->seg_unit[k]});
      c.cbs.push_back(cb);
    }
    s.chains.push_back(c);
  }
  for (u32 x = b->set_exec_off[i]; x < b->set_exec_off[i + 1]; x++)
    s.execs.push_back(Exec{b->exec_core[x], b->exec_prio[x], b->exec_wait[x]});
  for (u32 a = b->set_accel_off[i]; a < b->set_accel_off[i + 1]; a++)
    s.accels.push_back(Accel{b->accel_buckets[a], b->accel_units[a], b->accel_server_core[a],
                             b->accel_eps[a], b->accel_kappa[a]});
  return s;
}

inline System from_generated(const pg_set& g, u64 comm, u32 flags) {
  System s;
  s.comm = comm;
  s.flags = flags;
  for (u32 c = 0; c < g.m; c++) {
    Chain ch;
    ch.T = g.T[c]; ch.D = g.D[c]; ch.prio = g.prio[c]; ch.cls = g.cls[c];
    for (u32 j = 0; j < g.chain_ncb[c]; j++) {
      const u32 lc = c * g.K + j;
      Cb cb;
      cb.exec = g.cb_exec[lc];
      for (u32 k = 0; k < g.cb_nseg[lc]; k++) {
        const bool acc = (g.cb_nseg[lc] == 3 && k == 1);
        cb.segs.push_back(Seg{acc ? 1 : 0, g.cb_wcet[lc][k], acc ? g.cb_accel[lc] : 0, acc ? g.cb_unit[lc] : 0});
      }
      ch.cbs.push_back(cb);
    }
    s.chains.push_back(ch);
  }
  for (u32 x = 0; x < g.n_exec; x++) s.execs.push_back(Exec{g.exec_core[x], g.exec_prio[x], g.exec_wait[x]});
  for (u32 a = 0; a < g.n_accel; a++)
    s.accels.push_back(Accel{g.acc_buckets[a], g.acc_units[a], g.acc_server_core[a], g.acc_eps[a], g.acc_kappa[a]});
  return s;
}

// ------------------------------------------------------------------------------------------------
// Validation, rules checked in this order, first failure reported.
inline int validate(const System& s) {
  // 1. ERANGE: size caps and the time range (< 2^48 ns, A14).
  size_t n_cb = 0, n_seg = 0, n_aseg = 0;
  for (const Chain& c : s.chains) {
    n_cb += c.cbs.size();
    for (const Cb& cb : c.cbs) {
      n_seg += cb.segs.size();
      for (const Seg& g : cb.segs) n_aseg += (g.kind == 1);
    }
  }
  if (s.chains.size() > 32 || n_cb > 64 || n_seg > 192 || n_aseg > 64 || s.execs.size() > 32 ||
      s.accels.size() > 4)
    return OR_ERANGE;
  int units_total = 0;
  for (const Accel& a : s.accels) {
    if (a.buckets < 1 || a.buckets > 32 || a.units < 1 || a.units > 8) return OR_ERANGE;
    if (a.eps >= LIMT || a.kappa >= LIMT) return OR_ERANGE;
    units_total += a.units;
  }
  if (units_total > 8) return OR_ERANGE;
  for (const Chain& c : s.chains) {
    if (c.T == 0 || c.T >= LIMT || c.D >= LIMT) return OR_ERANGE;
    for (const Cb& cb : c.cbs)
      for (const Seg& g : cb.segs)
        if (g.wcet >= LIMT) return OR_ERANGE;
  }
  // 2. EDANGLING: empty chain / callback, executor or unit index out of range.
  for (const Chain& c : s.chains) {
    if (c.cbs.empty()) return OR_EDANGLING;
    for (const Cb& cb : c.cbs) {
      if (cb.segs.empty()) return OR_EDANGLING;
      if (cb.exec < 0 || (size_t)cb.exec >= s.execs.size()) return OR_EDANGLING;
      for (const Seg& g : cb.segs)
        if (g.kind == 1 && (size_t)g.accel < s.accels.size() && g.unit >= s.accels[g.accel].units)
          return OR_EDANGLING;
    }
  }
  // 3. EACCEL: accelerator segment on an undeclared accelerator.
  for (const Chain& c : s.chains)
    for (const Cb& cb : c.cbs)
      for (const Seg& g : cb.segs)
        if (g.kind == 1 && (size_t)g.accel >= s.accels.size()) return OR_EACCEL;
  // 4. ESHAPE: enum values, zero WCETs, alternation, contiguous executor visits.
  for (const Exec& x : s.execs)
    if (x.wait != 0 && x.wait != 1) return OR_ESHAPE;
  for (const Chain& c : s.chains) {
    if (c.cls != 0 && c.cls != 1) return OR_ESHAPE;
    for (const Cb& cb : c.cbs) {
      for (size_t k = 0; k < cb.segs.size(); k++) {
        if (cb.segs[k].kind != 0 && cb.segs[k].kind != 1) return OR_ESHAPE;
        if (cb.segs[k].wcet == 0) return OR_ESHAPE;
        if (k > 0 && cb.segs[k].kind == cb.segs[k - 1].kind) return OR_ESHAPE;
      }
    }
    for (size_t j = 1; j < c.cbs.size(); j++) {
      if (c.cbs[j].exec == c.cbs[j - 1].exec) continue;
      for (size_t i = 0; i + 1 < j; i++)
        if (c.cbs[i].exec == c.cbs[j].exec) return OR_ESHAPE;  // revisit after leaving (A13)
    }
  }
  // 4b. ERANGE: number of sub-chains.
  size_t n_sub = 0;
  for (const Chain& c : s.chains)
    for (size_t j = 0; j < c.cbs.size(); j++) n_sub += (j == 0 || c.cbs[j].exec != c.cbs[j - 1].exec);
  if (n_sub > 32) return OR_ERANGE;
  // 5. EDUPPRIO: unique chain priorities; unique process priority per core.
  for (size_t a = 0; a < s.chains.size(); a++)
    for (size_t b = a + 1; b < s.chains.size(); b++)
      if (s.chains[a].prio == s.chains[b].prio) return OR_EDUPPRIO;
  for (size_t a = 0; a < s.execs.size(); a++)
    for (size_t b = a + 1; b < s.execs.size(); b++)
      if (s.execs[a].core == s.execs[b].core && s.execs[a].prio == s.execs[b].prio) return OR_EDUPPRIO;
  // 6. EDEADLINE: constrained deadlines for CRITICAL chains, D >= 1 for all.
  for (const Chain& c : s.chains) {
    if (c.D == 0) return OR_EDEADLINE;
    if (c.cls == 0 && c.D > c.T) return OR_EDEADLINE;
  }
  // 7. ECORE: a server core never hosts a client executor (R1).
  for (const Accel& a : s.accels)
    for (const Exec& x : s.execs)
      if (x.core == a.server_core) return OR_ECORE;
  return OR_OK;
}

// Bucket of every (chain, accelerator) ("divides chain priorities into n evenly sized groups;
// the highest priority chains are assigned the highest priority buckets"; A5): the m_a
// chains that use accelerator a, ranked by priority, in groups of ceil(m_a / n); -1 if unused.
inline std::vector<std::vector<int>> bucket_map(const System& s) {
  const int m = (int)s.chains.size();
  std::vector<std::vector<int>> bucket(m, std::vector<int>(s.accels.size(), -1));
  for (int a = 0; a < (int)s.accels.size(); a++) {
    std::vector<int> users;
    for (int c = 0; c < m; c++) {
      bool uses = false;
      for (const Cb& cb : s.chains[c].cbs)
        for (const Seg& g : cb.segs) uses |= (g.kind == 1 && g.accel == a);
      if (uses) users.push_back(c);
    }
    std::sort(users.begin(), users.end(), [&](int x, int y) { return s.chains[x].prio > s.chains[y].prio; });
    const int ma = (int)users.size(), n = s.accels[a].buckets;
    const int g = (ma + n - 1) / n;
    for (int r = 0; r < ma; r++) bucket[users[r]][a] = n - 1 - r / g;
  }
  return bucket;
}

// Worst-Fit-Decreasing assignment of accelerator segments to units ("bin-packing heuristics
// such as WFD"): per accelerator, items = (callback, accelerator) with the callback's
// summed WCET on it (all its segments go to one unit), utilisation u = (A << 24) / T (integer, exact
// ordering key), sorted by u descending (ties: callback order), each placed on the unit with the least
// summed u (ties: lowest unit index).  Overrides the input units (flag PAAM_FLAG_WFD_UNITS).
inline void apply_wfd(System& s) {
  for (int a = 0; a < (int)s.accels.size(); a++) {
    struct Item { int c, j; u64 u; };
    std::vector<Item> items;
    for (int c = 0; c < (int)s.chains.size(); c++)
      for (int j = 0; j < (int)s.chains[c].cbs.size(); j++) {
        u64 A = 0;
        for (const Seg& g : s.chains[c].cbs[j].segs) if (g.kind == 1 && g.accel == a) A += g.wcet;
        if (A) items.push_back(Item{c, j, (A << 24) / s.chains[c].T});
      }
    std::stable_sort(items.begin(), items.end(), [](const Item& x, const Item& y) { return x.u > y.u; });
    std::vector<u64> load(s.accels[a].units, 0);
    for (const Item& it : items) {
      int best = 0;
      for (int k = 1; k < (int)load.size(); k++) if (load[k] < load[best]) best = k;
      load[best] += it.u;
      for (Seg& g : s.chains[it.c].cbs[it.j].segs) if (g.kind == 1 && g.accel == a) g.unit = best;
    }
  }
}

}  // namespace oracle_model
