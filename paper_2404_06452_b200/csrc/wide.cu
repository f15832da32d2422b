// wide.cu -- the exact u64 path: sets that have a time in [2^31 - 1, 2^48) ns ("wide" sets).
//
// The u32 kernels (fused.cu, pack.cu + analyze.cu) are exact for times below 2^31 - 1 ns (A14).  A set
// with a larger time is handed over to this kernel instead of being rejected: they append its index to
// a list, and wide_kernel -- one thread per listed set, state in local memory, u64 arithmetic saturating
// at 2^62 -- validates it in the documented order and runs the same analysis: sub-chains,
// A* = A + 2 kappa_eff (A6), rank-based buckets (A5), LP blocking, Lemma 2 per
// segment (Eq.3), Lemma 3 in union form (Eq.4, A1), H* = min(S, C) + eps
// (Eq.1), Eq.5 per sub-chain in dependency order (A7, A8), end to end and the
// verdict.  Times up to 2^48 keep every sum below 2^56; products saturate.
// It is a slow path by design (rare sets, division-based mu); nothing here is on the timed path.
#include "common.cuh"

namespace paam {

namespace {

constexpr uint64_t W_LIM = 1ull << 48;  // validation: every time < 2^48 ns
constexpr uint64_t W_SAT = 1ull << 62;  // saturation (UNB / UNSCHED inside the kernel)
constexpr uint64_t UNS = PAAM_UNSCHED;

__device__ __forceinline__ uint64_t wadd(uint64_t a, uint64_t b) {  // a, b <= W_SAT
  const uint64_t c = a + b;
  return c >= W_SAT ? W_SAT : c;
}
__device__ __forceinline__ uint64_t wmul(uint64_t a, uint64_t b) {
  return (__umul64hi(a, b) != 0 || a * b >= W_SAT) ? W_SAT : a * b;
}
// mu(t, T) = ceil(t / T) + 1 (Lemma 1, Eq.2), exact 64-bit division
__device__ __forceinline__ uint64_t wmu(uint64_t t, uint64_t T) { return t == 0 ? 1 : (t - 1) / T + 2; }

struct WSet {
  // chains (set-local index)
  uint64_t T[MAXC], D[MAXC];
  uint32_t prio[MAXC], rank[MAXC], cb0[MAXC], ncb[MAXC];
  uint8_t cls[MAXC];
  // callbacks
  uint64_t E[MAXCB];
  uint32_t seg0[MAXCB], nseg[MAXCB];
  uint8_t exec[MAXCB], chain[MAXCB];
  // accelerator segments, in callback order
  uint64_t A[MAXA], Astar[MAXA], LPB[MAXA], H[MAXA];
  uint8_t acc[MAXA], unit[MAXA], qcb[MAXA], qsub[MAXA];
  // executors, accelerators
  uint32_t xprio[MAXX];
  uint8_t xcore[MAXX], xwait[MAXX];
  uint32_t nb[4], nu[4], ub[4], server[4];
  uint64_t eps[4], keff[4];
  // W[rank][unit] (regrouped Lemma-2 / Lemma-3 sums), buckets per (chain, accelerator)
  uint64_t W[MAXC][MAXU];
  int8_t bucket[MAXC][4];
  // sub-chains, in callback order
  uint32_t scb0[MAXS], sncb[MAXS], sq0[MAXS], snq[MAXS], sumask[MAXS], shp[MAXS], shpp[MAXS], slp[MAXS];
  uint8_t schain[MAXS], sexec[MAXS];
  uint64_t sE[MAXS], smaxE[MAXS], seps[MAXS], sbase3[MAXS], sS[MAXS], sR[MAXS], sHs[MAXS];
};

// Validation in the order of include/paam.h; returns PAAM_SET_* and fills the set.  C32: b
// carries a compact batch (common.cuh ld_time).
template <bool C32>
__device__ int w_load(const paam_batch& b, uint32_t set, WSet& s, uint32_t& nch, uint32_t& ncb, uint32_t& nq,
                      uint32_t& nex, uint32_t& nac, uint32_t& nsub) {
  const uint32_t c0 = b.set_chain_off[set], c1 = b.set_chain_off[set + 1];
  const uint32_t x0 = b.set_exec_off[set], x1 = b.set_exec_off[set + 1];
  const uint32_t a0 = b.set_accel_off[set], a1 = b.set_accel_off[set + 1];
  nch = c1 - c0; nex = x1 - x0; nac = a1 - a0;
  const uint32_t cbA = b.chain_cb_off[c0], cbB = b.chain_cb_off[c1];
  const uint32_t sgA = b.cb_seg_off[cbA], sgB = b.cb_seg_off[cbB];
  ncb = cbB - cbA;
  const uint32_t nseg = sgB - sgA;
  nq = 0; nsub = 0;
  if (nch > MAXC || ncb > MAXCB || nseg > 192 || nex > MAXX || nac > 4) return PAAM_SET_ERANGE;
  if (b.set_bin && b.set_bin[set] >= b.n_bins) return PAAM_SET_ERANGE;
  // callbacks whose segment range leaves the set's (malformed CSR): a dangling reference, reported first
  for (uint32_t j = 0; j < ncb; j++) {
    const uint32_t so = b.cb_seg_off[cbA + j], se = b.cb_seg_off[cbA + j + 1];
    if (so < sgA || se < so || se > sgB) return PAAM_SET_EDANGLING;
  }
  bool erange = false, edang = false, eaccel = false, eshape = false;
  uint32_t units_total = 0;
  for (uint32_t a = 0; a < nac; a++) {
    const uint32_t n = b.accel_buckets[a0 + a], u = b.accel_units[a0 + a];
    const uint64_t e = ld_time<C32>(b.accel_eps, a0 + a), k = ld_time<C32>(b.accel_kappa, a0 + a);
    erange |= (n < 1 || n > 32 || u < 1 || u > 8 || e >= W_LIM || k >= W_LIM);
    s.nb[a] = n; s.nu[a] = u; s.ub[a] = units_total; s.server[a] = b.accel_server_core[a0 + a];
    s.eps[a] = e; s.keff[a] = n > 1 ? k : 0;  // A6
    units_total += u;
  }
  erange |= units_total > MAXU;
  for (uint32_t c = 0; c < nch; c++) {
    s.T[c] = ld_time<C32>(b.chain_T, c0 + c); s.D[c] = ld_time<C32>(b.chain_D, c0 + c); s.prio[c] = b.chain_prio[c0 + c];
    s.cls[c] = b.chain_class[c0 + c];
    erange |= (s.T[c] == 0 || s.T[c] >= W_LIM || s.D[c] >= W_LIM);
    const uint32_t o = b.chain_cb_off[c0 + c] - cbA, e = b.chain_cb_off[c0 + c + 1] - cbA;
    edang |= (e <= o) || (e > ncb);
    s.cb0[c] = o; s.ncb[c] = e > o ? e - o : 0;
    eshape |= s.cls[c] > 1;
  }
  for (uint32_t x = 0; x < nex; x++) {
    s.xcore[x] = b.exec_core[x0 + x]; s.xprio[x] = b.exec_prio[x0 + x]; s.xwait[x] = b.exec_wait[x0 + x];
    eshape |= s.xwait[x] > 1;
  }
  for (uint32_t j = 0; j < ncb; j++) {
    const uint32_t so = b.cb_seg_off[cbA + j], se = b.cb_seg_off[cbA + j + 1];
    const uint32_t x = ld_cb_exec<C32>(b, cbA + j);
    edang |= (se == so) || (x >= nex);
    s.exec[j] = (uint8_t)min(x, 255u);
    s.seg0[j] = nq; s.nseg[j] = 0;
    uint64_t E = 0;
    uint32_t prev = 0xffffffffu;
    for (uint32_t g = so; g < se; g++) {
      uint32_t kind, a, u;
      ld_seg<C32>(b, g, kind, a, u);
      const uint64_t w = ld_time<C32>(b.seg_wcet, g);
      erange |= w >= W_LIM;
      eshape |= (kind > 1) || (w == 0) || (kind == prev);
      prev = kind;
      if (kind == 0) E += w;  // < 192 * 2^48
      if (kind == 1) {
        if (a >= nac) eaccel = true;
        else edang |= u >= s.nu[a];
        if (nq < MAXA) {
          s.A[nq] = w; s.acc[nq] = (uint8_t)min(a, 3u); s.unit[nq] = (uint8_t)min(u, 7u); s.qcb[nq] = (uint8_t)j;
        }
        nq++;
      }
    }
    s.E[j] = E;
  }
  erange |= nq > MAXA;
  if (erange) return PAAM_SET_ERANGE;
  if (edang) return PAAM_SET_EDANGLING;
  if (eaccel) return PAAM_SET_EACCEL;
  // A13: a chain never re-enters an executor it left; sub-chains = maximal runs on one executor
  for (uint32_t c = 0; c < nch; c++) {
    for (uint32_t j = s.cb0[c]; j < s.cb0[c] + s.ncb[c]; j++) {
      s.chain[j] = (uint8_t)c;
      if (j == s.cb0[c] || s.exec[j] != s.exec[j - 1]) {
        for (uint32_t i = s.cb0[c]; i + 1 < j; i++) eshape |= s.exec[i] == s.exec[j];
        if (nsub < MAXS) { s.scb0[nsub] = j; s.sncb[nsub] = 0; s.schain[nsub] = (uint8_t)c; s.sexec[nsub] = s.exec[j]; }
        nsub++;
      }
      if (nsub <= MAXS) s.sncb[nsub - 1]++;
    }
  }
  if (eshape) return PAAM_SET_ESHAPE;
  if (nsub > MAXS) return PAAM_SET_ERANGE;
  for (uint32_t c = 0; c < nch; c++)
    for (uint32_t d = c + 1; d < nch; d++)
      if (s.prio[c] == s.prio[d]) return PAAM_SET_EDUPPRIO;
  for (uint32_t x = 0; x < nex; x++)
    for (uint32_t y = x + 1; y < nex; y++)
      if (s.xcore[x] == s.xcore[y] && s.xprio[x] == s.xprio[y]) return PAAM_SET_EDUPPRIO;
  for (uint32_t c = 0; c < nch; c++)
    if (s.D[c] == 0 || (s.cls[c] == 0 && s.D[c] > s.T[c])) return PAAM_SET_EDEADLINE;
  for (uint32_t a = 0; a < nac; a++)
    for (uint32_t x = 0; x < nex; x++)
      if (s.xcore[x] == s.server[a]) return PAAM_SET_ECORE;
  return PAAM_SET_OK;
}

// Lemma 2 (Eq.3): H = lfp of A* + LPB + sum_{HP chains k on the unit} mu(h, T_k) W[k][u],
// from the first two terms; W_SAT (UNB) once an iterate exceeds the cutoff min(D, T) (A4).
__device__ uint64_t w_lemma2(const WSet& s, uint32_t q, uint32_t nch) {
  const uint32_t c = s.chain[s.qcb[q]], r = s.rank[c], u = s.unit[q];
  const uint64_t cut = min(s.D[c], s.T[c]), base = wadd(s.Astar[q], s.LPB[q]);
  uint64_t h = base;
  while (h <= cut) {
    uint64_t g = base;
    for (uint32_t k = 0; k < nch; k++)
      if (s.rank[k] < r && s.W[s.rank[k]][u]) g = wadd(g, wmul(wmu(h, s.T[k]), s.W[s.rank[k]][u]));
    if (g == h) return h;
    h = g;
  }
  return W_SAT;
}

template <bool C32>
__global__ void __launch_bounds__(128) wide_kernel(paam_batch b, const uint32_t* __restrict__ list,
                                                   const uint32_t* __restrict__ count, int32_t* __restrict__ status_out,
                                                   uint64_t* __restrict__ out_wcrt, uint8_t* __restrict__ out_sched,
                                                   int64_t* __restrict__ out_bins, int32_t* __restrict__ out_fail) {
  const uint32_t total = *count;
  for (uint32_t li = blockIdx.x * blockDim.x + threadIdx.x; li < total; li += gridDim.x * blockDim.x) {
    const uint32_t set = list[li];
    if (set >= b.n_sets) continue;  // paam_analyze / paam_admit of the first n sets only
    WSet s;
    uint32_t nch, ncb, nq, nex, nac, nsub;
    const int st = w_load<C32>(b, set, s, nch, ncb, nq, nex, nac, nsub);
    const uint32_t c0 = b.set_chain_off[set], m = b.set_chain_off[set + 1] - c0;
    if (status_out) status_out[set] = st;
    uint32_t sched = 0;
    int32_t fail = -2 - st;
    if (st != PAAM_SET_OK) {
      if (out_wcrt) for (uint32_t c = 0; c < m; c++) out_wcrt[c0 + c] = UNS;
    } else {
      // ranks
      for (uint32_t c = 0; c < nch; c++) {
        uint32_t r = 0;
        for (uint32_t d = 0; d < nch; d++) r += s.prio[d] > s.prio[c];
        s.rank[c] = r;
      }
      // WFD units (PAAM_FLAG_WFD_UNITS): as pack.cu, items in callback order
      if (b.flags & PAAM_FLAG_WFD_UNITS) {
        uint64_t wu[MAXCB];
        uint8_t wo[MAXCB], wn[MAXCB], wc[MAXCB];
        for (uint32_t a = 0; a < nac; a++) {
          uint32_t ni = 0;
          for (uint32_t j = 0; j < ncb; j++) {
            uint64_t Aj = 0;
            for (uint32_t q = 0; q < nq; q++) if (s.qcb[q] == j && s.acc[q] == a) Aj += s.A[q];
            if (Aj) { wu[ni] = (Aj << 24) / s.T[s.chain[j]]; wc[ni] = (uint8_t)j; ni++; }
          }
          wfd_place(ni, wu, s.nu[a], wo, wn);
          for (uint32_t i = 0; i < ni; i++)
            for (uint32_t q = 0; q < nq; q++) if (s.qcb[q] == wc[i] && s.acc[q] == a) s.unit[q] = wn[i];
        }
      }
      // A* and global unit ids; sub-chain of every segment
      for (uint32_t q = 0; q < nq; q++) {
        const uint32_t a = s.acc[q];
        s.Astar[q] = s.A[q] + 2 * s.keff[a];
        s.unit[q] = (uint8_t)(s.ub[a] + s.unit[q]);
      }
      for (uint32_t i = 0; i < nsub; i++) {
        s.sq0[i] = s.seg0[s.scb0[i]];
        const uint32_t je = s.scb0[i] + s.sncb[i];
        s.snq[i] = (je < ncb ? s.seg0[je] : nq) - s.sq0[i];
        for (uint32_t q = s.sq0[i]; q < s.sq0[i] + s.snq[i]; q++) s.qsub[q] = (uint8_t)i;
      }
      // buckets (A5): the users of accelerator a ranked by priority, groups of ceil(m_a / n)
      for (uint32_t c = 0; c < nch; c++) for (uint32_t a = 0; a < 4; a++) s.bucket[c][a] = -1;
      for (uint32_t a = 0; a < nac; a++) {
        uint32_t users = 0, ma = 0;
        for (uint32_t q = 0; q < nq; q++) if (s.acc[q] == a) users |= 1u << s.chain[s.qcb[q]];
        ma = __popc(users);
        const uint32_t g = ma ? (ma + s.nb[a] - 1) / s.nb[a] : 1;
        for (uint32_t c = 0; c < nch; c++)
          if ((users >> c) & 1u) {
            uint32_t p = 0;  // position among the users by priority (0 = highest)
            for (uint32_t d = 0; d < nch; d++) p += ((users >> d) & 1u) && s.prio[d] > s.prio[c];
            s.bucket[c][a] = (int8_t)(s.nb[a] - 1 - p / g);
          }
      }
      // LP blocking and the regrouped sums W[rank][unit]
      for (uint32_t k = 0; k < nch; k++) for (uint32_t u = 0; u < MAXU; u++) s.W[k][u] = 0;
      for (uint32_t q = 0; q < nq; q++) {
        const uint32_t c = s.chain[s.qcb[q]], a = s.acc[q];
        uint64_t lpb = 0;
        for (uint32_t v = 0; v < nq; v++) {
          const uint32_t cv = s.chain[s.qcb[v]];
          if (s.unit[v] == s.unit[q] && s.prio[cv] < s.prio[c] && s.bucket[cv][a] == s.bucket[c][a])
            lpb = max(lpb, s.Astar[v]);
        }
        s.LPB[q] = lpb;
        s.W[s.rank[c]][s.unit[q]] = wadd(s.W[s.rank[c]][s.unit[q]], s.Astar[q]);
      }
      // sub-chain quantities; hp / lp (same executor) and hpp (same core, higher process priority)
      for (uint32_t i = 0; i < nsub; i++) {
        uint64_t E = 0, mE = 0, eps = 0, b3 = 0;
        uint32_t um = 0;
        for (uint32_t j = s.scb0[i]; j < s.scb0[i] + s.sncb[i]; j++) { E += s.E[j]; mE = max(mE, s.E[j]); }
        for (uint32_t q = s.sq0[i]; q < s.sq0[i] + s.snq[i]; q++) {
          eps += s.eps[s.acc[q]];
          b3 = wadd(b3, wadd(s.Astar[q], s.LPB[q]));
          um |= 1u << s.unit[q];
        }
        s.sE[i] = E; s.smaxE[i] = mE; s.seps[i] = eps; s.sbase3[i] = b3; s.sumask[i] = um;
      }
      for (uint32_t i = 0; i < nsub; i++) {
        uint32_t hp = 0, lp = 0, hpp = 0;
        const uint32_t xi = s.sexec[i];
        for (uint32_t l = 0; l < nsub; l++) {
          if (l == i) continue;
          const uint32_t xl = s.sexec[l];
          if (xl == xi) {
            if (s.prio[s.schain[l]] > s.prio[s.schain[i]]) hp |= 1u << l;
            else lp |= 1u << l;
          } else if (s.xcore[xl] == s.xcore[xi] && s.xprio[xl] > s.xprio[xi]) {
            hpp |= 1u << l;
          }
        }
        s.shp[i] = hp; s.slp[i] = lp; s.shpp[i] = hpp;
      }
      // Lemma 2 for every segment; S_c; the blocking term (or A10's sound variant)
      for (uint32_t q = 0; q < nq; q++) s.H[q] = w_lemma2(s, q, nch);
      for (uint32_t i = 0; i < nsub; i++) {
        uint64_t S = 0;
        for (uint32_t q = s.sq0[i]; q < s.sq0[i] + s.snq[i]; q++) S = wadd(S, s.H[q]);
        s.sS[i] = S;
      }
      // Eq.5 per sub-chain once its dependencies (hp, spinning hpp: A7, A8) are solved
      uint32_t solved = 0;
      const uint32_t all = nsub >= 32 ? 0xffffffffu : (1u << nsub) - 1u;
      while (solved != all) {
        for (uint32_t i = 0; i < nsub; i++) {
          if ((solved >> i) & 1u) continue;
          uint32_t dep = s.shp[i];
          for (uint32_t h = 0; h < nsub; h++) if (((s.shpp[i] >> h) & 1u) && s.xwait[s.sexec[h]] == 1) dep |= 1u << h;
          if (dep & ~solved) continue;
          const uint32_t c = s.schain[i], r = s.rank[c];
          const uint64_t cut = min(s.D[c], s.T[c]);
          uint64_t B = 0;
          for (uint32_t l = 0; l < nsub; l++) if ((s.slp[i] >> l) & 1u) B = max(B, s.smaxE[l]);
          if (b.flags & PAAM_FLAG_BLOCKING_SOUND) {  // A10: an LP callback also holds its accelerator wait
            for (uint32_t l = 0; l < nsub; l++) {
              if (!((s.slp[i] >> l) & 1u)) continue;
              for (uint32_t j = s.scb0[l]; j < s.scb0[l] + s.sncb[l]; j++) {
                uint64_t v = s.E[j];
                for (uint32_t q = 0; q < nq; q++) if (s.qcb[q] == j) v = wadd(v, wadd(s.H[q], s.eps[s.acc[q]]));
                B = max(B, v);
              }
            }
          }
          bool pois = false;
          for (uint32_t h = 0; h < nsub; h++) if (((dep >> h) & 1u) && s.sR[h] == W_SAT) pois = true;
          uint64_t R = 1, Hst = 0;
          auto C_of = [&](uint64_t t) {  // Lemma 3 (Eq.4, union form A1)
            uint64_t v = s.sbase3[i];
            for (uint32_t k = 0; k < nch; k++) {
              if (s.rank[k] >= r) continue;
              uint64_t wk = 0;
              for (uint32_t u = 0; u < MAXU; u++) if ((s.sumask[i] >> u) & 1u) wk = wadd(wk, s.W[s.rank[k]][u]);
              if (wk) v = wadd(v, wmul(wmu(t, s.T[k]), wk));
            }
            return v;
          };
          if (pois) {
            R = W_SAT;
          } else {
            for (;;) {
              const uint64_t Hs = wadd(min(s.sS[i], C_of(R)), s.seps[i]);  // Eq.1 with the min
              uint64_t F = wadd(wadd(B, s.sE[i]), Hs);
              for (uint32_t h = 0; h < nsub; h++) {
                if (!(((s.shp[i] | s.shpp[i]) >> h) & 1u)) continue;
                const bool dh = ((dep >> h) & 1u) != 0;  // spin()
                const uint64_t X = wadd(s.sE[h], dh ? s.sHs[h] : s.seps[h]);
                F = wadd(F, wmul(wmu(R, s.T[s.schain[h]]), X));
              }
              if (F > cut) { R = W_SAT; break; }  // A4
              if (F == R) { Hst = Hs; break; }
              R = F;
            }
          }
          s.sR[i] = R;
          s.sHs[i] = R == W_SAT ? W_SAT : Hst;
          solved |= 1u << i;
        }
      }
      // end to end (A9) and verdict
      bool ok = true;
      int32_t first_bad = -1;
      uint32_t best_rank = 0xffffffffu;
      for (uint32_t c = 0; c < nch; c++) {
        uint64_t sum = 0;
        uint32_t k = 0;
        bool uns = false;
        for (uint32_t i = 0; i < nsub; i++)
          if (s.schain[i] == c) { k++; if (s.sR[i] == W_SAT) uns = true; else sum += s.sR[i]; }
        const uint64_t Rstar = uns ? UNS : sum + b.comm_cost * (uint64_t)(k - 1);
        if (out_wcrt) out_wcrt[c0 + c] = Rstar;
        if (s.cls[c] == 0 && (Rstar == UNS || Rstar > s.D[c])) {
          ok = false;
          if (s.rank[c] < best_rank) { best_rank = s.rank[c]; first_bad = (int32_t)c; }
        }
      }
      sched = ok ? 1u : 0u;
      fail = ok ? -1 : first_bad;
    }
    if (out_sched) out_sched[set] = (uint8_t)sched;
    if (out_fail) out_fail[set] = fail;
    if (out_bins && b.set_bin && b.set_bin[set] < b.n_bins) {
      atomicAdd((unsigned long long*)&out_bins[2 * b.set_bin[set]], 1ull);
      if (sched) atomicAdd((unsigned long long*)&out_bins[2 * b.set_bin[set] + 1], 1ull);
    }
  }
}

}  // namespace

#ifndef PAAM_WARP_EMU
// The wide sets listed in list[0 .. *count) (count is device memory, written by the u32 kernels).
int launch_wide(const paam_batch* b, const uint32_t* list, const uint32_t* count, int32_t* status, uint64_t* out_wcrt,
                uint8_t* out_sched, int64_t* out_bins, int32_t* out_fail, cudaStream_t st, bool c32) {
  if (b->n_sets == 0) return PAAM_OK;
  if (c32) wide_kernel<true><<<148, 128, 0, st>>>(*b, list, count, status, out_wcrt, out_sched, out_bins, out_fail);
  else wide_kernel<false><<<148, 128, 0, st>>>(*b, list, count, status, out_wcrt, out_sched, out_bins, out_fail);
  count_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PAAM_OK : fail_cuda(e, "wide_kernel launch");
}
#endif

}  // namespace paam
