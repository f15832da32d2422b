// analyze.cu -- §8(a) steps 3-6: the WCRT fixed points of every chain set, one warp per set.
//
//   step 3  Lemma 2 / Eq.3: one lane per accelerator segment iterates
//           H <- A* + LPB + sum_{HP chains k} mu(H, T_k) * W[unit][k]     (start: first two terms)
//           to its least fixed point, or UNB (= SAT) once an iterate exceeds the cutoff (A4).
//           W[u][k] regroups the hps sum per interfering chain and unit (all segments of chain k on
//           unit u share T_k, so sum mu*A* = mu * sum A* exactly).  Computed on demand: step 4 first
//           uses the lower bound S_lb (sum of the start values) and asks for the exact S_c only where
//           the min(S_c, C_c) could depend on it (see step 4); the sound blocking flag computes all.
//   step 4  Theorem 1 / Eq.5: every sub-chain of the set at once, one lane each.  The
//           sub-chains depend on each other only through H*_h of their hp / spinning hpp sub-chains
//           (acyclic, A7), so the joint least fixed point of the whole system is the sequential one; it
//           is reached by Jacobi iteration from below (every lane evaluates F at its current R with the
//           H*_h of the previous iterate; stop when no R and no H* changes).  mu(R, T) = 2 +
//           floor((R-1)/T) (Eq.2 for R >= 1), and the floor term is non-zero only for periods T < R:
//           an iterate adds the mu = 2 part from pack (sA2, and 2 X_h) and walks the set's chains in
//           period order only up to the first T >= R.  H*_c(R) = min(S_c, C_c(R)) + sum eps (Eq.1,
//           P:1092), C_c = Lemma 3 in union form (Eq.4, A1).
//   step 5  R* = sum of sub-chain R_c + comm per executor crossing (A9); verdict = every
//           CRITICAL chain has R* <= D, voted with __all_sync.
//   step 6  per-warp shared-memory bin counts, flushed with one global atomic per bin at warp exit.
#include "common.cuh"

namespace paam {

namespace {

#ifndef ANA_AW
#define ANA_AW 8
#endif
#ifndef ANA_TICK
#define ANA_TICK 4
#endif
constexpr int AW = ANA_AW;     // warps per block
constexpr int WARP_BINS = 32;  // bins counted per warp in shared memory (more: direct global atomics)
constexpr uint32_t TICK = ANA_TICK;  // sets per work ticket
constexpr uint64_t UNS = PAAM_UNSCHED;

struct __align__(16) WarpSmem {
  Record rec;
  uint32_t H[MAXA];    // Lemma-2 value per accelerator segment (SAT = UNB)
  uint32_t R[MAXS];    // converged R_c (SAT = UNSCHED)
  uint32_t Hs[MAXS];   // H*_c at the sub-chain's current iterate (SAT once it is UNSCHED)
  uint8_t posOf[MAXC]; // period position of chain rank k
  uint8_t sPos[MAXS];  // period position of sub-chain h's chain
  unsigned long long sum[MAXC];  // end-to-end accumulation per chain
  uint32_t uns[MAXC];
};

constexpr uint32_t FULL = 0xffffffffu;
// Lemma 2 (Eq.3) for accelerator segment i: the least fixed point of
// G(h) = aBase2 + sum_{k<r} floor((h-1)/T_k) * W[k][u] from aBase2, or SAT (UNB) once an iterate
// exceeds the cutoff (A4).  aBase2 already holds A* + LPB + 2 sum_{k<r} W[k][u] (the "+2" of every mu),
// so the start is G's value for floor(.) = 0, <= the least fixed point (A3).  Products are 64-bit and
// < 2^62; the sum's high word is latched after each addition (a sum >= 2^32 is far above every cutoff,
// and one < 2^32 cannot wrap in one addition).
__device__ __forceinline__ uint32_t lemma2(const Record& r, uint32_t i) {
  const uint32_t misc = r.aMisc[i];
  const uint32_t rk = misc & 0xffu, u = (misc >> 8) & 0xffu;
  const uint32_t base = r.aBase2[i], cut = r.cCut[rk];
  uint32_t h = base;
  while (h <= cut) {
    const uint32_t h2 = (h - 1u) << 1;
    uint64_t acc = base;
    uint32_t hi = 0;
#pragma unroll 2
    for (uint32_t k = 0; k < rk; k++) {
      acc += (uint64_t)f_shr(__umulhi(h2, r.cM[k]), r.cMisc[k]) * r.W[k][u];
      hi |= (uint32_t)(acc >> 32);  // latched high word (eval_eq5)
    }
    if (hi || acc > cut) break;
    const uint32_t g = (uint32_t)acc;
    if (g == h) return h;
    h = g;
  }
  return SAT;
}

// Lemma 3's floor terms (Eq.4) for the periods T < R of lmask, walked from the shortest: bit
// 31 - position of lmask is pTab[position] (ascending periods), so the highest bit comes first.  WSEL:
// the weight is not the table's two-unit sum (see eval_eq5).  Overflow: every product is < 2^62 (q <=
// R - 1 < 2^31, every weight <= SAT), so a sum still < 2^32 cannot wrap in one addition; hi latches the
// sum's high word after each one and any nonzero latch saturates.  nm = min (q + 1) T (nxt - 1).
template <bool WSEL>
__device__ __forceinline__ uint64_t lemma3_terms(const Record& r, uint32_t R, uint32_t h2, uint32_t lmask,
                                                 uint32_t wsel, uint32_t umask, uint32_t& hi, uint32_t& nm) {
  uint64_t acc = 0;
  for (uint32_t m = lmask; m;) {
    const uint32_t i = f_hibit(m);
    const uint4 p = r.pTab[31u - i];  // {T, M, L | rank << 8, W[rank][0] + W[rank][1]}
    if (p.x >= R) { nm = min(nm, p.x); break; }  // this and every later period: floor((R-1)/T) = 0
    m ^= 1u << i;
    const uint32_t q = f_shr(__umulhi(h2, p.y), p.z);
    nm = min(nm, q * p.x + p.x);
    uint32_t wu = p.w;
    if (WSEL) {  // not both of units 0 and 1: one unit (wsel = unit + 1), or the general unit union
      const uint32_t k = p.z >> 8;
      if (wsel <= MAXU) {
        wu = r.W[k][wsel - 1];
      } else {
        wu = 0;
        for (uint32_t um = umask; um; um &= um - 1) wu = sadd(wu, r.W[k][__ffs(um) - 1]);
      }
    }
    acc += (uint64_t)q * wu;
    hi |= (uint32_t)(acc >> 32);
  }
  return acc;
}

// One Eq.5 evaluation F_c(R) (Theorem 1) for R >= 1, with mu(R, T) = 2 + floor((R-1)/T)
// (Eq.2): the mu = 2 parts come precomputed (A2 = base3 + 2 sum WU for Lemma 3, xs2 = 2 sum X_h of the
// static interferers), and the floor parts are added only for periods T < R -- for the Lemma-3 chains
// by walking their period positions (lmask) in ascending period order up to the first T >= R.
// C = C_c(R) (Eq.4, union form A1), nH = H*_c(R) = min(S, C) + eps (Eq.1), F = B + E + H* +
// the hp / hpp interference (SAT = above the cutoff: UNSCHED, A4; then H* = SAT poisons dependants, A8).
__device__ __forceinline__ void eval_eq5(const Record& r, const WarpSmem& w, uint32_t R, uint32_t lmask, uint32_t wsel,
                                         uint32_t umask, uint32_t A2, uint32_t S, uint32_t eps, uint32_t BE, uint32_t cut,
                                         uint32_t xm, uint32_t depm, uint32_t xs2, uint32_t xTmin, uint32_t& F,
                                         uint32_t& nH, uint32_t& C, uint32_t& nxt) {
  // nxt: the smallest R' > R at which a floor term floor((R' - 1) / T) differs from its value at R (a term
  // with q = floor((R - 1) / T) changes at (q + 1) T + 1 < 2^32); below it F and C are those at R while
  // the interferers' H* are unchanged (fused.cu f_eval).  nm = nxt - 1.
  const uint32_t h2 = (R - 1u) << 1;
  uint32_t hi = 0;
  uint32_t nm = 0xfffffffeu;
  uint64_t acc = wsel ? lemma3_terms<true>(r, R, h2, lmask, wsel, umask, hi, nm)
                      : lemma3_terms<false>(r, R, h2, lmask, wsel, umask, hi, nm);
  acc += A2;
  C = (hi || acc > SAT) ? SAT : (uint32_t)acc;  // C_c(R), Eq.4
  nH = sadd(min(S, C), eps);                     // H*_c(R), Eq.1
  uint64_t xs = xs2;  // CPU interference (hp, hpp): the mu = 2 part of the static interferers
  uint32_t xhi = 0;   // latched, as hi
  for (uint32_t m = depm; m;) {  // X_h = E_h + H*_h at h's current iterate (hp, spinning hpp); order-free
    const uint32_t h = f_hibit(m);
    m ^= 1u << h;
    const uint32_t X = sadd(r.sE[h], w.Hs[h]);
    const uint4 p = r.pTab[w.sPos[h]];
    const uint32_t q = p.x < R ? f_shr(__umulhi(h2, p.y), p.z) : 0u;
    nm = min(nm, q * p.x + p.x);
    xs += (uint64_t)(q + 2u) * X;
    xhi |= (uint32_t)(xs >> 32);
  }
  if (R > xTmin) {  // the floor terms of suspending hpp interferers with T_h < R: X_h = E_h + eps_h
    for (uint32_t m = xm & ~depm; m;) {
      const uint32_t h = f_hibit(m);
      m ^= 1u << h;
      const uint4 p = r.pTab[w.sPos[h]];
      if (p.x < R) {
        const uint32_t q = f_shr(__umulhi(h2, p.y), p.z);
        nm = min(nm, q * p.x + p.x);
        xs += (uint64_t)q * sadd(r.sE[h], r.sEps[h]);
        xhi |= (uint32_t)(xs >> 32);
      } else {
        nm = min(nm, p.x);
      }
    }
  } else if (xTmin != 0xffffffffu) {
    nm = min(nm, xTmin);
  }
  nxt = nm + 1u;
  const uint64_t f = (uint64_t)BE + nH + xs;
  F = (hi || xhi || f > cut) ? SAT : (uint32_t)f;  // above the cutoff: UNSCHED (A4)
  if (F == SAT) nH = SAT;                          // dependants become UNSCHED as well (A8)
}

// L2 prefetch of the next record while the current one is analysed.  Measured: 2.74 -> 2.63 ms per 2M
// sets, but the whole 4.4 KB slot is fetched where the staging reads only its live vectors (DRAM 3.24 ->
// 4.18 KB per set; restricting it to the live lines was slower, 2.82 ms), so it is off by default.
// The record's 16-byte vectors and which of them are live (analyze_kernel stages only those): the
// header's counts decide, per array, how many leading vectors are live (pack writes nothing past them,
// and nothing in analyze reads past them).
constexpr int REC_NV = sizeof(Record) / 16;
constexpr int V_CH = offsetof(Record, cCut) / 16, V_P = offsetof(Record, pTab) / 16;
constexpr int V_W = offsetof(Record, W) / 16;
constexpr int V_SUB = offsetof(Record, sE) / 16, V_SEG = offsetof(Record, aBase2) / 16;
constexpr int V_SND = offsetof(Record, aEps) / 16;  // aEps, aCbE: sound blocking only
static_assert(V_CH == 2 && V_P - V_CH == 4 * MAXC / 4 && V_W - V_P == MAXC && V_SEG - V_SUB == 10 * MAXS / 4 &&
                  V_SND - V_SEG == 2 * MAXA / 4 && REC_NV - V_SEG == 4 * MAXA / 4 && MAXU == 8 && MAXC == 32 &&
                  MAXS == 32,
              "live-vector map assumes the Record layout in common.cuh");
__device__ __forceinline__ void rec_counts(uint32_t hdr, uint32_t& nc, uint32_t& vc, uint32_t& vs, uint32_t& va) {
  nc = hdr & 0xffu;
  vc = (nc + 3) >> 2;
  vs = (((hdr >> 8) & 0xffu) + 3) >> 2;
  va = (((hdr >> 16) & 0xffu) + 3) >> 2;
}
__device__ __forceinline__ bool rec_live(int i, uint32_t nc, uint32_t vc, uint32_t vs, uint32_t va, bool sound) {
  return i < V_CH    ? true
         : i < V_P   ? (uint32_t)((i - V_CH) & (MAXC / 4 - 1)) < vc
         : i < V_W   ? (uint32_t)(i - V_P) < nc  // one period-table entry per vector
         : i < V_SUB ? (uint32_t)((i - V_W) >> 1) < nc  // W row k = 2 vectors
         : i < V_SEG ? (uint32_t)((i - V_SUB) & (MAXS / 4 - 1)) < vs
         : i < REC_NV ? (uint32_t)((i - V_SEG) & (MAXA / 4 - 1)) < va && (i < V_SND || sound)
                      : false;
}

#ifndef ANA_PF
// L2 prefetch of the next record (one line per lane) while this one is solved: measured 2.625 -> 2.524 ms
// per 2M sets; it also fetches the record's dead tails (tools/ana_pf_ab.sh; prefetching only the live
// lines cost more instructions than it saved: 2.649 ms)
#define ANA_PF 1
#endif
#ifndef ANA_MINB
#define ANA_MINB 4
#endif
__global__ void __launch_bounds__(AW * 32, ANA_MINB) analyze_kernel(const Record* __restrict__ recs, uint32_t n,
                                                          uint64_t comm, uint32_t flags, uint32_t n_bins,
                                                          uint64_t* __restrict__ out_wcrt,
                                                          uint8_t* __restrict__ out_sched,
                                                          int64_t* __restrict__ out_bins,
                                                          int32_t* __restrict__ out_fail,
                                                          unsigned int* __restrict__ ticket) {
  __shared__ WarpSmem smem[AW];
  __shared__ unsigned int wbins_all[AW][2 * WARP_BINS];
  const int lane = threadIdx.x & 31;
  WarpSmem& w = smem[threadIdx.x >> 5];
  unsigned int* wbins = wbins_all[threadIdx.x >> 5];
  const bool warp_bins = out_bins && n_bins <= WARP_BINS;  // per-warp counters, flushed at warp exit
  if (warp_bins) for (uint32_t i = lane; i < 2 * n_bins; i += 32) wbins[i] = 0;
  Record& r = w.rec;
  const bool sound = (flags & PAAM_FLAG_BLOCKING_SOUND) != 0;  // aEps / aCbE / sLp are read only then

  // Dynamic work distribution: warps take TICK consecutive sets per atomic ticket, so the per-set
  // cost variance does not leave warps (and their block's resources) idle at the end.
  // The next set's header word (its counts) is loaded one set ahead, so staging can skip the
  // record vectors past the live entries without a round trip in front of the set's loads.
  const uint32_t* hdr_base = reinterpret_cast<const uint32_t*>(recs);
  constexpr uint32_t HDR_STRIDE = sizeof(Record) / 4;
  uint32_t set, left;  // left: sets of the current ticket after `set`
  {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(ticket, TICK);
    set = __shfl_sync(FULL, t, 0);
    left = set < n ? min((uint32_t)TICK, n - set) - 1 : 0;
  }
  uint32_t hdr = set < n ? __ldg(hdr_base + (size_t)set * HDR_STRIDE) : 0u;
  while (set < n) {
    // ---- stage the record's live vectors in shared memory (16-byte vector loads, coalesced) -------
    // The header's counts decide, per array, how many leading 16-byte vectors are live (pack writes
    // nothing past them, and nothing below reads past them).  Config-3 sets use about 55% of the record.
    {
      const uint4* src = reinterpret_cast<const uint4*>(recs + set);
      uint4* dst = reinterpret_cast<uint4*>(&r);
      constexpr int NV = REC_NV;
      uint32_t nc, vc, vs, va;
      rec_counts(hdr, nc, vc, vs, va);
      // Predicated loads in groups of four, all issued before their stores (one round trip per group).
      constexpr int NK = (NV + 31) / 32;
#pragma unroll
      for (int k0 = 0; k0 < NK; k0 += 4) {
        uint4 v[4];
        uint32_t livem = 0;
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const int i = lane + 32 * (k0 + k);
          const bool live = rec_live(i, nc, vc, vs, va, sound);
          livem |= (uint32_t)live << k;
          v[k] = live ? __ldg(src + i) : uint4{0u, 0u, 0u, 0u};
        }
#pragma unroll
        for (int k = 0; k < 4; k++)
          if (livem >> k & 1u) dst[lane + 32 * (k0 + k)] = v[k];
      }
    }
    uint32_t nset, nleft;
    if (left) {
      nset = set + 1;
      nleft = left - 1;
    } else {
      uint32_t t = 0;
      if (lane == 0) t = atomicAdd(ticket, TICK);
      nset = __shfl_sync(FULL, t, 0);
      nleft = nset < n ? min((uint32_t)TICK, n - nset) - 1 : 0;
    }
    const uint32_t nhdr = nset < n ? __ldg(hdr_base + (size_t)nset * HDR_STRIDE) : 0u;
#if ANA_PF && !defined(PAAM_WARP_EMU)
    if (nset < n) {  // the next record into L2, one 128-byte line per lane
      const uintptr_t base = reinterpret_cast<uintptr_t>(recs + nset);
      const uintptr_t la = (base & ~(uintptr_t)127) + 128u * lane;
      if (la < base + sizeof(Record)) asm volatile("prefetch.global.L2 [%0];" ::"l"(la));
    }
#endif
    __syncwarp();
    const int32_t status = r.status;
    const bool handed = status == REC_STATUS_WIDE;  // a wide set: wide_kernel writes its outputs
    uint32_t sched = 0;
    if (handed) {
    } else if (status != PAAM_SET_OK) {
      if (out_wcrt)
        for (uint32_t i = lane; i < r.n_out; i += 32) out_wcrt[r.chain_base + i] = UNS;
      if (out_fail && lane == 0) out_fail[set] = -2 - status;  // admission: rejected by validation
    } else {
      const uint32_t nch = r.n_chain, nsub = r.n_sub, nas = r.n_aseg;

      // ---- step 3: Lemma 2, one lane per accelerator segment ----------------------------------------
      // Only the sound blocking term (A10) needs every H up front.  Otherwise S_c enters Eq.5 only as
      // min(S_c, C_c(R)) and C_c almost always wins, so step 4 starts from the lower bound
      // S_lb = sum of the Lemma-2 start values (pack's sSlb) and computes the exact S_c only for a
      // sub-chain whose C_c at the converged R exceeds S_lb (see step 4).
      // Segments are in rank order (rank = number of HP chains = loop length), so the loop cost of a
      // round is set by its highest rank: the first round takes segments [0, nas-32) (short loops),
      // the second the last 32 (nas <= 64).
      const bool lazy_s = !(flags & PAAM_FLAG_BLOCKING_SOUND);
      if (!lazy_s) {
        const uint32_t f = nas > 32 ? nas - 32 : 0;
        for (uint32_t i = lane < f ? lane : f + lane; i < nas; i = (i < f) ? f + lane : nas) w.H[i] = lemma2(r, i);
      }
      __syncwarp();
      // ---- per sub-chain constants (lane = sub-chain in canonical order) -----------------------------
      const bool act = lane < (int)nsub;
      uint32_t rk = 0, umask = 0, cut = 0, BE = 0, A2 = 0, S = 0, eps = 0, hpm = 0, hppm = 0;
      if (act) {
        const uint32_t misc = r.sMisc[lane];
        rk = misc & 0xffu;
        umask = (misc >> 8) & 0xffu;
        cut = r.cCut[rk];
        A2 = r.sA2[lane];
        eps = r.sEps[lane];
        hpm = r.sHp[lane];
        hppm = r.sHpp[lane];
        uint32_t B = r.sB[lane];
        if (lazy_s) {
          S = r.sSlb[lane];
        } else {  // exact S_c, and A10: an LP callback also holds its accelerator wait
          const uint32_t sg = r.sSeg[lane], a0 = sg & 0xffu, na = (sg >> 8) & 0xffu;
          for (uint32_t i = a0; i < a0 + na; i++) S = sadd(S, w.H[i]);
          uint32_t lp = r.sLp[lane];
          while (lp) {
            const uint32_t l = __ffs(lp) - 1;
            lp &= lp - 1;
            const uint32_t sl = r.sSeg[l], b0 = sl & 0xffu, bn = (sl >> 8) & 0xffu;
            uint32_t cur_cb = 0xffffffffu, v = 0;
            for (uint32_t i = b0; i < b0 + bn; i++) {
              const uint32_t cbid = r.aMisc[i] >> 24;
              if (cbid != cur_cb) {
                if (cur_cb != 0xffffffffu) B = max(B, v);
                cur_cb = cbid;
                v = r.aCbE[i];
              }
              v = sadd(v, sadd(w.H[i], r.aEps[i]));
            }
            if (cur_cb != 0xffffffffu) B = max(B, v);
          }
        }
        BE = sadd(B, r.sE[lane]);
      }
      const uint32_t spin_mask = __ballot_sync(FULL, act && ((r.sMisc[lane] >> 16) & 1u));
      const uint32_t depm = hpm | (hppm & spin_mask);  // X_h = E_h + H*_h (hp, spinning hpp: P:1132)
      const uint32_t xm = hpm | hppm;                   // every CPU interferer (Eq.5 sums)
      const bool critical = act && ((r.cMisc[rk] >> 8) & 0xffu) == 0;
      bool sexact = !lazy_s;
      // period positions of the chains (pTab is in ascending period order)
      if (lane < (int)nch) w.posOf[r.pTab[lane].z >> 8] = (uint8_t)lane;
      __syncwarp();
      // lmask: period positions of the chains of rank < rk (Lemma-3 interferers, Eq.4), an exclusive
      // OR-scan over ranks of 1 << (31 - position)
      uint32_t pb = lane < (int)nch ? (0x80000000u >> w.posOf[lane]) : 0u;  // bit 31 - position
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, pb, o);
        if (lane >= o) pb |= y;
      }
      uint32_t pex = __shfl_up_sync(FULL, pb, 1);
      if (lane == 0) pex = 0;
      const uint32_t lm_rk = __shfl_sync(FULL, pex, rk);  // every lane shuffles (rk = 0 when inactive)
      const uint32_t lmask = act ? lm_rk : 0u;
      const uint32_t n_unit = r.n_unit;
      // Lemma-3 weight of chain k for this sub-chain: W[k][0] + W[k][1] (pTab.w) when it uses exactly
      // units 0 and 1 of a <= 2-unit set (wsel = 0), W[k][u] for a single unit u (wsel = u + 1), else
      // the union over its units (wsel = MAXU + 1)
      const uint32_t wsel = (n_unit <= 2 && umask == (1u << n_unit) - 1u) ? 0u
                            : __popc(umask) == 1 ? (uint32_t)__ffs(umask) : (uint32_t)MAXU + 1u;
      // CPU interference of the suspending hpp interferers with every mu = 2 (2 (E_h + eps_h):
      // spin() = delta eps), and their smallest period; the dependencies (hp, spinning hpp)
      // are added per iterate
      uint32_t xs2 = 0, xTmin = 0xffffffffu;
      if (act) {
        w.sPos[lane] = w.posOf[rk];
        for (uint32_t m = xm & ~depm; m;) {
          const uint32_t h = f_hibit(m);
          m ^= 1u << h;
          xs2 = sadd(xs2, sadd(r.sE[h], r.sEps[h]));
          xTmin = min(xTmin, r.pTab[w.posOf[r.sMisc[h] & 0xffu]].x);
        }
        xs2 = sadd(xs2, xs2);
      }
      __syncwarp();

      // ---- step 4: Eq.5 for all sub-chains at once (Jacobi from below) -------------------------------
      // Start: R = 1 <= lfp (E_c + H*_c >= 1), with H*_h at R = 1 for the dependants.
      uint32_t R = act ? 1u : SAT, Hst = act ? sadd(min(S, A2), eps) : SAT, C = A2;
      if (act) w.Hs[lane] = Hst;
      __syncwarp();
      bool dirty = act;  // must be evaluated this iterate (own R or a dependency's H* changed)
      bool miss = false;
      for (;;) {
        uint32_t F = R, nH = Hst, nxt = 0u;
        if (dirty)  // one checked copy (the unchecked one doubled the loop's code)
          eval_eq5(r, w, R, lmask, wsel, umask, A2, S, eps, BE, cut, xm, depm, xs2, xTmin, F, nH, C, nxt);
        const bool chg = dirty && (F != R || nH != Hst);
        const uint32_t cm = __ballot_sync(FULL, chg);
        if (!cm) {
          // fixed point with the current S values; a lazy S_lb is exact enough unless C_c(R) > S_lb
          const bool need = act && !sexact && R != SAT && C > S;
          const uint32_t needm = __ballot_sync(FULL, need);
          if (!needm) break;
          for (uint32_t i = lane; i < nas; i += 32)  // lane per segment of the sub-chains that need it
            if ((needm >> ((r.aMisc[i] >> 16) & 0xffu)) & 1u) w.H[i] = lemma2(r, i);
          __syncwarp();
          if (need) {
            const uint32_t sg = r.sSeg[lane], a0 = sg & 0xffu, na = (sg >> 8) & 0xffu;
            uint32_t Sx = 0;
            for (uint32_t i = a0; i < a0 + na; i++) Sx = sadd(Sx, w.H[i]);
            S = Sx;
            sexact = true;
          }
          dirty = need;  // S only grew: F continues from the current R (still <= the new lfp)
          continue;
        }
        __syncwarp();  // every lane has read the H* of the previous iterate
        if (chg) {
          R = F;
          Hst = nH;
          w.Hs[lane] = nH;
        }
        __syncwarp();
        // a lane that moved below nxt has F(F) = F unless an interferer's H* changed (fused.cu)
        dirty = act && R != SAT && ((chg && R >= nxt) || (depm & cm) != 0u);
        if (flags & PAAM_FLAG_VERDICT_ONLY) {  // R_c > D_c of a CRITICAL chain => R* > D
          if (__any_sync(FULL, critical && R == SAT)) { miss = true; break; }
        }
      }
      if (act) w.R[lane] = R;
      __syncwarp();

      // ---- step 5: end to end and verdict ---------------------------------------------------------
      if (miss) goto verdict_done;  // verdict-only early exit: sched stays 0 (out_wcrt is NULL here)
      if (lane < nch) { w.sum[lane] = 0; w.uns[lane] = 0; }
      __syncwarp();
      if (act) {
        const uint32_t Rh = w.R[lane];
        if (Rh == SAT) w.uns[rk] = 1;
        else atomicAdd(&w.sum[rk], (unsigned long long)Rh);
      }
      __syncwarp();
      bool ok = true;
      if (lane < nch) {
        const uint32_t cm = r.cMisc[lane];
        const uint32_t nsc = cm >> 24;  // sub-chains of this chain
        const uint64_t Rstar = w.uns[lane] ? UNS : w.sum[lane] + comm * (uint64_t)(nsc - 1);
        if (out_wcrt) out_wcrt[r.chain_base + ((cm >> 16) & 0xffu)] = Rstar;
        const bool critical = ((cm >> 8) & 0xffu) == 0;
        ok = !critical || (Rstar != UNS && Rstar <= (uint64_t)r.cD[lane]);
      }
      sched = __all_sync(FULL, ok) ? 1u : 0u;
      if (out_fail) {  // admission: the first failing chain in priority order (lane = rank)
        const uint32_t bad = __ballot_sync(FULL, !ok);
        if (lane == 0) out_fail[set] = bad ? (int32_t)((r.cMisc[__ffs(bad) - 1] >> 16) & 0xffu) : -1;
      }
    }
  verdict_done:
    if (lane == 0 && !handed) {
      if (out_sched) out_sched[set] = (uint8_t)sched;
      if (out_bins && r.bin < n_bins) {  // (pack stores bin = ~0 for an out-of-range bin: ERANGE)
        if (warp_bins) {
          wbins[2 * r.bin]++;
          if (sched) wbins[2 * r.bin + 1]++;
        } else {
          atomicAdd((unsigned long long*)&out_bins[2 * r.bin], 1ull);
          if (sched) atomicAdd((unsigned long long*)&out_bins[2 * r.bin + 1], 1ull);
        }
      }
    }
    __syncwarp();
    set = nset;
    left = nleft;
    hdr = nhdr;
  }
  if (warp_bins) {
    __syncwarp();
    for (uint32_t i = lane; i < 2 * n_bins; i += 32)
      if (wbins[i]) atomicAdd((unsigned long long*)&out_bins[i], (unsigned long long)wbins[i]);
  }
}

}  // namespace

#ifndef PAAM_WARP_EMU
int launch_analyze(const Record* rec, uint32_t n, uint64_t comm, uint32_t flags, uint32_t n_bins,
                   uint64_t* out_wcrt, uint8_t* out_sched, int64_t* out_bins, unsigned int* ticket,
                   cudaStream_t st, int32_t* out_fail) {
  if (n == 0) return PAAM_OK;
  cudaMemsetAsync(ticket, 0, sizeof(unsigned int), st);
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, analyze_kernel, AW * 32, 0);
  if (per_sm < 1) per_sm = 1;
  const uint32_t need = (n + AW - 1) / AW;
  const uint32_t cap = (uint32_t)sms * (uint32_t)per_sm;
  const uint32_t grid = need < cap ? need : cap;
  analyze_kernel<<<grid, AW * 32, 0, st>>>(rec, n, comm, flags, n_bins, out_wcrt, out_sched, out_bins, out_fail,
                                           ticket);
  count_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PAAM_OK : fail_cuda(e, "analyze_kernel launch");
}

#endif  // PAAM_WARP_EMU

}  // namespace paam
