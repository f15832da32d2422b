// analyze.cu -- §8(a) steps 3-6: the WCRT fixed points of every chain set, one warp per set.
//
//   step 3  Lemma 2 / Eq.3: one lane per accelerator segment iterates
//           H <- A* + LPB + sum_{HP chains k} mu(H, T_k) * W[unit][k]     (start: first two terms)
//           to its least fixed point, or UNB (= SAT) once an iterate exceeds the cutoff (A4).
//           W[u][k] regroups the hps sum per interfering chain and unit (all segments of chain k on
//           unit u share T_k, so sum mu*A* = mu * sum A* exactly).  Computed on demand: step 4 first
//           uses the lower bound S_lb (sum of the start values) and asks for the exact S_c only where
//           the min(S_c, C_c) could depend on it (see step 4); the sound blocking flag computes all.
//   step 4  Theorem 1 / Eq.5 per sub-chain, in waves of up to four sub-chains whose
//           dependencies (hp, spinning hpp: earlier in the canonical order, A7) are solved, first
//           ready first, one 8-lane group per sub-chain: lanes take the Lemma-3 chains and the
//           hp / hpp sub-chains in turn, two saturating butterfly reductions per iterate give the
//           Lemma-3 interference (Eq.4, union form A1) and the CPU interference, and
//           H*_c(R) = min(S_c, C_c(R)) + sum eps (Eq.1).  Convergence / deadline miss are
//           group-uniform because every lane of a group holds the same reduced value.
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
#define ANA_TICK 2
#endif
constexpr int AW = ANA_AW;     // warps per block
constexpr int WARP_BINS = 32;  // bins counted per warp in shared memory (more: direct global atomics)
constexpr uint32_t TICK = ANA_TICK;  // sets per work ticket
constexpr uint64_t UNS = PAAM_UNSCHED;

struct __align__(16) WarpSmem {
  Record rec;
  uint32_t H[MAXA];    // Lemma-2 value per accelerator segment (SAT = UNB)
  uint32_t S[MAXS];    // per-segment bound summed over the sub-chain
  uint32_t Bc[MAXS];   // blocking term in use (as written, or the sound variant)
  uint32_t R[MAXS];    // converged R_c (SAT = UNSCHED)
  uint32_t Hs[MAXS];   // H*_c(R_c) of every solved sub-chain
  unsigned long long sum[MAXC];  // end-to-end accumulation per chain
  uint32_t uns[MAXC];
  uint8_t gpos[4];          // the sub-chains of the current Eq.5 wave, one per lane group
};

constexpr uint32_t FULL = 0xffffffffu;
// 8-lane group reductions (xor within aligned groups of 8)
__device__ __forceinline__ void gsum8x2(uint32_t& a, uint32_t& b) {
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    const uint32_t xa = __shfl_xor_sync(FULL, a, o), xb = __shfl_xor_sync(FULL, b, o);
    a = sadd(a, xa);
    b = sadd(b, xb);
  }
}
__device__ __forceinline__ bool gor8(bool p) {
  uint32_t v = p;
  v |= __shfl_xor_sync(FULL, v, 4);
  v |= __shfl_xor_sync(FULL, v, 2);
  v |= __shfl_xor_sync(FULL, v, 1);
  return v != 0;
}

// Lemma 2 (Eq.3) for accelerator segment i: the least fixed point of
// G(h) = aBase2 + sum_{k<r} floor((h-1)/T_k) * W[k][u] from aBase2, or SAT (UNB) once an iterate
// exceeds the cutoff (A4).  aBase2 already holds A* + LPB + 2 sum_{k<r} W[k][u] (the "+2" of every mu),
// so the start is G's value for floor(.) = 0, <= the least fixed point (A3).  Products are 64-bit; a
// product >= 2^32 (high word != 0) is far above every cutoff, and without one the 64-bit sum of <= 31
// products cannot overflow.
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
      const uint32_t q = __umulhi(h2, r.cM[k]) >> (r.cMisc[k] & 31u);
      const uint64_t p = (uint64_t)q * r.W[k][u];
      acc += p;
      hi |= (uint32_t)(p >> 32);
    }
    if (hi || acc > cut) break;
    const uint32_t g = (uint32_t)acc;
    if (g == h) return h;
    h = g;
  }
  return SAT;
}

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
      constexpr int NV = sizeof(Record) / 16;
      constexpr int V_CH = offsetof(Record, cCut) / 16, V_W = offsetof(Record, W) / 16;
      constexpr int V_SUB = offsetof(Record, sE) / 16, V_SEG = offsetof(Record, aBase2) / 16;
      static_assert(V_CH == 2 && V_W - V_CH == 4 * MAXC / 4 && V_SEG - V_SUB == 9 * MAXS / 4 &&
                        NV - V_SEG == 4 * MAXA / 4 && MAXU == 8,
                    "live-vector map assumes the Record layout in common.cuh");
      const uint32_t nc = hdr & 0xffu, vc = (nc + 3) >> 2, vs = (((hdr >> 8) & 0xffu) + 3) >> 2;
      const uint32_t va = (((hdr >> 16) & 0xffu) + 3) >> 2;
      // Predicated loads in groups of four, all issued before their stores (one round trip per group).
      constexpr int NK = (NV + 31) / 32;
#pragma unroll
      for (int k0 = 0; k0 < NK; k0 += 4) {
        uint4 v[4];
        uint32_t livem = 0;
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const int i = lane + 32 * (k0 + k);
          const bool live = i < V_CH    ? true
                            : i < V_W   ? (uint32_t)((i - V_CH) & (MAXC / 4 - 1)) < vc
                            : i < V_SUB ? (uint32_t)((i - V_W) >> 1) < nc  // W row k = 2 vectors
                            : i < V_SEG ? (uint32_t)((i - V_SUB) & (MAXS / 4 - 1)) < vs
                            : i < NV    ? (uint32_t)((i - V_SEG) & (MAXA / 4 - 1)) < va
                                        : false;
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
    __syncwarp();
    const int32_t status = r.status;
    uint32_t sched = 0;
    if (status != PAAM_SET_OK) {
      if (out_wcrt)
        for (uint32_t i = lane; i < r.n_out; i += 32) out_wcrt[r.chain_base + i] = UNS;
      if (out_fail && lane == 0) out_fail[set] = -2 - status;  // admission: rejected by validation
    } else {
      const uint32_t nch = r.n_chain, nsub = r.n_sub, nas = r.n_aseg;

      // ---- step 3: Lemma 2, one lane per accelerator segment ----------------------------------------
      // Only the sound blocking term (A10) needs every H up front.  Otherwise S_c enters Eq.5 only as
      // min(S_c, C_c(R)) and C_c almost always wins, so step 4 starts from the lower bound
      // S_lb = sum of the Lemma-2 start values and computes the exact S_c only for a sub-chain whose
      // C_c at the converged R exceeds S_lb (see step 4).
      // Segments are in rank order (rank = number of HP chains = loop length), so the loop cost of a
      // round is set by its highest rank: the first round takes segments [0, nas-32) (short loops),
      // the second the last 32 (nas <= 64).
      const bool lazy_s = !(flags & PAAM_FLAG_BLOCKING_SOUND);
      if (!lazy_s) {
        const uint32_t f = nas > 32 ? nas - 32 : 0;
        for (uint32_t i = lane < f ? lane : f + lane; i < nas; i = (i < f) ? f + lane : nas) w.H[i] = lemma2(r, i);
      }
      __syncwarp();
      // per-segment sums S_c and the blocking term in use
      if (lane < nsub) {
        const uint32_t sg = r.sSeg[lane], a0 = sg & 0xffu, na = (sg >> 8) & 0xffu;
        uint32_t S = 0;
        for (uint32_t i = a0; i < a0 + na; i++) S = sadd(S, lazy_s ? r.aBase2[i] : w.H[i]);  // S_lb or S_c
        w.S[lane] = S;
        uint32_t B = r.sB[lane];
        if (flags & PAAM_FLAG_BLOCKING_SOUND) {  // A10: an LP callback also holds its accelerator wait
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
        w.Bc[lane] = B;
      }
      __syncwarp();

      // ---- step 4: Eq.5, waves of up to four ready sub-chains, one 8-lane group each -------------------
      // A sub-chain's Eq.5 reads the results of its hp sub-chains and spinning hpp sub-chains only
      // (H*_h and R_h, A8); those precede it in the canonical order (A7).  The four 8-lane groups
      // (lanes 8g..8g+7) solve four ready sub-chains at a time.  Within a group, lane l handles the
      // Lemma-3 chains k = l, l+8, ... (< rank) and the hp/hpp sub-chains h = l, l+8, ...; the two
      // interference sums are reduced over the group with three xor-shuffles each.
      const uint32_t gi = lane >> 3, gl = lane & 7;
      const bool is_sub = lane < nsub;
      const uint32_t spin_mask = __ballot_sync(FULL, is_sub && ((r.sMisc[lane] >> 16) & 1u));
      const bool two_units = r.n_unit <= 2;  // set-uniform
      // Period magic constants of the interferers a group lane serves: chain k = gl + 8j (Lemma 3) and
      // the chain of sub-chain k (hp/hpp).  They depend on k only, so they are loaded once per set.
      uint32_t KM[4], KL[4], XM[4], XL[4];
#pragma unroll
      for (uint32_t j = 0; j < 4; j++) {
        const uint32_t k = gl + 8 * j;
        KM[j] = 1; KL[j] = 0; XM[j] = 1; XL[j] = 0;
        if (k < nch) { KM[j] = r.cM[k]; KL[j] = r.cMisc[k] & 31u; }
        if (k < nsub) {
          const uint32_t hm = r.sMisc[k] & 0xffu;
          XM[j] = r.cM[hm];
          XL[j] = r.cMisc[hm] & 31u;
        }
      }
      // solve(act, c): the group's sub-chain c (if act); returns the verdict-only early-exit vote
      auto solve = [&](const bool act, const uint32_t c) -> bool {
          const uint32_t cmisc = act ? r.sMisc[c] : 0u;
          const uint32_t rk = cmisc & 0xffu, umask = (cmisc >> 8) & 0xffu;
          const uint32_t hpm = act ? r.sHp[c] : 0u, hppm = act ? r.sHpp[c] : 0u;
          const uint32_t cpu_m = hpm | hppm, dep = hpm | (hppm & spin_mask);
          const uint32_t hibit = cpu_m ? 32u - __clz(cpu_m) : 0u;
          const uint32_t jmax = (__reduce_max_sync(FULL, max(rk, hibit)) + 7u) >> 3;
          // per-lane interferers: Lemma-3 chains and hp/hpp sub-chains (A8 poison on dependencies)
          uint32_t WU[4], X[4];
          bool pois = false;
#pragma unroll
          for (uint32_t j = 0; j < 4; j++) {
            WU[j] = 0; X[j] = 0;
            if (j < jmax) {
              const uint32_t k = gl + 8 * j;
              if (k < rk) {
                uint32_t wu = 0;
                if (two_units) {  // units 0 and 1 only: one 8-byte row load, two selects
                  const uint2 w01 = *reinterpret_cast<const uint2*>(&r.W[k][0]);
                  wu = sadd((umask & 1u) ? w01.x : 0u, (umask & 2u) ? w01.y : 0u);
                } else
                for (uint32_t um = umask; um; um &= um - 1)
                  wu = sadd(wu, r.W[k][__ffs(um) - 1]);  // union of hps over the sub-chain's units (A1)
                WU[j] = wu;
              }
              if ((cpu_m >> k) & 1u) {
                X[j] = sadd(r.sE[k], (((hpm | spin_mask) >> k) & 1u) ? w.Hs[k] : r.sEps[k]);  // spin() P:1132
                if ((dep >> k) & 1u) pois |= (w.R[k] == SAT);
              }
            }
          }
          // Start value (A3): R >= 1 on every iterate, so every mu >= 2 and
          // F(R) >= B + E + min(S, base3 + 2 sum WU) + eps + 2 sum X for all R >= 1; that value is
          // therefore <= the least fixed point and one iteration closer to it than the paper's start.
          uint32_t wu_sum = 0, x_sum = 0;
#pragma unroll
          for (uint32_t j = 0; j < 4; j++) { wu_sum = sadd(wu_sum, WU[j]); x_sum = sadd(x_sum, X[j]); }
          pois = gor8(pois);
          gsum8x2(wu_sum, x_sum);
          const uint32_t BE = act ? sadd(w.Bc[c], r.sE[c]) : 0u;
          uint32_t S = act ? w.S[c] : 0u;
          const uint32_t base3 = act ? r.sBase3[c] : 0u, eps = act ? r.sEps[c] : 0u;
          const uint32_t cut = act ? r.cCut[rk] : 0u;
          uint32_t R = sadd(sadd(BE, sadd(min(S, sadd(base3, sadd(wu_sum, wu_sum))), eps)), sadd(x_sum, x_sum)), Hst = 0;
          uint32_t C = 0;  // Lemma-3 term C_c(R) of the last iterate
          bool done = !act || pois;
          if (pois) R = SAT;
          auto iterate = [&]() {
          while (__any_sync(FULL, !done)) {
            if (!done && R > cut) { R = SAT; done = true; }
            const uint32_t h2 = (R - 1u) << 1;
            uint64_t aa = 0, bb = 0;
            uint32_t hi = 0;
#pragma unroll
            for (uint32_t j = 0; j < 4; j++) {
              if (j < jmax) {
                const uint64_t pa = (uint64_t)((__umulhi(h2, KM[j]) >> KL[j]) + 2u) * WU[j];
                const uint64_t pb = (uint64_t)((__umulhi(h2, XM[j]) >> XL[j]) + 2u) * X[j];
                aa += pa;
                bb += pb;
                hi |= (uint32_t)(pa >> 32) | (uint32_t)(pb >> 32);
              }
            }
            uint32_t a = (hi || aa > SAT) ? SAT : (uint32_t)aa;
            uint32_t bs = (hi || bb > SAT) ? SAT : (uint32_t)bb;
            gsum8x2(a, bs);
            if (!done) {
              C = sadd(base3, a);
              Hst = sadd(min(S, C), eps);
              const uint32_t F = sadd(sadd(BE, Hst), bs);
              if (F == R) done = true;
              else R = F;
            }
          }
          };
          iterate();
          // With S_lb <= S_c, F_lb <= F pointwise, so lfp(F_lb) <= lfp(F): a deadline miss under S_lb is a
          // miss, and a converged R with C_c(R) <= S_lb is also a fixed point of F (both mins pick C_c),
          // hence lfp(F).  Otherwise the group computes the exact S_c (lane per segment) and iterates F on
          // from R, a valid start below lfp(F).  need is uniform within a group.
          if (lazy_s) {
            const bool need = act && !pois && R != SAT && C > S;
            if (__any_sync(FULL, need)) {
              uint32_t Sx = 0, unused = 0;
              if (need) {
                const uint32_t sg = r.sSeg[c], a0 = sg & 0xffu, na = (sg >> 8) & 0xffu;
                for (uint32_t i = a0 + gl; i < a0 + na; i += 8) Sx = sadd(Sx, lemma2(r, i));
              }
              gsum8x2(Sx, unused);
              if (need) { S = Sx; done = false; }
              else done = true;
              iterate();
            }
          }
          if (act && gl == 0) {
            w.R[c] = R;
            w.Hs[c] = (R == SAT) ? SAT : Hst;
          }
          __syncwarp();
          if (flags & PAAM_FLAG_VERDICT_ONLY)  // R_c > D_c of a CRITICAL chain => R* > D
            return __any_sync(FULL, act && gl == 0 && R == SAT && ((r.cMisc[rk] >> 8) & 0xffu) == 0);
          return false;
      };
      bool miss = false;  // verdict-only: a CRITICAL sub-chain already exceeded its deadline
      // Waves: a sub-chain is ready once every sub-chain it depends on (hp, spinning hpp) is solved;
      // each wave solves the first four ready sub-chains in canonical order, one per group.  The first
      // unsolved sub-chain is always ready (its dependencies precede it, A7).
      {
        const uint32_t my_dep = is_sub ? (r.sHp[lane] | (r.sHpp[lane] & spin_mask)) : 0u;
        uint32_t todo = nsub >= 32 ? FULL : (1u << nsub) - 1u;
        while (todo && !miss) {
          const bool rdy = ((todo >> lane) & 1u) && (my_dep & todo) == 0u;
          const uint32_t ready = __ballot_sync(FULL, rdy);
          const uint32_t rnk = __popc(ready & ((1u << lane) - 1u));
          if (rdy && rnk < 4) w.gpos[rnk] = (uint8_t)lane;
          todo &= ~__ballot_sync(FULL, rdy && rnk < 4);
          __syncwarp();
          const bool act = gi < (uint32_t)__popc(ready);
          const uint32_t c = act ? w.gpos[gi] : 0u;
          __syncwarp();
          miss = solve(act, c);
        }
      }
      __syncwarp();

      // ---- step 5: end to end and verdict ---------------------------------------------------------
      if (miss) goto verdict_done;  // verdict-only early exit: sched stays 0 (out_wcrt is NULL here)
      if (lane < nch) { w.sum[lane] = 0; w.uns[lane] = 0; }
      __syncwarp();
      if (is_sub) {
        const uint32_t rk = r.sMisc[lane] & 0xffu, Rh = w.R[lane];
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
    if (lane == 0) {
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
