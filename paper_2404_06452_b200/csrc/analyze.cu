// analyze.cu -- §8(a) steps 3-6: the WCRT fixed points of every chain set, one warp per set.
//
//   step 3  Lemma 2 / Eq.3: one lane per accelerator segment iterates
//           H <- A* + LPB + sum_{HP chains k} mu(H, T_k) * W[unit][k]     (start: first two terms)
//           to its least fixed point, or UNB (= SAT) once an iterate exceeds the cutoff (A4).
//           W[u][k] regroups the hps sum per interfering chain and unit (all segments of chain k on
//           unit u share T_k, so sum mu*A* = mu * sum A* exactly).
//   step 4  Theorem 1 / Eq.5 per sub-chain in canonical order (A7).  One R-iteration
//           is warp-wide: lane k evaluates mu(R, T_k) for chain k, lane h the hp / hpp term of
//           sub-chain h (mu by shuffle from its chain's lane), two saturating butterfly reductions
//           give the Lemma-3 interference (Eq.4, union form A1) and the CPU interference, and
//           H*_c(R) = min(S_c, C_c(R)) + sum eps (Eq.1).  Convergence / deadline miss are
//           warp-uniform because every lane holds the same reduced value.
//   step 5  R* = sum of sub-chain R_c + comm per executor crossing (A9); verdict = every
//           CRITICAL chain has R* <= D, voted with __all_sync.
//   step 6  per-block shared-memory bin counts, flushed with one global atomic per bin per block.
#include "common.cuh"

namespace paam {

namespace {

constexpr int AW = 8;          // warps per block
constexpr int MAX_BINS = 256;  // bins accumulated in shared memory (more: direct global atomics)
constexpr uint64_t UNS = PAAM_UNSCHED;

struct __align__(16) WarpSmem {
  Record rec;
  uint32_t H[MAXA];    // Lemma-2 value per accelerator segment (SAT = UNB)
  uint32_t S[MAXS];    // per-segment bound summed over the sub-chain
  uint32_t Bc[MAXS];   // blocking term in use (as written, or the sound variant)
  uint32_t R[MAXS];    // converged R_c (SAT = UNSCHED)
};

// Exact saturating warp sums of values <= SAT via the integer reduction unit (REDUX): the 16-bit halves
// are summed separately (32 * 2^16 < 2^32, no wrap) and recombined in 64 bits.
__device__ __forceinline__ uint32_t wsum(uint32_t v) {
  const uint32_t lo = __reduce_add_sync(0xffffffffu, v & 0xffffu);
  const uint32_t hi = __reduce_add_sync(0xffffffffu, v >> 16);
  const uint64_t t = ((uint64_t)hi << 16) + lo;
  return t > SAT ? SAT : (uint32_t)t;
}
__device__ __forceinline__ void wsum2(uint32_t& a, uint32_t& b) {
  const uint32_t alo = __reduce_add_sync(0xffffffffu, a & 0xffffu);
  const uint32_t blo = __reduce_add_sync(0xffffffffu, b & 0xffffu);
  const uint32_t ahi = __reduce_add_sync(0xffffffffu, a >> 16);
  const uint32_t bhi = __reduce_add_sync(0xffffffffu, b >> 16);
  const uint64_t ta = ((uint64_t)ahi << 16) + alo, tb = ((uint64_t)bhi << 16) + blo;
  a = ta > SAT ? SAT : (uint32_t)ta;
  b = tb > SAT ? SAT : (uint32_t)tb;
}

__global__ void __launch_bounds__(AW * 32) analyze_kernel(const Record* __restrict__ recs, uint32_t n,
                                                          uint64_t comm, uint32_t flags, uint32_t n_bins,
                                                          uint64_t* __restrict__ out_wcrt,
                                                          uint8_t* __restrict__ out_sched,
                                                          int64_t* __restrict__ out_bins) {
  __shared__ WarpSmem smem[AW];
  __shared__ unsigned int sbins[2 * MAX_BINS];
  const bool smem_bins = out_bins && n_bins <= MAX_BINS;
  if (smem_bins)
    for (uint32_t i = threadIdx.x; i < 2 * n_bins; i += blockDim.x) sbins[i] = 0;
  __syncthreads();

  const int lane = threadIdx.x & 31;
  WarpSmem& w = smem[threadIdx.x >> 5];
  Record& r = w.rec;
  const uint32_t nwarps = gridDim.x * AW;

  for (uint32_t set = blockIdx.x * AW + (threadIdx.x >> 5); set < n; set += nwarps) {
    // ---- stage the record in shared memory (16-byte vector loads, coalesced) ---------------------
    {
      const uint4* src = reinterpret_cast<const uint4*>(recs + set);
      uint4* dst = reinterpret_cast<uint4*>(&r);
      constexpr int NV = sizeof(Record) / 16;
#pragma unroll 4
      for (int i = lane; i < NV; i += 32) dst[i] = __ldg(src + i);
    }
    __syncwarp();
    const int32_t status = r.status;
    uint32_t sched = 0;
    if (status != PAAM_SET_OK) {
      if (out_wcrt)
        for (uint32_t i = lane; i < r.n_out; i += 32) out_wcrt[r.chain_base + i] = UNS;
    } else {
      const uint32_t nch = r.n_chain, nsub = r.n_sub, nas = r.n_aseg;

      // ---- step 3: Lemma 2, one lane per accelerator segment ----------------------------------------
      // aBase2 already holds A* + LPB + 2 sum_{k<r} W[k][u] (the "+2" of every mu), so
      // G(h) = aBase2 + sum_{k<r} floor((h-1)/T_k) * W[k][u]; starting at G's value for
      // floor(.) = 0 is <= the least fixed point, so the lfp is unchanged (A3).  Products are
      // 64-bit; a product >= 2^32 (high word != 0) is far above every cutoff, and without one the
      // 64-bit sum of <= 31 products cannot overflow.
      for (uint32_t i = lane; i < nas; i += 32) {
        const uint32_t misc = r.aMisc[i];
        const uint32_t rk = misc & 0xffu, u = (misc >> 8) & 0xffu;
        const uint32_t base = r.aBase2[i], cut = r.cCut[rk];
        uint32_t h = base, H = SAT;
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
          if (g == h) { H = h; break; }
          h = g;
        }
        w.H[i] = H;
      }
      __syncwarp();
      // per-segment sums S_c and the blocking term in use
      if (lane < nsub) {
        const uint32_t sg = r.sSeg[lane], a0 = sg & 0xffu, na = (sg >> 8) & 0xffu;
        uint32_t S = 0;
        for (uint32_t i = a0; i < a0 + na; i++) S = sadd(S, w.H[i]);
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

      // ---- step 4: Eq.5 per sub-chain, canonical order ----------------------------------------------
      const bool is_chain = lane < nch;
      const uint32_t Mk = is_chain ? r.cM[lane] : 1u;
      const uint32_t Lk = is_chain ? (r.cMisc[lane] & 31u) : 0u;
      const bool is_sub = lane < nsub;
      const uint32_t hmisc = is_sub ? r.sMisc[lane] : 0u;
      const uint32_t h_rank = hmisc & 31u;
      const bool h_spin = (hmisc >> 16) & 1u;
      const uint32_t h_E = is_sub ? r.sE[lane] : 0u, h_eps = is_sub ? r.sEps[lane] : 0u;
      uint32_t h_R = 0, h_Hs = 0;  // this lane's sub-chain once solved
      for (uint32_t c = 0; c < nsub; c++) {
        const uint32_t cmisc = r.sMisc[c];
        const uint32_t rk = cmisc & 0xffu, umask = (cmisc >> 8) & 0xffu;
        const uint32_t in_hp = (r.sHp[c] >> lane) & 1u, in_hpp = (r.sHpp[c] >> lane) & 1u;
        const bool dep_unsched = (in_hp || (in_hpp && h_spin)) && h_R == SAT;
        uint32_t X = 0;
        if (in_hp) X = sadd(h_E, h_Hs);
        else if (in_hpp) X = sadd(h_E, h_spin ? h_Hs : h_eps);  // spin(Gamma_h)
        uint32_t WU = 0;  // Lemma-3 weight of chain `lane` over the units of c (union of hps, A1)
        if (lane < rk) {
          uint32_t um = umask;
          while (um) {
            const uint32_t u = __ffs(um) - 1;
            um &= um - 1;
            WU = sadd(WU, r.W[lane][u]);
          }
        }
        uint32_t Rc = SAT, Hsc = SAT;
        if (!__any_sync(0xffffffffu, dep_unsched)) {  // A8: an unschedulable dependency poisons c
          const uint32_t BE = sadd(w.Bc[c], r.sE[c]);
          const uint32_t S = w.S[c], base3 = r.sBase3[c], eps = r.sEps[c], cut = r.cCut[rk];
          // start: the first three terms B + E + H*(0), with mu(0) = 1
          const uint32_t A0 = wsum(WU);
          uint32_t R = sadd(BE, sadd(min(S, sadd(base3, A0)), eps));
          uint32_t Hst = 0;
          for (;;) {
            if (R > cut) { R = SAT; break; }
            const uint32_t mk = is_chain ? mu_magic(R, Mk, Lk) : 0u;
            uint32_t a = smul(mk, WU);
            const uint32_t mh = __shfl_sync(0xffffffffu, mk, h_rank);
            uint32_t bsum = smul(mh, X);
            wsum2(a, bsum);
            Hst = sadd(min(S, sadd(base3, a)), eps);
            const uint32_t F = sadd(sadd(BE, Hst), bsum);
            if (F == R) break;
            R = F;
          }
          Rc = R;
          Hsc = (R == SAT) ? SAT : Hst;
        }
        if (lane == c) { h_R = Rc; h_Hs = Hsc; }
      }
      if (is_sub) w.R[lane] = h_R;
      __syncwarp();

      // ---- step 5: end to end and verdict ---------------------------------------------------------
      bool ok = true;
      if (is_chain) {
        uint64_t sum = 0;
        uint32_t cnt = 0;
        bool uns = false;
        for (uint32_t h = 0; h < nsub; h++)
          if ((r.sMisc[h] & 0xffu) == (uint32_t)lane) {
            const uint32_t Rh = w.R[h];
            uns |= (Rh == SAT);
            sum += Rh;
            cnt++;
          }
        const uint64_t Rstar = uns ? UNS : sum + comm * (uint64_t)(cnt - 1);
        const uint32_t cm = r.cMisc[lane];
        if (out_wcrt) out_wcrt[r.chain_base + ((cm >> 16) & 0xffu)] = Rstar;
        const bool critical = ((cm >> 8) & 0xffu) == 0;
        ok = !critical || (Rstar != UNS && Rstar <= (uint64_t)r.cD[lane]);
      }
      sched = __all_sync(0xffffffffu, ok) ? 1u : 0u;
    }
    if (lane == 0) {
      if (out_sched) out_sched[set] = (uint8_t)sched;
      if (out_bins) {
        if (smem_bins) {
          atomicAdd(&sbins[2 * r.bin], 1u);
          if (sched) atomicAdd(&sbins[2 * r.bin + 1], 1u);
        } else {
          atomicAdd((unsigned long long*)&out_bins[2 * r.bin], 1ull);
          if (sched) atomicAdd((unsigned long long*)&out_bins[2 * r.bin + 1], 1ull);
        }
      }
    }
    __syncwarp();
  }
  if (smem_bins) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < 2 * n_bins; i += blockDim.x)
      if (sbins[i]) atomicAdd((unsigned long long*)&out_bins[i], (unsigned long long)sbins[i]);
  }
}

}  // namespace

#ifndef PAAM_WARP_EMU
int launch_analyze(const Record* rec, uint32_t n, uint64_t comm, uint32_t flags, uint32_t n_bins,
                   uint64_t* out_wcrt, uint8_t* out_sched, int64_t* out_bins, cudaStream_t st) {
  if (n == 0) return PAAM_OK;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, analyze_kernel, AW * 32, 0);
  if (per_sm < 1) per_sm = 1;
  const uint32_t need = (n + AW - 1) / AW;
  const uint32_t cap = (uint32_t)sms * (uint32_t)per_sm;
  const uint32_t grid = need < cap ? need : cap;
  analyze_kernel<<<grid, AW * 32, 0, st>>>(rec, n, comm, flags, n_bins, out_wcrt, out_sched, out_bins);
  count_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PAAM_OK : fail_cuda(e, "analyze_kernel launch");
}

#endif  // PAAM_WARP_EMU

}  // namespace paam
