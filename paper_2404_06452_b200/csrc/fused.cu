// fused.cu -- §8(a) steps 2-6 in one kernel: validate + derive (pack) and the WCRT fixed points
// (analyze) of each chain set, one warp per set, the derived per-set record never leaving shared
// memory and registers.  Used by paam_pack_analyze (and paam_sweep).
//
// Step 2 (pack) follows pack.cu phase by phase -- validation in the documented order,
// chain ranks, sub-chains, E, A* = A + 2 kappa_eff (A6),
// rank-based buckets (A5), LP blocking, W regrouping, B_c, hp / hpp / lp
// -- with two differences: sub-chains keep their callback order (the Jacobi solver below
// needs no canonical order), and nothing is written to a global record: every per-sub-chain quantity
// the analysis reads for its own lane (E, B, eps, A2, S_lb, masks, rank, units) stays in the lane's
// registers, and only what other lanes read (the period table, E / eps / H* of interferers, the
// segments for Lemma 2) goes to shared memory, into the space of the segment staging, which is dead by
// then.
// Steps 3-6 are analyze.cu's: Lemma 2 on demand (lazy S_lb), Eq.5 for all sub-chains at
// once by Jacobi iteration from below with mu(R, T) = 2 + floor((R-1)/T) and the floor terms walked in
// period order up to the first T >= R (Eq.4 union form A1, Eq.1), end to end
// (A9), verdict, per-warp bin counters.  DESIGN.md §1, §5.
#include "common.cuh"

namespace paam {

namespace {

// Block shape, measured (tools/fused_variants.sh, 2M config-3 sets): 2 blocks of 16 warps per SM beat 4 of
// 8 (8.02 vs 8.24 ms) and 8 of 4 (8.78 ms); one segment-staging pass per loop trip beats two (-0.05 ms).
#ifndef F_WARPS
#define F_WARPS 16
#endif
constexpr int FW = F_WARPS;  // warps per block
#ifndef F_PF
#define F_PF 1  // L2 prefetch of the next set's segment arrays
#endif
#ifndef F_CHUNK
#define F_CHUNK 8  // sets per work ticket (0: fixed per-warp ranges)
#endif
#ifndef F_SEG_UNROLL
#define F_SEG_UNROLL 1
#endif
constexpr int kFSegUnroll = F_SEG_UNROLL;  // segment-staging passes per loop trip
#ifndef F_CB_UNROLL
#define F_CB_UNROLL 1
#endif
constexpr int kFCbUnroll = F_CB_UNROLL;  // a callback's segments per trip of its walk
constexpr uint32_t FULL = 0xffffffffu;
constexpr uint32_t MAXSEG = 192;
constexpr int F_WARP_BINS = 32;
constexpr uint64_t UNS = PAAM_UNSCHED;

// Per-warp shared memory.  Arrays that die during the derivation share their space with the ones the
// analysis creates later (the unions below), which keeps a warp's share at ~7.4 KB.
struct FSmem {
  // chains by rank
  uint32_t rT[MAXC], rD[MAXC], rCbo[MAXC], rA0[MAXC];
  uint8_t rCls[MAXC], rIdx[MAXC], rNcb[MAXC], rNa[MAXC];
  uint8_t rank_of[MAXC];
  uint32_t cA0[MAXC];
  // callbacks (set-local order)
  uint32_t bE[MAXCB];
  uint8_t bExec[MAXCB], bNa[MAXCB], bA0[MAXCB + 1], bSub[MAXCB];
  union {
    struct {  // first accelerator segment of each callback: dead after the accelerator-segment pass
      uint32_t bFw[MAXCB];
      uint8_t bFa[MAXCB], bFu[MAXCB];
    };
    struct {  // chains by rank / period order (written after that pass)
      uint2 cML[MAXC];      // mu magic (M, L) by rank (Lemma 2)
      uint8_t posOf[MAXC];  // pTab slot (31 - period position) of chain rank k
      uint8_t sPos[MAXS];   // pTab slot of sub-chain h's chain
    };
  };
  // accelerator segments (rank order)
  uint32_t qAstar[MAXA];
  union {
    uint32_t qA[MAXA];  // raw WCET, for WFD only (dead after it)
    struct {
      uint32_t cmp[MAXC];    // LP-blocking scan buffer
      uint32_t sMaxE[MAXS];  // largest callback WCET of each sub-chain (B_c)
    };
  };
  uint8_t qUnit[MAXA], qAcc[MAXA], qCb[MAXA], qRank[MAXA];
  // executors, accelerators
  uint32_t xPrio[MAXX];
  uint8_t xCore[MAXX], xWait[MAXX], xPPrank[MAXX];
  uint32_t aN[4], aUnits[4], aUbase[4], aEps[4], aKeff[4], aServer[4];
  alignas(16) uint32_t W[MAXC][MAXU];  // sum of A* of chain rank k on unit u
  union {
    struct {  // derivation: dead once the sub-chains have their A2 / S_lb and the segments their aBase
      uint32_t maxA[MAXU][MAXC];  // becomes the LP blocking per (unit, rank)
      union {
        uint32_t pre2[MAXU][MAXC];  // 2 sum_{k < rank} W[k][u]
        struct {
          uint64_t wfdU[MAXCB];
          uint8_t wfdOrder[MAXCB], wfdUnit[MAXCB], wfdCb[MAXCB];
        };
      };
    };
    struct {  // analysis
      uint32_t Hs[MAXS];  // H*_h at the current iterate
      uint32_t H[MAXA];   // Lemma-2 value per accelerator segment (rank order)
      unsigned long long sum[MAXC];
      uint32_t uns[MAXC];
    };
  };
  uint8_t sRank[MAXS], sExec[MAXS], sJ0[MAXS];
  union {
    struct {  // the set's segments, staged by coalesced loads; dead after the accelerator-segment pass
      uint32_t gW[MAXSEG];
      uint8_t gMeta[MAXSEG];  // kind | accelerator << 1 | unit << 3 (the values of a valid set fit)
    };
    struct {  // what a lane reads of other lanes / chains
      uint4 pTab[MAXC];  // period order: {T, M, L | rank << 8, W[rank][0] + W[rank][1]} (f_shr: L < 32)
      uint32_t sE[MAXS], sEps[MAXS];
      uint32_t aBase[MAXA];  // Lemma-2 start value A* + LPB + 2 sum_{k<r} W[k][u] of each segment
    };
  };
};

static_assert(offsetof(FSmem, maxA) % 16 == 0 && sizeof(FSmem::maxA) >= MAXC * sizeof(uint2),
              "the chain-rank pass reads (priority, period) pairs from maxA's space as 16-byte vectors");
#ifdef PAAM_EMU_STATS
unsigned long long emu_stats[8];  // debugging statistics of the host emulation (never on the device)
#endif
__constant__ uint32_t kInv16F[33] = {0u, 65537u, 32769u, 21846u, 16385u, 13108u, 10923u, 9363u, 8193u, 7282u, 6554u, 5958u, 5462u, 5042u, 4682u, 4370u, 4097u, 3856u, 3641u, 3450u, 3277u, 3121u, 2979u, 2850u, 2731u, 2622u, 2521u, 2428u, 2341u, 2260u, 2185u, 2115u, 2049u};

__device__ __forceinline__ uint32_t f_scan_sat_incl(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v = sadd(v, y);
  }
  return v;
}
__device__ __forceinline__ uint32_t f_scan_excl(uint32_t v, int lane) {
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  return x - v;
}

__device__ PAAM_COLD void f_wfd_units(FSmem& s, uint32_t nac, uint32_t ncb, uint64_t cstart) {
  #pragma unroll 1
  for (uint32_t a = 0; a < nac; a++) {
    uint32_t ni = 0;
    #pragma unroll 1
    for (uint32_t j = 0; j < ncb; j++) {
      if (!s.bNa[j]) continue;
      const uint32_t c = __popcll(cstart & ((2ull << j) - 1)) - 1, rk = s.rank_of[c];
      const uint32_t q0 = s.rA0[rk] + (s.bA0[j] - s.cA0[c]);
      uint64_t A = 0;
      #pragma unroll 1
      for (uint32_t q = q0; q < q0 + s.bNa[j]; q++) if (s.qAcc[q] == a) A += s.qA[q];
      if (A) { s.wfdU[ni] = (A << 24) / s.rT[rk]; s.wfdCb[ni] = (uint8_t)j; ni++; }
    }
    wfd_place(ni, s.wfdU, s.aUnits[a], s.wfdOrder, s.wfdUnit);
    #pragma unroll 1
    for (uint32_t i = 0; i < ni; i++) {
      const uint32_t j = s.wfdCb[i];
      const uint32_t c = __popcll(cstart & ((2ull << j) - 1)) - 1, rk = s.rank_of[c];
      const uint32_t q0 = s.rA0[rk] + (s.bA0[j] - s.cA0[c]);
      #pragma unroll 1
      for (uint32_t q = q0; q < q0 + s.bNa[j]; q++)
        if (s.qAcc[q] == a) s.qUnit[q] = (uint8_t)(s.aUbase[a] + s.wfdUnit[i]);
    }
  }
}

// Lemma 2 (Eq.3) of accelerator segment q (rank order): lfp of
// G(h) = A* + LPB + 2 sum_{k<r} W[k][u] + sum_{k<r} floor((h-1)/T_k) W[k][u], or SAT (UNB) above the
// cutoff (A4); as analyze.cu's lemma2, with the record fields read from the pack scratch.
__device__ PAAM_COLD uint32_t f_lemma2(const FSmem& s, uint32_t q) {
  const uint32_t rk = s.qRank[q], u = s.qUnit[q];
  const uint32_t base = s.aBase[q];
  const uint32_t cut = min(s.rD[rk], s.rT[rk]);
  uint32_t h = base;
  while (h <= cut) {
    const uint32_t h2 = (h - 1u) << 1;
    uint64_t acc = base;
    uint32_t hi = 0;
#pragma unroll 1
    for (uint32_t k = 0; k < rk; k++) {
      const uint2 ml = s.cML[k];
      acc += (uint64_t)(__umulhi(h2, ml.x) >> ml.y) * s.W[k][u];
      hi |= (uint32_t)(acc >> 32);  // latched high word (f_eval: no wrap before a latch)
    }
    if (hi || acc > cut) break;
    const uint32_t g = (uint32_t)acc;
    if (g == h) return h;
    h = g;
  }
  return SAT;
}

// PAAM_FLAG_BLOCKING_SOUND (reading A10): B_c = max(B, max over the callbacks j of the LP sub-chains
// (lpm) of E_j + sum over j's segments of (H + eps)), from the Lemma-2 values in H.
__device__ PAAM_COLD uint32_t f_sound_blocking(const FSmem& s, uint32_t B, uint32_t lpm, uint32_t n_sub, uint32_t ncb) {
  #pragma unroll 1
  for (uint32_t lp = lpm; lp; lp &= lp - 1) {
    const uint32_t l = __ffs(lp) - 1;
    const uint32_t lrk = s.sRank[l], lj0 = s.sJ0[l];
    const uint32_t lq0 = s.rA0[lrk] + (s.bA0[lj0] - s.cA0[s.rIdx[lrk]]);
    const uint32_t lqn = s.bA0[l + 1 < n_sub ? s.sJ0[l + 1] : ncb] - s.bA0[lj0];
    uint32_t cur_cb = 0xffffffffu, v = 0;
    #pragma unroll 1
    for (uint32_t q = lq0; q < lq0 + lqn; q++) {
      const uint32_t cbid = s.qCb[q];
      if (cbid != cur_cb) {
        if (cur_cb != 0xffffffffu) B = max(B, v);
        cur_cb = cbid;
        v = s.bE[cbid];
      }
      v = sadd(v, sadd(s.H[q], s.aEps[s.qAcc[q]]));
    }
    if (cur_cb != 0xffffffffu) B = max(B, v);
  }
  return B;
}

// Eq.5 evaluation, as analyze.cu's eval_eq5 (see there), reading the shared period table.  nxt: the
// smallest R' > R at which one of the floor terms floor((R' - 1) / T) differs from its value at R (a term
// with q = floor((R - 1) / T) changes at R' = (q + 1) T + 1); below it F and C are those at R, as long
// as the interferers' H* are unchanged.  The loops track nm = nxt - 1 = min (q + 1) T (one multiply-add).
// Overflow: every product is < 2^62 (q <= R - 1 < 2^31, every weight <= SAT), so a 64-bit sum that is
// still < 2^32 cannot wrap in one addition; hi latches the sum's high word after each one, and any
// nonzero latch saturates (every intermediate sum only grows until then): one multiply-add and one OR
// per term.
// Lemma 3's floor terms: W = the weight column of the chain (WSEL false: the table's own
// two-unit sum; true: the sub-chain's units, wsel as in f_eval).
template <bool WSEL>
__device__ __forceinline__ uint64_t f_lemma3(const FSmem& s, uint32_t R, uint32_t h2, uint32_t lmask, uint32_t wsel,
                                             uint32_t umask, uint32_t& hi, uint32_t& nm) {
  uint64_t acc = 0;
  #pragma unroll 1
  for (uint32_t m = lmask; m;) {
    const uint32_t i = f_hibit(m);  // the shortest remaining period (pTab slot 31 - position)
    const uint4 p = s.pTab[i];
    if (p.x >= R) { nm = min(nm, p.x); break; }  // this and every later (longer) period: q = 0
    m ^= 1u << i;
#ifdef PAAM_EMU_STATS
    atomicAdd(&emu_stats[3], 1ull);  // Lemma-3 floor terms
#endif
    const uint32_t q = f_shr(__umulhi(h2, p.y), p.z);
    nm = min(nm, q * p.x + p.x);
    uint32_t wu = p.w;
    if (WSEL) {
      const uint32_t k = p.z >> 8;
      if (wsel <= MAXU) {
        wu = s.W[k][wsel - 1];
      } else {
        wu = 0;
        #pragma unroll 1
        for (uint32_t um = umask; um; um &= um - 1) wu = sadd(wu, s.W[k][__ffs(um) - 1]);
      }
    }
    acc += (uint64_t)q * wu;
    hi |= (uint32_t)(acc >> 32);
  }
  return acc;
}

__device__ __forceinline__ void f_eval(const FSmem& s, uint32_t R, uint32_t lmask, uint32_t wsel, uint32_t umask,
                                       uint32_t A2, uint32_t S, uint32_t eps, uint32_t BE, uint32_t cut, uint32_t xm,
                                       uint32_t depm, uint32_t xs2, uint32_t xTmin, uint32_t& F, uint32_t& nH,
                                       uint32_t& C, uint32_t& nxt) {
  const uint32_t h2 = (R - 1u) << 1;
  uint32_t hi = 0;
  uint32_t nm = 0xfffffffeu;  // (q + 1) T <= 2^32 - 4 for R, T < 2^31
  uint64_t acc = wsel ? f_lemma3<true>(s, R, h2, lmask, wsel, umask, hi, nm)
                      : f_lemma3<false>(s, R, h2, lmask, wsel, umask, hi, nm);
  acc += A2;
  C = (hi || acc > SAT) ? SAT : (uint32_t)acc;
  nH = sadd(min(S, C), eps);
  uint64_t xs = xs2;
  uint32_t xhi = 0;
  #pragma unroll 1
  for (uint32_t m = depm; m;) {  // order-free sums and minima: walked from the highest bit (one FLO)
    const uint32_t h = f_hibit(m);
    m ^= 1u << h;
    const uint32_t X = sadd(s.sE[h], s.Hs[h]);
    const uint4 p = s.pTab[s.sPos[h]];
    const uint32_t q = p.x < R ? (f_shr(__umulhi(h2, p.y), p.z)) : 0u;
    nm = min(nm, q * p.x + p.x);
    xs += (uint64_t)(q + 2u) * X;
    xhi |= (uint32_t)(xs >> 32);
  }
  if (R > xTmin) {
    #pragma unroll 1
    for (uint32_t m = xm & ~depm; m;) {
      const uint32_t h = f_hibit(m);
      m ^= 1u << h;
      const uint4 p = s.pTab[s.sPos[h]];
      if (p.x < R) {
        const uint32_t q = f_shr(__umulhi(h2, p.y), p.z);
        nm = min(nm, q * p.x + p.x);
        xs += (uint64_t)q * sadd(s.sE[h], s.sEps[h]);
        xhi |= (uint32_t)(xs >> 32);
      } else {
        nm = min(nm, p.x);
      }
    }
  } else if (xTmin != 0xffffffffu) {
    nm = min(nm, xTmin);  // every such interferer has T >= R: q = 0 up to its T
  }
  nxt = nm + 1u;
  const uint64_t f = (uint64_t)BE + nH + xs;
  F = (hi || xhi || f > cut) ? SAT : (uint32_t)f;
  if (F == SAT) nH = SAT;
}

#ifndef FUSED_MINB
#define FUSED_MINB 2  // 2 blocks of 16 warps (7 KB of shared memory per warp): 32 warps, 64 registers
#endif
// C32: b carries a compact batch (paam_batch32; common.cuh ld_time)
template <bool C32>
__global__ void __launch_bounds__(FW * 32, FUSED_MINB)
    fused_kernel(paam_batch b, uint32_t* __restrict__ wide_list, uint32_t* __restrict__ wide_count,
                 unsigned int* __restrict__ work_ticket,
                 int32_t* __restrict__ status_out, uint64_t* __restrict__ out_wcrt,
                 uint8_t* __restrict__ out_sched, int64_t* __restrict__ out_bins) {
#ifdef PAAM_WARP_EMU
  __shared__ FSmem smem[FW];
#else
  extern __shared__ __align__(16) unsigned char fsmem_raw[];  // FW * sizeof(FSmem), dynamic (> 48 KB)
  FSmem* smem = reinterpret_cast<FSmem*>(fsmem_raw);
#endif
  __shared__ unsigned int bbins[2 * F_WARP_BINS];  // the block's bin counters (shared-memory atomics)
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  FSmem& s = smem[threadIdx.x >> 5];
  const uint32_t flags = b.flags;
  const bool sound = (flags & PAAM_FLAG_BLOCKING_SOUND) != 0;
  const bool lazy_s = !sound;
  const uint32_t n_bins = b.set_bin ? b.n_bins : 0u;
  const bool blk_bins = out_bins && n_bins && n_bins <= F_WARP_BINS;  // uniform over the grid
  if (blk_bins) {
    for (uint32_t i = threadIdx.x; i < 2 * n_bins; i += FW * 32) bbins[i] = 0;
    __syncthreads();
  }
  const uint64_t comm = b.comm_cost;
  // Dynamic assignment: a warp takes F_CHUNK consecutive sets per ticket (a set's cost varies with its
  // chains and iterates, so fixed per-warp ranges leave the slowest warp ~8% behind the mean); within a
  // chunk each set's start offsets are the previous set's end offsets, whose dependent loads are
  // pipelined one set ahead.
#if F_CHUNK
  #pragma unroll 1
  for (;;) {
  uint32_t tk = 0;
  if (lane == 0) tk = atomicAdd(work_ticket, (unsigned)F_CHUNK);
  const uint32_t lo = __shfl_sync(FULL, tk, 0);
  if (lo >= b.n_sets) break;
  const uint32_t hi = min(lo + (uint32_t)F_CHUNK, b.n_sets);
#else
  const uint32_t nwarps = gridDim.x * FW, wid = blockIdx.x * FW + (threadIdx.x >> 5);
  const uint32_t lo = (uint32_t)((uint64_t)b.n_sets * wid / nwarps);
  const uint32_t hi = (uint32_t)((uint64_t)b.n_sets * (wid + 1) / nwarps);
#endif
  uint32_t c0 = 0, x0 = 0, a0 = 0, cb0 = 0, sg0 = 0;
  uint32_t nc = 0, nx = 0, na_ = 0, ncbo = 0, nsgo = 0;
  if (lo < hi) {
    c0 = b.set_chain_off[lo]; x0 = b.set_exec_off[lo]; a0 = b.set_accel_off[lo];
    nc = b.set_chain_off[lo + 1]; nx = b.set_exec_off[lo + 1]; na_ = b.set_accel_off[lo + 1];
    cb0 = b.chain_cb_off[c0]; ncbo = b.chain_cb_off[nc];
    sg0 = b.cb_seg_off[cb0]; nsgo = b.cb_seg_off[ncbo];
  }
  #pragma unroll 1
  for (uint32_t set = lo; set < hi; set++) {
    const uint32_t c1 = nc, x1 = nx, a1 = na_, cb1 = ncbo, sg1 = nsgo;
    const uint32_t nch = c1 - c0, nex = x1 - x0, nac = a1 - a0;
    const uint32_t ncb = cb1 - cb0;
    const uint32_t nseg = sg1 - sg0;
    const bool more = set + 1 < hi;
#if F_PF && !defined(PAAM_WARP_EMU)
    // L2 prefetch of the next set's segment WCETs (12 lines) and kinds (2 lines): this warp's next set follows
    // in memory, about as large as this one (measured: +0.9%; prefetching every array was slower, 7.52 ms,
    // the extra code costing more than the latency it hid)
    if (more && lane < 14) {
      const uint32_t esz = lane < 12 ? (C32 ? 4u : 8u) : 1u;
      const char* base = lane < 12 ? reinterpret_cast<const char*>(b.seg_wcet) : reinterpret_cast<const char*>(b.seg_kind);
      const uint64_t a0b = (uint64_t)(uintptr_t)base + (uint64_t)sg1 * esz;
      const uint64_t la = (a0b & ~127ull) + 128ull * (lane < 12 ? lane : lane - 12);
      if (la < a0b + (uint64_t)nseg * esz) asm volatile("prefetch.global.L2 [%0];" ::"l"(la));
    }
#endif
    uint32_t pc = c1, px = x1, pa = a1, pcb = cb1, psg = sg1;
    if (more) { pc = b.set_chain_off[set + 2]; px = b.set_exec_off[set + 2]; pa = b.set_accel_off[set + 2]; }
    bool st2 = !more, st3 = !more;
    int st = PAAM_SET_OK;
    const uint32_t bin = b.set_bin ? b.set_bin[set] : 0u;
    const bool bin_ok = n_bins && bin < n_bins;
    if (nch > MAXC || ncb > MAXCB || nseg > MAXSEG || nex > MAXX || nac > 4 || (b.set_bin && bin >= b.n_bins))
      st = PAAM_SET_ERANGE;
    uint32_t n_aseg = 0, n_sub = 0, n_unit = 0;
    uint64_t runstart = 0, cstart = 0;
    uint32_t T = 0, D = 0, prio = 0, cls = 0, cbo = 0, cbn = 0, rank = 0, ppos = 0;  // lane = chain index
    if (st == PAAM_SET_OK) {
      // ---- load + validate (as pack.cu) ---------------------------------------------------------------
      bool erange = false, edang = false, eaccel = false, eshape = false, edup = false, edl = false, ecore = false;
      bool wide = false;  // a time in [2^31 - 1, 2^48) ns: the set goes to the u64 path
      if (lane < (int)nch) {
        const uint64_t T64 = ld_time<C32>(b.chain_T, c0 + lane), D64 = ld_time<C32>(b.chain_D, c0 + lane);
        erange |= (T64 == 0 || T64 >= LIMW || D64 >= LIMW);
        wide |= (T64 >= LIM || D64 >= LIM);  // exact only on the u64 path (wide.cu)
        T = (uint32_t)min(T64, (uint64_t)SAT);
        D = (uint32_t)min(D64, (uint64_t)SAT);
        prio = b.chain_prio[c0 + lane];
        cls = b.chain_class[c0 + lane];
        cbo = b.chain_cb_off[c0 + lane] - cb0;
        cbn = b.chain_cb_off[c0 + lane + 1] - cb0 - cbo;
        edang |= (cbn == 0) || (cbo > ncb) || (cbn > ncb - cbo);
        eshape |= (cls > 1);
        edl |= (D == 0 || (cls == 0 && D > T));
      }
      if (lane < (int)nac) {
        const uint32_t n = b.accel_buckets[a0 + lane], u = b.accel_units[a0 + lane];
        const uint64_t e = ld_time<C32>(b.accel_eps, a0 + lane), kp = ld_time<C32>(b.accel_kappa, a0 + lane);
        erange |= (n < 1 || n > 32 || u < 1 || u > 8 || e >= LIMW || kp >= LIMW);
        wide |= (e >= LIM || kp >= LIM);
        s.aN[lane] = n;
        s.aUnits[lane] = u;
        s.aEps[lane] = (uint32_t)min(e, (uint64_t)SAT);
        s.aKeff[lane] = n > 1 ? (uint32_t)min(kp, (uint64_t)SAT) : 0u;  // A6
        s.aServer[lane] = b.accel_server_core[a0 + lane];
      }
      uint32_t xcore = 0xffffffffu, xprio = 0;
      if (lane < (int)nex) {
        xcore = b.exec_core[x0 + lane];
        xprio = b.exec_prio[x0 + lane];
        const uint32_t w = b.exec_wait[x0 + lane];
        eshape |= (w > 1);
        s.xCore[lane] = (uint8_t)xcore;
        s.xPrio[lane] = xprio;
        s.xWait[lane] = (uint8_t)w;
      }
      __syncwarp();
      uint32_t units_pack, servers_pack;  // byte a: the units / server core of accelerator a (a < nac <= 4)
      {
        const uint32_t u = lane < (int)nac ? s.aUnits[lane] : 0u;
        const uint32_t ub = f_scan_excl(u, lane);
        if (lane < (int)nac) s.aUbase[lane] = ub;
        n_unit = __reduce_add_sync(FULL, u);
        units_pack = __reduce_or_sync(FULL, lane < 4 ? u << (8 * lane) : 0u);
        const uint32_t sv = lane < (int)nac ? s.aServer[lane] : 0u;
        servers_pack = __reduce_or_sync(FULL, lane < 4 ? sv << (8 * lane) : 0u);
      }
      const uint64_t cstart_bit = (lane < (int)nch && cbo < 64) ? (1ull << cbo) : 0ull;
      cstart = ((uint64_t)__reduce_or_sync(FULL, (uint32_t)(cstart_bit >> 32)) << 32) |
               __reduce_or_sync(FULL, (uint32_t)cstart_bit);
      __syncwarp();
      // ---- segments: lane per segment, staged with their per-segment validation
      #pragma unroll kFSegUnroll
      for (uint32_t i = lane; i < nseg; i += 32) {
        const uint64_t w = ld_time<C32>(b.seg_wcet, sg0 + i);
        uint32_t kind, a, u;
        ld_seg<C32>(b, sg0 + i, kind, a, u);
        erange |= (w >= LIMW);
        wide |= (w >= LIM);
        eshape |= (kind > 1) || (w == 0);
        const bool isacc = kind == 1u;
        eaccel |= isacc && a >= nac;
        edang |= isacc && a < nac && u >= ((units_pack >> ((a & 3u) << 3)) & 0xffu);
        s.gW[i] = (uint32_t)w;  // exact unless the set is ERANGE or wide (its derived values are never used)
        // kind bit: an ACCEL segment (an undefined kind is ESHAPE, counted as no accelerator segment); the
        // accelerator / unit bits are read only for valid sets, where they fit
        s.gMeta[i] = (uint8_t)((kind == 1u ? 1u : 0u) | (a << 1) | (u << 3));
      }
      __syncwarp();
      // ---- callbacks: lane per callback, walking its staged segments
      uint32_t prev_exec = 0xffffffffu;
      bool malformed = false;
      #pragma unroll 1
      for (uint32_t pass = 0; pass * 32 < ncb; pass++) {
        const uint32_t j = pass * 32 + lane;
        uint32_t exec = 0xffffffffu, E = 0, na = 0, fa = 0, fu = 0, fw = 0;
        if (j < ncb) {
          exec = ld_cb_exec<C32>(b, cb0 + j);
          uint32_t so = b.cb_seg_off[cb0 + j], se = b.cb_seg_off[cb0 + j + 1];
          edang |= (se == so) || (exec >= nex);
          if (so < sg0 || se < so || se > sg1) { malformed = true; so = se = sg0; }
          uint32_t prev_kind = 0xffffffffu;
          #pragma unroll kFCbUnroll
          for (uint32_t k = so - sg0; k < se - sg0; k++) {
            const uint32_t meta = s.gMeta[k], kind = meta & 1u, w = s.gW[k];
            eshape |= (kind == prev_kind);
            prev_kind = kind;
            if (kind == 0) {
              E = sadd(E, w);
            } else {
              if (na == 0) { fa = (meta >> 1) & 3u; fu = meta >> 3; fw = w; }
              na++;
            }
          }
          // na <= nseg <= MAXSEG < 256, fa < 4, fu < 32; an executor >= 256 is EDANGLING, which precedes
          // the A13 rule that reads bExec
          s.bExec[j] = (uint8_t)exec;
          s.bE[j] = E;
          s.bNa[j] = (uint8_t)na;
          s.bFa[j] = (uint8_t)fa;
          s.bFu[j] = (uint8_t)fu;
          s.bFw[j] = fw;
        }
        uint32_t pe = __shfl_up_sync(FULL, exec, 1);
        if (lane == 0) pe = prev_exec;
        prev_exec = __shfl_sync(FULL, exec, 31);
        const bool first_of_chain = (j < ncb) && ((cstart >> j) & 1ull);
        const bool start = (j < ncb) && (first_of_chain || exec != pe);
        const uint32_t bal = __ballot_sync(FULL, start);
        runstart |= (uint64_t)bal << (pass * 32);
        n_aseg += __reduce_add_sync(FULL, na);
      }
      n_sub = __popcll(runstart);
      __syncwarp();
      if (runstart & ~cstart)  // some chain changes executor: A13 (no return to an executor it left)
      #pragma unroll 1
      for (uint32_t j = lane; j < ncb; j += 32) {  // A13
        if (((runstart >> j) & 1ull) && !((cstart >> j) & 1ull)) {
          const uint32_t first = 63 - __clzll(cstart & ((2ull << j) - 1));
          #pragma unroll 1
          for (uint32_t i = first; i + 1 < j; i++) eshape |= (s.bExec[i] == s.bExec[j]);
        }
      }
      // ---- ranks
      {  // chain ranks and period positions (ascending T; equal periods by chain index), one pass
        uint32_t rk = 0, below = 0;
        const uint32_t Tme = lane < (int)nch ? T : 0xffffffffu;
        // (priority, period) of every chain through maxA's space (dead until the per-chain pass of the
        // derivation; 16-byte aligned after W): one 16-byte broadcast load per two chains instead of four
        // shuffles
        uint2* const pt = reinterpret_cast<uint2*>(&s.maxA[0][0]);
        pt[lane] = uint2{prio, Tme};
        __syncwarp();
        uint32_t d = 0;
        #pragma unroll 1
        for (; d + 1 < nch; d += 2) {
          const uint4 v = reinterpret_cast<const uint4*>(pt)[d >> 1];  // chains d, d + 1
          rk += (uint32_t)(v.x > prio) + (uint32_t)(v.z > prio);
          below += (uint32_t)(v.y < Tme) + (uint32_t)(v.w < Tme);
        }
        if (d < nch) {
          const uint2 v = pt[d];
          rk += (v.x > prio);
          below += (v.y < Tme);
        }
        __syncwarp();  // pt is overwritten by the derivation
        rank = rk;
        ppos = below + __popc(__match_any_sync(FULL, Tme) & lt);
        const uint32_t valid = nch >= 32 ? FULL : (1u << nch) - 1u;
        const uint32_t same = __match_any_sync(FULL, prio) & valid & ~(1u << lane);
        edup |= (lane < (int)nch && same != 0);
      }
      {  // executors: duplicate (core, priority), process-priority rank, R1
        const uint32_t same_core = __match_any_sync(FULL, xcore) & ~(1u << lane);
        uint32_t pr = 0, m = lane < (int)nex ? same_core : 0u;
        while (m) {
          const uint32_t y = f_hibit(m);
          m ^= 1u << y;
          const uint32_t py = s.xPrio[y];
          edup |= (py == xprio);
          pr += (py > xprio);
        }
        if (lane < (int)nex) {
          s.xPPrank[lane] = (uint8_t)pr;
          const uint32_t vmask = nac >= 4 ? FULL : (1u << (8 * nac)) - 1u;  // the bytes of accelerators 0..nac-1
          ecore |= (__vcmpeq4(servers_pack, xcore * 0x01010101u) & vmask) != 0u;
        }
      }
      erange |= (n_aseg > MAXA) || (n_unit > MAXU);
      {  // the rules in order (include/paam.h): one OR-reduction, the first failing rule decides
        const uint32_t mine = (malformed ? 1u : 0u) | (erange ? 2u : 0u) | (wide ? 4u : 0u) | (edang ? 8u : 0u) |
                              (eaccel ? 16u : 0u) | (eshape ? 32u : 0u) | (edup ? 128u : 0u) | (edl ? 256u : 0u) |
                              (ecore ? 512u : 0u);
        const uint32_t err = __reduce_or_sync(FULL, mine) | (n_sub > MAXS ? 64u : 0u);
        if (err) {
          const uint32_t i = __ffs(err) - 1;  // nibble i: the status of rule i (rule 2 = the u64 handover)
          st = i == 2 ? REC_STATUS_WIDE : (int)((0x7651432012ull >> (4 * i)) & 0xfu);
        }
      }
    }
    if (!st2) { pcb = b.chain_cb_off[pc]; st2 = true; }
    if (st == REC_STATUS_WIDE) {  // every output of a handed-over set is wide_kernel's
      if (lane == 0) wide_list[atomicAdd(wide_count, 1u)] = set;
      if (!st3) psg = b.cb_seg_off[pcb];
      __syncwarp();
      c0 = c1; x0 = x1; a0 = a1; cb0 = cb1; sg0 = sg1;
      nc = pc; nx = px; na_ = pa; ncbo = pcb; nsgo = psg;
      continue;
    }
    if (lane == 0 && status_out) status_out[set] = st;
    uint32_t sched = 0;
    if (st != PAAM_SET_OK) {
      if (out_wcrt)
        #pragma unroll 1
        for (uint32_t i = lane; i < nch; i += 32) out_wcrt[c0 + i] = UNS;
      if (!st3) psg = b.cb_seg_off[pcb];
    } else {
      // ---- derivation (valid set) ======================================================================
      const bool is_chain = lane < (int)nch;
      if (is_chain) {
        s.rank_of[lane] = (uint8_t)rank;
        s.rT[rank] = T;
        s.rD[rank] = D;
        s.rCls[rank] = (uint8_t)cls;
        s.rIdx[rank] = (uint8_t)lane;
        s.rCbo[rank] = cbo;
        s.rNcb[rank] = (uint8_t)cbn;
      }
      {
        uint32_t carry = 0;
        #pragma unroll 1
        for (uint32_t pass = 0; pass * 32 < ncb; pass++) {
          const uint32_t j = pass * 32 + lane;
          const uint32_t na = j < ncb ? s.bNa[j] : 0u;
          const uint32_t ex = f_scan_excl(na, lane);
          if (j < ncb) s.bA0[j] = (uint8_t)(carry + ex);
          carry += __reduce_add_sync(FULL, na);
        }
        if (lane == 0) s.bA0[ncb] = (uint8_t)carry;
      }
      __syncwarp();
      {
        const uint32_t k = lane;
        uint32_t na = 0;
        if (k < nch) {
          const uint32_t o = s.rCbo[k];
          na = s.bA0[o + s.rNcb[k]] - s.bA0[o];
          s.cA0[s.rIdx[k]] = s.bA0[o];
        }
        const uint32_t f = f_scan_excl(na, lane);
        if (k < nch) { s.rA0[k] = f; s.rNa[k] = (uint8_t)na; }
      }
      #pragma unroll 1
      for (uint32_t j = lane; j < ncb; j += 32) {
        const uint32_t sid = __popcll(runstart & ((2ull << j) - 1)) - 1;
        s.bSub[j] = (uint8_t)sid;
        if ((runstart >> j) & 1ull) s.sJ0[sid] = (uint8_t)j;
      }
      __syncwarp();
      // ---- accelerator segments: A*, unit, rank, in rank order
      #pragma unroll 1
      for (uint32_t pass = 0; pass * 32 < ncb; pass++) {
        const uint32_t j = pass * 32 + lane;
        if (j < ncb && s.bNa[j]) {
          const uint32_t c = __popcll(cstart & ((2ull << j) - 1)) - 1;
          const uint32_t rk = s.rank_of[c];
          uint32_t q = s.rA0[rk] + (s.bA0[j] - s.cA0[c]);
          auto put = [&](uint32_t a, uint32_t u, uint32_t w) {
            s.qAstar[q] = sadd(w, sadd(s.aKeff[a], s.aKeff[a]));  // A* = A + 2 kappa_eff
            s.qA[q] = w;
            s.qUnit[q] = (uint8_t)(s.aUbase[a] + u);
            s.qAcc[q] = (uint8_t)a;
            s.qCb[q] = (uint8_t)j;
            s.qRank[q] = (uint8_t)rk;
            q++;
          };
          if (s.bNa[j] == 1) {
            put(s.bFa[j], s.bFu[j], s.bFw[j]);
          } else {
            const uint32_t so = b.cb_seg_off[cb0 + j] - sg0, se = b.cb_seg_off[cb0 + j + 1] - sg0;
            #pragma unroll 1
            for (uint32_t k = so; k < se; k++)
              if (s.gMeta[k] & 1u) put((s.gMeta[k] >> 1) & 3u, s.gMeta[k] >> 3, s.gW[k]);
          }
        }
      }
      __syncwarp();  // the staged segments are dead from here on (their space becomes analysis state)
      if ((flags & PAAM_FLAG_WFD_UNITS) && lane == 0) f_wfd_units(s, nac, ncb, cstart);
      __syncwarp();
      // ---- per chain (lane = rank): W[k][u], max A*[u][k], accelerator use mask
      uint32_t use = 0;
      #pragma unroll 1
      for (uint32_t u = 0; u < n_unit; u++) s.maxA[u][lane] = 0;
      if (is_chain) {
        const uint32_t k = lane;
        reinterpret_cast<uint4*>(s.W[k])[0] = uint4{0u, 0u, 0u, 0u};
        reinterpret_cast<uint4*>(s.W[k])[1] = uint4{0u, 0u, 0u, 0u};
        #pragma unroll 1
        for (uint32_t q = s.rA0[k]; q < s.rA0[k] + s.rNa[k]; q++) {
          const uint32_t u = s.qUnit[q], a = s.qAstar[q];
          use |= 1u << s.qAcc[q];
          s.maxA[u][k] = max(s.maxA[u][k], a);
          s.W[k][u] = sadd(s.W[k][u], a);
        }
      }
      __syncwarp();
      if (!st3) { psg = b.cb_seg_off[pcb]; st3 = true; }
      // ---- buckets (A5) and LP blocking per (unit, rank)
      #pragma unroll 1
      for (uint32_t a = 0; a < nac; a++) {
        const uint32_t U = __ballot_sync(FULL, (use >> a) & 1u);
        const uint32_t ma = __popc(U), n = s.aN[a];
        const uint32_t g = ma ? ((ma + n - 1) * kInv16F[n]) >> 16 : 1u;
        const uint32_t ginv = kInv16F[g];
        const bool user = (U >> lane) & 1u;
        const uint32_t p = __popc(U & lt);
        const uint32_t blk_end = min(((((uint32_t)lane * ginv) >> 16) + 1) * g, ma);
        #pragma unroll 1
        for (uint32_t u = s.aUbase[a]; u < s.aUbase[a] + s.aUnits[a]; u++) {
          if (user) s.cmp[p] = s.maxA[u][lane];
          __syncwarp();
          uint32_t v = (uint32_t)lane < ma ? s.cmp[lane] : 0u;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_down_sync(FULL, v, o);
            if ((uint32_t)lane + o < blk_end) v = max(v, y);
          }
          const uint32_t nxt = __shfl_down_sync(FULL, v, 1);
          const uint32_t ex = ((uint32_t)lane + 1 < blk_end) ? nxt : 0u;
          __syncwarp();
          if ((uint32_t)lane < ma) s.cmp[lane] = ex;
          __syncwarp();
          s.maxA[u][lane] = user ? s.cmp[p] : 0u;
          __syncwarp();
        }
      }
      #pragma unroll 1
      for (uint32_t u = 0; u < n_unit; u++) {
        const uint32_t w = is_chain ? s.W[lane][u] : 0u;
        const uint32_t incl = f_scan_sat_incl(w, lane);
        const uint32_t prev = __shfl_up_sync(FULL, incl, 1);
        const uint32_t ex = lane == 0 ? 0u : prev;
        s.pre2[u][lane] = sadd(ex, ex);
      }
      // ---- chains: mu constants, period table (lane = chain index; ppos from the rank pass)
      {
        uint32_t M = 0, L = 0;
        if (is_chain) {
          make_magic(T, &M, &L);
          s.cML[rank] = uint2{M, L};
          // slot 31 - ppos: the shortest period is a mask's highest bit (f_lemma3 walks down from it)
          s.pTab[31u - ppos] = uint4{T, M, L | (rank << 8), sadd(s.W[rank][0], s.W[rank][1])};
          s.posOf[rank] = (uint8_t)(31u - ppos);
        }
      }
      __syncwarp();

      // ---- sub-chains (lane = sub-chain id, callback order): everything stays in registers -----------
      const bool act = lane < (int)n_sub;
      uint32_t s_exec = 0, rk = 0, s_j0 = 0, s_nj = 0, E = 0;
      if (act) {
        s_j0 = s.sJ0[lane];
        s_nj = ((uint32_t)lane + 1 < n_sub ? s.sJ0[lane + 1] : ncb) - s_j0;
        const uint32_t c = __popcll(cstart & ((2ull << s_j0) - 1)) - 1;
        s_exec = s.bExec[s_j0];
        rk = s.rank_of[c];
        uint32_t mE = 0;
        #pragma unroll 1
        for (uint32_t j = s_j0; j < s_j0 + s_nj; j++) { mE = max(mE, s.bE[j]); E = sadd(E, s.bE[j]); }
        s.sMaxE[lane] = mE;
        s.sRank[lane] = (uint8_t)rk;
        s.sExec[lane] = (uint8_t)s_exec;
      }
      __syncwarp();
      const uint32_t same_exec = __match_any_sync(FULL, act ? s_exec : 0x100u + lane);
      const uint32_t my_core = act ? s.xCore[s_exec] : 0x100u + lane;
      const uint32_t same_core = __match_any_sync(FULL, my_core);
      uint32_t qa = 0, qn = 0, eps = 0, umask = 0, slb = 0, A2 = 0, hpm = 0, lpm = 0, hppm = 0, B = 0;
      bool spin = false;
      if (act) {
        const uint32_t c = s.rIdx[rk];
        qa = s.rA0[rk] + (s.bA0[s_j0] - s.cA0[c]);
        qn = s.bA0[s_j0 + s_nj] - s.bA0[s_j0];
        uint32_t base3 = 0;
        #pragma unroll 1
        for (uint32_t q = qa; q < qa + qn; q++) {
          const uint32_t u = s.qUnit[q];
          eps = sadd(eps, s.aEps[s.qAcc[q]]);
          const uint32_t bq = sadd(s.qAstar[q], s.maxA[u][rk]);
          base3 = sadd(base3, bq);
          const uint32_t ab = sadd(bq, s.pre2[u][rk]);  // the segment's Lemma-2 start value
          s.aBase[q] = ab;
          slb = sadd(slb, ab);
          umask |= 1u << u;
        }
        A2 = base3;
        #pragma unroll 1
        for (uint32_t um = umask; um;) {
          const uint32_t u = f_hibit(um);
          um ^= 1u << u;
          A2 = sadd(A2, s.pre2[u][rk]);
        }
        uint32_t m = same_exec & ~(1u << lane);
        while (m) {
          const uint32_t l = f_hibit(m);
          m ^= 1u << l;
          if (s.sRank[l] < rk) hpm |= 1u << l;
          else { lpm |= 1u << l; B = max(B, s.sMaxE[l]); }  // B_c
        }
        m = same_core & ~same_exec;
        const uint32_t mypp = s.xPPrank[s_exec];
        while (m) {
          const uint32_t l = f_hibit(m);
          m ^= 1u << l;
          if (s.xPPrank[s.sExec[l]] < mypp) hppm |= 1u << l;
        }
        spin = s.xWait[s_exec] == 1;
        s.sE[lane] = E;
        s.sEps[lane] = eps;
        s.sPos[lane] = s.posOf[rk];
      }
      // The set's CSR offsets and the prefetched next ones are not read again until step 5 / the end of the
      // set: they rest in the dead LP-blocking scan buffer, which frees their registers for the solve.
      uint32_t* const park = s.cmp;
      if (lane == 0) {
        park[0] = c0; park[1] = nc; park[2] = nx; park[3] = na_; park[4] = ncbo; park[5] = nsgo;
        park[6] = pc; park[7] = px; park[8] = pa; park[9] = pcb; park[10] = psg;
      }
      // ---- step 3: Lemma 2 (sound blocking: all segments up front) ------------------------------------
      __syncwarp();  // aBase / sE / sEps complete; maxA and pre2 are dead (H, Hs, sum, uns reuse them)
      if (!lazy_s)
        #pragma unroll 1
        for (uint32_t q = lane; q < n_aseg; q += 32) s.H[q] = f_lemma2(s, q);
      __syncwarp();
      uint32_t S = slb, cut = 0, BE = 0;
      if (act) {
        cut = min(s.rD[rk], s.rT[rk]);
        if (!lazy_s) {
          S = 0;
          #pragma unroll 1
          for (uint32_t q = qa; q < qa + qn; q++) S = sadd(S, s.H[q]);
          B = f_sound_blocking(s, B, lpm, n_sub, ncb);  // A10: an LP callback also holds its accelerator wait
        }
        BE = sadd(B, E);
      }
      const uint32_t spin_mask = __ballot_sync(FULL, act && spin);
      const uint32_t depm = hpm | (hppm & spin_mask);
      const uint32_t xm = hpm | hppm;
      const bool critical = act && s.rCls[rk] == 0;
      bool sexact = !lazy_s;
      // ---- lmask: pTab slots of the chains of rank < rk (exclusive OR-scan over ranks)
      uint32_t pb = is_chain ? (1u << s.posOf[lane]) : 0u;  // lane = rank
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, pb, o);
        if (lane >= o) pb |= y;
      }
      uint32_t pex = __shfl_up_sync(FULL, pb, 1);
      if (lane == 0) pex = 0;
      const uint32_t lm_rk = __shfl_sync(FULL, pex, rk);
      const uint32_t lmask = act ? lm_rk : 0u;
      const uint32_t wsel = (n_unit <= 2 && umask == (1u << n_unit) - 1u) ? 0u
                            : __popc(umask) == 1 ? (uint32_t)__ffs(umask) : (uint32_t)MAXU + 1u;
      uint32_t xs2 = 0, xTmin = 0xffffffffu;
      __syncwarp();
      if (act) {
        #pragma unroll 1
        for (uint32_t m = xm & ~depm; m;) {
          const uint32_t h = f_hibit(m);
          m ^= 1u << h;
          xs2 = sadd(xs2, sadd(s.sE[h], s.sEps[h]));
          xTmin = min(xTmin, s.pTab[s.sPos[h]].x);
        }
        xs2 = sadd(xs2, xs2);
      }

      // ---- step 4: Eq.5 for all sub-chains at once (Jacobi from below, see analyze.cu) -----------------
      uint32_t R = act ? 1u : SAT, Hst = act ? sadd(min(S, A2), eps) : SAT, C = A2;
      if (act) s.Hs[lane] = Hst;
      __syncwarp();
      bool dirty = act;
      bool miss = false;
#ifdef PAAM_EMU_STATS
      if (lane == 0) emu_stats[0]++;  // sets
#endif
      #pragma unroll 1
      for (;;) {
        uint32_t F = R, nH = Hst, nxt = 0u;
#ifdef PAAM_EMU_STATS
        if (lane == 0) emu_stats[1]++;  // warp iterates
        if (dirty) atomicAdd(&emu_stats[2], 1ull);  // lane evaluations
#endif
        if (dirty) {
          // one (checked) copy of the evaluation: the unchecked one for periods >= 64 ns saved one
          // instruction per floor term but doubled the loop's code (instruction-cache stalls)
          f_eval(s, R, lmask, wsel, umask, A2, S, eps, BE, cut, xm, depm, xs2, xTmin, F, nH, C, nxt);
        }
        const bool chg = dirty && (F != R || nH != Hst);
        const uint32_t cm = __ballot_sync(FULL, chg);
        if (!cm) {
          const bool need = act && !sexact && R != SAT && C > S;
          const uint32_t needm = __ballot_sync(FULL, need);
          if (!needm) break;
          #pragma unroll 1
          for (uint32_t q = lane; q < n_aseg; q += 32)
            if ((needm >> s.bSub[s.qCb[q]]) & 1u) s.H[q] = f_lemma2(s, q);
          __syncwarp();
          if (need) {
            uint32_t Sx = 0;
            #pragma unroll 1
            for (uint32_t q = qa; q < qa + qn; q++) Sx = sadd(Sx, s.H[q]);
            S = Sx;
            sexact = true;
          }
          dirty = need;
          continue;
        }
        __syncwarp();
        if (chg) {
          R = F;
          Hst = nH;
          s.Hs[lane] = nH;
        }
        __syncwarp();
        // A lane that moved to F below nxt has F(F) = F unless an interferer's H* changed: the floor terms,
        // hence C and H*, are those of the evaluation just done, so it is not re-evaluated for itself.
        dirty = act && R != SAT && ((chg && R >= nxt) || (depm & cm) != 0u);
        if (flags & PAAM_FLAG_VERDICT_ONLY) {
          if (__any_sync(FULL, critical && R == SAT)) { miss = true; break; }
        }
      }

      // ---- step 5: end to end and verdict ------------------------------------------------------------
      if (!miss) {
        if (is_chain) { s.sum[lane] = 0; s.uns[lane] = 0; }
        __syncwarp();
        if (act) {  // per chain: sum of R, and (sub-chains | unschedulable ones << 16)
          atomicAdd(&s.uns[rk], R == SAT ? 0x10001u : 1u);
          if (R != SAT) atomicAdd(&s.sum[rk], (unsigned long long)R);
        }
        __syncwarp();
        bool ok = true;
        if (is_chain) {
          const uint32_t k = lane;
          const uint32_t u = s.uns[k], nsc = u & 0xffffu;  // nsc: the chain's executor crossings + 1 (A9)
          const uint64_t Rstar = (u >> 16) ? UNS : s.sum[k] + comm * (uint64_t)(nsc - 1);
          if (out_wcrt) out_wcrt[park[0] + s.rIdx[k]] = Rstar;
          const bool crit = s.rCls[k] == 0;
          ok = !crit || (Rstar != UNS && Rstar <= (uint64_t)s.rD[k]);
        }
        sched = __all_sync(FULL, ok) ? 1u : 0u;
      }
      __syncwarp();
      c0 = park[0]; nc = park[1]; nx = park[2]; na_ = park[3]; ncbo = park[4]; nsgo = park[5];
      pc = park[6]; px = park[7]; pa = park[8]; pcb = park[9]; psg = park[10];
    }
    if (lane == 0) {
      if (out_sched) out_sched[set] = (uint8_t)sched;
      if (out_bins && bin_ok) {
        if (blk_bins) {
          atomicAdd(&bbins[2 * bin], 1u);
          if (sched) atomicAdd(&bbins[2 * bin + 1], 1u);
        } else {
          atomicAdd((unsigned long long*)&out_bins[2 * bin], 1ull);
          if (sched) atomicAdd((unsigned long long*)&out_bins[2 * bin + 1], 1ull);
        }
      }
    }
    __syncwarp();
    c0 = nc; x0 = nx; a0 = na_; cb0 = ncbo; sg0 = nsgo;
    nc = pc; nx = px; na_ = pa; ncbo = pcb; nsgo = psg;
  }
#if F_CHUNK
  }
#endif
  if (blk_bins) {  // every warp of the block is done: one global atomic per non-zero counter
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < 2 * n_bins; i += FW * 32)
      if (bbins[i]) atomicAdd((unsigned long long*)&out_bins[i], (unsigned long long)bbins[i]);
  }
}

}  // namespace

#ifndef PAAM_WARP_EMU
namespace {
template <bool C32>
int launch_fused_t(const paam_batch* b, uint32_t* wide_list, uint32_t* wide_count, int32_t* status, uint64_t* out_wcrt,
                   uint8_t* out_sched, int64_t* out_bins, cudaStream_t st) {
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  constexpr size_t SMEM = FW * sizeof(FSmem);
  static const cudaError_t attr =
      cudaFuncSetAttribute(fused_kernel<C32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
  if (attr != cudaSuccess) return fail_cuda(attr, "fused_kernel: shared memory attribute");
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_kernel<C32>, FW * 32, SMEM);
  if (per_sm < 1) per_sm = 1;
  const uint32_t need = (b->n_sets + FW - 1) / FW;
  const uint32_t cap = (uint32_t)sms * (uint32_t)per_sm;
  const uint32_t grid = need < cap ? need : cap;
  // the work ticket is the counter after wide_count (the callers zero both)
  fused_kernel<C32><<<grid, FW * 32, SMEM, st>>>(*b, wide_list, wide_count, wide_count + 1, status, out_wcrt, out_sched,
                                                  out_bins);
  count_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PAAM_OK : fail_cuda(e, "fused_kernel launch");
}
}  // namespace

int launch_fused(const paam_batch* b, uint32_t* wide_list, uint32_t* wide_count, int32_t* status, uint64_t* out_wcrt,
                 uint8_t* out_sched, int64_t* out_bins, cudaStream_t st, bool c32) {
  if (b->n_sets == 0) return PAAM_OK;
  return c32 ? launch_fused_t<true>(b, wide_list, wide_count, status, out_wcrt, out_sched, out_bins, st)
             : launch_fused_t<false>(b, wide_list, wide_count, status, out_wcrt, out_sched, out_bins, st);
}
#endif  // PAAM_WARP_EMU

}  // namespace paam
