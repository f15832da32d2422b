// pack.cu -- §8(a) step 2: validate each raw set and derive its analysis record (one warp per set).
//
// Reads the paper's system model from the flat CSR batch, checks the validation rules in
// the order documented in include/paam.h, and derives everything the fixed-point kernels
// need, so that they touch only integer arrays in shared memory:
//   * chain ranks (rank 0 = highest unique priority) and per-period mu constants (Eq.2);
//   * sub-chains = maximal runs of consecutive callbacks on one executor;
//   * E_i per callback, calligraphic E_c per sub-chain;
//   * A* = A + 2 kappa_eff with kappa_eff = 0 on a one-bucket accelerator (A6);
//   * the bucket of every (chain, accelerator): rank-based groups of ceil(m_a / n) (A5);
//   * LP blocking per segment: max A* of lower-priority segments in the same bucket and unit;
//   * W[k][u] = sum of A* of chain k on unit u (exact regrouping of the hps sums of Eq.3 / Eq.4);
//   * B_c as written, hp / hpp / lp sets as bit masks;
//   * the canonical analysis order: per core, process priority desc, then chain priority desc (A7).
// Mapping: lane = chain (ranked), lane = callback (two passes of 32), lane = sub-chain; relations are
// 32/64-bit masks built with ballot / match / warp reductions; the bucket LP-blocking maximum is a
// segmented suffix-max scan over the users of each unit (buckets are aligned blocks in rank order).
// Memory: sets are assigned to warps in contiguous blocks, so each set's CSR start offsets are the
// previous set's end offsets (its dependent offset loads are software-pipelined one set ahead); a
// set's segments are staged into shared memory with coalesced loads, into scratch that is dead until
// the W / WFD phase, and no integer divide runs per set (bucket sizes come from a reciprocal table).
#include "common.cuh"

namespace paam {

namespace {

#ifndef PACK_WARPS
#define PACK_WARPS 4
#endif
constexpr int WARPS = PACK_WARPS;
#ifndef PACK_SEG_UNROLL
#define PACK_SEG_UNROLL 1
#endif
constexpr int kSegUnroll = PACK_SEG_UNROLL;  // segment loop of the callback pass (measured: 1 < 3)
#ifndef PACK_STAGE_UNROLL
#define PACK_STAGE_UNROLL 2
#endif
constexpr int kStageUnroll = PACK_STAGE_UNROLL;  // coalesced segment staging loop (measured: 2 < 3 < 1 < 6)
constexpr uint32_t FULL = 0xffffffffu;
constexpr uint32_t MAXSEG = 192;  // segments per set (validation cap)

struct Scratch {
  // chains by rank
  uint32_t rT[MAXC], rD[MAXC], rCbo[MAXC], rA0[MAXC];  // rA0: first accelerator segment (rank order)
  uint8_t rCls[MAXC], rIdx[MAXC], rNcb[MAXC], rNa[MAXC];
  uint8_t rank_of[MAXC];  // chain index -> rank
  uint32_t cA0[MAXC];     // chain index -> first accelerator segment in callback order
  // callbacks (set-local order)
  uint32_t bE[MAXCB];
  uint8_t bExec[MAXCB], bNa[MAXCB], bA0[MAXCB + 1], bSub[MAXCB], bFa[MAXCB], bFu[MAXCB];
  uint32_t bFw[MAXCB];
  // accelerator segments (callback order)
  uint32_t qAstar[MAXA], qA[MAXA];
  uint8_t qUnit[MAXA], qAcc[MAXA], qCb[MAXA], qRank[MAXA];

  // executors
  uint32_t xPrio[MAXX];
  uint8_t xCore[MAXX], xWait[MAXX], xPPrank[MAXX];
  // accelerators
  uint32_t aN[4], aUnits[4], aUbase[4], aEps[4], aKeff[4], aServer[4];
  union {
    struct {
      // per (rank, unit) / (unit, rank)
      alignas(16) uint32_t W[MAXC][MAXU];
      uint32_t maxA[MAXU][MAXC];
      union {  // WFD scratch is dead before pre2 is computed
        uint32_t pre2[MAXU][MAXC];
        struct {
          uint64_t wfdU[MAXCB];
          uint8_t wfdOrder[MAXCB], wfdUnit[MAXCB], wfdCb[MAXCB];
        };
      };
    };
    struct {  // the set's segments, staged by coalesced loads; dead before WFD / W are written
      uint32_t gW[MAXSEG];  // WCET, saturated at SAT (a WCET >= LIM fails validation)
      uint8_t gKind[MAXSEG], gAcc[MAXSEG], gUnit[MAXSEG];
    };
  };
  uint32_t cmp[MAXC];
  // sub-chains (callback order of their first callback)
  uint8_t sRank[MAXS], sCanon[MAXS], sExec[MAXS], sJ0[MAXS];
  uint32_t sMaxE[MAXS];
};


// 2^16 / d + 1 for 1 <= d <= 32 (n of an accelerator, bucket group size g); warp-uniform index
__constant__ uint32_t kInv16[33] = {0u, 65537u, 32769u, 21846u, 16385u, 13108u, 10923u, 9363u, 8193u, 7282u, 6554u, 5958u, 5462u, 5042u, 4682u, 4370u, 4097u, 3856u, 3641u, 3450u, 3277u, 3121u, 2979u, 2850u, 2731u, 2622u, 2521u, 2428u, 2341u, 2260u, 2185u, 2115u, 2049u};
__device__ __forceinline__ uint32_t inv16(uint32_t d) { return kInv16[d]; }

// saturating inclusive prefix sum over lanes (Hillis-Steele; min(a+b, SAT) is associative on [0, SAT])
__device__ __forceinline__ uint32_t scan_sat_incl(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v = sadd(v, y);
  }
  return v;
}
__device__ __forceinline__ uint32_t scan_excl(uint32_t v, int lane) {  // plain exclusive prefix sum
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  return x - v;
}

// WFD unit assignment, per accelerator (PAAM_FLAG_WFD_UNITS; one lane, out of line: not the default path)
__device__ PAAM_COLD void wfd_units(Scratch& s, uint32_t nac, uint32_t ncb, uint64_t cstart) {
  for (uint32_t a = 0; a < nac; a++) {
    uint32_t ni = 0;
    for (uint32_t j = 0; j < ncb; j++) {
      if (!s.bNa[j]) continue;
      const uint32_t c = __popcll(cstart & ((2ull << j) - 1)) - 1, rk = s.rank_of[c];
      const uint32_t q0 = s.rA0[rk] + (s.bA0[j] - s.cA0[c]);
      uint64_t A = 0;
      for (uint32_t q = q0; q < q0 + s.bNa[j]; q++) if (s.qAcc[q] == a) A += s.qA[q];
      if (A) { s.wfdU[ni] = (A << 24) / s.rT[rk]; s.wfdCb[ni] = (uint8_t)j; ni++; }
    }
    wfd_place(ni, s.wfdU, s.aUnits[a], s.wfdOrder, s.wfdUnit);
    for (uint32_t i = 0; i < ni; i++) {
      const uint32_t j = s.wfdCb[i];
      const uint32_t c = __popcll(cstart & ((2ull << j) - 1)) - 1, rk = s.rank_of[c];
      const uint32_t q0 = s.rA0[rk] + (s.bA0[j] - s.cA0[c]);
      for (uint32_t q = q0; q < q0 + s.bNa[j]; q++)
        if (s.qAcc[q] == a) s.qUnit[q] = (uint8_t)(s.aUbase[a] + s.wfdUnit[i]);
    }
  }
}

#ifndef P_CHUNK
#define P_CHUNK 8  // sets per work ticket
#endif
#ifndef PACK_MINB
#define PACK_MINB 8
#endif
__global__ void __launch_bounds__(WARPS * 32, PACK_MINB) pack_kernel(paam_batch b, Record* __restrict__ recs,
                                                          int32_t* __restrict__ status_out,
                                                          uint32_t* __restrict__ wide_list,
                                                          uint32_t* __restrict__ wide_count,
                                                          unsigned int* __restrict__ work_ticket) {
  __shared__ Scratch smem[WARPS];
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  Scratch& s = smem[threadIdx.x >> 5];
  const bool sound = (b.flags & PAAM_FLAG_BLOCKING_SOUND) != 0;  // record fields of the sound B_c (A10)
  // Dynamic assignment: a warp takes P_CHUNK consecutive sets per ticket (as fused_kernel).  Consecutive
  // sets are adjacent in every CSR array, so the next set's start offsets are this set's end offsets:
  // after a chunk's first set no dependent offset loads remain.
  #pragma unroll 1
  for (;;) {
  uint32_t tk = 0;
  if (lane == 0) tk = atomicAdd(work_ticket, (unsigned)P_CHUNK);
  const uint32_t lo = __shfl_sync(0xffffffffu, tk, 0);
  if (lo >= b.n_sets) break;
  const uint32_t hi = min(lo + (uint32_t)P_CHUNK, b.n_sets);
  uint32_t c0 = 0, x0 = 0, a0 = 0, cb0 = 0, sg0 = 0;      // start offsets of the current set
  uint32_t nc = 0, nx = 0, na_ = 0, ncbo = 0, nsgo = 0;  // end offsets of the current set (prefetched)
  if (lo < hi) {
    c0 = b.set_chain_off[lo]; x0 = b.set_exec_off[lo]; a0 = b.set_accel_off[lo];
    nc = b.set_chain_off[lo + 1]; nx = b.set_exec_off[lo + 1]; na_ = b.set_accel_off[lo + 1];
    cb0 = b.chain_cb_off[c0]; ncbo = b.chain_cb_off[nc];
    sg0 = b.cb_seg_off[cb0]; nsgo = b.cb_seg_off[ncbo];
  }
  #pragma unroll 1
  for (uint32_t set = lo; set < hi; set++) {
    Record* r = recs + set;
    const uint32_t c1 = nc, x1 = nx, a1 = na_, cb1 = ncbo, sg1 = nsgo;
    const uint32_t nch = c1 - c0, nex = x1 - x0, nac = a1 - a0;
    const uint32_t ncb = cb1 - cb0;
    const uint32_t nseg = sg1 - sg0;
    // software pipeline of the next set's end offsets: its three dependent loads are issued at three
    // points of this set's work, so none of them is waited for
    const bool more = set + 1 < hi;
    uint32_t pc = c1, px = x1, pa = a1, pcb = cb1, psg = sg1;
    if (more) { pc = b.set_chain_off[set + 2]; px = b.set_exec_off[set + 2]; pa = b.set_accel_off[set + 2]; }
    bool st2 = !more, st3 = !more;
    int st = PAAM_SET_OK;

    const uint32_t bin = b.set_bin ? b.set_bin[set] : 0u;
    // size caps; a utilisation bin outside [0, n_bins) is a range error too (it is counted in no bin)
    if (nch > MAXC || ncb > MAXCB || nseg > MAXSEG || nex > MAXX || nac > 4 || (b.set_bin && bin >= b.n_bins))
      st = PAAM_SET_ERANGE;
    uint32_t n_aseg = 0, n_sub = 0, n_unit = 0;
    uint64_t runstart = 0;  // bit j: callback j starts a sub-chain
    uint64_t cstart = 0;    // bit j: callback j is the first of its chain
    // per-lane chain data (lane = chain index)
    uint32_t T = 0, D = 0, prio = 0, cls = 0, cbo = 0, cbn = 0, rank = 0;
    if (st == PAAM_SET_OK) {
      // ---- load: chains (lane), accelerators (lane), executors (lane) ---------------------------
      bool erange = false, edang = false, eaccel = false, eshape = false, edup = false, edl = false, ecore = false;
      bool wide = false;  // a time in [2^31 - 1, 2^48) ns: the set goes to the u64 path (wide.cu)
      if (lane < nch) {
        const uint64_t T64 = b.chain_T[c0 + lane], D64 = b.chain_D[c0 + lane];
        erange |= (T64 == 0 || T64 >= LIMW || D64 >= LIMW);
        wide |= (T64 >= LIM || D64 >= LIM);
        T = (uint32_t)min(T64, (uint64_t)SAT);
        D = (uint32_t)min(D64, (uint64_t)SAT);
        prio = b.chain_prio[c0 + lane];
        cls = b.chain_class[c0 + lane];
        cbo = b.chain_cb_off[c0 + lane] - cb0;
        cbn = b.chain_cb_off[c0 + lane + 1] - cb0 - cbo;
        edang |= (cbn == 0) || (cbo > ncb) || (cbn > ncb - cbo);  // (malformed CSR: no out-of-range indexing)
        eshape |= (cls > 1);
        edl |= (D == 0 || (cls == 0 && D > T));
      }
      if (lane < nac) {
        const uint32_t n = b.accel_buckets[a0 + lane], u = b.accel_units[a0 + lane];
        const uint64_t e = b.accel_eps[a0 + lane], kp = b.accel_kappa[a0 + lane];
        erange |= (n < 1 || n > 32 || u < 1 || u > 8 || e >= LIMW || kp >= LIMW);
        wide |= (e >= LIM || kp >= LIM);
        s.aN[lane] = n;
        s.aUnits[lane] = u;
        s.aEps[lane] = (uint32_t)min(e, (uint64_t)SAT);
        s.aKeff[lane] = n > 1 ? (uint32_t)min(kp, (uint64_t)SAT) : 0u;  // A6
        s.aServer[lane] = b.accel_server_core[a0 + lane];
      }
      uint32_t xcore = 0xffffffffu, xprio = 0;
      if (lane < nex) {
        xcore = b.exec_core[x0 + lane];
        xprio = b.exec_prio[x0 + lane];
        const uint32_t w = b.exec_wait[x0 + lane];
        eshape |= (w > 1);
        s.xCore[lane] = (uint8_t)xcore;
        s.xPrio[lane] = xprio;
        s.xWait[lane] = (uint8_t)w;
      }
      __syncwarp();
      // units: per-accelerator base and total
      {
        const uint32_t u = lane < nac ? s.aUnits[lane] : 0u;
        const uint32_t ub = scan_excl(u, lane);
        if (lane < nac) s.aUbase[lane] = ub;
        n_unit = __reduce_add_sync(FULL, u);
      }
      // chain start callbacks as a 64-bit mask (bit cbo of every chain)
      const uint64_t cstart_bit = (lane < nch && cbo < 64) ? (1ull << cbo) : 0ull;
      cstart = ((uint64_t)__reduce_or_sync(FULL, (uint32_t)(cstart_bit >> 32)) << 32) |
                              __reduce_or_sync(FULL, (uint32_t)cstart_bit);
      __syncwarp();
      // ---- segments: staged with coalesced loads (one round trip for the whole set), lane per segment,
      // with the per-segment validation (time range, kind, WCET > 0, declared accelerator and unit);
      // the set's callbacks cover [sg0, sg1) exactly unless a callback range is malformed (EDANGLING)
#ifndef PAAM_WARP_EMU
#pragma unroll kStageUnroll
#endif
      #pragma unroll 1
      for (uint32_t i = lane; i < nseg; i += 32) {
        const uint64_t w = b.seg_wcet[sg0 + i];
        const uint32_t kind = b.seg_kind[sg0 + i], a = b.seg_accel[sg0 + i], u = b.seg_unit[sg0 + i];
        erange |= (w >= LIMW);
        wide |= (w >= LIM);
        eshape |= (kind > 1) || (w == 0);
        if (kind == 1) {
          if (a >= nac) eaccel = true;
          else edang |= (u >= s.aUnits[a]);
        }
        s.gW[i] = (uint32_t)min(w, (uint64_t)SAT);
        s.gKind[i] = (uint8_t)kind;
        s.gAcc[i] = (uint8_t)a;
        s.gUnit[i] = (uint8_t)u;
      }
      __syncwarp();
      // ---- callbacks: two passes of 32 lanes; each lane walks its segments ----------------------
      uint32_t prev_exec = 0xffffffffu;
      bool malformed = false;  // a callback's segment range leaves the set's: EDANGLING before segment checks
      #pragma unroll 1
      for (uint32_t pass = 0; pass * 32 < ncb; pass++) {
        const uint32_t j = pass * 32 + lane;
        uint32_t exec = 0xffffffffu, E = 0, na = 0, fa = 0, fu = 0, fw = 0;  // fa/fu/fw: first ACCEL segment
        if (j < ncb) {
          exec = b.cb_exec[cb0 + j];
          uint32_t so = b.cb_seg_off[cb0 + j], se = b.cb_seg_off[cb0 + j + 1];
          edang |= (se == so) || (exec >= nex);
          if (so < sg0 || se < so || se > sg1) { malformed = true; so = se = sg0; }  // no staged reads
          uint32_t prev_kind = 0xffffffffu;
#pragma unroll kSegUnroll
          for (uint32_t k = so - sg0; k < se - sg0; k++) {
            const uint32_t kind = s.gKind[k], w = s.gW[k];
            eshape |= (kind == prev_kind);  // CPU / ACCEL segments alternate
            prev_kind = kind;
            if (kind == 0) {
              E = sadd(E, w);
            } else if (kind == 1) {  // an undefined kind (ESHAPE) is no accelerator segment
              if (na == 0) { fa = s.gAcc[k]; fu = s.gUnit[k]; fw = w; }
              na++;
            }
          }
          s.bExec[j] = (uint8_t)min(exec, 255u);
          s.bE[j] = E;
          s.bNa[j] = (uint8_t)min(na, 255u);
          s.bFa[j] = (uint8_t)min(fa, 255u);
          s.bFu[j] = (uint8_t)min(fu, 255u);
          s.bFw[j] = fw;
        }
        // previous callback's executor (shuffle; the pass boundary carries lane 31 over)
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
      // A13: a chain never re-enters an executor it left
      #pragma unroll 1
      for (uint32_t j = lane; j < ncb; j += 32) {
        if (((runstart >> j) & 1ull) && !((cstart >> j) & 1ull)) {
          const uint32_t first = 63 - __clzll(cstart & ((2ull << j) - 1));  // chain's first callback
          #pragma unroll 1
          for (uint32_t i = first; i + 1 < j; i++) eshape |= (s.bExec[i] == s.bExec[j]);
        }
      }
      // chain ranks and duplicate priorities
      {
        uint32_t rk = 0;
        #pragma unroll 1
        for (uint32_t d = 0; d < nch; d++) rk += (__shfl_sync(FULL, prio, d) > prio);
        rank = rk;
        const uint32_t valid = nch >= 32 ? FULL : (1u << nch) - 1u;
        const uint32_t same = __match_any_sync(FULL, prio) & valid & ~(1u << lane);
        edup |= (lane < nch && same != 0);
      }
      // executors: duplicate (core, priority) and process-priority rank on the core; R1 (ECORE)
      {  // executors sharing a core are found by match; only those are compared
        const uint32_t same_core = __match_any_sync(FULL, xcore) & ~(1u << lane);
        uint32_t pr = 0, m = lane < nex ? same_core : 0u;
        while (m) {
          const uint32_t y = __ffs(m) - 1;
          m &= m - 1;
          const uint32_t py = s.xPrio[y];
          edup |= (py == xprio);
          pr += (py > xprio);
        }
        if (lane < nex) {
          s.xPPrank[lane] = (uint8_t)pr;
          #pragma unroll 1
          for (uint32_t a = 0; a < nac; a++) ecore |= (xcore == s.aServer[a]);
        }
      }
      erange |= (n_aseg > MAXA) || (n_unit > MAXU);
      // first failing class, in the documented order (a malformed callback range is a dangling
      // reference: it is reported before the checks of the segments the callbacks no longer cover)
      if (__any_sync(FULL, malformed)) st = PAAM_SET_EDANGLING;
      else if (__any_sync(FULL, erange)) st = PAAM_SET_ERANGE;
      else if (__any_sync(FULL, wide)) st = REC_STATUS_WIDE;  // handed over: wide.cu validates and analyses it
      else if (__any_sync(FULL, edang)) st = PAAM_SET_EDANGLING;
      else if (__any_sync(FULL, eaccel)) st = PAAM_SET_EACCEL;
      else if (__any_sync(FULL, eshape)) st = PAAM_SET_ESHAPE;
      else if (n_sub > MAXS) st = PAAM_SET_ERANGE;
      else if (__any_sync(FULL, edup)) st = PAAM_SET_EDUPPRIO;
      else if (__any_sync(FULL, edl)) st = PAAM_SET_EDEADLINE;
      else if (__any_sync(FULL, ecore)) st = PAAM_SET_ECORE;
    }

    if (!st2) { pcb = b.chain_cb_off[pc]; st2 = true; }
    if (lane == 0) {
      r->status = st;
      r->chain_base = c0;
      r->bin = (b.set_bin && bin >= b.n_bins) ? 0xffffffffu : bin;  // analyze skips an out-of-range bin
      r->n_out = nch;
      if (status_out && st != REC_STATUS_WIDE) status_out[set] = st;
      if (st == REC_STATUS_WIDE) wide_list[atomicAdd(wide_count, 1u)] = set;
      if (st != PAAM_SET_OK) { r->n_chain = 0; r->n_sub = 0; r->n_aseg = 0; r->n_unit = 0; }
    }
    if (st != PAAM_SET_OK) {
      __syncwarp();
      if (!st3) psg = b.cb_seg_off[pcb];
      c0 = c1; x0 = x1; a0 = a1; cb0 = cb1; sg0 = sg1;
      nc = pc; nx = px; na_ = pa; ncbo = pcb; nsgo = psg;
      continue;
    }

    // ======================== derivation (valid set) =================================================
    const bool is_chain = lane < nch;
    // chain data by rank; accelerator-segment offsets (callback order) per chain
    if (is_chain) {
      s.rank_of[lane] = (uint8_t)rank;
      s.rT[rank] = T;
      s.rD[rank] = D;
      s.rCls[rank] = (uint8_t)cls;
      s.rIdx[rank] = (uint8_t)lane;
      s.rCbo[rank] = cbo;
      s.rNcb[rank] = (uint8_t)cbn;
    }
    // per-callback first accelerator segment (exclusive scan over the callback order)
    {
      uint32_t carry = 0;
      #pragma unroll 1
      for (uint32_t pass = 0; pass * 32 < ncb; pass++) {
        const uint32_t j = pass * 32 + lane;
        const uint32_t na = j < ncb ? s.bNa[j] : 0u;
        const uint32_t ex = scan_excl(na, lane);
        if (j < ncb) s.bA0[j] = (uint8_t)(carry + ex);
        carry += __reduce_add_sync(FULL, na);
      }
      if (lane == 0) s.bA0[ncb] = (uint8_t)carry;
    }
    __syncwarp();
    // per-chain accelerator-segment count, first index in callback order and in rank order
    {
      const uint32_t k = lane;  // rank
      uint32_t na = 0;
      if (k < nch) {
        const uint32_t o = s.rCbo[k];
        na = s.bA0[o + s.rNcb[k]] - s.bA0[o];
        s.cA0[s.rIdx[k]] = s.bA0[o];
      }
      const uint32_t f = scan_excl(na, lane);
      if (k < nch) { s.rA0[k] = f; s.rNa[k] = (uint8_t)na; }
    }
    // sub-chain id of every callback
    #pragma unroll 1
    for (uint32_t j = lane; j < ncb; j += 32) {
      const uint32_t sid = __popcll(runstart & ((2ull << j) - 1)) - 1;
      s.bSub[j] = (uint8_t)sid;
      if ((runstart >> j) & 1ull) s.sJ0[sid] = (uint8_t)j;  // first callback of each sub-chain
    }
    __syncwarp();
    // ---- accelerator segments: A*, unit, rank; written in rank order --------------------------------
    #pragma unroll 1
    for (uint32_t pass = 0; pass * 32 < ncb; pass++) {
      const uint32_t j = pass * 32 + lane;
      if (j < ncb && s.bNa[j]) {
        const uint32_t c = __popcll(cstart & ((2ull << j) - 1)) - 1;  // chain index of callback j
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
        if (s.bNa[j] == 1) {  // the common case: its one segment was kept by the callback pass
          put(s.bFa[j], s.bFu[j], s.bFw[j]);
        } else {
          const uint32_t so = b.cb_seg_off[cb0 + j] - sg0, se = b.cb_seg_off[cb0 + j + 1] - sg0;
          #pragma unroll 1
          for (uint32_t k = so; k < se; k++)  // the staged segments are intact until WFD / W
            if (s.gKind[k] == 1) put(s.gAcc[k], s.gUnit[k], s.gW[k]);
        }
      }
    }
    __syncwarp();
    if ((b.flags & PAAM_FLAG_WFD_UNITS) && lane == 0) wfd_units(s, nac, ncb, cstart);
    __syncwarp();
    // ---- per chain (lane = rank): W[k][u], max A*[u][k], accelerator use mask ------------------------
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
        s.W[k][u] = sadd(s.W[k][u], a);  // saturating sums are exact (associative on [0, SAT])
      }
    }
    __syncwarp();
    if (!st3) { psg = b.cb_seg_off[pcb]; st3 = true; }
    // ---- buckets (A5) and LP blocking per (unit, rank) ---------------------------------
    #pragma unroll 1
    for (uint32_t a = 0; a < nac; a++) {
      const uint32_t U = __ballot_sync(FULL, (use >> a) & 1u);
      const uint32_t ma = __popc(U), n = s.aN[a];
      // x / d == (x * (2^16 / d + 1)) >> 16 for x < 64, 1 <= d <= 32 (checked exhaustively): no divides
      const uint32_t g = ma ? ((ma + n - 1) * inv16(n)) >> 16 : 1u;
      const uint32_t ginv = inv16(g);
      const bool user = (U >> lane) & 1u;
      const uint32_t p = __popc(U & lt);  // position among users in rank order
      // users of a form aligned blocks of g consecutive positions, one block per bucket: the user at
      // position p is in bucket n - 1 - p / g (A5)
      const uint32_t blk_end = min(((((uint32_t)lane * ginv) >> 16) + 1) * g, ma);
      #pragma unroll 1
      for (uint32_t u = s.aUbase[a]; u < s.aUbase[a] + s.aUnits[a]; u++) {
        if (user) s.cmp[p] = s.maxA[u][lane];
        __syncwarp();
        uint32_t v = (uint32_t)lane < ma ? s.cmp[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {  // segmented inclusive suffix max
          const uint32_t y = __shfl_down_sync(FULL, v, o);
          if ((uint32_t)lane + o < blk_end) v = max(v, y);
        }
        const uint32_t nxt = __shfl_down_sync(FULL, v, 1);
        const uint32_t ex = ((uint32_t)lane + 1 < blk_end) ? nxt : 0u;  // exclusive: lower priorities only
        __syncwarp();
        if ((uint32_t)lane < ma) s.cmp[lane] = ex;
        __syncwarp();
        s.maxA[u][lane] = user ? s.cmp[p] : 0u;  // in place: maxA becomes LP blocking
        __syncwarp();
      }
    }
    // 2 * sum_{k < r} W[k][u]: the "+1 +1" of mu summed over the HP chains (exact, saturating)
    #pragma unroll 1
    for (uint32_t u = 0; u < n_unit; u++) {
      const uint32_t w = is_chain ? s.W[lane][u] : 0u;
      const uint32_t incl = scan_sat_incl(w, lane);
      const uint32_t prev = __shfl_up_sync(FULL, incl, 1);
      const uint32_t ex = lane == 0 ? 0u : prev;
      s.pre2[u][lane] = sadd(ex, ex);
    }
    __syncwarp();

    // ---- sub-chains (lane = sub-chain id, callback order) -------------------------------------------
    uint32_t s_exec = 0, s_rank = 0, s_key = 0xffffffffu, s_j0 = 0, s_nj = 0, s_E = 0;
    if ((uint32_t)lane < n_sub) {
      s_j0 = s.sJ0[lane];
      s_nj = ((uint32_t)lane + 1 < n_sub ? s.sJ0[lane + 1] : ncb) - s_j0;  // runs never span two chains
      const uint32_t c = __popcll(cstart & ((2ull << s_j0) - 1)) - 1;
      s_exec = s.bExec[s_j0];
      s_rank = s.rank_of[c];
      s_key = ((uint32_t)s.xCore[s_exec] << 16) | ((uint32_t)s.xPPrank[s_exec] << 8) | s_rank;
      uint32_t mE = 0;
      #pragma unroll 1
      for (uint32_t j = s_j0; j < s_j0 + s_nj; j++) { mE = max(mE, s.bE[j]); s_E = sadd(s_E, s.bE[j]); }
      s.sMaxE[lane] = mE;
      s.sRank[lane] = (uint8_t)s_rank;
      s.sExec[lane] = (uint8_t)s_exec;
    }
    // canonical order (A7): per core, process priority desc, chain rank asc
    {
      uint32_t pos = 0;
      #pragma unroll 1
      for (uint32_t l = 0; l < n_sub; l++) pos += (__shfl_sync(FULL, s_key, l) < s_key);
      if ((uint32_t)lane < n_sub) s.sCanon[lane] = (uint8_t)pos;
    }
    __syncwarp();
    const uint32_t same_exec = __match_any_sync(FULL, (uint32_t)lane < n_sub ? s_exec : 0x100u + lane);
    const uint32_t my_core = (uint32_t)lane < n_sub ? s.xCore[s_exec] : 0x100u + lane;
    const uint32_t same_core = __match_any_sync(FULL, my_core);
    if ((uint32_t)lane < n_sub) {
      const uint32_t k = s.sCanon[lane];
      const uint32_t c = s.rIdx[s_rank];
      // sub-chain's accelerator segments: contiguous in rank order
      const uint32_t qa = s.rA0[s_rank] + (s.bA0[s_j0] - s.cA0[c]);
      const uint32_t qn = s.bA0[s_j0 + s_nj] - s.bA0[s_j0];
      const uint32_t E = s_E;
      uint32_t eps = 0, base3 = 0, umask = 0, slb = 0;
      #pragma unroll 1
      for (uint32_t q = qa; q < qa + qn; q++) {
        const uint32_t u = s.qUnit[q];
        eps = sadd(eps, s.aEps[s.qAcc[q]]);
        const uint32_t b = sadd(s.qAstar[q], s.maxA[u][s_rank]);
        base3 = sadd(base3, b);
        slb = sadd(slb, sadd(b, s.pre2[u][s_rank]));  // aBase2 of the segment (Lemma-2 start value)
        umask |= 1u << u;
      }
      uint32_t a2 = base3;  // Eq.4 with every mu = 2 (the union of hps over the sub-chain's units, A1)
      #pragma unroll 1
      for (uint32_t um = umask; um; um &= um - 1) a2 = sadd(a2, s.pre2[__ffs(um) - 1][s_rank]);
      uint32_t hp = 0, lp = 0, hpp = 0, B = 0;
      uint32_t m = same_exec & ~(1u << lane);
      while (m) {
        const uint32_t l = __ffs(m) - 1;
        m &= m - 1;
        if (s.sRank[l] < s_rank) hp |= 1u << s.sCanon[l];
        else { lp |= 1u << s.sCanon[l]; B = max(B, s.sMaxE[l]); }  // B_c
      }
      m = same_core & ~same_exec;
      const uint32_t mypp = s.xPPrank[s_exec];
      while (m) {
        const uint32_t l = __ffs(m) - 1;
        m &= m - 1;
        if (s.xPPrank[s.sExec[l]] < mypp) hpp |= 1u << s.sCanon[l];
      }
      // position of this sub-chain inside its chain
      const uint32_t pos = __popcll(runstart & ((1ull << s_j0) - 1) & ~((1ull << s.rCbo[s_rank]) - 1));
      r->sE[k] = E;
      r->sB[k] = B;
      r->sEps[k] = eps;
      r->sHp[k] = hp;
      r->sHpp[k] = hpp;
      if (sound) r->sLp[k] = lp;
      r->sMisc[k] = s_rank | (umask << 8) | ((uint32_t)(s.xWait[s_exec] == 1) << 16) | (pos << 24);
      r->sSeg[k] = qa | (qn << 8) | (s_exec << 16) | ((uint32_t)s.xCore[s_exec] << 24);
      r->sA2[k] = a2;
      r->sSlb[k] = slb;
    }
    // ---- chains by rank ---------------------------------------------------------------------------------
    const uint32_t Tk = is_chain ? s.rT[lane] : 0xffffffffu;
    uint32_t M = 0, L = 0;
    if (is_chain) {
      const uint32_t k = lane;
      make_magic(Tk, &M, &L);
      const uint32_t o = s.rCbo[k], nb = s.rNcb[k];
      const uint64_t rng = (nb >= 64 ? ~0ull : ((1ull << nb) - 1)) << o;
      const uint32_t nsub = __popcll(runstart & rng);
      r->cCut[k] = min(s.rD[k], s.rT[k]);
      r->cD[k] = s.rD[k];
      r->cM[k] = M;
      r->cMisc[k] = L | ((uint32_t)s.rCls[k] << 8) | ((uint32_t)s.rIdx[k] << 16) | (nsub << 24);
      #pragma unroll 1
      for (uint32_t u = 0; u < n_unit; u++) r->W[k][u] = s.W[k][u];
    }
    {  // period order (ascending T, ties by rank)
      uint32_t pos = 0;
      #pragma unroll 1
      for (uint32_t j = 0; j < nch; j++) {
        const uint32_t Tj = __shfl_sync(FULL, Tk, j);
        pos += (Tj < Tk) || (Tj == Tk && j < (uint32_t)lane);
      }
      if (is_chain) r->pTab[pos] = uint4{Tk, M, L | ((uint32_t)lane << 8), sadd(s.W[lane][0], s.W[lane][1])};
      // every period >= 64 ns: q * W < 2^62 / 64, so 64 such products cannot overflow a u64 sum
      if (lane == 0) r->hflags = 0u;
    }
    // ---- accelerator segments (rank order) ------------------------------------------------------------
    #pragma unroll 1
    for (uint32_t q = lane; q < n_aseg; q += 32) {
      const uint32_t u = s.qUnit[q], rk = s.qRank[q];
      r->aBase2[q] = sadd(sadd(s.qAstar[q], s.maxA[u][rk]), s.pre2[u][rk]);
      if (sound) {
        r->aEps[q] = s.aEps[s.qAcc[q]];
        r->aCbE[q] = s.bE[s.qCb[q]];
      }
      r->aMisc[q] = rk | (u << 8) | ((uint32_t)s.sCanon[s.bSub[s.qCb[q]]] << 16) | ((uint32_t)s.qCb[q] << 24);
    }
    if (lane == 0) { r->n_chain = (uint8_t)nch; r->n_sub = (uint8_t)n_sub; r->n_aseg = (uint8_t)n_aseg; r->n_unit = (uint8_t)n_unit; }
    __syncwarp();
    c0 = c1; x0 = x1; a0 = a1; cb0 = cb1; sg0 = sg1;
    nc = pc; nx = px; na_ = pa; ncbo = pcb; nsgo = psg;
  }
  }
}

}  // namespace

#ifndef PAAM_WARP_EMU
int launch_pack(const paam_batch* b, Record* rec, int32_t* status, uint32_t* wide_list, uint32_t* wide_count,
                cudaStream_t st) {
  if (b->n_sets == 0) return PAAM_OK;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pack_kernel, WARPS * 32, 0);
  if (per_sm < 1) per_sm = 1;
  const uint32_t need = (b->n_sets + WARPS - 1) / WARPS;
  const uint32_t cap = (uint32_t)sms * (uint32_t)per_sm;
  const uint32_t grid = need < cap ? need : cap;
  pack_kernel<<<grid, WARPS * 32, 0, st>>>(*b, rec, status, wide_list, wide_count, wide_count + 1);
  count_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PAAM_OK : fail_cuda(e, "pack_kernel launch");
}

#endif  // PAAM_WARP_EMU

}  // namespace paam
