// simulate.cu -- §8(a) steps 7-8: discrete-event simulation of PAAM arbitration, one warp per set.
//
// Semantics: DESIGN.md App. A (rules D1-D17), derived from the paper's execution model
// (PiCAS executors P:135-136, fixed-priority cores P:136, PAAM server rules R1-R4 P:366-373,
// eps / kappa overheads P:374, bucket FIFO on equal priority P:320).  Lane ownership:
//   lane k  = chain of rank k (k = 0 highest priority): its <= QCAP live instances, release
//             schedule, statistics.  D14 queues every release of a chain (an unbounded backlog,
//             S:311); a release that finds all QCAP slots live stops the set's run and reports
//             PAAM_SIM_BACKLOG (everything up to that release is exact, so the outputs are lower
//             bounds of the full run's);
//   lane x  = executor x in canonical order (core asc, process priority desc): job, phase, work;
//   lane u  = accelerator unit u: state (idle / run / switch-out / switch-in), current request.
// Every timestamp is settled like this (D15): phase A = (1) unit phase ends and completions,
// (2) executor CPU / eps completions with enqueues sequenced by (chain, instance) (D7),
// (3) comm arrivals, (4) releases -- repeated until stable; phase B = (5) executor choice,
// (6) core dispatch, (7) unit dispatch; A/B repeat until nothing changes.  A pass is repeated only
// when something is provably left for it (zero-length work due now, an executor that just got its
// core with ready work), so every skipped pass would have been a no-op.  Each sub-phase is
// lane-parallel over the entities it touches (they touch disjoint state; shared statistics use
// shared-memory atomics); "best" choices are warp reductions over rank-ordered lanes, so the
// highest priority is the lowest set bit of a ballot.  Time then jumps to the warp-min next event.
// Instance slots are packed one byte per slot per chain (byte-compare scans).  The event digest is
// a sum of per-record FNV-1a-64 hashes (order independent), computed only when requested: the lane
// that makes an event appends its 16-byte record to the warp's event buffer (global scratch, L2-resident),
// and the warp hashes the buffered records 32 at a time, one per lane, whenever the buffer could not take
// another settle pass (and at the end of the run).
#include "../../gen/paam_gen.h"
#include "common.cuh"

struct paam_sets;  // defined in api.cu

namespace paam {

namespace {

// Block shape, measured (tools/des_variants.sh, 1M config-5 sets): 16 blocks of 2 warps per SM beat 8 of 4
// (317.5k vs 312k sets/s with digests), 4 of 8 (296k) and 32 of 1 (278k).
#ifndef SIM_WARPS
#define SIM_WARPS 2
#endif
constexpr int SW = SIM_WARPS;  // warps per block
constexpr int QCAP = PAAM_SIM_QCAP;  // instance slots per chain; one more live instance stops the run
constexpr int MAXG = 192;  // segments per set
constexpr uint32_t FULL = 0xffffffffu;
constexpr uint64_t NONE64 = ~0ull;
constexpr uint64_t STEP_CAP = PAAM_SIM_STEP_CAP;  // safety valve: a run past it stops (PAAM_SIM_STEPCAP)
// Event buffer per warp.  One phase-A pass makes at most 4 events per unit (ACC_DONE, SEG_DONE, CB_DONE,
// CHAIN_DONE), 3 per executor (SEG_DONE, CB_DONE, CHAIN_DONE; or REQ_ENQUEUE) and 5 per chain (QCAP
// drops + RELEASE): <= 8*4 + 32*3 + 32*5 = 288; a phase-B pass at most one CB_START per executor and two
// events per unit: <= 48.  The buffer is flushed before a pass that could overflow it.
constexpr uint32_t EVCAP = 512;
constexpr uint32_t EV_PASS_MAX = 288;

enum { EV_RELEASE = 0, EV_DROP, EV_OVERFLOW, EV_CB_START, EV_SEG_DONE, EV_REQ_ENQUEUE, EV_ACC_START,
       EV_ACC_PREEMPT, EV_ACC_RESUME, EV_ACC_DONE, EV_CB_DONE, EV_CHAIN_DONE };
enum { P_NONE = 0, P_CPU, P_EPS_SPIN, P_EPS_SUSP, P_WAIT };
enum { U_IDLE = 0, U_RUN, U_SWOUT, U_SWIN };
enum { I_FREE = 0, I_READY, I_RUN, I_TRANSIT };
constexpr uint32_t NOQ = 0xffu;  // wunit of a request that is not queued

// Instance slot q of chain c: the wide fields per slot, the byte fields packed per chain (byte q of
// a word), so that the per-lane scans over a chain's QCAP slots are one word load + a byte compare.
// The release time is not stored: instance k of chain c is released at phase_c + k T_c (D2).
struct InstWide {
  uint32_t k, seq;
  union {
    uint32_t ready_at;  // I_TRANSIT: arrival of the next callback (D13), low 32 bits (see Ctx::t32)
    uint32_t rem;       // a preempted request: its remaining accelerator work
  };
};
struct InstRef {
  uint8_t &state, &cb, &wunit, &started;  // wunit: the unit a waiting request is queued on, else NOQ
  uint32_t& ready_at;
  uint32_t &k, &seq, &rem;
};
__device__ __forceinline__ uint8_t& byte_of(uint32_t& w, uint32_t q) { return reinterpret_cast<uint8_t*>(&w)[q]; }
__device__ __forceinline__ uint32_t rep4(uint32_t v) { return v * 0x01010101u; }
// slots whose byte in w equals v: bit 8q set for slot q (iterate with m &= m - 1, slot_of(m))
__device__ __forceinline__ uint32_t slots_eq(uint32_t w, uint32_t v) { return __vcmpeq4(w, rep4(v)) & 0x01010101u; }
__device__ __forceinline__ uint32_t slot_of(uint32_t m) { return (uint32_t)(__ffs(m) - 1) >> 3; }

struct DesSmem {
  // static (per set)
  uint32_t cT[MAXC], cD[MAXC];
  uint64_t cPhase[MAXC];
  uint8_t cCls[MAXC], cLocal[MAXC], cCb0[MAXC], cNcb[MAXC];
  uint8_t bExec[MAXCB], bNseg[MAXCB];
  uint8_t bSeg0[MAXCB];
  uint32_t gW[MAXG];
  uint8_t gKind[MAXG], gUnit[MAXG], gBkt[MAXG];
  uint8_t cuBkt[MAXC][MAXU];  // bucket of chain rank k on unit u (per chain and accelerator)
  uint32_t xSameCore[MAXX];
  uint8_t xWait[MAXX];
  uint32_t uEps[MAXU], uKap[MAXU], uN[MAXU];
  // dynamic
  union {
    InstWide iw[MAXC][QCAP];
    struct {  // WFD scratch of the static staging (dead before the dynamic state exists)
      uint64_t wu[MAXCB];
      uint8_t wo[MAXCB], wn[MAXCB], wc[MAXCB];
    } wfd;
  };
  uint32_t iState[MAXC], iCb[MAXC], iWUnit[MAXC], iStarted[MAXC];
  __device__ __forceinline__ InstRef ref(uint32_t c, uint32_t q) {
    InstWide& w = iw[c][q];
    return InstRef{byte_of(iState[c], q), byte_of(iCb[c], q), byte_of(iWUnit[c], q), byte_of(iStarted[c], q),
                   w.ready_at, w.k, w.seq, w.rem};
  }
  uint32_t exRem[MAXX];
  uint32_t exTimer[MAXX];  // P_EPS_SUSP: end of the eps timer (low 32 bits)
  uint8_t exChain[MAXX], exSlot[MAXX], exSeg[MAXX], exPhase[MAXX];
  uint32_t unEnd[MAXU];  // end of the unit's current phase (run / switch-out / switch-in), low 32 bits
  uint8_t unState[MAXU], unChain[MAXU], unSlot[MAXU];
  uint32_t uQ[MAXU];  // requests queued on the unit (waiting, started or not; the running one included)
  uint8_t uDirty[MAXU];  // a running unit's queue or running request changed since its last preemption check
  unsigned long long maxResp[MAXC];
  uint32_t cnt[MAXC], miss[MAXC];
  uint32_t evN;  // records in the warp's event buffer
};

// FNV-1a-64 of a 32-byte event record (D17) in two parts: the state after the record's 8-byte time
// (the same for every record of a timestamp, so computed once per timestamp), then the 24 other bytes.
__device__ __forceinline__ uint64_t fnv_time(uint64_t t) {
  constexpr uint64_t P = 0x100000001b3ull, P3 = 0x08a97b0004e7feabull;  // P^3 mod 2^64
  uint64_t h = 0xcbf29ce484222325ull;
#pragma unroll
  for (int b = 0; b < 5; b++) h = (h ^ ((t >> (8 * b)) & 0xffu)) * P;
  if ((t >> 40) == 0) return h * P3;  // three zero bytes only multiply (t < 2^40 ns = 18 min)
#pragma unroll
  for (int b = 5; b < 8; b++) h = (h ^ ((t >> (8 * b)) & 0xffu)) * P;
  return h;
}
// One 4-byte field.  A field that does not apply (FULL at its call site) is recorded as 0xff (D17),
// and every real field is below 255, so each field's three high bytes are zero and only multiply:
// FNV-1a over the field's 4 bytes is (h ^ v) * P^4 (mod 2^64), one product.
__device__ __forceinline__ uint64_t fnv_field(uint64_t h, uint32_t v) {
  constexpr uint64_t P4 = 0x9ffaac085635bc91ull;  // P^4 mod 2^64, P = 0x100000001b3
  return (h ^ (v == 0xffffffffu ? 0xffu : v)) * P4;
}
// A record: {t low, t high, kind | chain << 8 | callback << 16 | segment << 24, unit | bucket << 8}, one
// byte per field (0xff: does not apply), chain = the set-local index (buffered as the rank).
__device__ __forceinline__ uint64_t fnv_record(uint4 e) {
  uint64_t h = fnv_time(((uint64_t)e.y << 32) | e.x);
  h = fnv_field(h, e.z & 0xffu);
  h = fnv_field(h, (e.z >> 8) & 0xffu);
  h = fnv_field(h, (e.z >> 16) & 0xffu);
  h = fnv_field(h, e.z >> 24);
  h = fnv_field(h, e.w & 0xffu);
  return fnv_field(h, e.w >> 8);
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

__device__ __forceinline__ uint32_t ev_byte(uint32_t v) { return v == 0xffffffffu ? 0xffu : v; }

// Every pending event lies less than 2^31 ns ahead of t (a period, eps, kappa, comm or remaining work,
// each < 2^31 - 1 ns), so the absolute times of pending events are kept as their low 32 bits: equality
// with t and the distance from t are exact in 32-bit arithmetic.
struct Ctx {
  DesSmem& S;
  uint64_t t, horizon, comm;
  __device__ uint32_t t32() const { return (uint32_t)t; }
  uint64_t dig;  // this lane's partial digest
  bool fifo;     // FIFO_DIRECT: no eps, no kappa, no buckets, arrival order
  bool want_dig; // the caller asked for digests (out_digest != NULL); otherwise events are not recorded
  uint4* evb;    // this warp's event buffer (EVCAP records)
  __device__ void ev(uint32_t kind, uint32_t c, uint32_t cb, uint32_t seg, uint32_t unit, uint32_t bk) {
    if (want_dig) {
      const uint32_t i = atomicAdd(&S.evN, 1u);
#ifdef PAAM_WARP_EMU
      if (i >= EVCAP) { fprintf(stderr, "simulate: event buffer overflow (%u, kind %u)\n", i, kind); abort(); }
#endif
      evb[i] = make_uint4((uint32_t)t, (uint32_t)(t >> 32),
                          kind | (c << 8) | (ev_byte(cb) << 16) | (ev_byte(seg) << 24),
                          ev_byte(unit) | (ev_byte(bk) << 8));
    }
  }
  // warp-converged, before a settle pass: could the pass overflow the buffer?  Lane 0's count decides for
  // the warp -- a lane that already started the pass could have added records that the others' reads would
  // see (no lane can pass the shuffle before every lane reached it, and no event is made between the
  // previous collective and this one).
  __device__ bool must_flush() { return __shfl_sync(0xffffffffu, S.evN, 0) > EVCAP - EV_PASS_MAX; }
  // warp-converged: hash the buffered records, one per lane, and empty the buffer
  __device__ void flush(uint32_t lane) {
    __syncwarp();
    const uint32_t n = S.evN;
    for (uint32_t i = lane; i < n; i += 32) {
      uint4 e = evb[i];
      e.z = (e.z & 0xffff00ffu) | ((uint32_t)S.cLocal[(e.z >> 8) & 0xffu] << 8);  // rank -> set-local chain
      dig += fnv_record(e);
    }
    __syncwarp();
    if (lane == 0) S.evN = 0;
    __syncwarp();
  }
  // executor x starts segment exSeg[x] of its job's callback; true: it has phase-A work due now (a
  // zero-length eps; CPU segments are never zero-length)
  __device__ bool begin_segment(uint32_t x) {
    const uint32_t c = S.exChain[x], sl = S.exSlot[x];
    const uint32_t j = S.cCb0[c] + S.ref(c, sl).cb;
    const uint32_t g = S.bSeg0[j] + S.exSeg[x];
    if (S.gKind[g] == 0) {
      S.exPhase[x] = P_CPU;
      S.exRem[x] = S.gW[g];
      return false;
    }
    const uint32_t eps = fifo ? 0u : S.uEps[S.gUnit[g]];
    if (S.xWait[x]) { S.exPhase[x] = P_EPS_SPIN; S.exRem[x] = eps; }
    else { S.exPhase[x] = P_EPS_SUSP; S.exTimer[x] = t32() + eps; }
    return eps == 0;
  }
  // executor x finished the current segment (D12, D13, D16); true: it has phase-A work due now
  __device__ bool advance_segment(uint32_t x) {
    const uint32_t c = S.exChain[x], sl = S.exSlot[x];
    InstRef I = S.ref(c, sl);
    const uint32_t j = S.cCb0[c] + I.cb;
    ev(EV_SEG_DONE, c, I.cb, S.exSeg[x], FULL, FULL);
    S.exSeg[x]++;
    if (S.exSeg[x] < S.bNseg[j]) return begin_segment(x);
    ev(EV_CB_DONE, c, I.cb, FULL, FULL, FULL);
    if (I.cb + 1u < S.cNcb[c]) {
      const uint32_t nx = S.bExec[j + 1];
      I.cb++;
      if (nx == x) I.state = I_READY;
      else { I.state = I_TRANSIT; I.ready_at = t32() + (uint32_t)comm; }
    } else {
      const uint64_t resp = t - (S.cPhase[c] + (uint64_t)I.k * S.cT[c]);  // D16
      atomicMax(&S.maxResp[c], (unsigned long long)resp);
      atomicAdd(&S.cnt[c], 1u);
      if (resp > S.cD[c]) atomicAdd(&S.miss[c], 1u);  // D16: deadline miss
      ev(EV_CHAIN_DONE, c, FULL, FULL, FULL, FULL);
      I.state = I_FREE;
    }
    S.exPhase[x] = P_NONE;
    S.exChain[x] = 0xff;
    return false;
  }
};

#ifndef SIM_MINB
#define SIM_MINB 16  // 16 blocks of 2 warps: 32 warps per SM (shared memory bounds it at 33)
#endif
__global__ void __launch_bounds__(SW * 32, SIM_MINB) simulate_kernel(paam_batch b, const Record* __restrict__ recs, uint32_t n,
                                                           uint64_t horizon, uint64_t seed, uint64_t first_index,
                                                           uint32_t sim_flags, paam_sim_out o,
                                                           unsigned int* __restrict__ ticket, uint4* __restrict__ evbuf) {
  uint64_t* __restrict__ out_resp = o.resp;
  uint64_t* __restrict__ out_count = o.count;
  uint64_t* __restrict__ out_digest = o.digest;
  const uint64_t* __restrict__ bound = o.bound;
  __shared__ DesSmem smem[SW];
  const uint32_t lane = threadIdx.x & 31;
  DesSmem& S = smem[threadIdx.x >> 5];
  // dynamic work distribution: a set's simulation cost varies by orders of magnitude (chains,
  // periods, horizon), so warps take one set per atomic ticket instead of a fixed stride
  auto next_set = [&]() {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1u);
    return __shfl_sync(0xffffffffu, t, 0);
  };
  for (uint32_t set = next_set(); set < n; set = next_set()) {
    const Record& rec = recs[set];
    const uint32_t c0 = b.set_chain_off[set], c1 = b.set_chain_off[set + 1];
    const uint32_t nch = c1 - c0;
    if (rec.status != PAAM_SET_OK) {
      for (uint32_t i = lane; i < nch; i += 32) {
        if (out_resp) out_resp[c0 + i] = 0;
        if (out_count) out_count[c0 + i] = 0;
        if (o.misses) o.misses[c0 + i] = 0;
        if (o.drops) o.drops[c0 + i] = 0;
      }
      if (lane == 0 && out_digest) out_digest[set] = 0;
      if (lane == 0 && o.status) o.status[set] = rec.status == REC_STATUS_WIDE ? PAAM_SIM_WIDE : PAAM_SIM_INVALID;
      continue;
    }
    const uint32_t x0 = b.set_exec_off[set], nex = b.set_exec_off[set + 1] - x0;
    const uint32_t a0 = b.set_accel_off[set], nac = b.set_accel_off[set + 1] - a0;
    const uint32_t cb0 = b.chain_cb_off[c0], ncb = b.chain_cb_off[c1] - cb0;
    const uint32_t sg0 = b.cb_seg_off[cb0], nseg = b.cb_seg_off[cb0 + ncb] - sg0;

    // ---- static staging ----------------------------------------------------------------------------
    // chains: rank = number of higher priorities
    uint32_t my_prio = lane < nch ? b.chain_prio[c0 + lane] : 0u, rank = 0;
    for (uint32_t d = 0; d < nch; d++) rank += (__shfl_sync(FULL, my_prio, d) > my_prio);
    uint32_t chain_of_rank_cb0 = 0;
    if (lane < nch) {
      const uint64_t T = b.chain_T[c0 + lane];
      S.cT[rank] = (uint32_t)T;
      S.cD[rank] = (uint32_t)b.chain_D[c0 + lane];
      S.cCls[rank] = b.chain_class[c0 + lane];
      S.cLocal[rank] = (uint8_t)lane;
      chain_of_rank_cb0 = b.chain_cb_off[c0 + lane] - cb0;
      S.cCb0[rank] = (uint8_t)chain_of_rank_cb0;
      S.cNcb[rank] = (uint8_t)(b.chain_cb_off[c0 + lane + 1] - cb0 - chain_of_rank_cb0);
      S.cPhase[rank] = pg_phase(seed, first_index + set, lane, T);  // D2
    }
    // executors: canonical order (core asc, process priority desc)
    uint32_t xcore = lane < nex ? b.exec_core[x0 + lane] : 0x100u + lane;
    uint32_t xprio = lane < nex ? b.exec_prio[x0 + lane] : 0u;
    uint32_t xpos = 0;
    for (uint32_t y = 0; y < nex; y++) {
      const uint32_t cy = __shfl_sync(FULL, xcore, y), py = __shfl_sync(FULL, xprio, y);
      xpos += (cy < xcore) || (cy == xcore && py > xprio);
    }
    __shared__ uint8_t xcanon_all[SW][MAXX];
    uint8_t* xcanon = xcanon_all[threadIdx.x >> 5];
    if (lane < nex) {
      xcanon[lane] = (uint8_t)xpos;
      S.xWait[xpos] = b.exec_wait[x0 + lane];
    }
    {
      const uint32_t same = __match_any_sync(FULL, xcore);
      // translate the same-core lane mask to canonical positions
      uint32_t m = 0;
      for (uint32_t y = 0; y < nex; y++) {
        const uint32_t py = __shfl_sync(FULL, xpos, y);  // every lane shuffles (no divergent shuffle)
        if ((same >> y) & 1u) m |= 1u << py;
      }
      if (lane < nex) S.xSameCore[xpos] = m;
    }
    __syncwarp();
    // accelerators / units
    __shared__ uint32_t ubase_all[SW][4];
    uint32_t* ubase = ubase_all[threadIdx.x >> 5];
    if (lane == 0) {
      uint32_t u = 0;
      for (uint32_t a = 0; a < nac; a++) {
        ubase[a] = u;
        const uint32_t nb = b.accel_buckets[a0 + a], nu = b.accel_units[a0 + a];
        const uint32_t e = (uint32_t)b.accel_eps[a0 + a];
        const uint32_t k = (nb > 1 && !(sim_flags & PAAM_SIM_FIFO_DIRECT)) ? (uint32_t)b.accel_kappa[a0 + a] : 0u;  // A6
        for (uint32_t v = 0; v < nu; v++, u++) { S.uEps[u] = e; S.uKap[u] = k; S.uN[u] = nb; }
      }
    }
    __syncwarp();
    const uint32_t n_unit = rec.n_unit;
    // callbacks and segments
    for (uint32_t j = lane; j < ncb; j += 32) {
      const uint32_t so = b.cb_seg_off[cb0 + j] - sg0;
      S.bExec[j] = xcanon[b.cb_exec[cb0 + j]];
      S.bSeg0[j] = (uint8_t)so;
      S.bNseg[j] = (uint8_t)(b.cb_seg_off[cb0 + j + 1] - sg0 - so);
    }
    for (uint32_t g = lane; g < nseg; g += 32) {
      const uint32_t kind = b.seg_kind[sg0 + g];
      S.gKind[g] = (uint8_t)kind;
      S.gW[g] = (uint32_t)b.seg_wcet[sg0 + g];
      S.gUnit[g] = kind == 1 ? (uint8_t)(ubase[b.seg_accel[sg0 + g]] + b.seg_unit[sg0 + g]) : (uint8_t)0;
    }
    __syncwarp();
    if ((b.flags & PAAM_FLAG_WFD_UNITS) && lane == 0) {  // WFD unit assignment, as pack_kernel
      uint64_t* wu = S.wfd.wu;
      uint8_t *wo = S.wfd.wo, *wn = S.wfd.wn, *wc = S.wfd.wc;
      for (uint32_t a = 0; a < nac; a++) {
        const uint32_t nu = b.accel_units[a0 + a];
        uint32_t ni = 0;
        for (uint32_t j = 0; j < ncb; j++) {
          uint32_t k = 0;
          for (uint32_t q = 0; q < nch; q++) if (S.cCb0[q] <= j && j < S.cCb0[q] + S.cNcb[q]) k = q;
          uint64_t A = 0;
          for (uint32_t g = S.bSeg0[j]; g < S.bSeg0[j] + S.bNseg[j]; g++)
            if (S.gKind[g] == 1 && b.seg_accel[sg0 + g] == a) A += S.gW[g];
          if (A) { wu[ni] = (A << 24) / S.cT[k]; wc[ni] = (uint8_t)j; ni++; }
        }
        wfd_place(ni, wu, nu, wo, wn);
        for (uint32_t i = 0; i < ni; i++) {
          const uint32_t j = wc[i];
          for (uint32_t g = S.bSeg0[j]; g < S.bSeg0[j] + S.bNseg[j]; g++)
            if (S.gKind[g] == 1 && b.seg_accel[sg0 + g] == a) S.gUnit[g] = (uint8_t)(ubase[a] + wn[i]);
        }
      }
    }
    __syncwarp();
    // buckets (A5): per accelerator, chains using it ranked by priority, groups of ceil(m_a/n)
    {
      uint32_t use = 0;  // lane = rank
      if (lane < nch) {
        for (uint32_t j = S.cCb0[lane]; j < S.cCb0[lane] + S.cNcb[lane]; j++)
          for (uint32_t g = S.bSeg0[j]; g < S.bSeg0[j] + S.bNseg[j]; g++)
            if (S.gKind[g] == 1) {
              uint32_t a = 0;
              for (uint32_t q = 1; q < nac; q++) if (ubase[q] <= S.gUnit[g]) a = q;
              use |= 1u << a;
            }
      }
      const uint32_t lt = lanemask_lt();
      uint32_t bk[4] = {0, 0, 0, 0};
      for (uint32_t a = 0; a < nac; a++) {
        const uint32_t U = __ballot_sync(FULL, (use >> a) & 1u);
        const uint32_t ma = __popc(U), nb = b.accel_buckets[a0 + a];
        const uint32_t gsz = ma ? (ma + nb - 1) / nb : 1u;
        bk[a] = nb - 1 - __popc(U & lt) / gsz;
      }
      if (lane < nch) {
        for (uint32_t j = S.cCb0[lane]; j < S.cCb0[lane] + S.cNcb[lane]; j++)
          for (uint32_t g = S.bSeg0[j]; g < S.bSeg0[j] + S.bNseg[j]; g++)
            if (S.gKind[g] == 1) {
              uint32_t a = 0;
              for (uint32_t q = 1; q < nac; q++) if (ubase[q] <= S.gUnit[g]) a = q;
              S.gBkt[g] = (sim_flags & PAAM_SIM_FIFO_DIRECT) ? (uint8_t)0 : (uint8_t)bk[a];
            }
        for (uint32_t u = 0; u < MAXU; u++) {
          uint32_t a = 0;
          for (uint32_t q = 1; q < nac; q++) if (ubase[q] <= u) a = q;
          S.cuBkt[lane][u] = (sim_flags & PAAM_SIM_FIFO_DIRECT) ? (uint8_t)0 : (uint8_t)bk[a];
        }
      }
    }
    // dynamic state
    if (lane < MAXC) {
      S.iState[lane] = rep4(I_FREE);
      S.iWUnit[lane] = rep4(NOQ);
      S.maxResp[lane] = 0;
      S.cnt[lane] = 0;
      S.miss[lane] = 0;
      S.exPhase[lane] = P_NONE;
      S.exChain[lane] = 0xff;
    }
    if (lane < MAXU) { S.unState[lane] = U_IDLE; S.uQ[lane] = 0; S.uDirty[lane] = 0; }
    if (lane == 0) S.evN = 0;
    __syncwarp();

    const bool fifo = (sim_flags & PAAM_SIM_FIFO_DIRECT) != 0;
    Ctx C{S, 0, horizon, b.comm_cost, 0, fifo, out_digest != nullptr && evbuf != nullptr,
          evbuf + ((size_t)blockIdx.x * SW + (threadIdx.x >> 5)) * EVCAP};
    uint32_t next_k = 0;  // lane = rank
    uint64_t next_rel = (uint32_t)lane < nch ? S.cPhase[lane] : NONE64;  // release time of instance next_k (D2)
    bool rel_live = (uint32_t)lane < nch && next_rel < horizon;  // a release is pending (below the horizon)
    uint32_t rel32 = (uint32_t)next_rel;                          // its low 32 bits (< 2^31 ahead of t)
    uint32_t seq = 0;     // warp-uniform
    bool on_core = false; // lane = canonical executor
    uint32_t drops = 0;
    uint32_t steps = 0;  // STEP_CAP < 2^32
    int32_t stop = PAAM_SIM_OK;  // warp-uniform: why the run stopped early (PAAM_SIM_BACKLOG / _STEPCAP)
    bool backlog = false;         // lane = chain: a release found every instance slot live
    const bool is_chain = lane < nch, is_exec = lane < nex, is_unit = lane < n_unit;
    // this lane's unit / executor / chain has an event due at the current t (set by the time advance from
    // the lane's own minima; a repeated pass of phase A runs with all three set)
    bool due_u = true, due_x = true, due_c = true;
    // lane-owned static facts of the set, kept in registers
    const uint32_t same_core = is_exec ? S.xSameCore[lane] : 0u;  // executors on this executor's core
    const uint32_t run_phases =  // phases (other than idle) in which this executor wants its core (D5)
        (1u << P_CPU) | (1u << P_EPS_SPIN) | ((is_exec && S.xWait[lane]) ? (1u << P_WAIT) : 0u);
    const bool preemptive = is_unit && S.uN[lane] > 1;  // a unit of a multi-bucket accelerator (D9)
    bool may_transit = false;  // chain lane: a callback of the chain is followed by one on another executor
    if (is_chain)
      for (uint32_t j = S.cCb0[lane]; j + 1 < (uint32_t)S.cCb0[lane] + S.cNcb[lane]; j++)
        may_transit |= S.bExec[j] != S.bExec[j + 1];
    const uint32_t one_x = is_chain ? 1u << S.bExec[S.cCb0[lane]] : 0u;  // its executor, if it has only one

    for (;;) {
      // ===================== settle time t (D15) =====================
      // A phase-A pass can leave work due at t only on an executor it advanced (a zero-length eps)
      // -- units settle in (1), transits made in (1)/(2) arrive in (3) of the same pass, and releases
      // are spaced by T -- and phase B can create due-now phase-A work only through a zero eps or
      // kappa.  Passes are repeated exactly when such work exists, so every skipped pass is a no-op.
      // The unit queues' occupancy (uQ) lets phase B skip units with no request to dispatch.
      bool run_a = true;
      for (;;) {
        while (run_a) {
          if (C.want_dig && C.must_flush()) C.flush(lane);
          // (1) units.  Only a unit whose phase end or completion is due at t has anything to do here.
          if (is_unit && due_u && S.unState[lane] != U_IDLE && S.unEnd[lane] == C.t32()) {
            const uint32_t u = lane;
            const uint32_t us = S.unState[u];
            if (us == U_SWOUT) S.unState[u] = U_IDLE;
            else if (us == U_SWIN) {
              S.unState[u] = U_RUN;
              S.unEnd[u] = C.t32() + S.ref(S.unChain[u], S.unSlot[u]).rem;  // > t: the rest of the request
              S.uDirty[u] = 1;
            } else if (us == U_RUN) {  // due: the request completes now
              const uint32_t c = S.unChain[u], sl = S.unSlot[u];
              InstRef I = S.ref(c, sl);
              const uint32_t j = S.cCb0[c] + I.cb;
              uint32_t x = S.bExec[j];
              // the request's segment: the executor's current segment
              const uint32_t g = S.bSeg0[j] + S.exSeg[x];
              C.ev(EV_ACC_DONE, c, I.cb, S.exSeg[x], u, S.gBkt[g]);
              I.wunit = NOQ;
              S.uQ[u]--;
              S.unState[u] = U_IDLE;
              C.advance_segment(x);  // the next segment is a CPU one or none: never due now
            }
          }
          __syncwarp();
          // (2) executors: CPU / eps completions; enqueues sequenced by (chain, instance) (D7)
          bool enq = false;
          uint32_t enq_key = 0xffffffffu;
          bool again_x = false;  // an executor (2) advanced is due again (its next segment is a zero-length eps)
          if (is_exec && due_x) {  // (1) leaves no executor due: a callback's next segment is never zero-length
            const uint32_t x = lane, ph = S.exPhase[x];
            if (ph == P_CPU && S.exRem[x] == 0) again_x = C.advance_segment(x);
            else if ((ph == P_EPS_SPIN && S.exRem[x] == 0) || (ph == P_EPS_SUSP && S.exTimer[x] == C.t32())) {
              S.exPhase[x] = P_WAIT;
              enq = true;
              enq_key = ((uint32_t)S.cLocal[S.exChain[x]] << 24) | (S.ref(S.exChain[x], S.exSlot[x]).k & 0xffffffu);
             
            }
          }
          // (2) served every executor that was due, and advance_segment(x) changes executor x only, so
          // only an executor (2) advanced can be due again; (3)/(4) leave executors alone
          const uint32_t enq_mask = __ballot_sync(FULL, enq);
          if (enq_mask) {
            uint32_t pos = 0;
            uint32_t mm = enq_mask;
            while (mm) {
              const uint32_t y = __ffs(mm) - 1;
              mm &= mm - 1;
              pos += (__shfl_sync(FULL, enq_key, y) < enq_key);
            }
            if (enq) {
              const uint32_t x = lane, c = S.exChain[x], sl = S.exSlot[x];
              InstRef I = S.ref(c, sl);
              const uint32_t g = S.bSeg0[S.cCb0[c] + I.cb] + S.exSeg[x];
              I.seq = seq + pos;
              I.wunit = S.gUnit[g];
              I.started = 0;
              atomicAdd(&S.uQ[S.gUnit[g]], 1u);
              S.uDirty[S.gUnit[g]] = 1;
              C.ev(EV_REQ_ENQUEUE, c, I.cb, S.exSeg[x], S.gUnit[g], S.gBkt[g]);
            }
            seq += __popc(enq_mask);
          }
          __syncwarp();
          // (3) comm arrivals, (4) releases (D2, D14)
          if (is_chain && due_c) {
            const uint32_t c = lane;
            if (may_transit)
              for (uint32_t tm = slots_eq(S.iState[c], I_TRANSIT); tm; tm &= tm - 1) {
                const uint32_t q = slot_of(tm);
                if (S.iw[c][q].ready_at == C.t32()) { byte_of(S.iState[c], q) = I_READY; }
              }
            if (rel_live && rel32 == C.t32()) {
              if (S.cCls[c] == 1)
                for (uint32_t dm = slots_eq(S.iState[c], I_READY) & slots_eq(S.iCb[c], 0); dm; dm &= dm - 1) {
                  byte_of(S.iState[c], slot_of(dm)) = I_FREE;
                  drops++;
                  C.ev(EV_DROP, c, FULL, FULL, FULL, FULL);
                }
              const uint32_t fm = slots_eq(S.iState[c], I_FREE);
              const int slot = fm ? (int)slot_of(fm) : -1;
              if (slot < 0) {
                backlog = true;  // D14: the new instance would be the chain's (QCAP+1)-th live one
              } else {
                InstRef I = S.ref(c, slot);
                I.state = I_READY; I.k = next_k; I.cb = 0; I.wunit = NOQ;
                C.ev(EV_RELEASE, c, FULL, FULL, FULL, FULL);
              }
              next_k++;
              next_rel += S.cT[c];
              rel_live = next_rel < horizon;
              rel32 = (uint32_t)next_rel;
            }
          }
          __syncwarp();
          // a backlog stop is checked only when the cheap vote fires (it almost never does)
          run_a = __any_sync(FULL, again_x || backlog);
          due_u = due_x = due_c = true;
          if (run_a && __any_sync(FULL, backlog)) { stop = PAAM_SIM_BACKLOG; goto sim_done; }
        }
        if (C.want_dig && C.must_flush()) C.flush(lane);
        // (5) executor choice (D4): per executor, the ready instance of the highest-priority chain
        bool needB = false, dueB = false;  // another phase-B pass could act / B left phase-A work due now
        uint32_t ready_x = 0;  // lane = rank: executors where this chain has a READY instance
        if (is_chain) {
          const uint32_t rm0 = slots_eq(S.iState[lane], I_READY);
          if (!may_transit) {
            ready_x = rm0 ? one_x : 0u;  // every callback of the chain runs on one executor
          } else {
            const uint32_t cbw = S.iCb[lane], cb0 = S.cCb0[lane];
            for (uint32_t rm = rm0; rm; rm &= rm - 1)
              ready_x |= 1u << S.bExec[cb0 + ((cbw >> (8 * slot_of(rm))) & 0xffu)];
          }
        }
        const uint32_t has_ready = __reduce_or_sync(FULL, ready_x);
        const uint32_t want = __ballot_sync(FULL, is_exec && on_core && S.exPhase[lane] == P_NONE && ((has_ready >> lane) & 1u));
        uint32_t wm = want;
        uint32_t hr = has_ready;  // (6) needs the chains' offers after (5)
        if (wm) {
        while (wm) {
          const uint32_t x = __ffs(wm) - 1;
          wm &= wm - 1;
          const uint32_t cand = __ballot_sync(FULL, (ready_x >> x) & 1u);
          const uint32_t c = __ffs(cand) - 1;
          if (lane == c) {
            int best = -1;
            const uint32_t cbw = S.iCb[c];
            for (uint32_t rm = slots_eq(S.iState[c], I_READY); rm; rm &= rm - 1) {
              const uint32_t q = slot_of(rm), qcb = (cbw >> (8 * q)) & 0xffu;
              if (S.bExec[S.cCb0[c] + qcb] != x) continue;
              if (best < 0) { best = (int)q; continue; }
              const uint32_t kq = S.iw[c][q].k, kb = S.iw[c][best].k;  // older release = smaller k
              if (kq < kb || (kq == kb && qcb < ((cbw >> (8 * best)) & 0xffu))) best = (int)q;
            }
            InstRef I = S.ref(c, best);
            I.state = I_RUN;
            S.exChain[x] = (uint8_t)c;
            S.exSlot[x] = (uint8_t)best;
            S.exSeg[x] = 0;
            C.ev(EV_CB_START, c, I.cb, 0, FULL, FULL);
            dueB |= C.begin_segment(x);
            // this chain no longer offers that instance
            ready_x = 0;
            {
              const uint32_t rm0 = slots_eq(S.iState[c], I_READY);
              if (!may_transit) {  // lane == c: this chain's own registers
                ready_x = rm0 ? one_x : 0u;
              } else {
                const uint32_t cbw2 = S.iCb[c], cb0 = S.cCb0[c];
                for (uint32_t rm = rm0; rm; rm &= rm - 1)
                  ready_x |= 1u << S.bExec[cb0 + ((cbw2 >> (8 * slot_of(rm))) & 0xffu)];
              }
            }
          }
          __syncwarp();
        }
        hr = __reduce_or_sync(FULL, ready_x);
        }
        // (6) core dispatch (D5): highest process priority runnable executor per core.  ready_x (hr) is
        // current: (5) recomputed it on every chain lane whose instance it started.
        {
          bool run = false;
          if (is_exec) {
            const uint32_t ph = S.exPhase[lane];
            run = ph == P_NONE ? ((hr >> lane) & 1u) : ((run_phases >> ph) & 1u);
          }
          const uint32_t R = __ballot_sync(FULL, run);
          const uint32_t cand = R & same_core;  // same_core = 0 on a lane that is no executor
          const bool oc = cand != 0 && (cand & (0u - cand)) == (1u << lane);  // the lowest is this lane
          // an executor that just got its core while idle with ready work is the only thing another
          // phase-B pass could act on ((5) serves every wanting executor once per pass; (7) units are
          // independent of each other)
          needB = oc && !on_core && is_exec && S.exPhase[lane] == P_NONE;
          on_core = oc;
        }
        // (7) unit dispatch (D8-D11).  Lane u decides whether unit u has anything to dispatch (queue
        // occupancy, state); only those units are visited (dispatch on one unit changes no other's).
        uint32_t umask;
        {
          bool cand = false;
          if (is_unit) {
            // an idle unit with requests always dispatches; a running one re-checks preemption (D9) only
            // if a request joined its queue or it resumed a request since its last check (otherwise the
            // check would repeat its last, negative, outcome)
            const uint32_t ust = S.unState[lane], q = S.uQ[lane];
            cand = fifo ? (ust == U_IDLE && q > 0)
                        : ((ust == U_IDLE && q > 0) || (ust == U_RUN && preemptive && q > 1 && S.uDirty[lane]));
            S.uDirty[lane] = 0;
          }
          umask = __ballot_sync(FULL, cand);
        }
        for (; umask; umask &= umask - 1) {
          const uint32_t u = __ffs(umask) - 1;
          const uint32_t ust = S.unState[u];
          if (fifo) {  // FIFO_DIRECT: an idle unit starts the oldest request; never preempts
            uint32_t myseq = 0xffffffffu;
            int fslot = -1;
            if (is_chain)
              for (uint32_t wm = slots_eq(S.iWUnit[lane], u); wm; wm &= wm - 1) {
                const uint32_t q = slot_of(wm);
                if (S.iw[lane][q].seq < myseq) { myseq = S.iw[lane][q].seq; fslot = (int)q; }
              }
            const uint32_t oldest = __reduce_min_sync(FULL, myseq);
            if (oldest == 0xffffffffu) continue;
            if (myseq == oldest) {
              InstRef I = S.ref(lane, fslot);
              const uint32_t j = S.cCb0[lane] + I.cb, x = S.bExec[j], seg = S.exSeg[x];
              S.unChain[u] = (uint8_t)lane;
              S.unSlot[u] = (uint8_t)fslot;
              I.started = 1;
              S.unState[u] = U_RUN;
              S.unEnd[u] = C.t32() + S.gW[S.bSeg0[j] + seg];
              C.ev(EV_ACC_START, lane, I.cb, seg, u, 0u);
            }
            __syncwarp();
            continue;
          }
          // best waiting request on u, excluding the running one: key = bucket | started | priority
          uint32_t key = 0;
          int bslot = -1;
          if (is_chain) {
            const uint32_t sw = S.iStarted[lane];
            for (uint32_t wm = slots_eq(S.iWUnit[lane], u); wm; wm &= wm - 1) {
              const int q = (int)slot_of(wm);
              if (ust == U_RUN && S.unChain[u] == lane && S.unSlot[u] == q) continue;
              if (bslot < 0) { bslot = q; continue; }
              const uint32_t sq = (sw >> (8 * q)) & 0xffu, sb = (sw >> (8 * bslot)) & 0xffu;
              if (sq != sb) { if (sq) bslot = q; }
              else if (S.iw[lane][q].seq < S.iw[lane][bslot].seq) bslot = q;
            }
            if (bslot >= 0) {
              InstRef I = S.ref(lane, bslot);
              const uint32_t bkt = S.cuBkt[lane][u];  // the bucket is per (chain, accelerator)
              key = 1u + ((bkt << 6) | ((uint32_t)I.started << 5) | (31u - lane));
            }
          }
          const uint32_t best = __reduce_max_sync(FULL, key);
          if (best == 0) continue;
          const uint32_t wc = 31u - ((best - 1u) & 31u);
          const uint32_t wbkt = (best - 1u) >> 6;
          if (lane == wc) {
            InstRef I = S.ref(wc, bslot);
            const uint32_t j = S.cCb0[wc] + I.cb;
            const uint32_t x = S.bExec[j];
            const uint32_t seg = S.exSeg[x];
            if (ust == U_IDLE) {
              S.unChain[u] = (uint8_t)wc;
              S.unSlot[u] = (uint8_t)bslot;
              if (I.started) {  // D10: switch back in
                S.unState[u] = U_SWIN;
                S.unEnd[u] = C.t32() + S.uKap[u];
                dueB |= S.uKap[u] == 0;
                C.ev(EV_ACC_RESUME, wc, I.cb, seg, u, wbkt);
              } else {
                I.started = 1;
                S.unState[u] = U_RUN;
                S.unEnd[u] = C.t32() + S.gW[S.bSeg0[j] + seg];
                C.ev(EV_ACC_START, wc, I.cb, seg, u, wbkt);
              }
            }
          }
          if (ust == U_RUN) {  // D9: preempt a lower bucket
            const uint32_t rc = S.unChain[u];
            InstRef R = S.ref(rc, S.unSlot[u]);
            const uint32_t rj = S.cCb0[rc] + R.cb, rx = S.bExec[rj], rseg = S.exSeg[rx];
            const uint32_t rbkt = S.gBkt[S.bSeg0[rj] + rseg];
            if (wbkt > rbkt) {
              if (lane == 0) {
                C.ev(EV_ACC_PREEMPT, rc, R.cb, rseg, u, rbkt);
                R.rem = S.unEnd[u] - C.t32();  // > 0: a request completing now finished in (1)
                S.unState[u] = U_SWOUT;
                S.unEnd[u] = C.t32() + S.uKap[u];
                dueB |= S.uKap[u] == 0;
              }
            }
          } else {
          }
          __syncwarp();
        }
        // the timestamp is settled unless B left phase-A work due now or gave an idle executor with
        // ready work its core (every other further A/B round would be a no-op)
        const uint32_t vb = __reduce_or_sync(FULL, (needB ? 1u : 0u) | (dueB ? 2u : 0u));
        if (!vb) break;
        run_a = (vb & 2u) != 0;
      }
      // ===================== advance time =====================
      // Every pending event lies less than 2^31 ns ahead (a period, eps, kappa, comm or remaining
      // work, each < 2^31 - 1 ns), so the next event is found as a 32-bit distance from t.
      uint32_t nd_c = 0xffffffffu, nd_x = 0xffffffffu, nd_u = 0xffffffffu;  // none
      bool run_x = false;  // executor whose remaining work shrinks with time
      if (is_chain) {
        if (rel_live) nd_c = rel32 - C.t32();
        if (may_transit)
          for (uint32_t tm = slots_eq(S.iState[lane], I_TRANSIT); tm; tm &= tm - 1)
            nd_c = min(nd_c, S.iw[lane][slot_of(tm)].ready_at - C.t32());
      }
      if (is_exec) {
        const uint32_t ph = S.exPhase[lane];
        run_x = (ph == P_CPU || ph == P_EPS_SPIN) && on_core;
        if (run_x) nd_x = S.exRem[lane];
        if (ph == P_EPS_SUSP) nd_x = S.exTimer[lane] - C.t32();
      }
      if (is_unit && S.unState[lane] != U_IDLE) nd_u = S.unEnd[lane] - C.t32();
      const uint32_t nd = __reduce_min_sync(FULL, min(nd_c, min(nd_x, nd_u)));
      if (nd == 0xffffffffu) break;
      // with comm = 0 a callback completing at t makes its successor arrive at t (D13), so every chain
      // lane checks its transits then
      due_c = nd_c == nd || C.comm == 0;
      due_x = nd_x == nd;
      due_u = nd_u == nd;
      if (++steps > STEP_CAP) { stop = PAAM_SIM_STEPCAP; break; }
      const uint64_t nt = C.t + nd;
      if (run_x) S.exRem[lane] -= nd;
      C.t = nt;
      __syncwarp();
    }

  sim_done:
    // ---- outputs ---------------------------------------------------------------------------------------
    // A stopped run's statistics cover the exact prefix up to the stop (lower bounds of the full run's);
    // its chains are not checked against the bound (census[stopped] counts it instead).
    if (C.want_dig) C.flush(lane);
    const uint64_t digest = warp_sum_u64(C.dig);
    bool viol = false, set_sched = bound != nullptr && stop == PAAM_SIM_OK;
    uint64_t bd = 0;
    if (is_chain) {
      const uint32_t local = S.cLocal[lane];
      if (out_resp) out_resp[c0 + local] = S.maxResp[lane];
      if (out_count) out_count[c0 + local] = S.cnt[lane];
      if (o.misses) o.misses[c0 + local] = S.miss[lane];
      if (o.drops) o.drops[c0 + local] = drops;
      if (bound) {
        bd = bound[c0 + local];
        if (S.cCls[lane] == 0 && (bd == PAAM_UNSCHED || bd > S.cD[lane])) set_sched = false;
        viol = S.cCls[lane] == 0 && S.maxResp[lane] > bd;
      }
    }
    set_sched = __all_sync(FULL, set_sched || !is_chain);
    const uint32_t vm = __ballot_sync(FULL, viol && set_sched);
    if (vm && o.violations) {  // sim > bound: count, and record the first max_witness witnesses
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd((unsigned long long*)o.violations, (unsigned long long)__popc(vm));
      base = __shfl_sync(FULL, base, 0);
      if ((vm >> lane) & 1u) {
        const unsigned long long w = base + __popc(vm & lanemask_lt());
        if (o.witness && w < o.max_witness) {
          o.witness[2 * w] = set;
          o.witness[2 * w + 1] = S.cLocal[lane];
        }
      }
    }
    if (lane == 0) {
      if (out_digest) out_digest[set] = digest;
      if (o.status) o.status[set] = stop;
      if (o.stopped && stop != PAAM_SIM_OK) atomicAdd((unsigned long long*)o.stopped, 1ull);
    }
    __syncwarp();
  }
}

}  // namespace

#ifndef PAAM_WARP_EMU
int launch_simulate(const paam_batch* b, const Record* rec, uint32_t n, uint64_t horizon, uint64_t seed,
                    uint64_t first_index, uint32_t sim_flags, const paam_sim_out* out, unsigned int* ticket,
                    void** scratch, size_t* scratch_bytes, cudaStream_t st) {
  if (n == 0) return PAAM_OK;
  cudaMemsetAsync(ticket, 0, sizeof(unsigned int), st);
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, simulate_kernel, SW * 32, 0);
  if (per_sm < 1) per_sm = 1;
  const uint32_t need = (n + SW - 1) / SW;
  const uint32_t cap = (uint32_t)sms * (uint32_t)per_sm;
  const uint32_t grid = need < cap ? need : cap;
  uint4* evbuf = nullptr;
  if (out->digest) {  // the event buffers of every resident warp (EVCAP records of 16 B each)
    const size_t bytes = (size_t)grid * SW * EVCAP * sizeof(uint4);
    if (*scratch_bytes < bytes) {
      if (*scratch) cudaFree(*scratch);
      *scratch = nullptr;
      *scratch_bytes = 0;
      const cudaError_t e = cudaMalloc(scratch, bytes);
      if (e != cudaSuccess) return fail_cuda(e, "simulate event buffers");
      *scratch_bytes = bytes;
    }
    evbuf = (uint4*)*scratch;
  }
  simulate_kernel<<<grid, SW * 32, 0, st>>>(*b, rec, n, horizon, seed, first_index, sim_flags, *out, ticket, evbuf);
  count_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PAAM_OK : fail_cuda(e, "simulate_kernel launch");
}

#endif  // PAAM_WARP_EMU

}  // namespace paam
