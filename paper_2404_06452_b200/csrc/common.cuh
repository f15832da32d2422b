// common.cuh -- device-side conventions of the PAAM product path (sm_100a).
//
// Integer time (A14): every input time is < 2^31 - 1 ns, every derived quantity is a u32 that
// saturates at SAT = 2^31 - 1.  Every cutoff (min(D, T)) is <= 2^31 - 2 < SAT, so a saturated value
// is "above every deadline" and no finite result or verdict can differ from exact u64 arithmetic.
// An unbounded Lemma-2 value (UNB) is represented by SAT as well: min(SAT, C) behaves exactly like
// the paper's min(UNB, C) because any C >= SAT is itself above the cutoff.
#pragma once
#include <cstddef>
#include <cstdint>
#ifdef PAAM_WARP_EMU
#include "../../tools/warp_emu/emu.h"  // host-side debugging emulation of the warp intrinsics
#else
#include <cuda_runtime.h>
#endif

#include "../../include/paam.h"

namespace paam {

#ifdef PAAM_WARP_EMU
#define PAAM_COLD
#else
#define PAAM_COLD __noinline__  // rarely taken paths: kept out of the hot loop's instruction stream
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
#endif

constexpr uint32_t SAT = 0x7FFFFFFFu;
constexpr uint64_t LIM = 0x7FFFFFFFull;  // the u32 kernels take the sets whose every time is < LIM (A14)

__device__ __forceinline__ uint32_t sadd(uint32_t a, uint32_t b) { return min(a + b, SAT); }  // a,b <= SAT

// Raw-batch loads for the u64 batch (C32 = false) or the compact batch (C32 = true, paam_batch32): a
// compact batch travels in a paam_batch whose pointers are paam_batch32's -- the times uint32_t,
// cb_exec uint8_t, seg_kind the packed segment byte kind | accel << 1 | unit << 3 (seg_accel / seg_unit
// unused).
template <bool C32>
__device__ __forceinline__ uint64_t ld_time(const uint64_t* p, size_t i) {
  if constexpr (C32) return reinterpret_cast<const uint32_t*>(p)[i];
  else return p[i];
}
template <bool C32>
__device__ __forceinline__ uint32_t ld_cb_exec(const paam_batch& b, size_t j) {
  if constexpr (C32) return reinterpret_cast<const uint8_t*>(b.cb_exec)[j];
  else return b.cb_exec[j];
}
template <bool C32>
__device__ __forceinline__ void ld_seg(const paam_batch& b, size_t g, uint32_t& kind, uint32_t& accel, uint32_t& unit) {
  if constexpr (C32) {
    const uint32_t m = b.seg_kind[g];
    kind = m & 1u; accel = (m >> 1) & 3u; unit = m >> 3;
  } else {
    kind = b.seg_kind[g]; accel = b.seg_accel[g]; unit = b.seg_unit[g];
  }
}
// x >> (z mod 32) in one funnel shift (wrap mode): a magic-division shift L = ceil(log2 T) <= 31 kept in
// the low 5 bits of a packed word (pTab.z, cMisc)
__device__ __forceinline__ uint32_t f_shr(uint32_t x, uint32_t z) { return __funnelshift_r(x, 0u, z); }
// the index of the highest set bit of m != 0 in one FLO (31 - __clz(m) compiles to three instructions)
__device__ __forceinline__ uint32_t f_hibit(uint32_t m) {
#ifdef PAAM_WARP_EMU
  return 31u - (uint32_t)__clz(m);
#else
  uint32_t i;
  asm("bfind.u32 %0, %1;" : "=r"(i) : "r"(m));
  return i;
#endif
}
__device__ __forceinline__ uint32_t smul(uint32_t a, uint32_t b) {
  const uint64_t p = (uint64_t)a * b;
  return p > SAT ? SAT : (uint32_t)p;
}

// mu(t) = ceil(t / T) + 1 (Lemma 1, Eq.2) for 1 <= t <= SAT, by multiply-high with the
// per-period constant (M, L) from make_magic: floor(n / T) = umulhi(2n, M) >> L for n < 2^31
// (Granlund-Montgomery with N = 31: M = ceil(2^(31+L) / T), L = ceil(log2 T)), and
// ceil(t / T) = floor((t - 1) / T) + 1 for t >= 1.
__device__ __forceinline__ uint32_t mu_magic(uint32_t t, uint32_t M, uint32_t L) {
  return (__umulhi((t - 1u) << 1, M) >> L) + 2u;
}
__host__ __device__ inline void make_magic(uint32_t T, uint32_t* M, uint32_t* L) {
#ifdef __CUDA_ARCH__
  const uint32_t l = T > 1 ? 32u - __clz(T - 1u) : 0u;  // ceil(log2 T)
  const uint64_t N = 1ull << (31 + l);
  // M = ceil(N / T): double reciprocal estimate (< 2^33, off by at most a few), then exact fix-up
  uint64_t m = (uint64_t)((double)N * __drcp_rn((double)T));
  while (m * T < N) m++;
  while (m > 0 && (m - 1) * T >= N) m--;
  *L = l;
  *M = (uint32_t)m;
#else
  uint32_t l = 0;
  while (l < 32 && (1ull << l) < T) l++;  // l = ceil(log2 T)
  *L = l;
  *M = (uint32_t)(((1ull << (31 + l)) + T - 1) / T);
#endif
}

// Worst-Fit-Decreasing unit assignment (flag PAAM_FLAG_WFD_UNITS), run by one
// lane: items (one per callback using accelerator a, in callback order) with utilisation key
// u = (sum A << 24) / T are taken by decreasing u (stable), each onto the least-loaded unit of a
// (ties: lowest unit).  Writes the chosen unit (0-based within a) to unit_of[item].
__device__ inline void wfd_place(uint32_t n_items, const uint64_t* u, uint32_t n_units, uint8_t* order, uint8_t* unit_of) {
  for (uint32_t i = 0; i < n_items; i++) order[i] = (uint8_t)i;
  for (uint32_t i = 1; i < n_items; i++) {  // stable insertion sort by u desc
    const uint8_t v = order[i];
    int k = (int)i - 1;
    while (k >= 0 && u[order[k]] < u[v]) { order[k + 1] = order[k]; k--; }
    order[k + 1] = v;
  }
  uint64_t load[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (uint32_t i = 0; i < n_items; i++) {
    const uint32_t it = order[i];
    uint32_t best = 0;
    for (uint32_t k = 1; k < n_units; k++) if (load[k] < load[best]) best = k;
    load[best] += u[it];
    unit_of[it] = (uint8_t)best;
  }
}

// ---- packed per-set record (written by pack.cu, read by analyze.cu / simulate.cu) ------------------
// Fixed stride, structure-of-arrays inside the record; everything a warp needs is one contiguous
// 16-byte-aligned block that it bulk-loads into shared memory.
constexpr int MAXC = 32;   // chains
constexpr int MAXS = 32;   // sub-chains
constexpr int MAXA = 64;   // accelerator segments
constexpr int MAXU = 8;    // accelerator units (all accelerators of the set)
constexpr int MAXX = 32;   // executors
constexpr int MAXCB = 64;  // callbacks
constexpr uint64_t LIMW = 1ull << 48;   // every input time must be < LIMW (else PAAM_SET_ERANGE); times >= LIM go
                                        // to the exact u64 path (wide.cu)
constexpr int32_t REC_STATUS_WIDE = 0x100;  // internal status: handed over to wide.cu

struct __align__(16) Record {
  // header
  uint8_t n_chain, n_sub, n_aseg, n_unit;
  int32_t status;       // PAAM_SET_*
  uint32_t chain_base;  // global index of the set's first chain (out_wcrt position)
  uint32_t bin;         // utilisation bin (0 when the batch has none)
  uint32_t n_out;       // chains of the set in the batch (== n_chain when valid)
  uint32_t hflags;      // reserved (0)
  uint32_t pad_[2];
  // chains by rank (rank 0 = highest priority)
  uint32_t cCut[MAXC];   // cutoff min(D, T) (A4, A12)
  uint32_t cD[MAXC];     // deadline (verdict)
  uint32_t cM[MAXC];     // mu magic multiplier for T
  uint32_t cMisc[MAXC];  // L (5 bits) | class << 8 | local index << 16 | n_sub << 24
  // the chains in period order (ascending T, ties by rank): mu(R, T) = 2 + floor((R-1)/T), and the
  // floor is non-zero only for T < R, so an Eq.5 iterate walks this list up to the first T >= R.
  // One 16-byte entry: {T, mu magic multiplier M, L | rank << 8, W[rank][0] + W[rank][1] (saturated)}
  uint4 pTab[MAXC];
  // W[k][u]: sum of A* of chain rank k's segments on unit u (exact regrouping of Eq.3/Eq.4 sums);
  // rank-major so that lanes reading different units of one chain hit different banks
  uint32_t W[MAXC][MAXU];
  // sub-chains in canonical analysis order (per core: process priority desc, chain rank asc; A7)
  uint32_t sE[MAXS];      // calligraphic E_c
  uint32_t sB[MAXS];      // B_c as written
  uint32_t sEps[MAXS];    // sum of eps over the sub-chain's segments (delta_c * eps, A11)
  uint32_t sHp[MAXS];     // bit h: h in hp(c)
  uint32_t sHpp[MAXS];    // bit h: h in hpp(c)
  uint32_t sLp[MAXS];     // bit h: h in lp(c) (PAAM_FLAG_BLOCKING_SOUND only)
  uint32_t sMisc[MAXS];   // rank | unitmask << 8 | spin << 16 | chain-position << 24
  uint32_t sSeg[MAXS];    // first accelerator segment | count << 8 | exec << 16 | core << 24
  uint32_t sA2[MAXS];     // Eq.4 with every mu = 2: base3 + 2 sum_{k<rank} sum_{u in units} W[k][u]
  uint32_t sSlb[MAXS];    // sum of the Lemma-2 start values aBase2 of the sub-chain's segments (<= S_c)
  // accelerator segments in chain-rank order (a sub-chain's segments are contiguous)
  uint32_t aBase2[MAXA];  // A* + LPB + 2 sum_{k<r} W[k][u]: Eq.3 with mu = floor((h-1)/T) + 2 split off
  uint32_t aMisc[MAXA];   // rank | unit << 8 | sub << 16 | callback << 24
  // written and read only under PAAM_FLAG_BLOCKING_SOUND (the sound B_c of reading A10)
  uint32_t aEps[MAXA];    // eps of the segment's accelerator
  uint32_t aCbE[MAXA];    // E_j of the segment's callback
};
static_assert(sizeof(Record) % 16 == 0, "record must be 16-byte aligned");
static_assert(offsetof(Record, W) % 16 == 0, "W rows are copied as 16-byte vectors");

// ---- launch bookkeeping ---------------------------------------------------------------------------
#ifndef PAAM_WARP_EMU
void count_launch();
int fail_cuda(cudaError_t e, const char* what);
int fail(int code, const char* what);

// launchers (defined in the kernel files)
// wide_count[1] is the kernel's work ticket: the caller zeroes wide_count[0..1] before the launch
int launch_pack(const paam_batch* dev_batch_fields, Record* rec, int32_t* status, uint32_t* wide_list,
                uint32_t* wide_count, cudaStream_t st);
// ticket: one device counter (zeroed by the launcher on `st`) for dynamic work distribution
int launch_analyze(const Record* rec, uint32_t n, uint64_t comm, uint32_t flags, uint32_t n_bins,
                   uint64_t* out_wcrt, uint8_t* out_sched, int64_t* out_bins, unsigned int* ticket,
                   cudaStream_t st, int32_t* out_fail = nullptr);
// §8(a) steps 2-6 in one kernel (fused.cu): no record is written
// c32: b carries a compact batch (paam_batch32, see ld_time).  wide_count[1] is the kernel's work ticket:
// the caller zeroes wide_count[0..1] on the stream before the launch.
int launch_fused(const paam_batch* b, uint32_t* wide_list, uint32_t* wide_count, int32_t* status, uint64_t* out_wcrt,
                 uint8_t* out_sched, int64_t* out_bins, cudaStream_t st, bool c32 = false);
// the exact u64 path over the sets listed by the u32 kernels (wide.cu); out_fail: admission decisions
int launch_wide(const paam_batch* b, const uint32_t* list, const uint32_t* count, int32_t* status, uint64_t* out_wcrt,
                uint8_t* out_sched, int64_t* out_bins, int32_t* out_fail, cudaStream_t st, bool c32 = false);
// scratch / scratch_bytes: the caller's device scratch for the DES event buffers (grown on demand)
int launch_simulate(const paam_batch* b, const Record* rec, uint32_t n, uint64_t horizon, uint64_t seed,
                    uint64_t first_index, uint32_t sim_flags, const paam_sim_out* out, unsigned int* ticket,
                    void** scratch, size_t* scratch_bytes, cudaStream_t st);
#endif

}  // namespace paam
