// generate.cu -- §8(a) step 1: device-side synthetic chain-set generation (paam_generate).
//
// The workload recipe is gen/paam_gen.h (input generation only -- it holds none of the analysed
// method).  Pass 1 sizes every set (pg_set_sizes: only the draws that decide sizes, one thread per
// set), five exclusive scans turn the sizes into CSR offsets, and pass 2 writes every set at its
// offsets.  Pass 2 is a warp-per-set re-implementation of pg_generate_set + pg_write_set: the same
// counter-based draws (each a pure function of (seed, set, purpose, index)) and the same integer
// steps, spread over lanes (lane = chain, lane = callback, lane = executor) so that the writes are
// coalesced and no per-thread set image lives in local memory; the short inherently sequential
// steps (Fisher-Yates swaps, worst-fit placement) run on lane 0 over shared memory.  The bytes equal
// the host generator's (tests/test_gpu_parity.py::test_device_generator_matches_host_bytes).
// Ranks generate disjoint index ranges with no communication.
#include <cstdlib>
#include <cstring>

#include "../../gen/paam_gen.h"
#include "common.cuh"

struct paam_raw {
  paam_batch b;
  void* buf;       // every array of the batch (capacity `bytes`)
  size_t bytes;
  void* scr;       // sizes / offsets / scan scratch (capacity `scr_bytes`)
  size_t scr_bytes;
  int device;
};

namespace paam {
namespace {

__global__ void gen_sizes_kernel(pg_params p, uint64_t seed, uint64_t first, uint32_t n, uint32_t* __restrict__ cnt) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t z[5];
  pg_set_sizes(&p, seed, first + i, z);
#pragma unroll
  for (int k = 0; k < 5; k++) cnt[k * (size_t)n + i] = z[k];
}

constexpr int GW = 4;  // warps per block of the fill kernel

// floor(x / d), exactly, without the 64-bit integer divide routine when both operands are exact
// doubles: the correctly rounded double quotient is within 1 of the true one, and one integer step
// corrects it.
__device__ __forceinline__ uint64_t udiv64(uint64_t x, uint64_t d) {
  if (x < (1ull << 52) && d < (1ull << 52)) {
    uint64_t q = (uint64_t)__ddiv_rn((double)x, (double)d);
    if (q * d > x) q--;
    else if ((q + 1) * d <= x) q++;
    return q;
  }
  return x / d;
}
constexpr uint32_t FULL = 0xffffffffu;

struct GenWarp {
  uint64_t ccpu[PG_MAX_CHAINS];   // CPU WCET per chain
  uint32_t sorted[PG_MAX_CHAINS]; // sorted cut points
  uint32_t prio[PG_MAX_CHAINS];
  uint32_t pk[PG_MAX_CHAINS];     // Fisher-Yates draw of step j
  uint8_t order[PG_MAX_CHAINS];   // chains by utilisation desc, index asc
  uint8_t best[PG_MAX_CHAINS], second[PG_MAX_CHAINS], split[PG_MAX_CHAINS];
};

// Lowest lane holding the minimum of v over the lanes with `valid` (worst-fit's "least loaded,
// ties to the lowest index").
__device__ __forceinline__ uint32_t argmin_lane(uint64_t v, bool valid) {
  const uint64_t x = valid ? v : ~0ull;
  const uint32_t hi = __reduce_min_sync(FULL, (uint32_t)(x >> 32));
  const uint32_t lo = __reduce_min_sync(FULL, (uint32_t)(x >> 32) == hi ? (uint32_t)x : 0xffffffffu);
  return __ffs(__ballot_sync(FULL, valid && (uint32_t)(x >> 32) == hi && (uint32_t)x == lo)) - 1;
}

// Warp-per-set generation; mirrors pg_generate_set + pg_write_set step for step (same draws, same
// integer expressions, same tie rules).
__global__ void __launch_bounds__(GW * 32) gen_fill_kernel(pg_params p, uint64_t seed, uint64_t first, uint32_t n,
                                                        pg_arrays o, const uint32_t* __restrict__ cb_off,
                                                        const uint32_t* __restrict__ sg_off) {
  __shared__ GenWarp smem[GW];
  GenWarp& w = smem[threadIdx.x >> 5];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t K = p.cbs_per_chain;
  const uint32_t invK = 65536u / K + 1u;  // cb / K == (cb * invK) >> 16 for cb < 64, K <= 32 (exhaustive check)
  const uint32_t units[PG_MAX_ACCEL] = {p.units[0], p.units[1], p.units[2], p.units[3]};
  for (uint32_t i = blockIdx.x * GW + (threadIdx.x >> 5); i < n; i += gridDim.x * GW) {
    const uint64_t index = first + i;
    const uint64_t key = pg_key(seed, index);
    const uint32_t bin = p.n_bins ? (uint32_t)(index % p.n_bins) : 0u;
    const uint64_t U = (uint64_t)p.u_lo_q20 + (uint64_t)bin * p.u_step_q20;
    const uint32_t m = p.m_lo + pg_bounded(pg_draw(key, PG_D_M, 0), p.m_hi - p.m_lo + 1);
    const bool isc = lane < m;
    const uint32_t ch0 = o.set_chain_off[i], cb0 = cb_off[i], sg0 = sg_off[i];
    const uint32_t ex0 = o.set_exec_off[i], ac0 = o.set_accel_off[i];

    // per-chain utilisation: the m-1 cut points, sorted (equal cut values are interchangeable)
    const bool iscut = lane + 1 < m;
    const uint32_t cutv = iscut ? pg_bounded(pg_draw(key, PG_D_CUT, lane), (uint32_t)U + 1u) : 0u;
    {
      uint32_t rk = 0;
      for (uint32_t j = 0; j + 1 < m; j++) {
        const uint32_t cj = __shfl_sync(FULL, cutv, j);
        rk += (cj < cutv) || (cj == cutv && j < lane);
      }
      if (iscut) w.sorted[rk] = cutv;
      if (isc) w.ccpu[lane] = 0;
    }
    __syncwarp();
    uint64_t share = 0, T = 0;
    if (isc) {
      const uint64_t hi = iscut ? (uint64_t)w.sorted[lane] : U;
      share = hi - (lane > 0 ? (uint64_t)w.sorted[lane - 1] : 0ull);
      // log-uniform period rounded to 1 us; D = T
      const uint32_t x = pg_bounded(pg_draw(key, PG_D_PERIOD, lane), p.period_span_q12 + 1);
      const uint32_t oct = x >> 12, frac = x & 4095u;
      uint64_t t_us = (((uint64_t)p.period_min_us * PG_TABLE(frac)) << oct) >> 30;
      if (t_us < 1) t_us = 1;
      T = t_us * 1000ull;
    }
    const uint64_t C = (share * T) >> 20;
    const uint64_t base = udiv64(C, K), rem = C - base * K;

    // callbacks (lane = callback, passes of 32): budget, segments, accelerator and unit draws
    const uint32_t ncb = m * K;
    uint32_t carry = 0;
    for (uint32_t pass = 0; pass * 32 < ncb; pass++) {
      const uint32_t cb = pass * 32 + lane;
      const bool iscb = cb < ncb;
      const uint32_t c = iscb ? (cb * invK) >> 16 : 0u, j = iscb ? cb - c * K : 0u;
      const uint64_t bc = __shfl_sync(FULL, base, c), rc = __shfl_sync(FULL, rem, c);
      const uint64_t budget = bc + (j < rc ? 1 : 0);
      uint32_t nseg = 0, acc = 0, unit = 0;
      uint64_t w0 = 0, w1 = 0, w2 = 0;
      if (iscb) {
        if (p.cpu_only_frac_q16 && pg_coin(pg_draw(key, PG_D_CPUONLY, cb), p.cpu_only_frac_q16)) {
          nseg = 1;
          w0 = budget ? budget : 1;
          atomicAdd((unsigned long long*)&w.ccpu[c], (unsigned long long)w0);
        } else {
          uint64_t A = udiv64(budget * p.ratio_acc, (uint32_t)(p.ratio_acc + p.ratio_cpu));
          uint64_t E = budget - A;
          uint64_t e1 = E / 2, e2 = E - E / 2;
          nseg = 3;
          w0 = e1 ? e1 : 1;
          w1 = A ? A : 1;
          w2 = e2 ? e2 : 1;
          acc = pg_bounded(pg_draw(key, PG_D_ACC, cb), p.n_accel);
          unit = pg_bounded(pg_draw(key, PG_D_UNIT, cb), units[acc]);
          atomicAdd((unsigned long long*)&w.ccpu[c], (unsigned long long)(w0 + w2));
        }
      }
      uint32_t incl = nseg;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, d);
        if (lane >= (uint32_t)d) incl += y;
      }
      const uint32_t sg = sg0 + carry + incl - nseg;
      carry += __shfl_sync(FULL, incl, 31);
      if (iscb) {
        o.cb_seg_off[cb0 + cb] = sg;
        if (nseg == 1) {
          o.seg_kind[sg] = 0; o.seg_wcet[sg] = w0; o.seg_accel[sg] = 0; o.seg_unit[sg] = 0;
        } else {
          o.seg_kind[sg] = 0; o.seg_wcet[sg] = w0; o.seg_accel[sg] = 0; o.seg_unit[sg] = 0;
          o.seg_kind[sg + 1] = 1; o.seg_wcet[sg + 1] = w1; o.seg_accel[sg + 1] = (uint8_t)acc; o.seg_unit[sg + 1] = (uint8_t)unit;
          o.seg_kind[sg + 2] = 0; o.seg_wcet[sg + 2] = w2; o.seg_accel[sg + 2] = 0; o.seg_unit[sg + 2] = 0;
        }
      }
    }
    __syncwarp();

    // unique priorities: rate-monotonic, or the CAPA-random Fisher-Yates permutation
    uint32_t prio = 0;
    if (p.rm_priorities) {
      uint32_t rank = 0;
      for (uint32_t d = 0; d < m; d++) {
        const uint64_t Td = __shfl_sync(FULL, T, d);
        rank += (Td < T) || (Td == T && d < lane);
      }
      prio = m - rank;
    } else {
      if (isc) {
        w.prio[lane] = lane + 1;
        w.pk[lane] = lane >= 1 ? pg_bounded(pg_draw(key, PG_D_PERM, lane), lane + 1) : 0u;
      }
      __syncwarp();
      if (lane == 0)
        for (uint32_t j = m - 1; j >= 1; j--) {
          const uint32_t k = w.pk[j], t = w.prio[j];
          w.prio[j] = w.prio[k];
          w.prio[k] = t;
        }
      __syncwarp();
      prio = isc ? w.prio[lane] : 0u;
    }
    const uint32_t n_be = (uint32_t)(((uint64_t)m * p.be_frac_q16) >> 16);

    // CPU utilisation and the worst-fit order (utilisation desc, index asc)
    const uint64_t util = isc ? udiv64(w.ccpu[lane] << 20, T) : 0ull;
    {
      uint32_t rk = 0;
      for (uint32_t d = 0; d < m; d++) {
        const uint64_t ud = __shfl_sync(FULL, util, d);
        rk += (ud > util) || (ud == util && d < lane);
      }
      if (isc) w.order[rk] = (uint8_t)lane;
    }
    __syncwarp();
    // Worst-fit placement in the order above; lane k holds the load of core / executor k, and each
    // step's least-loaded target (ties: lowest index, as the host loop) is a warp argmin.
    uint32_t n_exec, n_client, my_best = 0;
    uint64_t ld = 0;
    if (p.exec_mode == 0) {  // one executor per chain, worst-fit onto the client cores
      for (uint32_t jj = 0; jj < m; jj++) {
        const uint32_t c = w.order[jj];
        const uint64_t uc = __shfl_sync(FULL, util, c);
        const uint32_t best = argmin_lane(ld, lane < p.n_cores);
        if (lane == best) ld += uc;
        if (lane == c) my_best = best;
      }
      n_exec = m;
      n_client = p.n_cores;
    } else {  // n_exec single-threaded executors on their own cores; some chains split across two
      const uint32_t X = p.n_exec;
      const bool my_split = isc && p.xexec_frac_q16 && K >= 2 && pg_coin(pg_draw(key, PG_D_XEXEC, lane), p.xexec_frac_q16);
      uint32_t my_second = 0;
      for (uint32_t jj = 0; jj < m; jj++) {
        const uint32_t c = w.order[jj];
        const uint64_t uc = __shfl_sync(FULL, util, c);
        const bool split = __shfl_sync(FULL, (uint32_t)my_split, c) != 0;
        const uint32_t best = argmin_lane(ld, lane < X);
        if (!split) {
          if (lane == best) ld += uc;
        } else {
          const uint32_t second = argmin_lane(ld, lane < X && lane != best);
          if (lane == best) ld += uc / 2;
          if (lane == second) ld += uc - uc / 2;
          if (lane == c) my_second = second;
        }
        if (lane == c) my_best = best;
      }
      if (isc) { w.best[lane] = (uint8_t)my_best; w.second[lane] = (uint8_t)my_second; w.split[lane] = (uint8_t)my_split; }
      n_exec = X;
      n_client = X;
    }
    __syncwarp();

    // ---- writes (coalesced by lane) ----
    if (lane == 0 && o.set_bin) o.set_bin[i] = bin;
    if (isc) {
      o.chain_T[ch0 + lane] = T;
      o.chain_D[ch0 + lane] = T;
      o.chain_prio[ch0 + lane] = prio;
      o.chain_class[ch0 + lane] = (prio <= n_be) ? 1 : 0;
      o.chain_cb_off[ch0 + lane] = cb0 + lane * K;
    }
    for (uint32_t cb = lane; cb < ncb; cb += 32) {
      const uint32_t c = (cb * invK) >> 16, j = cb - c * K;
      uint32_t x;
      if (p.exec_mode == 0) x = c;
      else x = (w.split[c] && j >= (K + 1) / 2) ? w.second[c] : w.best[c];
      o.cb_exec[cb0 + cb] = (uint16_t)x;
    }
    if (lane < n_exec) {
      const uint32_t pr = (p.exec_mode == 0) ? prio : lane + 1;
      o.exec_core[ex0 + lane] = (p.exec_mode == 0) ? (uint8_t)my_best : (uint8_t)lane;
      o.exec_prio[ex0 + lane] = pr;
      o.exec_wait[ex0 + lane] = (uint8_t)(p.spin_frac_q16 && pg_coin(pg_draw(key, PG_D_SPIN, lane), p.spin_frac_q16));
    }
    if (lane < p.n_accel) {
      o.accel_buckets[ac0 + lane] = (uint8_t)p.buckets[lane];
      o.accel_units[ac0 + lane] = (uint8_t)units[lane];
      o.accel_server_core[ac0 + lane] = (uint8_t)(n_client + lane);
      o.accel_eps[ac0 + lane] = p.eps[lane];
      o.accel_kappa[ac0 + lane] = p.kappa[lane];
    }
    if (i == n - 1 && lane == 0) {  // CSR sentinels
      o.chain_cb_off[o.set_chain_off[n]] = cb_off[n];
      o.cb_seg_off[cb_off[n]] = sg_off[n];
    }
    __syncwarp();
  }
}

// ---- exclusive scan of u32 counts into [n+1] offsets (block scan + recursive block sums) -------------
constexpr int SB = 1024;

__global__ void scan_block_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint32_t n,
                                  uint32_t* __restrict__ block_sums) {
  __shared__ uint32_t warp_tot[SB / 32];
  const uint32_t i = blockIdx.x * SB + threadIdx.x;
  const uint32_t v = i < n ? in[i] : 0u;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t t = warp_tot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_tot[lane] = t;  // inclusive over warps
  }
  __syncthreads();
  const uint32_t excl = x - v + (wid > 0 ? warp_tot[wid - 1] : 0u);
  if (i < n) out[i] = excl;
  if (threadIdx.x == SB - 1) block_sums[blockIdx.x] = excl + v;
}

__global__ void scan_add_kernel(uint32_t* __restrict__ out, uint32_t n, const uint32_t* __restrict__ block_offs) {
  const uint32_t i = blockIdx.x * SB + threadIdx.x;
  if (i < n) out[i] += block_offs[blockIdx.x];
}

__global__ void set_total_kernel(uint32_t* out, uint32_t n, const uint32_t* in) {
  out[n] = (n ? out[n - 1] + in[n - 1] : 0u);
}

// out[0..n] = exclusive scan of in[0..n), out[n] = total.  `tmp` needs scan_tmp_words(n) words.
size_t scan_tmp_words(uint32_t n) {
  size_t words = 0;
  for (;;) {  // per level: nb block sums + (nb + 1) scanned offsets, then recurse on nb
    const uint32_t nb = (n + SB - 1) / SB;
    words += 2 * (size_t)nb + 1;
    if (nb <= 1) break;
    n = nb;
  }
  return words + 2;
}

void scan_rec(const uint32_t* in, uint32_t* out, uint32_t n, uint32_t* tmp, cudaStream_t st) {
  if (n == 0) return;
  const uint32_t nb = (n + SB - 1) / SB;
  uint32_t* sums = tmp;
  uint32_t* offs = tmp + nb;
  scan_block_kernel<<<nb, SB, 0, st>>>(in, out, n, sums);
  count_launch();
  if (nb > 1) {
    scan_rec(sums, offs, nb, offs + nb + 1, st);
    scan_add_kernel<<<nb, SB, 0, st>>>(out, n, offs);
    count_launch();
  }
}

void scan(const uint32_t* in, uint32_t* out, uint32_t n, uint32_t* tmp, cudaStream_t st) {
  scan_rec(in, out, n, tmp, st);
  set_total_kernel<<<1, 1, 0, st>>>(out, n, in);
  count_launch();
}

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace
}  // namespace paam

using namespace paam;

namespace paam {
namespace {

// Per-set upper bounds of the generator's sizes {chains, callbacks, segments, executors, accelerators}.
void size_caps(const pg_params& p, uint64_t cap[5]) {
  cap[0] = p.m_hi;
  cap[1] = (uint64_t)p.m_hi * p.cbs_per_chain;
  cap[2] = 3ull * p.m_hi * p.cbs_per_chain;
  cap[3] = p.exec_mode == 0 ? p.m_hi : p.n_exec;
  cap[4] = p.n_accel;
}

// Generate into `raw`, reusing its device buffers when the new batch fits (paam_regenerate).
// cap_sets > 0: lay the arrays out for cap_sets sets at the generator's per-set upper bounds instead
// of reading the totals back -- no host synchronisation (paam_sweep); the batch's totals are then
// those capacities, which no kernel reads.
int generate_into(paam_raw* raw, const pg_params& p, uint64_t seed, uint64_t first_index, uint32_t n,
                  uint64_t comm_cost, uint32_t flags, cudaStream_t st, uint32_t cap_sets = 0) {
  cudaError_t e;
  // pass 1: sizes, then offsets (scratch: cnt[5n], offs[5(n+1)], scan temporaries)
  const size_t nn = (size_t)n + 1;
  const size_t scr_words = 5 * (size_t)(n ? n : 1) + 5 * nn + scan_tmp_words(n);
  if (raw->scr_bytes < 4 * scr_words) {
    if (raw->scr) cudaFree(raw->scr);
    raw->scr = nullptr;
    raw->scr_bytes = 0;
    if ((e = cudaMalloc(&raw->scr, 4 * scr_words)) != cudaSuccess) return fail_cuda(e, "paam_generate: scratch cudaMalloc");
    raw->scr_bytes = 4 * scr_words;
  }
  uint32_t* cnt = (uint32_t*)raw->scr;
  uint32_t* offs = cnt + 5 * (size_t)(n ? n : 1);
  uint32_t* tmp = offs + 5 * nn;
  if (n) {
    gen_sizes_kernel<<<(n + 127) / 128, 128, 0, st>>>(p, seed, first_index, n, cnt);
    count_launch();
  }
  for (int k = 0; k < 5; k++) scan(cnt + (size_t)k * n, offs + (size_t)k * nn, n, tmp, st);
  uint32_t tot[5];
  if (cap_sets) {
    uint64_t cap[5];
    size_caps(p, cap);
    for (int k = 0; k < 5; k++) tot[k] = (uint32_t)(cap[k] * cap_sets);
  } else {
    for (int k = 0; k < 5; k++)
      cudaMemcpyAsync(&tot[k], offs + (size_t)k * nn + n, sizeof(uint32_t), cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return fail_cuda(e, "paam_generate: sizes");
  }

  // one allocation for every array of the raw batch
  const uint32_t nch = tot[0], ncb = tot[1], nsg = tot[2], nex = tot[3], nac = tot[4];
  const size_t nset = cap_sets ? (size_t)cap_sets + 1 : nn;
  struct Part { size_t elems, size; } parts[] = {
      {nset, 4}, {nset, 4}, {nset, 4},                            // set offsets
      {nch, 8}, {nch, 8}, {nch, 4}, {nch, 1}, {(size_t)nch + 1, 4},  // chains
      {ncb, 2}, {(size_t)ncb + 1, 4},                              // callbacks
      {nsg, 1}, {nsg, 8}, {nsg, 1}, {nsg, 1},                      // segments
      {nex, 1}, {nex, 4}, {nex, 1},                                // executors
      {nac, 1}, {nac, 1}, {nac, 1}, {nac, 8}, {nac, 8},            // accelerators
      {nset, 4}};                                                  // set_bin
  constexpr int NP = sizeof(parts) / sizeof(parts[0]);
  size_t off[NP], bytes = 0;
  for (int i = 0; i < NP; i++) { off[i] = bytes; bytes += align256(parts[i].elems * parts[i].size + 1); }
  if (raw->bytes < bytes) {
    if (raw->buf) cudaFree(raw->buf);
    raw->buf = nullptr;
    raw->bytes = 0;
    if ((e = cudaMalloc(&raw->buf, bytes)) != cudaSuccess) return fail_cuda(e, "paam_generate: cudaMalloc");
    raw->bytes = bytes;
  }
  char* base = (char*)raw->buf;
  pg_arrays o;
  void** slots[NP] = {(void**)&o.set_chain_off, (void**)&o.set_exec_off, (void**)&o.set_accel_off,
                      (void**)&o.chain_T, (void**)&o.chain_D, (void**)&o.chain_prio, (void**)&o.chain_class,
                      (void**)&o.chain_cb_off, (void**)&o.cb_exec, (void**)&o.cb_seg_off,
                      (void**)&o.seg_kind, (void**)&o.seg_wcet, (void**)&o.seg_accel, (void**)&o.seg_unit,
                      (void**)&o.exec_core, (void**)&o.exec_prio, (void**)&o.exec_wait,
                      (void**)&o.accel_buckets, (void**)&o.accel_units, (void**)&o.accel_server_core,
                      (void**)&o.accel_eps, (void**)&o.accel_kappa, (void**)&o.set_bin};
  for (int i = 0; i < NP; i++) *slots[i] = base + off[i];
  if (!p.n_bins) o.set_bin = nullptr;
  cudaMemcpyAsync(o.set_chain_off, offs + 0 * nn, nn * 4, cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(o.set_exec_off, offs + 3 * nn, nn * 4, cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(o.set_accel_off, offs + 4 * nn, nn * 4, cudaMemcpyDeviceToDevice, st);
  if (n) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gen_fill_kernel, GW * 32, 0);
    const uint32_t need = (n + GW - 1) / GW, cap = (uint32_t)sms * (uint32_t)(per_sm > 0 ? per_sm : 1);
    gen_fill_kernel<<<need < cap ? need : cap, GW * 32, 0, st>>>(p, seed, first_index, n, o, offs + 1 * nn, offs + 2 * nn);
    count_launch();
  } else {
    cudaMemsetAsync(o.chain_cb_off, 0, 4, st);
    cudaMemsetAsync(o.cb_seg_off, 0, 4, st);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e, "paam_generate: fill");

  paam_batch& b = raw->b;
  std::memset(&b, 0, sizeof(b));
  b.n_sets = n;
  b.mem = PAAM_MEM_DEVICE;
  b.n_chains = nch; b.n_cbs = ncb; b.n_segs = nsg; b.n_execs = nex; b.n_accels = nac;
  b.n_bins = p.n_bins;
  b.set_chain_off = o.set_chain_off; b.set_exec_off = o.set_exec_off; b.set_accel_off = o.set_accel_off;
  b.chain_T = o.chain_T; b.chain_D = o.chain_D; b.chain_prio = o.chain_prio; b.chain_class = o.chain_class;
  b.chain_cb_off = o.chain_cb_off; b.cb_exec = o.cb_exec; b.cb_seg_off = o.cb_seg_off;
  b.seg_kind = o.seg_kind; b.seg_wcet = o.seg_wcet; b.seg_accel = o.seg_accel; b.seg_unit = o.seg_unit;
  b.exec_core = o.exec_core; b.exec_prio = o.exec_prio; b.exec_wait = o.exec_wait;
  b.accel_buckets = o.accel_buckets; b.accel_units = o.accel_units; b.accel_server_core = o.accel_server_core;
  b.accel_eps = o.accel_eps; b.accel_kappa = o.accel_kappa;
  b.set_bin = o.set_bin;
  b.comm_cost = comm_cost;
  b.flags = flags;
  return PAAM_OK;
}

int check_gen_args(const paam_gen_params* params, uint64_t comm_cost, pg_params* p) {
  static_assert(sizeof(paam_gen_params) == sizeof(pg_params), "paam_gen_params must mirror pg_params");
  if (!params) return fail(PAAM_EINVAL, "paam_generate: NULL params");
  std::memcpy(p, params, sizeof(*p));
  if (pg_check_params(p)) return fail(PAAM_EINVAL, "paam_generate: generator parameters out of range");
  if (comm_cost >= LIM) return fail(PAAM_EINVAL, "paam_generate: comm_cost >= 2^31 - 1");
  return PAAM_OK;
}

}  // namespace
}  // namespace paam

extern "C" int paam_generate(const paam_gen_params* params, uint64_t seed, uint64_t first_index, uint32_t n,
                             uint64_t comm_cost, uint32_t flags, paam_raw** out, paam_stream_t stream) {
  if (!out) return fail(PAAM_EINVAL, "paam_generate: NULL out");
  *out = nullptr;
  pg_params p;
  if (int rc = check_gen_args(params, comm_cost, &p)) return rc;
  paam_raw* raw = (paam_raw*)std::calloc(1, sizeof(paam_raw));
  if (!raw) return fail(PAAM_ENOMEM, "paam_generate: host allocation");
  cudaGetDevice(&raw->device);
  if (int rc = generate_into(raw, p, seed, first_index, n, comm_cost, flags, (cudaStream_t)stream)) {
    paam_raw_free(raw);
    return rc;
  }
  *out = raw;
  return PAAM_OK;
}

extern "C" int paam_regenerate(paam_raw* raw, const paam_gen_params* params, uint64_t seed, uint64_t first_index,
                               uint32_t n, uint64_t comm_cost, uint32_t flags, paam_stream_t stream) {
  if (!raw) return fail(PAAM_EINVAL, "paam_regenerate: NULL handle");
  pg_params p;
  if (int rc = check_gen_args(params, comm_cost, &p)) return rc;
  cudaError_t e = cudaSetDevice(raw->device);
  if (e != cudaSuccess) return fail_cuda(e, "paam_regenerate: cudaSetDevice");
  return generate_into(raw, p, seed, first_index, n, comm_cost, flags, (cudaStream_t)stream);
}

extern "C" int paam_raw_batch(const paam_raw* raw, paam_batch* out) {
  if (!raw || !out) return fail(PAAM_EINVAL, "paam_raw_batch: NULL argument");
  *out = raw->b;
  return PAAM_OK;
}

extern "C" void paam_raw_free(paam_raw* raw) {
  if (!raw) return;
  cudaSetDevice(raw->device);
  if (raw->buf) cudaFree(raw->buf);
  if (raw->scr) cudaFree(raw->scr);
  std::free(raw);
}

// ---- paam_sweep: steps 1-6 over device-generated chunks, generation overlapped with analysis ------
struct paam_sweeper {
  uint32_t chunk;
  paam_raw raw[2];          // capacity-laid-out raw batches (ping-pong)
  uint32_t* wide[2];        // sets of the chunk handed over to the u64 path (wide.cu), one list per buffer
  unsigned int* tickets;    // per buffer: the wide-list count and fused_kernel's work ticket
  cudaStream_t sg, sa;      // generation / pack + analysis
  cudaEvent_t start, gen_done[2], ana_done[2], join[2];
  int device;
};

extern "C" int paam_sweep_create(uint32_t chunk, paam_sweeper** out) {
  if (!out || chunk == 0) return fail(PAAM_EINVAL, "paam_sweep_create: NULL out or chunk == 0");
  *out = nullptr;
  paam_sweeper* h = (paam_sweeper*)std::calloc(1, sizeof(paam_sweeper));
  if (!h) return fail(PAAM_ENOMEM, "paam_sweep_create: host allocation");
  h->chunk = chunk;
  cudaError_t e = cudaGetDevice(&h->device);
  for (int i = 0; i < 2 && e == cudaSuccess; i++) {
    h->raw[i].device = h->device;
    e = cudaMalloc((void**)&h->wide[i], sizeof(uint32_t) * (size_t)chunk);
  }
  if (e == cudaSuccess) e = cudaMalloc((void**)&h->tickets, sizeof(unsigned int) * 4);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->sg, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->sa, cudaStreamNonBlocking);
  cudaEvent_t* evs[7] = {&h->start, &h->gen_done[0], &h->gen_done[1], &h->ana_done[0], &h->ana_done[1], &h->join[0], &h->join[1]};
  for (int i = 0; i < 7 && e == cudaSuccess; i++) e = cudaEventCreateWithFlags(evs[i], cudaEventDisableTiming);
  if (e != cudaSuccess) {
    paam_sweep_free(h);
    return fail_cuda(e, "paam_sweep_create");
  }
  *out = h;
  return PAAM_OK;
}

extern "C" int paam_sweep(paam_sweeper* h, const paam_gen_params* params, uint64_t seed, uint64_t first_index,
                          uint32_t n, uint64_t comm_cost, uint32_t flags, uint8_t* out_sched, int64_t* out_bins,
                          paam_stream_t stream) {
  if (!h) return fail(PAAM_EINVAL, "paam_sweep: NULL handle");
  if (flags & ~(PAAM_FLAG_BLOCKING_SOUND | PAAM_FLAG_WFD_UNITS | PAAM_FLAG_VERDICT_ONLY))
    return fail(PAAM_EINVAL, "paam_sweep: unknown flag");
  pg_params p;
  if (int rc = check_gen_args(params, comm_cost, &p)) return rc;
  {
    uint64_t cap[5];
    size_caps(p, cap);
    for (int k = 0; k < 5; k++)
      if (cap[k] * h->chunk >= (1ull << 32)) return fail(PAAM_EINVAL, "paam_sweep: chunk too large for 32-bit offsets");
  }
  cudaError_t e = cudaSetDevice(h->device);
  if (e != cudaSuccess) return fail_cuda(e, "paam_sweep: cudaSetDevice");
  cudaStream_t st = (cudaStream_t)stream;
  cudaEventRecord(h->start, st);
  cudaStreamWaitEvent(h->sg, h->start, 0);
  cudaStreamWaitEvent(h->sa, h->start, 0);
  const uint32_t nchunks = (n + h->chunk - 1) / h->chunk;
  for (uint32_t i = 0; i < nchunks; i++) {
    const int bi = i & 1;
    const uint32_t lo = i * h->chunk, cnt = n - lo < h->chunk ? n - lo : h->chunk;
    if (i >= 2) cudaStreamWaitEvent(h->sg, h->ana_done[bi], 0);  // buffers of chunk i-2 consumed
    if (int rc = generate_into(&h->raw[bi], p, seed, first_index + lo, cnt, comm_cost, flags, h->sg, h->chunk)) return rc;
    cudaEventRecord(h->gen_done[bi], h->sg);
    cudaStreamWaitEvent(h->sa, h->gen_done[bi], 0);
    cudaMemsetAsync(h->tickets + 2 * bi, 0, 2 * sizeof(unsigned int), h->sa);  // wide count, work ticket
    if (int rc = launch_fused(&h->raw[bi].b, h->wide[bi], h->tickets + 2 * bi, nullptr, nullptr,
                              out_sched ? out_sched + lo : nullptr, p.n_bins ? out_bins : nullptr, h->sa))  // steps 2-6
      return rc;
    if (int rc = launch_wide(&h->raw[bi].b, h->wide[bi], h->tickets + 2 * bi, nullptr, nullptr,
                             out_sched ? out_sched + lo : nullptr, p.n_bins ? out_bins : nullptr, nullptr, h->sa))
      return rc;
    cudaEventRecord(h->ana_done[bi], h->sa);
  }
  cudaEventRecord(h->join[0], h->sg);
  cudaEventRecord(h->join[1], h->sa);
  cudaStreamWaitEvent(st, h->join[0], 0);
  cudaStreamWaitEvent(st, h->join[1], 0);
  e = cudaGetLastError();
  return e == cudaSuccess ? PAAM_OK : fail_cuda(e, "paam_sweep");
}

extern "C" void paam_sweep_free(paam_sweeper* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  for (int i = 0; i < 2; i++) {
    if (h->raw[i].buf) cudaFree(h->raw[i].buf);
    if (h->raw[i].scr) cudaFree(h->raw[i].scr);
    if (h->wide[i]) cudaFree(h->wide[i]);
  }
  if (h->tickets) cudaFree(h->tickets);
  if (h->sg) cudaStreamDestroy(h->sg);
  if (h->sa) cudaStreamDestroy(h->sa);
  cudaEvent_t evs[7] = {h->start, h->gen_done[0], h->gen_done[1], h->ana_done[0], h->ana_done[1], h->join[0], h->join[1]};
  for (int i = 0; i < 7; i++) if (evs[i]) cudaEventDestroy(evs[i]);
  std::free(h);
}
