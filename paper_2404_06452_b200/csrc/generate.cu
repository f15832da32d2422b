// generate.cu -- §8(a) step 1: device-side synthetic chain-set generation (paam_generate).
//
// Runs the shared counter-based generator gen/paam_gen.h (input generation only -- it holds none of
// the analysed method) on the device, one thread per set: pass 1 sizes every set, five exclusive
// scans turn the sizes into CSR offsets, pass 2 regenerates each set and writes it at its offsets.
// Every set is a pure function of (seed, global index), so ranks generate disjoint index ranges
// with no communication, and the bytes equal the host generator's (tests/test_gpu_parity.py).
#include <cstdlib>
#include <cstring>

#include "../../gen/paam_gen.h"
#include "common.cuh"

struct paam_raw {
  paam_batch b;
  void* buf;
  size_t bytes;
  int device;
};

namespace paam {
namespace {

__global__ void gen_sizes_kernel(pg_params p, uint64_t seed, uint64_t first, uint32_t n, uint32_t* __restrict__ cnt) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  pg_set s;
  pg_generate_set(&p, seed, first + i, &s);
  cnt[0 * (size_t)n + i] = s.m;
  cnt[1 * (size_t)n + i] = s.n_cb;
  cnt[2 * (size_t)n + i] = s.n_seg;
  cnt[3 * (size_t)n + i] = s.n_exec;
  cnt[4 * (size_t)n + i] = s.n_accel;
}

__global__ void gen_fill_kernel(pg_params p, uint64_t seed, uint64_t first, uint32_t n, pg_arrays o,
                                const uint32_t* __restrict__ cb_off, const uint32_t* __restrict__ sg_off) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  pg_set s;
  pg_generate_set(&p, seed, first + i, &s);
  pg_write_set(&s, i, o.set_chain_off[i], cb_off[i], sg_off[i], o.set_exec_off[i], o.set_accel_off[i], &o);
  if (i == n - 1) {  // CSR sentinels
    o.chain_cb_off[o.set_chain_off[n]] = cb_off[n];
    o.cb_seg_off[cb_off[n]] = sg_off[n];
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

extern "C" int paam_generate(const paam_gen_params* params, uint64_t seed, uint64_t first_index, uint32_t n,
                             uint64_t comm_cost, uint32_t flags, paam_raw** out, paam_stream_t stream) {
  static_assert(sizeof(paam_gen_params) == sizeof(pg_params), "paam_gen_params must mirror pg_params");
  if (!params || !out) return fail(PAAM_EINVAL, "paam_generate: NULL argument");
  *out = nullptr;
  pg_params p;
  std::memcpy(&p, params, sizeof(p));
  if (pg_check_params(&p)) return fail(PAAM_EINVAL, "paam_generate: generator parameters out of range");
  if (comm_cost >= LIM) return fail(PAAM_EINVAL, "paam_generate: comm_cost >= 2^31 - 1");
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;

  // pass 1: sizes, then offsets
  uint32_t *cnt = nullptr, *offs = nullptr, *tmp = nullptr;
  const size_t nn = (size_t)n + 1;
  const size_t tw = scan_tmp_words(n);
  if ((e = cudaMallocAsync((void**)&cnt, sizeof(uint32_t) * 5 * (size_t)(n ? n : 1), st)) != cudaSuccess)
    return fail_cuda(e, "paam_generate: cudaMallocAsync");
  if ((e = cudaMallocAsync((void**)&offs, sizeof(uint32_t) * 5 * nn, st)) != cudaSuccess)
    return fail_cuda(e, "paam_generate: cudaMallocAsync");
  if ((e = cudaMallocAsync((void**)&tmp, sizeof(uint32_t) * tw, st)) != cudaSuccess)
    return fail_cuda(e, "paam_generate: cudaMallocAsync");
  if (n) {
    gen_sizes_kernel<<<(n + 127) / 128, 128, 0, st>>>(p, seed, first_index, n, cnt);
    count_launch();
  }
  for (int k = 0; k < 5; k++) scan(cnt + (size_t)k * n, offs + (size_t)k * nn, n, tmp, st);
  uint32_t tot[5];
  for (int k = 0; k < 5; k++)
    cudaMemcpyAsync(&tot[k], offs + (size_t)k * nn + n, sizeof(uint32_t), cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return fail_cuda(e, "paam_generate: sizes");

  // one allocation for every array of the raw batch
  const uint32_t nch = tot[0], ncb = tot[1], nsg = tot[2], nex = tot[3], nac = tot[4];
  struct Part { size_t elems, size; } parts[] = {
      {nn, 4}, {nn, 4}, {nn, 4},                                  // set offsets
      {nch, 8}, {nch, 8}, {nch, 4}, {nch, 1}, {(size_t)nch + 1, 4},  // chains
      {ncb, 2}, {(size_t)ncb + 1, 4},                              // callbacks
      {nsg, 1}, {nsg, 8}, {nsg, 1}, {nsg, 1},                      // segments
      {nex, 1}, {nex, 4}, {nex, 1},                                // executors
      {nac, 1}, {nac, 1}, {nac, 1}, {nac, 8}, {nac, 8},            // accelerators
      {n, 4}};                                                     // set_bin
  constexpr int NP = sizeof(parts) / sizeof(parts[0]);
  size_t off[NP], bytes = 0;
  for (int i = 0; i < NP; i++) { off[i] = bytes; bytes += align256(parts[i].elems * parts[i].size + 1); }
  paam_raw* raw = (paam_raw*)std::calloc(1, sizeof(paam_raw));
  if (!raw) return fail(PAAM_ENOMEM, "paam_generate: host allocation");
  if ((e = cudaMalloc(&raw->buf, bytes)) != cudaSuccess) { std::free(raw); return fail_cuda(e, "paam_generate: cudaMalloc"); }
  raw->bytes = bytes;
  cudaGetDevice(&raw->device);
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
  cudaMemcpyAsync(o.set_chain_off, offs + 0 * nn, nn * 4, cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(o.set_exec_off, offs + 3 * nn, nn * 4, cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(o.set_accel_off, offs + 4 * nn, nn * 4, cudaMemcpyDeviceToDevice, st);
  if (n) {
    gen_fill_kernel<<<(n + 127) / 128, 128, 0, st>>>(p, seed, first_index, n, o, offs + 1 * nn, offs + 2 * nn);
    count_launch();
  } else {
    cudaMemsetAsync(o.chain_cb_off, 0, 4, st);
    cudaMemsetAsync(o.cb_seg_off, 0, 4, st);
  }
  cudaFreeAsync(cnt, st);
  cudaFreeAsync(offs, st);
  cudaFreeAsync(tmp, st);
  if ((e = cudaGetLastError()) != cudaSuccess) { cudaFree(raw->buf); std::free(raw); return fail_cuda(e, "paam_generate: fill"); }

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
  b.set_bin = p.n_bins ? o.set_bin : nullptr;
  b.comm_cost = comm_cost;
  b.flags = flags;
  *out = raw;
  return PAAM_OK;
}

extern "C" int paam_raw_batch(const paam_raw* raw, paam_batch* out) {
  if (!raw || !out) return fail(PAAM_EINVAL, "paam_raw_batch: NULL argument");
  *out = raw->b;
  return PAAM_OK;
}

extern "C" void paam_raw_free(paam_raw* raw) {
  if (!raw) return;
  cudaSetDevice(raw->device);
  cudaFree(raw->buf);
  std::free(raw);
}
