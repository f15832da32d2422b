// api.cu -- the C ABI of include/paam.h: handles, host staging, argument checks, error reporting.
// Every compute step runs in the kernels of pack.cu / analyze.cu / simulate.cu / generate.cu; this
// file only moves buffers and launches them.  There is no CPU fallback: without a CUDA device every
// entry point returns PAAM_ECUDA.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

struct paam_sets {
  uint32_t n_sets, n_chains, n_bins, cap;
  paam::Record* rec;
  uint64_t comm;
  uint32_t flags;
  void* stage;  // device staging of a host batch (grown on demand)
  size_t stage_bytes;
  int32_t* dstatus;  // device status staging for host batches
  uint32_t dstatus_cap;
  paam_batch dev;    // the packed batch with device pointers (paam_simulate reads its structure)
  cudaStream_t side[3];  // internal streams of paam_pack_analyze: pack, analyze, H2D copies (created on first use)
  cudaEvent_t ev[17], evc[8];  // evc: chunk copies done
  unsigned int* tickets;  // work-distribution counters: pipeline chunks [0, 16), analyze 16, admit 17, simulate 18,
                          // 20: number of wide sets listed (wide.cu), 21: fused_kernel's work ticket
  uint32_t* wide_list;    // [cap] the sets handed over to the u64 path by the last pack / fused launch
  int device;             // the CUDA device the handle lives on (made current by every call)
  void* ostage;           // device staging of host outputs of paam_pack_analyze (WCRTs, then verdicts)
  size_t ostage_bytes;
  void* sim_scratch;      // paam_simulate's event buffers (grown on demand)
  size_t sim_scratch_bytes;
  bool c32;               // dev is a compact batch (paam_pack_analyze32): nothing can pack it into records
  bool rec_valid;         // rec holds the records of `dev` (false after the fused paam_pack_analyze, which writes
                          // none: the next paam_analyze / paam_admit / paam_simulate packs them first)
};

namespace paam {

static std::atomic<uint64_t> g_launches{0};
static thread_local char g_err[512] = "";

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int fail(int code, const char* what) {
  std::snprintf(g_err, sizeof(g_err), "%s", what);
  return code;
}

int fail_cuda(cudaError_t e, const char* what) {
  std::snprintf(g_err, sizeof(g_err), "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? PAAM_ENOMEM : PAAM_ECUDA;
}

namespace {

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// Every call on a handle runs on the handle's device.  This library links its own CUDA runtime, whose
// per-thread current device is independent of the caller's (e.g. torch's), so it is set explicitly.
inline int use_device(const paam_sets* s) {
  const cudaError_t e = cudaSetDevice(s->device);
  return e == cudaSuccess ? PAAM_OK : fail_cuda(e, "cudaSetDevice");
}

struct Field { const void** ptr; size_t elems, size; };

// The array fields of a batch with their element counts (order of include/paam.h).
// c32: b carries a compact batch (paam_batch32 pointers: 4-byte times, 1-byte cb_exec, seg_kind = the
// packed segment byte, no seg_accel / seg_unit).
int batch_fields(paam_batch* b, Field* f, bool c32 = false) {
  const size_t nn = (size_t)b->n_sets + 1;
  const size_t tz = c32 ? 4 : 8, sa = c32 ? 0 : b->n_segs;
  Field t[] = {
      {(const void**)&b->set_chain_off, nn, 4}, {(const void**)&b->set_exec_off, nn, 4},
      {(const void**)&b->set_accel_off, nn, 4},
      {(const void**)&b->chain_T, b->n_chains, tz}, {(const void**)&b->chain_D, b->n_chains, tz},
      {(const void**)&b->chain_prio, b->n_chains, 4}, {(const void**)&b->chain_class, b->n_chains, 1},
      {(const void**)&b->chain_cb_off, (size_t)b->n_chains + 1, 4},
      {(const void**)&b->cb_exec, b->n_cbs, c32 ? 1u : 2u}, {(const void**)&b->cb_seg_off, (size_t)b->n_cbs + 1, 4},
      {(const void**)&b->seg_kind, b->n_segs, 1}, {(const void**)&b->seg_wcet, b->n_segs, tz},
      {(const void**)&b->seg_accel, sa, 1}, {(const void**)&b->seg_unit, sa, 1},
      {(const void**)&b->exec_core, b->n_execs, 1}, {(const void**)&b->exec_prio, b->n_execs, 4},
      {(const void**)&b->exec_wait, b->n_execs, 1},
      {(const void**)&b->accel_buckets, b->n_accels, 1}, {(const void**)&b->accel_units, b->n_accels, 1},
      {(const void**)&b->accel_server_core, b->n_accels, 1}, {(const void**)&b->accel_eps, b->n_accels, tz},
      {(const void**)&b->accel_kappa, b->n_accels, tz},
      {(const void**)&b->set_bin, b->set_bin ? (size_t)b->n_sets : 0, 4}};
  const int n = sizeof(t) / sizeof(t[0]);
  for (int i = 0; i < n; i++) f[i] = t[i];
  return n;
}

// Grow the device staging buffer of a host batch to `bytes`.
int ensure_stage(paam_sets* sets, size_t bytes) {
  if (bytes <= sets->stage_bytes) return PAAM_OK;
  if (sets->stage) cudaFree(sets->stage);
  sets->stage = nullptr;
  sets->stage_bytes = 0;
  const cudaError_t e = cudaMalloc(&sets->stage, bytes);
  if (e != cudaSuccess) return fail_cuda(e, "staging cudaMalloc");
  sets->stage_bytes = bytes;
  return PAAM_OK;
}
int ensure_dstatus(paam_sets* sets, uint32_t n) {
  if (sets->dstatus_cap >= n) return PAAM_OK;
  if (sets->dstatus) cudaFree(sets->dstatus);
  sets->dstatus = nullptr;
  sets->dstatus_cap = 0;
  const cudaError_t e = cudaMalloc((void**)&sets->dstatus, sizeof(int32_t) * (n ? n : 1));
  if (e != cudaSuccess) return fail_cuda(e, "status cudaMalloc");
  sets->dstatus_cap = n;
  return PAAM_OK;
}
// Is p host memory (pinned or pageable)?  Device and managed pointers are not.
bool is_host_ptr(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();  // pageable memory on old drivers reports an error: clear it
    return true;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeUnregistered;
}
int ensure_ostage(paam_sets* sets, size_t bytes) {
  if (sets->ostage_bytes >= bytes) return PAAM_OK;
  if (sets->ostage) cudaFree(sets->ostage);
  sets->ostage = nullptr;
  sets->ostage_bytes = 0;
  const cudaError_t e = cudaMalloc(&sets->ostage, bytes);
  if (e != cudaSuccess) return fail_cuda(e, "output staging cudaMalloc");
  sets->ostage_bytes = bytes;
  return PAAM_OK;
}
int ensure_streams(paam_sets* sets) {
  if (sets->side[0]) return PAAM_OK;
  cudaError_t e;
  for (int i = 0; i < 3; i++)
    if ((e = cudaStreamCreateWithFlags(&sets->side[i], cudaStreamNonBlocking)) != cudaSuccess) return fail_cuda(e, "stream");
  for (int i = 0; i < 17; i++)
    if ((e = cudaEventCreateWithFlags(&sets->ev[i], cudaEventDisableTiming)) != cudaSuccess) return fail_cuda(e, "event");
  for (int i = 0; i < 8; i++)
    if ((e = cudaEventCreateWithFlags(&sets->evc[i], cudaEventDisableTiming)) != cudaSuccess) return fail_cuda(e, "event");
  return PAAM_OK;
}

// Materialise the records of the handle's batch if the last call was the fused paam_pack_analyze.
int ensure_records(const paam_sets* cs, cudaStream_t st) {
  paam_sets* sets = const_cast<paam_sets*>(cs);
  if (sets->rec_valid) return PAAM_OK;
  if (sets->c32)
    return fail(PAAM_EINVAL, "the handle holds a compact batch (paam_pack_analyze32): paam_pack / paam_repack first");
  cudaMemsetAsync(sets->tickets + 20, 0, 2 * sizeof(unsigned int), st);  // wide count, work ticket
  if (int rc = launch_pack(&sets->dev, sets->rec, nullptr, sets->wide_list, sets->tickets + 20, st)) return rc;
  sets->rec_valid = true;
  return PAAM_OK;
}

int check_batch(const paam_batch* b, bool c32 = false) {
  if (!b) return fail(PAAM_EINVAL, "NULL batch");
  if (b->mem != PAAM_MEM_HOST && b->mem != PAAM_MEM_DEVICE) return fail(PAAM_EINVAL, "batch.mem must be HOST or DEVICE");
  if (b->comm_cost >= LIMW) return fail(PAAM_EINVAL, "batch.comm_cost must be < 2^48 ns");
  if (b->flags & ~(PAAM_FLAG_BLOCKING_SOUND | PAAM_FLAG_WFD_UNITS | PAAM_FLAG_VERDICT_ONLY))
    return fail(PAAM_EINVAL, "unknown flag");
  if (b->set_bin && b->n_bins == 0) return fail(PAAM_EINVAL, "set_bin given with n_bins == 0");
  paam_batch c = *b;
  Field f[32];
  const int nf = batch_fields(&c, f, c32);
  for (int i = 0; i < nf; i++)
    if (f[i].elems && !*f[i].ptr && f[i].ptr != (const void**)&c.set_bin)
      return fail(PAAM_EINVAL, "NULL array in a batch with a non-zero count");
  return PAAM_OK;
}

}  // namespace
}  // namespace paam

using namespace paam;

extern "C" int paam_repack(const paam_batch* batch, paam_sets* sets, int32_t* out_status, paam_stream_t stream) {
  int rc = check_batch(batch);
  if (rc) return rc;
  if (!sets) return fail(PAAM_EINVAL, "NULL handle");
  if (batch->n_sets > sets->cap) return fail(PAAM_EINVAL, "paam_repack: handle capacity too small");
  if ((rc = use_device(sets))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  paam_batch d = *batch;
  int32_t* status_dev = out_status;
  if (batch->mem == PAAM_MEM_HOST) {
    Field f[32];
    const int nf = batch_fields(&d, f);
    size_t bytes = 0;
    for (int i = 0; i < nf; i++) bytes += align256(f[i].elems * f[i].size);
    if ((rc = ensure_stage(sets, bytes))) return rc;
    char* base = (char*)sets->stage;
    size_t off = 0;
    for (int i = 0; i < nf; i++) {  // one cudaMemcpyAsync per array (no batched-copy APIs)
      const size_t nb = f[i].elems * f[i].size;
      if (nb) {
        if ((e = cudaMemcpyAsync(base + off, *f[i].ptr, nb, cudaMemcpyHostToDevice, st)) != cudaSuccess)
          return fail_cuda(e, "paam_pack: H2D copy");
        *f[i].ptr = base + off;
      }
      off += align256(nb);
    }
    if (out_status) {
      if ((rc = ensure_dstatus(sets, batch->n_sets))) return rc;
      status_dev = sets->dstatus;
    }
  }
  cudaMemsetAsync(sets->tickets + 20, 0, 2 * sizeof(unsigned int), st);  // wide count, work ticket
  rc = launch_pack(&d, sets->rec, status_dev, sets->wide_list, sets->tickets + 20, st);
  if (rc) return rc;
  // the wide sets (a time >= 2^31 - 1 ns): validated on the u64 path (statuses only here)
  rc = launch_wide(&d, sets->wide_list, sets->tickets + 20, status_dev, nullptr, nullptr, nullptr, nullptr, st);
  if (rc) return rc;
  if (batch->mem == PAAM_MEM_HOST) {
    if (out_status && batch->n_sets)
      if ((e = cudaMemcpyAsync(out_status, status_dev, sizeof(int32_t) * batch->n_sets, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        return fail_cuda(e, "paam_pack: status D2H");
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return fail_cuda(e, "paam_pack: synchronize");
  }
  sets->dev = d;
  sets->n_sets = batch->n_sets;
  sets->n_chains = batch->n_chains;
  sets->n_bins = batch->set_bin ? batch->n_bins : 0;
  sets->comm = batch->comm_cost;
  sets->flags = batch->flags;
  sets->rec_valid = true;
  sets->c32 = false;
  return PAAM_OK;
}

extern "C" int paam_pack(const paam_batch* batch, paam_sets** out, int32_t* out_status, paam_stream_t stream) {
  if (!out) return fail(PAAM_EINVAL, "NULL out");
  *out = nullptr;
  int rc = check_batch(batch);
  if (rc) return rc;
  paam_sets* s = (paam_sets*)std::calloc(1, sizeof(paam_sets));
  if (!s) return fail(PAAM_ENOMEM, "host allocation");
  s->cap = batch->n_sets;
  cudaError_t e = cudaGetDevice(&s->device);
  if (e != cudaSuccess) {
    std::free(s);
    return fail_cuda(e, "paam_pack: cudaGetDevice");
  }
  e = cudaMalloc((void**)&s->tickets, sizeof(unsigned int) * 32);
  if (e != cudaSuccess) {
    std::free(s);
    return fail_cuda(e, "paam_pack: ticket cudaMalloc");
  }
  e = cudaMalloc((void**)&s->rec, sizeof(Record) * (size_t)(batch->n_sets ? batch->n_sets : 1));
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->wide_list, sizeof(uint32_t) * (size_t)(batch->n_sets ? batch->n_sets : 1));
  if (e != cudaSuccess) {
    paam_free(s);  // releases the tickets
    return fail_cuda(e, "paam_pack: record cudaMalloc");
  }
  rc = paam_repack(batch, s, out_status, stream);
  if (rc) {
    paam_free(s);
    return rc;
  }
  *out = s;
  return PAAM_OK;
}

extern "C" int paam_analyze(const paam_sets* sets, uint32_t n, uint64_t* out_wcrt, uint8_t* out_sched,
                            int64_t* out_bins, paam_stream_t stream) {
  if (!sets) return fail(PAAM_EINVAL, "NULL handle");
  if (n > sets->n_sets) return fail(PAAM_EINVAL, "paam_analyze: n exceeds the packed sets");
  if ((sets->flags & PAAM_FLAG_VERDICT_ONLY) && out_wcrt)
    return fail(PAAM_EINVAL, "paam_analyze: PAAM_FLAG_VERDICT_ONLY writes no WCRTs (out_wcrt must be NULL)");
  if (int rc = use_device(sets)) return rc;
  if (int rc = ensure_records(sets, (cudaStream_t)stream)) return rc;
  int rc = launch_analyze(sets->rec, n, sets->comm, sets->flags, sets->n_bins, out_wcrt, out_sched,
                          sets->n_bins ? out_bins : nullptr, sets->tickets + 16, (cudaStream_t)stream);
  if (rc) return rc;
  paam_batch v = sets->dev;  // the wide sets of the first n
  v.n_sets = n;
  return launch_wide(&v, sets->wide_list, sets->tickets + 20, nullptr, out_wcrt, out_sched, sets->n_bins ? out_bins : nullptr,
                     nullptr, (cudaStream_t)stream);
}

extern "C" int paam_admit(const paam_sets* sets, uint32_t n, int32_t* out_decision, uint64_t* out_wcrt,
                          paam_stream_t stream) {
  if (!sets || !out_decision) return fail(PAAM_EINVAL, "paam_admit: NULL argument");
  if (n > sets->n_sets) return fail(PAAM_EINVAL, "paam_admit: n exceeds the packed sets");
  if (int rc = use_device(sets)) return rc;
  if (int rc = ensure_records(sets, (cudaStream_t)stream)) return rc;
  int rc = launch_analyze(sets->rec, n, sets->comm, sets->flags & ~PAAM_FLAG_VERDICT_ONLY, 0, out_wcrt, nullptr, nullptr,
                          const_cast<paam_sets*>(sets)->tickets + 17, (cudaStream_t)stream, out_decision);
  if (rc) return rc;
  paam_batch v = sets->dev;
  v.n_sets = n;
  return launch_wide(&v, sets->wide_list, sets->tickets + 20, nullptr, out_wcrt, nullptr, nullptr, out_decision,
                     (cudaStream_t)stream);
}

extern "C" int paam_simulate(const paam_sets* sets, uint32_t n, uint64_t horizon, uint64_t seed, uint64_t first_index,
                             uint32_t sim_flags, const paam_sim_out* out, paam_stream_t stream) {
  if (!sets) return fail(PAAM_EINVAL, "NULL handle");
  if (n > sets->n_sets) return fail(PAAM_EINVAL, "paam_simulate: n exceeds the packed sets");
  if (sim_flags & ~(uint32_t)PAAM_SIM_FIFO_DIRECT) return fail(PAAM_EINVAL, "paam_simulate: unknown sim flag");
  if (sets->dev.comm_cost >= LIM)
    return fail(PAAM_EINVAL, "paam_simulate: the DES needs comm_cost < 2^31 - 1 ns (32-bit time distances)");
  paam_sim_out o{};
  if (out) o = *out;
  if (o.witness && !o.violations) return fail(PAAM_EINVAL, "paam_simulate: witness needs violations");
  if (!o.witness) o.max_witness = 0;
  if (int rc = use_device(sets)) return rc;
  if (int rc = ensure_records(sets, (cudaStream_t)stream)) return rc;
  paam_sets* ms = const_cast<paam_sets*>(sets);
  return launch_simulate(&sets->dev, sets->rec, n, horizon, seed, first_index, sim_flags, &o, ms->tickets + 18,
                         &ms->sim_scratch, &ms->sim_scratch_bytes, (cudaStream_t)stream);
}

namespace paam {
namespace {
// paam_pack_analyze on a u64 batch or (c32) on a compact batch carried in a paam_batch
int pack_analyze_impl(const paam_batch* batch, bool c32, paam_sets* sets, int32_t* out_status, uint64_t* out_wcrt,
                      uint8_t* out_sched, int64_t* out_bins, paam_stream_t stream) {
  int rc = check_batch(batch, c32);
  if (rc) return rc;
  if (!sets) return fail(PAAM_EINVAL, "NULL handle");
  if (batch->n_sets > sets->cap) return fail(PAAM_EINVAL, "paam_pack_analyze: handle capacity too small");
  if ((batch->flags & PAAM_FLAG_VERDICT_ONLY) && out_wcrt)
    return fail(PAAM_EINVAL, "paam_pack_analyze: PAAM_FLAG_VERDICT_ONLY writes no WCRTs (out_wcrt must be NULL)");
  if ((rc = use_device(sets))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  const bool host = batch->mem == PAAM_MEM_HOST;
  const uint32_t n = batch->n_sets;
  const int64_t* bins = batch->set_bin ? out_bins : nullptr;
  paam_batch d = *batch;  // the batch the kernel reads (host: pointers into the staging buffer)
  d._pad = 0;
  int32_t* status_dev = out_status;
  const bool wcrt_host = out_wcrt && is_host_ptr(out_wcrt), sched_host = out_sched && is_host_ptr(out_sched);
  if (!host && (wcrt_host || sched_host))
    return fail(PAAM_EINVAL, "paam_pack_analyze: host out_wcrt / out_sched need a host batch");
  if (!host) {
    // steps 2-6 in one kernel (fused.cu): the derived records stay on chip
    cudaMemsetAsync(sets->tickets + 20, 0, 2 * sizeof(unsigned int), st);  // wide count, work ticket
    if ((rc = launch_fused(&d, sets->wide_list, sets->tickets + 20, status_dev, out_wcrt, out_sched,
                           const_cast<int64_t*>(bins), st, c32)))
      return rc;
    // the sets it handed over (a time >= 2^31 - 1 ns): exact u64 path
    if ((rc = launch_wide(&d, sets->wide_list, sets->tickets + 20, status_dev, out_wcrt, out_sched,
                          const_cast<int64_t*>(bins), nullptr, st, c32)))
      return rc;
  } else {
    // Host batch: K chunks; chunk i's slice of every array is copied H2D on side[2] while the kernel of
    // chunk i-1 runs on side[0] (copy engines alongside the SMs).
    static const int KH = [] {  // chunks (PAAM_H2D_CHUNKS overrides, for tuning)
      const char* ev = std::getenv("PAAM_H2D_CHUNKS");
      const int k = ev ? std::atoi(ev) : 8;  // measured: 8 > 6 > 4 (e2e 40.8 / 40.6 / 40.2M sets/s)
      return k < 1 ? 1 : (k > 8 ? 8 : k);
    }();
    const int K = n < 4096 ? 1 : KH;
    if ((rc = ensure_streams(sets))) return rc;
    Field f[32];
    const int nf = batch_fields(&d, f, c32);
    size_t foff[32];
    // The chunk copies read the host CSR offsets at chunk boundaries: they must be monotone and within
    // the declared totals (include/paam.h), else a copy range would be wrong or out of bounds.
    const paam_batch& hb = *batch;
    uint32_t pc = 0, pb = 0, ps = 0, px = 0, pa = 0;
    for (int i = 0; i <= K; i++) {
      const uint32_t sidx = (uint32_t)((uint64_t)n * i / K);
      const uint32_t c = hb.set_chain_off[sidx], x = hb.set_exec_off[sidx], a = hb.set_accel_off[sidx];
      if (c < pc || x < px || a < pa || c > hb.n_chains || x > hb.n_execs || a > hb.n_accels)
        return fail(PAAM_EINVAL, "paam_pack_analyze: host set offsets not monotone or beyond the batch totals");
      const uint32_t bcb = hb.chain_cb_off[c];
      if (bcb < pb || bcb > hb.n_cbs)
        return fail(PAAM_EINVAL, "paam_pack_analyze: host chain_cb_off not monotone or beyond n_cbs");
      const uint32_t sg = hb.cb_seg_off[bcb];
      if (sg < ps || sg > hb.n_segs)
        return fail(PAAM_EINVAL, "paam_pack_analyze: host cb_seg_off not monotone or beyond n_segs");
      pc = c; px = x; pa = a; pb = bcb; ps = sg;
    }
    size_t bytes = 0;
    for (int i = 0; i < nf; i++) { foff[i] = bytes; bytes += align256(f[i].elems * f[i].size); }
    if ((rc = ensure_stage(sets, bytes))) return rc;
    for (int i = 0; i < nf; i++) if (f[i].elems) *f[i].ptr = (char*)sets->stage + foff[i];
    if (out_status) {
      if ((rc = ensure_dstatus(sets, n))) return rc;
      status_dev = sets->dstatus;
    }
    // Host outputs: the kernels write a device staging copy and each chunk's WCRTs / verdicts go back on
    // side[1] as soon as the chunk's kernels are done, overlapping the next chunk's H2D (PCIe is duplex).
    uint64_t* wcrt_dev = out_wcrt;
    uint8_t* sched_dev = out_sched;
    if (wcrt_host || sched_host) {
      const size_t wb = wcrt_host ? align256(sizeof(uint64_t) * (size_t)batch->n_chains) : 0;
      if ((rc = ensure_ostage(sets, wb + (sched_host ? (size_t)n : 0) + 1))) return rc;
      if (wcrt_host) wcrt_dev = (uint64_t*)sets->ostage;
      if (sched_host) sched_dev = (uint8_t*)sets->ostage + wb;
    }
    cudaEventRecord(sets->ev[16], st);
    for (int i = 0; i < 3; i++) cudaStreamWaitEvent(sets->side[i], sets->ev[16], 0);
    for (int i = 0; i < K; i++) {
      const uint32_t lo = (uint32_t)((uint64_t)n * i / K), hi = (uint32_t)((uint64_t)n * (i + 1) / K);
      // element ranges of this chunk in every array (host CSR offsets), in batch_fields order
      const size_t cl = hb.set_chain_off[lo], ch = hb.set_chain_off[hi];
      const size_t xl = hb.set_exec_off[lo], xh = hb.set_exec_off[hi];
      const size_t al = hb.set_accel_off[lo], ah = hb.set_accel_off[hi];
      const size_t bl = hb.chain_cb_off[cl], bh = hb.chain_cb_off[ch];
      const size_t sl = hb.cb_seg_off[bl], sh = hb.cb_seg_off[bh];
      const size_t r[23][2] = {{lo, hi + 1ull}, {lo, hi + 1ull}, {lo, hi + 1ull},
                               {cl, ch}, {cl, ch}, {cl, ch}, {cl, ch}, {cl, ch + 1},
                               {bl, bh}, {bl, bh + 1},
                               {sl, sh}, {sl, sh}, {sl, sh}, {sl, sh},
                               {xl, xh}, {xl, xh}, {xl, xh},
                               {al, ah}, {al, ah}, {al, ah}, {al, ah}, {al, ah},
                               {lo, hi}};
      Field hf[32];
      paam_batch hcopy = *batch;
      batch_fields(&hcopy, hf, c32);
      for (int k = 0; k < nf; k++) {  // one cudaMemcpyAsync per array slice (no batched-copy APIs)
        if (!f[k].elems || r[k][1] <= r[k][0]) continue;
        const size_t sz = f[k].size;
        if ((e = cudaMemcpyAsync((char*)sets->stage + foff[k] + r[k][0] * sz, (const char*)*hf[k].ptr + r[k][0] * sz,
                                 (r[k][1] - r[k][0]) * sz, cudaMemcpyHostToDevice, sets->side[2])) != cudaSuccess)
          return fail_cuda(e, "paam_pack_analyze: H2D copy");
      }
      cudaEventRecord(sets->evc[i], sets->side[2]);
      cudaStreamWaitEvent(sets->side[0], sets->evc[i], 0);
      paam_batch view = d;  // CSR offsets stay global: a chunk is a shifted window of set offsets
      view.n_sets = hi - lo;
      view.set_chain_off += lo;
      view.set_exec_off += lo;
      view.set_accel_off += lo;
      if (view.set_bin) view.set_bin += lo;
      cudaMemsetAsync(sets->tickets + 20, 0, 2 * sizeof(unsigned int), sets->side[0]);  // wide count, work ticket
      if ((rc = launch_fused(&view, sets->wide_list, sets->tickets + 20, status_dev ? status_dev + lo : nullptr, wcrt_dev,
                             sched_dev ? sched_dev + lo : nullptr,
                             const_cast<int64_t*>(bins), sets->side[0], c32)))
        return rc;
      if ((rc = launch_wide(&view, sets->wide_list, sets->tickets + 20, status_dev ? status_dev + lo : nullptr, wcrt_dev,
                            sched_dev ? sched_dev + lo : nullptr, const_cast<int64_t*>(bins), nullptr, sets->side[0],
                            c32)))
        return rc;
      if (wcrt_host || sched_host) {
        cudaEventRecord(sets->ev[i], sets->side[0]);
        cudaStreamWaitEvent(sets->side[1], sets->ev[i], 0);
        if (wcrt_host && ch > cl &&
            (e = cudaMemcpyAsync(out_wcrt + cl, wcrt_dev + cl, sizeof(uint64_t) * (ch - cl), cudaMemcpyDeviceToHost,
                                 sets->side[1])) != cudaSuccess)
          return fail_cuda(e, "paam_pack_analyze: WCRT D2H");
        if (sched_host && hi > lo &&
            (e = cudaMemcpyAsync(out_sched + lo, sched_dev + lo, hi - lo, cudaMemcpyDeviceToHost, sets->side[1])) !=
                cudaSuccess)
          return fail_cuda(e, "paam_pack_analyze: verdict D2H");
      }
    }
    cudaEventRecord(sets->ev[9], sets->side[0]);
    cudaEventRecord(sets->ev[10], sets->side[2]);
    cudaEventRecord(sets->ev[11], sets->side[1]);
    cudaStreamWaitEvent(st, sets->ev[9], 0);
    cudaStreamWaitEvent(st, sets->ev[10], 0);
    cudaStreamWaitEvent(st, sets->ev[11], 0);
    if (out_status) {  // host status, as paam_repack: copied back, the call synchronises
      if ((e = cudaMemcpyAsync(out_status, status_dev, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        return fail_cuda(e, "paam_pack_analyze: status D2H");
      if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return fail_cuda(e, "paam_pack_analyze: synchronize");
    }
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e, "paam_pack_analyze");
  sets->dev = d;
  sets->n_sets = n;
  sets->n_chains = batch->n_chains;
  sets->n_bins = batch->set_bin ? batch->n_bins : 0;
  sets->comm = batch->comm_cost;
  sets->flags = batch->flags;
  sets->rec_valid = false;  // the fused kernel wrote no records
  sets->c32 = c32;
  return PAAM_OK;
}
}  // namespace
}  // namespace paam

extern "C" int paam_pack_analyze(const paam_batch* batch, paam_sets* sets, int32_t* out_status, uint64_t* out_wcrt,
                                 uint8_t* out_sched, int64_t* out_bins, paam_stream_t stream) {
  return pack_analyze_impl(batch, false, sets, out_status, out_wcrt, out_sched, out_bins, stream);
}

extern "C" int paam_pack_analyze32(const paam_batch32* b32, paam_sets* sets, int32_t* out_status, uint64_t* out_wcrt,
                                   uint8_t* out_sched, int64_t* out_bins, paam_stream_t stream) {
  if (!b32) return fail(PAAM_EINVAL, "NULL batch");
  // the compact arrays travel in a paam_batch (the kernels read them through ld_time / ld_seg)
  paam_batch b{};
  b.n_sets = b32->n_sets; b.mem = b32->mem;
  b.n_chains = b32->n_chains; b.n_cbs = b32->n_cbs; b.n_segs = b32->n_segs;
  b.n_execs = b32->n_execs; b.n_accels = b32->n_accels; b.n_bins = b32->n_bins;
  b.set_chain_off = b32->set_chain_off; b.set_exec_off = b32->set_exec_off; b.set_accel_off = b32->set_accel_off;
  b.chain_T = reinterpret_cast<const uint64_t*>(b32->chain_T);
  b.chain_D = reinterpret_cast<const uint64_t*>(b32->chain_D);
  b.chain_prio = b32->chain_prio; b.chain_class = b32->chain_class; b.chain_cb_off = b32->chain_cb_off;
  b.cb_exec = reinterpret_cast<const uint16_t*>(b32->cb_exec);
  b.cb_seg_off = b32->cb_seg_off;
  b.seg_kind = b32->seg_meta;
  b.seg_wcet = reinterpret_cast<const uint64_t*>(b32->seg_wcet);
  b.seg_accel = nullptr; b.seg_unit = nullptr;
  b.exec_core = b32->exec_core; b.exec_prio = b32->exec_prio; b.exec_wait = b32->exec_wait;
  b.accel_buckets = b32->accel_buckets; b.accel_units = b32->accel_units;
  b.accel_server_core = b32->accel_server_core;
  b.accel_eps = reinterpret_cast<const uint64_t*>(b32->accel_eps);
  b.accel_kappa = reinterpret_cast<const uint64_t*>(b32->accel_kappa);
  b.set_bin = b32->set_bin;
  b.comm_cost = b32->comm_cost; b.flags = b32->flags; b._pad = 0;
  return pack_analyze_impl(&b, true, sets, out_status, out_wcrt, out_sched, out_bins, stream);
}

extern "C" int paam_sets_info(const paam_sets* sets, uint32_t* n_sets, uint32_t* n_chains, uint32_t* n_bins) {
  if (!sets) return fail(PAAM_EINVAL, "NULL handle");
  if (n_sets) *n_sets = sets->n_sets;
  if (n_chains) *n_chains = sets->n_chains;
  if (n_bins) *n_bins = sets->n_bins;
  return PAAM_OK;
}

extern "C" void paam_free(paam_sets* sets) {
  if (!sets) return;
  cudaSetDevice(sets->device);
  if (sets->rec) cudaFree(sets->rec);
  if (sets->tickets) cudaFree(sets->tickets);
  if (sets->wide_list) cudaFree(sets->wide_list);
  if (sets->stage) cudaFree(sets->stage);
  if (sets->dstatus) cudaFree(sets->dstatus);
  if (sets->sim_scratch) cudaFree(sets->sim_scratch);
  if (sets->ostage) cudaFree(sets->ostage);
  if (sets->side[0]) {
    for (int i = 0; i < 3; i++) cudaStreamDestroy(sets->side[i]);
    for (int i = 0; i < 17; i++) cudaEventDestroy(sets->ev[i]);
    for (int i = 0; i < 8; i++) cudaEventDestroy(sets->evc[i]);
  }
  std::free(sets);
}

extern "C" const char* paam_strerror(int code) {
  switch (code) {
    case PAAM_OK: return "ok";
    case PAAM_EINVAL: return "invalid argument";
    case PAAM_ECUDA: return "CUDA error";
    case PAAM_ENOMEM: return "out of device memory";
    case PAAM_ERANGE: return "batch size out of range";
    default: return "unknown error";
  }
}

extern "C" const char* paam_last_error(void) { return g_err; }
extern "C" uint64_t paam_kernel_launches(void) { return g_launches.load(); }

extern "C" uint32_t paam_record_bytes(void) { return (uint32_t)sizeof(Record); }

extern "C" int paam_set_device(int device) {
  const cudaError_t e = cudaSetDevice(device);
  return e == cudaSuccess ? PAAM_OK : fail_cuda(e, "paam_set_device");
}

extern "C" int paam_copy(void* dst, const void* src, size_t bytes, paam_stream_t stream) {
  if ((!dst || !src) && bytes) return fail(PAAM_EINVAL, "paam_copy: NULL pointer");
  if (!bytes) return PAAM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? PAAM_OK : fail_cuda(e, "paam_copy");
}
