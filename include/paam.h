/* paam.h -- C ABI of the B200-native PAAM response-time analyser and arbitration simulator.
 *
 * What the library computes (PAPER.md = /root/reference/PAPER.md, "P:<line>"; SPEC.md "S:<line>"):
 *   For every chain set ("SystemConfig") of a batch, the worst-case end-to-end response
 *   time (WCRT) of every processing chain whose callbacks run on
 *   single-threaded, non-preemptive, priority-driven executors (PiCAS) and send their
 *   accelerator segments to a PAAM server (bucket downsampling P:279, rules R1-R4 P:366-373):
 *     Eq.1  H*_c = H_c + sum eps
 *     Eq.2  mu(t) = ceil(t/T) + 1                        (Lemma 1)
 *     Eq.3  per-segment handling-time fixed point        (Lemma 2)
 *     Eq.4  per-chain handling time, union of hps        (Lemma 3)
 *     H_c = min(Eq.3 summed, Eq.4)
 *     Eq.5  chain WCRT fixed point                       (Theorem 1)
 *     R*   = sum of sub-chain R_c + comm per crossing
 *   and the set's schedulability verdict (admission test).  The readings taken where the
 *   paper is silent or garbled are listed in DESIGN.md ("Readings", A1-A16).
 *   paam_simulate runs the discrete-event simulation of the PAAM arbitration (App. A
 *   rules D1-D17) and checks observed response times against the bounds.
 *
 * Conventions.
 *   - Every time is an unsigned 64-bit integer number of nanoseconds.  Each individual
 *     period, deadline, WCET, eps and kappa must be < 2^48 ns (about 78 hours; PAAM_SET_ERANGE
 *     otherwise), the comm cost too (PAAM_EINVAL).  A set whose times are all < 2^31 - 1 ns (about
 *     2.1 s) runs on the u32 kernels, whose sums saturate just above the deadline -- exact, because any
 *     value above the deadline is a miss; a set with a larger time is handed over
 *     to an exact u64 path (wide.cu) with the same results and statuses.  The DES computes in 32-bit
 *     time distances: it reports such a set PAAM_SIM_WIDE and needs comm cost < 2^31 - 1 ns.
 *   - Indices inside a set are set-local (executor, accelerator, unit); CSR offset arrays are global.
 *   - All calls are asynchronous on the given CUDA stream unless stated otherwise.  Exceptions that
 *     synchronise the stream: paam_pack / paam_repack with host-resident input, paam_pack_analyze
 *     with a host out_status, and paam_generate / paam_regenerate (they read the batch totals back to
 *     size the arrays).
 *   - Calls on one paam_sets handle share its work counters and staging buffers: order them (e.g.
 *     issue them on one stream).  Different handles are independent.
 *   - The caller owns every input and output buffer.  The library owns the opaque paam_sets handle
 *     (device memory) until paam_free.
 *   - Return value: 0 = OK, negative = the whole call failed (PAAM_E*).  Per-set validation failures
 *     do not fail the call; they are reported per set through out_status (PAAM_SET_*), and such a set
 *     gets sched = 0 and every WCRT = PAAM_UNSCHED.
 */
#ifndef PAAM_H
#define PAAM_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* paam_stream_t; /* a cudaStream_t (may be NULL = legacy default stream) */

/* ---- call-level return codes -------------------------------------------------------------- */
#define PAAM_OK 0
#define PAAM_EINVAL -1 /* bad argument (NULL pointer, n == 0 where not allowed, bad flag, ...) */
#define PAAM_ECUDA -2  /* a CUDA runtime call failed; paam_last_error() has the detail */
#define PAAM_ENOMEM -3 /* device allocation failed */
#define PAAM_ERANGE -4 /* batch-level size out of range (e.g. more than 2^32-1 chains) */

/* ---- per-set validation status (out_status[i]) -------------------------------------------- */
/* Checked in this order; the first failing rule is reported. */
#define PAAM_SET_OK 0
#define PAAM_SET_ERANGE 1    /* over the size caps below, T == 0, a time >= 2^48 ns, or a utilisation
                                bin >= n_bins (such a set is counted in no bin) */
#define PAAM_SET_EDANGLING 2 /* chain without callbacks, callback without segments, executor or
                                unit index out of range */
#define PAAM_SET_EACCEL 3    /* ACCEL segment on an undeclared accelerator */
#define PAAM_SET_ESHAPE 4    /* segment WCET == 0, CPU/ACCEL segments do not alternate, or a
                                chain revisits an executor non-contiguously (A13) */
#define PAAM_SET_EDUPPRIO 5  /* duplicate chain priority or duplicate process priority of
                                two executors on one core */
#define PAAM_SET_EDEADLINE 6 /* CRITICAL chain with D > T or D == 0 (P:128 constrained deadlines) */
#define PAAM_SET_ECORE 7     /* an accelerator's server core hosts a client executor (R1) */

/* ---- per-set size caps (one set = one warp, record staged in shared memory) ---------------- */
#define PAAM_MAX_CHAINS 32
#define PAAM_MAX_SUBCHAINS 32
#define PAAM_MAX_CALLBACKS 64
#define PAAM_MAX_ACCEL_SEGS 64
#define PAAM_MAX_SEGMENTS 192
#define PAAM_MAX_EXECUTORS 32
#define PAAM_MAX_ACCELS 4
#define PAAM_MAX_UNITS 8   /* summed over the set's accelerators */
#define PAAM_MAX_BUCKETS 32

#define PAAM_UNSCHED UINT64_MAX /* WCRT of a chain whose fixed point exceeds its deadline */

/* ---- flags (paam_batch.flags) --------------------------------------------------------------- */
#define PAAM_MEM_HOST 0
#define PAAM_MEM_DEVICE 1
#define PAAM_FLAG_BLOCKING_SOUND 0x1u /* B_c charges an LP callback's accelerator handling time
                                          (SURVEY.md §8(c) A10); default = the paper's B_c */
#define PAAM_FLAG_WFD_UNITS 0x2u      /* assign accelerator segments to units by Worst-Fit-Decreasing
                                           instead of seg_unit: per accelerator,
                                          callbacks by decreasing (sum A << 24) / T onto the least-
                                          loaded unit (ties: lowest unit); a callback's segments stay
                                          together */
#define PAAM_FLAG_VERDICT_ONLY 0x4u   /* verdict-only sweeps: the analysis of a
                                          set stops at its first CRITICAL sub-chain whose Eq.5 iterate
                                          exceeds D (R* > D follows), so out_sched and
                                          out_bins are identical to the full mode; out_wcrt must be
                                          NULL (PAAM_EINVAL otherwise).  paam_admit ignores the flag
                                          (its decision names the first failing chain). */

/* Raw batch: the paper's system model as flat CSR arrays.  `mem` says whether the
 * pointers are host or device memory.  Sizes n_chains..n_accels are the totals (= last entries
 * of the offset arrays).  Layout per set i:
 *   chains     [set_chain_off[i], set_chain_off[i+1])  : T, D, priority (unique, larger = higher),
 *                                                        class (0 CRITICAL, 1 BEST_EFFORT)
 *   callbacks of chain g [chain_cb_off[g], chain_cb_off[g+1]), in chain order
 *   segments of callback j [cb_seg_off[j], cb_seg_off[j+1]): kind 0 CPU / 1 ACCEL, WCET, and for
 *                                                        ACCEL the set-local accelerator and unit
 *   executors  [set_exec_off[i], set_exec_off[i+1])    : core, process priority (unique per core,
 *                                                        larger = higher), wait 0 SUSPEND / 1 SPIN
 *   accelerators [set_accel_off[i], ...)                : buckets n (>1 = preemptive GPU-like,
 *                                                        1 = TPU-like), units, server core, eps, kappa
 * Offset arrays must be non-decreasing.  Within a set, a chain's callback range or a callback's
 * segment range that leaves the set's own range is reported PAAM_SET_EDANGLING (never read out of
 * range); a set whose ranges exceed the caps is PAAM_SET_ERANGE.
 */
typedef struct {
  uint32_t n_sets;
  int32_t mem; /* PAAM_MEM_HOST | PAAM_MEM_DEVICE */
  uint32_t n_chains, n_cbs, n_segs, n_execs, n_accels, n_bins;
  const uint32_t *set_chain_off, *set_exec_off, *set_accel_off; /* [n_sets+1] */
  const uint64_t *chain_T, *chain_D;
  const uint32_t *chain_prio;
  const uint8_t *chain_class;
  const uint32_t *chain_cb_off; /* [n_chains+1] */
  const uint16_t *cb_exec;      /* set-local executor of each callback */
  const uint32_t *cb_seg_off;   /* [n_cbs+1] */
  const uint8_t *seg_kind;
  const uint64_t *seg_wcet;
  const uint8_t *seg_accel, *seg_unit;
  const uint8_t *exec_core;
  const uint32_t *exec_prio;
  const uint8_t *exec_wait;
  const uint8_t *accel_buckets, *accel_units, *accel_server_core;
  const uint64_t *accel_eps, *accel_kappa;
  const uint32_t *set_bin; /* utilisation bin of each set, < n_bins (may be NULL: no bin counts) */
  uint64_t comm_cost;      /* eps' per executor crossing (A9), default 100 us */
  uint32_t flags;          /* PAAM_FLAG_* */
  uint32_t _pad;
} paam_batch;

/* Generator knobs; integer only, reproduced bit-for-bit on host and device. */
typedef struct {
  uint32_t m_lo, m_hi, cbs_per_chain, n_bins;
  uint32_t u_lo_q20, u_step_q20;
  uint32_t ratio_acc, ratio_cpu;
  uint32_t period_min_us, period_span_q12;
  uint32_t exec_mode, n_cores, n_exec;
  uint32_t n_accel;
  uint32_t buckets[4], units[4];
  uint64_t eps[4], kappa[4];
  uint32_t be_frac_q16, spin_frac_q16, cpu_only_frac_q16, xexec_frac_q16, rm_priorities;
  uint32_t _pad;
} paam_gen_params;

/* Device-resident raw batch produced by paam_generate (owned by the library). */
typedef struct paam_raw paam_raw;
/* Device-resident packed records (owned by the library). */
typedef struct paam_sets paam_sets;

/* paam_generate -- §8(a) step 1.  Generates sets [first_index, first_index + n) of the stream
 * `seed` into a device raw batch.  Returns PAAM_EINVAL if the parameters exceed the generator's
 * caps.  *out receives a handle; paam_raw_batch() exposes its arrays as a paam_batch (mem = DEVICE). */
int paam_generate(const paam_gen_params* params, uint64_t seed, uint64_t first_index, uint32_t n,
                  uint64_t comm_cost, uint32_t flags, paam_raw** out, paam_stream_t stream);
/* paam_regenerate -- paam_generate into an existing handle (for timed loops): its device buffers are
 * reused when the new batch fits them (else they grow).  Same arguments and errors as paam_generate;
 * previously obtained paam_raw_batch views of the handle become invalid. */
int paam_regenerate(paam_raw* raw, const paam_gen_params* params, uint64_t seed, uint64_t first_index, uint32_t n,
                    uint64_t comm_cost, uint32_t flags, paam_stream_t stream);
int paam_raw_batch(const paam_raw* raw, paam_batch* out);

/* paam_sweep -- §8(a) steps 1-6 as one device-resident sweep over sets [first_index, first_index + n)
 * of the stream `seed`: chunks of `chunk` sets (paam_sweep_create) are generated, packed and analysed,
 * the generation of chunk i+1 overlapping the pack + analysis of chunk i on two internal streams;
 * the raw batches are laid out at the generator's per-set upper bounds, so nothing is read back to
 * the host and the call never synchronises.  Outputs: out_sched [n] (device, may be NULL) and
 * out_bins [n_bins*2] (device, ACCUMULATED, may be NULL); no WCRTs (flags as paam_batch.flags,
 * PAAM_FLAG_VERDICT_ONLY allowed).  The same verdicts and bins as paam_generate + paam_pack_analyze.
 * Errors: PAAM_EINVAL for bad parameters or a chunk whose capacity exceeds 32-bit offsets. */
typedef struct paam_sweeper paam_sweeper;
int paam_sweep_create(uint32_t chunk, paam_sweeper** out);
int paam_sweep(paam_sweeper* sweeper, const paam_gen_params* params, uint64_t seed, uint64_t first_index, uint32_t n,
               uint64_t comm_cost, uint32_t flags, uint8_t* out_sched, int64_t* out_bins, paam_stream_t stream);
void paam_sweep_free(paam_sweeper* sweeper);
void paam_raw_free(paam_raw* raw);

/* paam_pack -- §8(a) step 2.  Validates every set and derives the per-set record the analysis and
 * the simulator read: sub-chains (maximal runs of callbacks on one executor), E_c, delta_c,
 * A* = A + 2 kappa_eff, the bucket map, LP blocking per segment,
 * interference sets hps/hp/hpp and the per-core analysis order.
 * out_status: NULL or an array of n_sets int32 in the same memory space as the batch.
 * Host input is copied to the device on `stream` (the call then synchronises that stream). */
int paam_pack(const paam_batch* batch, paam_sets** out, int32_t* out_status, paam_stream_t stream);
/* Re-pack into an existing handle of sufficient capacity (no allocation; for timed loops). */
int paam_repack(const paam_batch* batch, paam_sets* sets, int32_t* out_status, paam_stream_t stream);

/* paam_analyze -- §8(a) steps 3-6.  For each of the first n sets of the handle:
 *   out_wcrt  [n_chains total, global chain order of the batch] R*_Gamma in ns or PAAM_UNSCHED;
 *             may be NULL (verdict-only sweeps).
 *   out_sched [n] 1 iff every CRITICAL chain has R* <= D (invalid sets: 0); may be NULL.
 *   out_bins  [n_bins*2] int64, ACCUMULATED (+=): bins[2b] += sets of bin b, bins[2b+1] += schedulable
 *             sets of bin b; may be NULL.  Integer sums, so the result is order-independent.
 * Device pointers only. */
int paam_analyze(const paam_sets* sets, uint32_t n, uint64_t* out_wcrt, uint8_t* out_sched,
                 int64_t* out_bins, paam_stream_t stream);

/* paam_admit -- batched admission test.  Each packed set is a what-if
 * "system plus candidate chain(s)"; the decision is computed by the same analysis as paam_analyze:
 *   out_decision[i] = -1            ACCEPT: every CRITICAL chain has R* <= D;
 *                   = c >= 0        REJECT: c is the set-local index of the highest-priority CRITICAL
 *                                   chain with R* > D (old chain or candidate);
 *                   = -2 - status   REJECT by validation (status = PAAM_SET_*, e.g. duplicate priority).
 *   out_wcrt as in paam_analyze (may be NULL).  Device pointers only. */
int paam_admit(const paam_sets* sets, uint32_t n, int32_t* out_decision, uint64_t* out_wcrt, paam_stream_t stream);

/* paam_pack_analyze -- steps 2-6 in one call: one fused kernel validates and derives each set and
 * solves its fixed points with the derived record on chip (no record is written), followed by the
 * exact u64 kernel for the sets it hands over (a time >= 2^31 - 1 ns).  A host batch is copied to the
 * device in chunks on an internal stream, each chunk's copy overlapping the kernel of the previous
 * chunk; with pinned host memory the copies are asynchronous, so the caller must not modify the batch
 * until `stream` has completed.  Same results as paam_repack followed by paam_analyze; `sets` must
 * have capacity for batch->n_sets (from paam_pack).  out_status is in the batch's memory space; a host
 * out_status makes the call synchronise `stream` (as paam_repack).  With a host batch, out_wcrt and
 * out_sched may be host memory too (pinned for asynchrony): the kernels write a device staging copy and
 * each chunk's WCRTs and verdicts are copied back as soon as its kernels finish, overlapping the next
 * chunk's H2D; they are complete when `stream` is.  With a device batch they must be device memory
 * (PAAM_EINVAL otherwise).  out_bins is always device memory (accumulated).  The handle keeps the batch
 * for a later paam_analyze / paam_admit / paam_simulate (which then pack it first). */
int paam_pack_analyze(const paam_batch* batch, paam_sets* sets, int32_t* out_status, uint64_t* out_wcrt,
                      uint8_t* out_sched, int64_t* out_bins, paam_stream_t stream);

/* Compact batch: paam_batch with 32-bit times and one byte per segment, 1.4 KB instead of 2.3 KB per
 * config-3 set, for host batches whose transfer bounds the call (the H2D copy of a host batch runs at
 * the PCIe rate).  Layout and meaning as paam_batch, except:
 *   chain_T, chain_D, seg_wcet, accel_eps, accel_kappa   uint32_t ns (a time below 2^32 ns; times
 *                                                        >= 2^31 - 1 ns take the exact u64 path);
 *   seg_meta   kind | accel << 1 | unit << 3 (kind 0 CPU / 1 ACCEL, set-local accelerator < 4,
 *              unit < 8; for a CPU segment accel and unit are ignored) -- replaces seg_kind,
 *              seg_accel and seg_unit;
 *   cb_exec    uint8_t.
 * Every value a paam_batch can express inside these ranges means the same; results are identical to
 * paam_pack_analyze on the equivalent paam_batch. */
typedef struct {
  uint32_t n_sets;
  int32_t mem; /* PAAM_MEM_HOST | PAAM_MEM_DEVICE */
  uint32_t n_chains, n_cbs, n_segs, n_execs, n_accels, n_bins;
  const uint32_t *set_chain_off, *set_exec_off, *set_accel_off; /* [n_sets+1] */
  const uint32_t *chain_T, *chain_D;
  const uint32_t *chain_prio;
  const uint8_t *chain_class;
  const uint32_t *chain_cb_off; /* [n_chains+1] */
  const uint8_t *cb_exec;
  const uint32_t *cb_seg_off;   /* [n_cbs+1] */
  const uint8_t *seg_meta;
  const uint32_t *seg_wcet;
  const uint8_t *exec_core;
  const uint32_t *exec_prio;
  const uint8_t *exec_wait;
  const uint8_t *accel_buckets, *accel_units, *accel_server_core;
  const uint32_t *accel_eps, *accel_kappa;
  const uint32_t *set_bin;
  uint64_t comm_cost;
  uint32_t flags;
  uint32_t _pad;
} paam_batch32;

/* paam_pack_analyze32 -- paam_pack_analyze on a compact batch (same outputs, same errors).  The handle
 * keeps no batch a later paam_analyze / paam_admit / paam_simulate could pack: those return
 * PAAM_EINVAL until a paam_pack / paam_repack / paam_pack_analyze. */
int paam_pack_analyze32(const paam_batch32* batch, paam_sets* sets, int32_t* out_status, uint64_t* out_wcrt,
                        uint8_t* out_sched, int64_t* out_bins, paam_stream_t stream);

/* paam_simulate -- §8(a) steps 7-8.  Discrete-event simulation of every set (DESIGN.md App. A,
 * rules D1-D17: PiCAS executors, fixed-priority cores, PAAM bucket queues with cross-bucket
 * preemption, eps per request, kappa per switch) over releases in [0, horizon), run until every
 * released instance completes.  Chain c of set i is released at phase + k*T with phase = 0 when
 * seed == 0, else pg_phase(seed, first_index + i, c, T) (gen/paam_gen.h).  sim_flags: 0 = PAAM, or
 * PAAM_SIM_FIFO_DIRECT (the direct-invocation baseline the paper compares against).
 * Overrun (D14): a CRITICAL chain queues every release (an unbounded backlog), a BE chain drops
 * its older pending, not-started instances.  The device keeps PAAM_SIM_QCAP instance slots per chain:
 * a release that would make a chain's (QCAP+1)-th live instance stops that set's run at that release
 * and reports PAAM_SIM_BACKLOG -- never a silently different simulation.  Up to the stop the run is
 * exact, so a stopped set's resp / count / misses / drops are lower bounds of the full run's.
 * Outputs (device pointers; every one may be NULL):
 *   resp     [n_chains total] maximum observed end-to-end response time per chain (0 if none) (D16).
 *   count    [n_chains total] completed instances per chain.
 *   misses   [n_chains total] completed instances whose response exceeded D (D16).
 *   drops    [n_chains total] BE instances dropped at a release (D14).
 *   digest   [n] order-independent FNV-1a-64 digest of the event records (D17); NULL: events are not
 *            hashed at all (faster).
 *   status   [n] PAAM_SIM_OK, or PAAM_SIM_INVALID (validation failed at pack: outputs 0),
 *            PAAM_SIM_BACKLOG or PAAM_SIM_STEPCAP (the run stopped early, see above).
 *   bound    [n_chains total] input: WCRTs from paam_analyze, or NULL.  In every set whose run did not
 *            stop and whose CRITICAL chains all have bound <= D (the analysis' schedulable sets,
 *            Lemma 1), each CRITICAL chain with resp > bound is a violation of P:533:
 *   violations [1] int64, += the violations;
 *   witness  [2*max_witness] u32 (set index in the batch, set-local chain index) of violations, in
 *            slot v = the value of *violations before that violation was added; slots >= max_witness
 *            are not written (zero *violations first for the first max_witness).  Needs violations.
 *   stopped  [1] int64, += sets whose run stopped early (BACKLOG / STEPCAP).
 * Reads the raw batch the handle was packed from: a DEVICE batch must still be alive (a HOST batch
 * was staged by paam_pack).  Errors: PAAM_EINVAL for an unknown sim flag, n beyond the handle, or
 * witness without violations. */
#define PAAM_SIM_FIFO_DIRECT 0x1u /* baseline arbitration: one FIFO per unit in arrival
                                     order, non-preemptive, no eps, no kappa, buckets ignored */
#define PAAM_SIM_QCAP 4           /* instance slots per chain on the device */
#define PAAM_SIM_STEP_CAP 50000000ull /* event timestamps per set before a run is stopped */
#define PAAM_SIM_OK 0
#define PAAM_SIM_INVALID 1
#define PAAM_SIM_BACKLOG 2
#define PAAM_SIM_STEPCAP 3
#define PAAM_SIM_WIDE 4    /* not simulated: the set has a time >= 2^31 - 1 ns (the DES computes in 32-bit time
                              distances); the analysis handles such sets exactly (u64 path) */
typedef struct {
  uint64_t *resp, *count, *misses, *drops;
  uint64_t* digest;
  int32_t* status;
  const uint64_t* bound;
  int64_t* violations;
  uint32_t* witness;
  int64_t* stopped;
  uint32_t max_witness, _pad;
} paam_sim_out;
int paam_simulate(const paam_sets* sets, uint32_t n, uint64_t horizon, uint64_t seed, uint64_t first_index,
                  uint32_t sim_flags, const paam_sim_out* out, paam_stream_t stream);

/* Handle queries (synchronous, small). */
int paam_sets_info(const paam_sets* sets, uint32_t* n_sets, uint32_t* n_chains, uint32_t* n_bins);
void paam_free(paam_sets* sets);

/* Make `device` current for this thread in the library's CUDA runtime.  paam_generate and paam_pack
 * allocate on the current device; every later call on a handle switches to the handle's device
 * itself.  (The library links its own runtime: a caller's cudaSetDevice does not reach it.) */
int paam_set_device(int device);

/* Utility: synchronous copy between any two memory spaces (cudaMemcpyDefault) on `stream`. */
int paam_copy(void* dst, const void* src, size_t bytes, paam_stream_t stream);
uint32_t paam_record_bytes(void); /* size of one packed per-set record in device memory */

const char* paam_strerror(int code);
const char* paam_last_error(void); /* thread-local detail of the last failure */
uint64_t paam_kernel_launches(void); /* kernels launched by this library since load (process-wide) */

#ifdef __cplusplus
}
#endif
#endif
