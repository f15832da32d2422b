// emu.h -- DEBUGGING AID ONLY: compiles the product's CUDA kernels as host C++ and runs every CUDA
// thread of a block as a host thread, with the warp intrinsics implemented as collectives over the
// warp's 32 threads (std::barrier).  A divergent collective deadlocks here, which is the point: it
// finds warp-synchronisation bugs on the CPU.  Never linked into libpaam.so; never used by tests
// that claim GPU parity.
#pragma once
#include <atomic>
#include <barrier>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <thread>
#include <vector>

#define __device__
#define __host__
#define __global__
#define __forceinline__ inline
#define __launch_bounds__(...)
#define __restrict__ __restrict
#define __align__(n) alignas(n)
#define __shared__ static
#define __constant__

struct dim3emu { unsigned x = 0, y = 0, z = 0; };
inline thread_local dim3emu threadIdx, blockIdx;
inline dim3emu gridDim{1, 1, 1}, blockDim{32, 1, 1};

struct uint4 { uint32_t x, y, z, w; };
inline uint4 make_uint4(uint32_t x, uint32_t y, uint32_t z, uint32_t w) { return uint4{x, y, z, w}; }
struct uint2 { uint32_t x, y; };
template <class T> inline T __ldg(const T* p) { return *p; }

namespace emu {
// A warp: one 32-thread barrier for full-warp collectives and one 16-thread barrier per half for
// the masks 0x0000ffff / 0xffff0000 (half-warp groups); any other mask is unsupported here.
struct Warp {
  std::barrier<> bar{32};
  std::barrier<> half[2] = {std::barrier<>(16), std::barrier<>(16)};
  uint64_t slot[32];
};
inline std::vector<Warp*>& warps() { static std::vector<Warp*> w; return w; }
inline std::barrier<>*& block_bar() { static std::barrier<>* b = nullptr; return b; }
inline Warp& W() { return *warps()[threadIdx.x / 32]; }
inline int lane() { return threadIdx.x & 31; }
inline std::barrier<>& bar_of(unsigned mask) {
  Warp& w = W();
  if (mask == 0xffffffffu) return w.bar;
  if (mask == 0x0000ffffu || mask == 0xffff0000u) {
    if (!((mask >> lane()) & 1u)) { std::fprintf(stderr, "emu: lane %d not in mask %08x\n", lane(), mask); std::abort(); }
    return w.half[mask == 0xffff0000u];
  }
  std::fprintf(stderr, "emu: unsupported collective mask %08x\n", mask);
  std::abort();
}
template <class T> inline uint64_t bits(T v) { uint64_t b = 0; std::memcpy(&b, &v, sizeof(T)); return b; }
template <class T> inline T unbits(uint64_t b) { T v; std::memcpy(&v, &b, sizeof(T)); return v; }
template <class T> inline T exch(unsigned mask, T v, int src) {
  Warp& w = W();
  std::barrier<>& b = bar_of(mask);
  w.slot[lane()] = bits(v);
  b.arrive_and_wait();
  const T r = unbits<T>(w.slot[src]);
  b.arrive_and_wait();
  return r;
}
template <class F> inline uint64_t collect(unsigned mask, uint64_t v, F f) {  // lanes in mask get f(slots, mask)
  Warp& w = W();
  std::barrier<>& b = bar_of(mask);
  w.slot[lane()] = v;
  b.arrive_and_wait();
  const uint64_t r = f(w.slot, mask);
  b.arrive_and_wait();
  return r;
}

// Run kernel body `k` for one block of `threads` host threads (one warp collective set per 32).
inline void launch_block(unsigned block, unsigned threads, const std::function<void()>& k) {
  for (auto* w : warps()) delete w;
  warps().clear();
  for (unsigned i = 0; i < threads / 32; i++) warps().push_back(new Warp());
  delete block_bar();
  block_bar() = new std::barrier<>(threads);
  blockDim.x = threads;
  std::vector<std::thread> th;
  for (unsigned t = 0; t < threads; t++)
    th.emplace_back([=, &k]() { threadIdx.x = t; blockIdx.x = block; k(); });
  for (auto& x : th) x.join();
}
}  // namespace emu

inline void __syncwarp(unsigned m = 0xffffffffu) { emu::bar_of(m).arrive_and_wait(); }
template <class T> inline T __shfl_sync(unsigned m, T v, int src, int width = 32) {
  return emu::exch(m, v, (emu::lane() & ~(width - 1)) + (src & (width - 1)));
}
template <class T> inline T __shfl_xor_sync(unsigned m, T v, int x, int width = 32) {
  const int s = emu::lane() ^ x;
  return emu::exch(m, v, ((s & ~(width - 1)) == (emu::lane() & ~(width - 1))) ? s : emu::lane());
}
template <class T> inline T __shfl_up_sync(unsigned m, T v, unsigned d, int width = 32) {
  const int s = emu::lane() - (int)d;
  return emu::exch(m, v, (s < (emu::lane() & ~(width - 1))) ? emu::lane() : s);
}
template <class T> inline T __shfl_down_sync(unsigned m, T v, unsigned d, int width = 32) {
  const int s = emu::lane() + (int)d;
  return emu::exch(m, v, (s > (emu::lane() | (width - 1))) ? emu::lane() : s);
}
inline unsigned __ballot_sync(unsigned m, int p) {
  return (unsigned)emu::collect(m, p ? 1 : 0, [](uint64_t* s, unsigned mk) {
    uint64_t r = 0; for (int i = 0; i < 32; i++) if ((mk >> i) & 1u) r |= (s[i] & 1) << i; return r; });
}
inline int __any_sync(unsigned m, int p) { return __ballot_sync(m, p) != 0; }
inline int __all_sync(unsigned m, int p) { return __ballot_sync(m, p) == m; }
inline unsigned __reduce_add_sync(unsigned m, unsigned v) {
  return (unsigned)emu::collect(m, v, [](uint64_t* s, unsigned mk) {
    uint32_t a = 0; for (int i = 0; i < 32; i++) if ((mk >> i) & 1u) a += (uint32_t)s[i]; return (uint64_t)a; });
}
inline unsigned __reduce_min_sync(unsigned m, unsigned v) {
  return (unsigned)emu::collect(m, v, [](uint64_t* s, unsigned mk) {
    uint32_t a = 0xffffffffu; for (int i = 0; i < 32; i++) if ((mk >> i) & 1u) a = std::min(a, (uint32_t)s[i]); return (uint64_t)a; });
}
inline unsigned __reduce_max_sync(unsigned m, unsigned v) {
  return (unsigned)emu::collect(m, v, [](uint64_t* s, unsigned mk) {
    uint32_t a = 0; for (int i = 0; i < 32; i++) if ((mk >> i) & 1u) a = std::max(a, (uint32_t)s[i]); return (uint64_t)a; });
}
inline unsigned __reduce_or_sync(unsigned m, unsigned v) {
  return (unsigned)emu::collect(m, v, [](uint64_t* s, unsigned mk) {
    uint32_t a = 0; for (int i = 0; i < 32; i++) if ((mk >> i) & 1u) a |= (uint32_t)s[i]; return (uint64_t)a; });
}
inline unsigned __reduce_and_sync(unsigned m, unsigned v) {
  return (unsigned)emu::collect(m, v, [](uint64_t* s, unsigned mk) {
    uint32_t a = 0xffffffffu; for (int i = 0; i < 32; i++) if ((mk >> i) & 1u) a &= (uint32_t)s[i]; return (uint64_t)a; });
}
inline unsigned __match_any_sync(unsigned m, unsigned long long v) {
  const int l = emu::lane();
  return (unsigned)emu::collect(m, v, [l](uint64_t* s, unsigned mk) {
    uint64_t r = 0; for (int i = 0; i < 32; i++) if ((mk >> i) & 1u) r |= (uint64_t)(s[i] == s[l]) << i; return r; });
}
inline unsigned __match_any_sync(unsigned m, unsigned v) {
  const int l = emu::lane();
  return (unsigned)emu::collect(m, v, [l](uint64_t* s, unsigned mk) {
    uint64_t r = 0; for (int i = 0; i < 32; i++) if ((mk >> i) & 1u) r |= (uint64_t)(s[i] == s[l]) << i; return r; });
}

inline int __popc(unsigned x) { return __builtin_popcount(x); }
inline int __popcll(unsigned long long x) { return __builtin_popcountll(x); }
inline int __clz(unsigned x) { return x ? __builtin_clz(x) : 32; }
inline int __clzll(unsigned long long x) { return x ? __builtin_clzll(x) : 64; }
inline int __ffs(unsigned x) { return x ? __builtin_ctz(x) + 1 : 0; }
inline unsigned __vcmpeq4(unsigned a, unsigned b) {  // per byte: 0xff where equal
  unsigned r = 0;
  for (int i = 0; i < 4; i++) if (((a >> (8 * i)) & 0xffu) == ((b >> (8 * i)) & 0xffu)) r |= 0xffu << (8 * i);
  return r;
}
inline int __ffsll(unsigned long long x) { return x ? __builtin_ctzll(x) + 1 : 0; }
inline unsigned __fns(unsigned mask, unsigned base, int offset) {
  for (unsigned i = base; i < 32; i++)
    if ((mask >> i) & 1u) { if (--offset == 0) return i; }
  return 0xffffffffu;
}
inline unsigned __umulhi(unsigned a, unsigned b) { return (unsigned)(((uint64_t)a * b) >> 32); }
inline unsigned __funnelshift_r(unsigned lo, unsigned hi, unsigned s) { return (unsigned)((((uint64_t)hi << 32) | lo) >> (s & 31u)); }
inline unsigned long long __umul64hi(unsigned long long a, unsigned long long b) {
  return (unsigned long long)(((unsigned __int128)a * b) >> 64);
}
inline double __drcp_rn(double x) { return 1.0 / x; }
inline uint32_t min(uint32_t a, uint32_t b) { return a < b ? a : b; }
inline uint32_t max(uint32_t a, uint32_t b) { return a > b ? a : b; }
inline uint64_t min(uint64_t a, uint64_t b) { return a < b ? a : b; }
inline uint64_t max(uint64_t a, uint64_t b) { return a > b ? a : b; }
inline unsigned long long min(unsigned long long a, unsigned long long b) { return a < b ? a : b; }
inline int min(int a, int b) { return a < b ? a : b; }
inline int max(int a, int b) { return a > b ? a : b; }
inline unsigned atomicAdd(unsigned* p, unsigned v) { return __atomic_fetch_add(p, v, __ATOMIC_RELAXED); }
inline unsigned long long atomicAdd(unsigned long long* p, unsigned long long v) { return __atomic_fetch_add(p, v, __ATOMIC_RELAXED); }
inline unsigned atomicOr(unsigned* p, unsigned v) { return __atomic_fetch_or(p, v, __ATOMIC_RELAXED); }
inline unsigned long long atomicMax(unsigned long long* p, unsigned long long v) {
  unsigned long long cur = __atomic_load_n(p, __ATOMIC_RELAXED);
  while (cur < v && !__atomic_compare_exchange_n(p, &cur, v, false, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {}
  return cur;
}
inline void __syncthreads() { emu::block_bar()->arrive_and_wait(); }

namespace paam {
inline uint32_t lanemask_lt() { return (1u << emu::lane()) - 1u; }
}
