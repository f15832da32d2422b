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

struct dim3emu { unsigned x = 0, y = 0, z = 0; };
inline thread_local dim3emu threadIdx, blockIdx;
inline dim3emu gridDim{1, 1, 1}, blockDim{32, 1, 1};

struct uint4 { uint32_t x, y, z, w; };
template <class T> inline T __ldg(const T* p) { return *p; }

namespace emu {
struct Warp {
  std::barrier<> bar{32};
  uint64_t slot[32];
};
inline std::vector<Warp*>& warps() { static std::vector<Warp*> w; return w; }
inline std::barrier<>*& block_bar() { static std::barrier<>* b = nullptr; return b; }
inline Warp& W() { return *warps()[threadIdx.x / 32]; }
inline int lane() { return threadIdx.x & 31; }
template <class T> inline uint64_t bits(T v) { uint64_t b = 0; std::memcpy(&b, &v, sizeof(T)); return b; }
template <class T> inline T unbits(uint64_t b) { T v; std::memcpy(&v, &b, sizeof(T)); return v; }
template <class T> inline T exch(T v, int src) {
  Warp& w = W();
  w.slot[lane()] = bits(v);
  w.bar.arrive_and_wait();
  const T r = unbits<T>(w.slot[src]);
  w.bar.arrive_and_wait();
  return r;
}
template <class F> inline uint64_t collect(uint64_t v, F f) {  // all lanes get f(slots)
  Warp& w = W();
  w.slot[lane()] = v;
  w.bar.arrive_and_wait();
  const uint64_t r = f(w.slot);
  w.bar.arrive_and_wait();
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

inline void __syncwarp(unsigned = 0xffffffffu) { emu::W().bar.arrive_and_wait(); }
template <class T> inline T __shfl_sync(unsigned, T v, int src, int width = 32) {
  return emu::exch(v, (emu::lane() & ~(width - 1)) + (src & (width - 1)));
}
template <class T> inline T __shfl_xor_sync(unsigned, T v, int m, int = 32) { return emu::exch(v, emu::lane() ^ m); }
template <class T> inline T __shfl_up_sync(unsigned, T v, unsigned d, int = 32) {
  const int s = emu::lane() - (int)d;
  const T r = emu::exch(v, s < 0 ? emu::lane() : s);
  return r;
}
template <class T> inline T __shfl_down_sync(unsigned, T v, unsigned d, int = 32) {
  const int s = emu::lane() + (int)d;
  return emu::exch(v, s > 31 ? emu::lane() : s);
}
inline unsigned __ballot_sync(unsigned, int p) {
  return (unsigned)emu::collect(p ? 1 : 0, [](uint64_t* s) { uint64_t m = 0; for (int i = 0; i < 32; i++) m |= (s[i] & 1) << i; return m; });
}
inline int __any_sync(unsigned m, int p) { return __ballot_sync(m, p) != 0; }
inline int __all_sync(unsigned m, int p) { return __ballot_sync(m, p) == 0xffffffffu; }
inline unsigned __reduce_add_sync(unsigned, unsigned v) {
  return (unsigned)emu::collect(v, [](uint64_t* s) { uint32_t a = 0; for (int i = 0; i < 32; i++) a += (uint32_t)s[i]; return (uint64_t)a; });
}
inline unsigned __reduce_min_sync(unsigned, unsigned v) {
  return (unsigned)emu::collect(v, [](uint64_t* s) { uint32_t a = 0xffffffffu; for (int i = 0; i < 32; i++) a = std::min(a, (uint32_t)s[i]); return (uint64_t)a; });
}
inline unsigned __reduce_max_sync(unsigned, unsigned v) {
  return (unsigned)emu::collect(v, [](uint64_t* s) { uint32_t a = 0; for (int i = 0; i < 32; i++) a = std::max(a, (uint32_t)s[i]); return (uint64_t)a; });
}
inline unsigned __reduce_or_sync(unsigned, unsigned v) {
  return (unsigned)emu::collect(v, [](uint64_t* s) { uint32_t a = 0; for (int i = 0; i < 32; i++) a |= (uint32_t)s[i]; return (uint64_t)a; });
}
inline unsigned __match_any_sync(unsigned, unsigned v) {
  const int l = emu::lane();
  return (unsigned)emu::collect(v, [l](uint64_t* s) { uint64_t m = 0; for (int i = 0; i < 32; i++) m |= (uint64_t)(s[i] == s[l]) << i; return m; });
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
