// tacos_device.cuh -- device helpers of the product path (Philox, bit select,
// warp reductions).  Product side only; the oracle has its own Philox.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "tacos_internal.h"

namespace tacos {

// last launch error text (thread-local), set by check_launch
char *cuda_error_buffer();
int check_launch(const char *what);

// ---------------------------------------------------------------------------
// Philox4x32-10 (R2; Salmon et al. SC'11).  Counter (t_lo, t_hi, link, sigma),
// key (seed_lo, seed_hi); word 0 = order key, word 1 = pick draw.
// ---------------------------------------------------------------------------
// Bounds-checked build (build.py --variant checked -DTACOS_CHECKED=1, loaded through
// TACOS_LIB): every shared-memory / global index of the search kernels is checked and a
// violation traps with its site.  Stands in for compute-sanitizer, which is closed on the
// GPU pool.
#ifndef TACOS_CHECKED
#define TACOS_CHECKED 0
#endif
#if TACOS_CHECKED
#define TCHECK(cond, what)                                                                              \
  do {                                                                                                  \
    if (!(cond)) {                                                                                      \
      printf("tacos check failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__, blockIdx.x, \
             threadIdx.x);                                                                              \
      __trap();                                                                                         \
    }                                                                                                   \
  } while (0)
#else
#define TCHECK(cond, what) \
  do {                     \
  } while (0)
#endif
__device__ __forceinline__ uint32_t dynamic_smem_bytes() {
  uint32_t r;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// Position of the r-th (0-based) set bit of x, x having more than r set bits:
// popc bisection, branch-free (predicated selects).
__device__ __forceinline__ uint32_t select_bit(uint32_t x, uint32_t r) {
  uint32_t pos = 0, c;
  bool m;
  c = __popc(x & 0xFFFFu); m = r >= c; r = m ? r - c : r; x = m ? x >> 16 : x; pos += m ? 16u : 0u;
  c = __popc(x & 0xFFu);   m = r >= c; r = m ? r - c : r; x = m ? x >> 8 : x;  pos += m ? 8u : 0u;
  c = __popc(x & 0xFu);    m = r >= c; r = m ? r - c : r; x = m ? x >> 4 : x;  pos += m ? 4u : 0u;
  c = __popc(x & 0x3u);    m = r >= c; r = m ? r - c : r; x = m ? x >> 2 : x;  pos += m ? 2u : 0u;
  c = x & 1u;              m = r >= c;                                         pos += m ? 1u : 0u;
  return pos;
}

// Same result without POPC (POPC issues on the XU pipe at a fraction of the ALU rate):
// SWAR bit counts of the 2-bit pairs, nibbles and bytes, the inclusive byte prefix by one
// multiply, then byte -> nibble -> pair -> bit, all on the ALU / FMA pipes.
__device__ __forceinline__ uint32_t select_bit_swar(uint32_t x, uint32_t r) {
  const uint32_t c1 = x - ((x >> 1) & 0x55555555u);                    // 2-bit counts
  const uint32_t c2 = (c1 & 0x33333333u) + ((c1 >> 2) & 0x33333333u);  // 4-bit counts
  const uint32_t c3 = (c2 + (c2 >> 4)) & 0x0F0F0F0Fu;                  // byte counts
  const uint32_t pre = c3 * 0x01010101u;  // byte i: set bits in bytes 0..i (monotone)
  const uint32_t p0 = pre & 0xFFu, p1 = (pre >> 8) & 0xFFu, p2 = (pre >> 16) & 0xFFu;
  uint32_t pos = 0, base = 0;
  if (r >= p0) { pos = 8u; base = p0; }
  if (r >= p1) { pos = 16u; base = p1; }
  if (r >= p2) { pos = 24u; base = p2; }
  r -= base;
  const uint32_t n = (c2 >> pos) & 0xFu;
  if (r >= n) { r -= n; pos += 4u; }
  const uint32_t q = (c1 >> pos) & 0x3u;
  if (r >= q) { r -= q; pos += 2u; }
  return pos + ((r >= ((x >> pos) & 1u)) ? 1u : 0u);
}

__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) { return __reduce_add_sync(0xFFFFFFFFu, v); }
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}
__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xFFFFFFFFu, v, o);
    v = y < v ? y : v;
  }
  return v;
}

// ---------------------------------------------------------------------------
// Distributed shared memory (thread-block clusters), explicit shared::cluster
// PTX: mapa for the peer address, ld.shared::cluster for reads, relaxed
// cluster-scope red for the exchanged counters (ordered by the cluster barrier).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t dsmem_addr(const void *p, uint32_t rank) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t dsmem_ld(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void dsmem_st_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void dsmem_st_u64(uint32_t addr, unsigned long long v) {
  asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ void dsmem_st_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void dsmem_st_u16(uint32_t addr, uint16_t v) {
  asm volatile("st.shared::cluster.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
__device__ __forceinline__ void dsmem_add_u32(uint32_t addr, uint32_t v) {
  asm volatile("red.relaxed.cluster.shared::cluster.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// 64-bit min/add on distributed shared memory are not used: on sm_100a a
// remote red.min.u64 was observed to be lost (measured), so 64-bit values are
// exchanged through per-rank slots written with plain remote stores.
__device__ __forceinline__ void dsmem_or_b32(uint32_t addr, uint32_t v) {
  asm volatile("red.relaxed.cluster.shared::cluster.or.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ uint4 andnot4(uint4 a, uint4 b) {
  return make_uint4(a.x & ~b.x, a.y & ~b.y, a.z & ~b.z, a.w & ~b.w);
}
__device__ __forceinline__ uint4 and4(uint4 a, uint4 b) { return make_uint4(a.x & b.x, a.y & b.y, a.z & b.z, a.w & b.w); }
__device__ __forceinline__ uint32_t popc4(uint4 a) { return __popc(a.x) + __popc(a.y) + __popc(a.z) + __popc(a.w); }

}  // namespace tacos
