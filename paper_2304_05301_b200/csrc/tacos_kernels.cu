// tacos_kernels.cu -- sm_100a kernels of the TACOS-Greedy hot path.
//
// PAPER.md citations "P:L<n>"; readings "R<n>" = DESIGN.md §3.
//
//   greedy_kernel     rows a2-a6: one CTA per (seed, orientation) job runs the
//                     whole event loop of one greedy synthesis (P:L249-253
//                     §VI.A, §VI.B) with its bitsets resident in
//                     shared memory when they fit (else in HBM/L2):
//                       PA arrivals at t (R7), done test
//                       PB free/live links, Philox draws (R2)
//                       PC shorter-link-first order of each destination's
//                          free in-links (R3)
//                       PD per-destination matching: P lanes per destination,
//                          128-bit row loads, popc + segmented scan rank-select
//                          of the Philox-drawn candidate, claims in registers (R4)
//                       PE next event time = min busy_until (warp shuffles),
//                          in-order send records via a link-id bitmap prefix
//   best_keys_kernel  row a7: best-of-S key (T << 20 | seed) (§VI.C)
//   emit_ag_kernel    row a8: winner's AG sends (optionally shifted by T_RS)
//   rs_* / radix_*    row a8: inversion into the RS (§VII.A), ordered by
//                     (t_start, link) with an LSD radix sort
//
// Nothing here is shared with the CPU oracle (oracle/): separate sources,
// separate Philox implementation.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "tacos_internal.h"

namespace tacos {

static thread_local char g_cuda_err[256];
const char *cuda_error_string() { return g_cuda_err; }

static int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", what, cudaGetErrorString(e));
    return -4;  // TACOS_E_CUDA
  }
  return 0;
}

// ---------------------------------------------------------------------------
// Philox4x32-10 (R2; Salmon et al. SC'11).  Counter (t_lo, t_hi, link, sigma),
// key (seed_lo, seed_hi); word 0 = order key, word 1 = pick draw.
// ---------------------------------------------------------------------------
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

// r-th (0-based) set bit of x (x has more than r set bits): popc bisection.
__device__ __forceinline__ uint32_t select_bit(uint32_t x, uint32_t r) {
  uint32_t pos = 0, c;
  c = __popc(x & 0xFFFFu); if (r >= c) { r -= c; x >>= 16; pos += 16; }
  c = __popc(x & 0xFFu);   if (r >= c) { r -= c; x >>= 8;  pos += 8; }
  c = __popc(x & 0xFu);    if (r >= c) { r -= c; x >>= 4;  pos += 4; }
  c = __popc(x & 0x3u);    if (r >= c) { r -= c; x >>= 2;  pos += 2; }
  c = x & 1u;              if (r >= c) { pos += 1; }
  return pos;
}

__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
  return __reduce_add_sync(0xFFFFFFFFu, v);
}
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}
__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long y = __shfl_xor_sync(0xFFFFFFFFu, v, o);
    v = y < v ? y : v;
  }
  return v;
}

__device__ __forceinline__ uint32_t u4_get(const uint4 &v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}
__device__ __forceinline__ void u4_or(uint4 &v, int i, uint32_t m) {
  if (i == 0) v.x |= m; else if (i == 1) v.y |= m; else if (i == 2) v.z |= m; else v.w |= m;
}
__device__ __forceinline__ uint4 andnot4(uint4 a, uint4 b) {
  return make_uint4(a.x & ~b.x, a.y & ~b.y, a.z & ~b.z, a.w & ~b.w);
}
__device__ __forceinline__ uint4 and4(uint4 a, uint4 b) {
  return make_uint4(a.x & b.x, a.y & b.y, a.z & b.z, a.w & b.w);
}
__device__ __forceinline__ uint32_t popc4(uint4 a) {
  return __popc(a.x) + __popc(a.y) + __popc(a.z) + __popc(a.w);
}

// ---------------------------------------------------------------------------
// The greedy synthesis kernel.  One CTA = one job (seed, orientation sigma).
// P = lanes per destination row (row = 4*P*VPL words); ROWS_SMEM / LINKS_SMEM
// place the bitset rows / per-position link state in shared memory.
// ---------------------------------------------------------------------------
template <int P, int V, bool ROWS_SMEM, bool LINKS_SMEM>
__global__ void __launch_bounds__(V > 1 ? 512 : 1024, 1)
greedy_kernel(const Job *__restrict__ jobs, JobOut *__restrict__ outs, const Layout lay) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned long long s_min, s_delivered, s_V, s_D, s_M;
  __shared__ uint32_t s_rec_base, s_next_base;

  const Job job = jobs[blockIdx.x];
  const DevTopo T = *job.topo;
  const uint32_t N = T.N, L = T.L, Wp = T.Wp;
  const uint32_t tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31u;
  const uint32_t *__restrict__ p_src = T.p_src;
  const uint32_t *__restrict__ p_dst = T.p_dst;
  const uint32_t *__restrict__ p_w = T.p_w;
  const uint32_t *__restrict__ p_lid = T.p_lid;
  const uint32_t *__restrict__ in_ptr = T.in_ptr;

  unsigned char *rows_base = ROWS_SMEM ? smem : reinterpret_cast<unsigned char *>(job.g_rows);
  unsigned char *links_base = LINKS_SMEM ? (smem + (ROWS_SMEM ? lay.rows_bytes : 0u)) : job.g_links;
  uint32_t *held = reinterpret_cast<uint32_t *>(rows_base);
  uint32_t *have = held + (size_t)N * Wp;  // held | pending | claimed (R4)
  unsigned long long *busy = reinterpret_cast<unsigned long long *>(links_base + lay.off_busy);
  uint32_t *cur = reinterpret_cast<uint32_t *>(links_base + lay.off_cur);
  uint32_t *ord = reinterpret_cast<uint32_t *>(links_base + lay.off_ord);
  uint32_t *pick = reinterpret_cast<uint32_t *>(links_base + lay.off_pick);
  uint32_t *seen = reinterpret_cast<uint32_t *>(links_base + lay.off_seen);
  uint32_t *order = reinterpret_cast<uint32_t *>(links_base + lay.off_order);
  unsigned char *lv = links_base + lay.off_lv;
  uint32_t *hver = reinterpret_cast<uint32_t *>(smem + lay.off_hver);
  uint32_t *nlive = reinterpret_cast<uint32_t *>(smem + lay.off_nlive);
  uint32_t *bitmap = reinterpret_cast<uint32_t *>(smem + lay.off_bitmap);
  uint32_t *wpre = reinterpret_cast<uint32_t *>(smem + lay.off_wpre);
  const uint32_t nbw = (L + 31u) / 32u;
  const uint32_t seed_lo = (uint32_t)job.seed, seed_hi = (uint32_t)(job.seed >> 32);
  Rec *rec = job.rec;

  // ---- a2: state init (P:L89 precondition; P:L212 start at t = 0) ----
  const uint32_t NW = N * Wp;
  for (uint32_t i = tid; i < NW; i += nthr) {
    uint32_t v;
    if (T.custom) {
      v = T.pre[i];
    } else {  // AG: chunks x*k .. x*k+k-1 (R12)
      const uint32_t x = i / Wp, q = i - x * Wp;
      const uint32_t lo = x * T.k, hi = lo + T.k, wlo = q * 32u, whi = wlo + 32u;
      const uint32_t a = lo > wlo ? lo : wlo, b = hi < whi ? hi : whi;
      v = 0u;
      if (a < b) v = ((b - a) == 32u ? 0xFFFFFFFFu : ((1u << (b - a)) - 1u)) << (a - wlo);
    }
    held[i] = v;
    have[i] = v;
  }
  for (uint32_t p = tid; p < L; p += nthr) {
    busy[p] = 0ull;
    cur[p] = kNone;
    seen[p] = kNone;
    lv[p] = 0;
  }
  for (uint32_t x = tid; x < N; x += nthr) {
    hver[x] = 0u;
    nlive[x] = 0u;
  }
  for (uint32_t i = tid; i < nbw; i += nthr) bitmap[i] = 0u;
  if (tid == 0) {
    s_delivered = 0ull;
    s_V = s_D = s_M = 0ull;
    s_rec_base = 0u;
    s_next_base = 0u;
  }
  __syncthreads();

  unsigned long long t = 0ull, t_prev = 0ull;
  uint32_t e = 0u, E = 0u;
  int status = 0;
  unsigned long long myV = 0, myD = 0, myM = 0;

  for (;;) {
    // ---- PA: records of the previous event (in link-id order), arrivals at t ----
    {
      const uint32_t rec_base = s_rec_base;
      uint32_t arr = 0;
      for (uint32_t p = tid; p < L; p += nthr) {
        const uint32_t c = cur[p];
        if (c == kNone) continue;
        const unsigned long long b = busy[p];
        if (rec != nullptr && e > 0u && b - p_w[p] == t_prev) {
          const uint32_t lid = p_lid[p];
          const uint32_t wi = lid >> 5;
          const uint32_t idx = rec_base + wpre[wi] + __popc(bitmap[wi] & ((1u << (lid & 31u)) - 1u));
          Rec r;
          r.chunk = c;
          r.link = lid;
          r.t_start = t_prev;
          rec[idx] = r;
        }
        if (b == t) {  // R7: held by dst from this instant
          const uint32_t d = p_dst[p];
          atomicOr(&held[(size_t)d * Wp + (c >> 5)], 1u << (c & 31u));
          hver[d] = e;
          cur[p] = kNone;
          ++arr;
        }
      }
      arr = warp_sum_u32(arr);
      if (lane == 0 && arr) atomicAdd(&s_delivered, (unsigned long long)arr);
    }
    __syncthreads();
    if (s_delivered == T.required) break;  // done test (postcondition holds)

    // ---- PB: free / live links, Philox draws ----
    if (tid == 0) {
      s_rec_base = s_next_base;
      s_min = ~0ull;
    }
    for (uint32_t i = tid; i < nbw; i += nthr) bitmap[i] = 0u;
    {
      uint32_t nfree = 0;
      for (uint32_t p = tid; p < L; p += nthr) {
        unsigned char f = 0;
        if (busy[p] <= t) {  // free: nothing in flight on it
          ++nfree;
          f = 1;
          if (seen[p] != hver[p_src[p]]) {  // else K = 0 for sure: src unchanged since its last empty visit
            const uint4 r = philox4x32_10(make_uint4((uint32_t)t, (uint32_t)(t >> 32), p_lid[p], job.sigma),
                                          seed_lo, seed_hi);
            ord[p] = r.x;
            pick[p] = r.y;
            f = 2;
          }
        }
        lv[p] = f;
      }
      myV += nfree;
    }
    ++E;
    __syncthreads();

    // ---- PC: shorter-link-first order of live in-links per destination (R3) ----
    for (uint32_t p = tid; p < L; p += nthr) {
      const unsigned char f = lv[p];
      if (!f) continue;
      const uint32_t d = p_dst[p];
      const uint32_t b0 = in_ptr[d], b1 = in_ptr[d + 1];
      bool first = true;
      for (uint32_t q = b0; q < p; ++q)
        if (lv[q]) { first = false; break; }
      if (first) ++myD;
      if (f == 2) {
        const uint32_t wp = p_w[p], op = ord[p];
        uint32_t rank = 0, nl = 0;
        for (uint32_t q = b0; q < b1; ++q) {
          if (lv[q] != 2) continue;
          ++nl;
          const uint32_t wq = p_w[q], oq = ord[q];
          // positions of a destination are in ascending link id: q < p <=> lid_q < lid_p
          rank += (wq < wp) || (wq == wp && (oq < op || (oq == op && q < p)));
        }
        order[b0 + rank] = p;
        if (rank == nl - 1u) nlive[d] = nl;
      }
    }
    __syncthreads();

    // ---- PD: matching (R1, R4, R13) ----
    {
      const uint32_t gl = lane & (P - 1);
      const uint32_t gmask = (P == 32) ? 0xFFFFFFFFu : (((1u << P) - 1u) << (lane & ~(uint32_t)(P - 1)));
      const uint32_t ngroups = nthr / P;
      for (uint32_t d = tid / P; d < N; d += ngroups) {
        const uint32_t nl = nlive[d];
        if (nl == 0u) continue;
        const uint32_t b0 = in_ptr[d];
        uint4 *have4 = reinterpret_cast<uint4 *>(have + (size_t)d * Wp);
        const uint4 *post4 = reinterpret_cast<const uint4 *>(T.post + (size_t)d * Wp);
        const bool custom = T.custom != 0u;
        uint4 hv[V];
#pragma unroll
        for (int v = 0; v < V; ++v) hv[v] = have4[v * P + gl];
        for (uint32_t s = 0; s < nl; ++s) {
          const uint32_t p = order[b0 + s];
          const uint32_t sp = p_src[p];
          const uint4 *held4 = reinterpret_cast<const uint4 *>(held + (size_t)sp * Wp);
          // Chunk order along the row is vector-major: vector v of lane gl holds
          // words (v*P + gl)*4 .. +3.  Count and scan per vector so the r-th
          // candidate is the r-th in ascending chunk id (R12).
          uint4 cv[V];
          uint32_t incl[V], tot[V];
          uint32_t K = 0;
#pragma unroll
          for (int v = 0; v < V; ++v) {
            cv[v] = andnot4(held4[v * P + gl], hv[v]);  // held[src] & ~have[d] (& post[d])
            if (custom) cv[v] = and4(cv[v], post4[v * P + gl]);
            incl[v] = popc4(cv[v]);
#pragma unroll
            for (int o = 1; o < P; o <<= 1) {
              const uint32_t y = __shfl_up_sync(gmask, incl[v], o, P);
              if (gl >= (uint32_t)o) incl[v] += y;
            }
            tot[v] = __shfl_sync(gmask, incl[v], P - 1, P);
            K += tot[v];
          }
          if (K == 0u) {
            if (gl == 0) seen[p] = hver[sp];
            continue;
          }
          const uint32_t r = __umulhi(pick[p], K);  // floor(u_pick * K / 2^32)
          bool mine = false;
          uint32_t chunk = 0;
          {
            uint32_t rv = r;  // rank within the vector that holds the r-th candidate
            bool placed = false;
#pragma unroll
            for (int v = 0; v < V; ++v) {
              if (!placed) {
                if (rv < tot[v]) {
                  placed = true;
                  const uint32_t kl = popc4(cv[v]);
                  const uint32_t excl = incl[v] - kl;
                  if (rv >= excl && rv < incl[v]) {
                    mine = true;
                    uint32_t rr = rv - excl;
                    bool found = false;
#pragma unroll
                    for (int cpt = 0; cpt < 4; ++cpt) {
                      if (!found) {
                        const uint32_t word = u4_get(cv[v], cpt);
                        const uint32_t pc = __popc(word);
                        if (rr < pc) {
                          const uint32_t bit = select_bit(word, rr);
                          chunk = ((uint32_t)(v * P + gl) * 4u + (uint32_t)cpt) * 32u + bit;
                          u4_or(hv[v], cpt, 1u << bit);  // claim: withheld from d's other in-links
                          found = true;
                        } else {
                          rr -= pc;
                        }
                      }
                    }
                  }
                } else {
                  rv -= tot[v];
                }
              }
            }
          }
          const uint32_t bal = __ballot_sync(gmask, mine);
          chunk = __shfl_sync(gmask, chunk, __ffs(bal) - 1);
          if (gl == 0) {
            cur[p] = chunk;
            busy[p] = t + p_w[p];
            ++myM;
            const uint32_t lid = p_lid[p];
            atomicOr(&bitmap[lid >> 5], 1u << (lid & 31u));
          }
        }
#pragma unroll
        for (int v = 0; v < V; ++v) have4[v * P + gl] = hv[v];
        if (gl == 0) nlive[d] = 0u;
      }
    }
    __syncthreads();

    // ---- PE: record offsets (bitmap prefix) and the next event time ----
    if (tid < 32) {
      uint32_t running = 0;
      for (uint32_t base = 0; base < nbw; base += 32u) {
        const uint32_t i = base + lane;
        const uint32_t v = i < nbw ? __popc(bitmap[i]) : 0u;
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
          if (lane >= (uint32_t)o) incl += y;
        }
        if (i < nbw) wpre[i] = running + incl - v;
        running += __shfl_sync(0xFFFFFFFFu, incl, 31);
      }
      if (lane == 0) s_next_base = s_rec_base + running;
    }
    {
      unsigned long long mn = ~0ull;
      for (uint32_t p = tid; p < L; p += nthr)
        if (cur[p] != kNone) {
          const unsigned long long b = busy[p];
          mn = b < mn ? b : mn;
        }
      mn = warp_min_u64(mn);
      if (lane == 0 && mn != ~0ull) atomicMin(&s_min, mn);
    }
    __syncthreads();
    const unsigned long long tn = s_min;
    if (tn == ~0ull) {  // nothing in flight and not done: stall (R17)
      status = -3;
      break;
    }
    if (tn >= kMaxTime) {
      status = -6;
      break;
    }
    t_prev = t;
    t = tn;
    ++e;
  }

  // ---- per-job counters ----
  myV = warp_sum_u64(myV);
  myD = warp_sum_u64(myD);
  myM = warp_sum_u64(myM);
  if (lane == 0) {
    if (myV) atomicAdd(&s_V, myV);
    if (myD) atomicAdd(&s_D, myD);
    if (myM) atomicAdd(&s_M, myM);
  }
  __syncthreads();
  if (tid == 0) {
    JobOut o;
    o.T = t;
    o.V = s_V;
    o.D = s_D;
    o.M = s_M;
    o.E = E;
    o.status = status;
    o.pad = 0;
    outs[job.out_slot] = o;
  }
}

// ---------------------------------------------------------------------------
Layout make_layout(uint32_t N, uint32_t L, uint32_t Wp, uint32_t P, uint32_t VPL, size_t smem_limit) {
  auto al = [](uint32_t x, uint32_t a) { return (x + a - 1u) / a * a; };
  Layout lay{};
  lay.rows_bytes = al(2u * N * Wp * 4u, 16u);
  uint32_t o = 0;
  lay.off_busy = o; o += al(L * 8u, 16u);
  lay.off_cur = o; o += al(L * 4u, 16u);
  lay.off_ord = o; o += al(L * 4u, 16u);
  lay.off_pick = o; o += al(L * 4u, 16u);
  lay.off_seen = o; o += al(L * 4u, 16u);
  lay.off_order = o; o += al(L * 4u, 16u);
  lay.off_lv = o; o += al(L, 16u);
  lay.links_bytes = o;
  const uint32_t nbw = (L + 31u) / 32u;
  const uint32_t small = al(N * 4u, 16u) * 2u + al(nbw * 4u, 16u) * 2u;
  const size_t lim = smem_limit;
  if ((size_t)lay.rows_bytes + lay.links_bytes + small <= lim) {
    lay.rows_in_smem = 1;
    lay.links_in_smem = 1;
  } else if ((size_t)lay.links_bytes + small <= lim) {
    lay.rows_in_smem = 0;
    lay.links_in_smem = 1;
  } else {
    lay.rows_in_smem = 0;
    lay.links_in_smem = 0;
  }
  uint32_t s = 0;
  if (lay.rows_in_smem) s += lay.rows_bytes;
  if (lay.links_in_smem) s += lay.links_bytes;
  lay.off_hver = s; s += al(N * 4u, 16u);
  lay.off_nlive = s; s += al(N * 4u, 16u);
  lay.off_bitmap = s; s += al(nbw * 4u, 16u);
  lay.off_wpre = s; s += al(nbw * 4u, 16u);
  lay.smem_bytes = s;
  uint32_t want = N * P > L ? N * P : L;
  uint32_t th = 128;
  const uint32_t th_max = VPL > 1 ? 512u : 1024u;  // matches the kernel's __launch_bounds__
  while (th < th_max && th < want / 2) th <<= 1;
  if (th < P) th = P;
  lay.threads = th;
  return lay;
}

template <int P, int V, bool R, bool K>
static int launch_one(const Layout &lay, const Job *d_jobs, uint32_t n_jobs, JobOut *d_outs, cudaStream_t st) {
  auto fn = greedy_kernel<P, V, R, K>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lay.smem_bytes);
  if (e != cudaSuccess) {
    snprintf(g_cuda_err, sizeof(g_cuda_err), "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return -4;
  }
  fn<<<n_jobs, lay.threads, lay.smem_bytes, st>>>(d_jobs, d_outs, lay);
  return check_launch("greedy_kernel");
}

template <int P, int V>
static int launch_p(const Layout &lay, const Job *d_jobs, uint32_t n_jobs, JobOut *d_outs, cudaStream_t st) {
  if (lay.rows_in_smem && lay.links_in_smem) return launch_one<P, V, true, true>(lay, d_jobs, n_jobs, d_outs, st);
  if (lay.links_in_smem) return launch_one<P, V, false, true>(lay, d_jobs, n_jobs, d_outs, st);
  return launch_one<P, V, false, false>(lay, d_jobs, n_jobs, d_outs, st);
}

int launch_greedy(const Layout &lay, uint32_t P, uint32_t VPL, const Job *d_jobs, uint32_t n_jobs, JobOut *d_outs,
                  void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (VPL == 1) {
    switch (P) {
      case 1: return launch_p<1, 1>(lay, d_jobs, n_jobs, d_outs, st);
      case 2: return launch_p<2, 1>(lay, d_jobs, n_jobs, d_outs, st);
      case 4: return launch_p<4, 1>(lay, d_jobs, n_jobs, d_outs, st);
      case 8: return launch_p<8, 1>(lay, d_jobs, n_jobs, d_outs, st);
      case 16: return launch_p<16, 1>(lay, d_jobs, n_jobs, d_outs, st);
      case 32: return launch_p<32, 1>(lay, d_jobs, n_jobs, d_outs, st);
      default: break;
    }
  } else if (P == 32 && VPL == 2) {
    return launch_p<32, 2>(lay, d_jobs, n_jobs, d_outs, st);
  } else if (P == 32 && VPL == 4) {
    return launch_p<32, 4>(lay, d_jobs, n_jobs, d_outs, st);
  }
  snprintf(g_cuda_err, sizeof(g_cuda_err), "unsupported row shape P=%u VPL=%u", P, VPL);
  return -1;
}

// ---------------------------------------------------------------------------
// a7: best-of-S keys and counters.  keys[0] over jobs [0, n_seeds), keys[1]
// over jobs [rs_base, rs_base + n_seeds) when has_rs (else = keys[0]).
// stats = {V, D, M, E, status(neg) as u64}.
// ---------------------------------------------------------------------------
__global__ void best_keys_kernel(const JobOut *__restrict__ outs, uint32_t n_seeds, uint32_t seed_offset,
                                 uint32_t rs_base, uint32_t has_rs, unsigned long long *keys,
                                 unsigned long long *stats, unsigned long long *times_ag,
                                 unsigned long long *times_rs) {
  __shared__ unsigned long long s_k0, s_k1, s_V, s_D, s_M, s_E;
  __shared__ int s_status;
  if (threadIdx.x == 0) {
    s_k0 = s_k1 = kNoKey;
    s_V = s_D = s_M = s_E = 0ull;
    s_status = 0;
  }
  __syncthreads();
  const uint32_t n_jobs = has_rs ? rs_base + n_seeds : n_seeds;
  unsigned long long k0 = kNoKey, k1 = kNoKey, V = 0, D = 0, M = 0, E = 0;
  int st = 0;
  for (uint32_t j = threadIdx.x; j < n_jobs; j += blockDim.x) {
    const JobOut o = outs[j];
    V += o.V;
    D += o.D;
    M += o.M;
    E += o.E;
    if (o.status != 0) st = o.status;
    const bool is_rs = has_rs && j >= rs_base;
    const uint32_t i = is_rs ? j - rs_base : j;
    const unsigned long long key =
        o.status == 0 ? ((o.T << kKeySeedBits) | (unsigned long long)(seed_offset + i)) : kNoKey;
    if (is_rs) {
      k1 = key < k1 ? key : k1;
      if (times_rs) times_rs[i] = o.T;
    } else {
      k0 = key < k0 ? key : k0;
      if (times_ag) times_ag[i] = o.T;
    }
  }
  atomicMin(&s_k0, k0);
  atomicMin(&s_k1, k1);
  atomicAdd(&s_V, V);
  atomicAdd(&s_D, D);
  atomicAdd(&s_M, M);
  atomicAdd(&s_E, E);
  if (st != 0) atomicMin(&s_status, st);
  __syncthreads();
  if (threadIdx.x == 0) {
    keys[0] = s_k0;
    keys[1] = has_rs ? s_k1 : s_k0;
    stats[0] = s_V;
    stats[1] = s_D;
    stats[2] = s_M;
    stats[3] = s_E;
    stats[4] = (unsigned long long)(long long)s_status;
  }
}

int launch_best_keys(const JobOut *d_outs, uint32_t n_seeds, uint32_t seed_offset, uint32_t rs_base,
                     uint32_t has_rs, uint64_t *d_keys, uint64_t *d_stats, uint64_t *d_times_ag,
                     uint64_t *d_times_rs, void *stream) {
  best_keys_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(
      d_outs, n_seeds, seed_offset, rs_base, has_rs, reinterpret_cast<unsigned long long *>(d_keys),
      reinterpret_cast<unsigned long long *>(d_stats), reinterpret_cast<unsigned long long *>(d_times_ag),
      reinterpret_cast<unsigned long long *>(d_times_rs));
  return check_launch("best_keys_kernel");
}

// ---------------------------------------------------------------------------
// a8: emission.  Output record = tacos_send {chunk, src, dst, link, t0, t1}.
// ---------------------------------------------------------------------------
struct Send32 {
  uint32_t chunk, src, dst, link;
  unsigned long long t0, t1;
};

__global__ void emit_ag_kernel(const Rec *__restrict__ rec, uint64_t M, const uint32_t *__restrict__ src,
                               const uint32_t *__restrict__ dst, const uint32_t *__restrict__ w, uint64_t shift,
                               Send32 *__restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < M; i += (uint64_t)gridDim.x * blockDim.x) {
    const Rec r = rec[i];
    Send32 s;
    s.chunk = r.chunk;
    s.link = r.link;
    s.src = src[r.link];
    s.dst = dst[r.link];
    s.t0 = r.t_start + shift;
    s.t1 = r.t_start + w[r.link] + shift;
    out[i] = s;
  }
}

static int grid_for(uint64_t n, int threads) {
  uint64_t g = (n + threads - 1) / threads;
  if (g > 148ull * 16ull) g = 148ull * 16ull;
  if (g == 0) g = 1;
  return (int)g;
}

int launch_emit_ag(const Rec *rec, uint64_t M, const uint32_t *src, const uint32_t *dst, const uint32_t *w,
                   uint64_t shift, void *out_sends, void *stream) {
  emit_ag_kernel<<<grid_for(M, 256), 256, 0, (cudaStream_t)stream>>>(rec, M, src, dst, w, shift,
                                                                      reinterpret_cast<Send32 *>(out_sends));
  return check_launch("emit_ag_kernel");
}

// RS = mirror of an AG: (c, a->b on l, t0, t1) -> (c, b->a on l', T-t1, T-t0)
// with l' = rev[l] when G is symmetric (AG searched on G), else l' = l (AG searched on G^T).
__global__ void rs_keys_kernel(const Rec *__restrict__ rec, uint64_t M, const uint32_t *__restrict__ w,
                               const int32_t *__restrict__ rev, uint64_t T_rs, uint32_t lbits,
                               unsigned long long *__restrict__ keys, uint32_t *__restrict__ vals) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < M; i += (uint64_t)gridDim.x * blockDim.x) {
    const Rec r = rec[i];
    const uint32_t l2 = rev ? (uint32_t)rev[r.link] : r.link;
    const unsigned long long t0 = T_rs - (r.t_start + w[r.link]);
    keys[i] = (t0 << lbits) | l2;
    vals[i] = (uint32_t)i;
  }
}

__global__ void rs_emit_kernel(const uint32_t *__restrict__ vals, const Rec *__restrict__ rec, uint64_t M,
                               const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                               const uint32_t *__restrict__ w, const int32_t *__restrict__ rev, uint64_t T_rs,
                               Send32 *__restrict__ out) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < M; j += (uint64_t)gridDim.x * blockDim.x) {
    const Rec r = rec[vals[j]];
    const uint32_t l2 = rev ? (uint32_t)rev[r.link] : r.link;
    Send32 s;
    s.chunk = r.chunk;
    s.link = l2;
    s.src = src[l2];
    s.dst = dst[l2];
    s.t0 = T_rs - (r.t_start + w[r.link]);
    s.t1 = T_rs - r.t_start;
    out[j] = s;
  }
}

// ---- LSD radix sort of (u64 key, u32 value), 8-bit digits, stable ----
constexpr int kRsThreads = 256;
constexpr int kRsItems = 16;
constexpr int kRsTile = kRsThreads * kRsItems;

__global__ void radix_hist_kernel(const unsigned long long *__restrict__ keys, uint64_t n, int shift,
                                  uint32_t *__restrict__ hist, uint32_t nblocks) {
  __shared__ uint32_t cnt[256];
  cnt[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kRsTile;
  for (int it = 0; it < kRsItems; ++it) {
    const uint64_t i = base + (uint64_t)it * kRsThreads + threadIdx.x;
    if (i < n) atomicAdd(&cnt[(keys[i] >> shift) & 255u], 1u);
  }
  __syncthreads();
  hist[(size_t)threadIdx.x * nblocks + blockIdx.x] = cnt[threadIdx.x];
}

// exclusive scan of hist[0..total) in place, one block of 1024 threads
__global__ void radix_scan_kernel(uint32_t *__restrict__ hist, uint32_t total) {
  __shared__ uint32_t s_part[1024];
  const uint32_t per = (total + 1023u) / 1024u;
  const uint32_t b = threadIdx.x * per, en = min(b + per, total);
  uint32_t sum = 0;
  for (uint32_t i = b; i < en; ++i) sum += hist[i];
  s_part[threadIdx.x] = sum;
  __syncthreads();
  for (uint32_t o = 1; o < 1024; o <<= 1) {
    uint32_t y = threadIdx.x >= o ? s_part[threadIdx.x - o] : 0u;
    __syncthreads();
    s_part[threadIdx.x] += y;
    __syncthreads();
  }
  uint32_t run = s_part[threadIdx.x] - sum;
  for (uint32_t i = b; i < en; ++i) {
    const uint32_t v = hist[i];
    hist[i] = run;
    run += v;
  }
}

__global__ void radix_scatter_kernel(const unsigned long long *__restrict__ keys_in,
                                     const uint32_t *__restrict__ vals_in, uint64_t n, int shift,
                                     const uint32_t *__restrict__ offs, uint32_t nblocks,
                                     unsigned long long *__restrict__ keys_out, uint32_t *__restrict__ vals_out) {
  constexpr int kWarps = kRsThreads / 32;
  __shared__ uint32_t s_off[256];
  __shared__ uint32_t s_wc[kWarps][256];
  __shared__ uint32_t s_tot[256];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  s_off[tid] = offs[(size_t)tid * nblocks + blockIdx.x];
  const uint64_t base = (uint64_t)blockIdx.x * kRsTile;
  for (int it = 0; it < kRsItems; ++it) {
    const uint64_t i = base + (uint64_t)it * kRsThreads + tid;
    const bool valid = i < n;
    const unsigned long long k = valid ? keys_in[i] : 0ull;
    const uint32_t d = valid ? (uint32_t)((k >> shift) & 255u) : 256u;
#pragma unroll
    for (int wv = 0; wv < kWarps; ++wv) s_wc[wv][tid] = 0u;
    __syncthreads();
    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
    const uint32_t rank_w = __popc(peers & ((1u << lane) - 1u));
    if (valid && (uint32_t)(__ffs(peers) - 1) == lane) s_wc[warp][d] = __popc(peers);
    __syncthreads();
    {
      uint32_t run = 0;
#pragma unroll
      for (int wv = 0; wv < kWarps; ++wv) {
        const uint32_t c = s_wc[wv][tid];
        s_wc[wv][tid] = run;
        run += c;
      }
      s_tot[tid] = run;
    }
    __syncthreads();
    if (valid) {
      const uint32_t pos = s_off[d] + s_wc[warp][d] + rank_w;
      keys_out[pos] = k;
      vals_out[pos] = vals_in[i];
    }
    __syncthreads();
    s_off[tid] += s_tot[tid];
    __syncthreads();
  }
}

size_t rs_sort_scratch_bytes(uint64_t M) {
  const uint64_t nb = (M + kRsTile - 1) / kRsTile;
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  return al(M * 8) * 2 + al(M * 4) * 2 + al(nb * 256 * 4 + 4);
}

int launch_rs_sort_emit(const Rec *rec, uint64_t M, const uint32_t *src, const uint32_t *dst, const uint32_t *w,
                        const int32_t *rev, uint64_t T_rs, uint32_t L, void *out_sends, void *scratch,
                        size_t scratch_bytes, uint32_t *launches, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (M == 0) return 0;
  if (scratch_bytes < rs_sort_scratch_bytes(M)) {
    snprintf(g_cuda_err, sizeof(g_cuda_err), "rs sort scratch too small");
    return -9;
  }
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  unsigned char *p = reinterpret_cast<unsigned char *>(scratch);
  unsigned long long *ka = reinterpret_cast<unsigned long long *>(p); p += al(M * 8);
  unsigned long long *kb = reinterpret_cast<unsigned long long *>(p); p += al(M * 8);
  uint32_t *va = reinterpret_cast<uint32_t *>(p); p += al(M * 4);
  uint32_t *vb = reinterpret_cast<uint32_t *>(p); p += al(M * 4);
  uint32_t *hist = reinterpret_cast<uint32_t *>(p);
  uint32_t lbits = 1;
  while ((1ull << lbits) < (unsigned long long)L) ++lbits;
  uint32_t tbits = 1;
  while ((1ull << tbits) <= T_rs) ++tbits;
  const uint32_t bits = lbits + tbits;
  if (bits > 64) {
    snprintf(g_cuda_err, sizeof(g_cuda_err), "rs key does not fit 64 bits");
    return -6;
  }
  uint32_t nl = 0;
  rs_keys_kernel<<<grid_for(M, 256), 256, 0, st>>>(rec, M, w, rev, T_rs, lbits, ka, va);
  ++nl;
  int rc = check_launch("rs_keys_kernel");
  if (rc) return rc;
  const uint32_t nb = (uint32_t)((M + kRsTile - 1) / kRsTile);
  for (uint32_t shift = 0; shift < bits; shift += 8) {
    radix_hist_kernel<<<nb, kRsThreads, 0, st>>>(ka, M, (int)shift, hist, nb);
    radix_scan_kernel<<<1, 1024, 0, st>>>(hist, nb * 256u);
    radix_scatter_kernel<<<nb, kRsThreads, 0, st>>>(ka, va, M, (int)shift, hist, nb, kb, vb);
    nl += 3;
    rc = check_launch("radix pass");
    if (rc) return rc;
    unsigned long long *tk = ka; ka = kb; kb = tk;
    uint32_t *tv = va; va = vb; vb = tv;
  }
  rs_emit_kernel<<<grid_for(M, 256), 256, 0, st>>>(va, rec, M, src, dst, w, rev, T_rs,
                                                   reinterpret_cast<Send32 *>(out_sends));
  ++nl;
  if (launches) *launches += nl;
  return check_launch("rs_emit_kernel");
}

// ---------------------------------------------------------------------------
__global__ void philox_probe_kernel(const uint32_t *in, uint32_t *out) {
  const uint4 r = philox4x32_10(make_uint4(in[0], in[1], in[2], in[3]), in[4], in[5]);
  out[0] = r.x;
  out[1] = r.y;
  out[2] = r.z;
  out[3] = r.w;
}

int launch_philox_probe(const uint32_t *d_in, uint32_t *d_out, void *stream) {
  philox_probe_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(d_in, d_out);
  return check_launch("philox_probe_kernel");
}

}  // namespace tacos
