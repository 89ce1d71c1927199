// literal_kernel.cu -- the paper-literal TACOS-Greedy variant (SURVEY §8 row f1,
// DESIGN.md reading R21) on sm_100a: chunk-first matching with chunk
// replacement.
//
//   chunk-first:  "first we choose a requested chunk and backtrack the NPU ...
//                 among candidate links, we can randomly select one"
//   shorter-link-first among the candidate links
//   arrival time: a chunk is forwarded only after it arrived
//   replacement:  "chunk 2 arrived NPU 2 already at t=1 ... this transmission is
//                 outdated ... TACOS-Greedy tries to replace this with another
//                 matching"
//
// One CTA per job (seed, sigma); one warp per destination.  Per event:
//   PA (thread per destination)  arrivals in ascending link id: a copy of a chunk
//                                 the destination already holds is dropped; the
//                                 others are delivered and recorded (records are
//                                 written at delivery, so cancelled sends never
//                                 appear; emission sorts them by (t_start, link))
//   -- barrier --                 done test (outstanding copies are outdated)
//   PM (warp per destination)     replacement of outdated in-flight copies; the
//                                 requested set R = post & ~held in the warp's
//                                 registers (lanes x 128-bit vectors); a Philox
//                                 rotation picks the first chunk; chunks are then
//                                 taken in cyclic order among those some free
//                                 unmatched in-link can provide (warp min-reduce
//                                 of the rotated distance); the in-link lanes test
//                                 the chunk bit of their source row, keep the
//                                 shortest cost, and a Philox draw picks among ties
//   -- barrier --
//   PE                            next event time (min busy_until)
//   -- barrier --
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "tacos_device.cuh"
#include "tacos_internal.h"

namespace tacos {

template <int V, bool ROWS_SMEM>
__global__ void __launch_bounds__(512, 1)
literal_kernel(const Job *__restrict__ jobs, JobOut *__restrict__ outs, const Layout lay) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned long long s_min, s_delivered, s_V, s_D, s_M, s_X;
  __shared__ uint32_t s_nrec;
  // per-event values with 32-bit shared atomics (64-bit ones are CAS loops on sm_100a)
  __shared__ uint32_t s_arr, s_min32;

  const Job job = jobs[blockIdx.x];
  const DevTopo T = *job.topo;
  const uint32_t N = T.N, Wp = T.Wp, C = T.C;
  const uint32_t Wr = ROWS_SMEM ? lay.row_stride : Wp;
  const uint32_t tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31u, warp = tid >> 5, nwarps = nthr >> 5;
  const uint32_t *__restrict__ in_ptr = T.in_ptr;
  const uint32_t *__restrict__ p_src = T.p_src;
  const uint32_t *__restrict__ p_w = T.p_w;
  const uint32_t *__restrict__ p_lid = T.p_lid;
  const bool custom = T.custom != 0u;
  uint32_t *held;
  if constexpr (ROWS_SMEM) held = reinterpret_cast<uint32_t *>(smem);
  else held = job.g_rows;
  unsigned char *links_base = smem + (ROWS_SMEM ? lay.rows_bytes : 0u);  // link state in shared memory
  unsigned long long *busy = reinterpret_cast<unsigned long long *>(links_base + lay.off_busy);
  uint32_t *cur = reinterpret_cast<uint32_t *>(links_base + lay.off_cur);
  const uint32_t seed_lo = (uint32_t)job.seed, seed_hi = (uint32_t)(job.seed >> 32);
  const uint32_t L = T.L;

  // ---- state init ----
  for (uint32_t i = tid; i < N * Wp; i += nthr) {
    const uint32_t x = i / Wp, q = i - x * Wp;
    uint32_t v;
    if (custom) {
      v = __ldg(&T.pre[i]);
    } else {
      const uint32_t lo = x * T.k, hi = lo + T.k, wlo = q * 32u, whi = wlo + 32u;
      const uint32_t a = lo > wlo ? lo : wlo, b = hi < whi ? hi : whi;
      v = 0u;
      if (a < b) v = ((b - a) == 32u ? 0xFFFFFFFFu : ((1u << (b - a)) - 1u)) << (a - wlo);
    }
    held[(size_t)x * Wr + q] = v;
  }
  for (uint32_t p = tid; p < L; p += nthr) {
    busy[p] = 0ull;
    cur[p] = kNone;
  }
  if (tid == 0) {
    s_delivered = 0ull;
    s_V = s_D = s_M = s_X = 0ull;
    s_nrec = 0u;
    s_min = ~0ull;
    s_arr = 0u;
    s_min32 = ~0u;
  }
  __syncthreads();

  unsigned long long t = 0ull;
  uint32_t E = 0;
  int status = 0;
  unsigned long long myV = 0, myD = 0, myM = 0, myX = 0;
  Rec *rec = job.rec;

  for (;;) {
    // ---- PA: arrivals (ascending link id per destination); duplicates dropped ----
    {
      uint32_t arr = 0;
      for (uint32_t d = tid; d < N; d += nthr) {
        const uint32_t b0 = __ldg(&in_ptr[d]), b1 = __ldg(&in_ptr[d + 1]);
        for (uint32_t p = b0; p < b1; ++p) {
          const uint32_t c = cur[p];
          if (c == kNone || busy[p] != t) continue;
          uint32_t &hw = held[(size_t)d * Wr + (c >> 5)];
          const uint32_t bit = 1u << (c & 31u);
          if (hw & bit) {
            ++myX;  // a copy arrived earlier (or at this instant on a lower link id)
          } else {
            hw |= bit;
            ++arr;
            if (rec != nullptr) {
              const uint32_t idx = atomicAdd(&s_nrec, 1u);
              Rec r;
              r.chunk = c;
              r.link = __ldg(&p_lid[p]);
              r.t_start = t - __ldg(&p_w[p]);
              TCHECK(idx < job.rec_cap && c < T.C, "literal record");
              rec[idx] = r;
            }
          }
          cur[p] = kNone;
        }
      }
      arr = warp_sum_u32(arr);
      if (lane == 0 && arr) atomicAdd(&s_arr, arr);
    }
    __syncthreads();
    if (s_delivered + s_arr == T.required) {  // done; copies still in flight are outdated
      for (uint32_t p = tid; p < L; p += nthr)
        if (cur[p] != kNone) ++myX;
      break;
    }
    ++E;
    if (tid == 0) s_min32 = ~0u;

    // ---- PM: one warp per destination ----
    for (uint32_t d = warp; d < N; d += nwarps) {
      const uint32_t b0 = __ldg(&in_ptr[d]), deg = __ldg(&in_ptr[d + 1]) - b0;
      const uint4 *h4 = reinterpret_cast<const uint4 *>(held + (size_t)d * Wr);
      const uint4 *post4 = reinterpret_cast<const uint4 *>(T.post + (size_t)d * Wp);
      // replacement of outdated copies, then the free in-links (lane j <-> in-link j; deg <= 32 per pass)
      uint32_t freemask = 0;  // bit j: in-link j free (same value on every lane)
      uint32_t nfree = 0;
      for (uint32_t base = 0; base < deg; base += 32u) {
        const uint32_t j = base + lane;
        bool f = false;
        if (j < deg) {
          const uint32_t p = b0 + j;
          const uint32_t c = cur[p];
          if (c != kNone && ((held[(size_t)d * Wr + (c >> 5)] >> (c & 31u)) & 1u)) {
            cur[p] = kNone;  // outdated: cancelled, the link is free now
            busy[p] = t;
            ++myX;
          }
          f = cur[p] == kNone;
        }
        const uint32_t b = __ballot_sync(0xFFFFFFFFu, f);
        nfree += __popc(b);
        if (base == 0) freemask = b;
      }
      if (lane == 0) {
        myV += nfree;
        myD += nfree ? 1u : 0u;
      }
      if (nfree == 0) continue;
      // requested set R = post & ~held (vector v of this lane = words (v*32 + lane)*4 .. +3)
      uint4 R[V];
      uint32_t cntR = 0;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const uint4 h = h4[v * 32 + lane];
        const uint4 pz = custom ? __ldg(&post4[v * 32 + lane]) : make_uint4(~0u, ~0u, ~0u, ~0u);
        R[v] = and4(andnot4(pz, h), pz);
        // chunks beyond C never requested (held rows carry no such bits; AG post is all-ones)
        const uint32_t w0 = (uint32_t)(v * 32 + lane) * 4u;
        uint32_t *rw = reinterpret_cast<uint32_t *>(&R[v]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t lo = (w0 + q) * 32u;
          if (lo >= C) rw[q] = 0u;
          else if (C - lo < 32u) rw[q] &= (1u << (C - lo)) - 1u;
        }
        cntR += popc4(R[v]);
      }
      const uint32_t nR = __reduce_add_sync(0xFFFFFFFFu, cntR);
      if (nR == 0u) continue;
      // rotation: start at the r0-th smallest member of R (vector-major order)
      const uint4 u0 = philox4x32_10(make_uint4((uint32_t)t, (uint32_t)(t >> 32), d, 0x80000000u | (job.sigma << 16)),
                                     seed_lo, seed_hi);
      uint32_t rr = __umulhi(u0.x, nR);
      uint32_t start = 0;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const uint32_t cv = popc4(R[v]);
        uint32_t incl = cv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
          if (lane >= (uint32_t)o) incl += y;
        }
        const uint32_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
        const bool here = rr < tot;
        if (here) {
          const uint32_t ex = incl - cv;
          uint32_t cand = 0xFFFFFFFFu;
          if (rr >= ex && rr < incl) {
            uint32_t k = rr - ex;
            const uint32_t *rw = reinterpret_cast<const uint32_t *>(&R[v]);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint32_t pc = __popc(rw[q]);
              if (cand == 0xFFFFFFFFu) {
                if (k < pc) cand = ((uint32_t)(v * 32 + lane) * 4u + q) * 32u + select_bit(rw[q], k);
                else k -= pc;
              }
            }
          }
          start = __reduce_min_sync(0xFFFFFFFFu, cand);
          rr = 0xFFFFFFFFu;  // found: later vectors skip
        } else {
          rr -= tot;
        }
      }
      // cyclic walk over the chunks some free unmatched in-link can provide
      uint32_t unmatched = freemask;  // in-links 0..31 (deg > 32: only the first 32 are matched)
      uint32_t dmin = 0;              // next rotated distance to consider
      uint32_t m = 0;
      while (unmatched != 0u && dmin < C) {
        // U = R & (union of the unmatched sources' rows); best = min rotated distance >= dmin
        uint32_t best = 0xFFFFFFFFu;
        const uint32_t A = start + dmin;  // chunks c >= A (if A < C) have distance c - start
        const uint32_t B = A > C ? A - C : 0u;  // chunks in [B, start) have distance c - start + C
#pragma unroll
        for (int v = 0; v < V; ++v) {
          uint4 U = make_uint4(0u, 0u, 0u, 0u);
          for (uint32_t mm = unmatched; mm; mm &= mm - 1u) {
            const uint32_t j = __ffs(mm) - 1u;
            const uint32_t sp = __ldg(&p_src[b0 + j]);
            const uint4 x = ROWS_SMEM ? reinterpret_cast<const uint4 *>(held + (size_t)sp * Wr)[v * 32 + lane]
                                      : __ldcg(&reinterpret_cast<const uint4 *>(held + (size_t)sp * Wr)[v * 32 + lane]);
            U.x |= x.x; U.y |= x.y; U.z |= x.z; U.w |= x.w;
          }
          U = and4(U, R[v]);
          const uint32_t *uw = reinterpret_cast<const uint32_t *>(&U);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t lo = ((uint32_t)(v * 32 + lane) * 4u + q) * 32u;
            uint32_t bits = uw[q];
            if (!bits) continue;
            // region 1: c >= A
            if (A < C) {
              uint32_t m1 = bits;
              if (A > lo) m1 = (A - lo >= 32u) ? 0u : (m1 & (~0u << (A - lo)));
              if (m1) {
                const uint32_t c = lo + __ffs(m1) - 1u;
                best = min(best, c - start);
              }
            }
            // region 2: B <= c < start (wrapped)
            uint32_t m2 = bits;
            if (B > lo) m2 = (B - lo >= 32u) ? 0u : (m2 & (~0u << (B - lo)));
            if (start < lo + 32u) m2 = (start <= lo) ? 0u : (m2 & ((1u << (start - lo)) - 1u));
            if (m2) {
              const uint32_t c = lo + __ffs(m2) - 1u;
              best = min(best, c + C - start);
            }
          }
        }
        best = __reduce_min_sync(0xFFFFFFFFu, best);
        if (best == 0xFFFFFFFFu) break;
        const uint32_t c = (start + best) % C;
        dmin = best + 1u;
        // candidate in-links: unmatched, source holds c; shortest cost first
        bool cand = false;
        uint32_t wj = 0xFFFFFFFFu;
        if (lane < deg && ((unmatched >> lane) & 1u)) {
          const uint32_t p = b0 + lane;
          const uint32_t sp = __ldg(&p_src[p]);
          const uint32_t word = ROWS_SMEM ? held[(size_t)sp * Wr + (c >> 5)] : __ldcg(&held[(size_t)sp * Wr + (c >> 5)]);
          cand = (word >> (c & 31u)) & 1u;
          if (cand) wj = __ldg(&p_w[p]);
        }
        const uint32_t wmin = __reduce_min_sync(0xFFFFFFFFu, wj);
        const uint32_t ties = __ballot_sync(0xFFFFFFFFu, cand && wj == wmin);
        if (ties == 0u) continue;  // cannot happen: c is in U
        ++m;
        const uint4 um = philox4x32_10(
            make_uint4((uint32_t)t, (uint32_t)(t >> 32), d, 0x80000000u | (job.sigma << 16) | m), seed_lo, seed_hi);
        uint32_t k = __umulhi(um.x, (uint32_t)__popc(ties));
        uint32_t tm = ties;
        while (k--) tm &= tm - 1u;
        const uint32_t j = __ffs(tm) - 1u;  // k-th tied in-link, ascending link id
        if (lane == j) {
          const uint32_t p = b0 + j;
          cur[p] = c;
          busy[p] = t + __ldg(&p_w[p]);
          ++myM;
        }
        unmatched &= ~(1u << j);
      }
      __syncwarp();
    }
    __syncthreads();
    if (tid == 0) {  // every thread has read this event's arrivals
      s_delivered += s_arr;
      s_arr = 0u;
    }

    // ---- PE: next event time (offset from t: in-flight copies end within w < 2^32) ----
    {
      unsigned long long mn = ~0ull;
      for (uint32_t p = tid; p < L; p += nthr)
        if (cur[p] != kNone) mn = busy[p] < mn ? busy[p] : mn;
      mn = warp_min_u64(mn);
      if (lane == 0 && mn != ~0ull) atomicMin(&s_min32, (uint32_t)(mn - t));
    }
    __syncthreads();
    const unsigned long long tn = s_min32 == ~0u ? ~0ull : t + s_min32;
    if (tn == ~0ull) {
      status = -3;
      break;
    }
    if (tn >= kMaxTime) {
      status = -6;
      break;
    }
    t = tn;
    __syncthreads();
  }
  myV = warp_sum_u64(myV);
  myD = warp_sum_u64(myD);
  myM = warp_sum_u64(myM);
  myX = warp_sum_u64(myX);
  if (lane == 0) {
    if (myV) atomicAdd(&s_V, myV);
    if (myD) atomicAdd(&s_D, myD);
    if (myM) atomicAdd(&s_M, myM);
    if (myX) atomicAdd(&s_X, myX);
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
    o.pad = (uint32_t)s_X;  // cancelled sends (duplicates + replaced outdated copies)
    o.Lv = 0;
    outs[job.out_slot] = o;
  }
}

template <int V, bool R>
static int launch_literal_one(const Layout &lay, const Job *d_jobs, uint32_t n_jobs, JobOut *d_outs, cudaStream_t st) {
  auto fn = literal_kernel<V, R>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lay.smem_bytes);
  if (e != cudaSuccess) {
    snprintf(cuda_error_buffer(), 256, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return -4;
  }
  fn<<<n_jobs, 512, lay.smem_bytes, st>>>(d_jobs, d_outs, lay);
  return check_launch("literal_kernel");
}

int launch_literal(const Layout &lay, uint32_t VPL, const Job *d_jobs, uint32_t n_jobs, JobOut *d_outs, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!lay.links_in_smem) {
    snprintf(cuda_error_buffer(), 256, "literal variant needs the link state in shared memory");
    return -6;
  }
  switch (VPL) {
    case 1: return lay.rows_in_smem ? launch_literal_one<1, true>(lay, d_jobs, n_jobs, d_outs, st)
                                    : launch_literal_one<1, false>(lay, d_jobs, n_jobs, d_outs, st);
    case 2: return lay.rows_in_smem ? launch_literal_one<2, true>(lay, d_jobs, n_jobs, d_outs, st)
                                    : launch_literal_one<2, false>(lay, d_jobs, n_jobs, d_outs, st);
    case 4: return lay.rows_in_smem ? launch_literal_one<4, true>(lay, d_jobs, n_jobs, d_outs, st)
                                    : launch_literal_one<4, false>(lay, d_jobs, n_jobs, d_outs, st);
    default:
      snprintf(cuda_error_buffer(), 256, "literal variant: unsupported vectors per lane %u", VPL);
      return -1;
  }
}

}  // namespace tacos
