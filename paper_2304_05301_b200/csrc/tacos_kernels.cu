// tacos_kernels.cu -- layout, launch dispatch and the small kernels of the
// TACOS-Greedy hot path (sm_100a).  The search kernel itself is in
// greedy_kernel.cuh (instantiated per lane count in greedy_p*.cu).
//
// PAPER.md citations "P:L<n>"; readings "R<n>" = DESIGN.md §3.
//
//   best_keys_kernel  row a7: best-of-S key (T << 20 | seed) (§VI.C)
//   emit_ag_kernel    row a8: winner's AG sends (optionally shifted by T_RS)
//   rs_* / radix_*    row a8: inversion into the RS (§VII.A), ordered by
//                     (t_start, link) with an LSD radix sort
//
// Nothing here is shared with the CPU oracle (oracle/): separate sources,
// separate Philox implementation.
#include <algorithm>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "greedy_kernel.cuh"
#include "tacos_device.cuh"
#include "tacos_internal.h"

namespace tacos {

static thread_local char g_cuda_err[256];
char *cuda_error_buffer() { return g_cuda_err; }
const char *cuda_error_string() { return g_cuda_err; }

int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", what, cudaGetErrorString(e));
    return -4;  // TACOS_E_CUDA
  }
  return 0;
}

// ---------------------------------------------------------------------------
// Shared-memory / scratch layout of one search job (see greedy_kernel.cuh).
// ---------------------------------------------------------------------------
thread_local int *g_occ_query = nullptr;

Layout make_layout(uint32_t N, uint32_t L, uint32_t Wp, uint32_t P, uint32_t VPL, size_t smem_limit, uint32_t n_jobs,
                   uint32_t n_sms, uint32_t q_force) {
  auto al = [](uint32_t x, uint32_t a) { return (x + a - 1u) / a * a; };
  Layout lay{};
  // pad the shared-memory row stride by one 16-byte vector when the row is an even
  // number of vectors: consecutive rows then start 4 banks apart
  lay.row_stride = ((Wp / 4u) % 2u == 0u) ? Wp + 4u : Wp;
  lay.rows_bytes = al(2u * N * lay.row_stride * 4u, 16u);
  uint32_t o = 0;
  lay.off_busy = o; o += al(L * 8u, 16u);
  lay.off_cur = o; o += al(L * 4u, 16u);
  lay.off_ord = o; o += al(L * 4u, 16u);
  lay.off_pick = o; o += al(L * 4u, 16u);
  lay.off_seen = o; o += al(L * 4u, 16u);
  lay.off_order = o; o += al(L * 2u, 16u);   // u16
  lay.off_rch = o; o += al(L * 4u, 16u);     // u16 x 2 parities
  lay.off_tsrc = o; o += al(L * 2u, 16u);    // u16 copies (shared-memory layout only)
  lay.off_tw = o; o += al(L * 4u, 16u);
  lay.off_tlid = o; o += al(L * 2u, 16u);
  lay.off_tdst = o; o += al(L * 2u, 16u);
  lay.off_lv = o; o += al(L, 16u);
  lay.links_bytes = o;
  const uint32_t nbw = (L + 31u) / 32u;
  const uint32_t act_words = (N + 31u) / 32u;
  const uint32_t small = al(N * 4u, 16u) + al(2u * nbw * 4u, 16u) + al(nbw * 4u, 16u) + al((N + 1u) * 4u, 16u) +
                         al(2u * act_words * 4u, 16u) + al(N * 4u, 16u) + al(N * 4u, 16u);
  const size_t lim = smem_limit;
  const bool ids16 = N < 65536u && L < 65536u;  // u16 NPU / link ids in the shared-memory link state
  if ((size_t)lay.rows_bytes + lay.links_bytes + small <= lim && ids16) {
    lay.rows_in_smem = 1;
    lay.links_in_smem = 1;
  } else if ((size_t)lay.links_bytes + small <= lim && ids16) {
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
  lay.off_bitmap = s; s += al(2u * nbw * 4u, 16u);
  lay.off_wpre = s; s += al(nbw * 4u, 16u);
  lay.off_inptr = s; s += al((N + 1u) * 4u, 16u);
  lay.off_act = s; s += al(2u * act_words * 4u, 16u);
  lay.off_list = s; s += al(N * 4u, 16u);
  lay.off_peers = s; s += al(N * 4u, 16u);
  lay.smem_bytes = s;
  // Cluster size: split each job over Q CTAs (SMs) while the grid still fits on
  // the chip and every CTA keeps >= 32 destinations.
  uint32_t Q = 1;
  // Q = 8 measured slower (barriers); >= 64 destinations per CTA (config 2: Q = 1 0.283 ms vs Q = 2 0.347 ms)
  while (Q < 4 && (uint64_t)n_jobs * Q * 2 <= n_sms && N / (Q * 2) >= 64) Q <<= 1;
  if (q_force) Q = q_force;
  if (const char *env = getenv("TACOS_CLUSTER")) {
    const uint32_t want = (uint32_t)atoi(env);
    if (want >= 1 && want <= kMaxCluster) Q = want;  // any cluster size (above 8: non-portable)
  }
  lay.cluster = Q;
  const uint32_t n_own = (N + Q - 1) / Q;
  // threads: one destination group per own destination in one pass when possible, plus
  // the warps that write the previous event's records meanwhile (about one thread per 16
  // own in-links; measured on configs 2, 3, 5)
  uint32_t th_max = VPL == 1 ? 768u : (P == 2 && VPL == 2) ? 640u
                    : VPL == 2 ? (uint32_t)TACOS_V2_THREADS
                    : P > 2u  ? (uint32_t)TACOS_WIDE_THREADS : (uint32_t)TACOS_V4_THREADS;  // = ThreadsFor<P, V>
  const uint32_t walkers = (n_own * P + 31u) & ~31u;
  const uint32_t recw = std::max<uint32_t>(64u, ((L / Q) / 16u + 31u) & ~31u);
  // one lane, four vectors, more own destinations than the default bound leaves walkers for: the
  // larger-bound instantiation (register path with on-chip state only; the host clears `big` for
  // the other paths, launch_greedy_pv), one destination per walker
  lay.big = 0u;
  if (P == 1u && VPL == 4u && walkers + 32u > th_max && !getenv("TACOS_NO_BIG")) {
    lay.big = 1u;
    th_max = (uint32_t)kBigThreads;
  }
  uint32_t th = std::max<uint32_t>(128u, walkers + recw);
  if (th > th_max) th = th_max;
  if (th < P) th = P;
  if (const char *env = getenv("TACOS_THREADS")) {  // tuning override (multiple of 32, <= the kernel bound)
    const uint32_t want = (uint32_t)atoi(env);
    if (want >= 64 && want <= th_max && want % 32 == 0 && want >= P) th = want;
  }
  lay.threads = th;
  lay.pre_draw = 0u;  // 1: draws made ahead in the previous event's record-offset phase (measured slower)
  if (const char *env = getenv("TACOS_PRE_DRAW")) lay.pre_draw = (uint32_t)atoi(env);
  return lay;
}

void add_window(Layout &lay, uint32_t N, uint32_t window, uint32_t deg) {
  auto al = [](uint32_t x, uint32_t a) { return (x + a - 1u) / a * a; };
  lay.window = window;
  lay.win_deg = deg;
  lay.win_ev = kWinEv;
  if (const char *env = getenv("TACOS_WIN_EV")) {  // testing: shorter windows (cut at the n-th event)
    const int n = atoi(env);
    if (n >= 1 && n <= (int)kWinEv) lay.win_ev = (uint32_t)n;
  }
  if (!window) return;
  uint32_t s = lay.smem_bytes;
  lay.off_wbm = s; s += al((window + 31u) / 32u * 4u, 16u);
  lay.off_wev = s; s += kWinEv * 4u;
  lay.off_wevc = s; s += kWinEv * 4u;
  lay.off_wevo = s; s += kWinEv * 4u;
  lay.off_wacnt = s; s += al(N * 4u, 16u);
  lay.off_waoff = s; s += al(N * deg * 4u, 16u);
  lay.off_wachk = s; s += al(N * deg * 2u, 16u);
  lay.smem_bytes = s;
}

void layout_drop_big(Layout &lay) {
  lay.big = 0u;
  lay.threads = std::min<uint32_t>(lay.threads, (uint32_t)TACOS_V4_THREADS);
}

bool add_lockstep(Layout &lay, uint32_t N, uint32_t L, uint32_t pos_cap, size_t smem_limit) {
  auto al = [](uint32_t x, uint32_t a) { return (x + a - 1u) / a * a; };
  // everything in shared memory (u16 NPU / link ids): the compact layout may fit where the
  // full one put the rows in global memory
  if (N >= 65536u || L >= 65536u || lay.window || lay.pre_draw) return false;
  Layout l = lay;
  l.rows_in_smem = 1u;
  l.links_in_smem = 1u;
  const uint32_t Q = l.cluster, n_own = (N + Q - 1u) / Q, Lc = pos_cap;
  l.rows_bytes = al((2u * N + n_own) * l.row_stride * 4u, 16u);  // held[2][N], have[n_own]
  uint32_t o = 0;
  l.off_busy = o; o += al(Lc * 8u, 16u);
  l.off_cur = o; o += al(Lc * 4u, 16u);
  l.off_ord = o; o += al(Lc * 4u, 16u);
  l.off_pick = o; o += al(Lc * 4u, 16u);
  l.off_seen = o; o += al(Lc * 4u, 16u);
  l.off_order = o; o += al(Lc * 2u, 16u);
  l.off_rch = o; o += al(Lc * 4u, 16u);
  l.off_tsrc = o; o += al(Lc * 2u, 16u);
  l.off_tw = o; o += al(Lc * 4u, 16u);
  l.off_tlid = o; o += al(Lc * 2u, 16u);
  l.off_tdst = o; o += al(Lc * 2u, 16u);
  l.off_lv = o; o += al(Lc, 16u);
  l.links_bytes = o;
  // the small arrays keep their sizes (hver doubles); shift them behind the new regions
  const uint32_t old_base = lay.off_hver, new_base = l.rows_bytes + l.links_bytes;
  const uint32_t hv_old = al(N * 4u, 16u), hv_new = al(2u * N * 4u, 16u);
  auto mv = [&](uint32_t off) { return off - old_base - hv_old + new_base + hv_new; };
  l.off_hver = new_base;
  l.off_bitmap = mv(lay.off_bitmap);
  l.off_wpre = mv(lay.off_wpre);
  l.off_inptr = mv(lay.off_inptr);
  l.off_act = mv(lay.off_act);
  l.off_list = mv(lay.off_list);
  l.off_peers = mv(lay.off_peers);
  l.smem_bytes = mv(lay.smem_bytes);
  if ((size_t)l.smem_bytes > smem_limit) return false;
  l.lockstep = 1u;
  l.pos_cap = pos_cap;
  lay = l;
  return true;
}

int launch_greedy(const Layout &lay, uint32_t P, uint32_t VPL, const Job *d_jobs, uint32_t n_jobs, JobOut *d_outs,
                  void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  switch (P) {
    case 1: return launch_greedy_p1(lay, VPL, d_jobs, n_jobs, d_outs, st);
    case 2: return launch_greedy_p2(lay, VPL, d_jobs, n_jobs, d_outs, st);
    case 4: return launch_greedy_p4(lay, VPL, d_jobs, n_jobs, d_outs, st);
    case 8: return launch_greedy_p8(lay, VPL, d_jobs, n_jobs, d_outs, st);
    case 16: return launch_greedy_p16(lay, VPL, d_jobs, n_jobs, d_outs, st);
    case 32: return launch_greedy_p32(lay, VPL, d_jobs, n_jobs, d_outs, st);
    default:
      snprintf(g_cuda_err, sizeof(g_cuda_err), "bad lanes-per-row %u", P);
      return -1;
  }
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
  // per-thread partials -> warp shuffles -> one slot per warp -> warp 0 (64-bit shared
  // atomics would be CAS loops on sm_100a)
  constexpr int kVals = 8;  // k0, k1 (min); V, D, M, E, X, Lv (sum)
  __shared__ unsigned long long s_w[32][kVals];
  __shared__ int s_st[32];
  const uint32_t n_jobs = has_rs ? rs_base + n_seeds : n_seeds;
  unsigned long long v[kVals] = {kNoKey, kNoKey, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
  int st = 0;
  for (uint32_t j = threadIdx.x; j < n_jobs; j += blockDim.x) {
    const JobOut o = outs[j];
    v[2] += o.V;
    v[3] += o.D;
    v[4] += o.M;
    v[5] += o.E;
    v[6] += o.pad;
    v[7] += o.Lv;
    if (o.status != 0) st = min(st, o.status);
    const bool is_rs = has_rs && j >= rs_base;
    const uint32_t i = is_rs ? j - rs_base : j;
    const unsigned long long key =
        o.status == 0 ? ((o.T << kKeySeedBits) | (unsigned long long)(seed_offset + i)) : kNoKey;
    if (is_rs) {
      v[1] = key < v[1] ? key : v[1];
      if (times_rs) times_rs[i] = o.T;
    } else {
      v[0] = key < v[0] ? key : v[0];
      if (times_ag) times_ag[i] = o.T;
    }
  }
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5, nw = (blockDim.x + 31u) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int q = 0; q < kVals; ++q) {
      const unsigned long long y = __shfl_xor_sync(0xFFFFFFFFu, v[q], o);
      v[q] = q < 2 ? (y < v[q] ? y : v[q]) : v[q] + y;
    }
    st = min(st, __shfl_xor_sync(0xFFFFFFFFu, st, o));
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < kVals; ++q) s_w[wid][q] = v[q];
    s_st[wid] = st;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint32_t w = 1; w < nw; ++w) {
#pragma unroll
      for (int q = 0; q < kVals; ++q) v[q] = q < 2 ? (s_w[w][q] < v[q] ? s_w[w][q] : v[q]) : v[q] + s_w[w][q];
      st = min(st, s_st[w]);
    }
    keys[0] = v[0];
    keys[1] = has_rs ? v[1] : v[0];
    stats[0] = v[2];
    stats[1] = v[3];
    stats[2] = v[4];
    stats[3] = v[5];
    stats[4] = (unsigned long long)(long long)st;
    stats[5] = v[6];
    stats[6] = v[7];
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

// limit: a send ending after it (a relay still in flight when the postcondition
// holds, R22) is written as a tombstone (chunk = kNone) for compact_sends.
// Winner chosen on the device (DevWin): the records of the job named by the best key, the
// shift of an AR's AG half = T of that key (a symmetric RS lasts as long as its AG), nothing
// written when the winning seed is not in this plan's shard.
__device__ __forceinline__ const Rec *dev_winner(const DevWin &dw, uint64_t &T) {
  const unsigned long long key = dw.keys[0];
  const uint64_t g = key & ((1ull << kKeySeedBits) - 1ull);
  T = key >> kKeySeedBits;
  if (key == kNoKey || g < dw.seed_offset || g - dw.seed_offset >= dw.n_seeds) return nullptr;
  return dw.rec_base + (g - dw.seed_offset) * dw.cap;
}

__global__ void emit_ag_kernel(const Rec *__restrict__ rec, uint64_t M, const uint32_t *__restrict__ src,
                               const uint32_t *__restrict__ dst, const uint32_t *__restrict__ w, uint64_t shift,
                               uint64_t limit, Send32 *__restrict__ out, DevWin dw) {
  if (dw.keys) {
    uint64_t T;
    rec = dev_winner(dw, T);
    if (!rec) return;
    shift = dw.shift_by_T ? T : 0ull;
  }
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < M; i += (uint64_t)gridDim.x * blockDim.x) {
    const Rec r = rec[i];
    Send32 s;
    s.chunk = r.t_start + w[r.link] > limit ? kNone : r.chunk;
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
                   uint64_t shift, void *out_sends, void *stream, uint64_t limit, const DevWin *dw) {
  emit_ag_kernel<<<grid_for(M, 256), 256, 0, (cudaStream_t)stream>>>(rec, M, src, dst, w, shift, limit,
                                                                      reinterpret_cast<Send32 *>(out_sends),
                                                                      dw ? *dw : DevWin{});
  return check_launch("emit_ag_kernel");
}

// Stream compaction of the tombstones left by the emitters (relay mode only, R22):
// one CTA walks the sends tile by tile, order preserved, in place (a kept send
// moves to an index <= its own, and a tile is read completely before it is written).
__global__ void compact_sends_kernel(Send32 *__restrict__ s, uint64_t n, unsigned long long *__restrict__ count) {
  __shared__ uint32_t warp_tot[32];
  __shared__ unsigned long long base;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, wid = tid >> 5, nw = blockDim.x >> 5;
  if (tid == 0) base = 0;
  __syncthreads();
  for (uint64_t t0 = 0; t0 < n; t0 += blockDim.x) {
    const uint64_t i = t0 + tid;
    Send32 v{};
    bool keep = false;
    if (i < n) {
      v = s[i];
      keep = v.chunk != kNone;
    }
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, keep);
    if (lane == 0) warp_tot[wid] = __popc(bal);
    __syncthreads();  // the whole tile is read (and counted) before any write
    uint32_t before = 0, total = 0;
    for (uint32_t j = 0; j < nw; ++j) {
      before += j < wid ? warp_tot[j] : 0u;
      total += warp_tot[j];
    }
    if (keep) s[base + before + __popc(bal & ((1u << lane) - 1u))] = v;
    __syncthreads();
    if (tid == 0) base += total;
    __syncthreads();
  }
  if (tid == 0) *count = base;
}

int launch_compact_sends(void *sends, uint64_t n, unsigned long long *d_count, void *stream) {
  compact_sends_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(reinterpret_cast<Send32 *>(sends), n, d_count);
  return check_launch("compact_sends_kernel");
}

// RS = mirror of an AG: (c, a->b on l, t0, t1) -> (c, b->a on l', T-t1, T-t0)
// with l' = rev[l] when G is symmetric (AG searched on G), else l' = l (AG searched on G^T).
__global__ void rs_keys_kernel(const Rec *__restrict__ rec, uint64_t M, const uint32_t *__restrict__ w,
                               const int32_t *__restrict__ rev, uint64_t T_rs, uint32_t lbits, uint32_t mirror,
                               unsigned long long *__restrict__ keys, uint32_t *__restrict__ vals) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < M; i += (uint64_t)gridDim.x * blockDim.x) {
    const Rec r = rec[i];
    const uint32_t l2 = (mirror && rev) ? (uint32_t)rev[r.link] : r.link;
    const bool late = mirror && r.t_start + w[r.link] > T_rs;  // relay in flight at the end (R22): sorted last
    const unsigned long long t0 = mirror ? T_rs - (r.t_start + w[r.link]) : r.t_start;
    keys[i] = late ? ~0ull : ((t0 << lbits) | l2);
    vals[i] = (uint32_t)i;
  }
}

__global__ void rs_emit_kernel(const uint32_t *__restrict__ vals, const Rec *__restrict__ rec, uint64_t M,
                               const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                               const uint32_t *__restrict__ w, const int32_t *__restrict__ rev, uint64_t T_rs,
                               uint32_t mirror, uint64_t shift, Send32 *__restrict__ out) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < M; j += (uint64_t)gridDim.x * blockDim.x) {
    const Rec r = rec[vals[j]];
    const uint32_t l2 = (mirror && rev) ? (uint32_t)rev[r.link] : r.link;
    Send32 s;
    s.chunk = (mirror && r.t_start + w[r.link] > T_rs) ? kNone : r.chunk;  // tombstone, see rs_keys_kernel
    s.link = l2;
    s.src = src[l2];
    s.dst = dst[l2];
    if (mirror) {
      s.t0 = T_rs - (r.t_start + w[r.link]);
      s.t1 = T_rs - r.t_start;
    } else {  // records in arbitrary order (paper-literal variant): sorted, shifted AG sends
      s.t0 = r.t_start + shift;
      s.t1 = r.t_start + w[r.link] + shift;
    }
    out[j] = s;
  }
}

// ---- LSD radix sort of (u64 key, u32 value), 8-bit digits, stable ----
constexpr int kRsThreads = 256;
constexpr int kRsItems = 4;
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

// Block-wide exclusive scan of one value per thread (blockDim = 256); returns
// the exclusive prefix and writes the block total to *total.
__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t v, uint32_t *s_warp, uint32_t *total) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= (uint32_t)o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < 8 ? s_warp[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, w, o);
      if (lane >= (uint32_t)o) w += y;
    }
    if (lane < 8) s_warp[8 + lane] = w;
  }
  __syncthreads();
  const uint32_t before = warp ? s_warp[8 + warp - 1] : 0u;
  *total = s_warp[15];
  __syncthreads();
  return before + incl - v;
}

// One block per digit: exclusive scan of that digit's per-tile counts
// hist[d][0..nb) in place (coalesced), digit total to totals[d].
__global__ void radix_rowscan_kernel(uint32_t *__restrict__ hist, uint32_t nb, uint32_t *__restrict__ totals) {
  __shared__ uint32_t s_warp[16];
  uint32_t *row = hist + (size_t)blockIdx.x * nb;
  uint32_t running = 0;
  for (uint32_t base = 0; base < nb; base += 256u) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t v = i < nb ? row[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan256(v, s_warp, &tot);
    if (i < nb) row[i] = running + ex;
    running += tot;
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = running;
}

__global__ void radix_scatter_kernel(const unsigned long long *__restrict__ keys_in,
                                     const uint32_t *__restrict__ vals_in, uint64_t n, int shift,
                                     const uint32_t *__restrict__ offs, const uint32_t *__restrict__ totals,
                                     uint32_t nblocks,
                                     unsigned long long *__restrict__ keys_out, uint32_t *__restrict__ vals_out) {
  constexpr int kWarps = kRsThreads / 32;
  __shared__ uint32_t s_off[256];
  __shared__ uint32_t s_wc[kWarps][256];
  __shared__ uint32_t s_tot[256];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  {
    __shared__ uint32_t s_warp[16];
    uint32_t tot;
    const uint32_t digit_base = block_excl_scan256(totals[tid], s_warp, &tot);
    s_off[tid] = digit_base + offs[(size_t)tid * nblocks + blockIdx.x];
  }
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
  return al(M * 8) * 2 + al(M * 4) * 2 + al(nb * 256 * 4 + 256 * 4 + 4);
}

int launch_rs_sort_emit(const Rec *rec, uint64_t M, const uint32_t *src, const uint32_t *dst, const uint32_t *w,
                        const int32_t *rev, uint64_t T_rs, uint32_t L, void *out_sends, void *scratch,
                        size_t scratch_bytes, uint32_t *launches, void *stream, uint32_t mirror, uint64_t shift) {
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
  const uint32_t nb0 = (uint32_t)((M + kRsTile - 1) / kRsTile);
  uint32_t *totals = hist + (size_t)nb0 * 256u;
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
  rs_keys_kernel<<<grid_for(M, 256), 256, 0, st>>>(rec, M, w, rev, T_rs, lbits, mirror, ka, va);
  ++nl;
  int rc = check_launch("rs_keys_kernel");
  if (rc) return rc;
  const uint32_t nb = (uint32_t)((M + kRsTile - 1) / kRsTile);
  for (uint32_t shift = 0; shift < bits; shift += 8) {
    radix_hist_kernel<<<nb, kRsThreads, 0, st>>>(ka, M, (int)shift, hist, nb);
    radix_rowscan_kernel<<<256, 256, 0, st>>>(hist, nb, totals);
    radix_scatter_kernel<<<nb, kRsThreads, 0, st>>>(ka, va, M, (int)shift, hist, totals, nb, kb, vb);
    nl += 3;
    rc = check_launch("radix pass");
    if (rc) return rc;
    unsigned long long *tk = ka; ka = kb; kb = tk;
    uint32_t *tv = va; va = vb; vb = tv;
  }
  rs_emit_kernel<<<grid_for(M, 256), 256, 0, st>>>(va, rec, M, src, dst, w, rev, T_rs, mirror, shift,
                                                   reinterpret_cast<Send32 *>(out_sends));
  ++nl;
  if (launches) *launches += nl;
  return check_launch("rs_emit_kernel");
}

// ---------------------------------------------------------------------------
// a8, uniform link cost: when every link costs the same w and G is symmetric (RS = the
// same-seed mirror on the reverse links, R9), the RS key (T_rs - t_start - w, rev[link])
// orders the AG events in reverse and, inside an event, by reverse link id.  The AG
// records are sorted by (t_start, link), so an event is a contiguous segment holding each
// link at most once: the RS position of record i is (M - end of its segment) + the rank of
// rev[link_i] among the segment's reverse links (a link-id bitmap prefix).  Same order as
// the radix sort, without it.
// ---------------------------------------------------------------------------
// starts: the segment starts (unordered); flags[i] = 1 where a segment starts (i < M), 0 up to
// the 16-byte padded end, so a CTA finds a segment's end with 16-flag vector loads
__global__ void seg_starts_kernel(const Rec *__restrict__ rec, uint64_t M, uint32_t *__restrict__ starts,
                                  unsigned int *__restrict__ n_seg, unsigned char *__restrict__ flags, uint64_t n_flags,
                                  DevWin dw) {
  if (dw.keys) {
    uint64_t T;
    rec = dev_winner(dw, T);
    if (!rec) return;
  }
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_flags; i += (uint64_t)gridDim.x * blockDim.x) {
    const bool b = i < M && (i == 0 || rec[i].t_start != rec[i - 1].t_start);
    flags[i] = b ? 1 : 0;
    if (b) starts[atomicAdd(n_seg, 1u)] = (uint32_t)i;
  }
}

// mirror = 0 (AG records of the lock-step loop, in (t_start, CTA, position) order): the same
// segment ranking with the identity link map puts record i at (start of its segment) + the rank
// of link_i among the segment's links, i.e. in (t_start, link) order, times shifted by T_rs.
// mirror = 2: both phases of an AR from one read of the records (RS at out[0, M), AG at
// out[M, 2M) shifted by T_rs = T_AG; a symmetric AR's two phases come from the same seed).
__global__ void rs_uniform_emit_kernel(const Rec *__restrict__ rec, uint64_t M, const uint32_t *__restrict__ starts,
                                       const unsigned int *__restrict__ n_seg, const unsigned char *__restrict__ flags,
                                       uint64_t n_flags, const uint32_t *__restrict__ src,
                                       const uint32_t *__restrict__ dst, uint32_t w0, const int32_t *__restrict__ rev,
                                       uint64_t T_rs, uint32_t L, Send32 *__restrict__ out, DevWin dw, uint32_t mirror) {
  extern __shared__ uint32_t sm[];
  if (dw.keys) {
    uint64_t T;
    rec = dev_winner(dw, T);
    if (!rec) return;
    T_rs = mirror ? T : (dw.shift_by_T ? T : 0ull);
  }
  const uint32_t nbw = (L + 31u) / 32u;
  const bool doR = mirror != 0u, doA = mirror != 1u;
  // side 0: reverse links (RS), side 1: link ids (AG); a bitmap and its prefix each
  uint32_t *bmR = sm, *preR = sm + nbw;
  uint32_t *bmA = doR ? sm + 2u * nbw : sm, *preA = bmA + nbw;
  __shared__ unsigned long long s_end;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const unsigned int nseg = *n_seg;
  for (uint32_t sg = blockIdx.x; sg < nseg; sg += gridDim.x) {
    const uint64_t s = starts[sg];
    for (uint32_t i = tid; i < (doR && doA ? 2u : 1u) * 2u * nbw; i += blockDim.x) sm[i] = 0u;
    if (tid == 0) s_end = M;
    __syncthreads();
    // segment end: the next segment start after s (16 flags per thread and pass)
    for (uint64_t c = (s + 1) & ~15ull; c < M; c += 16ull * blockDim.x) {
      const uint64_t i0 = c + 16ull * tid;
      if (i0 < n_flags) {
        const uint4 f = *reinterpret_cast<const uint4 *>(flags + i0);
        const uint32_t wv[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint32_t m = wv[k];
          // drop flags at or before s (the pass starts at the 16-aligned position below s + 1)
          while (m) {
            const uint32_t byte = (uint32_t)(__ffs(m) - 1) >> 3;
            const uint64_t i = i0 + 4u * k + byte;
            if (i > s && i < M) {
              atomicMin(&s_end, (unsigned long long)i);
              break;
            }
            m &= ~(0xFFu << (8u * byte));
          }
        }
      }
      if (__syncthreads_or(s_end != M)) break;
    }
    const uint64_t e = s_end;
    for (uint64_t i = s + tid; i < e; i += blockDim.x) {
      const uint32_t l = rec[i].link;
      if (doR) {
        const uint32_t l2 = (uint32_t)rev[l];
        atomicOr(&bmR[l2 >> 5], 1u << (l2 & 31u));
      }
      if (doA) atomicOr(&bmA[l >> 5], 1u << (l & 31u));
    }
    __syncthreads();
    // exclusive prefix of the bitmap word counts: warp 0 the RS side, warp 1 (or 0) the AG side
    if ((doR && warp == 0u) || (doA && warp == (doR ? 1u : 0u))) {
      uint32_t *bm = (doR && warp == 0u) ? bmR : bmA, *pre = (doR && warp == 0u) ? preR : preA;
      uint32_t running = 0;
      for (uint32_t b = 0; b < nbw; b += 32u) {
        const uint32_t i = b + lane;
        const uint32_t v = i < nbw ? __popc(bm[i]) : 0u;
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
          if (lane >= (uint32_t)o) incl += y;
        }
        if (i < nbw) pre[i] = running + incl - v;
        running += __shfl_sync(0xFFFFFFFFu, incl, 31);
      }
    }
    __syncthreads();
    Send32 *outA = mirror == 2u ? out + M : out;
    for (uint64_t i = s + tid; i < e; i += blockDim.x) {
      const Rec r = rec[i];
      if (doR) {
        const uint32_t l2 = (uint32_t)rev[r.link];
        const uint32_t rank = preR[l2 >> 5] + __popc(bmR[l2 >> 5] & ((1u << (l2 & 31u)) - 1u));
        Send32 o;
        o.chunk = r.chunk;
        o.link = l2;
        o.src = src[l2];
        o.dst = dst[l2];
        o.t0 = T_rs - (r.t_start + w0);
        o.t1 = T_rs - r.t_start;
        out[M - e + rank] = o;
      }
      if (doA) {
        const uint32_t l = r.link;
        const uint32_t rank = preA[l >> 5] + __popc(bmA[l >> 5] & ((1u << (l & 31u)) - 1u));
        Send32 o;
        o.chunk = r.chunk;
        o.link = l;
        o.src = src[l];
        o.dst = dst[l];
        o.t0 = r.t_start + T_rs;
        o.t1 = r.t_start + w0 + T_rs;
        outA[s + rank] = o;
      }
    }
    __syncthreads();
  }
}

int launch_rs_uniform_emit(const Rec *rec, uint64_t M, const uint32_t *src, const uint32_t *dst, uint32_t w0,
                           const int32_t *rev, uint64_t T_rs, uint32_t L, void *out_sends, void *scratch,
                           size_t scratch_bytes, uint32_t *launches, void *stream, const DevWin *dw, uint32_t mirror) {
  const DevWin dwv = dw ? *dw : DevWin{};
  cudaStream_t st = (cudaStream_t)stream;
  if (M == 0) return 0;
  if (scratch_bytes < 256 + ((M * 4 + 255) / 256) * 256 + M + 16 || M >= (1ull << 32)) {
    snprintf(g_cuda_err, sizeof(g_cuda_err), "rs uniform emit: scratch too small");
    return -9;
  }
  unsigned int *n_seg = reinterpret_cast<unsigned int *>(scratch);
  uint32_t *starts = reinterpret_cast<uint32_t *>(reinterpret_cast<unsigned char *>(scratch) + 256);
  const uint64_t n_flags = (M + 15u) & ~15ull;
  unsigned char *flags = reinterpret_cast<unsigned char *>(scratch) + 256 + ((M * 4 + 255) / 256) * 256;
  cudaMemsetAsync(n_seg, 0, sizeof(unsigned int), st);
  seg_starts_kernel<<<grid_for(n_flags, 256), 256, 0, st>>>(rec, M, starts, n_seg, flags, n_flags, dwv);
  int rc = check_launch("seg_starts_kernel");
  if (rc) return rc;
  const uint32_t nbw = (L + 31u) / 32u;
  const uint32_t smem = (mirror == 2u ? 4u : 2u) * nbw * 4u;  // link-id bitmap(s) + prefix(es)
  if (smem > 48u * 1024u) {
    const cudaError_t e = cudaFuncSetAttribute(rs_uniform_emit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      snprintf(g_cuda_err, sizeof(g_cuda_err), "rs_uniform_emit_kernel: %u B of shared memory: %s", smem,
               cudaGetErrorString(e));
      return -4;
    }
  }
  rs_uniform_emit_kernel<<<148, 1024, smem, st>>>(rec, M, starts, n_seg, flags, n_flags, src, dst, w0, rev, T_rs, L,
                                                   reinterpret_cast<Send32 *>(out_sends), dwv, mirror);
  if (launches) *launches += 2;
  return check_launch("rs_uniform_emit_kernel");
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
