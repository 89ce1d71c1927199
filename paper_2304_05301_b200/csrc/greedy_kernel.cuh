// greedy_kernel.cuh -- the TACOS-Greedy search kernel (rows a2-a6 of SURVEY §8).
//
// One CTA = one job (seed, orientation sigma) and runs the whole event loop of
// one greedy All-Gather synthesis (§VI.A, §VI.B),
// device-resident: no host round trip per event.  Per event, 3 block barriers:
//
//   PA  (per destination)    records of the previous event in link-id order;
//                            arrivals at t: held[dst] |= chunk (R7)
//       -- barrier --        done test: delivered == required
//                            (optionally the Philox draws run on PA's spare threads)
//   PM  (per destination,    free in-links (busy_until <= t); exact skip of a
//        P lanes each)       link whose source is unchanged since its last
//                            empty visit; Philox draws (R2); shorter-link-first
//                            order (w, u_ord, link) (R3); then the matching walk:
//                            have[d] row in registers, per in-link 128-bit loads
//                            of held[src], andnot + popc, segmented scan over the
//                            P lanes, r = umulhi(u_pick, K) (R13), branch-free
//                            rank-select of the r-th candidate, claim (R4)
//       -- barrier --
//   PE                       record offsets (link-id bitmap prefix), next event
//                            time = min busy_until (u64 warp shuffles)
//       -- barrier --
//
// Destinations are independent inside an event (a destination's walk writes
// only its own in-links' state and its own `have` row; `held` changes only in
// PA), so PM needs no block barrier between destinations.
//
// Thread-block clusters: a job may be split over a cluster of Q CTAs (Q SMs),
// each owning a contiguous range of destinations (their rows, in-links and
// link state).  A walk reads held[src] / hver[src] of a source owned by another
// CTA through distributed shared memory; the delivered count, the next event
// time and the record bitmap are exchanged with DSMEM atomics; the two
// event-level barriers become cluster barriers (release/acquire at cluster scope).
//
// Three event loops share the phases above:
//   per-event  the scheme above;
//   lock-step  one link cost, one lane per destination: every send started at t
//              ends at the next event t + w, so a walker writes d's next held row
//              (= have[d] after its walk) into the other buffer of held[2][N] and
//              pushes it to the mirroring CTAs -- no PA, one cluster barrier per
//              event; records in (t_start, CTA, position) order from a position
//              bitmap, ranked by link at emission;
//   windowed   several link costs, wide rows: all events of [T0, T0 + w_min)
//              run per destination between one set of cluster barriers.
#pragma once
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "tacos_device.cuh"

namespace tacos {

constexpr int kRegDeg = 8;  // in-degree handled in registers by the P == 1 path
// P == 1 register path: true = `have` row in shared memory (step_row), false = in registers
// (the lane-pair path with one lane)
constexpr bool kP1Smem = true;
#ifndef TACOS_P1_HAVE_REG  // 1: the P == 1 walk keeps have[d] in registers (experiment)
#define TACOS_P1_HAVE_REG 0
#endif

#ifndef TACOS_WIN_EAGER_HAVE  // 1: the windowed loop reads a destination's have row up front
#define TACOS_WIN_EAGER_HAVE 0
#endif
#ifndef TACOS_STEP1  // 1: the P == 1 walk step keeps per-word counts and selects the bit without POPC
#define TACOS_STEP1 1  // measured: config 2 0.283 -> 0.269 ms, config 3 0.745 -> 0.740, config 5 3.044 -> 3.015
#endif
#ifndef TACOS_MIN_BLOCKS  // resident CTAs per SM the register budget is sized for
#define TACOS_MIN_BLOCKS 1
#endif
#ifndef TACOS_P2_SPLIT_DRAWS  // 1: the two-lane path splits the Philox draws between its lanes
#define TACOS_P2_SPLIT_DRAWS 1
#endif
#ifndef TACOS_WIDE_PREFETCH  // 1: next-row prefetch in the wide-row register walk (needs registers)
#define TACOS_WIDE_PREFETCH 0
#endif
#ifndef TACOS_V4_THREADS  // thread bound of the 4-vector kernels (registers: 65536 / bound per thread)
#define TACOS_V4_THREADS 384
#endif
#ifndef TACOS_WIDE_THREADS  // thread bound of the wide-row kernels (P > 2 lanes, 4 vectors)
#define TACOS_WIDE_THREADS 512  // 128 registers: 32 lane groups of 16 in flight instead of 24 (config 4: 223 -> 213 ms)
#endif
#ifndef TACOS_V2_THREADS  // thread bound of the other 2-vector kernels (tuning; default as the 4-vector ones)
#define TACOS_V2_THREADS TACOS_V4_THREADS
#endif
// thread bound per kernel shape (registers per thread <= 65536 / bound): one vector per lane 768,
// two-lane groups of two vectors 640 (one group per destination of a 256-destination CTA plus
// the record warps), otherwise TACOS_V4_THREADS
template <int P, int V>
struct ThreadsFor {
  static constexpr int value = V == 1 ? 768 : (P == 2 && V == 2) ? 640 : V == 2 ? TACOS_V2_THREADS
                                : P > 2 ? TACOS_WIDE_THREADS : TACOS_V4_THREADS;
};
// MASKED (relays, R22): candidates are also and-ed with the
// per-position allow row, and only arrivals of chunks in post[dst] count.
// BIG: the one-lane four-vector register-path kernel bounded at kBigThreads (128 registers) for
// CTAs with more own destinations than the default bound leaves walker threads for (e.g. 512 NPUs
// on one SM): one destination per walker instead of two in sequence (the paper's 512-NPU
// Ring x FC x Switch: 8.1 -> 7.0 ms); the default bound stays faster where the destinations fit.
constexpr int kBigThreads = 512;
template <int P, int V, bool ROWS_SMEM, bool LINKS_SMEM, bool REG_PATH, bool MASKED, bool BIG = false>
__global__ void __launch_bounds__(BIG ? kBigThreads : ThreadsFor<P, V>::value, TACOS_MIN_BLOCKS)
greedy_kernel(const Job *__restrict__ jobs, JobOut *__restrict__ outs, const Layout lay) {
  static_assert(P >= 1 && P <= 32 && (P & (P - 1)) == 0, "P must be a power of two <= 32");
  // one thread per destination with shared-memory rows: `have` stays in shared memory and a
  // claim is one word update (no per-word predicated register updates)
  constexpr bool kHaveSmem = (P == 1) && ROWS_SMEM && !TACOS_P1_HAVE_REG;
  extern __shared__ __align__(16) unsigned char smem[];
  // 64-bit shared atomics are CAS loops on sm_100a: per-event values use 32-bit atomics
  // (arrivals of one event; next event time as an offset from t, < 2^32 since w < 2^32)
  __shared__ unsigned long long s_delivered, s_V, s_D, s_M, s_L;
  __shared__ uint32_t s_arr[2], s_min32[2], s_mcnt[2];
  // cluster exchange slots, indexed by the writer's rank (plain remote stores, no 64-bit DSMEM atomics)
  // s_slot_min2: event parity (the lock-step loop has one cluster barrier per event, so a peer may
  // publish event e + 1 before this CTA has read event e's slots)
  __shared__ unsigned long long s_slot_deliv[kMaxCluster], s_slot_min2[2][kMaxCluster], s_slot_cnt[kMaxCluster][4];

  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const uint32_t Q = cluster.num_blocks();
  const uint32_t crank = cluster.block_rank();
  const Job job = jobs[blockIdx.x / Q];
  const DevTopo T = *job.topo;
  const uint32_t N = T.N, L = T.L, Wp = T.Wp;
  // row stride in words: padded in shared memory so rows of different NPUs start in different
  // bank groups (a warp's 128-bit loads of random rows would otherwise 16-way conflict)
  const uint32_t Wr = ROWS_SMEM ? lay.row_stride : Wp;
  const uint32_t tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31u;
  const uint32_t *__restrict__ p_src = T.p_src;
  const uint32_t *__restrict__ p_w = T.p_w;
  const uint32_t *__restrict__ p_lid = T.p_lid;
  const uint32_t *__restrict__ in_ptr = T.in_ptr;
  const bool custom = T.custom != 0u;

  uint32_t *held;
  if constexpr (ROWS_SMEM) held = reinterpret_cast<uint32_t *>(smem);
  else held = job.g_rows;
  uint32_t *have = held + (size_t)N * Wr;  // held | pending | claimed (R4)
  unsigned char *links_base;
  if constexpr (LINKS_SMEM) links_base = smem + (ROWS_SMEM ? lay.rows_bytes : 0u);
  else links_base = job.g_links;
  unsigned long long *busy = reinterpret_cast<unsigned long long *>(links_base + lay.off_busy);
  uint32_t *cur = reinterpret_cast<uint32_t *>(links_base + lay.off_cur);
  uint32_t *ord = reinterpret_cast<uint32_t *>(links_base + lay.off_ord);
  uint32_t *pick = reinterpret_cast<uint32_t *>(links_base + lay.off_pick);
  uint32_t *seen = reinterpret_cast<uint32_t *>(links_base + lay.off_seen);
  uint16_t *order = reinterpret_cast<uint16_t *>(links_base + lay.off_order);  // walk order: position - b0
  uint16_t *rch = reinterpret_cast<uint16_t *>(links_base + lay.off_rch);      // chunk of a match, 2 event parities
  unsigned char *lv = links_base + lay.off_lv;
  // per-position topology (source, cost, link id, destination): staged into shared memory with
  // the link state, NPU and link ids as u16 there (the host keeps N, L < 2^16 for that layout)
  using IdT = typename std::conditional<LINKS_SMEM, uint16_t, uint32_t>::type;
  const IdT *t_src, *t_lid, *t_dst;
  const uint32_t *t_w = p_w;
  if constexpr (LINKS_SMEM) {
    t_src = reinterpret_cast<const IdT *>(links_base + lay.off_tsrc);
    t_w = reinterpret_cast<const uint32_t *>(links_base + lay.off_tw);
    t_lid = reinterpret_cast<const IdT *>(links_base + lay.off_tlid);
    t_dst = reinterpret_cast<const IdT *>(links_base + lay.off_tdst);
  } else {
    t_src = p_src;
    t_lid = p_lid;
    t_dst = T.p_dst;
  }
  uint32_t *hver = reinterpret_cast<uint32_t *>(smem + lay.off_hver);
  uint32_t *bitmap2 = reinterpret_cast<uint32_t *>(smem + lay.off_bitmap);  // 2 x nbw words (event parity)
  uint32_t *wpre = reinterpret_cast<uint32_t *>(smem + lay.off_wpre);
  uint32_t *s_inptr = reinterpret_cast<uint32_t *>(smem + lay.off_inptr);  // CSR offsets, own range
  uint32_t *s_list = reinterpret_cast<uint32_t *>(smem + lay.off_list);    // worklist entries
  __shared__ uint32_t s_nwork;
  __shared__ unsigned s_dbg[5];  // debug (TACOS_TRACE): slowest matching / record thread of an event
  if (tid < 5) s_dbg[tid] = 0u;
  const uint32_t nbw = (L + 31u) / 32u;
  const uint32_t seed_lo = (uint32_t)job.seed, seed_hi = (uint32_t)(job.seed >> 32);
  Rec *rec = job.rec;

  // destinations [d_lo, d_hi) and their in-link positions [p_lo, p_hi) belong to this CTA
  const uint32_t chunkN = (N + Q - 1u) / Q;
  const uint32_t d_lo = min(N, crank * chunkN), d_hi = min(N, d_lo + chunkN);
  const uint32_t p_lo = __ldg(&in_ptr[d_lo]), p_hi = __ldg(&in_ptr[d_hi]);
  const bool worklist = lay.worklist != 0u;
  TCHECK(lay.smem_bytes <= dynamic_smem_bytes(), "layout exceeds the dynamic shared memory");
  TCHECK(d_lo <= d_hi && p_lo <= p_hi && p_hi <= L, "CTA ranges");
  // Lock-step loop (one link cost, one lane per destination, AG-type, no relays; host: add_lockstep):
  // every send started at t ends at the next event t + w, so the walkers write the arrivals of the
  // next event themselves into the other held buffer (held[2][N], event parity) and an event needs
  // one cluster barrier.  Its layout keeps only the CTA's own have rows and in-link positions:
  // the pointers are shifted so that global indices address them.
  constexpr bool kLock = P == 1 && kP1Smem && ROWS_SMEM && LINKS_SMEM && !MASKED;
  const bool lockstep = kLock && lay.lockstep != 0u;
  uint32_t *const held_base = held, *const hver_base = hver;
  if (lockstep) {
    TCHECK(p_hi - p_lo <= lay.pos_cap, "lock-step position capacity");
    have = held + (size_t)2u * N * Wr - (size_t)d_lo * Wr;
    busy -= p_lo;
    cur -= p_lo;
    ord -= p_lo;
    pick -= p_lo;
    seen -= p_lo;
    order -= p_lo;
    rch -= 2u * p_lo;
    lv -= p_lo;
    t_src -= p_lo;
    t_w -= p_lo;
    t_lid -= p_lo;
    t_dst -= p_lo;
  }
  auto cluster_barrier = [&]() {
    if (Q > 1) cluster.sync();
    else __syncthreads();
  };

  // owner CTA of NPU x = x / chunkN, by a multiply-high with m = ceil(2^32 / chunkN):
  // exact while x * (m * chunkN - 2^32) < 2^32, i.e. for N < 2^16
  // (chunkN = 1 would need m = 2^32: the owner is x itself)
  const uint32_t own_magic = (uint32_t)((0xFFFFFFFFull + chunkN) / chunkN);
  auto owner_of = [&](uint32_t x) -> uint32_t {
    return chunkN == 1u ? x : (N < 65536u ? __umulhi(x, own_magic) : x / chunkN);
  };
  // Mirrors: a CTA keeps local copies of the held rows (shared-memory layout) and source
  // versions of the peers' NPUs that are sources of its in-links; the owner pushes every
  // arrival to them (DSMEM red.or / st) before the cluster barrier, so the matching phase
  // reads only its own shared memory.  s_peers[x] (own x): peer ranks that mirror x.
  uint32_t *s_peers = reinterpret_cast<uint32_t *>(smem + lay.off_peers);
  auto hver_of = [&](uint32_t x) -> uint32_t { return hver[x]; };

  // ---- a2: state init (P:L89 precondition; P:L212 start at t = 0) ----
  const uint32_t NW = N * Wp;
  // held: every row in shared memory (own rows and the mirrors), own rows only in global memory
  // (shared by the cluster); have: own rows
  const uint32_t i_lo = ROWS_SMEM ? 0u : d_lo * Wp, i_hi = ROWS_SMEM ? NW : d_hi * Wp;
  for (uint32_t i = i_lo + tid; i < i_hi; i += nthr) {
    uint32_t v, hv0;
    const uint32_t x = i / Wp, q = i - x * Wp;
    if (custom) {
      // chunks d does not require are never candidates: have[d] starts as pre | ~post
      // (with relays the per-link allow rows take that role)
      v = __ldg(&T.pre[i]);
      hv0 = MASKED ? v : (v | ~__ldg(&T.post[i]));
    } else {  // AG: chunks x*k .. x*k+k-1 (R12)
      const uint32_t xo = T.npu_orig ? T.npu_orig[x] : x;  // chunks of the NPU's original id (R12)
      const uint32_t lo = xo * T.k, hi = lo + T.k, wlo = q * 32u, whi = wlo + 32u;
      const uint32_t a = lo > wlo ? lo : wlo, b = hi < whi ? hi : whi;
      v = 0u;
      if (a < b) v = ((b - a) == 32u ? 0xFFFFFFFFu : ((1u << (b - a)) - 1u)) << (a - wlo);
      hv0 = v;
    }
    held[(size_t)x * Wr + q] = v;
    if (x - d_lo < d_hi - d_lo) have[(size_t)x * Wr + q] = hv0;
  }
  for (uint32_t p = p_lo + tid; p < p_hi; p += nthr) {
    busy[p] = 0ull;
    cur[p] = kNone;
    seen[p] = kNone;
    if constexpr (LINKS_SMEM) {
      const_cast<IdT *>(t_src)[p] = (IdT)__ldg(&p_src[p]);
      const_cast<uint32_t *>(t_w)[p] = __ldg(&p_w[p]);
      const_cast<IdT *>(t_lid)[p] = (IdT)__ldg(&p_lid[p]);
      const_cast<IdT *>(t_dst)[p] = (IdT)__ldg(&T.p_dst[p]);
    }
  }
  for (uint32_t x = tid; x < (lockstep ? 2u * N : N); x += nthr) hver[x] = 0u;
  for (uint32_t x = d_lo + tid; x < d_hi; x += nthr) s_peers[x] = 0u;
  for (uint32_t x = d_lo + tid; x <= d_hi; x += nthr) s_inptr[x] = __ldg(&in_ptr[x]);
  for (uint32_t i = tid; i < 2u * nbw; i += nthr) bitmap2[i] = 0u;
  if (tid == 0) {
    s_delivered = 0ull;
    s_arr[0] = s_arr[1] = 0u;
    s_V = s_D = s_M = s_L = 0ull;
  }
  cluster_barrier();  // peers may add to our counters / mirror lists from now on
  if (Q > 1) {  // register as a mirror of the remote sources of own in-links
    for (uint32_t q = p_lo + tid; q < p_hi; q += nthr) {
      const uint32_t sp = t_src[q];
      if (sp - d_lo >= d_hi - d_lo) dsmem_or_b32(dsmem_addr(s_peers + sp, owner_of(sp)), 1u << crank);
    }
    cluster_barrier();
  }

  unsigned long long t = 0ull, t_prev = 0ull;
  uint32_t e = 0u, E = 0u;
  int status = 0;
  unsigned long long myV = 0, myD = 0, myM = 0, myL = 0;  // myL: live visits (rows read)

  const uint32_t gl = lane & (P - 1);
  const uint32_t gmask = (P == 32) ? 0xFFFFFFFFu : (((1u << P) - 1u) << (lane & ~(uint32_t)(P - 1)));
  const uint32_t ngroups = nthr / P;
  const bool pre_draw = lay.pre_draw != 0u;
  const bool tracing = job.trace != nullptr && tid == 0;
  // Send records of the matches of event ev-1 (own positions; their index = base + rank of
  // the link id in the cluster-wide bitmap of ev-1, so records are ordered by (t_start, link)),
  // chunk from rch (parity of ev-1), by a group of `count` threads starting at `first` (a
  // multiple of 32; the whole CTA when first == 0): the group's first warp turns the bitmap
  // into word offsets, the group writes, then clears the bitmap for its reuse at ev+1.
  auto write_records = [&](uint32_t first, uint32_t count, uint32_t ev, uint32_t base,
                           unsigned long long t_start, bool clear) {
    if (rec == nullptr || ev == 0u) return;
    auto group_sync = [&]() {
      if (count == nthr) __syncthreads();
      else asm volatile("bar.sync 1, %0;" ::"r"(count) : "memory");
    };
    const uint32_t par = (ev + 1u) & 1u;
    uint32_t *bmp = bitmap2 + par * nbw;
    // bitmap keys: link ids (cluster-wide bitmap), or in the lock-step loop the CTA's own
    // positions q - p_lo (its records follow those of the lower cluster ranks: base)
    const uint32_t nkw = lockstep ? (p_hi - p_lo + 31u) / 32u : nbw;
    if (tid - first < 32u) {
      uint32_t running = 0;
      for (uint32_t b = 0; b < nkw; b += 32u) {
        const uint32_t i = b + lane;
        const uint32_t v = i < nkw ? __popc(bmp[i]) : 0u;
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
          if (lane >= (uint32_t)o) incl += y;
        }
        if (i < nkw) wpre[i] = running + incl - v;
        running += __shfl_sync(0xFFFFFFFFu, incl, 31);
      }
    }
    group_sync();
    for (uint32_t q = p_lo + (tid - first); q < p_hi; q += count) {
      const uint32_t lid = t_lid[q], key = lockstep ? q - p_lo : lid;
      const uint32_t wi = key >> 5, word = bmp[wi], bit = 1u << (key & 31u);
      if (word & bit) {
        Rec rc;
        rc.chunk = rch[2u * q + par];
        rc.link = lid;
        rc.t_start = t_start;
        TCHECK(base + wpre[wi] + __popc(word & (bit - 1u)) < job.rec_cap && q >= p_lo && q < p_hi, "send record");
        rec[base + wpre[wi] + __popc(word & (bit - 1u))] = rc;
      }
    }
    if (clear) {
      group_sync();
      for (uint32_t i = tid - first; i < nkw; i += count) bmp[i] = 0u;
    }
  };
  uint32_t rb = 0, rb_prev = 0;  // record offsets of the matches of events e and e-1 (cluster-wide)

  // pre_draw: Philox draws (R2) of every own link free at time tq, made ahead of the
  // event (t and busy_until are fixed by then; liveness is decided in PM after the
  // arrivals), kPB positions per pass so the Philox chains interleave.
  auto draw_ahead = [&](unsigned long long tq, uint32_t first, uint32_t stride) {
    constexpr int kPB = 4;
    for (uint32_t base = p_lo + first; base < p_hi; base += stride * kPB) {
      uint4 r[kPB];
#pragma unroll
      for (int u = 0; u < kPB; ++u) {
        const uint32_t q = base + (uint32_t)u * stride;
        r[u] = philox4x32_10(make_uint4((uint32_t)tq, (uint32_t)(tq >> 32), q < p_hi ? (uint32_t)t_lid[q] : 0u,
                                        job.sigma), seed_lo, seed_hi);
      }
#pragma unroll
      for (int u = 0; u < kPB; ++u) {
        const uint32_t q = base + (uint32_t)u * stride;
        if (q < p_hi && busy[q] <= tq) {
          ord[q] = r[u].x;
          pick[q] = r[u].y;
        }
      }
    }
  };
  if (pre_draw) {  // the draws of the first event (t = 0: every link is free)
    __syncthreads();
    draw_ahead(0ull, tid, nthr);
  }

  // ========================================================================================
  // Windowed event loop (lay.window = W > 0; wide rows on the register path, several link
  // costs, no relays).  Every arrival inside [T0, T0 + W), W <= the smallest link cost, comes
  // from a send that started before T0: a send started at t >= T0 ends at t + w >= T0 + W.
  // So at the window start T0 every event time of the window and every arrival at it are
  // known, and each destination can run all of the window's events on its own, in time
  // order, with one set of cluster barriers per window instead of per event:
  //   (1) event offsets of the window (own in-flight links; cluster OR of the bitmaps);
  //   (2) the sorted offsets (at most kWinEv; a longer window is cut at the next event);
  //   (3) all arrivals of the window applied to the held rows; each NPU's window arrivals
  //       (offset, chunk) listed (pushed to the CTAs that mirror it); per-event delivery
  //       counts summed over the cluster;
  //   (4) done test: the first event whose cumulative deliveries reach `required` ends the
  //       search there (no matching at it, as in the per-event loop);
  //   (5) per destination, per event t_k < done: free / live in-links at t_k, Philox draws
  //       (t_k, link, sigma), shorter-link-first ranks, the walk -- the source row at t_k is
  //       the row after the window's arrivals minus the source's arrivals later than t_k;
  //   (6) next window start = min busy_until of the links in flight (cluster MIN).
  // V / D / M / E are counted per event exactly as in the per-event loop; the source-change
  // versions count arrivals (hver[x] = arrivals at x before the window, plus its window
  // arrivals up to t_k).  Send records go to the destination's own record range
  // (Job::rec_off); emission sorts them by (t_start, link).
  // ========================================================================================
  bool windowed = false;
  if constexpr (REG_PATH && P > 2 && !MASKED) {
    if (lay.window != 0u) {
      windowed = true;
      uint32_t *w_bm = reinterpret_cast<uint32_t *>(smem + lay.off_wbm);
      uint32_t *w_ev = reinterpret_cast<uint32_t *>(smem + lay.off_wev);
      uint32_t *w_evc = reinterpret_cast<uint32_t *>(smem + lay.off_wevc);  // deliveries per event (cluster)
      uint32_t *w_evo = reinterpret_cast<uint32_t *>(smem + lay.off_wevo);  // own deliveries per event
      uint32_t *wa_cnt = reinterpret_cast<uint32_t *>(smem + lay.off_wacnt);
      uint32_t *wa_off = reinterpret_cast<uint32_t *>(smem + lay.off_waoff);
      uint16_t *wa_chk = reinterpret_cast<uint16_t *>(smem + lay.off_wachk);
      uint32_t *rcnt = s_list;  // records written per own destination
      const uint32_t Wwin = lay.window, DW = lay.win_deg, nbm = (Wwin + 31u) / 32u, kEv = lay.win_ev;
      const uint32_t *rec_off = job.rec_off;
      __shared__ uint32_t s_nev, s_wlim, s_kdone, s_wmin, s_wnext;
      __shared__ unsigned long long s_wdel;
      for (uint32_t i = tid; i < N; i += nthr) wa_cnt[i] = 0u;
      for (uint32_t i = tid; i < nbm; i += nthr) w_bm[i] = 0u;
      for (uint32_t i = tid; i < kWinEv; i += nthr) {
        w_evc[i] = 0u;
        w_evo[i] = 0u;
      }
      for (uint32_t i = d_lo + tid; i < d_hi; i += nthr) rcnt[i - d_lo] = 0u;
      if (tid == 0) s_dbg[1] = ~0u;
      cluster_barrier();  // peers push into our bitmap / lists from now on
      unsigned long long delivered = 0ull;  // cluster-wide deliveries before the window
      for (;;) {
        long long wts[9];  // debug (TACOS_TRACE): window phase timestamps, thread 0 of job 0
        const bool wtr = job.trace != nullptr && tid == 0;
        if (wtr) wts[0] = clock64();
        // ---- (1) event offsets of [t, t + W) ----
        for (uint32_t q = p_lo + tid; q < p_hi; q += nthr)
          if (cur[q] != kNone) {
            const unsigned long long off = busy[q] - t;
            if (off < Wwin) atomicOr(&w_bm[off >> 5], 1u << (off & 31u));
          }
        if (tid == 0) atomicOr(&w_bm[0], 1u);  // t itself
        if (Q > 1) {
          __syncthreads();
          for (uint32_t i = tid; i < nbm; i += nthr) {
            const uint32_t v = w_bm[i];
            if (v)
              for (uint32_t r = 0; r < Q; ++r)
                if (r != crank) dsmem_or_b32(dsmem_addr(&w_bm[i], r), v);
          }
        }
        if (wtr) wts[1] = clock64();
        cluster_barrier();
        if (wtr) wts[2] = clock64();
        // ---- (2) sorted offsets, the window limit (first offset left out) ----
        // warp 0: lane l takes the words [l cw, (l + 1) cw) (ascending offsets lane by lane), one
        // scan of the lane counts places every offset
        if (tid < 32) {
          const uint32_t cw = (nbm + 31u) / 32u, w0 = lane * cw, w1 = min(nbm, w0 + cw);
          uint32_t c = 0;
          for (uint32_t i = w0; i < w1; ++i) c += __popc(w_bm[i]);
          uint32_t incl = c;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= (uint32_t)o) incl += y;
          }
          const uint32_t n = __shfl_sync(0xFFFFFFFFu, incl, 31);
          if (lane == 0) {
            s_nev = n < kEv ? n : kEv;
            s_wlim = Wwin;
          }
          __syncwarp();
          uint32_t pos = incl - c;
          for (uint32_t i = w0; i < w1 && pos <= kEv; ++i)
            for (uint32_t m = w_bm[i]; m && pos <= kEv; m &= m - 1u, ++pos) {
              const uint32_t off = i * 32u + (uint32_t)(__ffs(m) - 1);
              if (pos < kEv) w_ev[pos] = off;
              else s_wlim = off;  // the first offset of the next window
            }
        }
        __syncthreads();
        if (wtr) wts[3] = clock64();
        const uint32_t n_ev = s_nev, wlim = s_wlim;
        for (uint32_t i = tid; i < nbm; i += nthr) w_bm[i] = 0u;  // peers write it again after (6)
        TCHECK(n_ev >= 1u && n_ev <= kEv && kEv <= kWinEv && w_ev[0] == 0u, "window events");
        // ---- (3) arrivals of the window ----
        {
          uint32_t arr = 0;
          for (uint32_t q = p_lo + tid; q < p_hi; q += nthr) {
            const uint32_t c = cur[q];
            if (c == kNone) continue;
            const unsigned long long off64 = busy[q] - t;
            if (off64 >= wlim) continue;
            const uint32_t off = (uint32_t)off64, d = t_dst[q];
            TCHECK(d < N && c < T.C, "window arrival");
            atomicOr(&held[(size_t)d * Wr + (c >> 5)], 1u << (c & 31u));
            const uint32_t j = atomicAdd(&wa_cnt[d], 1u);
            TCHECK(j < DW, "window arrivals per NPU");
            wa_off[d * DW + j] = off;
            wa_chk[d * DW + j] = (uint16_t)c;
            uint32_t lo = 0, hi = n_ev;  // event index of off (present in the list)
            while (lo < hi) {
              const uint32_t mid = (lo + hi) >> 1;
              if (w_ev[mid] < off) lo = mid + 1u;
              else hi = mid;
            }
            atomicAdd(&w_evo[lo], 1u);
            cur[q] = kNone;
            ++arr;
            if (Q > 1)
              for (uint32_t pm = s_peers[d]; pm; pm &= pm - 1u) {
                const uint32_t r = __ffs(pm) - 1u;
                if constexpr (ROWS_SMEM) dsmem_or_b32(dsmem_addr(&held[(size_t)d * Wr + (c >> 5)], r), 1u << (c & 31u));
                dsmem_st_u32(dsmem_addr(&wa_off[d * DW + j], r), off);
                dsmem_st_u16(dsmem_addr(&wa_chk[d * DW + j], r), (uint16_t)c);
                dsmem_add_u32(dsmem_addr(&wa_cnt[d], r), 1u);
              }
          }
          (void)arr;
          __syncthreads();
          for (uint32_t k = tid; k < n_ev; k += nthr) {  // per-event deliveries, summed over the cluster
            const uint32_t v = w_evo[k];
            if (v) {
              atomicAdd(&w_evc[k], v);
              for (uint32_t r = 0; r < Q; ++r)
                if (r != crank) dsmem_add_u32(dsmem_addr(&w_evc[k], r), v);
            }
          }
        }
        if (wtr) wts[4] = clock64();
        cluster_barrier();
        if (wtr) wts[5] = clock64();
        // ---- (4) done test inside the window ----
        if (tid < 32) {  // warp 0: cumulative deliveries per event (a scan per 32 events)
          unsigned long long acc = delivered;
          uint32_t kd = kNone;
          for (uint32_t b = 0; b < n_ev; b += 32u) {
            const uint32_t i = b + lane;
            const uint32_t v = i < n_ev ? w_evc[i] : 0u;
            uint32_t incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
              if (lane >= (uint32_t)o) incl += y;
            }
            const uint32_t hit = __ballot_sync(0xFFFFFFFFu, i < n_ev && acc + incl == T.required);
            if (hit && kd == kNone) kd = b + (uint32_t)(__ffs(hit) - 1);
            acc += __shfl_sync(0xFFFFFFFFu, incl, 31);
          }
          if (lane == 0) {
            s_kdone = kd;
            s_wdel = acc - delivered;
            s_wmin = ~0u;
            s_wnext = 0u;
          }
        }
        __syncthreads();
        const uint32_t k_done = s_kdone;
        const uint32_t n_run = k_done == kNone ? n_ev : k_done;
        E += n_run;
        if (wtr) wts[6] = clock64();
        const long long g_t0 = job.trace != nullptr ? clock64() : 0;  // debug: per-group phase time
        // ---- (5) destinations: every event of the window before done ----
        constexpr int SL = (kRegDeg + P - 1) / P;
        // destinations are taken from a shared counter, one group at a time: their costs differ
        // widely inside a window, and a static split left groups waiting at the barrier
        for (;;) {
          uint32_t wi = 0;
          if (gl == 0) wi = atomicAdd(&s_wnext, 1u);
          wi = __shfl_sync(gmask, wi, 0, P);
          if (wi >= d_hi - d_lo) break;
          const uint32_t d = d_lo + wi, b0 = s_inptr[d], b1 = s_inptr[d + 1], deg = b1 - b0;
          TCHECK(b0 >= p_lo && b1 <= p_hi && deg <= kRegDeg, "window destination");
          uint4 *have4 = reinterpret_cast<uint4 *>(have + (size_t)d * Wr);
          uint4 hv[V];
          bool hv_loaded = false;  // the have row (L2 with global rows) is read at the first live event
#if TACOS_WIN_EAGER_HAVE
#pragma unroll
          for (int v = 0; v < V; ++v) hv[v] = have4[v * P + gl];
          hv_loaded = true;
#endif
          const uint32_t rbase = rec != nullptr ? __ldg(&rec_off[d]) : 0u;  // issued early: an L2 round trip
          unsigned long long bq[SL];
          uint32_t sq[SL], srq[SL], hq[SL], nq[SL];
          // the first kWinReg window-arrival offsets of each slot's source, in registers (~0 = none)
          constexpr int kWinReg = 4;
          uint32_t ao[SL][kWinReg];
#pragma unroll
          for (int sl = 0; sl < SL; ++sl) {
            const uint32_t j = (uint32_t)sl * P + gl, q = b0 + j;
            const bool in = j < deg;
            bq[sl] = in ? busy[q] : ~0ull;
            sq[sl] = in ? seen[q] : 0u;
            srq[sl] = in ? (uint32_t)t_src[q] : 0u;
            hq[sl] = in ? hver[srq[sl]] : 0u;
            nq[sl] = in ? wa_cnt[srq[sl]] : 0u;
#pragma unroll
            for (int a = 0; a < kWinReg; ++a) ao[sl][a] = (uint32_t)a < nq[sl] ? wa_off[srq[sl] * DW + a] : ~0u;
          }
          uint32_t rc = rcnt[wi];
          bool any_claim = false;
          // Only the events at which this destination's state can change are run: an arrival
          // at d (an in-link frees) or at the source of an in-link (the source's row grows).  In
          // between, no in-link is live (each was matched, is busy or has an unchanged source
          // since its last empty visit), so those events only add the free-link count to V / D.
          uint32_t k = 0;
          while (k < n_run) {
            const uint32_t offk = w_ev[k];
            const unsigned long long tk = t + offk;
            unsigned long long key[SL];
            uint32_t pk[SL], ver[SL];
            uint32_t nfree = 0, nlive = 0;
#pragma unroll
            for (int sl = 0; sl < SL; ++sl) {
              key[sl] = ~0ull;
              pk[sl] = 0u;
              ver[sl] = hq[sl];
              const uint32_t j = (uint32_t)sl * P + gl;
              if (j < deg && bq[sl] <= tk) {
                ++nfree;
#pragma unroll
                for (int a = 0; a < kWinReg; ++a) ver[sl] += ao[sl][a] <= offk ? 1u : 0u;
                for (uint32_t a = kWinReg; a < nq[sl]; ++a) ver[sl] += wa_off[srq[sl] * DW + a] <= offk ? 1u : 0u;
                if (sq[sl] != ver[sl]) {
                  const uint32_t q = b0 + j;
                  const uint4 r = philox4x32_10(
                      make_uint4((uint32_t)tk, (uint32_t)(tk >> 32), t_lid[q], job.sigma), seed_lo, seed_hi);
                  key[sl] = ((unsigned long long)t_w[q] << 32) | r.x;  // (w, u_ord), R3
                  pk[sl] = r.y;
                  ++nlive;
                }
              }
            }
            {  // one group reduction for both counts (each <= kRegDeg)
              const uint32_t both = __reduce_add_sync(gmask, (nfree << 16) | nlive);
              nfree = both >> 16;
              nlive = both & 0xFFFFu;
            }
            if (gl == 0) {
              myV += nfree;
              myD += nfree ? 1u : 0u;
              myL += nlive;
              if (job.trace != nullptr) {  // debug: processed events, walked in-links
                atomicAdd(&s_dbg[2], 1u);
                atomicAdd(&s_dbg[3], nlive);
              }
            }
            const uint32_t rc_event = rc;
            if (nlive != 0u && !hv_loaded) {
#pragma unroll
              for (int v = 0; v < V; ++v) hv[v] = have4[v * P + gl];
              hv_loaded = true;
            }
            if (nlive != 0u) {
            uint32_t rk[SL];
#pragma unroll
            for (int sl = 0; sl < SL; ++sl) rk[sl] = 0u;
#pragma unroll
            for (int i = 0; i < kRegDeg; ++i) {
              const int isl = i / P, ilane = i % P;
              const unsigned long long ki = __shfl_sync(gmask, key[isl], ilane, P);
#pragma unroll
              for (int sl = 0; sl < SL; ++sl) {
                const uint32_t j = (uint32_t)sl * P + gl;
                rk[sl] += (ki < key[sl] || (ki == key[sl] && (uint32_t)i < j)) ? 1u : 0u;
              }
            }
#pragma unroll
            for (int sl = 0; sl < SL; ++sl) rk[sl] = key[sl] != ~0ull ? rk[sl] : 0xFFu;
            for (uint32_t s = 0; s < nlive; ++s) {
              // the in-link of rank s: its slot, pick draw and source version (owner lane broadcasts)
              uint32_t jj = 0, pp = 0, vv = 0;
              bool own = false;
#pragma unroll
              for (int sl = 0; sl < SL; ++sl) {
                const bool m = rk[sl] == s;
                own = own || m;
                jj = m ? (uint32_t)sl * P + gl : jj;
                pp = m ? pk[sl] : pp;
                vv = m ? ver[sl] : vv;
              }
              const int src_lane = __ffs(__ballot_sync(gmask, own)) - 1;
              jj = __shfl_sync(gmask, jj, src_lane);
              pp = __shfl_sync(gmask, pp, src_lane);
              vv = __shfl_sync(gmask, vv, src_lane);
              const uint32_t q = b0 + jj, sp = t_src[q];
              uint4 cv[V];
              const uint4 *h4 = reinterpret_cast<const uint4 *>(held + (size_t)sp * Wr);
#pragma unroll
              for (int v = 0; v < V; ++v) cv[v] = ROWS_SMEM ? h4[v * P + gl] : __ldcg(&h4[v * P + gl]);
              // the source's arrivals after t_k are not held yet at t_k
              const uint32_t na = wa_cnt[sp];
              for (uint32_t a = 0; a < na; ++a) {
                if (wa_off[sp * DW + a] <= offk) continue;
                const uint32_t c = wa_chk[sp * DW + a], wd = c >> 5, vec = wd >> 2;
                if (vec % P != gl) continue;
                const uint32_t vi = vec / P, comp = wd & 3u, nb = ~(1u << (c & 31u));
#pragma unroll
                for (int v = 0; v < V; ++v) {
                  if ((uint32_t)v != vi) continue;
                  cv[v].x &= comp == 0u ? nb : ~0u;
                  cv[v].y &= comp == 1u ? nb : ~0u;
                  cv[v].z &= comp == 2u ? nb : ~0u;
                  cv[v].w &= comp == 3u ? nb : ~0u;
                }
              }
              uint32_t incl[V], tot[V], K = 0;
#pragma unroll
              for (int v = 0; v < V; ++v) {
                cv[v] = andnot4(cv[v], hv[v]);  // held[src](t_k) & ~have[d]
                incl[v] = popc4(cv[v]);
#pragma unroll
                for (int o = 1; o < P; o <<= 1) {
                  const uint32_t y = __shfl_up_sync(gmask, incl[v], o, P);
                  if (gl >= (uint32_t)o) incl[v] += y;
                }
                tot[v] = __shfl_sync(gmask, incl[v], P - 1, P);
                K += tot[v];
              }
              const uint32_t osl = jj / P;  // slot of the in-link on its owner lane
              if (K == 0u) {  // exact skip from here on while the source is unchanged
                if (gl == jj % P) {
#pragma unroll
                  for (int sl = 0; sl < SL; ++sl)
                    if ((uint32_t)sl == osl) sq[sl] = vv;
                  seen[q] = vv;
                }
                continue;
              }
              uint32_t rv = __umulhi(pp, K);  // floor(u_pick * K / 2^32), R13
              int vsel = 0;
#pragma unroll
              for (int v = 0; v + 1 < V; ++v) {
                const bool adv = (vsel == v) && (rv >= tot[v]);
                rv = adv ? rv - tot[v] : rv;
                vsel = adv ? v + 1 : vsel;
              }
              uint4 x = cv[0];
              uint32_t inc = incl[0];
#pragma unroll
              for (int v = 1; v < V; ++v) {
                x = (vsel == v) ? cv[v] : x;
                inc = (vsel == v) ? incl[v] : inc;
              }
              const uint32_t cx = __popc(x.x), cy = __popc(x.y), cz = __popc(x.z);
              const uint32_t excl = inc - (cx + cy + cz + __popc(x.w));
              const bool mine = (rv >= excl) && (rv < inc);
              uint32_t rr = rv - excl, wsel = 0, word = x.x;
              bool m = rr >= cx;
              rr = m ? rr - cx : rr; wsel = m ? 1u : wsel; word = m ? x.y : word;
              m = m && rr >= cy;
              rr = m ? rr - cy : rr; wsel = m ? 2u : wsel; word = m ? x.z : word;
              m = m && rr >= cz;
              rr = m ? rr - cz : rr; wsel = m ? 3u : wsel; word = m ? x.w : word;
              const uint32_t bit = select_bit_swar(word, rr);
              const uint32_t mask = mine ? (1u << bit) : 0u;
#pragma unroll
              for (int v = 0; v < V; ++v) {
                if (vsel != v) continue;
                hv[v].x |= wsel == 0u ? mask : 0u;
                hv[v].y |= wsel == 1u ? mask : 0u;
                hv[v].z |= wsel == 2u ? mask : 0u;
                hv[v].w |= wsel == 3u ? mask : 0u;
              }
              uint32_t chunk = (((uint32_t)vsel * P + gl) * 4u + wsel) * 32u + bit;
              chunk = __shfl_sync(gmask, chunk, __ffs(__ballot_sync(gmask, mine)) - 1);
              TCHECK(chunk < T.C, "window claim");
              const uint32_t wp = t_w[q];
              if (gl == jj % P) {  // the slot's owner lane: link state
#pragma unroll
                for (int sl = 0; sl < SL; ++sl)
                  if ((uint32_t)sl == osl) bq[sl] = tk + wp;
                cur[q] = chunk;
                busy[q] = tk + wp;
              }
              if (gl == 0) {
                ++myM;
                if (rec != nullptr) {
                  TCHECK(rbase + rc < rec_off[d + 1], "window record");
                  Rec r;
                  r.chunk = chunk;
                  r.link = t_lid[q];
                  r.t_start = tk;
                  rec[rbase + rc] = r;
                }
              }
              ++rc;
              any_claim = true;
            }
            }  // nlive
            // the next event that can change this destination's state, and the free in-links
            // until then (this event's claims are busy now)
            const uint32_t nf = nfree - (rc - rc_event);  // every claim of this event took a free in-link
            // (a busy in-link matters again only when it frees -- its source's state is read
            // then -- so source arrivals count for the free in-links only)
            uint32_t nx = ~0u;
#pragma unroll
            for (int sl = 0; sl < SL; ++sl) {
              const uint32_t j = (uint32_t)sl * P + gl;
              if (j >= deg) continue;
              if (bq[sl] > tk) {
                const unsigned long long o = bq[sl] - t;
                if (o < wlim && (uint32_t)o < nx) nx = (uint32_t)o;
                continue;
              }
#pragma unroll
              for (int a = 0; a < kWinReg; ++a) {
                const uint32_t o = ao[sl][a];
                if (o > offk && o < nx) nx = o;
              }
              for (uint32_t a = kWinReg; a < nq[sl]; ++a) {
                const uint32_t o = wa_off[srq[sl] * DW + a];
                if (o > offk && o < nx) nx = o;
              }
            }
            nx = __reduce_min_sync(gmask, nx);
            uint32_t lo = k + 1u, hi = n_run;  // first event at or after offset nx
            while (lo < hi) {
              const uint32_t mid = (lo + hi) >> 1;
              if (w_ev[mid] < nx) lo = mid + 1u;
              else hi = mid;
            }
            if (gl == 0) {
              myV += (unsigned long long)nf * (lo - k - 1u);
              myD += nf ? (unsigned long long)(lo - k - 1u) : 0ull;
            }
            k = lo;
          }
          if (any_claim) {
#pragma unroll
            for (int v = 0; v < V; ++v) have4[v * P + gl] = hv[v];
            if (gl == 0) rcnt[wi] = rc;
          }
        }
        if (job.trace != nullptr && gl == 0) {
          atomicMax(&s_dbg[0], (unsigned)(clock64() - g_t0));
          atomicMin(&s_dbg[1], (unsigned)(clock64() - g_t0));
        }
        if (wtr) wts[7] = clock64();
        __syncthreads();
        // ---- (6) end of the window ----
        delivered += s_wdel;
        for (uint32_t x = tid; x < N; x += nthr) {
          const uint32_t a = wa_cnt[x];
          if (a) {
            hver[x] += a;
            wa_cnt[x] = 0u;
          }
        }
        for (uint32_t k = tid; k < n_ev; k += nthr) {
          w_evc[k] = 0u;
          w_evo[k] = 0u;
        }
        if (k_done != kNone) {
          t += w_ev[k_done];
          break;
        }
        // next window start: min busy_until over the links in flight (offsets < 2^32: w < 2^31)
        uint32_t mo = ~0u;
        for (uint32_t q = p_lo + tid; q < p_hi; q += nthr)
          if (cur[q] != kNone) {
            const uint32_t o = (uint32_t)(busy[q] - t);
            mo = o < mo ? o : mo;
          }
        mo = __reduce_min_sync(0xFFFFFFFFu, mo);
        if (lane == 0 && mo != ~0u) atomicMin(&s_wmin, mo);
        __syncthreads();
        if (Q > 1 && tid < Q) dsmem_st_u64(dsmem_addr(&s_slot_min2[0][crank], tid), (unsigned long long)s_wmin << 32);
        cluster_barrier();
        uint32_t mo_all = s_wmin;
        if (Q > 1) {
          mo_all = ~0u;
          for (uint32_t r = 0; r < Q; ++r) {
            const uint32_t hi = (uint32_t)(s_slot_min2[0][r] >> 32);
            mo_all = hi < mo_all ? hi : mo_all;
          }
        }
        if (mo_all == ~0u) {  // nothing in flight and not done: stall (R17)
          status = -3;
          break;
        }
        if (wtr && e % job.trace_stride == 0u && e / job.trace_stride < kTraceEvents) {
          wts[8] = clock64();
          unsigned long long *tr = job.trace + ((size_t)crank * kTraceEvents + e / job.trace_stride) * kTraceWords;
          tr[0] = t;
          tr[1] = n_ev;
          tr[2] = n_run;
          tr[3] = wlim;
          for (int i = 1; i < 9; ++i) tr[3 + i] = (unsigned long long)(wts[i] - wts[i - 1]);
          tr[12] = s_dbg[0];  // slowest group's destination phase
          tr[13] = s_dbg[1];  // fastest group's
          tr[14] = s_dbg[2];  // processed (destination, event) pairs of this CTA
          tr[15] = s_dbg[3];  // walked in-links
          tr[16] = 0;
          s_dbg[0] = s_dbg[2] = s_dbg[3] = 0u;
          s_dbg[1] = ~0u;
        }
        t += mo_all;
        if (t >= kMaxTime) {
          status = -6;
          break;
        }
        ++e;
      }
    }
  }

  unsigned long long ls_delivered = 0ull;  // lock-step loop: cluster-wide deliveries up to t
  if (!windowed)
  for (;;) {
    long long ts[9];  // debug phase timestamps (TACOS_TRACE), thread 0
    if (tracing) ts[0] = clock64();
    // ================= PA: arrivals at t =================
    if (tid == 0) {  // this event's counters (their parity was last read two events ago)
      s_min32[e & 1u] = ~0u;
      s_mcnt[e & 1u] = 0u;
    }
    if (worklist && tid == 0) s_nwork = 0u;  // read in PW, after the cluster barrier
    if (lockstep) {  // the arrivals at t are in held[e & 1] (written by the walkers of event e - 1)
      held = held_base + (size_t)(e & 1u) * N * Wr;
      hver = hver_base + (size_t)(e & 1u) * N;
    } else {
      uint32_t arr = 0;
      // one thread per in-link position: the arrival (a shared-memory atomicOr on the
      // destination's held row).  With pre_draw the Philox draws of this event were made
      // at the end of the previous one (draw_ahead); the records of event e-1 are written
      // during PM (write_records), away from the cluster barrier's fence.
      // kPA positions per pass: their link state is loaded before any arrival is applied
      // (the DSMEM pushes are asm volatile with memory clobbers, which would otherwise
      // serialize the loads of the next position behind them)
      constexpr int kPA = 5;
      for (uint32_t qb = p_lo + tid; qb < p_hi; qb += nthr * kPA) {
        uint32_t cq[kPA], dq[kPA], pq[kPA];
        bool arrq[kPA];
#pragma unroll
        for (int u = 0; u < kPA; ++u) {
          const uint32_t q = qb + (uint32_t)u * nthr;
          cq[u] = q < p_hi ? cur[q] : kNone;
          arrq[u] = cq[u] != kNone && busy[q] == t;  // R7: held by dst from this instant
          dq[u] = arrq[u] ? (uint32_t)t_dst[q] : 0u;
          pq[u] = (Q > 1 && arrq[u]) ? s_peers[dq[u]] : 0u;
        }
#pragma unroll
        for (int u = 0; u < kPA; ++u) {
          if (!arrq[u]) continue;
          const uint32_t q = qb + (uint32_t)u * nthr, c = cq[u], d = dq[u];
          TCHECK(d < N && c < T.C && q >= p_lo && q < p_hi, "arrival");
          atomicOr(&held[(size_t)d * Wr + (c >> 5)], 1u << (c & 31u));
          hver[d] = e;
          cur[q] = kNone;
          // push to the mirrors of d (ordered before the peers' reads by the cluster barrier)
          for (uint32_t pm = pq[u]; pm; pm &= pm - 1u) {
            const uint32_t r = __ffs(pm) - 1u;
            if constexpr (ROWS_SMEM) dsmem_or_b32(dsmem_addr(&held[(size_t)d * Wr + (c >> 5)], r), 1u << (c & 31u));
            dsmem_st_u32(dsmem_addr(&hver[d], r), e);
          }
          // a relayed chunk (not in post[d]) is held but not required
          if (!MASKED || ((__ldg(&T.post[(size_t)d * Wp + (c >> 5)]) >> (c & 31u)) & 1u)) ++arr;
        }
      }
      arr = warp_sum_u32(arr);
      if (lane == 0 && arr) atomicAdd(&s_arr[e & 1u], arr);  // own deliveries of this event
      if (Q > 1) {
        __syncthreads();
        if (tid < Q) dsmem_st_u64(dsmem_addr(&s_slot_deliv[crank], tid), s_delivered + s_arr[e & 1u]);
      }
    }
    if (tracing) ts[1] = clock64();
    if (!lockstep) cluster_barrier();
    if (tracing) ts[2] = clock64();
    unsigned long long delivered = lockstep ? ls_delivered : s_delivered + s_arr[e & 1u];  // own, cumulative
    if (Q > 1 && !lockstep) {
      delivered = 0;
      for (uint32_t r = 0; r < Q; ++r) delivered += s_slot_deliv[r];
    }
    if (delivered == T.required) {  // done test (postcondition holds)
      write_records(0u, nthr, e, rb_prev, t_prev, false);  // the last event's matches
      break;
    }
    ++E;

    // ================= PW (optional): worklist of destinations with a live in-link =================
    // For sparse events (heterogeneous costs free few links per event) the destination
    // phase then visits only the destinations that can match; V and D are counted here.
    uint32_t n_work = d_hi - d_lo;
    uint32_t mo_w = ~0u;  // min offset (busy - t) of own in-flight links (PW / walkers; else PE scans)
    if (worklist) {
      // one thread per own destination: free and live in-links (busy <= t; source changed since
      // the last empty visit), the min next-free offset of the busy ones; active destinations are
      // appended with warp-aggregated atomics (their order does not matter: destinations of one
      // event are independent and the records are ordered by the link-id bitmap)
      uint32_t nfree = 0, nd = 0;
      for (uint32_t i0 = 0; i0 < d_hi - d_lo; i0 += nthr) {
        const uint32_t i = i0 + tid;
        bool active = false;
        if (i < d_hi - d_lo) {
          const uint32_t d = d_lo + i, b0 = s_inptr[d], b1 = s_inptr[d + 1];
          uint32_t f = 0;
          if constexpr (REG_PATH) {  // in-degree <= kRegDeg: every slot's state loaded up front
            unsigned long long bq[kRegDeg];
            uint32_t sq[kRegDeg], srq[kRegDeg];
#pragma unroll
            for (int j = 0; j < kRegDeg; ++j) {
              const uint32_t q = b0 + (uint32_t)j;
              const bool in = q < b1;
              bq[j] = in ? busy[q] : ~0ull;
              sq[j] = in ? seen[q] : 0u;
              srq[j] = in ? (uint32_t)t_src[q] : 0u;
            }
#pragma unroll
            for (int j = 0; j < kRegDeg; ++j) {
              const bool in = b0 + (uint32_t)j < b1;
              if (in && bq[j] <= t) {
                ++f;
                active = active || sq[j] != hver_of(srq[j]);
              } else if (in) {
                mo_w = (uint32_t)(bq[j] - t) < mo_w ? (uint32_t)(bq[j] - t) : mo_w;
              }
            }
          } else {
            for (uint32_t q = b0; q < b1; ++q) {
              const unsigned long long bq = busy[q];
              if (bq <= t) {
                ++f;
                active = active || seen[q] != hver_of(t_src[q]);
              } else {
                mo_w = (uint32_t)(bq - t) < mo_w ? (uint32_t)(bq - t) : mo_w;
              }
            }
          }
          nfree += f;
          nd += f ? 1u : 0u;
        }
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, active);
        uint32_t base = 0;
        if (lane == 0 && bal) base = atomicAdd(&s_nwork, (uint32_t)__popc(bal));
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
        TCHECK(!active || base + __popc(bal & ((1u << lane) - 1u)) < d_hi - d_lo, "worklist");
        if (active) s_list[base + __popc(bal & ((1u << lane) - 1u))] = d_lo + i;
      }
      myV += nfree;
      myD += nd;
      __syncthreads();
      n_work = s_nwork;
    }
    if (tracing) ts[3] = clock64();

    // ================= PM: per-destination draws, order and matching =================
    // threads beyond the destination groups write the records of event e-1 meanwhile
    const uint32_t pm_thr = min(nthr, (n_work * P + 31u) & ~31u);
    const long long pm_t0 = job.trace != nullptr ? clock64() : 0;  // debug: slowest thread of the phase
    uint32_t my_claims = 0;  // this event's matches of this thread (published with the next time)
    // one-thread register path: the walker also takes the minimum next-free offset of its in-links
    // (busy beyond t, or claimed now), so PE needs no second pass over the link state
    constexpr bool kWalkMin = REG_PATH && P == 1 && kP1Smem;
    if (tid >= pm_thr) {
      write_records(pm_thr, nthr - pm_thr, e, rb_prev, t_prev, true);
      if (job.trace != nullptr) atomicMax(&s_dbg[1], (unsigned)(clock64() - pm_t0));
    }
    {
      uint32_t *bm = bitmap2 + (e & 1u) * nbw;
      for (uint32_t wi = tid / P; wi < n_work; wi += ngroups) {
        const uint32_t d = worklist ? s_list[wi] : d_lo + wi;
        const uint32_t b0 = s_inptr[d], b1 = s_inptr[d + 1];
        const uint32_t deg = b1 - b0;
        TCHECK(d >= d_lo && d < d_hi && b0 >= p_lo && b1 <= p_hi && b0 <= b1, "destination range");
        uint4 *have4 = reinterpret_cast<uint4 *>(have + (size_t)d * Wr);
        uint4 hv[V];
        uint32_t pmask = 0;  // lock-step loop: matched in-link slots of d (bit p - b0)

        // One step of the matching walk (a5) on in-link position p with pick draw pk.
        // held[src] row of in-link p into registers (own shared memory, a peer's via DSMEM, or L2)
        auto load_row = [&](uint32_t p, uint4 (&cv)[V]) {
          const uint32_t sp = t_src[p];
          TCHECK(sp < N && p >= p_lo && p < p_hi, "walk row");
          // Row chunk order is vector-major: vector v of lane gl holds words (v*P + gl)*4 .. +3.
          const uint4 *h4 = reinterpret_cast<const uint4 *>(held + (size_t)sp * Wr);
          if (!ROWS_SMEM) {  // rows in HBM/L2, written by other SMs of the cluster: L2-coherent loads
#pragma unroll
            for (int v = 0; v < V; ++v) cv[v] = __ldcg(&h4[v * P + gl]);
          } else {  // shared-memory rows: own, or a peer's mirrored copy (pushed in PA)
#pragma unroll
            for (int v = 0; v < V; ++v) cv[v] = h4[v * P + gl];
          }
        };
        // One lane per destination (P == 1): the per-word counts of the candidate row are kept
        // for the selection (vector -> word -> bit), and the bit select runs without POPC.
        auto step_row1 = [&](uint32_t p, uint32_t pk, uint4 (&cv)[V]) {
          uint32_t wd[4 * V], pc[4 * V], vt[V];
          uint32_t K = 0;
#pragma unroll
          for (int v = 0; v < V; ++v) {
            if constexpr (kHaveSmem) cv[v] = andnot4(cv[v], have4[v]);  // held[src] & ~have[d]
            else cv[v] = andnot4(cv[v], hv[v]);
            if constexpr (MASKED)  // & allow[p]: post[d] plus the relays of this link
              cv[v] = and4(cv[v], __ldg(reinterpret_cast<const uint4 *>(T.allow + (size_t)p * Wp) + v));
            wd[4 * v + 0] = cv[v].x;
            wd[4 * v + 1] = cv[v].y;
            wd[4 * v + 2] = cv[v].z;
            wd[4 * v + 3] = cv[v].w;
          }
#pragma unroll
          for (int i = 0; i < 4 * V; ++i) pc[i] = __popc(wd[i]);
#pragma unroll
          for (int v = 0; v < V; ++v) {
            vt[v] = (pc[4 * v] + pc[4 * v + 1]) + (pc[4 * v + 2] + pc[4 * v + 3]);
            K += vt[v];
          }
          if (K == 0u) {
            seen[p] = hver_of(t_src[p]);
            return;
          }
          uint32_t rv = __umulhi(pk, K);  // floor(u_pick * K / 2^32)
          uint32_t vsel = 0;
#pragma unroll
          for (int v = 0; v + 1 < V; ++v) {
            const bool adv = (vsel == (uint32_t)v) && (rv >= vt[v]);
            rv = adv ? rv - vt[v] : rv;
            vsel = adv ? (uint32_t)v + 1u : vsel;
          }
          uint32_t q0 = pc[0], q1 = pc[1], q2 = pc[2];
          uint4 x = cv[0];
#pragma unroll
          for (int v = 1; v < V; ++v) {
            const bool m = vsel == (uint32_t)v;
            q0 = m ? pc[4 * v] : q0;
            q1 = m ? pc[4 * v + 1] : q1;
            q2 = m ? pc[4 * v + 2] : q2;
            x = m ? cv[v] : x;
          }
          uint32_t wi = 0, word = x.x;
          bool m = rv >= q0;
          rv = m ? rv - q0 : rv; wi = m ? 1u : wi; word = m ? x.y : word;
          m = m && rv >= q1;
          rv = m ? rv - q1 : rv; wi = m ? 2u : wi; word = m ? x.z : word;
          m = m && rv >= q2;
          rv = m ? rv - q2 : rv; wi = m ? 3u : wi; word = m ? x.w : word;
          const uint32_t bit = select_bit_swar(word, rv);
          const uint32_t mask = 1u << bit;
          // claim: withheld from d's other in-links (R4)
          if constexpr (kHaveSmem) {
            reinterpret_cast<uint32_t *>(have4)[vsel * 4u + wi] |= mask;  // one word, dynamic index
          } else {
            const uint32_t sel = vsel * 4u + wi;  // flat word index: independent predicated ORs
#pragma unroll
            for (int v = 0; v < V; ++v) {
              hv[v].x |= sel == (uint32_t)(4 * v + 0) ? mask : 0u;
              hv[v].y |= sel == (uint32_t)(4 * v + 1) ? mask : 0u;
              hv[v].z |= sel == (uint32_t)(4 * v + 2) ? mask : 0u;
              hv[v].w |= sel == (uint32_t)(4 * v + 3) ? mask : 0u;
            }
          }
          const uint32_t chunk = (vsel * 4u + wi) * 32u + bit;
          TCHECK(chunk < T.C && t_lid[p] < L, "claimed chunk");
          if (!lockstep) cur[p] = chunk;  // (the lock-step loop has no arrival phase)
          rch[2u * p + (e & 1u)] = (uint16_t)chunk;
          const uint32_t wp = t_w[p];
          busy[p] = t + wp;
          mo_w = wp < mo_w ? wp : mo_w;
          ++myM;
          ++my_claims;
          if (lockstep) {  // position bits, set once per destination after the walk (in-degree <= 32)
            if (REG_PATH || deg <= 32u) pmask |= 1u << (p - b0);  // (register path: in-degree <= 8)
            else atomicOr(&bm[(p - p_lo) >> 5], 1u << ((p - p_lo) & 31u));
          } else {
            const uint32_t lid = t_lid[p];
            atomicOr(&bm[lid >> 5], 1u << (lid & 31u));
          }
        };

        // One step of the matching walk (a5) on in-link p, pick draw pk, loaded row cv.
        auto step_row = [&](uint32_t p, uint32_t pk, uint4 (&cv)[V]) {
#if TACOS_STEP1
          if constexpr (P == 1) {
            step_row1(p, pk, cv);
            return;
          }
#endif
          uint32_t incl[V], tot[V];
          uint32_t K = 0;
#pragma unroll
          for (int v = 0; v < V; ++v) {
            if constexpr (kHaveSmem) cv[v] = andnot4(cv[v], have4[v * P + gl]);  // held[src] & ~have[d]
            else cv[v] = andnot4(cv[v], hv[v]);
            if constexpr (MASKED)  // & allow[p]: post[d] plus the relays of this link
              cv[v] = and4(cv[v], __ldg(reinterpret_cast<const uint4 *>(T.allow + (size_t)p * Wp) + v * P + gl));
            incl[v] = popc4(cv[v]);
#pragma unroll
            for (int o = 1; o < P; o <<= 1) {
              const uint32_t y = __shfl_up_sync(gmask, incl[v], o, P);
              if (gl >= (uint32_t)o) incl[v] += y;
            }
            tot[v] = (P > 1) ? __shfl_sync(gmask, incl[v], P - 1, P) : incl[v];
            K += tot[v];
          }
          if (K == 0u) {
            if (gl == 0) seen[p] = hver_of(t_src[p]);
            return;
          }
          const uint32_t r = __umulhi(pk, K);  // floor(u_pick * K / 2^32)
          // vector holding the r-th candidate, rank inside it
          uint32_t rv = r;
          int vsel = 0;
#pragma unroll
          for (int v = 0; v + 1 < V; ++v) {
            const bool adv = (vsel == v) && (rv >= tot[v]);
            rv = adv ? rv - tot[v] : rv;
            vsel = adv ? v + 1 : vsel;
          }
          uint4 x = cv[0];
          uint32_t inc = incl[0];
#pragma unroll
          for (int v = 1; v < V; ++v) {
            x = (vsel == v) ? cv[v] : x;
            inc = (vsel == v) ? incl[v] : inc;
          }
          const uint32_t cx = __popc(x.x), cy = __popc(x.y), cz = __popc(x.z);
          const uint32_t excl = inc - (cx + cy + cz + __popc(x.w));
          const bool mine = (rv >= excl) && (rv < inc);
          uint32_t rr = rv - excl;
          // word inside the lane's vector, branch-free
          uint32_t wi = 0, word = x.x;
          bool m = rr >= cx;
          rr = m ? rr - cx : rr; wi = m ? 1u : wi; word = m ? x.y : word;
          m = m && rr >= cy;
          rr = m ? rr - cy : rr; wi = m ? 2u : wi; word = m ? x.z : word;
          m = m && rr >= cz;
          rr = m ? rr - cz : rr; wi = m ? 3u : wi; word = m ? x.w : word;
          const uint32_t bit = select_bit(word, rr);
          const uint32_t mask = mine ? (1u << bit) : 0u;
          // claim: withheld from d's other in-links (R4)
          if constexpr (kHaveSmem) {
            reinterpret_cast<uint32_t *>(have4)[(uint32_t)vsel * 4u + wi] |= mask;  // one word, dynamic index
          } else {
            const uint32_t sel = (uint32_t)vsel * 4u + wi;  // flat word index: independent predicated ORs
#pragma unroll
            for (int v = 0; v < V; ++v) {
              hv[v].x |= sel == (uint32_t)(4 * v + 0) ? mask : 0u;
              hv[v].y |= sel == (uint32_t)(4 * v + 1) ? mask : 0u;
              hv[v].z |= sel == (uint32_t)(4 * v + 2) ? mask : 0u;
              hv[v].w |= sel == (uint32_t)(4 * v + 3) ? mask : 0u;
            }
          }
          uint32_t chunk = (((uint32_t)vsel * P + gl) * 4u + wi) * 32u + bit;
          if (P > 1) chunk = __shfl_sync(gmask, chunk, __ffs(__ballot_sync(gmask, mine)) - 1);
          TCHECK(chunk < T.C && t_lid[p] < L, "claimed chunk");
          if (gl == 0) {
            cur[p] = chunk;
            rch[2u * p + (e & 1u)] = (uint16_t)chunk;
            const uint32_t wp = t_w[p];
            busy[p] = t + wp;
            mo_w = wp < mo_w ? wp : mo_w;
            ++myM;
            ++my_claims;
            const uint32_t lid = t_lid[p];
            atomicOr(&bm[lid >> 5], 1u << (lid & 31u));
          }
        };

        auto step = [&](uint32_t p, uint32_t pk) {
          uint4 cv[V];
          load_row(p, cv);
          step_row(p, pk, cv);
        };

        // REG_PATH (every in-degree <= kRegDeg): ranks in registers; else shared memory
        // lock-step loop: d's held row at the next event = have[d] after the walk (at t every
        // earlier send has arrived, so have == held; the claims of t arrive at t + w, the next
        // event), written to the other held buffer and pushed to the CTAs that mirror d
        auto ls_push = [&](bool arrived) {
          const uint32_t nb = (e + 1u) & 1u;
          uint4 *hn = reinterpret_cast<uint4 *>(held_base + ((size_t)nb * N + d) * Wr);
          uint32_t *hvn = hver_base + (size_t)nb * N + d;
          uint4 r[V];
#pragma unroll
          for (int v = 0; v < V; ++v) r[v] = have4[v];
#pragma unroll
          for (int v = 0; v < V; ++v) hn[v] = r[v];
          const uint32_t ver = arrived ? e + 1u : hver[d];
          *hvn = ver;
          if (Q > 1)
            for (uint32_t pm = s_peers[d]; pm; pm &= pm - 1u) {
              const uint32_t rk = __ffs(pm) - 1u;
#pragma unroll
              for (int v = 0; v < V; ++v) dsmem_st_v4(dsmem_addr(hn + v, rk), r[v]);
              dsmem_st_u32(dsmem_addr(hvn, rk), ver);
            }
        };
        // lock-step loop: this event's matched positions (bit q - p_lo of the CTA's position
        // bitmap; in-degree > 32 sets them per match): the records are written in position order,
        // ranked by link at emission
        auto ls_positions = [&]() {
          const uint32_t o = b0 - p_lo, sh = o & 31u;
          if (pmask) atomicOr(&bm[o >> 5], pmask << sh);
          if (sh != 0u && (pmask >> (32u - sh)) != 0u) atomicOr(&bm[(o >> 5) + 1u], pmask >> (32u - sh));
        };
        if constexpr (REG_PATH && P == 1 && kP1Smem) {
          // ---- one thread per destination: in-link j in slot j (static), ranks by pairwise
          //      comparisons, walk order packed 4 bits per rank, and the next in-link's source
          //      row loaded while the current one is matched.  The slot count is specialised:
          //      D = 6 (15 comparisons, e.g. every 3-D torus) or 8 (28) ----
          uint32_t nfree = 0, nlive = 0, ordp = 0;  // ordp: slot of rank s in bits [4s, 4s + 4)
          auto prologue = [&](auto degc) {
            constexpr int D = decltype(degc)::value;
            unsigned long long key[D];
            uint32_t o32[D];
            // the link state of every slot is loaded before any draw, so the loads of later
            // slots do not wait behind the Philox chains of earlier ones
            uint32_t live = 0;  // bit j: slot j is live
            {
              unsigned long long bq[D];
              uint32_t sq[D], srq[D];
#pragma unroll
              for (int j = 0; j < D; ++j) {
                const uint32_t q = b0 + (uint32_t)j;
                const bool in = (uint32_t)j < deg;
                bq[j] = in ? busy[q] : ~0ull;
                sq[j] = in ? seen[q] : 0u;
                srq[j] = in ? (uint32_t)t_src[q] : 0u;
              }
#pragma unroll
              for (int j = 0; j < D; ++j) {
                const bool in = (uint32_t)j < deg;
                const bool isfree = in && bq[j] <= t;
                if (in && !isfree) mo_w = (uint32_t)(bq[j] - t) < mo_w ? (uint32_t)(bq[j] - t) : mo_w;
                nfree += isfree ? 1u : 0u;
                if (isfree && sq[j] != hver_of(srq[j])) live |= 1u << j;
              }
            }
            uint32_t wlo = ~0u, whi = 0u;
            bool ord_max = false;  // a live u_ord of 2^32 - 1 (then the 32-bit keys could tie a dead slot)
#pragma unroll
            for (int j = 0; j < D; ++j) {
              key[j] = ~0ull;
              o32[j] = ~0u;
              if ((live >> j) & 1u) {
                const uint32_t q = b0 + (uint32_t)j;
                uint32_t o;
                if (pre_draw) {
                  o = ord[q];
                } else {
                  const uint4 r = philox4x32_10(
                      make_uint4((uint32_t)t, (uint32_t)(t >> 32), t_lid[q], job.sigma), seed_lo, seed_hi);
                  o = r.x;
                  pick[q] = r.y;
                }
                ++nlive;
                const uint32_t wq = t_w[q];
                wlo = wq < wlo ? wq : wlo;
                whi = wq > whi ? wq : whi;
                ord_max = ord_max || o == ~0u;
                o32[j] = o;
                key[j] = ((unsigned long long)wq << 32) | o;  // (w, u_ord), R3
              }
            }
            if (nlive == 0u) return;
            // rank of slot j = #{i : key_i < key_j or (key_i == key_j and i < j)}; dead keys (~0,
            // above every live key: w < 2^32 - 1 is enforced on the host) rank last.  With one
            // cost among the live slots the order is that of u_ord alone (32-bit compares).
            uint32_t rk[D];
#pragma unroll
            for (int j = 0; j < D; ++j) rk[j] = 0u;
            if (wlo == whi && !ord_max) {
#pragma unroll
              for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = i + 1; j < D; ++j) {
                  const bool jfirst = o32[j] < o32[i];
                  rk[i] += jfirst ? 1u : 0u;
                  rk[j] += jfirst ? 0u : 1u;
                }
            } else {
#pragma unroll
              for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = i + 1; j < D; ++j) {
                  const bool jfirst = key[j] < key[i];
                  rk[i] += jfirst ? 1u : 0u;
                  rk[j] += jfirst ? 0u : 1u;
                }
            }
#pragma unroll
            for (int j = 0; j < D; ++j) ordp |= (uint32_t)j << (4u * rk[j]);
          };
          const uint32_t claims0 = my_claims;
          if (deg <= 6u) prologue(std::integral_constant<int, 6>());
          else prologue(std::integral_constant<int, kRegDeg>());
          if (!worklist) {
            myV += nfree;
            myD += nfree ? 1u : 0u;
          }
          if (gl == 0) myL += nlive;
          if (nlive == 0u) {
            if (lockstep) ls_push(false);
            continue;
          }
          const long long dbg_pro = job.trace != nullptr ? clock64() : 0;  // debug (TACOS_TRACE)
          uint4 nxt[V];
          if constexpr (!kHaveSmem) {
#pragma unroll
            for (int v = 0; v < V; ++v) hv[v] = have4[v];
          }
          load_row(b0 + (ordp & 15u), nxt);
          uint32_t pk_nxt = pick[b0 + (ordp & 15u)];  // the pick draw travels with the row prefetch
          for (uint32_t s = 0; s < nlive; ++s) {
            const uint32_t p = b0 + ((ordp >> (4u * s)) & 15u);
            uint4 cv[V];
#pragma unroll
            for (int v = 0; v < V; ++v) cv[v] = nxt[v];
            const uint32_t pk = pk_nxt;
            if (s + 1u < nlive) {
              const uint32_t pn = b0 + ((ordp >> (4u * s + 4u)) & 15u);
              load_row(pn, nxt);
              pk_nxt = pick[pn];
            }
            step_row(p, pk, cv);
          }
          if (job.trace != nullptr) {
            atomicMax(&s_dbg[2], (unsigned)(dbg_pro - pm_t0));
            atomicMax(&s_dbg[3], (unsigned)(clock64() - dbg_pro));
            atomicMax(&s_dbg[4], nlive);
          }
          if constexpr (!kHaveSmem) {
#pragma unroll
            for (int v = 0; v < V; ++v) have4[v] = hv[v];
          }
          if (lockstep) {
            ls_push(my_claims != claims0);
            ls_positions();
          }
        } else if constexpr (REG_PATH && P <= 2) {
          // ---- a group of P lanes per destination: every lane ranks the in-links itself
          //      (redundant, no shuffles); the row is split lane-major (lane gl holds the
          //      vectors gl*V .. gl*V+V-1, chunks in ascending order across the lanes), so a
          //      step needs one inclusive scan of the lane counts; the lane holding the r-th
          //      candidate claims it and writes the link; the next in-link's row is loaded
          //      while the current one is matched ----
          unsigned long long key[kRegDeg];
          uint32_t nfree = 0, nlive = 0;
#if TACOS_P2_SPLIT_DRAWS
          if constexpr (P == 2) {
            // the two lanes split the draws (slot j drawn by lane j & 1) and exchange u_ord
            uint32_t live = 0, od[kRegDeg];
#pragma unroll
            for (int j = 0; j < kRegDeg; ++j) {
              od[j] = 0u;
              if ((uint32_t)j < deg) {
                const uint32_t q = b0 + (uint32_t)j;
                const bool isfree = busy[q] <= t;
                const bool islive = isfree && seen[q] != hver_of(t_src[q]);
                nfree += isfree ? 1u : 0u;
                if (islive) {
                  live |= 1u << j;
                  if (pre_draw) {
                    od[j] = ord[q];
                  } else if ((uint32_t)(j & 1) == gl) {
                    const uint4 r = philox4x32_10(
                        make_uint4((uint32_t)t, (uint32_t)(t >> 32), t_lid[q], job.sigma), seed_lo, seed_hi);
                    od[j] = r.x;
                    pick[q] = r.y;
                  }
                }
              }
            }
#pragma unroll
            for (int j = 0; j < kRegDeg; ++j) {
              const uint32_t o = pre_draw ? od[j] : __shfl_sync(gmask, od[j], j & 1, P);
              key[j] = ((live >> j) & 1u) ? (((unsigned long long)t_w[b0 + (uint32_t)j] << 32) | o) : ~0ull;
            }
            nlive = __popc(live);
          } else
#endif
#pragma unroll
          for (int j = 0; j < kRegDeg; ++j) {
            key[j] = ~0ull;
            if ((uint32_t)j < deg) {
              const uint32_t q = b0 + (uint32_t)j;
              const bool isfree = busy[q] <= t;
              const bool islive = isfree && seen[q] != hver_of(t_src[q]);
              nfree += isfree ? 1u : 0u;
              if (islive) {
                uint32_t o;
                if (pre_draw) {
                  o = ord[q];
                } else {
                  const uint4 r = philox4x32_10(
                      make_uint4((uint32_t)t, (uint32_t)(t >> 32), t_lid[q], job.sigma), seed_lo, seed_hi);
                  o = r.x;
                  if (gl == 0) pick[q] = r.y;
                }
                ++nlive;
                key[j] = ((unsigned long long)t_w[q] << 32) | o;  // (w, u_ord), R3
              }
            }
          }
          if (gl == 0 && !worklist) {
            myV += nfree;
            myD += nfree ? 1u : 0u;
          }
          if (gl == 0) myL += nlive;
          if (nlive == 0u) continue;
          uint32_t rk[kRegDeg];
#pragma unroll
          for (int j = 0; j < kRegDeg; ++j) rk[j] = 0u;
#pragma unroll
          for (int i = 0; i < kRegDeg; ++i)
#pragma unroll
            for (int j = i + 1; j < kRegDeg; ++j) {
              const bool jfirst = key[j] < key[i];
              rk[i] += jfirst ? 1u : 0u;
              rk[j] += jfirst ? 0u : 1u;
            }
          uint32_t ordp = 0;
#pragma unroll
          for (int j = 0; j < kRegDeg; ++j) ordp |= (uint32_t)j << (4u * rk[j]);
          auto load_half = [&](uint32_t pp, uint4 (&cv)[V]) {
            const uint32_t sp = t_src[pp];
            const uint4 *h4 = reinterpret_cast<const uint4 *>(held + (size_t)sp * Wr);
            if (!ROWS_SMEM) {
#pragma unroll
              for (int v = 0; v < V; ++v) cv[v] = __ldcg(&h4[gl * V + v]);
            } else {  // own or mirrored row
#pragma unroll
              for (int v = 0; v < V; ++v) cv[v] = h4[gl * V + v];
            }
          };
          uint4 hl[V];
#pragma unroll
          for (int v = 0; v < V; ++v) hl[v] = have4[gl * V + v];
          uint4 nxt[V];
          load_half(b0 + (ordp & 15u), nxt);
          if (!pre_draw) __syncwarp(gmask);  // lane 0's pick draws visible to lane 1
          for (uint32_t s = 0; s < nlive; ++s) {
            const uint32_t pp = b0 + ((ordp >> (4u * s)) & 15u);
            uint4 cv[V];
#pragma unroll
            for (int v = 0; v < V; ++v) cv[v] = nxt[v];
            if (s + 1u < nlive) load_half(b0 + ((ordp >> (4u * s + 4u)) & 15u), nxt);
            uint32_t tot[V], k = 0;
#pragma unroll
            for (int v = 0; v < V; ++v) {
              cv[v] = andnot4(cv[v], hl[v]);  // held[src] & ~have[d], this lane's half
              if constexpr (MASKED)
                cv[v] = and4(cv[v], __ldg(reinterpret_cast<const uint4 *>(T.allow + (size_t)pp * Wp) + gl * V + v));
              tot[v] = popc4(cv[v]);
              k += tot[v];
            }
            uint32_t incl = k;  // inclusive scan of the lane counts over the group
#pragma unroll
            for (int o = 1; o < P; o <<= 1) {
              const uint32_t y = __shfl_up_sync(gmask, incl, o, P);
              if (gl >= (uint32_t)o) incl += y;
            }
            const uint32_t K = P > 1 ? __shfl_sync(gmask, incl, P - 1, P) : incl;
            if (K == 0u) {
              if (gl == 0u) seen[pp] = hver_of(t_src[pp]);
              continue;
            }
            const uint32_t r = __umulhi(pick[pp], K);  // floor(u_pick * K / 2^32), R13
            const uint32_t excl = incl - k;
            const bool mine = r >= excl && r < incl;
            uint32_t rv = r - excl;
            int vsel = 0;
#pragma unroll
            for (int v = 0; v + 1 < V; ++v) {
              const bool adv = (vsel == v) && (rv >= tot[v]);
              rv = adv ? rv - tot[v] : rv;
              vsel = adv ? v + 1 : vsel;
            }
            uint4 x = cv[0];
#pragma unroll
            for (int v = 1; v < V; ++v) x = (vsel == v) ? cv[v] : x;
            const uint32_t cx = __popc(x.x), cy = __popc(x.y), cz = __popc(x.z);
            uint32_t rr = rv, wi = 0, word = x.x;
            bool m = rr >= cx;
            rr = m ? rr - cx : rr; wi = m ? 1u : wi; word = m ? x.y : word;
            m = m && rr >= cy;
            rr = m ? rr - cy : rr; wi = m ? 2u : wi; word = m ? x.z : word;
            m = m && rr >= cz;
            rr = m ? rr - cz : rr; wi = m ? 3u : wi; word = m ? x.w : word;
            const uint32_t bit = select_bit(word, rr);
            const uint32_t mask = mine ? (1u << bit) : 0u;
#pragma unroll
            for (int v = 0; v < V; ++v) {
              if (vsel == v) {
                hl[v].x |= wi == 0u ? mask : 0u;
                hl[v].y |= wi == 1u ? mask : 0u;
                hl[v].z |= wi == 2u ? mask : 0u;
                hl[v].w |= wi == 3u ? mask : 0u;
              }
            }
            if (mine) {  // claim (R4): the owning lane writes the link
              const uint32_t chunk = ((((uint32_t)(gl * V) + (uint32_t)vsel) * 4u + wi) * 32u) + bit;
              TCHECK(chunk < T.C && pp >= p_lo && pp < p_hi, "claimed chunk (lane pair)");
              cur[pp] = chunk;
              rch[2u * pp + (e & 1u)] = (uint16_t)chunk;
              const uint32_t wp = t_w[pp];
              busy[pp] = t + wp;
              mo_w = wp < mo_w ? wp : mo_w;
              ++myM;
              ++my_claims;
              const uint32_t lid = t_lid[pp];
              atomicOr(&bm[lid >> 5], 1u << (lid & 31u));
            }
          }
#pragma unroll
          for (int v = 0; v < V; ++v) have4[gl * V + v] = hl[v];
        } else if constexpr (REG_PATH) {
          // ---- register path for wide rows (P > 2, measured faster there than the lane-major
          //      group path): the group owns the destination's <= kRegDeg in-links, in-link j
          //      in slot j / P of lane j % P; ranks and the walk order stay in registers ----
          constexpr int SL = (kRegDeg + P - 1) / P;  // slots per lane
          // the destination's have row (L2 when the rows live in global memory) is loaded
          // first, so its latency overlaps the draws and the ranking
#pragma unroll
          for (int v = 0; v < V; ++v) if (!kHaveSmem) hv[v] = have4[v * P + gl];
          unsigned long long key[SL];
          uint32_t pk[SL];
          uint32_t nfree = 0, nlive = 0;
#pragma unroll
          for (int sl = 0; sl < SL; ++sl) {
            key[sl] = ~0ull;
            pk[sl] = 0u;
            const uint32_t j = (uint32_t)sl * P + gl;
            if (j < deg) {
              const uint32_t q = b0 + j;
              bool isfree, islive;
              uint32_t o = 0;
              if (pre_draw) {  // draws made in PA; liveness needs the arrivals of PA
                isfree = busy[q] <= t;
                islive = isfree && seen[q] != hver_of(t_src[q]);
                if (islive) {
                  o = ord[q];
                  pk[sl] = pick[q];
                }
              } else {
                isfree = busy[q] <= t;
                islive = isfree && seen[q] != hver_of(t_src[q]);
                if (islive) {
                  const uint4 r = philox4x32_10(
                      make_uint4((uint32_t)t, (uint32_t)(t >> 32), t_lid[q], job.sigma), seed_lo, seed_hi);
                  o = r.x;
                  pk[sl] = r.y;
                }
              }
              nfree += isfree ? 1u : 0u;
              if (islive) {
                ++nlive;
                key[sl] = ((unsigned long long)t_w[q] << 32) | o;  // (w, u_ord), R3
              }
            }
          }
          if (P > 1) {
            nfree = __reduce_add_sync(gmask, nfree);
            nlive = __reduce_add_sync(gmask, nlive);
          }
          if (gl == 0 && !worklist) {
            myV += nfree;
            myD += nfree ? 1u : 0u;
          }
          if (gl == 0) myL += nlive;
          if (nlive == 0u) continue;
          // ranks among live in-links by (w, u_ord, position); positions ascend with link id.
          // Non-live keys are ~0 > every live key (w < 2^32 - 1 is enforced on the host).
          uint32_t rk[SL];
#pragma unroll
          for (int sl = 0; sl < SL; ++sl) rk[sl] = 0u;
#pragma unroll
          for (int i = 0; i < kRegDeg; ++i) {
            const int isl = i / P, ilane = i % P;
            const unsigned long long ki =
                (P > 1) ? __shfl_sync(gmask, key[isl], ilane, P) : key[isl];
#pragma unroll
            for (int sl = 0; sl < SL; ++sl) {
              const uint32_t j = (uint32_t)sl * P + gl;
              rk[sl] += (ki < key[sl] || (ki == key[sl] && (uint32_t)i < j)) ? 1u : 0u;
            }
          }
#pragma unroll
          for (int sl = 0; sl < SL; ++sl) rk[sl] = key[sl] != ~0ull ? rk[sl] : 0xFFu;
          // walk order: in-link of rank s (owning lane broadcasts position and pick draw)
          auto link_of_rank = [&](uint32_t s, uint32_t &jj, uint32_t &pp) {
            jj = 0;
            pp = 0;
            bool own = false;
#pragma unroll
            for (int sl = 0; sl < SL; ++sl) {
              const bool m = rk[sl] == s;
              own = own || m;
              jj = m ? (uint32_t)sl * P + gl : jj;
              pp = m ? pk[sl] : pp;
            }
            if (P > 1) {
              const int src_lane = __ffs(__ballot_sync(gmask, own)) - 1;
              jj = __shfl_sync(gmask, jj, src_lane);
              pp = __shfl_sync(gmask, pp, src_lane);
            }
          };
#if TACOS_WIDE_PREFETCH
          // the next in-link's source row is loaded while the current one is matched
          uint32_t jj, pp;
          link_of_rank(0u, jj, pp);
          uint4 nxt[V];
          load_row(b0 + jj, nxt);
          for (uint32_t s = 0; s < nlive; ++s) {
            const uint32_t pc = b0 + jj, pkc = pp;
            uint4 cv[V];
#pragma unroll
            for (int v = 0; v < V; ++v) cv[v] = nxt[v];
            if (s + 1u < nlive) {
              link_of_rank(s + 1u, jj, pp);
              load_row(b0 + jj, nxt);
            }
            step_row(pc, pkc, cv);
          }
#else
          for (uint32_t s = 0; s < nlive; ++s) {
            uint32_t jj, pp;
            link_of_rank(s, jj, pp);
            step(b0 + jj, pp);
          }
#endif
#pragma unroll
          for (int v = 0; v < V; ++v) if (!kHaveSmem) have4[v * P + gl] = hv[v];
        } else {
        // ---- shared-memory path: per-position draws, ranks and order ----
        uint32_t nfree = 0, nl = 0;
        for (uint32_t q = b0 + gl; q < b1; q += P) {
          unsigned char f;
          if (pre_draw) {  // draws made in PA
            f = busy[q] <= t ? (seen[q] != hver_of(t_src[q]) ? 2 : 1) : 0;
            lv[q] = f;
          } else {
            f = 0;
            if (busy[q] <= t) {  // free: nothing in flight on it
              f = 1;
              // exact skip: K stays 0 while src is unchanged since its last empty visit
              if (seen[q] != hver_of(t_src[q])) {
                const uint4 r = philox4x32_10(
                    make_uint4((uint32_t)t, (uint32_t)(t >> 32), t_lid[q], job.sigma), seed_lo, seed_hi);
                ord[q] = r.x;
                pick[q] = r.y;
                f = 2;
              }
            }
            lv[q] = f;
          }
          nfree += f ? 1u : 0u;
          if (P == 1 && f == 2) order[b0 + nl] = (uint16_t)(q - b0);  // one lane: compact list of the live in-links
          nl += f == 2 ? 1u : 0u;
        }
        if (P > 1) {
          nfree = __reduce_add_sync(gmask, nfree);
          nl = __reduce_add_sync(gmask, nl);
        }
        if (gl == 0 && !worklist) {
          myV += nfree;
          myD += nfree ? 1u : 0u;
        }
        if (gl == 0) myL += nl;
        if (nl == 0u) {
          if (lockstep) ls_push(false);
          continue;
        }
        if constexpr (P == 1) {
          const uint32_t claims0 = my_claims;
          // one lane per destination: the walk takes the live in-links in shorter-link-first order
          // (R3: smallest (w, u_ord, position) first, positions ascend with the link id) by a
          // selection over the compact live list -- O(live^2) instead of O(live x in-degree)
#pragma unroll
          for (int v = 0; v < V; ++v) if (!kHaveSmem) hv[v] = have4[v];
          for (uint32_t s = 0; s < nl; ++s) {
            uint32_t bi = s, bp = b0 + order[b0 + s];
            unsigned long long bk = ((unsigned long long)t_w[bp] << 32) | ord[bp];
            for (uint32_t i = s + 1; i < nl; ++i) {
              const uint32_t qi = b0 + order[b0 + i];
              const unsigned long long ki = ((unsigned long long)t_w[qi] << 32) | ord[qi];
              const bool better = ki < bk || (ki == bk && qi < bp);
              bi = better ? i : bi;
              bp = better ? qi : bp;
              bk = better ? ki : bk;
            }
            if (bi != s) {
              const uint16_t tmp = order[b0 + s];
              order[b0 + s] = order[b0 + bi];
              order[b0 + bi] = tmp;
            }
            step(bp, pick[bp]);
          }
#pragma unroll
          for (int v = 0; v < V; ++v) if (!kHaveSmem) have4[v] = hv[v];
          if (lockstep) {
            ls_push(my_claims != claims0);
            ls_positions();
          }
          continue;
        }
        if (P > 1) __syncwarp(gmask);
        // shorter-link-first order of the live in-links (R3): rank by (w, u_ord, link)
        for (uint32_t q = b0 + gl; q < b1; q += P) {
          if (lv[q] != 2) continue;
          const uint32_t wq = t_w[q], oq = ord[q];
          uint32_t rank = 0;
          for (uint32_t u = b0; u < b1; ++u) {
            if (lv[u] != 2) continue;
            const uint32_t wu = t_w[u], ou = ord[u];
            // positions of a destination are in ascending link id: u < q <=> lid_u < lid_q
            rank += (wu < wq) || (wu == wq && (ou < oq || (ou == oq && u < q)));
          }
          order[b0 + rank] = (uint16_t)(q - b0);
        }
        if (P > 1) __syncwarp(gmask);
#pragma unroll
        for (int v = 0; v < V; ++v) if (!kHaveSmem) hv[v] = have4[v * P + gl];
        for (uint32_t s = 0; s < nl; ++s) {
          const uint32_t p = b0 + order[b0 + s];
          step(p, pick[p]);
        }
#pragma unroll
        for (int v = 0; v < V; ++v) if (!kHaveSmem) have4[v * P + gl] = hv[v];
        }
      }
    }
    if (job.trace != nullptr && tid < pm_thr) atomicMax(&s_dbg[0], (unsigned)(clock64() - pm_t0));
    if (pm_thr == nthr) write_records(0u, nthr, e, rb_prev, t_prev, true);
    my_claims = __reduce_add_sync(0xFFFFFFFFu, my_claims);
    if (lane == 0 && my_claims) atomicAdd(&s_mcnt[e & 1u], my_claims);
    // lock-step loop: the walkers' minimum next-free offset joins the same block barrier
    if (lockstep) {
      const uint32_t mo = __reduce_min_sync(0xFFFFFFFFu, mo_w);
      if (lane == 0 && mo != ~0u) atomicMin(&s_min32[e & 1u], mo);
    }
    if (tracing) ts[4] = clock64();
    __syncthreads();
    if (tracing) ts[5] = clock64();
    if (tid == 0) {  // every thread has read this event's arrivals (done test, publication)
      s_delivered += s_arr[e & 1u];
      s_arr[e & 1u] = 0u;
    }

    // ================= PE: next event time, this event's match count =================
    {
      uint32_t *bm = bitmap2 + (e & 1u) * nbw;
      // publish: own matched links into the peers' bitmaps; own min busy_until (as an offset
      // from t, < 2^32) and own match count into every CTA's slot
      if (Q > 1 && !lockstep) {
        for (uint32_t i = tid; i < nbw; i += nthr) {
          const uint32_t wbits = bm[i];
          if (wbits)
            for (uint32_t r = 0; r < Q; ++r)
              if (r != crank) dsmem_or_b32(dsmem_addr(bm + i, r), wbits);
        }
      }
      // (with the worklist only the active destinations were walked: full pass)
      const bool walk_min = kWalkMin || worklist;
      uint32_t mo = walk_min ? mo_w : ~0u;
      if (!walk_min && !lockstep)
      for (uint32_t p = p_lo + tid; p < p_hi; p += nthr)
        if (cur[p] != kNone) {
          const uint32_t o = (uint32_t)(busy[p] - t);
          mo = o < mo ? o : mo;
        }
      if (!lockstep) {
        mo = __reduce_min_sync(0xFFFFFFFFu, mo);
        if (lane == 0 && mo != ~0u) atomicMin(&s_min32[e & 1u], mo);
        __syncthreads();
      }
      if (Q > 1 && tid < Q)
        dsmem_st_u64(dsmem_addr(&s_slot_min2[e & 1u][crank], tid),
                     ((unsigned long long)s_min32[e & 1u] << 32) | s_mcnt[e & 1u]);
      if (tracing) ts[6] = clock64();
      if (Q > 1) cluster.sync();
      if (tracing) ts[7] = clock64();
    }
    uint32_t mo_all = s_min32[e & 1u], m_all = s_mcnt[e & 1u], m_lower = 0u;
    if (Q > 1) {
      mo_all = ~0u;
      m_all = 0u;
      for (uint32_t r = 0; r < Q; ++r) {
        const unsigned long long v = s_slot_min2[e & 1u][r];
        const uint32_t hi = (uint32_t)(v >> 32);
        mo_all = hi < mo_all ? hi : mo_all;
        m_all += (uint32_t)v;
        if (r < crank) m_lower += (uint32_t)v;  // matches of the lower cluster ranks at this event
      }
    }
    const unsigned long long tn = mo_all == ~0u ? ~0ull : t + mo_all;
    rb_prev = lockstep ? rb + m_lower : rb;  // lock-step: this CTA's first record of the event
    rb += m_all;
    if (lockstep) ls_delivered += m_all;  // AG without relays: every send is a delivery at t + w
    if (pre_draw && tn != ~0ull) draw_ahead(tn, tid, nthr);  // (optional) the next event's draws
    if (tracing && e % job.trace_stride == 0u && e / job.trace_stride < kTraceEvents) {
      ts[8] = clock64();
      unsigned long long *tr = job.trace + ((size_t)crank * kTraceEvents + e / job.trace_stride) * kTraceWords;
      tr[0] = t;
      tr[1] = delivered;
      tr[2] = tn;
      tr[3] = m_all;
      for (int i = 1; i < 9; ++i) tr[3 + i] = (unsigned long long)(ts[i] - ts[i - 1]);
      tr[12] = s_dbg[0];
      tr[13] = s_dbg[1];
      tr[14] = s_dbg[2];
      tr[15] = s_dbg[3];
      tr[16] = s_dbg[4];
      s_dbg[0] = s_dbg[1] = s_dbg[2] = s_dbg[3] = s_dbg[4] = 0u;
    }
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
  myL = warp_sum_u64(myL);
  if (lane == 0) {
    if (myV) atomicAdd(&s_V, myV);
    if (myD) atomicAdd(&s_D, myD);
    if (myM) atomicAdd(&s_M, myM);
    if (myL) atomicAdd(&s_L, myL);
  }
  __syncthreads();
  if (Q > 1) {
    if (tid == 0) {
      const uint32_t a = dsmem_addr(&s_slot_cnt[crank][0], 0);
      dsmem_st_u64(a, s_V);
      dsmem_st_u64(a + 8u, s_D);
      dsmem_st_u64(a + 16u, s_M);
      dsmem_st_u64(a + 24u, s_L);
    }
    cluster.sync();  // also keeps every CTA's shared memory alive until the peers are done with it
    if (tid == 0 && crank == 0) {
      s_V = s_D = s_M = s_L = 0ull;
      for (uint32_t r = 0; r < Q; ++r) {
        s_V += s_slot_cnt[r][0];
        s_D += s_slot_cnt[r][1];
        s_M += s_slot_cnt[r][2];
        s_L += s_slot_cnt[r][3];
      }
    }
  }
  if (tid == 0 && crank == 0) {
    JobOut o;
    o.T = t;
    o.V = s_V;
    o.D = s_D;
    o.M = s_M;
    o.E = E;
    o.Lv = s_L;
    o.status = status;
    o.pad = 0;
    outs[job.out_slot] = o;
  }
}

template <int P, int V, bool R, bool K, bool G, bool M = false, bool B = false>
int launch_greedy_one(const Layout &lay, const Job *d_jobs, uint32_t n_jobs, JobOut *d_outs, cudaStream_t st) {
  auto fn = greedy_kernel<P, V, R, K, G, M, B>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lay.smem_bytes);
  // clusters beyond the portable 8 CTAs (B200: up to 16) are opt-in per kernel
  if (e == cudaSuccess && lay.cluster > 8u) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  // all of the unified L1 / shared array as shared memory (the kernels stage their state there;
  // global row loads bypass L1 with ld.cg), so several CTAs can be resident when they fit
  if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) {
    snprintf(cuda_error_buffer(), 256, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return -4;
  }
  const uint32_t Q = lay.cluster ? lay.cluster : 1u;
  if (g_occ_query) {  // occupancy query (plan build): co-resident clusters / CTAs, no launch
    int n = 0;
    if (Q > 1) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(n_jobs * Q, 1, 1);
      cfg.blockDim = dim3(lay.threads, 1, 1);
      cfg.dynamicSmemBytes = lay.smem_bytes;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = Q;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) n = 0;
    } else {
      int b = 0, dev = 0, sms = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, (int)lay.threads, lay.smem_bytes) == cudaSuccess) n = b * sms;
    }
    cudaGetLastError();
    *g_occ_query = n;
    return 0;
  }
  if (Q > 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(n_jobs * Q, 1, 1);
    cfg.blockDim = dim3(lay.threads, 1, 1);
    cfg.dynamicSmemBytes = lay.smem_bytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = Q;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (getenv("TACOS_DEBUG_OCC")) {  // debug: co-resident clusters of this shape
      int ncl = -1;
      cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg);
      fprintf(stderr, "tacos: cluster %u x %u threads, %u B smem: max active clusters %d (jobs %u)\n", Q, lay.threads,
              lay.smem_bytes, ncl, n_jobs);
    }
    e = cudaLaunchKernelEx(&cfg, fn, d_jobs, d_outs, lay);
    if (e != cudaSuccess) {
      snprintf(cuda_error_buffer(), 256, "cudaLaunchKernelEx (cluster %u): %s", Q, cudaGetErrorString(e));
      cudaGetLastError();
      return -4;
    }
  } else {
    fn<<<n_jobs, lay.threads, lay.smem_bytes, st>>>(d_jobs, d_outs, lay);
  }
  return check_launch("greedy_kernel");
}

template <int P, int V>
int launch_greedy_pv(const Layout &lay, const Job *d_jobs, uint32_t n_jobs, JobOut *d_outs, cudaStream_t st) {
  if (lay.masked) {  // relays: shared-memory ranking path only
    if (lay.rows_in_smem && lay.links_in_smem) return launch_greedy_one<P, V, true, true, false, true>(lay, d_jobs, n_jobs, d_outs, st);
    if (lay.links_in_smem) return launch_greedy_one<P, V, false, true, false, true>(lay, d_jobs, n_jobs, d_outs, st);
    return launch_greedy_one<P, V, false, false, false, true>(lay, d_jobs, n_jobs, d_outs, st);
  }
  if (lay.reg_path) {
    if constexpr (P == 1 && V == 4)
      if (lay.big && lay.rows_in_smem && lay.links_in_smem)
        return launch_greedy_one<P, V, true, true, true, false, true>(lay, d_jobs, n_jobs, d_outs, st);
    if (lay.rows_in_smem && lay.links_in_smem) return launch_greedy_one<P, V, true, true, true>(lay, d_jobs, n_jobs, d_outs, st);
    if (lay.links_in_smem) return launch_greedy_one<P, V, false, true, true>(lay, d_jobs, n_jobs, d_outs, st);
    return launch_greedy_one<P, V, false, false, true>(lay, d_jobs, n_jobs, d_outs, st);
  }
  if (lay.rows_in_smem && lay.links_in_smem) return launch_greedy_one<P, V, true, true, false>(lay, d_jobs, n_jobs, d_outs, st);
  if (lay.links_in_smem) return launch_greedy_one<P, V, false, true, false>(lay, d_jobs, n_jobs, d_outs, st);
  return launch_greedy_one<P, V, false, false, false>(lay, d_jobs, n_jobs, d_outs, st);
}

// One translation unit per P (greedy_p<P>.cu) instantiates these.
template <int P>
int launch_greedy_p(const Layout &lay, uint32_t V, const Job *d_jobs, uint32_t n_jobs, JobOut *d_outs,
                    cudaStream_t st) {
  switch (V) {
    case 1: return launch_greedy_pv<P, 1>(lay, d_jobs, n_jobs, d_outs, st);
    case 2: return launch_greedy_pv<P, 2>(lay, d_jobs, n_jobs, d_outs, st);
    case 4: return launch_greedy_pv<P, 4>(lay, d_jobs, n_jobs, d_outs, st);
    default:
      snprintf(cuda_error_buffer(), 256, "unsupported vectors per lane %u", V);
      return -1;
  }
}

int launch_greedy_p1(const Layout &, uint32_t, const Job *, uint32_t, JobOut *, cudaStream_t);
int launch_greedy_p2(const Layout &, uint32_t, const Job *, uint32_t, JobOut *, cudaStream_t);
int launch_greedy_p4(const Layout &, uint32_t, const Job *, uint32_t, JobOut *, cudaStream_t);
int launch_greedy_p8(const Layout &, uint32_t, const Job *, uint32_t, JobOut *, cudaStream_t);
int launch_greedy_p16(const Layout &, uint32_t, const Job *, uint32_t, JobOut *, cudaStream_t);
int launch_greedy_p32(const Layout &, uint32_t, const Job *, uint32_t, JobOut *, cudaStream_t);

}  // namespace tacos
