// tacos_internal.h -- shared between the host runtime (tacos_api.cpp) and the
// CUDA kernels (tacos_kernels.cu).  Product side only; the oracle never
// includes this file.
#pragma once
#include <cstdint>
#include <cstddef>

namespace tacos {

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr int kKeySeedBits = 20;              // best key = (T << 20) | global seed index
constexpr unsigned long long kNoKey = 0x7FFFFFFFFFFFFFFFull;  // no finished seed (also max as int64)
constexpr uint64_t kMaxTime = 1ull << 40;     // T must stay below 2^40 time units
constexpr int kMaxVPL = 4;                    // uint4 vectors per lane: C <= 32*4*32*4 = 16384
constexpr uint32_t kMaxChunks = 32u * 4u * 32u * kMaxVPL;

// Topology as the kernels see it, for one orientation sigma (0 = G, 1 = G^T).
// Positions p index the links grouped by destination (CSR): in-links of d are
// positions in_ptr[d] .. in_ptr[d+1]-1, in ascending link id.
struct DevTopo {
  uint32_t N, L, C, k;
  uint32_t Wp;       // padded words per row = 4 * P * VPL
  uint32_t P, VPL;   // lanes per destination, uint4 vectors per lane
  uint32_t custom;   // 1: pre/post rows given
  uint32_t max_deg;  // maximum in-degree
  uint64_t required; // deliveries needed
  const uint32_t *in_ptr; // [N+1]
  const uint32_t *p_src;  // [L] source NPU of position p
  const uint32_t *p_dst;  // [L]
  const uint32_t *p_w;    // [L] cost in time units
  const uint32_t *p_lid;  // [L] link id (input index)
  const uint32_t *pre;    // [N*Wp] custom only
  const uint32_t *post;   // [N*Wp] custom only
  const uint32_t *allow;  // [L*Wp] relays only (R22): chunks position p may carry, else nullptr
  const uint32_t *npu_orig;  // [N] original id of kernel NPU x when the plan relabels NPUs, else nullptr
};

// Compact send record written by the search (16 B): ordered by (t_start, link)
// within a job.
struct Rec {
  uint32_t chunk, link;
  uint64_t t_start;
};

struct Job {
  const DevTopo *topo;   // device pointer
  uint64_t seed;
  uint32_t sigma;
  uint32_t out_slot;
  const uint32_t *rec_off;  // windowed loop: records of destination d at [rec_off[d], rec_off[d+1])
  Rec *rec;              // nullptr: recording off
  uint64_t rec_cap;      // records the job may write (bounds-checked build)
  uint32_t *g_rows;      // global rows (held | have) when they do not fit in smem
  unsigned char *g_links;// global per-position arrays when they do not fit in smem
  unsigned long long *trace;  // debug (TACOS_TRACE): per CTA rank, per event {t, delivered, local min, matches}
  uint32_t trace_stride;      // debug: trace every trace_stride-th event (TACOS_TRACE_STRIDE, default 1)
};
constexpr uint32_t kTraceEvents = 4096;
constexpr uint32_t kTraceWords = 17;  // t, delivered, t_next, matches, 8 phase durations, slowest PM / record thread

struct JobOut {
  uint64_t T, V, D, M, E;
  uint64_t Lv;  // live visits: free links whose candidate row was read (the others were skipped exactly)
  int32_t status;
  uint32_t pad;
};
constexpr uint32_t kSmallWords = 16;  // per part: keys[2], stats {V, D, M, E, status, X, Lv}

// Byte offsets of the per-block arrays, either in dynamic shared memory or in
// the job's global scratch (rows / links regions).
struct Layout {
  uint32_t rows_bytes;   // 2*N*row_stride*4 (held then have)
  uint32_t row_stride;   // words between consecutive rows in shared memory (Wp, padded)
  uint32_t links_bytes;  // per-position arrays
  // within the links region
  uint32_t off_busy, off_cur, off_ord, off_pick, off_seen, off_order, off_lv, off_rch;
  uint32_t off_tsrc, off_tw, off_tlid, off_tdst;  // per-position topology copies (src, w, link id, dst)
  // always in shared memory, after [rows][links] when those are resident
  uint32_t off_hver, off_bitmap, off_wpre, off_inptr, off_act, off_list, off_peers;  // bitmap: 2 x ceil(L/32) words (event parity)
  uint32_t smem_bytes;   // total dynamic smem
  uint32_t rows_in_smem, links_in_smem;
  uint32_t threads;
  uint32_t pre_draw;     // 1: draws per position by all threads before the destination phase
  uint32_t cluster;      // CTAs per job (thread-block cluster size), 1 = one CTA per job
  uint32_t reg_path;     // 1: every in-degree <= 8 (register ranking path)
  uint32_t worklist;     // 1: compact the destinations with a live in-link before matching
  uint32_t masked;       // 1: relays (R22): candidates & allow[p], only required arrivals count
  // windowed event loop (greedy_window.cuh): window length W in time units (0 = one event per
  // iteration), max in-degree, and its shared-memory arrays (after the others)
  uint32_t window, win_deg, win_ev;  // win_ev: events per window at most (<= kWinEv; TACOS_WIN_EV)
  uint32_t off_wbm, off_wev, off_wevc, off_wevo, off_wacnt, off_waoff, off_wachk;
  // lock-step event loop (one link cost, one lane per destination): held rows
  // double-buffered by event parity (held[2][N], then the own have rows), link state of the
  // CTA's own in-link positions only (pos_cap per CTA), hver[2][N]
  uint32_t lockstep, pos_cap;
  // 1: the one-lane four-vector register-path kernel with the larger thread bound (kBigThreads)
  uint32_t big;
};
constexpr uint32_t kMaxCluster = 16;  // CTAs per job at most (non-portable cluster sizes above 8)
constexpr uint32_t kWinEv = 256;      // events per window at most (a longer window is cut there)
constexpr uint32_t kWinBits = 16384;  // window length cap (bitmap of event offsets)
// Append the windowed loop's shared-memory arrays to a layout (window = W, deg = max in-degree).
void add_window(Layout &lay, uint32_t N, uint32_t window, uint32_t deg);
// Switch a one-lane shared-memory layout to the lock-step loop's (pos_cap = the most in-link
// positions a CTA of the cluster owns); false (layout unchanged) when it does not fit.
bool add_lockstep(Layout &lay, uint32_t N, uint32_t L, uint32_t pos_cap, size_t smem_limit);
// The larger-bound kernel exists for the register path with on-chip state only: otherwise back
// to the default bound.
void layout_drop_big(Layout &lay);

// q_force: cluster size to use (0: the automatic choice; TACOS_CLUSTER overrides both)
Layout make_layout(uint32_t N, uint32_t L, uint32_t Wp, uint32_t P, uint32_t VPL, size_t smem_limit, uint32_t n_jobs,
                   uint32_t n_sms, uint32_t q_force = 0);
// When set, launch_greedy writes the number of co-resident clusters (CTAs when Q = 1) of the
// kernel the layout selects into *g_occ_query and launches nothing.
extern thread_local int *g_occ_query;

// ---- kernel launch wrappers (tacos_kernels.cu) ----
int launch_greedy(const Layout &lay, uint32_t P, uint32_t VPL, const Job *d_jobs, uint32_t n_jobs, JobOut *d_outs, void *stream);
int launch_best_keys(const JobOut *d_outs, uint32_t n_seeds, uint32_t seed_offset, uint32_t rs_base,
                     uint32_t has_rs, uint64_t *d_keys, uint64_t *d_stats, uint64_t *d_times_ag,
                     uint64_t *d_times_rs, void *stream);
// Winner resolved on the device from the (possibly all-reduced) best keys, so the emitters
// can follow the search without a host round trip: keys == nullptr = the host passed rec / T.
struct DevWin {
  const unsigned long long *keys;  // keys[0]: (T << 20) | global seed index
  const Rec *rec_base;             // records of job 0 of the plan part
  uint64_t cap;                    // records per job
  uint32_t seed_offset, n_seeds;   // the shard's global seed range
  uint32_t shift_by_T;             // emit_ag: shift the sends by the key's T (AR on a symmetric graph)
};
int launch_emit_ag(const Rec *rec, uint64_t M, const uint32_t *src, const uint32_t *dst, const uint32_t *w,
                   uint64_t shift, void *out_sends, void *stream, uint64_t limit = ~0ull, const DevWin *dw = nullptr);
int launch_compact_sends(void *sends, uint64_t n, unsigned long long *d_count, void *stream);
int launch_rs_sort_emit(const Rec *rec, uint64_t M, const uint32_t *src, const uint32_t *dst, const uint32_t *w,
                        const int32_t *rev, uint64_t T_rs, uint32_t L, void *out_sends, void *scratch,
                        size_t scratch_bytes, uint32_t *launches, void *stream, uint32_t mirror = 1,
                        uint64_t shift = 0);
int launch_rs_uniform_emit(const Rec *rec, uint64_t M, const uint32_t *src, const uint32_t *dst, uint32_t w0,
                           const int32_t *rev, uint64_t T_rs, uint32_t L, void *out_sends, void *scratch,
                           size_t scratch_bytes, uint32_t *launches, void *stream, const DevWin *dw = nullptr,
                           uint32_t mirror = 1);
int launch_literal(const Layout &lay, uint32_t VPL, const Job *d_jobs, uint32_t n_jobs, JobOut *d_outs, void *stream);
size_t rs_sort_scratch_bytes(uint64_t M);
int launch_philox_probe(const uint32_t *d_in, uint32_t *d_out, void *stream);

const char *cuda_error_string();

}  // namespace tacos
