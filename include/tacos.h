/*
 * tacos.h -- C ABI of libtacos.so, the B200-native TACOS-Greedy synthesizer.
 *
 * Method: TACOS-Greedy (Won et al., arXiv 2304.05301).  Citations are
 * "P:L<n>" = /root/reference/PAPER.md line n (LaTeX source), with the paper
 * section, and "R<n>" = the readings listed in DESIGN.md §3.
 *
 *   - A topology is a directed graph of NPUs with alpha-beta link costs
 *     (§II.C "alpha + beta * n"; §IV.A base graph G = (V, E)).
 *   - A collective is a pre/postcondition over (NPU, chunk) pairs (§II.A).
 *   - tacos_synthesize runs the greedy link-chunk matching over the implicit
 *     time-expanded network (§VI.A, Fig. GreedyMatching;
 *     shorter-link-first and arrival-time rules P:L263-267 §VI.B) for a batch
 *     of seeds, keeps the best one (§VI.C "initiating multiple
 *     independent search instances concurrently and choose the best"), and
 *     derives Reduce-Scatter by inversion and All-Reduce as RS followed by AG
 *     (§VII.A; §II.A).
 *   - tacos_eval replays a schedule and checks it (§IV.B: a
 *     collective algorithm is a set of TEN links each matched with a chunk).
 *
 * Conventions (whole ABI):
 *   - Every function returns TACOS_OK (0) or a negative tacos_status.  No C++
 *     exception crosses the ABI.  tacos_last_error() gives a thread-local
 *     one-line detail of the last failure on the calling thread.
 *   - Out-parameters (`*out`) are written only on success; on failure they
 *     are set to NULL when they are handle pointers.
 *   - All input arrays are copied; the caller keeps ownership of them.
 *   - Handles are immutable after creation and may be shared between threads
 *     (distinct handles are fully independent).  Output arrays belong to the
 *     handle and stay valid until the handle is freed.
 *   - Time is integer, in units of time_unit_ns (R5).  Bandwidth is integer
 *     bytes per ns (= decimal GB/s, R6).  A send on link l occupies
 *     [t_start, t_start + w_l) (R8) with
 *         w_l = ceil((alpha_l * bw_l + chunk_bytes) / (bw_l * time_unit_ns))
 *     (P:L104 delay alpha + n/bw; §IV.C discretization ceil(l/f)).
 *   - Chunks: C = N * chunks_per_npu for AG/RS/AR, chunk c = owner*k + j
 *     (R12).  Bitsets are rows of ceil(C/32) uint32 words per NPU, chunk c at
 *     bit (c & 31) of word (c >> 5).
 *   - The CUDA path runs on the current CUDA device of the calling thread.
 *     There is no CPU fallback: without a usable sm_100 device the synthesis
 *     entry points return TACOS_E_CUDA.
 */
#ifndef TACOS_H
#define TACOS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TACOS_ABI_VERSION 1

typedef enum {
  TACOS_OK = 0,
  TACOS_E_INVALID_ARG = -1, /* null pointer, N < 2, k < 1, n = 0, S < 1, bad collective ... */
  TACOS_E_TOPOLOGY = -2,    /* self-loop, duplicate (src,dst) pair, id out of range, bw = 0, w = 0 */
  TACOS_E_UNREACHABLE = -3, /* G not strongly connected (AG/RS/AR) or greedy stall (CUSTOM, R17) */
  TACOS_E_CUDA = -4,        /* CUDA runtime error or no usable device */
  TACOS_E_NOMEM = -5,       /* host or device allocation failed */
  TACOS_E_OVERFLOW = -6,    /* w >= 2^32 - 1, time >= 2^40 units, C > 16384, L >= 2^24 ... */
  TACOS_E_VERIFY = -7,      /* internal verification failed */
  TACOS_E_NCCL = -8,        /* reserved: cross-GPU selection failed */
  TACOS_E_CAPACITY = -9     /* caller-provided output buffer too small */
} tacos_status;

typedef enum {
  TACOS_ALL_GATHER = 0,
  TACOS_REDUCE_SCATTER = 1, /* mirror of the AG on G^T (R9) */
  TACOS_ALL_REDUCE = 2,     /* RS then AG, T = T_RS + T_AG (R10) */
  TACOS_CUSTOM = 3          /* caller pre/post bitsets, same greedy rule, may stall (R17) */
} tacos_collective;

enum {
  TACOS_FLAG_NO_SCHEDULE = 1u,   /* search only: no send records, time and seed only */
  TACOS_FLAG_KEEP_SEED_TIMES = 2u, /* keep the per-seed collective times */
  /* Paper-literal variant (reading R21): chunk-first
   * matching with replacement of outdated transmissions
   * instead of the link-first walk with persistent claims (R1, R4).  One CTA per
   * seed, in-degree <= 32; cancelled transmissions leave the schedule. */
  TACOS_FLAG_LITERAL = 4u
};

typedef struct tacos_topology tacos_topology; /* opaque */
typedef struct tacos_schedule tacos_schedule; /* opaque */
typedef struct tacos_plan tacos_plan;         /* opaque, device-resident synthesis plan */

/* One send of a schedule: chunk `chunk` leaves `src` over input link `link`
 * (= index into the arrays given to tacos_load_topology, src -> dst) at
 * t_start and is held by dst from t_end = t_start + w_link. */
typedef struct {
  uint32_t chunk, src, dst, link;
  uint64_t t_start, t_end;
} tacos_send; /* 32 bytes */

typedef struct {
  int32_t collective;      /* tacos_collective */
  uint32_t chunks_per_npu; /* k >= 1 (AG/RS/AR) */
  uint64_t chunk_bytes;    /* n > 0 */
  uint32_t time_unit_ns;   /* f >= 1 (0 is read as 1) */
  uint32_t n_seeds;        /* S >= 1: seeds base_seed + seed_offset + i, i < n_seeds */
  uint64_t base_seed;
  uint32_t seed_offset;    /* first global seed index of this shard (multi-GPU, 0 otherwise) */
  uint32_t n_chunks;       /* CUSTOM only: C */
  const uint32_t *pre_bits;  /* CUSTOM only: N rows of ceil(C/32) words, copied */
  const uint32_t *post_bits; /* CUSTOM only: N rows of ceil(C/32) words, copied; pre subset of post */
  uint32_t flags;            /* TACOS_FLAG_* */
  uint32_t reserved;
} tacos_synth_params;

/* Summary of one synthesis. */
typedef struct {
  uint64_t T;          /* collective time in time units (AR: T_RS + T_AG) */
  uint64_t T_ag, T_rs; /* phase times (0 when the phase is absent) */
  uint64_t seed;       /* winning AG seed (64-bit Philox key, R2) */
  uint64_t rs_seed;    /* winning RS seed (== seed when G is symmetric) */
  uint64_t n_sends;    /* sends in the schedule (0 when not emitted here) */
  uint64_t matches;    /* link-chunk matches committed over all searched seeds (M) */
  uint64_t visits;     /* free-link visits over all searched seeds (V) */
  uint64_t dest_events;/* (destination, event) pairs with a free in-link (D) */
  uint64_t events;     /* events at which matching ran, summed over seeds (E) */
  int32_t status;      /* TACOS_OK or the failure of the search */
  uint32_t winner_local; /* bit 0: the AG phase was emitted here; bit 1: the RS phase was emitted here
                            (the winning seed of that phase belongs to this shard) */
  uint64_t best_key_ag, best_key_rs; /* (T << 20) | global seed index, see tacos_plan_best_keys */
  uint64_t cancelled;  /* TACOS_FLAG_LITERAL: transmissions dropped as duplicates or replaced */
} tacos_result;

typedef enum {
  TACOS_V_NO_SUCH_LINK = 0,
  TACOS_V_WRONG_DURATION = 1,
  TACOS_V_LINK_OVERLAP = 2,
  TACOS_V_UNHELD_AT_DEPART = 3,
  TACOS_V_DUPLICATE_DELIVERY = 4,
  TACOS_V_POST_UNMET = 5,
  TACOS_V_PHASE_ORDER = 6, /* AR: an AG send starts before the RS phase ends (R10) */
  TACOS_V_COUNT = 7
} tacos_violation;

typedef struct {
  uint64_t T;               /* max t_end */
  uint64_t T_rs;            /* AR: end of the RS phase */
  uint64_t n_violations;    /* total */
  uint64_t per_kind[TACOS_V_COUNT];
  int32_t first_kind;       /* -1 if clean */
  uint32_t reserved;
  uint64_t first_index;     /* index of the first offending send (or NPU*C+chunk for POST_UNMET) */
} tacos_eval_report;

/* ---------------------------------------------------------------------- */
/* Topology                                                                */
/* ---------------------------------------------------------------------- */

/* Load a directed topology.  Link id = array index.  src/dst in [0, N);
 * src != dst; at most one link per ordered pair; bw > 0;
 * 2 <= N; 1 <= L < 2^24.  Builds the CSR by destination (and by source for
 * G^T), the reverse-link map (symmetry, R9) and strong connectivity, and
 * uploads the arrays to the current CUDA device when one is present.
 * Errors: TACOS_E_INVALID_ARG (null, sizes), TACOS_E_TOPOLOGY (rules above),
 * TACOS_E_CUDA (upload failed), TACOS_E_NOMEM. */
int tacos_load_topology(int32_t n_npus, int32_t n_links, const int32_t *src, const int32_t *dst,
                        const uint32_t *alpha_ns, const uint32_t *bw_bytes_per_ns, tacos_topology **out);
void tacos_free_topology(tacos_topology *topo);
int32_t tacos_topology_num_npus(const tacos_topology *topo);
int32_t tacos_topology_num_links(const tacos_topology *topo);
int tacos_topology_strongly_connected(const tacos_topology *topo); /* 1 / 0 */

/* a1: quantized link costs w[L] for (chunk_bytes, time_unit_ns) into caller
 * memory (host).  Errors: TACOS_E_OVERFLOW if some w >= 2^32,
 * TACOS_E_TOPOLOGY if some w = 0 (alpha = n = 0). */
int tacos_link_costs(const tacos_topology *topo, uint64_t chunk_bytes, uint32_t time_unit_ns, uint32_t *w_out);
/* 1 if every link a->b has a reverse b->a with equal cost for these params (R9). */
int tacos_is_symmetric(const tacos_topology *topo, uint64_t chunk_bytes, uint32_t time_unit_ns);

/* ---------------------------------------------------------------------- */
/* One-call synthesis (host in, host out)                                  */
/* ---------------------------------------------------------------------- */

/* Best-of-S synthesis (all seeds of the params) on the current device; the
 * schedule is copied to host memory owned by *out, sorted by (t_start, link).
 * Errors: as listed above; TACOS_E_UNREACHABLE before any kernel runs when
 * an AG/RS/AR is requested on a graph that is not strongly connected. */
int tacos_synthesize(const tacos_topology *topo, const tacos_synth_params *p, tacos_schedule **out);

/* Same for n_topos topologies sharing the params, searched in one batched
 * launch; outs[i] receives topology i's schedule (all or nothing). */
int tacos_synthesize_batch(const tacos_topology *const *topos, uint32_t n_topos, const tacos_synth_params *p,
                           tacos_schedule **outs);

/* Same as tacos_synthesize but writes into caller memory: `sends` may be a
 * host pointer (pinned or pageable) or a device pointer of the current
 * device; capacity in sends (see tacos_max_sends).  `result` is host memory.
 * `stream` is a cudaStream_t (NULL = legacy default stream).
 * Errors additionally: TACOS_E_CAPACITY. */
int tacos_synthesize_into(const tacos_topology *topo, const tacos_synth_params *p, tacos_send *sends,
                          uint64_t capacity, tacos_result *result, void *stream);
/* Number of sends the schedule will have (AG/RS: M, AR: 2M; M = C(N-1) or
 * sum |post - pre| for CUSTOM). */
int tacos_max_sends(const tacos_topology *topo, const tacos_synth_params *p, uint64_t *n_out);

uint64_t tacos_schedule_num_sends(const tacos_schedule *s);
const tacos_send *tacos_schedule_sends(const tacos_schedule *s); /* valid until free */
uint64_t tacos_schedule_time(const tacos_schedule *s);            /* T (AR: T_RS + T_AG) */
uint64_t tacos_schedule_seed(const tacos_schedule *s);            /* winning AG seed */
const tacos_result *tacos_schedule_result(const tacos_schedule *s);
/* per-seed collective times (only with TACOS_FLAG_KEEP_SEED_TIMES), n_seeds entries */
const uint64_t *tacos_schedule_seed_times(const tacos_schedule *s);
void tacos_free_schedule(tacos_schedule *s);

/* ---------------------------------------------------------------------- */
/* Device-resident plan (inputs in HBM; used by multi-GPU sharding)        */
/* ---------------------------------------------------------------------- */

/* Allocate the device state for (topo, params) on the current device:
 * per-seed bitsets, link state, send records.  Reusable across calls. */
int tacos_plan_create(const tacos_topology *topo, const tacos_synth_params *p, tacos_plan **out);
void tacos_plan_destroy(tacos_plan *plan);
/* Run the batched greedy search of all local seeds on `stream` (async) and
 * compute the local best keys into device memory:
 *   keys[0] = min over local seeds of (T_AG(s) << 20) | s   (AR symmetric: T_AG)
 *   keys[1] = same for the RS search on G^T (asymmetric RS/AR), else keys[0]
 * A seed that did not finish contributes 0x7FFFFFFFFFFFFFFF (max as int64 and
 * as uint64, so a MIN all-reduce works in either type).
 * where s = seed_offset + i is the global seed index.  A MIN all-reduce of
 * these two uint64 over ranks selects the global winner. */
int tacos_plan_search(tacos_plan *plan, void *stream);
/* Device pointer to the two uint64 keys (valid for the plan's lifetime). */
uint64_t *tacos_plan_best_keys(tacos_plan *plan);
/* Emit the schedule of the seed named by the (possibly all-reduced) keys if
 * this shard owns it: writes up to `capacity` sends to device memory `d_sends`
 * sorted by (t_start, link) and fills *result (host).  Synchronizes `stream`
 * once to read the keys.  Only the phases whose winning seed is local are
 * written (result->winner_local bits); an AR's RS phase goes to d_sends[0, M)
 * and its AG phase to d_sends[M, 2M). */
int tacos_plan_emit(tacos_plan *plan, tacos_send *d_sends, uint64_t capacity, tacos_result *result, void *stream);
/* Winner of a (possibly all-reduced) pair of best keys. */
typedef struct {
  uint64_t T, T_ag, T_rs;       /* T = T_rs + T_ag (R10); a phase absent from the collective has 0 */
  uint64_t seed_index_ag;       /* global seed index of the AG phase winner */
  uint64_t seed_index_rs;       /* global seed index of the RS phase winner (= AG winner on a symmetric graph) */
  uint32_t local;               /* bit 0: AG winner in [seed_offset, seed_offset + n_seeds); bit 1: RS winner */
  uint32_t reserved;
} tacos_winner;
/* Decode best keys (see tacos_plan_search) into the winning seeds and times,
 * host only (P:L274 best-of-S; R9 symmetric RS = mirror of the AG winner;
 * R11 ties to the lowest seed index).  `symmetric` as tacos_is_symmetric.
 * Errors: TACOS_E_UNREACHABLE if a needed key says no seed finished,
 * TACOS_E_OVERFLOW if T >= 2^40, TACOS_E_INVALID_ARG. */
int tacos_select_winner(const uint64_t keys[2], int32_t collective, int symmetric, uint32_t seed_offset,
                        uint32_t n_seeds, tacos_winner *out);
/* Per-seed finish times (device pointer, n_seeds uint64: AG on G) and, for an
 * asymmetric RS/AR, the RS search times (second pointer, else NULL). */
const uint64_t *tacos_plan_seed_times_device(const tacos_plan *plan, const uint64_t **rs_times);
/* Number of CUDA kernels the last search / emit launched. */
uint32_t tacos_plan_last_launches(const tacos_plan *plan);
/* Algorithmic bytes of the last search:
 *   B = V*(R + 16) + D*(2R) + M*48 with R = C/8, summed over seeds;
 * requires the stats of a completed search (synchronizes). */
int tacos_plan_stats(tacos_plan *plan, tacos_result *result, void *stream);

/* ---------------------------------------------------------------------- */
/* Verification                                                            */
/* ---------------------------------------------------------------------- */

/* Replay `sends` (host memory) as the collective of `p` on `topo` (host-side):
 * link exists and t_end - t_start == w; link intervals disjoint; the source
 * holds the chunk (arrived) at t_start; every required (chunk, NPU) delivered
 * exactly once; postcondition met; AR: the first half is the RS (mirrored back
 * it must verify as an AG on G^T) and every AG send starts at or after T_RS.
 * Returns TACOS_OK when the replay ran (violations are data in *out). */
int tacos_eval(const tacos_topology *topo, const tacos_synth_params *p, const tacos_send *sends, uint64_t n_sends,
               tacos_eval_report *out);

/* ---------------------------------------------------------------------- */
/* Continuous-time evaluation and baselines (host)       */
/* ---------------------------------------------------------------------- */

/* Replay `sends` in continuous time ("time domain translator",
 * P:L299 queueing link congestion): a send on link l lasts
 * alpha_l + chunk_bytes / bw_l ns (unrounded); each link serves its
 * sends one at a time, first come first served in the schedule's order of
 * (t_start, position in the array); a send starts when its link is free and
 * its input is ready:
 *   AG-type send (c, a->b): chunk c available at a (initially held, or the end
 *     of the send that delivered it to a);
 *   RS-type send (c, a->b) (RS phase of an RS/AR): every RS send of chunk c
 *     into a has ended (a's partial sum is complete; mirror of the AG rule);
 *   AR: the first half of the (t_start, link)-sorted sends is the RS phase;
 *     in the AG phase the owner of c starts from the end of its RS inputs.
 * The schedule's own order must be a topological order of these
 * dependencies (true for TACOS and baseline schedules).  Reports the
 * collective time and the RS phase end, in ns (double). */
typedef struct {
  double T_ns;        /* last arrival */
  double T_rs_ns;     /* AR/RS: end of the RS phase */
  double max_link_busy_ns; /* busiest link's total occupancy */
  uint64_t n_sends;
} tacos_cont_report;
int tacos_eval_continuous(const tacos_topology *topo, const tacos_synth_params *p, const tacos_send *sends,
                          uint64_t n_sends, tacos_cont_report *out);

/* Baseline collective algorithms as schedules ("Ring and Direct
 * collective communication algorithms as two baselines"; P:L120 xy-routing):
 *   TACOS_BASELINE_RING:   logical ring over NPU ids 0..N-1; in step j NPU i
 *                          forwards the chunks of NPU (i - j) mod N to NPU i+1;
 *   TACOS_BASELINE_DIRECT: every NPU sends each of its chunks to every NPU.
 * Each logical transfer follows a shortest path in hops (BFS visiting out-links
 * in link-id order; on a mesh in canonical order this is xy routing); every hop
 * is one send.  t_start is a logical order key (step and hop), t_end =
 * t_start + w: evaluate them with tacos_eval_continuous (they are not
 * congestion-free).  RS = time mirror of the AG on G^T, AR = RS then AG.
 * Call with capacity 0 to get *n_out. */
enum { TACOS_BASELINE_RING = 0, TACOS_BASELINE_DIRECT = 1 };
int tacos_baseline(const tacos_topology *topo, const tacos_synth_params *p, int32_t algorithm, tacos_send *out,
                   uint64_t capacity, uint64_t *n_out);

/* ---------------------------------------------------------------------- */
/* Topology front-end (host)                             */
/* ---------------------------------------------------------------------- */

/* One dimension of a hierarchical topology ("3D topology of
 * Ring_FullyConnected_Switch"; SPEC S:L84-91 composition).
 *   TACOS_DIM_RING:   i -> i+1 (mod n); bidirectional adds i -> i-1 (a 2-node
 *                     ring has one link per direction)
 *   TACOS_DIM_FC:     every ordered pair
 *   TACOS_DIM_SWITCH: switch unwound with degree d (§IV.D):
 *                     i -> i+1 .. i+d (mod n), each link bw / d (bw must be a
 *                     multiple of d); d = 1 with `bidirectional` is the paper's
 *                     bi-directional ring variation at full bandwidth
 *   TACOS_DIM_PATH:   1-D mesh, i -> i+1 and i -> i-1 where they exist
 * Every link of a dimension gets that dimension's alpha and bandwidth. */
enum { TACOS_DIM_RING = 0, TACOS_DIM_FC = 1, TACOS_DIM_SWITCH = 2, TACOS_DIM_PATH = 3 };
typedef struct {
  int32_t kind;
  uint32_t n;             /* NPUs along this dimension (>= 2) */
  uint32_t degree;        /* SWITCH only: 1 <= d <= n - 1 */
  uint32_t bidirectional; /* RING / SWITCH with d = 1 */
  uint32_t alpha_ns;
  uint32_t bw;            /* bytes per ns (total per NPU for SWITCH) */
} tacos_dim_spec;

/* Product of the dimensions: NPU id = c_0 + n_0 (c_1 + n_1 (c_2 + ...)) (dimension
 * 0 fastest).  Links in canonical order: NPU by NPU, then dimension by dimension,
 * then the dimension's own link order from c_i.  Writes up to `capacity` links to
 * src/dst/alpha/bw (caller host memory) and the counts to *n_npus / *n_links;
 * call with capacity 0 (arrays may be NULL) to get the sizes.
 * Errors: TACOS_E_INVALID_ARG (bad spec, N >= 2^31), TACOS_E_CAPACITY. */
int tacos_build_hierarchical(const tacos_dim_spec *dims, uint32_t n_dims, int32_t *n_npus, int32_t *n_links,
                             int32_t *src, int32_t *dst, uint32_t *alpha_ns, uint32_t *bw, int64_t capacity);

/* Remove NPUs (and every link touching them), renumbering the remaining NPUs
 * densely in ascending order and keeping the relative link order (PAPER
 * P:L406, Table IV: a mesh with failed NPUs is re-synthesized on the
 * reduced topology).  Outputs as tacos_build_hierarchical; `old_id` (may be
 * NULL, capacity >= N - n_removed) receives the original id of each new NPU. */
int tacos_remove_npus(int32_t n_npus, int32_t n_links, const int32_t *src, const int32_t *dst, const uint32_t *alpha_ns,
                      const uint32_t *bw, const int32_t *removed, uint32_t n_removed, int32_t *out_n_npus,
                      int32_t *out_n_links, int32_t *out_src, int32_t *out_dst, uint32_t *out_alpha, uint32_t *out_bw,
                      int64_t capacity, int32_t *old_id);

/* ---------------------------------------------------------------------- */
/* Misc                                                                    */
/* ---------------------------------------------------------------------- */
const char *tacos_strerror(int code);
const char *tacos_last_error(void);
int tacos_abi_version(void);
/* Philox4x32-10 of the product path (R2), exposed for known-answer tests:
 * out[4] = Philox(ctr[4], key[2]) computed by a device kernel. */
int tacos_philox_device(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

#ifdef __cplusplus
}
#endif
#endif /* TACOS_H */
