/*
 * tacos_oracle.c -- plain, slow, obviously-correct CPU oracle for TACOS-Greedy.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this code.
 * It shares no source, header, table or helper with the CUDA product path
 * (paper_2304_05301_b200/csrc); neither includes the other.
 *
 * What it computes (PAPER.md = "P:L<line>", SURVEY.md §8(c) = "R<n>"):
 *   - a1  link cost  w = ceil((alpha*bw + n) / (bw*f))           P:L104 (§II.C), P:L172 (§IV.C), R5, R6
 *   - R2  Philox4x32-10 (Salmon et al., SC'11) for every random draw P:L253 "randomly select"
 *   - a2-a6 one greedy All-Gather synthesis, step by step in the order of
 *         SURVEY §8(c)'s pseudo-code: arrivals, done test, per-destination
 *         link-first matching in shorter-link-first order, advance.      P:L249-253 (§VI.A), P:L263-270 (§VI.B)
 * All arithmetic is integer.  No blocking, fusion or reordering beyond the
 * pseudo-code.  The All-Reduce composition (mirror, shift, best-of-S; P:L284,
 * P:L274) lives in oracle/__init__.py (numpy), also part of the oracle.
 *
 * Readings taken where the paper is silent (listed in DESIGN.md §3):
 *   R1 link-first walk; R2 Philox ctr=(t_lo,t_hi,link,sigma) key=(seed_lo,seed_hi),
 *   word0 = order key, word1 = pick draw; R3 sort free in-links by (w, u_ord, link);
 *   R4 claims persist until arrival; R7 arrivals at t before matching at t;
 *   R8 link busy on [t, t+w); R12 chunk c at bit c&31 of word c>>5, r-th = ascending;
 *   R13 r = floor(u_pick*K / 2^32); R19 T = time of the last arrival.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_E_INVALID_ARG -1
#define ORACLE_E_UNREACHABLE -3
#define ORACLE_E_NOMEM -5
#define ORACLE_E_OVERFLOW -6
#define ORACLE_E_CAPACITY -9

#define NONE 0xFFFFFFFFu

typedef struct {
  uint32_t chunk, src, dst, link;
  uint64_t t_start, t_end;
} oracle_send; /* 32 bytes, same field order as the public tacos_send */

/* ------------------------------------------------------------------------ */
/* a1: cost quantization.  P:L104 delay = alpha + beta*n with beta = 1/bw    */
/* (R6: bw in bytes/ns); P:L172 re-calculated into ceil(l/f).  In integer   */
/* form l/f = (alpha + n/bw)/f = (alpha*bw + n)/(bw*f).  Exact (128-bit).   */
/* ------------------------------------------------------------------------ */
int oracle_link_cost(uint32_t alpha_ns, uint32_t bw, uint64_t n_bytes, uint32_t f_ns, uint64_t *w_out) {
  if (bw == 0 || f_ns == 0 || w_out == NULL) return ORACLE_E_INVALID_ARG;
  unsigned __int128 num = (unsigned __int128)alpha_ns * bw + n_bytes;
  unsigned __int128 den = (unsigned __int128)bw * f_ns;
  unsigned __int128 w = (num + den - 1) / den; /* ceiling */
  if (w == 0) return ORACLE_E_INVALID_ARG;     /* alpha = n = 0: no time passes */
  if (w > (unsigned __int128)0xFFFFFFFFu) return ORACLE_E_OVERFLOW;
  *w_out = (uint64_t)w;
  return ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* R2: Philox4x32-10.  Round: (hi1^c1^k0, lo1, hi0^c3^k1, lo0) with        */
/* (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2; key bumped by the Weyl constants   */
/* between rounds.                                                          */
/* ------------------------------------------------------------------------ */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { k0 += W0; k1 += W1; }
    uint64_t p0 = (uint64_t)M0 * c[0];
    uint64_t p1 = (uint64_t)M1 * c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c[3] ^ k1;
    uint32_t n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
  }
  out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

/* ---- small bitset helpers (plain loops) -------------------------------- */
static int bit_get(const uint32_t *row, uint32_t c) { return (row[c >> 5] >> (c & 31)) & 1u; }
static void bit_set(uint32_t *row, uint32_t c) { row[c >> 5] |= 1u << (c & 31); }
static void bit_clr(uint32_t *row, uint32_t c) { row[c >> 5] &= ~(1u << (c & 31)); }

typedef struct {
  uint64_t w;
  uint32_t u_ord;
  uint32_t link;
  uint32_t u_pick;
} free_link;

/* R3: ascending (w, u_ord, link id) */
static int cmp_free_link(const void *pa, const void *pb) {
  const free_link *a = (const free_link *)pa, *b = (const free_link *)pb;
  if (a->w != b->w) return a->w < b->w ? -1 : 1;
  if (a->u_ord != b->u_ord) return a->u_ord < b->u_ord ? -1 : 1;
  if (a->link != b->link) return a->link < b->link ? -1 : 1;
  return 0;
}

/*
 * One greedy synthesis for one seed.
 *   pre_bits == NULL: All-Gather with k chunks per NPU: chunk c = owner*k + j
 *     (R12), held[x] = {x*k .. x*k+k-1}, post[x] = all C = N*k chunks.
 *   pre_bits != NULL: CUSTOM pre/post (N rows of ceil(C/32) words each);
 *     requires pre[x] subset of post[x].
 * Outputs the sends in production order (event by event, destination by
 * destination, in walk order), the finish time T (R19) and the counters
 * stats[0]=V free-link visits, [1]=D (destination,event) pairs with a free
 * in-link, [2]=M matches, [3]=E events at which matching ran.
 */
/*
 * allow_bits (NULL, or CUSTOM only): L rows of ceil(C/32) words, row l = the
 * chunks link l may carry (reading R22: post[dst]
 * plus the chunks dst may relay).  The candidate set then reads allow[l]
 * instead of post[d], and only arrivals of chunks in post[dst] count towards
 * the postcondition (a relayed chunk is held, so it can be forwarded, but it
 * is not required at the relay).
 */
static int greedy_impl(int32_t n_npus, int32_t n_links, const int32_t *src, const int32_t *dst, const uint64_t *w,
                       uint32_t n_chunks, uint32_t k, const uint32_t *pre_bits, const uint32_t *post_bits,
                       const uint32_t *allow_bits, uint64_t seed, uint32_t sigma, oracle_send *sends, uint64_t cap,
                       uint64_t *n_sends_out, uint64_t *T_out, uint64_t *stats) {
  if (n_npus < 1 || n_links < 0 || n_chunks < 1) return ORACLE_E_INVALID_ARG;
  if (allow_bits != NULL && pre_bits == NULL) return ORACLE_E_INVALID_ARG;
  const uint32_t N = (uint32_t)n_npus, L = (uint32_t)n_links, C = n_chunks;
  const uint32_t W = (C + 31) / 32;
  int rc = ORACLE_OK;

  uint32_t *held = calloc((size_t)N * W, 4);
  uint32_t *pending = calloc((size_t)N * W, 4);
  uint32_t *post = calloc((size_t)N * W, 4);
  uint32_t *claimed = calloc(W, 4);
  uint32_t *cand = calloc(W, 4);
  uint64_t *busy_until = calloc(L ? L : 1, 8);
  uint32_t *cur = malloc((size_t)(L ? L : 1) * 4);
  free_link *F = malloc((size_t)(L ? L : 1) * sizeof(free_link));
  uint32_t *in_start = calloc((size_t)N + 1, 4); /* in-links of d: in_list[in_start[d] .. in_start[d+1]) */
  uint32_t *in_list = malloc((size_t)(L ? L : 1) * 4);
  if (!held || !pending || !post || !claimed || !cand || !busy_until || !cur || !F || !in_start || !in_list) {
    rc = ORACLE_E_NOMEM;
    goto done;
  }

  /* a2: state init (P:L89 pre/postcondition; P:L212 start at t = 0) */
  uint64_t required = 0;
  if (pre_bits == NULL) {
    if ((uint64_t)N * k != C) { rc = ORACLE_E_INVALID_ARG; goto done; }
    for (uint32_t x = 0; x < N; ++x) {
      for (uint32_t j = 0; j < k; ++j) bit_set(&held[(size_t)x * W], x * k + j);
      for (uint32_t c = 0; c < C; ++c) bit_set(&post[(size_t)x * W], c);
    }
    required = (uint64_t)C * (N - 1);
  } else {
    memcpy(held, pre_bits, (size_t)N * W * 4);
    memcpy(post, post_bits, (size_t)N * W * 4);
    for (uint32_t x = 0; x < N; ++x)
      for (uint32_t c = 0; c < C; ++c) {
        int in_pre = bit_get(&held[(size_t)x * W], c), in_post = bit_get(&post[(size_t)x * W], c);
        if (in_pre && !in_post) { rc = ORACLE_E_INVALID_ARG; goto done; }
        if (in_post && !in_pre) required++;
      }
    /* bits beyond C must be clear */
    for (uint32_t x = 0; x < N; ++x)
      for (uint32_t c = C; c < W * 32; ++c)
        if (bit_get(&held[(size_t)x * W], c) || bit_get(&post[(size_t)x * W], c)) { rc = ORACLE_E_INVALID_ARG; goto done; }
  }
  for (uint32_t l = 0; l < L; ++l) {
    if (src[l] < 0 || src[l] >= n_npus || dst[l] < 0 || dst[l] >= n_npus || w[l] < 1) { rc = ORACLE_E_INVALID_ARG; goto done; }
    busy_until[l] = 0;
    cur[l] = NONE;
  }
  /* in-link lists per destination, ascending link id (plain counting) */
  for (uint32_t l = 0; l < L; ++l) in_start[dst[l] + 1]++;
  for (uint32_t d = 0; d < N; ++d) in_start[d + 1] += in_start[d];
  {
    uint32_t *fill = calloc((size_t)N, 4);
    if (!fill) { rc = ORACLE_E_NOMEM; goto done; }
    for (uint32_t l = 0; l < L; ++l) in_list[in_start[dst[l]] + fill[dst[l]]++] = l;
    free(fill);
  }

  uint64_t t = 0, delivered = 0, n_sends = 0;
  uint64_t V = 0, D = 0, M = 0, E = 0;
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};

  for (;;) {
    /* (1) arrivals at t (R7): the chunk is held by dst from this instant */
    for (uint32_t l = 0; l < L; ++l) {
      if (cur[l] != NONE && busy_until[l] == t) {
        bit_set(&held[(size_t)dst[l] * W], cur[l]);
        bit_clr(&pending[(size_t)dst[l] * W], cur[l]);
        if (bit_get(&post[(size_t)dst[l] * W], cur[l])) delivered += 1; /* a relay arrival is not required */
        cur[l] = NONE;
      }
    }
    /* (2) done test: postcondition holds */
    if (delivered == required) { *T_out = t; break; }

    /* (3) matching, destination by destination (R1, R3, R4) */
    E += 1;
    for (uint32_t d = 0; d < N; ++d) {
      uint32_t *held_d = &held[(size_t)d * W];
      uint32_t *post_d = &post[(size_t)d * W];
      memcpy(claimed, &pending[(size_t)d * W], (size_t)W * 4);
      uint32_t nf = 0;
      for (uint32_t e = in_start[d]; e < in_start[d + 1]; ++e) {
        uint32_t l = in_list[e];
        if (cur[l] == NONE) {
          uint32_t ctr[4] = {(uint32_t)t, (uint32_t)(t >> 32), l, sigma};
          uint32_t out[4];
          oracle_philox4x32_10(ctr, key, out);
          F[nf].w = w[l];
          F[nf].u_ord = out[0];
          F[nf].u_pick = out[1];
          F[nf].link = l;
          nf++;
        }
      }
      if (nf == 0) continue;
      D += 1;
      qsort(F, nf, sizeof(free_link), cmp_free_link); /* shorter-link-first */
      for (uint32_t i = 0; i < nf; ++i) {
        uint32_t l = F[i].link;
        const uint32_t *held_s = &held[(size_t)src[l] * W];
        V += 1;
        /* cand = post[d] & held[src] & ~held[d] & ~claimed  (allow[l] in place of post[d] with relays) */
        const uint32_t *mask = allow_bits ? &allow_bits[(size_t)l * W] : post_d;
        uint64_t K = 0;
        for (uint32_t q = 0; q < W; ++q) {
          cand[q] = mask[q] & held_s[q] & ~held_d[q] & ~claimed[q];
          K += (uint64_t)__builtin_popcount(cand[q]);
        }
        if (K == 0) continue;
        /* R13: r = floor(u_pick * K / 2^32), 0 <= r < K */
        uint64_t r = ((uint64_t)F[i].u_pick * K) >> 32;
        /* r-th smallest member of cand (0-based, ascending chunk id, R12) */
        uint32_t c = NONE;
        for (uint32_t q = 0; q < W && c == NONE; ++q) {
          uint64_t pc = (uint64_t)__builtin_popcount(cand[q]);
          if (r >= pc) { r -= pc; continue; }
          for (uint32_t b = 0; b < 32; ++b) {
            if ((cand[q] >> b) & 1u) {
              if (r == 0) { c = q * 32 + b; break; }
              r--;
            }
          }
        }
        if (t > UINT64_MAX / 2 - w[l]) { rc = ORACLE_E_OVERFLOW; goto done; }
        bit_set(claimed, c);
        cur[l] = c;
        busy_until[l] = t + w[l];
        if (sends) {
          if (n_sends >= cap) { rc = ORACLE_E_CAPACITY; goto done; }
          sends[n_sends].chunk = c;
          sends[n_sends].src = (uint32_t)src[l];
          sends[n_sends].dst = d;
          sends[n_sends].link = l;
          sends[n_sends].t_start = t;
          sends[n_sends].t_end = t + w[l];
        }
        n_sends += 1;
        M += 1;
      }
      memcpy(&pending[(size_t)d * W], claimed, (size_t)W * 4);
    }

    /* (4) advance to the next event; nothing in flight and not done = stall */
    uint64_t t_next = UINT64_MAX;
    for (uint32_t l = 0; l < L; ++l)
      if (cur[l] != NONE && busy_until[l] < t_next) t_next = busy_until[l];
    if (t_next == UINT64_MAX) { rc = ORACLE_E_UNREACHABLE; *T_out = t; break; }
    t = t_next;
  }
  /* Relays (R22): a send still in flight when the postcondition holds carries a
   * chunk nobody requires any more (every required chunk has arrived); it leaves
   * the schedule.  Without relays nothing is in flight at that point. */
  if (rc == ORACLE_OK && sends) {
    uint64_t kept = 0;
    for (uint64_t i = 0; i < n_sends; ++i)
      if (sends[i].t_end <= *T_out) sends[kept++] = sends[i];
    n_sends = kept;
  }
  *n_sends_out = n_sends;
  if (stats) { stats[0] = V; stats[1] = D; stats[2] = M; stats[3] = E; }

done:
  free(held); free(pending); free(post); free(claimed); free(cand);
  free(busy_until); free(cur); free(F); free(in_start); free(in_list);
  return rc;
}

int oracle_greedy(int32_t n_npus, int32_t n_links, const int32_t *src, const int32_t *dst, const uint64_t *w,
                  uint32_t n_chunks, uint32_t k, const uint32_t *pre_bits, const uint32_t *post_bits,
                  uint64_t seed, uint32_t sigma, oracle_send *sends, uint64_t cap, uint64_t *n_sends_out,
                  uint64_t *T_out, uint64_t *stats) {
  return greedy_impl(n_npus, n_links, src, dst, w, n_chunks, k, pre_bits, post_bits, NULL, seed, sigma, sends, cap,
                     n_sends_out, T_out, stats);
}

/* CUSTOM with a per-link allow mask (relays, R22); see greedy_impl. */
int oracle_greedy_relay(int32_t n_npus, int32_t n_links, const int32_t *src, const int32_t *dst, const uint64_t *w,
                        uint32_t n_chunks, const uint32_t *pre_bits, const uint32_t *post_bits,
                        const uint32_t *allow_bits, uint64_t seed, uint32_t sigma, oracle_send *sends, uint64_t cap,
                        uint64_t *n_sends_out, uint64_t *T_out, uint64_t *stats) {
  if (allow_bits == NULL) return ORACLE_E_INVALID_ARG;
  return greedy_impl(n_npus, n_links, src, dst, w, n_chunks, 0, pre_bits, post_bits, allow_bits, seed, sigma, sends,
                     cap, n_sends_out, T_out, stats);
}

/*
 * Paper-literal variant (reading R21).
 *   chunk-first matching ("first we choose a requested chunk and
 *   backtrack the NPU ... among candidate links, we can randomly select one"),
 *   shorter-link-first among the candidates, the arrival-time rule
 *    and chunk replacement of outdated transmissions:
 * At each event t:
 *  (1) arrivals in ascending link id; a copy of a chunk its destination already
 *      holds (a duplicate) is dropped: its send leaves the schedule;
 *  (2) done test;
 *  (3) replacement: an in-flight send whose chunk its destination already holds
 *      is outdated: cancelled (leaves the schedule), its link is free at t;
 *  (4) per destination d: R = post[d] - held[d] (chunks in flight to d are
 *      requested again); Philox block (t_lo, t_hi, d, 0x80000000 | sigma<<16 | 0),
 *      word 0 -> r0 = floor(u * |R| / 2^32); chunks are visited in ascending id
 *      from the r0-th smallest member of R, cyclically; for chunk c the
 *      candidates are d's free in-links not matched at t whose source holds c;
 *      the candidates of minimal w are kept, and the m-th match (m = 1, 2, ...)
 *      takes the floor(u * n / 2^32)-th of them (ascending link id) with u = word 0
 *      of block (t_lo, t_hi, d, 0x80000000 | sigma<<16 | m); stop when d has no
 *      free unmatched in-link;
 *  (5) advance to the next busy_until.
 * stats: [0]=V free in-links at (4), [1]=D, [2]=M sends issued, [3]=E, [4]=X cancelled.
 * Output: the delivered sends (production order of their issue).
 */
int oracle_greedy_literal(int32_t n_npus, int32_t n_links, const int32_t *src, const int32_t *dst, const uint64_t *w,
                          uint32_t n_chunks, uint32_t k, const uint32_t *pre_bits, const uint32_t *post_bits,
                          uint64_t seed, uint32_t sigma, oracle_send *sends, uint64_t cap, uint64_t *n_sends_out,
                          uint64_t *T_out, uint64_t *stats) {
  if (n_npus < 1 || n_links < 0 || n_chunks < 1) return ORACLE_E_INVALID_ARG;
  const uint32_t N = (uint32_t)n_npus, L = (uint32_t)n_links, C = n_chunks;
  const uint32_t W = (C + 31) / 32;
  int rc = ORACLE_OK;
  uint32_t *held = calloc((size_t)N * W, 4);
  uint32_t *post = calloc((size_t)N * W, 4);
  uint64_t *busy_until = calloc(L ? L : 1, 8);
  uint32_t *cur = malloc((size_t)(L ? L : 1) * 4);
  uint64_t *issue = malloc((size_t)(L ? L : 1) * 8);   /* index of the link's in-flight send */
  char *used = calloc(L ? L : 1, 1);
  uint32_t *in_start = calloc((size_t)N + 1, 4);
  uint32_t *in_list = malloc((size_t)(L ? L : 1) * 4);
  uint32_t *cands = malloc((size_t)(L ? L : 1) * 4);
  /* every issued send, with a cancelled flag; capacity grows */
  uint64_t n_issued = 0, cap_issued = 1024;
  oracle_send *issued = malloc(cap_issued * sizeof(oracle_send));
  char *cancelled = calloc(cap_issued, 1);
  if (!held || !post || !busy_until || !cur || !issue || !used || !in_start || !in_list || !cands || !issued ||
      !cancelled) {
    rc = ORACLE_E_NOMEM;
    goto done;
  }
  uint64_t required = 0;
  if (pre_bits == NULL) {
    if ((uint64_t)N * k != C) { rc = ORACLE_E_INVALID_ARG; goto done; }
    for (uint32_t x = 0; x < N; ++x) {
      for (uint32_t j = 0; j < k; ++j) bit_set(&held[(size_t)x * W], x * k + j);
      for (uint32_t c = 0; c < C; ++c) bit_set(&post[(size_t)x * W], c);
    }
    required = (uint64_t)C * (N - 1);
  } else {
    memcpy(held, pre_bits, (size_t)N * W * 4);
    memcpy(post, post_bits, (size_t)N * W * 4);
    for (uint32_t x = 0; x < N; ++x)
      for (uint32_t c = 0; c < C; ++c) {
        int a = bit_get(&held[(size_t)x * W], c), b = bit_get(&post[(size_t)x * W], c);
        if (a && !b) { rc = ORACLE_E_INVALID_ARG; goto done; }
        if (b && !a) required++;
      }
  }
  for (uint32_t l = 0; l < L; ++l) {
    if (src[l] < 0 || src[l] >= n_npus || dst[l] < 0 || dst[l] >= n_npus || w[l] < 1) { rc = ORACLE_E_INVALID_ARG; goto done; }
    cur[l] = NONE;
    busy_until[l] = 0;
  }
  for (uint32_t l = 0; l < L; ++l) in_start[dst[l] + 1]++;
  for (uint32_t d = 0; d < N; ++d) in_start[d + 1] += in_start[d];
  {
    uint32_t *fill = calloc((size_t)N, 4);
    if (!fill) { rc = ORACLE_E_NOMEM; goto done; }
    for (uint32_t l = 0; l < L; ++l) in_list[in_start[dst[l]] + fill[dst[l]]++] = l;
    free(fill);
  }
  uint64_t t = 0, delivered = 0, V = 0, D = 0, M = 0, E = 0, X = 0;
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  for (;;) {
    /* (1) arrivals, ascending link id; duplicates dropped */
    for (uint32_t l = 0; l < L; ++l) {
      if (cur[l] != NONE && busy_until[l] == t) {
        uint32_t *hd = &held[(size_t)dst[l] * W];
        if (bit_get(hd, cur[l])) {
          cancelled[issue[l]] = 1;
          X += 1;
        } else {
          bit_set(hd, cur[l]);
          delivered += 1;
        }
        cur[l] = NONE;
      }
    }
    /* (2) done: copies still in flight are outdated and leave the schedule */
    if (delivered == required) {
      *T_out = t;
      for (uint32_t l = 0; l < L; ++l)
        if (cur[l] != NONE) {
          cancelled[issue[l]] = 1;
          X += 1;
          cur[l] = NONE;
        }
      break;
    }
    /* (3) replacement of outdated in-flight sends */
    for (uint32_t l = 0; l < L; ++l) {
      if (cur[l] != NONE && bit_get(&held[(size_t)dst[l] * W], cur[l])) {
        cancelled[issue[l]] = 1;
        X += 1;
        cur[l] = NONE;
        busy_until[l] = t;
      }
    }
    /* (4) chunk-first matching */
    E += 1;
    for (uint32_t d = 0; d < N; ++d) {
      uint32_t n_free = 0;
      for (uint32_t e = in_start[d]; e < in_start[d + 1]; ++e) {
        uint32_t l = in_list[e];
        used[l] = 0;
        if (cur[l] == NONE) n_free++;
      }
      if (n_free == 0) continue;
      D += 1;
      V += n_free;
      const uint32_t *hd = &held[(size_t)d * W], *pd = &post[(size_t)d * W];
      uint64_t nR = 0;
      for (uint32_t c = 0; c < C; ++c)
        if (bit_get(pd, c) && !bit_get(hd, c)) nR++;
      if (nR == 0) continue;
      uint32_t ctr[4] = {(uint32_t)t, (uint32_t)(t >> 32), d, 0x80000000u | (sigma << 16)};
      uint32_t out[4];
      oracle_philox4x32_10(ctr, key, out);
      uint64_t r0 = ((uint64_t)out[0] * nR) >> 32;
      /* start chunk: the r0-th smallest member of R */
      uint32_t start = 0;
      {
        uint64_t seen = 0;
        for (uint32_t c = 0; c < C; ++c)
          if (bit_get(pd, c) && !bit_get(hd, c)) {
            if (seen == r0) { start = c; break; }
            seen++;
          }
      }
      uint32_t m = 0, n_unmatched = n_free;
      for (uint32_t i = 0; i < C && n_unmatched > 0; ++i) {
        const uint32_t c = (start + i) % C;
        if (!(bit_get(pd, c) && !bit_get(hd, c))) continue;
        /* candidates: free, unmatched in-links whose source holds c; keep minimal w */
        uint32_t nc = 0;
        uint64_t wmin = UINT64_MAX;
        for (uint32_t e = in_start[d]; e < in_start[d + 1]; ++e) {
          uint32_t l = in_list[e];
          if (cur[l] != NONE || used[l]) continue;
          if (!bit_get(&held[(size_t)src[l] * W], c)) continue;
          if (w[l] < wmin) { wmin = w[l]; nc = 0; }
          if (w[l] == wmin) cands[nc++] = l;
        }
        if (nc == 0) continue;
        m += 1;
        uint32_t ctr2[4] = {(uint32_t)t, (uint32_t)(t >> 32), d, 0x80000000u | (sigma << 16) | m};
        oracle_philox4x32_10(ctr2, key, out);
        const uint32_t l = cands[((uint64_t)out[0] * nc) >> 32];
        if (t > UINT64_MAX / 2 - w[l]) { rc = ORACLE_E_OVERFLOW; goto done; }
        used[l] = 1;
        n_unmatched--;
        cur[l] = c;
        busy_until[l] = t + w[l];
        if (n_issued == cap_issued) {
          cap_issued *= 2;
          oracle_send *ni = realloc(issued, cap_issued * sizeof(oracle_send));
          char *nc2 = realloc(cancelled, cap_issued);
          if (!ni || !nc2) { rc = ORACLE_E_NOMEM; if (ni) issued = ni; if (nc2) cancelled = nc2; goto done; }
          issued = ni;
          cancelled = nc2;
          memset(cancelled + n_issued, 0, cap_issued - n_issued);
        }
        issued[n_issued].chunk = c;
        issued[n_issued].src = (uint32_t)src[l];
        issued[n_issued].dst = d;
        issued[n_issued].link = l;
        issued[n_issued].t_start = t;
        issued[n_issued].t_end = t + w[l];
        issue[l] = n_issued;
        n_issued++;
        M += 1;
      }
    }
    /* (5) advance */
    uint64_t t_next = UINT64_MAX;
    for (uint32_t l = 0; l < L; ++l)
      if (cur[l] != NONE && busy_until[l] < t_next) t_next = busy_until[l];
    if (t_next == UINT64_MAX) { rc = ORACLE_E_UNREACHABLE; *T_out = t; break; }
    t = t_next;
  }
  {
    uint64_t n_out = 0;
    for (uint64_t i = 0; i < n_issued; ++i) {
      if (cancelled[i]) continue;
      if (sends) {
        if (n_out >= cap) { rc = ORACLE_E_CAPACITY; goto done; }
        sends[n_out] = issued[i];
      }
      n_out++;
    }
    *n_sends_out = n_out;
  }
  if (stats) { stats[0] = V; stats[1] = D; stats[2] = M; stats[3] = E; stats[4] = X; }
done:
  free(held); free(post); free(busy_until); free(cur); free(issue); free(used);
  free(in_start); free(in_list); free(cands); free(issued); free(cancelled);
  return rc;
}
