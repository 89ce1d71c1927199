// tacos_api.cpp -- host runtime behind include/tacos.h (C ABI).
//
// Validation, cost quantization (a1), CSR construction,
// strong connectivity, plan / device memory management (a caching device and
// pinned-host allocator), orchestration of the kernels in tacos_kernels.cu
// (a2-a8), and the host verifier behind tacos_eval.
// Product side only: nothing here is shared with the CPU oracle (oracle/).
#include "tacos.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <thread>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <unordered_map>
#include <tuple>
#include <unordered_set>
#include <vector>

#include "tacos_internal.h"
#include "tacos_nccl.h"

using namespace tacos;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_last_error;

static int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                        \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess) return fail(TACOS_E_CUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

// ---------------------------------------------------------------------------
// caching allocators (device and pinned host): freed blocks are kept per
// (device, size class) and reused, so repeated synthesize calls do not pay
// cudaMalloc / cudaMallocHost.
// ---------------------------------------------------------------------------
namespace {
size_t size_class(size_t n) {
  if (n <= 4096) return 4096;
  if (n <= (2u << 20)) {
    size_t c = 4096;
    while (c < n) c <<= 1;
    return c;
  }
  return (n + (2u << 20) - 1) / (2u << 20) * (2u << 20);
}

struct Pool {
  std::mutex mu;
  std::multimap<std::pair<int, size_t>, void *> free_blocks;
  bool pinned;
  explicit Pool(bool pinned_) : pinned(pinned_) {}
  void *alloc(int dev, size_t n, size_t *cls_out) {
    const size_t cls = size_class(n);
    *cls_out = cls;
    {
      std::lock_guard<std::mutex> g(mu);
      auto it = free_blocks.find({dev, cls});
      if (it != free_blocks.end()) {
        void *p = it->second;
        free_blocks.erase(it);
        return p;
      }
    }
    void *p = nullptr;
    cudaError_t e = pinned ? cudaMallocHost(&p, cls) : cudaMalloc(&p, cls);
    if (e != cudaSuccess) {
      cudaGetLastError();
      // trim the cache and retry once
      std::vector<std::pair<int, void *>> drop;
      {
        std::lock_guard<std::mutex> g(mu);
        for (auto &kv : free_blocks) drop.push_back({kv.first.first, kv.second});
        free_blocks.clear();
      }
      for (auto &d : drop) {
        if (pinned) cudaFreeHost(d.second);
        else cudaFree(d.second);
      }
      e = pinned ? cudaMallocHost(&p, cls) : cudaMalloc(&p, cls);
      if (e != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
      }
    }
    return p;
  }
  void release(int dev, void *p, size_t cls) {
    if (!p) return;
    std::lock_guard<std::mutex> g(mu);
    free_blocks.insert({{dev, cls}, p});
  }
};

Pool &device_pool() {
  static Pool *p = new Pool(false);  // intentionally leaked: lives until process exit
  return *p;
}
Pool &pinned_pool() {
  static Pool *p = new Pool(true);
  return *p;
}

struct DevBuf {
  void *p = nullptr;
  size_t cls = 0;
  int dev = -1;
};

int cuda_device_ok(int *dev_out) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(TACOS_E_CUDA, "no CUDA device available (%s)", e != cudaSuccess ? cudaGetErrorString(e) : "0 devices");
  }
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  *dev_out = dev;
  return TACOS_OK;
}
}  // namespace

// ---------------------------------------------------------------------------
// topology
// ---------------------------------------------------------------------------
struct tacos_topology {
  int32_t N = 0, L = 0;
  std::vector<int32_t> src, dst;
  std::vector<uint32_t> alpha, bw;
  std::vector<int32_t> rev;  // link dst->src or -1
  bool strongly_connected = false;
  // orientation 0 = G (grouped by dst), 1 = G^T (grouped by src)
  std::vector<uint32_t> in_ptr[2], pos_lid[2], pos_src[2], pos_dst[2];
  int device = -1;  // device current at load time, -1 without a GPU
  // per-device copies of the CSR arrays (tacos_synthesize with n_devices > 1 uses several),
  // created on first use under the mutex; the handle stays logically immutable
  struct Dev {
    int dev = -1;
    uint32_t *d_in_ptr[2] = {nullptr, nullptr}, *d_pos_lid[2] = {nullptr, nullptr};
    uint32_t *d_pos_src[2] = {nullptr, nullptr}, *d_pos_dst[2] = {nullptr, nullptr};
    uint32_t *d_src = nullptr, *d_dst = nullptr;
    int32_t *d_rev = nullptr;
    std::vector<DevBuf> bufs;
    DevBuf stage;               // pinned staging block of the upload (kept until the handle is freed)
    cudaEvent_t ready = nullptr;  // recorded after the upload on the stream of the first user
  };
  mutable std::mutex mu;
  mutable std::vector<std::unique_ptr<Dev>> devs;
  ~tacos_topology() {
    // the blocks go back to a caching pool (no implicit synchronization as with cudaFree):
    // wait for every kernel that may still read them (a plan built from this topology)
    int cur = -1;
    const bool have_cur = cudaGetDevice(&cur) == cudaSuccess;
    for (auto &d : devs) {
      if (cudaSetDevice(d->dev) == cudaSuccess) cudaDeviceSynchronize();
      for (auto &b : d->bufs) device_pool().release(b.dev, b.p, b.cls);
      if (d->stage.p) pinned_pool().release(d->stage.dev, d->stage.p, d->stage.cls);
      if (d->ready) cudaEventDestroy(d->ready);
    }
    if (have_cur) cudaSetDevice(cur);
    cudaGetLastError();
  }
};
using TopoDev = tacos_topology::Dev;

namespace {
// The topology's arrays on device `dev` (the calling thread's current device), uploaded on
// first use: one pinned staging copy + one H2D copy on `st`, not waited for; later users on
// other streams wait for it (event), so nothing here synchronizes.
int topo_on_device(const tacos_topology *t, int dev, const TopoDev **out, cudaStream_t st);
}  // namespace

namespace {
template <typename T>
int upload(std::vector<DevBuf> &bufs, int dev, const T *h, size_t n, T **d_out, cudaStream_t st = nullptr) {
  DevBuf b;
  b.dev = dev;
  b.p = device_pool().alloc(dev, n * sizeof(T) + 16, &b.cls);
  if (!b.p) return fail(TACOS_E_NOMEM, "device allocation of %zu bytes failed", n * sizeof(T));
  bufs.push_back(b);
  if (n) CUDA_TRY(cudaMemcpyAsync(b.p, h, n * sizeof(T), cudaMemcpyHostToDevice, st));
  *d_out = reinterpret_cast<T *>(b.p);
  return TACOS_OK;
}

// Batched host->device upload: arrays are packed into one pinned staging block and
// copied with a single cudaMemcpyAsync into one device block (pageable copies of many
// small arrays each cost a staged, synchronous transfer).
struct Stager {
  struct Part {
    const void *h;
    size_t off, bytes;
  };
  std::vector<Part> parts;
  size_t total = 0;
  unsigned char *d_base = nullptr;
  size_t reserve(size_t bytes) {
    const size_t off = total;
    total += (bytes + 255) / 256 * 256;
    return off;
  }
  // the device address of a reserved region (valid after alloc)
  template <typename T>
  T *at(size_t off) const {
    return reinterpret_cast<T *>(d_base + off);
  }
  int alloc(std::vector<DevBuf> &bufs, int dev) {
    DevBuf b;
    b.dev = dev;
    b.p = device_pool().alloc(dev, total + 16, &b.cls);
    if (!b.p) return fail(TACOS_E_NOMEM, "device allocation of %zu bytes failed", total);
    bufs.push_back(b);
    d_base = reinterpret_cast<unsigned char *>(b.p);
    return TACOS_OK;
  }
  void put(size_t off, const void *h, size_t bytes) { parts.push_back(Part{h, off, bytes}); }
  // one pinned staging copy + one H2D copy on `st`, an event recorded after it; the pinned
  // block is handed to the caller (released once the copy is known complete)
  int copy_async(int dev, cudaStream_t st, DevBuf *stage, cudaEvent_t *ev) {
    if (total == 0) return TACOS_OK;
    stage->dev = dev;
    stage->p = pinned_pool().alloc(dev, total, &stage->cls);
    if (!stage->p) return fail(TACOS_E_NOMEM, "pinned allocation of %zu bytes failed", total);
    for (const Part &q : parts) std::memcpy(reinterpret_cast<unsigned char *>(stage->p) + q.off, q.h, q.bytes);
    cudaError_t e = cudaMemcpyAsync(d_base, stage->p, total, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(*ev, st);
    if (e != cudaSuccess) return fail(TACOS_E_CUDA, "staged upload: %s", cudaGetErrorString(e));
    return TACOS_OK;
  }
};

int dev_alloc(std::vector<DevBuf> &bufs, int dev, size_t n, void **d_out) {
  DevBuf b;
  b.dev = dev;
  b.p = device_pool().alloc(dev, n + 16, &b.cls);
  if (!b.p) return fail(TACOS_E_NOMEM, "device allocation of %zu bytes failed", n);
  bufs.push_back(b);
  *d_out = b.p;
  return TACOS_OK;
}

bool reach_all(int32_t N, const std::vector<uint32_t> &ptr, const std::vector<uint32_t> &pos_src) {
  // BFS from 0 following reversed CSR edges (in-links): reaches every node that can reach 0
  std::vector<char> seen(N, 0);
  std::vector<int32_t> stack{0};
  seen[0] = 1;
  int32_t cnt = 1;
  while (!stack.empty()) {
    int32_t v = stack.back();
    stack.pop_back();
    for (uint32_t p = ptr[v]; p < ptr[v + 1]; ++p) {
      int32_t u = (int32_t)pos_src[p];
      if (!seen[u]) {
        seen[u] = 1;
        ++cnt;
        stack.push_back(u);
      }
    }
  }
  return cnt == N;
}

// a1: w = ceil((alpha*bw + n) / (bw*f)) exactly (P:L104 alpha + n/bw; P:L172 ceil(l/f))
int quantize(uint32_t alpha, uint32_t bw, uint64_t n, uint32_t f, uint32_t *w_out) {
  if (bw == 0) return TACOS_E_TOPOLOGY;
  const uint64_t ab = (uint64_t)alpha * bw, den64 = (uint64_t)bw * (f ? f : 1u);  // both < 2^64
  unsigned __int128 q;
  if (n <= ~0ull - ab) {  // the numerator fits 64 bits: the same quotient without 128-bit division
    const uint64_t num64 = ab + n;
    q = num64 / den64 + (num64 % den64 != 0 ? 1u : 0u);
  } else {
    const unsigned __int128 num = (unsigned __int128)ab + n;
    q = num / den64 + (num % den64 != 0 ? 1 : 0);
  }
  if (q == 0) return TACOS_E_TOPOLOGY;
  if (q >= 0xFFFFFFFFull) return TACOS_E_OVERFLOW;  // w < 2^32 - 1 (the search packs (w, u_ord) into 64 bits)
  *w_out = (uint32_t)q;
  return TACOS_OK;
}

int link_costs(const tacos_topology *t, uint64_t n, uint32_t f, std::vector<uint32_t> &w) {
  w.resize(t->L);
  uint32_t pa = 0, pb = 0, pw = 0;  // the previous link's (alpha, bw) and cost: uniform runs reuse it
  bool have_prev = false;
  for (int32_t l = 0; l < t->L; ++l) {
    if (have_prev && t->alpha[l] == pa && t->bw[l] == pb) {
      w[l] = pw;
      continue;
    }
    int rc = quantize(t->alpha[l], t->bw[l], n, f, &w[l]);
    if (rc == TACOS_OK) {
      pa = t->alpha[l];
      pb = t->bw[l];
      pw = w[l];
      have_prev = true;
    }
    if (rc == TACOS_E_TOPOLOGY) return fail(rc, "link %d has zero cost (alpha = n = 0)", l);
    if (rc == TACOS_E_OVERFLOW) return fail(rc, "link %d cost exceeds 2^32 - 2 time units", l);
    if (rc) return fail(rc, "link %d: bad cost", l);
  }
  return TACOS_OK;
}

bool symmetric_for(const tacos_topology *t, const std::vector<uint32_t> &w) {
  for (int32_t l = 0; l < t->L; ++l) {
    if (t->rev[l] < 0 || w[t->rev[l]] != w[l]) return false;
  }
  return true;
}
}  // namespace

namespace {
int topo_on_device(const tacos_topology *t, int dev, const TopoDev **out, cudaStream_t st) {
  std::lock_guard<std::mutex> g(t->mu);
  for (auto &d : t->devs)
    if (d->dev == dev) {
      if (d->ready) CUDA_TRY(cudaStreamWaitEvent(st, d->ready, 0));
      *out = d.get();
      return TACOS_OK;
    }
  std::unique_ptr<TopoDev> d(new TopoDev());
  d->dev = dev;
  Stager sg;
  const size_t lb = (size_t)t->L * 4;
  size_t o_ptr[2], o_lid[2], o_src[2], o_dst[2];
  for (int o = 0; o < 2; ++o) {
    o_ptr[o] = sg.reserve(t->in_ptr[o].size() * 4);
    o_lid[o] = sg.reserve(lb);
    o_src[o] = sg.reserve(lb);
    o_dst[o] = sg.reserve(lb);
  }
  const size_t o_s = sg.reserve(lb), o_d = sg.reserve(lb), o_r = sg.reserve(lb);
  int rc;
  if ((rc = sg.alloc(d->bufs, dev))) {
    for (auto &b : d->bufs) device_pool().release(b.dev, b.p, b.cls);
    return rc;
  }
  for (int o = 0; o < 2; ++o) {
    sg.put(o_ptr[o], t->in_ptr[o].data(), t->in_ptr[o].size() * 4);
    sg.put(o_lid[o], t->pos_lid[o].data(), lb);
    sg.put(o_src[o], t->pos_src[o].data(), lb);
    sg.put(o_dst[o], t->pos_dst[o].data(), lb);
    d->d_in_ptr[o] = sg.at<uint32_t>(o_ptr[o]);
    d->d_pos_lid[o] = sg.at<uint32_t>(o_lid[o]);
    d->d_pos_src[o] = sg.at<uint32_t>(o_src[o]);
    d->d_pos_dst[o] = sg.at<uint32_t>(o_dst[o]);
  }
  sg.put(o_s, t->src.data(), lb);  // int32 ids < 2^31: the same bytes as uint32
  sg.put(o_d, t->dst.data(), lb);
  sg.put(o_r, t->rev.data(), lb);
  d->d_src = sg.at<uint32_t>(o_s);
  d->d_dst = sg.at<uint32_t>(o_d);
  d->d_rev = sg.at<int32_t>(o_r);
  if ((rc = sg.copy_async(dev, st, &d->stage, &d->ready))) {
    for (auto &b : d->bufs) device_pool().release(b.dev, b.p, b.cls);
    if (d->stage.p) pinned_pool().release(d->stage.dev, d->stage.p, d->stage.cls);
    return rc;
  }
  *out = d.get();
  t->devs.push_back(std::move(d));
  return TACOS_OK;
}
}  // namespace

extern "C" int tacos_load_topology(int32_t n_npus, int32_t n_links, const int32_t *src, const int32_t *dst,
                                   const uint32_t *alpha_ns, const uint32_t *bw, tacos_topology **out) {
  if (out) *out = nullptr;
  if (!out || !src || !dst || !alpha_ns || !bw) return fail(TACOS_E_INVALID_ARG, "null argument");
  if (n_npus < 2) return fail(TACOS_E_INVALID_ARG, "n_npus = %d < 2", n_npus);
  if (n_links < 1 || n_links >= (1 << 24)) return fail(TACOS_E_INVALID_ARG, "n_links = %d out of [1, 2^24)", n_links);
  std::unique_ptr<tacos_topology> t(new (std::nothrow) tacos_topology());
  if (!t) return fail(TACOS_E_NOMEM, "host allocation failed");
  t->N = n_npus;
  t->L = n_links;
  t->src.assign(src, src + n_links);
  t->dst.assign(dst, dst + n_links);
  t->alpha.assign(alpha_ns, alpha_ns + n_links);
  t->bw.assign(bw, bw + n_links);
  // (src, dst) -> link id: open addressing, linear probing, load <= 1/2
  size_t cap = 16;
  uint32_t lg = 4;
  while (cap < (size_t)n_links * 2) {
    cap <<= 1;
    ++lg;
  }
  std::vector<uint64_t> hkey(cap, ~0ull);
  std::vector<int32_t> hval(cap, -1);
  auto slot_of = [&](uint64_t key) {  // Fibonacci hashing: the top lg bits of the product
    size_t h = (size_t)((key * 0x9E3779B97F4A7C15ull) >> (64u - lg));
    while (hkey[h] != ~0ull && hkey[h] != key) h = (h + 1) & (cap - 1);
    return h;
  };
  for (int32_t l = 0; l < n_links; ++l) {
    const int32_t a = src[l], b = dst[l];
    if (a < 0 || a >= n_npus || b < 0 || b >= n_npus)
      return fail(TACOS_E_TOPOLOGY, "link %d: endpoint out of range (%d -> %d)", l, a, b);
    if (a == b) return fail(TACOS_E_TOPOLOGY, "link %d: self-loop on NPU %d", l, a);
    if (bw[l] == 0) return fail(TACOS_E_TOPOLOGY, "link %d: bandwidth 0", l);
    const uint64_t key = ((uint64_t)(uint32_t)a << 32) | (uint32_t)b;
    const size_t h = slot_of(key);
    if (hkey[h] == key) return fail(TACOS_E_TOPOLOGY, "link %d duplicates link %d (%d -> %d)", l, hval[h], a, b);
    hkey[h] = key;
    hval[h] = l;
  }
  t->rev.assign(n_links, -1);
  for (int32_t l = 0; l < n_links; ++l) {
    const uint64_t key = ((uint64_t)(uint32_t)dst[l] << 32) | (uint32_t)src[l];
    const size_t h = slot_of(key);
    if (hkey[h] == key) t->rev[l] = hval[h];
  }
  // CSR per orientation; within a destination, positions in ascending link id
  for (int o = 0; o < 2; ++o) {
    const int32_t *key = o == 0 ? dst : src;
    const int32_t *oth = o == 0 ? src : dst;
    auto &ptr = t->in_ptr[o];
    ptr.assign(n_npus + 1, 0);
    for (int32_t l = 0; l < n_links; ++l) ptr[key[l] + 1]++;
    for (int32_t d = 0; d < n_npus; ++d) ptr[d + 1] += ptr[d];
    std::vector<uint32_t> fill(ptr.begin(), ptr.end() - 1);
    t->pos_lid[o].resize(n_links);
    t->pos_src[o].resize(n_links);
    t->pos_dst[o].resize(n_links);
    for (int32_t l = 0; l < n_links; ++l) {
      const uint32_t p = fill[key[l]]++;
      t->pos_lid[o][p] = (uint32_t)l;
      t->pos_src[o][p] = (uint32_t)oth[l];
      t->pos_dst[o][p] = (uint32_t)key[l];
    }
  }
  t->strongly_connected = reach_all(n_npus, t->in_ptr[0], t->pos_src[0]) && reach_all(n_npus, t->in_ptr[1], t->pos_src[1]);

  // (the device copy is made by the first plan that uses the topology, on its stream)
  int dev = -1;
  int n = 0;
  if (cudaGetDeviceCount(&n) == cudaSuccess && n > 0 && cudaGetDevice(&dev) == cudaSuccess) t->device = dev;
  else cudaGetLastError();
  *out = t.release();
  return TACOS_OK;
}

extern "C" void tacos_free_topology(tacos_topology *t) { delete t; }
extern "C" int32_t tacos_topology_num_npus(const tacos_topology *t) { return t ? t->N : -1; }
extern "C" int32_t tacos_topology_num_links(const tacos_topology *t) { return t ? t->L : -1; }
extern "C" int tacos_topology_strongly_connected(const tacos_topology *t) { return t && t->strongly_connected ? 1 : 0; }

extern "C" int tacos_link_costs(const tacos_topology *t, uint64_t chunk_bytes, uint32_t f, uint32_t *w_out) {
  if (!t || !w_out) return fail(TACOS_E_INVALID_ARG, "null argument");
  std::vector<uint32_t> w;
  int rc = link_costs(t, chunk_bytes, f ? f : 1u, w);
  if (rc) return rc;
  std::memcpy(w_out, w.data(), w.size() * 4);
  return TACOS_OK;
}

extern "C" int tacos_is_symmetric(const tacos_topology *t, uint64_t chunk_bytes, uint32_t f) {
  if (!t) return 0;
  std::vector<uint32_t> w;
  if (link_costs(t, chunk_bytes, f ? f : 1u, w)) return 0;
  return symmetric_for(t, w) ? 1 : 0;
}

// ---------------------------------------------------------------------------
// plan: device state for a batch of topologies sharing the params
// ---------------------------------------------------------------------------
namespace {
struct Part {
  const tacos_topology *topo = nullptr;
  const TopoDev *td = nullptr;  // the topology's arrays on the plan's device
  uint32_t N = 0, L = 0, C = 0, k = 0, Wp = 0, P = 0, VPL = 0;
  bool custom = false, symmetric = false, rs_search = false;
  uint32_t rs_base = 0;  // first job of the G^T (sigma 1) search: S, or 0 when only the RS phase is searched
  bool windowed = false;  // searched by the windowed event loop (records per destination, sorted at emission)
  bool lockstep = false;  // lock-step loop: records in (t_start, CTA, position) order, ranked by link at emission
  uint64_t required = 0;
  uint64_t cap = 0;  // send records per job (= required without relays)
  std::vector<uint32_t> w;
  DevTopo htopo[2];
  DevTopo *d_topo[2] = {nullptr, nullptr};
  uint32_t *d_w = nullptr;
  uint32_t job_base = 0, n_jobs = 0;  // jobs [job_base, job_base + n_jobs): S (sigma 0) then S (sigma 1)
  Rec *d_rec = nullptr;               // n_jobs * required records
  const uint32_t *d_rec_off = nullptr;  // windowed loop: per-destination record offsets (N + 1)
  uint64_t *d_keys = nullptr;         // 2
  uint64_t *d_stats = nullptr;        // 5
  uint64_t *d_times_ag = nullptr, *d_times_rs = nullptr;
};
struct Group {
  uint32_t P, VPL;
  Layout lay;
  uint32_t job_begin, job_end;
};
}  // namespace

struct tacos_plan {
  int device = -1;
  tacos_synth_params p{};
  std::vector<uint32_t> pre, post;  // CUSTOM copies (unpadded rows)
  std::vector<Part> parts;
  std::vector<Group> groups;
  std::vector<Job> jobs;
  Job *d_jobs = nullptr;
  JobOut *d_outs = nullptr;
  unsigned char *d_rows = nullptr, *d_links = nullptr;
  void *d_sort = nullptr;
  size_t sort_bytes = 0;
  uint64_t *h_small = nullptr;  // pinned: per part kSmallWords {keys[2], stats}
  DevBuf h_small_buf;
  DevBuf stage_buf;             // pinned staging block of the plan's one H2D upload
  std::vector<DevBuf> bufs;
  uint32_t last_launches = 0;
  unsigned long long *d_trace = nullptr;
  unsigned long long *d_count = nullptr;  // compact_sends result (relays)
  cudaEvent_t done = nullptr;             // recorded after the last search / emit work on its stream
  ~tacos_plan() {
    // blocks return to the caching pool: wait for the plan's in-flight kernels first
    if (done) {
      cudaEventSynchronize(done);
      cudaEventDestroy(done);
      cudaGetLastError();
    }
    for (auto &b : bufs) device_pool().release(b.dev, b.p, b.cls);
    if (h_small_buf.p) pinned_pool().release(h_small_buf.dev, h_small_buf.p, h_small_buf.cls);
    if (stage_buf.p) pinned_pool().release(stage_buf.dev, stage_buf.p, stage_buf.cls);
  }
};

namespace {
// collective classes (tacos.h): named = rooted collectives of row f2
bool coll_named(int c) { return c >= TACOS_BROADCAST && c <= TACOS_GATHER; }
bool coll_custom(int c) { return c == TACOS_CUSTOM || coll_named(c); }
bool coll_need_rs(int c) {
  return c == TACOS_REDUCE_SCATTER || c == TACOS_ALL_REDUCE || c == TACOS_REDUCE || c == TACOS_GATHER;
}
bool coll_need_ag(int c) { return !(c == TACOS_REDUCE_SCATTER || c == TACOS_REDUCE || c == TACOS_GATHER); }
bool coll_relay(const tacos_synth_params *p) {
  return (p->flags & TACOS_FLAG_RELAY) != 0u || p->collective == TACOS_SCATTER || p->collective == TACOS_GATHER;
}

// Pre/post rows (W0 = ceil(C/32) words per NPU) of the searched forward problem
// (§II.A; P:L70 Fig. CollectiveDefinition): the caller's for CUSTOM; for
// BROADCAST / REDUCE the Broadcast from root, for SCATTER / GATHER the Scatter
// from root (REDUCE and GATHER are its inverse on G^T).
int problem_bits(uint32_t N, const tacos_synth_params *p, uint32_t &C, std::vector<uint32_t> &pre,
                 std::vector<uint32_t> &post) {
  const int c = p->collective;
  if (c == TACOS_CUSTOM) {
    C = p->n_chunks;
    const uint32_t W0 = (C + 31u) / 32u;
    pre.assign(p->pre_bits, p->pre_bits + (size_t)N * W0);
    post.assign(p->post_bits, p->post_bits + (size_t)N * W0);
    return TACOS_OK;
  }
  const uint32_t k = p->chunks_per_npu, root = p->root;
  if (root >= N) return fail(TACOS_E_INVALID_ARG, "root %u out of range", root);
  const bool bcast = c == TACOS_BROADCAST || c == TACOS_REDUCE;
  const uint64_t C64 = bcast ? (uint64_t)k : (uint64_t)N * k;
  if (C64 > kMaxChunks) return fail(TACOS_E_OVERFLOW, "C = %llu chunks exceeds %u", (unsigned long long)C64, kMaxChunks);
  C = (uint32_t)C64;
  const uint32_t W0 = (C + 31u) / 32u;
  pre.assign((size_t)N * W0, 0u);
  post.assign((size_t)N * W0, 0u);
  auto set = [&](std::vector<uint32_t> &v, uint32_t x, uint32_t ch) { v[(size_t)x * W0 + (ch >> 5)] |= 1u << (ch & 31u); };
  for (uint32_t ch = 0; ch < C; ++ch) {
    set(pre, root, ch);
    set(post, root, ch);
    if (bcast)
      for (uint32_t x = 0; x < N; ++x) set(post, x, ch);
    else
      set(post, ch / k, ch);  // Scatter: NPU x requires chunks x*k .. x*k+k-1
  }
  return TACOS_OK;
}

// R22 relay masks in the position order of orientation o (0: links as given,
// 1: reversed): allow[q] = post[d] plus the chunks c that d may relay, i.e. d does
// not require c and is one hop closer than s to some NPU r that requires c and
// lacks it at the start (chunks every NPU requires have no relays).  Wp words per row.
// One backward BFS per distinct requirer r gives the positions on its shortest paths
// (dist_r[s] = dist_r[d] + 1) as a bitset over positions; a chunk's relay positions are
// the OR of its requirers' bitsets: O(R (N + L) + C R L / 64) instead of a BFS per
// (chunk, requirer) pair.
void relay_allow(const tacos_topology *t, int o, uint32_t C, uint32_t Wp, const std::vector<uint32_t> &pre,
                 const std::vector<uint32_t> &post, std::vector<uint32_t> &allow) {
  const uint32_t N = (uint32_t)t->N, L = (uint32_t)t->L, W0 = (C + 31u) / 32u;
  const uint32_t LW = (L + 63u) / 64u;  // u64 words of a position bitset
  const auto &ptr = t->in_ptr[o];
  const auto &ps = t->pos_src[o];
  const auto &pd = t->pos_dst[o];
  auto bit = [&](const std::vector<uint32_t> &v, uint32_t x, uint32_t ch) {
    return ((v[(size_t)x * W0 + (ch >> 5)] >> (ch & 31u)) & 1u) != 0u;
  };
  allow.assign((size_t)L * Wp, 0u);
  for (uint32_t q = 0; q < L; ++q)
    for (uint32_t i = 0; i < W0; ++i) allow[(size_t)q * Wp + i] = post[(size_t)pd[q] * W0 + i];
  // chunks with relays: some NPU requires and lacks c, and some NPU does not require c
  std::vector<std::vector<uint32_t>> req(C);
  std::vector<char> need_bfs(N, 0);
  for (uint32_t ch = 0; ch < C; ++ch) {
    bool relayable = false;
    for (uint32_t x = 0; x < N && !relayable; ++x) relayable = !bit(post, x, ch);
    if (!relayable) continue;
    for (uint32_t x = 0; x < N; ++x)
      if (bit(post, x, ch) && !bit(pre, x, ch)) {
        req[ch].push_back(x);
        need_bfs[x] = 1;
      }
  }
  // per requirer: positions on its shortest paths (BFS backwards along in-links from r)
  std::vector<uint32_t> slot(N, ~0u);
  std::vector<uint64_t> onpath;
  std::vector<int32_t> dist(N);
  std::vector<uint32_t> queue;
  uint32_t n_req = 0;
  for (uint32_t r = 0; r < N; ++r) {
    if (!need_bfs[r]) continue;
    slot[r] = n_req++;
    onpath.resize((size_t)n_req * LW, 0ull);
    std::fill(dist.begin(), dist.end(), -1);
    queue.assign(1, r);
    dist[r] = 0;
    for (size_t h = 0; h < queue.size(); ++h) {
      const uint32_t y = queue[h];
      for (uint32_t q = ptr[y]; q < ptr[y + 1]; ++q) {
        const uint32_t x = ps[q];
        if (dist[x] < 0) {
          dist[x] = dist[y] + 1;
          queue.push_back(x);
        }
      }
    }
    uint64_t *row = &onpath[(size_t)slot[r] * LW];
    for (uint32_t q = 0; q < L; ++q) {
      const int32_t ds = dist[ps[q]], dd = dist[pd[q]];
      if (dd >= 0 && ds == dd + 1) row[q >> 6] |= 1ull << (q & 63u);
    }
  }
  std::vector<uint64_t> acc(LW);
  for (uint32_t ch = 0; ch < C; ++ch) {
    if (req[ch].empty()) continue;
    std::fill(acc.begin(), acc.end(), 0ull);
    for (uint32_t r : req[ch]) {
      const uint64_t *row = &onpath[(size_t)slot[r] * LW];
      for (uint32_t i = 0; i < LW; ++i) acc[i] |= row[i];
    }
    for (uint32_t i = 0; i < LW; ++i)
      for (uint64_t m = acc[i]; m; m &= m - 1) {
        const uint32_t q = i * 64u + (uint32_t)__builtin_ctzll(m);
        if (!bit(post, pd[q], ch)) allow[(size_t)q * Wp + (ch >> 5)] |= 1u << (ch & 31u);
      }
  }
}

int validate_params(const tacos_synth_params *p) {
  if (!p) return fail(TACOS_E_INVALID_ARG, "null params");
  if (p->collective < TACOS_ALL_GATHER || p->collective > TACOS_GATHER)
    return fail(TACOS_E_INVALID_ARG, "bad collective %d", p->collective);
  if (coll_relay(p) && !coll_custom(p->collective))
    return fail(TACOS_E_INVALID_ARG, "relays apply to CUSTOM and rooted collectives");
  if (coll_relay(p) && (p->flags & TACOS_FLAG_LITERAL))
    return fail(TACOS_E_INVALID_ARG, "relays are not supported by the paper-literal variant");
  if (p->chunk_bytes == 0) return fail(TACOS_E_INVALID_ARG, "chunk_bytes = 0");
  if (p->n_seeds < 1) return fail(TACOS_E_INVALID_ARG, "n_seeds = 0");
  if ((uint64_t)p->seed_offset + p->n_seeds > (1ull << kKeySeedBits))
    return fail(TACOS_E_OVERFLOW, "seed index beyond 2^%d", kKeySeedBits);
  if (p->collective == TACOS_CUSTOM) {
    if (!p->pre_bits || !p->post_bits || p->n_chunks < 1) return fail(TACOS_E_INVALID_ARG, "CUSTOM needs pre/post/n_chunks");
  } else if (p->chunks_per_npu < 1) {
    return fail(TACOS_E_INVALID_ARG, "chunks_per_npu = 0");
  }
  return TACOS_OK;
}

uint32_t pow2_at_least(uint32_t x) {
  uint32_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// st: the stream the plan's first search will run on; the one staged upload of the plan's
// host-built arrays is ordered on it (no synchronization).  nullptr: upload on the legacy
// stream and synchronize (tacos_plan_create, whose caller's stream is not known yet).
// Cluster size chosen for a launch shape (per device), so repeated syntheses skip the
// occupancy queries.
struct ClusterKey {
  int dev;
  uint32_t N, L, W, P, V, jobs, reg_path, masked, worklist, smem, win, deg;
  bool operator<(const ClusterKey &o) const {
    return std::tie(dev, N, L, W, P, V, jobs, reg_path, masked, worklist, smem, win, deg) <
           std::tie(o.dev, o.N, o.L, o.W, o.P, o.V, o.jobs, o.reg_path, o.masked, o.worklist, o.smem, o.win, o.deg);
  }
};
std::mutex g_cluster_mu;
std::map<ClusterKey, uint32_t> &cluster_cache() {
  static auto *m = new std::map<ClusterKey, uint32_t>();
  return *m;
}
bool cluster_cache_get(const ClusterKey &k, uint32_t *q) {
  std::lock_guard<std::mutex> g(g_cluster_mu);
  auto it = cluster_cache().find(k);
  if (it == cluster_cache().end()) return false;
  *q = it->second;
  return true;
}
void cluster_cache_put(const ClusterKey &k, uint32_t q) {
  std::lock_guard<std::mutex> g(g_cluster_mu);
  cluster_cache()[k] = q;
}

// Host-built arrays of a plan, staged into one host buffer and shipped with one H2D copy
// into one device block: reserve() / add() return byte offsets; device addresses are
// base + offset once the block exists (structs holding device pointers are written into
// their reserved slots after that).
struct PlanStage {
  std::vector<unsigned char> host;
  size_t add(const void *src, size_t n) {
    const size_t off = reserve(n);
    if (n) std::memcpy(host.data() + off, src, n);
    return off;
  }
  size_t reserve(size_t n) {
    const size_t off = (host.size() + 255) / 256 * 256;
    host.resize(off + n + 16, 0);
    return off;
  }
  template <typename T>
  void put(size_t off, const T &v) { std::memcpy(host.data() + off, &v, sizeof(T)); }
};

int plan_build(const tacos_topology *const *topos, uint32_t n_topos, const tacos_synth_params *p, tacos_plan **out,
               cudaStream_t st = nullptr, bool sync = true) {
  *out = nullptr;
  int rc = validate_params(p);
  if (rc) return rc;
  int dev = -1;
  if ((rc = cuda_device_ok(&dev))) return rc;
  std::unique_ptr<tacos_plan> pl(new (std::nothrow) tacos_plan());
  if (!pl) return fail(TACOS_E_NOMEM, "host allocation failed");
  pl->device = dev;
  pl->p = *p;
  if (pl->p.time_unit_ns == 0) pl->p.time_unit_ns = 1;
  const uint32_t S = p->n_seeds;
  const bool custom = coll_custom(p->collective);
  const bool need_rs = coll_need_rs(p->collective);
  const bool relay = coll_relay(p);
  const bool record = (p->flags & TACOS_FLAG_NO_SCHEDULE) == 0;

  // ---- per-topology host preparation ----
  pl->parts.resize(n_topos);
  uint32_t n_jobs = 0;
  for (uint32_t i = 0; i < n_topos; ++i) {
    const tacos_topology *t = topos[i];
    if (!t) return fail(TACOS_E_INVALID_ARG, "null topology %u", i);
    Part &pt = pl->parts[i];
    pt.topo = t;
    if ((rc = topo_on_device(t, dev, &pt.td, st))) return rc;
    pt.N = (uint32_t)t->N;
    pt.L = (uint32_t)t->L;
    pt.custom = custom;
    if (custom) {
      if (n_topos != 1) return fail(TACOS_E_INVALID_ARG, "CUSTOM and rooted collectives are not batched over topologies");
      if ((rc = problem_bits(pt.N, p, pt.C, pl->pre, pl->post))) return rc;
      pt.k = 0;
    } else {
      const uint64_t C = (uint64_t)pt.N * p->chunks_per_npu;
      if (C > kMaxChunks) return fail(TACOS_E_OVERFLOW, "C = %llu chunks exceeds %u", (unsigned long long)C, kMaxChunks);
      pt.C = (uint32_t)C;
      pt.k = p->chunks_per_npu;
      if (!t->strongly_connected)
        return fail(TACOS_E_UNREACHABLE, "topology %u is not strongly connected", i);
    }
    if (pt.C > kMaxChunks) return fail(TACOS_E_OVERFLOW, "C = %u chunks exceeds %u", pt.C, kMaxChunks);
    if ((rc = link_costs(t, p->chunk_bytes, pl->p.time_unit_ns, pt.w))) return rc;
    pt.symmetric = symmetric_for(t, pt.w);
    pt.rs_search = need_rs && !pt.symmetric;
    const uint32_t W0 = (pt.C + 31u) / 32u;
    const uint32_t vec = (W0 + 3u) / 4u;
    pt.P = std::min<uint32_t>(32u, pow2_at_least((vec + 3u) / 4u));  // up to 4 vectors per lane
    if (p->flags & TACOS_FLAG_LITERAL) pt.P = 32u;  // literal variant: one warp per destination
    if (const char *env = getenv("TACOS_LANES")) {  // tuning override: lanes per destination row
      const uint32_t want = (uint32_t)atoi(env);
      if (want >= 1 && want <= 32 && (want & (want - 1)) == 0 && want <= pow2_at_least(vec) &&
          (vec + want - 1) / want <= 4)
        pt.P = want;
    }
    pt.VPL = (vec + pt.P - 1u) / pt.P;
    if (pt.VPL == 3) pt.VPL = 4;
    if (pt.VPL > (uint32_t)kMaxVPL) return fail(TACOS_E_OVERFLOW, "C too large");
    pt.Wp = 4u * pt.P * pt.VPL;
    if (custom) {
      const size_t words = (size_t)pt.N * W0;
      uint64_t req = 0, held0 = 0;
      for (size_t q = 0; q < words; ++q) {
        if (pl->pre[q] & ~pl->post[q]) return fail(TACOS_E_INVALID_ARG, "pre is not a subset of post (row %zu)", q / W0);
        const uint32_t valid = (q % W0 == W0 - 1 && (pt.C & 31u)) ? ((1u << (pt.C & 31u)) - 1u) : 0xFFFFFFFFu;
        if ((pl->pre[q] | pl->post[q]) & ~valid) return fail(TACOS_E_INVALID_ARG, "bits beyond C set");
        req += (uint64_t)__builtin_popcount(pl->post[q] & ~pl->pre[q]);
        held0 += (uint64_t)__builtin_popcount(pl->pre[q]);
      }
      pt.required = req;
      // records per job: every (NPU, chunk) pair is delivered at most once (relays add sends)
      pt.cap = relay ? (uint64_t)pt.N * pt.C - held0 : req;
    } else {
      pt.required = (uint64_t)pt.C * (pt.N - 1u);
      pt.cap = pt.required;
    }
    pt.job_base = n_jobs;
    // jobs: S forward searches on G (sigma 0) unless only the RS phase is needed and it is
    // searched on G^T, then S searches on G^T (sigma 1) for an asymmetric RS phase (R9)
    const bool fwd = !pt.rs_search || coll_need_ag(p->collective);
    pt.rs_base = fwd ? S : 0u;
    pt.n_jobs = (fwd ? S : 0u) + (pt.rs_search ? S : 0u);
    n_jobs += pt.n_jobs;
  }

  // ---- groups by row shape: one launch each, max layout over members ----
  std::vector<uint32_t> order(n_topos);
  for (uint32_t i = 0; i < n_topos; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
    return std::make_pair(pl->parts[a].P, pl->parts[a].VPL) < std::make_pair(pl->parts[b].P, pl->parts[b].VPL);
  });
  int smem_optin = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const size_t smem_limit = (size_t)smem_optin > 1024 ? (size_t)smem_optin - 1024 : 0;
  int n_sms = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, dev));
  // re-number jobs in group order
  n_jobs = 0;
  for (size_t gi = 0; gi < order.size();) {
    const uint32_t P0 = pl->parts[order[gi]].P, V0 = pl->parts[order[gi]].VPL;
    uint32_t maxN = 0, maxL = 0, maxW = 0;
    size_t gj = gi;
    const uint32_t begin = n_jobs;
    while (gj < order.size() && pl->parts[order[gj]].P == P0 && pl->parts[order[gj]].VPL == V0) {
      Part &pt = pl->parts[order[gj]];
      maxN = std::max(maxN, pt.N);
      maxL = std::max(maxL, pt.L);
      maxW = std::max(maxW, pt.Wp);
      pt.job_base = n_jobs;
      n_jobs += pt.n_jobs;
      ++gj;
    }
    Group g;
    g.P = P0;
    g.VPL = V0;
    g.lay = make_layout(maxN, maxL, maxW, P0, V0, smem_limit, n_jobs - begin, (uint32_t)n_sms);
    uint32_t max_deg = 0;
    for (size_t gk = gi; gk < gj; ++gk) {
      const tacos_topology *tt = pl->parts[order[gk]].topo;
      for (int o = 0; o < 2; ++o)
        for (int32_t d = 0; d < tt->N; ++d) max_deg = std::max(max_deg, tt->in_ptr[o][d + 1] - tt->in_ptr[o][d]);
    }
    g.lay.reg_path = max_deg <= 8u ? 1u : 0u;
    if (p->flags & TACOS_FLAG_LITERAL) {
      if (max_deg > 32u) return fail(TACOS_E_INVALID_ARG, "literal variant supports in-degree <= 32 (got %u)", max_deg);
      if (!g.lay.links_in_smem) return fail(TACOS_E_OVERFLOW, "literal variant: link state does not fit shared memory");
      g.lay.cluster = 1;
    }
    if (const char *env = getenv("TACOS_REG_PATH")) g.lay.reg_path = (uint32_t)atoi(env);
    g.lay.masked = relay ? 1u : 0u;
    if (relay) g.lay.reg_path = 0u;  // the masked kernels are instantiated on the shared-memory ranking path
    // worklist for sparse events: several distinct link costs free only some links per event
    bool multi_w = false;
    for (size_t gk = gi; gk < gj && !multi_w; ++gk) {
      const auto &wv = pl->parts[order[gk]].w;
      for (size_t l = 1; l < wv.size(); ++l)
        if (wv[l] != wv[0]) {
          multi_w = true;
          break;
        }
    }
    g.lay.worklist = (multi_w && g.lay.reg_path) ? 1u : 0u;  // measured: helps the mesh (config 4), not config 5
    if (const char *env = getenv("TACOS_WORKLIST")) g.lay.worklist = (uint32_t)atoi(env);
    // Windowed event loop (greedy_kernel.cuh): several link costs, wide rows on the
    // register path, no relays, link-first; window W = the group's smallest link cost (capped),
    // every cost < 2^31 (busy offsets from a window start stay below 2^32).  TACOS_WINDOW=0: off.
    uint32_t win = 0;
    {
      uint32_t w_min = ~0u, w_max = 0;
      for (size_t gk = gi; gk < gj; ++gk)
        for (uint32_t x : pl->parts[order[gk]].w) {
          w_min = std::min(w_min, x);
          w_max = std::max(w_max, x);
        }
      const char *env = getenv("TACOS_WINDOW");
      const bool want = env ? atoi(env) != 0 : true;
      if (want && multi_w && g.lay.reg_path && P0 > 2 && !relay && !(p->flags & TACOS_FLAG_LITERAL) &&
          w_max < (1u << 31))
        win = std::min<uint32_t>(w_min, kWinBits);
    }
    auto finish_layout = [&](Layout &lq) {
      lq.reg_path = g.lay.reg_path;
      lq.masked = g.lay.masked;
      lq.worklist = g.lay.worklist;
      add_window(lq, maxN, win, max_deg);
      if (win && (size_t)lq.smem_bytes > smem_limit) {  // does not fit: the per-event loop
        Layout l2 = make_layout(maxN, maxL, maxW, P0, V0, smem_limit, n_jobs - begin, (uint32_t)n_sms, lq.cluster);
        l2.reg_path = lq.reg_path;
        l2.masked = lq.masked;
        l2.worklist = lq.worklist;
        add_window(l2, maxN, 0, 0);
        lq = l2;
      }
      // Lock-step loop (greedy_kernel.cuh): one link cost per topology, one lane per
      // destination (register or shared-memory ranking path), AG-type problem without relays: every send started at t
      // ends at the next event t + w, so the walkers write the arrivals themselves (held rows
      // double-buffered by event parity) and an event needs one cluster barrier.  TACOS_LOCKSTEP=0: off.
      const char *env_ls = getenv("TACOS_LOCKSTEP");
      if (!win && !multi_w && P0 == 1u && !relay && !custom && !(p->flags & TACOS_FLAG_LITERAL) &&
          !lq.worklist && (!env_ls || atoi(env_ls) != 0)) {
        const uint32_t Q = lq.cluster;
        uint32_t pos_cap = 0;
        for (size_t gk = gi; gk < gj; ++gk) {
          const tacos_topology *tt = pl->parts[order[gk]].topo;
          const uint32_t n = (uint32_t)tt->N, chunk_n = (n + Q - 1u) / Q;
          for (int o = 0; o < 2; ++o)
            for (uint32_t r = 0; r < Q; ++r) {
              const uint32_t lo = std::min(n, r * chunk_n), hi = std::min(n, lo + chunk_n);
              pos_cap = std::max(pos_cap, tt->in_ptr[o][hi] - tt->in_ptr[o][lo]);
            }
        }
        add_lockstep(lq, maxN, maxL, std::max(pos_cap, 1u), smem_limit);
      }
      if (lq.big && !(lq.reg_path && lq.rows_in_smem && lq.links_in_smem && !lq.masked)) layout_drop_big(lq);
    };
    finish_layout(g.lay);
    // Cluster size: the largest Q <= 8 (any size, not only powers of two) with jobs * Q <= #SMs,
    // >= 64 destinations per CTA, and every job's cluster co-resident on the chip (asked of the
    // occupancy calculator for the kernel this layout selects: only 15 clusters of 8 fit on a
    // B200, so config 4's 16 jobs take Q = 6, 579 ms vs 625 ms at Q = 4; waves of clusters
    // would double the time). TACOS_CLUSTER overrides.
    // (the choice is cached per shape: the occupancy queries cost more than a small synthesis)
    const ClusterKey ck{dev, maxN, maxL, maxW, P0, V0, n_jobs - begin, g.lay.reg_path, g.lay.masked, g.lay.worklist,
                        (uint32_t)smem_limit, win, max_deg};
    uint32_t cached_q = 0;
    if (!(p->flags & TACOS_FLAG_LITERAL) && !getenv("TACOS_CLUSTER") && cluster_cache_get(ck, &cached_q)) {
      if (cached_q != g.lay.cluster) {
        Layout lq = make_layout(maxN, maxL, maxW, P0, V0, smem_limit, n_jobs - begin, (uint32_t)n_sms, cached_q);
        finish_layout(lq);
        g.lay = lq;
      }
    } else if (!(p->flags & TACOS_FLAG_LITERAL) && !getenv("TACOS_CLUSTER")) {
      const uint32_t jobs = n_jobs - begin;
      for (uint32_t q = kMaxCluster; q > g.lay.cluster; --q) {
        if ((uint64_t)jobs * q > (uint64_t)n_sms || maxN / q < 64u) continue;
        Layout lq = make_layout(maxN, maxL, maxW, P0, V0, smem_limit, jobs, (uint32_t)n_sms, q);
        finish_layout(lq);
        int n_active = 0;
        g_occ_query = &n_active;
        launch_greedy(lq, P0, V0, nullptr, jobs, nullptr, nullptr);
        g_occ_query = nullptr;
        if ((uint32_t)n_active >= jobs) {
          g.lay = lq;
          break;
        }
      }
      cluster_cache_put(ck, g.lay.cluster);
    }
    if ((size_t)g.lay.smem_bytes > smem_limit)  // the per-NPU / per-link arrays that always stay on chip
      return fail(TACOS_E_OVERFLOW, "search state needs %u B of shared memory per CTA (limit %zu)", g.lay.smem_bytes,
                  smem_limit);
    g.job_begin = begin;
    g.job_end = n_jobs;
    for (size_t gk = gi; gk < gj; ++gk) {
      pl->parts[order[gk]].windowed = g.lay.window != 0u;
      pl->parts[order[gk]].lockstep = g.lay.lockstep != 0u;
    }
    pl->groups.push_back(g);
    gi = gj;
  }

  // ---- device memory: big scratch blocks, then one staged block for everything host-built ----
  auto &bufs = pl->bufs;
  void *vp = nullptr;
  size_t rows_total = 0, links_total = 0;
  for (auto &g : pl->groups) {
    const size_t nj = g.job_end - g.job_begin;
    if (!g.lay.rows_in_smem) rows_total += nj * g.lay.rows_bytes;
    if (!g.lay.links_in_smem) links_total += nj * g.lay.links_bytes;
  }
  if (rows_total) {
    if ((rc = dev_alloc(bufs, dev, rows_total, &vp))) return rc;
    pl->d_rows = reinterpret_cast<unsigned char *>(vp);
  }
  if (links_total) {
    if ((rc = dev_alloc(bufs, dev, links_total, &vp))) return rc;
    pl->d_links = reinterpret_cast<unsigned char *>(vp);
  }
  uint64_t max_M = 0;
  for (uint32_t i = 0; i < n_topos; ++i) {
    Part &pt = pl->parts[i];
    if (record) {
      if ((rc = dev_alloc(bufs, dev, sizeof(Rec) * pt.cap * pt.n_jobs, &vp))) return rc;
      pt.d_rec = reinterpret_cast<Rec *>(vp);
    }
    if ((need_rs || (p->flags & TACOS_FLAG_LITERAL) || pt.windowed || pt.lockstep) && record) max_M = std::max(max_M, pt.cap);
  }
  if (max_M) {
    pl->sort_bytes = rs_sort_scratch_bytes(max_M);
    if ((rc = dev_alloc(bufs, dev, pl->sort_bytes, &pl->d_sort))) return rc;
  }
  PlanStage sg;
  const size_t o_outs = sg.reserve(sizeof(JobOut) * n_jobs), o_count = sg.reserve(8);
  struct PartOffs {
    size_t w, pos_w[2], allow[2] = {0, 0}, pre = 0, post = 0, topo[2], keys, times_ag, times_rs = 0, rec_off = 0;
    size_t orig = 0, in_ptr[2] = {0, 0}, pos_lid[2] = {0, 0}, pos_src[2] = {0, 0}, pos_dst[2] = {0, 0};
    bool relabel = false;
  };
  std::vector<PartOffs> po(n_topos);
  for (uint32_t i = 0; i < n_topos; ++i) {
    Part &pt = pl->parts[i];
    const tacos_topology *t = pt.topo;
    PartOffs &o = po[i];
    o.w = sg.add(pt.w.data(), pt.w.size() * 4);
    // Windowed parts on a cluster: NPUs relabeled so that each CTA's contiguous block of kernel
    // ids holds several id blocks spread over the topology (block b of ~N / (Q m) ids goes to CTA
    // b mod Q), balancing the CTAs of a cluster (a CTA of border NPUs was the slowest).  The result
    // is unchanged: chunk ids (the AG init reads the original id), link ids, the Philox counters
    // and the in-link order of every NPU stay the same; records carry link ids.
    std::vector<uint32_t> orig;  // kernel id -> original id
    uint32_t Qg = 1;
    for (const Group &g : pl->groups)
      if (pt.job_base >= g.job_begin && pt.job_base < g.job_end) Qg = g.lay.cluster ? g.lay.cluster : 1u;
    uint32_t mil = 8;  // blocks per CTA (config 4: 249 / 235 / 233 / 231 ms at 0 (off) / 4 / 2 / 8)
    if (const char *env = getenv("TACOS_INTERLEAVE")) mil = (uint32_t)std::max(0, atoi(env));
    o.relabel = pt.windowed && Qg > 1 && mil > 0 && pt.N >= 2 * Qg * mil;
    std::vector<uint32_t> newid;
    if (o.relabel) {
      const uint32_t nb = Qg * mil, bs = (pt.N + nb - 1) / nb;
      orig.resize(pt.N);
      for (uint32_t x = 0; x < pt.N; ++x) orig[x] = x;
      std::stable_sort(orig.begin(), orig.end(), [&](uint32_t a, uint32_t b) {
        return (a / bs) % Qg < (b / bs) % Qg || ((a / bs) % Qg == (b / bs) % Qg && a < b);
      });
      newid.resize(pt.N);
      for (uint32_t x = 0; x < pt.N; ++x) newid[orig[x]] = x;
      o.orig = sg.add(orig.data(), orig.size() * 4);
      for (int q = 0; q < 2; ++q) {  // the CSR in kernel ids, each NPU's in-links in their original order
        std::vector<uint32_t> ip(pt.N + 1, 0u), lid(pt.L), src(pt.L), dst(pt.L);
        uint32_t k = 0;
        for (uint32_t x2 = 0; x2 < pt.N; ++x2) {
          const uint32_t x = orig[x2];
          ip[x2] = k;
          for (uint32_t p = t->in_ptr[q][x]; p < t->in_ptr[q][x + 1]; ++p, ++k) {
            lid[k] = t->pos_lid[q][p];
            src[k] = newid[t->pos_src[q][p]];
            dst[k] = x2;
          }
        }
        ip[pt.N] = k;
        o.in_ptr[q] = sg.add(ip.data(), ip.size() * 4);
        o.pos_lid[q] = sg.add(lid.data(), lid.size() * 4);
        o.pos_src[q] = sg.add(src.data(), src.size() * 4);
        o.pos_dst[q] = sg.add(dst.data(), dst.size() * 4);
        std::vector<uint32_t> pw(pt.L);
        for (uint32_t x = 0; x < pt.L; ++x) pw[x] = pt.w[lid[x]];
        o.pos_w[q] = sg.add(pw.data(), pw.size() * 4);
      }
    } else {
      for (int q = 0; q < 2; ++q) {  // per-position costs of both orientations
        std::vector<uint32_t> pw(pt.L);
        for (uint32_t x = 0; x < pt.L; ++x) pw[x] = pt.w[t->pos_lid[q][x]];
        o.pos_w[q] = sg.add(pw.data(), pw.size() * 4);
      }
    }
    auto kid = [&](uint32_t x2) { return o.relabel ? orig[x2] : x2; };  // original id of kernel NPU x2
    if (relay) {
      for (int q = 0; q < 2; ++q) {
        std::vector<uint32_t> allow;
        relay_allow(t, q, pt.C, pt.Wp, pl->pre, pl->post, allow);
        o.allow[q] = sg.add(allow.data(), allow.size() * 4);
      }
    }
    if (custom) {
      const uint32_t W0 = (pt.C + 31u) / 32u;
      std::vector<uint32_t> pre_p((size_t)pt.N * pt.Wp, 0u), post_p((size_t)pt.N * pt.Wp, 0u);
      for (uint32_t x = 0; x < pt.N; ++x)
        for (uint32_t q = 0; q < W0; ++q) {
          pre_p[(size_t)x * pt.Wp + q] = pl->pre[(size_t)kid(x) * W0 + q];
          post_p[(size_t)x * pt.Wp + q] = pl->post[(size_t)kid(x) * W0 + q];
        }
      o.pre = sg.add(pre_p.data(), pre_p.size() * 4);
      o.post = sg.add(post_p.data(), post_p.size() * 4);
    }
    if (pt.windowed) {  // records of destination x at [rec_off[x], rec_off[x+1]): |post[x] - pre[x]| each
      std::vector<uint32_t> ro(pt.N + 1, 0u);
      const uint32_t W0 = (pt.C + 31u) / 32u;
      for (uint32_t x = 0; x < pt.N; ++x) {
        uint32_t need;
        if (custom) {
          need = 0;
          for (uint32_t q = 0; q < W0; ++q)
            need += (uint32_t)__builtin_popcount(pl->post[(size_t)kid(x) * W0 + q] & ~pl->pre[(size_t)kid(x) * W0 + q]);
        } else {
          need = pt.C - pt.k;
        }
        ro[x + 1] = ro[x] + need;
      }
      o.rec_off = sg.add(ro.data(), ro.size() * 4);
    }
    for (int q = 0; q < 2; ++q) o.topo[q] = sg.reserve(sizeof(DevTopo));
    o.keys = sg.reserve(8 * kSmallWords);
    o.times_ag = sg.reserve(8 * (size_t)S);
    if (pt.rs_search) o.times_rs = sg.reserve(8 * (size_t)S);
  }
  const size_t o_jobs = sg.reserve(sizeof(Job) * n_jobs);
  if ((rc = dev_alloc(bufs, dev, sg.host.size(), &vp))) return rc;
  unsigned char *base = reinterpret_cast<unsigned char *>(vp);
  pl->d_outs = reinterpret_cast<JobOut *>(base + o_outs);
  pl->d_count = reinterpret_cast<unsigned long long *>(base + o_count);
  for (uint32_t i = 0; i < n_topos; ++i) {
    Part &pt = pl->parts[i];
    const PartOffs &o = po[i];
    pt.d_w = reinterpret_cast<uint32_t *>(base + o.w);
    for (int q = 0; q < 2; ++q) {
      DevTopo &h = pt.htopo[q];
      h.N = pt.N;
      h.L = pt.L;
      h.C = pt.C;
      h.k = pt.k;
      h.Wp = pt.Wp;
      h.P = pt.P;
      h.VPL = pt.VPL;
      h.custom = custom ? 1u : 0u;
      h.required = pt.required;
      h.in_ptr = o.relabel ? reinterpret_cast<const uint32_t *>(base + o.in_ptr[q]) : pt.td->d_in_ptr[q];
      h.p_src = o.relabel ? reinterpret_cast<const uint32_t *>(base + o.pos_src[q]) : pt.td->d_pos_src[q];
      h.p_dst = o.relabel ? reinterpret_cast<const uint32_t *>(base + o.pos_dst[q]) : pt.td->d_pos_dst[q];
      h.p_w = reinterpret_cast<const uint32_t *>(base + o.pos_w[q]);
      h.p_lid = o.relabel ? reinterpret_cast<const uint32_t *>(base + o.pos_lid[q]) : pt.td->d_pos_lid[q];
      h.npu_orig = o.relabel ? reinterpret_cast<const uint32_t *>(base + o.orig) : nullptr;
      h.pre = custom ? reinterpret_cast<const uint32_t *>(base + o.pre) : nullptr;
      h.post = custom ? reinterpret_cast<const uint32_t *>(base + o.post) : nullptr;
      h.allow = relay ? reinterpret_cast<const uint32_t *>(base + o.allow[q]) : nullptr;
      sg.put(o.topo[q], h);
      pt.d_topo[q] = reinterpret_cast<DevTopo *>(base + o.topo[q]);
    }
    pt.d_rec_off = pt.windowed ? reinterpret_cast<const uint32_t *>(base + o.rec_off) : nullptr;
    pt.d_keys = reinterpret_cast<uint64_t *>(base + o.keys);
    pt.d_stats = pt.d_keys + 2;
    pt.d_times_ag = reinterpret_cast<uint64_t *>(base + o.times_ag);
    if (pt.rs_search) pt.d_times_rs = reinterpret_cast<uint64_t *>(base + o.times_rs);
  }
  // ---- job table ----
  pl->jobs.resize(n_jobs);
  size_t rows_off = 0, links_off = 0;
  for (auto &g : pl->groups) {
    for (uint32_t i = 0; i < n_topos; ++i) {
      Part &pt = pl->parts[i];
      if (pt.job_base < g.job_begin || pt.job_base >= g.job_end) continue;
      for (uint32_t j = 0; j < pt.n_jobs; ++j) {
        const uint32_t sigma = (pt.rs_search && j >= pt.rs_base) ? 1u : 0u;
        const uint32_t si = j % S;
        Job &jb = pl->jobs[pt.job_base + j];
        jb.topo = pt.d_topo[sigma];
        jb.seed = p->base_seed + p->seed_offset + si;
        jb.sigma = sigma;
        jb.out_slot = pt.job_base + j;
        jb.rec = record ? pt.d_rec + (size_t)j * pt.cap : nullptr;
        jb.rec_cap = record ? pt.cap : 0;
        jb.rec_off = pt.d_rec_off;
        jb.g_rows = nullptr;
        jb.g_links = nullptr;
        jb.trace = nullptr;
        jb.trace_stride = 1u;
        if (!g.lay.rows_in_smem) {
          jb.g_rows = reinterpret_cast<uint32_t *>(pl->d_rows + rows_off);
          rows_off += g.lay.rows_bytes;
        }
        if (!g.lay.links_in_smem) {
          jb.g_links = pl->d_links + links_off;
          links_off += g.lay.links_bytes;
        }
      }
    }
  }
  if (getenv("TACOS_TRACE") && !pl->jobs.empty()) {
    if ((rc = dev_alloc(bufs, dev, 8ull * kTraceWords * kTraceEvents * 8, &vp))) return rc;
    CUDA_TRY(cudaMemsetAsync(vp, 0xFF, 8ull * kTraceWords * kTraceEvents * 8, st));
    pl->jobs[0].trace = reinterpret_cast<unsigned long long *>(vp);
    pl->jobs[0].trace_stride = 1u;
    if (const char *env = getenv("TACOS_TRACE_STRIDE")) pl->jobs[0].trace_stride = std::max(1, atoi(env));
    pl->d_trace = pl->jobs[0].trace;
  }
  std::memcpy(sg.host.data() + o_jobs, pl->jobs.data(), sizeof(Job) * n_jobs);
  pl->d_jobs = reinterpret_cast<Job *>(base + o_jobs);
  // one pinned staging copy + one H2D on `st`; the pinned block stays with the plan (released
  // after its last work completes), so nothing here waits for the copy
  pl->stage_buf.dev = dev;
  pl->stage_buf.p = pinned_pool().alloc(dev, sg.host.size(), &pl->stage_buf.cls);
  if (!pl->stage_buf.p) return fail(TACOS_E_NOMEM, "pinned allocation failed");
  std::memcpy(pl->stage_buf.p, sg.host.data(), sg.host.size());
  CUDA_TRY(cudaEventCreateWithFlags(&pl->done, cudaEventDisableTiming));
  CUDA_TRY(cudaMemcpyAsync(base, pl->stage_buf.p, sg.host.size(), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaEventRecord(pl->done, st));
  pl->h_small_buf.dev = dev;
  pl->h_small_buf.p = pinned_pool().alloc(dev, 8 * kSmallWords * (size_t)n_topos, &pl->h_small_buf.cls);
  if (!pl->h_small_buf.p) return fail(TACOS_E_NOMEM, "pinned allocation failed");
  pl->h_small = reinterpret_cast<uint64_t *>(pl->h_small_buf.p);
  if (sync) CUDA_TRY(cudaStreamSynchronize(st));
  *out = pl.release();
  return TACOS_OK;
}

int plan_search(tacos_plan *pl, cudaStream_t st) {
  int rc;
  pl->last_launches = 0;
  const bool literal = (pl->p.flags & TACOS_FLAG_LITERAL) != 0;
  for (auto &g : pl->groups) {
    rc = literal ? launch_literal(g.lay, g.VPL, pl->d_jobs + g.job_begin, g.job_end - g.job_begin, pl->d_outs, st)
                 : launch_greedy(g.lay, g.P, g.VPL, pl->d_jobs + g.job_begin, g.job_end - g.job_begin, pl->d_outs, st);
    if (rc) return fail(rc, "%s", cuda_error_string());
    pl->last_launches++;
  }
  const uint32_t S = pl->p.n_seeds;
  for (auto &pt : pl->parts) {
    if ((rc = launch_best_keys(pl->d_outs + pt.job_base, S, pl->p.seed_offset, pt.rs_base, pt.rs_search ? 1u : 0u, pt.d_keys,
                               pt.d_stats, pt.d_times_ag, pt.d_times_rs, st)))
      return fail(rc, "%s", cuda_error_string());
    pl->last_launches++;
  }
  CUDA_TRY(cudaEventRecord(pl->done, st));
  return TACOS_OK;
}

// Read keys + stats of every part (one D2H, one sync).
int plan_read_small(tacos_plan *pl, cudaStream_t st) {
  for (size_t i = 0; i < pl->parts.size(); ++i)
    CUDA_TRY(cudaMemcpyAsync(pl->h_small + kSmallWords * i, pl->parts[i].d_keys, 8 * kSmallWords, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return TACOS_OK;
}

// upper bound of the sends of one result (exact without relays)
uint64_t sends_per_result(const tacos_plan *pl, const Part &pt) {
  if (pl->p.flags & TACOS_FLAG_NO_SCHEDULE) return 0;
  return pl->p.collective == TACOS_ALL_REDUCE ? 2 * pt.cap : pt.cap;
}

// Emission that follows the search on the stream without a host round trip: the emitters
// read the best keys on the device (DevWin).  For one part, no relays, not the literal or the
// windowed loop (their records need a sort whose pass count depends on T), AG-type, or an
// RS-type phase on a symmetric graph with one link cost (the sort-free mirror).  The host
// decodes the keys afterwards (plan_emit_part with dev_launched).
bool dev_emit_eligible(const tacos_plan *pl) {
  if (pl->parts.size() != 1) return false;
  const Part &pt = pl->parts[0];
  if (pl->p.flags & (TACOS_FLAG_NO_SCHEDULE | TACOS_FLAG_LITERAL)) return false;
  if (coll_relay(&pl->p) || pt.windowed || pt.d_rec == nullptr) return false;
  if (pt.lockstep && (size_t)16 * ((pt.L + 31u) / 32u) > (size_t)200 * 1024) return false;
  if (coll_need_rs(pl->p.collective)) {
    if (!pt.symmetric || pt.w.empty() || (size_t)8 * ((pt.L + 31u) / 32u) > (size_t)200 * 1024) return false;
    for (uint32_t x : pt.w)
      if (x != pt.w[0]) return false;
  }
  return true;
}

int plan_emit_dev_launch(tacos_plan *pl, tacos_send *d_sends, uint64_t capacity, cudaStream_t st) {
  Part &pt = pl->parts[0];
  const uint64_t nsend = sends_per_result(pl, pt);
  if (nsend == 0 || capacity < nsend) return TACOS_OK;  // (the capacity error is raised by plan_emit_part)
  const int coll = pl->p.collective;
  DevWin dw{reinterpret_cast<const unsigned long long *>(pt.d_keys), pt.d_rec, pt.cap, pl->p.seed_offset,
            pl->p.n_seeds, coll == TACOS_ALL_REDUCE ? 1u : 0u};
  const uint64_t M = pt.required;
  int rc;
  if (coll == TACOS_ALL_REDUCE && pt.lockstep) {  // both phases from one pass over the records
    uint32_t nl = 0;
    if ((rc = launch_rs_uniform_emit(nullptr, M, pt.td->d_src, pt.td->d_dst, pt.w[0], pt.td->d_rev, 0, pt.L, d_sends,
                                     pl->d_sort, pl->sort_bytes, &nl, st, &dw, /*mirror=*/2u)))
      return fail(rc, "%s", cuda_error_string());
    pl->last_launches += nl;
    return TACOS_OK;
  }
  if (coll_need_rs(coll)) {
    uint32_t nl = 0;
    if ((rc = launch_rs_uniform_emit(nullptr, M, pt.td->d_src, pt.td->d_dst, pt.w[0], pt.td->d_rev, 0, pt.L, d_sends,
                                     pl->d_sort, pl->sort_bytes, &nl, st, &dw)))
      return fail(rc, "%s", cuda_error_string());
    pl->last_launches += nl;
  }
  if (coll_need_ag(coll)) {
    const uint64_t base = coll == TACOS_ALL_REDUCE ? M : 0;
    if (pt.lockstep) {  // records in (t_start, CTA, position) order: ranked by link inside each event
      uint32_t nl = 0;
      if ((rc = launch_rs_uniform_emit(nullptr, M, pt.td->d_src, pt.td->d_dst, pt.w[0], nullptr, 0, pt.L, d_sends + base,
                                       pl->d_sort, pl->sort_bytes, &nl, st, &dw, /*mirror=*/0u)))
        return fail(rc, "%s", cuda_error_string());
      pl->last_launches += nl;
    } else {
      if ((rc = launch_emit_ag(nullptr, M, pt.td->d_src, pt.td->d_dst, pt.d_w, 0, d_sends + base, st, ~0ull, &dw)))
        return fail(rc, "%s", cuda_error_string());
      pl->last_launches += 1;
    }
  }
  return TACOS_OK;
}

// Emit part i's schedule into device memory d_sends; fill res from the keys in h_small.
int plan_emit_part(tacos_plan *pl, size_t i, tacos_send *d_sends, uint64_t capacity, tacos_result *res,
                   cudaStream_t st, bool dev_launched = false) {
  Part &pt = pl->parts[i];
  const uint64_t *hs = pl->h_small + kSmallWords * i;
  const uint64_t key_ag = hs[0], key_rs = hs[1];
  const uint64_t *stats = hs + 2;
  std::memset(res, 0, sizeof(*res));
  res->visits = stats[0];
  res->dest_events = stats[1];
  res->matches = stats[2];
  res->events = stats[3];
  res->cancelled = stats[5];
  res->live_visits = stats[6];
  res->best_key_ag = key_ag;
  res->best_key_rs = key_rs;
  const int32_t st_status = (int32_t)(int64_t)stats[4];
  const int coll = pl->p.collective;
  const bool need_rs = coll_need_rs(coll);
  const bool need_ag = coll_need_ag(coll);
  tacos_winner win;
  const uint64_t keys[2] = {key_ag, key_rs};
  int rc0 = tacos_select_winner(keys, coll, pt.symmetric ? 1 : 0, pl->p.seed_offset, pl->p.n_seeds, &win);
  if (rc0 == TACOS_E_UNREACHABLE) {
    res->status = st_status ? st_status : TACOS_E_UNREACHABLE;
    return fail(res->status, "no seed finished the synthesis (status %d)", res->status);
  }
  if (rc0) return rc0;
  const uint64_t T_ag = win.T_ag, g_ag = win.seed_index_ag, T_rs = win.T_rs, g_rs = win.seed_index_rs;
  res->T_ag = T_ag;
  res->T_rs = T_rs;
  res->T = win.T;
  res->rs_seed = pl->p.base_seed + g_rs;
  res->seed = need_ag ? pl->p.base_seed + g_ag : res->rs_seed;
  const uint32_t off = pl->p.seed_offset;
  const bool ag_local = (win.local & 1u) != 0;
  const bool rs_local = (win.local & 2u) != 0;
  res->winner_local = win.local;
  res->status = TACOS_OK;
  const uint64_t nsend = sends_per_result(pl, pt);
  if (nsend == 0) return TACOS_OK;
  if (capacity < nsend) return fail(TACOS_E_CAPACITY, "capacity %llu < %llu sends", (unsigned long long)capacity, (unsigned long long)nsend);
  if (dev_launched) {  // emitted by plan_emit_dev_launch, winner resolved on the device
    res->n_sends = (need_rs && rs_local ? pt.required : 0) + (need_ag && ag_local ? pt.required : 0);
    return TACOS_OK;
  }
  int rc;
  uint64_t emitted = 0;
  // matches of a winning job: `required` without relays, else read back from its JobOut
  auto job_matches = [&](uint32_t job, uint64_t *m) -> int {
    if (!coll_relay(&pl->p)) {
      *m = pt.required;
      return TACOS_OK;
    }
    JobOut o;
    CUDA_TRY(cudaMemcpyAsync(&o, pl->d_outs + pt.job_base + job, sizeof(o), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    *m = o.M;
    return TACOS_OK;
  };
  // relays (R22): drop the sends still in flight when the postcondition held (tombstones
  // written by the emitters), order preserved; *m = the sends kept
  auto drop_late = [&](tacos_send *first, uint64_t *m) -> int {
    if (!coll_relay(&pl->p) || *m == 0) return TACOS_OK;
    int r = launch_compact_sends(first, *m, pl->d_count, st);
    if (r) return fail(r, "%s", cuda_error_string());
    pl->last_launches += 1;
    unsigned long long kept = 0;
    CUDA_TRY(cudaMemcpyAsync(&kept, pl->d_count, sizeof(kept), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    *m = kept;
    return TACOS_OK;
  };
  if (need_rs && rs_local) {
    const uint32_t job = pt.symmetric ? (uint32_t)(g_rs - off) : pt.rs_base + (uint32_t)(g_rs - off);
    uint64_t M;
    if ((rc = job_matches(job, &M))) return rc;
    const Rec *rec = pt.d_rec + (size_t)job * pt.cap;
    uint32_t nl = 0;
    // one link cost, symmetric, no relays: the mirror order needs no sort (launch_rs_uniform_emit)
    // (its link-id bitmap lives in shared memory: 2 bits per link, at most 200 KB)
    const bool uniform = pt.symmetric && !coll_relay(&pl->p) && !pt.windowed && !pt.w.empty() &&
                         (size_t)8 * ((pt.L + 31u) / 32u) <= (size_t)200 * 1024 &&
                         std::all_of(pt.w.begin(), pt.w.end(), [&](uint32_t x) { return x == pt.w[0]; });
    if (uniform) {
      if ((rc = launch_rs_uniform_emit(rec, M, pt.td->d_src, pt.td->d_dst, pt.w[0], pt.td->d_rev, T_rs, pt.L, d_sends, pl->d_sort,
                                       pl->sort_bytes, &nl, st)))
        return fail(rc, "%s", cuda_error_string());
    } else if ((rc = launch_rs_sort_emit(rec, M, pt.td->d_src, pt.td->d_dst, pt.d_w, pt.symmetric ? pt.td->d_rev : nullptr, T_rs,
                                         pt.L, d_sends, pl->d_sort, pl->sort_bytes, &nl, st)))
      return fail(rc, "%s", cuda_error_string());
    pl->last_launches += nl;
    if ((rc = drop_late(d_sends, &M))) return rc;
    emitted += M;
  }
  if (need_ag && ag_local) {
    uint64_t M;
    if ((rc = job_matches((uint32_t)(g_ag - off), &M))) return rc;
    const Rec *rec = pt.d_rec + (size_t)(g_ag - off) * pt.cap;
    const uint64_t base = coll == TACOS_ALL_REDUCE ? pt.required : 0;  // AR: after the RS half (no relays)
    if ((pl->p.flags & TACOS_FLAG_LITERAL) || pt.windowed) {  // records not in (t_start, link) order: sort
      uint32_t nl = 0;
      if ((rc = launch_rs_sort_emit(rec, M, pt.td->d_src, pt.td->d_dst, pt.d_w, nullptr, T_ag, pt.L, d_sends + base, pl->d_sort,
                                    pl->sort_bytes, &nl, st, /*mirror=*/0u, /*shift=*/T_rs)))
        return fail(rc, "%s", cuda_error_string());
      pl->last_launches += nl;
    } else if (pt.lockstep && (size_t)8 * ((pt.L + 31u) / 32u) <= (size_t)200 * 1024) {
      // records in (t_start, CTA, position) order: ranked by link inside each event (no relays)
      uint32_t nl = 0;
      if ((rc = launch_rs_uniform_emit(rec, M, pt.td->d_src, pt.td->d_dst, pt.w[0], nullptr, T_rs, pt.L, d_sends + base,
                                       pl->d_sort, pl->sort_bytes, &nl, st, nullptr, /*mirror=*/0u)))
        return fail(rc, "%s", cuda_error_string());
      pl->last_launches += nl;
    } else if (pt.lockstep) {  // (a link-id bitmap beyond 200 KB) sort
      uint32_t nl = 0;
      if ((rc = launch_rs_sort_emit(rec, M, pt.td->d_src, pt.td->d_dst, pt.d_w, nullptr, T_ag, pt.L, d_sends + base, pl->d_sort,
                                    pl->sort_bytes, &nl, st, /*mirror=*/0u, /*shift=*/T_rs)))
        return fail(rc, "%s", cuda_error_string());
      pl->last_launches += nl;
    } else {
      if ((rc = launch_emit_ag(rec, M, pt.td->d_src, pt.td->d_dst, pt.d_w, T_rs, d_sends + base, st, T_rs + T_ag)))
        return fail(rc, "%s", cuda_error_string());
      pl->last_launches += 1;
    }
    if ((rc = drop_late(d_sends + base, &M))) return rc;
    emitted += M;
  }
  res->n_sends = emitted;
  return TACOS_OK;
}
}  // namespace

extern "C" int tacos_select_winner(const uint64_t keys[2], int32_t collective, int symmetric, uint32_t seed_offset,
                                   uint32_t n_seeds, tacos_winner *out) {
  if (!keys || !out) return fail(TACOS_E_INVALID_ARG, "null argument");
  if (collective < TACOS_ALL_GATHER || collective > TACOS_GATHER) return fail(TACOS_E_INVALID_ARG, "bad collective");
  std::memset(out, 0, sizeof(*out));
  const bool need_rs = coll_need_rs(collective);
  const bool need_ag = coll_need_ag(collective);
  // the RS phase of a symmetric graph is the mirror of the AG winner (R9); else its own search (key 1)
  const bool rs_own = need_rs && !symmetric;
  const uint64_t k_ag = keys[0], k_rs = rs_own ? keys[1] : keys[0];
  if ((need_ag || !rs_own) && k_ag == kNoKey) return fail(TACOS_E_UNREACHABLE, "no AG seed finished");
  if (rs_own && k_rs == kNoKey) return fail(TACOS_E_UNREACHABLE, "no RS seed finished");
  const uint64_t mask = (1ull << kKeySeedBits) - 1ull;
  out->T_ag = need_ag ? (k_ag >> kKeySeedBits) : 0;
  out->seed_index_ag = k_ag & mask;
  out->T_rs = need_rs ? (k_rs >> kKeySeedBits) : 0;
  out->seed_index_rs = need_rs ? (k_rs & mask) : out->seed_index_ag;
  out->T = out->T_ag + out->T_rs;  // R10: AR = RS then AG
  if (out->T >= kMaxTime) return fail(TACOS_E_OVERFLOW, "collective time beyond 2^40 time units");
  auto local = [&](uint64_t g) { return g >= seed_offset && g < (uint64_t)seed_offset + n_seeds; };
  out->local = (need_ag && local(out->seed_index_ag) ? 1u : 0u) | (need_rs && local(out->seed_index_rs) ? 2u : 0u);
  return TACOS_OK;
}

extern "C" int tacos_plan_create(const tacos_topology *topo, const tacos_synth_params *p, tacos_plan **out) {
  if (!out) return fail(TACOS_E_INVALID_ARG, "null out");
  const tacos_topology *ts[1] = {topo};
  try {
    return plan_build(ts, 1, p, out);
  } catch (const std::bad_alloc &) {
    return fail(TACOS_E_NOMEM, "host allocation failed");
  } catch (...) {
    return fail(TACOS_E_INVALID_ARG, "internal error");
  }
}

extern "C" void tacos_plan_destroy(tacos_plan *pl) { delete pl; }

extern "C" int tacos_plan_search(tacos_plan *pl, void *stream) {
  if (!pl) return fail(TACOS_E_INVALID_ARG, "null plan");
  return plan_search(pl, (cudaStream_t)stream);
}

extern "C" uint64_t *tacos_plan_best_keys(tacos_plan *pl) { return pl ? pl->parts[0].d_keys : nullptr; }

extern "C" int tacos_plan_emit(tacos_plan *pl, tacos_send *d_sends, uint64_t capacity, tacos_result *result,
                               void *stream) {
  if (!pl || !result) return fail(TACOS_E_INVALID_ARG, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  pl->last_launches = 0;
  const bool dev = dev_emit_eligible(pl) && d_sends != nullptr;
  int rc = dev ? plan_emit_dev_launch(pl, d_sends, capacity, st) : TACOS_OK;
  if (rc) return rc;
  if ((rc = plan_read_small(pl, st))) return rc;
  rc = plan_emit_part(pl, 0, d_sends, capacity, result, st, dev);
  cudaEventRecord(pl->done, st);
  return rc;
}

extern "C" int tacos_plan_emit_async(tacos_plan *pl, tacos_send *d_sends, uint64_t capacity, void *stream) {
  if (!pl || !d_sends) return fail(TACOS_E_INVALID_ARG, "null argument");
  if (!dev_emit_eligible(pl)) return fail(TACOS_E_INVALID_ARG, "this plan's emission needs the keys on the host (tacos_plan_emit)");
  if (capacity < sends_per_result(pl, pl->parts[0]))
    return fail(TACOS_E_CAPACITY, "capacity %llu < %llu sends", (unsigned long long)capacity,
                (unsigned long long)sends_per_result(pl, pl->parts[0]));
  cudaStream_t st = (cudaStream_t)stream;
  pl->last_launches = 0;
  int rc = plan_emit_dev_launch(pl, d_sends, capacity, st);
  cudaEventRecord(pl->done, st);
  return rc;
}

extern "C" int tacos_plan_result(tacos_plan *pl, uint64_t capacity, tacos_result *result, void *stream) {
  if (!pl || !result) return fail(TACOS_E_INVALID_ARG, "null argument");
  if (!dev_emit_eligible(pl)) return fail(TACOS_E_INVALID_ARG, "not a device-resolved emission (tacos_plan_emit)");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = plan_read_small(pl, st);
  if (rc) return rc;
  return plan_emit_part(pl, 0, nullptr, capacity, result, st, true);
}

extern "C" int tacos_plan_stats(tacos_plan *pl, tacos_result *result, void *stream) {
  if (!pl || !result) return fail(TACOS_E_INVALID_ARG, "null argument");
  int rc = plan_read_small(pl, (cudaStream_t)stream);
  if (rc) return rc;
  const uint64_t *hs = pl->h_small;
  std::memset(result, 0, sizeof(*result));
  result->visits = hs[2];
  result->dest_events = hs[3];
  result->matches = hs[4];
  result->events = hs[5];
  result->status = (int32_t)(int64_t)hs[6];
  result->cancelled = hs[7];
  result->live_visits = hs[8];
  result->best_key_ag = hs[0];
  result->best_key_rs = hs[1];
  return TACOS_OK;
}

extern "C" const uint64_t *tacos_plan_seed_times_device(const tacos_plan *pl, const uint64_t **rs_times) {
  if (!pl) return nullptr;
  if (rs_times) *rs_times = pl->parts[0].d_times_rs;
  return pl->parts[0].d_times_ag;
}

extern "C" uint32_t tacos_plan_last_launches(const tacos_plan *pl) { return pl ? pl->last_launches : 0; }

extern "C" int tacos_plan_info_get(const tacos_plan *pl, tacos_plan_info *out) {
  if (!pl || !out) return fail(TACOS_E_INVALID_ARG, "null argument");
  std::memset(out, 0, sizeof(*out));
  const Group *big = nullptr;
  for (const Group &g : pl->groups) {
    const uint32_t nj = g.job_end - g.job_begin, q = g.lay.cluster ? g.lay.cluster : 1u;
    out->n_jobs += nj;
    out->ctas += nj * q;
    out->launches += 1;
    if (!g.lay.rows_in_smem) out->rows_bytes += (uint64_t)nj * g.lay.rows_bytes;
    if (!big || nj > big->job_end - big->job_begin) big = &g;
  }
  if (big) {
    out->cluster = big->lay.cluster ? big->lay.cluster : 1u;
    out->threads = big->lay.threads;
    out->smem_bytes = big->lay.smem_bytes;
    out->rows_in_smem = big->lay.rows_in_smem;
    out->links_in_smem = big->lay.links_in_smem;
    out->event_loop = big->lay.window ? 1u : big->lay.lockstep ? 2u : 0u;
  }
  return TACOS_OK;
}

// ---------------------------------------------------------------------------
// one-call synthesis
// ---------------------------------------------------------------------------
struct tacos_schedule {
  tacos_result result{};
  uint64_t n_sends = 0;
  tacos_send *sends = nullptr;  // pinned pool block
  DevBuf host_buf;
  std::vector<uint64_t> seed_times;
  ~tacos_schedule() {
    if (host_buf.p) pinned_pool().release(host_buf.dev, host_buf.p, host_buf.cls);
  }
};

extern "C" int tacos_max_sends(const tacos_topology *topo, const tacos_synth_params *p, uint64_t *n_out) {
  if (!topo || !p || !n_out) return fail(TACOS_E_INVALID_ARG, "null argument");
  int rc = validate_params(p);
  if (rc) return rc;
  uint64_t M;
  if (coll_custom(p->collective)) {
    uint32_t C = 0;
    std::vector<uint32_t> pre, post;
    try {
      if ((rc = problem_bits((uint32_t)topo->N, p, C, pre, post))) return rc;
    } catch (const std::bad_alloc &) {
      return fail(TACOS_E_NOMEM, "host allocation failed");
    }
    M = 0;
    uint64_t held0 = 0;
    for (size_t q = 0; q < pre.size(); ++q) {
      M += (uint64_t)__builtin_popcount(post[q] & ~pre[q]);
      held0 += (uint64_t)__builtin_popcount(pre[q]);
    }
    if (coll_relay(p)) M = (uint64_t)topo->N * C - held0;  // upper bound: each (NPU, chunk) delivered at most once
  } else {
    M = (uint64_t)topo->N * p->chunks_per_npu * (uint64_t)(topo->N - 1);
  }
  if (p->flags & TACOS_FLAG_NO_SCHEDULE) M = 0;
  *n_out = p->collective == TACOS_ALL_REDUCE ? 2 * M : M;
  return TACOS_OK;
}

namespace {
bool is_device_ptr(const void *ptr) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Search + emit for n_topos topologies; per topology: sends into dst[i] (host or
// device, capacity caps[i]) and results[i]; seed times optional.
// Per-seed collective times (tacos_schedule_seed_times) of a part from the AG-on-G and
// AG-on-G^T search times: AG-type T_AG(s); RS-type T_RS(s); AR T_RS(s) + T_AG(s) (R10),
// where on a symmetric graph T_RS(s) = T_AG(s) (R9).
void combine_seed_times(const Part &pt, int coll, uint32_t S, const std::vector<uint64_t> &t_ag,
                        const std::vector<uint64_t> &t_rs, uint64_t *out) {
  const bool fwd_jobs = !pt.rs_search || pt.rs_base > 0;
  for (uint32_t s = 0; s < S; ++s) {
    const uint64_t ta = fwd_jobs ? t_ag[s] : 0, tr = pt.rs_search ? t_rs[s] : ta;
    out[s] = !coll_need_rs(coll) ? ta : (coll == TACOS_ALL_REDUCE ? tr + ta : tr);
  }
}

// D2H of a part's per-seed search times (async on st; read after a synchronize)
int read_seed_times_async(const Part &pt, uint32_t S, std::vector<uint64_t> &t_ag, std::vector<uint64_t> &t_rs,
                          cudaStream_t st) {
  const bool fwd_jobs = !pt.rs_search || pt.rs_base > 0;
  if (fwd_jobs) {
    t_ag.resize(S);
    CUDA_TRY(cudaMemcpyAsync(t_ag.data(), pt.d_times_ag, 8 * (size_t)S, cudaMemcpyDeviceToHost, st));
  }
  if (pt.rs_search) {
    t_rs.resize(S);
    CUDA_TRY(cudaMemcpyAsync(t_rs.data(), pt.d_times_rs, 8 * (size_t)S, cudaMemcpyDeviceToHost, st));
  }
  return TACOS_OK;
}

// One part, emission resolved on the device: search, emission, D2H of the schedule (host
// destination), keys and seed times are all queued on the stream, then one synchronization.
int synth_one_dev(tacos_plan *pl, tacos_send *dst, tacos_result *res, std::vector<uint64_t> *seed_times,
                  cudaStream_t st) {
  const Part &pt = pl->parts[0];
  const uint64_t need = sends_per_result(pl, pt);
  const bool dev_out = need > 0 && is_device_ptr(dst);
  tacos_send *d_out = dev_out ? dst : nullptr;
  DevBuf tmp;
  if (need > 0 && !dev_out) {
    tmp.dev = pl->device;
    tmp.p = device_pool().alloc(pl->device, need * sizeof(tacos_send), &tmp.cls);
    if (!tmp.p) return fail(TACOS_E_NOMEM, "device allocation failed");
    d_out = reinterpret_cast<tacos_send *>(tmp.p);
  }
  int rc = plan_emit_dev_launch(pl, d_out, need, st);
  // the whole schedule (the winner is always local on one device; a failed search writes nothing)
  if (rc == TACOS_OK && need > 0 && !dev_out) {
    cudaError_t e = cudaMemcpyAsync(dst, d_out, need * sizeof(tacos_send), cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) rc = fail(TACOS_E_CUDA, "D2H of the schedule: %s", cudaGetErrorString(e));
  }
  std::vector<uint64_t> t_ag, t_rs;
  if (rc == TACOS_OK && seed_times) rc = read_seed_times_async(pt, pl->p.n_seeds, t_ag, t_rs, st);
  if (rc == TACOS_OK) rc = plan_read_small(pl, st);  // one synchronization for all of it
  if (rc == TACOS_OK) rc = plan_emit_part(pl, 0, d_out, need, res, st, true);
  if (tmp.p) device_pool().release(tmp.dev, tmp.p, tmp.cls);
  if (rc) return rc;
  if (seed_times) {
    seed_times[0].resize(pl->p.n_seeds);
    combine_seed_times(pt, pl->p.collective, pl->p.n_seeds, t_ag, t_rs, seed_times[0].data());
  }
  return TACOS_OK;
}

int synth_many(const tacos_topology *const *topos, uint32_t n_topos, const tacos_synth_params *p, tacos_send **dst,
               const uint64_t *caps, tacos_result *results, std::vector<uint64_t> *seed_times, cudaStream_t st) {
  tacos_plan *raw = nullptr;
  int rc = plan_build(topos, n_topos, p, &raw, st, false);
  if (rc) return rc;
  std::unique_ptr<tacos_plan> pl(raw);
  if ((rc = plan_search(pl.get(), st))) return rc;
  if (pl->d_trace) {  // debug dump of job 0's event trace (TACOS_TRACE=path)
    std::vector<unsigned long long> tr((size_t)kTraceWords * kTraceEvents * 8);
    cudaMemcpy(tr.data(), pl->d_trace, tr.size() * 8, cudaMemcpyDeviceToHost);
    if (FILE *f = fopen(getenv("TACOS_TRACE"), "w")) {
      for (uint32_t r = 0; r < 8; ++r)
        for (uint32_t ev = 0; ev < kTraceEvents; ++ev) {
          const unsigned long long *x = &tr[(r * kTraceEvents + ev) * kTraceWords];
          if (x[0] == ~0ull) continue;
          fprintf(f, "%u %u", r, ev);
          for (uint32_t w = 0; w < kTraceWords; ++w) fprintf(f, " %llu", x[w]);
          fprintf(f, "\n");
        }
      fclose(f);
    }
  }
  if (dev_emit_eligible(pl.get()) && caps[0] >= sends_per_result(pl.get(), pl->parts[0]))
    return synth_one_dev(pl.get(), dst[0], results, seed_times, st);
  if ((rc = plan_read_small(pl.get(), st))) return rc;
  for (uint32_t i = 0; i < n_topos; ++i) {
    const Part &pt = pl->parts[i];
    const uint64_t need = sends_per_result(pl.get(), pt);
    if (caps[i] < need) return fail(TACOS_E_CAPACITY, "capacity %llu < %llu sends", (unsigned long long)caps[i], (unsigned long long)need);
    const bool dev_out = need > 0 && is_device_ptr(dst[i]);
    tacos_send *d_out = dev_out ? dst[i] : nullptr;
    DevBuf tmp;
    if (need > 0 && !dev_out) {
      tmp.dev = pl->device;
      tmp.p = device_pool().alloc(pl->device, need * sizeof(tacos_send), &tmp.cls);
      if (!tmp.p) return fail(TACOS_E_NOMEM, "device allocation failed");
      d_out = reinterpret_cast<tacos_send *>(tmp.p);
    }
    rc = plan_emit_part(pl.get(), i, d_out, need, &results[i], st);
    if (rc == TACOS_OK && results[i].n_sends > 0 && !dev_out) {
      cudaError_t e = cudaMemcpyAsync(dst[i], d_out, results[i].n_sends * sizeof(tacos_send), cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) rc = fail(TACOS_E_CUDA, "D2H of the schedule: %s", cudaGetErrorString(e));
    }
    // per-seed collective times (tacos_schedule_seed_times): AG-type T_AG(s); RS-type T_RS(s);
    // AR T_RS(s) + T_AG(s) (R10), where on a symmetric graph T_RS(s) = T_AG(s) (R9)
    std::vector<uint64_t> t_ag, t_rs;
    if (rc == TACOS_OK && seed_times) rc = read_seed_times_async(pt, p->n_seeds, t_ag, t_rs, st);
    if (rc == TACOS_OK) {
      cudaError_t e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) rc = fail(TACOS_E_CUDA, "synchronize: %s", cudaGetErrorString(e));
    }
    if (tmp.p) device_pool().release(tmp.dev, tmp.p, tmp.cls);
    if (rc) return rc;
    if (seed_times) {
      seed_times[i].resize(p->n_seeds);
      combine_seed_times(pt, p->collective, p->n_seeds, t_ag, t_rs, seed_times[i].data());
    }
  }
  return TACOS_OK;
}
}  // namespace

// ---------------------------------------------------------------------------
// several GPUs of one process: seed sharding + one NCCL MIN
// ---------------------------------------------------------------------------
namespace {
int resolve_devices(const tacos_synth_params *p, uint32_t *D) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    return fail(TACOS_E_CUDA, "no CUDA device available");
  }
  uint32_t want = p->n_devices == TACOS_ALL_DEVICES ? (uint32_t)n : p->n_devices;
  if (want <= 1) want = 1;
  if (want > (uint32_t)n) return fail(TACOS_E_INVALID_ARG, "n_devices = %u but %d devices are visible", want, n);
  *D = want;
  return TACOS_OK;
}

// NCCL communicators over devices 0 .. D-1 (ncclCommInitAll), created on first use and
// kept for the life of the process (creation costs far more than a synthesis).
int nccl_clique(uint32_t D, const NcclApi *api, std::vector<ncclComm_t> **out) {
  static std::mutex mu;
  static std::map<uint32_t, std::vector<ncclComm_t>> *cliques = new std::map<uint32_t, std::vector<ncclComm_t>>();
  std::lock_guard<std::mutex> g(mu);
  auto it = cliques->find(D);
  if (it == cliques->end()) {
    std::vector<ncclComm_t> comms(D);
    std::vector<int> devs(D);
    for (uint32_t i = 0; i < D; ++i) devs[i] = (int)i;
    int cur = 0;
    cudaGetDevice(&cur);
    const ncclResult_t r = api->CommInitAll(comms.data(), (int)D, devs.data());
    cudaSetDevice(cur);
    if (r != ncclSuccess) return fail(TACOS_E_NCCL, "ncclCommInitAll(%u): %s", D, api->GetErrorString(r));
    it = cliques->emplace(D, std::move(comms)).first;
  }
  *out = &it->second;
  return TACOS_OK;
}

// All threads of a sharded synthesis meet here before the collective: a failure on one
// device must not leave the others waiting inside ncclAllReduce.
struct Rendezvous {
  std::mutex m;
  std::condition_variable cv;
  uint32_t n, arrived = 0;
  bool failed = false;
  explicit Rendezvous(uint32_t n_) : n(n_) {}
  bool arrive(bool fail_here) {
    std::unique_lock<std::mutex> lk(m);
    failed = failed || fail_here;
    if (++arrived == n) cv.notify_all();
    else cv.wait(lk, [&] { return arrived == n; });
    return !failed;
  }
};

struct ShardOut {
  int rc = 0;
  std::string err;
  tacos_result res{};
  std::vector<uint64_t> times;  // the shard's per-seed collective times
};

// One topology, the seeds sharded over devices 0 .. G-1: each device's thread builds its
// plan (seed block [g S / G, (g+1) S / G)), searches on its own stream, takes part in one
// ncclAllReduce(MIN) of the two best keys, and emits the phases whose winning seed it
// owns into `dst` (host or device memory, same offsets as a one-device emission).
int synth_sharded(const tacos_topology *topo, const tacos_synth_params *p, uint32_t D, tacos_send *dst, uint64_t cap,
                  tacos_result *result, std::vector<uint64_t> *seed_times) {
  const uint32_t S = p->n_seeds, G = std::min(D, S);
  std::string nerr;
  const NcclApi *api = nccl_api(&nerr);
  if (!api) return fail(TACOS_E_NCCL, "%s", nerr.c_str());
  std::vector<ncclComm_t> *comms = nullptr;
  int rc = nccl_clique(G, api, &comms);
  if (rc) return rc;
  uint64_t need = 0;
  if ((rc = tacos_max_sends(topo, p, &need))) return rc;
  if (cap < need) return fail(TACOS_E_CAPACITY, "capacity %llu < %llu sends", (unsigned long long)cap, (unsigned long long)need);
  int caller = 0;
  CUDA_TRY(cudaGetDevice(&caller));
  std::vector<ShardOut> outs(G);
  Rendezvous rv(G);
  auto work = [&](uint32_t g) {
    ShardOut &o = outs[g];
    int r = TACOS_OK;
    cudaStream_t st = nullptr;
    tacos_plan *raw = nullptr;
    tacos_synth_params pg = *p;
    pg.n_devices = 1;
    const uint32_t lo = (uint32_t)((uint64_t)g * S / G), hi = (uint32_t)((uint64_t)(g + 1) * S / G);
    pg.seed_offset = p->seed_offset + lo;
    pg.n_seeds = hi - lo;
    if (cudaSetDevice((int)g) != cudaSuccess || cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
      r = fail(TACOS_E_CUDA, "device %u: %s", g, cudaGetErrorString(cudaGetLastError()));
    std::unique_ptr<tacos_plan> pl;
    try {  // no exception may leave a worker thread, and every worker must reach the rendezvous
      if (!r) r = plan_build(&topo, 1, &pg, &raw, st, false);
      pl.reset(raw);
      if (!r) r = plan_search(pl.get(), st);
    } catch (...) {
      r = TACOS_E_NOMEM;
    }
    const bool go = rv.arrive(r != 0);
    if (go) {
      uint64_t *keys = pl->parts[0].d_keys;
      const ncclResult_t nr = api->AllReduce(keys, keys, 2, ncclUint64, ncclMin, (*comms)[g], st);
      if (nr != ncclSuccess) r = fail(TACOS_E_NCCL, "ncclAllReduce: %s", api->GetErrorString(nr));
    }
    if (go && !r) r = plan_read_small(pl.get(), st);
    DevBuf tmp;
    std::vector<uint64_t> t_ag, t_rs;
    if (go && !r) {
      const Part &pt = pl->parts[0];
      const uint64_t n_out = sends_per_result(pl.get(), pt);
      tacos_send *d_out = nullptr;
      if (n_out) {
        tmp.dev = (int)g;
        tmp.p = device_pool().alloc((int)g, n_out * sizeof(tacos_send), &tmp.cls);
        if (!tmp.p) r = fail(TACOS_E_NOMEM, "device allocation failed");
        d_out = reinterpret_cast<tacos_send *>(tmp.p);
      }
      if (!r) r = plan_emit_part(pl.get(), 0, d_out, n_out, &o.res, st);
      if (!r && n_out && o.res.winner_local) {  // copy the phases emitted here (same offsets)
        auto copy = [&](uint64_t off, uint64_t n) {
          if (!r && n && cudaMemcpyAsync(dst + off, d_out + off, n * sizeof(tacos_send), cudaMemcpyDefault, st) != cudaSuccess)
            r = fail(TACOS_E_CUDA, "copy of the schedule: %s", cudaGetErrorString(cudaGetLastError()));
        };
        if (p->collective == TACOS_ALL_REDUCE) {  // RS half [0, M), AG half [M, 2M) (no relays)
          if (o.res.winner_local & 2u) copy(0, pt.required);
          if (o.res.winner_local & 1u) copy(pt.required, pt.required);
        } else {
          copy(0, o.res.n_sends);
        }
      }
      if (!r && seed_times) r = read_seed_times_async(pt, pg.n_seeds, t_ag, t_rs, st);
      if (!r && cudaStreamSynchronize(st) != cudaSuccess)
        r = fail(TACOS_E_CUDA, "synchronize: %s", cudaGetErrorString(cudaGetLastError()));
      if (!r && seed_times) {
        o.times.resize(pg.n_seeds);
        combine_seed_times(pt, p->collective, pg.n_seeds, t_ag, t_rs, o.times.data());
      }
    }
    if (tmp.p) device_pool().release(tmp.dev, tmp.p, tmp.cls);
    pl.reset();
    if (st) cudaStreamDestroy(st);
    if (!go && !r) r = fail(TACOS_E_CUDA, "another device failed before the selection");
    o.rc = r;
    if (r) o.err = g_last_error;
  };
  {
    std::vector<std::thread> th;
    for (uint32_t g = 0; g < G; ++g)
      th.emplace_back([&, g] {
        try {
          work(g);
        } catch (...) {  // (past the rendezvous: only host allocations can throw here)
          outs[g].rc = TACOS_E_NOMEM;
          outs[g].err = "host allocation failed";
        }
      });
    for (auto &t : th) t.join();
  }
  cudaSetDevice(caller);
  for (uint32_t g = 0; g < G; ++g)  // report a real failure before the knock-on ones
    if (outs[g].rc && outs[g].err.find("another device failed") == std::string::npos)
      return fail(outs[g].rc, "device %u: %s", g, outs[g].err.c_str());
  for (uint32_t g = 0; g < G; ++g)
    if (outs[g].rc) return fail(outs[g].rc, "device %u: %s", g, outs[g].err.c_str());
  tacos_result res = outs[0].res;
  res.visits = res.dest_events = res.matches = res.events = res.cancelled = res.n_sends = res.live_visits = 0;
  for (const ShardOut &o : outs) {
    res.visits += o.res.visits;
    res.dest_events += o.res.dest_events;
    res.matches += o.res.matches;
    res.events += o.res.events;
    res.cancelled += o.res.cancelled;
    res.live_visits += o.res.live_visits;
    res.n_sends += o.res.n_sends;
  }
  res.winner_local = (p->collective == TACOS_ALL_REDUCE) ? 3u : (coll_need_ag(p->collective) ? 1u : 2u);
  *result = res;
  if (seed_times) {
    seed_times->clear();
    for (const ShardOut &o : outs) seed_times->insert(seed_times->end(), o.times.begin(), o.times.end());
  }
  return TACOS_OK;
}
}  // namespace

extern "C" int tacos_synthesize_into(const tacos_topology *topo, const tacos_synth_params *p, tacos_send *sends,
                                     uint64_t capacity, tacos_result *result, void *stream) {
  if (!topo || !p || !result) return fail(TACOS_E_INVALID_ARG, "null argument");
  try {
    uint32_t D = 1;
    int rc = resolve_devices(p, &D);
    if (rc) return rc;
    if (D > 1) {  // seeds sharded over devices 0 .. D-1 (`stream` is not used: one stream per device)
      if ((rc = validate_params(p))) return rc;
      return synth_sharded(topo, p, D, sends, sends ? capacity : 0, result, nullptr);
    }
    const tacos_topology *ts[1] = {topo};
    tacos_send *d[1] = {sends};
    uint64_t caps[1] = {sends ? capacity : 0};
    return synth_many(ts, 1, p, d, caps, result, nullptr, (cudaStream_t)stream);
  } catch (const std::bad_alloc &) {
    return fail(TACOS_E_NOMEM, "host allocation failed");
  }
}

extern "C" int tacos_synthesize_batch(const tacos_topology *const *topos, uint32_t n_topos, const tacos_synth_params *p,
                                      tacos_schedule **outs) {
  if (!topos || !outs || n_topos == 0) return fail(TACOS_E_INVALID_ARG, "null argument");
  for (uint32_t i = 0; i < n_topos; ++i) outs[i] = nullptr;
  try {
    std::vector<std::unique_ptr<tacos_schedule>> sch(n_topos);
    std::vector<tacos_send *> dst(n_topos, nullptr);
    std::vector<uint64_t> caps(n_topos, 0);
    std::vector<tacos_result> res(n_topos);
    std::vector<std::vector<uint64_t>> times(n_topos);
    int dev = -1;
    int rc = cuda_device_ok(&dev);
    if (rc) return rc;
    for (uint32_t i = 0; i < n_topos; ++i) {
      uint64_t n = 0;
      if (!topos[i]) return fail(TACOS_E_INVALID_ARG, "null topology %u", i);
      if ((rc = tacos_max_sends(topos[i], p, &n))) return rc;
      sch[i].reset(new tacos_schedule());
      if (n) {
        sch[i]->host_buf.dev = dev;
        sch[i]->host_buf.p = pinned_pool().alloc(dev, n * sizeof(tacos_send), &sch[i]->host_buf.cls);
        if (!sch[i]->host_buf.p) return fail(TACOS_E_NOMEM, "pinned allocation failed");
        sch[i]->sends = reinterpret_cast<tacos_send *>(sch[i]->host_buf.p);
      }
      dst[i] = sch[i]->sends;
      caps[i] = n;
    }
    const bool keep = (p->flags & TACOS_FLAG_KEEP_SEED_TIMES) != 0;
    uint32_t D = 1;
    if ((rc = resolve_devices(p, &D))) return rc;
    if (D > 1 && n_topos == 1) {  // one topology: its seeds sharded over the devices
      if ((rc = validate_params(p))) return rc;
      rc = synth_sharded(topos[0], p, D, dst[0], caps[0], &res[0], keep ? &times[0] : nullptr);
    } else if (D > 1) {  // topologies dealt round-robin to the devices, all seeds of one on one device
      const uint32_t G = std::min(D, n_topos);
      std::vector<int> rcs(G, 0);
      std::vector<std::string> errs(G);
      auto work = [&](uint32_t g) {
        std::vector<const tacos_topology *> tg;
        std::vector<tacos_send *> dg;
        std::vector<uint64_t> cg;
        std::vector<uint32_t> idx;
        for (uint32_t i = g; i < n_topos; i += G) {
          tg.push_back(topos[i]);
          dg.push_back(dst[i]);
          cg.push_back(caps[i]);
          idx.push_back(i);
        }
        std::vector<tacos_result> rg(tg.size());
        std::vector<std::vector<uint64_t>> tmg(tg.size());
        tacos_synth_params pg = *p;
        pg.n_devices = 1;
        int r = cudaSetDevice((int)g) == cudaSuccess ? TACOS_OK : fail(TACOS_E_CUDA, "cudaSetDevice(%u)", g);
        try {  // no exception may leave a worker thread
          if (!r) r = synth_many(tg.data(), (uint32_t)tg.size(), &pg, dg.data(), cg.data(), rg.data(),
                                 keep ? tmg.data() : nullptr, nullptr);
        } catch (...) {
          r = fail(TACOS_E_NOMEM, "host allocation failed");
        }
        if (!r)
          for (size_t j = 0; j < idx.size(); ++j) {
            res[idx[j]] = rg[j];
            times[idx[j]] = std::move(tmg[j]);
          }
        rcs[g] = r;
        if (r) errs[g] = g_last_error;
      };
      int caller = 0;
      cudaGetDevice(&caller);
      std::vector<std::thread> th;
      for (uint32_t g = 0; g < G; ++g)
        th.emplace_back([&, g] {
          try {
            work(g);
          } catch (...) {
            rcs[g] = TACOS_E_NOMEM;
            errs[g] = "host allocation failed";
          }
        });
      for (auto &t : th) t.join();
      cudaSetDevice(caller);
      for (uint32_t g = 0; g < G && !rc; ++g)
        if (rcs[g]) rc = fail(rcs[g], "device %u: %s", g, errs[g].c_str());
    } else {
      rc = synth_many(topos, n_topos, p, dst.data(), caps.data(), res.data(), keep ? times.data() : nullptr, nullptr);
    }
    if (rc) return rc;
    for (uint32_t i = 0; i < n_topos; ++i) {
      sch[i]->result = res[i];
      sch[i]->n_sends = res[i].n_sends;
      sch[i]->seed_times = std::move(times[i]);
      outs[i] = sch[i].release();
    }
    return TACOS_OK;
  } catch (const std::bad_alloc &) {
    return fail(TACOS_E_NOMEM, "host allocation failed");
  }
}

extern "C" int tacos_synthesize(const tacos_topology *topo, const tacos_synth_params *p, tacos_schedule **out) {
  if (out) *out = nullptr;
  if (!topo || !out) return fail(TACOS_E_INVALID_ARG, "null argument");
  const tacos_topology *ts[1] = {topo};
  return tacos_synthesize_batch(ts, 1, p, out);
}

extern "C" uint64_t tacos_schedule_num_sends(const tacos_schedule *s) { return s ? s->n_sends : 0; }
extern "C" const tacos_send *tacos_schedule_sends(const tacos_schedule *s) { return s ? s->sends : nullptr; }
extern "C" uint64_t tacos_schedule_time(const tacos_schedule *s) { return s ? s->result.T : 0; }
extern "C" uint64_t tacos_schedule_seed(const tacos_schedule *s) { return s ? s->result.seed : 0; }
extern "C" const tacos_result *tacos_schedule_result(const tacos_schedule *s) { return s ? &s->result : nullptr; }
extern "C" const uint64_t *tacos_schedule_seed_times(const tacos_schedule *s) {
  return s && !s->seed_times.empty() ? s->seed_times.data() : nullptr;
}
extern "C" void tacos_free_schedule(tacos_schedule *s) { delete s; }

// ---------------------------------------------------------------------------
// NCCL communicator of a multi-process job (one rank per GPU) and the exchange step
// ---------------------------------------------------------------------------
struct tacos_comm {
  ncclComm_t comm = nullptr;
  int device = -1;
  const NcclApi *api = nullptr;
};

extern "C" int tacos_nccl_version(int32_t *version) {
  if (!version) return fail(TACOS_E_INVALID_ARG, "null argument");
  std::string err;
  const NcclApi *api = nccl_api(&err);
  if (!api) return fail(TACOS_E_NCCL, "%s", err.c_str());
  int v = 0;
  if (api->GetVersion(&v) != ncclSuccess) return fail(TACOS_E_NCCL, "ncclGetVersion failed");
  *version = v;
  return TACOS_OK;
}

extern "C" int tacos_comm_unique_id(uint8_t id[TACOS_COMM_ID_BYTES]) {
  if (!id) return fail(TACOS_E_INVALID_ARG, "null argument");
  static_assert(sizeof(ncclUniqueId) == TACOS_COMM_ID_BYTES, "NCCL unique id size");
  std::string err;
  const NcclApi *api = nccl_api(&err);
  if (!api) return fail(TACOS_E_NCCL, "%s", err.c_str());
  ncclUniqueId u;
  const ncclResult_t r = api->GetUniqueId(&u);
  if (r != ncclSuccess) return fail(TACOS_E_NCCL, "ncclGetUniqueId: %s", api->GetErrorString(r));
  std::memcpy(id, &u, sizeof(u));
  return TACOS_OK;
}

extern "C" int tacos_comm_init_rank(const uint8_t id[TACOS_COMM_ID_BYTES], int32_t n_ranks, int32_t rank,
                                    tacos_comm **out) {
  if (out) *out = nullptr;
  if (!id || !out || n_ranks < 1 || rank < 0 || rank >= n_ranks) return fail(TACOS_E_INVALID_ARG, "bad argument");
  int dev = -1, rc;
  if ((rc = cuda_device_ok(&dev))) return rc;
  std::string err;
  const NcclApi *api = nccl_api(&err);
  if (!api) return fail(TACOS_E_NCCL, "%s", err.c_str());
  std::unique_ptr<tacos_comm> c(new (std::nothrow) tacos_comm());
  if (!c) return fail(TACOS_E_NOMEM, "host allocation failed");
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  const ncclResult_t r = api->CommInitRank(&c->comm, n_ranks, u, rank);
  if (r != ncclSuccess) return fail(TACOS_E_NCCL, "ncclCommInitRank: %s", api->GetErrorString(r));
  c->device = dev;
  c->api = api;
  *out = c.release();
  return TACOS_OK;
}

extern "C" void tacos_comm_destroy(tacos_comm *c) {
  if (!c) return;
  if (c->comm && c->api) c->api->CommDestroy(c->comm);
  delete c;
}

extern "C" int tacos_plan_allreduce_keys(tacos_plan *pl, tacos_comm *c, void *stream) {
  if (!pl || !c || !c->comm) return fail(TACOS_E_INVALID_ARG, "null argument");
  if (pl->device != c->device)
    return fail(TACOS_E_INVALID_ARG, "plan on device %d, communicator on device %d", pl->device, c->device);
  uint64_t *keys = pl->parts[0].d_keys;
  const ncclResult_t r = c->api->AllReduce(keys, keys, 2, ncclUint64, ncclMin, c->comm, (cudaStream_t)stream);
  if (r != ncclSuccess) return fail(TACOS_E_NCCL, "ncclAllReduce: %s", c->api->GetErrorString(r));
  return TACOS_OK;
}

// ---------------------------------------------------------------------------
// tacos_eval: host replay ("a TEN link matched with a chunk";
// P:L266-267 arrival before departure; P:L89 postcondition; R8 occupancy)
// ---------------------------------------------------------------------------
namespace {
struct Checker {
  tacos_eval_report *rep;
  void add(int kind, uint64_t idx) {
    rep->per_kind[kind]++;
    rep->n_violations++;
    if (rep->first_kind < 0) {
      rep->first_kind = kind;
      rep->first_index = idx;
    }
  }
};

// Greedy rules of one AG-like phase (P:L253 maximal matching per
// event, P:L263-264 shorter-link-first): replay the events t < T (t = 0 and every
// arrival time) in order; at t, after the arrivals at t (R7), every idle link a->b
// (no send on it covers t) must have each candidate c in post[b] & held[a] - held[b]
// - in flight to b claimed for b by a send starting at t, on a link no costlier than
// itself.  A link is re-examined only when its source gained a chunk since its last
// idle examination: its candidates then were all claimed (or reported) and every
// later candidate must be a newer arrival at the source (held and in-flight sets only
// grow).  Sends with structural violations are excluded (`ok`).
void check_greedy_rules(const tacos_topology *t, const std::vector<uint32_t> &w, int o,
                        const std::vector<tacos_send> &s, const std::vector<size_t> &ok, uint32_t C,
                        const std::vector<uint32_t> &pre, const std::vector<uint32_t> &post, uint32_t W0,
                        Checker &ck) {
  const uint32_t N = (uint32_t)t->N, L = (uint32_t)t->L;
  if (ok.empty()) return;
  std::vector<size_t> by_start(ok), by_end(ok);
  std::stable_sort(by_start.begin(), by_start.end(), [&](size_t x, size_t y) { return s[x].t_start < s[y].t_start; });
  std::stable_sort(by_end.begin(), by_end.end(), [&](size_t x, size_t y) { return s[x].t_end < s[y].t_end; });
  uint64_t T = 0;
  for (size_t i : ok) T = std::max<uint64_t>(T, s[i].t_end);
  std::vector<uint32_t> held(pre), pend((size_t)N * W0, 0u);
  (void)C;
  std::vector<uint32_t> ver(N, 1u), seen(L, 0u);  // source version at the link's last idle examination
  std::vector<uint64_t> busy_until(L, 0ull);      // end of the latest send started on the link
  std::vector<std::vector<std::pair<uint32_t, uint32_t>>> claims(N);  // per dst at t: (chunk, cost)
  std::vector<uint32_t> touched;
  std::vector<char> starting(L, 0);
  size_t ia = 0, is = 0;
  uint64_t tcur = 0;
  for (;;) {
    // arrivals at tcur (R7): held by dst, no longer in flight
    while (ia < by_end.size() && s[by_end[ia]].t_end <= tcur) {
      const tacos_send &e = s[by_end[ia++]];
      const size_t wd = (size_t)e.dst * W0 + (e.chunk >> 5);
      const uint32_t m = 1u << (e.chunk & 31u);
      held[wd] |= m;
      pend[wd] &= ~m;
      ++ver[e.dst];
    }
    if (tcur >= T) break;
    // the matching of event tcur: sends starting at tcur
    const size_t is0 = is;
    while (is < by_start.size() && s[by_start[is]].t_start == tcur) {
      const tacos_send &e = s[by_start[is++]];
      if (claims[e.dst].empty()) touched.push_back(e.dst);
      claims[e.dst].push_back({e.chunk, w[e.link]});
      starting[e.link] = 1;
    }
    for (uint32_t l = 0; l < L; ++l) {
      if (starting[l] || busy_until[l] > tcur) continue;  // not idle at tcur
      const uint32_t a = (uint32_t)(o == 0 ? t->src[l] : t->dst[l]);
      const uint32_t b = (uint32_t)(o == 0 ? t->dst[l] : t->src[l]);
      if (seen[l] == ver[a]) continue;  // source unchanged since its last idle examination
      seen[l] = ver[a];
      const uint32_t *ha = &held[(size_t)a * W0], *hb = &held[(size_t)b * W0], *pb = &pend[(size_t)b * W0];
      const uint32_t *qb = &post[(size_t)b * W0];
      bool bad_max = false, bad_sf = false;
      for (uint32_t i = 0; i < W0; ++i) {
        for (uint32_t m = ha[i] & qb[i] & ~hb[i] & ~pb[i]; m; m &= m - 1) {
          const uint32_t c = i * 32u + (uint32_t)__builtin_ctz(m);
          const auto &cl = claims[b];
          auto it = std::find_if(cl.begin(), cl.end(), [&](const std::pair<uint32_t, uint32_t> &x) { return x.first == c; });
          if (it == cl.end()) bad_max = true;
          else if (it->second > w[l]) bad_sf = true;
        }
      }
      if (bad_max) ck.add(TACOS_V_NOT_MAXIMAL, l);
      if (bad_sf) ck.add(TACOS_V_NOT_SHORTER_FIRST, l);
    }
    // this event's sends are in flight from now on
    for (size_t j = is0; j < is; ++j) {
      const tacos_send &e = s[by_start[j]];
      pend[(size_t)e.dst * W0 + (e.chunk >> 5)] |= 1u << (e.chunk & 31u);
      busy_until[e.link] = std::max<uint64_t>(busy_until[e.link], e.t_end);
      starting[e.link] = 0;
    }
    for (uint32_t x : touched) claims[x].clear();
    touched.clear();
    // next event: the next arrival time (matching runs only at arrivals, R20)
    if (ia >= by_end.size()) break;
    tcur = s[by_end[ia]].t_end;
  }
}

// One AG-like phase on orientation o (0: links as given, 1: reversed).
void check_phase(const tacos_topology *t, const std::vector<uint32_t> &w, int o, const std::vector<tacos_send> &s,
                 const std::vector<uint64_t> &index, uint32_t C, const std::vector<uint32_t> &pre,
                 const std::vector<uint32_t> &post, uint32_t W0, Checker &ck, bool greedy) {
  const uint32_t N = (uint32_t)t->N;
  const uint64_t kNever = ~0ull;
  std::vector<uint64_t> arrive((size_t)N * C, kNever);
  for (uint32_t x = 0; x < N; ++x)
    for (uint32_t c = 0; c < C; ++c)
      if ((pre[(size_t)x * W0 + (c >> 5)] >> (c & 31)) & 1u) arrive[(size_t)x * C + c] = 0;
  std::vector<size_t> ok;
  ok.reserve(s.size());
  for (size_t i = 0; i < s.size(); ++i) {
    const tacos_send &e = s[i];
    if (e.link >= (uint32_t)t->L || e.chunk >= C || e.src >= N || e.dst >= N) {
      ck.add(TACOS_V_NO_SUCH_LINK, index[i]);
      continue;
    }
    const uint32_t a = (uint32_t)(o == 0 ? t->src[e.link] : t->dst[e.link]);
    const uint32_t b = (uint32_t)(o == 0 ? t->dst[e.link] : t->src[e.link]);
    if (a != e.src || b != e.dst) {
      ck.add(TACOS_V_NO_SUCH_LINK, index[i]);
      continue;
    }
    if (e.t_end < e.t_start || e.t_end - e.t_start != w[e.link]) ck.add(TACOS_V_WRONG_DURATION, index[i]);
    ok.push_back(i);
  }
  // link intervals disjoint
  std::vector<size_t> by_link(ok);
  std::sort(by_link.begin(), by_link.end(), [&](size_t x, size_t y) {
    return s[x].link != s[y].link ? s[x].link < s[y].link : s[x].t_start < s[y].t_start;
  });
  for (size_t j = 1; j < by_link.size(); ++j) {
    const tacos_send &a = s[by_link[j - 1]], &b = s[by_link[j]];
    if (a.link == b.link && b.t_start < a.t_end) ck.add(TACOS_V_LINK_OVERLAP, index[by_link[j]]);
  }
  // deliveries in arrival order; exactly once
  std::vector<size_t> by_end(ok);
  std::stable_sort(by_end.begin(), by_end.end(), [&](size_t x, size_t y) { return s[x].t_end < s[y].t_end; });
  for (size_t j : by_end) {
    const tacos_send &e = s[j];
    uint64_t &a = arrive[(size_t)e.dst * C + e.chunk];
    if (a != kNever) ck.add(TACOS_V_DUPLICATE_DELIVERY, index[j]);
    else a = e.t_end;
  }
  for (size_t j : ok) {
    const tacos_send &e = s[j];
    const uint64_t a = arrive[(size_t)e.src * C + e.chunk];
    if (a == kNever || a > e.t_start) ck.add(TACOS_V_UNHELD_AT_DEPART, index[j]);
  }
  for (uint32_t x = 0; x < N; ++x)
    for (uint32_t c = 0; c < C; ++c)
      if (((post[(size_t)x * W0 + (c >> 5)] >> (c & 31)) & 1u) && arrive[(size_t)x * C + c] == kNever)
        ck.add(TACOS_V_POST_UNMET, (uint64_t)x * C + c);
  if (greedy) check_greedy_rules(t, w, o, s, ok, C, pre, post, W0, ck);
}
}  // namespace

extern "C" int tacos_eval(const tacos_topology *t, const tacos_synth_params *p, const tacos_send *sends,
                          uint64_t n_sends, tacos_eval_report *out) {
  if (!t || !p || !out || (!sends && n_sends)) return fail(TACOS_E_INVALID_ARG, "null argument");
  int rc = validate_params(p);
  if (rc) return rc;
  try {
    std::memset(out, 0, sizeof(*out));
    out->first_kind = -1;
    std::vector<uint32_t> w;
    if ((rc = link_costs(t, p->chunk_bytes, p->time_unit_ns ? p->time_unit_ns : 1u, w))) return rc;
    const uint32_t N = (uint32_t)t->N;
    uint32_t C;
    std::vector<uint32_t> pre, post;
    uint32_t W0;
    if (coll_custom(p->collective)) {  // REDUCE / GATHER: the forward problem, checked on G^T below
      if ((rc = problem_bits(N, p, C, pre, post))) return rc;
      W0 = (C + 31) / 32;
    } else {
      C = N * p->chunks_per_npu;
      W0 = (C + 31) / 32;
      pre.assign((size_t)N * W0, 0u);
      post.assign((size_t)N * W0, 0u);
      for (uint32_t x = 0; x < N; ++x)
        for (uint32_t c = 0; c < C; ++c) {
          post[(size_t)x * W0 + (c >> 5)] |= 1u << (c & 31);
          if (c / p->chunks_per_npu == x) pre[(size_t)x * W0 + (c >> 5)] |= 1u << (c & 31);
        }
    }
    Checker ck{out};
    // the greedy rules hold for link-first searches without relays (R1, R4); the literal
    // variant (R21) and relay collectives (R22) follow other rules
    const bool greedy = (p->flags & TACOS_FLAG_LITERAL) == 0 && !coll_relay(p);
    uint64_t T = 0;
    for (uint64_t i = 0; i < n_sends; ++i) T = std::max<uint64_t>(T, sends[i].t_end);
    out->T = T;
    std::vector<tacos_send> all(sends, sends + n_sends);
    std::vector<uint64_t> idx(n_sends);
    for (uint64_t i = 0; i < n_sends; ++i) idx[i] = i;
    if (!coll_need_rs(p->collective)) {  // AG, CUSTOM, BROADCAST, SCATTER
      check_phase(t, w, 0, all, idx, C, pre, post, W0, ck, greedy);
      return TACOS_OK;
    }
    // RS part (all of an RS; the earliest half of an AR): mirror back into an AG on G^T
    std::vector<uint64_t> order(n_sends);
    for (uint64_t i = 0; i < n_sends; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) {
      return all[a].t_start != all[b].t_start ? all[a].t_start < all[b].t_start : all[a].link < all[b].link;
    });
    const uint64_t n_rs = p->collective == TACOS_ALL_REDUCE ? n_sends / 2 : n_sends;
    uint64_t T_rs = 0;
    for (uint64_t j = 0; j < n_rs; ++j) T_rs = std::max<uint64_t>(T_rs, all[order[j]].t_end);
    out->T_rs = T_rs;
    std::vector<tacos_send> rs(n_rs), ag;
    std::vector<uint64_t> rs_idx(n_rs), ag_idx;
    for (uint64_t j = 0; j < n_rs; ++j) {
      const tacos_send &e = all[order[j]];
      tacos_send m = e;
      m.src = e.dst;
      m.dst = e.src;
      m.t_start = T_rs - std::min<uint64_t>(T_rs, e.t_end);
      m.t_end = T_rs - std::min<uint64_t>(T_rs, e.t_start);
      rs[j] = m;
      rs_idx[j] = order[j];
    }
    check_phase(t, w, 1, rs, rs_idx, C, pre, post, W0, ck, greedy);
    if (p->collective == TACOS_ALL_REDUCE) {
      for (uint64_t j = n_rs; j < n_sends; ++j) {
        tacos_send e = all[order[j]];
        if (e.t_start < T_rs) {
          ck.add(TACOS_V_PHASE_ORDER, order[j]);
          continue;
        }
        e.t_start -= T_rs;
        e.t_end -= T_rs;
        ag.push_back(e);
        ag_idx.push_back(order[j]);
      }
      check_phase(t, w, 0, ag, ag_idx, C, pre, post, W0, ck, greedy);
    }
    return TACOS_OK;
  } catch (const std::bad_alloc &) {
    return fail(TACOS_E_NOMEM, "host allocation failed");
  }
}

// ---------------------------------------------------------------------------
extern "C" const char *tacos_strerror(int code) {
  switch (code) {
    case TACOS_OK: return "ok";
    case TACOS_E_INVALID_ARG: return "invalid argument";
    case TACOS_E_TOPOLOGY: return "invalid topology";
    case TACOS_E_UNREACHABLE: return "postcondition unreachable";
    case TACOS_E_CUDA: return "CUDA error";
    case TACOS_E_NOMEM: return "out of memory";
    case TACOS_E_OVERFLOW: return "value out of supported range";
    case TACOS_E_VERIFY: return "verification failed";
    case TACOS_E_NCCL: return "NCCL error";
    case TACOS_E_CAPACITY: return "output buffer too small";
    default: return "unknown error";
  }
}
extern "C" const char *tacos_last_error(void) { return g_last_error.c_str(); }
extern "C" int tacos_abi_version(void) { return TACOS_ABI_VERSION; }

extern "C" int tacos_philox_device(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  if (!ctr || !key || !out) return fail(TACOS_E_INVALID_ARG, "null argument");
  int dev, rc;
  if ((rc = cuda_device_ok(&dev))) return rc;
  uint32_t h[6] = {ctr[0], ctr[1], ctr[2], ctr[3], key[0], key[1]};
  uint32_t *d = nullptr;
  CUDA_TRY(cudaMalloc(&d, 64));
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  rc = launch_philox_probe(d, d + 8, nullptr);
  if (rc == 0) {
    cudaError_t e = cudaMemcpy(out, d + 8, 16, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = fail(TACOS_E_CUDA, "%s", cudaGetErrorString(e));
  } else {
    rc = fail(rc, "%s", cuda_error_string());
  }
  cudaFree(d);
  return rc;
}

// ---------------------------------------------------------------------------
// Topology front-end (f4): hierarchical products of dimensions with switch
// unwinding (§IV.D), NPU removal.
// ---------------------------------------------------------------------------
namespace {
struct DimLink {
  uint32_t a, b, alpha, bw;
};

int dim_links(const tacos_dim_spec &d, std::vector<DimLink> &out) {
  out.clear();
  const uint32_t n = d.n;
  if (n < 2) return fail(TACOS_E_INVALID_ARG, "dimension of size %u < 2", n);
  if (d.bw == 0) return fail(TACOS_E_INVALID_ARG, "dimension bandwidth 0");
  switch (d.kind) {
    case TACOS_DIM_RING:
      for (uint32_t i = 0; i < n; ++i) {
        out.push_back({i, (i + 1) % n, d.alpha_ns, d.bw});
        if (d.bidirectional && n > 2) out.push_back({i, (i + n - 1) % n, d.alpha_ns, d.bw});
      }
      return TACOS_OK;
    case TACOS_DIM_FC:
      for (uint32_t i = 0; i < n; ++i)
        for (uint32_t j = 0; j < n; ++j)
          if (i != j) out.push_back({i, j, d.alpha_ns, d.bw});
      return TACOS_OK;
    case TACOS_DIM_SWITCH: {
      const uint32_t deg = d.degree;
      if (deg < 1 || deg > n - 1) return fail(TACOS_E_INVALID_ARG, "switch degree %u outside [1, %u]", deg, n - 1);
      if (d.bw % deg != 0) return fail(TACOS_E_INVALID_ARG, "switch bandwidth %u not divisible by degree %u", d.bw, deg);
      if (deg == 1 && d.bidirectional) {  // the paper's bi-directional ring variation, full bandwidth
        for (uint32_t i = 0; i < n; ++i) {
          out.push_back({i, (i + 1) % n, d.alpha_ns, d.bw});
          if (n > 2) out.push_back({i, (i + n - 1) % n, d.alpha_ns, d.bw});
        }
        return TACOS_OK;
      }
      for (uint32_t i = 0; i < n; ++i)
        for (uint32_t s = 1; s <= deg; ++s) out.push_back({i, (i + s) % n, d.alpha_ns, d.bw / deg});
      return TACOS_OK;
    }
    case TACOS_DIM_PATH:
      for (uint32_t i = 0; i < n; ++i) {
        if (i + 1 < n) out.push_back({i, i + 1, d.alpha_ns, d.bw});
        if (i >= 1) out.push_back({i, i - 1, d.alpha_ns, d.bw});
      }
      return TACOS_OK;
    default:
      return fail(TACOS_E_INVALID_ARG, "unknown dimension kind %d", d.kind);
  }
}
}  // namespace

extern "C" int tacos_build_hierarchical(const tacos_dim_spec *dims, uint32_t n_dims, int32_t *n_npus,
                                        int32_t *n_links, int32_t *src, int32_t *dst, uint32_t *alpha_ns,
                                        uint32_t *bw, int64_t capacity) {
  if (!dims || n_dims == 0 || !n_npus || !n_links) return fail(TACOS_E_INVALID_ARG, "null argument");
  try {
    std::vector<std::vector<DimLink>> per(n_dims);
    std::vector<std::vector<uint32_t>> start(n_dims);  // per dim: links of coordinate c at [start[c], start[c+1])
    uint64_t N = 1;
    for (uint32_t i = 0; i < n_dims; ++i) {
      int rc = dim_links(dims[i], per[i]);
      if (rc) return rc;
      N *= dims[i].n;
      if (N >= (1ull << 31)) return fail(TACOS_E_INVALID_ARG, "too many NPUs");
      auto &st = start[i];
      st.assign(dims[i].n + 1, 0u);
      for (const DimLink &l : per[i]) st[l.a + 1]++;
      for (uint32_t c = 0; c < dims[i].n; ++c) st[c + 1] += st[c];
      std::stable_sort(per[i].begin(), per[i].end(), [](const DimLink &x, const DimLink &y) { return x.a < y.a; });
    }
    uint64_t L = 0;
    for (uint32_t i = 0; i < n_dims; ++i) L += per[i].size() * (N / dims[i].n);
    if (L >= (1ull << 31)) return fail(TACOS_E_INVALID_ARG, "too many links");
    *n_npus = (int32_t)N;
    *n_links = (int32_t)L;
    if (capacity == 0) return TACOS_OK;
    if ((uint64_t)capacity < L) return fail(TACOS_E_CAPACITY, "capacity %lld < %llu links", (long long)capacity, (unsigned long long)L);
    if (!src || !dst || !alpha_ns || !bw) return fail(TACOS_E_INVALID_ARG, "null output array");
    uint64_t k = 0;
    std::vector<uint32_t> coord(n_dims);
    for (uint64_t x = 0; x < N; ++x) {
      uint64_t r = x;
      for (uint32_t i = 0; i < n_dims; ++i) {
        coord[i] = (uint32_t)(r % dims[i].n);
        r /= dims[i].n;
      }
      uint64_t stride = 1;
      for (uint32_t i = 0; i < n_dims; ++i) {
        const uint32_t c = coord[i];
        for (uint32_t e = start[i][c]; e < start[i][c + 1]; ++e) {
          const DimLink &l = per[i][e];
          src[k] = (int32_t)x;
          dst[k] = (int32_t)(x + ((int64_t)l.b - (int64_t)c) * (int64_t)stride);
          alpha_ns[k] = l.alpha;
          bw[k] = l.bw;
          ++k;
        }
        stride *= dims[i].n;
      }
    }
    return TACOS_OK;
  } catch (const std::bad_alloc &) {
    return fail(TACOS_E_NOMEM, "host allocation failed");
  }
}

extern "C" int tacos_remove_npus(int32_t n_npus, int32_t n_links, const int32_t *src, const int32_t *dst,
                                 const uint32_t *alpha_ns, const uint32_t *bw, const int32_t *removed,
                                 uint32_t n_removed, int32_t *out_n_npus, int32_t *out_n_links, int32_t *out_src,
                                 int32_t *out_dst, uint32_t *out_alpha, uint32_t *out_bw, int64_t capacity,
                                 int32_t *old_id) {
  if (n_npus < 1 || n_links < 0 || !out_n_npus || !out_n_links || (n_links && (!src || !dst || !alpha_ns || !bw)) ||
      (n_removed && !removed))
    return fail(TACOS_E_INVALID_ARG, "bad argument");
  try {
    std::vector<char> gone(n_npus, 0);
    for (uint32_t i = 0; i < n_removed; ++i) {
      if (removed[i] < 0 || removed[i] >= n_npus) return fail(TACOS_E_INVALID_ARG, "removed NPU %d out of range", removed[i]);
      gone[removed[i]] = 1;
    }
    std::vector<int32_t> nid(n_npus, -1);
    int32_t n2 = 0;
    for (int32_t x = 0; x < n_npus; ++x)
      if (!gone[x]) {
        if (old_id && capacity > n2) old_id[n2] = x;
        nid[x] = n2++;
      }
    int64_t L2 = 0;
    for (int32_t l = 0; l < n_links; ++l)
      if (src[l] >= 0 && src[l] < n_npus && dst[l] >= 0 && dst[l] < n_npus && !gone[src[l]] && !gone[dst[l]]) ++L2;
    *out_n_npus = n2;
    *out_n_links = (int32_t)L2;
    if (capacity == 0) return TACOS_OK;
    if (capacity < L2) return fail(TACOS_E_CAPACITY, "capacity %lld < %lld links", (long long)capacity, (long long)L2);
    if (!out_src || !out_dst || !out_alpha || !out_bw) return fail(TACOS_E_INVALID_ARG, "null output array");
    int64_t k = 0;
    for (int32_t l = 0; l < n_links; ++l) {
      if (src[l] < 0 || src[l] >= n_npus || dst[l] < 0 || dst[l] >= n_npus) continue;
      if (gone[src[l]] || gone[dst[l]]) continue;
      out_src[k] = nid[src[l]];
      out_dst[k] = nid[dst[l]];
      out_alpha[k] = alpha_ns[l];
      out_bw[k] = bw[l];
      ++k;
    }
    return TACOS_OK;
  } catch (const std::bad_alloc &) {
    return fail(TACOS_E_NOMEM, "host allocation failed");
  }
}

// ---------------------------------------------------------------------------
// Multi-tenant merge (f2; Table VI; reading R23)
// ---------------------------------------------------------------------------
extern "C" int tacos_multi_tenant(uint32_t N, const tacos_tenant *tn, uint32_t n_tenants, uint32_t *n_chunks,
                                  uint32_t *pre, uint32_t *post, uint32_t *first, uint64_t capacity_words) {
  if (!tn || !n_chunks || n_tenants == 0) return fail(TACOS_E_INVALID_ARG, "null argument or no tenant");
  if (N < 2) return fail(TACOS_E_INVALID_ARG, "n_npus = %u < 2", N);
  uint64_t C = 0;
  for (uint32_t i = 0; i < n_tenants; ++i) {
    const tacos_tenant &t = tn[i];
    if (t.kind != TACOS_ALL_GATHER && t.kind != TACOS_BROADCAST && t.kind != TACOS_SCATTER && t.kind != TACOS_GATHER &&
        t.kind != TACOS_REDUCE)
      return fail(TACOS_E_INVALID_ARG, "tenant %u: unknown kind %d", i, t.kind);
    if (t.k < 1) return fail(TACOS_E_INVALID_ARG, "tenant %u: k = 0", i);
    if (t.kind != TACOS_ALL_GATHER && t.root >= N) return fail(TACOS_E_INVALID_ARG, "tenant %u: root %u >= N", i, t.root);
    C += t.kind == TACOS_BROADCAST ? (uint64_t)t.k : (uint64_t)N * t.k;
    if (C > kMaxChunks) return fail(TACOS_E_OVERFLOW, "merged tenants need more than %u chunks", kMaxChunks);
  }
  *n_chunks = (uint32_t)C;
  if (capacity_words == 0) return TACOS_OK;
  const uint32_t W0 = ((uint32_t)C + 31u) / 32u;
  if (capacity_words < (uint64_t)N * W0)
    return fail(TACOS_E_CAPACITY, "capacity %llu < %llu words", (unsigned long long)capacity_words,
                (unsigned long long)N * W0);
  if (!pre || !post || !first) return fail(TACOS_E_INVALID_ARG, "null output array");
  std::memset(pre, 0, sizeof(uint32_t) * (size_t)N * W0);
  std::memset(post, 0, sizeof(uint32_t) * (size_t)N * W0);
  auto set = [&](uint32_t *v, uint32_t x, uint32_t c) { v[(size_t)x * W0 + (c >> 5)] |= 1u << (c & 31u); };
  uint32_t base = 0;
  for (uint32_t i = 0; i < n_tenants; ++i) {
    const tacos_tenant &t = tn[i];
    const uint32_t span = t.kind == TACOS_BROADCAST ? t.k : N * t.k;
    first[i] = base;
    for (uint32_t j = 0; j < span; ++j) {
      const uint32_t c = base + j, owner = j / t.k;
      switch (t.kind) {
        case TACOS_ALL_GATHER:
          set(pre, owner, c);
          for (uint32_t x = 0; x < N; ++x) set(post, x, c);
          break;
        case TACOS_BROADCAST:
          set(pre, t.root, c);
          for (uint32_t x = 0; x < N; ++x) set(post, x, c);
          break;
        case TACOS_SCATTER:
          set(pre, t.root, c);
          set(post, t.root, c);
          set(post, owner, c);
          break;
        default:  // GATHER, REDUCE (R23)
          set(pre, owner, c);
          set(post, owner, c);
          set(post, t.root, c);
      }
    }
    base += span;
  }
  return TACOS_OK;
}

// ---------------------------------------------------------------------------
// Continuous-time evaluation (f3) and the Ring
// / Direct baselines.
// ---------------------------------------------------------------------------
namespace {
int params_chunks(const tacos_topology *t, const tacos_synth_params *p, uint32_t &C, std::vector<uint32_t> &pre,
                  uint32_t &W0) {
  const uint32_t N = (uint32_t)t->N;
  if (coll_custom(p->collective)) {
    std::vector<uint32_t> post;
    int rc = problem_bits(N, p, C, pre, post);
    if (rc) return rc;
    W0 = (C + 31) / 32;
  } else {
    C = N * p->chunks_per_npu;
    W0 = (C + 31) / 32;
    pre.assign((size_t)N * W0, 0u);
    for (uint32_t c = 0; c < C; ++c) {
      const uint32_t x = c / p->chunks_per_npu;
      pre[(size_t)x * W0 + (c >> 5)] |= 1u << (c & 31);
    }
  }
  return TACOS_OK;
}
}  // namespace

extern "C" int tacos_eval_continuous(const tacos_topology *t, const tacos_synth_params *p, const tacos_send *sends,
                                     uint64_t n_sends, tacos_cont_report *out) {
  if (!t || !p || !out || (!sends && n_sends)) return fail(TACOS_E_INVALID_ARG, "null argument");
  int rc = validate_params(p);
  if (rc) return rc;
  try {
    std::memset(out, 0, sizeof(*out));
    const uint32_t N = (uint32_t)t->N, L = (uint32_t)t->L;
    std::vector<double> dur(L);
    for (uint32_t l = 0; l < L; ++l) dur[l] = (double)t->alpha[l] + (double)p->chunk_bytes / (double)t->bw[l];
    uint32_t C, W0;
    std::vector<uint32_t> pre;
    if ((rc = params_chunks(t, p, C, pre, W0))) return rc;
    std::vector<uint64_t> ord(n_sends);
    for (uint64_t i = 0; i < n_sends; ++i) {
      const tacos_send &s = sends[i];
      if (s.link >= L || s.chunk >= C || s.src != (uint32_t)t->src[s.link] || s.dst != (uint32_t)t->dst[s.link])
        return fail(TACOS_E_VERIFY, "send %llu does not match its link", (unsigned long long)i);
      ord[i] = i;
    }
    std::stable_sort(ord.begin(), ord.end(), [&](uint64_t a, uint64_t b) { return sends[a].t_start < sends[b].t_start; });
    // reduction-phase replay for RS / REDUCE / GATHER (a node sends a chunk once everything it
    // receives of that chunk has arrived; GATHER receives each chunk at most once)
    const bool ar = p->collective == TACOS_ALL_REDUCE, rs = coll_need_rs(p->collective) && !ar;
    uint64_t n_rs = ar ? n_sends / 2 : (rs ? n_sends : 0);
    if (ar) {  // phase split by (t_start, link), as tacos_eval
      std::vector<uint64_t> o2(ord);
      std::stable_sort(o2.begin(), o2.end(), [&](uint64_t a, uint64_t b) {
        return sends[a].t_start != sends[b].t_start ? sends[a].t_start < sends[b].t_start : sends[a].link < sends[b].link;
      });
      std::vector<char> in_rs(n_sends, 0);
      for (uint64_t j = 0; j < n_rs; ++j) in_rs[o2[j]] = 1;
      std::stable_partition(ord.begin(), ord.end(), [&](uint64_t i) { return in_rs[i] != 0; });
    }
    const double kInf = std::numeric_limits<double>::infinity();
    std::vector<double> link_free(L, 0.0), busy(L, 0.0);
    std::vector<double> rs_in((size_t)N * C, 0.0);
    double T_rs = 0.0, T = 0.0;
    for (uint64_t j = 0; j < n_rs; ++j) {  // reduction phase: a sends once its partial is complete
      const tacos_send &s = sends[ord[j]];
      const double ready = rs_in[(size_t)s.src * C + s.chunk];
      const double st = std::max(ready, link_free[s.link]);
      const double en = st + dur[s.link];
      link_free[s.link] = en;
      busy[s.link] += dur[s.link];
      double &r = rs_in[(size_t)s.dst * C + s.chunk];
      r = std::max(r, en);
      T_rs = std::max(T_rs, en);
    }
    std::vector<double> avail((size_t)N * C, kInf);
    for (uint32_t x = 0; x < N; ++x)
      for (uint32_t c = 0; c < C; ++c)
        if ((pre[(size_t)x * W0 + (c >> 5)] >> (c & 31)) & 1u) avail[(size_t)x * C + c] = ar ? std::max(T_rs, rs_in[(size_t)x * C + c]) : 0.0;
    T = T_rs;
    for (uint64_t j = n_rs; j < n_sends; ++j) {  // data movement phase
      const tacos_send &s = sends[ord[j]];
      const double ready = avail[(size_t)s.src * C + s.chunk];
      if (ready == kInf)
        return fail(TACOS_E_VERIFY, "send %llu (chunk %u at NPU %u) departs before its chunk is available",
                    (unsigned long long)ord[j], s.chunk, s.src);
      const double st = std::max(ready, link_free[s.link]);
      const double en = st + dur[s.link];
      link_free[s.link] = en;
      busy[s.link] += dur[s.link];
      double &a = avail[(size_t)s.dst * C + s.chunk];
      a = std::min(a, en);
      T = std::max(T, en);
    }
    out->T_ns = T;
    out->T_rs_ns = T_rs;
    out->n_sends = n_sends;
    for (uint32_t l = 0; l < L; ++l) out->max_link_busy_ns = std::max(out->max_link_busy_ns, busy[l]);
    return TACOS_OK;
  } catch (const std::bad_alloc &) {
    return fail(TACOS_E_NOMEM, "host allocation failed");
  }
}

namespace {
// Shortest paths in hops from s: BFS visiting out-links in link-id order
// (orientation o: 0 = G, 1 = G^T).  parent[x] = link into x on the path.
void bfs_parents(const tacos_topology *t, int o, uint32_t s, std::vector<int32_t> &parent) {
  const uint32_t N = (uint32_t)t->N;
  parent.assign(N, -1);
  std::vector<char> seen(N, 0);
  std::vector<uint32_t> q{s};
  seen[s] = 1;
  // out-links of x in G are the in-links of x in G^T's CSR (orientation 1 groups by src)
  const int oo = 1 - o;
  for (size_t h = 0; h < q.size(); ++h) {
    const uint32_t x = q[h];
    for (uint32_t e = t->in_ptr[oo][x]; e < t->in_ptr[oo][x + 1]; ++e) {
      const uint32_t y = t->pos_src[oo][e];  // other endpoint
      if (!seen[y]) {
        seen[y] = 1;
        parent[y] = (int32_t)t->pos_lid[oo][e];
        q.push_back(y);
      }
    }
  }
}

struct LSend {
  uint32_t chunk, a, b, link;
  uint64_t key;
};

// AG baseline on orientation o (links as given for o = 0, reversed for o = 1).
int baseline_ag(const tacos_topology *t, uint32_t k, int alg, int o, std::vector<LSend> &out) {
  const uint32_t N = (uint32_t)t->N;
  out.clear();
  std::vector<std::vector<int32_t>> par(N);
  for (uint32_t s = 0; s < N; ++s) bfs_parents(t, o, s, par[s]);
  auto path = [&](uint32_t s, uint32_t d, std::vector<uint32_t> &links) -> bool {
    links.clear();
    uint32_t x = d;
    while (x != s) {
      const int32_t l = par[s][x];
      if (l < 0) return false;
      links.push_back((uint32_t)l);
      x = (uint32_t)(o == 0 ? t->src[l] : t->dst[l]);
    }
    std::reverse(links.begin(), links.end());
    return true;
  };
  auto ends = [&](uint32_t l, uint32_t &a, uint32_t &b) {
    a = (uint32_t)(o == 0 ? t->src[l] : t->dst[l]);
    b = (uint32_t)(o == 0 ? t->dst[l] : t->src[l]);
  };
  std::vector<uint32_t> hops;
  if (alg == TACOS_BASELINE_RING) {
    // logical ring i -> i+1 on G; on G^T (the RS, mirrored back onto G) i -> i-1, so
    // the mirrored reduction ring runs i-1 -> i along G's own direction
    auto succ = [&](uint32_t i) { return o == 0 ? (i + 1) % N : (i + N - 1) % N; };
    auto pred_owner = [&](uint32_t i, uint32_t j) { return o == 0 ? (i + N - j) % N : (i + j) % N; };
    uint64_t H = 1;
    for (uint32_t i = 0; i < N; ++i) {
      if (!path(i, succ(i), hops)) return fail(TACOS_E_UNREACHABLE, "no path %u -> %u", i, succ(i));
      H = std::max<uint64_t>(H, hops.size());
    }
    for (uint32_t j = 0; j + 1 < N; ++j)
      for (uint32_t i = 0; i < N; ++i) {
        const uint32_t owner = pred_owner(i, j);
        path(i, succ(i), hops);
        for (uint32_t h = 0; h < hops.size(); ++h)
          for (uint32_t q = 0; q < k; ++q) {
            LSend s;
            s.chunk = owner * k + q;
            ends(hops[h], s.a, s.b);
            s.link = hops[h];
            s.key = (uint64_t)j * H + h;
            out.push_back(s);
          }
      }
  } else {
    for (uint32_t owner = 0; owner < N; ++owner)
      for (uint32_t d = 0; d < N; ++d) {
        if (d == owner) continue;
        if (!path(owner, d, hops)) return fail(TACOS_E_UNREACHABLE, "no path %u -> %u", owner, d);
        for (uint32_t h = 0; h < hops.size(); ++h)
          for (uint32_t q = 0; q < k; ++q) {
            LSend s;
            s.chunk = owner * k + q;
            ends(hops[h], s.a, s.b);
            s.link = hops[h];
            s.key = h;
            out.push_back(s);
          }
      }
  }
  std::stable_sort(out.begin(), out.end(), [](const LSend &x, const LSend &y) { return x.key < y.key; });
  return TACOS_OK;
}
}  // namespace

extern "C" int tacos_baseline(const tacos_topology *t, const tacos_synth_params *p, int32_t algorithm, tacos_send *out,
                              uint64_t capacity, uint64_t *n_out) {
  if (!t || !p || !n_out) return fail(TACOS_E_INVALID_ARG, "null argument");
  int rc = validate_params(p);
  if (rc) return rc;
  if (coll_custom(p->collective)) return fail(TACOS_E_INVALID_ARG, "baselines are defined for AG / RS / AR");
  if (algorithm != TACOS_BASELINE_RING && algorithm != TACOS_BASELINE_DIRECT)
    return fail(TACOS_E_INVALID_ARG, "unknown baseline %d", algorithm);
  try {
    std::vector<uint32_t> w;
    if ((rc = link_costs(t, p->chunk_bytes, p->time_unit_ns ? p->time_unit_ns : 1u, w))) return rc;
    std::vector<LSend> ag, rsv;
    const int coll = p->collective;
    if (coll != TACOS_REDUCE_SCATTER)
      if ((rc = baseline_ag(t, p->chunks_per_npu, algorithm, 0, ag))) return rc;
    if (coll != TACOS_ALL_GATHER)
      if ((rc = baseline_ag(t, p->chunks_per_npu, algorithm, 1, rsv))) return rc;
    const uint64_t n = ag.size() + rsv.size();
    *n_out = n;
    if (capacity == 0) return TACOS_OK;
    if (capacity < n) return fail(TACOS_E_CAPACITY, "capacity %llu < %llu sends", (unsigned long long)capacity, (unsigned long long)n);
    if (!out) return fail(TACOS_E_INVALID_ARG, "null output");
    uint64_t kmax = 0;
    for (const LSend &s : rsv) kmax = std::max(kmax, s.key);
    uint64_t i = 0;
    // RS: time mirror of the AG on G^T, landing on G's links (R9)
    for (auto it = rsv.rbegin(); it != rsv.rend(); ++it) {
      tacos_send s;
      s.chunk = it->chunk;
      s.src = it->b;
      s.dst = it->a;
      s.link = it->link;
      s.t_start = kmax - it->key;
      s.t_end = s.t_start + w[s.link];
      out[i++] = s;
    }
    const uint64_t shift = rsv.empty() ? 0 : kmax + 1;
    for (const LSend &x : ag) {
      tacos_send s;
      s.chunk = x.chunk;
      s.src = x.a;
      s.dst = x.b;
      s.link = x.link;
      s.t_start = x.key + shift;
      s.t_end = s.t_start + w[s.link];
      out[i++] = s;
    }
    return TACOS_OK;
  } catch (const std::bad_alloc &) {
    return fail(TACOS_E_NOMEM, "host allocation failed");
  }
}
