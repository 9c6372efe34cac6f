// C-ABI implementation: plans, task-list construction and phase orchestration
// for the batched HODLR build / factor / solve / GMRES on one B200.
//
// Level-synchronous restatement of the reference recursion:
//   build   every off-diagonal block of every front in ONE launch (ACA) or
//           one skeleton launch (BDLR)                     src/hodlr.py:239-242
//   factor  Z gather -> batched leaf LU + inverse -> leaf GEMM  (:222-232)
//           then for each level bottom-up: H = V^T [c | d] (GEMM), coupling
//           LU + inverse, Q = S^{-1} rhs (GEMM), c -= d y (GEMM)  (:264-282)
//   solve   leaf apply, then per level V^T x, S^{-1}, x -= d y     (:285-306)
//
// Extension layout: one column-major n x W buffer Y per front with the
// ancestors' U factors FARTHEST FIRST.  Node p at level l then owns the
// rectangle Y[lo_p:hi_p, 0:w_p] (w_p = sum of ancestor ranks on its side),
// and its children's d blocks are Y[rows, w_p : w_p + r].  Nothing is ever
// concatenated (the reference's hstack/vstack at :244-245, :282 disappear).
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/hodlr_b200.h"
#include "hk_graph.h"
#include "hk_internal.h"

// ------------------------------------------------------------------ errors, counters
static thread_local std::string g_err;

// HK_HOST_PROFILE=1: print host-side phase times (planning vs launching vs
// waiting) of build / factor / solve to stderr.
static bool host_profile() {
  static int on = -1;
  if (on < 0) on = getenv("HK_HOST_PROFILE") ? 1 : 0;
  return on == 1;
}
// NVTX range over an API entry point (SURVEY.md §5 tracing): a no-op unless a
// tool that injects NVTX (ncu --nvtx, nsys) is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
struct HostClock {
  const char* what;
  NvtxRange range;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  explicit HostClock(const char* w) : what(w), range(w) {}
  void mark(const char* phase) {
    if (!host_profile()) return;
    auto t1 = std::chrono::steady_clock::now();
    fprintf(stderr, "[hk host] %s %s %.1f us\n", what, phase,
            std::chrono::duration<double, std::micro>(t1 - t0).count());
    t0 = t1;
  }
};
static std::atomic<long long> g_launches{0};

void hk_count_launch(int k) { g_launches += k; }

static hk_status fail(hk_status code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CU(expr)                                                                      \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess)                                                            \
      return fail(HK_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));   \
  } while (0)

#define CHK(expr)                    \
  do {                               \
    hk_status _s = (expr);           \
    if (_s != HK_OK) return _s;      \
  } while (0)

extern "C" const char* hk_last_error(void) { return g_err.c_str(); }
extern "C" const char* hk_version(void) { return "hodlr_b200 0.1.0 sm_100a"; }
extern "C" int hk_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}
extern "C" int64_t hk_launch_count(void) { return g_launches.load(); }

// ------------------------------------------------------------------ device buffers
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t need, cudaStream_t st) {
    if (need <= bytes && p) return cudaSuccess;
    if (p) hk_dev_free(p, st);
    p = nullptr;
    bytes = 0;
    size_t alloc = need < 256 ? 256 : need;
    cudaError_t e = hk_dev_malloc(&p, alloc, st);
    if (e == cudaSuccess) bytes = alloc;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const { return reinterpret_cast<T*>(p); }
};

template <class T>
static cudaError_t upload(DevBuf& b, const std::vector<T>& v, cudaStream_t st) {
  cudaError_t e = b.ensure(v.size() * sizeof(T) + 16, st);
  if (e != cudaSuccess) return e;
  if (v.empty()) return cudaSuccess;
  return cudaMemcpyAsync(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st);
}

// Pinned host staging for task arrays.  An API call packs the task arrays of
// one phase into pinned memory, moves them to the device with ONE asynchronous
// copy (commit) and launches that phase; the host then plans the next phase
// while the GPU runs this one.  Storage is a list of fixed segments (pinned
// host + device twin) so that committed regions never move; segments are
// reused by the next call only after that call's own synchronisation point.
struct Staging {
  struct Seg {
    char* host = nullptr;
    char* dev = nullptr;
    size_t cap = 0, used = 0, committed = 0;
  };
  std::vector<Seg> segs;
  size_t cur = 0;
  static constexpr size_t kSeg = size_t(4) << 20;
  void reset() {
    for (auto& g : segs) g.used = g.committed = 0;
    cur = 0;
  }
  // returns a device pointer valid for launches enqueued after the next commit()
  void* push(const void* src, size_t bytes, cudaStream_t st) {
    for (;;) {
      if (cur == segs.size()) {
        Seg g;
        g.cap = std::max(kSeg, bytes + 256);
        if (cudaHostAlloc((void**)&g.host, g.cap, cudaHostAllocDefault) != cudaSuccess) return nullptr;
        if (hk_dev_malloc((void**)&g.dev, g.cap, st) != cudaSuccess) {
          cudaFreeHost(g.host);
          return nullptr;
        }
        segs.push_back(g);
      }
      Seg& g = segs[cur];
      const size_t off = (g.used + 255) & ~size_t(255);
      if (off + bytes <= g.cap) {
        if (bytes) memcpy(g.host + off, src, bytes);
        g.used = off + bytes;
        return g.dev + off;
      }
      if (commit_seg(g, st) != cudaSuccess) return nullptr;   // full: flush, next segment
      ++cur;
    }
  }
  template <class T>
  T* push(const std::vector<T>& v, cudaStream_t st) {
    if (hk_validate_enabled())
      for (const T& t : v) hk_validate(t);
    return reinterpret_cast<T*>(push(v.data(), v.size() * sizeof(T), st));
  }
  static cudaError_t commit_seg(Seg& g, cudaStream_t st) {
    if (g.used <= g.committed) return cudaSuccess;
    cudaError_t e = cudaMemcpyAsync(g.dev + g.committed, g.host + g.committed, g.used - g.committed,
                                    cudaMemcpyHostToDevice, st);
    g.committed = g.used;
    return e;
  }
  cudaError_t commit(cudaStream_t st) {
    for (size_t i = 0; i <= cur && i < segs.size(); ++i) {
      cudaError_t e = commit_seg(segs[i], st);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  void release() {
    for (auto& g : segs) {
      if (g.host) cudaFreeHost(g.host);
      if (g.dev) cudaFree(g.dev);
    }
    segs.clear();
    cur = 0;
  }
};

static void init_pool_once() {
  static bool done = false;
  if (done) return;
  done = true;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

// ------------------------------------------------------------------ plan
struct Node {
  int level;
  int64_t lo, hi;
  int left, right;
};

struct BlockGeom {
  int node;       // slot
  int side;       // 0 upper, 1 lower
  int64_t row0, col0;
  int m, n, cap;
  int ldu, ldv;          // leading dimensions of the column-major U (m x cap) and V (n x cap)
  int ldu_log, ldv_log;  // both are powers of two >= 64 (compile-time strides in aca.cu)
  int64_t u_off, v_off;   // doubles, within one front's UV region
  int64_t t_off;          // ints, within one front's trace region
};

struct AcaPlanKey {
  const void* ptr[6];
  int64_t v[4];
  bool operator==(const AcaPlanKey& o) const {
    for (int i = 0; i < 6; ++i) if (ptr[i] != o.ptr[i]) return false;
    for (int i = 0; i < 4; ++i) if (v[i] != o.v[i]) return false;
    return true;
  }
};
struct AcaPlanCache {
  AcaPlanKey key{};
  DevBuf tasks;
  size_t ncl_tasks = 0;
  int ngroups = 0;
  int cl_P[4], cl_begin[4], cl_cnt[4], cl_cap[4], cl_m[4];
  int cls_begin[5], cls_cap[4], cls_m[4];
};

struct NodeRec {  // per (front, node) factor storage
  int64_t inv = -1, h = -1, q = -1, m = -1;         // doubles in F pool
  int64_t status = -1;                              // ints in I pool
  int64_t g = -1, yv = -1;                          // solve scratch (doubles) per rhs column
  int R = 0, rl = 0, ru = 0;
  int64_t w = 0, hcols = 0;
};

// A cached solve program: task arrays in the plan's program staging (pstage),
// valid until the next factorization drops them.
struct SolveProg {
  bool small = true;
  int s = 0;
  // small-s: split skinny kernels (pdot -> sgemv(S^-1) -> sgemv(update) per level)
  struct Sg {   // one sgemv launch
    const SgemvTask* t = nullptr;
    const int32_t* items = nullptr;
    int nitems = 0, max_k = 0;
  };
  Sg leaf;
  struct Level {
    const PdotTask* pdot_t = nullptr;
    const int32_t* pdot_items = nullptr;
    int n_pdot = 0;
    Sg sinv, upd;
    // gemm variant
    const GemmTask *g1 = nullptr, *g2 = nullptr, *g3 = nullptr;
    const int32_t *g1map = nullptr, *g2map = nullptr, *g3map = nullptr;
    int t1 = 0, t2 = 0, t3 = 0;
  };
  std::vector<Level> levels;
  const GemmTask* leaf_g = nullptr;
  const int32_t* leaf_map = nullptr;
  int leaf_tiles = 0;
  DevBuf pbuf;          // partial dot products of one level (levels reuse it in stream order)
  // the kernel sequence is captured into a CUDA graph at its second use (a
  // GMRES run applies the same program every iteration); one graph launch
  // then replaces 3 launches per level
  int uses = 0;
  cudaGraphExec_t gexec = nullptr;
  int gkernels = 0;
  // device memory is returned stream-ordered by drop_progs (a plain cudaFree
  // would synchronise the whole device, stalling copies on other streams)
  void free_async(cudaStream_t st) {
    if (pbuf.p) hk_dev_free(pbuf.p, st);
    pbuf.p = nullptr;
    pbuf.bytes = 0;
  }
  ~SolveProg() {
    pbuf.release();
    if (gexec) cudaGraphExecDestroy(gexec);
  }
};

struct GmresGraph;
static void destroy_gmres_graph(GmresGraph* g);

struct hk_plan {
  int64_t n = 0, leaf = 0, batch = 0;
  std::vector<Node> nodes;
  std::vector<int> internal;        // slots, preorder
  std::vector<int> iidx;            // slot -> internal index or -1
  std::vector<int> leaves;          // slots, preorder
  std::vector<int> post;            // slot -> DFS event index (failure ordering)
  int depth = 0;

  // build
  int scheme = -1;
  bool built = false, factored = false;
  const double* A = nullptr;
  int64_t lda = 0, fstride = 0;
  std::vector<BlockGeom> blocks;
  std::vector<int> block_order;     // largest first
  int64_t uv_per_front = 0, trace_per_front = 0;
  DevBuf At, UV, ranks_d, trace_d, tasks_d, aca_scr, aca_cnt;
  cudaStream_t side[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaStream_t cl_side[4] = {nullptr, nullptr, nullptr, nullptr};   // cluster ACA groups
  std::vector<cudaEvent_t> fev;     // factor: staging-commit events (front-group streams)
  // BDLR selection cache (graph hash, depth)
  std::vector<AcaPlanCache> aca_plans;   // cached ACA task lists (hk_build_aca)
  int* started_h = nullptr;         // mapped pinned residency counter of the largest ACA clusters
  int* started_d = nullptr;
  bool sel_valid = false;
  DevBuf gidx_d, selout_d, seltask_d;   // device graph CSR and GPU selection outputs
  uint64_t sel_key = 0;
  std::vector<int64_t> probe_off, probe_cnt;
  int sel_max_k = 0, sel_max_kc = 0;
  size_t gjs_need = 0;              // factor: large-GJ global scratch bytes (0 = none)
  cudaEvent_t cl_side_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t side_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<int32_t> ranks;       // batch * nblocks
  bool have_trace = false;
  // bdlr
  std::vector<std::vector<int64_t>> rsel, csel;  // per block
  DevBuf sel_d, work_d, perm_d, skel_status_d, probe_d;
  std::vector<int64_t> sel_off_r, sel_off_c;     // per block offsets into sel_d
  std::vector<int64_t> perm_off;                  // per (front, block) into perm_d
  // factor
  std::vector<int64_t> W;           // per front
  std::vector<int64_t> y_off;       // per front (doubles)
  std::vector<NodeRec> rec;         // batch * nodes
  DevBuf Y, Ytmp, F, I, ftask_d, fmap_d, gj_d, gj2_d, gjs_d;
  Staging stage;                    // pinned task arena of the current build / factor call
  Staging pstage;                   // task arrays of the cached solve programs
  int64_t g_per_col = 0;            // doubles of G/Yv scratch per rhs column (all fronts)
  std::map<std::pair<int, int>, SolveProg*> progs;
  std::vector<GmresGraph*> gmres_graphs;   // cached device-resident GMRES loops (hk_gmres_batch)
  // TMA tensor map of the fronts for the leaf Gauss-Jordan (hk_gj_leaf_map)
  alignas(64) unsigned char leafmap[128] = {};
  const double* leafmap_base = nullptr;
  int64_t leafmap_key[3] = {0, 0, 0};   // lda, fstride, batch
  bool leafmap_ok = false;
  DevBuf Xin, X2, G, Yv;
  // timings
  double t_lowrank = 0, t_leaf = 0, t_schur = 0, t_aca = 0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};

  int nblocks() const { return (int)blocks.size(); }
  ~hk_plan() {
    for (GmresGraph* g : gmres_graphs) destroy_gmres_graph(g);
    for (auto& kv : progs) delete kv.second;
    for (auto& x : side)
      if (x) cudaStreamDestroy(x);
    for (auto& x : side_ev)
      if (x) cudaEventDestroy(x);
    for (auto& x : cl_side)
      if (x) cudaStreamDestroy(x);
    for (auto& x : cl_side_ev)
      if (x) cudaEventDestroy(x);
    for (auto& x : fev)
      if (x) cudaEventDestroy(x);
    for (auto& c : aca_plans) c.tasks.release();
    if (started_h) cudaFreeHost(started_h);
    DevBuf* bufs[] = {&gidx_d, &selout_d, &seltask_d, &aca_cnt, &aca_scr, &At, &UV, &ranks_d, &trace_d, &tasks_d, &sel_d, &work_d, &perm_d,
                      &skel_status_d, &probe_d, &Y, &Ytmp, &F, &I, &ftask_d, &fmap_d, &gj_d, &gj2_d, &gjs_d,
                      &Xin, &X2, &G, &Yv};
    for (DevBuf* b : bufs) b->release();
    stage.release();
    pstage.release();
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }
};

static void build_tree(hk_plan* p) {
  // preorder, split at ceil(size/2), leaf iff size <= threshold (hodlr.py:76-102)
  struct Item { int level; int64_t lo, hi; int parent, side; };
  std::vector<Item> stack{{0, 0, p->n, -1, 0}};
  while (!stack.empty()) {
    Item it = stack.back();
    stack.pop_back();
    int slot = (int)p->nodes.size();
    p->nodes.push_back({it.level, it.lo, it.hi, -1, -1});
    if (it.parent >= 0) {
      if (it.side == 0) p->nodes[it.parent].left = slot;
      else p->nodes[it.parent].right = slot;
    }
    if (it.hi - it.lo > p->leaf) {
      int64_t mid = it.lo + (it.hi - it.lo + 1) / 2;
      stack.push_back({it.level + 1, mid, it.hi, slot, 1});
      stack.push_back({it.level + 1, it.lo, mid, slot, 0});
    }
  }
  p->iidx.assign(p->nodes.size(), -1);
  for (int s = 0; s < (int)p->nodes.size(); ++s) {
    p->depth = std::max(p->depth, p->nodes[s].level);
    if (p->nodes[s].left >= 0) {
      p->iidx[s] = (int)p->internal.size();
      p->internal.push_back(s);
    } else {
      p->leaves.push_back(s);
    }
  }
  // DFS event order of the reference recursion: compress at entry, leaf LU at
  // entry, Schur at exit (hodlr.py:217-282).  Failure precedence uses the
  // exit/leaf index.
  p->post.assign(p->nodes.size(), 0);
  int cnt = 0;
  std::vector<std::pair<int, int>> st{{0, 0}};
  while (!st.empty()) {
    auto& top = st.back();
    int s = top.first;
    const Node& nd = p->nodes[s];
    if (nd.left < 0) {
      p->post[s] = cnt++;
      st.pop_back();
      continue;
    }
    if (top.second == 0) { top.second = 1; st.push_back({nd.left, 0}); continue; }
    if (top.second == 1) { top.second = 2; st.push_back({nd.right, 0}); continue; }
    p->post[s] = cnt++;
    st.pop_back();
  }
  // block geometry
  for (int k = 0; k < (int)p->internal.size(); ++k) {
    const Node& nd = p->nodes[p->internal[k]];
    const Node& a = p->nodes[nd.left];
    const Node& b = p->nodes[nd.right];
    BlockGeom up{};
    up.node = p->internal[k]; up.side = 0; up.row0 = a.lo; up.col0 = b.lo;
    up.m = (int)(a.hi - a.lo); up.n = (int)(b.hi - b.lo);
    BlockGeom lw{};
    lw.node = p->internal[k]; lw.side = 1; lw.row0 = b.lo; lw.col0 = a.lo;
    lw.m = (int)(b.hi - b.lo); lw.n = (int)(a.hi - a.lo);
    p->blocks.push_back(up);
    p->blocks.push_back(lw);
  }
}

static void set_caps(hk_plan* p, int64_t max_rank) {
  int64_t off = 0, toff = 0;
  for (auto& b : p->blocks) {
    int64_t cap = std::min(b.m, b.n);
    if (max_rank > 0) cap = std::min(cap, max_rank);
    b.cap = (int)cap;
    auto pow2log = [](int v) { int l = 6; while ((1 << l) < v) ++l; return l; };
    // one shared power-of-two leading dimension for U and V (aca.cu template)
    b.ldu_log = b.ldv_log = std::max(pow2log(b.m), pow2log(b.n));
    b.ldu = 1 << b.ldu_log;
    b.ldv = 1 << b.ldv_log;
    // +8 columns of slack: the ACA prefetches whole 8-column chunks
    b.u_off = off;
    off += (int64_t)b.ldu * (cap + 8);
    b.v_off = off;
    off += (int64_t)b.ldv * (cap + 8);
    b.t_off = toff;
    toff += 2 + (b.m + cap + 1) + (cap + 1);
  }
  p->uv_per_front = off;
  p->trace_per_front = toff;
  p->block_order.resize(p->blocks.size());
  for (size_t i = 0; i < p->blocks.size(); ++i) p->block_order[i] = (int)i;
  std::stable_sort(p->block_order.begin(), p->block_order.end(), [&](int a, int b) {
    const BlockGeom &x = p->blocks[a], &y = p->blocks[b];
    return (int64_t)(x.m + x.n) * x.cap > (int64_t)(y.m + y.n) * y.cap;
  });
}

extern "C" hk_status hk_plan_create(int64_t n, int64_t leaf_threshold, int64_t batch,
                                    hk_plan** out) {
  if (!out) return fail(HK_ERR_VALUE, "out is null");
  if (n < 1) return fail(HK_ERR_VALUE, "n must be >= 1");
  if (leaf_threshold < 1) return fail(HK_ERR_VALUE, "leaf_threshold must be >= 1");
  if (batch < 1) return fail(HK_ERR_VALUE, "batch must be >= 1");
  hk_plan* p = new hk_plan();
  p->n = n;
  p->leaf = leaf_threshold;
  p->batch = batch;
  build_tree(p);
  *out = p;
  return HK_OK;
}

extern "C" hk_status hk_plan_destroy(hk_plan* plan) {
  if (plan) {
    cudaDeviceSynchronize();
    delete plan;
  }
  return HK_OK;
}

extern "C" int64_t hk_plan_num_nodes(const hk_plan* p) { return p ? (int64_t)p->nodes.size() : 0; }

extern "C" hk_status hk_plan_tree(const hk_plan* p, int32_t* level, int64_t* lo, int64_t* hi,
                                  int32_t* left, int32_t* right) {
  if (!p) return fail(HK_ERR_VALUE, "null plan");
  for (size_t s = 0; s < p->nodes.size(); ++s) {
    level[s] = p->nodes[s].level;
    lo[s] = p->nodes[s].lo;
    hi[s] = p->nodes[s].hi;
    left[s] = p->nodes[s].left;
    right[s] = p->nodes[s].right;
  }
  return HK_OK;
}

extern "C" hk_status hk_block_shape(const hk_plan* p, int64_t block, int64_t* m, int64_t* n,
                                    int64_t* cap) {
  if (!p || block < 0 || block >= (int64_t)p->blocks.size())
    return fail(HK_ERR_VALUE, "block out of range");
  *m = p->blocks[block].m;
  *n = p->blocks[block].n;
  *cap = p->blocks[block].cap;
  return HK_OK;
}

// callers synchronise the stream first: the programs' task arrays are reused
static void drop_progs(hk_plan* p, cudaStream_t st) {
  // the cached GMRES graphs replay the programs' kernels: drop them too
  for (GmresGraph* g : p->gmres_graphs) destroy_gmres_graph(g);
  p->gmres_graphs.clear();
  for (auto& kv : p->progs) {
    kv.second->free_async(st);
    delete kv.second;
  }
  p->progs.clear();
  p->pstage.reset();
}

// Side streams of the four ACA size classes.  Stream priorities steer the CTA
// scheduler when the classes do not all fit at once.  Smallest first: the
// short class-2/3 chains (high L1 hit rates, little L2 traffic) take the SMs at
// t = 0 beside class 0, and the class-1 chains start as those retire, late and
// with little competition.  Measured on config 3 (64 fronts): offsets 0,0,0,1
// (largest first, round 1) 3.98 ms; 1,2,0,0 3.47 ms; 1,1,0,0 / 2,3,1,0 / 2,4,0,0
// equal; the 512-front level is neutral (24.3 ms either way).  With everything
// launched at once the large classes ran their last, L2-heaviest steps all in
// phase; per-chain times under that load were 25 us per step against 15 us
// for the late class-1 chains of this order (HK_ACA_PROFILE).
// HK_ACA_PRIO="p0,p1,p2,p3" (offsets from the greatest priority) overrides.
static hk_status ensure_side_streams(hk_plan* p) {
  int least = 0, greatest = 0;
  cudaDeviceGetStreamPriorityRange(&least, &greatest);
  int off[4] = {1, 2, 0, 0};
  if (const char* e = getenv("HK_ACA_PRIO"))
    sscanf(e, "%d,%d,%d,%d", &off[0], &off[1], &off[2], &off[3]);
  for (int c = 0; c < 4; ++c) {
    int prio = greatest + off[c];
    if (prio > least) prio = least;
    if (!p->side[c]) CU(cudaStreamCreateWithPriority(&p->side[c], cudaStreamNonBlocking, prio));
    if (!p->side_ev[c]) CU(cudaEventCreateWithFlags(&p->side_ev[c], cudaEventDisableTiming));
    if (!p->cl_side[c]) CU(cudaStreamCreateWithPriority(&p->cl_side[c], cudaStreamNonBlocking, greatest));
    if (!p->cl_side_ev[c]) CU(cudaEventCreateWithFlags(&p->cl_side_ev[c], cudaEventDisableTiming));
  }
  return HK_OK;
}

static hk_status ensure_events(hk_plan* p) {
  for (auto& e : p->ev)
    if (!e) CU(cudaEventCreate(&e));
  return HK_OK;
}

static hk_status timed_begin(hk_plan* p, cudaStream_t st) {
  CHK(ensure_events(p));
  CU(cudaEventRecord(p->ev[0], st));
  return HK_OK;
}

static hk_status prepare_build(hk_plan* p, const double* A, int64_t ld, int64_t fstride,
                               int64_t max_rank, cudaStream_t st) {
  if (!A) return fail(HK_ERR_VALUE, "fronts pointer is null");
  if (ld < p->n) return fail(HK_ERR_DIMENSION, "leading dimension smaller than n");
  if (p->batch > 1 && fstride < ld * p->n) return fail(HK_ERR_DIMENSION, "front stride too small");
  if (hk_device_count() == 0) return fail(HK_ERR_CUDA, "no CUDA device visible");
  init_pool_once();
  p->A = A;
  p->lda = ld;
  p->fstride = fstride;
  p->built = false;
  p->factored = false;
  if (!p->progs.empty()) {
    CU(cudaStreamSynchronize(st));
    drop_progs(p, st);
  }
  set_caps(p, max_rank);
  const size_t nb = p->blocks.size();
  CU(p->UV.ensure((size_t)p->batch * p->uv_per_front * 8 + 8, st));
  CU(p->ranks_d.ensure((size_t)p->batch * nb * 4 + 4, st));
  CU(cudaMemsetAsync(p->ranks_d.p, 0, (size_t)p->batch * nb * 4 + 4, st));
  p->ranks.assign((size_t)p->batch * nb, 0);
  return HK_OK;
}

static hk_status fetch_ranks(hk_plan* p, cudaStream_t st) {
  if (!p->ranks.empty())
    CU(cudaMemcpyAsync(p->ranks.data(), p->ranks_d.p, p->ranks.size() * 4, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return HK_OK;
}

extern "C" hk_status hk_build_aca(hk_plan* p, const double* A, int64_t ld, int64_t fstride,
                                  double tol, double tol2, int64_t max_rank, int record_trace,
                                  void* stream) {
  if (!p) return fail(HK_ERR_VALUE, "null plan");
  if (!(tol > 0.0 && tol < 1.0)) return fail(HK_ERR_VALUE, "tol must lie strictly between 0 and 1");
  cudaStream_t st = (cudaStream_t)stream;
  HostClock hc("build_aca");
  CHK(prepare_build(p, A, ld, fstride, max_rank, st));
  CHK(timed_begin(p, st));
  const int64_t n = p->n;
  // transposed copy with the same ld/stride as the fronts: At[j*ld + i] = A[i*ld + j]
  const int64_t atstride = p->batch > 1 ? fstride : 0;
  // HK_ACA_AT=0: no transposed copy; the column gathers read the front with stride ld
  static int use_at = -1;
  if (use_at < 0) {
    const char* e = getenv("HK_ACA_AT");
    use_at = e ? atoi(e) : 1;
  }
  if (use_at) {
    CU(p->At.ensure((size_t)((p->batch - 1) * atstride + ld * n) * 8 + 8, st));
    CU(hk_launch_transpose(A, p->At.as<double>(), n, ld, p->batch, atstride, st));
  }
  const int64_t ldat = ld;
  p->have_trace = record_trace != 0;
  if (p->have_trace) CU(p->trace_d.ensure((size_t)p->batch * p->trace_per_front * 4 + 4, st));
  const size_t nb = p->blocks.size();
  size_t scr_per_front = 0;
  std::vector<size_t> scr_off(nb);
  for (size_t bi = 0; bi < nb; ++bi) {
    scr_off[bi] = scr_per_front;
    const BlockGeom& b = p->blocks[bi];
    const int P = hk_aca_cluster_size(b.m, b.n);
    scr_per_front += P > 1 ? hk_aca_scratch_doubles_cl(b.cap, P) : hk_aca_scratch_doubles(b.cap);
  }
  CU(p->aca_scr.ensure((size_t)p->batch * scr_per_front * 8 + 8, st));
  const char* prof = getenv("HK_ACA_PROFILE");
  // The task list depends only on the fronts pointer, the plan's buffers and
  // the caps: a batch rebuilt in the same device buffers (every step of a
  // level streamed through two buffers) reuses its device copy instead of
  // planning and staging it again (~0.25 ms of host time with the GPU idle).
  AcaPlanKey key{};
  key.ptr[0] = A; key.ptr[1] = p->At.p; key.ptr[2] = p->UV.p; key.ptr[3] = p->ranks_d.p;
  key.ptr[4] = p->have_trace ? p->trace_d.p : nullptr; key.ptr[5] = p->aca_scr.p;
  key.v[0] = ld; key.v[1] = fstride; key.v[2] = max_rank; key.v[3] = use_at;
  AcaPlanCache* hitc = nullptr;
  if (!prof)
    for (auto& c : p->aca_plans)
      if (c.key == key) hitc = &c;
  const AcaTask* tasks_dev = nullptr;
  std::vector<AcaTask> tasks;
  std::vector<int64_t> task_key;
  size_t ncl_tasks = 0;
  int cl_P[4] = {0, 0, 0, 0}, cl_begin[4] = {0, 0, 0, 0}, cl_cnt[4] = {0, 0, 0, 0};
  int cl_cap[4] = {0, 0, 0, 0}, cl_m[4] = {0, 0, 0, 0};
  int ngroups = 0;
  int cls_begin[5] = {0, 0, 0, 0, 0}, cls_cap[4] = {0, 0, 0, 0}, cls_m[4] = {0, 0, 0, 0};
  DevBuf clk;
  if (hitc) {
    tasks_dev = hitc->tasks.as<AcaTask>();
    ncl_tasks = hitc->ncl_tasks;
    ngroups = hitc->ngroups;
    memcpy(cl_P, hitc->cl_P, sizeof cl_P); memcpy(cl_begin, hitc->cl_begin, sizeof cl_begin);
    memcpy(cl_cnt, hitc->cl_cnt, sizeof cl_cnt); memcpy(cl_cap, hitc->cl_cap, sizeof cl_cap);
    memcpy(cl_m, hitc->cl_m, sizeof cl_m);
    memcpy(cls_begin, hitc->cls_begin, sizeof cls_begin); memcpy(cls_cap, hitc->cls_cap, sizeof cls_cap);
    memcpy(cls_m, hitc->cls_m, sizeof cls_m);
  } else {
  tasks.reserve((size_t)p->batch * p->blocks.size());
  int max_cap = 0, max_m = 0, max_mn = 0;
  for (int64_t f = 0; f < p->batch; ++f) {
    for (int bi : p->block_order) {
      const BlockGeom& b = p->blocks[bi];
      AcaTask t{};
      t.A = A + f * fstride + b.row0 * ld + b.col0;
      t.At = use_at ? p->At.as<double>() + f * atstride + b.col0 * ldat + b.row0 : nullptr;
      t.U = p->UV.as<double>() + f * p->uv_per_front + b.u_off;
      t.V = p->UV.as<double>() + f * p->uv_per_front + b.v_off;
      t.rank = p->ranks_d.as<int32_t>() + f * nb + bi;
      t.trace = p->have_trace ? p->trace_d.as<int32_t>() + f * p->trace_per_front + b.t_off : nullptr;
      t.scratch = p->aca_scr.as<double>() + f * scr_per_front + scr_off[bi];
      t.lda = ld;
      t.m = b.m;
      t.n = b.n;
      t.cap = b.cap;
      t.ldu = b.ldu_log;
      t.ldv = b.ldv_log;
      if (b.ldu_log > 13 || b.ldv_log > 13) return fail(HK_ERR_VALUE, "block too large for the ACA kernel (max 8192 rows)");
      max_cap = std::max(max_cap, b.cap);
      max_m = std::max(max_m, b.m);
      max_mn = std::max(max_mn, b.m + b.n);
      tasks.push_back(t);
      task_key.push_back(f * (int64_t)nb + bi);
    }
  }
  // global largest-first order across fronts: the long root chains start first
  std::vector<size_t> order(tasks.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = i;
  // group key: cluster tasks first (largest cluster first), then the
  // single-CTA size classes
  auto group_of = [](const AcaTask& a) {
    const int P = hk_aca_cluster_size(a.m, a.n);
    return P > 1 ? -P : hk_aca_class(a.m, a.n);
  };
  std::stable_sort(order.begin(), order.end(), [&](size_t x, size_t y) {
    const AcaTask &a = tasks[x], &b = tasks[y];
    const int ca = group_of(a), cb = group_of(b);
    if (ca != cb) return ca < cb;
    return (int64_t)(a.m + a.n) * a.cap > (int64_t)(b.m + b.n) * b.cap;
  });
  std::vector<AcaTask> sorted(tasks.size());
  std::vector<size_t> tidx(tasks.size());   // sorted position -> (f * nb + block) key
  std::vector<int64_t> skey(tasks.size());
  for (size_t i = 0; i < order.size(); ++i) { sorted[i] = tasks[order[i]]; skey[i] = task_key[order[i]]; }
  tasks.swap(sorted);
  task_key.swap(skey);
  (void)tidx;
  if (prof) {
    CU(clk.ensure(tasks.size() * 24 + 8, st));
    for (size_t i = 0; i < tasks.size(); ++i) tasks[i].clock = clk.as<int64_t>() + 3 * i;
  }
  p->stage.reset();
  tasks_dev = p->stage.push(tasks, st);
  if (!tasks_dev) return fail(HK_ERR_CUDA, "pinned staging allocation failed");
  CU(p->stage.commit(st));
  // cluster groups (P = 16, 8, 4, 2) then the four single-CTA classes
  while (ncl_tasks < tasks.size()) {
    const AcaTask& t = tasks[ncl_tasks];
    const int P = hk_aca_cluster_size(t.m, t.n);
    if (P == 1) break;
    if (ngroups == 0 || cl_P[ngroups - 1] != P) {
      if (ngroups == 4) return fail(HK_ERR_VALUE, "internal: more than four ACA cluster groups");
      cl_P[ngroups] = P;
      cl_begin[ngroups] = (int)ncl_tasks;
      ++ngroups;
    }
    const int g = ngroups - 1;
    cl_cnt[g]++;
    cl_cap[g] = std::max(cl_cap[g], t.cap);
    cl_m[g] = std::max(cl_m[g], t.m);
    if ((size_t)(4 * t.cap + 32) * 8 + t.m + 1024 > 220 * 1024)
      return fail(HK_ERR_VALUE, "block too large for the cluster ACA kernel");
    ++ncl_tasks;
  }
  for (size_t i = ncl_tasks; i < tasks.size(); ++i) {
    const AcaTask& t = tasks[i];
    const int c = hk_aca_class(t.m, t.n);
    cls_begin[c + 1]++;
    cls_cap[c] = std::max(cls_cap[c], t.cap);
    cls_m[c] = std::max(cls_m[c], t.m);
    if ((size_t)(2 * t.cap + 32) * 8 + t.m + 1024 > 220 * 1024)
      return fail(HK_ERR_VALUE, "block too large for the single-CTA ACA kernel");
  }
  for (int c = 0; c < 4; ++c) cls_begin[c + 1] += cls_begin[c];
  if (!prof) {   // keep a device copy of this task list (at most 4 cached)
    if (p->aca_plans.size() >= 4) {
      p->aca_plans.front().tasks.release();
      p->aca_plans.erase(p->aca_plans.begin());
    }
    p->aca_plans.emplace_back();
    AcaPlanCache& c = p->aca_plans.back();
    c.key = key;
    CU(c.tasks.ensure(tasks.size() * sizeof(AcaTask) + 16, st));
    CU(cudaMemcpyAsync(c.tasks.p, tasks_dev, tasks.size() * sizeof(AcaTask), cudaMemcpyDeviceToDevice, st));
    c.ncl_tasks = ncl_tasks;
    c.ngroups = ngroups;
    memcpy(c.cl_P, cl_P, sizeof cl_P); memcpy(c.cl_begin, cl_begin, sizeof cl_begin);
    memcpy(c.cl_cnt, cl_cnt, sizeof cl_cnt); memcpy(c.cl_cap, cl_cap, sizeof cl_cap);
    memcpy(c.cl_m, cl_m, sizeof cl_m);
    memcpy(c.cls_begin, cls_begin, sizeof cls_begin); memcpy(c.cls_cap, cls_cap, sizeof cls_cap);
    memcpy(c.cls_m, cls_m, sizeof cls_m);
  }
  }
  CHK(ensure_side_streams(p));
  if (ngroups > 0 && !p->started_h) {
    if (cudaHostAlloc((void**)&p->started_h, 64, cudaHostAllocMapped) == cudaSuccess) {
      if (cudaHostGetDevicePointer((void**)&p->started_d, p->started_h, 0) != cudaSuccess) {
        cudaFreeHost(p->started_h);
        p->started_h = nullptr;
        p->started_d = nullptr;
      }
    } else {
      p->started_h = nullptr;
    }
    (void)cudaGetLastError();
  }
  CU(p->aca_cnt.ensure(64, st));
  CU(cudaMemsetAsync(p->aca_cnt.p, 0, 64, st));
  CU(cudaEventRecord(p->ev[3], st));
  cudaStream_t ss[4];
  for (int c = 0; c < 4; ++c) {   // fork
    ss[c] = p->side[c];
    CU(cudaStreamWaitEvent(ss[c], p->ev[3], 0));
  }
  for (int g = 0; g < ngroups; ++g) {   // the long chains launch first
    CU(cudaStreamWaitEvent(p->cl_side[g], p->ev[3], 0));
    int* started_d = nullptr;
    if (g == 0 && p->started_h) {
      *(volatile int*)p->started_h = 0;
      started_d = p->started_d;
    }
    int max_active = 0;
    CU(hk_launch_aca_cluster(tasks_dev + cl_begin[g], cl_cnt[g], cl_P[g], cl_cap[g], cl_m[g],
                             tol2, p->cl_side[g], started_d, &max_active));
    if (g == 0 && started_d && (ngroups > 1 || cls_begin[4] > 0)) {
      // The largest clusters (config 4: two 16-CTA clusters on the root
      // blocks, the longest chains) need 16 free SMs of one GPC at once; when
      // the other groups and classes launched beside them got the SMs first,
      // the root chains started only after ~5.7 ms.  Hold the other launches
      // until those clusters are resident (bounded wait).
      const int want = std::min(cl_cnt[0], std::max(max_active, 1));
      const auto t0 = std::chrono::steady_clock::now();
      while (*(volatile int*)p->started_h < want &&
             std::chrono::steady_clock::now() - t0 < std::chrono::milliseconds(20)) {
      }
    }
  }
  CU(hk_launch_aca_classes(tasks_dev + ncl_tasks, cls_begin, cls_cap, cls_m, tol2,
                           p->aca_cnt.as<int>(), ss));
  for (int c = 0; c < 4; ++c) {   // join
    CU(cudaEventRecord(p->side_ev[c], ss[c]));
    CU(cudaStreamWaitEvent(st, p->side_ev[c], 0));
  }
  for (int g = 0; g < ngroups; ++g) {
    CU(cudaEventRecord(p->cl_side_ev[g], p->cl_side[g]));
    CU(cudaStreamWaitEvent(st, p->cl_side_ev[g], 0));
  }
  CU(cudaEventRecord(p->ev[1], st));
  hc.mark("plan+launch");
  CHK(fetch_ranks(p, st));
  hc.mark("wait");
  if (prof) {
    std::vector<int64_t> h(tasks.size() * 3);
    CU(cudaMemcpy(h.data(), clk.p, h.size() * 8, cudaMemcpyDeviceToHost));
    FILE* fo = fopen(prof, "w");
    if (fo) {
      for (size_t i = 0; i < tasks.size(); ++i)
        fprintf(fo, "%d %d %d %d %lld %lld %lld\n", tasks[i].m, tasks[i].n,
                p->ranks[task_key[i]], (int)(task_key[i] % nb), (long long)h[3 * i],
                (long long)h[3 * i + 1], (long long)h[3 * i + 2]);
      fclose(fo);
    }
    clk.release();
  }
  float ms = 0, ms_aca = 0;
  CU(cudaEventElapsedTime(&ms, p->ev[0], p->ev[1]));
  CU(cudaEventElapsedTime(&ms_aca, p->ev[3], p->ev[1]));
  p->t_lowrank = ms * 1e-3;
  p->t_aca = ms_aca * 1e-3;
  p->scheme = HK_SCHEME_ACA;
  p->built = true;
  return HK_OK;
}

// numpy.linspace(0, m-1, num=min(m, 8)).astype(intp), then unique (lowrank.py:325)
static std::vector<int64_t> probe_rows(int64_t m) {
  std::vector<int64_t> out;
  int64_t num = std::min<int64_t>(m, 8);
  if (num <= 0) return out;
  if (num == 1) {
    out.push_back(0);
    return out;
  }
  double stop = (double)(m - 1);
  double step = stop / (double)(num - 1);
  for (int64_t i = 0; i < num; ++i) {
    double y = (double)i * step;
    if (i == num - 1) y = stop;
    out.push_back((int64_t)y);
  }
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
  return out;
}

extern "C" hk_status hk_build_bdlr(hk_plan* p, const double* A, int64_t ld, int64_t fstride,
                                   double tol, int32_t depth, int64_t max_rank,
                                   const int64_t* indptr, const int64_t* indices, void* stream) {
  NvtxRange nvtx_range("hk_build_bdlr");
  if (!p) return fail(HK_ERR_VALUE, "null plan");
  if (!(tol > 0.0 && tol < 1.0)) return fail(HK_ERR_VALUE, "tol must lie strictly between 0 and 1");
  if (depth < 0) return fail(HK_ERR_VALUE, "depth must be >= 0");
  if (!indptr || !indices) return fail(HK_ERR_VALUE, "bdlr compression requires a graph view on the block");
  cudaStream_t st = (cudaStream_t)stream;
  CHK(prepare_build(p, A, ld, fstride, max_rank, st));
  CHK(timed_begin(p, st));
  const size_t nb = p->blocks.size();
  // the selections depend only on (graph, tree, depth): reuse them when the
  // same graph comes back (FNV-1a over the CSR arrays; every batch of a
  // multifrontal level shares one separator graph)
  uint64_t key = 1469598103934665603ull;
  auto mix = [&](const void* data, size_t bytes) {
    const unsigned char* c = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < bytes; ++i) key = (key ^ c[i]) * 1099511628211ull;
  };
  const int64_t nnz = indptr[p->n];
  mix(&p->n, sizeof(p->n));
  mix(&depth, sizeof(depth));
  mix(indptr, (size_t)(p->n + 1) * 8);
  mix(indices, (size_t)nnz * 8);
  const bool hit = p->sel_valid && p->sel_key == key;
  std::vector<int64_t> sel_all, probes;
  std::vector<int64_t>& probe_off = p->probe_off;
  std::vector<int64_t>& probe_cnt = p->probe_cnt;
  int& max_k = p->sel_max_k;
  int& max_kc = p->sel_max_kc;
  if (!hit) {
  p->sel_valid = false;
  p->rsel.assign(nb, {});
  p->csel.assign(nb, {});
  p->sel_off_r.assign(nb, 0);
  p->sel_off_c.assign(nb, 0);
  probe_off.assign(nb, 0);
  probe_cnt.assign(nb, 0);
  max_k = 0;
  max_kc = 0;
  // selections of every block: on the GPU (select.cu; default) or by the
  // host BFS (graph.cpp; HK_BDLR_SELECT=host) -- identical results
  std::vector<std::vector<int64_t>> all_rs(nb), all_cs(nb);
  static int gpu_sel = -1;
  if (gpu_sel < 0) {
    const char* e = getenv("HK_BDLR_SELECT");
    gpu_sel = (e && std::string(e) == "host") ? 0 : 1;
  }
  if (gpu_sel) {
    CU(p->gidx_d.ensure((size_t)(p->n + 1 + nnz) * 8 + 8, st));
    int64_t* gip = p->gidx_d.as<int64_t>();
    CU(cudaMemcpyAsync(gip, indptr, (size_t)(p->n + 1) * 8, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(gip + p->n + 1, indices, (size_t)nnz * 8, cudaMemcpyHostToDevice, st));
    std::vector<SelTask> sts;
    std::vector<int64_t> off;
    int64_t cap = 0;
    int max_own = 1;
    for (size_t bi = 0; bi < nb; ++bi) {
      const BlockGeom& b = p->blocks[bi];
      for (int side = 0; side < 2; ++side) {
        SelTask t{};
        t.own0 = side == 0 ? b.row0 : b.col0;
        t.n_own = side == 0 ? b.m : b.n;
        t.oth0 = side == 0 ? b.col0 : b.row0;
        t.n_oth = side == 0 ? b.n : b.m;
        off.push_back(cap);
        cap += t.n_own;
        max_own = std::max(max_own, t.n_own);
        sts.push_back(t);
      }
    }
    CU(p->selout_d.ensure((size_t)cap * 8 + (size_t)sts.size() * 4 + 64, st));
    int64_t* outd = p->selout_d.as<int64_t>();
    int32_t* cntd = reinterpret_cast<int32_t*>(outd + cap);
    for (size_t i = 0; i < sts.size(); ++i) {
      sts[i].out = outd + off[i];
      sts[i].count = cntd + i;
    }
    CU(upload(p->seltask_d, sts, st));
    CU(hk_launch_select(p->seltask_d.as<SelTask>(), (int)sts.size(), max_own, gip, gip + p->n + 1,
                        depth, st));
    std::vector<int64_t> outh((size_t)cap);
    std::vector<int32_t> cnth(sts.size());
    CU(cudaMemcpyAsync(outh.data(), outd, (size_t)cap * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(cnth.data(), cntd, cnth.size() * 4, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    for (size_t bi = 0; bi < nb; ++bi) {
      all_rs[bi].assign(outh.begin() + off[2 * bi], outh.begin() + off[2 * bi] + cnth[2 * bi]);
      all_cs[bi].assign(outh.begin() + off[2 * bi + 1],
                        outh.begin() + off[2 * bi + 1] + cnth[2 * bi + 1]);
    }
  } else {
    for (size_t bi = 0; bi < nb; ++bi) {
      const BlockGeom& b = p->blocks[bi];
      std::vector<int64_t> rv(b.m), cv(b.n);
      for (int i = 0; i < b.m; ++i) rv[i] = b.row0 + i;
      for (int j = 0; j < b.n; ++j) cv[j] = b.col0 + j;
      hk::select_by_depth(p->n, indptr, indices, rv.data(), b.m, cv.data(), b.n, depth,
                          all_rs[bi], all_cs[bi]);
    }
  }
  for (size_t bi = 0; bi < nb; ++bi) {
    const BlockGeom& b = p->blocks[bi];
    const std::vector<int64_t>& rs = all_rs[bi];
    const std::vector<int64_t>& cs = all_cs[bi];
    // EmptySelectionError -> rank-0 factor (lowrank.py:345-348)
    if (rs.empty() || cs.empty()) continue;
    p->rsel[bi] = rs;
    p->csel[bi] = cs;
    p->sel_off_r[bi] = (int64_t)sel_all.size();
    sel_all.insert(sel_all.end(), rs.begin(), rs.end());
    p->sel_off_c[bi] = (int64_t)sel_all.size();
    sel_all.insert(sel_all.end(), cs.begin(), cs.end());
    auto pr = probe_rows(b.m);
    probe_off[bi] = (int64_t)probes.size();
    probe_cnt[bi] = (int64_t)pr.size();
    probes.insert(probes.end(), pr.begin(), pr.end());
    max_k = std::max(max_k, (int)rs.size());
    max_kc = std::max(max_kc, (int)cs.size());
  }
  CU(upload(p->sel_d, sel_all, st));
  CU(upload(p->probe_d, probes, st));
  p->sel_key = key;
  p->sel_valid = true;
  }
  // scratch per (front, block) with a selection
  std::vector<SkelTask> tasks;
  int64_t work_total = 0, perm_total = 0;
  p->perm_off.assign((size_t)p->batch * nb, -1);
  std::vector<int64_t> work_off((size_t)p->batch * nb, 0);
  for (int64_t f = 0; f < p->batch; ++f)
    for (size_t bi = 0; bi < nb; ++bi) {
      if (p->rsel[bi].empty()) continue;
      work_off[f * nb + bi] = work_total;
      work_total += (int64_t)p->rsel[bi].size() * p->csel[bi].size();
      p->perm_off[f * nb + bi] = perm_total;
      perm_total += (int64_t)p->rsel[bi].size() + p->csel[bi].size();
    }
  CU(p->work_d.ensure((size_t)work_total * 8 + 8, st));
  CU(p->perm_d.ensure((size_t)perm_total * 8 + 8, st));
  CU(p->skel_status_d.ensure((size_t)p->batch * nb * 4 + 4, st));
  CU(cudaMemsetAsync(p->skel_status_d.p, 0, (size_t)p->batch * nb * 4 + 4, st));
  for (int64_t f = 0; f < p->batch; ++f)
    for (int bi : p->block_order) {
      if (p->rsel[bi].empty()) continue;
      const BlockGeom& b = p->blocks[bi];
      SkelTask t{};
      t.A = A + f * fstride + b.row0 * ld + b.col0;
      t.lda = ld;
      t.rsel = p->sel_d.as<int64_t>() + p->sel_off_r[bi];
      t.csel = p->sel_d.as<int64_t>() + p->sel_off_c[bi];
      t.work = p->work_d.as<double>() + work_off[f * nb + bi];
      t.rperm = p->perm_d.as<int64_t>() + p->perm_off[f * nb + bi];
      t.cperm = t.rperm + p->rsel[bi].size();
      t.U = p->UV.as<double>() + f * p->uv_per_front + b.u_off;
      t.V = p->UV.as<double>() + f * p->uv_per_front + b.v_off;
      t.rank = p->ranks_d.as<int32_t>() + f * nb + bi;
      t.status = p->skel_status_d.as<int32_t>() + f * nb + bi;
      t.probe = p->probe_d.as<int64_t>() + probe_off[bi];
      t.nprobe = (int32_t)probe_cnt[bi];
      t.m = b.m;
      t.n = b.n;
      t.k = (int)p->rsel[bi].size();
      t.kc = (int)p->csel[bi].size();
      t.cap = b.cap;
      t.ldu = b.ldu;
      t.ldv = b.ldv;
      t.tol = tol;
      tasks.push_back(t);
    }
  int max_bm = 0, max_bn = 0;
  for (const SkelTask& t : tasks) {
    max_bm = std::max(max_bm, t.m);
    max_bn = std::max(max_bn, t.n);
  }
  CU(upload(p->tasks_d, tasks, st));
  CU(hk_launch_skeleton(p->tasks_d.as<SkelTask>(), (int)tasks.size(), max_k, max_kc, max_bm,
                        max_bn, st));
  CU(cudaEventRecord(p->ev[1], st));
  CHK(fetch_ranks(p, st));
  std::vector<int32_t> status((size_t)p->batch * nb, 0);
  CU(cudaMemcpy(status.data(), p->skel_status_d.p, status.size() * 4, cudaMemcpyDeviceToHost));
  for (int64_t f = 0; f < p->batch; ++f)
    for (size_t bi = 0; bi < nb; ++bi)   // preorder, upper before lower
      if (status[f * nb + bi] == HK_ERR_DEGENERATE) {
        char msg[160];
        snprintf(msg, sizeof msg,
                 "skeleton rank 0 but sampled block magnitude exceeds tolerance "
                 "(front %lld, block %zu); selection depth is too small", (long long)f, bi);
        return fail(HK_ERR_DEGENERATE, msg);
      }
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, p->ev[0], p->ev[1]));
  p->t_lowrank = ms * 1e-3;
  p->scheme = HK_SCHEME_BDLR;
  p->built = true;
  return HK_OK;
}

extern "C" hk_status hk_build_external_begin(hk_plan* p, const double* A, int64_t ld,
                                             int64_t fstride, void* stream) {
  if (!p) return fail(HK_ERR_VALUE, "null plan");
  cudaStream_t st = (cudaStream_t)stream;
  CHK(prepare_build(p, A, ld, fstride, 0, st));
  p->t_lowrank = 0;
  p->scheme = HK_SCHEME_SVD;
  p->built = true;
  return HK_OK;
}

extern "C" hk_status hk_set_block_factor(hk_plan* p, int64_t f, int64_t bi, int64_t rank,
                                         const double* U, int64_t ldu, const double* V,
                                         int64_t ldv, void* stream) {
  if (!p || !p->built) return fail(HK_ERR_STATE, "build not started");
  if (f < 0 || f >= p->batch || bi < 0 || bi >= (int64_t)p->blocks.size())
    return fail(HK_ERR_VALUE, "front/block out of range");
  const BlockGeom& b = p->blocks[bi];
  if (rank < 0 || rank > b.cap) return fail(HK_ERR_VALUE, "rank exceeds block cap");
  cudaStream_t st = (cudaStream_t)stream;
  double* Ud = p->UV.as<double>() + f * p->uv_per_front + b.u_off;
  double* Vd = p->UV.as<double>() + f * p->uv_per_front + b.v_off;
  if (rank > 0) {   // column-major input -> row-major pool
    std::vector<CopyTask> ct(2);
    ct[0] = CopyTask{U, Ud, 1, ldu, 1, b.ldu, b.m, (int32_t)rank};
    ct[1] = CopyTask{V, Vd, 1, ldv, 1, b.ldv, b.n, (int32_t)rank};
    DevBuf tb;
    CU(upload(tb, ct, st));
    CU(hk_launch_copy(tb.as<CopyTask>(), 2, st));
    CU(cudaStreamSynchronize(st));
    tb.release();
  }
  const size_t nb = p->blocks.size();
  p->ranks[f * nb + bi] = (int32_t)rank;
  int32_t r32 = (int32_t)rank;
  CU(cudaMemcpyAsync(p->ranks_d.as<int32_t>() + f * nb + bi, &r32, 4, cudaMemcpyHostToDevice, st));
  CU(cudaStreamSynchronize(st));
  return HK_OK;
}

extern "C" hk_status hk_get_ranks(hk_plan* p, int32_t* out) {
  if (!p || !p->built) return fail(HK_ERR_STATE, "plan not built");
  std::memcpy(out, p->ranks.data(), p->ranks.size() * 4);
  return HK_OK;
}

extern "C" hk_status hk_get_aca_trace(hk_plan* p, int64_t f, int64_t bi, int32_t* rows,
                                      int64_t* nrows, int32_t* cols, int64_t* ncols) {
  if (!p || !p->built || !p->have_trace) return fail(HK_ERR_STATE, "no ACA trace recorded");
  const BlockGeom& b = p->blocks[bi];
  const int64_t len = 2 + (b.m + b.cap + 1) + (b.cap + 1);
  std::vector<int32_t> h(len);
  CU(cudaMemcpy(h.data(), p->trace_d.as<int32_t>() + f * p->trace_per_front + b.t_off, len * 4,
                cudaMemcpyDeviceToHost));
  *nrows = h[0];
  *ncols = h[1];
  if (rows) std::memcpy(rows, h.data() + 2, (size_t)h[0] * 4);
  if (cols) std::memcpy(cols, h.data() + 2 + (b.m + b.cap + 1), (size_t)h[1] * 4);
  return HK_OK;
}

extern "C" hk_status hk_get_skeleton(hk_plan* p, int64_t f, int64_t bi, int64_t* rank,
                                     int64_t* rows, int64_t* cols, int64_t cap) {
  if (!p || !p->built || p->scheme != HK_SCHEME_BDLR) return fail(HK_ERR_STATE, "no BDLR build");
  const size_t nb = p->blocks.size();
  const int64_t r = p->ranks[f * nb + bi];
  *rank = r;
  if (r == 0) return HK_OK;
  if (r > cap) return fail(HK_ERR_VALUE, "output too small");
  const size_t k = p->rsel[bi].size(), kc = p->csel[bi].size();
  std::vector<int64_t> perm(k + kc);
  CU(cudaMemcpy(perm.data(), p->perm_d.as<int64_t>() + p->perm_off[f * nb + bi], (k + kc) * 8,
                cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < r; ++i) {
    rows[i] = p->rsel[bi][perm[i]];
    cols[i] = p->csel[bi][perm[k + i]];
  }
  return HK_OK;
}

extern "C" hk_status hk_get_block_factor(hk_plan* p, int64_t f, int64_t bi, double* U, double* V) {
  if (!p || !p->built) return fail(HK_ERR_STATE, "plan not built");
  const BlockGeom& b = p->blocks[bi];
  const int64_t r = p->ranks[f * p->blocks.size() + bi];
  const double* base = p->UV.as<double>() + f * p->uv_per_front;
  if (r > 0) {   // padded column-major pool -> dense column-major host (m x r, n x r)
    CU(cudaMemcpy2D(U, (size_t)b.m * 8, base + b.u_off, (size_t)b.ldu * 8, (size_t)b.m * 8, r,
                    cudaMemcpyDeviceToHost));
    CU(cudaMemcpy2D(V, (size_t)b.n * 8, base + b.v_off, (size_t)b.ldv * 8, (size_t)b.n * 8, r,
                    cudaMemcpyDeviceToHost));
  }
  return HK_OK;
}

// ------------------------------------------------------------------ factor
struct TileList {
  std::vector<GemmTask> tasks;
  std::vector<int32_t> map;
  void add(const GemmTask& t) {
    if (t.m <= 0 || t.n <= 0) return;
    if (t.k <= 0 && t.beta == 1.0) return;
    const int id = (int)tasks.size();
    tasks.push_back(t);
    const int tm = (t.m + 63) / 64, tn = (t.n + 63) / 64;
    for (int a = 0; a < tm; ++a)
      for (int b = 0; b < tn; ++b) {
        map.push_back(id);
        map.push_back(a);
        map.push_back(b);
      }
  }
  int ntiles() const { return (int)(map.size() / 3); }
};

// A factorization phase is planned on the host into a list of ops whose task
// arrays live in the pinned staging; flush() commits and launches them.
struct Op {
  enum Kind { COPY, GEMM, GJ, GJ_LEAF_TMA, EVENT } kind;
  const void* a = nullptr;   // device task array
  const int32_t* map = nullptr;
  int n = 0, maxN = 0;       // tasks / tiles, largest GJ order
  int ev = 0;
  double flops = 0;          // GEMM: sum of 2 m n k over the tasks (profile labels)
  int kmin = 0, kmax = 0;    // GEMM: range of the tasks' k (profile labels)
};

static hk_status stage_tiles(hk_plan* p, std::vector<Op>& ops, const TileList& tl, cudaStream_t st) {
  if (tl.ntiles() == 0) return HK_OK;
  Op o{Op::GEMM};
  o.a = p->stage.push(tl.tasks, st);
  o.map = p->stage.push(tl.map, st);
  if (!o.a || !o.map) return fail(HK_ERR_CUDA, "pinned staging allocation failed");
  o.n = tl.ntiles();
  if (host_profile()) {
    o.kmin = 1 << 30;
    for (const GemmTask& t : tl.tasks) {
      o.flops += 2.0 * t.m * t.n * t.k;
      o.kmin = std::min(o.kmin, t.k);
      o.kmax = std::max(o.kmax, t.k);
    }
  }
  ops.push_back(o);
  return HK_OK;
}

static GemmTask gemm(const double* A, int64_t lda, int transA, const double* B, int64_t ldb,
                     double* C, int64_t ldc, int m, int n, int k, double alpha, double beta,
                     double diag = 0.0) {
  GemmTask t{};
  t.diag = diag;
  t.A = A; t.lda = lda; t.transA = transA;
  t.B = B; t.ldb = ldb;
  t.C = C; t.ldc = ldc;
  t.m = m; t.n = n; t.k = k;
  t.alpha = alpha; t.beta = beta;
  t.vec = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) % 16 == 0) &&
          lda % 2 == 0 && ldb % 2 == 0;
  return t;
}

// Batched Gauss-Jordan inversions: SMEM/register-resident tasks and large
// tasks (global scratch at p->gjs_d, shared by every stage since the stages
// run in stream order) in separate launches.
static hk_status stage_gj(hk_plan* p, std::vector<Op>& ops, std::vector<GjTask>& tasks,
                          cudaStream_t st) {
  if (tasks.empty()) return HK_OK;
  std::vector<GjTask> small, large;
  size_t scratch = 0;
  int ms = 0, ml = 0;
  for (auto& t : tasks) {
    size_t b = hk_gj_scratch_bytes(t.N);
    if (b == 0) { small.push_back(t); ms = std::max(ms, t.N); }
    else {
      t.scratch = (double*)(p->gjs_d.as<char>() + scratch);
      scratch += (b + 255) / 256 * 256;
      large.push_back(t);
      ml = std::max(ml, t.N);
    }
  }
  if (scratch > p->gjs_d.bytes) return fail(HK_ERR_STATE, "internal: GJ scratch undersized");
  for (auto* v : {&small, &large}) {
    if (v->empty()) continue;
    Op o{Op::GJ};
    o.a = p->stage.push(*v, st);
    if (!o.a) return fail(HK_ERR_CUDA, "pinned staging allocation failed");
    o.n = (int)v->size();
    o.maxN = v == &small ? ms : ml;
    ops.push_back(o);
  }
  return HK_OK;
}

// Leaf Gauss-Jordan through the TMA (HK_GJ_LEAF_TMA=0 turns it off): every leaf
// is a row-major block of <= 64 of the fronts, and a tensor map of the fronts
// can be encoded (16-byte aligned base and strides).  The map is cached per
// (fronts pointer, lda, fstride, batch).
static bool leaf_tma_ok(hk_plan* p, const std::vector<GjTask>& gts) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("HK_GJ_LEAF_TMA");
    on = e ? atoi(e) : 1;
  }
  if (!on || gts.empty()) return false;
  // the box origin's inner coordinate must sit on a 16-byte boundary (the TMA
  // raises an illegal instruction otherwise): every leaf offset even
  for (const GjTask& t : gts)
    if (t.N > 64 || t.mode != 0 || t.src_ld != p->lda || ((t.src - p->A) & 1)) return false;
  const int64_t key[3] = {p->lda, p->fstride, p->batch};
  if (!(p->leafmap_ok && p->leafmap_base == p->A && key[0] == p->leafmap_key[0] &&
        key[1] == p->leafmap_key[1] && key[2] == p->leafmap_key[2])) {
    p->leafmap_ok = hk_gj_leaf_map(p->leafmap, p->A, p->n, p->lda, p->fstride, p->batch) == 0;
    p->leafmap_base = p->A;
    for (int i = 0; i < 3; ++i) p->leafmap_key[i] = key[i];
  }
  return p->leafmap_ok;
}

// HK_HOST_PROFILE: an event after every launched op gives in-situ per-op GPU
// times (kernel + any idle gap before it) for the factorization.
struct OpProfile {
  std::vector<cudaEvent_t> ev;
  std::vector<std::string> label;
  size_t used = 0;
  void reset() { used = 0; label.clear(); }
  void mark(const std::string& l, cudaStream_t st) {
    if (used == ev.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev.push_back(e);
    }
    cudaEventRecord(ev[used++], st);
    label.push_back(l);
  }
  void print(const char* what) {
    for (size_t i = 1; i < used; ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
      fprintf(stderr, "[hk gpu] %s %-28s %8.1f us\n", what, label[i].c_str(), ms * 1e3);
    }
  }
};
static OpProfile g_opprof;

// commit the staged task arrays and launch the ops planned so far
static hk_status launch_ops(hk_plan* p, std::vector<Op>& ops, cudaStream_t st) {
  const bool prof = host_profile();
  for (const Op& o : ops) {
    char lbl[64] = "";
    switch (o.kind) {
      case Op::COPY: CU(hk_launch_copy((const CopyTask*)o.a, o.n, st)); snprintf(lbl, 64, "copy x%d", o.n); break;
      case Op::GEMM: CU(hk_launch_gemm((const GemmTask*)o.a, o.map, o.n, st)); snprintf(lbl, 64, "gemm %d tiles %.0f MF k %d-%d", o.n, o.flops * 1e-6, o.kmin, o.kmax); break;
      case Op::GJ: CU(hk_launch_gj((const GjTask*)o.a, o.n, o.maxN, st)); snprintf(lbl, 64, "gj x%d N<=%d", o.n, o.maxN); break;
      case Op::GJ_LEAF_TMA:
        CU(hk_launch_gj_leaf_tma((const GjTask*)o.a, o.n, p->leafmap, p->A, p->lda, p->fstride, st));
        snprintf(lbl, 64, "gj leaves (TMA) x%d N<=%d", o.n, o.maxN);
        break;
      case Op::EVENT: CU(cudaEventRecord(p->ev[o.ev], st)); break;
    }
    if (prof && lbl[0]) g_opprof.mark(lbl, st);
  }
  ops.clear();
  return HK_OK;
}

static hk_status flush(hk_plan* p, std::vector<Op>& ops, cudaStream_t st) {
  CU(p->stage.commit(st));
  return launch_ops(p, ops, st);
}

static hk_status lu_on_demand(const LuTask& proto, int N, double* lu_host, int32_t* piv_host,
                              int* singular, double* inv_host = nullptr);
struct SolveProg;
static hk_status build_solve_prog(hk_plan* p, int front, int s, SolveProg*& out, cudaStream_t st);
static hk_status ensure_solve_scratch(hk_plan* p, int s, cudaStream_t st);

extern "C" hk_status hk_factor_ext(hk_plan* p, const double* Zext, int64_t ldz, int64_t wext,
                                   void* stream) {
  if (!p || !p->built) return fail(HK_ERR_STATE, "factor requires a build");
  if (wext < 0) return fail(HK_ERR_VALUE, "negative extension width");
  if (wext > 0 && (p->batch != 1 || !Zext || ldz < p->n))
    return fail(HK_ERR_VALUE, "an external extension needs batch 1, a device pointer and ldz >= n");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = p->n;
  const size_t nb = p->blocks.size();
  const int nn = (int)p->nodes.size();
  if (!p->progs.empty()) {
    CU(cudaStreamSynchronize(st));
    drop_progs(p, st);
  }
  p->factored = false;
  HostClock hc("factor");
  CHK(ensure_events(p));
  CU(cudaEventRecord(p->ev[0], st));
  if (host_profile()) {
    g_opprof.reset();
    g_opprof.mark("start", st);
  }
  // ---- widths and storage layout
  p->W.assign(p->batch, 0);
  p->y_off.assign(p->batch, 0);
  p->rec.assign((size_t)p->batch * nn, NodeRec());
  int64_t ytot = 0, ftot = 0, itot = 0, gtot = 0;
  for (int64_t f = 0; f < p->batch; ++f) {
    std::vector<int64_t> w(nn, 0);
    w[0] = wext;                    // the root's extension (subtree sharding, §6)
    int64_t W = 0;
    for (int s = 0; s < nn; ++s) {  // preorder: parents before children
      const Node& nd = p->nodes[s];
      NodeRec& r = p->rec[f * nn + s];
      r.w = w[s];
      if (nd.left < 0) {
        W = std::max(W, w[s]);
        const int64_t b = nd.hi - nd.lo;
        r.inv = ftot; ftot += b * b;
        r.status = itot; itot += 1;
        continue;
      }
      const int k = p->iidx[s];
      const int ru = p->ranks[f * nb + 2 * k], rl = p->ranks[f * nb + 2 * k + 1];
      w[nd.left] = w[s] + ru;
      w[nd.right] = w[s] + rl;
      r.ru = ru; r.rl = rl; r.R = ru + rl;
      r.hcols = w[s] + std::max(ru, rl);
      const int64_t R = r.R;
      const int64_t sm = std::min(ru, rl);
      r.h = ftot; ftot += R * r.hcols;
      r.q = ftot; ftot += R * w[s];
      r.inv = ftot; ftot += R * R;
      r.m = ftot; ftot += sm * sm;
      r.status = itot; itot += 1;
      r.g = gtot; gtot += R;
      r.yv = gtot; gtot += R;
    }
    p->W[f] = W;
    p->y_off[f] = ytot;
    ytot += n * std::max<int64_t>(W, 1);
  }
  p->g_per_col = gtot;
  CU(p->Y.ensure((size_t)ytot * 8 + 8, st));
  CU(p->Ytmp.ensure((size_t)ytot * 8 + 8, st));
  CU(p->F.ensure((size_t)ftot * 8 + 8, st));
  // statuses [0, itot) and near-singular flags of the coupling systems [itot, 2 itot)
  CU(p->I.ensure((size_t)2 * itot * 4 + 4, st));
  CU(cudaMemsetAsync(p->I.p, 0, (size_t)2 * itot * 4 + 4, st));
  // large Gauss-Jordan scratch: the largest single stage (stages run in order)
  {
    size_t need = 0, leaf_need = 0;
    for (int s : p->leaves) {
      const size_t b = hk_gj_scratch_bytes((int)(p->nodes[s].hi - p->nodes[s].lo));
      leaf_need += (b + 255) / 256 * 256;
    }
    need = leaf_need * p->batch;
    for (int lvl = 0; lvl < p->depth; ++lvl) {
      size_t lv = 0;
      for (int64_t f = 0; f < p->batch; ++f)
        for (int s : p->internal) {
          if (p->nodes[s].level != lvl) continue;
          const NodeRec& r = p->rec[f * nn + s];
          if (r.R == 0) continue;
          const size_t b = hk_gj_scratch_bytes(std::min(r.ru, r.rl));
          lv += (b + 255) / 256 * 256;
        }
      need = std::max(need, lv);
    }
    p->gjs_need = need;
    if (need) CU(p->gjs_d.ensure(need + 256, st));
  }
  p->stage.reset();
  // Front groups: the fronts of a batch are independent, so G groups run
  // their factorization chains on G streams and one group's latency-bound
  // Gauss-Jordan phases overlap another's GEMMs (HK_FACTOR_GROUPS, default 2
  // for batches of >= 4 fronts; 1 when large GJ systems share the scratch).
  int G = 1;
  {
    const char* e = getenv("HK_FACTOR_GROUPS");
    const int want = e ? atoi(e) : 2;
    if (want > 1 && p->batch >= 2 * want && p->gjs_need == 0 && wext == 0) G = std::min(want, 4);
  }
  std::vector<std::vector<Op>> gops((size_t)G);
  std::vector<cudaStream_t> gst((size_t)G, st);
  if (G > 1) {
    CHK(ensure_side_streams(p));
    CU(cudaEventRecord(p->ev[3], st));
    for (int g = 0; g < G; ++g) {
      gst[g] = p->side[g];
      CU(cudaStreamWaitEvent(gst[g], p->ev[3], 0));
    }
  }
  auto grp_lo = [&](int g) { return p->batch * g / G; };
  auto grp_hi = [&](int g) { return p->batch * (g + 1) / G; };
  // commit the staged task arrays on `st`, then launch every group's ops on its stream
  int phase = 0;
  auto launch_groups = [&]() -> hk_status {
    if (G == 1) return flush(p, gops[0], st);
    CU(p->stage.commit(st));
    if ((int)p->fev.size() <= phase) {
      cudaEvent_t e;
      CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      p->fev.push_back(e);
    }
    CU(cudaEventRecord(p->fev[phase], st));
    for (int g = 0; g < G; ++g) {
      CU(cudaStreamWaitEvent(gst[g], p->fev[phase], 0));
      CHK(launch_ops(p, gops[g], gst[g]));
    }
    ++phase;
    return HK_OK;
  };
  double* Y = p->Y.as<double>();
  double* Yt = p->Ytmp.as<double>();
  double* F = p->F.as<double>();
  int32_t* I = p->I.as<int32_t>();
  const double* UV = p->UV.as<double>();

  // ---- leaves first: the Gauss-Jordan inverses of the diagonal blocks need only the
  // front, so they are staged and launched before the (larger) Z gather and leaf GEMM
  // task lists are planned; the GPU inverts the leaves meanwhile (hodlr.py:222-232)
  for (int g = 0; g < G; ++g) {
  std::vector<Op>& ops = gops[g];
  {
    std::vector<GjTask> gts;
    for (int64_t f = grp_lo(g); f < grp_hi(g); ++f)
      for (int s : p->leaves) {
        const Node& nd = p->nodes[s];
        const NodeRec& r = p->rec[f * nn + s];
        GjTask t{};
        t.src = p->A + f * p->fstride + nd.lo * p->lda + nd.lo;
        t.src_ld = p->lda;
        t.out = F + r.inv;
        t.out_ld = nd.hi - nd.lo;
        t.status = I + r.status;
        t.N = (int)(nd.hi - nd.lo);
        t.mode = 0;
        gts.push_back(t);
      }
    if (leaf_tma_ok(p, gts)) {
      Op o{Op::GJ_LEAF_TMA};
      o.a = p->stage.push(gts, st);
      if (!o.a) return fail(HK_ERR_CUDA, "pinned staging allocation failed");
      o.n = (int)gts.size();
      o.maxN = 64;
      ops.push_back(o);
    } else {
      CHK(stage_gj(p, ops, gts, st));
    }
  }
  }
  CHK(launch_groups());
  // ---- Z gather: U of every block into the rows of its child, columns [w_p, w_p + r),
  // then Y = K^{-1} Z
  for (int g = 0; g < G; ++g) {
  std::vector<Op>& ops = gops[g];
  std::vector<CopyTask> copies;
  for (int64_t f = grp_lo(g); f < grp_hi(g); ++f)
    for (int k = 0; k < (int)p->internal.size(); ++k) {
      const int s = p->internal[k];
      const NodeRec& r = p->rec[f * nn + s];
      for (int side = 0; side < 2; ++side) {
        const BlockGeom& b = p->blocks[2 * k + side];
        const int rank = side == 0 ? r.ru : r.rl;
        if (rank == 0) continue;
        CopyTask c{};
        c.src = UV + f * p->uv_per_front + b.u_off;   // column-major m x cap, ld ldu
        c.src_rs = 1;
        c.src_cs = b.ldu;
        c.dst = Yt + p->y_off[f] + b.row0 + r.w * n;   // column-major, ld n
        c.dst_rs = 1;
        c.dst_cs = n;
        c.rows = b.m;
        c.cols = rank;
        copies.push_back(c);
      }
    }
  if (wext > 0) {                 // the caller's extension columns come first (farthest)
    CopyTask c{};
    c.src = Zext; c.src_rs = 1; c.src_cs = ldz;
    c.dst = Yt + p->y_off[0]; c.dst_rs = 1; c.dst_cs = n;
    c.rows = n; c.cols = wext;
    copies.push_back(c);
  }
  if (!copies.empty()) {
    Op o{Op::COPY};
    o.a = p->stage.push(copies, st);
    if (!o.a) return fail(HK_ERR_CUDA, "pinned staging allocation failed");
    o.n = (int)copies.size();
    ops.push_back(o);
  }

  {
    TileList tl;
    for (int64_t f = grp_lo(g); f < grp_hi(g); ++f)
      for (int s : p->leaves) {
        const Node& nd = p->nodes[s];
        const NodeRec& r = p->rec[f * nn + s];
        const int b = (int)(nd.hi - nd.lo);
        if (r.w == 0) continue;
        tl.add(gemm(F + r.inv, b, 0, Yt + p->y_off[f] + nd.lo, n, Y + p->y_off[f] + nd.lo, n, b,
                    (int)r.w, b, 1.0, 0.0));
      }
    CHK(stage_tiles(p, ops, tl, st));
  }
  if (g == 0) {
    Op o{Op::EVENT};
    o.ev = 1;
    ops.push_back(o);
  }
  }
  hc.mark("plan leaves");
  CHK(launch_groups());          // the GPU starts on the leaves while the levels are planned

  // ---- upward sweep, deepest internal level first (hodlr.py:264-282).
  // The coupling system S = [[I, X], [Y, I]] (X = V_low^T d_left, Y = V_up^T
  // d_right) is inverted by block elimination of one identity block: only the
  // Woodbury capacitance M = I - Y X (or I - X Y, whichever is smaller) is
  // factored, with partial pivoting; S^{-1} is assembled by GEMMs and kept
  // for the solve phase.  det S = det M, so singular S <=> singular M.
  for (int lvl = p->depth - 1; lvl >= 0; --lvl) {
  for (int g = 0; g < G; ++g) {
    std::vector<Op>& ops = gops[g];
    TileList th, tm, t4, t5, tq, tu;
    std::vector<GjTask> gts;
    for (int64_t f = grp_lo(g); f < grp_hi(g); ++f)
      for (int k = 0; k < (int)p->internal.size(); ++k) {
        const int s = p->internal[k];
        const Node& nd = p->nodes[s];
        if (nd.level != lvl) continue;
        const NodeRec& r = p->rec[f * nn + s];
        if (r.R == 0) continue;
        const Node& a = p->nodes[nd.left];
        const Node& b = p->nodes[nd.right];
        const int na = (int)(a.hi - a.lo), nbr = (int)(b.hi - b.lo);
        const BlockGeom& bu = p->blocks[2 * k];
        const BlockGeom& bl = p->blocks[2 * k + 1];
        const double* Vup = UV + f * p->uv_per_front + bu.v_off;   // nb x ru
        const double* Vlow = UV + f * p->uv_per_front + bl.v_off;  // na x rl
        double* Yf = Y + p->y_off[f];
        double* H = F + r.h;
        double* Si = F + r.inv;
        double* M = F + r.m;
        const int R = r.R, rl = r.rl, ru = r.ru;
        const int w = (int)r.w;
        // H[0:rl, 0:w+ru] = V_low^T Y[a, 0:w+ru];  H[rl:R, 0:w+rl] = V_up^T Y[b, 0:w+rl]
        if (rl > 0) th.add(gemm(Vlow, bl.ldv, 1, Yf + a.lo, n, H, R, rl, w + ru, na, 1.0, 0.0));
        if (ru > 0) th.add(gemm(Vup, bu.ldv, 1, Yf + b.lo, n, H + rl, R, ru, w + rl, nbr, 1.0, 0.0));
        const double* X = H + (int64_t)w * R;          // rl x ru
        const double* Yc = H + rl + (int64_t)w * R;    // ru x rl
        GjTask g{};
        g.src_ld = 0;
        g.out_ld = R;
        g.status = I + r.status;
        g.near = I + itot + r.status;
        g.mode = 1;
        if (ru <= rl) {
          // M = I_u - Y X ; S^{-1} = [[I - X (-M^{-1} Y), -X M^{-1}], [-M^{-1} Y, M^{-1}]]
          tm.add(gemm(Yc, R, 0, X, R, M, ru, ru, ru, rl, -1.0, 0.0, 1.0));
          g.src = M; g.src_ld = ru; g.out = Si + rl + (int64_t)rl * R; g.N = ru;
          const double* Mi = Si + rl + (int64_t)rl * R;
          t4.add(gemm(Mi, R, 0, Yc, R, Si + rl, R, ru, rl, ru, -1.0, 0.0));
          t4.add(gemm(X, R, 0, Mi, R, Si + (int64_t)rl * R, R, rl, ru, ru, -1.0, 0.0));
          t5.add(gemm(X, R, 0, Si + rl, R, Si, R, rl, rl, ru, -1.0, 0.0, 1.0));
        } else {
          // M = I_l - X Y ; S^{-1} = [[M^{-1}, -M^{-1} X], [-Y M^{-1}, I - Y (-M^{-1} X)]]
          tm.add(gemm(X, R, 0, Yc, R, M, rl, rl, rl, ru, -1.0, 0.0, 1.0));
          g.src = M; g.src_ld = rl; g.out = Si; g.N = rl;
          t4.add(gemm(Si, R, 0, X, R, Si + (int64_t)rl * R, R, rl, ru, rl, -1.0, 0.0));
          t4.add(gemm(Yc, R, 0, Si, R, Si + rl, R, ru, rl, rl, -1.0, 0.0));
          t5.add(gemm(Yc, R, 0, Si + (int64_t)rl * R, R, Si + rl + (int64_t)rl * R, R, ru, ru, rl,
                      -1.0, 0.0, 1.0));
        }
        gts.push_back(g);
        if (w > 0) {
          double* Q = F + r.q;
          tq.add(gemm(Si, R, 0, H, R, Q, R, R, w, R, 1.0, 0.0));
          // top -= d_left y_up ; bottom -= d_right y_low
          if (ru > 0) tu.add(gemm(Yf + a.lo + (int64_t)w * n, n, 0, Q + rl, R, Yf + a.lo, n, na, w, ru, -1.0, 1.0));
          if (rl > 0) tu.add(gemm(Yf + b.lo + (int64_t)w * n, n, 0, Q, R, Yf + b.lo, n, nbr, w, rl, -1.0, 1.0));
        }
      }
    CHK(stage_tiles(p, ops, th, st));
    CHK(stage_tiles(p, ops, tm, st));
    CHK(stage_gj(p, ops, gts, st));
    CHK(stage_tiles(p, ops, t4, st));
    CHK(stage_tiles(p, ops, t5, st));
    CHK(stage_tiles(p, ops, tq, st));
    CHK(stage_tiles(p, ops, tu, st));
  }
    CHK(launch_groups());
  }
  if (G > 1) {                   // join the group streams
    for (int g = 0; g < G; ++g) {
      CU(cudaEventRecord(p->side_ev[g], gst[g]));
      CU(cudaStreamWaitEvent(st, p->side_ev[g], 0));
    }
  }
  CU(cudaEventRecord(p->ev[2], st));
  hc.mark("plan+launch levels");
  // The usual next call -- one solve of every front, one rhs -- gets its
  // program planned now, on the host, while the GPU still runs the levels
  // (otherwise ~0.2 ms of host planning per batch with the GPU idle).
  if (wext == 0) {
    SolveProg* sp = nullptr;
    if (ensure_solve_scratch(p, 1, st) == HK_OK) (void)build_solve_prog(p, -1, 1, sp, st);
    hc.mark("solve program");
  }
  // ---- statuses: first failure in the reference's DFS event order
  std::vector<int32_t> ih((size_t)2 * itot);
  if (itot) CU(cudaMemcpyAsync(ih.data(), I, (size_t)2 * itot * 4, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  // A coupling system whose capacitance matrix M had a pivot below
  // HK_NEAR_PIVOT (or none above 1e-300) is re-decided the reference's way:
  // partial-pivot LU of S itself, singular iff min |U_kk| < 1e-300
  // (hodlr.py:272-277, dense.py:76-77).  det S = det M, but the pivots of the
  // two eliminations differ, so only this keeps the raise/no-raise decision
  // identical near singularity.  Never triggered on well-conditioned fronts.
  for (int64_t f = 0; f < p->batch; ++f)
    for (int s : p->internal) {
      const NodeRec& r = p->rec[f * nn + s];
      if (r.status < 0 || r.R == 0) continue;
      if (ih[r.status] == 0 && ih[itot + r.status] == 0) continue;
      LuTask t{};
      t.src = F + r.h;
      t.src_ld = r.R;
      t.mode = 1;
      t.rl = r.rl;
      t.ru = r.ru;
      t.h_col0 = r.w;
      int sing = 0;
      CHK(lu_on_demand(t, r.R, nullptr, nullptr, &sing));
      // an exactly singular M cannot be inverted: it stays singular even if
      // S's rounding gave pivots above the floor (measure-zero case)
      ih[r.status] = (sing || ih[r.status]) ? 1 : 0;
    }
  hc.mark("wait");
  if (host_profile()) g_opprof.print("factor");
  float ms1 = 0, ms2 = 0;
  CU(cudaEventElapsedTime(&ms1, p->ev[0], p->ev[1]));
  CU(cudaEventElapsedTime(&ms2, p->ev[1], p->ev[2]));
  p->t_leaf = ms1 * 1e-3;
  p->t_schur = ms2 * 1e-3;
  for (int64_t f = 0; f < p->batch; ++f) {
    int best = -1;
    for (int s = 0; s < nn; ++s) {
      const NodeRec& r = p->rec[f * nn + s];
      if (r.status < 0) continue;
      if (ih[r.status] != 0 && (best < 0 || p->post[s] < p->post[best])) best = s;
    }
    if (best >= 0) {
      const Node& nd = p->nodes[best];
      char msg[200];
      if (nd.left < 0) {
        snprintf(msg, sizeof msg, "leaf block [%lld, %lld) is singular (front %lld)",
                 (long long)nd.lo, (long long)nd.hi, (long long)f);
        return fail(HK_ERR_SINGULAR_LEAF, msg);
      }
      snprintf(msg, sizeof msg,
               "coupling system singular at node [%lld, %lld) (front %lld); compression "
               "tolerance is too loose", (long long)nd.lo, (long long)nd.hi, (long long)f);
      return fail(HK_ERR_SINGULAR_SCHUR, msg);
    }
  }
  p->factored = true;
  return HK_OK;
}

extern "C" hk_status hk_factor(hk_plan* p, void* stream) {
  return hk_factor_ext(p, nullptr, 0, 0, stream);
}

extern "C" hk_status hk_get_extension(hk_plan* p, int64_t front, double** Y, int64_t* ld,
                                      int64_t* width) {
  if (!p || !p->factored) return fail(HK_ERR_STATE, "extension requires a factorization");
  if (front < 0 || front >= p->batch) return fail(HK_ERR_VALUE, "front out of range");
  *Y = p->Y.as<double>() + p->y_off[front];
  *ld = p->n;
  *width = p->W[front];
  return HK_OK;
}

extern "C" hk_status hk_copy_extension(hk_plan* p, int64_t front, int64_t col0, int64_t ncols,
                                       double* dst, int64_t ldd, void* stream) {
  if (!p || !p->factored) return fail(HK_ERR_STATE, "extension requires a factorization");
  if (front < 0 || front >= p->batch) return fail(HK_ERR_VALUE, "front out of range");
  if (col0 < 0 || ncols < 0 || col0 + ncols > std::max<int64_t>(p->W[front], 0))
    return fail(HK_ERR_VALUE, "extension columns out of range");
  if (ncols == 0) return HK_OK;
  if (ldd < p->n) return fail(HK_ERR_DIMENSION, "destination leading dimension smaller than n");
  const double* src = p->Y.as<double>() + p->y_off[front] + col0 * p->n;
  CU(cudaMemcpy2DAsync(dst, ldd * 8, src, p->n * 8, p->n * 8, ncols, cudaMemcpyDeviceToDevice,
                       (cudaStream_t)stream));
  return HK_OK;
}

extern "C" hk_status hk_dgemm(int transa, int64_t m, int64_t n, int64_t k, double alpha,
                              const double* A, int64_t lda, const double* B, int64_t ldb,
                              double beta, double* C, int64_t ldc, void* stream) {
  if (m < 0 || n < 0 || k < 0) return fail(HK_ERR_VALUE, "negative GEMM dimension");
  if (m == 0 || n == 0) return HK_OK;
  if (m > INT32_MAX || n > INT32_MAX || k > INT32_MAX) return fail(HK_ERR_VALUE, "GEMM too large");
  cudaStream_t st = (cudaStream_t)stream;
  TileList tl;
  tl.add(gemm(A, lda, transa ? 1 : 0, B, ldb, C, ldc, (int)m, (int)n, (int)k, alpha, beta));
  if (tl.ntiles() == 0) return HK_OK;
  char* d = nullptr;
  const size_t tb = sizeof(GemmTask), mb = tl.map.size() * 4;
  CU(hk_dev_malloc((void**)&d, tb + 256 + mb, st));
  CU(cudaMemcpyAsync(d, tl.tasks.data(), tb, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(d + 256, tl.map.data(), mb, cudaMemcpyHostToDevice, st));
  CU(hk_launch_gemm((const GemmTask*)d, (const int32_t*)(d + 256), tl.ntiles(), st));
  CU(hk_dev_free(d, st));
  return HK_OK;
}

extern "C" hk_status hk_get_aca_time(hk_plan* p, double* seconds) {
  if (!p) return fail(HK_ERR_VALUE, "null plan");
  *seconds = p->t_aca;
  return HK_OK;
}

extern "C" hk_status hk_get_timings(hk_plan* p, double* lowrank, double* leaf_lu, double* schur) {
  if (!p) return fail(HK_ERR_VALUE, "null plan");
  *lowrank = p->t_lowrank;
  *leaf_lu = p->t_leaf;
  *schur = p->t_schur;
  return HK_OK;
}

static void colmajor_to_rowmajor(const std::vector<double>& cm, int64_t rows, int64_t cols,
                                 int64_t ld, double* out) {
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) out[i * cols + j] = cm[i + j * ld];
}

// On-demand partial-pivot LU (inspection of leaf_lus / couplings[].schur_lu;
// the hot path keeps explicit inverses instead).
static hk_status lu_on_demand(const LuTask& proto, int N, double* lu_host, int32_t* piv_host,
                              int* singular, double* inv_host) {
  if (singular) *singular = 0;
  if (N == 0) return HK_OK;
  double* lu = nullptr;
  double* inv = nullptr;
  if (inv_host) CU(cudaMalloc(&inv, (size_t)N * N * 8));
  int32_t *ip = nullptr, *pm = nullptr, *stt = nullptr;
  LuTask* td = nullptr;
  CU(cudaMalloc(&lu, (size_t)N * N * 8));
  CU(cudaMalloc(&ip, (size_t)N * 4));
  CU(cudaMalloc(&pm, (size_t)N * 4));
  CU(cudaMalloc(&stt, 8));
  CU(cudaMalloc(&td, sizeof(LuTask)));
  LuTask t = proto;
  t.lu = lu; t.ipiv = ip; t.perm = pm; t.status = stt; t.inv = inv; t.N = N;
  CU(cudaMemcpy(td, &t, sizeof(LuTask), cudaMemcpyHostToDevice));
  CU(hk_launch_lu(td, 1, N, 0));
  if (lu_host) {
    std::vector<double> h((size_t)N * N);
    CU(cudaMemcpy(h.data(), lu, h.size() * 8, cudaMemcpyDeviceToHost));
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) lu_host[(int64_t)i * N + j] = h[i + (int64_t)j * N];
  }
  if (piv_host) CU(cudaMemcpy(piv_host, ip, (size_t)N * 4, cudaMemcpyDeviceToHost));
  int32_t sg = 0;
  CU(cudaMemcpy(&sg, stt, 4, cudaMemcpyDeviceToHost));
  if (singular) *singular = sg != 0;
  if (inv_host && !sg) {   // column-major inverse -> row-major host copy
    std::vector<double> h((size_t)N * N);
    CU(cudaMemcpy(h.data(), inv, h.size() * 8, cudaMemcpyDeviceToHost));
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) inv_host[(int64_t)i * N + j] = h[i + (int64_t)j * N];
  }
  if (inv) cudaFree(inv);
  cudaFree(lu); cudaFree(ip); cudaFree(pm); cudaFree(stt); cudaFree(td);
  return HK_OK;
}

extern "C" hk_status hk_get_leaf_lu(hk_plan* p, int64_t f, int64_t slot, double* lu, int32_t* perm,
                                    double* inv) {
  if (!p || !p->factored) return fail(HK_ERR_STATE, "plan not factored");
  const Node& nd = p->nodes[slot];
  if (nd.left >= 0) return fail(HK_ERR_VALUE, "not a leaf");
  LuTask t{};
  t.src = p->A + f * p->fstride + nd.lo * p->lda + nd.lo;
  t.src_ld = p->lda;
  t.mode = 0;
  return lu_on_demand(t, (int)(nd.hi - nd.lo), lu, perm, nullptr, inv);
}

extern "C" hk_status hk_get_coupling(hk_plan* p, int64_t f, int64_t slot, double* dl, double* dr,
                                     double* slu, int32_t* sperm, double* sinv) {
  if (!p || !p->factored) return fail(HK_ERR_STATE, "plan not factored");
  const Node& nd = p->nodes[slot];
  if (nd.left < 0) return fail(HK_ERR_VALUE, "not an internal node");
  const NodeRec& r = p->rec[f * p->nodes.size() + slot];
  const Node& a = p->nodes[nd.left];
  const Node& b = p->nodes[nd.right];
  const int64_t n = p->n;
  const double* Yf = p->Y.as<double>() + p->y_off[f];
  if (dl && r.ru > 0) {
    std::vector<double> h((size_t)n * r.ru);
    CU(cudaMemcpy2D(h.data(), (a.hi - a.lo) * 8, Yf + a.lo + r.w * n, n * 8, (a.hi - a.lo) * 8,
                    r.ru, cudaMemcpyDeviceToHost));
    colmajor_to_rowmajor(h, a.hi - a.lo, r.ru, a.hi - a.lo, dl);
  }
  if (dr && r.rl > 0) {
    std::vector<double> h((size_t)n * r.rl);
    CU(cudaMemcpy2D(h.data(), (b.hi - b.lo) * 8, Yf + b.lo + r.w * n, n * 8, (b.hi - b.lo) * 8,
                    r.rl, cudaMemcpyDeviceToHost));
    colmajor_to_rowmajor(h, b.hi - b.lo, r.rl, b.hi - b.lo, dr);
  }
  if (slu && r.R > 0) {
    LuTask t{};
    t.src = p->F.as<double>() + r.h;
    t.src_ld = r.R;
    t.mode = 1;
    t.rl = r.rl;
    t.ru = r.ru;
    t.h_col0 = r.w;
    CHK(lu_on_demand(t, r.R, slu, sperm, nullptr, sinv));
  }
  return HK_OK;
}

// ------------------------------------------------------------------ solve
// Build (and cache) the task lists of one solve program for `front` (-1 =
// every front) and s right-hand sides.  Scratch: Xin/X2 (n x s per front),
// G/Yv (R x s per node).
static hk_status build_solve_prog(hk_plan* p, int front, int s, SolveProg*& out, cudaStream_t st) {
  auto key = std::make_pair(front, s);
  auto it = p->progs.find(key);
  if (it != p->progs.end()) {
    out = it->second;
    return HK_OK;
  }
  SolveProg* sp = new SolveProg();
  sp->s = s;
  sp->small = s <= 16;
  const int64_t n = p->n;
  const int nn = (int)p->nodes.size();
  const size_t nb = p->blocks.size();
  const double* UV = p->UV.as<double>();
  double* F = p->F.as<double>();
  const double* Xin = p->Xin.as<double>();
  double* X2 = p->X2.as<double>();
  double* G = p->G.as<double>();
  double* Yv = p->Yv.as<double>();
  const int64_t xs = n * s;  // per-front stride of Xin/X2
  int64_t f0 = front < 0 ? 0 : front, f1 = front < 0 ? p->batch : front + 1;
  // leaves
  {
    std::vector<SgemvTask> sg;
    std::vector<int32_t> items;
    TileList tl;
    for (int64_t f = f0; f < f1; ++f) {
      for (int slot : p->leaves) {
        const Node& nd = p->nodes[slot];
        const NodeRec& r = p->rec[f * nn + slot];
        const int b = (int)(nd.hi - nd.lo);
        if (sp->small) {
          SgemvTask t{};
          t.M = F + r.inv; t.ldm = b;
          t.v0 = Xin + f * xs + nd.lo; t.ldv = n;
          t.y = X2 + f * xs + nd.lo; t.ldy = n;
          t.rows = b; t.K = b; t.mode = 0;
          for (int rb = 0; rb * HK_SGEMV_ROWS < b; ++rb) {
            items.push_back((int32_t)sg.size());
            items.push_back(rb);
          }
          sg.push_back(t);
          sp->leaf.max_k = std::max(sp->leaf.max_k, b);
        } else {
          tl.add(gemm(F + r.inv, b, 0, Xin + f * xs + nd.lo, n, X2 + f * xs + nd.lo, n, b, s, b, 1.0, 0.0));
        }
      }
    }
    if (sp->small) {
      sp->leaf.t = p->pstage.push(sg, st);
      sp->leaf.items = p->pstage.push(items, st);
      sp->leaf.nitems = (int)(items.size() / 2);
      if (!sp->leaf.t || !sp->leaf.items) { delete sp; return fail(HK_ERR_CUDA, "pinned staging allocation failed"); }
    } else {
      sp->leaf_tiles = tl.ntiles();
      sp->leaf_g = p->pstage.push(tl.tasks, st);
      sp->leaf_map = p->pstage.push(tl.map, st);
      if (!sp->leaf_g || !sp->leaf_map) { delete sp; return fail(HK_ERR_CUDA, "pinned staging allocation failed"); }
    }
  }
  // partial-dot scratch: the largest level (levels run in stream order)
  if (sp->small) {
    int64_t need = 0;
    for (int lvl = 0; lvl < p->depth; ++lvl) {
      int64_t lv = 0;
      for (int64_t f = f0; f < f1; ++f)
        for (int k = 0; k < (int)p->internal.size(); ++k) {
          const Node& nd = p->nodes[p->internal[k]];
          if (nd.level != lvl) continue;
          const NodeRec& r = p->rec[f * nn + p->internal[k]];
          const int64_t na = p->nodes[nd.left].hi - p->nodes[nd.left].lo;
          const int64_t nbr = p->nodes[nd.right].hi - p->nodes[nd.right].lo;
          lv += ((na + HK_PDOT_ROWS - 1) / HK_PDOT_ROWS) * r.rl + ((nbr + HK_PDOT_ROWS - 1) / HK_PDOT_ROWS) * r.ru;
        }
      need = std::max(need, lv);
    }
    if (sp->pbuf.ensure((size_t)need * s * 8 + 64, st) != cudaSuccess) {
      delete sp;
      return fail(HK_ERR_CUDA, "solve scratch allocation failed");
    }
  }
  for (int lvl = p->depth - 1; lvl >= 0; --lvl) {
    SolveProg::Level L;
    std::vector<PdotTask> pd;
    std::vector<int32_t> pitems, sitems, uitems;
    std::vector<SgemvTask> sv, up;
    TileList t1, t2, t3;
    int64_t poff = 0;   // doubles into pbuf (levels reuse it in stream order)
    double* P = sp->pbuf.as<double>();
    for (int64_t f = f0; f < f1; ++f) {
      for (int k = 0; k < (int)p->internal.size(); ++k) {
        const int slot = p->internal[k];
        const Node& nd = p->nodes[slot];
        if (nd.level != lvl) continue;
        const NodeRec& r = p->rec[f * nn + slot];
        if (r.R == 0) continue;
        const Node& a = p->nodes[nd.left];
        const Node& b = p->nodes[nd.right];
        const int na = (int)(a.hi - a.lo), nbr = (int)(b.hi - b.lo);
        const BlockGeom& bu = p->blocks[2 * k];
        const BlockGeom& bl = p->blocks[2 * k + 1];
        const double* Vup = UV + f * p->uv_per_front + bu.v_off;
        const double* Vlow = UV + f * p->uv_per_front + bl.v_off;
        const double* Yf = p->Y.as<double>() + p->y_off[f];
        double* Xf = X2 + f * xs;
        double* g = G + r.g * s;     // R x s, ld R
        double* yv = Yv + r.g * s;   // R x s, ld R
        const int R = r.R, rl = r.rl, ru = r.ru;
        const double* dleft = Yf + a.lo + r.w * n;
        const double* dright = Yf + b.lo + r.w * n;
        if (sp->small) {
          // g = [V_low^T x_a ; V_up^T x_b] as partial dots, reduced inside the S^-1 sgemv
          const int nchA = (na + HK_PDOT_ROWS - 1) / HK_PDOT_ROWS;
          const int nchB = (nbr + HK_PDOT_ROWS - 1) / HK_PDOT_ROWS;
          double* PA = P + poff;
          poff += (int64_t)nchA * rl * s;
          double* PB = P + poff;
          poff += (int64_t)nchB * ru * s;
          auto add_pdot = [&](const double* M, int64_t ldm, const double* x, int rows, int cols, double* Pp) {
            if (cols == 0) return;
            const int ti = (int)pd.size();
            pd.push_back(PdotTask{M, x, Pp, ldm, (int64_t)n, rows, cols});
            for (int ch = 0; ch * HK_PDOT_ROWS < rows; ++ch)
              for (int cb = 0; cb * HK_PDOT_COLS < cols; ++cb) {
                pitems.push_back(ti);
                pitems.push_back(ch);
                pitems.push_back(cb);
              }
          };
          add_pdot(Vlow, bl.ldv, Xf + a.lo, na, rl, PA);
          add_pdot(Vup, bu.ldv, Xf + b.lo, nbr, ru, PB);
          SgemvTask t{};
          t.M = F + r.inv; t.ldm = R;
          t.v0 = nullptr; t.PA = PA; t.PB = PB; t.KA = rl; t.nchA = nchA; t.nchB = nchB;
          t.y = yv; t.ldy = R; t.rows = R; t.K = R; t.mode = 0;
          for (int rb = 0; rb * HK_SGEMV_ROWS < R; ++rb) {
            sitems.push_back((int32_t)sv.size());
            sitems.push_back(rb);
          }
          sv.push_back(t);
          L.sinv.max_k = std::max(L.sinv.max_k, R);
          // top -= d_left y_up ; bottom -= d_right y_low
          auto add_upd = [&](const double* M, const double* v, double* y, int rows, int K) {
            if (K == 0 || rows == 0) return;
            SgemvTask u{};
            u.M = M; u.ldm = n; u.v0 = v; u.ldv = R; u.y = y; u.ldy = n;
            u.rows = rows; u.K = K; u.mode = 1;
            for (int rb = 0; rb * HK_SGEMV_ROWS < rows; ++rb) {
              uitems.push_back((int32_t)up.size());
              uitems.push_back(rb);
            }
            up.push_back(u);
            L.upd.max_k = std::max(L.upd.max_k, K);
          };
          add_upd(dleft, yv + rl, Xf + a.lo, na, ru);
          add_upd(dright, yv, Xf + b.lo, nbr, rl);
        } else {
          if (rl > 0) t1.add(gemm(Vlow, bl.ldv, 1, Xf + a.lo, n, g, R, rl, s, na, 1.0, 0.0));
          if (ru > 0) t1.add(gemm(Vup, bu.ldv, 1, Xf + b.lo, n, g + rl, R, ru, s, nbr, 1.0, 0.0));
          t2.add(gemm(F + r.inv, R, 0, g, R, yv, R, R, s, R, 1.0, 0.0));
          if (ru > 0) t3.add(gemm(dleft, n, 0, yv + rl, R, Xf + a.lo, n, na, s, ru, -1.0, 1.0));
          if (rl > 0) t3.add(gemm(dright, n, 0, yv, R, Xf + b.lo, n, nbr, s, rl, -1.0, 1.0));
        }
      }
    }
    bool ok = true;
    if (sp->small) {
      L.n_pdot = (int)(pitems.size() / 3);
      L.pdot_t = p->pstage.push(pd, st);
      L.pdot_items = p->pstage.push(pitems, st);
      L.sinv.t = p->pstage.push(sv, st);
      L.sinv.items = p->pstage.push(sitems, st);
      L.sinv.nitems = (int)(sitems.size() / 2);
      L.upd.t = p->pstage.push(up, st);
      L.upd.items = p->pstage.push(uitems, st);
      L.upd.nitems = (int)(uitems.size() / 2);
      ok = L.pdot_t && L.pdot_items && L.sinv.t && L.sinv.items && L.upd.t && L.upd.items;
    } else {
      L.t1 = t1.ntiles(); L.t2 = t2.ntiles(); L.t3 = t3.ntiles();
      L.g1 = p->pstage.push(t1.tasks, st); L.g1map = p->pstage.push(t1.map, st);
      L.g2 = p->pstage.push(t2.tasks, st); L.g2map = p->pstage.push(t2.map, st);
      L.g3 = p->pstage.push(t3.tasks, st); L.g3map = p->pstage.push(t3.map, st);
      ok = L.g1 && L.g1map && L.g2 && L.g2map && L.g3 && L.g3map;
    }
    if (!ok) { delete sp; return fail(HK_ERR_CUDA, "pinned staging allocation failed"); }
    sp->levels.push_back(std::move(L));
  }
  (void)nb;
  CU(p->pstage.commit(st));
  p->progs[key] = sp;
  out = sp;
  return HK_OK;
}

static hk_status ensure_solve_scratch(hk_plan* p, int s, cudaStream_t st) {
  const size_t need_x = (size_t)p->batch * p->n * s * 8 + 8;
  const size_t need_g = (size_t)p->g_per_col * s * 8 + 8;
  if (p->Xin.bytes < need_x || p->X2.bytes < need_x || p->G.bytes < need_g || p->Yv.bytes < need_g) {
    // buffers move: cached programs hold raw pointers -> drop them
    CU(cudaStreamSynchronize(st));
    drop_progs(p, st);
    CU(p->Xin.ensure(need_x, st));
    CU(p->X2.ensure(need_x, st));
    CU(p->G.ensure(need_g, st));
    CU(p->Yv.ensure(need_g, st));
  }
  return HK_OK;
}

// The solve program's kernel sequence: leaf solve, then per level (deepest
// first) V^T x partial dots -> S^{-1} g -> x -= d y  (hodlr.py:298-306).
static hk_status launch_solve_kernels(SolveProg* sp, int s, cudaStream_t st, bool prof) {
  if (sp->small) {
    CU(hk_launch_sgemv(sp->leaf.t, sp->leaf.items, sp->leaf.nitems, s, sp->leaf.max_k, st));
    if (prof) g_opprof.mark("leaf sgemv", st);
  } else {
    if (sp->leaf_tiles) CU(hk_launch_gemm(sp->leaf_g, sp->leaf_map, sp->leaf_tiles, st));
  }
  for (auto& L : sp->levels) {
    if (sp->small) {
      CU(hk_launch_pdot(L.pdot_t, L.pdot_items, L.n_pdot, s, st));
      if (prof) g_opprof.mark("pdot " + std::to_string(L.n_pdot), st);
      CU(hk_launch_sgemv(L.sinv.t, L.sinv.items, L.sinv.nitems, s, L.sinv.max_k, st));
      if (prof) g_opprof.mark("sinv " + std::to_string(L.sinv.nitems), st);
      CU(hk_launch_sgemv(L.upd.t, L.upd.items, L.upd.nitems, s, L.upd.max_k, st));
      if (prof) g_opprof.mark("upd " + std::to_string(L.upd.nitems), st);
    } else {
      if (L.t1) CU(hk_launch_gemm(L.g1, L.g1map, L.t1, st));
      if (L.t2) CU(hk_launch_gemm(L.g2, L.g2map, L.t2, st));
      if (L.t3) CU(hk_launch_gemm(L.g3, L.g3map, L.t3, st));
    }
  }
  return HK_OK;
}

static hk_status run_solve(hk_plan* p, int front, double* rhs, int64_t ld, int64_t s,
                           int64_t rhs_stride, cudaStream_t st) {
  if (!p || !p->factored) return fail(HK_ERR_STATE, "solve requires a factorization");
  if (s <= 0) return HK_OK;
  const int64_t n = p->n;
  if (ld < n) return fail(HK_ERR_DIMENSION, "rhs leading dimension smaller than n");
  HostClock hc("solve");
  CHK(ensure_solve_scratch(p, (int)s, st));
  SolveProg* sp = nullptr;
  CHK(build_solve_prog(p, front, (int)s, sp, st));
  hc.mark("prog");
  const int64_t xs = n * s;
  const int64_t f0 = front < 0 ? 0 : front, f1 = front < 0 ? p->batch : front + 1;
  // one copy when the fronts' rhs blocks are packed like Xin (ld = n, stride = n*s)
  const bool packed = ld == n && (f1 - f0 == 1 || rhs_stride == xs);
  if (packed) {
    CU(cudaMemcpyAsync(p->Xin.as<double>() + f0 * xs, rhs, (size_t)(f1 - f0) * xs * 8,
                       cudaMemcpyDeviceToDevice, st));
  } else {
    for (int64_t f = f0; f < f1; ++f)
      CU(cudaMemcpy2DAsync(p->Xin.as<double>() + f * xs, n * 8, rhs + (f - f0) * rhs_stride, ld * 8,
                           n * 8, s, cudaMemcpyDeviceToDevice, st));
  }
  const bool prof = host_profile();
  if (prof) {
    g_opprof.reset();
    g_opprof.mark("start", st);
    CHK(launch_solve_kernels(sp, (int)s, st, true));
  } else if (++sp->uses >= 2) {
    if (!sp->gexec) {
      CHK(ensure_side_streams(p));
      cudaStream_t cs = p->side[0];
      const long long before = hk_launch_count();
      CU(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
      const hk_status h = launch_solve_kernels(sp, (int)s, cs, false);
      cudaGraph_t graph = nullptr;
      const cudaError_t e = cudaStreamEndCapture(cs, &graph);
      if (h != HK_OK) {
        if (graph) cudaGraphDestroy(graph);
        return h;
      }
      CU(e);
      sp->gkernels = (int)(hk_launch_count() - before);
      hk_count_launch(-sp->gkernels);       // captured, not executed
      const cudaError_t ei = cudaGraphInstantiate(&sp->gexec, graph, 0);
      cudaGraphDestroy(graph);
      CU(ei);
    }
    CU(cudaGraphLaunch(sp->gexec, st));
    hk_count_launch(sp->gkernels);
  } else {
    CHK(launch_solve_kernels(sp, (int)s, st, false));
  }
  if (packed) {
    CU(cudaMemcpyAsync(rhs, p->X2.as<double>() + f0 * xs, (size_t)(f1 - f0) * xs * 8,
                       cudaMemcpyDeviceToDevice, st));
  } else {
    for (int64_t f = f0; f < f1; ++f)
      CU(cudaMemcpy2DAsync(rhs + (f - f0) * rhs_stride, ld * 8, p->X2.as<double>() + f * xs, n * 8,
                           n * 8, s, cudaMemcpyDeviceToDevice, st));
  }
  hc.mark("launch");
  if (prof) {
    CU(cudaStreamSynchronize(st));
    g_opprof.print("solve");
  }
  return HK_OK;
}

extern "C" hk_status hk_solve(hk_plan* p, double* rhs, int64_t ld, int64_t nrhs, int64_t stride,
                              void* stream) {
  if (p && p->batch > 1 && stride < ld * nrhs) return fail(HK_ERR_DIMENSION, "rhs stride too small");
  return run_solve(p, -1, rhs, ld, nrhs, stride, (cudaStream_t)stream);
}

extern "C" hk_status hk_solve_front(hk_plan* p, int64_t front, double* rhs, int64_t ld,
                                    int64_t nrhs, void* stream) {
  if (!p || front < 0 || front >= p->batch) return fail(HK_ERR_VALUE, "front out of range");
  return run_solve(p, (int)front, rhs, ld, nrhs, 0, (cudaStream_t)stream);
}

// ------------------------------------------------------------------ GMRES
// Device-resident GMRES (krylov.py:69-166) for s <= 16 right-hand sides of one
// front, advanced in lock step.  One CUDA graph per (front, s, operator,
// preconditioner, tol, max_iter):
//
//   pre   ||b_c||, r0 = M^{-1} b, beta_c = ||r0_c||, Q_c[:,0] = r0_c / beta_c
//   WHILE (any system active and k < min(max_iter, n))        krylov.py:107
//         W = A V (one s-column GEMV, the front streamed once)   :110
//         W = M^{-1} W (the s-column HODLR sweep, factor streamed once)
//         Arnoldi/MGS/Givens per system; the last CTA updates the flags,
//         the history and the loop condition (cudaGraphSetConditional)  :111-145
//   post  x_c = Q_c y_c, true residuals                          :147-156
//
// The host launches the graph and reads the state once, after the loop:
// no per-iteration round trip.  Per system the arithmetic is that of a
// single-rhs run (the GEMV and the sweep treat columns independently), so
// iterates, counts and flags do not depend on s.  The Krylov basis starts
// with room for min(mmax, 64) vectors; when a system needs more, the loop
// stops at the capacity, the host grows the buffers (copying the basis,
// Hessenberg and rotations) and relaunches the loop alone.
struct GmresGraph {
  int64_t front = 0;
  int s = 0, precond = 0;
  const double* A = nullptr;
  int64_t lda = 0;
  const double* diag = nullptr;
  double tol = 0;
  int64_t max_iter = 0, mmax = 0, cap = 0;
  DevBuf basis, hess, cs, sn, g, V, W, B, X, hist, y, state;
  cudaGraphExec_t main = nullptr, resume = nullptr;
  long long k_pre = 0, k_body = 0, k_post = 0;   // kernels per part (launch counter)
};

static void destroy_gmres_graph(GmresGraph* g) {
  if (!g) return;
  if (g->main) cudaGraphExecDestroy(g->main);
  if (g->resume) cudaGraphExecDestroy(g->resume);
  DevBuf* all[] = {&g->basis, &g->hess, &g->cs, &g->sn, &g->g, &g->V, &g->W, &g->B, &g->X,
                   &g->hist, &g->y, &g->state};
  for (DevBuf* d : all) d->release();
  delete g;
}

static GmParams gm_params(const hk_plan* p, const GmresGraph* g) {
  GmParams P{};
  P.n = p->n;
  P.cap = g->cap;
  P.mmax = g->mmax;
  P.max_iter = g->max_iter;
  P.s = g->s;
  P.tol = g->tol;
  P.vs = g->cap + 1;
  P.bstride = p->n * (g->cap + 1);
  P.hstride = (g->cap + 1) * g->cap;
  P.basis = g->basis.as<double>();
  P.hess = g->hess.as<double>();
  P.cs = g->cs.as<double>();
  P.sn = g->sn.as<double>();
  P.g = g->g.as<double>();
  P.V = g->V.as<double>();
  P.hist = g->hist.as<double>();
  P.y = g->y.as<double>();
  P.st = g->state.as<GmState>();
  return P;
}

// Krylov buffers for capacity `cap` (fresh allocations; the caller copies).
static cudaError_t gm_alloc_krylov(const hk_plan* p, GmresGraph* g, int64_t cap, DevBuf* basis,
                                   DevBuf* hess, DevBuf* cs, DevBuf* sn, DevBuf* gv, DevBuf* y,
                                   cudaStream_t st) {
  const size_t s = (size_t)g->s, vs = (size_t)cap + 1;
  cudaError_t e;
  if ((e = basis->ensure(s * p->n * vs * 8, st)) != cudaSuccess) return e;
  if ((e = hess->ensure(s * vs * cap * 8, st)) != cudaSuccess) return e;
  if ((e = cs->ensure(s * vs * 8, st)) != cudaSuccess) return e;
  if ((e = sn->ensure(s * vs * 8, st)) != cudaSuccess) return e;
  if ((e = gv->ensure(s * vs * 8, st)) != cudaSuccess) return e;
  return y->ensure(s * vs * 8, st);
}

// body of the WHILE loop: W = M^{-1} A V, then the Arnoldi step of every system
static hk_status gm_body_ops(hk_plan* p, GmresGraph* g, SolveProg* sp, const GmParams& P,
                             cudaGraphConditionalHandle h, cudaStream_t cs) {
  const int64_t n = p->n;
  double* W = g->W.as<double>();
  if (g->precond == 1) {
    double* xin = p->Xin.as<double>() + g->front * n * g->s;
    CU(hk_launch_gemv_rowmajor(g->A, g->lda, n, n, P.V, n, g->s, xin, n, cs));
    CHK(launch_solve_kernels(sp, g->s, cs, false));
    W = p->X2.as<double>() + g->front * n * g->s;
  } else {
    CU(hk_launch_gemv_rowmajor(g->A, g->lda, n, n, P.V, n, g->s, W, n, cs));
    if (g->precond == 2) CU(hk_launch_vdiv(W, g->diag, W, n, g->s, cs));
  }
  CU(hk_launch_gm_arnoldi(P, W, h, cs));
  return HK_OK;
}

// Capture one executable graph: [pre] -> WHILE(body) -> post.  The resume
// variant (with_pre = false) starts the loop with the condition set.
static hk_status gm_capture(hk_plan* p, GmresGraph* g, SolveProg* sp, bool with_pre,
                            cudaGraphExec_t* out) {
  CHK(ensure_side_streams(p));
  cudaStream_t cs = p->side[0], bs = p->side[1];
  const int64_t n = p->n;
  const int s = g->s;
  const GmParams P = gm_params(p, g);
  GmState* stt = g->state.as<GmState>();
  const long long c0 = hk_launch_count();
  long long c_pre = 0, c_body = 0;
  CU(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
  auto record = [&]() -> hk_status {
    cudaStreamCaptureStatus cst;
    cudaGraph_t cg = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    CU(cudaStreamGetCaptureInfo(cs, &cst, nullptr, &cg, &deps, &nd));
    cudaGraphConditionalHandle h;
    CU(cudaGraphConditionalHandleCreate(&h, cg, with_pre ? 0u : 1u, cudaGraphCondAssignDefault));
    if (with_pre) {
      CU(cudaMemsetAsync(stt, 0, sizeof(GmState), cs));
      CU(cudaMemsetAsync(P.hess, 0, (size_t)s * P.hstride * 8, cs));
      CU(cudaMemsetAsync(P.g, 0, (size_t)s * P.vs * 8, cs));
      const double* B = g->B.as<double>();
      CU(hk_launch_norms(B, n, n, s, stt->nb, cs));
      const double* R0 = B;
      if (g->precond == 1) {
        double* xin = p->Xin.as<double>() + g->front * n * s;
        CU(cudaMemcpyAsync(xin, B, (size_t)n * s * 8, cudaMemcpyDeviceToDevice, cs));
        CHK(launch_solve_kernels(sp, s, cs, false));
        R0 = p->X2.as<double>() + g->front * n * s;
      } else if (g->precond == 2) {
        CU(hk_launch_vdiv(B, g->diag, g->W.as<double>(), n, s, cs));
        R0 = g->W.as<double>();
      }
      CU(hk_launch_norms(R0, n, n, s, stt->beta, cs));
      CU(hk_launch_gm_start(P, R0, h, cs));
      c_pre = hk_launch_count() - c0;
    }
    CU(cudaStreamGetCaptureInfo(cs, &cst, nullptr, &cg, &deps, &nd));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    CU(cudaGraphAddNode(&cnode, cg, deps, nd, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CU(cudaStreamUpdateCaptureDependencies(cs, &cnode, 1, cudaStreamSetCaptureDependencies));
    const long long cb0 = hk_launch_count();
    CU(cudaStreamBeginCaptureToGraph(bs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    const hk_status rb = gm_body_ops(p, g, sp, P, h, bs);
    cudaGraph_t tmp = nullptr;
    const cudaError_t eb = cudaStreamEndCapture(bs, &tmp);
    if (rb != HK_OK) return rb;
    CU(eb);
    c_body = hk_launch_count() - cb0;
    // post: x = Q y, true residuals (both no-ops unless the loop finished)
    CU(hk_launch_gm_combine(P, g->X.as<double>(), cs));
    CU(hk_launch_gemv_rowmajor(g->A, g->lda, n, n, g->X.as<double>(), n, s, g->W.as<double>(), n, cs));
    CU(hk_launch_gm_resid(P, g->B.as<double>(), g->W.as<double>(), cs));
    return HK_OK;
  };
  const hk_status rc = record();
  cudaGraph_t graph = nullptr;
  const cudaError_t ee = cudaStreamEndCapture(cs, &graph);
  const long long captured = hk_launch_count() - c0;
  hk_count_launch(-(int)captured);          // captured, not executed
  if (rc != HK_OK) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  CU(ee);
  const cudaError_t ei = cudaGraphInstantiate(out, graph, 0);
  cudaGraphDestroy(graph);
  CU(ei);
  g->k_pre = c_pre;
  g->k_body = c_body;
  g->k_post = captured - c_pre - c_body;
  return HK_OK;
}

// Grow the Krylov capacity of a graph to cap2 columns, keeping the first
// k+1 basis vectors, the Hessenberg columns and the rotations.
static hk_status gm_grow(hk_plan* p, GmresGraph* g, int64_t cap2, cudaStream_t st) {
  DevBuf basis, hess, cs, sn, gv, y;
  CU(gm_alloc_krylov(p, g, cap2, &basis, &hess, &cs, &sn, &gv, &y, st));
  const int64_t n = p->n, cap = g->cap, vs = cap + 1, vs2 = cap2 + 1;
  const size_t s = (size_t)g->s;
  CU(cudaMemsetAsync(hess.p, 0, s * vs2 * cap2 * 8, st));
  CU(cudaMemsetAsync(gv.p, 0, s * vs2 * 8, st));
  CU(cudaMemcpy2DAsync(basis.p, (size_t)n * vs2 * 8, g->basis.p, (size_t)n * vs * 8, (size_t)n * vs * 8,
                       s, cudaMemcpyDeviceToDevice, st));
  // Hessenberg: s * cap columns of length vs -> ld vs2, per-system stride vs2 * cap2
  for (size_t c = 0; c < s; ++c)
    CU(cudaMemcpy2DAsync(hess.as<double>() + c * vs2 * cap2, (size_t)vs2 * 8,
                         g->hess.as<double>() + c * vs * cap, (size_t)vs * 8, (size_t)vs * 8, cap,
                         cudaMemcpyDeviceToDevice, st));
  DevBuf* src[3] = {&g->cs, &g->sn, &g->g};
  DevBuf* dst[3] = {&cs, &sn, &gv};
  for (int i = 0; i < 3; ++i)
    CU(cudaMemcpy2DAsync(dst[i]->p, (size_t)vs2 * 8, src[i]->p, (size_t)vs * 8, (size_t)vs * 8, s,
                         cudaMemcpyDeviceToDevice, st));
  CU(cudaStreamSynchronize(st));
  std::swap(g->basis, basis);
  std::swap(g->hess, hess);
  std::swap(g->cs, cs);
  std::swap(g->sn, sn);
  std::swap(g->g, gv);
  std::swap(g->y, y);
  DevBuf* old[] = {&basis, &hess, &cs, &sn, &gv, &y};
  for (DevBuf* d : old) d->release();
  g->cap = cap2;
  if (g->main) cudaGraphExecDestroy(g->main);
  if (g->resume) cudaGraphExecDestroy(g->resume);
  g->main = g->resume = nullptr;
  return HK_OK;
}

static hk_status gmres_run(hk_plan* p, int64_t front, const double* A, int64_t lda, int64_t n,
                           const double* B, int64_t s, double tol, int64_t max_iter, int precond,
                           const double* diag, double* X, int64_t* iterations, double* history,
                           double* true_residual, int32_t* flags, cudaStream_t st) {
  if (!(tol > 0.0 && tol < 1.0)) return fail(HK_ERR_VALUE, "tol must lie strictly between 0 and 1");
  if (max_iter < 1) return fail(HK_ERR_VALUE, "max_iter must be >= 1");
  if (s < 1 || s > HK_GM_MAXS) return fail(HK_ERR_VALUE, "gmres takes 1..16 right-hand sides");
  if (!p) return fail(HK_ERR_VALUE, "null plan");
  if (n != p->n) return fail(HK_ERR_DIMENSION, "operator size differs from the preconditioner's");
  if (lda < n) return fail(HK_ERR_DIMENSION, "operator leading dimension smaller than n");
  if (precond < 0 || precond > 2) return fail(HK_ERR_VALUE, "precond must be 0, 1 or 2");
  if (precond == 1 && !p->factored) return fail(HK_ERR_STATE, "HODLR preconditioner not factored");
  if (precond == 1 && (front < 0 || front >= p->batch)) return fail(HK_ERR_VALUE, "front out of range");
  if (precond == 2 && !diag) return fail(HK_ERR_VALUE, "diagonal preconditioner needs its diagonal");
  if (!A || !B || !X) return fail(HK_ERR_VALUE, "null operand");
  if (hk_device_count() == 0) return fail(HK_ERR_CUDA, "no CUDA device visible");
  init_pool_once();
  const int64_t mmax = std::min<int64_t>(max_iter, n);
  SolveProg* sp = nullptr;
  if (precond == 1) {
    CHK(ensure_solve_scratch(p, (int)s, st));        // may drop cached programs and graphs
    CHK(build_solve_prog(p, (int)front, (int)s, sp, st));
  }
  GmresGraph* g = nullptr;
  for (GmresGraph* c : p->gmres_graphs)
    if (c->front == (precond == 1 ? front : 0) && c->s == s && c->precond == precond && c->A == A &&
        c->lda == lda && c->diag == (precond == 2 ? diag : nullptr) && c->tol == tol &&
        c->max_iter == max_iter) {
      g = c;
      break;
    }
  if (!g) {
    g = new GmresGraph();
    g->front = precond == 1 ? front : 0;
    g->s = (int)s;
    g->precond = precond;
    g->A = A;
    g->lda = lda;
    g->diag = precond == 2 ? diag : nullptr;
    g->tol = tol;
    g->max_iter = max_iter;
    g->mmax = mmax;
    g->cap = std::min<int64_t>(mmax, 64);
    cudaError_t e = gm_alloc_krylov(p, g, g->cap, &g->basis, &g->hess, &g->cs, &g->sn, &g->g, &g->y, st);
    const size_t ns = (size_t)n * s * 8;
    if (e == cudaSuccess) e = g->V.ensure(ns, st);
    if (e == cudaSuccess) e = g->W.ensure(ns, st);
    if (e == cudaSuccess) e = g->B.ensure(ns, st);
    if (e == cudaSuccess) e = g->X.ensure(ns, st);
    if (e == cudaSuccess) e = g->hist.ensure((size_t)s * max_iter * 8, st);
    if (e == cudaSuccess) e = g->state.ensure(sizeof(GmState), st);
    if (e != cudaSuccess) {
      cudaStreamSynchronize(st);
      destroy_gmres_graph(g);
      return fail(HK_ERR_CUDA, std::string("GMRES buffers: ") + cudaGetErrorString(e));
    }
    p->gmres_graphs.push_back(g);
  }
  if (!g->main) {
    CU(cudaStreamSynchronize(st));              // buffers allocated on st are ready for capture
    CHK(gm_capture(p, g, sp, true, &g->main));
  }
  CU(cudaMemcpyAsync(g->B.p, B, (size_t)n * s * 8, cudaMemcpyDeviceToDevice, st));
  CU(cudaGraphLaunch(g->main, st));
  // the state, the iterates and the histories in one round trip (the usual
  // case: the loop finished inside the first graph launch)
  GmState hs{};
  CU(cudaMemcpyAsync(&hs, g->state.p, sizeof(GmState), cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(X, g->X.p, (size_t)n * s * 8, cudaMemcpyDeviceToDevice, st));
  CU(cudaMemcpyAsync(history, g->hist.p, (size_t)s * max_iter * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  long long launched = g->k_pre + g->k_post + g->k_body * hs.k;
  const bool resumed = !hs.finished;
  while (!hs.finished) {                        // Krylov capacity exhausted: grow, resume
    const int64_t k0 = hs.k;
    CHK(gm_grow(p, g, std::min<int64_t>(mmax, 4 * g->cap), st));
    CHK(gm_capture(p, g, sp, false, &g->resume));
    CU(cudaGraphLaunch(g->resume, st));
    CU(cudaMemcpyAsync(&hs, g->state.p, sizeof(GmState), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    launched += g->k_post + g->k_body * (hs.k - k0);
    if (g->main) cudaGraphExecDestroy(g->main);   // recaptured at the new capacity on next use
    g->main = nullptr;
  }
  hk_count_launch((int)launched);
  if (resumed) {
    CU(cudaMemcpyAsync(X, g->X.p, (size_t)n * s * 8, cudaMemcpyDeviceToDevice, st));
    CU(cudaMemcpyAsync(history, g->hist.p, (size_t)s * max_iter * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
  }
  hk_status rc = HK_OK;
  for (int64_t c = 0; c < s; ++c) {
    iterations[c] = hs.m[c];
    flags[2 * c] = flags[2 * c + 1] = 0;
    true_residual[c] = hs.tres[c];
    if (hs.zero[c]) {                            // krylov.py:85-87
      iterations[c] = 0;
      history[c * max_iter] = 0.0;
      true_residual[c] = 0.0;
      flags[2 * c] = 1;
      continue;
    }
    if (hs.err[c]) {                             // krylov.py:91-92
      rc = fail(HK_ERR_BREAKDOWN, "preconditioned rhs is exactly zero");
      continue;
    }
    const double tr = hs.tres[c];
    bool cv = hs.conv[c] != 0;
    const bool bk = hs.brk[c] != 0;
    if (bk && tr > 10.0 * tol) {                 // krylov.py:157-159
      char msg[160];
      snprintf(msg, sizeof msg, "Arnoldi norm underflow at iteration %lld with true residual %.3e",
               (long long)(hs.m[c] + 1), tr);
      rc = fail(HK_ERR_BREAKDOWN, msg);
    }
    if (cv && tr > 10.0 * tol) cv = false;       // true-residual guard, :160-163
    if (bk) cv = true;
    flags[2 * c] = cv ? 1 : 0;
    flags[2 * c + 1] = bk ? 1 : 0;
  }
  return rc;
}

extern "C" hk_status hk_gmres(hk_plan* p, int64_t front, const double* A, int64_t lda, int64_t n,
                              const double* b, double tol, int64_t max_iter, int precond,
                              const double* diag, double* x, int64_t* iterations, double* history,
                              double* true_residual, int32_t* flags, void* stream) {
  NvtxRange nvtx_range("hk_gmres");
  return gmres_run(p, front, A, lda, n, b, 1, tol, max_iter, precond, diag, x, iterations, history,
                   true_residual, flags, (cudaStream_t)stream);
}

extern "C" hk_status hk_gmres_batch(hk_plan* p, int64_t front, const double* A, int64_t lda,
                                    int64_t n, const double* B, int64_t s, double tol,
                                    int64_t max_iter, int precond, const double* diag, double* X,
                                    int64_t* iterations, double* history, double* true_residual,
                                    int32_t* flags, void* stream) {
  NvtxRange nvtx_range("hk_gmres_batch");
  return gmres_run(p, front, A, lda, n, B, s, tol, max_iter, precond, diag, X, iterations, history,
                   true_residual, flags, (cudaStream_t)stream);
}

extern "C" hk_status hk_arnoldi_step(int64_t n, int64_t j, int64_t mmax, double* basis,
                                     double* hess, double* cs, double* sn, double* g, double* w,
                                     double beta, double* out_host, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  double* outd = nullptr;
  CU(hk_dev_malloc(&outd, 32, st));
  CU(hk_launch_arnoldi(n, j, mmax, basis, hess, cs, sn, g, w, beta, outd, st));
  CU(cudaMemcpyAsync(out_host, outd, 24, cudaMemcpyDeviceToHost, st));
  CU(hk_dev_free(outd, st));
  CU(cudaStreamSynchronize(st));
  return HK_OK;
}

// s systems' Arnoldi steps in one launch (one CTA each), device-only: the
// caller reads out_dev (3 doubles per system) once per iteration for all of
// them.  System c: basis + c*bstride (n x (mmax+1)), hess + c*hstride,
// cs/sn/g + c*(mmax+1), w + c*n, beta_dev[c]; systems with active_dev[c] == 0
// are skipped.
extern "C" hk_status hk_arnoldi_step_batch(int64_t n, int64_t j, int64_t mmax, double* basis,
                                           int64_t bstride, double* hess, int64_t hstride,
                                           double* cs, double* sn, double* g, double* w,
                                           const double* beta_dev, double* out_dev,
                                           const int32_t* active_dev, int64_t s, void* stream) {
  if (s < 1 || s > 1024) return fail(HK_ERR_VALUE, "1..1024 systems");
  if (j < 0 || j >= mmax) return fail(HK_ERR_VALUE, "column index out of range");
  CU(hk_launch_arnoldi_batch(n, j, mmax, basis, bstride, hess, hstride, cs, sn, g, w, beta_dev,
                             out_dev, active_dev, (int)s, (cudaStream_t)stream));
  return HK_OK;
}

extern "C" hk_status hk_gmres_combine(int64_t n, int64_t m, int64_t mmax, const double* basis,
                                      const double* hess, const double* g, double* x, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  double* y = nullptr;
  CU(hk_dev_malloc(&y, (size_t)(m + 1) * 8, st));
  CU(hk_launch_combine(n, m, mmax, basis, hess, g, x, y, st));
  CU(hk_dev_free(y, st));
  return HK_OK;
}

// ------------------------------------------------------------------ dense entry points
extern "C" hk_status hk_copy_h2d_streaming(const void* src_host, void* dst_dev, int64_t bytes,
                                           int ctas, void* stream) {
  if (bytes < 0 || ctas < 1) return fail(HK_ERR_VALUE, "bad copy size or CTA count");
  if ((reinterpret_cast<uintptr_t>(src_host) | reinterpret_cast<uintptr_t>(dst_dev)) & 15)
    return fail(HK_ERR_VALUE, "copy buffers must be 16-byte aligned");
  CU(hk_launch_h2d_stream(src_host, dst_dev, bytes, ctas, (cudaStream_t)stream));
  return HK_OK;
}

extern "C" hk_status hk_gemv(const double* A, int64_t lda, int64_t m, int64_t n, const double* x,
                             int64_t ldx, int64_t s, double* y, int64_t ldy, void* stream) {
  if (hk_device_count() == 0) return fail(HK_ERR_CUDA, "no CUDA device visible");
  CU(hk_launch_gemv_rowmajor(A, lda, m, n, x, ldx, s, y, ldy, (cudaStream_t)stream));
  return HK_OK;
}

extern "C" hk_status hk_lu_full(double* a, int64_t m, int64_t n, int64_t ld, int64_t* rp,
                                int64_t* cp, double* piv, int64_t* npiv, void* stream) {
  if (hk_device_count() == 0) return fail(HK_ERR_CUDA, "no CUDA device visible");
  cudaStream_t st = (cudaStream_t)stream;
  int64_t* d = nullptr;
  CU(hk_dev_malloc(&d, 8, st));
  CU(hk_launch_lu_full(a, m, n, ld, rp, cp, piv, d, st));
  CU(cudaMemcpyAsync(npiv, d, 8, cudaMemcpyDeviceToHost, st));
  CU(hk_dev_free(d, st));
  CU(cudaStreamSynchronize(st));
  return HK_OK;
}

extern "C" hk_status hk_lu_partial(double* a, int64_t n, int64_t ld, int32_t* perm, double* inv,
                                   void* stream) {
  if (hk_device_count() == 0) return fail(HK_ERR_CUDA, "no CUDA device visible");
  if (n == 0) return HK_OK;
  if (ld != n) return fail(HK_ERR_VALUE, "lu_partial needs a contiguous matrix");
  cudaStream_t st = (cudaStream_t)stream;
  double *lu = nullptr, *iv = nullptr;
  int32_t *ip = nullptr, *stt = nullptr;
  CU(hk_dev_malloc(&lu, (size_t)n * n * 8, st));
  CU(hk_dev_malloc(&iv, (size_t)n * n * 8, st));
  CU(hk_dev_malloc(&ip, (size_t)n * 4 + 4, st));
  CU(hk_dev_malloc(&stt, 8, st));
  LuTask t{};
  t.src = a; t.src_ld = ld; t.lu = lu; t.inv = inv ? iv : nullptr;
  t.perm = ip; t.ipiv = perm; t.status = stt; t.N = (int)n; t.mode = 0;
  LuTask* td = nullptr;
  CU(hk_dev_malloc(&td, sizeof(LuTask), st));
  CU(cudaMemcpyAsync(td, &t, sizeof(LuTask), cudaMemcpyHostToDevice, st));
  CU(hk_launch_lu(td, 1, (int)n, st));
  // column-major results -> row-major outputs
  CU(hk_launch_transpose(lu, a, n, n, 1, 0, st));
  if (inv) CU(hk_launch_transpose(iv, inv, n, n, 1, 0, st));
  int32_t sing = 0;
  CU(cudaMemcpyAsync(&sing, stt, 4, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  hk_dev_free(lu, st); hk_dev_free(iv, st); hk_dev_free(ip, st);
  hk_dev_free(stt, st); hk_dev_free(td, st);
  if (sing) return fail(HK_ERR_SINGULAR, "pivot magnitude below 1e-300");
  return HK_OK;
}

// Batched explicit inverses by the factor's Gauss-Jordan kernels (the
// capacitance-matrix path of hodlr.py:273; implicit partial pivoting, so the
// singularity test is dense.py:76-77's).  A: `batch` row-major n x n matrices
// (leading dimension lda, matrix stride `stride` elements); out: column-major
// inverses (leading dimension n, stride n*n).  status_host[b] = 1 if matrix b
// is singular.
extern "C" hk_status hk_gj_inverse(const double* A, int64_t n, int64_t lda, int64_t batch,
                                   int64_t stride, double* out, int32_t* status_host,
                                   void* stream) {
  if (hk_device_count() == 0) return fail(HK_ERR_CUDA, "no CUDA device visible");
  if (n < 0 || batch < 0 || lda < n) return fail(HK_ERR_VALUE, "bad gj_inverse dimensions");
  if (n == 0 || batch == 0) return HK_OK;
  if (n > INT32_MAX) return fail(HK_ERR_VALUE, "gj_inverse matrix too large");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t scr = hk_gj_scratch_bytes((int)n);
  char* scratch = nullptr;
  int32_t* stt = nullptr;
  GjTask* td = nullptr;
  if (scr) CU(hk_dev_malloc((void**)&scratch, scr * (size_t)batch, st));
  CU(hk_dev_malloc((void**)&stt, (size_t)batch * 4, st));
  std::vector<GjTask> tasks((size_t)batch);
  for (int64_t b = 0; b < batch; ++b) {
    GjTask& t = tasks[(size_t)b];
    t.src = A + b * stride;
    t.src_ld = lda;
    t.out = out + b * n * n;
    t.out_ld = n;
    t.scratch = scr ? reinterpret_cast<double*>(scratch + scr * (size_t)b) : nullptr;
    t.status = stt + b;
    t.N = (int32_t)n;
    t.mode = 0;
  }
  CU(hk_dev_malloc((void**)&td, sizeof(GjTask) * tasks.size(), st));
  CU(cudaMemcpyAsync(td, tasks.data(), sizeof(GjTask) * tasks.size(), cudaMemcpyHostToDevice, st));
  CU(hk_launch_gj(td, (int)batch, (int)n, st));
  CU(cudaMemcpyAsync(status_host, stt, (size_t)batch * 4, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  hk_dev_free(td, st);
  hk_dev_free(stt, st);
  if (scratch) hk_dev_free(scratch, st);
  return HK_OK;
}

// In-place inverses of `batch` symmetric positive definite n x n matrices
// (column-major view, leading dimension lda, matrix stride `stride`) by block
// Gauss-Jordan with 64 x 64 pivot blocks (128 for n > 2048): per block k, P = A_kk^{-1}
// (Gauss-Jordan kernel, partial pivoting inside the block), R = P A_k*,
// A_ij -= A_ik R_kj (DMMA GEMM, the 2 n^2 b flops of the step), A_ik = -A_ik P,
// A_kj = R_kj, A_kk = P -- every front of the batch in the same launches.
// No pivoting across blocks: the fronts' plane Schur complements are SPD.
// Used by frontgen's plane-by-plane elimination (the step before the path,
// SURVEY.md §8(f)#1).  status_host[b] = 1 if a pivot block of matrix b was
// singular.  A row-major matrix is the transpose of its column-major view, and
// (A^T)^{-1} = (A^{-1})^T, so row-major input works unchanged.
extern "C" hk_status hk_spd_inverse(double* A, int64_t n, int64_t lda, int64_t batch,
                                    int64_t stride, int32_t* status_host, void* stream) {
  NvtxRange nvtx_range("hk_spd_inverse");
  if (hk_device_count() == 0) return fail(HK_ERR_CUDA, "no CUDA device visible");
  if (n < 0 || batch < 0 || lda < n) return fail(HK_ERR_VALUE, "bad spd_inverse dimensions");
  if (n == 0 || batch == 0) return HK_OK;
  if (n > INT32_MAX / 2) return fail(HK_ERR_VALUE, "spd_inverse matrix too large");
  if (batch > 1 && stride < lda * n) return fail(HK_ERR_DIMENSION, "matrix stride too small");
  cudaStream_t st = (cudaStream_t)stream;
  // pivot blocks of 64 (128 above n = 2048: the trailing GEMMs' K doubles,
  // which lifts the DMMA kernel from ~10 to ~20 TFLOP/s; the register-resident
  // Gauss-Jordan still takes 128 x 128)
  const int64_t NB = n > 2048 ? 128 : 64;
  const int64_t per = NB * NB + 2 * NB * n;             // P, R (NB x n), Cc (n x NB)
  double* scr = nullptr;
  int32_t* stt = nullptr;
  CU(hk_dev_malloc((void**)&scr, (size_t)batch * per * 8, st));
  const int64_t nsteps = (n + NB - 1) / NB;   // one status per (front, pivot block)
  CU(hk_dev_malloc((void**)&stt, (size_t)batch * nsteps * 4, st));
  CU(cudaMemsetAsync(stt, 0, (size_t)batch * nsteps * 4, st));
  // task arrays of every block step of one call, in one pinned arena (the call
  // synchronises at the end, before a later call may rewrite it)
  static Staging stage;
  stage.reset();
  std::vector<Op> ops;
  hk_status rc = HK_OK;
  for (int64_t k0 = 0; k0 < n && rc == HK_OK; k0 += NB) {
    const int64_t k1 = std::min(n, k0 + NB), b = k1 - k0;
    std::vector<GjTask> gts;
    TileList trc, tup;
    std::vector<CopyTask> cps;
    for (int64_t f = 0; f < batch; ++f) {
      double* Af = A + f * stride;
      double* P = scr + f * per;
      double* R = P + NB * NB;            // b x n, ld NB
      double* Cc = R + NB * n;            // n x b, ld n
      GjTask g{};
      g.src = Af + k0 + k0 * lda; g.src_ld = lda; g.mode = 1;
      g.out = P; g.out_ld = NB; g.status = stt + f * nsteps + k0 / NB; g.N = (int32_t)b;
      gts.push_back(g);
      // R = P A[k, :];  Cc = -A[:, k] P   (both read the pre-step A)
      trc.add(gemm(P, NB, 0, Af + k0, lda, R, NB, (int)b, (int)n, (int)b, 1.0, 0.0));
      trc.add(gemm(Af + k0 * lda, lda, 0, P, NB, Cc, n, (int)n, (int)b, (int)b, -1.0, 0.0));
      // A_ij -= A_ik R_kj for i, j outside block k
      const int64_t rr[2][2] = {{0, k0}, {k1, n}};
      for (auto& ri : rr)
        for (auto& cj : rr) {
          const int64_t mi = ri[1] - ri[0], nj = cj[1] - cj[0];
          if (mi <= 0 || nj <= 0) continue;
          tup.add(gemm(Af + k0 * lda + ri[0], lda, 0, R + cj[0] * NB, NB, Af + ri[0] + cj[0] * lda,
                       lda, (int)mi, (int)nj, (int)b, -1.0, 1.0));
        }
      // write back: column block (rows outside k) <- Cc, row block <- R, A_kk <- P
      for (auto& ri : rr) {
        if (ri[1] <= ri[0]) continue;
        CopyTask c{};
        c.src = Cc + ri[0]; c.src_rs = 1; c.src_cs = n;
        c.dst = Af + ri[0] + k0 * lda; c.dst_rs = 1; c.dst_cs = lda;
        c.rows = (int)(ri[1] - ri[0]); c.cols = (int)b;
        cps.push_back(c);
        CopyTask d{};
        d.src = R + ri[0] * NB; d.src_rs = 1; d.src_cs = NB;
        d.dst = Af + k0 + ri[0] * lda; d.dst_rs = 1; d.dst_cs = lda;
        d.rows = (int)b; d.cols = (int)(ri[1] - ri[0]);
        cps.push_back(d);
      }
      CopyTask e{};
      e.src = P; e.src_rs = 1; e.src_cs = NB;
      e.dst = Af + k0 + k0 * lda; e.dst_rs = 1; e.dst_cs = lda;
      e.rows = (int)b; e.cols = (int)b;
      cps.push_back(e);
    }
    // the GJ tasks read A_kk; the copies rewrite it last
    {
      Op o{Op::GJ};
      o.a = stage.push(gts, st);
      o.n = (int)gts.size();
      o.maxN = (int)b;
      if (!o.a) { rc = fail(HK_ERR_CUDA, "pinned staging allocation failed"); break; }
      ops.push_back(o);
    }
    for (TileList* tl : {&trc, &tup}) {
      if (tl->ntiles() == 0) continue;
      Op o{Op::GEMM};
      o.a = stage.push(tl->tasks, st);
      o.map = stage.push(tl->map, st);
      o.n = tl->ntiles();
      if (!o.a || !o.map) { rc = fail(HK_ERR_CUDA, "pinned staging allocation failed"); break; }
      ops.push_back(o);
    }
    if (rc != HK_OK) break;
    Op o{Op::COPY};
    o.a = stage.push(cps, st);
    o.n = (int)cps.size();
    if (!o.a) { rc = fail(HK_ERR_CUDA, "pinned staging allocation failed"); break; }
    ops.push_back(o);
    if (stage.commit(st) != cudaSuccess) { rc = fail(HK_ERR_CUDA, "staging commit failed"); break; }
    for (const Op& op : ops) {
      cudaError_t e = cudaSuccess;
      switch (op.kind) {
        case Op::GJ: e = hk_launch_gj((const GjTask*)op.a, op.n, op.maxN, st); break;
        case Op::GEMM: e = hk_launch_gemm((const GemmTask*)op.a, op.map, op.n, st); break;
        case Op::COPY: e = hk_launch_copy((const CopyTask*)op.a, op.n, st); break;
        default: break;
      }
      if (e != cudaSuccess) { rc = fail(HK_ERR_CUDA, cudaGetErrorString(e)); break; }
    }
    ops.clear();
  }
  std::vector<int32_t> sh((size_t)batch * nsteps, 0);
  if (rc == HK_OK)
    CU(cudaMemcpyAsync(sh.data(), stt, sh.size() * 4, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  for (int64_t f = 0; f < batch; ++f) {
    int32_t any = 0;
    for (int64_t k = 0; k < nsteps; ++k) any |= sh[(size_t)(f * nsteps + k)];
    status_host[f] = any ? 1 : 0;
  }
  hk_dev_free(scr, st);
  hk_dev_free(stt, st);
  return rc;
}

extern "C" hk_status hk_aca_block(const double* a, int64_t m, int64_t n, int64_t ld, double tol2,
                                  int64_t cap, double* U, double* V, int64_t* rank,
                                  int32_t* trows, int64_t* nrows, int32_t* tcols, int64_t* ncols,
                                  void* stream) {
  if (hk_device_count() == 0) return fail(HK_ERR_CUDA, "no CUDA device visible");
  cudaStream_t st = (cudaStream_t)stream;
  if (m == 0 || n == 0 || cap == 0) {
    *rank = 0;
    if (nrows) *nrows = 0;
    if (ncols) *ncols = 0;
    return HK_OK;
  }
  if ((size_t)(cap + 16) * 8 + m + 1024 > 200 * 1024) return fail(HK_ERR_VALUE, "block too large for the ACA kernel");
  // square zero-padded copy of the block and its transpose, both ld = sq
  const int64_t sq = std::max(m, n);
  const int64_t tlen = 2 + (m + cap + 1) + (cap + 1);
  double *sqbuf = nullptr, *at = nullptr;
  int32_t *rk = nullptr, *tr = nullptr;
  CU(hk_dev_malloc(&sqbuf, (size_t)sq * sq * 8, st));
  CU(hk_dev_malloc(&at, (size_t)sq * sq * 8, st));
  CU(hk_dev_malloc(&rk, 8, st));
  CU(hk_dev_malloc(&tr, (size_t)tlen * 4, st));
  CU(cudaMemsetAsync(sqbuf, 0, (size_t)sq * sq * 8, st));
  CU(cudaMemcpy2DAsync(sqbuf, sq * 8, a, ld * 8, n * 8, m, cudaMemcpyDeviceToDevice, st));
  CU(hk_launch_transpose(sqbuf, at, sq, sq, 1, 0, st));
  double* scr = nullptr;
  {
    const int P = hk_aca_cluster_size((int)std::max(m, n), (int)std::max(m, n));
    const size_t sd = P > 1 ? hk_aca_scratch_doubles_cl((int)cap, P) : hk_aca_scratch_doubles((int)cap);
    CU(hk_dev_malloc(&scr, sd * 8, st));
  }
  int lmu = 6;
  while ((1 << lmu) < std::max(m, n)) ++lmu;
  const int lmv = lmu;
  if (lmu > 13 || lmv > 13) return fail(HK_ERR_VALUE, "block too large for the ACA kernel (max 8192 rows)");
  double *Ur = nullptr, *Vr = nullptr;
  CU(hk_dev_malloc(&Ur, ((size_t)1 << lmu) * (cap + 8) * 8, st));
  CU(hk_dev_malloc(&Vr, ((size_t)1 << lmv) * (cap + 8) * 8, st));
  AcaTask t{};
  t.scratch = scr;
  t.A = sqbuf;
  t.At = at;
  t.lda = sq;
  t.U = Ur;
  t.V = Vr;
  t.ldu = lmu;
  t.ldv = lmv;
  t.rank = rk;
  t.trace = tr;
  t.m = (int)m;
  t.n = (int)n;
  t.cap = (int)cap;
  AcaTask* td = nullptr;
  CU(hk_dev_malloc(&td, sizeof(AcaTask), st));
  CU(cudaMemcpyAsync(td, &t, sizeof(AcaTask), cudaMemcpyHostToDevice, st));
  CU(hk_launch_aca(td, 1, (int)cap, (int)m, tol2, st, (int)std::max(m, n)));
  std::vector<int32_t> h(tlen);
  int32_t r32 = 0;
  CU(cudaMemcpyAsync(&r32, rk, 4, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(h.data(), tr, tlen * 4, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (r32 > 0) {   // row-major working factors -> the caller's column-major buffers
    std::vector<CopyTask> ct(2);
    ct[0] = CopyTask{Ur, U, 1, (int64_t)1 << lmu, 1, m, (int32_t)m, r32};
    ct[1] = CopyTask{Vr, V, 1, (int64_t)1 << lmv, 1, n, (int32_t)n, r32};
    CopyTask* ctd = nullptr;
    CU(hk_dev_malloc(&ctd, sizeof(CopyTask) * 2, st));
    CU(cudaMemcpyAsync(ctd, ct.data(), sizeof(CopyTask) * 2, cudaMemcpyHostToDevice, st));
    CU(hk_launch_copy(ctd, 2, st));
    CU(cudaStreamSynchronize(st));
    hk_dev_free(ctd, st);
  }
  hk_dev_free(Ur, st);
  hk_dev_free(Vr, st);
  *rank = r32;
  if (nrows) *nrows = h[0];
  if (ncols) *ncols = h[1];
  if (trows) std::memcpy(trows, h.data() + 2, (size_t)h[0] * 4);
  if (tcols) std::memcpy(tcols, h.data() + 2 + (m + cap + 1), (size_t)h[1] * 4);
  hk_dev_free(at, st); hk_dev_free(rk, st); hk_dev_free(tr, st);
  hk_dev_free(sqbuf, st); hk_dev_free(td, st); hk_dev_free(scr, st);
  return HK_OK;
}

extern "C" hk_status hk_skeleton_block(const double* a, int64_t m, int64_t n, int64_t ld,
                                       const int64_t* rsel, int64_t k, const int64_t* csel,
                                       int64_t kc, double tol, int64_t cap, double* U, double* V,
                                       int64_t* rank, int64_t* rows_out, int64_t* cols_out,
                                       void* stream) {
  if (hk_device_count() == 0) return fail(HK_ERR_CUDA, "no CUDA device visible");
  cudaStream_t st = (cudaStream_t)stream;
  *rank = 0;
  if (k == 0 || kc == 0 || m == 0 || n == 0) return HK_OK;
  std::vector<int64_t> sel(rsel, rsel + k);
  sel.insert(sel.end(), csel, csel + kc);
  auto pr = probe_rows(m);
  sel.insert(sel.end(), pr.begin(), pr.end());
  int64_t *seld = nullptr, *perm = nullptr;
  double* work = nullptr;
  int32_t* small = nullptr;  // [rank, status]
  CU(hk_dev_malloc(&seld, sel.size() * 8, st));
  CU(hk_dev_malloc(&perm, (size_t)(k + kc) * 8, st));
  CU(hk_dev_malloc(&work, (size_t)k * kc * 8, st));
  CU(hk_dev_malloc(&small, 8, st));
  CU(cudaMemcpyAsync(seld, sel.data(), sel.size() * 8, cudaMemcpyHostToDevice, st));
  SkelTask t{};
  t.A = a; t.lda = ld;
  t.rsel = seld; t.csel = seld + k;
  t.work = work; t.rperm = perm; t.cperm = perm + k;
  t.U = U; t.V = V; t.ldu = (int32_t)m; t.ldv = (int32_t)n;
  t.rank = small; t.status = small + 1;
  t.probe = seld + k + kc; t.nprobe = (int32_t)pr.size();
  t.m = (int)m; t.n = (int)n; t.k = (int)k; t.kc = (int)kc; t.cap = (int)cap; t.tol = tol;
  SkelTask* td = nullptr;
  CU(hk_dev_malloc(&td, sizeof(SkelTask), st));
  CU(cudaMemcpyAsync(td, &t, sizeof(SkelTask), cudaMemcpyHostToDevice, st));
  CU(hk_launch_skeleton(td, 1, (int)k, (int)kc, (int)m, (int)n, st));
  int32_t hs[2] = {0, 0};
  std::vector<int64_t> ph((size_t)(k + kc));
  CU(cudaMemcpyAsync(hs, small, 8, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(ph.data(), perm, ph.size() * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  hk_dev_free(seld, st); hk_dev_free(perm, st); hk_dev_free(work, st);
  hk_dev_free(small, st); hk_dev_free(td, st);
  *rank = hs[0];
  for (int64_t i = 0; i < hs[0]; ++i) {
    if (rows_out) rows_out[i] = rsel[ph[i]];
    if (cols_out) cols_out[i] = csel[ph[k + i]];
  }
  if (hs[1] == HK_ERR_DEGENERATE)
    return fail(HK_ERR_DEGENERATE, "skeleton rank 0 but sampled block magnitude exceeds the "
                                   "tolerance; selection depth is too small");
  return HK_OK;
}

// ------------------------------------------------------------------ graph
extern "C" hk_status hk_graph_distance(int64_t nverts, const int64_t* indptr, const int64_t* indices,
                                       const int64_t* own, int64_t n_own, const int64_t* other,
                                       int64_t n_other, int64_t* dist_out) {
  std::vector<int64_t> d;
  hk::side_distance(nverts, indptr, indices, own, n_own, other, n_other, d);
  std::memcpy(dist_out, d.data(), d.size() * 8);
  return HK_OK;
}

extern "C" hk_status hk_select_by_depth(int64_t nverts, const int64_t* indptr,
                                        const int64_t* indices, const int64_t* row_verts,
                                        int64_t n_rows, const int64_t* col_verts, int64_t n_cols,
                                        int32_t depth, int64_t* row_sel, int64_t* n_row_sel,
                                        int64_t* col_sel, int64_t* n_col_sel) {
  if (depth < 0) return fail(HK_ERR_VALUE, "depth must be >= 0");
  std::vector<int64_t> rs, cs;
  bool ok = hk::select_by_depth(nverts, indptr, indices, row_verts, n_rows, col_verts, n_cols,
                                depth, rs, cs);
  *n_row_sel = (int64_t)rs.size();
  *n_col_sel = (int64_t)cs.size();
  std::memcpy(row_sel, rs.data(), rs.size() * 8);
  std::memcpy(col_sel, cs.data(), cs.size() * 8);
  if (!ok) return fail(HK_ERR_EMPTY_SELECTION, "no vertices within requested depth of the boundary");
  return HK_OK;
}
