// Task-extent validation (HK_VALIDATE=1): the memcheck substitute for this
// library's own kernels.  compute-sanitizer is closed on the GPU pool, so
// instead every task array a kernel will read is checked on the host when it
// is staged (Staging::push in api.cpp): each matrix region a task touches --
// from its pointer, leading dimension and extents, exactly as the kernel
// indexes it -- must lie inside ONE device allocation.  The allocation of a
// pointer comes from the driver (cuMemGetAddressRange, fetched through
// cudaGetDriverEntryPoint so the library still needs no libcuda at link
// time).  In validation mode the library's own buffers are plain cudaMalloc
// allocations (hk_dev_malloc), so their ranges are exact; torch tensors are
// exact with PYTORCH_NO_CUDA_MEMORY_CACHING=1 (the caching allocator would
// otherwise report a whole cached segment).  Violations are printed to
// stderr and counted (hk_debug_violations).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>

#include "../../include/hodlr_b200.h"
#include "hk_internal.h"

namespace {

std::atomic<long long> g_viol{0};
std::atomic<long long> g_checked{0};

typedef int (*GetRangeFn)(unsigned long long* base, size_t* size, unsigned long long ptr);

GetRangeFn range_fn() {
  static GetRangeFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<GetRangeFn>(p);
  }
  return fn;
}

// [p, p + bytes) inside one allocation?
void check_region(const char* what, const void* p, long long bytes) {
  if (bytes <= 0 || p == nullptr) return;
  g_checked.fetch_add(1);
  GetRangeFn fn = range_fn();
  if (!fn) return;
  unsigned long long base = 0;
  size_t size = 0;
  const int rc = fn(&base, &size, (unsigned long long)p);
  const unsigned long long lo = (unsigned long long)p, hi = lo + (unsigned long long)bytes;
  if (rc != 0 || hi > base + size) {
    const long long n = g_viol.fetch_add(1);
    if (n < 20)
      fprintf(stderr,
              "[hk validate] %s: region [%p, +%lld B) %s allocation [0x%llx, +%zu B)\n", what, p,
              bytes, rc ? "outside any" : "overruns its", base, size);
  }
}

// column-major rows x cols with leading dimension ld (elements)
long long cm_bytes(long long rows, long long cols, long long ld, long long esz = 8) {
  if (rows <= 0 || cols <= 0) return 0;
  return ((cols - 1) * ld + rows) * esz;
}

}  // namespace

bool hk_validate_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HK_VALIDATE");
    v = e ? atoi(e) : 0;
  }
  return v != 0;
}

cudaError_t hk_dev_malloc_raw(void** p, size_t bytes, cudaStream_t st) {
  if (hk_validate_enabled()) return cudaMalloc(p, bytes);
  return cudaMallocAsync(p, bytes, st);
}

cudaError_t hk_dev_free(void* p, cudaStream_t st) {
  if (!p) return cudaSuccess;
  if (hk_validate_enabled()) {
    cudaStreamSynchronize(st);
    return cudaFree(p);
  }
  return cudaFreeAsync(p, st);
}

void hk_validate(const GemmTask& t) {
  const long long ar = t.transA ? t.k : t.m, ac = t.transA ? t.m : t.k;
  check_region("gemm A", t.A, cm_bytes(ar, ac, t.lda));
  check_region("gemm B", t.B, cm_bytes(t.k, t.n, t.ldb));
  check_region("gemm C", t.C, cm_bytes(t.m, t.n, t.ldc));
}

void hk_validate(const CopyTask& t) {
  if (t.rows <= 0 || t.cols <= 0) return;
  check_region("copy src", t.src,
               ((long long)(t.rows - 1) * t.src_rs + (long long)(t.cols - 1) * t.src_cs + 1) * 8);
  check_region("copy dst", t.dst,
               ((long long)(t.rows - 1) * t.dst_rs + (long long)(t.cols - 1) * t.dst_cs + 1) * 8);
}

void hk_validate(const AcaTask& t) {
  // row i of the block: A[i*lda + j]; column j (transposed copy): At[j*lda + i]
  check_region("aca A", t.A, cm_bytes(t.n, t.m, t.lda));
  if (t.At) check_region("aca At", t.At, cm_bytes(t.m, t.n, t.lda));
  const long long ldu = 1ll << t.ldu, ldv = 1ll << t.ldv;
  check_region("aca U", t.U, cm_bytes(ldu, t.cap + 8, ldu));   // + the 8 prefetch slack columns
  check_region("aca V", t.V, cm_bytes(ldv, t.cap + 8, ldv));
  check_region("aca rank", t.rank, 4);
}

void hk_validate(const SkelTask& t) {
  check_region("skel rsel", t.rsel, (long long)t.k * 8);
  check_region("skel csel", t.csel, (long long)t.kc * 8);
  check_region("skel work", t.work, (long long)t.k * t.kc * 8);
  check_region("skel U", t.U, cm_bytes(t.m, t.cap, t.ldu));
  check_region("skel V", t.V, cm_bytes(t.n, t.cap, t.ldv));
}

void hk_validate(const GjTask& t) {
  check_region("gj src", t.src, cm_bytes(t.N, t.N, t.src_ld));
  check_region("gj out", t.out, cm_bytes(t.N, t.N, t.out_ld));
  check_region("gj status", t.status, 4);
}

void hk_validate(const LuTask& t) {
  if (t.mode == 0) check_region("lu src", t.src, cm_bytes(t.N, t.N, t.src_ld));
  check_region("lu lu", t.lu, (long long)t.N * t.N * 8);
  if (t.inv) check_region("lu inv", t.inv, (long long)t.N * t.N * 8);
}

void hk_validate(const PdotTask& t) {
  check_region("pdot M", t.M, cm_bytes(t.rows, t.cols, t.ldm));
  check_region("pdot x", t.x, (long long)t.rows * 8);
  const long long nch = (t.rows + HK_PDOT_ROWS - 1) / HK_PDOT_ROWS;
  check_region("pdot P", t.P, nch * t.cols * 8);
}

void hk_validate(const SgemvTask& t) {
  check_region("sgemv M", t.M, cm_bytes(t.rows, t.K, t.ldm));
  if (t.v0) check_region("sgemv v", t.v0, (long long)t.K * 8);
  if (t.PA) check_region("sgemv PA", t.PA, (long long)t.nchA * t.KA * 8);
  if (t.PB) check_region("sgemv PB", t.PB, (long long)t.nchB * (t.K - t.KA) * 8);
  check_region("sgemv y", t.y, (long long)t.rows * 8);
}

void hk_validate(const MatVecTask& t) {
  check_region("matvec M", t.M, cm_bytes(t.rows, t.K, t.ldm));
  check_region("matvec x", t.x, (long long)t.K * 8);
  check_region("matvec y", t.y, (long long)t.rows * 8);
}

void hk_validate(const DotTask& t) {
  check_region("dot M", t.M, cm_bytes(t.rows, t.cols, t.ldm));
  check_region("dot x", t.x, (long long)t.rows * 8);
}

void hk_validate(const SelTask& t) {
  check_region("select out", t.out, (long long)t.n_own * 8);
  check_region("select count", t.count, 4);
}

extern "C" int64_t hk_debug_violations(int64_t* checked) {
  if (checked) *checked = g_checked.load();
  return g_viol.load();
}
