// Device-resident GMRES pieces (src/krylov.py:69-166): the Arnoldi column with
// modified Gram-Schmidt (+ one conditional re-orthogonalisation pass), the
// Givens update and the convergence scalars in one single-CTA kernel, so the
// host reads back three doubles per iteration and nothing else.
#include "hk_common.cuh"
#include "hk_internal.h"

namespace {

constexpr int KR_NT = 1024;

__device__ double block_dot(const double* a, const double* b, int64_t n, double* red) {
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += KR_NT) s += a[i] * b[i];
  return block_sum<KR_NT>(s, red);
}

// w -= h * q  (own elements only; no sync needed between calls on the same w)
__device__ void block_axpy(double* w, const double* q, double h, int64_t n) {
  for (int64_t i = threadIdx.x; i < n; i += KR_NT) w[i] -= h * q[i];
}

__device__ __forceinline__ void arnoldi_body(int64_t n, int64_t j, int64_t mmax, double* basis,
                                             double* hess, double* cs, double* sn, double* g,
                                             double* w, double beta, double* out, double* vout) {
  __shared__ double red[KR_NT / 32];
  const int64_t k = j + 1;
  const int64_t ldh = mmax + 1;
  double* hcol = hess + j * ldh;
  const double norm_in = sqrt(block_dot(w, w, n, red));
  for (int64_t i = 0; i < k; ++i) {                 // MGS, krylov.py:111-114
    const double* q = basis + i * n;
    const double h = block_dot(q, w, n, red);
    if (threadIdx.x == 0) hcol[i] = h;
    block_axpy(w, q, h, n);
    __syncthreads();
  }
  double nw = sqrt(block_dot(w, w, n, red));
  if (nw < norm_in / sqrt(2.0)) {                   // re-orthogonalise, :115-119
    for (int64_t i = 0; i < k; ++i) {
      const double* q = basis + i * n;
      const double e = block_dot(q, w, n, red);
      if (threadIdx.x == 0) hcol[i] += e;
      block_axpy(w, q, e, n);
      __syncthreads();
    }
    nw = sqrt(block_dot(w, w, n, red));
  }
  const double hk = nw;
  const bool happy = hk <= 1e-14 * fmax(norm_in, 1e-300);   // :122
  if (!happy) {
    double* qn = basis + k * n;
    for (int64_t i = threadIdx.x; i < n; i += KR_NT) {
      const double q = w[i] / hk;
      qn[i] = q;
      if (vout) vout[i] = q;
    }
  }
  if (threadIdx.x == 0) {
    hcol[k] = hk;
    for (int64_t i = 0; i < j; ++i) {               // apply previous rotations, :126-129
      const double temp = cs[i] * hcol[i] + sn[i] * hcol[i + 1];
      hcol[i + 1] = -sn[i] * hcol[i] + cs[i] * hcol[i + 1];
      hcol[i] = temp;
    }
    const double denom = hypot(hcol[j], hcol[k]);
    double brk = 0.0, rel = 0.0;
    if (denom == 0.0) {
      brk = 1.0;
    } else {
      cs[j] = hcol[j] / denom;
      sn[j] = hcol[k] / denom;
      hcol[j] = denom;
      hcol[k] = 0.0;
      g[k] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      rel = fabs(g[k]) / beta;
    }
    out[0] = rel;
    out[1] = happy ? 1.0 : 0.0;
    out[2] = brk;
  }
}

// Register-resident variant for n <= WPT * KR_NT (every config): the new
// vector w lives in registers (WPT entries per thread), so an MGS step is one
// pass over q_i with the dot and the update fused, and every block reduction
// takes one barrier (double-buffered SMEM partials reduced by every warp in a
// fixed order).  Same algorithm and step order as arnoldi_body.
template <int WPT>
__device__ __forceinline__ void arnoldi_body_reg(int64_t n, int64_t j, int64_t mmax, double* basis,
                                                 double* hess, double* cs, double* sn, double* g,
                                                 double* w, double beta, double* out, double* vout) {
  constexpr int NW = KR_NT / 32;
  __shared__ double red[2][NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int par = 0;
  auto bsum = [&](double v) -> double {
    v = warp_sum(v);
    if (lane == 0) red[par][warp] = v;
    __syncthreads();
    double t = lane < NW ? red[par][lane] : 0.0;
    t = warp_sum(t);
    par ^= 1;
    return __shfl_sync(0xffffffffu, t, 0);
  };
  const int64_t k = j + 1;
  const int64_t ldh = mmax + 1;
  double* hcol = hess + j * ldh;
  double wr[WPT];
#pragma unroll
  for (int q = 0; q < WPT; ++q) {
    const int64_t i = tid + (int64_t)q * KR_NT;
    wr[q] = i < n ? w[i] : 0.0;
  }
  auto sumsq = [&]() {
    double a = 0.0;
#pragma unroll
    for (int q = 0; q < WPT; ++q) a += wr[q] * wr[q];
    return a;
  };
  auto mgs_pass = [&](bool add) {
    for (int64_t i = 0; i < k; ++i) {             // MGS, krylov.py:111-114 (:115-119)
      const double* qv = basis + i * n;
      double d = 0.0;
#pragma unroll
      for (int q = 0; q < WPT; ++q) {
        const int64_t e = tid + (int64_t)q * KR_NT;
        d += (e < n ? qv[e] : 0.0) * wr[q];
      }
      const double h = bsum(d);
      if (tid == 0) hcol[i] = add ? hcol[i] + h : h;
#pragma unroll
      for (int q = 0; q < WPT; ++q) {             // q_i again, from L1
        const int64_t e = tid + (int64_t)q * KR_NT;
        wr[q] -= h * (e < n ? qv[e] : 0.0);
      }
    }
  };
  const double norm_in = sqrt(bsum(sumsq()));
  mgs_pass(false);
  double nw = sqrt(bsum(sumsq()));
  if (nw < norm_in / sqrt(2.0)) {                 // re-orthogonalise
    mgs_pass(true);
    nw = sqrt(bsum(sumsq()));
  }
  const double hk = nw;
  const bool happy = hk <= 1e-14 * fmax(norm_in, 1e-300);   // :122
  double* qn = basis + k * n;
#pragma unroll
  for (int q = 0; q < WPT; ++q) {
    const int64_t i = tid + (int64_t)q * KR_NT;
    if (i < n) {
      w[i] = wr[q];
      if (!happy) {
        const double v = wr[q] / hk;
        qn[i] = v;
        if (vout) vout[i] = v;
      }
    }
  }
  if (tid == 0) {
    hcol[k] = hk;
    for (int64_t i = 0; i < j; ++i) {               // apply previous rotations, :126-129
      const double temp = cs[i] * hcol[i] + sn[i] * hcol[i + 1];
      hcol[i + 1] = -sn[i] * hcol[i] + cs[i] * hcol[i + 1];
      hcol[i] = temp;
    }
    const double denom = hypot(hcol[j], hcol[k]);
    double brk = 0.0, rel = 0.0;
    if (denom == 0.0) {
      brk = 1.0;
    } else {
      cs[j] = hcol[j] / denom;
      sn[j] = hcol[k] / denom;
      hcol[j] = denom;
      hcol[k] = 0.0;
      g[k] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      rel = fabs(g[k]) / beta;
    }
    out[0] = rel;
    out[1] = happy ? 1.0 : 0.0;
    out[2] = brk;
  }
}

// dispatch: registers for n <= 16 * 1024, the streaming body above that
__device__ __forceinline__ void arnoldi_dispatch(int64_t n, int64_t j, int64_t mmax, double* basis,
                                                 double* hess, double* cs, double* sn, double* g,
                                                 double* w, double beta, double* out,
                                                 double* vout = nullptr) {
  if (n <= 1 * KR_NT) arnoldi_body_reg<1>(n, j, mmax, basis, hess, cs, sn, g, w, beta, out, vout);
  else if (n <= 3 * KR_NT) arnoldi_body_reg<3>(n, j, mmax, basis, hess, cs, sn, g, w, beta, out, vout);
  else if (n <= 5 * KR_NT) arnoldi_body_reg<5>(n, j, mmax, basis, hess, cs, sn, g, w, beta, out, vout);
  else if (n <= 10 * KR_NT) arnoldi_body_reg<10>(n, j, mmax, basis, hess, cs, sn, g, w, beta, out, vout);
  else if (n <= 16 * KR_NT) arnoldi_body_reg<16>(n, j, mmax, basis, hess, cs, sn, g, w, beta, out, vout);
  else arnoldi_body(n, j, mmax, basis, hess, cs, sn, g, w, beta, out, vout);
}

__global__ void __launch_bounds__(KR_NT) arnoldi_kernel(int64_t n, int64_t j, int64_t mmax,
                                                        double* basis, double* hess, double* cs,
                                                        double* sn, double* g, double* w,
                                                        double beta, double* out) {
  arnoldi_dispatch(n, j, mmax, basis, hess, cs, sn, g, w, beta, out);
}

// s independent GMRES systems advanced together (one CTA each): system c owns
// basis + c*bstride, hess + c*hstride, cs/sn/g + c*(mmax+1), w + c*n, beta[c],
// out + 3c; systems whose flag active[c] is 0 (converged) are skipped.
__global__ void __launch_bounds__(KR_NT) arnoldi_batch_kernel(
    int64_t n, int64_t j, int64_t mmax, double* basis, int64_t bstride, double* hess,
    int64_t hstride, double* cs, double* sn, double* g, double* w, const double* beta,
    double* out, const int32_t* active) {
  const int c = blockIdx.x;
  if (!active[c]) return;
  const int64_t vs = mmax + 1;
  arnoldi_dispatch(n, j, mmax, basis + c * bstride, hess + c * hstride, cs + c * vs, sn + c * vs,
                   g + c * vs, w + c * n, beta[c], out + 3 * c);
}

// per-column 2-norms of an n x s column-major block (ld), one CTA per column
__global__ void __launch_bounds__(KR_NT) norms_kernel(const double* x, int64_t n, int64_t ld,
                                                     double* out) {
  __shared__ double red[KR_NT / 32];
  const double* xc = x + blockIdx.x * ld;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += KR_NT) s += xc[i] * xc[i];
  s = block_sum<KR_NT>(s, red);
  if (threadIdx.x == 0) out[blockIdx.x] = sqrt(s);
}

// y = back substitution (krylov.py:147-151) by one thread, then x = Q[:, :m] y.
__global__ void __launch_bounds__(KR_NT) combine_kernel(int64_t n, int64_t m, int64_t mmax,
                                                        const double* basis, const double* hess,
                                                        const double* g, double* x, double* y) {
  const int64_t ldh = mmax + 1;
  if (threadIdx.x == 0) {
    for (int64_t i = m - 1; i >= 0; --i) {
      double s = 0.0;
      for (int64_t l = i + 1; l < m; ++l) s += hess[i + l * ldh] * y[l];
      y[i] = (g[i] - s) / hess[i + i * ldh];
    }
  }
  __syncthreads();
  for (int64_t r = (int64_t)blockIdx.x * KR_NT + threadIdx.x; r < n; r += (int64_t)gridDim.x * KR_NT) {
    double s = 0.0;
    for (int64_t l = 0; l < m; ++l) s += basis[r + l * n] * y[l];
    x[r] = s;
  }
}

__global__ void __launch_bounds__(KR_NT) norm_kernel(const double* x, int64_t n, double* out) {
  __shared__ double red[KR_NT / 32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += KR_NT) s += x[i] * x[i];
  s = block_sum<KR_NT>(s, red);
  if (threadIdx.x == 0) *out = sqrt(s);
}

// y = x / num[0] (invert=0) -- the r0 / beta scaling
__global__ void scale_kernel(const double* x, int64_t n, const double* num, double* y) {
  const double d = *num;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] / d;
}

__global__ void axpby_kernel(const double* x, const double* y, double* z, int64_t n, double a,
                             double b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    z[i] = a * x[i] + b * y[i];
}

// y = x / diag(A), zero diagonal entries treated as 1 (krylov.py:44-62)
__global__ void diag_scale_kernel(const double* A, int64_t lda, const double* x, double* y,
                                  int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double d = A[i * lda + i];
    if (d == 0.0) d = 1.0;
    y[i] = x[i] / d;
  }
}

// ---------------------------------------------------------------- device-resident GMRES
// Loop bookkeeping of krylov.py:121-145 after an Arnoldi step (first = false)
// or at the start (first = true), then the WHILE condition of the graph.
// Runs on one thread after every system's step is visible.
__device__ void gm_control(const GmParams& P, cudaGraphConditionalHandle h, bool first) {
  GmState* st = P.st;
  int k = st->k;
  if (!first) {
    ++k;                                              // iteration k just completed
    for (int c = 0; c < P.s; ++c) {
      if (!st->active[c]) continue;
      const volatile double* o = st->out + 3 * c;
      if (o[2] != 0.0) {                              // Givens breakdown: m = k - 1
        st->brk[c] = 1;
        st->m[c] = k - 1;
        st->active[c] = 0;
        continue;
      }
      P.hist[c * P.max_iter + (k - 1)] = o[0];
      st->m[c] = k;
      if (o[0] <= P.tol || o[1] != 0.0) {             // converged or happy breakdown
        st->conv[c] = 1;
        st->active[c] = 0;
      }
    }
    st->k = k;
  }
  int any = 0;
  for (int c = 0; c < P.s; ++c) any |= st->active[c];
  const int cont = any && k < P.mmax && k < P.cap;
  st->cont = cont;
  st->finished = (!any || k >= P.mmax) ? 1 : 0;
  cudaGraphSetConditional(h, cont ? 1u : 0u);
}

// the last CTA of the grid to arrive runs the control step
__device__ __forceinline__ void gm_last_cta(const GmParams& P, cudaGraphConditionalHandle h, bool first) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const int t = atomicAdd(&P.st->counter, 1);
    if (t == (int)gridDim.x - 1) {
      __threadfence();
      gm_control(P, h, first);
      P.st->counter = 0;
      __threadfence();
    }
  }
}

__global__ void __launch_bounds__(256) gm_start_kernel(GmParams P, const double* R0,
                                                       cudaGraphConditionalHandle h) {
  const int c = blockIdx.x;
  GmState* st = P.st;
  const double nb = st->nb[c], beta = st->beta[c];
  const bool zero = nb == 0.0, err = !zero && beta == 0.0, go = !zero && !err;
  if (go) {                                          // Q[:,0] = r0 / beta (krylov.py:89-93)
    const double* r = R0 + (int64_t)c * P.n;
    double* q = P.basis + c * P.bstride;
    double* v = P.V + (int64_t)c * P.n;
    for (int64_t i = threadIdx.x; i < P.n; i += blockDim.x) {
      const double x = r[i] / beta;
      q[i] = x;
      v[i] = x;
    }
  }
  if (threadIdx.x == 0) {
    st->zero[c] = zero;
    st->err[c] = err;
    st->active[c] = go;
    st->m[c] = st->conv[c] = st->brk[c] = 0;
    st->tres[c] = 0.0;
    if (go) P.g[c * P.vs] = beta;
  }
  gm_last_cta(P, h, true);
}

__global__ void __launch_bounds__(KR_NT) gm_arnoldi_kernel(GmParams P, double* W,
                                                           cudaGraphConditionalHandle h) {
  const int c = blockIdx.x;
  GmState* st = P.st;
  const int64_t j = *(volatile int32_t*)&st->k;     // read before this CTA's arrival count
  if (*(volatile int32_t*)&st->active[c]) {
    const int64_t vs = P.vs;
    arnoldi_dispatch(P.n, j, P.cap, P.basis + c * P.bstride, P.hess + c * P.hstride, P.cs + c * vs,
                     P.sn + c * vs, P.g + c * vs, W + c * P.n, st->beta[c], st->out + 3 * c,
                     P.V + c * P.n);
  }
  gm_last_cta(P, h, false);
}

// back substitution (krylov.py:147-151) and x = Q[:, :m] y (:152)
__global__ void __launch_bounds__(KR_NT) gm_combine_kernel(GmParams P, double* X) {
  const GmState* st = P.st;
  if (!st->finished) return;
  const int c = blockIdx.x;
  const int64_t m = st->m[c], n = P.n, ldh = P.cap + 1;
  double* x = X + (int64_t)c * n;
  if (st->zero[c] || st->err[c] || m == 0) {
    for (int64_t r = threadIdx.x; r < n; r += KR_NT) x[r] = 0.0;
    return;
  }
  const double* hess = P.hess + c * P.hstride;
  const double* g = P.g + c * P.vs;
  double* y = P.y + c * P.vs;
  if (threadIdx.x == 0) {
    for (int64_t i = m - 1; i >= 0; --i) {
      double s = 0.0;
      for (int64_t l = i + 1; l < m; ++l) s += hess[i + l * ldh] * y[l];
      y[i] = (g[i] - s) / hess[i + i * ldh];
    }
  }
  __syncthreads();
  const double* basis = P.basis + c * P.bstride;
  for (int64_t r = threadIdx.x; r < n; r += KR_NT) {
    double s = 0.0;
    for (int64_t l = 0; l < m; ++l) s += basis[r + l * n] * y[l];
    x[r] = s;
  }
}

__global__ void __launch_bounds__(KR_NT) gm_resid_kernel(GmParams P, const double* B, const double* AX) {
  __shared__ double red[KR_NT / 32];
  GmState* st = P.st;
  if (!st->finished) return;
  const int c = blockIdx.x;
  const double* b = B + (int64_t)c * P.n;
  const double* ax = AX + (int64_t)c * P.n;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < P.n; i += KR_NT) {
    const double d = b[i] - ax[i];
    s += d * d;
  }
  s = block_sum<KR_NT>(s, red);
  if (threadIdx.x == 0) st->tres[c] = st->zero[c] ? 0.0 : sqrt(s) / st->nb[c];
}

__global__ void vdiv_kernel(const double* x, const double* d, double* y, int64_t n, int s) {
  const int64_t total = n * s;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x)
    y[t] = x[t] / d[t % n];
}

int grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 2048) b = 2048;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace

cudaError_t hk_launch_arnoldi(int64_t n, int64_t j, int64_t mmax, double* basis, double* hess,
                              double* cs, double* sn, double* g, double* w, double beta,
                              double* out_dev, cudaStream_t st) {
  arnoldi_kernel<<<1, KR_NT, 0, st>>>(n, j, mmax, basis, hess, cs, sn, g, w, beta, out_dev);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_combine(int64_t n, int64_t m, int64_t mmax, const double* basis,
                              const double* hess, const double* g, double* x, double* y_scratch,
                              cudaStream_t st) {
  combine_kernel<<<1, KR_NT, 0, st>>>(n, m, mmax, basis, hess, g, x, y_scratch);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_norm(const double* x, int64_t n, double* out, cudaStream_t st) {
  norm_kernel<<<1, KR_NT, 0, st>>>(x, n, out);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_scale(const double* x, int64_t n, const double* num, double* y, int invert,
                            cudaStream_t st) {
  (void)invert;
  scale_kernel<<<grid_for(n), 256, 0, st>>>(x, n, num, y);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_axpby(const double* x, const double* y, double* z, int64_t n, double a,
                            double b, cudaStream_t st) {
  axpby_kernel<<<grid_for(n), 256, 0, st>>>(x, y, z, n, a, b);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_diag_scale(const double* A, int64_t lda, const double* x, double* y,
                                 int64_t n, cudaStream_t st) {
  diag_scale_kernel<<<grid_for(n), 256, 0, st>>>(A, lda, x, y, n);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_arnoldi_batch(int64_t n, int64_t j, int64_t mmax, double* basis,
                                    int64_t bstride, double* hess, int64_t hstride, double* cs,
                                    double* sn, double* g, double* w, const double* beta,
                                    double* out, const int32_t* active, int s, cudaStream_t st) {
  if (s <= 0) return cudaSuccess;
  arnoldi_batch_kernel<<<s, KR_NT, 0, st>>>(n, j, mmax, basis, bstride, hess, hstride, cs, sn, g,
                                            w, beta, out, active);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_norms(const double* x, int64_t n, int64_t ld, int s, double* out,
                            cudaStream_t st) {
  if (s <= 0) return cudaSuccess;
  norms_kernel<<<s, KR_NT, 0, st>>>(x, n, ld, out);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_gm_start(const GmParams& P, const double* R0, cudaGraphConditionalHandle h,
                               cudaStream_t st) {
  gm_start_kernel<<<P.s, 256, 0, st>>>(P, R0, h);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_gm_arnoldi(const GmParams& P, double* W, cudaGraphConditionalHandle h,
                                 cudaStream_t st) {
  gm_arnoldi_kernel<<<P.s, KR_NT, 0, st>>>(P, W, h);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_gm_combine(const GmParams& P, double* X, cudaStream_t st) {
  gm_combine_kernel<<<P.s, KR_NT, 0, st>>>(P, X);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_gm_resid(const GmParams& P, const double* B, const double* AX, cudaStream_t st) {
  gm_resid_kernel<<<P.s, KR_NT, 0, st>>>(P, B, AX);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_vdiv(const double* x, const double* d, double* y, int64_t n, int s,
                           cudaStream_t st) {
  if (n <= 0 || s <= 0) return cudaSuccess;
  vdiv_kernel<<<grid_for(n * s), 256, 0, st>>>(x, d, y, n, s);
  hk_count_launch();
  return cudaGetLastError();
}
