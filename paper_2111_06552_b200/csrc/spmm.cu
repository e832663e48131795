// MatDotMultiVec on B200: fp64 CSR x row-major multivector (SpMM).
//
// Reference: CsrOperator.apply (operators.py:103-111) -> kernels.csr_matvec
// (_cy.pyx:11-23: column-by-column scalar CSR loop) and ShiftedOperator.apply
// (operators.py:149-156: A x - theta (B x or x)).
//
// B200 design.  X is row-major, so the k values a nonzero (i, j) needs are one
// contiguous run X[j*ldx : j*ldx+k].  A group of LPR lanes owns one row and
// reads those runs with 16-byte vector loads (NV column chunks per lane); a
// warp holds 32/LPR rows.  The row's (column index, value) stream is loaded
// once, cooperatively (one nonzero per lane, 12 B/nnz from HBM), and broadcast
// inside the group with shuffles.
//
// At the BASELINE shapes the kernel is latency-bound (a row is a 3-deep chain:
// row pointer -> index/value -> X gathers), so it is software-pipelined: while
// a warp gathers X for its current rows it already holds the row pointers and
// the index/value chunk of its NEXT rows in registers, leaving only the X
// gathers on the critical path; all gathers of a row batch (up to 8 nonzeros)
// are issued before the first FMA.
//
// The epilogue fuses the shifted-operator term (gamma*Z, Z = X for A - theta*I),
// an axpby with a second input (beta*Yin, used for r = rhs - op x) and an
// optional per-column dot product reduced deterministically (p'q and ||r||^2
// for block CG), so CG never makes a separate pass for them.
//
// Roofline: HBM.  Algorithmic bytes per launch = 12*nnz + 4*(n+1) + 16*n*k
// (+8*n*k per extra epilogue stream); flops = 2*nnz*k.

#include <stdlib.h>

#include "common.cuh"

namespace gcg {

extern int64_t g_launches;

struct SpmmArgs {
  long long n;
  const int* __restrict__ rowptr;
  const int* __restrict__ colidx;
  const double* __restrict__ val;
  int k;
  const double* __restrict__ X;
  long long ldx;
  double alpha, gamma, beta;
  const double* __restrict__ Z;
  long long ldz;
  const double* Yin;
  long long ldyin;
  double* Y;
  long long ldy;
  int dot_mode;
  const double* __restrict__ W;
  long long ldw;
  double* partials;   // [gridDim.x][k]
  const int* skip;    // device flag: nonzero -> kernel is a no-op (CG early exit)
  int* prof_skipped;  // profiling: set when the launch was a no-op
};

template <int VEC>
struct VecT;
template <>
struct VecT<1> {
  static __device__ __forceinline__ void load(const double* p, double* o) { o[0] = __ldg(p); }
};
template <>
struct VecT<2> {
  static __device__ __forceinline__ void load(const double* p, double* o) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(p));
    o[0] = v.x;
    o[1] = v.y;
  }
};

constexpr int kSpmmThreads = 256;
constexpr int kSpmmMinBlocks = 4;  // <= 64 registers: 32 resident warps per SM

template <int LPR, int VEC, int NV>
__global__ void __launch_bounds__(kSpmmThreads, kSpmmMinBlocks) spmm_csr_kernel(SpmmArgs a) {
  if (a.skip != nullptr && *a.skip) {
    if (a.prof_skipped && blockIdx.x == 0 && threadIdx.x == 0) *a.prof_skipped = 1;
    return;
  }
  constexpr int G = 32 / LPR;  // rows per warp step
  constexpr int COLS = LPR * VEC * NV;
  // gathers in flight per batch: <= 16 doubles of X per lane, a power of 2 dividing LPR
  constexpr int UB = 16 / (NV * VEC);
  constexpr int U0 = UB >= 8 ? 8 : (UB >= 4 ? 4 : 2);
  constexpr int U = U0 < LPR ? U0 : LPR;
  constexpr int NW = kSpmmThreads / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / LPR, sub = lane % LPR;
  const long long stride = (long long)gridDim.x * NW * G;
  const int k = a.k;

  __shared__ double sdot[NW][COLS];
  double dacc[NV][VEC];
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int e = 0; e < VEC; ++e) dacc[q][e] = 0.0;

  // prefetched state of the row this lane group handles next
  long long rb = ((long long)blockIdx.x * NW + warp) * G;
  int nstart = 0, nlen = 0, ncol = 0;
  double nval = 0.0;
  auto fetch_rowptr = [&](long long base, int& st, int& ln) {
    const long long r = base + g;
    st = 0;
    ln = 0;
    if (r < a.n) {
      st = __ldg(a.rowptr + r);
      ln = __ldg(a.rowptr + r + 1) - st;
    }
  };
  auto fetch_chunk = [&](int st, int ln, int off, int& cidx, double& cval) {
    cidx = 0;
    cval = 0.0;
    if (off + sub < ln) {
      cidx = __ldg(a.colidx + st + off + sub);
      cval = __ldg(a.val + st + off + sub);
    }
  };
  if (rb < a.n) {
    fetch_rowptr(rb, nstart, nlen);
    fetch_chunk(nstart, nlen, 0, ncol, nval);
  }

  for (; rb < a.n; rb += stride) {
    const long long r = rb + g;
    const int start = nstart, len = nlen;
    int mycol = ncol;
    double myval = nval;
    const long long rbn = rb + stride;
    if (rbn < a.n) fetch_rowptr(rbn, nstart, nlen);  // lands during the gathers below
    const int maxlen = __reduce_max_sync(0xffffffffu, len);
    double acc[NV][VEC];
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[q][e] = 0.0;

    for (int off = 0; off < maxlen; off += LPR) {
      if (off > 0) fetch_chunk(start, len, off, mycol, myval);  // rows longer than LPR
      const int tmax = min(LPR, maxlen - off);
      for (int t0 = 0; t0 < tmax; t0 += U) {
        int j[U];
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          j[u] = __shfl_sync(0xffffffffu, mycol, t0 + u, LPR);
          v[u] = __shfl_sync(0xffffffffu, myval, t0 + u, LPR);
          if (t0 + u >= tmax || off + t0 + u >= len) v[u] = 0.0;
        }
        double xv[U][NV][VEC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool ok = (t0 + u < tmax) && (off + t0 + u < len);
          const double* xr = a.X + (long long)j[u] * a.ldx;
#pragma unroll
          for (int q = 0; q < NV; ++q) {
            const int c = (q * LPR + sub) * VEC;
            if (ok && c < k) {
              VecT<VEC>::load(xr + c, xv[u][q]);
            } else {
#pragma unroll
              for (int e = 0; e < VEC; ++e) xv[u][q][e] = 0.0;
            }
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int q = 0; q < NV; ++q)
#pragma unroll
            for (int e = 0; e < VEC; ++e) acc[q][e] = fma(v[u], xv[u][q][e], acc[q][e]);
      }
    }
    // first index/value chunk of the next rows (their row pointers have arrived)
    if (rbn < a.n) fetch_chunk(nstart, nlen, 0, ncol, nval);
    if (r < a.n) {
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const int c = (q * LPR + sub) * VEC;
        if (c < k) {
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            double y = a.alpha * acc[q][e];
            if (a.gamma != 0.0) y = fma(a.gamma, a.Z[r * a.ldz + c + e], y);
            if (a.beta != 0.0) y = fma(a.beta, a.Yin[r * a.ldyin + c + e], y);
            a.Y[r * a.ldy + c + e] = y;
            if (a.dot_mode == 1) dacc[q][e] = fma(y, a.W[r * a.ldw + c + e], dacc[q][e]);
            else if (a.dot_mode == 2) dacc[q][e] = fma(y, y, dacc[q][e]);
          }
        }
      }
    }
  }

  if (a.dot_mode == 0) return;
  // reduce over the row groups of the warp (lanes with equal `sub`), then warps
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      double v = dacc[q][e];
#pragma unroll
      for (int o = LPR; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      dacc[q][e] = v;
    }
  if (g == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
      for (int e = 0; e < VEC; ++e) sdot[warp][(q * LPR + sub) * VEC + e] = dacc[q][e];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k && c < COLS; c += kSpmmThreads) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += sdot[w][c];
    a.partials[(long long)blockIdx.x * k + c] = s;
  }
}

// out[c*out_stride] = sum_b partials[b*k + c] in fixed b order (deterministic).
__global__ void reduce_partials_kernel(const double* __restrict__ partials, int nparts, int k,
                                       double* out, int out_stride, int mode) {
  const int c = blockIdx.x;
  double s = 0.0;
  for (int b = threadIdx.x; b < nparts; b += blockDim.x) s += partials[(long long)b * k + c];
  __shared__ double sm[128];  // fixed-shape tree over the 128 threads
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int w = 64; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double v = sm[0];
    if (mode == 1) v += out[(long long)c * out_stride];
    out[(long long)c * out_stride] = v;
  }
}

int reduce_partials(Ctx* c, const double* partials, int nparts, int k, double* out,
                    int out_stride, int mode) {
  if (k <= 0) return GCG_OK;
  reduce_partials_kernel<<<k, 128, 0, c->stream>>>(partials, nparts, k, out, out_stride, mode);
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

template <int LPR, int VEC>
static int launch_nv(Ctx* c, SpmmArgs a, int nv, int grid) {
  switch (nv) {
    case 1: spmm_csr_kernel<LPR, VEC, 1><<<grid, kSpmmThreads, 0, c->stream>>>(a); break;
    case 2: spmm_csr_kernel<LPR, VEC, 2><<<grid, kSpmmThreads, 0, c->stream>>>(a); break;
    case 3: spmm_csr_kernel<LPR, VEC, 3><<<grid, kSpmmThreads, 0, c->stream>>>(a); break;
    default: spmm_csr_kernel<LPR, VEC, 4><<<grid, kSpmmThreads, 0, c->stream>>>(a); break;
  }
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

template <int VEC>
static int launch_lpr(Ctx* c, SpmmArgs a, int lpr, int nv, int grid) {
  switch (lpr) {
    case 4: return launch_nv<4, VEC>(c, a, nv, grid);
    case 8: return launch_nv<8, VEC>(c, a, nv, grid);
    case 16: return launch_nv<16, VEC>(c, a, nv, grid);
    default: return launch_nv<32, VEC>(c, a, nv, grid);
  }
}

static inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// exactly one wave of kSpmmMinBlocks CTAs per SM (grid-stride over rows)
int spmm_grid(Ctx* c, long long n) { return grid_for(n, 64, kSpmmMinBlocks, c->num_sms); }

// One SpMM over all k columns, split into passes of at most 256 columns.  With
// dot_mode != 0 and `partials` given, per-CTA partials ([grid][k], k <= 256)
// are left for the caller to reduce; otherwise they are reduced into `dots`.
int spmm_launch_impl(Ctx* c, long long n, long long nnz, const int* rowptr, const int* colidx,
                     const double* val, int k, const double* X, long long ldx, double alpha,
                     double gamma, const double* Z, long long ldz, double beta, const double* Yin,
                     long long ldyin, double* Y, long long ldy, int dot_mode, const double* W,
                     long long ldw, double* dots, double* partials_ext, int* grid_out,
                     const int* skip) {
  if (n <= 0 || k <= 0) return GCG_OK;
  constexpr int kMaxPass = 256;
  const int grid = spmm_grid(c, n);
  if (grid_out) *grid_out = grid;
  if (partials_ext && k > kMaxPass) return GCG_ERR_ARG;
  double* partials = partials_ext;
  if (dot_mode && !partials) {
    GCG_TRY(ensure(c->partials, sizeof(double) * (size_t)grid * (size_t)kMaxPass));
    partials = (double*)c->partials.ptr;
  }
  for (int c0 = 0; c0 < k; c0 += kMaxPass) {
    const int kc = (k - c0) < kMaxPass ? (k - c0) : kMaxPass;
    const bool vec2 = (kc % 2 == 0) && (ldx % 2 == 0) && aligned16(X + c0);
    const int vec = vec2 ? 2 : 1;
    const int lanes_needed = (kc + vec - 1) / vec;
    // small lane groups keep more rows (independent gather chains) per warp:
    // about two column chunks per lane, at most four
    int lpr = 4;
    while (lpr < 32 && 2 * lpr < lanes_needed) lpr <<= 1;
    const int nv = (lanes_needed + lpr - 1) / lpr;
    SpmmArgs a;
    a.n = n;
    a.rowptr = rowptr;
    a.colidx = colidx;
    a.val = val;
    a.k = kc;
    a.X = X + c0;
    a.ldx = ldx;
    a.alpha = alpha;
    a.gamma = gamma;
    a.Z = Z ? Z + c0 : nullptr;
    a.ldz = ldz;
    a.beta = beta;
    a.Yin = Yin ? Yin + c0 : nullptr;
    a.ldyin = ldyin;
    a.Y = Y + c0;
    a.ldy = ldy;
    a.dot_mode = dot_mode;
    a.W = W ? W + c0 : nullptr;
    a.ldw = ldw;
    a.partials = partials;
    a.skip = skip;
    // algorithmic bytes: index/value stream + X once + Y once + each extra distinct stream
    double bytes = 12.0 * nnz + 4.0 * (n + 1) + 16.0 * n * kc;
    if (gamma != 0.0 && Z != X) bytes += 8.0 * n * kc;
    if (beta != 0.0) bytes += 8.0 * n * kc;
    if (dot_mode == 1 && W != X && W != Z) bytes += 8.0 * n * kc;
    const int ps = prof_start(c, PROF_SPMM, bytes);
    a.prof_skipped = prof_skip_slot(c, ps);
    const int s = vec2 ? launch_lpr<2>(c, a, lpr, nv, grid) : launch_lpr<1>(c, a, lpr, nv, grid);
    prof_stop(c, ps);
    if (s != GCG_OK) return s;
    if (dot_mode && !partials_ext) {
      GCG_TRY(reduce_partials(c, partials, grid, kc, dots + c0, 1, 0));
      ++g_launches;
    }
  }
  return GCG_OK;
}

int spmm_launch_parts(Ctx* c, long long n, long long nnz, const int* rowptr, const int* colidx,
                      const double* val, int k, const double* X, long long ldx, double alpha,
                      double gamma, const double* Z, long long ldz, double beta,
                      const double* Yin, long long ldyin, double* Y, long long ldy, int dot_mode,
                      const double* W, long long ldw, double* partials, int* grid_out,
                      const int* skip) {
  return spmm_launch_impl(c, n, nnz, rowptr, colidx, val, k, X, ldx, alpha, gamma, Z, ldz, beta,
                          Yin, ldyin, Y, ldy, dot_mode, W, ldw, nullptr, partials, grid_out, skip);
}

}  // namespace gcg
