// Tall-skinny multivector kernels on B200 (fp64, row-major multivectors).
//
//  gram     G = alpha X'Y + beta G   MultiVecInnerProd   multivec.py:84-112, _cy.pyx:26-50,
//                                                        orth.py:139-140,164,242,288
//  lincomb  Y = alpha X C + beta Y   MultiVecLinearComb  solver.py:300,333,376; orth.py:144,175,184
//  axpby    Y = alpha X + beta Y     MultiVecAxpby       multivec.py:62-73, _cy.pyx:53-65
//  + strided copy / column scaling / column dots / fill
//
// Gram: the n-long contraction is split into row slabs (a multiple of the SM
// count); each CTA stages a 16-row chunk of X and Y tiles in shared memory
// and accumulates a register micro-tile, then slab partials are reduced in
// fixed order — the result is bit-identical run to run, which is the
// reference's `deterministic` contract (test_kernels.py:74-85) for free.
// Roofline: HBM for k1*k2/(k1+k2) small (bytes 8n(k1+k2)), FP64 otherwise
// (flops 2n k1 k2).
//
// LinComb: classic row-panel GEMM; each CTA owns BM rows x BN columns of Y and
// walks m in BK chunks with X and C tiles in shared memory.  Bytes 8n(m+d)
// (+8nd if beta != 0), flops 2nmd.

#include "common.cuh"

namespace gcg {

int64_t g_launches = 0;

// ---------------------------------------------------------------------------
// Gram

template <int BM, int BN, int TM, int TN>
__global__ void __launch_bounds__(256) gram_kernel(long long n, int k1, int k2,
                                                   const double* __restrict__ X, long long ldx,
                                                   const double* __restrict__ Y, long long ldy,
                                                   long long rows_per_slab, double* part) {
  constexpr int BK = 16;
  constexpr int TX = BN / TN;  // threads along columns
  constexpr int TY = BM / TM;
  static_assert(TX * TY == 256, "256 threads");
  __shared__ double Xs[BK][BM];
  __shared__ double Ys[BK][BN];
  const int tm0 = blockIdx.x * BM;
  const int tn0 = blockIdx.y * BN;
  const int slab = blockIdx.z;
  const long long r0 = (long long)slab * rows_per_slab;
  long long r1 = r0 + rows_per_slab;
  if (r1 > n) r1 = n;
  const int tx = threadIdx.x % TX;
  const int ty = threadIdx.x / TX;
  double acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0;

  for (long long rb = r0; rb < r1; rb += BK) {
    // cooperative loads (coalesced along the contiguous column direction)
    for (int e = threadIdx.x; e < BK * BM; e += 256) {
      const int rr = e / BM, cc = e % BM;
      const long long row = rb + rr;
      const int col = tm0 + cc;
      Xs[rr][cc] = (row < r1 && col < k1) ? __ldg(X + row * ldx + col) : 0.0;
    }
    for (int e = threadIdx.x; e < BK * BN; e += 256) {
      const int rr = e / BN, cc = e % BN;
      const long long row = rb + rr;
      const int col = tn0 + cc;
      Ys[rr][cc] = (row < r1 && col < k2) ? __ldg(Y + row * ldy + col) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double xv[TM], yv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) xv[i] = Xs[kk][ty + i * TY];
#pragma unroll
      for (int j = 0; j < TN; ++j) yv[j] = Ys[kk][tx + j * TX];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(xv[i], yv[j], acc[i][j]);
    }
    __syncthreads();
  }
  double* out = part + (long long)slab * k1 * k2;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int r = tm0 + ty + i * TY;
    if (r >= k1) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int c = tn0 + tx + j * TX;
      if (c < k2) out[(long long)r * k2 + c] = acc[i][j];
    }
  }
}

// G[r*grs + c*gcs] = alpha * sum_s part[s][r][c] + beta * G  (fixed slab order)
__global__ void gram_finish_kernel(int k1, int k2, int nslab, const double* __restrict__ part,
                                   double alpha, double beta, double* G, long long grs,
                                   long long gcs) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)k1 * k2) return;
  const int r = (int)(e / k2), c = (int)(e % k2);
  double s = 0.0;
  for (int q = 0; q < nslab; ++q) s += part[(long long)q * k1 * k2 + e];
  double* g = G + r * grs + c * gcs;
  *g = (beta == 0.0) ? alpha * s : fma(alpha, s, beta * *g);
}

int col_dots_launch(Ctx* c, long long n, int k, const double* X, long long ldx, const double* Y,
                    long long ldy, double* out);

int gram_launch(Ctx* c, long long n, int k1, int k2, const double* X, long long ldx,
                const double* Y, long long ldy, double alpha, double beta, double* G,
                long long grs, long long gcs) {
  if (k1 <= 0 || k2 <= 0) return GCG_OK;
  const bool big = (k1 > 32 && k2 > 32);
  const int BM = big ? 64 : 32, BN = big ? 64 : 32;
  const int tiles = ((k1 + BM - 1) / BM) * ((k2 + BN - 1) / BN);
  // enough slabs for ~4 CTAs per SM, but keep >= 256 rows per slab
  long long nslab = (4LL * c->num_sms + tiles - 1) / tiles;
  long long max_slab = (n + 255) / 256;
  if (nslab > max_slab) nslab = max_slab;
  if (nslab < 1) nslab = 1;
  if (nslab > 65535) nslab = 65535;
  long long rps = (n + nslab - 1) / nslab;
  rps = (rps + 15) / 16 * 16;
  nslab = (n + rps - 1) / rps;
  if (nslab < 1) nslab = 1;
  GCG_TRY(ensure(c->partials, sizeof(double) * (size_t)nslab * k1 * k2));
  double* part = (double*)c->partials.ptr;
  dim3 grid((k1 + BM - 1) / BM, (k2 + BN - 1) / BN, (unsigned)nslab);
  const int ps = prof_start(c, PROF_GRAM, 8.0 * n * (X == Y ? k1 : k1 + k2));
  if (big)
    gram_kernel<64, 64, 4, 4><<<grid, 256, 0, c->stream>>>(n, k1, k2, X, ldx, Y, ldy, rps, part);
  else
    gram_kernel<32, 32, 2, 2><<<grid, 256, 0, c->stream>>>(n, k1, k2, X, ldx, Y, ldy, rps, part);
  prof_stop(c, ps);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  const long long tot = (long long)k1 * k2;
  gram_finish_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, c->stream>>>(
      k1, k2, (int)nslab, part, alpha, beta, G, grs, gcs);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

// ---------------------------------------------------------------------------
// LinComb  Y = alpha X C + beta Y

template <int BM, int BN, int TM, int TN>
__global__ void __launch_bounds__(256) lincomb_kernel(long long n, int m, int d, double alpha,
                                                      const double* __restrict__ X, long long ldx,
                                                      const double* __restrict__ C, long long ldc,
                                                      double beta, double* Y, long long ldy) {
  constexpr int BK = 16;
  constexpr int TX = BN / TN;
  constexpr int TY = BM / TM;
  static_assert(TX * TY == 256, "256 threads");
  __shared__ double Xs[BK][BM + 1];
  __shared__ double Cs[BK][BN];
  const long long r0 = (long long)blockIdx.x * BM;
  const int c0 = blockIdx.y * BN;
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  double acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0;
  for (int kb = 0; kb < m; kb += BK) {
    for (int e = threadIdx.x; e < BM * BK; e += 256) {
      const int rr = e / BK, kk = e % BK;
      const long long row = r0 + rr;
      Xs[kk][rr] = (row < n && kb + kk < m) ? __ldg(X + row * ldx + kb + kk) : 0.0;
    }
    for (int e = threadIdx.x; e < BK * BN; e += 256) {
      const int kk = e / BN, cc = e % BN;
      Cs[kk][cc] = (kb + kk < m && c0 + cc < d) ? __ldg(C + (long long)(kb + kk) * ldc + c0 + cc)
                                                : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double xv[TM], cv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) xv[i] = Xs[kk][ty + i * TY];
#pragma unroll
      for (int j = 0; j < TN; ++j) cv[j] = Cs[kk][tx + j * TX];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(xv[i], cv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const long long row = r0 + ty + i * TY;
    if (row >= n) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int col = c0 + tx + j * TX;
      if (col >= d) continue;
      double* y = Y + row * ldy + col;
      *y = (beta == 0.0) ? alpha * acc[i][j] : fma(alpha, acc[i][j], beta * *y);
    }
  }
}

int lincomb_launch(Ctx* c, long long n, int m, int d, double alpha, const double* X,
                   long long ldx, const double* C, long long ldc, double beta, double* Y,
                   long long ldy) {
  if (n <= 0 || d <= 0) return GCG_OK;
  const int ps = prof_start(c, PROF_LINCOMB, 8.0 * n * (m + d) + (beta != 0.0 ? 8.0 * n * d : 0.0));
  if (d <= 32) {
    dim3 grid((unsigned)((n + 127) / 128), (d + 31) / 32);
    lincomb_kernel<128, 32, 4, 4><<<grid, 256, 0, c->stream>>>(n, m, d, alpha, X, ldx, C, ldc,
                                                                beta, Y, ldy);
  } else {
    dim3 grid((unsigned)((n + 63) / 64), (d + 63) / 64);
    lincomb_kernel<64, 64, 4, 4><<<grid, 256, 0, c->stream>>>(n, m, d, alpha, X, ldx, C, ldc,
                                                               beta, Y, ldy);
  }
  prof_stop(c, ps);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

// ---------------------------------------------------------------------------
// elementwise multivector kernels: one thread per element, grid-stride

__global__ void axpby_kernel(long long n, int k, double alpha, const double* __restrict__ X,
                             long long ldx, double beta, double* Y, long long ldy) {
  const long long tot = n * k;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / k;
    const int c = (int)(e % k);
    double* y = Y + i * ldy + c;
    double v;
    if (beta == 0.0) v = (alpha == 0.0) ? 0.0 : alpha * X[i * ldx + c];
    else {
      v = *y;
      if (beta != 1.0) v *= beta;
      if (alpha != 0.0) v += alpha * X[i * ldx + c];
    }
    *y = v;
  }
}

__global__ void copy_kernel(long long n, int k, const double* __restrict__ X, long long ldx,
                            double* Y, long long ldy) {
  const long long tot = n * k;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / k;
    const int c = (int)(e % k);
    Y[i * ldy + c] = X[i * ldx + c];
  }
}

__global__ void fill_kernel(long long n, int k, double v, double* Y, long long ldy) {
  const long long tot = n * k;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    Y[(e / k) * ldy + (e % k)] = v;
  }
}

__global__ void col_scale_kernel(long long n, int k, const double* __restrict__ s, double* X,
                                 long long ldx) {
  const long long tot = n * k;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e % k);
    X[(e / k) * ldx + c] *= s[c];
  }
}

// per-CTA column dot partials over a contiguous row range; threads map to
// (row-lane, column) with the column fastest so loads are coalesced.
__global__ void __launch_bounds__(256) col_dots_kernel(long long n, int k,
                                                       const double* __restrict__ X, long long ldx,
                                                       const double* __restrict__ Y, long long ldy,
                                                       long long rows_per_cta, double* part) {
  extern __shared__ double sm[];
  const int kc = k < 256 ? k : 256;  // columns handled per pass
  const int lanes = 256 / kc;        // row lanes
  const long long r0 = (long long)blockIdx.x * rows_per_cta;
  long long r1 = r0 + rows_per_cta;
  if (r1 > n) r1 = n;
  for (int cb = 0; cb < k; cb += kc) {
    const int c = cb + threadIdx.x % kc;
    const int rl = threadIdx.x / kc;
    double s = 0.0;
    if (rl < lanes && c < k) {
      for (long long i = r0 + rl; i < r1; i += lanes) s = fma(X[i * ldx + c], Y[i * ldy + c], s);
    }
    sm[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x < kc && c < k) {
      double t = 0.0;
      for (int l = 0; l < lanes; ++l) t += sm[l * kc + threadIdx.x];
      part[(long long)blockIdx.x * k + c] = t;
    }
    __syncthreads();
  }
}

static int elem_grid(Ctx* c, long long tot) { return grid_for(tot, 256 * 4, 8, c->num_sms); }

int axpby_launch(Ctx* c, long long n, int k, double alpha, const double* X, long long ldx,
                 double beta, double* Y, long long ldy) {
  if (n <= 0 || k <= 0) return GCG_OK;
  axpby_kernel<<<elem_grid(c, n * k), 256, 0, c->stream>>>(n, k, alpha, X, ldx, beta, Y, ldy);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

int copy_launch(Ctx* c, long long n, int k, const double* X, long long ldx, double* Y,
                long long ldy) {
  if (n <= 0 || k <= 0 || X == Y) return GCG_OK;
  copy_kernel<<<elem_grid(c, n * k), 256, 0, c->stream>>>(n, k, X, ldx, Y, ldy);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

int fill_launch(Ctx* c, long long n, int k, double v, double* Y, long long ldy) {
  if (n <= 0 || k <= 0) return GCG_OK;
  fill_kernel<<<elem_grid(c, n * k), 256, 0, c->stream>>>(n, k, v, Y, ldy);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

int col_scale_launch(Ctx* c, long long n, int k, const double* s, double* X, long long ldx) {
  if (n <= 0 || k <= 0) return GCG_OK;
  col_scale_kernel<<<elem_grid(c, n * k), 256, 0, c->stream>>>(n, k, s, X, ldx);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

int col_dots_launch(Ctx* c, long long n, int k, const double* X, long long ldx, const double* Y,
                    long long ldy, double* out) {
  if (k <= 0) return GCG_OK;
  if (n <= 0) return fill_launch(c, 1, k, 0.0, out, k);
  int grid = grid_for(n, 1024, 4, c->num_sms);
  long long rpc = (n + grid - 1) / grid;
  grid = (int)((n + rpc - 1) / rpc);
  GCG_TRY(ensure(c->partials, sizeof(double) * (size_t)grid * k));
  double* part = (double*)c->partials.ptr;
  col_dots_kernel<<<grid, 256, 256 * sizeof(double), c->stream>>>(n, k, X, ldx, Y, ldy, rpc,
                                                                   part);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  GCG_TRY(reduce_partials(c, part, grid, k, out, 1, 0));
  ++g_launches;
  return GCG_OK;
}

// ---------------------------------------------------------------------------
// small dense GEMM (row-major; matrices of order <= a few thousand)

__global__ void dgemm_small_kernel(int ta, int tb, int M, int N, int K, double alpha,
                                   const double* __restrict__ A, long long lda,
                                   const double* __restrict__ B, long long ldb, double beta,
                                   double* C, long long ldc) {
  __shared__ double As[16][17];
  __shared__ double Bs[16][17];
  const int row = blockIdx.y * 16 + threadIdx.y;
  const int col = blockIdx.x * 16 + threadIdx.x;
  double acc = 0.0;
  for (int kb = 0; kb < K; kb += 16) {
    {
      const int kk = kb + threadIdx.x;  // A(row, kk)
      double v = 0.0;
      if (row < M && kk < K) v = ta ? A[(long long)kk * lda + row] : A[(long long)row * lda + kk];
      As[threadIdx.y][threadIdx.x] = v;
    }
    {
      const int kk = kb + threadIdx.y;  // B(kk, col)
      double v = 0.0;
      if (col < N && kk < K) v = tb ? B[(long long)col * ldb + kk] : B[(long long)kk * ldb + col];
      Bs[threadIdx.y][threadIdx.x] = v;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) acc = fma(As[threadIdx.y][q], Bs[q][threadIdx.x], acc);
    __syncthreads();
  }
  if (row < M && col < N) {
    double* cp = C + (long long)row * ldc + col;
    *cp = (beta == 0.0) ? alpha * acc : fma(alpha, acc, beta * *cp);
  }
}

int dgemm_launch(Ctx* c, int ta, int tb, int M, int N, int K, double alpha, const double* A,
                 long long lda, const double* B, long long ldb, double beta, double* C,
                 long long ldc) {
  if (M <= 0 || N <= 0) return GCG_OK;
  dim3 block(16, 16), grid((N + 15) / 16, (M + 15) / 16);
  dgemm_small_kernel<<<grid, block, 0, c->stream>>>(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta,
                                                    C, ldc);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

__global__ void symmetrize_kernel(int m, double* A, long long lda) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)m * m) return;
  const int i = (int)(e / m), j = (int)(e % m);
  if (j <= i) return;
  double a = A[(long long)i * lda + j], b = A[(long long)j * lda + i];
  double s = (a + b) / 2.0;
  A[(long long)i * lda + j] = s;
  A[(long long)j * lda + i] = (b + a) / 2.0;
}

int symmetrize_launch(Ctx* c, int m, double* A, long long lda) {
  if (m <= 1) return GCG_OK;
  const long long tot = (long long)m * m;
  symmetrize_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, c->stream>>>(m, A, lda);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

}  // namespace gcg
