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
                                                       long long rows_per_cta, double* part,
                                                       const int* skip) {
  if (skip && *skip) return;
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

// out[i*ldo + c] = X[idx[i]*ldx + c]  (halo send packing)
__global__ void gather_rows_kernel(int nidx, const int* __restrict__ idx, int k,
                                   const double* __restrict__ X, long long ldx, double* out,
                                   long long ldo) {
  const long long tot = (long long)nidx * k;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / k), c = (int)(e % k);
    out[(long long)i * ldo + c] = X[(long long)idx[i] * ldx + c];
  }
}

static int elem_grid(Ctx* c, long long tot) { return grid_for(tot, 256 * 4, 8, c->num_sms); }

int gather_rows_launch(Ctx* c, int nidx, const int* idx, int k, const double* X, long long ldx,
                       double* out, long long ldo) {
  if (nidx <= 0 || k <= 0) return GCG_OK;
  gather_rows_kernel<<<elem_grid(c, (long long)nidx * k), 256, 0, c->stream>>>(nidx, idx, k, X,
                                                                              ldx, out, ldo);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

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

// Y[i, c] = s[c] * X[i, c] in one pass (the block-CG right-hand side scale * X)
__global__ void col_scale_copy_kernel(long long n, int k, const double* __restrict__ s,
                                      const double* __restrict__ X, long long ldx, double* Y,
                                      long long ldy) {
  const long long tot = n * k;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / k;
    const int c = (int)(e - i * k);
    Y[i * ldy + c] = s[c] * X[i * ldx + c];
  }
}

int col_scale_copy_launch(Ctx* c, long long n, int k, const double* s, const double* X,
                          long long ldx, double* Y, long long ldy) {
  if (n <= 0 || k <= 0) return GCG_OK;
  col_scale_copy_kernel<<<elem_grid(c, n * k), 256, 0, c->stream>>>(n, k, s, X, ldx, Y, ldy);
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
                                                                   part, c->skip);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  GCG_TRY(reduce_partials(c, part, grid, k, out, 1, 0));
  ++g_launches;
  return GCG_OK;
}

// ---------------------------------------------------------------------------
// small dense GEMM (row-major; matrices of order <= a few thousand)

// One 16 x 16 output tile per CTA, K walked in slabs of 64: every thread requests its
// four A and four B elements of a slab before the barrier (eight independent loads in
// flight instead of two), so an order-200 product costs 4 exposed memory latencies, not
// 13 — these launches are latency-bound (a few hundred kflop).  The k-order of each
// output's fma chain is unchanged.
constexpr int kGemmKT = 64;
__global__ void dgemm_small_kernel(int ta, int tb, int M, int N, int K, double alpha,
                                   const double* __restrict__ A, long long lda,
                                   const double* __restrict__ B, long long ldb, double beta,
                                   double* C, long long ldc) {
  __shared__ double As[16][kGemmKT + 1];
  __shared__ double Bs[kGemmKT][17];
  pdl_wait();     // launched with programmatic stream serialization (chains of tiny products)
  pdl_trigger();  // a few CTAs: the successor may become resident at once
  const int row = blockIdx.y * 16 + threadIdx.y;
  const int col = blockIdx.x * 16 + threadIdx.x;
  double acc = 0.0;
  for (int kb = 0; kb < K; kb += kGemmKT) {
    double av[kGemmKT / 16], bv[kGemmKT / 16];
#pragma unroll
    for (int u = 0; u < kGemmKT / 16; ++u) {
      const int ka = kb + u * 16 + threadIdx.x;  // A(row, ka)
      av[u] = 0.0;
      if (row < M && ka < K) av[u] = ta ? A[(long long)ka * lda + row] : A[(long long)row * lda + ka];
      const int kk = kb + u * 16 + threadIdx.y;  // B(kk, col)
      bv[u] = 0.0;
      if (col < N && kk < K) bv[u] = tb ? B[(long long)col * ldb + kk] : B[(long long)kk * ldb + col];
    }
#pragma unroll
    for (int u = 0; u < kGemmKT / 16; ++u) {
      As[threadIdx.y][u * 16 + threadIdx.x] = av[u];
      Bs[u * 16 + threadIdx.y][threadIdx.x] = bv[u];
    }
    __syncthreads();
    const int kend = K - kb < kGemmKT ? K - kb : kGemmKT;
    if (kend == kGemmKT) {
#pragma unroll 16
      for (int q = 0; q < kGemmKT; ++q) acc = fma(As[threadIdx.y][q], Bs[q][threadIdx.x], acc);
    } else {
      // same chain as the 16-wide slabs of the previous kernel: zero-padded up to a multiple of 16
      const int kpad = (kend + 15) / 16 * 16;
      for (int q = 0; q < kpad; ++q) acc = fma(As[threadIdx.y][q], Bs[q][threadIdx.x], acc);
    }
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
  pdl_launch(dgemm_small_kernel, grid, block, 0, c->stream, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta,
             C, ldc);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

// ---------------------------------------------------------------------------
// FP64 peak probes (roofline denominators; MEASURED_PEAKS.json has no FP64 entry):
// every thread runs `iters` x 8 independent chains of DMMA.8x8x4 (mode 1, 512 flop
// per warp-instruction per chain) or DFMA (mode 0, 2 flop per lane).
__global__ void fp64_peak_kernel(int mode, int iters, double* sink) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  if (mode == 1) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile(
            "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
            : "+d"(c[i][0]), "+d"(c[i][1])
            : "d"(a), "d"(b));
    }
  } else {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        c[i][0] = fma(a, c[i][0], b);
        c[i][1] = fma(b, c[i][1], a);
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) sink[0] = s;  // keep the chains live
}

int fp64_peak_launch(Ctx* c, int mode, int iters, double* sink, int* grid_out, int* block_out) {
  const int block = 256, grid = c->num_sms * 4;
  fp64_peak_kernel<<<grid, block, 0, c->stream>>>(mode, iters, sink);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  *grid_out = grid;
  *block_out = block;
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
