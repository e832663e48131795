// Tall-skinny fp64 GEMMs on B200: Gram (MultiVecInnerProd) and LinComb
// (MultiVecLinearComb).
//
//  gram     G = alpha X'Y + beta G   multivec.py:84-112, _cy.pyx:26-50, orth.py:139-140,164,242,288
//  lincomb  Y = alpha X C + beta Y   solver.py:300,333,376; orth.py:144,175,184,264,291
//
// Both stream an n-long, k-wide row-major panel once from HBM.  Shapes on the
// hot path are k ~ 16..600, so they are HBM-bound (Gram with k1*k2/(k1+k2)
// small, LinComb with small d) up to FP64-bound (RR update m x d = 200 x 160).
// B200 has no FP64 tcgen05 kind, so the FP64 work runs on the FFMA64 pipe;
// the design goal is to keep enough bytes in flight: every CTA streams its
// panel through a 3-stage cp.async (LDGSTS) shared-memory ring (16-byte copies
// when the row runs are 16-byte aligned), and each thread keeps a 4x4 register
// micro-tile so shared-memory reads stay at 1 LDS.64 per 2 FMAs.
//
// Gram splits the n-long contraction into row slabs (grid = tiles x slabs, a
// few CTAs per SM); each CTA reduces its row groups in shared memory and writes
// one partial tile; a second kernel sums the slab partials with one warp per
// output in a fixed order.  The result is bit-identical run to run (the
// reference's `deterministic` contract, test_kernels.py:74-85).

#include "common.cuh"

namespace gcg {

extern int64_t g_launches;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Copy `cols` doubles of row `row` (global, starting at src) into smem dst,
// element stride 1; zero-fill beyond `valid`.  VEC16: 16-byte copies (src and
// dst 16-byte aligned, cols even).
template <bool VEC16>
__device__ __forceinline__ void stage_row_elems(double* dst, const double* src, int idx,
                                                int valid, const double* safe) {
  if (VEC16) {
    const int e = idx * 2;
    const int nb = valid - e >= 2 ? 16 : (valid - e == 1 ? 8 : 0);
    cp_async16(dst + e, nb ? src + e : safe, nb);
  } else {
    cp_async8(dst + idx, idx < valid ? src + idx : safe, idx < valid);
  }
}

// ---------------------------------------------------------------------------
// Gram

constexpr int kStages = 3;

template <int BM, int BN, int R, bool VEC16>
__global__ void __launch_bounds__(256) gram2_kernel(long long n, int k1, int k2,
                                                    const double* __restrict__ X, long long ldx,
                                                    const double* __restrict__ Y, long long ldy,
                                                    long long rows_per_slab, double* part) {
  constexpr int TM = 4, TN = 4;
  constexpr int TX = BN / TN, TY = BM / TM, TT = TX * TY, G = 256 / TT;
  constexpr int W = BM + BN + 2;  // padded smem row (doubles)
  constexpr int V = VEC16 ? 2 : 1;
  extern __shared__ __align__(16) double smg[];
  const int tm0 = blockIdx.x * BM, tn0 = blockIdx.y * BN;
  const long long r0 = (long long)blockIdx.z * rows_per_slab;
  long long r1 = r0 + rows_per_slab;
  if (r1 > n) r1 = n;
  const int tid = threadIdx.x;
  const int grp = tid / TT, t = tid % TT, tx = t % TX, ty = t / TX;
  const int vx = min(BM, k1 - tm0), vy = min(BN, k2 - tn0);  // valid columns of the tiles
  const int nch = (int)((r1 - r0 + R - 1) / R);

  auto load = [&](int ch, int st) {
    const long long rb = r0 + (long long)ch * R;
    constexpr int PX = BM / V, PY = BN / V, P = PX + PY;
    for (int e = tid; e < R * P; e += 256) {
      const int rr = e / P, cc = e % P;
      const long long row = rb + rr;
      double* dst = smg + (st * R + rr) * W;
      const bool ok = row < r1;
      if (cc < PX)
        stage_row_elems<VEC16>(dst, X + (ok ? row : r0) * ldx + tm0, cc, ok ? vx : 0, X);
      else
        stage_row_elems<VEC16>(dst + BM, Y + (ok ? row : r0) * ldy + tn0, cc - PX, ok ? vy : 0, Y);
    }
  };

  double acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0;

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nch) load(s, s);
    cp_commit();
  }
  for (int ch = 0; ch < nch; ++ch) {
    cp_wait<kStages - 2>();
    __syncthreads();
    if (ch + kStages - 1 < nch) load(ch + kStages - 1, (ch + kStages - 1) % kStages);
    cp_commit();
    const double* base = smg + (ch % kStages) * R * W;
#pragma unroll 2
    for (int rr = grp; rr < R; rr += G) {
      const double* rowp = base + rr * W;
      double xv[TM], yv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) xv[i] = rowp[ty + i * TY];
#pragma unroll
      for (int j = 0; j < TN; ++j) yv[j] = rowp[BM + tx + j * TX];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(xv[i], yv[j], acc[i][j]);
    }
  }
  cp_wait<0>();
  __syncthreads();
  // combine the G row groups in a fixed order
  double* red = smg;  // G * BM * BN doubles (<= 4096)
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) red[(grp * BM + ty + i * TY) * BN + tx + j * TX] = acc[i][j];
  __syncthreads();
  double* out = part + (long long)blockIdx.z * k1 * k2;
  for (int e = tid; e < BM * BN; e += 256) {
    const int rr = e / BN, cc = e % BN;
    double s = 0.0;
#pragma unroll
    for (int g = 0; g < G; ++g) s += red[g * BM * BN + e];
    if (tm0 + rr < k1 && tn0 + cc < k2) out[(long long)(tm0 + rr) * k2 + tn0 + cc] = s;
  }
}

// one warp per output: lanes stride the slabs, fixed shuffle tree (deterministic)
__global__ void gram_finish2_kernel(int k1, int k2, int nslab, const double* __restrict__ part,
                                    double alpha, double beta, double* G, long long grs,
                                    long long gcs) {
  const long long e = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (e >= (long long)k1 * k2) return;
  const long long kk = (long long)k1 * k2;
  double s = 0.0;
  for (int q = lane; q < nslab; q += 32) s += part[q * kk + e];
  s = warp_sum(s);
  if (lane == 0) {
    const int r = (int)(e / k2), c = (int)(e % k2);
    double* g = G + r * grs + c * gcs;
    *g = (beta == 0.0) ? alpha * s : fma(alpha, s, beta * *g);
  }
}

static inline bool al16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

template <int BM, int BN>
static int gram_go(Ctx* c, long long n, int k1, int k2, const double* X, long long ldx,
                   const double* Y, long long ldy, double* part, long long rps, int nslab,
                   bool vec) {
  constexpr int R = 32;
  const size_t sm = sizeof(double) * (size_t)kStages * R * (BM + BN + 2);
  const size_t need = sm > 4096 * sizeof(double) ? sm : 4096 * sizeof(double);
  dim3 grid((k1 + BM - 1) / BM, (k2 + BN - 1) / BN, nslab);
  if (vec) {
    auto kern = gram2_kernel<BM, BN, R, true>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need);
    kern<<<grid, 256, need, c->stream>>>(n, k1, k2, X, ldx, Y, ldy, rps, part);
  } else {
    auto kern = gram2_kernel<BM, BN, R, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need);
    kern<<<grid, 256, need, c->stream>>>(n, k1, k2, X, ldx, Y, ldy, rps, part);
  }
  return GCG_OK;
}

int gram_launch(Ctx* c, long long n, int k1, int k2, const double* X, long long ldx,
                const double* Y, long long ldy, double alpha, double beta, double* G,
                long long grs, long long gcs) {
  if (k1 <= 0 || k2 <= 0) return GCG_OK;
  const int BM = k1 <= 16 ? 16 : (k1 <= 32 ? 32 : 64);
  const int BN = k2 <= 16 ? 16 : (k2 <= 32 ? 32 : 64);
  const long long tiles = (long long)((k1 + BM - 1) / BM) * ((k2 + BN - 1) / BN);
  // ~3 CTAs per SM in total, slabs a multiple of the 32-row stage
  long long nslab = (3LL * c->num_sms + tiles - 1) / tiles;
  const long long max_slab = (n + 127) / 128;
  if (nslab > max_slab) nslab = max_slab;
  if (nslab < 1) nslab = 1;
  if (nslab > 65535) nslab = 65535;
  long long rps = (n + nslab - 1) / nslab;
  rps = (rps + 31) / 32 * 32;
  nslab = (n + rps - 1) / rps;
  if (nslab < 1) nslab = 1;
  GCG_TRY(ensure(c->partials, sizeof(double) * (size_t)nslab * k1 * k2));
  double* part = (double*)c->partials.ptr;
  const bool vec = (ldx % 2 == 0) && (ldy % 2 == 0) && al16(X) && al16(Y) && (BM % 2 == 0);
  const int ps = prof_start(c, PROF_GRAM, 8.0 * n * (X == Y ? k1 : k1 + k2));
#define GRAM_CASE(bm, bn) \
  if (BM == bm && BN == bn) gram_go<bm, bn>(c, n, k1, k2, X, ldx, Y, ldy, part, rps, (int)nslab, vec)
  GRAM_CASE(16, 16);
  else GRAM_CASE(16, 32);
  else GRAM_CASE(16, 64);
  else GRAM_CASE(32, 16);
  else GRAM_CASE(32, 32);
  else GRAM_CASE(32, 64);
  else GRAM_CASE(64, 16);
  else GRAM_CASE(64, 32);
  else GRAM_CASE(64, 64);
#undef GRAM_CASE
  prof_stop(c, ps);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  const long long outs = (long long)k1 * k2;
  gram_finish2_kernel<<<(unsigned)((outs * 32 + 255) / 256), 256, 0, c->stream>>>(
      k1, k2, (int)nslab, part, alpha, beta, G, grs, gcs);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

// ---------------------------------------------------------------------------
// LinComb  Y = alpha X C + beta Y

template <int BM, int BN, bool VEC16>
__global__ void __launch_bounds__(256) lincomb2_kernel(long long n, int m, int d, double alpha,
                                                       const double* __restrict__ X,
                                                       long long ldx,
                                                       const double* __restrict__ C,
                                                       long long ldc, double beta, double* Y,
                                                       long long ldy) {
  constexpr int BK = 16;
  constexpr int TM = 4, TN = 4, TX = BN / TN, TY = BM / TM;
  static_assert(TX * TY == 256, "256 threads");
  constexpr int XW = BK + 2;  // padded X row in smem
  constexpr int CW = BN + 2;
  constexpr int XS = BM * XW, CS = BK * CW;  // doubles per stage
  constexpr int V = VEC16 ? 2 : 1;
  extern __shared__ __align__(16) double sml[];
  double* xs = sml;
  double* cs = sml + kStages * XS;
  const long long r0 = (long long)blockIdx.x * BM;
  const int c0 = blockIdx.y * BN;
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  const int nk = (m + BK - 1) / BK;
  const int vc = min(BN, d - c0);

  auto load = [&](int kb, int st) {
    const int k0 = kb * BK;
    const int vk = min(BK, m - k0);
    constexpr int PX = BK / V;
    for (int e = tid; e < BM * PX; e += 256) {
      const int rr = e / PX, cc = e % PX;
      const long long row = r0 + rr;
      const bool ok = row < n;
      stage_row_elems<VEC16>(xs + st * XS + rr * XW, X + (ok ? row : 0) * ldx + k0, cc,
                             ok ? vk : 0, X);
    }
    for (int e = tid; e < BK * BN; e += 256) {
      const int kk = e / BN, cc = e % BN;
      const bool ok = kk < vk && cc < vc;
      cp_async8(cs + st * CS + kk * CW + cc, ok ? C + (long long)(k0 + kk) * ldc + c0 + cc : C,
                ok);
    }
  };

  double acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0;
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nk) load(s, s);
    cp_commit();
  }
  for (int kb = 0; kb < nk; ++kb) {
    cp_wait<kStages - 2>();
    __syncthreads();
    if (kb + kStages - 1 < nk) load(kb + kStages - 1, (kb + kStages - 1) % kStages);
    cp_commit();
    const double* xb = xs + (kb % kStages) * XS;
    const double* cb = cs + (kb % kStages) * CS;
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double xv[TM], cv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) xv[i] = xb[(ty + i * TY) * XW + kk];
#pragma unroll
      for (int j = 0; j < TN; ++j) cv[j] = cb[kk * CW + tx + j * TX];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(xv[i], cv[j], acc[i][j]);
    }
  }
  cp_wait<0>();
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

template <int BM, int BN>
static void lincomb_go(Ctx* c, long long n, int m, int d, double alpha, const double* X,
                       long long ldx, const double* C, long long ldc, double beta, double* Y,
                       long long ldy, bool vec) {
  const size_t sm = sizeof(double) * (size_t)kStages * (BM * (16 + 2) + 16 * (BN + 2));
  dim3 grid((unsigned)((n + BM - 1) / BM), (d + BN - 1) / BN);
  if (vec) {
    auto kern = lincomb2_kernel<BM, BN, true>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    kern<<<grid, 256, sm, c->stream>>>(n, m, d, alpha, X, ldx, C, ldc, beta, Y, ldy);
  } else {
    auto kern = lincomb2_kernel<BM, BN, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    kern<<<grid, 256, sm, c->stream>>>(n, m, d, alpha, X, ldx, C, ldc, beta, Y, ldy);
  }
}

int lincomb_launch(Ctx* c, long long n, int m, int d, double alpha, const double* X,
                   long long ldx, const double* C, long long ldc, double beta, double* Y,
                   long long ldy) {
  if (n <= 0 || d <= 0) return GCG_OK;
  const int ps =
      prof_start(c, PROF_LINCOMB, 8.0 * n * (m + d) + (beta != 0.0 ? 8.0 * n * d : 0.0));
  // 16-byte staging needs every X row run 16-byte aligned (XW = 18 keeps smem aligned)
  const bool vec = (ldx % 2 == 0) && al16(X);
  if (d <= 16)
    lincomb_go<256, 16>(c, n, m, d, alpha, X, ldx, C, ldc, beta, Y, ldy, vec);
  else if (d <= 32)
    lincomb_go<128, 32>(c, n, m, d, alpha, X, ldx, C, ldc, beta, Y, ldy, vec);
  else
    lincomb_go<64, 64>(c, n, m, d, alpha, X, ldx, C, ldc, beta, Y, ldy, vec);
  prof_stop(c, ps);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

}  // namespace gcg
