// Dense symmetric eigensolver for the Rayleigh-Ritz matrices on B200.
//
// Reference: sym_eig_full (dense.py:74-82: scipy.linalg.eigh -> LAPACK ?syevr)
// with the sign rule _fix_signs (dense.py:63-71).  At the BASELINE shapes the
// projected matrix has order m = 120..500; cuSOLVER syevd spends ~1.9 ms on
// m = 200 (a blocked tridiagonalisation of many small launches, then divide and
// conquer) — 15-20 % of a cfg2 solve.  This path replaces it for m <= 224 with
// five short kernels and no host synchronisation:
//
//   1. tridiag_kernel   Householder reduction A = Q T Q' (LAPACK dsytd2, lower)
//                       in ONE CTA: the packed lower triangle (m(m+1)/2
//                       doubles, 201 KB at m = 224) lives in shared memory, so
//                       each of the m-2 steps (reflector, symmetric mat-vec,
//                       rank-2 update) runs at shared-memory speed with a few
//                       block barriers instead of kernel launches.
//   2. bisect_kernel    eigenvalues of T by Sturm-count multisection: one warp
//                       per eigenvalue, 32 points per round (log33 of the
//                       range, ~11 rounds), dstebz's pivmin safeguard.
//   3. invit_kernel     eigenvectors of T by inverse iteration (dstein): one
//                       thread per eigenvalue, LU of T - lambda I with partial
//                       pivoting (dlagtf / dlagts, tiny pivots perturbed); the
//                       second pass reuses the factors.
//   4. cluster_kernel   classical Gram-Schmidt twice inside each tight cluster
//                       (gaps <= 1e-7 ||T||_1), then normalisation; (3)+(4) run
//                       twice; then a global first-order Loewdin step.
//   5. backtr_kernel    Z = Q Z_T, reflectors applied in reverse order, each warp
//                       holding 4 columns of Z in registers.
// then the reference's sign rule (vec_fix_kernel in dense.cu).
//
// Every reduction has a fixed order (bit-stable run to run).  Eigenvalues agree
// with LAPACK to O(eps ||A||); eigenvectors of (near-)degenerate eigenvalues are
// any orthonormal basis of their invariant subspace, as with any eigensolver.

#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "async.cuh"
#include "common.cuh"

namespace gcg {

extern int64_t g_launches;

constexpr int kTriThreads = 1024;
constexpr int kEigMaxM = 224;

__host__ __device__ inline int tri_off(int m, int j) { return j * m - (j * (j - 1)) / 2; }

static size_t tri_smem(int m) {
  // packed lower triangle | (v, w) previous step | (v, w) current | p | slots
  return sizeof(double) * ((size_t)m * (m + 1) / 2 + 1 + 9 * (size_t)m + 64);
}

// 1. Householder tridiagonalisation (dsytd2, UPLO = 'L') in one CTA, the packed
// lower triangle in shared memory.  Step j:
//   B  (warps 0-7, a thread per row) column j gets the deferred rank-2 update of
//      step j-1, then the reflector v_j, tau_j (dlarfg; rsqrt / reciprocals);
//   C1 row i (4 warps: columns split mod 4, lane = row so one access reads 32
//      consecutive rows of a column) applies step j-1's deferred update to its
//      lower-part elements L(i, c), s0 <= c <= i, stores them and accumulates
//      sum_c L(i, c) v_c;
//   C2 after a barrier the same threads add the upper part sum_{c > i} L(c, i) v_c
//      (column i of the packed storage, already updated), so p = A22 v needs no
//      scatter: each row's sum is its 4 quarter partials, added in fixed order;
//   D  (warps 0-7) w = tau p - (tau^2 / 2)(p'v) v, the next deferred update; D of
//      step j and B of step j+1 run back to back between named barriers.
// Every element is read and written once per step; all sums have a fixed order.
// Outputs: d[m], e[m-1], tau[m-1] and the reflectors in Vr (column-major m x m,
// column j holds v_j in rows j+1..m-1, v_j[j+1] = 1).
__global__ void __launch_bounds__(kTriThreads)
    tridiag_kernel(int m, const double* __restrict__ A, long long lda, int sym, double* d,
                   double* e, double* tau, double* Vr) {
  extern __shared__ double tsm[];
  double* L = tsm;                          // packed lower triangle, by columns
  // (v, w) pairs: previous step's (the deferred update) and the current step's
  double2* P = reinterpret_cast<double2*>(L + (((size_t)m * (m + 1) / 2 + 1) & ~(size_t)1));
  double2* Q = P + m;
  double* part = reinterpret_cast<double*>(Q + m);  // [4][m] row partial sums of p
  double* vcur = part + 4 * m;                    // this step's v as plain doubles (C2's
                                                  // per-lane reads: 8-byte stride)
  double* slot = vcur + m;                        // scalars
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // load: coalesced row-major reads, scattered shared-memory writes
  for (int idx = tid; idx < m * m; idx += kTriThreads) {
    const int i = idx / m, c = idx - i * m;
    if (i >= c) {
      double x = A[(long long)i * lda + c];
      if (sym) x = 0.5 * (x + A[(long long)c * lda + i]);
      L[tri_off(m, c) + (i - c)] = x;
    }
  }
  for (int i = tid; i < m; i += kTriThreads) P[i] = make_double2(0.0, 0.0);
  __syncthreads();
  const int row = 32 * (warp & 7) + lane, q = warp >> 3;  // C1: row, column residue mod 4
  double* redb = slot + 8;   // [8] warp partials of B's norm
  double* redd = slot + 16;  // [8] warp partials of D's p'v
  // B. column j: deferred update with (v_{j-1}, w_{j-1}), then the reflector (dlarfg;
  // rsqrt / reciprocals instead of divisions).  Warps 0-7, thread t owns row j + t;
  // the norm is a fixed-order sum of 8 warp partials (named barrier 1).
  auto phase_B = [&](int j) {
    const int oj = tri_off(m, j);
    const double2 pj = P[j];
    const int i = j + tid;
    double x = 0.0;
    if (i < m) {
      const double2 pi = P[i];
      x = L[oj + tid] - fma(pi.x, pj.y, pi.y * pj.x);
      L[oj + tid] = x;
    }
    double sq = (tid >= 2 && i < m) ? x * x : 0.0;
    sq = warp_sum(sq);
    if (lane == 0) redb[warp] = sq;
    if (tid == 0) slot[2] = x;  // d_j
    if (tid == 1) slot[3] = x;  // alpha
    asm volatile("bar.sync 1, 256;" ::: "memory");
    double s = 0.0;
#pragma unroll
    for (int w2 = 0; w2 < 8; ++w2) s += redb[w2];
    const double alpha = slot[3], djj = slot[2];
    double t = 0.0, beta = alpha, scal = 0.0;
    if (s > 0.0) {
      const double nrm2 = fma(alpha, alpha, s);
      const double rn = rsqrt(nrm2);  // beta = -sign(alpha) ||x||
      beta = alpha >= 0.0 ? -nrm2 * rn : nrm2 * rn;
      t = (beta - alpha) * __drcp_rn(beta);
      scal = __drcp_rn(alpha - beta);
    }
    if (i < m) {
      const double vi = i == j ? 0.0 : (i == j + 1 ? 1.0 : x * scal);
      Q[i].x = t != 0.0 ? vi : 0.0;
      vcur[i] = t != 0.0 ? vi : 0.0;
      if (i > j) Vr[(long long)j * m + i] = vi;
    }
    if (tid == 0) {
      d[j] = djj;
      e[j] = beta;
      tau[j] = t;
      slot[0] = t;
    }
  };
  // D. p = t * (sum of the 4 row partials, fixed order), w = p - (t/2)(p'v) v; warps 0-7
  auto phase_D = [&](int s0, double t) {
    const int i = s0 + tid;
    double pl = 0.0, dv = 0.0;
    if (i < m) {
      pl = t * (((part[i] + part[m + i]) + part[2 * m + i]) + part[3 * m + i]);
      dv = pl * Q[i].x;
    }
    dv = warp_sum(dv);
    if (lane == 0) redd[warp] = dv;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    double ds = 0.0;
#pragma unroll
    for (int w2 = 0; w2 < 8; ++w2) ds += redd[w2];
    const double a2 = -0.5 * t * ds;
    if (i < m) Q[i].y = fma(a2, Q[i].x, pl);
    asm volatile("bar.sync 1, 256;" ::: "memory");  // w_{s0} is read by every B thread
  };
  if (warp < 8) phase_B(0);
  __syncthreads();
  for (int j = 0; j + 2 < m; ++j) {
    const int s0 = j + 1;
    const double t = slot[0];
    // C1. lower-part elements L(row, c), s0 <= c <= row: warp w takes row block
    // (w & 7) (lane = row: 32 consecutive rows of one column per access, conflict-
    // free) and the columns c = s0 + (w >> 3) mod 4; 4-way unrolled.
    double acc = 0.0;
    const bool rok = row >= s0 && row < m;
    if (rok) {
      const double2 pr = P[row];
      const double vpi = pr.x, wpi = pr.y;
      int c = s0 + q;
      int a = tri_off(m, c) + (row - c);
      int da = 4 * m - 4 * c - 10;  // a(c + 4) - a(c)
      for (; c + 12 <= row; c += 16) {
        const int a0 = a, a1 = a0 + da, a2 = a1 + da - 16, a3 = a2 + da - 32;
        double x0 = L[a0], x1 = L[a1], x2 = L[a2], x3 = L[a3];
        const double2 q0 = P[c], q1 = P[c + 4], q2 = P[c + 8], q3 = P[c + 12];
        x0 -= fma(vpi, q0.y, wpi * q0.x);
        x1 -= fma(vpi, q1.y, wpi * q1.x);
        x2 -= fma(vpi, q2.y, wpi * q2.x);
        x3 -= fma(vpi, q3.y, wpi * q3.x);
        L[a0] = x0;
        L[a1] = x1;
        L[a2] = x2;
        L[a3] = x3;
        acc = fma(x0, Q[c].x, acc);
        acc = fma(x1, Q[c + 4].x, acc);
        acc = fma(x2, Q[c + 8].x, acc);
        acc = fma(x3, Q[c + 12].x, acc);
        a = a3 + da - 48;
        da -= 64;
      }
      for (; c <= row; c += 4) {
        const double2 qc = P[c];
        const double x = L[a] - fma(vpi, qc.y, wpi * qc.x);
        L[a] = x;
        acc = fma(x, Q[c].x, acc);
        a += da;
        da -= 16;
      }
    }
    __syncthreads();
    // C2. upper part of the same row: L(c, row), c = row + 1 + q + 4k — column `row`
    // of the packed storage (already updated), walked by the same thread
    if (rok) {
      const double* colr = L + tri_off(m, row) - row;
      int c = row + 1 + q;
      for (; c + 12 < m; c += 16) {
        const double y0 = colr[c], y1 = colr[c + 4], y2 = colr[c + 8], y3 = colr[c + 12];
        acc = fma(y0, vcur[c], acc);
        acc = fma(y1, vcur[c + 4], acc);
        acc = fma(y2, vcur[c + 8], acc);
        acc = fma(y3, vcur[c + 12], acc);
      }
      for (; c < m; c += 4) acc = fma(colr[c], vcur[c], acc);
    }
    if (row < m) part[q * m + row] = acc;
    __syncthreads();
    if (warp < 8) phase_D(s0, t);
    double2* tq = P;  // the current (v, w) become the deferred update of the next step
    P = Q;
    Q = tq;
    if (warp < 8 && j + 3 < m) phase_B(j + 1);
    __syncthreads();
  }
  // deferred update of the last 2 x 2 block, then its entries
  if (tid == 0) {
    if (m >= 2) {
      const int o2 = tri_off(m, m - 2), o1 = tri_off(m, m - 1);
      const double2 p2 = P[m - 2], p1 = P[m - 1];
      const double a = L[o2] - fma(p2.x, p2.y, p2.y * p2.x);
      const double b = L[o2 + 1] - fma(p1.x, p2.y, p1.y * p2.x);
      const double c = L[o1] - fma(p1.x, p1.y, p1.y * p1.x);
      d[m - 2] = a;
      e[m - 2] = b;
      tau[m - 2] = 0.0;
      d[m - 1] = c;
    } else {
      d[0] = L[0];
    }
  }
}

// Sturm count (number of eigenvalues of T below x) by the three-term determinant
// recurrence p_k = (d_k - x) p_{k-1} - e_{k-1}^2 p_{k-2}: one FMA on the dependent
// chain per step instead of a division.  T is pre-scaled to ||T|| ~ 1 and the
// pair (p_k, p_{k-1}) is rescaled by exact powers of two every 8 steps; an exact
// zero takes a tiny value of the opposite sign (dstebz's -pivmin).
__device__ __forceinline__ int sturm_count(int m, const double* d, const double* e2, double x) {
  double p2 = 1.0, p1 = d[0] - x;
  if (p1 == 0.0) p1 = -0x1p-60;
  int cnt = p1 < 0.0;
#pragma unroll 8
  for (int k = 1; k < m; ++k) {
    double p = fma(d[k] - x, p1, -e2[k - 1] * p2);
    if (p == 0.0) p = -0x1p-60 * p1;
    cnt += signbit(p) != signbit(p1);
    p2 = p1;
    p1 = p;
    if ((k & 7) == 0) {
      const double a = fabs(p1);
      if (a > 0x1p400 || a < 0x1p-400) {
        const double sc = ldexp(1.0, -ilogb(a));
        p1 *= sc;
        p2 *= sc;
      }
    }
  }
  return cnt;
}

// 2. Eigenvalue idx (0-based, ascending) by 33-way multisection, one warp each.
__global__ void __launch_bounds__(256) bisect_kernel(int m, const double* __restrict__ d,
                                                     const double* __restrict__ e, double* lam,
                                                     double* norms) {
  __shared__ double sd[kEigMaxM], se2[kEigMaxM];
  __shared__ double rlo[8], rhi[8], rone[8];
  __shared__ double sgl, sgu, sscale;
  // Gershgorin interval and ||T||_1 (= ||T||_inf), block-parallel
  double gl = INFINITY, gu = -INFINITY, one = 0.0;
  for (int k = threadIdx.x; k < m; k += blockDim.x) {
    const double r = (k > 0 ? fabs(e[k - 1]) : 0.0) + (k + 1 < m ? fabs(e[k]) : 0.0);
    gl = fmin(gl, d[k] - r);
    gu = fmax(gu, d[k] + r);
    one = fmax(one, fabs(d[k]) + r);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    gl = fmin(gl, __shfl_xor_sync(0xffffffffu, gl, o));
    gu = fmax(gu, __shfl_xor_sync(0xffffffffu, gu, o));
    one = fmax(one, __shfl_xor_sync(0xffffffffu, one, o));
  }
  if ((threadIdx.x & 31) == 0) {
    rlo[threadIdx.x >> 5] = gl;
    rhi[threadIdx.x >> 5] = gu;
    rone[threadIdx.x >> 5] = one;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      gl = fmin(gl, rlo[w]);
      gu = fmax(gu, rhi[w]);
      one = fmax(one, rone[w]);
    }
    const double tn = fmax(fabs(gl), fabs(gu));
    const double sc = tn > 0.0 ? ldexp(1.0, -ilogb(tn)) : 1.0;  // exact power of two
    sscale = sc;
    sgl = gl * sc;
    sgu = gu * sc;
    if (blockIdx.x == 0) norms[0] = one;
  }
  __syncthreads();
  const double sc = sscale;
  for (int k = threadIdx.x; k < m; k += blockDim.x) {
    sd[k] = d[k] * sc;
    const double ek = k + 1 < m ? e[k] * sc : 0.0;
    se2[k] = ek * ek;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int idx = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (idx >= m) return;
  const double eps = 1.1102230246251565e-16;  // 2^-53
  const double tn = fmax(fabs(sgl), fabs(sgu));
  const double pad = 2.0 * eps * tn * m + 0x1p-900;
  double lo = sgl - pad, hi = sgu + pad;  // count(lo) = 0 <= idx < m = count(hi)
  for (int round = 0; round < 40; ++round) {
    const double width = hi - lo;
    if (width <= 2.0 * eps * fmax(fabs(lo), fabs(hi)) || width <= eps * tn) break;
    const double x = lo + width * (double)(lane + 1) / 33.0;
    const int cnt = sturm_count(m, sd, se2, x);
    const unsigned above = __ballot_sync(0xffffffffu, cnt > idx);
    const int f = above ? __ffs(above) - 1 : 32;  // first point above eigenvalue idx
    const double nlo = f == 0 ? lo : lo + width * (double)f / 33.0;
    const double nhi = f == 32 ? hi : lo + width * (double)(f + 1) / 33.0;
    if (!(nhi < hi || nlo > lo)) break;  // no progress (rounding): converged
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) lam[idx] = 0.5 * (lo + hi) / sc;
}

// deterministic pseudo-random start vector entry (dstein starts from uniform(-1, 1))
__device__ __forceinline__ double start_entry(int j, int k) {
  uint64_t x = ((uint64_t)(j + 1) << 32) ^ (uint64_t)(k + 0x9E3779B9u);
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return (double)(x >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

// 3. Inverse iteration for eigenvector j of T: solve (T - lam_j I) z = b by LU with
// partial pivoting (dlagtf), b = start vector (pass 0) or the current column of Z
// (pass 1); writes z (unnormalised) into column j of Z (column-major, ld m).
// Per-thread factors interleaved [k][m] in W (coalesced across threads).  Pass 0
// factors (one reciprocal per step on the dependent chain) and keeps the
// multipliers and row swaps; pass 1 only re-runs the substitutions (one FMA per
// step on the chain).  The backward pass multiplies by stored reciprocal pivots.
__global__ void __launch_bounds__(32) invit_kernel(int m, const double* d, const double* e,
                                                   const double* __restrict__ lam,
                                                   double* __restrict__ Z, double* __restrict__ W,
                                                   int pass,
                                                   const double* __restrict__ norms) {
  __shared__ double sdv[kEigMaxM], sev[kEigMaxM];
  extern __shared__ double ysm[];  // [m][32]: this thread's forward-substituted rhs
  for (int k = threadIdx.x; k < m; k += blockDim.x) {
    sdv[k] = d[k];
    sev[k] = k + 1 < m ? e[k] : 0.0;
  }
  __syncthreads();
  d = sdv;
  e = sev;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const size_t mm = (size_t)m * m;
  double* R1 = W;            // 1 / U(k, k)
  double* U2 = W + mm;
  double* U3 = W + 2 * mm;
  double* const Yb = ysm + threadIdx.x;  // Yb[k * 32]
#define YS(k) Yb[(size_t)(k) * 32]
  double* ML = W + 4 * mm;   // multipliers; negative zero-bias flag in SW
  double* SW = W + 5 * mm;   // 1.0 where rows k, k+1 were swapped
  double* z = Z + (size_t)j * m;
  if (pass == 0) {
    const double lj = lam[j];
    const double tnorm = norms[0];
    const double tiny = fmax(tnorm, 1e-300) * 2.220446049250313e-16;
    auto fixp = [&](double u) { return fabs(u) < tiny ? (u < 0.0 ? -tiny : tiny) : u; };
    double dg = d[0] - lj;            // current pivot-row diagonal
    double sp = m > 1 ? e[0] : 0.0;   // current pivot-row superdiagonal
    double yk = start_entry(j, 0);
#pragma unroll 4
    for (int k = 0; k + 1 < m; ++k) {
      const double sub = e[k];                        // T(k+1, k)
      const double a1 = d[k + 1] - lj;                // T(k+1, k+1)
      const double s1 = k + 2 < m ? e[k + 1] : 0.0;   // T(k+1, k+2)
      const double bk1 = start_entry(j, k + 1);
      const size_t o = (size_t)k * m + j;
      // partial pivoting without divergence: swap rows k, k+1 when |sub| > |dg|
      const bool sw = fabs(sub) > fabs(dg);
      const double rp = __drcp_rn(sw ? sub : fixp(dg));
      const double mult = (sw ? dg : sub) * rp;
      R1[o] = rp;
      U2[o] = sw ? a1 : sp;
      U3[o] = sw ? s1 : 0.0;
      YS(k) = sw ? bk1 : yk;
      ML[o] = mult;
      SW[o] = sw ? 1.0 : 0.0;
      yk = fma(-mult, sw ? bk1 : yk, sw ? yk : bk1);
      dg = fma(-mult, sw ? a1 : sp, sw ? sp : a1);
      sp = sw ? -mult * s1 : s1;
    }
    R1[(size_t)(m - 1) * m + j] = __drcp_rn(fixp(dg));
    YS(m - 1) = yk;
  } else {
    // forward substitution of the new right-hand side with the stored factors
    // loads are batched 8 steps ahead of the chain: the stores to Y would otherwise
    // keep the compiler from hoisting the ML / SW / z loads (same base pointer)
    double yk = z[0];
    constexpr int B = 8;
    int k = 0;
    for (; k + B < m; k += B) {
      double mlb[B], swb[B], bb[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const size_t o = (size_t)(k + u) * m + j;
        mlb[u] = ML[o];
        swb[u] = SW[o];
        bb[u] = z[k + u + 1];
      }
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const bool sw = swb[u] != 0.0;
        YS(k + u) = sw ? bb[u] : yk;
        yk = fma(-mlb[u], sw ? bb[u] : yk, sw ? yk : bb[u]);
      }
    }
    for (; k + 1 < m; ++k) {
      const size_t o = (size_t)k * m + j;
      const double bk1 = z[k + 1];
      const bool sw = SW[o] != 0.0;
      YS(k) = sw ? bk1 : yk;
      yk = fma(-ML[o], sw ? bk1 : yk, sw ? yk : bk1);
    }
    YS(m - 1) = yk;
  }
  double x2 = 0.0, x1 = YS(m - 1) * R1[(size_t)(m - 1) * m + j];
  z[m - 1] = x1;
  {
    constexpr int B = 8;
    int k = m - 2;
    for (; k - B + 1 >= 0; k -= B) {
      double yb[B], u2[B], u3[B], r1[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const size_t o = (size_t)(k - u) * m + j;
        yb[u] = YS(k - u);
        u2[u] = U2[o];
        u3[u] = U3[o];
        r1[u] = R1[o];
      }
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const double x0 = (yb[u] - u2[u] * x1 - u3[u] * x2) * r1[u];
        z[k - u] = x0;
        x2 = x1;
        x1 = x0;
      }
    }
    for (; k >= 0; --k) {
      const size_t o = (size_t)k * m + j;
      const double x0 = (YS(k) - U2[o] * x1 - U3[o] * x2) * R1[o];
      z[k] = x0;
      x2 = x1;
      x1 = x0;
    }
  }
#undef YS
  // no normalisation here: the cluster kernel normalises every column (2-norm);
  // the unnormalised solution is at most ~1/eps times the start vector
}

// Eigenvalues closer than kTightGap ||T|| form a tight cluster: inverse iteration
// gives them vectors that are arbitrary inside the (near-)invariant subspace, so
// they are Gram-Schmidt orthogonalised.  Every other pair is already orthogonal to
// ~eps ||T|| / gap <= ~1e-9 and is finished by the global first-order Loewdin step
// (loewdin_*), which, like Gram-Schmidt, moves each vector only along eigenvectors
// whose eigenvalue differs by the gap that caused the error — residuals stay at
// eps ||T|| (dstein clusters at 1e-3 ||T|| instead, which on Rayleigh-Ritz spectra
// chains most eigenvalues into one long sequential Gram-Schmidt).
constexpr double kTightGap = 1e-7;

// 4. Orthonormalise each tight cluster (consecutive eigenvalues, gaps <= ortol):
// one CTA per potential cluster start; classical Gram-Schmidt twice per vector
// against the earlier members, then 2-norm normalisation (fixed-order sums).
__global__ void __launch_bounds__(256) cluster_kernel(int m, const double* __restrict__ lam,
                                                      double* Z, const double* __restrict__ norms) {
  __shared__ double red[8][33];
  __shared__ double coef[kEigMaxM];
  const int b = blockIdx.x;
  const double ortol = kTightGap * norms[0];
  if (b > 0 && lam[b] - lam[b - 1] <= ortol) return;  // not a cluster start
  int end = b + 1;
  while (end < m && lam[end] - lam[end - 1] <= ortol) ++end;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int jj = b; jj < end; ++jj) {
    double* zj = Z + (size_t)jj * m;
    for (int pass = 0; pass < 2 && jj > b; ++pass) {
      // coefficients c_i = z_i' z_j, one warp per earlier member (fixed order)
      for (int i = b + warp; i < jj; i += 8) {
        const double* zi = Z + (size_t)i * m;
        double s = 0.0;
        for (int k = lane; k < m; k += 32) s = fma(zi[k], zj[k], s);
        s = warp_sum(s);
        if (lane == 0) coef[i - b] = s;
      }
      __syncthreads();
      for (int k = tid; k < m; k += 256) {
        double x = zj[k];
        for (int i = b; i < jj; ++i) x = fma(-coef[i - b], Z[(size_t)i * m + k], x);
        zj[k] = x;
      }
      __syncthreads();
    }
    double s = 0.0;
    for (int k = tid; k < m; k += 256) s = fma(zj[k], zj[k], s);
    s = warp_sum(s);
    if (lane == 0) red[warp][0] = s;
    __syncthreads();
    double nrm2 = 0.0;
    for (int w2 = 0; w2 < 8; ++w2) nrm2 += red[w2][0];
    const double inv = nrm2 > 0.0 ? 1.0 / sqrt(nrm2) : 0.0;
    for (int k = tid; k < m; k += 256) zj[k] *= inv;
    __syncthreads();
  }
}

// 5. Z <- Q Z with Q = H_0 H_1 ... H_{m-3}: each warp owns kBtCols columns of Z in
// registers (lane holds rows lane + 32 s) and applies all reflectors last-first,
// with the next reflector's loads issued before the current one's reductions; no
// block barriers.
constexpr int kBtWarps = 8;
constexpr int kBtCols = 4;
constexpr int kBtRows = (kEigMaxM + 31) / 32;
constexpr int kBtChunk = 16;  // reflectors per shared-memory stage
static size_t backtr_smem(int m) { return sizeof(double) * 2 * kBtChunk * ((size_t)m + 1); }
__global__ void __launch_bounds__(32 * kBtWarps) backtr_kernel(int m, const double* __restrict__ Vr,
                                                               const double* __restrict__ tau,
                                                               double* Z) {
  extern __shared__ __align__(16) double bsm[];  // [2][kBtChunk][m] reflectors + [2][kBtChunk] tau
  double* vbuf = bsm;
  double* tbuf = bsm + 2 * kBtChunk * (size_t)m;
  const int lane = threadIdx.x & 31;
  const int col0 = (blockIdx.x * kBtWarps + (threadIdx.x >> 5)) * kBtCols;
  const bool live = col0 < m;
  double r[kBtCols][kBtRows];
#pragma unroll
  for (int cc = 0; cc < kBtCols; ++cc)
#pragma unroll
    for (int s = 0; s < kBtRows; ++s) {
      const int k = lane + 32 * s;
      r[cc][s] = (live && k < m && col0 + cc < m) ? Z[(size_t)(col0 + cc) * m + k] : 0.0;
    }
  // reflectors are applied last-first: chunk c covers j = jtop - c*kBtChunk down to ..-kBtChunk+1
  const int jtop = m - 3;
  const int nchunks = jtop >= 0 ? jtop / kBtChunk + 1 : 0;
  auto stage = [&](int cidx, int buf) {
    const int jhi = jtop - cidx * kBtChunk;
    const int cnt = min(kBtChunk, jhi + 1);
    double* dst = vbuf + (size_t)buf * kBtChunk * m;
    for (int e = threadIdx.x; e < cnt * m; e += blockDim.x) {
      const int q = e / m, k = e - q * m;
      const int j = jhi - q;
      cp_async8(dst + (size_t)q * m + k, Vr + (size_t)j * m + k, k > j);
    }
    if (threadIdx.x < cnt) cp_async8(tbuf + buf * kBtChunk + threadIdx.x, tau + jhi - threadIdx.x, true);
    cp_commit();
  };
  if (nchunks > 0) stage(0, 0);
  for (int cidx = 0; cidx < nchunks; ++cidx) {
    const int buf = cidx & 1;
    if (cidx + 1 < nchunks) {
      stage(cidx + 1, buf ^ 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const int jhi = jtop - cidx * kBtChunk;
    const int cnt = min(kBtChunk, jhi + 1);
    const double* vb = vbuf + (size_t)buf * kBtChunk * m;
    if (live) {
      for (int q = 0; q < cnt; ++q) {
        const double t = tbuf[buf * kBtChunk + q];
        if (t == 0.0) continue;
        const double* vj = vb + (size_t)q * m;
        double vv[kBtRows];
#pragma unroll
        for (int s = 0; s < kBtRows; ++s) {
          const int k = lane + 32 * s;
          vv[s] = k < m ? vj[k] : 0.0;  // zero-filled above the reflector's first row
        }
        double dot[kBtCols];
#pragma unroll
        for (int cc = 0; cc < kBtCols; ++cc) {
          dot[cc] = 0.0;
#pragma unroll
          for (int s = 0; s < kBtRows; ++s) dot[cc] = fma(vv[s], r[cc][s], dot[cc]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int cc = 0; cc < kBtCols; ++cc) dot[cc] += __shfl_xor_sync(0xffffffffu, dot[cc], o);
#pragma unroll
        for (int cc = 0; cc < kBtCols; ++cc) {
          const double f = t * dot[cc];
#pragma unroll
          for (int s = 0; s < kBtRows; ++s) r[cc][s] = fma(-f, vv[s], r[cc][s]);
        }
      }
    }
    __syncthreads();  // buffer 'buf' is restaged two chunks later
  }
  if (!live) return;
#pragma unroll
  for (int cc = 0; cc < kBtCols; ++cc)
#pragma unroll
    for (int s = 0; s < kBtRows; ++s) {
      const int k = lane + 32 * s;
      if (k < m && col0 + cc < m) Z[(size_t)(col0 + cc) * m + k] = r[cc][s];
    }
}

// 4b. Global first-order Loewdin orthonormalisation Z <- Z (3/2 I - 1/2 Z'Z) (the
// residual non-orthogonality after 4 is <= ~1e-9, so the result is orthonormal to
// ~1e-18).  G = Z'Z: one CTA per column j of G, one warp per entry (fixed order).
__global__ void __launch_bounds__(256) loewdin_gram_kernel(int m, const double* __restrict__ Z,
                                                           double* __restrict__ G) {
  const int j = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* zj = Z + (size_t)j * m;
  for (int i = warp; i < m; i += 8) {
    const double* zi = Z + (size_t)i * m;
    double s = 0.0;
    for (int k = lane; k < m; k += 32) s = fma(zi[k], zj[k], s);
    s = warp_sum(s);
    if (lane == 0) G[(size_t)j * m + i] = s;
  }
}
// Z2[:, j] = 3/2 z_j - 1/2 sum_i z_i G[i, j]; one CTA per column j, thread per row
__global__ void __launch_bounds__(256) loewdin_apply_kernel(int m, const double* __restrict__ Z,
                                                            const double* __restrict__ G,
                                                            double* __restrict__ Z2) {
  __shared__ double gj[kEigMaxM];
  const int j = blockIdx.x;
  for (int i = threadIdx.x; i < m; i += blockDim.x) gj[i] = G[(size_t)j * m + i];
  __syncthreads();
  for (int k = threadIdx.x; k < m; k += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s = fma(Z[(size_t)i * m + k], gj[i], s);
    Z2[(size_t)j * m + k] = fma(1.5, Z[(size_t)j * m + k], -0.5 * s);
  }
}

__global__ void vec_fix_kernel(int m, const double* Vcm, double* V, long long ldv);

bool dense_syev_tridiag_ok(int m) {
  static const char* impl = getenv("GCG_SYEV");
  if (impl && impl[0] == 'c') return false;  // GCG_SYEV=cusolver: A/B switch
  return m >= 3 && m <= kEigMaxM;
}

// w (m, ascending) and V (row-major, ldv; eigenvector j in column j, sign rule
// applied) of the symmetric m x m row-major A (symmetrised first when sym != 0).
int dense_syev_tridiag(Ctx* c, int m, const double* A, long long lda, int sym, double* w,
                       double* V, long long ldv) {
  if (m < 3 || m > kEigMaxM) return GCG_ERR_ARG;
  const size_t mm = (size_t)m * m;
  // workspace: d, e, tau (3m) | Vr (m^2) | Z (m^2) | inverse-iteration factors (6 m^2) | norms
  GCG_TRY(ensure(c->dense, sizeof(double) * (3 * (size_t)m + 8 * mm + 8) + 256));
  double* dd = (double*)c->dense.ptr;
  double* ee = dd + m;
  double* tt = ee + m;
  double* Vr = tt + m;
  double* Z = Vr + mm;
  double* W = Z + mm;
  double* norms = W + 6 * mm;
  const size_t smem = tri_smem(m);
  kernel_smem((const void*)tridiag_kernel, smem);
  tridiag_kernel<<<1, kTriThreads, smem, c->stream>>>(m, A, lda, sym, dd, ee, tt, Vr);
  bisect_kernel<<<(m + 7) / 8, 256, 0, c->stream>>>(m, dd, ee, w, norms);
  for (int pass = 0; pass < 2; ++pass) {
    const size_t ysm = sizeof(double) * 32 * (size_t)m;
    kernel_smem((const void*)invit_kernel, ysm);
    invit_kernel<<<(m + 31) / 32, 32, ysm, c->stream>>>(m, dd, ee, w, Z, W, pass, norms);
    cluster_kernel<<<m, 256, 0, c->stream>>>(m, w, Z, norms);
  }
  double* G = W;            // the inverse-iteration factors are dead now
  double* Z2 = W + mm;
  loewdin_gram_kernel<<<m, 256, 0, c->stream>>>(m, Z, G);
  loewdin_apply_kernel<<<m, 256, 0, c->stream>>>(m, Z, G, Z2);
  Z = Z2;
  kernel_smem((const void*)backtr_kernel, backtr_smem(m));
  backtr_kernel<<<(m + kBtWarps * kBtCols - 1) / (kBtWarps * kBtCols), 32 * kBtWarps,
                  backtr_smem(m), c->stream>>>(m, Vr, tt, Z);
  vec_fix_kernel<<<m, 256, 0, c->stream>>>(m, Z, V, ldv);
  g_launches += 10;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

}  // namespace gcg
