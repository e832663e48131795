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

#include <cooperative_groups.h>

#include "async.cuh"
#include "common.cuh"

namespace gcg {

extern int64_t g_launches;

constexpr int kTriThreads = 1024;
constexpr int kEigMaxM = 224;    // one-CTA tridiagonalisation (packed triangle in smem)
constexpr int kEigMaxBig = 1024; // multi-CTA path (tridiag_multi_kernel)

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
                                                     double* norms, int i0, int K) {
  extern __shared__ double bsd[];  // d, e^2 of the scaled T (2m doubles)
  double* sd = bsd;
  double* se2 = bsd + m;
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
  const int jl = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (jl >= K) return;
  const int idx = i0 + jl;  // eigenvalue index (0-based, ascending) of this warp
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
  if (lane == 0) lam[jl] = 0.5 * (lo + hi) / sc;
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
// (pass 1); writes z (unnormalised) into column j of Z.
// Per-thread factors interleaved [k][K] in W (coalesced across threads).  Pass 0
// factors (one reciprocal per step on the dependent chain) and keeps the
// multipliers and row swaps; pass 1 only re-runs the substitutions (one FMA per
// step on the chain).  The backward pass multiplies by stored reciprocal pivots.
// K vectors (eigenvalues lam[0..K-1], global indices j0..j0+K-1: the start vector
// depends on the global index, so a slice equals the same columns of the full
// solve).  Z layout: ldz == 0 -> column-major m x K (vector j at Z + j*m), else
// row-major (element (k, j) at Z[k*ldz + j]).  The forward-substituted rhs lives
// in dynamic shared memory ([m][blockDim]) when ys_shared, else in W (after the
// six factor arrays, [m][K]).
struct InvitZ {
  double* Z;
  long long ldz;
  int m;
  __device__ __forceinline__ double& at(int k, int j) const {
    return ldz ? Z[(long long)k * ldz + j] : Z[(long long)j * m + k];
  }
};
__global__ void __launch_bounds__(32) invit_kernel(int m, int K, int j0, const double* d,
                                                   const double* e,
                                                   const double* __restrict__ lam, InvitZ zz,
                                                   double* __restrict__ W, int pass,
                                                   const double* __restrict__ norms,
                                                   int ys_shared) {
  __shared__ double sdv[kEigMaxBig], sev[kEigMaxBig];
  extern __shared__ double ysm[];  // [m][32]: this thread's forward-substituted rhs
  for (int k = threadIdx.x; k < m; k += blockDim.x) {
    sdv[k] = d[k];
    sev[k] = k + 1 < m ? e[k] : 0.0;
  }
  __syncthreads();
  d = sdv;
  e = sev;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= K) return;
  const size_t mk = (size_t)m * K;
  double* R1 = W;            // 1 / U(k, k)
  double* U2 = W + mk;
  double* U3 = W + 2 * mk;
  double* const Yb = ys_shared ? ysm + threadIdx.x : W + 6 * mk + j;
  const size_t ysd = ys_shared ? blockDim.x : (size_t)K;
#define YS(k) Yb[(size_t)(k) * ysd]
  double* ML = W + 4 * mk;   // multipliers; negative zero-bias flag in SW
  double* SW = W + 5 * mk;   // 1.0 where rows k, k+1 were swapped
#define ZV(k) zz.at((k), j)
  if (pass == 0) {
    const double lj = lam[j];
    const double tnorm = norms[0];
    const double tiny = fmax(tnorm, 1e-300) * 2.220446049250313e-16;
    auto fixp = [&](double u) { return fabs(u) < tiny ? (u < 0.0 ? -tiny : tiny) : u; };
    const int jg = j0 + j;
    double dg = d[0] - lj;            // current pivot-row diagonal
    double sp = m > 1 ? e[0] : 0.0;   // current pivot-row superdiagonal
    double yk = start_entry(jg, 0);
#pragma unroll 4
    for (int k = 0; k + 1 < m; ++k) {
      const double sub = e[k];                        // T(k+1, k)
      const double a1 = d[k + 1] - lj;                // T(k+1, k+1)
      const double s1 = k + 2 < m ? e[k + 1] : 0.0;   // T(k+1, k+2)
      const double bk1 = start_entry(jg, k + 1);
      const size_t o = (size_t)k * K + j;
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
    R1[(size_t)(m - 1) * K + j] = __drcp_rn(fixp(dg));
    YS(m - 1) = yk;
  } else {
    // forward substitution of the new right-hand side with the stored factors
    // loads are batched 8 steps ahead of the chain: the stores to Y would otherwise
    // keep the compiler from hoisting the ML / SW / z loads (same base pointer)
    double yk = ZV(0);
    constexpr int B = 8;
    int k = 0;
    for (; k + B < m; k += B) {
      double mlb[B], swb[B], bb[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const size_t o = (size_t)(k + u) * K + j;
        mlb[u] = ML[o];
        swb[u] = SW[o];
        bb[u] = ZV(k + u + 1);
      }
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const bool sw = swb[u] != 0.0;
        YS(k + u) = sw ? bb[u] : yk;
        yk = fma(-mlb[u], sw ? bb[u] : yk, sw ? yk : bb[u]);
      }
    }
    for (; k + 1 < m; ++k) {
      const size_t o = (size_t)k * K + j;
      const double bk1 = ZV(k + 1);
      const bool sw = SW[o] != 0.0;
      YS(k) = sw ? bk1 : yk;
      yk = fma(-ML[o], sw ? bk1 : yk, sw ? yk : bk1);
    }
    YS(m - 1) = yk;
  }
  double x2 = 0.0, x1 = YS(m - 1) * R1[(size_t)(m - 1) * K + j];
  ZV(m - 1) = x1;
  {
    constexpr int B = 8;
    int k = m - 2;
    for (; k - B + 1 >= 0; k -= B) {
      double yb[B], u2[B], u3[B], r1[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const size_t o = (size_t)(k - u) * K + j;
        yb[u] = YS(k - u);
        u2[u] = U2[o];
        u3[u] = U3[o];
        r1[u] = R1[o];
      }
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const double x0 = (yb[u] - u2[u] * x1 - u3[u] * x2) * r1[u];
        ZV(k - u) = x0;
        x2 = x1;
        x1 = x0;
      }
    }
    for (; k >= 0; --k) {
      const size_t o = (size_t)k * K + j;
      const double x0 = (YS(k) - U2[o] * x1 - U3[o] * x2) * R1[o];
      ZV(k) = x0;
      x2 = x1;
      x1 = x0;
    }
  }
#undef YS
#undef ZV
  // no normalisation here: the cluster kernel normalises every column (2-norm);
  // the unnormalised solution is at most ~1/eps times the start vector
}

// 3'. Inverse iteration with the factors in shared memory: each pass factors
// T - lambda_j I again (the same operations, so the same factors as a stored copy)
// while eliminating the right-hand side — start vector (pass 0) or the current
// column of Z (pass 1, preloaded into the rhs array) — then back-substitutes from
// shared memory.  T threads per block (one eigenvalue each), [k][T] interleaved
// arrays: R1 (1/pivot), U2, U3, Y.  Bitwise the same result as invit_kernel.
static int invit_threads(int m) {
  int t = 32;
  while (t > 1 && 4 * sizeof(double) * (size_t)m * t > 160 * 1024) t >>= 1;
  return t;
}
__global__ void invit_smem_kernel(int m, int K, int j0, const double* __restrict__ d,
                                  const double* __restrict__ e, const double* __restrict__ lam,
                                  InvitZ zz, int pass, const double* __restrict__ norms) {
  __shared__ double sdv[kEigMaxBig], sev[kEigMaxBig];
  extern __shared__ double fsm[];
  const int T = blockDim.x;
  for (int k = threadIdx.x; k < m; k += T) {
    sdv[k] = d[k];
    sev[k] = k + 1 < m ? e[k] : 0.0;
  }
  const int j = blockIdx.x * T + threadIdx.x;
  double* R1 = fsm + threadIdx.x;
  double* U2 = R1 + (size_t)m * T;
  double* U3 = U2 + (size_t)m * T;
  double* Y = U3 + (size_t)m * T;
#define FS(arr, k) arr[(size_t)(k) * T]
  if (pass == 1 && j < K)
    for (int k = 0; k < m; ++k) FS(Y, k) = zz.at(k, j);
  __syncthreads();
  if (j >= K) return;
  const double lj = lam[j];
  const double tnorm = norms[0];
  const double tiny = fmax(tnorm, 1e-300) * 2.220446049250313e-16;
  auto fixp = [&](double u) { return fabs(u) < tiny ? (u < 0.0 ? -tiny : tiny) : u; };
  const int jg = j0 + j;
  double dg = sdv[0] - lj;
  double sp = m > 1 ? sev[0] : 0.0;
  double yk = pass == 0 ? start_entry(jg, 0) : FS(Y, 0);
#pragma unroll 4
  for (int k = 0; k + 1 < m; ++k) {
    const double sub = sev[k];
    const double a1 = sdv[k + 1] - lj;
    const double s1 = k + 2 < m ? sev[k + 1] : 0.0;
    const double bk1 = pass == 0 ? start_entry(jg, k + 1) : FS(Y, k + 1);
    const bool sw = fabs(sub) > fabs(dg);
    const double rp = __drcp_rn(sw ? sub : fixp(dg));
    const double mult = (sw ? dg : sub) * rp;
    FS(R1, k) = rp;
    FS(U2, k) = sw ? a1 : sp;
    FS(U3, k) = sw ? s1 : 0.0;
    FS(Y, k) = sw ? bk1 : yk;
    yk = fma(-mult, sw ? bk1 : yk, sw ? yk : bk1);
    dg = fma(-mult, sw ? a1 : sp, sw ? sp : a1);
    sp = sw ? -mult * s1 : s1;
  }
  FS(R1, m - 1) = __drcp_rn(fixp(dg));
  FS(Y, m - 1) = yk;
  double x2 = 0.0, x1 = FS(Y, m - 1) * FS(R1, m - 1);
  zz.at(m - 1, j) = x1;
#pragma unroll 4
  for (int k = m - 2; k >= 0; --k) {
    const double x0 = (FS(Y, k) - FS(U2, k) * x1 - FS(U3, k) * x2) * FS(R1, k);
    zz.at(k, j) = x0;
    x2 = x1;
    x1 = x0;
  }
#undef FS
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
// K vectors of length m in the InvitZ layout.
__global__ void __launch_bounds__(256) cluster_kernel(int m, int K, const double* __restrict__ lam,
                                                      InvitZ zz, const double* __restrict__ norms) {
  __shared__ double red[8][33];
  __shared__ double coef[kEigMaxBig];
  const int b = blockIdx.x;
  const double ortol = kTightGap * norms[0];
  if (b > 0 && lam[b] - lam[b - 1] <= ortol) return;  // not a cluster start
  int end = b + 1;
  while (end < K && lam[end] - lam[end - 1] <= ortol) ++end;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int jj = b; jj < end; ++jj) {
    for (int pass = 0; pass < 2 && jj > b; ++pass) {
      // coefficients c_i = z_i' z_j, one warp per earlier member (fixed order)
      for (int i = b + warp; i < jj; i += 8) {
        double s = 0.0;
        for (int k = lane; k < m; k += 32) s = fma(zz.at(k, i), zz.at(k, jj), s);
        s = warp_sum(s);
        if (lane == 0) coef[i - b] = s;
      }
      __syncthreads();
      for (int k = tid; k < m; k += 256) {
        double x = zz.at(k, jj);
        for (int i = b; i < jj; ++i) x = fma(-coef[i - b], zz.at(k, i), x);
        zz.at(k, jj) = x;
      }
      __syncthreads();
    }
    double s = 0.0;
    for (int k = tid; k < m; k += 256) s = fma(zz.at(k, jj), zz.at(k, jj), s);
    s = warp_sum(s);
    if (lane == 0) red[warp][0] = s;
    __syncthreads();
    double nrm2 = 0.0;
    for (int w2 = 0; w2 < 8; ++w2) nrm2 += red[w2][0];
    const double inv = nrm2 > 0.0 ? 1.0 / sqrt(nrm2) : 0.0;
    for (int k = tid; k < m; k += 256) zz.at(k, jj) *= inv;
    __syncthreads();
  }
}

// 5. Z <- Q Z with Q = H_0 H_1 ... H_{m-3}: each warp owns COLS columns of Z in
// registers (lane holds rows lane + 32 s, s < ROWS) and applies all reflectors
// last-first, with the next reflector's loads issued before the current one's
// reductions; no block barriers inside a chunk of CHUNK reflectors (staged in shared
// memory, double-buffered).  K columns of Z in the InvitZ layout.
// m <= 224: 4 columns x 7 rows per lane; m <= 1024: 1 column x 32 rows.
constexpr int kBtWarps = 8;
template <int CHUNK>
static size_t backtr_smem(int m) { return sizeof(double) * 2 * CHUNK * ((size_t)m + 1); }
template <int COLS, int ROWS, int CHUNK>
__global__ void __launch_bounds__(32 * kBtWarps) backtr_kernel(int m, int K,
                                                               const double* __restrict__ Vr,
                                                               const double* __restrict__ tau,
                                                               InvitZ zz) {
  extern __shared__ __align__(16) double bsm[];  // [2][CHUNK][m] reflectors + [2][CHUNK] tau
  double* vbuf = bsm;
  double* tbuf = bsm + 2 * CHUNK * (size_t)m;
  const int lane = threadIdx.x & 31;
  const int col0 = (blockIdx.x * kBtWarps + (threadIdx.x >> 5)) * COLS;
  const bool live = col0 < K;
  double r[COLS][ROWS];
#pragma unroll
  for (int cc = 0; cc < COLS; ++cc)
#pragma unroll
    for (int s = 0; s < ROWS; ++s) {
      const int k = lane + 32 * s;
      r[cc][s] = (live && k < m && col0 + cc < K) ? zz.at(k, col0 + cc) : 0.0;
    }
  // reflectors are applied last-first: chunk c covers j = jtop - c*CHUNK down to ..-CHUNK+1
  const int jtop = m - 3;
  const int nchunks = jtop >= 0 ? jtop / CHUNK + 1 : 0;
  auto stage = [&](int cidx, int buf) {
    const int jhi = jtop - cidx * CHUNK;
    const int cnt = min(CHUNK, jhi + 1);
    double* dst = vbuf + (size_t)buf * CHUNK * m;
    for (int e = threadIdx.x; e < cnt * m; e += blockDim.x) {
      const int q = e / m, k = e - q * m;
      const int j = jhi - q;
      cp_async8(dst + (size_t)q * m + k, Vr + (size_t)j * m + k, k > j);
    }
    if (threadIdx.x < cnt) cp_async8(tbuf + buf * CHUNK + threadIdx.x, tau + jhi - threadIdx.x, true);
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
    const int jhi = jtop - cidx * CHUNK;
    const int cnt = min(CHUNK, jhi + 1);
    const double* vb = vbuf + (size_t)buf * CHUNK * m;
    if (live) {
      for (int q = 0; q < cnt; ++q) {
        const double t = tbuf[buf * CHUNK + q];
        if (t == 0.0) continue;
        const double* vj = vb + (size_t)q * m;
        // rows above the reflector's first row (k <= j) are zero-filled: skip whole
        // register rows below the first nonzero 32-row block
        const int s0 = (jhi - q + 1) >> 5;
        double vv[ROWS];
#pragma unroll
        for (int s = 0; s < ROWS; ++s) {
          const int k = lane + 32 * s;
          vv[s] = (s >= s0 && k < m) ? vj[k] : 0.0;
        }
        double dot[COLS];
#pragma unroll
        for (int cc = 0; cc < COLS; ++cc) {
          dot[cc] = 0.0;
#pragma unroll
          for (int s = 0; s < ROWS; ++s) dot[cc] = fma(vv[s], r[cc][s], dot[cc]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int cc = 0; cc < COLS; ++cc) dot[cc] += __shfl_xor_sync(0xffffffffu, dot[cc], o);
#pragma unroll
        for (int cc = 0; cc < COLS; ++cc) {
          const double f = t * dot[cc];
#pragma unroll
          for (int s = 0; s < ROWS; ++s) r[cc][s] = fma(-f, vv[s], r[cc][s]);
        }
      }
    }
    __syncthreads();  // buffer 'buf' is restaged two chunks later
  }
  if (!live) return;
#pragma unroll
  for (int cc = 0; cc < COLS; ++cc)
#pragma unroll
    for (int s = 0; s < ROWS; ++s) {
      const int k = lane + 32 * s;
      if (k < m && col0 + cc < K) zz.at(k, col0 + cc) = r[cc][s];
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

// ---------------------------------------------------------------------------
// Orders 224 < m <= 1024 (cfg3 / cfg4 / cfg5 Rayleigh-Ritz: m = 400 / 500 / 1000):
// the packed triangle (up to 4 MB) no longer fits one SM, so the Householder
// reduction runs on G co-resident CTAs (cooperative launch, G ~ m / 8 <= #SMs).
//
// 1'. tridiag_grid_kernel  Row i of the full symmetric matrix lives in the shared
//     memory of CTA i mod G (cyclic: the trailing block stays balanced), one warp
//     per row.  Step j:
//       A  each CTA applies the deferred rank-2 update of step j-1 to its trailing
//          rows (x -= v_i w_c + w_i v_c, the product sum commutative, so the stored
//          matrix stays bitwise symmetric), forms p_i = tau_j sum_c A(i, c) v_c and
//          publishes p_i, its partial sum of p_i v_i and — the owner of row j+1 —
//          that row (= column j+1 by symmetry) to global memory (L2, double
//          buffered by step parity);
//       one grid barrier (monotone counter, release / acquire);
//       B  every CTA redundantly reduces the G partials in a fixed order, forms
//          w_j = p - (tau/2)(p'v) v, applies step j's update to column j+1 and
//          computes reflector v_{j+1} (dlarfg) — identical bits in every CTA.
//     One barrier and a few L2 round trips per step; every element is read and
//     written once per step from shared memory.  Same outputs as tridiag_kernel.
constexpr int kTgRows = 8;  // rows per CTA of the grid variant; G = ceil(m / kTgRows)

struct TgArgs {
  int m;
  const double* A;
  long long lda;
  int sym;
  double* d;
  double* e;
  double* tau;
  double* Vr;
  double* pbuf;    // grid: [2][m]  p of the current step (by parity)
  double* rowbuf;  // grid: [2][m]  row j+1 of A^(j)
  double* part;    // grid: [2][G]  per-CTA partial p'v
  double* dlast;   // grid: A^(m-3)(m-1, m-1)
  unsigned* bar;   // grid: barrier counter (zeroed before the launch)
  int G;           // CTAs (grid size / cluster size)
  int R;           // rows per CTA = ceil(m / G)
};

__device__ __forceinline__ double tg_sym_at(const TgArgs& a, int i, int c) {
  const int r = i >= c ? i : c, s = i >= c ? c : i;  // the lower triangle of row-major A
  double x = a.A[(long long)r * a.lda + s];
  if (a.sym) x = 0.5 * (x + a.A[(long long)s * a.lda + r]);
  return x;
}
// x - (v_i w_c + w_i v_c), symmetric in (i, c) bit for bit
__device__ __forceinline__ double tg_upd(double x, double vi, double wc, double wi, double vc) {
  return x - __dadd_rn(__dmul_rn(vi, wc), __dmul_rn(wi, vc));
}
// fixed-order block sum (every thread gets the same value); red: NT/32 slots
template <int NT>
__device__ __forceinline__ double tg_block_sum(double v, double* red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) s += red[w];
  return s;
}
// reflector of column j (x[j..m-1] in shared memory) into vout; block 0 records d, e,
// tau and the reflector column of Vr.  Returns tau.
template <int NT>
__device__ double tg_reflector(const TgArgs& a, int j, const double* x, double* vout,
                               double* red) {
  const int m = a.m;
  double sq = 0.0;
  for (int i = j + 2 + (int)threadIdx.x; i < m; i += NT) sq = fma(x[i], x[i], sq);
  const double s = tg_block_sum<NT>(sq, red);
  const double alpha = x[j + 1], djj = x[j];
  double t = 0.0, beta = alpha, scal = 0.0;
  if (s > 0.0) {
    const double nrm2 = fma(alpha, alpha, s);
    const double rn = rsqrt(nrm2);  // beta = -sign(alpha) ||x||
    beta = alpha >= 0.0 ? -nrm2 * rn : nrm2 * rn;
    t = (beta - alpha) * __drcp_rn(beta);
    scal = __drcp_rn(alpha - beta);
  }
  for (int i = threadIdx.x; i < m; i += NT) {
    const double vi = i <= j ? 0.0 : (i == j + 1 ? 1.0 : x[i] * scal);
    vout[i] = t != 0.0 ? vi : 0.0;
    if (blockIdx.x == 0 && i > j) a.Vr[(long long)j * m + i] = vi;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.d[j] = djj;
    a.e[j] = beta;
    a.tau[j] = t;
  }
  __syncthreads();
  return t;
}

template <int NT>
static size_t tg_smem(int m, int R) {
  return sizeof(double) * ((size_t)R * m + 4 * (size_t)m + 4 * (NT / 32) + 16);
}

// The multi-CTA Householder reduction; CLUSTER = false: G co-resident CTAs exchanging
// through L2 with a grid barrier (1'), true: one thread-block cluster exchanging
// through distributed shared memory with the cluster barrier (1'').  Per step: phase
// A (no block barrier) processes a warp's rows in pairs — the shared vector loads
// serve both, two independent reduction chains — and leaves per-warp partials of
// p'v; one cluster / grid barrier; phase B issues every remote load first, each warp
// reduces p'v itself (fixed order, identical everywhere), each thread forms w_i, the
// updated column entry x_i and its share of ||x||^2 in registers; one block barrier
// for the norm, the reflector is formed redundantly by every thread, a second block
// barrier publishes it.  Entries are owned by thread i - (j + 1) mod NT; their (owner
// CTA, slot) pairs advance incrementally with j (no divisions on the step path).
constexpr int kTbSlots = 4;  // phase-B entries per thread: m <= NT * kTbSlots
template <int NT, bool CLUSTER>
__global__ void __launch_bounds__(NT, 1) tridiag_multi_kernel(TgArgs a) {
  namespace cgx = cooperative_groups;
  constexpr int NW = NT / 32;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ double gsm[];
  const int m = a.m, G = a.G, R = a.R;
  const int cta = CLUSTER ? (int)cgx::this_cluster().block_rank() : (int)blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* S = gsm;  // [R][m]: local row r = global row cta + G r
  double* vb[4];
  for (int q = 0; q < 4; ++q) vb[q] = S + (size_t)R * m + (size_t)q * m;
  double* part = vb[3] + m;  // cluster: [2][NW] per-warp partials of p'v, by step parity
  double* red = part + 2 * NW;  // [0, NW) ||x||^2 warps, [NW, 2 NW) p'v warps (grid), [2 NW, +2) d, alpha
  for (int r = 0; r < R; ++r) {
    const int i = cta + G * r;
    if (i >= m) break;
    for (int c = tid; c < m; c += NT) S[(size_t)r * m + c] = tg_sym_at(a, i, c);
  }
  for (int c = tid; c < m; c += NT) {
    vb[0][c] = 0.0;  // v_{-1}
    vb[1][c] = 0.0;  // w_{-1}
    vb[3][c] = tg_sym_at(a, c, 0);  // column 0
  }
  __syncthreads();
  double* vprev = vb[0];
  double* wprev = vb[1];
  double* vcur = vb[2];
  double* wnew = vb[3];
  double t = tg_reflector<NT>(a, 0, wnew, vcur, red);
  // phase-B entries i_q = j + 1 + tid + q NT: owner CTA and local slot, advanced per step
  int own[kTbSlots], slt[kTbSlots];
#pragma unroll
  for (int q = 0; q < kTbSlots; ++q) {
    const int i = 1 + tid + q * NT;
    own[q] = i % G;
    slt[q] = i / G;
  }
  int own1 = 1 % G, slt1 = 1 / G;  // row j + 1
  if constexpr (CLUSTER) cgx::this_cluster().sync();  // rows loaded before remote reads
  for (int j = 0; j + 2 < m; ++j) {
    const int par = j & 1;
    // A: deferred update + p on this CTA's trailing rows, two rows per pass
    double mypv = 0.0;
    const int rfirst = (j + 1 - cta + G - 1) / G > 0 ? (j + 1 - cta + G - 1) / G : 0;
    for (int r0 = rfirst + warp; r0 < R; r0 += 2 * NW) {
      const int r1 = r0 + NW;
      const int i0 = cta + G * r0, i1 = cta + G * r1;
      const bool ok0 = i0 < m, ok1 = r1 < R && i1 < m;
      if (!ok0) break;
      double* S0 = S + (size_t)r0 * m;
      double* S1 = S + (size_t)(ok1 ? r1 : r0) * m;
      const double vp0 = vprev[i0], wp0 = wprev[i0];
      const double vp1 = ok1 ? vprev[i1] : 0.0, wp1 = ok1 ? wprev[i1] : 0.0;
      double acc0 = 0.0, acc1 = 0.0;
      for (int c = j + 1 + lane; c < m; c += 32) {
        const double wc = wprev[c], vc = vprev[c], uc = vcur[c];
        const double x0 = tg_upd(S0[c], vp0, wc, wp0, vc);
        S0[c] = x0;
        acc0 = fma(x0, uc, acc0);
        double x1 = 0.0;
        if (ok1) {
          x1 = tg_upd(S1[c], vp1, wc, wp1, vc);
          S1[c] = x1;
          acc1 = fma(x1, uc, acc1);
        }
        if constexpr (!CLUSTER) {
          if (i0 == j + 1) __stcg(a.rowbuf + (size_t)par * m + c, x0);
          if (ok1 && i1 == j + 1) __stcg(a.rowbuf + (size_t)par * m + c, x1);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc0 += __shfl_xor_sync(FULL, acc0, o);
        acc1 += __shfl_xor_sync(FULL, acc1, o);
      }
      __syncwarp();
      if (lane == 0) {
        const double p0 = t * acc0, p1 = t * acc1;
        if constexpr (CLUSTER) {
          // p_i lives in column j of row i's own storage: dead since step j-1
          S0[j] = p0;
          if (ok1) S1[j] = p1;
        } else {
          __stcg(a.pbuf + (size_t)par * m + i0, p0);
          if (ok1) __stcg(a.pbuf + (size_t)par * m + i1, p1);
          if (j == m - 3) {
            if (i0 == m - 1) __stcg(a.dlast, S0[m - 1]);
            if (ok1 && i1 == m - 1) __stcg(a.dlast, S1[m - 1]);
          }
        }
        mypv = fma(p0, vcur[i0], mypv);
        if (ok1) mypv = fma(p1, vcur[i1], mypv);
      }
    }
    if constexpr (CLUSTER) {
      if (lane == 0) part[par * NW + warp] = mypv;
      cgx::this_cluster().sync();
    } else {
      if (lane == 0) red[NW + warp] = mypv;
      __syncthreads();
      if (tid == 0) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) s += red[NW + w];
        __stcg(a.part + (size_t)par * G + cta, s);
        __threadfence();
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.bar) : "memory");
        const unsigned target = (unsigned)G * (unsigned)(j + 1);
        unsigned v;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.bar) : "memory");
        } while (v < target);
      }
      __syncthreads();
    }
    // B: remote loads first
    double pv = 0.0, p1 = 0.0;
    double pr[kTbSlots], rw[kTbSlots];
    if constexpr (CLUSTER) {
      cgx::cluster_group cl = cgx::this_cluster();
      for (int idx = lane; idx < G * NW; idx += 32)
        pv += *cl.map_shared_rank(part + par * NW + (idx % NW), idx / NW);
      p1 = *cl.map_shared_rank(S + (size_t)slt1 * m + j, own1);
      const double* rowj1 = cl.map_shared_rank(S + (size_t)slt1 * m, own1);
#pragma unroll
      for (int q = 0; q < kTbSlots; ++q) {
        if (j + 1 + q * NT >= m) break;  // uniform: no thread of the CTA has slot q
        const int i = j + 1 + tid + q * NT;
        pr[q] = i < m ? *cl.map_shared_rank(S + (size_t)slt[q] * m + j, own[q]) : 0.0;
        rw[q] = i < m ? rowj1[i] : 0.0;
      }
    } else {
      for (int q = lane; q < G; q += 32) pv += __ldcg(a.part + (size_t)par * G + q);
      p1 = __ldcg(a.pbuf + (size_t)par * m + j + 1);
#pragma unroll
      for (int q = 0; q < kTbSlots; ++q) {
        if (j + 1 + q * NT >= m) break;  // uniform: no thread of the CTA has slot q
        const int i = j + 1 + tid + q * NT;
        pr[q] = i < m ? __ldcg(a.pbuf + (size_t)par * m + i) : 0.0;
        rw[q] = i < m ? __ldcg(a.rowbuf + (size_t)par * m + i) : 0.0;
      }
    }
    pv = warp_sum(pv);  // every warp, same order
    const double a2 = -0.5 * t * pv;
    const double vj1 = vcur[j + 1];
    const double wj1 = fma(a2, vj1, p1);
    double xq[kTbSlots];
    double sq = 0.0;
#pragma unroll
    for (int q = 0; q < kTbSlots; ++q) {
      xq[q] = 0.0;
      if (j + 1 + q * NT >= m) break;
      const int i = j + 1 + tid + q * NT;
      if (i < m) {
        const double vi = vcur[i];
        const double wi = fma(a2, vi, pr[q]);
        wnew[i] = wi;
        const double x = tg_upd(rw[q], vi, wj1, wi, vj1);
        xq[q] = x;
        if (i >= j + 3) sq = fma(x, x, sq);
        if (i == j + 1) red[2 * NW] = x;
        if (i == j + 2) red[2 * NW + 1] = x;
      }
    }
    sq = warp_sum(sq);
    if (lane == 0) red[warp] = sq;
    __syncthreads();
    const double djj = red[2 * NW], alpha = red[2 * NW + 1];
    if (j + 3 < m) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) s += red[w];
      double tn = 0.0, beta = alpha, scal = 0.0;
      if (s > 0.0) {
        const double nrm2 = fma(alpha, alpha, s);
        const double rn = rsqrt(nrm2);  // beta = -sign(alpha) ||x||
        beta = alpha >= 0.0 ? -nrm2 * rn : nrm2 * rn;
        tn = (beta - alpha) * __drcp_rn(beta);
        scal = __drcp_rn(alpha - beta);
      }
      double* vn = vprev;  // dead after A: v_{j+1}
#pragma unroll
      for (int q = 0; q < kTbSlots; ++q) {
        if (j + 1 + q * NT >= m) break;  // uniform: no thread of the CTA has slot q
        const int i = j + 1 + tid + q * NT;
        if (i < m) {
          const double vi = i == j + 1 ? 0.0 : (i == j + 2 ? 1.0 : xq[q] * scal);
          vn[i] = tn != 0.0 ? vi : 0.0;
          if (blockIdx.x == 0 && i > j + 1) a.Vr[(long long)(j + 1) * m + i] = vi;
        }
      }
      if (blockIdx.x == 0 && tid == 0) {
        a.d[j + 1] = djj;
        a.e[j + 1] = beta;
        a.tau[j + 1] = tn;
      }
      t = tn;
    } else if (blockIdx.x == 0 && tid == 0) {  // last 2 x 2 block
      double dl;
      if constexpr (CLUSTER)
        dl = *cgx::this_cluster().map_shared_rank(S + (size_t)((m - 1) / G) * m + (m - 1),
                                                  (m - 1) % G);
      else
        dl = __ldcg(a.dlast);
      a.d[m - 2] = djj;
      a.e[m - 2] = alpha;
      a.tau[m - 2] = 0.0;
      a.d[m - 1] = tg_upd(dl, vcur[m - 1], wnew[m - 1], wnew[m - 1], vcur[m - 1]);
    }
    __syncthreads();
    // rotate: (v_j, w_j) become the deferred update, v_{j+1} the current reflector
    double* old_w = wprev;
    double* old_v = vprev;
    vprev = vcur;
    wprev = wnew;
    vcur = old_v;
    wnew = old_w;
#pragma unroll
    for (int q = 0; q < kTbSlots; ++q)
      if (++own[q] == G) {
        own[q] = 0;
        ++slt[q];
      }
    if (++own1 == G) {
      own1 = 0;
      ++slt1;
    }
  }
  if constexpr (CLUSTER) cgx::this_cluster().sync();  // nobody leaves while read remotely
}

constexpr int kTgThreads = 256;  // grid variant
constexpr int kTcThreads = 256;  // cluster variant (m <= 256: one phase-B slot per thread)

// V[i*ldv + j] = sign_j * Z[i*ldz + j] (row-major Z, column j) with the sign rule
__global__ void vec_fix_rm_kernel(int m, const double* Z, long long ldz, double* V, long long ldv) {
  const int j = blockIdx.x;
  double best = -1.0;
  int lead = 0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double x = fabs(Z[(long long)i * ldz + j]);
    if (x > best) {
      best = x;
      lead = i;
    }
  }
  __shared__ double bv[256];
  __shared__ int bi[256];
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = lead;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const double o = bv[threadIdx.x + w];
      const int oi = bi[threadIdx.x + w];
      if (o > bv[threadIdx.x] || (o == bv[threadIdx.x] && oi < bi[threadIdx.x])) {
        bv[threadIdx.x] = o;
        bi[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  const double sg = Z[(long long)bi[0] * ldz + j] < 0.0 ? -1.0 : 1.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) V[(long long)i * ldv + j] = sg * Z[(long long)i * ldz + j];
}

int gram_launch(Ctx* c, long long n, int k1, int k2, const double* X, long long ldx,
                const double* Y, long long ldy, double alpha, double beta, double* G,
                long long grs, long long gcs);
int lincomb_launch(Ctx* c, long long n, int m, int d, double alpha, const double* X,
                   long long ldx, const double* C, long long ldc, double beta, double* Y,
                   long long ldy);
int copy_launch(Ctx* c, long long n, int k, const double* X, long long ldx, double* Y,
                long long ldy);

__global__ void vec_fix_kernel(int m, const double* Vcm, double* V, long long ldv);

bool dense_syev_tridiag_ok(int m) {
  static const char* impl = getenv("GCG_SYEV");
  if (impl && impl[0] == 'c') return false;  // GCG_SYEV=cusolver: A/B switch
  return m >= 3 && m <= kEigMaxBig;
}

// Tridiagonalisation variant by order: 'o' one CTA (m <= 224), 'c' one cluster
// (m <= 600), 'g' co-resident grid.  GCG_TRIMODE=o|c|g forces one where it applies (A/B).
constexpr int kTcMaxM = 600;
static char tridiag_mode(int m) {
  static const char* env = getenv("GCG_TRIMODE");
  static const char force = env ? env[0] : 0;
  static const bool legacy_grid = getenv("GCG_TRIGRID") && getenv("GCG_TRIGRID")[0] == '1';
  if (legacy_grid) return 'g';
  if (force == 'o' && m <= kEigMaxM) return 'o';
  if (force == 'g') return 'g';
  if (force == 'c' && m <= kTcMaxM) return 'c';
  // measured (scripts/eig_bench.py, profiles/r02_eig_modes.txt): the 8-CTA cluster from
  // m = 100 (0.385 vs 0.436 ms one-CTA) to 256, the co-resident grid above (a 16-CTA
  // cluster runs out of phase-A parallelism past ~300); one CTA only for tiny orders
  if (m < 48) return 'o';
  return m <= 256 ? 'c' : 'g';
}
static bool use_grid_tridiag(int m) { return tridiag_mode(m) != 'o'; }

static int tridiag_cluster_launch(Ctx* c, int m, const double* A, long long lda, int sym,
                                  double* dd, double* ee, double* tt, double* Vr) {
  static const int env_c = getenv("GCG_TRIC") ? atoi(getenv("GCG_TRIC")) : 0;  // A/B
  const int C = (env_c == 4 || env_c == 8 || env_c == 16) ? env_c : (m <= 256 ? 8 : 16);
  const int R = (m + C - 1) / C;
  TgArgs a = {};
  a.m = m;
  a.A = A;
  a.lda = lda;
  a.sym = sym;
  a.d = dd;
  a.e = ee;
  a.tau = tt;
  a.Vr = Vr;
  a.G = C;
  a.R = R;
  const size_t smem = tg_smem<kTcThreads>(m, R);
  auto kern = tridiag_multi_kernel<kTcThreads, true>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr_done = true;
  }
  kernel_smem((const void*)kern, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  GCG_TRY(cuda_status(cudaLaunchKernelEx(&cfg, kern, a)));
  ++g_launches;
  return GCG_OK;
}

static int tridiag_grid_launch(Ctx* c, int m, const double* A, long long lda, int sym, double* dd,
                               double* ee, double* tt, double* Vr, double* gw) {
  int G = (m + kTgRows - 1) / kTgRows;
  if (G > c->num_sms) G = c->num_sms;
  const int R = (m + G - 1) / G;
  if (R > 2 * kTgRows) return GCG_ERR_ARG;
  TgArgs a;
  a.m = m;
  a.A = A;
  a.lda = lda;
  a.sym = sym;
  a.d = dd;
  a.e = ee;
  a.tau = tt;
  a.Vr = Vr;
  a.pbuf = gw;
  a.rowbuf = gw + 2 * (size_t)m;
  a.part = gw + 4 * (size_t)m;
  a.dlast = a.part + 2 * (size_t)G;
  a.bar = (unsigned*)(a.dlast + 2);
  a.G = G;
  a.R = R;
  GCG_TRY(cuda_status(cudaMemsetAsync(a.bar, 0, sizeof(unsigned), c->stream)));
  const size_t smem = tg_smem<kTgThreads>(m, R);
  auto kern = tridiag_multi_kernel<kTgThreads, false>;
  kernel_smem((const void*)kern, smem);
  void* args[] = {&a};
  GCG_TRY(cuda_status(cudaLaunchCooperativeKernel((const void*)kern, dim3(G), dim3(kTgThreads),
                                                  args, smem, c->stream)));
  ++g_launches;
  return GCG_OK;
}

// back-transform for m <= 224: COLS columns per warp (GCG_BTCOLS=1|2|4, default 2):
// fewer columns per warp = more CTAs and a shorter per-reflector chain
static int backtr_small(Ctx* c, int m, int K, const double* Vr, const double* tt, InvitZ zz) {
  static const int cols = getenv("GCG_BTCOLS") ? atoi(getenv("GCG_BTCOLS")) : 2;
  constexpr int RW = (kEigMaxM + 31) / 32;
#define BT(C)                                                                               \
  do {                                                                                      \
    auto bt = backtr_kernel<C, RW, 16>;                                                     \
    kernel_smem((const void*)bt, backtr_smem<16>(m));                                       \
    bt<<<(K + kBtWarps * C - 1) / (kBtWarps * C), 32 * kBtWarps, backtr_smem<16>(m),        \
         c->stream>>>(m, K, Vr, tt, zz);                                                    \
  } while (0)
  if (cols == 1) BT(1);
  else if (cols == 4) BT(4);
  else BT(2);
#undef BT
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

// Eigenpairs il..iu (1-based inclusive; K = iu - il + 1) of the symmetric m x m
// row-major A (symmetrised first when sym != 0): w (K values, ascending) and V
// (row-major m x K, ldv; the sign rule applied).  No cuSOLVER:
//   tridiagonalisation (one CTA, one cluster or a co-resident grid: tridiag_mode), bisection
//   of the requested indices only, inverse iteration + tight-cluster Gram-Schmidt
//   (twice), Loewdin, back-transform, sign rule.
// The full spectrum of an order <= 224 keeps the column-major one-CTA kernels; every
// other case (larger orders, index slices) works on a row-major Z (m x K) whose
// Loewdin step is one DMMA Gram Z'Z and one LinComb Z (3/2 I - 1/2 G).
int dense_syev_tridiag_range(Ctx* c, int m, const double* A, long long lda, int sym, int il,
                             int iu, double* w, double* V, long long ldv) {
  if (m < 3 || m > kEigMaxBig || il < 1 || iu < il || iu > m) return GCG_ERR_ARG;
  const int K = iu - il + 1;
  const bool grid = use_grid_tridiag(m);
  const bool small = m <= kEigMaxM && K == m;  // column-major Z, one-CTA Loewdin kernels
  const size_t mm = (size_t)m * m, mk = (size_t)m * K;
  const bool ys_shared = 32 * (size_t)m * sizeof(double) <= 64 * 1024;
  // workspace: d, e, tau (3m) | Vr (m^2) | Z (mK) | inverse-iteration factors (6 mK)
  // [+ rhs (mK)] | Z2 (mK) | G (K^2) | grid scratch (6m + 2G + 8) | norms
  const size_t words = 3 * (size_t)m + mm + mk + 6 * mk + (ys_shared ? 0 : mk) + mk +
                       (size_t)K * K + 6 * (size_t)m + 2 * kNumSMs + 16 + 8;
  GCG_TRY(ensure(c->dense, sizeof(double) * words + 512));
  double* dd = (double*)c->dense.ptr;
  double* ee = dd + m;
  double* tt = ee + m;
  double* Vr = tt + m;
  double* Z = Vr + mm;
  double* W = Z + mk;
  double* Z2 = W + 6 * mk + (ys_shared ? 0 : mk);
  double* Gm = Z2 + mk;
  double* gw = Gm + (size_t)K * K;
  double* norms = gw + 6 * (size_t)m + 2 * kNumSMs + 16;
  if (grid && tridiag_mode(m) == 'c') {
    GCG_TRY(tridiag_cluster_launch(c, m, A, lda, sym, dd, ee, tt, Vr));
  } else if (grid) {
    GCG_TRY(tridiag_grid_launch(c, m, A, lda, sym, dd, ee, tt, Vr, gw));
  } else {
    const size_t smem = tri_smem(m);
    kernel_smem((const void*)tridiag_kernel, smem);
    tridiag_kernel<<<1, kTriThreads, smem, c->stream>>>(m, A, lda, sym, dd, ee, tt, Vr);
    ++g_launches;
  }
  bisect_kernel<<<(K + 7) / 8, 256, 2 * sizeof(double) * m, c->stream>>>(m, dd, ee, w, norms,
                                                                          il - 1, K);
  InvitZ zz;
  zz.Z = Z;
  zz.ldz = small ? 0 : K;
  zz.m = m;
  static const bool invit_global = getenv("GCG_INVIT") && getenv("GCG_INVIT")[0] == 'g';
  const size_t ysm = ys_shared ? sizeof(double) * 32 * (size_t)m : 0;
  const int it = invit_threads(m);
  const size_t fsm = 4 * sizeof(double) * (size_t)m * it;
  for (int pass = 0; pass < 2; ++pass) {
    if (invit_global) {  // A/B: factors stored in global memory by pass 0, reused by pass 1
      kernel_smem((const void*)invit_kernel, ysm);
      invit_kernel<<<(K + 31) / 32, 32, ysm, c->stream>>>(m, K, il - 1, dd, ee, w, zz, W, pass,
                                                          norms, ys_shared ? 1 : 0);
    } else {
      kernel_smem((const void*)invit_smem_kernel, fsm);
      invit_smem_kernel<<<(K + it - 1) / it, it, fsm, c->stream>>>(m, K, il - 1, dd, ee, w, zz,
                                                                   pass, norms);
    }
    cluster_kernel<<<K, 256, 0, c->stream>>>(m, K, w, zz, norms);
  }
  g_launches += 5;
  GCG_CHECK_LAUNCH();
  if (small) {
    double* G = W;  // the inverse-iteration factors are dead now
    double* Zs = W + mm;
    loewdin_gram_kernel<<<m, 256, 0, c->stream>>>(m, Z, G);
    loewdin_apply_kernel<<<m, 256, 0, c->stream>>>(m, Z, G, Zs);
    zz.Z = Zs;
    GCG_TRY(backtr_small(c, m, K, Vr, tt, zz));
    vec_fix_kernel<<<m, 256, 0, c->stream>>>(m, Zs, V, ldv);
    g_launches += 4;
    GCG_CHECK_LAUNCH();
    return GCG_OK;
  }
  // Loewdin on the row-major Z: G = Z'Z, Z2 = 3/2 Z - 1/2 Z G (LinComb in <= 256-column panels)
  GCG_TRY(gram_launch(c, m, K, K, Z, K, Z, K, 1.0, 0.0, Gm, K, 1));
  GCG_TRY(copy_launch(c, m, K, Z, K, Z2, K));
  for (int c0 = 0; c0 < K; c0 += 256) {
    const int dk = K - c0 < 256 ? K - c0 : 256;
    GCG_TRY(lincomb_launch(c, m, K, dk, -0.5, Z, K, Gm + c0, K, 1.5, Z2 + c0, K));
  }
  zz.Z = Z2;
  if (m <= kEigMaxM) {
    GCG_TRY(backtr_small(c, m, K, Vr, tt, zz));
  } else {
    auto bt = backtr_kernel<1, kEigMaxBig / 32, 8>;
    kernel_smem((const void*)bt, backtr_smem<8>(m));
    bt<<<(K + kBtWarps - 1) / kBtWarps, 32 * kBtWarps, backtr_smem<8>(m), c->stream>>>(m, K, Vr,
                                                                                      tt, zz);
  }
  vec_fix_rm_kernel<<<K, 256, 0, c->stream>>>(m, Z2, K, V, ldv);
  g_launches += 2;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

// w (m, ascending) and V (row-major, ldv; eigenvector j in column j, sign rule
// applied) of the symmetric m x m row-major A (symmetrised first when sym != 0).
int dense_syev_tridiag(Ctx* c, int m, const double* A, long long lda, int sym, double* w,
                       double* V, long long ldv) {
  return dense_syev_tridiag_range(c, m, A, lda, sym, 1, m, w, V, ldv);
}

}  // namespace gcg
