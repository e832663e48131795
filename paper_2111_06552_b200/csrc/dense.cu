// Small dense symmetric eigenproblems and the orthogonalisation / convergence
// decision kernels, all on device (no CPU fallback).
//
// Reference: dense.py:63-133 (sym_eig_full / sym_eig_range / gram_svd via
// LAPACK, eigenvalues ascending, each eigenvector's largest-|entry| made
// positive, first index on ties), orth.py:155-188 (_leaf_svqb), orth.py:124-152
// (_deflate_against repeat test), solver.py:129-164 (_rel_residual,
// _count_converged).
//
// B200 design.  Orders <= 64 (SVQB leaves of width <= 16, the post-pass Gram
// of a block of bs <= 64 columns, the momentum Gram) are solved by one CTA with
// a parallel cyclic Jacobi sweep in shared memory (round-robin pairing, all
// m/2 rotations of a round applied at once) — a few tens of microseconds, no
// library call, fused with the SVQB bookkeeping so one kernel turns a Gram
// block into the SVQB coefficient matrix plus a 3-double status record.
// Larger orders (the Rayleigh-Ritz matrix, m <= 1000) use cuSOLVER syevd on
// the context stream followed by an on-device transpose + sign fix.

#include <math.h>
#include <stdlib.h>

#include <vector>

#include "common.cuh"

namespace gcg {

extern int64_t g_launches;

constexpr int kJacMax = 64;

// Parallel cyclic Jacobi on a[mp][kJacMax+1] (symmetric), accumulating v.
// mp is even; rows/cols >= m are zero padding.  All threads of the CTA call it.
//
// Per round (mp/2 disjoint rotations, round-robin pairing): (1) one thread
// per pair computes (c, s) with reciprocal/sqrt only, plus the exact new
// diagonal (Rutishauser: a_pq becomes exactly 0); (2) every 2x2 block (P, R)
// of pair rows x pair columns is transformed in one step, B' = J_P^T B J_R,
// reading and writing each element once, together with V <- V J.  Two
// barriers per round; each thread's block / row assignments are fixed for the
// whole solve and kept in registers (no integer division in the loop).
// kJacThreads threads for orders up to MMAX: 256 threads serve order 64 (4 blocks and 8 V
// items per thread); orders <= 32 can run on 128 threads (2 and 4) with cheaper barriers.
template <int kJacThreads, int MMAX>
__device__ void jacobi_sweeps(int mp, double (*a)[kJacMax + 1], double (*v)[kJacMax + 1],
                              double* cs, double* sn, int* pp, int* qq, double* red) {
  constexpr int kJacMaxBlk = ((MMAX / 2) * (MMAX / 2) + kJacThreads - 1) / kJacThreads;
  constexpr int kJacMaxVrow = (MMAX * (MMAX / 2) + kJacThreads - 1) / kJacThreads;
  const int tid = threadIdx.x;
  const int half = mp / 2;
  // fixed work lists: blocks (P <= R) and V items (row i, pair R)
  // thread tid owns blocks e = tid + b*kJacThreads (kept only when P <= R) and V
  // items e = tid + b*kJacThreads; -1 marks an empty slot
  int blkP[kJacMaxBlk], blkR[kJacMaxBlk];
#pragma unroll
  for (int b = 0; b < kJacMaxBlk; ++b) {
    const int e = tid + b * kJacThreads;
    const int P = e / half, R = e % half;
    const bool ok = e < half * half && P <= R;
    blkP[b] = ok ? P : -1;
    blkR[b] = R;
  }
  int vI[kJacMaxVrow], vR[kJacMaxVrow];
#pragma unroll
  for (int b = 0; b < kJacMaxVrow; ++b) {
    const int e = tid + b * kJacThreads;
    vI[b] = e < mp * half ? e / half : -1;
    vR[b] = e % half;
  }
  for (int sweep = 0; sweep < 40; ++sweep) {
    // convergence: off-diagonal vs diagonal mass (accumulated separately)
    double off = 0.0, dia = 0.0;
    for (int e = tid; e < mp * mp; e += kJacThreads) {
      const int i = e / mp, j = e % mp;
      const double x = a[i][j];
      if (i == j) dia += x * x;
      else off += x * x;
    }
    off = warp_sum(off);
    dia = warp_sum(dia);
    if ((tid & 31) == 0) {
      red[2 * (tid >> 5)] = off;
      red[2 * (tid >> 5) + 1] = dia;
    }
    __syncthreads();
    double toff = 0.0, tdia = 0.0;
    for (int w = 0; w < kJacThreads / 32; ++w) {
      toff += red[2 * w];
      tdia += red[2 * w + 1];
    }
    __syncthreads();
    // relative off-diagonal norm <= 1e-14: eigenvalues/vectors at rounding level
    if (toff <= 1e-28 * tdia || toff == 0.0) break;
    for (int round = 0; round < mp - 1; ++round) {
      if (tid < half) {
        int p, q;
        if (tid == 0) {
          p = round;
          q = mp - 1;
        } else {
          p = round + tid;
          if (p >= mp - 1) p -= mp - 1;
          q = round - tid;
          if (q < 0) q += mp - 1;
        }
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        const double apq = a[p][q], app = a[p][p], aqq = a[q][q];
        double c = 1.0, s = 0.0, t = 0.0;
        if (fabs(apq) > 1e-18 * sqrt(fabs(app * aqq)) && apq != 0.0) {
          // Rutishauser's rotation with reciprocals instead of divisions (the
          // rotation chain is the round's critical path: ~4 long-latency ops)
          const double theta = (aqq - app) * (0.5 * __drcp_rn(apq));
          const double h2 = fma(theta, theta, 1.0);
          const double h = h2 * rsqrt(h2);  // sqrt(1 + theta^2)
          t = __drcp_rn(fabs(theta) + h);
          if (theta < 0.0) t = -t;
          c = rsqrt(fma(t, t, 1.0));
          s = t * c;
        }
        cs[tid] = c;
        sn[tid] = s;
        pp[tid] = p;
        qq[tid] = q;
        red[64 + 2 * tid] = app - t * apq;
        red[64 + 2 * tid + 1] = aqq + t * apq;
      }
      __syncthreads();
#pragma unroll
      for (int b = 0; b < kJacMaxBlk; ++b) {
        const int P = blkP[b], R = blkR[b];
        if (P < 0) continue;
        const double cP = cs[P], sP = sn[P];
        const int p = pp[P], q = qq[P];
        if (P == R) {
          if (sP != 0.0) {
            a[p][p] = red[64 + 2 * P];
            a[q][q] = red[64 + 2 * P + 1];
            a[p][q] = 0.0;
            a[q][p] = 0.0;
          }
          continue;
        }
        const double cR = cs[R], sR = sn[R];
        if (sP == 0.0 && sR == 0.0) continue;
        const int r = pp[R], u = qq[R];
        const double b00 = a[p][r], b01 = a[p][u], b10 = a[q][r], b11 = a[q][u];
        const double u0 = cP * b00 - sP * b10, u1 = cP * b01 - sP * b11;
        const double w0 = sP * b00 + cP * b10, w1 = sP * b01 + cP * b11;
        const double n00 = cR * u0 - sR * u1, n01 = sR * u0 + cR * u1;
        const double n10 = cR * w0 - sR * w1, n11 = sR * w0 + cR * w1;
        a[p][r] = n00;
        a[p][u] = n01;
        a[q][r] = n10;
        a[q][u] = n11;
        a[r][p] = n00;
        a[u][p] = n01;
        a[r][q] = n10;
        a[u][q] = n11;
      }
#pragma unroll
      for (int b = 0; b < kJacMaxVrow; ++b) {
        const int i = vI[b], R = vR[b];
        if (i < 0) continue;
        const double cR = cs[R], sR = sn[R];
        if (sR == 0.0) continue;
        const int r = pp[R], u = qq[R];
        const double vr = v[i][r], vu = v[i][u];
        v[i][r] = cR * vr - sR * vu;
        v[i][u] = sR * vr + cR * vu;
      }
      __syncthreads();
    }
  }
}

// Sort eigenpairs ascending (stable by index) and apply the sign rule;
// writes w[m] and V (row-major, ldv) from a/v (m x m, padded).
__device__ void sort_and_sign(int m, double (*a)[kJacMax + 1], double (*v)[kJacMax + 1],
                              double* wout, double* Vout, long long ldv, int* rank) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < m; i += nt) {
    const double di = a[i][i];
    int r = 0;
    for (int j = 0; j < m; ++j) {
      const double dj = a[j][j];
      r += (dj < di) || (dj == di && j < i);
    }
    rank[i] = r;
  }
  __syncthreads();
  for (int i = tid; i < m; i += nt) {
    const int r = rank[i];
    wout[r] = a[i][i];
    // sign rule on source column i
    int lead = 0;
    double best = -1.0;
    for (int row = 0; row < m; ++row) {
      const double x = fabs(v[row][i]);
      if (x > best) {
        best = x;
        lead = row;
      }
    }
    const double sg = v[lead][i] < 0.0 ? -1.0 : 1.0;
    for (int row = 0; row < m; ++row) Vout[(long long)row * ldv + r] = sg * v[row][i];
  }
  __syncthreads();
}

// threads of the one-CTA Jacobi by order (GCG_JAC_NT=64|128|256 forces it for orders <= 32)
static int jac_threads(int m) {
  static const int env = getenv("GCG_JAC_NT") ? atoi(getenv("GCG_JAC_NT")) : 0;
  if (m > 32) return 256;
  if (env == 64 || env == 128 || env == 256) return env;
  return 128;  // measured: order 16 86.9 -> 72.3 us, order 20 111 -> 100 us (64 threads: 93 / 155 us)
}

struct JacSmem {
  double a[kJacMax][kJacMax + 1];
  double v[kJacMax][kJacMax + 1];
  double cs[kJacMax / 2], sn[kJacMax / 2];
  int pp[kJacMax / 2], qq[kJacMax / 2];
  int rank[kJacMax];
  double red[128];  // [0,64): block reductions; [64,128): exact post-rotation diagonals
  double w[kJacMax];
  double Vs[kJacMax * kJacMax];
};

__device__ void jac_load(JacSmem& S, int m, int mp, const double* A, long long lda, bool sym) {
  for (int e = threadIdx.x; e < mp * mp; e += blockDim.x) {
    const int i = e / mp, j = e % mp;
    double x = 0.0;
    if (i < m && j < m) {
      x = A[(long long)i * lda + j];
      if (sym) x = (x + A[(long long)j * lda + i]) / 2.0;
    }
    S.a[i][j] = x;
    S.v[i][j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
}

template <int NT, int MMAX>
__global__ void __launch_bounds__(NT) syev_jacobi_kernel(int m, const double* A, long long lda,
                                                         double* w, double* V, long long ldv) {
  extern __shared__ __align__(16) unsigned char smraw[];
  JacSmem& S = *reinterpret_cast<JacSmem*>(smraw);
  const int mp = (m + 1) & ~1;
  jac_load(S, m, mp, A, lda, false);
  jacobi_sweeps<NT, MMAX>(mp, S.a, S.v, S.cs, S.sn, S.pp, S.qq, S.red);
  sort_and_sign(m, S.a, S.v, w, V, ldv, S.rank);
}

int dense_syev_jacobi(Ctx* c, int m, const double* A, long long lda, double* w, double* V,
                      long long ldv) {
  if (m <= 0 || m > kJacMax) return GCG_ERR_ARG;
  const size_t sm = sizeof(JacSmem);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(syev_jacobi_kernel<256, kJacMax>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(syev_jacobi_kernel<128, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm);
    cudaFuncSetAttribute(syev_jacobi_kernel<64, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm);
    attr = true;
  }
  const int nt = jac_threads(m);
  if (nt == 64) syev_jacobi_kernel<64, 32><<<1, 64, sm, c->stream>>>(m, A, lda, w, V, ldv);
  else if (nt == 128) syev_jacobi_kernel<128, 32><<<1, 128, sm, c->stream>>>(m, A, lda, w, V, ldv);
  else syev_jacobi_kernel<256, kJacMax><<<1, 256, sm, c->stream>>>(m, A, lda, w, V, ldv);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

// ---------------------------------------------------------------------------
// SVQB leaf step, fused (orth.py:155-188): defect of the raw Gram, Jacobi on
// its symmetric part, dependence count and the coefficient matrix
// Q = V[:, nbad:] / sqrt(lambda[nbad:]).
template <int NT, int MMAX>
__global__ void __launch_bounds__(NT) svqb_prepare_kernel(int m, const double* G, long long ldg,
                                                           double dep_tol, double skip_tol,
                                                           double* Q,
                                                           long long ldq, double* status,
                                                           const int* skip, int* stop_out) {
  pdl_wait();
  pdl_trigger();  // one CTA: let the successor's CTAs become resident while it runs
  // speculative pass (orth.cu): a no-op whose stop flag propagates the "stop"
  if (skip && *skip) {
    if (threadIdx.x == 0 && stop_out) *stop_out = 1;
    return;
  }
  extern __shared__ __align__(16) unsigned char smraw[];
  JacSmem& S = *reinterpret_cast<JacSmem*>(smraw);
  const int mp = (m + 1) & ~1;
  // defect = max |G - I| on the raw (unsymmetrised) Gram
  double dmax = 0.0;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int i = e / m, j = e % m;
    dmax = fmax(dmax, fabs(G[(long long)i * ldg + j] - (i == j ? 1.0 : 0.0)));
  }
  dmax = warp_max(dmax);
  if ((threadIdx.x & 31) == 0) S.red[threadIdx.x >> 5] = dmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)blockDim.x / 32; ++w) t = fmax(t, S.red[w]);
    status[0] = t;
    S.red[127] = t;
  }
  __syncthreads();
  // the caller stops when the Gram is already the identity to reorth_tol
  // (orth.py:170-171): skip the factorisation then
  if (S.red[127] <= skip_tol) {
    if (threadIdx.x == 0 && stop_out) *stop_out = 1;  // converged: the caller returns
    return;
  }
  jac_load(S, m, mp, G, ldg, true);
  jacobi_sweeps<NT, MMAX>(mp, S.a, S.v, S.cs, S.sn, S.pp, S.qq, S.red);
  sort_and_sign(m, S.a, S.v, S.w, S.Vs, m, S.rank);
  __shared__ int nbad_s;
  if (threadIdx.x == 0) {
    const double wmax = S.w[m - 1];
    const double floor = dep_tol * fmax(wmax, 0.0);
    int nb = 0;
    while (nb < m && S.w[nb] <= floor) ++nb;  // searchsorted(..., side="right")
    nbad_s = nb;
    status[1] = (double)nb;
    status[2] = wmax;
    // the next pass follows on the device only for a full-rank block (dependent
    // columns are replaced on the host first, orth.py:176-186)
    if (stop_out) *stop_out = nb != 0;
  }
  __syncthreads();
  const int nb = nbad_s;
  const int kept = m - nb;
  for (int e = threadIdx.x; e < m * kept; e += blockDim.x) {
    const int i = e / kept, j = e % kept;
    Q[(long long)i * ldq + j] = S.Vs[i * m + nb + j] / sqrt(S.w[nb + j]);
  }
}

int svqb_prepare_small(Ctx* c, int m, const double* G, long long ldg, double dep_tol,
                       double skip_tol, double* Q,
                       long long ldq, double* status, int* stop_out) {
  const size_t sm = sizeof(JacSmem);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(svqb_prepare_kernel<256, kJacMax>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(svqb_prepare_kernel<128, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm);
    cudaFuncSetAttribute(svqb_prepare_kernel<64, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm);
    attr = true;
  }
  const int nt = jac_threads(m);
  if (nt == 64)
    pdl_launch(svqb_prepare_kernel<64, 32>, dim3(1), dim3(64), sm, c->stream, m, G, ldg, dep_tol,
               skip_tol, Q, ldq, status, c->skip, stop_out);
  else if (nt == 128)
    pdl_launch(svqb_prepare_kernel<128, 32>, dim3(1), dim3(128), sm, c->stream, m, G, ldg, dep_tol,
               skip_tol, Q, ldq, status, c->skip, stop_out);
  else
    pdl_launch(svqb_prepare_kernel<256, kJacMax>, dim3(1), dim3(256), sm, c->stream, m, G, ldg,
               dep_tol, skip_tol, Q, ldq, status, c->skip, stop_out);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

// ---------------------------------------------------------------------------
// cuSOLVER path for larger orders

__global__ void sym_copy_kernel(int m, const double* A, long long lda, double* B, int sym,
                                double* status) {
  // B (dense m x m, ld m) = A or (A + A^T)/2 ; optional defect max|A - I| into status[0]
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)m * m) return;
  const int i = (int)(e / m), j = (int)(e % m);
  const double x = A[(long long)i * lda + j];
  B[e] = sym ? (x + A[(long long)j * lda + i]) / 2.0 : x;
}

__global__ void max_offeye_kernel(int m, const double* A, long long lda, double* out) {
  double dmax = 0.0;
  for (long long e = threadIdx.x; e < (long long)m * m; e += blockDim.x) {
    const int i = (int)(e / m), j = (int)(e % m);
    dmax = fmax(dmax, fabs(A[(long long)i * lda + j] - (i == j ? 1.0 : 0.0)));
  }
  dmax = warp_max(dmax);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)blockDim.x / 32; ++w) t = fmax(t, red[w]);
    *out = t;
  }
}

// V_out[i*ldv + j] = sign_j * Vcm[i + j*m]  (sign rule per column j)
__global__ void vec_fix_kernel(int m, const double* Vcm, double* V, long long ldv) {
  const int j = blockIdx.x;
  const double* col = Vcm + (long long)j * m;
  double best = -1.0;
  int lead = 0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double x = fabs(col[i]);
    if (x > best) {  // strict: first index wins within a thread
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
  const double sg = col[bi[0]] < 0.0 ? -1.0 : 1.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) V[(long long)i * ldv + j] = sg * col[i];
}

bool dense_syev_tridiag_ok(int m);
int dense_syev_tridiag(Ctx* c, int m, const double* A, long long lda, int sym, double* w,
                       double* V, long long ldv);
int dense_syev_tridiag_range(Ctx* c, int m, const double* A, long long lda, int sym, int il,
                             int iu, double* w, double* V, long long ldv);

int64_t g_cusolver_calls = 0;

int dense_syev_cusolver_sym(Ctx* c, int m, const double* A, long long lda, int symmetrize,
                            double* w, double* V, long long ldv) {
  if (m <= 0) return GCG_ERR_ARG;
  // orders 3..1024 (every BASELINE Rayleigh-Ritz order): eig.cu, no cuSOLVER; cuSOLVER
  // syevd only beyond (or with GCG_SYEV=cusolver for A/B)
  if (dense_syev_tridiag_ok(m)) return dense_syev_tridiag(c, m, A, lda, symmetrize, w, V, ldv);
  ++g_cusolver_calls;
  cusolverDnSetStream(c->solver, c->stream);
  int lwork = 0;
  const size_t mat = (size_t)m * m;
  GCG_TRY(ensure(c->dense, sizeof(double) * mat + 64));
  double* B = (double*)c->dense.ptr;
  if (cusolverDnDsyevd_bufferSize(c->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m,
                                  B, m, w, &lwork) != CUSOLVER_STATUS_SUCCESS)
    return GCG_ERR_SOLVER;
  // GCG_SYEV=syevj selects cuSOLVER's Jacobi driver (A/B experiment: 3x slower at
  // m = 200); default syevd.  (cusolverDnXsyevBatched measured identical to syevd.)
  static const char* impl = getenv("GCG_SYEV");
  const bool jac = impl && impl[0] == 's' && impl[4] == 'j';
  static syevjInfo_t jparams = nullptr;
  if (jac && !jparams) {
    cusolverDnCreateSyevjInfo(&jparams);
    cusolverDnXsyevjSetTolerance(jparams, 1e-15);
    cusolverDnXsyevjSetMaxSweeps(jparams, 30);
  }
  if (jac && cusolverDnDsyevj_bufferSize(c->solver, CUSOLVER_EIG_MODE_VECTOR,
                                         CUBLAS_FILL_MODE_LOWER, m, B, m, w, &lwork,
                                         jparams) != CUSOLVER_STATUS_SUCCESS)
    return GCG_ERR_SOLVER;
  GCG_TRY(ensure(c->eigwork, sizeof(double) * ((size_t)lwork + 8)));
  double* work = (double*)c->eigwork.ptr;
  int* info = (int*)(work + lwork);
  sym_copy_kernel<<<(unsigned)((mat + 255) / 256), 256, 0, c->stream>>>(m, A, lda, B, symmetrize,
                                                                        nullptr);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  const bool x64 = impl && impl[0] == 'x';  // A/B: the 64-bit generic API (host workspace)
  cusolverStatus_t st;
  if (x64) {
    static cusolverDnParams_t prm = nullptr;
    if (!prm) cusolverDnCreateParams(&prm);
    size_t dws = 0, hws = 0;
    if (cusolverDnXsyevd_bufferSize(c->solver, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                                    m, CUDA_R_64F, B, m, CUDA_R_64F, w, CUDA_R_64F, &dws,
                                    &hws) != CUSOLVER_STATUS_SUCCESS)
      return GCG_ERR_SOLVER;
    GCG_TRY(ensure(c->eigwork, dws + 64));
    static std::vector<char> hbuf;
    if (hbuf.size() < hws + 1) hbuf.resize(hws + 1);
    int* xinfo = (int*)((char*)c->eigwork.ptr + dws);
    st = cusolverDnXsyevd(c->solver, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m,
                          CUDA_R_64F, B, m, CUDA_R_64F, w, CUDA_R_64F, c->eigwork.ptr, dws,
                          hbuf.data(), hws, xinfo);
  } else {
    st = jac ? cusolverDnDsyevj(c->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, B,
                                m, w, work, lwork, info, jparams)
             : cusolverDnDsyevd(c->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, B,
                                m, w, work, lwork, info);
  }
  if (st != CUSOLVER_STATUS_SUCCESS) return GCG_ERR_SOLVER;
  // row-major symmetric input == its column-major transpose, so B now holds
  // eigenvector j in column-major column j
  vec_fix_kernel<<<m, 256, 0, c->stream>>>(m, B, V, ldv);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

int dense_syev_cusolver(Ctx* c, int m, const double* A, long long lda, double* w, double* V,
                        long long ldv) {
  return dense_syev_cusolver_sym(c, m, A, lda, 0, w, V, ldv);
}

// Eigenpairs il..iu (1-based inclusive) — sym_eig_range (dense.py:86-117): for orders
// 3..1024 eig.cu's tridiagonalisation, bisection of the requested indices only,
// inverse iteration and back-transformation of those columns (the split-range RR of
// each slice is independent); cuSOLVER syevdx beyond.
// w receives iu - il + 1 values, V (m x (iu - il + 1), row-major) the sign-fixed vectors.
int dense_syev_range(Ctx* c, int m, const double* A, long long lda, int il, int iu, double* w,
                     double* V, long long ldv) {
  if (m <= 0 || il < 1 || iu < il || iu > m) return GCG_ERR_ARG;
  if (dense_syev_tridiag_ok(m)) return dense_syev_tridiag_range(c, m, A, lda, 0, il, iu, w, V, ldv);
  ++g_cusolver_calls;
  cusolverDnSetStream(c->solver, c->stream);
  const size_t mat = (size_t)m * m;
  GCG_TRY(ensure(c->dense, sizeof(double) * (mat + (size_t)m) + 64));
  double* B = (double*)c->dense.ptr;
  double* wall = B + mat;  // syevdx writes the selected values into the head of an m-array
  int lwork = 0, meig = 0;
  if (cusolverDnDsyevdx_bufferSize(c->solver, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I,
                                   CUBLAS_FILL_MODE_LOWER, m, B, m, 0.0, 0.0, il, iu, &meig, wall,
                                   &lwork) != CUSOLVER_STATUS_SUCCESS)
    return GCG_ERR_SOLVER;
  GCG_TRY(ensure(c->eigwork, sizeof(double) * ((size_t)lwork + 8)));
  double* work = (double*)c->eigwork.ptr;
  int* info = (int*)(work + lwork);
  sym_copy_kernel<<<(unsigned)((mat + 255) / 256), 256, 0, c->stream>>>(m, A, lda, B, 0, nullptr);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  if (cusolverDnDsyevdx(c->solver, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I,
                        CUBLAS_FILL_MODE_LOWER, m, B, m, 0.0, 0.0, il, iu, &meig, wall, work, lwork,
                        info) != CUSOLVER_STATUS_SUCCESS)
    return GCG_ERR_SOLVER;
  const int k = iu - il + 1;
  if (meig != k) return GCG_ERR_SOLVER;
  GCG_TRY(cuda_status(cudaMemcpyAsync(w, wall, sizeof(double) * k, cudaMemcpyDeviceToDevice,
                                      c->stream)));
  vec_fix_kernel<<<k, 256, 0, c->stream>>>(m, B, V, ldv);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

// count of vals[j] <= rel * max(max(vals), 0)  (vals ascending; searchsorted side=right)
__global__ void count_le_kernel(int len, const double* vals, double rel, double* out) {
  __shared__ double red[32];
  double mx = -INFINITY;
  for (int i = threadIdx.x; i < len; i += blockDim.x) mx = fmax(mx, vals[i]);
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;  // max(values.max(initial=0.0), 0.0)
    for (int w = 0; w < (int)blockDim.x / 32; ++w) t = fmax(t, red[w]);
    const double floor = rel * fmax(t, 0.0);
    int nb = 0;
    while (nb < len && vals[nb] <= floor) ++nb;
    out[0] = (double)nb;
    out[1] = t;
  }
}

// out[i, j] = V[i, off + j] / sqrt(w[off + j])
__global__ void scale_rsqrt_kernel(int m, int off, const double* V, long long ldv,
                                   const double* w, double* out, long long ldo) {
  const int kept = m - off;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)m * kept) return;
  const int i = (int)(e / kept), j = (int)(e % kept);
  out[(long long)i * ldo + j] = V[(long long)i * ldv + off + j] / sqrt(w[off + j]);
}

__global__ void scale_rsqrt_devoff_kernel(int m, const double* offp, const double* V,
                                          long long ldv, const double* w, double* out,
                                          long long ldo) {
  const int off = (int)offp[0];
  const int kept = m - off;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (kept <= 0 || e >= (long long)m * kept) return;
  const int i = (int)(e / kept), j = (int)(e % kept);
  out[(long long)i * ldo + j] = V[(long long)i * ldv + off + j] / sqrt(w[off + j]);
}

int count_le_launch(Ctx* c, int len, const double* vals, double rel, double* out) {
  count_le_kernel<<<1, 256, 0, c->stream>>>(len, vals, rel, out);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

int scale_rsqrt_launch(Ctx* c, int m, int off, const double* V, long long ldv, const double* w,
                       double* out, long long ldo) {
  const long long tot = (long long)m * (m - off);
  if (tot <= 0) return GCG_OK;
  scale_rsqrt_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, c->stream>>>(m, off, V, ldv, w, out,
                                                                           ldo);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

int svqb_prepare_launch(Ctx* c, int m, const double* G, long long ldg, double dep_tol,
                        double skip_tol, double* Q,
                        long long ldq, double* status) {
  if (m <= kJacMax)
    return svqb_prepare_small(c, m, G, ldg, dep_tol, skip_tol, Q, ldq, status, nullptr);
  // large leaf: defect, cuSOLVER on the symmetric part, count, scale
  max_offeye_kernel<<<1, 256, 0, c->stream>>>(m, G, ldg, status);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  const size_t mat = (size_t)m * m;
  // V + w staging after the solver's own matrix in a separate scratch
  GCG_TRY(ensure(c->host_tmp4, sizeof(double) * (mat + m)));
  double* V = (double*)c->host_tmp4.ptr;
  double* w = V + mat;
  GCG_TRY(dense_syev_cusolver_sym(c, m, G, ldg, 1, w, V, m));
  GCG_TRY(count_le_launch(c, m, w, dep_tol, status + 1));
  // Q = V[:, nbad:] / sqrt(w[nbad:]) with nbad read on device from status[1]
  scale_rsqrt_devoff_kernel<<<(unsigned)((mat + 255) / 256), 256, 0, c->stream>>>(
      m, status + 1, V, m, w, Q, ldq);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

// speculative-chain form (orth.cu): small leaves only, stop flag for the next pass
int svqb_prepare_spec_launch(Ctx* c, int m, const double* G, long long ldg, double dep_tol,
                             double skip_tol, double* Q, long long ldq, double* status,
                             int* stop_out) {
  if (m > kJacMax) return GCG_ERR_ARG;
  return svqb_prepare_small(c, m, G, ldg, dep_tol, skip_tol, Q, ldq, status, stop_out);
}
bool svqb_spec_ok(int m) { return m <= kJacMax; }

// deflation repeat test (orth.py:138-152)
__global__ void deflate_status_kernel(int K, int w, const double* R, long long ldr,
                                      const double* dnew, long long dstride, double dgks,
                                      double* status, const int* skip, double stop_tol,
                                      int* stop_out) {
  pdl_wait();
  pdl_trigger();  // one CTA: let the successor's CTAs become resident while it runs
  if (skip && *skip) {  // speculative pass after a "stop": propagate it
    if (threadIdx.x == 0 && stop_out) *stop_out = 1;
    return;
  }
  __shared__ double red[32];
  __shared__ double colsum[256];
  __shared__ int anyf;
  if (threadIdx.x == 0) anyf = 0;
  // one pass over R: thread (lane l, column c) takes rows l, l + L, ... (L = 256 / w lanes
  // per column when w <= 256), so a column's K loads are spread over L threads instead of
  // one thread walking it; the lane sums of a column are added in lane order
  double mx = 0.0;
  if (w <= (int)blockDim.x) {
    const int L = (int)blockDim.x / w;
    const int c = threadIdx.x % w, l = threadIdx.x / w;
    double lost = 0.0;
    if (l < L) {
      for (int r = l; r < K; r += L) {
        const double x = R[(long long)r * ldr + c];
        mx = fmax(mx, fabs(x));
        lost += x * x;
      }
    }
    colsum[threadIdx.x] = lost;
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < w) {
      double t = 0.0;
      for (int q = 0; q < L; ++q) t += colsum[q * w + threadIdx.x];
      if (t > dgks * fmax(dnew[threadIdx.x * dstride], 1e-300)) atomicExch(&anyf, 1);
    }
  } else {
    for (long long e = threadIdx.x; e < (long long)K * w; e += blockDim.x)
      mx = fmax(mx, fabs(R[(e / w) * ldr + (e % w)]));
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    for (int col = threadIdx.x; col < w; col += blockDim.x) {
      double lost = 0.0;
      for (int r = 0; r < K; ++r) {
        const double x = R[(long long)r * ldr + col];
        lost += x * x;
      }
      if (lost > dgks * fmax(dnew[col * dstride], 1e-300)) atomicExch(&anyf, 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < (int)blockDim.x / 32; ++q) t = fmax(t, red[q]);
    status[0] = t;
    status[1] = (double)anyf;
    if (stop_out) *stop_out = (t <= stop_tol || anyf == 0) ? 1 : 0;  // orth.py:148-152
  }
}

int deflate_status_launch(Ctx* c, int K, int w, const double* R, long long ldr,
                          const double* dnew, long long dstride, double dgks, double* status) {
  pdl_launch(deflate_status_kernel, dim3(1), dim3(256), 0, c->stream, K, w, R, ldr, dnew, dstride, dgks,
             status, (const int*)nullptr, 0.0, (int*)nullptr);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

int deflate_status_spec_launch(Ctx* c, int K, int w, const double* R, long long ldr,
                               const double* dnew, long long dstride, double dgks,
                               double* status, double stop_tol, int* stop_out) {
  pdl_launch(deflate_status_kernel, dim3(1), dim3(256), 0, c->stream, K, w, R, ldr, dnew, dstride, dgks,
             status, c->skip, stop_tol, stop_out);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

// ---------------------------------------------------------------------------
// structured projected matrix (solver.py:281-290) + symmetrisation
__global__ void abar_assemble_kernel(int d, int np, int nw, const double* lam, const double* Pc,
                                     long long ldp, const double* cross, long long ldc,
                                     double* A, long long lda) {
  const int m = d + np + nw;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)m * m) return;
  const int i = (int)(e / m), j = (int)(e % m);
  auto raw = [&](int r, int cc) -> double {
    if (cc >= d + np) return cross[(long long)r * ldc + (cc - d - np)];
    if (r >= d + np) return cross[(long long)cc * ldc + (r - d - np)];
    if (r < d && cc < d) return r == cc ? lam[r] : 0.0;
    if (r >= d && cc >= d) return Pc[(long long)(r - d) * ldp + (cc - d)];
    return 0.0;
  };
  // abar[d+np:, :] = cross.T overrides the cross rows (solver.py:288-289), then (A + A^T)/2
  const double a = raw(i, j), b = raw(j, i);
  A[(long long)i * lda + j] = (a + b) / 2.0;
}

int abar_assemble_launch(Ctx* c, int d, int np, int nw, const double* lam, const double* Pc,
                         long long ldp, const double* cross, long long ldc, double* Abar,
                         long long lda) {
  const long long m = d + np + nw;
  if (m <= 0) return GCG_OK;
  abar_assemble_kernel<<<(unsigned)((m * m + 255) / 256), 256, 0, c->stream>>>(
      d, np, nw, lam, Pc, ldp, cross, ldc, Abar, lda);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

__global__ void max_abs_diff_kernel(int m, int n, const double* A, long long lda,
                                    const double* B, long long ldb, double* out) {
  double mx = 0.0;
  for (long long e = threadIdx.x; e < (long long)m * n; e += blockDim.x) {
    const int i = (int)(e / n), j = (int)(e % n);
    const double b = B ? B[(long long)i * ldb + j] : (i == j ? 1.0 : 0.0);
    mx = fmax(mx, fabs(A[(long long)i * lda + j] - b));
  }
  mx = warp_max(mx);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)blockDim.x / 32; ++w) t = fmax(t, red[w]);
    *out = t;
  }
}

int max_abs_diff_launch(Ctx* c, int m, int n, const double* A, long long lda, const double* B,
                        long long ldb, double* out) {
  max_abs_diff_kernel<<<1, 1024, 0, c->stream>>>(m, n, A, lda, B, ldb, out);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

// ---------------------------------------------------------------------------
// Ritz residuals (solver.py:129-141); per-CTA partials of
// s0 = ||AX - lam BX||^2 (or AX - lam X), s1 = X.X, s2 = X.BX, s3 = BX.BX
__global__ void __launch_bounds__(256) ritz_partials_kernel(long long n, int k,
                                                            const double* AX, long long ldax,
                                                            const double* X, long long ldx,
                                                            const double* BX, long long ldbx,
                                                            const double* lam, int mode,
                                                            long long rows_per_cta,
                                                            double* part) {
  __shared__ double sm[4][256];
  const int kc = k;  // <= 256
  const int lanes = 256 / kc;
  const int c = threadIdx.x % kc, rl = threadIdx.x / kc;
  const long long r0 = (long long)blockIdx.x * rows_per_cta;
  long long r1 = r0 + rows_per_cta;
  if (r1 > n) r1 = n;
  // B = I: BX is X itself — one stream fewer
  const bool same = (BX == X) && (ldbx == ldx);
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  if (rl < lanes) {
    const double l = lam[c];
    auto add = [&](double ax, double x, double bx) {
      const double res = (mode == 0) ? ax - l * x : ax - l * bx;
      s0 = fma(res, res, s0);
      s1 = fma(x, x, s1);
      s2 = fma(x, bx, s2);
      s3 = fma(bx, bx, s3);
    };
    constexpr int U = 8;  // rows in flight per thread
    long long i = r0 + rl;
    for (; i + (U - 1) * lanes < r1; i += U * lanes) {
      double av[U], xv[U], bv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long ii = i + u * lanes;
        av[u] = AX[ii * ldax + c];
        xv[u] = X[ii * ldx + c];
        bv[u] = same ? xv[u] : BX[ii * ldbx + c];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) add(av[u], xv[u], bv[u]);
    }
    for (; i < r1; i += lanes) {
      const double x = X[i * ldx + c];
      add(AX[i * ldax + c], x, same ? x : BX[i * ldbx + c]);
    }
  }
  sm[0][threadIdx.x] = s0;
  sm[1][threadIdx.x] = s1;
  sm[2][threadIdx.x] = s2;
  sm[3][threadIdx.x] = s3;
  __syncthreads();
  if (threadIdx.x < kc) {
    for (int q = 0; q < 4; ++q) {
      double t = 0.0;
      for (int l = 0; l < lanes; ++l) t += sm[q][l * kc + threadIdx.x];
      part[((long long)blockIdx.x * 4 + q) * k + threadIdx.x] = t;
    }
  }
}

// one 128-thread block per column: the 4 sums over the per-CTA partials in a fixed
// order (thread t: parts t, t + 128, ...; then a fixed tree), then the residual
__global__ void __launch_bounds__(128) ritz_finish_kernel(int k, int nparts, const double* part,
                                                          const double* lam, int mode,
                                                          double* out) {
  __shared__ double sm[4][128];
  const int c = blockIdx.x;
  double s[4] = {0, 0, 0, 0};
  for (int b = threadIdx.x; b < nparts; b += 128)
#pragma unroll
    for (int q = 0; q < 4; ++q) s[q] += part[((long long)b * 4 + q) * k + c];
#pragma unroll
  for (int q = 0; q < 4; ++q) sm[q][threadIdx.x] = s[q];
  __syncthreads();
  for (int w = 64; w > 0; w >>= 1) {
    if (threadIdx.x < w)
#pragma unroll
      for (int q = 0; q < 4; ++q) sm[q][threadIdx.x] += sm[q][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double l = lam[c];
    double den;
    if (mode == 2) {
      den = fabs(l) * sqrt(sm[3][0]);
    } else if (mode == 1) {
      den = sqrt(fmax(sm[2][0], 0.0));
      if (l > 0.0) den *= l;
    } else {
      den = sqrt(sm[1][0]);
    }
    if (den == 0.0) den = 1.0;
    out[c] = sqrt(sm[0][0]) / den;
  }
}

int ritz_residuals_launch(Ctx* c, long long n, int k, const double* AX, long long ldax,
                          const double* X, long long ldx, const double* BX, long long ldbx,
                          const double* lam, int mode, double* out) {
  if (k <= 0) return GCG_OK;
  if (k > 256) return GCG_ERR_ARG;
  int grid = grid_for(n, 1024, 4, c->num_sms);
  long long rpc = (n + grid - 1) / grid;
  grid = (int)((n + rpc - 1) / rpc);
  GCG_TRY(ensure(c->partials, sizeof(double) * (size_t)grid * 4 * k));
  double* part = (double*)c->partials.ptr;
  ritz_partials_kernel<<<grid, 256, 0, c->stream>>>(n, k, AX, ldax, X, ldx, BX, ldbx, lam, mode,
                                                     rpc, part);
  ritz_finish_kernel<<<k, 128, 0, c->stream>>>(k, grid, part, lam, mode, out);
  g_launches += 2;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

// split form for row-partitioned runs: local column sums [4][k] ...
int ritz_sums_launch(Ctx* c, long long n, int k, const double* AX, long long ldax,
                     const double* X, long long ldx, const double* BX, long long ldbx,
                     const double* lam, int mode, double* sums) {
  if (k <= 0) return GCG_OK;
  if (k > 256) return GCG_ERR_ARG;
  if (n <= 0) {
    cudaMemsetAsync(sums, 0, sizeof(double) * 4 * k, c->stream);
    return GCG_OK;
  }
  int grid = grid_for(n, 1024, 4, c->num_sms);
  long long rpc = (n + grid - 1) / grid;
  grid = (int)((n + rpc - 1) / rpc);
  GCG_TRY(ensure(c->partials, sizeof(double) * (size_t)grid * 4 * k));
  double* part = (double*)c->partials.ptr;
  ritz_partials_kernel<<<grid, 256, 0, c->stream>>>(n, k, AX, ldax, X, ldx, BX, ldbx, lam, mode,
                                                     rpc, part);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  GCG_TRY(reduce_partials(c, part, grid, 4 * k, sums, 1, 0));
  ++g_launches;
  return GCG_OK;
}

// ... and the residuals from (globally reduced) sums
int ritz_finish_launch(Ctx* c, int k, const double* sums, const double* lam, int mode,
                       double* out) {
  if (k <= 0) return GCG_OK;
  ritz_finish_kernel<<<k, 128, 0, c->stream>>>(k, 1, sums, lam, mode, out);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

}  // namespace gcg
