// Block CG for the damped inverse power step (GCG STEP 6) on B200.
//
// Reference: block_cg (cg.py:33-99).  k independent CG recurrences share one
// operator application per sweep; a column stops once ||r|| <= rel_tol*||r0||
// (cg.py:55-57, 86-88) and freezes when p'op p <= 0 (cg.py:73-82).
//
// B200 design.  The reference compacts the still-active columns every sweep
// (gather copies, cg.py:67-71).  Here all k columns stay in place and
// per-column flags live on the device, and a sweep is TWO kernels:
//
//   1. the fused sweep SpMM (spmm.cu, CG mode) gathers r and, from own-row values,
//      applies the previous sweep's x += alpha p, forms p = r + beta p and
//      q = (A + shift) r + beta q — which equals (A + shift) p without gathering p
//      (Chronopoulos-Gear) — and the p'q partials; its prologue reduces the
//      ||r||^2 partials and takes the stop / beta decisions (cg.py:86-96);
//   2. the r-update: prologue reduces p'q, freezes columns with p'q <= 0 or forms
//      alpha (cg.py:73-84); body r -= alpha q and the ||r||^2 partials.
//
// The SpMM is bound by its L1/L2 gather stream with HBM mostly idle (round-1 ncu:
// DRAM 24 %), so the x / p / q streams ride along in its epilogue instead of a
// third kernel.  Per sweep HBM traffic ~ 12 nnz + 56nk (SpMM) + 24nk (r-update),
// against SpMM + 24nk + 40nk (+8nk own-row p re-read) with a separate p/x kernel.
// No host sync happens inside the solve: once every column has stopped, device
// flags turn the remaining launches into no-ops, and the sweep count is read
// back lazily by the caller.

#include <stdlib.h>

#include "async.cuh"
#include "cgstate.cuh"
#include "common.cuh"

namespace gcg {

extern int64_t g_launches;
int spmm_launch_parts(Ctx* c, long long n, long long nnz, const int* rowptr, const int* colidx,
                      const double* val, int k, const double* X, long long ldx, double alpha,
                      double gamma, const double* Z, long long ldz, double beta,
                      const double* Yin, long long ldyin, double* Y, long long ldy, int dot_mode,
                      const double* W, long long ldw, double* partials, int* grid_out,
                      const int* skip);
int spmm_grid(Ctx* c, long long n);
int spmm_cg_sweep_launch(Ctx* c, long long n, long long nnz, const int* rowptr,
                         const int* colidx, const double* val, int k, const double* R,
                         double shift, double* partials, int* grid_out, const CgSweep& cg);
int fill_launch(Ctx* c, long long n, int k, double v, double* Y, long long ldy);
int copy_launch(Ctx* c, long long n, int k, const double* X, long long ldx, double* Y,
                long long ldy);


// Fixed-order reduction of one column's per-CTA partials by a 128-thread block:
// thread t sums partials t, t+128, ... then a fixed tree — deterministic.
__device__ double block_sum_parts(const double* part, int nparts, int k, int c, double* sm) {
  double v = 0.0;
  for (int b = threadIdx.x; b < nparts; b += blockDim.x) v += part[(long long)b * k + c];
  sm[threadIdx.x] = v;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  const double t = sm[0];
  __syncthreads();
  return t;
}

// Last-block epilogue: block-level counts are combined with an atomic ticket;
// the block that arrives last publishes the skip flag and resets the counters.
__device__ void publish_active(const CgState& s, int k, int my_active, bool reset_sweeps) {
  __shared__ int last;
  if (threadIdx.x == 0) {
    if (my_active) atomicAdd(s.nact, 1);
    __threadfence();
    last = (atomicAdd(s.ticket, 1) == k - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    const int na = atomicAdd(s.nact, 0);
    if (na == 0) *s.skip1 = 1;
    if (reset_sweeps) *s.sweeps = 0;
    *s.nact = 0;
    *s.ticket = 0;
  }
}

// one block per column: ||r0||, target, initial flags
__global__ void cg_init_fin(int k, const double* part, int nparts, double rel_tol, CgState s) {
  __shared__ double sm[128];
  const int c = blockIdx.x;
  const double rr = block_sum_parts(part, nparts, k, c, sm);
  int cv = 0;
  if (threadIdx.x == 0) {
    const double r0 = sqrt(rr);
    s.rn0[c] = r0;
    s.rn[c] = r0;
    s.target[c] = rel_tol * r0;
    cv = r0 <= rel_tol * r0;
    s.conv[c] = cv;
    s.frozen[c] = 0;
    s.rz[c] = rr;
    s.upd[c] = 0;
  }
  if (c == 0 && threadIdx.x == 0) {
    *s.skip1 = 0;
    *s.skip2 = 0;
    *s.pending = 0;
  }
  // skip1 is only raised by the last block, after every block passed this point
  publish_active(s, k, !cv, true);
}

__constant__ int c_prefetch_upd = 0;
__device__ __forceinline__ bool prefetch_upd() { return c_prefetch_upd != 0; }

// r -= alpha q and the ||r||^2 partials, with the alpha step of the recurrence
// (cg.py:73-84) folded in: every CTA reduces the sweep SpMM's p'q partials itself
// and takes the per-column decisions (freeze when p'q <= 0, else alpha = r'r / p'q);
// CTA 0 publishes them.  x += alpha p is left to the next sweep SpMM (or the final
// copy-back): `pending` says it is owed.
__global__ void __launch_bounds__(256) cg_update_kernel(long long n, int k, double* r,
                                                        const double* __restrict__ q,
                                                        long long rows_per_cta,
                                                        const double* spart, int nsp,
                                                        double* part, CgState s, int par,
                                                        int* prof_skipped) {
  // Pull this CTA's r and q rows into L2 while the sweep SpMM drains and the p'q
  // partials are reduced (L2 is the point of coherence, so prefetching lines the
  // predecessor is still writing is safe).
  if (prefetch_upd()) {
    const long long b0 = (long long)blockIdx.x * rows_per_cta * k;
    long long b1 = b0 + rows_per_cta * k;
    if (b1 > n * k) b1 = n * k;
    for (long long e = b0 + threadIdx.x * 16; e < b1; e += 256 * 16) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(r + e));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(q + e));
    }
  }
  pdl_wait();
  if (*s.skip2) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      *s.skip1 = 1;  // propagate: the next sweep SpMM is a no-op too
      if (prof_skipped) *prof_skipped = 1;
    }
    return;
  }
  __shared__ double sm[256];
  __shared__ double s_al[256];
  __shared__ int s_up[256];
  __shared__ int nup;
  if (threadIdx.x == 0) nup = 0;
  cta_column_sums(spart, nsp, k, sm, s_al);
  if (threadIdx.x < k) {
    const int cc = threadIdx.x;
    const double den = s_al[cc];
    int u = 0;
    double al = 0.0;
    if (!s.conv[cc] && !s.frozen[cc]) {
      if (den <= 0.0) {
        if (blockIdx.x == 0) s.frozen[cc] = 1;
      } else {
        al = s.rz[par * k + cc] / den;
        u = 1;
      }
    }
    s_al[cc] = al;
    s_up[cc] = u;
    if (u) atomicAdd(&nup, 1);
    if (blockIdx.x == 0) {
      s.alpha[cc] = al;
      s.upd[cc] = u;
    }
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *s.sweeps += 1;
    *s.pending = 1;
    if (nup == 0) *s.skip1 = 1;  // every column froze: nothing left to sweep
  }
  const int kc = k;  // k <= 256 (checked by the launcher)
  const int lanes = 256 / kc;
  const int c = threadIdx.x % kc;
  const int rl = threadIdx.x / kc;
  const long long r0 = (long long)blockIdx.x * rows_per_cta;
  long long r1 = r0 + rows_per_cta;
  if (r1 > n) r1 = n;
  double acc = 0.0;
  if (rl < lanes && s_up[c]) {
    const double al = s_al[c];
    constexpr int U = 8;  // rows in flight per thread
    long long i = r0 + rl;
    for (; i + (U - 1) * lanes < r1; i += U * lanes) {
      double qv[U], rv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        qv[u] = q[(i + u * lanes) * k + c];
        rv[u] = r[(i + u * lanes) * k + c];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double nr = fma(-al, qv[u], rv[u]);
        r[(i + u * lanes) * k + c] = nr;
        acc = fma(nr, nr, acc);
      }
    }
    for (; i < r1; i += lanes) {
      const double nr = fma(-al, q[i * k + c], r[i * k + c]);
      r[i * k + c] = nr;
      acc = fma(nr, nr, acc);
    }
  }
  pdl_trigger();  // late: see spmm_csr_kernel
  sm[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < kc) {
    double t = 0.0;
    for (int l = 0; l < lanes; ++l) t += sm[l * kc + threadIdx.x];
    part[(long long)blockIdx.x * k + threadIdx.x] = t;
  }
}

// The r-update as a bulk-copy pipeline: one CTA per SM walks a contiguous row range in
// stages of ~16 KB per stream; thread 0 keeps kUpdStages stages of r and q in flight
// (cp.async.bulk into shared memory, completion on the stage's mbarrier) — issued before
// the prologue, so the fixed-order reduction of the sweep's p'q partials and the alpha
// decisions overlap the first loads, and HBM latency is covered by bytes in flight
// instead of by resident warps.  Same per-element arithmetic as cg_update_kernel; the
// ||r||^2 partials are one row per CTA (148 instead of 512 for the sweep's prologue).
constexpr int kUpdStages = 4;
__global__ void __launch_bounds__(256, 1)
    cg_update_bulk_kernel(long long n, int k, double* r, const double* __restrict__ q,
                          long long rows_per_cta, int rows_per_stage, int order,
                          const double* spart, int nsp, double* part, CgState s, int par,
                          int* prof_skipped) {
  extern __shared__ __align__(128) unsigned char upd_smem[];
  __shared__ unsigned long long full[kUpdStages];
  pdl_wait();
  if (*s.skip2) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      *s.skip1 = 1;  // propagate: the next sweep SpMM is a no-op too
      if (prof_skipped) *prof_skipped = 1;
    }
    return;
  }
  // order 0: one contiguous row range per CTA; 1 / 2: stage-sized chunks dealt round-robin
  // over the CTAs, walked from the last rows down (1) or from the first up (2) — the grid
  // then moves through the block as one window, in the direction opposite to the sweep
  // SpMM's (whose last-written rows of q are the freshest lines in L2)
  long long r0 = (long long)blockIdx.x * rows_per_cta;
  long long r1 = r0 + rows_per_cta;
  if (r1 > n) r1 = n;
  const long long nrows = r1 > r0 ? r1 - r0 : 0;
  int nst = (int)((nrows + rows_per_stage - 1) / rows_per_stage);
  const long long nch = (n + rows_per_stage - 1) / rows_per_stage;
  if (order) {
    r1 = n;
    nst = blockIdx.x < nch ? (int)((nch - blockIdx.x + gridDim.x - 1) / gridDim.x) : 0;
  }
  auto stage_row = [&](int st) -> long long {
    if (!order) return r0 + (long long)st * rows_per_stage;
    const long long j = (long long)blockIdx.x + (long long)st * gridDim.x;
    return (order == 1 ? nch - 1 - j : j) * rows_per_stage;
  };
  const size_t sbytes = (size_t)rows_per_stage * k * sizeof(double);  // per stream
  auto issue = [&](int st) {  // thread 0: stage st of this CTA's rows into slot st % kUpdStages
    const long long row = stage_row(st);
    const long long rows = (r1 - row) < rows_per_stage ? (r1 - row) : rows_per_stage;
    const unsigned bytes = (unsigned)(rows * k * sizeof(double));
    const int slot = st % kUpdStages;
    unsigned char* dst = upd_smem + (size_t)slot * 2 * sbytes;
    mbar_expect(&full[slot], 2 * bytes);
    bulk_g2s(dst, r + row * k, bytes, &full[slot]);
    bulk_g2s(dst + sbytes, q + row * k, bytes, &full[slot]);
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < kUpdStages; ++i) mbar_init(&full[i]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < kUpdStages && i < nst; ++i) issue(i);
  }
  __shared__ double sm[256];
  __shared__ double s_al[256];
  __shared__ int s_up[256];
  __shared__ int nup;
  if (threadIdx.x == 0) nup = 0;
  cta_column_sums(spart, nsp, k, sm, s_al);
  if (threadIdx.x < k) {
    const int cc = threadIdx.x;
    const double den = s_al[cc];
    int u = 0;
    double al = 0.0;
    if (!s.conv[cc] && !s.frozen[cc]) {
      if (den <= 0.0) {
        if (blockIdx.x == 0) s.frozen[cc] = 1;
      } else {
        al = s.rz[par * k + cc] / den;
        u = 1;
      }
    }
    s_al[cc] = al;
    s_up[cc] = u;
    if (u) atomicAdd(&nup, 1);
    if (blockIdx.x == 0) {
      s.alpha[cc] = al;
      s.upd[cc] = u;
    }
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *s.sweeps += 1;
    *s.pending = 1;
    if (nup == 0) *s.skip1 = 1;  // every column froze: nothing left to sweep
  }
  const int lanes = 256 / k;
  const int c = threadIdx.x % k;
  const int rl = threadIdx.x / k;
  const bool upd = rl < lanes && s_up[c];
  const double al = s_al[c];
  double acc = 0.0;
  for (int st = 0; st < nst; ++st) {
    const int slot = st % kUpdStages;
    mbar_wait(&full[slot], (unsigned)((st / kUpdStages) & 1));
    const long long row = stage_row(st);
    const int rows = (int)((r1 - row) < rows_per_stage ? (r1 - row) : rows_per_stage);
    const double* sr = reinterpret_cast<const double*>(upd_smem + (size_t)slot * 2 * sbytes);
    const double* sq = reinterpret_cast<const double*>(upd_smem + (size_t)slot * 2 * sbytes + sbytes);
    if (upd) {
      double* rout = r + row * k + c;
#pragma unroll 4
      for (int i = rl; i < rows; i += lanes) {
        const double nr = fma(-al, sq[i * k + c], sr[i * k + c]);
        rout[(long long)i * k] = nr;
        acc = fma(nr, nr, acc);
      }
    }
    __syncthreads();  // every thread is done with the slot: refill it
    if (threadIdx.x == 0 && st + kUpdStages < nst) issue(st + kUpdStages);
  }
  pdl_trigger();  // late: see spmm_csr_kernel
  sm[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < k) {
    double t = 0.0;
    for (int l = 0; l < lanes; ++l) t += sm[l * k + threadIdx.x];
    part[(long long)blockIdx.x * k + threadIdx.x] = t;
  }
}

// After the last sweep (256 threads, one CTA): when the last r-update's stop test is
// still owed (no sweep SpMM followed it), reduce its ||r||^2 partials exactly as the
// sweep SpMM's prologue would and test; then the report (cg.py:98-99).
__global__ void __launch_bounds__(256) cg_final(int k, CgState s, const double* rpart, int nrp,
                                                int* d_sweeps, int8_t* conv, int8_t* frozen,
                                                double* relres) {
  __shared__ double sm[256], rr[256];
  const int pend = *s.pending;
  if (pend) cta_column_sums(rpart, nrp, k, sm, rr);
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    double rn = s.rn[c];
    int cv = s.conv[c];
    if (pend && s.upd[c]) {
      rn = sqrt(rr[c]);
      if (rn <= s.target[c]) cv = 1;
    }
    const double r0 = s.rn0[c];
    relres[c] = rn / (r0 > 0.0 ? r0 : 1.0);
    conv[c] = (int8_t)cv;
    frozen[c] = (int8_t)s.frozen[c];
  }
  if (threadIdx.x == 0) atomicMax(d_sweeps, *s.sweeps);  // max over column chunks
}

// x_user = X + alpha P for the columns whose last x-update is still owed, else X.
__global__ void __launch_bounds__(256) cg_xout_kernel(long long n, int k,
                                                      const double* __restrict__ X,
                                                      const double* __restrict__ P, double* x,
                                                      long long ldx, long long rows_per_cta,
                                                      CgState s) {
  __shared__ double s_al[256];
  __shared__ int s_use[256];
  if (threadIdx.x < k) {
    const int use = *s.pending && s.upd[threadIdx.x];
    s_use[threadIdx.x] = use;
    s_al[threadIdx.x] = use ? s.alpha[threadIdx.x] : 0.0;
  }
  __syncthreads();
  const int lanes = 256 / k;
  const int c = threadIdx.x % k, rl = threadIdx.x / k;
  if (rl >= lanes) return;
  const long long r0 = (long long)blockIdx.x * rows_per_cta;
  long long r1 = r0 + rows_per_cta;
  if (r1 > n) r1 = n;
  const bool use = s_use[c];
  const double al = s_al[c];
  for (long long i = r0 + rl; i < r1; i += lanes) {
    const double xv = X[i * k + c];
    x[i * ldx + c] = use ? fma(al, P[i * k + c], xv) : xv;
  }
}

int block_cg_chunk(Ctx* c, long long n, long long nnz, const int* rowptr, const int* colidx,
                   const double* val, double shift, int k, const double* rhs, long long ldr,
                   const double* x0, long long ldx0, double* x, long long ldx, int max_iters,
                   double rel_tol, int* d_sweeps, int8_t* d_conv, int8_t* d_frozen,
                   double* d_relres, const gcg_cg_dist* dist);

// The k CG recurrences are independent, so they can run in column chunks (each
// chunk's sweep count is the same as in the joint run).  GCG_CG_CHUNK=w forces
// chunks of w columns — e.g. to keep a chunk's x, r, p, q and the CSR streams
// resident in the 126 MB L2.  Measured at cfg2 (k = 20) that is slower (the
// sweep is latency-bound, and chunking multiplies launches), so the default
// is one chunk.
int block_cg_launch(Ctx* c, long long n, long long nnz, const int* rowptr, const int* colidx,
                    const double* val, double shift, int k, const double* rhs, long long ldr,
                    const double* x0, long long ldx0, double* x, long long ldx, int max_iters,
                    double rel_tol, int* d_sweeps, int8_t* d_conv, int8_t* d_frozen,
                    double* d_relres, const gcg_cg_dist* dist) {
  if (k <= 0 || n <= 0) return GCG_ERR_ARG;
  static const bool pf_set = [] {
    const int v = getenv("GCG_CG_UPD_PREFETCH") ? atoi(getenv("GCG_CG_UPD_PREFETCH")) : 0;
    return cudaMemcpyToSymbol(c_prefetch_upd, &v, sizeof(int)) == cudaSuccess;
  }();
  (void)pf_set;
  GCG_TRY(cuda_status(cudaMemsetAsync(d_sweeps, 0, sizeof(int), c->stream)));
  static const char* env = getenv("GCG_CG_CHUNK");
  int kc = env ? atoi(env) : k;
  if (kc < 1 || kc > k) kc = k;
  // the sweep kernels hold one column per thread slot of a 256-thread CTA: wider
  // blocks (block_size > 256, e.g. nev > 1280) run in column chunks, each with
  // the same sweep count as the joint run (the reported count is the max)
  if (kc > 256) kc = (k + (k + 255) / 256 - 1) / ((k + 255) / 256);
  // A column count that is not a multiple of 4 (the last iterations of a solve, when
  // fewer than block_size pairs are left) loses the 32-byte row gathers and the bulk
  // r-update: at cfg2 a sweep pair costs 142 / 110 / 123 us at k = 19 / 18 / 17 against
  // 88 us at k = 20.  Such a block runs padded with zero right-hand sides instead — a zero
  // column converges at sweep 0 and is never touched again (cg.py:56-60), the other
  // columns' recurrences are unchanged.  GCG_CG_PAD=0 disables; not for row-partitioned
  // runs (their halo buffers are sized for k).
  static const bool pad_on = !(getenv("GCG_CG_PAD") && getenv("GCG_CG_PAD")[0] == '0');
  for (int c0 = 0; c0 < k; c0 += kc) {
    const int w = (k - c0) < kc ? (k - c0) : kc;
    const int wp = (w + 3) & ~3;
    if (pad_on && !dist && w > 4 && wp != w && wp <= 256) {
      const size_t blk = (size_t)n * wp;
      GCG_TRY(ensure(c->cgpad, sizeof(double) * (2 * blk + wp) + 2 * (size_t)wp + 256));
      double* rhs_p = (double*)c->cgpad.ptr;
      double* x_p = rhs_p + blk;
      double* relres_p = x_p + blk;
      int8_t* conv_p = (int8_t*)(relres_p + wp);
      int8_t* frozen_p = conv_p + wp;
      GCG_TRY(fill_launch(c, n, wp - w, 0.0, rhs_p + w, wp));
      GCG_TRY(fill_launch(c, n, wp - w, 0.0, x_p + w, wp));
      GCG_TRY(copy_launch(c, n, w, rhs + c0, ldr, rhs_p, wp));
      GCG_TRY(copy_launch(c, n, w, x0 ? x0 + c0 : x + c0, x0 ? ldx0 : ldx, x_p, wp));
      GCG_TRY(block_cg_chunk(c, n, nnz, rowptr, colidx, val, shift, wp, rhs_p, wp, nullptr, 0, x_p,
                             wp, max_iters, rel_tol, d_sweeps, conv_p, frozen_p, relres_p, nullptr));
      GCG_TRY(copy_launch(c, n, w, x_p, wp, x + c0, ldx));
      GCG_TRY(cuda_status(cudaMemcpyAsync(d_conv + c0, conv_p, (size_t)w, cudaMemcpyDeviceToDevice, c->stream)));
      GCG_TRY(cuda_status(cudaMemcpyAsync(d_frozen + c0, frozen_p, (size_t)w, cudaMemcpyDeviceToDevice, c->stream)));
      GCG_TRY(cuda_status(cudaMemcpyAsync(d_relres + c0, relres_p, sizeof(double) * (size_t)w,
                                          cudaMemcpyDeviceToDevice, c->stream)));
      continue;
    }
    GCG_TRY(block_cg_chunk(c, n, nnz, rowptr, colidx, val, shift, w, rhs + c0, ldr,
                           x0 ? x0 + c0 : nullptr, ldx0, x + c0, ldx, max_iters, rel_tol,
                           d_sweeps, d_conv + c0, d_frozen + c0, d_relres + c0, dist));
  }
  return GCG_OK;
}

int gather_rows_launch(Ctx* c, int nidx, const int* idx, int k, const double* X, long long ldx,
                       double* out, long long ldo);

// Row-partitioned runs: refresh the ghost rows [n, n + nghost) of a block
// (ld) from the neighbours — gather the owned rows they need into send_buf,
// let the host exchange send_buf -> recv_buf, scatter into the ghost rows.
int nccl_cg_halo(Ctx* c, const gcg_cg_dist* d, int k);
int nccl_cg_allreduce(Ctx* c, const gcg_cg_dist* d, int k);

static int dist_halo(Ctx* c, const gcg_cg_dist* d, long long n, int k, double* X, long long ld) {
  if (d->nsend > 0) GCG_TRY(gather_rows_launch(c, d->nsend, d->send_idx, k, X, ld, d->send_buf, k));
  if (d->nccl_comm) {
    GCG_TRY(nccl_cg_halo(c, d, k));  // grouped send / recv on the context stream
  } else if (d->callback(0, k, d->user) != 0) {
    return GCG_ERR_ARG;
  }
  if (d->nghost > 0) GCG_TRY(copy_launch(c, d->nghost, k, d->recv_buf, k, X + n * ld, ld));
  return GCG_OK;
}

// Combine per-CTA partials into k local column sums, then the global sums
// (host allreduce into red_buf); the finish kernels read them as 1 partial.
static int dist_reduce(Ctx* c, const gcg_cg_dist* d, const double* part, int nparts, int k) {
  GCG_TRY(reduce_partials(c, part, nparts, k, d->red_buf, 1, 0));
  ++g_launches;
  if (d->nccl_comm) return nccl_cg_allreduce(c, d, k);
  if (d->callback(1, k, d->user) != 0) return GCG_ERR_ARG;
  return GCG_OK;
}

int block_cg_chunk(Ctx* c, long long n, long long nnz, const int* rowptr, const int* colidx,
                   const double* val, double shift, int k, const double* rhs, long long ldr,
                   const double* x0, long long ldx0, double* x, long long ldx, int max_iters,
                   double rel_tol, int* d_sweeps, int8_t* d_conv, int8_t* d_frozen,
                   double* d_relres, const gcg_cg_dist* dist) {
  if (k <= 0 || k > 256) return GCG_ERR_ARG;
  const int sgrid = spmm_grid(c, n);
  int ugrid = grid_for(n, 512, 4, c->num_sms);
  long long rpc = (n + ugrid - 1) / ugrid;
  ugrid = (int)((n + rpc - 1) / rpc);
  const int nparts_max = sgrid > ugrid ? sgrid : ugrid;
  // bulk-copy r-update: one CTA per SM over an even number of rows, stages of <= 16 KB per
  // stream in whole row-lane rounds (GCG_CG_UPD_BULK=0: the register-streamed kernel)
  // (even k only: bulk copies move 16-byte multiples, and a range's last stage may hold an
  // odd number of rows)
  static const bool upd_bulk_env = !(getenv("GCG_CG_UPD_BULK") && getenv("GCG_CG_UPD_BULK")[0] == '0');
  const bool upd_bulk = upd_bulk_env && k % 2 == 0;
  long long brpc = ((n + c->num_sms - 1) / c->num_sms + 1) & ~1LL;
  if (brpc < 64) brpc = 64;
  const int bgrid = (int)((n + brpc - 1) / brpc);
  int brps = (int)(16384 / (sizeof(double) * k));
  if (brps >= 256 / k) brps -= brps % (256 / k);
  brps &= ~1;
  if (brps < 2) brps = 2;
  const size_t bsmem = (size_t)kUpdStages * 2 * brps * k * sizeof(double);
  if (upd_bulk) {
    static size_t smem_set = 0;
    if (bsmem > smem_set) {
      GCG_TRY(cuda_status(cudaFuncSetAttribute(cg_update_bulk_kernel,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem)));
      smem_set = bsmem;
    }
  }
  static const int upd_order = getenv("GCG_CG_UPD_ORDER") ? atoi(getenv("GCG_CG_UPD_ORDER")) : 1;
  const int rgrid = upd_bulk ? bgrid : ugrid;  // CTAs (= partial rows) of the r-update
  const long long nghost = dist ? dist->nghost : 0;
  // workspace: R and X ((n + ghosts) x k: both are gathered by an SpMM), P, Q (n x k)
  // + partials + state.  The iterate lives in the dense X (ld = k) during the sweeps —
  // a strided arena view streams noticeably slower — and is copied back into x at the
  // end.  Block starts kept 32-byte aligned so the SpMM can gather rows with 256-bit
  // loads.
  const size_t vec = ((size_t)n * k + 3) & ~(size_t)3;
  const size_t pvec = ((size_t)(n + nghost) * k + 3) & ~(size_t)3;
  const size_t bytes =
      sizeof(double) * (2 * vec + 2 * pvec + 2 * (size_t)nparts_max * k + 7 * (size_t)k) +
      sizeof(int) * (3 * (size_t)k + 8) + 256;
  GCG_TRY(ensure(c->cg, bytes));
  double* R = (double*)c->cg.ptr;
  double* Xc = R + pvec;
  double* Q = Xc + pvec;
  double* P = Q + vec;
  double* part = P + vec;
  double* const x_user = x;
  const long long ldx_user = ldx;
  // initial guess: x0 when given (the caller's X block), else the iterate's own input
  GCG_TRY(copy_launch(c, n, k, x0 ? x0 : x_user, x0 ? ldx0 : ldx_user, Xc, k));
  double* upart = part + (size_t)nparts_max * k;  // r-update partials (SpMM's stay readable)
  double* sd = upart + (size_t)nparts_max * k;
  CgState s;
  s.rz = sd;  // 2k
  s.rn = sd + 2 * k;
  s.rn0 = sd + 3 * k;
  s.target = sd + 4 * k;
  s.alpha = sd + 5 * k;
  int* si = (int*)(sd + 7 * k);
  s.conv = si;
  s.frozen = si + k;
  s.upd = si + 2 * k;
  s.skip1 = si + 3 * k;
  s.skip2 = si + 3 * k + 1;
  s.pending = si + 3 * k + 2;
  s.sweeps = si + 3 * k + 3;
  s.nact = si + 3 * k + 4;
  s.ticket = si + 3 * k + 5;
  GCG_TRY(cuda_status(cudaMemsetAsync(s.skip1, 0, 6 * sizeof(int), c->stream)));

  // r = rhs - op(x) = -(A x) - shift*x + rhs ; ||r0||^2 partials
  int g = 0;
  if (dist) GCG_TRY(dist_halo(c, dist, n, k, Xc, k));
  GCG_TRY(spmm_launch_parts(c, n, nnz, rowptr, colidx, val, k, Xc, k, -1.0, -shift, Xc, k, 1.0,
                            rhs, ldr, R, k, 2, nullptr, 0, part, &g, nullptr));
  const double* red = part;
  int nred = g;
  if (dist) {
    GCG_TRY(dist_reduce(c, dist, part, g, k));
    red = dist->red_buf;
    nred = 1;
  }
  cg_init_fin<<<k, 128, 0, c->stream>>>(k, red, nred, rel_tol, s);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  const double* rred = nullptr;  // ||r||^2 partials of the last r-update
  int nrred = 0;
  for (int it = 0; it < max_iters; ++it) {
    // sweep SpMM: x += alpha p (owed), p = r + beta p, q = (A + shift) r + beta q, p'q
    if (dist) GCG_TRY(dist_halo(c, dist, n, k, R, k));
    CgSweep sw;
    sw.s = s;
    sw.rpart = rred;
    sw.nrp = nrred;
    sw.k = k;
    sw.par = it & 1;
    sw.first = it == 0;
    sw.x = Xc;
    sw.P = P;
    sw.Q = Q;
    GCG_TRY(spmm_cg_sweep_launch(c, n, nnz, rowptr, colidx, val, k, R, shift, part, &g, sw));
    red = part;
    nred = g;
    if (dist) {
      GCG_TRY(dist_reduce(c, dist, part, g, k));
      red = dist->red_buf;
      nred = 1;
    }
    // r-update: alpha = r'r / p'q (freeze on p'q <= 0), r -= alpha q, ||r||^2 partials
    const int ps = prof_start(c, PROF_CG_UPDATE, 24.0 * n * k);
    if (upd_bulk)
      pdl_launch(cg_update_bulk_kernel, dim3(bgrid), dim3(256), bsmem, c->stream, n, k, R,
                 (const double*)Q, (long long)brpc, brps, upd_order, red, nred, upart, s, (it & 1) ^ 1,
                 prof_skip_slot(c, ps));
    else
      pdl_launch(cg_update_kernel, dim3(ugrid), dim3(256), 0, c->stream, n, k, R, (const double*)Q,
                 (long long)rpc, red, nred, upart, s, (it & 1) ^ 1, prof_skip_slot(c, ps));
    prof_stop(c, ps);
    ++g_launches;
    GCG_CHECK_LAUNCH();
    rred = upart;
    nrred = rgrid;
    if (dist) {
      GCG_TRY(dist_reduce(c, dist, upart, rgrid, k));
      rred = dist->red_buf;
      nrred = 1;
    }
  }
  const int ps = prof_start(c, PROF_CG_XOUT, 24.0 * n * k);
  cg_xout_kernel<<<ugrid, 256, 0, c->stream>>>(n, k, Xc, P, x_user, ldx_user, (long long)rpc, s);
  prof_stop(c, ps);
  cg_final<<<1, 256, 0, c->stream>>>(k, s, rred ? rred : part, rred ? nrred : 0, d_sweeps, d_conv,
                                     d_frozen, d_relres);
  g_launches += 2;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

}  // namespace gcg
