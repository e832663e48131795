// Block CG for the damped inverse power step (GCG STEP 6) on B200.
//
// Reference: block_cg (cg.py:33-99).  k independent CG recurrences share one
// operator application per sweep; a column stops once ||r|| <= rel_tol*||r0||
// (cg.py:55-57, 86-88) and freezes when p'op p <= 0 (cg.py:73-82).
//
// B200 design.  The reference compacts the still-active columns every sweep
// (gather copies, cg.py:67-71).  Here all k columns stay in place and
// per-column flags live on the device: the SpMM is done on the full row-major
// block (an active subset costs the same HBM sectors as the whole row run),
// the p'q and ||r||^2 reductions are fused into the SpMM / update epilogues,
// and the scalar recurrences run in 1-CTA "finish" kernels.  No host sync
// happens inside the solve: once every column has stopped, a device flag turns
// the remaining launches into no-ops and the sweep count is read back lazily
// by the caller.  Per sweep HBM traffic ~ SpMM + 24nk (r -= alpha q) + 40nk
// (x += alpha p, p = r + beta p).

#include <stdlib.h>

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
int copy_launch(Ctx* c, long long n, int k, const double* X, long long ldx, double* Y,
                long long ldy);

struct CgState {
  double* rz;
  double* rn;
  double* rn0;
  double* target;
  double* alpha;
  double* beta;
  int* conv;
  int* frozen;
  int* upd;
  int* pup;
  int* skip;
  int* sweeps;
  int* nact;
  int* ticket;
  int* live;
};

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
    if (na == 0) *s.skip = 1;
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
    s.pup[c] = 0;
  }
  if (c == 0 && threadIdx.x == 0) *s.skip = 0;
  // skip is only raised by the last block, after every block passed this point
  publish_active(s, k, !cv, true);
}

// den = p'q per active column; freeze on den <= 0, else alpha = rz / den.
__global__ void cg_fin1(int k, const double* part, int nparts, CgState s) {
  // `live` tells cg_pupdate_kernel whether this sweep ran (its deferred x update
  // must still happen in the sweep that raises `skip`)
  if (*s.skip) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *s.live = 0;
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *s.live = 1;
  __shared__ double sm[128];
  const int c = blockIdx.x;
  const double den = block_sum_parts(part, nparts, k, c, sm);
  if (threadIdx.x == 0) {
    if (c == 0) *s.sweeps += 1;
    int u = 0;
    if (!s.conv[c] && !s.frozen[c]) {
      if (den <= 0.0) {
        s.frozen[c] = 1;
      } else {
        s.alpha[c] = s.rz[c] / den;
        u = 1;
      }
    }
    s.upd[c] = u;
  }
}

// rn = ||r||; converge, else beta = rz_new / rz.  Raises the skip flag when no
// column remains active (the reference's loop exit, cg.py:67-69).
__global__ void cg_fin2(int k, const double* part, int nparts, CgState s) {
  if (*s.skip) return;
  __shared__ double sm[128];
  const int c = blockIdx.x;
  const double rr = block_sum_parts(part, nparts, k, c, sm);
  int active = 0;
  if (threadIdx.x == 0) {
    int p = 0;
    if (s.upd[c]) {
      const double rn = sqrt(rr);
      s.rn[c] = rn;
      if (rn <= s.target[c]) {
        s.conv[c] = 1;
      } else {
        s.beta[c] = rr / s.rz[c];
        s.rz[c] = rr;
        p = 1;
      }
    }
    s.pup[c] = p;
    active = !s.conv[c] && !s.frozen[c];
  }
  publish_active(s, k, active, false);
}

// r -= alpha q ; partial ||r||^2 (updated columns only).  The matching
// x += alpha p is deferred to cg_pupdate_kernel, which reads the old p anyway:
// per sweep 24nk + 40nk bytes instead of 48nk + 24nk.
__global__ void __launch_bounds__(256) cg_update_kernel(long long n, int k, double* r,
                                                        const double* __restrict__ q,
                                                        long long rows_per_cta, double* part,
                                                        CgState s, int* prof_skipped) {
  if (*s.skip) {
    if (prof_skipped && blockIdx.x == 0 && threadIdx.x == 0) *prof_skipped = 1;
    return;
  }
  __shared__ double sm[256];
  const int kc = k;  // k <= 256 (checked by the launcher)
  const int lanes = 256 / kc;
  const int c = threadIdx.x % kc;
  const int rl = threadIdx.x / kc;
  const long long r0 = (long long)blockIdx.x * rows_per_cta;
  long long r1 = r0 + rows_per_cta;
  if (r1 > n) r1 = n;
  double acc = 0.0;
  if (rl < lanes && s.upd[c]) {
    const double al = s.alpha[c];
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
  sm[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < kc) {
    double t = 0.0;
    for (int l = 0; l < lanes; ++l) t += sm[l * kc + threadIdx.x];
    part[(long long)blockIdx.x * k + threadIdx.x] = t;
  }
}

// x += alpha p (columns updated this sweep) then p = r + beta p (columns still iterating)
__global__ void __launch_bounds__(256) cg_pupdate_kernel(long long n, int k, double* x,
                                                         long long ldx,
                                                         const double* __restrict__ r, double* p,
                                                         long long rows_per_cta, CgState s,
                                                         int* prof_skipped) {
  if (!*s.live) {
    if (prof_skipped && blockIdx.x == 0 && threadIdx.x == 0) *prof_skipped = 1;
    return;
  }
  // same (row lane, column) mapping as cg_update_kernel: flags and scalars are
  // per-thread constants, U rows in flight per thread
  const int lanes = 256 / k;
  const int c = threadIdx.x % k;
  const int rl = threadIdx.x / k;
  if (rl >= lanes) return;
  const long long r0 = (long long)blockIdx.x * rows_per_cta;
  long long r1 = r0 + rows_per_cta;
  if (r1 > n) r1 = n;
  const bool ux = s.upd[c], up = s.pup[c];
  if (!ux && !up) return;
  const double al = s.alpha[c], be = s.beta[c];
  constexpr int U = 8;
  long long i = r0 + rl;
  for (; i + (U - 1) * lanes < r1; i += U * lanes) {
    double pv[U], xv[U], rv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long ii = i + u * lanes;
      pv[u] = p[ii * k + c];
      if (ux) xv[u] = x[ii * ldx + c];
      if (up) rv[u] = r[ii * k + c];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long ii = i + u * lanes;
      if (ux) x[ii * ldx + c] = fma(al, pv[u], xv[u]);
      if (up) p[ii * k + c] = fma(be, pv[u], rv[u]);
    }
  }
  for (; i < r1; i += lanes) {
    const double pv = p[i * k + c];
    if (ux) x[i * ldx + c] = fma(al, pv, x[i * ldx + c]);
    if (up) p[i * k + c] = fma(be, pv, r[i * k + c]);
  }
}

__global__ void cg_final(int k, CgState s, int* d_sweeps, int8_t* conv, int8_t* frozen,
                         double* relres) {
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    const double r0 = s.rn0[c];
    relres[c] = s.rn[c] / (r0 > 0.0 ? r0 : 1.0);
    conv[c] = (int8_t)s.conv[c];
    frozen[c] = (int8_t)s.frozen[c];
  }
  if (threadIdx.x == 0) atomicMax(d_sweeps, *s.sweeps);  // max over column chunks
}

int block_cg_chunk(Ctx* c, long long n, long long nnz, const int* rowptr, const int* colidx,
                   const double* val, double shift, int k, const double* rhs, long long ldr,
                   double* x, long long ldx, int max_iters, double rel_tol, int* d_sweeps,
                   int8_t* d_conv, int8_t* d_frozen, double* d_relres, const gcg_cg_dist* dist);

// The k CG recurrences are independent, so they can run in column chunks (each
// chunk's sweep count is the same as in the joint run).  GCG_CG_CHUNK=w forces
// chunks of w columns — e.g. to keep a chunk's x, r, p, q and the CSR streams
// resident in the 126 MB L2.  Measured at cfg2 (k = 20) that is slower (the
// sweep is latency-bound, and chunking multiplies launches), so the default
// is one chunk.
int block_cg_launch(Ctx* c, long long n, long long nnz, const int* rowptr, const int* colidx,
                    const double* val, double shift, int k, const double* rhs, long long ldr,
                    double* x, long long ldx, int max_iters, double rel_tol, int* d_sweeps,
                    int8_t* d_conv, int8_t* d_frozen, double* d_relres, const gcg_cg_dist* dist) {
  if (k <= 0 || k > 256 || n <= 0) return GCG_ERR_ARG;
  GCG_TRY(cuda_status(cudaMemsetAsync(d_sweeps, 0, sizeof(int), c->stream)));
  static const char* env = getenv("GCG_CG_CHUNK");
  int kc = env ? atoi(env) : k;
  if (kc < 1 || kc > k || dist) kc = k;
  for (int c0 = 0; c0 < k; c0 += kc) {
    const int w = (k - c0) < kc ? (k - c0) : kc;
    GCG_TRY(block_cg_chunk(c, n, nnz, rowptr, colidx, val, shift, w, rhs + c0, ldr, x + c0, ldx,
                           max_iters, rel_tol, d_sweeps, d_conv + c0, d_frozen + c0,
                           d_relres + c0, dist));
  }
  return GCG_OK;
}

int gather_rows_launch(Ctx* c, int nidx, const int* idx, int k, const double* X, long long ldx,
                       double* out, long long ldo);

// Row-partitioned runs: refresh the ghost rows [n, n + nghost) of a block
// (ld) from the neighbours — gather the owned rows they need into send_buf,
// let the host exchange send_buf -> recv_buf, scatter into the ghost rows.
static int dist_halo(Ctx* c, const gcg_cg_dist* d, long long n, int k, double* X, long long ld) {
  if (d->nsend > 0) GCG_TRY(gather_rows_launch(c, d->nsend, d->send_idx, k, X, ld, d->send_buf, k));
  if (d->callback(0, k, d->user) != 0) return GCG_ERR_ARG;
  if (d->nghost > 0) GCG_TRY(copy_launch(c, d->nghost, k, d->recv_buf, k, X + n * ld, ld));
  return GCG_OK;
}

// Combine per-CTA partials into k local column sums, then the global sums
// (host allreduce into red_buf); the finish kernels read them as 1 partial.
static int dist_reduce(Ctx* c, const gcg_cg_dist* d, const double* part, int nparts, int k) {
  GCG_TRY(reduce_partials(c, part, nparts, k, d->red_buf, 1, 0));
  ++g_launches;
  if (d->callback(1, k, d->user) != 0) return GCG_ERR_ARG;
  return GCG_OK;
}

int block_cg_chunk(Ctx* c, long long n, long long nnz, const int* rowptr, const int* colidx,
                   const double* val, double shift, int k, const double* rhs, long long ldr,
                   double* x, long long ldx, int max_iters, double rel_tol, int* d_sweeps,
                   int8_t* d_conv, int8_t* d_frozen, double* d_relres, const gcg_cg_dist* dist) {
  const int sgrid = spmm_grid(c, n);
  int ugrid = grid_for(n, 512, 4, c->num_sms);
  long long rpc = (n + ugrid - 1) / ugrid;
  ugrid = (int)((n + rpc - 1) / rpc);
  const int nparts_max = sgrid > ugrid ? sgrid : ugrid;
  const long long nghost = dist ? dist->nghost : 0;
  // workspace: R, Q (n x k), P and X ((n + ghosts) x k) + partials + state.  The
  // iterate lives in the dense X (ld = k) during the sweeps — a strided arena view
  // streams noticeably slower — and is copied back into x at the end.
  // block starts kept 32-byte aligned so the SpMM can gather rows with 256-bit loads
  const size_t vec = ((size_t)n * k + 3) & ~(size_t)3;
  const size_t pvec = ((size_t)(n + nghost) * k + 3) & ~(size_t)3;
  const size_t bytes =
      sizeof(double) * (2 * vec + 2 * pvec + (size_t)nparts_max * k + 6 * (size_t)k) +
      sizeof(int) * (4 * (size_t)k + 5) + 256;
  GCG_TRY(ensure(c->cg, bytes));
  double* R = (double*)c->cg.ptr;
  double* Q = R + vec;
  double* P = Q + vec;
  double* Xc = P + pvec;
  double* part = Xc + pvec;
  double* const x_user = x;
  const long long ldx_user = ldx;
  GCG_TRY(copy_launch(c, n, k, x_user, ldx_user, Xc, k));
  x = Xc;
  ldx = k;
  double* sd = part + (size_t)nparts_max * k;
  CgState s;
  s.rz = sd;
  s.rn = sd + k;
  s.rn0 = sd + 2 * k;
  s.target = sd + 3 * k;
  s.alpha = sd + 4 * k;
  s.beta = sd + 5 * k;
  int* si = (int*)(sd + 6 * k);
  s.conv = si;
  s.frozen = si + k;
  s.upd = si + 2 * k;
  s.pup = si + 3 * k;
  s.skip = si + 4 * k;
  s.sweeps = si + 4 * k + 1;
  s.nact = si + 4 * k + 2;
  s.ticket = si + 4 * k + 3;
  s.live = si + 4 * k + 4;
  GCG_TRY(cuda_status(cudaMemsetAsync(s.skip, 0, 5 * sizeof(int), c->stream)));
  const int fin_threads = k < 32 ? 32 : (k + 31) / 32 * 32;

  // r = rhs - op(x) = -(A x) - shift*x + rhs ; ||r0||^2 partials
  int g = 0;
  if (dist) GCG_TRY(dist_halo(c, dist, n, k, x, ldx));
  GCG_TRY(spmm_launch_parts(c, n, nnz, rowptr, colidx, val, k, x, ldx, -1.0, -shift, x, ldx, 1.0,
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
  GCG_TRY(copy_launch(c, n, k, R, k, P, k));
  for (int it = 0; it < max_iters; ++it) {
    if (dist) GCG_TRY(dist_halo(c, dist, n, k, P, k));
    GCG_TRY(spmm_launch_parts(c, n, nnz, rowptr, colidx, val, k, P, k, 1.0, shift, P, k, 0.0,
                              nullptr, 0, Q, k, 1, P, k, part, &g, s.skip));
    red = part;
    nred = g;
    if (dist) {
      GCG_TRY(dist_reduce(c, dist, part, g, k));
      red = dist->red_buf;
      nred = 1;
    }
    cg_fin1<<<k, 128, 0, c->stream>>>(k, red, nred, s);
    int ps = prof_start(c, PROF_CG_UPDATE, 24.0 * n * k);
    cg_update_kernel<<<ugrid, 256, 0, c->stream>>>(n, k, R, Q, rpc, part, s, prof_skip_slot(c, ps));
    prof_stop(c, ps);
    red = part;
    nred = ugrid;
    if (dist) {
      GCG_TRY(dist_reduce(c, dist, part, ugrid, k));
      red = dist->red_buf;
      nred = 1;
    }
    cg_fin2<<<k, 128, 0, c->stream>>>(k, red, nred, s);
    ps = prof_start(c, PROF_CG_PUPDATE, 40.0 * n * k);
    cg_pupdate_kernel<<<ugrid, 256, 0, c->stream>>>(n, k, x, ldx, R, P, rpc, s,
                                                    prof_skip_slot(c, ps));
    prof_stop(c, ps);
    g_launches += 4;
    GCG_CHECK_LAUNCH();
  }
  GCG_TRY(copy_launch(c, n, k, Xc, k, x_user, ldx_user));
  cg_final<<<1, fin_threads, 0, c->stream>>>(k, s, d_sweeps, d_conv, d_frozen, d_relres);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

}  // namespace gcg
