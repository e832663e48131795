/*
 * gcgb200 — C ABI of the B200-native GCG hot path (sm_100a, fp64).
 *
 * Two tiers of entry points, both plain `extern "C"` with pointers + sizes and
 * an int status (0 = ok; never a C++ exception across the ABI):
 *
 *  1. Reference-FFI mirror (host buffers).  `gcgeig_csr_matvec`,
 *     `gcgeig_inner_product` and `gcgeig_axpby` take exactly the arguments of
 *     the reference's kernel-backend functions
 *         csr_matvec(indptr, indices, data, x, out)        _kernels/__init__.py:54-55, _cy.pyx:11-23
 *         inner_product(x, y, out, chunk, deterministic)   _kernels/__init__.py:58-59, _cy.pyx:26-50
 *         axpby(alpha, x, beta, y)                         _kernels/__init__.py:62-63, _cy.pyx:53-65
 *     (column-major host arrays, int64 CSR indices, a strided `out`), copy to
 *     HBM, run the device kernels and copy back.  They back the `sm100`
 *     backend registered in gcgeig._kernels._IMPLS.
 *
 *  2. Device tier (device pointers, row-major multivectors, caller stream).
 *     Element (i, c) of a multivector lives at X[i*ld + c]; small dense
 *     matrices are row-major with leading dimension ld.  These are the GCGE
 *     ops surface:
 *         MatDotMultiVec      -> gcg_spmm_csr          (operators.py:103-111, 149-156)
 *         MultiVecInnerProd   -> gcg_gram              (multivec.py:84-112)
 *         MultiVecLinearComb  -> gcg_lincomb           (solver.py:300,333,376; orth.py:144,175,184)
 *         MultiVecAxpby       -> gcg_axpby             (multivec.py:62-73)
 *         block CG (STEP 6)   -> gcg_block_cg          (cg.py:33-99)
 *         dense RR eigensolve -> gcg_syev              (dense.py:74-133, sign rule dense.py:63-71)
 *     plus fused decision kernels for the B-orthogonalisation
 *     (orth.py:124-188) and the convergence test (solver.py:129-164).
 *
 * Every device entry point is asynchronous on the context's stream and never
 * allocates user-visible memory (workspace lives in the context).
 */
#ifndef GCGB200_H
#define GCGB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  GCG_OK = 0,
  GCG_ERR_ARG = 1,     /* bad argument (maps to InvalidShape / InvalidRange)   */
  GCG_ERR_CUDA = 2,    /* CUDA runtime error                                    */
  GCG_ERR_SOLVER = 3,  /* dense eigensolver failure (maps to NoConvergence)     */
  GCG_ERR_ALLOC = 4,   /* device allocation failed                              */
  GCG_ERR_NODEV = 5,   /* no CUDA device                                        */
  GCG_ERR_IO = 6,      /* file could not be read (maps to IoError)              */
  GCG_ERR_PARSE = 7,   /* malformed input file (maps to ParseError + line)      */
  GCG_ERR_UNSUPPORTED = 8 /* well-formed but unhandled input (Unsupported)      */
};

#define GCG_ABI_VERSION 1

int gcg_abi_version(void);
const char* gcg_status_string(int status);

/* ---- context ------------------------------------------------------------ */
int gcg_ctx_create(void** ctx, void* cuda_stream);
int gcg_ctx_destroy(void* ctx);
int gcg_ctx_set_stream(void* ctx, void* cuda_stream);
int gcg_ctx_sync(void* ctx);
/* number of kernels this library has launched since load (instrumentation) */
int64_t gcg_launch_count(void);
/* number of cuSOLVER eigensolver calls since load (0 for every order <= 1024) */
int64_t gcg_cusolver_calls(void);
/* Live kernel timing: between begin and end every SpMM / Gram / LinComb / CG-update /
 * CG-p-update launch on this ctx is bracketed by CUDA events on the ctx stream.
 * end() synchronises and writes out[3*cls + {0,1,2}] = {total ms, launches,
 * algorithmic HBM bytes} for cls = 0..5: SpMM, Gram, LinComb, CG r-update, CG
 * x-copy-out, fused CG sweep SpMM. */
int gcg_prof_begin(void* ctx);
int gcg_prof_end(void* ctx, double* out);
/* time only every stride-th launch of each class (stride >= 1, default 1): the
 * event records then perturb a timed region by 1/stride as much; ms, launches
 * and bytes in gcg_prof_end refer to the sampled launches. */
int gcg_prof_sample(void* ctx, int stride);

/* ---- tier 1: reference-FFI mirror (host buffers, column-major) ----------- */
/* out[:, c] = A @ x[:, c];  A is nrow x ncol CSR (int64 indptr/indices, f64 data);
 * x is ncol x k with column stride ldx; out is nrow x k with column stride ldo. */
int gcgeig_csr_matvec(const int64_t* indptr, const int64_t* indices, const double* data,
                      int64_t nrow, int64_t ncol, const double* x, int64_t k, int64_t ldx,
                      double* out, int64_t ldo);
/* A CSR operator kept resident in HBM — replaces CsrOperator.apply
 * (operators.py:103-111; the reference's `kernels.csr_matvec` per call re-reads
 * the matrix).  create uploads indptr/indices (int64, validated: monotone row
 * pointers, column indices in [0, ncol)) and data once; apply computes
 * out[:, c] = A @ x[:, c] for F-order host blocks (x: ncol x k, column stride
 * ldx; out: nrow x k, column stride ldo); destroy frees it (NULL is a no-op). */
int gcgeig_csr_create(const int64_t* indptr, const int64_t* indices, const double* data,
                      int64_t nrow, int64_t ncol, void** handle);
int gcgeig_csr_apply(void* handle, const double* x, int64_t k, int64_t ldx, double* out,
                     int64_t ldo);
int gcgeig_csr_destroy(void* handle);
/* out[r*out_rs + c*out_cs] = sum_i x[i + r*ldx] * y[i + c*ldy]  (x: n x kx, y: n x ky).
 * Always bit-stable run to run; `chunk`/`deterministic` are accepted for interface parity. */
int gcgeig_inner_product(const double* x, int64_t n, int64_t kx, int64_t ldx, const double* y,
                         int64_t ky, int64_t ldy, double* out, int64_t out_rs, int64_t out_cs,
                         int64_t chunk, int deterministic);
/* y <- alpha x + beta y on n x k column-major blocks; beta == 0 never reads y. */
int gcgeig_axpby(double alpha, const double* x, int64_t n, int64_t k, int64_t ldx, double beta,
                 double* y, int64_t ldy);

/* ---- tier 2: device ops --------------------------------------------------- */
/* Y = alpha*(A X) + gamma*Z + beta*Yin, rows 0..n-1, k columns; A is CSR with
 * int32 indices.  beta == 0 never reads Yin; gamma == 0 never reads Z.
 * dot_mode 0: none; 1: dots[c] = sum_i Y[i,c] W[i,c]; 2: dots[c] = sum_i Y[i,c]^2
 * (deterministic fixed-order reduction). */
int gcg_spmm_csr(void* ctx, int64_t n, int64_t nnz, const int32_t* rowptr, const int32_t* colidx,
                 const double* val, int64_t k, const double* X, int64_t ldx, double alpha,
                 double gamma, const double* Z, int64_t ldz, double beta, const double* Yin,
                 int64_t ldyin, double* Y, int64_t ldy, int dot_mode, const double* W,
                 int64_t ldw, double* dots);

/* G[r*g_rs + c*g_cs] = alpha * sum_i X[i,r] Y[i,c] + beta * G[...]  (beta == 0: no read)
 * optional fused column dots: dots[c] = sum_i T[i,c] Y[i,c] (T may equal Y). */
/* SELL-C-sigma form of a CSR matrix (C = 32; sigma 1 keeps the row order, any other
 * value sorts rows by length inside windows of 1024 rows).  gcg_sell_size returns the
 * slice count and the padded entry count (synchronises); gcg_csr_to_sell fills the
 * caller's arrays: slice_ptr (nslices + 1), perm (n: sorted position -> row),
 * sell_col / sell_val (nnz_padded; sell_val may be NULL for a pattern-only copy).
 * gcg_spmm_sell has gcg_spmm_csr's epilogue and dot modes and gives the same
 * results.  SURVEY §8(b) MatDotMultiVec -> gcg_spmm_sell; operators.py:103-111. */
int gcg_sell_size(void* ctx, int64_t n, const int32_t* rowptr, int32_t sigma, int64_t* nslices,
                  int64_t* nnz_padded);
int gcg_csr_to_sell(void* ctx, int64_t n, const int32_t* rowptr, const int32_t* colidx,
                    const double* val, int32_t sigma, int64_t* slice_ptr, int32_t* perm,
                    int32_t* sell_col, double* sell_val);
int gcg_spmm_sell(void* ctx, int64_t n, int64_t nslices, const int64_t* slice_ptr,
                  const int32_t* perm, const int32_t* sell_col, const double* sell_val, int64_t k,
                  const double* X, int64_t ldx, double alpha, double gamma, const double* Z,
                  int64_t ldz, double beta, const double* Yin, int64_t ldyin, double* Y,
                  int64_t ldy, int dot_mode, const double* W, int64_t ldw, double* dots);

int gcg_gram(void* ctx, int64_t n, int64_t k1, int64_t k2, const double* X, int64_t ldx,
             const double* Y, int64_t ldy, double alpha, double beta, double* G, int64_t g_rs,
             int64_t g_cs, const double* T, int64_t ldt, double* dots);

/* Y = alpha * X C + beta * Y;  X: n x m, C: m x d (row-major, ldc), Y: n x d.
 * Y may share rows with X (same row stride): column ranges disjoint, or in
 * place (Y row i inside X row i) when d <= 256 — one CTA owns all output
 * columns of its rows; any other overlap is GCG_ERR_ARG. */
int gcg_lincomb(void* ctx, int64_t n, int64_t m, int64_t d, double alpha, const double* X,
                int64_t ldx, const double* C, int64_t ldc, double beta, double* Y, int64_t ldy);

/* Y = alpha X + beta Y (n x k); beta == 0 never reads Y. */
int gcg_axpby(void* ctx, int64_t n, int64_t k, double alpha, const double* X, int64_t ldx,
              double beta, double* Y, int64_t ldy);
/* Y = X (n x k strided copy). */
int gcg_copy(void* ctx, int64_t n, int64_t k, const double* X, int64_t ldx, double* Y,
             int64_t ldy);
/* X[:, c] *= s[c]  (s on device) */
int gcg_col_scale(void* ctx, int64_t n, int64_t k, const double* s, double* X, int64_t ldx);
/* out[c] = sum_i X[i,c] Y[i,c] */
int gcg_col_dots(void* ctx, int64_t n, int64_t k, const double* X, int64_t ldx, const double* Y,
                 int64_t ldy, double* out);
/* fill n x k with 0 */
int gcg_fill(void* ctx, int64_t n, int64_t k, double value, double* X, int64_t ldx);

/* Block CG on op = A + diag_shift*I (A = the shifted-value CSR A - theta*B when B is
 * stored on A's pattern).  x holds x0 on entry and the iterate on exit.  Per column:
 * stop at rel_tol*||r0|| or after max_iters sweeps, freeze on p'op p <= 0 (cg.py:33-99).
 * Outputs stay on device: *d_sweeps, d_converged[k], d_frozen[k], d_relres[k]. */
int gcg_block_cg(void* ctx, int64_t n, int64_t nnz, const int32_t* rowptr, const int32_t* colidx,
                 const double* val, double diag_shift, int64_t k, const double* rhs,
                 int64_t ldr, double* x, int64_t ldx, int32_t max_iters, double rel_tol,
                 int32_t* d_sweeps, int8_t* d_converged, int8_t* d_frozen, double* d_relres);

/* gcg_block_cg with the initial guess read from x0 (ldx0) instead of x: the iterate is
 * written to x only (saves the caller's copy of the X block into the W block). */
int gcg_block_cg_x0(void* ctx, int64_t n, int64_t nnz, const int32_t* rowptr,
                    const int32_t* colidx, const double* val, double diag_shift, int64_t k,
                    const double* rhs, int64_t ldr, const double* x0, int64_t ldx0, double* x,
                    int64_t ldx, int32_t max_iters, double rel_tol, int32_t* d_sweeps,
                    int8_t* d_converged, int8_t* d_frozen, double* d_relres);

/* Y[i, c] = s[c] * X[i, c] (one pass; the block-CG right-hand side (Lambda - theta) X). */
int gcg_col_scale_copy(void* ctx, int64_t n, int64_t k, const double* s, const double* X,
                       int64_t ldx, double* Y, int64_t ldy);

/* Row-partitioned (multi-GPU) block CG.  Rows [0, n) are owned; rows [n, n + nghost)
 * of x (and of the internal direction block) are ghost copies of neighbours' rows
 * that the local CSR references (column indices >= n).  The host exchanges them:
 *   callback(0, k, user): halo — send_buf (nsend x k, packed) -> recv_buf (nghost x k),
 *                          the library gathers rows send_idx[] before and scatters
 *                          recv_buf into the ghost rows after;
 *   callback(1, k, user): allreduce — red_buf[0:k] holds this rank's column sums on
 *                          entry and must hold the global sums on return.
 * Both are called from the enqueuing thread, stream-ordered on the context stream.
 * With nccl_comm set (gcg_nccl_comm_create) there is no callback: the library
 * exchanges the halo itself (grouped ncclSend / ncclRecv with each of the npeer
 * neighbours: send_buf rows [peer_send_off[q], peer_send_off[q+1]) to peer_rank[q],
 * recv_buf rows [peer_recv_off[q], ...) from it) and sums red_buf with ncclAllReduce,
 * all on the context stream — no host round trip inside the CG. */
typedef struct gcg_cg_dist {
  int64_t nghost;
  int64_t nsend;
  const int32_t* send_idx; /* device [nsend], local row indices */
  double* send_buf;        /* device [nsend * k] */
  double* recv_buf;        /* device [nghost * k] */
  double* red_buf;         /* device [k] */
  int (*callback)(int op, int k, void* user);
  void* user;
  void* nccl_comm;              /* ncclComm_t or NULL (host callbacks) */
  int32_t npeer;
  const int32_t* peer_rank;     /* host [npeer] */
  const int64_t* peer_send_off; /* host [npeer + 1], rows of send_buf */
  const int64_t* peer_recv_off; /* host [npeer + 1], rows of recv_buf */
} gcg_cg_dist;

/* ---- native NCCL (loaded at run time; gcg_nccl_available() == 0 without it) ---- */
int gcg_nccl_available(void);                       /* NCCL version code, 0 if absent */
int gcg_nccl_unique_id(uint8_t* out128);            /* rank 0: the bootstrap id */
int gcg_nccl_comm_create(void* ctx, int32_t nranks, int32_t rank, const uint8_t* id128,
                         void** comm);
int gcg_nccl_comm_destroy(void* comm);
/* in-place sum of count doubles over the communicator, on the context stream */
int gcg_nccl_allreduce_sum(void* ctx, void* comm, double* buf, int64_t count);

int gcg_block_cg_dist(void* ctx, int64_t n, int64_t nnz, const int32_t* rowptr,
                      const int32_t* colidx, const double* val, double diag_shift, int64_t k,
                      const double* rhs, int64_t ldr, double* x, int64_t ldx, int32_t max_iters,
                      double rel_tol, int32_t* d_sweeps, int8_t* d_converged, int8_t* d_frozen,
                      double* d_relres, const gcg_cg_dist* dist);

/* FP64 peak probe (roofline denominator): mode 1 = DMMA.8x8x4 chains, 0 = DFMA chains;
 * *flops_per_launch receives the flop count of the launch (time it with events). */
int gcg_fp64_peak(void* ctx, int mode, int32_t iters, double* flops_per_launch, double* sink);

/* out[i, :] = X[idx[i], :]  (row gather, k columns; halo send packing) */
int gcg_gather_rows(void* ctx, int64_t nidx, const int32_t* idx, int64_t k, const double* X,
                    int64_t ldx, double* out, int64_t ldo);

/* Ritz-residual column sums (row-partitioned form of gcg_ritz_residuals):
 * sums[q*k + j], q = 0..3: ||AX - lam (X or BX)||^2, X.X, X.BX, BX.BX; then
 * gcg_ritz_finish turns (globally reduced) sums into the residuals. */
int gcg_ritz_sums(void* ctx, int64_t n, int64_t k, const double* AX, int64_t ldax,
                  const double* X, int64_t ldx, const double* BX, int64_t ldbx,
                  const double* lam, int mode, double* sums);
int gcg_ritz_finish(void* ctx, int64_t k, const double* sums, const double* lam, int mode,
                    double* out);

/* ---- small dense (device, row-major) -------------------------------------- */
/* full symmetric eigendecomposition: w ascending, V[:, j] its eigenvector with the
 * largest-|entry| made positive (dense.py:63-82).  A is read only.  m <= 64: one-CTA
 * Jacobi; 65..1024: csrc/eig.cu (Householder tridiagonalisation in one CTA, one
 * cluster or a co-resident grid; bisection; inverse iteration); cuSOLVER syevd above. */
int gcg_syev(void* ctx, int64_t m, const double* A, int64_t lda, double* w, double* V,
             int64_t ldv);
/* eigenpairs il..iu (1-based inclusive, dense.py:86-117 sym_eig_range): w gets
 * iu - il + 1 ascending values, V (m x (iu - il + 1), row-major) the sign-fixed
 * vectors.  csrc/eig.cu for 3 <= m <= 1024 (only the requested indices are bisected,
 * inverse-iterated and back-transformed), cuSOLVER syevdx otherwise. */
int gcg_syev_range(void* ctx, int64_t m, const double* A, int64_t lda, int64_t il, int64_t iu,
                   double* w, double* V, int64_t ldv);
/* C = alpha op(A) op(B) + beta C, op = transpose when t* != 0. */
int gcg_dgemm(void* ctx, int ta, int tb, int64_t M, int64_t N, int64_t K, double alpha,
              const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
              double* C, int64_t ldc);
/* A <- (A + A^T)/2 */
int gcg_symmetrize(void* ctx, int64_t m, double* A, int64_t lda);

/* Leaf SVQB step (orth.py:155-188) for a w x w Gram block G:
 *   status[0] = max|G - I|, status[1] = #eigenvalues <= dep_tol*max(lambda_max,0),
 *   status[2] = lambda_max; Q (w x (w - nbad)) = V[:, nbad:] / sqrt(lambda[nbad:]). */
int gcg_svqb_prepare(void* ctx, int64_t w, const double* G, int64_t ldg, double dep_tol,
                     double skip_tol, double* Q, int64_t ldq, double* status);
/* (skip_tol: when max|G - I| <= skip_tol the caller is done — orth.py:170-171 — and
 *  only status[0] is written; pass a negative value to always factorise) */
/* Deflation repeat test (orth.py:146-152): R is K x w coefficients, dnew[w] squared norms.
 *   status[0] = max|R|, status[1] = any(sum_r R[r,c]^2 > dgks * max(dnew[c], 1e-300)). */
int gcg_deflate_status(void* ctx, int64_t K, int64_t w, const double* R, int64_t ldr,
                       const double* dnew, int64_t dstride, double dgks, double* status);
/* out = #{ j : vals[j] <= rel * max(max(vals), 0) } written as a double. */
/* solver._build_p (solver.py:167-199) on one device: writes the momentum block's
 * coefficients (m x kept, row-major, ldp) into phat and kept into *kept_out (0 = no
 * momentum block).  coeffs is the m x d Ritz coefficient block (ldc); the group is
 * columns gs..gs+gw-1 with its first num_x_rows rows zeroed.  Two host reads. */
int gcg_build_p(void* ctx, int64_t m, int64_t d, const double* coeffs, int64_t ldc,
                int64_t num_x_rows, int64_t gs, int64_t gw, double dep_tol, double* phat,
                int64_t ldp, int64_t* kept_out);
int gcg_count_le(void* ctx, int64_t len, const double* vals, double rel, double* out);
/* out[:, j] = V[:, off + j] / sqrt(w[off + j]) for j < m - off. */
int gcg_scale_rsqrt(void* ctx, int64_t m, int64_t off, const double* V, int64_t ldv,
                    const double* w, double* out, int64_t ldo);

/* Structured projected matrix (solver.py:281-290): Abar (m x m, m = d + np + nw) =
 *   [diag(lam[0:d]) 0 cross[0:d]; 0 Pc cross[d:d+np]; cross^T] then (Abar + Abar^T)/2,
 * where cross is m x nw (row-major, ldc) and Pc is np x np (ldp). */
int gcg_abar_assemble(void* ctx, int64_t d, int64_t np, int64_t nw, const double* lam,
                      const double* Pc, int64_t ldp, const double* cross, int64_t ldc,
                      double* Abar, int64_t lda);
/* out[0] = max |A - B| over an m x n block (B == NULL: B = identity). */
int gcg_max_abs_diff(void* ctx, int64_t m, int64_t n, const double* A, int64_t lda,
                     const double* B, int64_t ldb, double* out);

/* Ritz residuals (solver.py:129-141): per column j,
 *   mode 0: ||AX - lam X|| / ||X||                        (reference, B = I)
 *   mode 1: ||AX - lam BX|| / (lam^+ sqrt(X'BX))          (reference, generalized)
 *   mode 2: ||AX - lam BX|| / (|lam| ||BX||)              (north-star criterion)
 * BX may equal X (B = I). */
int gcg_ritz_residuals(void* ctx, int64_t n, int64_t k, const double* AX, int64_t ldax,
                       const double* X, int64_t ldx, const double* BX, int64_t ldbx,
                       const double* lam, int mode, double* out);

/* ---- B-orthogonalisation, natively driven (one GPU) ------------------------
 * The reference's Alg. 3 control flow (orth.py:124-226, 339-372) run by the
 * library: every repeat / dependence decision is a pinned read of the fused
 * status record, every long-vector step a library kernel.  B = CSR (n x n,
 * rowptr/colidx int32 on device) or b_rowptr == NULL for B = I.  Outputs: the
 * kept column count (0 = all dependent), the reduction count, and the slots
 * refilled from the rear (first `cap` written, total in *nrep). */
typedef struct gcg_orth_opts {
  int64_t svd_leaf;        /* <= 0: min(width, 16) */
  double reorth_tol;       /* orth.py:59 */
  double dependence_tol;   /* orth.py:60 */
  int32_t max_passes;      /* orth.py:61 */
  int32_t pad_;
} gcg_orth_opts;
/* recursive_orth_svd on columns [lo, hi) of X (orth.py:207-226) */
int gcg_orth_recursive(void* ctx, int64_t n, double* X, int64_t ldx, int64_t lo, int64_t hi,
                       int64_t b_nnz, const int* b_rowptr, const int* b_colidx,
                       const double* b_val, const gcg_orth_opts* opts, int64_t* kept,
                       int64_t* reductions, int64_t* replaced, int64_t cap, int64_t* nrep);
/* orth_against: X[:, 0:w] against the B-orthonormal basis (n x K, ldb) (orth.py:339-372) */
int gcg_orth_against(void* ctx, int64_t n, double* X, int64_t ldx, int64_t w,
                     const double* basis, int64_t ldb, int64_t K, int64_t b_nnz,
                     const int* b_rowptr, const int* b_colidx, const double* b_val,
                     const gcg_orth_opts* opts, int64_t* kept, int64_t* reductions,
                     int64_t* replaced, int64_t cap, int64_t* nrep);

/* ---- BASELINE operators assembled on the device (problems.py generators) ----
 * Structured grid n0 x n1 x n2 (n2 fastest; n0 = 1 for 2-D), noff <= 27 offsets
 * (host int32 triples d0,d1,d2), Dirichlet truncation, rows in lexicographic
 * order, columns sorted.  Weights: w[t] constant per offset (host), or wrow[t]
 * a device array of n per-row values (host array of device pointers).  rowptr
 * (n + 1), colidx and val (nnz, from gcg_stencil_nnz) are caller-owned device
 * buffers.  Bit-identical to problems.stencil_csr. */
int gcg_stencil_nnz(int64_t n0, int64_t n1, int64_t n2, int32_t noff, const int32_t* offs,
                    int64_t* nnz);
int gcg_stencil_csr(void* ctx, int64_t n0, int64_t n1, int64_t n2, int32_t noff,
                    const int32_t* offs, const double* w, const double* const* wrow,
                    int32_t* rowptr, int32_t* colidx, double* val);
/* per-row weights of the var-coef 7-pt operator (problems.py varcoef_diffusion_3d)
 * from the N^3 cell field kc (device): out = [diag | -face(ax, s) for (ax, s) in
 * (0,-1),(0,+1),(1,-1),(1,+1),(2,-1),(2,+1)], 7 arrays of N^3. */
int gcg_varcoef7_weights(void* ctx, int64_t N, const double* kc, double* out);
/* One rank's z-slab of the same stencil for a row-partitioned run:
 * rows [row0, row1) with columns in the local layout of distributed.local_part —
 * owned rows 0..nloc-1, then the ghost plane below (global [row0 - nprev, row0)),
 * then the one above ([row1, row1 + nnext)); a plane is n1*n2 rows (n2 for n0 = 1).
 * Pass 1 (colidx == NULL): fills rowptr (nloc + 1) and *nnz_out = the slab's nnz.
 * Pass 2: fills colidx/val; *nnz_out = nprev + nnext (ghost rows); GCG_ERR_ARG if
 * the stencil reaches beyond one ghost plane.  wrow (per-row weights) are indexed by
 * GLOBAL row. */
int gcg_stencil_slab(void* ctx, int64_t n0, int64_t n1, int64_t n2, int32_t noff,
                     const int32_t* offs, const double* w, const double* const* wrow, int64_t row0,
                     int64_t row1, int32_t* rowptr, int32_t* colidx, double* val,
                     int64_t* nnz_out);
/* Device validation of a square CSR operator (operators.py:56-66, 79-87; rows sorted):
 * out[4] (host) = {max |a_ij|, max |a_ij - a_ji| (missing = 0), #non-finite values,
 * #column indices outside [0, n)}.  Synchronous. */
int gcg_csr_check(void* ctx, int64_t n, const int32_t* rowptr, const int32_t* colidx,
                  const double* val, double* out);
/* X[i, c] = N(0,1) from Philox4x32-10 keyed by seed at counter (row0 + i, c / 2)
 * (Box-Muller): a seeded block that every row partition draws identically. */
int gcg_fill_normal(void* ctx, int64_t n, int64_t k, int64_t row0, uint64_t seed, double* X,
                    int64_t ldx);

/* ---- MatrixMarket ingestion (host; io.py:108-216 read_matrix_market) ------
 * gcg_mm_open parses the whole file (coordinate entries tokenised by
 * `nthreads` host threads, 0 = all cores) into a handle; on a malformed file it
 * returns GCG_ERR_PARSE with info->err_line (1-based) and info->err_msg set,
 * GCG_ERR_UNSUPPORTED / GCG_ERR_IO likewise, and no handle.  gcg_mm_fetch
 * copies the parsed data into caller buffers: coordinate -> nentries (row,
 * col, value) triples, 0-based, symmetric storage already mirrored (duplicates
 * NOT yet summed); array -> the dense nrows x ncols matrix, column-major. */
typedef struct gcg_mm_info {
  int64_t nrows, ncols;
  int64_t nentries;   /* coordinate: triples after mirroring; array: nrows * ncols */
  int32_t format;     /* 0 coordinate, 1 array */
  int32_t symmetric;
  int32_t err_kind;   /* 0 none, 1 parse, 2 unsupported, 3 io */
  int32_t pad_;
  int64_t err_line;
  char err_msg[240];
} gcg_mm_info;
int gcg_mm_open(const char* path, int nthreads, void** handle, gcg_mm_info* info);
int gcg_mm_fetch(void* handle, int64_t* rows, int64_t* cols, double* vals);
/* COO -> CSR on the device (the assembly half of MatrixMarket ingestion): device
 * 0-based int64 rows / cols and f64 vals in any order, duplicates allowed ->
 * rowptr (n + 1), colidx / val (capacity nnz) with sorted columns and duplicates summed
 * in input order; *nnz_out = stored entries.  Synchronises the context stream. */
int gcg_coo_to_csr(void* ctx, int64_t n, int64_t ncols, int64_t nnz, const int64_t* rows,
                   const int64_t* cols, const double* vals, int32_t* rowptr, int32_t* colidx,
                   double* val, int64_t* nnz_out);
void gcg_mm_close(void* handle);

#ifdef __cplusplus
}
#endif

#endif /* GCGB200_H */
