// extern "C" boundary of libgcgb200.so (declared in include/gcgb200.h).
//
// No C++ exception crosses this boundary; every entry point returns an int
// status.  The device tier is asynchronous on the context stream; the
// reference-FFI tier (gcgeig_*) is synchronous, like the reference's own
// kernel-backend calls (_cy.pyx:11-65).

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <vector>

#include "common.cuh"

namespace gcg {

extern int64_t g_launches;
extern int64_t g_cusolver_calls;

int sell_size(Ctx* c, long long n, const int* rowptr, int sigma, long long* nslices,
              long long* nnz_padded);
int csr_to_sell(Ctx* c, long long n, const int* rowptr, const int* colidx, const double* val,
                int sigma, long long* sptr, int* perm, int* scol, double* sval);
int spmm_sell_launch(Ctx* c, long long n, long long nslices, const long long* sptr,
                     const int* perm, const int* scol, const double* sval, int k,
                     const double* X, long long ldx, double alpha, double gamma, const double* Z,
                     long long ldz, double beta, const double* Yin, long long ldyin, double* Y,
                     long long ldy, int dot_mode, const double* W, long long ldw, double* dots);
int spmm_launch_impl(Ctx* c, long long n, long long nnz, const int* rowptr, const int* colidx,
                     const double* val, int k, const double* X, long long ldx, double alpha,
                     double gamma, const double* Z, long long ldz, double beta, const double* Yin,
                     long long ldyin, double* Y, long long ldy, int dot_mode, const double* W,
                     long long ldw, double* dots, double* partials_ext, int* grid_out,
                     const int* skip);
int gram_launch(Ctx* c, long long n, int k1, int k2, const double* X, long long ldx,
                const double* Y, long long ldy, double alpha, double beta, double* G,
                long long grs, long long gcs);
int lincomb_launch(Ctx* c, long long n, int m, int d, double alpha, const double* X,
                   long long ldx, const double* C, long long ldc, double beta, double* Y,
                   long long ldy);
int axpby_launch(Ctx* c, long long n, int k, double alpha, const double* X, long long ldx,
                 double beta, double* Y, long long ldy);
int copy_launch(Ctx* c, long long n, int k, const double* X, long long ldx, double* Y,
                long long ldy);
int fill_launch(Ctx* c, long long n, int k, double v, double* Y, long long ldy);
int col_scale_copy_launch(Ctx* c, long long n, int k, const double* s, const double* X,
                          long long ldx, double* Y, long long ldy);
int col_scale_launch(Ctx* c, long long n, int k, const double* s, double* X, long long ldx);
int col_dots_launch(Ctx* c, long long n, int k, const double* X, long long ldx, const double* Y,
                    long long ldy, double* out);
int dgemm_launch(Ctx* c, int ta, int tb, int M, int N, int K, double alpha, const double* A,
                 long long lda, const double* B, long long ldb, double beta, double* C,
                 long long ldc);
int symmetrize_launch(Ctx* c, int m, double* A, long long lda);
int block_cg_launch(Ctx* c, long long n, long long nnz, const int* rowptr, const int* colidx,
                    const double* val, double shift, int k, const double* rhs, long long ldr,
                    const double* x0, long long ldx0, double* x, long long ldx, int max_iters,
                    double rel_tol, int* d_sweeps, int8_t* d_conv, int8_t* d_frozen,
                    double* d_relres, const gcg_cg_dist* dist);
int gather_rows_launch(Ctx* c, int nidx, const int* idx, int k, const double* X, long long ldx,
                       double* out, long long ldo);
int fp64_peak_launch(Ctx* c, int mode, int iters, double* sink, int* grid_out, int* block_out);
int ritz_sums_launch(Ctx* c, long long n, int k, const double* AX, long long ldax,
                     const double* X, long long ldx, const double* BX, long long ldbx,
                     const double* lam, int mode, double* sums);
int ritz_finish_launch(Ctx* c, int k, const double* sums, const double* lam, int mode,
                       double* out);
int svqb_prepare_launch(Ctx* c, int m, const double* G, long long ldg, double dep_tol,
                        double skip_tol, double* Q,
                        long long ldq, double* status);
int deflate_status_launch(Ctx* c, int K, int w, const double* R, long long ldr,
                          const double* dnew, long long dstride, double dgks, double* status);
int abar_assemble_launch(Ctx* c, int d, int np, int nw, const double* lam, const double* Pc,
                         long long ldp, const double* cross, long long ldc, double* Abar,
                         long long lda);
int max_abs_diff_launch(Ctx* c, int m, int n, const double* A, long long lda, const double* B,
                        long long ldb, double* out);
int count_le_launch(Ctx* c, int len, const double* vals, double rel, double* out);
int scale_rsqrt_launch(Ctx* c, int m, int off, const double* V, long long ldv, const double* w,
                       double* out, long long ldo);
int ritz_residuals_launch(Ctx* c, long long n, int k, const double* AX, long long ldax,
                          const double* X, long long ldx, const double* BX, long long ldbx,
                          const double* lam, int mode, double* out);

// GCG_PDL=0 turns programmatic dependent launch off (A/B switch)
// Programmatic dependent launch: off by default since the CG sweep became two kernels —
// at cfg4 (n = 2.1 M, k = 100: many waves) the early-launched dependent CTAs occupy SM
// slots while they wait, 5.08 -> 4.05 ms per sweep without PDL; cfg2 within noise
// (bench 0.2751 vs 0.2742 s).  GCG_PDL=1 re-enables it.
int ensure_mapped(Ctx* c) {
  if (c->mapped) return GCG_OK;
  if (cudaHostAlloc((void**)&c->mapped, 64 * sizeof(double), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&c->mapped_dev, c->mapped, 0) != cudaSuccess) {
    cudaGetLastError();
    if (c->mapped) cudaFreeHost(c->mapped);
    c->mapped = c->mapped_dev = nullptr;
    return GCG_ERR_ALLOC;
  }
  return GCG_OK;
}

// (Turning it on only for small CG blocks, n k <= 8 M, measured no better at cfg2:
// bench 0.268-0.270 vs 0.267 s.)
bool pdl_enabled() {
  // on by default since the CG kernels trigger late (at the end of their row loops): the
  // successor's CTAs are scheduled while the grid drains instead of competing with it —
  // cfg2 93.1 -> 89.2 us per sweep pair, cfg4 unchanged (an early trigger cost 40 % there)
  static const bool on = !(getenv("GCG_PDL") && getenv("GCG_PDL")[0] == '0');
  return on;
}

void kernel_smem(const void* kern, size_t bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, size_t>> done;
  std::lock_guard<std::mutex> lk(mu);
  for (auto& e : done) {
    if (e.first != kern) continue;
    if (e.second >= bytes) return;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    e.second = bytes;
    return;
  }
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  done.emplace_back(kern, bytes);
}

int kernel_occupancy(const void* kern, int threads, size_t smem) {
  static std::mutex mu;
  struct Key {
    const void* k;
    int t;
    size_t s;
    int occ;
  };
  static std::vector<Key> cache;
  std::lock_guard<std::mutex> lk(mu);
  for (const auto& e : cache)
    if (e.k == kern && e.t == threads && e.s == smem) return e.occ;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
  if (occ < 1) occ = 1;
  cache.push_back({kern, threads, smem, occ});
  return occ;
}

int ensure(Scratch& s, size_t bytes) {
  if (bytes <= s.bytes) return GCG_OK;
  // the scratch may still be in use by queued work on any stream of this ctx
  cudaDeviceSynchronize();
  if (s.ptr) cudaFree(s.ptr);
  s.ptr = nullptr;
  s.bytes = 0;
  size_t want = bytes + bytes / 4 + 4096;
  if (cudaMalloc(&s.ptr, want) != cudaSuccess) {
    cudaGetLastError();
    return GCG_ERR_ALLOC;
  }
  s.bytes = want;
  return GCG_OK;
}

int prof_start(Ctx* c, int cls, double bytes) {
  Prof& p = c->prof;
  if (!p.on) return -1;
  if (p.stride > 1 && (p.seen[cls]++ % p.stride) != 0) return -1;
  if (p.used == p.cap) {
    // grow: only between profiled regions is the device flag array reallocated safely,
    // so allocate generously up front and stop recording when full
    return -1;
  }
  const int slot = p.used++;
  p.cls[slot] = cls;
  p.bytes[slot] = bytes;
  cudaEventRecord(p.ev[2 * slot], c->stream);
  return slot;
}

int* prof_skip_slot(Ctx* c, int slot) {
  return slot < 0 ? nullptr : c->prof.d_skipped + slot;
}

static int prof_reserve(Prof& p, int cap) {
  if (p.cap >= cap) return GCG_OK;
  cudaEvent_t* ev = (cudaEvent_t*)realloc(p.ev, sizeof(cudaEvent_t) * 2 * cap);
  int* cl = (int*)realloc(p.cls, sizeof(int) * cap);
  double* by = (double*)realloc(p.bytes, sizeof(double) * cap);
  if (!ev || !cl || !by) return GCG_ERR_ALLOC;
  for (int i = 2 * p.cap; i < 2 * cap; ++i) cudaEventCreate(&ev[i]);
  p.ev = ev;
  p.cls = cl;
  p.bytes = by;
  if (p.d_skipped) cudaFree(p.d_skipped);
  if (cudaMalloc(&p.d_skipped, sizeof(int) * cap) != cudaSuccess) return GCG_ERR_ALLOC;
  p.cap = cap;
  return GCG_OK;
}

void prof_stop(Ctx* c, int slot) {
  if (slot < 0) return;
  cudaEventRecord(c->prof.ev[2 * slot + 1], c->stream);
}

static void release(Scratch& s) {
  if (s.ptr) cudaFree(s.ptr);
  s.ptr = nullptr;
  s.bytes = 0;
}

// --- transposes used by the column-major reference-FFI tier ----------------
// out_rm[i*k + c] = in_cm[i + c*ld]
__global__ void cm_to_rm_kernel(long long n, int k, const double* in, long long ld, double* out) {
  const long long tot = n * k;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / k;
    const int c = (int)(e % k);
    out[e] = in[i + (long long)c * ld];
  }
}
// out_cm[i + c*n] = in_rm[i*k + c]
__global__ void rm_to_cm_kernel(long long n, int k, const double* in, double* out) {
  const long long tot = n * k;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e / n);
    const long long i = e % n;
    out[e] = in[i * k + c];
  }
}
__global__ void i64_to_i32_kernel(long long n, const long long* in, int* out) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = (int)in[e];
}

}  // namespace gcg

using namespace gcg;

#define CTX(p) reinterpret_cast<gcg::Ctx*>(p)

extern "C" {

int gcg_abi_version(void) { return GCG_ABI_VERSION; }

const char* gcg_status_string(int status) {
  switch (status) {
    case GCG_OK: return "ok";
    case GCG_ERR_ARG: return "invalid argument";
    case GCG_ERR_CUDA: return "CUDA error";
    case GCG_ERR_SOLVER: return "dense eigensolver failure";
    case GCG_ERR_ALLOC: return "device allocation failed";
    case GCG_ERR_NODEV: return "no CUDA device";
    case GCG_ERR_IO: return "file could not be read";
    case GCG_ERR_PARSE: return "malformed input file";
    case GCG_ERR_UNSUPPORTED: return "unsupported input";
    default: return "unknown status";
  }
}

int64_t gcg_launch_count(void) { return g_launches; }
int64_t gcg_cusolver_calls(void) { return g_cusolver_calls; }

int gcg_ctx_create(void** out, void* stream) {
  if (!out) return GCG_ERR_ARG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return GCG_ERR_NODEV;
  }
  Ctx* c = new (std::nothrow) Ctx();
  if (!c) return GCG_ERR_ALLOC;
  c->stream = (cudaStream_t)stream;
  cudaGetDevice(&c->device);
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device) == cudaSuccess &&
      sms > 0)
    c->num_sms = sms;
  int l2 = 0;
  if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, c->device) == cudaSuccess) c->l2_bytes = l2;
  if (cusolverDnCreate(&c->solver) != CUSOLVER_STATUS_SUCCESS) {
    delete c;
    return GCG_ERR_SOLVER;
  }
  cusolverDnSetStream(c->solver, c->stream);
  *out = c;
  return GCG_OK;
}

int gcg_ctx_destroy(void* p) {
  Ctx* c = CTX(p);
  if (!c) return GCG_OK;
  cudaStreamSynchronize(c->stream);
  release(c->partials);
  release(c->eigwork);
  release(c->cg);
  release(c->cgpad);
  release(c->host_tmp);
  release(c->host_tmp2);
  release(c->host_tmp3);
  release(c->host_tmp4);
  release(c->dense);
  release(c->orth);
  release(c->buildp);
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->mapped) cudaFreeHost(c->mapped);
  if (c->spec) cudaFree(c->spec);
  for (cudaEvent_t e : c->spec_ev)
    if (e) cudaEventDestroy(e);
  if (c->solver) cusolverDnDestroy(c->solver);
  delete c;
  return GCG_OK;
}

int gcg_ctx_set_stream(void* p, void* stream) {
  Ctx* c = CTX(p);
  if (!c) return GCG_ERR_ARG;
  c->stream = (cudaStream_t)stream;
  cusolverDnSetStream(c->solver, c->stream);
  return GCG_OK;
}

int gcg_ctx_sync(void* p) {
  Ctx* c = CTX(p);
  if (!c) return GCG_ERR_ARG;
  return cuda_status(cudaStreamSynchronize(c->stream));
}

int gcg_prof_begin(void* p) {
  Ctx* c = CTX(p);
  if (!c) return GCG_ERR_ARG;
  cudaStreamSynchronize(c->stream);
  GCG_TRY(prof_reserve(c->prof, 1 << 18));
  GCG_TRY(cuda_status(cudaMemsetAsync(c->prof.d_skipped, 0, sizeof(int) * c->prof.cap,
                                      c->stream)));
  c->prof.on = true;
  c->prof.used = 0;
  for (long long& v : c->prof.seen) v = 0;
  return GCG_OK;
}

int gcg_prof_sample(void* p, int stride) {
  Ctx* c = CTX(p);
  if (!c || stride < 1) return GCG_ERR_ARG;
  c->prof.stride = stride;
  return GCG_OK;
}

int gcg_prof_end(void* p, double* out) {
  Ctx* c = CTX(p);
  if (!c || !out) return GCG_ERR_ARG;
  Prof& pr = c->prof;
  pr.on = false;
  GCG_TRY(cuda_status(cudaStreamSynchronize(c->stream)));
  double ms[PROF_NCLASS] = {0}, by[PROF_NCLASS] = {0}, nl[PROF_NCLASS] = {0};
  std::vector<int> skipped(pr.used > 0 ? pr.used : 1, 0);
  if (pr.used > 0)
    GCG_TRY(cuda_status(cudaMemcpy(skipped.data(), pr.d_skipped, sizeof(int) * pr.used,
                                   cudaMemcpyDeviceToHost)));
  for (int s = 0; s < pr.used; ++s) {
    if (skipped[s]) continue;  // CG early-exit no-op: no work, no bytes
    float t = 0.f;
    if (cudaEventElapsedTime(&t, pr.ev[2 * s], pr.ev[2 * s + 1]) == cudaSuccess) {
      ms[pr.cls[s]] += t;
      by[pr.cls[s]] += pr.bytes[s];
      nl[pr.cls[s]] += 1.0;
    }
  }
  cudaGetLastError();
  for (int i = 0; i < PROF_NCLASS; ++i) {
    out[3 * i + 0] = ms[i];
    out[3 * i + 1] = nl[i];
    out[3 * i + 2] = by[i];
  }
  return GCG_OK;
}

// ---- device tier ------------------------------------------------------------

int gcg_spmm_csr(void* p, int64_t n, int64_t nnz, const int32_t* rowptr, const int32_t* colidx,
                 const double* val, int64_t k, const double* X, int64_t ldx, double alpha,
                 double gamma, const double* Z, int64_t ldz, double beta, const double* Yin,
                 int64_t ldyin, double* Y, int64_t ldy, int dot_mode, const double* W,
                 int64_t ldw, double* dots) {
  Ctx* c = CTX(p);
  if (!c || n < 0 || k < 0 || (n > 0 && (!rowptr || !X || !Y))) return GCG_ERR_ARG;
  if (ldx < k || ldy < k) return GCG_ERR_ARG;
  if (gamma != 0.0 && !Z) return GCG_ERR_ARG;
  if (beta != 0.0 && !Yin) return GCG_ERR_ARG;
  if (dot_mode < 0 || dot_mode > 2 || (dot_mode && !dots) || (dot_mode == 1 && !W))
    return GCG_ERR_ARG;
  return spmm_launch_impl(c, n, nnz, rowptr, colidx, val, (int)k, X, ldx, alpha, gamma, Z, ldz, beta,
                          Yin, ldyin, Y, ldy, dot_mode, W, ldw, dots, nullptr, nullptr, nullptr);
}

int gcg_sell_size(void* p, int64_t n, const int32_t* rowptr, int32_t sigma, int64_t* nslices,
                  int64_t* nnz_padded) {
  Ctx* c = CTX(p);
  if (!c || n <= 0 || !rowptr || !nslices || !nnz_padded) return GCG_ERR_ARG;
  long long ns = 0, nz = 0;
  const int st = sell_size(c, n, rowptr, sigma, &ns, &nz);
  *nslices = ns;
  *nnz_padded = nz;
  return st;
}

int gcg_csr_to_sell(void* p, int64_t n, const int32_t* rowptr, const int32_t* colidx,
                    const double* val, int32_t sigma, int64_t* slice_ptr, int32_t* perm,
                    int32_t* sell_col, double* sell_val) {
  Ctx* c = CTX(p);
  if (!c) return GCG_ERR_ARG;
  return csr_to_sell(c, n, rowptr, colidx, val, sigma, (long long*)slice_ptr, perm, sell_col,
                     sell_val);
}

int gcg_spmm_sell(void* p, int64_t n, int64_t nslices, const int64_t* slice_ptr,
                  const int32_t* perm, const int32_t* sell_col, const double* sell_val, int64_t k,
                  const double* X, int64_t ldx, double alpha, double gamma, const double* Z,
                  int64_t ldz, double beta, const double* Yin, int64_t ldyin, double* Y,
                  int64_t ldy, int dot_mode, const double* W, int64_t ldw, double* dots) {
  Ctx* c = CTX(p);
  if (!c || n < 0 || k < 0 || nslices < 0 || (n > 0 && (!slice_ptr || !perm || !sell_col ||
                                                        !sell_val || !X || !Y)))
    return GCG_ERR_ARG;
  if (ldx < k || ldy < k || (gamma != 0.0 && !Z) || (beta != 0.0 && !Yin)) return GCG_ERR_ARG;
  if (dot_mode < 0 || dot_mode > 2 || (dot_mode && !dots) || (dot_mode == 1 && !W))
    return GCG_ERR_ARG;
  return spmm_sell_launch(c, n, nslices, (const long long*)slice_ptr, perm, sell_col, sell_val,
                          (int)k, X, ldx, alpha, gamma, Z, ldz, beta, Yin, ldyin, Y, ldy,
                          dot_mode, W, ldw, dots);
}

int gcg_gram(void* p, int64_t n, int64_t k1, int64_t k2, const double* X, int64_t ldx,
             const double* Y, int64_t ldy, double alpha, double beta, double* G, int64_t g_rs,
             int64_t g_cs, const double* T, int64_t ldt, double* dots) {
  Ctx* c = CTX(p);
  if (!c || n < 0 || k1 < 0 || k2 < 0 || ldx < k1 || ldy < k2) return GCG_ERR_ARG;
  if (k1 > 0 && k2 > 0 && !G) return GCG_ERR_ARG;
  if (n == 0) {
    // empty contraction: G = beta * G
    if (k1 > 0 && k2 > 0) {
      if (g_cs == 1) GCG_TRY(axpby_launch(c, k1, (int)k2, 0.0, G, g_rs, beta, G, g_rs));
      else GCG_TRY(axpby_launch(c, k2, (int)k1, 0.0, G, g_cs, beta, G, g_cs));
    }
    if (dots) GCG_TRY(fill_launch(c, 1, (int)k2, 0.0, dots, k2));
    return GCG_OK;
  }
  GCG_TRY(gram_launch(c, n, (int)k1, (int)k2, X, ldx, Y, ldy, alpha, beta, G, g_rs, g_cs));
  if (dots) GCG_TRY(col_dots_launch(c, n, (int)k2, T ? T : Y, T ? ldt : ldy, Y, ldy, dots));
  return GCG_OK;
}

int gcg_lincomb(void* p, int64_t n, int64_t m, int64_t d, double alpha, const double* X,
                int64_t ldx, const double* C, int64_t ldc, double beta, double* Y, int64_t ldy) {
  Ctx* c = CTX(p);
  if (!c || n < 0 || m < 0 || d < 0 || ldx < m || ldc < d || ldy < d) return GCG_ERR_ARG;
  if (m == 0) {
    if (beta == 0.0) return fill_launch(c, n, (int)d, 0.0, Y, ldy);
    return axpby_launch(c, n, (int)d, 0.0, Y, ldy, beta, Y, ldy);
  }
  return lincomb_launch(c, n, (int)m, (int)d, alpha, X, ldx, C, ldc, beta, Y, ldy);
}

int gcg_axpby(void* p, int64_t n, int64_t k, double alpha, const double* X, int64_t ldx,
              double beta, double* Y, int64_t ldy) {
  Ctx* c = CTX(p);
  if (!c || n < 0 || k < 0 || ldy < k || (alpha != 0.0 && ldx < k)) return GCG_ERR_ARG;
  return axpby_launch(c, n, (int)k, alpha, X, ldx, beta, Y, ldy);
}

int gcg_copy(void* p, int64_t n, int64_t k, const double* X, int64_t ldx, double* Y,
             int64_t ldy) {
  Ctx* c = CTX(p);
  if (!c || n < 0 || k < 0 || ldx < k || ldy < k) return GCG_ERR_ARG;
  return copy_launch(c, n, (int)k, X, ldx, Y, ldy);
}

int gcg_col_scale(void* p, int64_t n, int64_t k, const double* s, double* X, int64_t ldx) {
  Ctx* c = CTX(p);
  if (!c || n < 0 || k < 0 || ldx < k) return GCG_ERR_ARG;
  return col_scale_launch(c, n, (int)k, s, X, ldx);
}

int gcg_col_dots(void* p, int64_t n, int64_t k, const double* X, int64_t ldx, const double* Y,
                 int64_t ldy, double* out) {
  Ctx* c = CTX(p);
  if (!c || n < 0 || k < 0 || ldx < k || ldy < k) return GCG_ERR_ARG;
  return col_dots_launch(c, n, (int)k, X, ldx, Y, ldy, out);
}

int gcg_fill(void* p, int64_t n, int64_t k, double value, double* X, int64_t ldx) {
  Ctx* c = CTX(p);
  if (!c || n < 0 || k < 0 || ldx < k) return GCG_ERR_ARG;
  return fill_launch(c, n, (int)k, value, X, ldx);
}

int gcg_block_cg(void* p, int64_t n, int64_t nnz, const int32_t* rowptr, const int32_t* colidx,
                 const double* val, double diag_shift, int64_t k, const double* rhs,
                 int64_t ldr, double* x, int64_t ldx, int32_t max_iters, double rel_tol,
                 int32_t* d_sweeps, int8_t* d_converged, int8_t* d_frozen, double* d_relres) {
  Ctx* c = CTX(p);
  if (!c || n <= 0 || k <= 0 || ldr < k || ldx < k || max_iters < 0)
    return GCG_ERR_ARG;
  if (!d_sweeps || !d_converged || !d_frozen || !d_relres) return GCG_ERR_ARG;
  return block_cg_launch(c, n, nnz, rowptr, colidx, val, diag_shift, (int)k, rhs, ldr, nullptr, 0,
                         x, ldx, max_iters, rel_tol, d_sweeps, d_converged, d_frozen, d_relres,
                         nullptr);
}

int gcg_block_cg_x0(void* p, int64_t n, int64_t nnz, const int32_t* rowptr,
                    const int32_t* colidx, const double* val, double diag_shift, int64_t k,
                    const double* rhs, int64_t ldr, const double* x0, int64_t ldx0, double* x,
                    int64_t ldx, int32_t max_iters, double rel_tol, int32_t* d_sweeps,
                    int8_t* d_converged, int8_t* d_frozen, double* d_relres) {
  Ctx* c = CTX(p);
  if (!c || n <= 0 || k <= 0 || ldr < k || ldx < k || ldx0 < k || !x0 ||
      max_iters < 0)
    return GCG_ERR_ARG;
  if (!d_sweeps || !d_converged || !d_frozen || !d_relres) return GCG_ERR_ARG;
  return block_cg_launch(c, n, nnz, rowptr, colidx, val, diag_shift, (int)k, rhs, ldr, x0, ldx0,
                         x, ldx, max_iters, rel_tol, d_sweeps, d_converged, d_frozen, d_relres,
                         nullptr);
}

int gcg_col_scale_copy(void* p, int64_t n, int64_t k, const double* s, const double* X,
                       int64_t ldx, double* Y, int64_t ldy) {
  Ctx* c = CTX(p);
  if (!c || n < 0 || k < 0 || ldx < k || ldy < k || (n > 0 && k > 0 && (!s || !X || !Y)))
    return GCG_ERR_ARG;
  return col_scale_copy_launch(c, n, (int)k, s, X, ldx, Y, ldy);
}

int gcg_block_cg_dist(void* p, int64_t n, int64_t nnz, const int32_t* rowptr,
                      const int32_t* colidx, const double* val, double diag_shift, int64_t k,
                      const double* rhs, int64_t ldr, double* x, int64_t ldx, int32_t max_iters,
                      double rel_tol, int32_t* d_sweeps, int8_t* d_converged, int8_t* d_frozen,
                      double* d_relres, const gcg_cg_dist* dist) {
  Ctx* c = CTX(p);
  if (!c || n <= 0 || k <= 0 || ldr < k || ldx < k || max_iters < 0 || !dist ||
      (!dist->callback && !dist->nccl_comm) || !dist->red_buf)
    return GCG_ERR_ARG;
  if (dist->nccl_comm && dist->npeer > 0 &&
      (!dist->peer_rank || !dist->peer_send_off || !dist->peer_recv_off))
    return GCG_ERR_ARG;
  if (!d_sweeps || !d_converged || !d_frozen || !d_relres) return GCG_ERR_ARG;
  return block_cg_launch(c, n, nnz, rowptr, colidx, val, diag_shift, (int)k, rhs, ldr, nullptr, 0, x, ldx,
                         max_iters, rel_tol, d_sweeps, d_converged, d_frozen, d_relres, dist);
}

int gcg_fp64_peak(void* p, int mode, int32_t iters, double* flops_per_launch, double* sink) {
  Ctx* c = CTX(p);
  if (!c || (mode != 0 && mode != 1) || iters <= 0 || !flops_per_launch || !sink)
    return GCG_ERR_ARG;
  int grid = 0, block = 0;
  GCG_TRY(fp64_peak_launch(c, mode, iters, sink, &grid, &block));
  const double warps = (double)grid * block / 32.0;
  *flops_per_launch = mode == 1 ? warps * iters * 8.0 * 512.0          // 8x8x4 x 2 flop
                                : (double)grid * block * iters * 8.0 * 4.0;  // 2 fma x 2 flop
  return GCG_OK;
}

int gcg_gather_rows(void* p, int64_t nidx, const int32_t* idx, int64_t k, const double* X,
                    int64_t ldx, double* out, int64_t ldo) {
  Ctx* c = CTX(p);
  if (!c || nidx < 0 || k < 0 || ldx < k || ldo < k) return GCG_ERR_ARG;
  return gather_rows_launch(c, (int)nidx, idx, (int)k, X, ldx, out, ldo);
}

int gcg_ritz_sums(void* p, int64_t n, int64_t k, const double* AX, int64_t ldax,
                  const double* X, int64_t ldx, const double* BX, int64_t ldbx,
                  const double* lam, int mode, double* sums) {
  Ctx* c = CTX(p);
  if (!c || n < 0 || k < 0 || k > 256 || mode < 0 || mode > 2) return GCG_ERR_ARG;
  return ritz_sums_launch(c, n, (int)k, AX, ldax, X, ldx, BX, ldbx, lam, mode, sums);
}

int gcg_ritz_finish(void* p, int64_t k, const double* sums, const double* lam, int mode,
                    double* out) {
  Ctx* c = CTX(p);
  if (!c || k < 0 || mode < 0 || mode > 2) return GCG_ERR_ARG;
  return ritz_finish_launch(c, (int)k, sums, lam, mode, out);
}

int gcg_syev(void* p, int64_t m, const double* A, int64_t lda, double* w, double* V,
             int64_t ldv) {
  Ctx* c = CTX(p);
  if (!c || m <= 0 || lda < m || ldv < m) return GCG_ERR_ARG;
  static const char* impl = getenv("GCG_SYEV");
  const bool tri_small = impl && impl[0] == 't';  // GCG_SYEV=tri: tridiagonal path for m <= 64 too
  if (m <= 64 && !tri_small) return dense_syev_jacobi(c, (int)m, A, lda, w, V, ldv);
  return dense_syev_cusolver(c, (int)m, A, lda, w, V, ldv);
}

int gcg_syev_range(void* p, int64_t m, const double* A, int64_t lda, int64_t il, int64_t iu,
                   double* w, double* V, int64_t ldv) {
  Ctx* c = CTX(p);
  const int64_t k = iu - il + 1;
  if (!c || m <= 0 || lda < m || il < 1 || iu < il || iu > m || ldv < k) return GCG_ERR_ARG;
  return dense_syev_range(c, (int)m, A, lda, (int)il, (int)iu, w, V, ldv);
}

int gcg_dgemm(void* p, int ta, int tb, int64_t M, int64_t N, int64_t K, double alpha,
              const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
              double* C, int64_t ldc) {
  Ctx* c = CTX(p);
  if (!c || M < 0 || N < 0 || K < 0 || ldc < N) return GCG_ERR_ARG;
  return dgemm_launch(c, ta, tb, (int)M, (int)N, (int)K, alpha, A, lda, B, ldb, beta, C, ldc);
}

int gcg_symmetrize(void* p, int64_t m, double* A, int64_t lda) {
  Ctx* c = CTX(p);
  if (!c || m < 0 || lda < m) return GCG_ERR_ARG;
  return symmetrize_launch(c, (int)m, A, lda);
}

int gcg_svqb_prepare(void* p, int64_t w, const double* G, int64_t ldg, double dep_tol,
                     double skip_tol, double* Q, int64_t ldq, double* status) {
  Ctx* c = CTX(p);
  if (!c || w <= 0 || ldg < w || ldq < w || !status) return GCG_ERR_ARG;
  return svqb_prepare_launch(c, (int)w, G, ldg, dep_tol, skip_tol, Q, ldq, status);
}

int gcg_deflate_status(void* p, int64_t K, int64_t w, const double* R, int64_t ldr,
                       const double* dnew, int64_t dstride, double dgks, double* status) {
  Ctx* c = CTX(p);
  if (!c || K < 0 || w < 0 || ldr < w || !status) return GCG_ERR_ARG;
  return deflate_status_launch(c, (int)K, (int)w, R, ldr, dnew, dstride, dgks, status);
}

int gcg_abar_assemble(void* p, int64_t d, int64_t np, int64_t nw, const double* lam,
                      const double* Pc, int64_t ldp, const double* cross, int64_t ldc,
                      double* Abar, int64_t lda) {
  Ctx* c = CTX(p);
  const int64_t m = d + np + nw;
  if (!c || d < 0 || np < 0 || nw < 0 || lda < m || (nw > 0 && ldc < nw) || (np > 0 && ldp < np))
    return GCG_ERR_ARG;
  return abar_assemble_launch(c, (int)d, (int)np, (int)nw, lam, Pc, ldp, cross, ldc, Abar, lda);
}

int gcg_max_abs_diff(void* p, int64_t m, int64_t n, const double* A, int64_t lda,
                     const double* B, int64_t ldb, double* out) {
  Ctx* c = CTX(p);
  if (!c || m < 0 || n < 0 || lda < n || (B && ldb < n) || !out) return GCG_ERR_ARG;
  return max_abs_diff_launch(c, (int)m, (int)n, A, lda, B, ldb, out);
}

// ---- native momentum block -------------------------------------------------

static int syev_dispatch(Ctx* c, int m, const double* A, long long lda, double* w, double* V,
                         long long ldv) {
  static const char* impl = getenv("GCG_SYEV");
  const bool tri_small = impl && impl[0] == 't';
  if (m <= 64 && !tri_small) return dense_syev_jacobi(c, m, A, lda, w, V, ldv);
  return dense_syev_cusolver(c, m, A, lda, w, V, ldv);
}


static int read_pinned(Ctx* c, const double* dev, int count) {
  if (!c->pinned) {
    if (cudaHostAlloc((void**)&c->pinned, 64 * sizeof(double), cudaHostAllocDefault) !=
        cudaSuccess) {
      cudaGetLastError();
      return GCG_ERR_ALLOC;
    }
  }
  GCG_TRY(cuda_status(cudaMemcpyAsync(c->pinned, dev, sizeof(double) * count,
                                      cudaMemcpyDeviceToHost, c->stream)));
  return cuda_status(cudaStreamSynchronize(c->stream));
}

// solver._orthonormalize_small (solver.py:167-199 helper): g = pt'pt, eigh, drop
// eigenvalues <= rel * max, q = pt V / sqrt(w) over the kept ones; one host read.
static int orth_small(Ctx* c, int m, int gw, const double* pt, long long ldpt, double rel,
                      double* q, long long ldq, int* kept, double* g, double* V, double* w,
                      double* scaled, double* status) {
  GCG_TRY(dgemm_launch(c, 1, 0, gw, gw, m, 1.0, pt, ldpt, pt, ldpt, 0.0, g, gw));
  GCG_TRY(symmetrize_launch(c, gw, g, gw));
  GCG_TRY(syev_dispatch(c, gw, g, gw, w, V, gw));
  GCG_TRY(ensure_mapped(c));
  (void)status;
  GCG_TRY(count_le_launch(c, gw, w, rel, c->mapped_dev));
  GCG_TRY(cuda_status(cudaStreamSynchronize(c->stream)));
  const int bad = (int)c->mapped[0];
  *kept = 0;
  if (bad >= gw) return GCG_OK;
  const int k = gw - bad;
  GCG_TRY(scale_rsqrt_launch(c, gw, bad, V, gw, w, scaled, k));
  GCG_TRY(dgemm_launch(c, 0, 0, m, k, gw, 1.0, pt, ldpt, scaled, k, 0.0, q, ldq));
  *kept = k;
  return GCG_OK;
}

// solver._build_p (solver.py:167-199) for one device: the momentum block's Ritz
// coefficients, projected against the new X coefficients (twice), orthonormalised
// (dropping dependent directions, dep_tol), projected once more and
// re-orthonormalised (1e-4).  Same operations and decisions as the Python
// driver's build_p, two pinned host reads instead of two Python round trips.
int gcg_build_p(void* p, int64_t m, int64_t d, const double* coeffs, int64_t ldc,
                int64_t num_x_rows, int64_t gs, int64_t gw, double dep_tol, double* phat,
                int64_t ldp, int64_t* kept_out) {
  Ctx* c = CTX(p);
  if (!c || !kept_out) return GCG_ERR_ARG;
  *kept_out = 0;
  if (gw <= 0 || m <= num_x_rows) return GCG_OK;
  if (m <= 0 || d <= 0 || gs < 0 || gs + gw > d || ldc < d || !coeffs || !phat || ldp < gw ||
      num_x_rows < 0 || gw > 1024)
    return GCG_ERR_ARG;
  const size_t sz_pt = (size_t)m * gw, sz_tmp = (size_t)d * gw, sz_g = (size_t)gw * gw;
  GCG_TRY(ensure(c->buildp, sizeof(double) * (2 * sz_pt + sz_tmp + 3 * sz_g + gw + 8) + 256));
  double* pt = (double*)c->buildp.ptr;
  double* q = pt + sz_pt;
  double* tmp = q + sz_pt;
  double* g = tmp + sz_tmp;
  double* V = g + sz_g;
  double* scaled = V + sz_g;
  double* w = scaled + sz_g;
  double* status = w + gw;
  const int M = (int)m, D = (int)d, GW = (int)gw;
  GCG_TRY(copy_launch(c, m, GW, coeffs + gs, ldc, pt, GW));
  if (num_x_rows > 0) GCG_TRY(fill_launch(c, num_x_rows, GW, 0.0, pt, GW));
  for (int rep = 0; rep < 2; ++rep) {
    GCG_TRY(dgemm_launch(c, 1, 0, D, GW, M, 1.0, coeffs, ldc, pt, GW, 0.0, tmp, GW));
    GCG_TRY(dgemm_launch(c, 0, 0, M, GW, D, -1.0, coeffs, ldc, tmp, GW, 1.0, pt, GW));
  }
  int kept = 0;
  GCG_TRY(orth_small(c, M, GW, pt, GW, dep_tol, q, GW, &kept, g, V, w, scaled, status));
  if (kept == 0) return GCG_OK;
  GCG_TRY(dgemm_launch(c, 1, 0, D, kept, M, 1.0, coeffs, ldc, q, GW, 0.0, tmp, kept));
  GCG_TRY(dgemm_launch(c, 0, 0, M, kept, D, -1.0, coeffs, ldc, tmp, kept, 1.0, q, GW));
  int kept2 = 0;
  GCG_TRY(orth_small(c, M, kept, q, GW, 1e-4, phat, ldp, &kept2, g, V, w, scaled, status));
  *kept_out = kept2;
  return GCG_OK;
}

int gcg_count_le(void* p, int64_t len, const double* vals, double rel, double* out) {
  Ctx* c = CTX(p);
  if (!c || len < 0 || !out) return GCG_ERR_ARG;
  return count_le_launch(c, (int)len, vals, rel, out);
}

int gcg_scale_rsqrt(void* p, int64_t m, int64_t off, const double* V, int64_t ldv,
                    const double* w, double* out, int64_t ldo) {
  Ctx* c = CTX(p);
  if (!c || m < 0 || off < 0 || off > m || ldv < m || ldo < m - off) return GCG_ERR_ARG;
  return scale_rsqrt_launch(c, (int)m, (int)off, V, ldv, w, out, ldo);
}

int gcg_ritz_residuals(void* p, int64_t n, int64_t k, const double* AX, int64_t ldax,
                       const double* X, int64_t ldx, const double* BX, int64_t ldbx,
                       const double* lam, int mode, double* out) {
  Ctx* c = CTX(p);
  if (!c || n <= 0 || k < 0 || k > 256 || mode < 0 || mode > 2) return GCG_ERR_ARG;
  return ritz_residuals_launch(c, n, (int)k, AX, ldax, X, ldx, BX, ldbx, lam, mode, out);
}

// ---- reference-FFI tier (host buffers) --------------------------------------

static std::mutex g_host_mu;
static Ctx* g_host_ctx = nullptr;

static int host_ctx(Ctx** out) {
  if (!g_host_ctx) {
    void* p = nullptr;
    int s = gcg_ctx_create(&p, nullptr);
    if (s != GCG_OK) return s;
    g_host_ctx = CTX(p);
  }
  *out = g_host_ctx;
  return GCG_OK;
}

static int h2d_cm(Ctx* c, const double* host, long long rows, long long cols, long long ld,
                  double* dev) {
  // pack a column-major host block (rows x cols, column stride ld) densely
  if (rows == 0 || cols == 0) return GCG_OK;
  return cuda_status(cudaMemcpy2DAsync(dev, rows * sizeof(double), host, ld * sizeof(double),
                                       rows * sizeof(double), cols, cudaMemcpyHostToDevice,
                                       c->stream));
}

static int d2h_cm(Ctx* c, const double* dev, long long rows, long long cols, double* host,
                  long long ld) {
  if (rows == 0 || cols == 0) return GCG_OK;
  return cuda_status(cudaMemcpy2DAsync(host, ld * sizeof(double), dev, rows * sizeof(double),
                                       rows * sizeof(double), cols, cudaMemcpyDeviceToHost,
                                       c->stream));
}

static int elem_grid_host(Ctx* c, long long tot) { return grid_for(tot, 1024, 8, c->num_sms); }

int gcgeig_csr_matvec(const int64_t* indptr, const int64_t* indices, const double* data,
                      int64_t nrow, int64_t ncol, const double* x, int64_t k, int64_t ldx,
                      double* out, int64_t ldo) {
  if (nrow < 0 || ncol < 0 || k < 0 || ldx < ncol || ldo < nrow) return GCG_ERR_ARG;
  if (nrow == 0 || k == 0) return GCG_OK;
  const long long nnz = indptr[nrow] - indptr[0];
  if (indptr[0] != 0 || nnz < 0 || nnz >= (1LL << 31) || ncol >= (1LL << 31)) return GCG_ERR_ARG;
  std::lock_guard<std::mutex> lock(g_host_mu);
  Ctx* c;
  GCG_TRY(host_ctx(&c));
  // staging: indptr/indices as int64 then int32; values; x (cm, rm); y (rm, cm)
  const size_t b_idx = sizeof(long long) * ((size_t)nrow + 1 + (size_t)nnz);
  const size_t b_i32 = sizeof(int) * ((size_t)nrow + 1 + (size_t)nnz);
  const size_t b_val = sizeof(double) * (size_t)(nnz > 0 ? nnz : 1);
  const size_t b_x = sizeof(double) * (size_t)ncol * k;
  const size_t b_y = sizeof(double) * (size_t)nrow * k;
  GCG_TRY(ensure(c->host_tmp, b_idx + b_i32 + b_val + 64));
  GCG_TRY(ensure(c->host_tmp2, 2 * b_x + 64));
  GCG_TRY(ensure(c->host_tmp3, 2 * b_y + 64));
  char* base = (char*)c->host_tmp.ptr;
  long long* d_i64 = (long long*)base;
  int* d_i32 = (int*)(base + b_idx);
  double* d_val = (double*)(base + b_idx + b_i32 + (8 - (b_idx + b_i32) % 8) % 8);
  double* d_xcm = (double*)c->host_tmp2.ptr;
  double* d_xrm = d_xcm + (size_t)ncol * k;
  double* d_yrm = (double*)c->host_tmp3.ptr;
  double* d_ycm = d_yrm + (size_t)nrow * k;
  cudaStream_t s = c->stream;
  GCG_TRY(cuda_status(cudaMemcpyAsync(d_i64, indptr, sizeof(long long) * (nrow + 1),
                                      cudaMemcpyHostToDevice, s)));
  if (nnz > 0) {
    GCG_TRY(cuda_status(cudaMemcpyAsync(d_i64 + nrow + 1, indices, sizeof(long long) * nnz,
                                        cudaMemcpyHostToDevice, s)));
    GCG_TRY(cuda_status(
        cudaMemcpyAsync(d_val, data, sizeof(double) * nnz, cudaMemcpyHostToDevice, s)));
  }
  const long long nidx = nrow + 1 + nnz;
  i64_to_i32_kernel<<<elem_grid_host(c, nidx), 256, 0, s>>>(nidx, d_i64, d_i32);
  ++g_launches;
  GCG_TRY(h2d_cm(c, x, ncol, k, ldx, d_xcm));
  cm_to_rm_kernel<<<elem_grid_host(c, ncol * k), 256, 0, s>>>(ncol, (int)k, d_xcm, ncol, d_xrm);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  GCG_TRY(spmm_launch_impl(c, nrow, nnz, d_i32, d_i32 + nrow + 1, d_val, (int)k, d_xrm, k, 1.0, 0.0,
                           nullptr, 0, 0.0, nullptr, 0, d_yrm, k, 0, nullptr, 0, nullptr, nullptr,
                           nullptr, nullptr));
  rm_to_cm_kernel<<<elem_grid_host(c, nrow * k), 256, 0, s>>>(nrow, (int)k, d_yrm, d_ycm);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  GCG_TRY(d2h_cm(c, d_ycm, nrow, k, out, ldo));
  return cuda_status(cudaStreamSynchronize(s));
}

// A CSR operator resident in HBM for the reference's operator protocol
// (CsrOperator.apply, operators.py:103-111): the pattern and values are uploaded
// once, each apply moves only the F-order multivector in and the product out.
struct HostCsr {
  long long n = 0, ncol = 0, nnz = 0;
  int* rowptr = nullptr;  // n + 1, then nnz column indices (one allocation)
  double* val = nullptr;
};

int gcgeig_csr_create(const int64_t* indptr, const int64_t* indices, const double* data,
                      int64_t nrow, int64_t ncol, void** handle) {
  if (!handle) return GCG_ERR_ARG;
  *handle = nullptr;
  if (nrow < 0 || ncol < 0 || !indptr || nrow >= (1LL << 31) || ncol >= (1LL << 31))
    return GCG_ERR_ARG;
  const long long nnz = indptr[nrow] - indptr[0];
  if (indptr[0] != 0 || nnz < 0 || nnz >= (1LL << 31)) return GCG_ERR_ARG;
  for (long long i = 0; i < nrow; ++i)
    if (indptr[i + 1] < indptr[i]) return GCG_ERR_ARG;
  for (long long e = 0; e < nnz; ++e)
    if (indices[e] < 0 || indices[e] >= ncol) return GCG_ERR_ARG;
  std::lock_guard<std::mutex> lock(g_host_mu);
  Ctx* c;
  GCG_TRY(host_ctx(&c));
  HostCsr* h = new HostCsr();
  h->n = nrow;
  h->ncol = ncol;
  h->nnz = nnz;
  const size_t nidx = (size_t)nrow + 1 + (size_t)nnz;
  if (cudaMalloc((void**)&h->rowptr, sizeof(int) * nidx) != cudaSuccess ||
      cudaMalloc((void**)&h->val, sizeof(double) * (size_t)(nnz > 0 ? nnz : 1)) != cudaSuccess) {
    cudaFree(h->rowptr);
    delete h;
    return GCG_ERR_ALLOC;
  }
  GCG_TRY(ensure(c->host_tmp, sizeof(long long) * nidx + 64));
  long long* d_i64 = (long long*)c->host_tmp.ptr;
  cudaStream_t s = c->stream;
  GCG_TRY(cuda_status(cudaMemcpyAsync(d_i64, indptr, sizeof(long long) * (nrow + 1),
                                      cudaMemcpyHostToDevice, s)));
  if (nnz > 0) {
    GCG_TRY(cuda_status(cudaMemcpyAsync(d_i64 + nrow + 1, indices, sizeof(long long) * nnz,
                                        cudaMemcpyHostToDevice, s)));
    GCG_TRY(cuda_status(
        cudaMemcpyAsync(h->val, data, sizeof(double) * nnz, cudaMemcpyHostToDevice, s)));
  }
  i64_to_i32_kernel<<<elem_grid_host(c, (long long)nidx), 256, 0, s>>>((long long)nidx, d_i64,
                                                                       h->rowptr);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  GCG_TRY(cuda_status(cudaStreamSynchronize(s)));
  *handle = h;
  return GCG_OK;
}

int gcgeig_csr_apply(void* handle, const double* x, int64_t k, int64_t ldx, double* out,
                     int64_t ldo) {
  HostCsr* h = (HostCsr*)handle;
  if (!h || k < 0 || ldx < h->ncol || ldo < h->n) return GCG_ERR_ARG;
  if (h->n == 0 || k == 0) return GCG_OK;
  std::lock_guard<std::mutex> lock(g_host_mu);
  Ctx* c;
  GCG_TRY(host_ctx(&c));
  const size_t b_x = sizeof(double) * (size_t)h->ncol * k;
  const size_t b_y = sizeof(double) * (size_t)h->n * k;
  GCG_TRY(ensure(c->host_tmp2, 2 * b_x + 64));
  GCG_TRY(ensure(c->host_tmp3, 2 * b_y + 64));
  double* d_xcm = (double*)c->host_tmp2.ptr;
  double* d_xrm = d_xcm + (size_t)h->ncol * k;
  double* d_yrm = (double*)c->host_tmp3.ptr;
  double* d_ycm = d_yrm + (size_t)h->n * k;
  cudaStream_t s = c->stream;
  GCG_TRY(h2d_cm(c, x, h->ncol, k, ldx, d_xcm));
  cm_to_rm_kernel<<<elem_grid_host(c, h->ncol * k), 256, 0, s>>>(h->ncol, (int)k, d_xcm,
                                                                 h->ncol, d_xrm);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  GCG_TRY(spmm_launch_impl(c, h->n, h->nnz, h->rowptr, h->rowptr + h->n + 1, h->val, (int)k,
                           d_xrm, k, 1.0, 0.0, nullptr, 0, 0.0, nullptr, 0, d_yrm, k, 0, nullptr,
                           0, nullptr, nullptr, nullptr, nullptr));
  rm_to_cm_kernel<<<elem_grid_host(c, h->n * k), 256, 0, s>>>(h->n, (int)k, d_yrm, d_ycm);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  GCG_TRY(d2h_cm(c, d_ycm, h->n, k, out, ldo));
  return cuda_status(cudaStreamSynchronize(s));
}

int gcgeig_csr_destroy(void* handle) {
  HostCsr* h = (HostCsr*)handle;
  if (!h) return GCG_OK;
  std::lock_guard<std::mutex> lock(g_host_mu);
  if (g_host_ctx) cudaStreamSynchronize(g_host_ctx->stream);
  cudaFree(h->rowptr);
  cudaFree(h->val);
  delete h;
  return GCG_OK;
}

int gcgeig_inner_product(const double* x, int64_t n, int64_t kx, int64_t ldx, const double* y,
                         int64_t ky, int64_t ldy, double* out, int64_t out_rs, int64_t out_cs,
                         int64_t chunk, int deterministic) {
  (void)chunk;
  (void)deterministic;  // the device reduction order is fixed: always bit-stable
  if (n < 0 || kx < 0 || ky < 0 || ldx < n || ldy < n) return GCG_ERR_ARG;
  if (kx == 0 || ky == 0) return GCG_OK;
  std::lock_guard<std::mutex> lock(g_host_mu);
  Ctx* c;
  GCG_TRY(host_ctx(&c));
  const size_t bx = (size_t)n * kx, by = (size_t)n * ky, bg = (size_t)kx * ky;
  GCG_TRY(ensure(c->host_tmp2, sizeof(double) * (2 * bx + 8)));
  GCG_TRY(ensure(c->host_tmp3, sizeof(double) * (2 * by + 8)));
  GCG_TRY(ensure(c->host_tmp, sizeof(double) * (bg + 8)));
  double* d_xcm = (double*)c->host_tmp2.ptr;
  double* d_xrm = d_xcm + bx;
  double* d_ycm = (double*)c->host_tmp3.ptr;
  double* d_yrm = d_ycm + by;
  double* d_g = (double*)c->host_tmp.ptr;
  cudaStream_t s = c->stream;
  GCG_TRY(h2d_cm(c, x, n, kx, ldx, d_xcm));
  GCG_TRY(h2d_cm(c, y, n, ky, ldy, d_ycm));
  if (n > 0) {
    cm_to_rm_kernel<<<elem_grid_host(c, bx), 256, 0, s>>>(n, (int)kx, d_xcm, n, d_xrm);
    cm_to_rm_kernel<<<elem_grid_host(c, by), 256, 0, s>>>(n, (int)ky, d_ycm, n, d_yrm);
    g_launches += 2;
    GCG_CHECK_LAUNCH();
    GCG_TRY(gram_launch(c, n, (int)kx, (int)ky, d_xrm, kx, d_yrm, ky, 1.0, 0.0, d_g, ky, 1));
  } else {
    GCG_TRY(fill_launch(c, kx, (int)ky, 0.0, d_g, ky));
  }
  std::vector<double> g(bg);
  GCG_TRY(cuda_status(
      cudaMemcpyAsync(g.data(), d_g, sizeof(double) * bg, cudaMemcpyDeviceToHost, s)));
  GCG_TRY(cuda_status(cudaStreamSynchronize(s)));
  for (long long r = 0; r < kx; ++r)
    for (long long cc = 0; cc < ky; ++cc) out[r * out_rs + cc * out_cs] = g[r * ky + cc];
  return GCG_OK;
}

int gcgeig_axpby(double alpha, const double* x, int64_t n, int64_t k, int64_t ldx, double beta,
                 double* y, int64_t ldy) {
  if (n < 0 || k < 0 || ldx < n || ldy < n) return GCG_ERR_ARG;
  if (n == 0 || k == 0) return GCG_OK;
  std::lock_guard<std::mutex> lock(g_host_mu);
  Ctx* c;
  GCG_TRY(host_ctx(&c));
  const size_t b = (size_t)n * k;
  GCG_TRY(ensure(c->host_tmp2, sizeof(double) * (b + 8)));
  GCG_TRY(ensure(c->host_tmp3, sizeof(double) * (b + 8)));
  double* d_x = (double*)c->host_tmp2.ptr;
  double* d_y = (double*)c->host_tmp3.ptr;
  cudaStream_t s = c->stream;
  GCG_TRY(h2d_cm(c, x, n, k, ldx, d_x));
  if (beta != 0.0) GCG_TRY(h2d_cm(c, y, n, k, ldy, d_y));
  // a packed column-major n x k block is a row-major k x n block with ld n
  GCG_TRY(axpby_launch(c, k, (int)n, alpha, d_x, n, beta, d_y, n));
  GCG_TRY(d2h_cm(c, d_y, n, k, y, ldy));
  return cuda_status(cudaStreamSynchronize(s));
}

}  // extern "C"
