// Native orchestration of the B-orthogonalisation (Alg. 3 and orth_against) on one GPU.
//
// Reference: orth.py — _deflate_against (:124-152), _leaf_svqb (:155-188),
// _recurse_svd (:191-204), recursive_orth_svd (:207-226), orth_against
// (:339-372), _Ctx.pull_rear (:95-108).
//
// The control flow is the reference's (and orth.py's, which keeps it for the
// row-partitioned path and for Alg. 2): recursion, repeat-until tests,
// dependent-column replacement, reduction counts.  Each decision needs a few
// doubles from the device; driving the loop from C++ turns every such round
// trip into one pinned 32-byte read (~10 us) instead of a Python step
// (~40 us of interpreter time between the read and the next launch, during
// which the GPU idles).  All arithmetic is the library's kernels: Gram with the
// squared norms riding along as the diagonal of the bottom block, LinComb
// (in place for the SVQB update), the fused deflation status and the one-CTA
// Jacobi SVQB kernel.

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace gcg {

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
int copy_launch(Ctx* c, long long n, int k, const double* X, long long ldx, double* Y,
                long long ldy);
int col_dots_launch(Ctx* c, long long n, int k, const double* X, long long ldx, const double* Y,
                    long long ldy, double* out);
int svqb_prepare_launch(Ctx* c, int m, const double* G, long long ldg, double dep_tol,
                        double skip_tol, double* Q, long long ldq, double* status);
int deflate_status_launch(Ctx* c, int K, int w, const double* R, long long ldr,
                          const double* dnew, long long dstride, double dgks, double* status);

namespace {

constexpr double kDgks = 0.5;  // orth.py:43

struct Run {
  Ctx* c;
  long long n;
  double* x;
  long long ldx;
  long long bnnz;
  const int* brp;
  const int* bci;
  const double* bv;
  gcg_orth_opts o;
  long long start, active_end;
  long long reductions = 0;
  std::vector<long long> replaced;
  long long leaf = 16;
  // scratch (from c->orth): status | g | q | bt
  double* status;
  double* g;
  double* q;
  double* bt;
  double* host;

  double* col(long long j) const { return x + j; }

  // B y into scratch (or y itself when B = I); returns the pointer and its ld
  int bdot(const double* y, long long w, const double** out, long long* ld) {
    if (!brp) {
      *out = y;
      *ld = ldx;
      return GCG_OK;
    }
    GCG_TRY(spmm_launch_impl(c, n, bnnz, brp, bci, bv, (int)w, y, ldx, 1.0, 0.0, nullptr, 0, 0.0,
                             nullptr, 0, bt, w, 0, nullptr, 0, nullptr, nullptr, nullptr,
                             nullptr));
    *out = bt;
    *ld = w;
    return GCG_OK;
  }

  // the status kernels wrote into host-mapped slots: the decision read is the stream
  // synchronisation alone (no copy launch between the kernel and the host)
  int read(int count) {
    (void)count;
    return cuda_status(cudaStreamSynchronize(c->stream));
  }

  bool pull_rear(long long slot) {
    replaced.push_back(slot);
    if (active_end - 1 > slot) {
      --active_end;
      copy_launch(c, n, 1, col(active_end), ldx, col(slot), ldx);
      return true;
    }
    active_end = slot;
    return false;
  }

  // orth.py:124-152; basis is n x K (ldb), target x[:, lo:hi]
  int deflate(const double* basis, long long ldb, long long K, long long lo, long long hi,
              int* passes_out) {
    int passes = 0;
    while (passes < o.max_passes) {
      hi = std::min(hi, active_end);
      if (lo >= hi || K == 0) break;
      const long long w = hi - lo;
      double* target = col(lo);
      const double* bt_p;
      long long bt_ld;
      GCG_TRY(bdot(target, w, &bt_p, &bt_ld));
      const double* coef = g;
      const double* dnew;
      long long dstride;
      if (basis + K == target && ldb == ldx) {
        // [basis | target]' (B target): coefficients on top, squared norms on the
        // diagonal of the bottom w x w block — one fused reduction
        GCG_TRY(gram_launch(c, n, (int)(K + w), (int)w, basis, ldb, bt_p, bt_ld, 1.0, 0.0, g, w,
                            1));
        dnew = g + K * w;
        dstride = w + 1;
      } else {
        GCG_TRY(gram_launch(c, n, (int)K, (int)w, basis, ldb, bt_p, bt_ld, 1.0, 0.0, g, w, 1));
        double* dn = g + K * w;
        GCG_TRY(col_dots_launch(c, n, (int)w, target, ldx, bt_p, bt_ld, dn));
        dnew = dn;
        dstride = 1;
      }
      ++reductions;
      ++passes;
      GCG_TRY(lincomb_launch(c, n, (int)K, (int)w, -1.0, basis, ldb, coef, w, 1.0, target, ldx));
      GCG_TRY(deflate_status_launch(c, (int)K, (int)w, coef, w, dnew, dstride, kDgks, status));
      GCG_TRY(read(2));
      if (host[0] <= o.reorth_tol) break;
      if (host[1] == 0.0) break;
    }
    if (passes_out) *passes_out = passes;
    return GCG_OK;
  }

  // orth.py:155-188
  int leaf_svqb(long long lo, long long hi) {
    int passes = 0;
    while (true) {
      hi = std::min(hi, active_end);
      if (lo >= hi) return GCG_OK;
      const long long w = hi - lo;
      double* block = col(lo);
      const double* bb;
      long long bb_ld;
      GCG_TRY(bdot(block, w, &bb, &bb_ld));
      GCG_TRY(gram_launch(c, n, (int)w, (int)w, block, ldx, bb, bb_ld, 1.0, 0.0, g, w, 1));
      ++reductions;
      ++passes;
      GCG_TRY(svqb_prepare_launch(c, (int)w, g, w, o.dependence_tol, o.reorth_tol, q, w, status));
      GCG_TRY(read(2));
      if (host[0] <= o.reorth_tol) return GCG_OK;
      const long long bad = (long long)host[1];
      const long long kept = w - bad;
      if (kept > 0) {
        if (kept <= 256) {  // in place: every output row is produced from its own input row
          GCG_TRY(lincomb_launch(c, n, (int)w, (int)kept, 1.0, block, ldx, q, w, 0.0, block, ldx));
        } else {
          GCG_TRY(lincomb_launch(c, n, (int)w, (int)kept, 1.0, block, ldx, q, w, 0.0, bt, kept));
          GCG_TRY(copy_launch(c, n, (int)kept, bt, kept, block, ldx));
        }
      }
      if (bad == 0) {
        if (passes >= o.max_passes) return GCG_OK;
        continue;
      }
      for (long long slot = lo + kept; slot < hi; ++slot)
        if (!pull_rear(slot)) break;
      passes = 0;
    }
  }

  // orth.py:191-204
  int recurse(long long lo, long long hi) {
    hi = std::min(hi, active_end);
    if (lo >= hi) return GCG_OK;
    const long long width = hi - lo;
    if (width <= leaf) return leaf_svqb(lo, hi);
    long long mid = lo + width / 2;
    GCG_TRY(recurse(lo, mid));
    mid = std::min(mid, active_end);
    if (lo < mid && mid < active_end) GCG_TRY(deflate(col(lo), ldx, mid - lo, mid, hi, nullptr));
    return recurse(mid, hi);
  }
};

int setup(Ctx* c, Run& r, long long wmax, long long kmax) {
  if (!c->pinned) {
    if (cudaHostAlloc((void**)&c->pinned, 64 * sizeof(double), cudaHostAllocDefault) !=
        cudaSuccess) {
      cudaGetLastError();
      return GCG_ERR_ALLOC;
    }
  }
  const size_t gsz = (size_t)(kmax + wmax) * wmax + wmax;
  const size_t qsz = (size_t)wmax * wmax;
  const size_t bsz = (r.brp || wmax > 256) ? (size_t)r.n * wmax : 0;
  GCG_TRY(ensure(c->orth, sizeof(double) * (8 + gsz + qsz + bsz) + 256));
  double* base = (double*)c->orth.ptr;
  GCG_TRY(ensure_mapped(c));
  r.status = c->mapped_dev;
  r.g = base + 8;
  r.q = r.g + gsz;
  r.bt = r.q + qsz;
  r.host = c->mapped;
  return GCG_OK;
}

void fill_out(const Run& r, long long kept, int64_t* kept_out, int64_t* red_out,
              int64_t* replaced, int64_t cap, int64_t* nrep) {
  *kept_out = kept;
  *red_out = r.reductions;
  const long long nr = (long long)r.replaced.size();
  if (nrep) *nrep = nr;
  if (replaced)
    for (long long i = 0; i < nr && i < cap; ++i) replaced[i] = r.replaced[i];
}

}  // namespace
}  // namespace gcg

using namespace gcg;

extern "C" {

int gcg_orth_recursive(void* ctx, int64_t n, double* X, int64_t ldx, int64_t lo, int64_t hi,
                       int64_t b_nnz, const int* b_rowptr, const int* b_colidx,
                       const double* b_val, const gcg_orth_opts* opts, int64_t* kept,
                       int64_t* reductions, int64_t* replaced, int64_t cap, int64_t* nrep) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !opts || !kept || !reductions || n < 0 || lo < 0 || hi <= lo || ldx < hi)
    return GCG_ERR_ARG;
  Run r{c, n, X, ldx, b_nnz, b_rowptr, b_colidx, b_val, *opts, lo, hi};
  if (r.o.max_passes < 1) r.o.max_passes = 1;
  r.leaf = opts->svd_leaf > 0 ? opts->svd_leaf : std::min<long long>(hi - lo, 16);
  GCG_TRY(setup(c, r, hi - lo, hi - lo));
  GCG_TRY(r.recurse(lo, hi));
  fill_out(r, r.active_end - lo, kept, reductions, replaced, cap, nrep);
  return GCG_OK;
}

int gcg_orth_against(void* ctx, int64_t n, double* X, int64_t ldx, int64_t w,
                     const double* basis, int64_t ldb, int64_t K, int64_t b_nnz,
                     const int* b_rowptr, const int* b_colidx, const double* b_val,
                     const gcg_orth_opts* opts, int64_t* kept, int64_t* reductions,
                     int64_t* replaced, int64_t cap, int64_t* nrep) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !opts || !kept || !reductions || n < 0 || w <= 0 || ldx < w || K < 0 ||
      (K > 0 && (!basis || ldb < K)))
    return GCG_ERR_ARG;
  gcg_orth_opts o = *opts;
  if (o.max_passes < 1) o.max_passes = 1;
  // deflation against the basis (orth.py:356-357)
  const long long kmax = std::max<long long>(K, w);  // one scratch layout for all three phases
  Run st{c, n, X, ldx, b_nnz, b_rowptr, b_colidx, b_val, o, 0, w};
  GCG_TRY(setup(c, st, w, kmax));
  if (K > 0) GCG_TRY(st.deflate(basis, ldb, K, 0, w, nullptr));
  // Alg. 3 on the block (orth.py:358)
  Run in{c, n, X, ldx, b_nnz, b_rowptr, b_colidx, b_val, o, 0, w};
  in.leaf = o.svd_leaf > 0 ? o.svd_leaf : std::min<long long>(w, 16);
  GCG_TRY(setup(c, in, w, kmax));
  GCG_TRY(in.recurse(0, w));
  long long k_out = in.active_end;
  std::vector<long long> rep = in.replaced;
  long long extra = 0;
  // re-deflate at unit scale and re-true the kept block (orth.py:361-371)
  if (K > 0 && k_out > 0) {
    Run post{c, n, X, ldx, b_nnz, b_rowptr, b_colidx, b_val, o, 0, k_out};
    GCG_TRY(setup(c, post, w, kmax));
    GCG_TRY(post.deflate(basis, ldb, K, 0, k_out, nullptr));
    GCG_TRY(post.leaf_svqb(0, k_out));
    k_out = post.active_end;
    rep.insert(rep.end(), post.replaced.begin(), post.replaced.end());
    extra = post.reductions;
  }
  Run tot = in;
  tot.replaced = rep;
  tot.reductions = st.reductions + in.reductions + extra;
  fill_out(tot, k_out, kept, reductions, replaced, cap, nrep);
  return GCG_OK;
}

}  // extern "C"
