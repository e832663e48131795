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
int deflate_status_spec_launch(Ctx* c, int K, int w, const double* R, long long ldr,
                               const double* dnew, long long dstride, double dgks,
                               double* status, double stop_tol, int* stop_out);
int svqb_prepare_spec_launch(Ctx* c, int m, const double* G, long long ldg, double dep_tol,
                             double skip_tol, double* Q, long long ldq, double* status,
                             int* stop_out);
bool svqb_spec_ok(int m);

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

  // Speculative passes.  A repeat-until loop (DGKS deflation passes, SVQB passes) has
  // the same shapes in every pass, so the next pass is enqueued BEFORE the host reads
  // the current pass's decision: its kernels take the current pass's device stop flag
  // (Ctx::skip) and return at once when it is set, and the host waits on an event
  // recorded after the current pass's status kernel instead of on the whole stream.
  // The decision round trip then overlaps the next pass instead of idling the GPU;
  // a pass after a "stop" costs a few no-op launches.  Same passes, same arithmetic,
  // same reduction counts as the synchronous loop (GCG_ORTH_SPEC=0).
  long long pc = 0;  // passes enqueued by this run: status slot / event parity
  int dsite = 1, lsite = 3;  // call sites (Ctx::spec_hist): recursion by default
  static bool spec_on() {
    static const bool on = !(getenv("GCG_ORTH_SPEC") && getenv("GCG_ORTH_SPEC")[0] == '0');
    return on;
  }
  int* next_stop() { return c->spec + (c->spec_seq++ % kSpecRing); }
  double* slot_dev(long long k) { return status + 4 * (k & 1); }
  const double* slot_host(long long k) const { return host + 4 * (k & 1); }
  int mark(long long k) { return cuda_status(cudaEventRecord(c->spec_ev[k & 1], c->stream)); }
  int wait(long long k) { return cuda_status(cudaEventSynchronize(c->spec_ev[k & 1])); }

  // one deflation pass of x[:, lo:lo+w] against basis (K columns), status into slot k
  int deflate_pass(const double* basis, long long ldb, long long K, long long lo, long long w,
                   long long k, int* stop) {
    double* target = col(lo);
    const double* bt_p;
    long long bt_ld;
    if (!brp) {
      bt_p = target;
      bt_ld = ldx;
    } else {
      GCG_TRY(spmm_launch_impl(c, n, bnnz, brp, bci, bv, (int)w, target, ldx, 1.0, 0.0, nullptr,
                               0, 0.0, nullptr, 0, bt, w, 0, nullptr, 0, nullptr, nullptr,
                               nullptr, c->skip));
      bt_p = bt;
      bt_ld = w;
    }
    const double* dnew;
    long long dstride;
    if (basis + K == target && ldb == ldx) {
      GCG_TRY(gram_launch(c, n, (int)(K + w), (int)w, basis, ldb, bt_p, bt_ld, 1.0, 0.0, g, w, 1));
      dnew = g + K * w;
      dstride = w + 1;
    } else {
      GCG_TRY(gram_launch(c, n, (int)K, (int)w, basis, ldb, bt_p, bt_ld, 1.0, 0.0, g, w, 1));
      double* dn = g + K * w;
      GCG_TRY(col_dots_launch(c, n, (int)w, target, ldx, bt_p, bt_ld, dn));
      dnew = dn;
      dstride = 1;
    }
    GCG_TRY(lincomb_launch(c, n, (int)K, (int)w, -1.0, basis, ldb, g, w, 1.0, target, ldx));
    return deflate_status_spec_launch(c, (int)K, (int)w, g, w, dnew, dstride, kDgks, slot_dev(k),
                                      o.reorth_tol, stop);
  }

  // orth.py:124-152 with the next pass speculatively in flight
  int deflate_spec(const double* basis, long long ldb, long long K, long long lo, long long hi,
                   int* passes_out) {
    int passes = 0;
    hi = std::min(hi, active_end);
    if (lo < hi && K > 0) {
      const long long w = hi - lo;
      const int* prev = nullptr;  // stop flag of the newest enqueued pass
      int launched = 0;
      const long long k0 = pc;
      auto enqueue = [&]() -> int {
        int* stop = next_stop();
        c->skip = prev;
        const int rc = deflate_pass(basis, ldb, K, lo, w, pc, stop);
        c->skip = nullptr;
        GCG_TRY(rc);
        prev = stop;
        GCG_TRY(mark(pc));
        ++pc;
        ++launched;
        return GCG_OK;
      };
      const int predict = c->spec_hist[dsite];
      GCG_TRY(enqueue());
      while (true) {
        if (launched < o.max_passes && launched < predict) GCG_TRY(enqueue());
        GCG_TRY(wait(k0 + passes));
        const double* h = slot_host(k0 + passes);
        ++reductions;
        ++passes;
        if (h[0] <= o.reorth_tol || h[1] == 0.0 || passes >= o.max_passes) break;
        if (launched == passes) GCG_TRY(enqueue());  // not predicted: enqueue it now
      }
      c->spec_hist[dsite] = passes;
    }
    if (passes_out) *passes_out = passes;
    return GCG_OK;
  }

  // one SVQB Gram + prepare of x[:, lo:lo+w] (small leaves), status into slot k
  int svqb_pass(long long lo, long long w, long long k, int* stop) {
    double* block = col(lo);
    const double* bb;
    long long bb_ld;
    if (!brp) {
      bb = block;
      bb_ld = ldx;
    } else {
      GCG_TRY(spmm_launch_impl(c, n, bnnz, brp, bci, bv, (int)w, block, ldx, 1.0, 0.0, nullptr, 0,
                               0.0, nullptr, 0, bt, w, 0, nullptr, 0, nullptr, nullptr, nullptr,
                               c->skip));
      bb = bt;
      bb_ld = w;
    }
    GCG_TRY(gram_launch(c, n, (int)w, (int)w, block, ldx, bb, bb_ld, 1.0, 0.0, g, w, 1));
    return svqb_prepare_spec_launch(c, (int)w, g, w, o.dependence_tol, o.reorth_tol, q, w,
                                    slot_dev(k), stop);
  }

  // orth.py:155-188 with the next pass (update + Gram + prepare) speculatively in flight
  int leaf_svqb_spec(long long lo, long long hi) {
    int passes = 0;
    while (true) {
      hi = std::min(hi, active_end);
      if (lo >= hi) return GCG_OK;
      const long long w = hi - lo;
      double* block = col(lo);
      const int predict = c->spec_hist[lsite];
      int* stop = next_stop();
      long long k = pc++;
      GCG_TRY(svqb_pass(lo, w, k, stop));
      GCG_TRY(mark(k));
      while (true) {
        bool ahead = false;
        int* stop2 = nullptr;
        if (passes + 1 < o.max_passes && passes + 1 < predict) {
          // this pass's in-place update and the next pass: no-ops unless the block was
          // neither converged nor rank-deficient
          stop2 = next_stop();
          c->skip = stop;
          int rc = lincomb_launch(c, n, (int)w, (int)w, 1.0, block, ldx, q, w, 0.0, block, ldx);
          if (rc == GCG_OK) rc = svqb_pass(lo, w, pc, stop2);
          c->skip = nullptr;
          GCG_TRY(rc);
          GCG_TRY(mark(pc));
          ++pc;
          ahead = true;
        }
        GCG_TRY(wait(k));
        const double* h = slot_host(k);
        ++reductions;
        ++passes;
        if (h[0] <= o.reorth_tol) {
          c->spec_hist[lsite] = passes;
          return GCG_OK;
        }
        const long long bad = (long long)h[1];
        const long long kept = w - bad;
        if (bad == 0 && ahead) {  // the update ran, the next pass is in flight
          k = k + 1;
          stop = stop2;
          continue;
        }
        if (kept > 0)
          GCG_TRY(lincomb_launch(c, n, (int)w, (int)kept, 1.0, block, ldx, q, w, 0.0, block, ldx));
        if (bad == 0) {
          if (passes >= o.max_passes) {
            c->spec_hist[lsite] = passes;
            return GCG_OK;
          }
          stop = next_stop();  // not predicted: the next pass, enqueued now
          k = pc++;
          GCG_TRY(svqb_pass(lo, w, k, stop));
          GCG_TRY(mark(k));
          continue;
        }
        for (long long slot = lo + kept; slot < hi; ++slot)
          if (!pull_rear(slot)) break;
        passes = 0;
        break;
      }
    }
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
    if (spec_on()) return deflate_spec(basis, ldb, K, lo, hi, passes_out);
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
    if (spec_on() && svqb_spec_ok((int)std::min(hi, active_end) - (int)lo) &&
        std::min(hi, active_end) - lo <= 256)
      return leaf_svqb_spec(lo, hi);
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
  if (!c->spec) {
    if (cudaMalloc((void**)&c->spec, sizeof(int) * kSpecRing) != cudaSuccess ||
        cudaMemset(c->spec, 0, sizeof(int) * kSpecRing) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->spec_ev[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->spec_ev[1], cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      return GCG_ERR_ALLOC;
    }
  }
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
  st.dsite = 0;
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
    post.dsite = 2;
    post.lsite = 4;
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
