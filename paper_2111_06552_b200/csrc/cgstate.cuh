// Device state of the block-CG sweeps (cg.cu) shared with the fused sweep SpMM
// (spmm.cu): per-column scalars and flags, and the fixed-order column sums every
// consumer CTA computes from a producer's per-CTA partials.
#pragma once

#include "common.cuh"

namespace gcg {

struct CgState {
  double* rz;      // [2][k]: r'r of the current sweep at one parity, the next at the other
  double* rn;      // ||r|| (last tested)
  double* rn0;     // ||r0||
  double* target;  // rel_tol * ||r0||
  double* alpha;   // alpha of the last r-update (its x-update is deferred to the next SpMM)
  int* conv;
  int* frozen;
  int* upd;        // column updated by the last r-update
  int* skip1;      // set: the next sweep SpMM is a no-op (written by the r-update / init)
  int* skip2;      // set: the next r-update is a no-op (written by the sweep SpMM)
  int* pending;    // the last r-update's x += alpha p has not been applied yet
  int* sweeps;
  int* nact;
  int* ticket;
};

// Extra arguments of the fused sweep SpMM (spmm.cu, CG mode): it gathers r, and from
// own-row values forms x += alpha p (deferred from the previous sweep),
// p = r + beta p and q = (A + shift) r + beta q (so q = (A + shift) p without a
// second gather), plus the p'q partials.
struct CgSweep {
  CgState s;
  const double* rpart;  // ||r||^2 partials of the previous r-update ([nrp][k])
  int nrp;
  int k;                // total CG columns (the SpMM may run in column passes)
  int par;              // rz parity read (old) — the new value goes to par ^ 1
  int first;            // sweep 0: p = r, q = (A + shift) r, no x-update
  double* x;            // iterate, dense n x k
  double* P;            // search directions, dense n x k
  double* Q;            // (A + shift) P, dense n x k
};

// Fixed-order column sums of an nparts x k block of per-CTA partials, computed
// redundantly by every CTA of the consumer kernel (256 threads, k <= 256): thread t
// sums column t % k over parts t / k, t / k + L, ... (L = 256 / k), then the L
// partials of each column are added in lane order — the same bits in every CTA and
// run to run.  Replaces a separate 1-CTA "finish" launch per reduction.
__device__ __forceinline__ void cta_column_sums(const double* part, int nparts, int k, double* sm,
                                                double* out) {
  const int L = blockDim.x / k;
  const int c = threadIdx.x % k, l = threadIdx.x / k;
  double v = 0.0;
  if (l < L) {
    // 16 independent loads in flight per round (the tail round predicated, not serial),
    // added in index order
    constexpr int U = 16;
    for (int b = l; b < nparts; b += U * L) {
      double t[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        t[u] = b + u * L < nparts ? part[(long long)(b + u * L) * k + c] : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) v += t[u];
    }
  }
  sm[threadIdx.x] = v;
  __syncthreads();
  if (threadIdx.x < k) {
    double t = 0.0;
    for (int j = 0; j < L; ++j) t += sm[j * k + threadIdx.x];
    out[threadIdx.x] = t;
  }
  __syncthreads();
}

}  // namespace gcg
