// BASELINE operators assembled directly in HBM.
//
// The host generators (problems.py stencil_csr / varcoef_diffusion_3d) build the
// structured-grid matrices with numpy: config 5 (27-pt, 256^3) alone needs
// ~6 GB of host temporaries and minutes, then 5.4 GB of H2D.  Here the same
// CSR — identical index order and bit-identical values — is written by the
// device: one thread per row counts its in-grid neighbours, a device prefix
// sum (CUB) turns the counts into row pointers, and a second pass writes
// column indices (offsets visited in increasing linear order, so rows come out
// sorted) and values (a constant per offset, or a per-row array).  The
// variable-coefficient 7-pt operator's per-row weights (harmonic-mean faces of
// the cell field, Dirichlet faces on the diagonal) are computed on the device
// in the host generator's exact operation order.

#include <cub/cub.cuh>

#include "common.cuh"

namespace gcg {

extern int64_t g_launches;

constexpr int kMaxOff = 27;

struct StencilDesc {
  int n0, n1, n2, noff;
  int d0[kMaxOff], d1[kMaxOff], d2[kMaxOff];
  long long lin[kMaxOff];
  double w[kMaxOff];
  const double* wrow[kMaxOff];
};

__device__ __forceinline__ bool in_grid(const StencilDesc& s, int z, int y, int x, int t) {
  const int a = z + s.d0[t], b = y + s.d1[t], c = x + s.d2[t];
  return a >= 0 && a < s.n0 && b >= 0 && b < s.n1 && c >= 0 && c < s.n2;
}

__global__ void stencil_count_kernel(const __grid_constant__ StencilDesc s, long long n,
                                     int* len) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % s.n2), y = (int)((i / s.n2) % s.n1), z = (int)(i / ((long long)s.n2 * s.n1));
    int cnt = 0;
    for (int t = 0; t < s.noff; ++t) cnt += in_grid(s, z, y, x, t);
    len[i] = cnt;
  }
}

__global__ void stencil_fill_kernel(const __grid_constant__ StencilDesc s, long long n,
                                    const int* __restrict__ rowptr, int* colidx, double* val) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % s.n2), y = (int)((i / s.n2) % s.n1), z = (int)(i / ((long long)s.n2 * s.n1));
    long long p = i == 0 ? 0 : rowptr[i];
    for (int t = 0; t < s.noff; ++t) {
      if (!in_grid(s, z, y, x, t)) continue;
      colidx[p] = (int)(i + s.lin[t]);
      val[p] = s.wrow[t] ? s.wrow[t][i] : s.w[t];
      ++p;
    }
  }
}

// Per-row weights of the cell-centred variable-coefficient 7-pt operator
// (problems.py varcoef_diffusion_3d): out[0] = diagonal, out[1 + 2*ax + (s>0)] =
// -face for direction (ax, s).  Same operation order as the numpy generator:
// face = 2*k*knb/(k+knb) (0 on a Dirichlet face), diag += face, diag += k on a
// Dirichlet face, directions in the order (ax 0..2) x (s = -1, +1).
__global__ void varcoef7_weights_kernel(int N, const double* __restrict__ kc, double* out) {
  const long long n = (long long)N * N * N;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int c[3] = {(int)(i / ((long long)N * N)), (int)((i / N) % N), (int)(i % N)};
    const long long st[3] = {(long long)N * N, N, 1};
    const double k = kc[i];
    double diag = 0.0;
    for (int ax = 0; ax < 3; ++ax) {
      for (int h = 0; h < 2; ++h) {
        const int sg = h ? 1 : -1;
        const bool bnd = sg < 0 ? c[ax] == 0 : c[ax] == N - 1;
        double face = 0.0;
        if (!bnd) {
          const double nb = kc[i + sg * st[ax]];
          face = 2.0 * k * nb / (k + nb);
        }
        diag = diag + face;
        diag = diag + (bnd ? k : 0.0);
        out[(long long)(1 + 2 * ax + h) * n + i] = -face;
      }
    }
    out[i] = diag;
  }
}

static int fill_desc(StencilDesc& s, int64_t n0, int64_t n1, int64_t n2, int noff,
                     const int* offs, const double* w, const double* const* wrow) {
  if (noff < 1 || noff > kMaxOff || n0 < 1 || n1 < 1 || n2 < 1) return GCG_ERR_ARG;
  s.n0 = (int)n0;
  s.n1 = (int)n1;
  s.n2 = (int)n2;
  s.noff = noff;
  // visit offsets in increasing linear order (sorted columns)
  int order[kMaxOff];
  long long lin[kMaxOff];
  for (int t = 0; t < noff; ++t) {
    lin[t] = (long long)offs[3 * t] * n1 * n2 + (long long)offs[3 * t + 1] * n2 + offs[3 * t + 2];
    order[t] = t;
  }
  for (int a = 1; a < noff; ++a)  // stable insertion sort
    for (int b = a; b > 0 && lin[order[b - 1]] > lin[order[b]]; --b) {
      const int tmp = order[b];
      order[b] = order[b - 1];
      order[b - 1] = tmp;
    }
  for (int q = 0; q < noff; ++q) {
    const int t = order[q];
    s.d0[q] = offs[3 * t];
    s.d1[q] = offs[3 * t + 1];
    s.d2[q] = offs[3 * t + 2];
    s.lin[q] = lin[t];
    s.w[q] = w ? w[t] : 0.0;
    s.wrow[q] = wrow ? wrow[t] : nullptr;
  }
  return GCG_OK;
}

}  // namespace gcg

using namespace gcg;

extern "C" {

int gcg_stencil_nnz(int64_t n0, int64_t n1, int64_t n2, int32_t noff, const int32_t* offs,
                    int64_t* nnz) {
  if (!offs || !nnz || noff < 1 || n0 < 1 || n1 < 1 || n2 < 1) return GCG_ERR_ARG;
  long long tot = 0;
  for (int t = 0; t < noff; ++t) {
    long long c = 1;
    const int64_t dims[3] = {n0, n1, n2};
    for (int a = 0; a < 3; ++a) {
      const long long d = offs[3 * t + a] < 0 ? -offs[3 * t + a] : offs[3 * t + a];
      c *= dims[a] > d ? dims[a] - d : 0;
    }
    tot += c;
  }
  *nnz = tot;
  return GCG_OK;
}

int gcg_stencil_csr(void* ctx, int64_t n0, int64_t n1, int64_t n2, int32_t noff,
                    const int32_t* offs, const double* w, const double* const* wrow, int32_t* rowptr,
                    int32_t* colidx, double* val) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !offs || !rowptr || !colidx || !val || (!w && !wrow)) return GCG_ERR_ARG;
  StencilDesc s;
  GCG_TRY(fill_desc(s, n0, n1, n2, noff, offs, w, wrow));
  const long long n = (long long)n0 * n1 * n2;
  int64_t nnz = 0;
  GCG_TRY(gcg_stencil_nnz(n0, n1, n2, noff, offs, &nnz));
  if (n >= (1LL << 31) || nnz >= (1LL << 31)) return GCG_ERR_ARG;
  const int grid = grid_for(n, 256, 8, c->num_sms);
  // row lengths into rowptr[1..n], inclusive scan in place, rowptr[0] = 0
  stencil_count_kernel<<<grid, 256, 0, c->stream>>>(s, n, rowptr + 1);
  GCG_CHECK_LAUNCH();
  size_t tmp = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp, rowptr + 1, rowptr + 1, (int)n, c->stream);
  GCG_TRY(ensure(c->host_tmp, tmp + 16));
  if (cub::DeviceScan::InclusiveSum(c->host_tmp.ptr, tmp, rowptr + 1, rowptr + 1, (int)n,
                                    c->stream) != cudaSuccess)
    return GCG_ERR_CUDA;
  GCG_TRY(cuda_status(cudaMemsetAsync(rowptr, 0, sizeof(int32_t), c->stream)));
  stencil_fill_kernel<<<grid, 256, 0, c->stream>>>(s, n, rowptr, colidx, val);
  g_launches += 3;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

int gcg_varcoef7_weights(void* ctx, int64_t N, const double* kc, double* out) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || N < 1 || !kc || !out) return GCG_ERR_ARG;
  const long long n = (long long)N * N * N;
  varcoef7_weights_kernel<<<grid_for(n, 256, 8, c->num_sms), 256, 0, c->stream>>>((int)N, kc, out);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

}  // extern "C"
