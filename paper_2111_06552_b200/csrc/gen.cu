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

#include <string.h>

#include <cub/device/device_radix_sort.cuh>
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

// One rank's slab [row0, row1) of the stencil, columns remapped to the local layout
// of a row-partitioned run (distributed.local_part): owned rows 0..nloc-1, then the
// ghost plane below the slab (global rows [row0 - nprev, row0)), then the one above
// ([row1, row1 + nnext)).  Offsets are visited in increasing linear order, as in the
// global generator, so each row's entries keep the global column order.
struct SlabMap {
  long long row0, row1, nprev, nnext;
};

__global__ void slab_count_kernel(const __grid_constant__ StencilDesc s, SlabMap m, int* len) {
  const long long nloc = m.row1 - m.row0;
  for (long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x; l < nloc;
       l += (long long)gridDim.x * blockDim.x) {
    const long long i = m.row0 + l;
    const int x = (int)(i % s.n2), y = (int)((i / s.n2) % s.n1), z = (int)(i / ((long long)s.n2 * s.n1));
    int cnt = 0;
    for (int t = 0; t < s.noff; ++t) cnt += in_grid(s, z, y, x, t);
    len[l] = cnt;
  }
}

__global__ void slab_fill_kernel(const __grid_constant__ StencilDesc s, SlabMap m,
                                 const int* __restrict__ rowptr, int* colidx, double* val,
                                 int* bad) {
  const long long nloc = m.row1 - m.row0;
  for (long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x; l < nloc;
       l += (long long)gridDim.x * blockDim.x) {
    const long long i = m.row0 + l;
    const int x = (int)(i % s.n2), y = (int)((i / s.n2) % s.n1), z = (int)(i / ((long long)s.n2 * s.n1));
    long long p = l == 0 ? 0 : rowptr[l];
    for (int t = 0; t < s.noff; ++t) {
      if (!in_grid(s, z, y, x, t)) continue;
      const long long j = i + s.lin[t];
      long long c;
      if (j >= m.row0 && j < m.row1) {
        c = j - m.row0;
      } else if (j < m.row0 && j >= m.row0 - m.nprev) {
        c = nloc + (j - (m.row0 - m.nprev));
      } else if (j >= m.row1 && j < m.row1 + m.nnext) {
        c = nloc + m.nprev + (j - m.row1);
      } else {
        c = 0;
        atomicExch(bad, 1);  // stencil reaches beyond one ghost plane
      }
      colidx[p] = (int)c;
      val[p] = s.wrow[t] ? s.wrow[t][i] : s.w[t];
      ++p;
    }
  }
}

// Validation of a square CSR operator on the device (the reference's CsrOperator /
// DenseOperator checks, operators.py:56-66, 79-87): out = {max |a_ij|, max |a_ij - a_ji|,
// #non-finite entries, #column indices out of range}.  Rows must be sorted (canonical
// CSR): a_ji is found by binary search in row j; a missing transposed entry counts as 0.
__device__ __forceinline__ void atomic_max_nonneg(double* a, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(a), (unsigned long long)__double_as_longlong(v));
}

__global__ void csr_check_kernel(long long n, const int* __restrict__ rowptr,
                                 const int* __restrict__ colidx, const double* __restrict__ val,
                                 double* out, unsigned long long* counts) {
  double mx = 0.0, md = 0.0;
  unsigned long long nonfin = 0, badcol = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    for (int e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      const double v = val[e];
      const int j = colidx[e];
      if (!isfinite(v)) {
        ++nonfin;
        continue;
      }
      if (j < 0 || j >= n) {
        ++badcol;
        continue;
      }
      mx = fmax(mx, fabs(v));
      int lo = rowptr[j], hi = rowptr[j + 1];
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (colidx[mid] < i) lo = mid + 1;
        else hi = mid;
      }
      const double vt = (lo < rowptr[j + 1] && colidx[lo] == i) ? val[lo] : 0.0;
      md = fmax(md, fabs(v - vt));
    }
  }
  mx = warp_max(mx);
  md = warp_max(md);
  if ((threadIdx.x & 31) == 0) {
    if (mx > 0.0) atomic_max_nonneg(out, mx);
    if (md > 0.0) atomic_max_nonneg(out + 1, md);
  }
  if (nonfin) atomicAdd(counts, nonfin);
  if (badcol) atomicAdd(counts + 1, badcol);
}

// Seeded N(0,1) block on the device: Philox4x32-10 keyed by the seed, counter = (global
// row, column pair); Box-Muller on two 53-bit uniforms.  Entry (i, c) depends only on
// (seed, row0 + i, c), so any row partition draws the same global block.
__device__ __forceinline__ void philox10(uint32_t ctr[4], uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t h0 = __umulhi(M0, ctr[0]), l0 = M0 * ctr[0];
    const uint32_t h1 = __umulhi(M1, ctr[2]), l1 = M1 * ctr[2];
    const uint32_t n0 = h1 ^ ctr[1] ^ k0, n2 = h0 ^ ctr[3] ^ k1;
    ctr[0] = n0;
    ctr[1] = l1;
    ctr[2] = n2;
    ctr[3] = l0;
    k0 += W0;
    k1 += W1;
  }
}

__global__ void fill_normal_kernel(long long n, int k, long long row0, unsigned long long seed,
                                   double* X, long long ldx) {
  const int pairs = (k + 1) / 2;
  const long long tot = n * pairs;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < tot;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / pairs;
    const int cp = (int)(t % pairs);
    const unsigned long long g = (unsigned long long)(row0 + i);
    uint32_t ctr[4] = {(uint32_t)g, (uint32_t)(g >> 32), (uint32_t)cp, 0x6763672du};
    philox10(ctr, (uint32_t)seed, (uint32_t)(seed >> 32));
    const unsigned long long a = ((unsigned long long)ctr[0] << 21) ^ ctr[1];
    const unsigned long long b = ((unsigned long long)ctr[2] << 21) ^ ctr[3];
    const double u1 = ((double)(a & ((1ULL << 53) - 1)) + 1.0) * 0x1.0p-53;  // (0, 1]
    const double u2 = (double)(b & ((1ULL << 53) - 1)) * 0x1.0p-53;          // [0, 1)
    const double rad = sqrt(-2.0 * log(u1));
    double s, c;
    sincospi(2.0 * u2, &s, &c);
    const int c0 = 2 * cp;
    X[i * ldx + c0] = rad * c;
    if (c0 + 1 < k) X[i * ldx + c0 + 1] = rad * s;
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

static inline double __longlong_as_double_host(unsigned long long b) {
  double d;
  memcpy(&d, &b, sizeof(d));
  return d;
}

}  // namespace gcg

using namespace gcg;

// ---- COO -> CSR on the device (MatrixMarket ingestion, io.py:108-250) ----------------
// keys row * ncols + col, stable radix sort (duplicates keep their file order), one
// segment-head thread sums each run of equal keys in that order, row lengths counted and
// scanned into the row pointers.
__global__ void coo_keys_kernel(long long nnz, long long ncols, const long long* __restrict__ rows,
                                const long long* __restrict__ cols, unsigned long long* keys,
                                int* idx) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x) {
    keys[e] = (unsigned long long)rows[e] * (unsigned long long)ncols + (unsigned long long)cols[e];
    idx[e] = (int)e;
  }
}
// head[e] = 1 where a new key starts (sorted keys)
__global__ void coo_heads_kernel(long long nnz, const unsigned long long* __restrict__ keys,
                                 int* head) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x)
    head[e] = (e == 0 || keys[e] != keys[e - 1]) ? 1 : 0;
}
// seg = inclusive scan of head (1-based unique index); each head sums its run in order
__global__ void coo_reduce_kernel(long long nnz, long long ncols,
                                  const unsigned long long* __restrict__ keys,
                                  const int* __restrict__ idx, const int* __restrict__ seg,
                                  const double* __restrict__ vals, int* row_len, int* colidx,
                                  double* val) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x) {
    if (e > 0 && keys[e] == keys[e - 1]) continue;
    const unsigned long long k = keys[e];
    double s = vals[idx[e]];
    for (long long f = e + 1; f < nnz && keys[f] == k; ++f) s += vals[idx[f]];
    const int u = seg[e] - 1;
    colidx[u] = (int)(k % (unsigned long long)ncols);
    val[u] = s;
    atomicAdd(row_len + (k / (unsigned long long)ncols), 1);
  }
}

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

int gcg_stencil_slab(void* ctx, int64_t n0, int64_t n1, int64_t n2, int32_t noff,
                     const int32_t* offs, const double* w, const double* const* wrow, int64_t row0,
                     int64_t row1, int32_t* rowptr, int32_t* colidx, double* val,
                     int64_t* nnz_out) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !offs || !rowptr || (!w && !wrow)) return GCG_ERR_ARG;
  StencilDesc s;
  GCG_TRY(fill_desc(s, n0, n1, n2, noff, offs, w, wrow));
  const long long n = (long long)n0 * n1 * n2;
  if (row0 < 0 || row1 > n || row0 >= row1 || n >= (1LL << 31)) return GCG_ERR_ARG;
  const long long plane = n0 > 1 ? (long long)n1 * n2 : (long long)n2;
  SlabMap m;
  m.row0 = row0;
  m.row1 = row1;
  m.nprev = row0 > 0 ? (plane < row0 ? plane : row0) : 0;
  m.nnext = row1 < n ? (plane < n - row1 ? plane : n - row1) : 0;
  const long long nloc = row1 - row0;
  const int grid = grid_for(nloc, 256, 8, c->num_sms);
  if (!colidx) {  // pass 1: row pointers and the slab's nonzero count
    slab_count_kernel<<<grid, 256, 0, c->stream>>>(s, m, rowptr + 1);
    GCG_CHECK_LAUNCH();
    size_t tmp = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp, rowptr + 1, rowptr + 1, (int)nloc, c->stream);
    GCG_TRY(ensure(c->host_tmp, tmp + 16));
    if (cub::DeviceScan::InclusiveSum(c->host_tmp.ptr, tmp, rowptr + 1, rowptr + 1, (int)nloc,
                                      c->stream) != cudaSuccess)
      return GCG_ERR_CUDA;
    GCG_TRY(cuda_status(cudaMemsetAsync(rowptr, 0, sizeof(int32_t), c->stream)));
    g_launches += 2;
    int last = 0;
    GCG_TRY(cuda_status(cudaMemcpyAsync(&last, rowptr + nloc, sizeof(int), cudaMemcpyDeviceToHost,
                                        c->stream)));
    GCG_TRY(cuda_status(cudaStreamSynchronize(c->stream)));
    if (nnz_out) *nnz_out = last;
    return GCG_OK;
  }
  if (!val) return GCG_ERR_ARG;
  GCG_TRY(ensure(c->host_tmp, 64));
  int* bad = (int*)c->host_tmp.ptr;
  GCG_TRY(cuda_status(cudaMemsetAsync(bad, 0, sizeof(int), c->stream)));
  slab_fill_kernel<<<grid, 256, 0, c->stream>>>(s, m, rowptr, colidx, val, bad);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  int hbad = 0;
  GCG_TRY(cuda_status(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream)));
  GCG_TRY(cuda_status(cudaStreamSynchronize(c->stream)));
  if (nnz_out) *nnz_out = (int64_t)(m.nprev + m.nnext);  // ghost rows of the slab
  return hbad ? GCG_ERR_ARG : GCG_OK;
}

int gcg_csr_check(void* ctx, int64_t n, const int32_t* rowptr, const int32_t* colidx,
                  const double* val, double* out) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || n < 0 || !out || (n > 0 && (!rowptr || !colidx || !val))) return GCG_ERR_ARG;
  GCG_TRY(ensure(c->host_tmp, 64));
  double* d = (double*)c->host_tmp.ptr;
  GCG_TRY(cuda_status(cudaMemsetAsync(d, 0, 4 * sizeof(double), c->stream)));
  if (n > 0) {
    csr_check_kernel<<<grid_for(n, 256, 8, c->num_sms), 256, 0, c->stream>>>(
        n, rowptr, colidx, val, d, (unsigned long long*)(d + 2));
    ++g_launches;
    GCG_CHECK_LAUNCH();
  }
  unsigned long long h[4];
  GCG_TRY(cuda_status(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, c->stream)));
  GCG_TRY(cuda_status(cudaStreamSynchronize(c->stream)));
  out[0] = __longlong_as_double_host(h[0]);
  out[1] = __longlong_as_double_host(h[1]);
  out[2] = (double)h[2];
  out[3] = (double)h[3];
  return GCG_OK;
}

int gcg_fill_normal(void* ctx, int64_t n, int64_t k, int64_t row0, uint64_t seed, double* X,
                    int64_t ldx) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || n < 0 || k < 0 || row0 < 0 || ldx < k || (n > 0 && k > 0 && !X)) return GCG_ERR_ARG;
  if (n == 0 || k == 0) return GCG_OK;
  const long long tot = n * ((k + 1) / 2);
  fill_normal_kernel<<<grid_for(tot, 256, 8, c->num_sms), 256, 0, c->stream>>>(n, (int)k, row0,
                                                                               seed, X, ldx);
  ++g_launches;
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


// COO (device, 0-based int64 row / col, any order, duplicates allowed) -> CSR with sorted
// column indices and duplicates summed (in input order).  rowptr: n + 1 entries;
// colidx / val: capacity nnz (the first *nnz_out used).
int gcg_coo_to_csr(void* ctx, int64_t n, int64_t ncols, int64_t nnz, const int64_t* rows,
                   const int64_t* cols, const double* vals, int32_t* rowptr, int32_t* colidx,
                   double* val, int64_t* nnz_out) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || n < 0 || ncols <= 0 || nnz < 0 || !rowptr || !nnz_out || nnz >= (1LL << 31) ||
      n >= (1LL << 31))
    return GCG_ERR_ARG;
  if (nnz > 0 && (!rows || !cols || !vals || !colidx || !val)) return GCG_ERR_ARG;
  GCG_TRY(cuda_status(cudaMemsetAsync(rowptr, 0, sizeof(int32_t) * (size_t)(n + 1), c->stream)));
  if (nnz == 0) {
    *nnz_out = 0;
    return cuda_status(cudaStreamSynchronize(c->stream));
  }
  const int N = (int)nnz;
  // workspace: keys[2] (u64), idx[2] (int), head, seg (int) | cub temp
  const size_t kb = sizeof(unsigned long long) * (size_t)N, ib = sizeof(int) * (size_t)N;
  size_t t_sort = 0, t_scan = 0, t_scan2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t_sort, (unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (int*)nullptr, (int*)nullptr, N,
                                  0, 64, c->stream);
  cub::DeviceScan::InclusiveSum(nullptr, t_scan, (int*)nullptr, (int*)nullptr, N, c->stream);
  cub::DeviceScan::InclusiveSum(nullptr, t_scan2, (int*)nullptr, (int*)nullptr, (int)n, c->stream);
  size_t tmp = t_sort > t_scan ? t_sort : t_scan;
  if (t_scan2 > tmp) tmp = t_scan2;
  GCG_TRY(ensure(c->host_tmp2, 2 * kb + 4 * ib + tmp + 256));
  char* base = (char*)c->host_tmp2.ptr;
  unsigned long long* k0 = (unsigned long long*)base;
  unsigned long long* k1 = k0 + N;
  int* i0 = (int*)(k1 + N);
  int* i1 = i0 + N;
  int* head = i1 + N;
  int* seg = head + N;
  void* temp = (void*)(((uintptr_t)(seg + N) + 255) & ~(uintptr_t)255);
  const int grid = grid_for(nnz, 256, 8, c->num_sms);
  coo_keys_kernel<<<grid, 256, 0, c->stream>>>(nnz, ncols, (const long long*)rows,
                                               (const long long*)cols, k0, i0);
  GCG_CHECK_LAUNCH();
  int bits = 1;
  while (bits < 64 && ((unsigned long long)n * (unsigned long long)ncols) >> bits) ++bits;
  size_t ts = t_sort;
  if (cub::DeviceRadixSort::SortPairs(temp, ts, k0, k1, i0, i1, N, 0, bits, c->stream) !=
      cudaSuccess)
    return GCG_ERR_CUDA;
  coo_heads_kernel<<<grid, 256, 0, c->stream>>>(nnz, k1, head);
  GCG_CHECK_LAUNCH();
  size_t tsc = t_scan;
  if (cub::DeviceScan::InclusiveSum(temp, tsc, head, seg, N, c->stream) != cudaSuccess)
    return GCG_ERR_CUDA;
  coo_reduce_kernel<<<grid, 256, 0, c->stream>>>(nnz, ncols, k1, i1, seg, vals, rowptr + 1, colidx,
                                                 val);
  GCG_CHECK_LAUNCH();
  size_t tsc2 = t_scan2;
  if (n > 0 && cub::DeviceScan::InclusiveSum(temp, tsc2, rowptr + 1, rowptr + 1, (int)n,
                                             c->stream) != cudaSuccess)
    return GCG_ERR_CUDA;
  int uniq = 0;
  GCG_TRY(cuda_status(cudaMemcpyAsync(&uniq, seg + N - 1, sizeof(int), cudaMemcpyDeviceToHost,
                                      c->stream)));
  GCG_TRY(cuda_status(cudaStreamSynchronize(c->stream)));
  *nnz_out = uniq;
  g_launches += 5;
  return GCG_OK;
}

}  // extern "C"
