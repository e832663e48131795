// Shared definitions for the gcgb200 CUDA library (sm_100a, fp64).
//
// Layout convention (B200 design): a multivector block is
// ROW-MAJOR in HBM — element (row i, column c) lives at X[i * ld + c] — so a
// CSR row gather reads one contiguous run of k doubles per neighbour and a
// column range [c0, c0+k) of the arena is just the pointer X + c0 with the
// same ld.  Small dense matrices (projected matrix, Ritz coefficients, Gram
// blocks) are row-major too.
#pragma once

#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <stdint.h>

#include "../../include/gcgb200.h"

namespace gcg {

constexpr int kNumSMs = 148;

// Per-context scratch: grows monotonically, never shrinks during a solve.
struct Scratch {
  void* ptr = nullptr;
  size_t bytes = 0;
};

// Live per-kernel-class timing (CUDA events on the ctx stream around each
// launch) + algorithmic byte counts, for bench.py's roofline.  Off by default.
enum ProfClass { PROF_SPMM = 0, PROF_GRAM, PROF_LINCOMB, PROF_CG_UPDATE, PROF_CG_XOUT,
                 PROF_CG_SWEEP, PROF_NCLASS };

struct Prof {
  bool on = false;
  cudaEvent_t* ev = nullptr;   // pool of events, pairs (start, stop)
  int* cls = nullptr;          // class of each pair
  double* bytes = nullptr;     // algorithmic bytes of each pair
  int* d_skipped = nullptr;    // device flags: the launch was a CG early-exit no-op
  int cap = 0;                 // pairs
  int used = 0;
  int stride = 1;              // time every stride-th launch of each class
  long long seen[PROF_NCLASS] = {0};
};

struct Ctx {
  Prof prof;
  cudaStream_t stream = nullptr;
  cusolverDnHandle_t solver = nullptr;
  int num_sms = kNumSMs;
  int device = 0;
  long long l2_bytes = 0;
  // generic workspaces (slots are owned by one op at a time; ops on one ctx
  // are stream-ordered so reuse across ops is safe)
  Scratch partials;   // per-CTA partial sums for deterministic reductions
  Scratch eigwork;    // cuSOLVER work + info
  Scratch cg;         // block-CG vectors r, p, q and per-column state
  Scratch cgpad;      // block CG on a column count padded to a multiple of 4 (rhs, iterate)
  Scratch host_tmp;   // device staging for the host-buffer (reference FFI) entry points
  Scratch host_tmp2;
  Scratch host_tmp3;
  Scratch host_tmp4;
  Scratch dense;      // small dense temporaries (eigensolver staging)
  Scratch orth;       // native orthogonalisation: status, Gram, SVQB coefficients, B*block
  Scratch buildp;     // native momentum block (gcg_build_p)
  double* pinned = nullptr;  // pinned host slots for decision reads
  // host-mapped (zero-copy) decision slots: the status kernels store straight into
  // host memory, so a decision read is one stream synchronisation — no copy launch
  double* mapped = nullptr;      // host view
  double* mapped_dev = nullptr;  // device view of the same 64 doubles
  int* sync_flag = nullptr;
  cudaEvent_t ev = nullptr;
  // speculative passes (orth.cu): while `skip` is set, the Gram / LinComb / column-dot
  // launchers pass it to their kernels, which return at once when *skip != 0 — a pass
  // enqueued before the host has read the previous pass's decision is a device no-op
  // when that decision was "stop"
  const int* skip = nullptr;
  int* spec = nullptr;  // device ring of per-pass stop flags (kSpecRing ints)
  unsigned spec_seq = 0;
  cudaEvent_t spec_ev[2] = {nullptr, nullptr};
  // passes the last loop at each call site ran (orth.cu): a pass is speculated only
  // where the previous loop there went on past it
  int spec_hist[8] = {2, 2, 2, 2, 2, 2, 2, 2};
};
constexpr int kSpecRing = 64;

// kernel side of Ctx::skip: `flag` is the stop flag of the previous pass (nullptr: run),
// `prof` the profiling slot's no-op marker (launches that did nothing carry no bytes)
struct Skip {
  const int* flag;
  int* prof;
};
__device__ __forceinline__ bool skip_now(const Skip& s) {
  if (s.flag && *s.flag) {
    if (s.prof && threadIdx.x == 0) *s.prof = 1;
    return true;
  }
  return false;
}

int ensure(Scratch& s, size_t bytes);
// allocates the mapped decision slots on first use
int ensure_mapped(Ctx* c);

// cudaFuncSetAttribute / the occupancy query are host API calls of several
// microseconds; the launchers call these cached forms instead (keyed by kernel).
void kernel_smem(const void* kern, size_t bytes);
int kernel_occupancy(const void* kern, int threads, size_t smem);

inline int cuda_status(cudaError_t e) {
  return e == cudaSuccess ? GCG_OK : GCG_ERR_CUDA;
}

#define GCG_CHECK_LAUNCH()                                  \
  do {                                                      \
    cudaError_t _e = cudaGetLastError();                    \
    if (_e != cudaSuccess) return GCG_ERR_CUDA;             \
  } while (0)

#define GCG_TRY(x)                                          \
  do {                                                      \
    int _s = (x);                                           \
    if (_s != GCG_OK) return _s;                            \
  } while (0)

// ---------------------------------------------------------------------------
// warp / block reduction helpers

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Grid sizing: a multiple of the SM count, capped by the work available.
inline int grid_for(long long work_items, int items_per_cta, int ctas_per_sm, int num_sms) {
  long long need = (work_items + items_per_cta - 1) / items_per_cta;
  long long cap = (long long)num_sms * ctas_per_sm;
  if (need < 1) need = 1;
  return (int)(need < cap ? need : cap);
}

// Programmatic dependent launch (sm_90+): a kernel launched with pdl_launch may be
// scheduled while its predecessor on the stream drains; it must call pdl_wait()
// before touching anything the predecessor writes (the wait returns once the
// predecessor grid has completed and its memory is visible; a no-op for ordinary
// launches).  pdl_trigger() lets the successor start launching early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args... args) {
  if (!pdl_enabled()) {
    kern<<<grid, block, smem, stream>>>(args...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// profiling: prof_start returns a pair slot (or -1 when off), prof_stop closes it
int prof_start(Ctx* c, int cls, double bytes);
void prof_stop(Ctx* c, int slot);
// device flag slot of a prof_start pair (nullptr when profiling is off)
int* prof_skip_slot(Ctx* c, int slot);
inline Skip skip_of(Ctx* c, int prof_slot) {
  return Skip{c->skip, c->skip ? prof_skip_slot(c, prof_slot) : nullptr};
}

// internal launchers shared between translation units
int reduce_partials(Ctx* c, const double* partials, int nparts, int k, double* out,
                    int out_stride, int mode);
int dense_syev_jacobi(Ctx* c, int m, const double* A, long long lda, double* w, double* V,
                      long long ldv);
int dense_syev_cusolver(Ctx* c, int m, const double* A, long long lda, double* w, double* V,
                        long long ldv);
int dense_syev_range(Ctx* c, int m, const double* A, long long lda, int il, int iu, double* w,
                     double* V, long long ldv);

}  // namespace gcg
