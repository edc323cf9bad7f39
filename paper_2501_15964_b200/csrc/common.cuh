// Shared host/device plumbing of libcluspath_b200: errors, device buffers,
// the per-device context (stream, workspace, pinned scalar mailbox, kernel
// statistics) and deterministic warp/block reductions.
//
// The whole library is compiled with -fmad=false so that every elementwise
// expression rounds exactly like the reference's SSE2 build (no FMA
// contraction, proj/src/CMakeLists.txt:19).  Reductions are fixed-order
// (run-to-run bitwise reproducible) but, being parallel, do not reproduce
// Eigen's sequential order; the kNN distances, which must be bitwise, use the
// exact Eigen order (graph.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "cluspath_b200.h"

namespace cpb {

// ---- errors ----------------------------------------------------------------
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void invalid(const std::string& m) { throw Error(CP_EINVAL, m); }
[[noreturn]] inline void runtime(const std::string& m) { throw Error(CP_ERUNTIME, m); }

#define CPB_CUDA(call)                                                                      \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      throw ::cpb::Error(CP_ECUDA, std::string("CUDA error ") + cudaGetErrorString(e_) +    \
                                       " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)
// Every kernel launch of the library is followed by exactly one
// CPB_LAUNCH_CHECK, which also counts it (cp_launch_count; CUB's internal
// sort/scan kernels are not counted).
extern unsigned long long g_launches;
#define CPB_LAUNCH_CHECK()              \
  do {                                  \
    ++::cpb::g_launches;                \
    CPB_CUDA(cudaGetLastError());       \
  } while (0)

// ---- device buffers --------------------------------------------------------
// Caching device allocator: freed blocks are kept in a per-device, size-keyed
// free list and handed back to later requests of up to 2x smaller size, so
// rebuilding a graph or re-growing a workspace never calls cudaFree (which
// synchronises the device) or cudaMalloc in steady state (C3 path steps
// varied 2.5-3.7 s with cudaFree in the graph rebuild, 2.49 s without).
// Stream ordering: a free records an event on the freeing thread's current
// library stream (tl_stream, set by the C-ABI for the call's context); a
// reuse makes its own stream wait on that event, so a block is never touched
// before the work of another context that used it has finished.
extern thread_local cudaStream_t tl_stream;
struct StreamScope {  // sets tl_stream for the current thread
  cudaStream_t prev;
  explicit StreamScope(cudaStream_t s) : prev(tl_stream) { tl_stream = s; }
  ~StreamScope() { tl_stream = prev; }
};
void* dev_alloc(size_t bytes);
void dev_free(void* p, size_t bytes);
void dev_cache_trim();

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  explicit DBuf(size_t count) { resize(count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p, n = o.n;
      o.p = nullptr, o.n = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p) dev_free(p, n * sizeof(T));
    p = nullptr, n = 0;
  }
  // Grow-only (contents are not preserved on growth).
  void resize(size_t count) {
    if (count <= n && p) return;
    release();
    if (count == 0) count = 1;
    p = static_cast<T*>(dev_alloc(count * sizeof(T)));
    n = count;
  }
  T* get() const { return p; }
};

inline void swap_buf(DBuf<double>& a, DBuf<double>& b) {
  std::swap(a.p, b.p);
  std::swap(a.n, b.n);
}

// ---- kernel statistics (CUDA events on the launching stream) --------------
struct KStat {
  int64_t launches = 0;
  double ms = 0.0, bytes = 0.0;
};

struct Ctx {
  int device = 0;
  int sm_count = 148;
  int sm_major = 0, sm_minor = 0;
  cudaStream_t s = nullptr;
  double* hscal = nullptr;   // pinned scalar mailbox (host)
  double* dscal = nullptr;   // device scalar area
  static constexpr int kScal = 4096;
  std::map<std::string, DBuf<char>> ws;  // named workspace buffers
  bool stats_on = false;
  std::map<std::string, KStat> stats;
  struct Pending {
    std::string name;
    cudaEvent_t a, b;
    double bytes;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  cudaEvent_t timer_a = nullptr, timer_b = nullptr;  // cp_timer_start / cp_timer_stop
  std::map<std::string, int> cg_hint;                 // last PCG iteration count per operator
  std::vector<cp_trace_row> trace;                    // Solution::trace of the current / last solve
  struct KnnInfo {
    int64_t overflow_rows;  // rows re-done by the exact FP64 tile kernel
    double worst_ratio;     // max |d2~ - d2| / delta_i over re-checked candidates
    int segments;           // column segments of the tensor-core pass (0 = exact path only)
    int tensor_cores;       // 1 when the tcgen05 candidate pass ran
  } knn_last{0, 0.0, 0, 0};
  int64_t knn_band_rows = 0;  // rows settled by the tensor-core threshold (band) pass
  // Multi-GPU: the NCCL communicator (comm.cuh) and, while the partitioned PCG
  // runs, the node rows [own_v0, own_v1) this rank's Hessian applies cover
  // (own_v1 < 0: every node).
  std::unique_ptr<struct Comm> comm;
  int64_t own_v0 = 0, own_v1 = -1;
  cudaStream_t cs = nullptr;                          // device->host copy stream (lazily created)
  cudaStream_t copy_stream() {
    if (!cs) CPB_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    return cs;
  }

  explicit Ctx(int dev);
  ~Ctx();

  template <class T>
  T* buf(const std::string& name, size_t count) {
    auto& b = ws[name];
    b.resize(count * sizeof(T));
    return reinterpret_cast<T*>(b.p);
  }
  // Copy `count` device scalars from dscal[off..] to the host and wait.
  void fetch(int off, int count, double* out);
  void sync() { CPB_CUDA(cudaStreamSynchronize(s)); }
  // Timed-launch bracket for the hot kernels (no-op when stats are off).
  struct Timer {
    Ctx* c;
    cudaEvent_t a = nullptr, b = nullptr;
    std::string name;
    double bytes;
    Timer(Ctx* c_, const char* n, double by);
    ~Timer();
  };
  cudaEvent_t get_event();
  void drain_stats();
  // Drop the last `count` pending timings named `name` (launches that no-oped).
  void discard_pending(const std::string& name, int count);
};

// ---- launch geometry -------------------------------------------------------
inline int cdiv(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

// ---- device reductions (fixed order) ---------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// Block-wide sum in a fixed tree over the linear thread id (1-D or 2-D
// blocks, size a multiple of 32); every thread receives the result.
// `sh` must hold >= 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* sh) {
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5, nw = (blockDim.x * blockDim.y + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = (tid < nw) ? sh[tid] : 0.0;
  if (wid == 0) t = warp_sum(t);
  if (tid == 0) sh[0] = t;
  __syncthreads();
  const double r = sh[0];
  __syncthreads();
  return r;
}
__device__ __forceinline__ double block_max(double v, double* sh) {
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5, nw = (blockDim.x * blockDim.y + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = (tid < nw) ? sh[tid] : 0.0;
  if (wid == 0) t = warp_max(t);
  if (tid == 0) sh[0] = t;
  __syncthreads();
  const double r = sh[0];
  __syncthreads();
  return r;
}

// Row groups: a row (node or edge) of length d is owned by blockDim.x <= 32
// lanes of one warp (blockDim.x a power of two); blockDim.y rows per block.
__device__ __forceinline__ unsigned group_mask() {
  const unsigned dx = blockDim.x;
  if (dx >= 32) return 0xffffffffu;
  const unsigned lin = threadIdx.y * dx + threadIdx.x;
  return ((1u << dx) - 1u) << ((lin & 31u) & ~(dx - 1u));
}
__device__ __forceinline__ double group_sum(double v, unsigned m) {
  for (int o = blockDim.x >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(m, v, o, blockDim.x);
  return v;
}
__device__ __forceinline__ double group_max(double v, unsigned m) {
  for (int o = blockDim.x >> 1; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(m, v, o, blockDim.x));
  return v;
}

// CPB_TRACE=1: host wall-clock trace lines "[cpb] <tag> +<ms since previous>"
// on stderr (diagnostics for host-side stalls; off by default).
void trace(const char* tag);
bool trace_on();

// True the first time `tag` is seen for the calling thread's current device
// (kernel attributes such as the >48 KB shared-memory opt-in are per device;
// thread-safe, so in-process ranks on several devices each set their own).
bool first_on_device(const char* tag);

// Host helpers implemented in common.cu.
// Deterministic sum of `count` doubles at `src` into dst[0] (one block).
void reduce_sum(Ctx& c, const double* src, int64_t count, double* dst);
void reduce_max(Ctx& c, const double* src, int64_t count, double* dst);
// Column sums of a (rows x cols) row-major block of partials: dst[c] = sum_r src[r*cols+c].
void reduce_cols(Ctx& c, const double* src, int64_t rows, int64_t cols, double* dst);
void fill(Ctx& c, double* p, int64_t count, double v);
void h2d(Ctx& c, void* dst, const void* src, size_t bytes);
void d2h(Ctx& c, void* dst, const void* src, size_t bytes);

}  // namespace cpb
