// Context, statistics and the fixed-order reduction kernels (see common.cuh).
#include "common.cuh"
#include "comm.cuh"

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <set>
#include <string>

namespace cpb {

thread_local cudaStream_t tl_stream = nullptr;

bool first_on_device(const char* tag) {
  static std::mutex mu;
  static std::set<std::pair<int, std::string>> seen;
  int dev = 0;
  CPB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  return seen.emplace(dev, tag).second;
}

bool trace_on() {
  static const bool on = std::getenv("CPB_TRACE") != nullptr;
  return on;
}

void trace(const char* tag) {
  if (!trace_on()) return;
  static auto last = std::chrono::steady_clock::now();
  const auto now = std::chrono::steady_clock::now();
  std::fprintf(stderr, "[cpb] %s +%.3f ms\n", tag, std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}

namespace {
struct Block {
  void* p;
  cudaEvent_t ready;  // recorded on the freeing stream (null: no pending work known)
};
std::mutex g_cache_mu;
std::map<std::pair<int, size_t>, std::vector<Block>>& cache() {
  static auto* m = new std::map<std::pair<int, size_t>, std::vector<Block>>();  // outlives static dtors
  return *m;
}
}  // namespace

void* dev_alloc(size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  Block b{nullptr, nullptr};
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto& m = cache();
    auto it = m.lower_bound({dev, bytes});
    if (it != m.end() && it->first.first == dev && it->first.second <= 2 * bytes && !it->second.empty()) {
      b = it->second.back();
      it->second.pop_back();
      if (it->second.empty()) m.erase(it);
    }
  }
  if (b.p) {
    if (b.ready) {
      if (tl_stream)
        cudaStreamWaitEvent(tl_stream, b.ready, 0);
      else
        cudaEventSynchronize(b.ready);
      cudaEventDestroy(b.ready);
    }
    return b.p;
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {  // out of memory: return the cache to CUDA and retry once
    cudaGetLastError();
    dev_cache_trim();
    CPB_CUDA(cudaMalloc(&p, bytes));
  }
  return p;
}
void dev_free(void* p, size_t bytes) {
  if (!p) return;
  int dev = 0;
  cudaGetDevice(&dev);
  Block b{p, nullptr};
  if (tl_stream && cudaEventCreateWithFlags(&b.ready, cudaEventDisableTiming) == cudaSuccess) {
    if (cudaEventRecord(b.ready, tl_stream) != cudaSuccess) {
      cudaGetLastError();
      cudaEventDestroy(b.ready);
      b.ready = nullptr;
    }
  } else {
    cudaGetLastError();
    b.ready = nullptr;
  }
  std::lock_guard<std::mutex> lk(g_cache_mu);
  cache()[{dev, bytes}].push_back(b);
}
void dev_cache_trim() {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& kv : cache()) {
    cudaSetDevice(kv.first.first);
    for (auto& b : kv.second) {
      if (b.ready) {
        cudaEventSynchronize(b.ready);
        cudaEventDestroy(b.ready);
      }
      cudaFree(b.p);
    }
  }
  cache().clear();
  cudaSetDevice(cur);
}

unsigned long long g_launches = 0;

Ctx::Ctx(int dev) : device(dev) {
  int count = 0;
  CPB_CUDA(cudaGetDeviceCount(&count));
  if (count == 0) runtime("no CUDA device is visible (libcluspath_b200 has no CPU fallback)");
  if (dev < 0 || dev >= count) invalid("cp_ctx_create: device index out of range");
  CPB_CUDA(cudaSetDevice(dev));
  cudaDeviceProp prop;
  CPB_CUDA(cudaGetDeviceProperties(&prop, dev));
  sm_count = prop.multiProcessorCount;
  sm_major = prop.major;
  sm_minor = prop.minor;
  if (sm_major != 10)
    runtime("libcluspath_b200 is built for sm_100a (B200); device reports sm_" + std::to_string(sm_major) +
            std::to_string(sm_minor));
  CPB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CPB_CUDA(cudaMallocHost(&hscal, kScal * sizeof(double)));
  CPB_CUDA(cudaMalloc(&dscal, kScal * sizeof(double)));
  CPB_CUDA(cudaMemset(dscal, 0, kScal * sizeof(double)));
}

Ctx::~Ctx() {
  cudaSetDevice(device);
  if (s) cudaStreamSynchronize(s);
  for (auto& p : pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : event_pool) cudaEventDestroy(e);
  if (cs) {
    cudaStreamSynchronize(cs);
    cudaStreamDestroy(cs);
  }
  if (timer_a) cudaEventDestroy(timer_a);
  if (timer_b) cudaEventDestroy(timer_b);
  ws.clear();
  if (hscal) cudaFreeHost(hscal);
  if (dscal) cudaFree(dscal);
  if (s) cudaStreamDestroy(s);
}

void Ctx::fetch(int off, int count, double* out) {
  CPB_CUDA(cudaMemcpyAsync(hscal + off, dscal + off, count * sizeof(double), cudaMemcpyDeviceToHost, s));
  CPB_CUDA(cudaStreamSynchronize(s));
  std::memcpy(out, hscal + off, count * sizeof(double));
}

cudaEvent_t Ctx::get_event() {
  if (!event_pool.empty()) {
    cudaEvent_t e = event_pool.back();
    event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CPB_CUDA(cudaEventCreate(&e));
  return e;
}

Ctx::Timer::Timer(Ctx* c_, const char* n, double by) : c(c_), name(n), bytes(by) {
  if (!c->stats_on) return;
  a = c->get_event();
  b = c->get_event();
  CPB_CUDA(cudaEventRecord(a, c->s));
}
Ctx::Timer::~Timer() {
  if (!a) return;
  cudaEventRecord(b, c->s);
  c->pending.push_back({name, a, b, bytes});
  if (c->pending.size() > 4096) c->drain_stats();
}

void Ctx::discard_pending(const std::string& name, int count) {
  for (int k = static_cast<int>(pending.size()) - 1; k >= 0 && count > 0; --k) {
    if (pending[k].name != name) continue;
    event_pool.push_back(pending[k].a);
    event_pool.push_back(pending[k].b);
    pending.erase(pending.begin() + k);
    --count;
  }
}

void Ctx::drain_stats() {
  for (auto& p : pending) {
    cudaEventSynchronize(p.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    KStat& k = stats[p.name];
    k.launches += 1;
    k.ms += ms;
    k.bytes += p.bytes;
    event_pool.push_back(p.a);
    event_pool.push_back(p.b);
  }
  pending.clear();
}

// ---- reductions --------------------------------------------------------------
namespace {
constexpr int kRedThreads = 1024;

__global__ void k_reduce_sum(const double* __restrict__ src, int64_t count, double* dst) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t k = threadIdx.x; k < count; k += blockDim.x) acc = __dadd_rn(acc, src[k]);
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) *dst = acc;
}
__global__ void k_reduce_max(const double* __restrict__ src, int64_t count, double* dst) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t k = threadIdx.x; k < count; k += blockDim.x) acc = fmax(acc, src[k]);
  acc = block_max(acc, sh);
  if (threadIdx.x == 0) *dst = acc;
}
__global__ void k_reduce_cols(const double* __restrict__ src, int64_t rows, int64_t cols, double* dst) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= cols) return;
  double acc = 0.0;
  for (int64_t r = 0; r < rows; ++r) acc = __dadd_rn(acc, src[r * cols + c]);
  dst[c] = acc;
}
__global__ void k_fill(double* p, int64_t count, double v) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < count;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[k] = v;
}
}  // namespace

void reduce_sum(Ctx& c, const double* src, int64_t count, double* dst) {
  k_reduce_sum<<<1, kRedThreads, 0, c.s>>>(src, count, dst);
  CPB_LAUNCH_CHECK();
}
void reduce_max(Ctx& c, const double* src, int64_t count, double* dst) {
  k_reduce_max<<<1, kRedThreads, 0, c.s>>>(src, count, dst);
  CPB_LAUNCH_CHECK();
}
void reduce_cols(Ctx& c, const double* src, int64_t rows, int64_t cols, double* dst) {
  if (cols <= 0) return;
  k_reduce_cols<<<cdiv(cols, 256), 256, 0, c.s>>>(src, rows, cols, dst);
  CPB_LAUNCH_CHECK();
}
void fill(Ctx& c, double* p, int64_t count, double v) {
  if (count <= 0) return;
  const int grid = std::min(cdiv(count, 256), c.sm_count * 8);
  k_fill<<<grid, 256, 0, c.s>>>(p, count, v);
  CPB_LAUNCH_CHECK();
}
void h2d(Ctx& c, void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  CPB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c.s));
}
void d2h(Ctx& c, void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  CPB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c.s));
  CPB_CUDA(cudaStreamSynchronize(c.s));
}

}  // namespace cpb
