// The extern "C" boundary (include/cluspath_b200.h).  Every entry point maps
// host buffers to device state, runs the sm_100a kernels and maps exceptions
// to return codes (CP_EINVAL = std::invalid_argument, CP_ERUNTIME =
// std::runtime_error) with a thread-local message.  There is no CPU fallback:
// without a CUDA device cp_ctx_create fails with CP_ERUNTIME.
#include <sys/mman.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <random>
#include <string>
#include <vector>

#include "comm.cuh"
#include "gather.cuh"
#include "linalg.cuh"
#include "solve.cuh"

struct cp_ctx {
  std::unique_ptr<cpb::Ctx> c;
};
struct cp_data {
  cpb::Data d;
  cudaStream_t s = nullptr;  // stream of the creating context (stream-ordered frees)
  int device = 0;
};
struct cp_graph {
  std::unique_ptr<cpb::Graph> g;
  cudaStream_t s = nullptr;
  int device = 0;
};
struct cp_linop {
  cpb::LinOp op;
  int device = 0;
};
struct cp_factor {
  cpb::LinOp M;    // I + rho L (CSR rows)
  cpb::LinOp pre;  // Jacobi diagonal of M
  double rho = 0.0;
  int device = 0;
};

namespace {
thread_local std::string g_err;

// page-locked blocks made by mmap + cudaHostRegister: user pointer -> (mapping base, length)
std::map<void*, std::pair<void*, size_t>>& host_blocks() {
  static std::map<void*, std::pair<void*, size_t>> m;
  return m;
}
std::mutex& host_blocks_mu() {
  static std::mutex mu;
  return mu;
}

template <class F>
int guard(cp_ctx* ctx, F f) {
  try {
    if (ctx && ctx->c) cudaSetDevice(ctx->c->device);
    cpb::StreamScope scope(ctx && ctx->c ? ctx->c->s : nullptr);
    f();
    return CP_OK;
  } catch (const cpb::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return CP_EINVAL;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return CP_ERUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CP_ERUNTIME;
  }
}

void need(const void* p, const char* what) {
  if (!p) cpb::invalid(std::string(what) + " must not be null");
}
void check_q(int q) {
  if (q != 0 && q != 1 && q != 2)
    cpb::invalid("penalty norm exponent must be 1, 2 or 0 (infinity), got " + std::to_string(q));
}

double* upload(cpb::Ctx& c, const char* name, const double* h, int64_t count) {
  double* d = c.buf<double>(name, count + 1);
  cpb::h2d(c, d, h, count * sizeof(double));
  return d;
}

__global__ void k_finite(const double* a, int64_t m, int* bad) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < m;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (!isfinite(a[p])) atomicOr(bad, 1);
}

// ProblemInstance validation (objective.cpp:26-33)
cpb::Prob make_prob(cp_ctx* ctx, const cp_data* A, const cp_graph* g, double gamma, int q) {
  need(A, "data");
  need(g, "graph");
  check_q(q);
  if (A->d.n != g->g->n)
    cpb::invalid("instance: graph has " + std::to_string(g->g->n) + " nodes for " + std::to_string(A->d.n) +
                 " samples");
  if (!(gamma >= 0.0) || !std::isfinite(gamma)) cpb::invalid("instance: gamma must be finite and >= 0");
  cpb::Prob P;
  P.c = ctx->c.get();
  P.A = const_cast<cpb::Data*>(&A->d);
  P.g = g->g.get();
  P.gamma = gamma;
  P.q = q;
  P.rad = P.c->buf<double>("api.rad", g->g->E + 1);
  cpb::make_radii(*P.c, *P.g, gamma, P.rad);
  return P;
}

}  // namespace

extern "C" {

const char* cp_last_error(void) { return g_err.c_str(); }

void cp_solver_config_default(cp_solver_config* c) {
  std::memset(c, 0, sizeof(*c));
  c->algorithm = 2;
  c->epsilon = 1e-6;
  c->kkt_factor = 10.0;
  c->max_iter = 0;
  c->time_limit = 0.0;
  c->admm_rho = 1.0;
  c->ama_step_safety = 0.99;
  c->ssnal_sigma0 = 1.0;
  c->armijo_mu = 1e-4;
  c->backtrack_beta = 0.5;
  c->ssnal_newton_max = 50;
  c->pcg_max_iter = 500;
}
void cp_path_options_default(cp_path_options* o) {
  o->warm_start = 1;
  o->require_connected = 0;
  o->fuse_tol = 1e-3;
}

int cp_ctx_create(int device, cp_ctx** out) {
  return guard(nullptr, [&] {
    need(out, "out");
    auto* c = new cp_ctx;
    try {
      c->c = std::make_unique<cpb::Ctx>(device);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}
void cp_ctx_destroy(cp_ctx* ctx) {
  if (!ctx) return;
  try {
    delete ctx;
  } catch (...) {
  }
}
int cp_ctx_synchronize(cp_ctx* ctx) {
  return guard(ctx, [&] { ctx->c->sync(); });
}
int cp_device_info(cp_ctx* ctx, int* sm_major, int* sm_minor, int* sm_count, int* built_arch) {
  return guard(ctx, [&] {
    if (sm_major) *sm_major = ctx->c->sm_major;
    if (sm_minor) *sm_minor = ctx->c->sm_minor;
    if (sm_count) *sm_count = ctx->c->sm_count;
    if (built_arch) *built_arch = 100;
  });
}
int cp_knn_info(cp_ctx* ctx, int* tensor_cores, int* segments, int64_t* band_rows, int64_t* exact_rows,
                double* worst_ratio) {
  return guard(ctx, [&] {
    const auto& k = ctx->c->knn_last;
    if (tensor_cores) *tensor_cores = k.tensor_cores;
    if (segments) *segments = k.segments;
    if (band_rows) *band_rows = ctx->c->knn_band_rows;
    if (exact_rows) *exact_rows = k.overflow_rows;
    if (worst_ratio) *worst_ratio = k.worst_ratio;
  });
}
unsigned long long cp_launch_count(void) { return cpb::g_launches; }

int cp_timer_start(cp_ctx* ctx) {
  return guard(ctx, [&] {
    cpb::Ctx& c = *ctx->c;
    c.timer_a = c.timer_a ? c.timer_a : c.get_event();
    c.timer_b = c.timer_b ? c.timer_b : c.get_event();
    CPB_CUDA(cudaEventRecord(c.timer_a, c.s));
  });
}
int cp_timer_stop(cp_ctx* ctx, double* ms) {
  return guard(ctx, [&] {
    cpb::Ctx& c = *ctx->c;
    if (!c.timer_a) cpb::invalid("cp_timer_stop without cp_timer_start");
    CPB_CUDA(cudaEventRecord(c.timer_b, c.s));
    CPB_CUDA(cudaEventSynchronize(c.timer_b));
    float f = 0.f;
    CPB_CUDA(cudaEventElapsedTime(&f, c.timer_a, c.timer_b));
    if (ms) *ms = f;
  });
}
int cp_flush_l2(cp_ctx* ctx) {
  return guard(ctx, [&] {
    cpb::Ctx& c = *ctx->c;
    const size_t bytes = size_t(512) << 20;  // 4x the 126 MB L2
    char* p = c.buf<char>("api.flush", bytes);
    CPB_CUDA(cudaMemsetAsync(p, 1, bytes, c.s));
    c.sync();
  });
}

// Large blocks (the path's output pool: 89 GB at C3) are page-locked from transparent huge
// pages: anonymous mmap aligned to 2 MB, MADV_HUGEPAGE, first touch by parallel threads, then
// cudaHostRegister (portable, mapped).  Measured on the B200 box: 48 GB in 3.8 s against
// 19.9 s for cudaHostAlloc (tools/pin_probe.py), which is most of a cold run_path.
int cp_host_alloc(uint64_t bytes, void** out) {
  return guard(nullptr, [&] {
    need(out, "out");
    *out = nullptr;
    if (bytes < (uint64_t(64) << 20)) {
      CPB_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable | cudaHostAllocMapped));
      return;
    }
    const size_t huge = size_t(2) << 20;
    const size_t len = static_cast<size_t>(bytes) + huge;
    void* base = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (base == MAP_FAILED) throw std::bad_alloc();
    char* p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(base) + huge - 1) & ~(uintptr_t(huge) - 1));
    madvise(p, static_cast<size_t>(bytes), MADV_HUGEPAGE);
    const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    const size_t chunk = (static_cast<size_t>(bytes) / nt + huge - 1) / huge * huge;
    for (unsigned k = 0; k < nt; ++k) {
      const size_t a = k * chunk;
      if (a >= bytes) break;
      const size_t b = std::min(static_cast<size_t>(bytes), a + chunk);
      pool.emplace_back([p, a, b] { std::memset(p + a, 0, b - a); });
    }
    for (auto& t : pool) t.join();
    const cudaError_t e = cudaHostRegister(p, static_cast<size_t>(bytes), cudaHostRegisterPortable | cudaHostRegisterMapped);
    if (e != cudaSuccess) {
      munmap(base, len);
      CPB_CUDA(e);
    }
    {
      std::lock_guard<std::mutex> lk(host_blocks_mu());
      host_blocks()[p] = {base, len};
    }
    *out = p;
  });
}
void cp_host_free(void* p) {
  if (!p) return;
  std::pair<void*, size_t> blk{nullptr, 0};
  {
    std::lock_guard<std::mutex> lk(host_blocks_mu());
    auto it = host_blocks().find(p);
    if (it != host_blocks().end()) {
      blk = it->second;
      host_blocks().erase(it);
    }
  }
  if (blk.first) {
    cudaHostUnregister(p);
    munmap(blk.first, blk.second);
  } else {
    cudaFreeHost(p);
  }
}

int cp_gaussian_mixture(const double* centers, int64_t d, int64_t m, double spread, int64_t per_center, uint64_t seed,
                        double* out) {
  return guard(nullptr, [&] {
    if (m < 1) cpb::invalid("mixture needs at least one center");
    if (per_center < 1) cpb::invalid("mixture needs per_center >= 1");
    if (!(spread >= 0.0)) cpb::invalid("mixture spread must be >= 0");
    need(centers, "centers");
    need(out, "out");
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    int64_t col = 0;
    for (int64_t c = 0; c < m; ++c)
      for (int64_t s = 0; s < per_center; ++s, ++col)
        for (int64_t r = 0; r < d; ++r) out[col * d + r] = centers[c * d + r] + spread * gauss(rng);
  });
}
int cp_normals(uint64_t seed, int64_t count, double* out) {
  return guard(nullptr, [&] {
    need(out, "out");
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    for (int64_t k = 0; k < count; ++k) out[k] = gauss(rng);
  });
}

int cp_stats_enable(cp_ctx* ctx, int on) {
  return guard(ctx, [&] { ctx->c->stats_on = on != 0; });
}
int cp_stats_reset(cp_ctx* ctx) {
  return guard(ctx, [&] {
    ctx->c->sync();
    ctx->c->drain_stats();
    ctx->c->stats.clear();
  });
}
int cp_stats_get(cp_ctx* ctx, cp_kernel_stat* out, int max_entries, int* count) {
  return guard(ctx, [&] {
    ctx->c->sync();
    ctx->c->drain_stats();
    int k = 0;
    for (auto& [name, st] : ctx->c->stats) {
      if (k < max_entries && out) {
        std::memset(&out[k], 0, sizeof(cp_kernel_stat));
        std::strncpy(out[k].name, name.c_str(), sizeof(out[k].name) - 1);
        out[k].launches = st.launches;
        out[k].ms = st.ms;
        out[k].alg_bytes = st.bytes;
      }
      ++k;
    }
    if (count) *count = k;
  });
}

// ---- data ---------------------------------------------------------------------
int cp_data_create(cp_ctx* ctx, const double* A, int64_t d, int64_t n, cp_data** out) {
  return guard(ctx, [&] {
    need(out, "out");
    if (d < 1 || n < 1) cpb::invalid("data matrix must have at least one feature and one sample");
    need(A, "A");
    cpb::Ctx& c = *ctx->c;
    auto p = std::make_unique<cp_data>();
    p->s = ctx->c->s;
    p->device = ctx->c->device;
    p->d.d = d;
    p->d.n = n;
    p->d.A.resize(d * n);
    cpb::h2d(c, p->d.A.p, A, d * n * sizeof(double));
    int* bad = c.buf<int>("api.bad", 1);
    CPB_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), c.s));
    k_finite<<<std::max(1, std::min(cpb::cdiv(d * n, 256), c.sm_count * 4)), 256, 0, c.s>>>(p->d.A.p, d * n, bad);
    CPB_LAUNCH_CHECK();
    int h = 0;
    cpb::d2h(c, &h, bad, sizeof(int));
    if (h) cpb::invalid("data matrix contains non-finite entries");
    *out = p.release();
  });
}
void cp_data_destroy(cp_data* data) {
  if (!data) return;
  cudaSetDevice(data->device);
  cpb::StreamScope scope(data->s);
  delete data;
}

// ---- graph --------------------------------------------------------------------
int cp_knn_graph(cp_ctx* ctx, const cp_data* data, int64_t k, double phi, cp_graph** out) {
  return guard(ctx, [&] {
    need(data, "data");
    need(out, "out");
    auto g = std::make_unique<cp_graph>();
    g->s = ctx->c->s;
    g->device = ctx->c->device;
    g->g = cpb::knn_graph(*ctx->c, data->d, k, phi);
    *out = g.release();
  });
}
int cp_graph_laplacian(cp_ctx* ctx, const cp_graph* g, int64_t* colptr, int64_t* rowidx, double* values,
                       int64_t* nnz) {
  return guard(ctx, [&] {
    need(g, "graph");
    const int64_t z = cpb::laplacian_csc(*ctx->c, *g->g, colptr, rowidx, values);
    if (nnz) *nnz = z;
  });
}
int cp_knn_rows(cp_ctx* ctx, const cp_data* data, int64_t k, int64_t r0, int64_t r1, double* kd_dev,
                int32_t* kj_dev) {
  return guard(ctx, [&] {
    need(data, "data");
    need(kd_dev, "kd");
    need(kj_dev, "kj");
    cpb::knn_validate(data->d, k, 0.0);
    cpb::knn_rows_dev(*ctx->c, data->d, k, r0, r1, kd_dev, kj_dev);
    ctx->c->sync();
  });
}
int cp_graph_from_knn(cp_ctx* ctx, int64_t n, int64_t k, double phi, const double* kd_dev, const int32_t* kj_dev,
                      cp_graph** out) {
  return guard(ctx, [&] {
    need(kd_dev, "kd");
    need(kj_dev, "kj");
    need(out, "out");
    if (n < 2) cpb::invalid("graph from kNN lists: n must be >= 2");
    auto g = std::make_unique<cp_graph>();
    g->s = ctx->c->s;
    g->device = ctx->c->device;
    g->g = cpb::graph_from_knn_dev(*ctx->c, n, k, phi, kd_dev, kj_dev);
    *out = g.release();
  });
}
int cp_nccl_unique_id(char out[128]) {
  return guard(nullptr, [&] {
    need(out, "out");
    cpb::comm_unique_id(out);
  });
}
int cp_ctx_set_comm(cp_ctx* ctx, int nranks, int rank, const char id[128]) {
  return guard(ctx, [&] {
    need(id, "id");
    cpb::comm_init(*ctx->c, nranks, rank, id);
  });
}
int cp_local_group_create(int nranks, cp_local_group** out) {
  return guard(nullptr, [&] {
    need(out, "out");
    *out = reinterpret_cast<cp_local_group*>(cpb::local_group_create(nranks));
  });
}
void cp_local_group_destroy(cp_local_group* g) { cpb::local_group_destroy(reinterpret_cast<cpb::LocalGroup*>(g)); }
int cp_ctx_set_local_comm(cp_ctx* ctx, cp_local_group* g, int rank) {
  return guard(ctx, [&] {
    need(g, "group");
    cpb::comm_init_local(*ctx->c, reinterpret_cast<cpb::LocalGroup*>(g), rank);
  });
}
int cp_shard_rows(int64_t n, int nranks, int rank, int64_t* r0, int64_t* r1) {
  if (n < 0 || nranks < 1 || rank < 0 || rank >= nranks || !r0 || !r1) {
    g_err = "cp_shard_rows: invalid arguments";
    return CP_EINVAL;
  }
  const int64_t chunk = (n + nranks - 1) / nranks;
  *r0 = std::min<int64_t>(n, chunk * rank);
  *r1 = std::min<int64_t>(n, chunk * (rank + 1));
  return CP_OK;
}
int cp_graph_from_edges(cp_ctx* ctx, int64_t n, const int64_t* i, const int64_t* j, const double* w, int64_t E,
                        cp_graph** out) {
  return guard(ctx, [&] {
    need(out, "out");
    if (E < 0) cpb::invalid("edge count must be nonnegative");
    if (E > 0) {
      need(i, "i");
      need(j, "j");
      need(w, "w");
    }
    auto g = std::make_unique<cp_graph>();
    g->s = ctx->c->s;
    g->device = ctx->c->device;
    g->g = cpb::graph_from_edges(*ctx->c, n, i, j, w, E);
    *out = g.release();
  });
}
void cp_graph_destroy(cp_graph* g) {
  if (!g) return;
  cudaSetDevice(g->device);
  cpb::StreamScope scope(g->s);
  delete g;
}
int64_t cp_graph_nodes(const cp_graph* g) { return g ? g->g->n : 0; }
int64_t cp_graph_edge_count(const cp_graph* g) { return g ? g->g->E : 0; }
int cp_graph_export(cp_ctx* ctx, const cp_graph* g, int64_t* i, int64_t* j, double* w, double* d2) {
  return guard(ctx, [&] {
    need(g, "graph");
    cpb::Ctx& c = *ctx->c;
    const int64_t E = g->g->E;
    if (E == 0) return;
    std::vector<int> tmp(static_cast<size_t>(E));
    if (i) {
      cpb::d2h(c, tmp.data(), g->g->ei.p, E * sizeof(int));
      for (int64_t l = 0; l < E; ++l) i[l] = tmp[static_cast<size_t>(l)];
    }
    if (j) {
      cpb::d2h(c, tmp.data(), g->g->ej.p, E * sizeof(int));
      for (int64_t l = 0; l < E; ++l) j[l] = tmp[static_cast<size_t>(l)];
    }
    if (w) cpb::d2h(c, w, g->g->w.p, E * sizeof(double));
    if (d2) cpb::d2h(c, d2, g->g->d2.p, E * sizeof(double));
  });
}
int cp_graph_degrees(cp_ctx* ctx, const cp_graph* g, int64_t* degree) {
  return guard(ctx, [&] {
    need(g, "graph");
    need(degree, "degree");
    const int64_t n = g->g->n;
    std::vector<int> off(static_cast<size_t>(n + 1));
    cpb::d2h(*ctx->c, off.data(), g->g->off.p, (n + 1) * sizeof(int));
    for (int64_t v = 0; v < n; ++v) degree[v] = off[static_cast<size_t>(v + 1)] - off[static_cast<size_t>(v)];
  });
}

int cp_incidence_apply(cp_ctx* ctx, const cp_graph* g, const double* X, int64_t d, int64_t n, double* out) {
  return guard(ctx, [&] {
    need(g, "graph");
    if (n != g->g->n)
      cpb::invalid("incidence apply: operand has " + std::to_string(n) + " columns, graph has " +
                   std::to_string(g->g->n) + " nodes");
    if (d < 0) cpb::invalid("incidence apply: negative row count");
    cpb::Ctx& c = *ctx->c;
    const int64_t E = g->g->E;
    if (E * d == 0) return;
    double* dx = upload(c, "api.x", X, d * n);
    double* dout = c.buf<double>("api.o", E * d);
    cpb::incidence_apply_dev(c, *g->g, dx, d, dout);
    cpb::d2h(c, out, dout, E * d * sizeof(double));
  });
}
int cp_incidence_apply_t(cp_ctx* ctx, const cp_graph* g, const double* Z, int64_t d, int64_t E, double* out) {
  return guard(ctx, [&] {
    need(g, "graph");
    if (E != g->g->E)
      cpb::invalid("incidence adjoint: operand has " + std::to_string(E) + " columns, graph has " +
                   std::to_string(g->g->E) + " edges");
    if (d < 0) cpb::invalid("incidence adjoint: negative row count");
    cpb::Ctx& c = *ctx->c;
    const int64_t n = g->g->n;
    if (n * d == 0) return;
    double* dz = upload(c, "api.z", Z, d * E);
    double* dout = c.buf<double>("api.o", n * d);
    cpb::incidence_apply_t_dev(c, *g->g, dz, d, dout);
    cpb::d2h(c, out, dout, n * d * sizeof(double));
  });
}
int cp_connected_components(cp_ctx* ctx, const cp_graph* g, int64_t* labels, int64_t* K) {
  return guard(ctx, [&] {
    need(g, "graph");
    cpb::Ctx& c = *ctx->c;
    const int64_t n = g->g->n;
    int* lab = c.buf<int>("api.lab", n + 1);
    const int64_t k = cpb::components_dev(c, *g->g, nullptr, lab);
    std::vector<int> h(static_cast<size_t>(n));
    cpb::d2h(c, h.data(), lab, n * sizeof(int));
    if (labels)
      for (int64_t v = 0; v < n; ++v) labels[v] = h[static_cast<size_t>(v)];
    if (K) *K = k;
  });
}
int cp_laplacian_lambda_max(cp_ctx* ctx, const cp_graph* g, double tol, int64_t max_iter, double* lambda) {
  return guard(ctx, [&] {
    need(g, "graph");
    need(lambda, "lambda");
    *lambda = cpb::laplacian_lambda_max(*ctx->c, *g->g, tol, max_iter);
  });
}

// ---- prox ---------------------------------------------------------------------
}  // extern "C"
namespace {
void check_thresholds(const double* t, int64_t E, const char* what) {
  for (int64_t l = 0; l < E; ++l)
    if (!(t[l] >= 0.0) || !std::isfinite(t[l]))
      cpb::invalid(std::string(what) + ": threshold must be finite and >= 0");
}
template <class F>
int columns_call(cp_ctx* ctx, int q, const double* V, const double* t, int64_t d, int64_t E, double* out,
                 const char* what, F f) {
  return guard(ctx, [&] {
    check_q(q);
    if (d < 0 || E < 0) cpb::invalid(std::string(what) + ": negative shape");
    if (E > 0) need(t, "thresholds");
    check_thresholds(t, E, what);
    if (d * E == 0) return;
    cpb::Ctx& c = *ctx->c;
    double* dv = upload(c, "api.v", V, d * E);
    double* dt = upload(c, "api.t", t, E);
    double* dout = c.buf<double>("api.o", d * E);
    f(c, dv, dt, dout);
    cpb::d2h(c, out, dout, d * E * sizeof(double));
  });
}
}  // namespace
extern "C" {

int cp_prox_columns(cp_ctx* ctx, int q, const double* V, const double* thresholds, int64_t d, int64_t E,
                    double* out) {
  return columns_call(ctx, q, V, thresholds, d, E, out, "prox_norm",
                      [&](cpb::Ctx& c, double* v, double* t, double* o) { cpb::prox_columns_dev(c, q, v, t, d, E, o); });
}
int cp_project_columns(cp_ctx* ctx, int q, const double* Z, const double* radii, int64_t d, int64_t E, double* out) {
  return columns_call(ctx, q, Z, radii, d, E, out, "project_dual_ball", [&](cpb::Ctx& c, double* v, double* t, double* o) {
    cpb::project_columns_dev(c, q, v, t, d, E, o);
  });
}
int cp_prox_jacobian_apply(cp_ctx* ctx, int q, const double* V, const double* thresholds, const double* W,
                           int64_t d, int64_t E, double* out) {
  return columns_call(ctx, q, V, thresholds, d, E, out, "prox_jacobian",
                      [&](cpb::Ctx& c, double* v, double* t, double* o) {
                        need(W, "W");
                        double* w = upload(c, "api.w", W, d * E);
                        cpb::prox_jacobian_apply_dev(c, q, v, t, w, d, E, o);
                      });
}
int cp_prox_jacobian_diag(cp_ctx* ctx, int q, const double* V, const double* thresholds, int64_t d, int64_t E,
                          double* out) {
  return columns_call(ctx, q, V, thresholds, d, E, out, "prox_jacobian",
                      [&](cpb::Ctx& c, double* v, double* t, double* o) {
                        cpb::prox_jacobian_diag_dev(c, q, v, t, d, E, o);
                      });
}

// ---- objectives -----------------------------------------------------------------
int cp_primal_objective(cp_ctx* ctx, const cp_data* A, const cp_graph* g, double gamma, int q, const double* X,
                        double* out) {
  return guard(ctx, [&] {
    cpb::Prob P = make_prob(ctx, A, g, gamma, q);
    double* dx = upload(*P.c, "api.x", X, P.d() * P.n());
    *out = cpb::primal_objective_dev(P, dx);
  });
}
int cp_dual_objective(cp_ctx* ctx, const cp_data* A, const cp_graph* g, double gamma, int q, const double* Z,
                      double* out) {
  return guard(ctx, [&] {
    cpb::Prob P = make_prob(ctx, A, g, gamma, q);
    double* dz = upload(*P.c, "api.z", Z, P.d() * P.E());
    *out = cpb::dual_objective_dev(P, dz);
  });
}
int cp_kkt_residual(cp_ctx* ctx, const cp_data* A, const cp_graph* g, double gamma, int q, const double* X,
                    const double* Z, double* out) {
  return guard(ctx, [&] {
    cpb::Prob P = make_prob(ctx, A, g, gamma, q);
    double* dx = upload(*P.c, "api.x", X, P.d() * P.n());
    double* dz = upload(*P.c, "api.z", Z, P.d() * P.E());
    *out = cpb::kkt_residual_dev(P, dx, dz);
  });
}

}  // extern "C"
namespace {
// eval_phi at (Z, sigma, X) into api buffers; returns phi.
double phi_at(cpb::Prob& P, const double* Z, double sigma, const double* X, double** V, double** nv, double** thr,
              double** dx) {
  if (!(sigma > 0.0)) cpb::invalid("ssnal: sigma must be positive");
  cpb::Ctx& c = *P.c;
  const int64_t d = P.d(), n = P.n(), E = P.E();
  *dx = upload(c, "api.x", X, d * n);
  double* dz = upload(c, "api.z", Z, d * E);
  *thr = c.buf<double>("api.thr", E + 1);
  *V = c.buf<double>("api.V", d * E + 1);
  *nv = c.buf<double>("api.nv", 2 * E + 1);
  cpb::make_thr(c, E, P.rad, sigma, *thr);
  const double zz = cpb::dot_dev(c, dz, dz, d * E);
  return cpb::eval_phi(P, *dx, nullptr, 0.0, nullptr, dz, sigma, *thr, zz, *V, *nv);
}
}  // namespace
extern "C" {

int cp_ssnal_phi_value(cp_ctx* ctx, const cp_data* A, const cp_graph* g, double gamma, int q, const double* Z,
                       double sigma, const double* X, double* out) {
  return guard(ctx, [&] {
    cpb::Prob P = make_prob(ctx, A, g, gamma, q);
    double *V, *nv, *thr, *dx;
    *out = phi_at(P, Z, sigma, X, &V, &nv, &thr, &dx);
  });
}
int cp_ssnal_phi_gradient(cp_ctx* ctx, const cp_data* A, const cp_graph* g, double gamma, int q, const double* Z,
                          double sigma, const double* X, double* out) {
  return guard(ctx, [&] {
    cpb::Prob P = make_prob(ctx, A, g, gamma, q);
    cpb::Ctx& c = *P.c;
    double *V, *nv, *thr, *dx;
    phi_at(P, Z, sigma, X, &V, &nv, &thr, &dx);
    const int64_t E = P.E(), m = P.d() * P.n();
    double* ps = c.buf<double>("api.ps", E + 1);
    double* jal = c.buf<double>("api.jal", E + 1);
    double* jbe = c.buf<double>("api.jbe", E + 1);
    double* G = c.buf<double>("api.G", m);
    double* diag = c.buf<double>("api.diag", m);
    cpb::jac_params(P, nv, thr, ps, jal, jbe);
    cpb::grad_diag(P, dx, V, ps, jal, jbe, thr, sigma, G, diag, false);
    cpb::d2h(c, out, G, m * sizeof(double));
  });
}
int cp_ssnal_hessian_apply(cp_ctx* ctx, const cp_data* A, const cp_graph* g, double gamma, int q, const double* Z,
                           double sigma, const double* X, const double* D, double* out) {
  return guard(ctx, [&] {
    cpb::Prob P = make_prob(ctx, A, g, gamma, q);
    cpb::Ctx& c = *P.c;
    double *V, *nv, *thr, *dx;
    phi_at(P, Z, sigma, X, &V, &nv, &thr, &dx);
    const int64_t E = P.E(), m = P.d() * P.n();
    double* ps = c.buf<double>("api.ps", E + 1);
    double* jal = c.buf<double>("api.jal", E + 1);
    double* jbe = c.buf<double>("api.jbe", E + 1);
    cpb::jac_params(P, nv, thr, ps, jal, jbe);
    double* dd = upload(c, "api.D", D, m);
    double* Ap = c.buf<double>("api.Ap", m);
    double* part = c.buf<double>("api.hpart", 2 * static_cast<size_t>(c.sm_count) * 8 + 2);
    unsigned *mask = nullptr, *sgn = nullptr;  // q = 1 / inf: the solver's bit-mask Hessian path
    if (q != 2 && E > 0) {
      const size_t words = static_cast<size_t>(E) * ((P.d() + 31) / 32);
      mask = c.buf<unsigned>("api.mask", words + 1);
      sgn = c.buf<unsigned>("api.sgn", words + 1);
      cpb::edge_masks(c, *P.g, V, q == 1 ? thr : jal, P.d(), q, mask, sgn);
    }
    cpb::hess_apply(P, dd, V, jal, jbe, thr, sigma, Ap, part, nullptr, mask, sgn);
    cpb::d2h(c, out, Ap, m * sizeof(double));
  });
}

// ---- solve / path ---------------------------------------------------------------
int cp_solve(cp_ctx* ctx, const cp_data* A, const cp_graph* g, double gamma, int q, const cp_solver_config* cfg,
             const double* warmX, int64_t warm_d, int64_t warm_n, const double* warmZ, int64_t warm_E, double* X,
             double* Z, cp_termination* term) {
  return guard(ctx, [&] {
    cp_solver_config def;
    cp_solver_config_default(&def);
    const cp_solver_config& cf = cfg ? *cfg : def;
    cpb::Prob P = make_prob(ctx, A, g, gamma, q);
    cpb::validate_config(cf);
    cpb::Ctx& c = *P.c;
    const int64_t d = P.d(), n = P.n(), E = P.E();
    double* dx = c.buf<double>("api.sX", d * n + 1);
    double* dz = c.buf<double>("api.sZ", d * E + 1);
    const bool trivial = !(gamma > 0.0) || E == 0;
    const bool warm = warmX && warmZ && !trivial;
    if (warm) {
      if (warm_d != d || warm_n != n || warm_E != E) cpb::invalid("warm start does not match the instance shapes");
      cpb::h2d(c, dx, warmX, d * n * sizeof(double));
      cpb::h2d(c, dz, warmZ, d * E * sizeof(double));
    }
    cpb::SolveCache cache;
    cp_termination t = cpb::solve_dev(P, cf, warm, dx, dz, cache);
    if (X) cpb::d2h(c, X, dx, d * n * sizeof(double));
    if (Z && d > 0 && E > 0) cpb::d2h(c, Z, dz, d * E * sizeof(double));
    if (term) *term = t;
  });
}

int cp_make_schedule(double start, double end, int64_t count, int geometric, double* out) {
  return guard(nullptr, [&] {
    if (!(start > 0.0) || !(end > 0.0) || !std::isfinite(start) || !std::isfinite(end))
      cpb::invalid("schedule endpoints must be positive and finite");
    if (count < 1) cpb::invalid("schedule count must be >= 1");
    if (count > 1 && start == end) cpb::invalid("schedule with count > 1 needs distinct endpoints");
    need(out, "out");
    if (count == 1) {
      out[0] = start;
      return;
    }
    const double lo = std::min(start, end), hi = std::max(start, end);
    if (!geometric) {
      for (int64_t t = 0; t < count; ++t)
        out[t] = lo + (hi - lo) * static_cast<double>(t) / static_cast<double>(count - 1);
    } else {
      const double lr = std::log(hi / lo) / static_cast<double>(count - 1);
      for (int64_t t = 0; t < count; ++t) out[t] = lo * std::exp(static_cast<double>(t) * lr);
    }
    out[0] = lo;
    out[count - 1] = hi;
    for (int64_t t = 1; t < count; ++t)
      if (!(out[t] > out[t - 1])) cpb::invalid("schedule endpoints too close: values are not strictly increasing");
  });
}

int cp_extract_clusters(cp_ctx* ctx, const cp_graph* g, const double* X, int64_t d, int64_t n, double fuse_tol,
                        int64_t* labels, int64_t* K, double* centroids) {
  return guard(ctx, [&] {
    need(g, "graph");
    if (n != g->g->n) cpb::invalid("extract_clusters: X column count != node count");
    if (!(fuse_tol > 0.0)) cpb::invalid("extract_clusters: fuse_tol must be positive");
    cpb::Ctx& c = *ctx->c;
    double* dx = upload(c, "api.x", X, d * n);
    int* lab = c.buf<int>("api.lab", n + 1);
    double* cent = centroids ? c.buf<double>("api.cent", d * n + 1) : nullptr;
    const int64_t k = cpb::extract_clusters_dev(c, *g->g, dx, d, fuse_tol, lab, cent);
    std::vector<int> h(static_cast<size_t>(n));
    cpb::d2h(c, h.data(), lab, n * sizeof(int));
    if (labels)
      for (int64_t v = 0; v < n; ++v) labels[v] = h[static_cast<size_t>(v)];
    if (K) *K = k;
    if (centroids) cpb::d2h(c, centroids, cent, d * k * sizeof(double));
  });
}

int cp_run_path(cp_ctx* ctx, const cp_data* A, const cp_graph* g, int q, const double* gammas, int64_t T,
                const cp_solver_config* cfg, const cp_path_options* opt, double* X_out, double* Z_out,
                int64_t* labels_out, int64_t* K_out, cp_termination* terms_out) {
  return cp_run_path_ex(ctx, A, g, q, gammas, T, cfg, opt, X_out, Z_out, labels_out, K_out, terms_out, nullptr);
}

int cp_run_path_ex(cp_ctx* ctx, const cp_data* A, const cp_graph* g, int q, const double* gammas, int64_t T,
                   const cp_solver_config* cfg, const cp_path_options* opt, double* X_out, double* Z_out,
                   int64_t* labels_out, int64_t* K_out, cp_termination* terms_out, const cp_path_sink* sink) {
  return guard(ctx, [&] {
    need(A, "data");
    need(g, "graph");
    check_q(q);
    if (T > 0) need(gammas, "gammas");
    cp_solver_config defc;
    cp_solver_config_default(&defc);
    cp_path_options defo;
    cp_path_options_default(&defo);
    cpb::run_path_dev(*ctx->c, const_cast<cpb::Data&>(A->d), *g->g, q, gammas, T, cfg ? *cfg : defc,
                      opt ? *opt : defo, X_out, Z_out, labels_out, K_out, terms_out, sink);
  });
}

int cp_last_trace(cp_ctx* ctx, cp_trace_row* rows, int64_t max_rows, int64_t* count) {
  return guard(ctx, [&] {
    need(ctx, "ctx");
    const auto& tr = ctx->c->trace;
    if (count) *count = static_cast<int64_t>(tr.size());
    if (rows)
      for (size_t k = 0; k < tr.size() && static_cast<int64_t>(k) < max_rows; ++k) rows[k] = tr[k];
  });
}

// ---- linalg (linalg.hpp:17-87) --------------------------------------------------------
}  // extern "C"
namespace {
template <class F>
int make_linop(cp_ctx* ctx, cp_linop** out, F fill) {
  return guard(ctx, [&] {
    need(ctx, "ctx");
    need(out, "out");
    auto h = std::make_unique<cp_linop>();
    h->device = ctx->c->device;
    fill(h->op);
    *out = h.release();
  });
}
void check_op(cp_ctx* ctx, const cp_linop* op) {
  need(ctx, "ctx");
  need(op, "operator");
  if (op->device != ctx->c->device) cpb::invalid("operator belongs to another device");
}
}  // namespace
extern "C" {

int cp_linop_identity(cp_ctx* ctx, int64_t n, cp_linop** out) {
  return make_linop(ctx, out, [&](cpb::LinOp& op) {
    if (n < 0) cpb::invalid("LinearOperator: negative dimension");
    op.kind = cpb::LinOp::Identity;
    op.n = n;
    op.symmetric = op.positive_definite = true;
  });
}
int cp_linop_dense(cp_ctx* ctx, const double* M, int64_t n, int positive_definite, cp_linop** out) {
  return make_linop(ctx, out, [&](cpb::LinOp& op) {
    if (n < 0) cpb::invalid("LinearOperator::dense: matrix must be square");
    if (n > 0) need(M, "M");
    // symmetric flag as linalg.cpp:82-84: ||M - M^T||_inf-entry <= 1e-12 (1 + ||M||_inf-entry)
    double asym = 0.0, scale = 0.0;
    for (int64_t r = 0; r < n; ++r)
      for (int64_t c = 0; c < n; ++c) {
        asym = std::max(asym, std::abs(M[c * n + r] - M[r * n + c]));
        scale = std::max(scale, std::abs(M[c * n + r]));
      }
    op.kind = cpb::LinOp::Dense;
    op.n = n;
    op.symmetric = asym <= 1e-12 * (1.0 + scale);
    op.positive_definite = positive_definite != 0;
    op.vals.resize(static_cast<size_t>(n * n) + 1);
    if (n > 0) cpb::h2d(*ctx->c, op.vals.p, M, static_cast<size_t>(n * n) * sizeof(double));
    ctx->c->sync();
  });
}
int cp_linop_sparse(cp_ctx* ctx, int64_t n, const int64_t* colptr, const int64_t* rowidx, const double* values,
                    int positive_definite, cp_linop** out) {
  return make_linop(ctx, out, [&](cpb::LinOp& op) {
    need(colptr, "colptr");
    cpb::linop_set_sparse(*ctx->c, op, n, colptr, rowidx, values, 1.0, 0.0);
    op.symmetric = true;
    op.positive_definite = positive_definite != 0;
  });
}
int cp_linop_jacobi(cp_ctx* ctx, const double* diag, int64_t rows, int64_t cols, cp_linop** out) {
  return make_linop(ctx, out, [&](cpb::LinOp& op) {
    if (rows < 0 || cols < 1) cpb::invalid("jacobi: bad diagonal shape");
    const int64_t m = rows * cols;
    if (m > 0) need(diag, "diag");
    for (int64_t k = 0; k < m; ++k)
      if (!(diag[k] > 0.0)) cpb::invalid("jacobi: diagonal must be positive");
    op.kind = cpb::LinOp::Jacobi;
    op.n = rows;
    op.jcols = cols;
    op.symmetric = op.positive_definite = true;
    op.vals.resize(static_cast<size_t>(m) + 1);
    if (m > 0) cpb::h2d(*ctx->c, op.vals.p, diag, static_cast<size_t>(m) * sizeof(double));
    ctx->c->sync();
  });
}
int cp_linop_callback(cp_ctx* ctx, int64_t rows, cp_apply_fn fn, void* user, int symmetric, int positive_definite,
                      cp_linop** out) {
  return make_linop(ctx, out, [&](cpb::LinOp& op) {
    if (rows < 0) cpb::invalid("LinearOperator: negative dimension");
    if (!fn) cpb::invalid("LinearOperator: empty apply function");
    op.kind = cpb::LinOp::Callback;
    op.n = rows;
    op.fn = fn;
    op.user = user;
    op.symmetric = symmetric != 0;
    op.positive_definite = positive_definite != 0;
  });
}
int cp_linop_info(const cp_linop* op, int64_t* rows, int* symmetric, int* positive_definite) {
  return guard(nullptr, [&] {
    need(op, "operator");
    if (rows) *rows = op->op.n;
    if (symmetric) *symmetric = op->op.symmetric;
    if (positive_definite) *positive_definite = op->op.positive_definite;
  });
}
void cp_linop_destroy(cp_linop* op) {
  if (!op) return;
  cudaSetDevice(op->device);
  delete op;
}
int cp_linop_apply(cp_ctx* ctx, const cp_linop* op, const double* X, int64_t cols, double* out) {
  return guard(ctx, [&] {
    check_op(ctx, op);
    if (cols < 0) cpb::invalid("LinearOperator::apply: operand has wrong row count");
    cpb::Ctx& c = *ctx->c;
    const int64_t m = op->op.n * cols;
    double* dx = upload(c, "la.x", X, m);
    double* dy = c.buf<double>("la.y", m + 1);
    cpb::linop_apply(c, op->op, dx, cols, dy);
    cpb::d2h(c, out, dy, m * sizeof(double));
  });
}
int cp_pcg(cp_ctx* ctx, const cp_linop* op, const double* rhs, int64_t cols, const cp_linop* pre, double tol,
           int64_t max_iter, double* x, int64_t* iterations, double* residual, int32_t* converged) {
  return guard(ctx, [&] {
    check_op(ctx, op);
    if (pre) check_op(ctx, pre);
    if (cols < 0) cpb::invalid("pcg: rhs row count does not match the operator");
    cpb::Ctx& c = *ctx->c;
    const int64_t m = op->op.n * cols;
    double* db = upload(c, "la.b", rhs, m);
    double* dx = c.buf<double>("la.xo", m + 1);
    const cpb::PcgResultDev r = cpb::pcg_generic(c, op->op, db, cols, pre ? &pre->op : nullptr, tol, max_iter, dx);
    if (x) cpb::d2h(c, x, dx, m * sizeof(double));
    if (iterations) *iterations = r.iterations;
    if (residual) *residual = r.residual;
    if (converged) *converged = r.converged ? 1 : 0;
  });
}
int cp_power_iteration(cp_ctx* ctx, const cp_linop* op, double tol, int64_t max_iter, double* lambda) {
  return guard(ctx, [&] {
    check_op(ctx, op);
    need(lambda, "lambda");
    *lambda = cpb::power_generic(*ctx->c, op->op, tol, max_iter);
  });
}
int cp_factor_create(cp_ctx* ctx, int64_t n, const int64_t* colptr, const int64_t* rowidx, const double* values,
                     double rho, cp_factor** out) {
  return guard(ctx, [&] {
    need(ctx, "ctx");
    need(out, "out");
    need(colptr, "colptr");
    if (!(rho > 0.0) || !std::isfinite(rho)) cpb::invalid("cholesky: rho must be positive and finite");
    if (n < 0) cpb::invalid("cholesky: matrix must be square");
    // check_square_symmetric (linalg.cpp:14-28): max |L^T - L| <= 1e-12 (1 + max |L|)
    std::map<std::pair<int64_t, int64_t>, double> ent;
    double scale = 0.0;
    for (int64_t j = 0; j < n; ++j)
      for (int64_t q = colptr[j]; q < colptr[j + 1]; ++q) {
        if (rowidx[q] < 0 || rowidx[q] >= n) cpb::invalid("cholesky: row index out of range");
        ent[{rowidx[q], j}] += values[q];
        scale = std::max(scale, std::abs(values[q]));
      }
    double asym = 0.0;
    for (const auto& [rc, v] : ent) {
      auto it = ent.find({rc.second, rc.first});
      asym = std::max(asym, std::abs(v - (it == ent.end() ? 0.0 : it->second)));
    }
    if (asym > 1e-12 * (1.0 + scale)) cpb::invalid("cholesky: matrix is not symmetric");
    auto f = std::make_unique<cp_factor>();
    f->device = ctx->c->device;
    f->rho = rho;
    cpb::Ctx& c = *ctx->c;
    cpb::linop_set_sparse(c, f->M, n, colptr, rowidx, values, rho, 1.0);  // M = I + rho L (linalg.cpp:40-42)
    std::vector<double> dg(static_cast<size_t>(n), 1.0);
    for (const auto& [rc, v] : ent)
      if (rc.first == rc.second) dg[static_cast<size_t>(rc.first)] += rho * v;
    for (double x : dg)
      if (!(x > 0.0)) cpb::runtime("cholesky: factorization of I + rho*L failed");
    f->pre.kind = cpb::LinOp::Jacobi;
    f->pre.n = n;
    f->pre.vals.resize(static_cast<size_t>(n) + 1);
    if (n > 0) cpb::h2d(c, f->pre.vals.p, dg.data(), static_cast<size_t>(n) * sizeof(double));
    c.sync();
    *out = f.release();
  });
}
int cp_factor_solve(cp_ctx* ctx, const cp_factor* f, const double* rhs, int64_t cols, double* out) {
  return guard(ctx, [&] {
    need(ctx, "ctx");
    need(f, "factor");
    if (f->device != ctx->c->device) cpb::invalid("factor belongs to another device");
    if (cols < 0) cpb::invalid("cholesky solve: rhs has wrong row count");
    cpb::Ctx& c = *ctx->c;
    const int64_t n = f->M.n, m = n * cols;
    double* db = upload(c, "fa.b", rhs, m);
    double* dx = c.buf<double>("fa.x", m + 1);
    const cpb::PcgResultDev r = cpb::pcg_generic(c, f->M, db, cols, &f->pre, 1e-14, 20 * n + 100, dx, 1);
    if (!r.converged && r.residual > 1e-10) cpb::runtime("cholesky: solve of I + rho*L did not converge");
    cpb::d2h(c, out, dx, m * sizeof(double));
  });
}
void cp_factor_destroy(cp_factor* f) {
  if (!f) return;
  cudaSetDevice(f->device);
  delete f;
}
int cp_norm_values(cp_ctx* ctx, int q, const double* V, int64_t d, int64_t cols, double* norm, double* dual) {
  return guard(ctx, [&] {
    need(ctx, "ctx");
    check_q(q);
    if (d < 0 || cols < 0) cpb::invalid("norm_value: bad shape");
    cpb::Ctx& c = *ctx->c;
    double* dv = upload(c, "nv.v", V, d * cols);
    double* dn = c.buf<double>("nv.n", 2 * cols + 2);
    cpb::norm_values_dev(c, q, dv, d, cols, dn, dn + cols);
    std::vector<double> h(static_cast<size_t>(2 * cols));
    if (cols) cpb::d2h(c, h.data(), dn, 2 * cols * sizeof(double));
    for (int64_t k = 0; k < cols; ++k) {
      if (norm) norm[k] = h[static_cast<size_t>(k)];
      if (dual) dual[k] = h[static_cast<size_t>(cols + k)];
    }
  });
}

}  // extern "C"
