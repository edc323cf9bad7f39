// NCCL through dlopen (see comm.cuh).
#include <dlfcn.h>

#include <cstdlib>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <mutex>
#include <vector>

#include "comm.cuh"

namespace cpb {

namespace {

struct Nccl {
  decltype(&ncclGetUniqueId) get_id = nullptr;
  decltype(&ncclCommInitRank) init = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllReduce) allreduce = nullptr;
  decltype(&ncclAllGather) allgather = nullptr;
  decltype(&ncclGetErrorString) errstr = nullptr;
  decltype(&ncclBroadcast) bcast = nullptr;
  decltype(&ncclGroupStart) gstart = nullptr;
  decltype(&ncclGroupEnd) gend = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    // an NCCL already in the process (torch's), then CPB_NCCL_LIB (the Python layer points it at
    // torch's wheel), then the loader's search path
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h)
      if (const char* p = std::getenv("CPB_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.get_id = reinterpret_cast<decltype(n.get_id)>(dlsym(h, "ncclGetUniqueId"));
    n.init = reinterpret_cast<decltype(n.init)>(dlsym(h, "ncclCommInitRank"));
    n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(h, "ncclCommDestroy"));
    n.allreduce = reinterpret_cast<decltype(n.allreduce)>(dlsym(h, "ncclAllReduce"));
    n.allgather = reinterpret_cast<decltype(n.allgather)>(dlsym(h, "ncclAllGather"));
    n.errstr = reinterpret_cast<decltype(n.errstr)>(dlsym(h, "ncclGetErrorString"));
    n.bcast = reinterpret_cast<decltype(n.bcast)>(dlsym(h, "ncclBroadcast"));
    n.gstart = reinterpret_cast<decltype(n.gstart)>(dlsym(h, "ncclGroupStart"));
    n.gend = reinterpret_cast<decltype(n.gend)>(dlsym(h, "ncclGroupEnd"));
    n.send = reinterpret_cast<decltype(n.send)>(dlsym(h, "ncclSend"));
    n.recv = reinterpret_cast<decltype(n.recv)>(dlsym(h, "ncclRecv"));
  });
  if (!n.get_id || !n.init || !n.destroy || !n.allreduce || !n.allgather || !n.bcast || !n.gstart || !n.gend ||
      !n.send || !n.recv)
    throw Error(CP_ENCCL, "NCCL (libnccl.so.2) is not available in this process");
  return n;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(CP_ENCCL, std::string(what) + ": " + (nccl().errstr ? nccl().errstr(r) : "NCCL error"));
}

}  // namespace

struct LocalGroup {
  int n = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  std::vector<double*> ptrs;
  std::vector<const std::vector<int64_t>*> offs;
  std::vector<std::vector<double>> host;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const unsigned long long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

LocalGroup* local_group_create(int nranks) {
  if (nranks < 1) invalid("local group: nranks must be >= 1");
  auto* g = new LocalGroup();
  g->n = nranks;
  g->ptrs.assign(static_cast<size_t>(nranks), nullptr);
  g->offs.assign(static_cast<size_t>(nranks), nullptr);
  g->host.resize(static_cast<size_t>(nranks));
  return g;
}
void local_group_destroy(LocalGroup* g) { delete g; }

Comm::~Comm() {
  if (nccl) {
    try {
      cpb::nccl().destroy(static_cast<ncclComm_t>(nccl));
    } catch (...) {
    }
  }
}

void comm_unique_id(char out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
  ncclUniqueId id;
  check(nccl().get_id(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
}

void comm_init(Ctx& c, int nranks, int rank, const char id[128]) {
  if (nranks < 1 || rank < 0 || rank >= nranks) invalid("communicator: rank out of range");
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  auto cm = std::make_unique<Comm>();
  ncclComm_t comm = nullptr;
  check(nccl().init(&comm, nranks, uid, rank), "ncclCommInitRank");
  cm->nccl = comm;
  cm->rank = rank;
  cm->nranks = nranks;
  c.comm = std::move(cm);
}

void comm_init_local(Ctx& c, LocalGroup* g, int rank) {
  if (!g || rank < 0 || rank >= g->n) invalid("communicator: rank out of range");
  auto cm = std::make_unique<Comm>();
  cm->local = g;
  cm->rank = rank;
  cm->nranks = g->n;
  c.comm = std::move(cm);
}

void comm_allreduce_sum(Ctx& c, double* buf, size_t count) {
  if (!c.comm || count == 0) return;
  if (LocalGroup* g = c.comm->local) {  // host sum in rank order: identical on every rank
    const int r = c.comm->rank;
    g->host[r].resize(count);
    d2h(c, g->host[r].data(), buf, count * sizeof(double));
    g->barrier();
    std::vector<double> sum(count, 0.0);
    for (int q = 0; q < g->n; ++q)
      for (size_t i = 0; i < count; ++i) sum[i] += g->host[q][i];
    g->barrier();  // nobody refills its host slot before every rank has read it
    h2d(c, buf, sum.data(), count * sizeof(double));
    return;
  }
  check(nccl().allreduce(buf, buf, count, ncclFloat64, ncclSum, static_cast<ncclComm_t>(c.comm->nccl), c.s),
        "ncclAllReduce");
}

void comm_allreduce_max(Ctx& c, double* buf, size_t count) {
  if (!c.comm || count == 0) return;
  if (LocalGroup* g = c.comm->local) {
    const int r = c.comm->rank;
    g->host[r].resize(count);
    d2h(c, g->host[r].data(), buf, count * sizeof(double));
    g->barrier();
    std::vector<double> mx(g->host[0]);
    for (int q = 1; q < g->n; ++q)
      for (size_t i = 0; i < count; ++i) mx[i] = std::max(mx[i], g->host[q][i]);
    g->barrier();
    h2d(c, buf, mx.data(), count * sizeof(double));
    return;
  }
  check(nccl().allreduce(buf, buf, count, ncclFloat64, ncclMax, static_cast<ncclComm_t>(c.comm->nccl), c.s),
        "ncclAllReduce(max)");
}

void comm_allreduce_host(Ctx& c, std::vector<double>& v, const std::vector<int>& max_cols) {
  if (!c.comm || v.empty()) return;
  const size_t k = v.size();
  std::vector<double> buf(2 * k, 0.0);
  for (size_t i = 0; i < k; ++i) buf[i] = v[i], buf[k + i] = -1e300;
  for (int mcol : max_cols) buf[k + mcol] = v[static_cast<size_t>(mcol)], buf[static_cast<size_t>(mcol)] = 0.0;
  double* d = c.buf<double>("comm.host", 2 * k);
  h2d(c, d, buf.data(), 2 * k * sizeof(double));
  comm_allreduce_sum(c, d, k);
  comm_allreduce_max(c, d + k, k);
  d2h(c, buf.data(), d, 2 * k * sizeof(double));
  for (size_t i = 0; i < k; ++i) v[i] = buf[i];
  for (int mcol : max_cols) v[static_cast<size_t>(mcol)] = buf[k + mcol];
}

void comm_allgatherv_rows(Ctx& c, double* base, const std::vector<int64_t>& row0, const std::vector<int64_t>& rows,
                          int64_t d) {
  if (!c.comm) return;
  if (LocalGroup* g = c.comm->local) {
    const int r = c.comm->rank;
    c.sync();
    g->ptrs[r] = base;
    g->barrier();
    for (int q = 0; q < g->n; ++q)
      if (q != r && rows[q] > 0)
        CPB_CUDA(cudaMemcpyAsync(base + row0[q] * d, g->ptrs[q] + row0[q] * d, rows[q] * d * sizeof(double),
                                 cudaMemcpyDeviceToDevice, c.s));
    c.sync();
    g->barrier();
    return;
  }
  const Nccl& n = nccl();
  check(n.gstart(), "ncclGroupStart");
  for (int q = 0; q < c.comm->nranks; ++q)
    if (rows[q] > 0)
      check(n.bcast(base + row0[q] * d, base + row0[q] * d, static_cast<size_t>(rows[q] * d), ncclFloat64, q,
                    static_cast<ncclComm_t>(c.comm->nccl), c.s),
            "ncclBroadcast");
  check(n.gend(), "ncclGroupEnd");
}

void comm_exchange(Ctx& c, const double* sbuf, const std::vector<int64_t>& send_off, double* rbuf,
                   const std::vector<int64_t>& recv_off, int64_t d) {
  if (!c.comm || c.comm->nranks == 1) return;
  const int r = c.comm->rank, P = c.comm->nranks;
  if (LocalGroup* g = c.comm->local) {  // pull my segment of every peer's send buffer
    c.sync();
    g->ptrs[r] = const_cast<double*>(sbuf);
    g->offs[r] = &send_off;
    g->barrier();
    for (int q = 0; q < P; ++q) {
      if (q == r) continue;
      const int64_t rows = recv_off[q + 1] - recv_off[q];
      if (rows == 0) continue;
      const int64_t at = (*g->offs[q])[r];  // peer q's rows destined to me start here
      CPB_CUDA(cudaMemcpyAsync(rbuf + recv_off[q] * d, g->ptrs[q] + at * d, rows * d * sizeof(double),
                               cudaMemcpyDeviceToDevice, c.s));
    }
    c.sync();
    g->barrier();
    return;
  }
  const Nccl& n = nccl();
  ncclComm_t cm = static_cast<ncclComm_t>(c.comm->nccl);
  check(n.gstart(), "ncclGroupStart");
  for (int q = 0; q < P; ++q) {
    if (q == r) continue;
    const int64_t ns = send_off[q + 1] - send_off[q], nr = recv_off[q + 1] - recv_off[q];
    if (ns) check(n.send(sbuf + send_off[q] * d, static_cast<size_t>(ns * d), ncclFloat64, q, cm, c.s), "ncclSend");
    if (nr) check(n.recv(rbuf + recv_off[q] * d, static_cast<size_t>(nr * d), ncclFloat64, q, cm, c.s), "ncclRecv");
  }
  check(n.gend(), "ncclGroupEnd");
}

void comm_allgather_bytes(Ctx& c, void* base_, size_t chunk_bytes) {
  if (!c.comm || chunk_bytes == 0) return;
  char* base = static_cast<char*>(base_);
  if (LocalGroup* g = c.comm->local) {
    const int r = c.comm->rank;
    c.sync();
    g->ptrs[r] = reinterpret_cast<double*>(base);
    g->barrier();
    for (int q = 0; q < g->n; ++q)
      if (q != r)
        CPB_CUDA(cudaMemcpyAsync(base + q * chunk_bytes, reinterpret_cast<char*>(g->ptrs[q]) + q * chunk_bytes,
                                 chunk_bytes, cudaMemcpyDeviceToDevice, c.s));
    c.sync();
    g->barrier();
    return;
  }
  check(nccl().allgather(base + static_cast<size_t>(c.comm->rank) * chunk_bytes, base, chunk_bytes, ncclChar,
                         static_cast<ncclComm_t>(c.comm->nccl), c.s),
        "ncclAllGather(bytes)");
}

void comm_allgather(Ctx& c, double* base, size_t chunk_elems) {
  if (!c.comm || chunk_elems == 0) return;
  if (LocalGroup* g = c.comm->local) {  // device-to-device copies of the other ranks' chunks
    const int r = c.comm->rank;
    c.sync();
    g->ptrs[r] = base;
    g->barrier();
    for (int q = 0; q < g->n; ++q)
      if (q != r)
        CPB_CUDA(cudaMemcpyAsync(base + q * chunk_elems, g->ptrs[q] + q * chunk_elems, chunk_elems * sizeof(double),
                                 cudaMemcpyDeviceToDevice, c.s));
    c.sync();
    g->barrier();  // every rank has copied before anyone writes its chunk again
    return;
  }
  check(nccl().allgather(base + static_cast<size_t>(c.comm->rank) * chunk_elems, base, chunk_elems, ncclFloat64,
                         static_cast<ncclComm_t>(c.comm->nccl), c.s),
        "ncclAllGather");
}

}  // namespace cpb
