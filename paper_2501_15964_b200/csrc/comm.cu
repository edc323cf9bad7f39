// NCCL through dlopen (see comm.cuh).
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

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
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.get_id = reinterpret_cast<decltype(n.get_id)>(dlsym(h, "ncclGetUniqueId"));
    n.init = reinterpret_cast<decltype(n.init)>(dlsym(h, "ncclCommInitRank"));
    n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(h, "ncclCommDestroy"));
    n.allreduce = reinterpret_cast<decltype(n.allreduce)>(dlsym(h, "ncclAllReduce"));
    n.allgather = reinterpret_cast<decltype(n.allgather)>(dlsym(h, "ncclAllGather"));
    n.errstr = reinterpret_cast<decltype(n.errstr)>(dlsym(h, "ncclGetErrorString"));
  });
  if (!n.get_id || !n.init || !n.destroy || !n.allreduce || !n.allgather)
    throw Error(CP_ENCCL, "NCCL (libnccl.so.2) is not available in this process");
  return n;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(CP_ENCCL, std::string(what) + ": " + (nccl().errstr ? nccl().errstr(r) : "NCCL error"));
}

}  // namespace

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

void comm_allreduce_sum(Ctx& c, double* buf, size_t count) {
  if (!c.comm || count == 0) return;
  check(nccl().allreduce(buf, buf, count, ncclFloat64, ncclSum, static_cast<ncclComm_t>(c.comm->nccl), c.s),
        "ncclAllReduce");
}

void comm_allgather(Ctx& c, double* base, size_t chunk_elems) {
  if (!c.comm || chunk_elems == 0) return;
  check(nccl().allgather(base + static_cast<size_t>(c.comm->rank) * chunk_elems, base, chunk_elems, ncclFloat64,
                         static_cast<ncclComm_t>(c.comm->nccl), c.s),
        "ncclAllGather");
}

}  // namespace cpb
