// Multi-GPU plumbing for the node-partitioned PCG: one
// process per GPU, an NCCL communicator per context (libnccl.so.2 is loaded
// at run time, so the library has no link-time NCCL dependency and a process
// without NCCL simply cannot create a communicator).
//
// Partition: rank r owns node rows [r * chunk, min(n, (r + 1) * chunk)) with
// chunk = ceil(n / P); node arrays are full size on every rank (padded to
// P * chunk rows) so an in-place ncclAllGather of the owned chunk refreshes
// the rows other ranks gather from.  Reductions all-reduce the fixed-shape
// block-partial tables, so every rank takes identical control decisions.
#pragma once

#include "common.cuh"

namespace cpb {

struct Comm {
  void* nccl = nullptr;  // ncclComm_t
  int rank = 0, nranks = 1;
  ~Comm();
  int64_t chunk(int64_t n) const { return (n + nranks - 1) / nranks; }
  int64_t v0(int64_t n) const { return std::min<int64_t>(n, chunk(n) * rank); }
  int64_t v1(int64_t n) const { return std::min<int64_t>(n, chunk(n) * (rank + 1)); }
};

// 128-byte NCCL unique id (rank 0 creates it, the caller distributes it).
void comm_unique_id(char out[128]);
void comm_init(Ctx& c, int nranks, int rank, const char id[128]);
// In-place sum over the ranks of `count` doubles on the context stream.
void comm_allreduce_sum(Ctx& c, double* buf, size_t count);
// In-place all-gather: rank r's `chunk_elems` doubles at base + r * chunk_elems.
void comm_allgather(Ctx& c, double* base, size_t chunk_elems);

}  // namespace cpb
