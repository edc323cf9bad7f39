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

#include <vector>

namespace cpb {

// In-process group: P contexts driven by P host threads (tests on one GPU).
// Collectives synchronise the ranks' streams and meet at a host barrier; no
// kernel ever waits on another rank, so ranks sharing a GPU cannot deadlock.
struct LocalGroup;
LocalGroup* local_group_create(int nranks);
void local_group_destroy(LocalGroup* g);

struct Comm {
  void* nccl = nullptr;         // ncclComm_t
  LocalGroup* local = nullptr;  // or an in-process group
  int rank = 0, nranks = 1;
  ~Comm();
  int64_t chunk(int64_t n) const { return (n + nranks - 1) / nranks; }
  int64_t v0(int64_t n) const { return std::min<int64_t>(n, chunk(n) * rank); }
  int64_t v1(int64_t n) const { return std::min<int64_t>(n, chunk(n) * (rank + 1)); }
};

// 128-byte NCCL unique id (rank 0 creates it, the caller distributes it).
void comm_unique_id(char out[128]);
void comm_init(Ctx& c, int nranks, int rank, const char id[128]);
void comm_init_local(Ctx& c, LocalGroup* g, int rank);
// In-place sum over the ranks of `count` doubles on the context stream.
void comm_allreduce_sum(Ctx& c, double* buf, size_t count);
// In-place all-gather: rank r's `chunk_elems` doubles at base + r * chunk_elems.
void comm_allgather(Ctx& c, double* base, size_t chunk_elems);
// In-place all-gather of raw bytes (rank r's chunk at base + r * chunk_bytes).
void comm_allgather_bytes(Ctx& c, void* base, size_t chunk_bytes);
// Point-to-point exchange: rows [send_off[s], send_off[s+1]) of sbuf go to
// rank s, rows [recv_off[s], recv_off[s+1]) of rbuf come from rank s (width d).
void comm_exchange(Ctx& c, const double* sbuf, const std::vector<int64_t>& send_off, double* rbuf,
                   const std::vector<int64_t>& recv_off, int64_t d);
// In-place max over the ranks.
void comm_allreduce_max(Ctx& c, double* buf, size_t count);
// In-place all-gather of variable row ranges: rank q owns rows [row0[q], row0[q] + rows[q]) of width d.
void comm_allgatherv_rows(Ctx& c, double* base, const std::vector<int64_t>& row0, const std::vector<int64_t>& rows,
                          int64_t d);
// Host values: sums except the entries in max_cols, which are maxed.
void comm_allreduce_host(Ctx& c, std::vector<double>& v, const std::vector<int>& max_cols = {});

}  // namespace cpb
