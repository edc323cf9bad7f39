// SSNAL Hessian apply (ssnal.cpp:56-64) with TMA-staged rows.
//
//   Ap_v = p_v + sigma * sum_{l ni v} +-( w_l - (alpha_l w_l + beta_l <v_l, w_l> v_l) ),
//   w_l = p_i(l) - p_j(l)
//
// Work item = a segment of <= 64 incident edges of one node; one warp owns the
// node's whole feature row (lane l holds features l + 32 k, k < NK) so the
// per-edge dot <v_l, w_l> is a warp reduction and V is read once per
// endpoint (the two-pass edge_dot + gather reads it three times).  Rows
// p_other and v_l are streamed into a per-warp shared-memory ring by
// cp.async.bulk (the TMA engine) with mbarrier completion: one lane issues
// the next stages' copies while the warp computes, so every warp keeps
// STAGES x 2 rows (2 x 6.3 KB at d = 784) in flight independent of its
// register budget.  Nodes with more than 64 edges are split into segments
// whose partial sums a second kernel combines in segment order
// (deterministic).  Items run in node-id order, so both endpoints of an edge
// of a clustered graph tend to read v_l within the L2 window.
#include <algorithm>
#include <cstdlib>
#include <queue>
#include <string>
#include <vector>

#include "gather.cuh"
#include "graph.cuh"
#include "ops.cuh"
#include "ptx.cuh"

namespace cpb {

namespace {

constexpr int kSegEdges = 64;
constexpr int kMaxStages = 8;  // ring depth per warp: 2 at d = 784, up to 8 for short rows


// Per-warp shared memory: a metadata table for the current segment (<= 64
// edges: id, other endpoint, 1 - alpha, beta) filled with two coalesced
// rounds at segment start, and an S-deep ring of {p_other row, v row}.
// Per edge, with w = p_v - p_o and c = <v_l, w> (sign-free), the edge adds
//   (1 - alpha) w - beta c v_l
// to node v: one FMA per feature for the dot, two for the update (w is kept
// in registers, so the update reads only v_l back from shared memory).  An
// edge with beta = 0 (prox zero) adds (1 - alpha)(p_v - p_o): its p_v part is
// folded into one final FMA.
// FULL: d >= 32 (NK - 1), so the first NK - 1 feature chunks of a row are complete and only
// the last needs the f < d predicate (d = 784: 24 full chunks + 16 lanes).
template <int NK, bool FULL>
__global__ void __launch_bounds__(128) k_hess_tma(const double* __restrict__ P, const double* __restrict__ V,
                                                  const double* __restrict__ jal, const double* __restrict__ jbe,
                                                  const int* __restrict__ adj_e, const int* __restrict__ adj_o,
                                                  const int* __restrict__ seg_node, const int* __restrict__ seg_beg,
                                                  const int* __restrict__ seg_end, const int* __restrict__ seg_slot,
                                                  int nseg, int d, int dp, double sigma, double* __restrict__ Ap,
                                                  double* __restrict__ partial, double* part, const int* active,
                                                  int S, const int* __restrict__ wrange) {
  if (active && !*active) return;
  auto in_row = [d](int k, int f) { return (FULL && k < NK - 1) || f < d; };
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ double sh[32];
  __shared__ uint64_t bars[4][kMaxStages];
  __shared__ int m_le[4][kSegEdges], m_lo[4][kSegEdges];
  __shared__ double m_ca[4][kSegEdges], m_be[4][kSegEdges];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* ring = reinterpret_cast<double*>(smraw) + static_cast<size_t>(warp) * S * 2 * dp;
  uint64_t* bar = bars[warp];
  int* le = m_le[warp];
  int* lo = m_lo[warp];
  double* ca = m_ca[warp];
  double* mb = m_be[warp];
  if (lane == 0)
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
  fence_mbar_init();
  fence_proxy_async();
  __syncwarp();
  const unsigned row_bytes = static_cast<unsigned>(d) * 8u;
  int cst = 0;        // next ring slot to consume
  unsigned cph = 0;   // its mbarrier phase parity
  double s_a = 0.0, s_b = 0.0;
  auto issue = [&](int q, int st) {  // lane 0: stream edge q's rows into stage st
    const bool nv = mb[q] != 0.0;
    mbar_expect_tx(&bar[st], nv ? 2 * row_bytes : row_bytes);
    bulk_g2s(ring + st * 2 * dp, P + static_cast<int64_t>(lo[q]) * d, row_bytes, &bar[st]);
    if (nv) bulk_g2s(ring + st * 2 * dp + dp, V + static_cast<int64_t>(le[q]) * d, row_bytes, &bar[st]);
  };
  const int wid = blockIdx.x * (blockDim.x >> 5) + warp, nw = gridDim.x * (blockDim.x >> 5);
  // each warp walks its balanced item list (wrange: offsets, then items) or, without it, every nw-th item
  const int j0 = wrange ? wrange[wid] : wid, j1 = wrange ? wrange[wid + 1] : nseg, jstep = wrange ? 1 : nw;
  for (int j = j0; j < j1; j += jstep) {
    const int it = wrange ? wrange[j] : j;
    const int v = seg_node[it], e0 = seg_beg[it], ne = seg_end[it] - e0, slot = seg_slot[it];
    const int64_t base = static_cast<int64_t>(v) * d;
    // segment metadata: coalesced loads, then gathers of alpha / beta
    for (int q = lane; q < ne; q += 32) {
      const int l = adj_e[e0 + q];
      le[q] = l;
      lo[q] = adj_o[e0 + q];
      ca[q] = 1.0 - jal[l];
      mb[q] = jbe[l];
    }
    __syncwarp();
    if (lane == 0) {
      for (int s = 0, t = cst; s < S && s < ne; ++s, t = (t + 1 == S) ? 0 : t + 1) issue(s, t);
    }
    double pv[NK], acc[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      const int f = lane + 32 * k;
      pv[k] = in_row(k, f) ? P[base + f] : 0.0;
      acc[k] = 0.0;
    }
    double dsum = 0.0;
    for (int q = 0; q < ne; ++q) {
      const int st = cst;
      const double cq = ca[q], be = mb[q];
      mbar_wait(&bar[st], cph);
      if (++cst == S) cst = 0, cph ^= 1u;
      const double* po = ring + st * 2 * dp;
      const double* vl = po + dp;
      if (be != 0.0) {
        // w = p_v - p_o stays in registers: the update re-reads only v_l
        double w[NK];
        double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
#pragma unroll
        for (int k = 0; k < NK; ++k) {
          const int f = lane + 32 * k;
          w[k] = in_row(k, f) ? pv[k] - po[f] : 0.0;
          if (in_row(k, f)) {
            if ((k & 3) == 0) c0 = __fma_rn(vl[f], w[k], c0);
            if ((k & 3) == 1) c1 = __fma_rn(vl[f], w[k], c1);
            if ((k & 3) == 2) c2 = __fma_rn(vl[f], w[k], c2);
            if ((k & 3) == 3) c3 = __fma_rn(vl[f], w[k], c3);
          }
        }
        const double bc = be * warp_sum((c0 + c1) + (c2 + c3));
#pragma unroll
        for (int k = 0; k < NK; ++k) {
          const int f = lane + 32 * k;
          if (in_row(k, f)) acc[k] = __fma_rn(cq, w[k], __fma_rn(-bc, vl[f], acc[k]));
        }
      } else {
        dsum += cq;
#pragma unroll
        for (int k = 0; k < NK; ++k) {
          const int f = lane + 32 * k;
          if (in_row(k, f)) acc[k] = __fma_rn(-cq, po[f], acc[k]);
        }
      }
      // the warp's reads of this slot are ordered before the refill by the
      // warp barrier (only reads: no generic->async proxy fence is needed)
      __syncwarp();
      if (lane == 0 && q + S < ne) issue(q + S, st);
    }
    __syncwarp();  // metadata table is rewritten by the next segment
    if (slot < 0) {
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        const int f = lane + 32 * k;
        if (!in_row(k, f)) continue;
        const double o = pv[k] + sigma * __fma_rn(dsum, pv[k], acc[k]);
        Ap[base + f] = o;
        a += pv[k] * o;
        b += pv[k] * pv[k];
      }
      s_a += a;
      s_b += b;
    } else {
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        const int f = lane + 32 * k;
        if (in_row(k, f)) partial[static_cast<int64_t>(slot) * d + f] = __fma_rn(dsum, pv[k], acc[k]);
      }
    }
  }
  s_a = block_sum(s_a, sh);
  s_b = block_sum(s_b, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s_a;
    part[2 * blockIdx.x + 1] = s_b;
  }
}

// Hub nodes: Ap = p + sigma * (sum of segment partials, in segment order).
__global__ void __launch_bounds__(256) k_hess_combine(const double* __restrict__ P, const double* __restrict__ partial,
                                                      const int* __restrict__ hub_node, const int* __restrict__ hub_slot0,
                                                      const int* __restrict__ hub_nslots, int nhub, int d, double sigma,
                                                      double* __restrict__ Ap, double* part, const int* active) {
  if (active && !*active) return;
  __shared__ double sh[32];
  double s_a = 0.0, s_b = 0.0;
  for (int h = blockIdx.x; h < nhub; h += gridDim.x) {
    const int v = hub_node[h], s0 = hub_slot0[h], ns = hub_nslots[h];
    const int64_t base = static_cast<int64_t>(v) * d;
    for (int f = threadIdx.x; f < d; f += blockDim.x) {
      // segment order; 8 slots' loads in flight at a time (a hub has up to ~20 slots)
      double acc = 0.0;
      int s = 0;
      for (; s + 8 <= ns; s += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = partial[static_cast<int64_t>(s0 + s + u) * d + f];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u];
      }
      for (; s < ns; ++s) acc += partial[static_cast<int64_t>(s0 + s) * d + f];
      const double pv = P[base + f];
      const double o = pv + sigma * acc;
      Ap[base + f] = o;
      s_a += pv * o;
      s_b += pv * pv;
    }
  }
  s_a = block_sum(s_a, sh);
  s_b = block_sum(s_b, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s_a;
    part[2 * blockIdx.x + 1] = s_b;
  }
}

// Segments per graph (host-built once from the CSR).  Items run in a
// breadth-first (Cuthill-McKee-like) node order by default, so the nodes in
// flight at any time are graph neighbours of each other and the second
// endpoint's read of V_l and the gathered p rows tend to hit L2
// (CPB_HESS_ORDER=id keeps node-id order).
struct SegPlan {
  uint64_t uid = 0;
  int64_t v0 = 0, v1 = -1;  // node range the items cover (v1 < 0: all nodes)
  int nseg = 0, nhub = 0, nslots = 0;
  DBuf<int> node, beg, end, slot, hub_node, hub_slot0, hub_nslots;
  std::vector<int64_t> cost_prefix;  // per-item cost prefix (edges + fixed overhead)
  int split_nw = 0;                  // warp count `wrange` was cut for
  DBuf<int> wrange;  // nw + 1 list offsets, then the items of every warp's list
};

// Per-warp item lists (lpt_lists): windows of nw consecutive breadth-first
// items, so all warps work on neighbouring nodes at the same time (L2 reuse
// of V_l and the gathered p rows, as with round-robin), and inside each
// window the largest items go to the least-loaded warps so the warps finish
// together (round-robin left the longest warp ~15 % behind; C3 H-apply
// 1.43 -> 1.20 ms).
const int* warp_ranges(Ctx& c, SegPlan& p, int nw) {
  if (p.split_nw == nw) return p.wrange.p;
  std::vector<int64_t> cost(static_cast<size_t>(p.nseg));
  for (int i = 0; i < p.nseg; ++i) cost[i] = p.cost_prefix[i + 1] - p.cost_prefix[i];
  trace("warp_ranges begin");
  const std::vector<int> flat = lpt_lists(cost, nw, nw);  // windows of one item per warp
  trace("warp_ranges lpt done");
  p.wrange.resize(flat.size());
  h2d(c, p.wrange.p, flat.data(), flat.size() * sizeof(int));
  c.sync();
  p.split_nw = nw;
  return p.wrange.p;
}

SegPlan& seg_plan(Ctx& c, const Graph& g) {
  static thread_local std::vector<std::unique_ptr<SegPlan>> plans;
  for (auto& p : plans)
    if (p->uid == g.uid && p->v0 == c.own_v0 && p->v1 == c.own_v1) return *p;
  auto p = std::make_unique<SegPlan>();
  p->uid = g.uid;
  p->v0 = c.own_v0;
  p->v1 = c.own_v1;
  trace("seg_plan begin");
  std::vector<int> off, seq;
  if (g.E > 0) {
    seq = bfs_sequence(c, g, &off);
    trace("seg_plan bfs done");
  } else {
    off.resize(static_cast<size_t>(g.n + 1));
    d2h(c, off.data(), g.off.p, off.size() * sizeof(int));
    seq.resize(static_cast<size_t>(g.n));
    for (int v = 0; v < g.n; ++v) seq[v] = v;
  }
  std::vector<int> node, beg, end, slot, hn, hs, hc;
  int slots = 0;
  for (int v : seq) {
    if (c.own_v1 >= 0 && (v < c.own_v0 || v >= c.own_v1)) continue;  // another rank's node
    const int a = off[v], b = off[v + 1];
    if (b - a <= kSegEdges) {
      node.push_back(v), beg.push_back(a), end.push_back(b), slot.push_back(-1);
      continue;
    }
    hn.push_back(v), hs.push_back(slots);
    int ns = 0;
    for (int e = a; e < b; e += kSegEdges, ++ns)
      node.push_back(v), beg.push_back(e), end.push_back(std::min(b, e + kSegEdges)), slot.push_back(slots + ns);
    hc.push_back(ns);
    slots += ns;
  }
  auto up = [&](DBuf<int>& buf, const std::vector<int>& h) {
    buf.resize(h.size() + 1);
    if (!h.empty()) h2d(c, buf.p, h.data(), h.size() * sizeof(int));
  };
  up(p->node, node), up(p->beg, beg), up(p->end, end), up(p->slot, slot);
  up(p->hub_node, hn), up(p->hub_slot0, hs), up(p->hub_nslots, hc);
  c.sync();
  p->nseg = static_cast<int>(node.size());
  p->cost_prefix.assign(node.size() + 1, 0);
  for (size_t i = 0; i < node.size(); ++i) p->cost_prefix[i + 1] = p->cost_prefix[i] + (end[i] - beg[i]) + 4;
  p->nhub = static_cast<int>(hn.size());
  p->nslots = slots;
  if (plans.size() > 8) plans.erase(plans.begin());
  plans.push_back(std::move(p));
  trace("seg_plan built");
  return *plans.back();
}

#define NK_DISPATCH(nk, full, KERNEL, ...)                                     \
  switch (nk * 2 + (full ? 1 : 0)) {                                           \
    case 2 * 8: KERNEL<8, false> __VA_ARGS__; break;                           \
    case 2 * 8 + 1: KERNEL<8, true> __VA_ARGS__; break;                        \
    case 2 * 16: KERNEL<16, false> __VA_ARGS__; break;                         \
    case 2 * 16 + 1: KERNEL<16, true> __VA_ARGS__; break;                      \
    case 2 * 25: KERNEL<25, false> __VA_ARGS__; break;                         \
    case 2 * 25 + 1: KERNEL<25, true> __VA_ARGS__; break;                      \
    case 2 * 32 + 1: KERNEL<32, true> __VA_ARGS__; break;                      \
    default: KERNEL<32, false> __VA_ARGS__; break;                             \
  }

template <int NK, bool FULL>
void set_smem(int bytes) {
  CPB_CUDA(cudaFuncSetAttribute(k_hess_tma<NK, FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

int nk_bucket(int64_t d) {
  const int need = static_cast<int>((d + 31) / 32);
  for (int b : {8, 16, 25, 32})
    if (need <= b) return b;
  return 0;
}

}  // namespace

// Even d in [256, 1024]: below that the per-edge rows are too short for a
// two-deep ring to cover the copy latency (C5, d = 64: 17.4 ms vs 9.7 ms for
// the warp-chunk path).
bool hess_tma_supported(int64_t d) { return d >= 256 && d % 2 == 0 && nk_bucket(d) != 0; }

// Returns the number of (pAp, pp) block partials written to `part`.
int hess_tma(Ctx& c, const Graph& g, const double* P, const double* V, const double* jal, const double* jbe,
             int64_t d, double sigma, double* Ap, double* part, const int* active) {
  SegPlan& sp = seg_plan(c, g);
  const int nk = nk_bucket(d);
  const int dp = static_cast<int>((d + 1) / 2 * 2);
  const int warps = 4;
  // ring depth 2 (deeper rings measured slower: C5 with 8 stages 38.8 vs 17.4 ms;
  // an L2 evict_first policy on the streamed V_l rows measured neutral-to-worse
  // at C3, 1586 vs 1541 us)
  const int S = 2;
  const size_t smem = static_cast<size_t>(warps) * S * 2 * dp * sizeof(double);
  if (smem > 220 * 1024) invalid("hessian: shared-memory ring exceeds 220 KB");
  const bool full = d >= 32 * (nk - 1);
  NK_DISPATCH(nk, full, set_smem, (static_cast<int>(smem)));
  double* partial = c.buf<double>("hess.partial", static_cast<size_t>(sp.nslots) * d + 1);
  // partitioned PCG: every rank launches the same grid so the partial tables line up
  const bool parted = c.own_v1 >= 0;
  const int grid = parted ? c.sm_count * 2 : std::max(1, std::min(cdiv(sp.nseg, warps), c.sm_count * 2));
  const int* wr = warp_ranges(c, sp, grid * warps);
  NK_DISPATCH(nk, full, k_hess_tma, <<<grid, 32 * warps, smem, c.s>>>(P, V, jal, jbe, g.adj_e.p, g.adj_o.p, sp.node.p,
                                                                sp.beg.p, sp.end.p, sp.slot.p, sp.nseg,
                                                                static_cast<int>(d), dp, sigma, Ap, partial, part,
                                                                active, S, wr));
  CPB_LAUNCH_CHECK();
  int nb = grid;
  if (sp.nhub > 0 || parted) {
    const int gh = parted ? c.sm_count * 4 : std::max(1, std::min(sp.nhub, c.sm_count * 4));
    k_hess_combine<<<gh, 256, 0, c.s>>>(P, partial, sp.hub_node.p, sp.hub_slot0.p, sp.hub_nslots.p, sp.nhub,
                                         static_cast<int>(d), sigma, Ap, part + 2 * grid, active);
    CPB_LAUNCH_CHECK();
    nb += gh;
  }
  return nb;
}

}  // namespace cpb
