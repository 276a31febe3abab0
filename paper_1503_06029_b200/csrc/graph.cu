// graph.cu -- f4: the cell graph as CSR and a breadth-first path query.
//
// The paper builds G_X so that motion planning can "find a path in such a
// graph", naming GPU graph traversal as the next step.
// Input: the canonical edge list of cg_build (u32 pairs (i, j), i < j,
// ascending).  Output CSR: row_ptr[v] .. row_ptr[v+1] index col[], the
// neighbours of v in ascending order.
//
// Because the list is sorted by (i, j), the HIGHER neighbours of v (edges
// (v, w)) are one contiguous, sorted run of it; the LOWER neighbours (edges
// (u, v)) are the run of v in the same list re-sorted by (j, i).  With
// hi_off[v] / lo_off[v] the first position of v in the two lists,
// row_ptr[v] = hi_off[v] + lo_off[v] (every edge is counted once from each
// side), so no scan is needed; one thread per vertex copies its two runs.
//
// BFS is level-synchronous: one warp per frontier vertex walks its adjacency
// (coalesced), claims unvisited neighbours with atomicCAS on dist and appends
// them to the next frontier with one warp-aggregated atomicAdd.  The BFS
// tree is not unique, so the parent returned is canonical: the smallest
// neighbour one level closer to the source (a pass after the search).
#include "kernels.cuh"

namespace cgk {
namespace {

// off[v] = first position p with key(p) >= v, v in [0, nv]; keys sorted
// ascending: key(p) = the u32 at edges[2p + comp] (comp 0: i, 1: j after the
// swap into (j, i) order)
__global__ void k_run_bounds(const uint32_t* __restrict__ pairs, int comp, int64_t m, int64_t nv,
                             uint64_t* __restrict__ off) {
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p <= m;
       p += int64_t(gridDim.x) * blockDim.x) {
    const int64_t cur = p < m ? int64_t(pairs[2 * p + comp]) : nv;
    const int64_t prev = p > 0 ? int64_t(pairs[2 * (p - 1) + comp]) : -1;
    for (int64_t v = prev + 1; v <= cur && v <= nv; ++v) off[v] = uint64_t(p);
  }
}

// (i, j) pairs -> u64 keys (j << 32 | i) for the transpose sort
__global__ void k_swap_keys(const uint32_t* __restrict__ e, int64_t m, uint64_t* __restrict__ k) {
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < m;
       p += int64_t(gridDim.x) * blockDim.x)
    k[p] = (uint64_t(e[2 * p + 1]) << 32) | e[2 * p];
}

__global__ void k_csr_fill(const uint32_t* __restrict__ e, const uint64_t* __restrict__ ji,
                           const uint64_t* __restrict__ hi_off, const uint64_t* __restrict__ lo_off,
                           int64_t nv, uint64_t* __restrict__ row_ptr, uint32_t* __restrict__ col) {
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v <= nv;
       v += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t base = hi_off[v] + lo_off[v];
    row_ptr[v] = base;
    if (v == nv) break;
    uint64_t o = base;
    for (uint64_t q = lo_off[v]; q < lo_off[v + 1]; ++q) col[o++] = uint32_t(ji[q]);  // lower: i
    for (uint64_t q = hi_off[v]; q < hi_off[v + 1]; ++q) col[o++] = e[2 * q + 1];     // higher: j
  }
}

__global__ void k_bfs_init(int32_t* __restrict__ dist, int64_t nv, int64_t src,
                           uint32_t* __restrict__ frontier) {
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < nv;
       v += int64_t(gridDim.x) * blockDim.x)
    dist[v] = v == src ? 0 : -1;
  if (blockIdx.x == 0 && threadIdx.x == 0) frontier[0] = uint32_t(src);
}

// one warp per frontier vertex
__global__ void __launch_bounds__(256)
    k_bfs_expand(const uint64_t* __restrict__ row_ptr, const uint32_t* __restrict__ col,
                 const uint32_t* __restrict__ cur, uint32_t ncur, int32_t level,
                 int32_t* __restrict__ dist, uint32_t* __restrict__ next, uint32_t* __restrict__ nnext) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t f = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; f < ncur; f += nw) {
    const uint32_t v = cur[f];
    const uint64_t b = row_ptr[v], e = row_ptr[v + 1];
    for (uint64_t q0 = b; q0 < e; q0 += 32) {
      const uint64_t q = q0 + lane;
      bool claim = false;
      uint32_t w = 0;
      if (q < e) {
        w = col[q];
        claim = dist[w] < 0 && atomicCAS(&dist[w], -1, level + 1) == -1;
      }
      const uint32_t bal = __ballot_sync(kFull, claim);
      if (bal) {
        uint32_t base = 0;
        if (lane == __ffs(bal) - 1) base = atomicAdd(nnext, uint32_t(__popc(bal)));
        base = __shfl_sync(kFull, base, __ffs(bal) - 1);
        if (claim) next[base + __popc(bal & lt)] = w;
      }
    }
  }
}

// canonical parent: the smallest neighbour one level closer (-1: source or
// unreachable)
__global__ void k_bfs_parent(const uint64_t* __restrict__ row_ptr, const uint32_t* __restrict__ col,
                             const int32_t* __restrict__ dist, int64_t nv,
                             int32_t* __restrict__ parent) {
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < nv;
       v += int64_t(gridDim.x) * blockDim.x) {
    const int32_t d = dist[v];
    int32_t p = -1;
    if (d > 0)
      for (uint64_t q = row_ptr[v]; q < row_ptr[v + 1]; ++q)
        if (dist[col[q]] == d - 1) {
          p = int32_t(col[q]);
          break;
        }
    parent[v] = p;
  }
}

int grid1(int64_t n) {
  return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 16)));
}

}  // namespace

void build_csr(const uint32_t* edges, int64_t m, int64_t nv, uint64_t* row_ptr, uint32_t* col,
               cudaStream_t s) {
  DevBuf<uint64_t> hi_off(size_t(nv) + 1, s), lo_off(size_t(nv) + 1, s);
  DevBuf<uint64_t> ji(std::max<size_t>(1, size_t(m)), s), ji_alt(std::max<size_t>(1, size_t(m)), s);
  k_run_bounds<<<grid1(m + 1), 256, 0, s>>>(edges, 0, m, nv, hi_off.p);
  CG_LAUNCH_CHECK();
  uint64_t* jis = ji.p;
  if (m > 0) {
    k_swap_keys<<<grid1(m), 256, 0, s>>>(edges, m, ji.p);
    CG_LAUNCH_CHECK();
    // (j << 32 | i): sorted by j, then i -- the lower neighbours in order
    radix_sort<uint64_t>(ji.p, ji_alt.p, nullptr, nullptr, nullptr, false, m, 64, &jis, nullptr, s,
                         nullptr);
  }
  // the high word of each key is j: view the sorted keys as (i, j) u32 pairs
  k_run_bounds<<<grid1(m + 1), 256, 0, s>>>(reinterpret_cast<const uint32_t*>(jis), 1, m, nv,
                                             lo_off.p);
  CG_LAUNCH_CHECK();
  k_csr_fill<<<grid1(nv + 1), 256, 0, s>>>(edges, jis, hi_off.p, lo_off.p, nv, row_ptr, col);
  CG_LAUNCH_CHECK();
}

int bfs(const uint64_t* row_ptr, const uint32_t* col, int64_t nv, int64_t src, int32_t* dist,
        int32_t* parent, cudaStream_t s) {
  DevBuf<uint32_t> fa(size_t(nv), s), fb(size_t(nv), s), cnt(1, s);
  k_bfs_init<<<grid1(nv), 256, 0, s>>>(dist, nv, src, fa.p);
  CG_LAUNCH_CHECK();
  uint32_t* cur = fa.p;
  uint32_t* nxt = fb.p;
  uint32_t ncur = 1;
  int32_t level = 0;
  uint32_t* h = static_cast<uint32_t*>(host_stage(sizeof(uint32_t)));
  while (ncur > 0) {
    CG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(uint32_t), s));
    const int64_t blocks = std::min<int64_t>((int64_t(ncur) * 32 + 255) / 256, int64_t(num_sms()) * 16);
    k_bfs_expand<<<unsigned(std::max<int64_t>(1, blocks)), 256, 0, s>>>(row_ptr, col, cur, ncur,
                                                                        level, dist, nxt, cnt.p);
    CG_LAUNCH_CHECK();
    CG_CUDA(cudaMemcpyAsync(h, cnt.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaStreamSynchronize(s));
    ncur = h[0];
    std::swap(cur, nxt);
    ++level;
  }
  if (parent) {
    k_bfs_parent<<<grid1(nv), 256, 0, s>>>(row_ptr, col, dist, nv, parent);
    CG_LAUNCH_CHECK();
  }
  return level - 1;  // eccentricity of the source within its component
}

}  // namespace cgk
