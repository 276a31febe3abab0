// edges.cu -- a7: canonical edge list from the probe's unordered hits
// without a full sort.
//
// The probe appends hits (i << 32 | j) in arbitrary order.  The canonical list
// is ascending by (i, j) (DESIGN G4).  Instead of radix-sorting all m
// keys (8 passes), the edges are placed by their source cell:
//   1. count    deg[i] += 1 per edge (atomics into a u32 array of n_c)
//   2. scan     off = exclusive prefix sum of deg (one-sweep, look-back)
//   3. place    pos = off[i] + atomicAdd(cur[i], 1); write (i, j) there
//   4. fix      each cell's segment (its out-degree, <= ell and usually
//               0..2) is insertion-sorted by j
// Traffic: ~4 passes over m edges plus 3 over n_c counters, and no global
// multi-pass sort.  The output is unique: (i, j) pairs are distinct, so the
// order inside a segment after step 4 does not depend on the atomics.
#include "kernels.cuh"

namespace cgk {
namespace {

__global__ void k_edge_count(const uint64_t* __restrict__ e, int64_t m, uint32_t* __restrict__ deg) {
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < m;
       t += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(deg + (e[t] >> 32), 1u);
}

constexpr int kScanThreads = 256;
constexpr int kScanIPT = 16;

// exclusive scan of u32 (total < 2^32), in place; tiles by atomic ticket
__global__ void __launch_bounds__(kScanThreads)
    k_scan_u32(uint32_t* __restrict__ v, int64_t n, uint64_t* status, uint32_t* ticket) {
  constexpr int TILE = kScanThreads * kScanIPT;
  __shared__ uint32_t s_scan[33];
  __shared__ uint32_t s_base;
  __shared__ uint32_t s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t g0 = tile * TILE + int64_t(threadIdx.x) * kScanIPT;
  uint32_t x[kScanIPT];
  uint32_t sum = 0;
#pragma unroll
  for (int i = 0; i < kScanIPT; ++i) {
    x[i] = (g0 + i < n) ? v[g0 + i] : 0u;
    sum += x[i];
  }
  uint32_t total;
  const uint32_t excl = block_excl_scan(sum, s_scan, &total);
  if (threadIdx.x < 32) {
    const uint32_t b = lookback_warp(status, tile, total, 1);
    if (threadIdx.x == 0) s_base = b;
  }
  __syncthreads();
  uint32_t run = s_base + excl;
#pragma unroll
  for (int i = 0; i < kScanIPT; ++i) {
    if (g0 + i < n) v[g0 + i] = run;
    run += x[i];
  }
}

__global__ void k_edge_place(const uint64_t* __restrict__ e, int64_t m, const uint32_t* __restrict__ off,
                             uint32_t* __restrict__ cur, uint64_t* __restrict__ out) {
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < m;
       t += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = e[t];
    const uint32_t i = uint32_t(k >> 32);
    const uint32_t pos = off[i] + atomicAdd(cur + i, 1u);
    out[pos] = (k >> 32) | (k << 32);  // little-endian (i, j) u32 pair
  }
}

// sort each cell's segment [off[i], off[i] + deg) by j (insertion sort; the
// segment holds the cell's out-edges, at most ell of them)
__global__ void k_edge_fix(const uint32_t* __restrict__ off, const uint32_t* __restrict__ cur,
                           int64_t nc, uint64_t* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nc;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t len = cur[i];
    if (len < 2) continue;
    uint64_t* s = out + off[i];
    for (uint32_t a = 1; a < len; ++a) {
      const uint64_t v = s[a];
      const uint32_t jv = uint32_t(v >> 32);
      uint32_t b = a;
      while (b > 0 && uint32_t(s[b - 1] >> 32) > jv) {
        s[b] = s[b - 1];
        --b;
      }
      s[b] = v;
    }
  }
}

int blocks_for(int64_t n, int threads, int per_sm) {
  int64_t b = (n + threads - 1) / threads;
  return int(std::max<int64_t>(1, std::min<int64_t>(b, int64_t(num_sms()) * per_sm)));
}

}  // namespace

void launch_scan_u32(uint32_t* v, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  constexpr int TILE = kScanThreads * kScanIPT;
  const int64_t tiles = (n + TILE - 1) / TILE;
  DevBuf<uint64_t> status(size_t(tiles), s);
  DevBuf<uint32_t> ticket(1, s);
  CG_CUDA(cudaMemsetAsync(status.p, 0, size_t(tiles) * 8, s));
  CG_CUDA(cudaMemsetAsync(ticket.p, 0, 4, s));
  k_scan_u32<<<unsigned(tiles), kScanThreads, 0, s>>>(v, n, status.p, ticket.p);
  CG_LAUNCH_CHECK();
}

void place_edges(const uint64_t* hits, int64_t m, int64_t nc, uint64_t* out, cudaStream_t s) {
  if (m <= 0) return;
  DevBuf<uint32_t> deg(size_t(nc), s), cur(size_t(nc), s);
  CG_CUDA(cudaMemsetAsync(deg.p, 0, size_t(nc) * 4, s));
  CG_CUDA(cudaMemsetAsync(cur.p, 0, size_t(nc) * 4, s));
  k_edge_count<<<blocks_for(m, 256, 16), 256, 0, s>>>(hits, m, deg.p);
  CG_LAUNCH_CHECK();
  constexpr int TILE = kScanThreads * kScanIPT;
  const int64_t tiles = (nc + TILE - 1) / TILE;
  DevBuf<uint64_t> status(size_t(tiles), s);
  DevBuf<uint32_t> ticket(1, s);
  CG_CUDA(cudaMemsetAsync(status.p, 0, size_t(tiles) * 8, s));
  CG_CUDA(cudaMemsetAsync(ticket.p, 0, 4, s));
  k_scan_u32<<<unsigned(tiles), kScanThreads, 0, s>>>(deg.p, nc, status.p, ticket.p);
  CG_LAUNCH_CHECK();
  k_edge_place<<<blocks_for(m, 256, 16), 256, 0, s>>>(hits, m, deg.p, cur.p, out);
  CG_LAUNCH_CHECK();
  k_edge_fix<<<blocks_for(nc, 256, 16), 256, 0, s>>>(deg.p, cur.p, nc, out);
  CG_LAUNCH_CHECK();
}

}  // namespace cgk
