// layers.cu -- a4 popcount layering and a5 dictionary build.
//
// a4: a single-bit flip changes the popcount by exactly one,
// so the cells at distance 1 from a cell of popcount p lie in layers p-1 and
// p+1, and the 0->1 flips that emit each edge once (DESIGN G3) only look in
// layer p+1.  The layer-major order (popcount, canonical index) comes from a
// stable radix sort of (popc, index) pairs (radix.cu); this file turns it
// into layer offsets and gathers the rows and lcp values into that order.
//
// a5: the dictionary is the layer-major sorted array itself plus, per layer,
// a 2^b_p-entry prefix index T_p (b_p chosen so a bucket holds ~2^bucket_log2
// cells): T_p[x] = first row of layer p whose top b_p bits are >= x.  A
// lookup reads two T entries and binary-searches the bucket (DESIGN a5: the
// NS's "sorted-array binary search" option, prefix-accelerated).  It plays
// the role of the paper's leaf-only 2^r-ary tree:
// both map a prefix to the contiguous range of sorted vectors carrying it
// (P:280); here a whole b_p-bit prefix is resolved by one table read instead
// of b_p/r tree levels.
#include "kernels.cuh"

namespace cgk {
namespace {

__global__ void k_layer_offsets(const uint32_t* __restrict__ sp, int64_t nc, int ell,
                                uint32_t* __restrict__ off) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < nc;
       j += int64_t(gridDim.x) * blockDim.x) {
    const int p = int(sp[j]);
    const int pp = j == 0 ? -1 : int(sp[j - 1]);
    for (int q = pp + 1; q <= p; ++q) off[q] = uint32_t(j);
    if (j == nc - 1)
      for (int q = p + 1; q <= ell + 1; ++q) off[q] = uint32_t(nc);
  }
}

__global__ void k_gather_rows(const uint64_t* __restrict__ in, const uint32_t* __restrict__ idx,
                              int64_t n, int W, uint64_t* __restrict__ out) {
  const int64_t total = n * W;
  for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < total;
       g += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = g / W;
    const int w = int(g - r * W);
    out[g] = in[int64_t(idx[r]) * W + w];
  }
}

__global__ void k_gather_u16(const uint16_t* __restrict__ in, const uint32_t* __restrict__ idx,
                             int64_t n, uint16_t* __restrict__ out) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
       j += int64_t(gridDim.x) * blockDim.x)
    out[j] = in[idx[j]];
}

__device__ __forceinline__ int64_t prefix_of(uint64_t w0, int b) {
  return b ? int64_t(w0 >> (64 - b)) : 0;
}

__global__ void k_prefix_index(DictView d, const uint32_t* __restrict__ sp, uint32_t* __restrict__ T,
                               uint32_t* __restrict__ F) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < d.n_cells;
       j += int64_t(gridDim.x) * blockDim.x) {
    const int p = int(sp[j]);
    const uint32_t o = d.layer_off[p], e = d.layer_off[p + 1];
    const int b = d.tbits[p];
    uint32_t* Tp = T + d.tbase[p];
    const uint64_t w0 = d.keys[j * d.W];
    // filter bit of the cell's (b + fextra)-bit prefix
    const uint64_t y = w0 >> (64 - (b + d.fextra));
    atomicOr(F + d.fbase[p] + (y >> 5), 1u << (y & 31));
    const int64_t x = prefix_of(w0, b);
    const int64_t xp = (uint32_t(j) == o) ? -1 : prefix_of(d.keys[(j - 1) * d.W], b);
    for (int64_t q = xp + 1; q <= x; ++q) Tp[q] = uint32_t(j);
    if (uint32_t(j) + 1 == e) {
      const int64_t top = int64_t(1) << b;
      for (int64_t q = x + 1; q <= top; ++q) Tp[q] = e;
    }
  }
}

__global__ void k_prefix_index_empty(DictView d, uint32_t* __restrict__ T) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p <= d.ell; p += gridDim.x * blockDim.x) {
    const uint32_t o = d.layer_off[p], e = d.layer_off[p + 1];
    if (o != e) continue;
    const int64_t top = int64_t(1) << d.tbits[p];
    for (int64_t q = 0; q <= top; ++q) T[d.tbase[p] + q] = o;
  }
}

int blocks_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  return int(std::max<int64_t>(1, std::min<int64_t>(b, int64_t(num_sms()) * 16)));
}

}  // namespace

void launch_layer_offsets(const uint32_t* sorted_popc, int64_t nc, int ell, uint32_t* layer_off,
                          cudaStream_t s) {
  k_layer_offsets<<<blocks_for(nc, 256), 256, 0, s>>>(sorted_popc, nc, ell, layer_off);
  CG_LAUNCH_CHECK();
}

void launch_gather_rows(const uint64_t* in, const uint32_t* idx, int64_t n, int W, uint64_t* out,
                        cudaStream_t s) {
  k_gather_rows<<<blocks_for(n * W, 256), 256, 0, s>>>(in, idx, n, W, out);
  CG_LAUNCH_CHECK();
}

void launch_gather_u16(const uint16_t* in, const uint32_t* idx, int64_t n, uint16_t* out,
                       cudaStream_t s) {
  k_gather_u16<<<blocks_for(n, 256), 256, 0, s>>>(in, idx, n, out);
  CG_LAUNCH_CHECK();
}

void launch_build_prefix_index(const DictView& d, const uint32_t* sorted_popc, uint32_t* T,
                               uint32_t* F, cudaStream_t s) {
  k_prefix_index_empty<<<blocks_for(d.ell + 1, 128), 128, 0, s>>>(d, T);
  CG_LAUNCH_CHECK();
  if (d.n_cells > 0) {
    k_prefix_index<<<blocks_for(d.n_cells, 256), 256, 0, s>>>(d, sorted_popc, T, F);
    CG_LAUNCH_CHECK();
  }
}

}  // namespace cgk
