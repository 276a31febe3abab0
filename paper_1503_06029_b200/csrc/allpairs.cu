// allpairs.cu -- f3: the all-pairs methods of the paper on the GPU, as an
// independent in-GPU cross-check of the flip-probe path.
//
// The naive method compares every pair.  Alg. 1-2 add
// h anchors: d(x_a, x_j) is computed once for every anchor a < h and every
// vector j (ComputeDist), and a pair (i, j) is skipped when the triangle
// inequality d(x_i, x_j) >= |d(x_a, x_i) - d(x_a, x_j)| already
// exceeds 1 for some anchor (the sound form of the guard, DESIGN G15 /
// S:271); the rest are compared word by word with an early exit once the
// count passes 1.  Input is the canonical cell table (distinct vectors), so
// the output -- every pair at distance exactly 1, canonical (i, j) -- must
// equal the edge list of cg_build.
//
// B200 mapping: a CTA owns a 128 x 128 tile (i-block, j-block) of the upper
// triangle; the j-block's rows and anchor distances are staged in shared
// memory, each thread takes one i row (registers) against the 128 columns.
// Hits are appended with warp-aggregated atomics as (i << 32 | j) and the
// list is radix-sorted afterwards (the only ordering step).
#include "kernels.cuh"

namespace cgk {
namespace {

constexpr int kApTile = 128;
constexpr int kMaxAnchors = 8;

__global__ void k_anchor_dist(const uint64_t* __restrict__ cells, int64_t n, int W, int h,
                              uint16_t* __restrict__ ad) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
       j += int64_t(gridDim.x) * blockDim.x) {
    for (int a = 0; a < h; ++a) {
      int d = 0;
      for (int w = 0; w < W; ++w) d += __popcll(cells[j * W + w] ^ cells[int64_t(a) * W + w]);
      ad[j * h + a] = uint16_t(d);
    }
  }
}

template <int WC>  // WC > 0: words per row known at compile time
__global__ void __launch_bounds__(kApTile)
    k_allpairs(const uint64_t* __restrict__ cells, int64_t n, int Wrt, int h,
               const uint16_t* __restrict__ ad, int64_t nblk, uint64_t* __restrict__ out,
               uint64_t cap, unsigned long long* __restrict__ count,
               unsigned long long* __restrict__ compared) {
  extern __shared__ __align__(16) uint64_t sj[];  // [kApTile][W]
  __shared__ uint16_t sad[kApTile * kMaxAnchors];
  const int W = WC > 0 ? WC : Wrt;
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t lt = lanemask_lt();
  unsigned long long my_cmp = 0;
  // upper-triangle tile index -> (bi, bj), bi <= bj
  for (int64_t t = blockIdx.x; t < nblk * (nblk + 1) / 2; t += gridDim.x) {
    int64_t bi = int64_t((sqrt(8.0 * double(t) + 1.0) - 1.0) / 2.0);
    while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
    while (bi * (bi + 1) / 2 > t) --bi;
    const int64_t bj = t - bi * (bi + 1) / 2;  // bj <= bi: swap roles below
    const int64_t I0 = bj * kApTile, J0 = bi * kApTile;  // I0 <= J0
    __syncthreads();
    for (int q = tid; q < kApTile * W; q += kApTile) {
      const int64_t r = J0 + q / W;
      sj[q] = r < n ? cells[r * W + q % W] : 0ull;
    }
    for (int q = tid; q < kApTile * h; q += kApTile) {
      const int64_t r = J0 + q / h;
      sad[q] = r < n ? ad[r * h + q % h] : uint16_t(0);
    }
    __syncthreads();
    const int64_t i = I0 + tid;
    const bool vi = i < n;
    uint64_t xi[WC > 0 ? WC : 1];
    if (WC > 0)
#pragma unroll
      for (int w = 0; w < (WC > 0 ? WC : 1); ++w) xi[w] = vi ? cells[i * W + w] : 0ull;
    uint16_t ai[kMaxAnchors];
#pragma unroll
    for (int a = 0; a < kMaxAnchors; ++a) ai[a] = (vi && a < h) ? ad[i * h + a] : uint16_t(0);
    const int jlo = (I0 == J0) ? tid + 1 : 0;  // diagonal tile: j > i only
    const int jn = int(n - J0 < kApTile ? n - J0 : int64_t(kApTile));
    for (int jj = 0; jj < kApTile; ++jj) {
      bool hit = false;
      if (vi && jj >= jlo && jj < jn) {
        bool skip = false;
#pragma unroll
        for (int a = 0; a < kMaxAnchors; ++a)
          if (a < h) skip |= abs(int(ai[a]) - int(sad[jj * h + a])) > 1;
        if (!skip) {
          ++my_cmp;
          int d = 0;
          if (WC > 0) {
#pragma unroll
            for (int w = 0; w < (WC > 0 ? WC : 1); ++w) d += __popcll(xi[w] ^ sj[jj * WC + w]);
          } else {  // long rows: early exit once the distance exceeds 1
            for (int w = 0; w < W && d <= 1; ++w) d += __popcll(cells[i * W + w] ^ sj[jj * W + w]);
          }
          hit = d == 1;
        }
      }
      const uint32_t bal = __ballot_sync(kFull, hit);
      if (bal) {
        unsigned long long base = 0;
        if (lane == __ffs(bal) - 1) base = atomicAdd(count, (unsigned long long)__popc(bal));
        base = __shfl_sync(kFull, base, __ffs(bal) - 1);
        if (hit) {
          const unsigned long long pos = base + __popc(bal & lt);
          if (pos < cap) out[pos] = (uint64_t(i) << 32) | uint64_t(J0 + jj);
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) my_cmp += __shfl_xor_sync(kFull, my_cmp, o);
  if (lane == 0 && my_cmp) atomicAdd(compared, my_cmp);
}

}  // namespace

int allpairs_max_anchors() { return kMaxAnchors; }

// hits (unsorted (i << 32 | j)) -> returns the count (may exceed cap: rerun)
uint64_t launch_allpairs(const uint64_t* cells, int64_t n, int W, int h, uint64_t* out,
                         uint64_t cap, uint64_t* n_compared, cudaStream_t s) {
  DevBuf<uint16_t> ad(std::max<size_t>(1, size_t(n) * std::max(h, 1)), s);
  DevBuf<unsigned long long> ctr(2, s);
  CG_CUDA(cudaMemsetAsync(ctr.p, 0, 2 * sizeof(unsigned long long), s));
  if (h > 0) {
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 16);
    k_anchor_dist<<<unsigned(std::max<int64_t>(1, blocks)), 256, 0, s>>>(cells, n, W, h, ad.p);
    CG_LAUNCH_CHECK();
  }
  const int64_t nblk = (n + kApTile - 1) / kApTile;
  const int64_t tiles = nblk * (nblk + 1) / 2;
  const int grid = int(std::min<int64_t>(tiles, int64_t(num_sms()) * 16));
  const size_t smem = size_t(kApTile) * W * 8;
  auto go = [&](auto kern) {
    if (smem > (48u << 10))
      CG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<grid, kApTile, smem, s>>>(cells, n, W, h, ad.p, nblk, out, cap, ctr.p, ctr.p + 1);
  };
  switch (W) {
    case 1: go(k_allpairs<1>); break;
    case 2: go(k_allpairs<2>); break;
    case 4: go(k_allpairs<4>); break;
    default: go(k_allpairs<0>); break;
  }
  CG_LAUNCH_CHECK();
  unsigned long long* h2 = static_cast<unsigned long long*>(host_stage(2 * sizeof(unsigned long long)));
  CG_CUDA(cudaMemcpyAsync(h2, ctr.p, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaStreamSynchronize(s));
  if (n_compared) *n_compared = h2[1];
  return h2[0];
}

}  // namespace cgk
