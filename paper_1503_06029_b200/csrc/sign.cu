// sign.cu -- f1: on-device cell signatures, fused with the bit packing.
//
// "Each point P of the configuration space is assigned a binary vector v_P:
// the i-th bit of v_P is 1 iff P satisfies the inequality c_i"; the
// samples come from a point generator.  Here the constraints are
// half-spaces c_i: a_i . p + b_i >= 0 over R^dim (a tie counts as satisfied,
// DESIGN G12), points are f64[n][dim], planes f64[ell][dim + 1] =
// (a_i0 .. a_i(dim-1), b_i).  The value is evaluated in ONE fixed IEEE-754
// order, v = b; v = fma(a_t, p_t, v) for t = 0 .. dim-1 (DESIGN G21), so the
// CPU oracle (std::fma, same order) reproduces every bit exactly.  Inputs
// must be finite with magnitude <= 2^60 (then no value can overflow); any
// other input raises *err (CG_EINPUT).
//
// The output is the packed key layout of pack.cu (bit k at word k/64,
// position 63 - k%64), so the sort consumes it directly and the n*ell-byte
// signature matrix never exists (8.6 GB at C5).  One thread per point: it
// loads its point once (coalesced) and evaluates the planes word by word from
// shared memory (warp-uniform plane index: broadcast loads).  Like k_pack it
// can count the MSD sort's top digits of word 0 on the way.
#include "kernels.cuh"

namespace cgk {
namespace {

constexpr int kSignThreads = 256;
constexpr int kMaxDim = 16;
// |coordinate|, |coefficient| <= 2^60: the fma chain of <= 16 terms then
// stays below 2^125 in magnitude, far from overflow, so every value is finite
constexpr double kMaxMag = 1152921504606846976.0;  // 2^60

template <int DIM>  // DIM > 0: compile-time dimension; 0: runtime dim
__global__ void __launch_bounds__(kSignThreads)
    k_signatures(const double* __restrict__ pts, int64_t n, int dim_rt,
                 const double* __restrict__ planes, int ell, int W,
                 uint64_t* __restrict__ keys, uint32_t* __restrict__ err,
                 uint32_t* __restrict__ hist, int dlo, int planes_in_smem) {
  extern __shared__ __align__(16) double spl[];
  __shared__ uint32_t sh[3][256];
  const int dim = DIM > 0 ? DIM : dim_rt;
  const int pl = dim + 1;
  const double* P = planes;
  bool bad = false;
  // inputs bounded by kMaxMag keep every fma chain finite (checked once per
  // value instead of per result)
  for (int i = threadIdx.x; i < ell * pl; i += blockDim.x) {
    const double c = planes[i];
    bad |= !(fabs(c) <= kMaxMag);
    if (planes_in_smem) spl[i] = c;
  }
  if (planes_in_smem) P = spl;
  const int nd = hist ? 8 - dlo : 0;
  if (hist)
    for (int i = threadIdx.x; i < 3 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  uint32_t last[3] = {0, 0, 0}, cnt[3] = {0, 0, 0};
  // thread per group of R consecutive points: all lanes of a warp evaluate
  // the same plane at the same time (shared-memory broadcast loads), and each
  // plane's coefficients are loaded once for R points (register blocking)
  constexpr int R = 4;
  const int64_t ngroups = (n + R - 1) / R;
  for (int64_t gq = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; gq < ngroups;
       gq += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r0 = gq * R;
    double p[R][DIM > 0 ? DIM : kMaxDim];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int64_t r = r0 + q < n ? r0 + q : n - 1;
#pragma unroll
      for (int t = 0; t < (DIM > 0 ? DIM : kMaxDim); ++t)
        if (t < dim) p[q][t] = __ldg(pts + r * dim + t);
    }
#pragma unroll
    for (int q = 0; q < R; ++q)
#pragma unroll
      for (int t = 0; t < (DIM > 0 ? DIM : kMaxDim); ++t)
        if (t < dim) bad |= !(fabs(p[q][t]) <= kMaxMag);
    for (int w = 0; w < W; ++w) {
      const int k0 = 64 * w, len = min(64, ell - k0);
      // bits shifted in MSB-first: plane k0 + j ends at position 63 - j
      uint32_t hi[R], lo[R];
#pragma unroll
      for (int q = 0; q < R; ++q) hi[q] = lo[q] = 0u;
#pragma unroll 4
      for (int j = 0; j < len; ++j) {
        const double* a = P + (k0 + j) * pl;
        double v[R];
#pragma unroll
        for (int q = 0; q < R; ++q) v[q] = a[dim];  // b_k
#pragma unroll
        for (int t = 0; t < (DIM > 0 ? DIM : kMaxDim); ++t) {
          if (t < dim) {
            const double at = a[t];
#pragma unroll
            for (int q = 0; q < R; ++q) v[q] = __fma_rn(at, p[q][t], v[q]);
          }
        }
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const uint32_t bit = v[q] >= 0.0 ? 1u : 0u;
          if (j < 32) hi[q] = 2u * hi[q] + bit;
          else lo[q] = 2u * lo[q] + bit;
        }
      }
      uint64_t word[R];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        // left-align a short last word (len < 64)
        const uint64_t wv = len > 32 ? (uint64_t(hi[q]) << (len - 32)) | lo[q] : uint64_t(hi[q]);
        word[q] = wv << (64 - len);
      }
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if (r0 + q < n) {
          keys[(r0 + q) * W + w] = word[q];
          if (nd && w == 0) {
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              if (d < nd) {
                const uint32_t bin = uint32_t(word[q] >> (8 * (dlo + d))) & 255u;
                if (bin != last[d]) {
                  if (cnt[d]) atomicAdd(&sh[d][last[d]], cnt[d]);
                  last[d] = bin;
                  cnt[d] = 0;
                }
                ++cnt[d];
              }
            }
          }
        }
      }
    }
  }
  if (bad) atomicOr(err, 1u);
  if (hist) {
#pragma unroll
    for (int d = 0; d < 3; ++d)
      if (d < nd && cnt[d]) atomicAdd(&sh[d][last[d]], cnt[d]);
    __syncthreads();
    for (int i = threadIdx.x; i < nd * 256; i += blockDim.x) {
      const uint32_t v = (&sh[0][0])[i];
      if (v) atomicAdd(&hist[i], v);
    }
  }
}

}  // namespace

int signatures_max_dim() { return kMaxDim; }

void launch_signatures(const double* pts, int64_t n, int dim, const double* planes, int ell,
                       uint64_t* keys, uint32_t* err, cudaStream_t s, uint32_t* hist, int dlo) {
  const int W = (ell + 63) / 64;
  int64_t blocks = std::min<int64_t>((n + 4 * kSignThreads - 1) / (4 * kSignThreads),
                                     int64_t(num_sms()) * 8);
  if (blocks < 1) blocks = 1;
  if (hist && (dlo < 5 || dlo > 7)) hist = nullptr;
  const size_t pbytes = size_t(ell) * (dim + 1) * sizeof(double);
  const int in_smem = pbytes <= (96u << 10) ? 1 : 0;  // else read through L1
  const size_t smem = in_smem ? pbytes : 0;
  auto go = [&](auto kern) {
    if (smem > (48u << 10))
      CG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<unsigned(blocks), kSignThreads, smem, s>>>(pts, n, dim, planes, ell, W, keys, err, hist,
                                                      dlo, in_smem);
  };
  switch (dim) {
    case 2: go(k_signatures<2>); break;
    case 3: go(k_signatures<3>); break;
    case 4: go(k_signatures<4>); break;
    default: go(k_signatures<0>); break;
  }
  CG_LAUNCH_CHECK();
}

}  // namespace cgk
