// pack.cu -- a1: bit-pack the cell signatures.
//
// Input: uint8[n][ell], byte k of row r = x_r(k) in {0,1} ("the i-th bit of
// v_P is 1 iff P satisfies the inequality c_i"; the paper stores each
// vector "as a continuous array of bytes").  Output: u64[n][W],
// W = ceil(ell/64), bit k at word k/64, bit position 63-(k%64) (MSB-first),
// so unsigned word-by-word comparison is the canonical order (DESIGN G1) and
// pad bits are zero (G6).  Any byte > 1 raises *err (CG_EINPUT, G5).
//
// HBM-streaming kernel: one thread per output word reads the word's <= 64
// input bytes with 16-byte (ell % 16 == 0), 8-byte (ell % 8 == 0) or 1-byte
// loads, turns each group of 8 bytes into 8 MSB-first bits with one multiply
// (x * 0x8040201008040201 >> 56 places byte j at bit 7-j: the 64 partial
// products land on distinct bit positions, so there are no carries), and
// writes the word.  Consecutive threads read consecutive 64-byte spans.
#include "kernels.cuh"

namespace cgk {
namespace {

__device__ __forceinline__ uint32_t bits8_msb(uint64_t x) {
  return uint32_t((x * 0x8040201008040201ull) >> 56);
}

constexpr uint64_t kHi7 = 0xfefefefefefefefeull;

// Optionally (hist != nullptr) also counts the 8-bit digits dlo..7 of word 0
// (the top bits the MSD sort partitions on), run-length accumulated per
// thread so constant digits do not serialise shared-memory atomics; this
// saves the sort's separate histogram read of the keys.
//
// With tile_hist (the MSD sort's first one-sweep pass then needs no
// look-back): the CTA walks whole tiles of tile_rows rows (the sort's tiles)
// and also writes each tile's count of digit dlo, tile_hist[t][256].
template <int VEC>
__global__ void __launch_bounds__(256) k_pack(const uint8_t* __restrict__ vecs, int64_t n,
                                              int ell, int W, uint64_t* __restrict__ keys,
                                              uint32_t* __restrict__ err,
                                              uint32_t* __restrict__ hist, int dlo,
                                              uint32_t* __restrict__ tile_hist, int tile_rows) {
  __shared__ uint32_t sh[3][256];
  __shared__ uint32_t st[256];
  const int nd = hist ? 8 - dlo : 0;
  if (hist) {
    for (int i = threadIdx.x; i < 3 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
    __syncthreads();
  }
  uint32_t last[3] = {0, 0, 0}, cnt[3] = {0, 0, 0};
  const int64_t total = n * W;
  uint64_t bad = 0;
  const int64_t ntiles = tile_hist ? (n + tile_rows - 1) / tile_rows : 1;
  const int64_t twords = tile_hist ? int64_t(tile_rows) * W : total;
  // without tile_hist: one "tile" = all words, grid-strided over all CTAs
  for (int64_t t = tile_hist ? blockIdx.x : 0; t < ntiles; t += tile_hist ? gridDim.x : 1) {
  if (tile_hist) {
    st[threadIdx.x] = 0u;
    __syncthreads();
  }
  const int64_t g0 = t * twords, gend = min(total, g0 + twords);
  const int64_t gstep = tile_hist ? int64_t(blockDim.x) : int64_t(gridDim.x) * blockDim.x;
  for (int64_t g = g0 + (tile_hist ? 0 : int64_t(blockIdx.x) * blockDim.x) + threadIdx.x; g < gend;
       g += gstep) {
    const int64_t r = g / W;
    const int w = int(g - r * W);
    const int len = min(64, ell - 64 * w);
    const uint8_t* src = vecs + r * ell + 64 * w;
    uint64_t word = 0;
    if (VEC == 16) {
      const uint4* p = reinterpret_cast<const uint4*>(src);
      uint4 v[4];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (16 * c < len) v[c] = __ldcs(p + c);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (16 * c < len) {
          const uint64_t lo = (uint64_t(v[c].y) << 32) | v[c].x;
          const uint64_t hi = (uint64_t(v[c].w) << 32) | v[c].z;
          bad |= (lo | hi) & kHi7;
          word |= uint64_t(bits8_msb(lo)) << (56 - 16 * c);
          word |= uint64_t(bits8_msb(hi)) << (48 - 16 * c);
        }
      }
    } else if (VEC == 8) {
      const uint2* p = reinterpret_cast<const uint2*>(src);
      uint2 v[8];
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (8 * c < len) v[c] = __ldcs(p + c);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (8 * c < len) {
          const uint64_t x = (uint64_t(v[c].y) << 32) | v[c].x;
          bad |= x & kHi7;
          word |= uint64_t(bits8_msb(x)) << (56 - 8 * c);
        }
      }
    } else {
      for (int k = 0; k < len; ++k) {
        const uint8_t b = src[k];
        bad |= b & 0xfe;
        word |= uint64_t(b & 1) << (63 - k);
      }
    }
    keys[g] = word;
    if (tile_hist && w == 0) atomicAdd(&st[uint32_t(word >> (8 * dlo)) & 255u], 1u);
    if (nd && w == 0) {
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        if (d < nd) {
          const uint32_t bin = uint32_t(word >> (8 * (dlo + d))) & 255u;
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
  if (tile_hist) {
    __syncthreads();
    tile_hist[t * 256 + threadIdx.x] = st[threadIdx.x];
    __syncthreads();
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

__global__ void k_check_pad(const uint64_t* __restrict__ words, int64_t n, int W, uint64_t pad,
                            uint32_t* __restrict__ err) {
  uint64_t bad = 0;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x)
    bad |= words[r * W + W - 1] & pad;
  if (bad) atomicOr(err, 1u);
}

}  // namespace

void launch_pack(const uint8_t* vecs, int64_t n, int ell, uint64_t* keys, uint32_t* err,
                 cudaStream_t s, uint32_t* hist, int dlo, uint32_t* tile_hist, int tile_rows) {
  const int W = (ell + 63) / 64;
  const int64_t total = n * W;
  const int threads = 256;
  int64_t blocks = tile_hist ? (n + tile_rows - 1) / tile_rows : (total + threads - 1) / threads;
  blocks = std::min<int64_t>(blocks, int64_t(num_sms()) * 8);
  if (blocks < 1) blocks = 1;
  if (hist && (dlo < 5 || dlo > 7)) hist = nullptr;  // at most 3 top digits
  if (!hist) tile_hist = nullptr;
  const uintptr_t a = reinterpret_cast<uintptr_t>(vecs);
  if (ell % 16 == 0 && a % 16 == 0) {
    k_pack<16><<<unsigned(blocks), threads, 0, s>>>(vecs, n, ell, W, keys, err, hist, dlo, tile_hist, tile_rows);
  } else if (ell % 8 == 0 && a % 8 == 0) {
    k_pack<8><<<unsigned(blocks), threads, 0, s>>>(vecs, n, ell, W, keys, err, hist, dlo, tile_hist, tile_rows);
  } else {
    k_pack<1><<<unsigned(blocks), threads, 0, s>>>(vecs, n, ell, W, keys, err, hist, dlo, tile_hist, tile_rows);
  }
  CG_LAUNCH_CHECK();
}

void launch_check_pad(const uint64_t* words, int64_t n, int ell, uint32_t* err, cudaStream_t s) {
  if (ell % 64 == 0) return;
  const int W = (ell + 63) / 64;
  const uint64_t pad = ~uint64_t(0) >> (ell % 64);
  int64_t blocks = std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 8);
  k_check_pad<<<unsigned(std::max<int64_t>(1, blocks)), 256, 0, s>>>(words, n, W, pad, err);
  CG_LAUNCH_CHECK();
}

}  // namespace cgk
