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
// k_pack_sweep (the sweep path) also does the MSD sort's first partition.
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

// ---------------------------------------------------------------- pack + first MSD partition
// The MSD sort's first pass fused into the pack ("sweep"
// path; ell = 64 W, W <= 2, 16-byte aligned input).  A CTA of kSweepThreads
// threads packs a tile of kSweepRows rows into shared memory -- fully
// coalesced 16-byte loads (a warp reads 512 contiguous bytes per
// instruction), each chunk's 16 bits OR-combined over the 4 lanes that hold
// one 64-bit word -- then ranks the rows by the top byte of word 0 with
// shared atomics (the order inside a digit is free: every top-16-bit bucket
// is sorted completely by the bucket pass), reserves each digit's run in
// that digit's region with ONE global atomicAdd per (tile, digit) (no
// look-back, no histogram pass: region d is over-allocated to capr rows),
// reorders the tile in shared memory and writes the runs.  A region that
// would overflow sets *ovf and is clipped; the caller then re-packs and
// takes the exact path.
#ifndef SWEEP_NT
#define SWEEP_NT 256  // threads per CTA (A/B at C5: 512 x 2 CTAs 1.66 ms, 256 x 4 1.54, 256 x 3 1.71)
#endif
#ifndef SWEEP_RPT
#define SWEEP_RPT 8  // rows per thread in the rank phase
#endif
#ifndef SWEEP_MINB
#define SWEEP_MINB 4  // resident CTAs per SM (register bound: 64 registers)
#endif
#ifndef SWEEP_U
#define SWEEP_U 8  // 16-byte loads in flight per thread
#endif
constexpr int kSweepThreads = SWEEP_NT;
constexpr int kSweepRPT = SWEEP_RPT;
constexpr int kSweepRows = kSweepThreads * kSweepRPT;

template <int W>
__global__ void __launch_bounds__(kSweepThreads, SWEEP_MINB) k_pack_sweep(
    const uint8_t* __restrict__ vecs, int64_t n, uint64_t* __restrict__ regions, uint32_t capr,
    uint32_t* __restrict__ rcnt, uint32_t* __restrict__ err, uint32_t* __restrict__ ovf) {
  constexpr int C = 4 * W;  // 16-byte chunks per row (ell = 64 W bytes)
  constexpr int TR = kSweepRows, NT = kSweepThreads;
  constexpr int STEPS = TR * C / NT;  // chunk loads per thread
  constexpr int U = SWEEP_U;          // loads in flight per thread
  static_assert(STEPS % U == 0, "sweep tile");
  extern __shared__ __align__(16) uint64_t sk[];  // [TR][W]
  __shared__ uint32_t hc[256], dex[256], lim[256], s_scan[33];
  __shared__ uint64_t gb[256];
  const int tid = threadIdx.x;
  const int64_t r0 = int64_t(blockIdx.x) * TR;
  const int rows = int(min(int64_t(TR), n - r0));
  const int nch = rows * C;
  if (tid < 256) hc[tid] = 0u;
  const uint4* src = reinterpret_cast<const uint4*>(vecs + r0 * (64 * W));
  uint64_t bad = 0;
  const int j = tid & (C - 1);        // chunk of the row this thread reads (NT % C == 0)
  const int sh = 48 - 16 * (j & 3);   // its 16 bits inside the word
  for (int s0 = 0; s0 < STEPS; s0 += U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = (s0 + u) * NT + tid;
      // (cached loads: A/B at C5 1.527 vs 1.547 ms with evict-first __ldcs)
      v[u] = c < nch ? __ldg(src + c) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = (s0 + u) * NT + tid;
      const uint64_t lo = (uint64_t(v[u].y) << 32) | v[u].x;
      const uint64_t hi = (uint64_t(v[u].w) << 32) | v[u].z;
      bad |= (lo | hi) & kHi7;
      uint64_t p = (uint64_t(bits8_msb(lo)) << (sh + 8)) | (uint64_t(bits8_msb(hi)) << sh);
      p |= __shfl_xor_sync(kFull, p, 1);
      p |= __shfl_xor_sync(kFull, p, 2);
      if ((tid & 3) == 0 && c < nch) sk[(c / C) * W + (j >> 2)] = p;
    }
  }
  __syncthreads();
  uint64_t key[kSweepRPT][W];
  uint32_t rk[kSweepRPT];
#pragma unroll
  for (int k = 0; k < kSweepRPT; ++k) {
    const int r = k * NT + tid;
    rk[k] = 0u;
#pragma unroll
    for (int w = 0; w < W; ++w) key[k][w] = r < rows ? sk[r * W + w] : 0ull;
    if (r < rows) rk[k] = atomicAdd(&hc[uint32_t(key[k][0] >> 56)], 1u);
  }
  __syncthreads();
  // digit d = tid (< 256): tile count, local start, region reservation
  const uint32_t c = tid < 256 ? hc[tid] : 0u;
  uint32_t tot;
  const uint32_t ex = block_excl_scan(c, s_scan, &tot);
  if (tid < 256) {
    uint32_t base = 0;
    if (c) {
      base = atomicAdd(&rcnt[tid], c);
      if (uint64_t(base) + c > capr) atomicOr(ovf, 1u);
    }
    dex[tid] = ex;
    gb[tid] = uint64_t(tid) * capr + base - ex;  // region row of local position ex + q = gb + ex + q
    lim[tid] = ex + (base < capr ? capr - base : 0u);  // local positions below lim fit
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kSweepRPT; ++k) {
    const int r = k * NT + tid;
    if (r < rows) {
      const uint32_t pos = dex[uint32_t(key[k][0] >> 56)] + rk[k];
#pragma unroll
      for (int w = 0; w < W; ++w) sk[pos * W + w] = key[k][w];
    }
  }
  __syncthreads();
  for (int q = tid; q < rows; q += NT) {
    const uint32_t d = uint32_t(sk[q * W] >> 56);
    if (uint32_t(q) < lim[d]) {
      const uint64_t g = gb[d] + uint64_t(q);
      if (W == 2) {
        *reinterpret_cast<ulonglong2*>(regions + 2 * g) =
            *reinterpret_cast<const ulonglong2*>(sk + 2 * q);
      } else {
        regions[g] = sk[q];
      }
    }
  }
  if (bad) atomicOr(err, 1u);
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

bool pack_sweep_ok(const uint8_t* vecs, int64_t n, int ell) {
  return (ell == 64 || ell == 128) && (reinterpret_cast<uintptr_t>(vecs) % 16) == 0 &&
         n < (int64_t(1) << 32);
}

int sweep_bits(int64_t n) {
  if (n <= (int64_t(1) << 18) || n > (int64_t(1) << 26)) return 0;
  int c = 0;
  while ((int64_t(1) << c) < n) ++c;  // ceil(log2 n)
  return std::min(8, std::max(1, c - 18));
}

uint32_t pack_sweep_capr(int64_t n) {
  // mean region + 1/16 + two tiles: uniform top bytes never come close
  // mean + 1/16 (+ 1/2 below 2^24 rows, where a sample screens skewed inputs
  // first and memory is no concern) + two tiles; even (16-byte bulk copies)
  const int64_t mean = (n + 255) / 256;
  const int64_t slack = n < (int64_t(1) << 24) ? mean / 2 : mean / 16;
  return uint32_t((mean + slack + 2 * kSweepRows + 1) & ~int64_t(1));
}

void launch_pack_sweep(const uint8_t* vecs, int64_t n, int ell, uint64_t* regions, uint32_t capr,
                       uint32_t* rcnt, uint32_t* err, uint32_t* ovf, cudaStream_t s) {
  const int W = ell / 64;
  const int64_t tiles = (n + kSweepRows - 1) / kSweepRows;
  const size_t smem = size_t(kSweepRows) * W * 8;
  CG_CUDA(cudaMemsetAsync(rcnt, 0, 256 * sizeof(uint32_t), s));
  if (W == 2) {
    CG_CUDA(cudaFuncSetAttribute(k_pack_sweep<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    k_pack_sweep<2><<<unsigned(tiles), kSweepThreads, smem, s>>>(vecs, n, regions, capr, rcnt, err, ovf);
  } else {
    CG_CUDA(cudaFuncSetAttribute(k_pack_sweep<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    k_pack_sweep<1><<<unsigned(tiles), kSweepThreads, smem, s>>>(vecs, n, regions, capr, rcnt, err, ovf);
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
