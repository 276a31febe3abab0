// small.cu -- the whole path (a1 pack, a2 sort, a3 dedupe, a6 probes, a7
// canonical edges) in ONE CTA for small inputs: n <= 2048 rows, ell <= 256.
//
// At these sizes (CFG1: 1000 vectors; the paper's range starts at thousands
// of vectors) the multi-kernel path is latency-bound: ~15 launches
// and three host round trips for ~1 MB of work.  Here the rows live in
// shared memory from pack to output:
//   a1  thread per (row, word): bytes -> MSB-first words, bytes in {0,1}
//       checked (G5);
//   a2  bitonic sort of the rows (padded to a power of two with all-ones
//       rows, which sort last) = canonical order (G1);
//   a3  first row of each run of equal rows -> cell index by a block scan
//       (P:274);
//   a6  per cell, every zero bit k <= lcp(V_i, V_{i+1}) (exact pruning, G3:
//       0->1 flips only) is looked up by binary search among the later cells
//       (the targets are larger than V_i; Alg. 4's lookup);
//   a7  counts per cell, a block scan, then the same loop writes each cell's
//       hits at its offset, flips from the least significant candidate up =
//       ascending j: the list comes out in canonical (i, j) order (G4).
// One launch and one host read-back of (n_c, m, error) per build.
#include "kernels.cuh"

namespace cgk {
namespace {

constexpr int kSmallMaxN = 2048;
constexpr int kSmallMaxW = 4;
constexpr int kSmallThreads = 1024;

#ifndef SMALL_CLK
#define SMALL_CLK 0
#endif
template <int W>
__global__ void __launch_bounds__(kSmallThreads, 1)
    k_small_build(const uint8_t* __restrict__ vecs, int n, int ell, int lcp_prune,
                  uint64_t* __restrict__ cells, uint64_t* __restrict__ edges,
                  int64_t* __restrict__ res) {
  extern __shared__ __align__(16) uint64_t sk[];  // [NP][W] rows
  __shared__ uint16_t uidx[kSmallMaxN];           // cell -> sorted row
  __shared__ uint32_t cnt[kSmallMaxN];            // hits per cell -> offsets
  __shared__ uint16_t stab[kSmallMaxN + 2];       // prefix index
  __shared__ uint32_t s_scan[33];
  __shared__ uint32_t s_bad;
  const int tid = threadIdx.x, nt = blockDim.x;
  int NP = 1;
  while (NP < n) NP <<= 1;
  if (tid == 0) s_bad = 0;
#if SMALL_CLK
  long long ck[6];
  ck[0] = clock64();
#define SCLK(q) ck[q] = clock64()
#else
#define SCLK(q)
#endif
  // ---- a1 pack: thread per (row, word), its <= 8 eight-byte chunks loaded
  // independently (one round trip); 8 bytes -> 8 bits by one multiply:
  // byte j (0/1) of x lands on bit 63 - j of x * 0x8040201008040201 (the
  // partial products sit on distinct bits, so no carries reach bits 56-63)
  const bool al8 = ((reinterpret_cast<uintptr_t>(vecs) | uintptr_t(ell)) & 7) == 0;
  uint64_t bad = 0;
  for (int t = tid; t < NP * W; t += nt) {
    const int r = t / W, w = t - r * W;
    uint64_t word = ~0ull;  // padding rows (r >= n) sort after every cell
    if (r < n) {
      word = 0;
      const uint8_t* p = vecs + int64_t(r) * ell + 64 * w;
      const int len = min(64, ell - 64 * w);
      uint64_t x[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        x[q] = 0;
        const int lq = min(8, len - 8 * q);
        if (lq == 8 && al8) {
          x[q] = *reinterpret_cast<const uint64_t*>(p + 8 * q);
        } else {
          for (int j = 0; j < lq; ++j) x[q] |= uint64_t(p[8 * q + j]) << (8 * j);
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        bad |= x[q] & ~0x0101010101010101ull;
        word |= ((x[q] * 0x8040201008040201ull) >> 56) << (56 - 8 * q);
      }
    }
    sk[t] = word;
  }
  if (bad) atomicOr(&s_bad, 1u);
  __syncthreads();
  SCLK(1);
  // ---- a2 bitonic sort, rows compared as W-word unsigned sequences
  for (int k = 2; k <= NP; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < NP; i += nt) {
        const int ixj = i ^ j;
        if (ixj > i) {
          uint64_t* A = sk + i * W;
          uint64_t* B = sk + ixj * W;
          int c = 0;
#pragma unroll
          for (int w = 0; w < W; ++w)
            if (c == 0) c = A[w] < B[w] ? -1 : (A[w] > B[w] ? 1 : 0);
          const bool up = (i & k) == 0;
          if (up ? c > 0 : c < 0) {
#pragma unroll
            for (int w = 0; w < W; ++w) {
              const uint64_t x = A[w];
              A[w] = B[w];
              B[w] = x;
            }
          }
        }
      }
      __syncthreads();
    }
  }
  SCLK(2);
  // ---- a3 dedupe: rows 2*tid, 2*tid + 1
  auto differs = [&](int i) -> uint32_t {
    if (i >= n) return 0u;
    if (i == 0) return 1u;
    uint32_t d = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) d |= sk[i * W + w] != sk[(i - 1) * W + w];
    return d;
  };
  const int i0 = 2 * tid;
  const uint32_t f0 = differs(i0), f1 = differs(i0 + 1);
  uint32_t nc_u = 0;
  const uint32_t ex = block_excl_scan(f0 + f1, s_scan, &nc_u);
  if (f0) uidx[ex] = uint16_t(i0);
  if (f1) uidx[ex + f0] = uint16_t(i0 + 1);
  __syncthreads();
  const int nc = int(nc_u);
  auto row = [&](int c) -> const uint64_t* { return sk + int(uidx[c]) * W; };
  // ---- a5 prefix index over the cells: T[x] = first cell whose top b bits
  // are >= x, b = floor(log2 n_c) (1-2 cells per bucket)
  int b = 0;
  while ((nc >> (b + 1)) >= 1) ++b;
  auto pre = [&](int c) -> int { return b ? int(row(c)[0] >> (64 - b)) : 0; };
  for (int c = tid; c < nc; c += nt) {
    const int x = pre(c), xp = c ? pre(c - 1) : -1;
    for (int q = xp + 1; q <= x; ++q) stab[q] = uint16_t(c);
    if (c == nc - 1)
      for (int q = x + 1; q <= (1 << b); ++q) stab[q] = uint16_t(nc);
  }
  __syncthreads();
  SCLK(3);
  // ---- a6 + a7: count, scan, write
  uint32_t m_u = 0;
  for (int pass = 0; pass < 2; ++pass) {
    for (int c = tid; c < nc; c += nt) {
      const uint64_t* V = row(c);
      int kmax = -1;
      if (!lcp_prune) {
        kmax = ell - 1;
      } else if (c + 1 < nc) {
        const uint64_t* N = row(c + 1);
        int l = -1;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const uint64_t x = V[w] ^ N[w];
          if (l < 0 && x) l = 64 * w + __clzll(x);
        }
        kmax = min(l, ell - 1);
      }
      uint32_t h = 0;
      const uint32_t base = pass ? cnt[c] : 0u;
      // zero bits k <= kmax, word by word from the last, least significant
      // first: largest k first = ascending targets
      for (int fw = kmax >> 6; fw >= 0; --fw) {
        uint64_t z = ~V[fw];
        if (fw == (kmax >> 6)) z &= ~0ull << (63 - (kmax & 63));
        while (z) {
        const uint64_t bm = z & (~z + 1);
        z ^= bm;
        // the target's prefix bucket; short buckets are scanned
        const uint64_t t0 = V[0] | (fw == 0 ? bm : 0ull);
        const int xb = b ? int(t0 >> (64 - b)) : 0;
        int lo = stab[xb], len = int(stab[xb + 1]) - lo;
        if (len <= 8) {
          int r = lo;
          for (; r < lo + len; ++r) {
            const uint64_t* R = row(r);
            int cmp = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) {
              const uint64_t tv = V[w] | (w == fw ? bm : 0ull);
              if (cmp == 0) cmp = R[w] < tv ? -1 : (R[w] > tv ? 1 : 0);
            }
            if (cmp >= 0) break;
          }
          lo = r;
          len = 0;
          if (lo >= int(stab[xb + 1])) lo = nc;  // not in the bucket
        }
        while (len > 0) {
          const int half = len >> 1;
          const uint64_t* R = row(lo + half);
          int cmp = 0;
#pragma unroll
          for (int w = 0; w < W; ++w) {
            const uint64_t tv = V[w] | (w == fw ? bm : 0ull);
            if (cmp == 0) cmp = R[w] < tv ? -1 : (R[w] > tv ? 1 : 0);
          }
          if (cmp < 0) {
            lo += half + 1;
            len -= half + 1;
          } else {
            len = half;
          }
        }
        if (lo < nc) {
          const uint64_t* R = row(lo);
          bool eq = true;
#pragma unroll
          for (int w = 0; w < W; ++w) eq = eq && R[w] == (V[w] | (w == fw ? bm : 0ull));
          if (eq) {
            if (pass) edges[base + h] = uint64_t(uint32_t(c)) | (uint64_t(uint32_t(lo)) << 32);
            ++h;
          }
        }
        }
      }
      if (!pass) cnt[c] = h;
    }
    __syncthreads();
    if (!pass) {
      const uint32_t a = i0 < nc ? cnt[i0] : 0u, b2 = i0 + 1 < nc ? cnt[i0 + 1] : 0u;
      const uint32_t e0 = block_excl_scan(a + b2, s_scan, &m_u);
      if (i0 < nc) cnt[i0] = e0;
      if (i0 + 1 < nc) cnt[i0 + 1] = e0 + a;
      __syncthreads();
    }
  }
  SCLK(4);
  // ---- outputs
  for (int t = tid; t < nc * W; t += nt) cells[t] = sk[int(uidx[t / W]) * W + t % W];
  if (tid == 0) {
    res[0] = nc;
    res[1] = int64_t(m_u);
    res[2] = s_bad;
#if SMALL_CLK
    for (int q = 1; q < 5; ++q) res[2 + q] = ck[q] - ck[q - 1];
#endif
  }
}

}  // namespace

bool small_build_ok(int64_t n, int ell) {
  return n >= 1 && n <= kSmallMaxN && (ell + 63) / 64 <= kSmallMaxW;
}

void launch_small_build(const uint8_t* vecs, int64_t n, int ell, int lcp_prune, uint64_t* cells,
                        uint64_t* edges, int64_t* res, cudaStream_t s) {
  const int W = (ell + 63) / 64;
  int NP = 1;
  while (NP < n) NP <<= 1;
  const size_t smem = size_t(NP) * W * 8;
#define CG_SMALL(WW)                                                                          \
  do {                                                                                        \
    CG_CUDA(cudaFuncSetAttribute(k_small_build<WW>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                 int(kSmallMaxN * kSmallMaxW * 8)));                          \
    k_small_build<WW><<<1, kSmallThreads, smem, s>>>(vecs, int(n), ell, lcp_prune, cells,     \
                                                     edges, res);                             \
  } while (0)
  switch (W) {
    case 1: CG_SMALL(1); break;
    case 2: CG_SMALL(2); break;
    case 3: CG_SMALL(3); break;
    default: CG_SMALL(4); break;
  }
#undef CG_SMALL
  CG_LAUNCH_CHECK();
}

}  // namespace cgk
