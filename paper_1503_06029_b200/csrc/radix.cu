// radix.cu -- the radix sort engine (a2 cell sort, a4 popcount layering, a7
// canonical edge sort).
//
// "As these vectors are binary, the sorting can clearly be done in O(n*ell)
// time, using the radix sort algorithm".  The paper does not say
// which radix sort.  This file implements, for sm_100a:
//
// (1) a stable one-sweep LSD pass engine over 8-bit digits:
//   * one histogram kernel reads the keys once and counts the digits of all
//     requested passes (run-length accumulated in registers so constant
//     digits do not serialise shared-memory atomics); passes whose histogram
//     is a single bucket are skipped (pad bits, small indices, narrow
//     popcounts);
//   * each pass: a CTA takes a tile by atomic ticket, loads it warp-striped
//     (coalesced), ranks digits per warp with __match_any_sync, publishes
//     per-digit tile counts through a decoupled look-back, reorders the tile
//     in shared memory by digit and writes each digit run contiguously.
//   Keys are u32, u64 or 128-bit rows (ulonglong2: .x = word 0, the most
//   significant); digits are taken from the most significant word.
//
// (2) the cell sort for W <= 2 words (MSD fast path): LSD passes over only
//   the top B bits move the whole keys into 2^B prefix buckets (the first
//   pass takes its tile offsets from the pack kernel's per-tile digit
//   counts, so it needs no look-back); the bucket starts are found by one
//   binary search per bucket; each bucket (~2^10 keys for uniform keys) is
//   then sorted in shared memory by a rank-in-digit pass (k_bucket_rank: the
//   first varying bit, an 11-bit digit count, ranks within a digit) with the
//   dedupe of a3 fused in.  Skewed buckets go to a stable byte-pass kernel
//   (k_bucket_sort); a bucket larger than its capacity makes the caller fall
//   back to the full LSD sort (skewed data), which is always correct.
//
// (3) the multi-word LSD (W > 2): per word (least significant first) a
//   stable sort of (word, u32 row index) pairs, then a row gather.
//
// (4) the sweep path (W <= 2, ell = 64/128, 2^18 < n <= 2^26; DESIGN
//   section 6): the pack kernel (pack.cu: k_pack_sweep) already moved the
//   rows into 256 over-allocated top-byte regions; k_region_sweep splits
//   each region by the next B2 bits into slots of ~2^10 rows (one atomicAdd
//   per tile and slot, no look-back: the order inside a slot is free), and
//   k_bucket_rank reads each slot and writes its bucket sorted, deduplicated
//   and -- for the global dictionary -- with its slices of the prefix index
//   T and filter F.  A region or slot overflow (skewed top bits) makes the
//   caller re-run the exact path.
#include <algorithm>
#include <vector>

#include "kernels.cuh"

namespace cgk {
namespace {

constexpr int kRadix = 256;
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;

template <class K>
struct KT;
template <>
struct KT<uint32_t> {
  __device__ __forceinline__ static uint64_t top(const uint32_t& k) { return k; }
  __device__ __forceinline__ static uint32_t zero_val() { return 0; }
};
template <>
struct KT<uint64_t> {
  __device__ __forceinline__ static uint64_t top(const uint64_t& k) { return k; }
};
template <>
struct KT<ulonglong2> {
  __device__ __forceinline__ static uint64_t top(const ulonglong2& k) { return k.x; }
};

template <class K>
__device__ __forceinline__ uint32_t digit_of(const K& k, int shift) {
  return uint32_t(KT<K>::top(k) >> shift) & 255u;
}

#ifndef OS_IPT16
#define OS_IPT16 12  // 16-byte keys per thread and one-sweep tile
#endif
#ifndef OS_MINB
#define OS_MINB 3  // resident one-sweep CTAs per SM (register bound)
#endif
template <class K, bool V>
struct TileCfg {
  static constexpr int IPT = sizeof(K) == 16 ? OS_IPT16 : (V ? 12 : 16);
  static constexpr int TILE = kSortThreads * IPT;
  static constexpr size_t SMEM = size_t(TILE) * (sizeof(K) + (V ? 4 : 0));
};

// hist[(d - dlo) * 256 + bin] for digits d in [dlo, dhi) of the top word
template <class K>
__global__ void __launch_bounds__(256) k_digit_hist(const K* __restrict__ keys, int64_t n,
                                                    int dlo, int dhi, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[8][kRadix];
  const int nd = dhi - dlo;
  for (int i = threadIdx.x; i < 8 * kRadix; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  uint32_t last[8], cnt[8];
#pragma unroll
  for (int d = 0; d < 8; ++d) {
    last[d] = 0;
    cnt[d] = 0;
  }
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t k = KT<K>::top(keys[i]);
#pragma unroll
    for (int d = 0; d < 8; ++d) {
      if (d < nd) {
        const uint32_t b = uint32_t(k >> (8 * (d + dlo))) & 255u;
        if (b != last[d]) {
          if (cnt[d]) atomicAdd(&h[d][last[d]], cnt[d]);
          last[d] = b;
          cnt[d] = 0;
        }
        ++cnt[d];
      }
    }
  }
#pragma unroll
  for (int d = 0; d < 8; ++d)
    if (d < nd && cnt[d]) atomicAdd(&h[d][last[d]], cnt[d]);
  __syncthreads();
  for (int i = threadIdx.x; i < nd * kRadix; i += blockDim.x) {
    const uint32_t v = (&h[0][0])[i];
    if (v) atomicAdd(&hist[i], v);
  }
}

#ifndef MW_PREFIX32
#define MW_PREFIX32 1  // W > 2: sort on (32-bit prefix, index) first (4 passes)
#endif
#ifndef OS_UNSTABLE1
#define OS_UNSTABLE1 1
#endif
template <class K, bool V>
__global__ void __launch_bounds__(kSortThreads, OS_MINB)
    k_onesweep(const K* __restrict__ kin, K* __restrict__ kout, const uint32_t* __restrict__ vin,
               uint32_t* __restrict__ vout, int64_t n, int shift,
               const uint32_t* __restrict__ bucket_base, uint64_t* status,
               uint32_t* tile_counter, uint32_t epoch,
               const uint32_t* __restrict__ tile_pre) {
  constexpr int IPT = TileCfg<K, V>::IPT;
  constexpr int TILE = TileCfg<K, V>::TILE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* skeys = reinterpret_cast<K*>(smem_raw);
  uint32_t* svals = reinterpret_cast<uint32_t*>(smem_raw + size_t(TILE) * sizeof(K));
  __shared__ uint32_t wcnt[kSortWarps][kRadix];
  __shared__ uint32_t s_dexcl[kRadix];
  __shared__ uint32_t s_gbase[kRadix];
  __shared__ uint32_t s_scan[33];
  __shared__ uint32_t s_tile;

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < kSortWarps * kRadix; i += kSortThreads) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * TILE;
  const int64_t wbase = base + int64_t(w) * 32 * IPT;

  K key[IPT];
  uint32_t val[IPT];
  uint32_t rank[IPT];
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int64_t g = wbase + i * 32 + lane;
    if (g < n) {
      key[i] = kin[g];
      if (V) val[i] = vin ? vin[g] : uint32_t(g);
    } else {
      key[i] = K{};
      val[i] = 0;
    }
  }
  // warp-level stable ranking: items are visited in index order
  // (item i of every lane precedes item i+1; lanes in order within an item).
  // The first LSD pass (tile_pre given) needs no stability -- the input
  // order is arbitrary -- so a shared atomic per item ranks it there
  const uint32_t lt = lanemask_lt();
  if (OS_UNSTABLE1 && tile_pre) {
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const bool valid = wbase + i * 32 + lane < n;
      if (valid) rank[i] = atomicAdd(&wcnt[w][digit_of(key[i], shift)], 1u);
    }
  } else
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const bool valid = wbase + i * 32 + lane < n;
    const uint32_t d = valid ? digit_of(key[i], shift) : 256u;
    const uint32_t peers = __match_any_sync(kFull, d);
    uint32_t prev = 0;
    if (valid) prev = wcnt[w][d];
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) wcnt[w][d] = prev + __popc(peers);
    __syncwarp();
    rank[i] = prev + __popc(peers & lt);
  }
  __syncthreads();
  // thread tid owns digit tid: warp-exclusive prefixes and the tile total
  uint32_t total = 0;
#pragma unroll
  for (int ww = 0; ww < kSortWarps; ++ww) {
    const uint32_t c = wcnt[ww][tid];
    wcnt[ww][tid] = total;
    total += c;
  }
  // earlier tiles' count of digit tid: precomputed (the pack kernel counted
  // this pass's digit per tile) or by decoupled look-back
  const uint32_t excl_tiles = tile_pre ? tile_pre[tile * kRadix + tid]
                                       : lookback(status, tile, kRadix, tid, total, epoch);
  uint32_t tile_n_u;
  const uint32_t dex = block_excl_scan(total, s_scan, &tile_n_u);
  s_dexcl[tid] = dex;
  s_gbase[tid] = bucket_base[tid] + excl_tiles - dex;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const bool valid = wbase + i * 32 + lane < n;
    if (valid) {
      const uint32_t d = digit_of(key[i], shift);
      const uint32_t pos = s_dexcl[d] + wcnt[w][d] + rank[i];
      skeys[pos] = key[i];
      if (V) svals[pos] = val[i];
    }
  }
  __syncthreads();
  const int tile_n = int(tile_n_u);
  for (int j = tid; j < tile_n; j += kSortThreads) {
    const K k = skeys[j];
    const uint32_t d = digit_of(k, shift);
    const uint32_t gp = s_gbase[d] + uint32_t(j);
    kout[gp] = k;
    if (V) vout[gp] = svals[j];
  }
}

// Second partition of the sweep path (after k_pack_sweep): region x (top
// byte x) is split by the next byte into the buckets (x, d) of the top 16
// bits.  The tile structure of k_onesweep, but the order inside a bucket is
// free (the bucket pass sorts each bucket completely), so ranks come from
// shared atomics and each (tile, bucket) run is reserved in the bucket's
// slot of cap16 rows with one global atomicAdd -- no look-back.  Block
// x * tpr + t takes tile t of region x.
#ifndef RS_IPT
#define RS_IPT 12  // region sweep: 16-byte keys per thread and tile
#endif
#ifndef RS_MINB
#define RS_MINB 3  // region sweep: resident CTAs per SM
#endif
#ifndef RS_PERSIST
#define RS_PERSIST 1  // region sweep as a persistent kernel with TMA prefetch of the next tile
#endif
template <class K>
struct RsCfg {
  static constexpr int IPT = sizeof(K) == 16 ? RS_IPT : 2 * RS_IPT;
  static constexpr int TILE = kSortThreads * IPT;
  static constexpr size_t SMEM = size_t(TILE) * sizeof(K);
};
// the region sweep's digit: the B2 bits after the top byte
template <class K>
__device__ __forceinline__ uint32_t rs_digit(const K& k, int B2) {
  return uint32_t(KT<K>::top(k) >> (56 - B2)) & ((1u << B2) - 1u);
}
template <class K, int B2T>  // B2T: the digit width at compile time (8 at 2^26 rows), 0 = B2
__global__ void __launch_bounds__(kSortThreads, RS_MINB)
    k_region_sweep(const K* __restrict__ regions, uint32_t capr, const uint32_t* __restrict__ rcnt,
                   uint32_t tpr, K* __restrict__ slots, uint32_t cap16,
                   uint32_t* __restrict__ cnt16, uint32_t* __restrict__ ovf, int B2arg) {
  const int B2 = B2T ? B2T : B2arg;
  if (*ovf) return;  // a region overflowed in the pack: the caller re-runs the exact path
  constexpr int IPT = RsCfg<K>::IPT;
  constexpr int TILE = RsCfg<K>::TILE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* skeys = reinterpret_cast<K*>(smem_raw);
  __shared__ uint32_t wcnt[kSortWarps][kRadix];
  __shared__ uint32_t s_dexcl[kRadix], s_lim[kRadix], s_gbase[kRadix];
  __shared__ uint32_t s_scan[33];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t x = blockIdx.x / tpr, t = blockIdx.x % tpr;
  const uint32_t cnt = min(rcnt[x], capr);
  const uint32_t beg = t * uint32_t(TILE);
  if (beg >= cnt) return;  // (block-uniform)
  const int nt = int(min(uint32_t(TILE), cnt - beg));
  for (int i = tid; i < kSortWarps * kRadix; i += kSortThreads) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const K* kin = regions + size_t(x) * capr + beg;
  const int wb = w * 32 * IPT;
  K key[IPT];
  uint32_t rank[IPT];
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int g = wb + i * 32 + lane;
    key[i] = g < nt ? kin[g] : K{};
  }
#pragma unroll
  for (int i = 0; i < IPT; ++i)
    if (wb + i * 32 + lane < nt) rank[i] = atomicAdd(&wcnt[w][rs_digit(key[i], B2)], 1u);
  __syncthreads();
  uint32_t total = 0;
#pragma unroll
  for (int ww = 0; ww < kSortWarps; ++ww) {
    const uint32_t c = wcnt[ww][tid];
    wcnt[ww][tid] = total;
    total += c;
  }
  uint32_t tile_n;
  const uint32_t dex = block_excl_scan(total, s_scan, &tile_n);
  // the reservation's result is first used after the shared-memory scatter:
  // its L2 round trip overlaps the scatter
  uint32_t base = 0;
  const uint32_t q = (x << B2) | uint32_t(tid);
  if (total) base = atomicAdd(&cnt16[q], total);
  s_dexcl[tid] = dex;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    if (wb + i * 32 + lane < nt) {
      const uint32_t d = rs_digit(key[i], B2);
      skeys[s_dexcl[d] + wcnt[w][d] + rank[i]] = key[i];
    }
  }
  if (total && uint64_t(base) + total > cap16) atomicOr(ovf, 1u);
  s_gbase[tid] = q * cap16 + base - dex;  // slot row of local position dex + r: s_gbase + dex + r
  s_lim[tid] = dex + (base < cap16 ? cap16 - base : 0u);
  __syncthreads();
  for (int j = tid; j < nt; j += kSortThreads) {
    const K k = skeys[j];
    const uint32_t d = rs_digit(k, B2);
    if (uint32_t(j) < s_lim[d]) slots[s_gbase[d] + uint32_t(j)] = k;
  }
}

// off[q] = min(cnt16[q], cap) (then scanned), off[nb] = 0
__global__ void k_clip_counts(const uint32_t* __restrict__ cnt, int64_t nb, uint32_t cap,
                              uint32_t* __restrict__ off) {
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q <= nb;
       q += int64_t(gridDim.x) * blockDim.x)
    off[q] = q < nb ? min(cnt[q], cap) : 0u;
}

__global__ void k_iota(uint32_t* v, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    v[i] = uint32_t(i);
}

__global__ void k_gather_word(const uint64_t* __restrict__ keys, int W, int w,
                              const uint32_t* __restrict__ idx, int64_t n,
                              uint64_t* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = idx ? int64_t(idx[i]) : i;
    out[i] = keys[r * W + w];
  }
}

// ---------------------------------------------------------------- MSD fast path
// off[b] = first row whose top-B prefix is >= b, b in [0, 2^B]
// off[q] = first row whose top B bits are >= q, q in [0, 2^B] (off[2^B] = n),
// for keys sorted on their top B bits: one lower-bound binary search per
// bucket (thread per q), ~log2(n) dependent loads that neighbouring threads
// share through L1/L2 -- 22 us at C5 instead of 0.17 ms for streaming every
// key through the SMs to find the run heads
template <class K>
__global__ void k_bucket_bounds_search(const K* __restrict__ keys, int64_t n, int B,
                                       uint32_t* __restrict__ off, int skip = 0) {
  // buckets = bits [skip, skip + B) of the top word (the top `skip` bits are
  // common to all keys: a prefix chunk of the distributed merge)
  const int sh = 64 - B;
  const int64_t nb = int64_t(1) << B;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q <= nb;
       q += int64_t(gridDim.x) * blockDim.x) {
    int64_t lo = 0, len = n;
    while (len > 0) {
      const int64_t half = len >> 1;
      const uint64_t p = (KT<K>::top(__ldg(keys + lo + half)) << skip) >> sh;
      if (p < uint64_t(q)) {
        lo += half + 1;
        len -= half + 1;
      } else {
        len = half;
      }
    }
    off[q] = uint32_t(lo);
  }
}

// the same for rows of W words (word 0 carries the prefix)
__global__ void k_row_bounds_search(const uint64_t* __restrict__ rows, int64_t n, int W, int B,
                                    uint32_t* __restrict__ off) {
  const int sh = 64 - B;
  const int64_t nb = int64_t(1) << B;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q <= nb;
       q += int64_t(gridDim.x) * blockDim.x) {
    int64_t lo = 0, len = n;
    while (len > 0) {
      const int64_t half = len >> 1;
      const uint64_t p = __ldg(rows + (lo + half) * W) >> sh;
      if (p < uint64_t(q)) {
        lo += half + 1;
        len -= half + 1;
      } else {
        len = half;
      }
    }
    off[q] = uint32_t(lo);
  }
}

__device__ __forceinline__ bool key_less(const uint64_t& a, const uint64_t& b) { return a < b; }
__device__ __forceinline__ bool key_less(const ulonglong2& a, const ulonglong2& b) {
  return a.x < b.x || (a.x == b.x && a.y < b.y);
}
template <class K>
__device__ __forceinline__ K key_max();
template <>
__device__ __forceinline__ uint64_t key_max<uint64_t>() { return ~0ull; }
template <>
__device__ __forceinline__ ulonglong2 key_max<ulonglong2>() { return make_ulonglong2(~0ull, ~0ull); }

// byte P of the key, P = 0 the most significant byte of word 0
__device__ __forceinline__ uint32_t key_byte(const uint64_t& k, int P) {
  return uint32_t(k >> (56 - 8 * P)) & 255u;
}
__device__ __forceinline__ uint32_t key_byte(const ulonglong2& k, int P) {
  return P < 8 ? uint32_t(k.x >> (56 - 8 * P)) & 255u : uint32_t(k.y >> (56 - 8 * (P - 8))) & 255u;
}
// the key's bits from (MSB-first) position f on, left-aligned in 64 bits
__device__ __forceinline__ uint64_t key_bits_at(const uint64_t& k, int f) {
  return f < 64 ? (k << f) : 0ull;
}
__device__ __forceinline__ uint64_t key_bits_at(const ulonglong2& k, int f) {
  if (f == 0) return k.x;
  if (f < 64) return (k.x << f) | (k.y >> (64 - f));
  return f < 128 ? (k.y << (f - 64)) : 0ull;
}
__device__ __forceinline__ void key_andor(const uint64_t& k, uint64_t* a, uint64_t* o) {
  a[0] &= k;
  o[0] |= k;
}
__device__ __forceinline__ void key_andor(const ulonglong2& k, uint64_t* a, uint64_t* o) {
  a[0] &= k.x;
  o[0] |= k.x;
  a[1] &= k.y;
  o[1] |= k.y;
}

constexpr int kBktThreads = 256;
constexpr int kBktWarps = kBktThreads / 32;
constexpr int kBktMaxRounds = 64;

// One CTA sorts one prefix bucket at a time (persistent loop), entirely in
// shared memory.  The keys stay in place; u16 row indices move:
//   1. block AND/OR reduction finds the bytes that vary inside the bucket;
//   2. stable LSD passes over the two most significant varying bytes
//      (warp ranking with __match_any_sync, as in the global passes);
//   3. odd-even transposition rounds on the whole key finish the order
//      (ties of the two bytes are short runs: planted pairs, duplicates);
//      a bucket that does not settle within kBktMaxRounds, or is larger than
//      CAP, raises *overflow and the caller runs the full LSD sort instead.
template <class K, int MAXC>  // MAXC chunks of 32 rows per warp: CAP <= 8 * 32 * MAXC
__global__ void __launch_bounds__(kBktThreads)
    k_bucket_sort(K* __restrict__ keys, const uint32_t* __restrict__ off, int64_t nbuckets,
                  int CAP, int B, uint32_t* __restrict__ overflow, uint32_t* __restrict__ ucnt,
                  const uint32_t* __restrict__ blist, const uint32_t* __restrict__ nlist) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* s = reinterpret_cast<K*>(smem_raw);
  uint16_t* ia = reinterpret_cast<uint16_t*>(smem_raw + size_t(CAP) * sizeof(K));
  uint16_t* ib = ia + CAP;
  __shared__ uint32_t cnt[kBktWarps][kRadix];
  __shared__ uint32_t s_scan[33];
  __shared__ uint64_t s_red[2][kBktWarps][2];
  constexpr int NW = sizeof(K) / 8;
  constexpr int NBYTES = sizeof(K);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t lt = lanemask_lt();
  // blist: only the listed buckets (the ones k_bucket_rank handed over)
  const int64_t nwork = blist ? int64_t(*nlist) : nbuckets;
  for (int64_t x = blockIdx.x; x < nwork; x += gridDim.x) {
    const int64_t bk = blist ? int64_t(blist[x]) : x;
    const uint32_t lo = off[bk], hi = off[bk + 1];
    const int S = int(hi - lo);
    if (S <= 1) {
      if (ucnt && tid == 0) ucnt[bk] = uint32_t(S);
      continue;
    }
    if (S > CAP) {
      if (tid == 0) atomicOr(overflow, 1u);
      continue;
    }
    // ---- load + AND/OR of the key words
    uint64_t av[2] = {~0ull, ~0ull}, ov[2] = {0ull, 0ull};
    for (int i = tid; i < S; i += kBktThreads) {
      const K k = keys[lo + i];
      s[i] = k;
      ia[i] = uint16_t(i);
      key_andor(k, av, ov);
    }
#pragma unroll
    for (int w = 0; w < NW; ++w) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        av[w] &= __shfl_xor_sync(kFull, av[w], o);
        ov[w] |= __shfl_xor_sync(kFull, ov[w], o);
      }
    }
    if (lane == 0) {
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        s_red[0][wid][w] = av[w];
        s_red[1][wid][w] = ov[w];
      }
    }
    __syncthreads();
    uint64_t dif[2] = {0ull, 0ull};
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      uint64_t a = ~0ull, o = 0ull;
      for (int ww = 0; ww < kBktWarps; ++ww) {
        a &= s_red[0][ww][w];
        o |= s_red[1][ww][w];
      }
      dif[w] = a ^ o;  // bits that vary inside the bucket
    }
    int P1 = -1, P2 = -1;  // two most significant varying bytes
    for (int P = B / 8; P < NBYTES; ++P) {
      const uint64_t wv = dif[P >> 3];
      if ((wv >> (56 - 8 * (P & 7))) & 255u) {
        if (P1 < 0) P1 = P;
        else if (P2 < 0) P2 = P;
      }
    }
    uint16_t* cur = ia;
    uint16_t* nxt = ib;
    // ---- fast path: ONE unstable counting pass on the most significant
    // varying byte P1 (shared-memory atomics give the slot), then the thread
    // owning each digit insertion-sorts that digit's run on the whole key
    // (runs hold ~S/256 keys).  A run longer than 32 (skewed data) sends the
    // bucket to the stable two-byte path below.
    bool fast_done = false;
    if (P1 >= 0) {
      // 11-bit digit starting at the most significant varying bit: with
      // ~1024 keys per bucket the runs are 0-2 keys long
      constexpr int kDBits = 11, kBins = 1 << kDBits, kPer = kBins / kBktThreads;
      int f = 0;
      if (dif[0]) f = __clzll(dif[0]);
      else if (NW > 1) f = 64 + __clzll(dif[NW > 1 ? 1 : 0]);
      auto dig = [&](const K& k) -> uint32_t { return key_bits_at(k, f) >> (64 - kDBits); };
      uint32_t* h = &cnt[0][0];  // 8 * 256 = 2048 counters
#pragma unroll
      for (int q = 0; q < kPer; ++q) h[tid * kPer + q] = 0;
      __syncthreads();
      uint32_t rk[MAXC], dg[MAXC];
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        const int i = c * kBktThreads + tid;
        dg[c] = kBins;
        if (i < S) {
          dg[c] = dig(s[i]);
          rk[c] = atomicAdd(&h[dg[c]], 1u);
        }
      }
      __syncthreads();
      uint32_t rl[kPer];
      uint32_t loc = 0;
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        rl[q] = h[tid * kPer + q];
        loc += rl[q];
      }
      uint32_t all;
      const uint32_t rb0 = block_excl_scan(loc, s_scan, &all);
      uint32_t rbq[kPer];
      {
        uint32_t run = rb0;
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
          rbq[q] = run;
          h[tid * kPer + q] = run;
          run += rl[q];
        }
      }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        const int i = c * kBktThreads + tid;
        if (i < S) nxt[h[dg[c]] + rk[c]] = uint16_t(i);
      }
      __syncthreads();
      int too_long = 0;
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const uint32_t rb = rbq[q], len = rl[q];
        if (len > 32) {
          too_long = 1;
        } else {
          for (uint32_t a = rb + 1; a < rb + len; ++a) {
            const uint16_t v = nxt[a];
            const K kv = s[v];
            uint32_t z = a;
            while (z > rb && key_less(kv, s[nxt[z - 1]])) {
              nxt[z] = nxt[z - 1];
              --z;
            }
            nxt[z] = v;
          }
        }
      }
      if (!__syncthreads_or(too_long)) {
        cur = nxt;
        nxt = ia;
        fast_done = true;
      }
    }
    // ---- stable LSD passes: P2 then P1
    const int seg = ((S + kBktWarps * 32 - 1) / (kBktWarps * 32)) * 32;  // rows per warp
    for (int pass = 0; pass < 2 && !fast_done; ++pass) {
      const int P = pass == 0 ? P2 : P1;
      if (P < 0) continue;
      for (int i = tid; i < kBktWarps * kRadix; i += kBktThreads) (&cnt[0][0])[i] = 0;
      __syncthreads();
      uint32_t rk[MAXC], dg[MAXC];
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        const int i = wid * seg + c * 32 + lane;
        const bool in_seg = c * 32 < seg;
        const bool valid = in_seg && i < S;
        const uint32_t d = valid ? key_byte(s[cur[i]], P) : 256u;
        dg[c] = d;
        rk[c] = 0;
        if (in_seg) {  // warp-uniform
          const uint32_t peers = __match_any_sync(kFull, d);
          uint32_t prev = 0;
          if (valid) prev = cnt[wid][d];
          __syncwarp();
          if (valid && lane == __ffs(peers) - 1) cnt[wid][d] = prev + __popc(peers);
          __syncwarp();
          rk[c] = prev + __popc(peers & lt);
        }
      }
      __syncthreads();
      uint32_t tot = 0;
#pragma unroll
      for (int ww = 0; ww < kBktWarps; ++ww) {
        const uint32_t c = cnt[ww][tid];
        cnt[ww][tid] = tot;
        tot += c;
      }
      uint32_t all;
      const uint32_t dbase = block_excl_scan(tot, s_scan, &all);
#pragma unroll
      for (int ww = 0; ww < kBktWarps; ++ww) cnt[ww][tid] += dbase;
      __syncthreads();
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        const int i = wid * seg + c * 32 + lane;
        if (c * 32 < seg && i < S) nxt[cnt[wid][dg[c]] + rk[c]] = cur[i];
      }
      __syncthreads();
      uint16_t* t = cur;
      cur = nxt;
      nxt = t;
    }
    // ---- finish the order.  Keys are now sorted by (byte P1, byte P2), and
    // every byte before P2 other than P1 is constant, so keys that tie on
    // (P1, P2) form contiguous runs that only need sorting internally: the
    // thread at the head of each run insertion-sorts it on the whole key.
    // Runs longer than 32 (skewed data) fall back to odd-even rounds.
    int long_run = 0;
    if (P2 >= 0 && !fast_done) {
      auto tb = [&](int i) -> uint32_t {
        const K k = s[cur[i]];
        return (key_byte(k, P1) << 8) | key_byte(k, P2);
      };
      // find the run heads first (read-only), then sort after a barrier
      int hd[MAXC], hl[MAXC];
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        hl[c] = 0;
        const int i = c * kBktThreads + tid;
        hd[c] = i;
        if (i + 1 >= S) continue;
        const uint32_t bi = tb(i);
        if (bi != tb(i + 1) || (i > 0 && tb(i - 1) == bi)) continue;  // not a run head
        int j = i + 2;
        while (j < S && j - i <= 32 && tb(j) == bi) ++j;
        if (j - i > 32) long_run = 1;
        else hl[c] = j - i;
      }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        const int i = hd[c], j = hd[c] + hl[c];
        for (int a = i + 1; a < j; ++a) {
          const uint16_t v = cur[a];
          const K kv = s[v];
          int q = a;
          while (q > i && key_less(kv, s[cur[q - 1]])) {
            cur[q] = cur[q - 1];
            --q;
          }
          cur[q] = v;
        }
      }
    }
    const bool need_rounds = __syncthreads_or(long_run) != 0;
    bool settled = !need_rounds;
    for (int round = 0; need_rounds && round < kBktMaxRounds; ++round) {
      int changed = 0;
      for (int ph = 0; ph < 2; ++ph) {
        for (int i = 2 * tid + ph; i + 1 < S; i += 2 * kBktThreads) {
          const uint16_t a = cur[i], c = cur[i + 1];
          if (key_less(s[c], s[a])) {
            cur[i] = c;
            cur[i + 1] = a;
            changed = 1;
          }
        }
        __syncthreads();
      }
      if (!__syncthreads_or(changed)) {
        settled = true;
        break;
      }
    }
    if (!settled) {
      if (tid == 0) atomicOr(overflow, 1u);
      __syncthreads();
      continue;
    }
    if (!ucnt) {
      for (int i = tid; i < S; i += kBktThreads) keys[lo + i] = s[cur[i]];
    } else {
      // a3 fused: keep the first of each run of equal keys, written
      // compacted at the front of the bucket's range; ucnt[b] = unique count.
      // (Keys of different buckets differ in their prefix, so the first key
      // of a bucket is always new.)
      // chunk c, thread t -> sorted position c*256 + t (coalesced writes);
      // per-(chunk, warp) ballot counts, one scan over them in (c, w) order
      uint32_t* wc = &cnt[1][0];  // MAXC * 8 <= 128 counters
      uint32_t bl[MAXC];
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        const int i = c * kBktThreads + tid;
        const bool f = i < S && (i == 0 || key_less(s[cur[i - 1]], s[cur[i]]));
        bl[c] = __ballot_sync(kFull, f);
        if (lane == 0) wc[c * kBktWarps + wid] = __popc(bl[c]);
      }
      __syncthreads();
      if (tid < 32) {  // exclusive scan of MAXC * 8 counts by one warp
        constexpr int NWC = MAXC * kBktWarps;
        constexpr int PER = (NWC + 31) / 32;
        uint32_t v[PER], sum = 0;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
          v[q] = (tid * PER + q < NWC) ? wc[tid * PER + q] : 0u;
          sum += v[q];
        }
        uint32_t inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, inc, o);
          if (tid >= o) inc += y;
        }
        uint32_t run = inc - sum;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
          if (tid * PER + q < NWC) wc[tid * PER + q] = run;
          run += v[q];
        }
        if (tid == 31) ucnt[bk] = inc;
      }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        if ((bl[c] >> lane) & 1u) {
          const int i = c * kBktThreads + tid;
          keys[lo + wc[c * kBktWarps + wid] + __popc(bl[c] & lt)] = s[cur[i]];
        }
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- bucket rank sort
// The default bucket pass.  One CTA per prefix bucket (persistent loop), the
// NEXT bucket prefetched into the other half of a double buffer with
// cp.async while the current one is sorted:
//   1. AND/OR reduction -> f, the first bit that varies inside the bucket;
//   2. one counting pass on the 11-bit digit starting at f (shared atomics
//      give each key a slot inside its digit's range);
//   3. each key's final position = its digit's offset + the number of keys
//      of the same digit that are smaller (equal keys: lower index first);
//      digits hold ~S/2048 keys, so this is ~1 full-key compare per key;
//   4. (ucnt) first key of each run of equal keys kept, written compacted at
//      the front of the bucket's range, ucnt[b] = unique count.
// A digit holding more than kRankRun keys (skewed data) or a bucket larger
// than CAP is listed in blist for k_bucket_sort (stable byte passes).
constexpr int kRankRun = 24;
constexpr int kRankBits = 11;

template <class K>
__device__ __forceinline__ void cp_async_key(K* dst, const K* src) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  if (sizeof(K) == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// TMA bulk copies (cp.async.bulk, 1-D) completing on an mbarrier: one thread
// moves a whole bucket global -> shared; the CTA waits on the barrier phase.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

__device__ __forceinline__ bool key_eq(const uint64_t& a, const uint64_t& b) { return a == b; }
__device__ __forceinline__ bool key_eq(const ulonglong2& a, const ulonglong2& b) {
  return a.x == b.x && a.y == b.y;
}

// (a, ia) before (b, ib): key order, equal keys by index (branch-free)
__device__ __forceinline__ uint32_t key_before(const uint64_t& a, int ia, const uint64_t& b, int ib) {
  return uint32_t(a < b) | (uint32_t(a == b) & uint32_t(ia < ib));
}
__device__ __forceinline__ uint32_t key_before(const ulonglong2& a, int ia, const ulonglong2& b,
                                               int ib) {
  const uint32_t ex = uint32_t(a.x == b.x);
  return uint32_t(a.x < b.x) | (ex & uint32_t(a.y < b.y)) | (ex & uint32_t(a.y == b.y) & uint32_t(ia < ib));
}

#ifndef BKT_RCAP
#define BKT_RCAP 1152  // bucket-rank capacity (keys) for a ~1024-key mean bucket: 4 CTAs/SM
#endif
template <class K, int MAXC, bool PREF>
__global__ void __launch_bounds__(kBktThreads, PREF ? (MAXC <= 5 ? 4 : 3) : 4)
    k_bucket_rank(K* __restrict__ keys, const uint32_t* __restrict__ off, int64_t nbuckets, int CAP,
                  uint32_t* __restrict__ ucnt, uint32_t* __restrict__ blist,
                  uint32_t* __restrict__ nlist, const K* __restrict__ src, uint32_t scap,
                  uint32_t* __restrict__ Tix, uint32_t* __restrict__ Fix, int ib, int ibits,
                  const uint32_t* __restrict__ abort_flag) {
  // (sweep path) a region or slot overflowed: the caller re-runs the exact path
  if (abort_flag && *abort_flag) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // PREF: the next bucket is prefetched (cp.async) into a second buffer;
  // otherwise one buffer and more resident CTAs hide the load latency
  K* buf0 = reinterpret_cast<K*>(smem_raw);
  K* buf1 = PREF ? buf0 + CAP : buf0;
  uint16_t* nxt = reinterpret_cast<uint16_t*>(buf1 + CAP);
  uint16_t* pos_of = nxt + CAP;
  uint32_t* mlist = reinterpret_cast<uint32_t*>(pos_of + CAP);  // keys of digits holding > 2
  const uint32_t mcap = PREF ? uint32_t(CAP) : uint32_t(CAP / 2);
  constexpr int kBins = 1 << kRankBits, kPer = kBins / kBktThreads;
  // histogram slot of digit d: thread t owns digits kPer*t .. kPer*t+kPer-1
  // for the scan; storing digit d at (d % kPer) * 256 + d / kPer makes those
  // accesses conflict-free (one row per q, consecutive threads, banks)
  auto hx = [](uint32_t d) -> uint32_t {
    return d >= uint32_t(kBins) ? uint32_t(kBins) : (d % kPer) * kBktThreads + d / kPer;
  };
  __shared__ uint32_t s_nmany, s_eq;
  __shared__ __align__(16) uint32_t h[kBins + 1];
  __shared__ uint32_t s_scan[33];
  __shared__ uint64_t s_red[2][kBktWarps][2];
  __shared__ uint32_t s_wc[MAXC * kBktWarps];
  constexpr int NW = sizeof(K) / 8;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t lt = lanemask_lt();

  // 16-byte keys: the next bucket arrives by one TMA bulk copy per bucket
  // (mbarrier completion); 8-byte keys: per-thread cp.async
  constexpr bool BULK = PREF && sizeof(K) == 16;
  __shared__ uint64_t s_bar[2];
  if (BULK) {
    if (tid == 0) {
      mbar_init(&s_bar[0], 1);
      mbar_init(&s_bar[1], 1);
      mbar_fence_init();
    }
    __syncthreads();
  }
  // the bucket's input rows: in place (src == nullptr) or, on the sweep
  // path, bucket bk's slot of scap rows in src; the output always goes to
  // keys + off[bk]
  // (scap = 0: src has the output's bucket offsets -- the distributed merge)
  auto rsrc = [&](int64_t bk, uint32_t lo) -> const K* {
    return src ? (scap ? src + size_t(bk) * scap : src + lo) : keys + lo;
  };
  auto prefetch = [&](int64_t bk, K* dst, uint64_t* bar) {
    if (BULK) {
      if (tid == 0) {
        uint32_t S = 0, lo = 0;
        if (bk < nbuckets) {
          lo = off[bk];
          S = off[bk + 1] - lo;
        }
        if (S > 0 && S <= uint32_t(CAP)) {
          // the buffer was last written by the threads (generic proxy): order
          // those writes before the async-proxy (TMA) writes
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive_expect_tx(bar, S * uint32_t(sizeof(K)));
          bulk_g2s(dst, rsrc(bk, lo), S * uint32_t(sizeof(K)), bar);
        } else {
          mbar_arrive(bar);  // nothing to move: complete the phase
        }
      }
      return;
    }
    if (PREF && bk < nbuckets) {
      const uint32_t lo = off[bk];
      const int S = int(off[bk + 1] - lo);
      if (S <= CAP)
        for (int i = tid; i < S; i += kBktThreads) cp_async_key(dst + i, rsrc(bk, lo) + i);
    }
    cp_async_commit();
  };
  prefetch(blockIdx.x, buf0, &s_bar[0]);
  int it = 0;
  for (int64_t bk = blockIdx.x; bk < nbuckets; bk += gridDim.x, ++it) {
    K* s = (it & 1) ? buf1 : buf0;
    prefetch(bk + gridDim.x, (it & 1) ? buf0 : buf1, &s_bar[(it + 1) & 1]);
    if (BULK) {
      mbar_wait(&s_bar[it & 1], uint32_t(it >> 1) & 1u);  // use it/2 of this buffer
    } else {
      cp_async_wait1();
    }
    __syncthreads();
    const uint32_t lo = off[bk], hi = off[bk + 1];
    const int S = int(hi - lo);
    // a listed bucket is finished in place by the byte-pass kernel: on the
    // sweep path its rows are first copied to their output range
    // Fused prefix index (sweep path): bucket bk owns the
    // 2^(ib - ibits) <= 1024 entries of T and words of F (b + 5-bit filter)
    // under its top ibits bits; its distinct cells are counted per ib-bit prefix and OR'ed
    // into the filter words in shared memory (h is free at those points),
    // then T (bucket start + exclusive count) and F are written once --
    // no separate pass over the table, no global atomics, no memset of F.
    const int ixs = Tix ? ib - ibits : 0, ixn = 1 << ixs;
    uint32_t* ixc = h;           // [ixn] cells per ib-bit prefix
    uint32_t* ixf = h + 1024;    // [ixn] filter words
    auto ix_zero = [&]() {
      for (int q = tid; q < ixn; q += kBktThreads) ixc[q] = ixf[q] = 0u;
    };
    auto ix_add = [&](const K& k) {
      const uint64_t t = KT<K>::top(k);
      const uint32_t x = uint32_t(t >> (64 - ib)) & uint32_t(ixn - 1);
      atomicAdd(&ixc[x], 1u);
      atomicOr(&ixf[x], 1u << (uint32_t(t >> (64 - ib - 5)) & 31u));
    };
    auto ix_write = [&](int64_t b2, uint32_t base) {  // after a barrier
      constexpr int PER = 1024 / kBktThreads;
      uint32_t cv[PER], loc = 0;
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int q = tid * PER + u;
        cv[u] = q < ixn ? ixc[q] : 0u;
        loc += cv[u];
      }
      uint32_t tot;
      uint32_t run = block_excl_scan(loc, s_scan, &tot);
      const size_t g0 = size_t(b2) << ixs;
      static_assert(PER == 4, "one 16-byte store per array and thread");
      if (tid * PER < ixn) {  // (ixn >= 4 when ixs >= 2; else one entry per thread)
        uint4 tv, fv;
        tv.x = base + run;
        tv.y = tv.x + cv[0];
        tv.z = tv.y + cv[1];
        tv.w = tv.z + cv[2];
        if (ixn >= 4) {
          fv = *reinterpret_cast<const uint4*>(ixf + tid * PER);
          *reinterpret_cast<uint4*>(Tix + g0 + tid * PER) = tv;
          *reinterpret_cast<uint4*>(Fix + g0 + tid * PER) = fv;
        } else {
          const uint32_t t4[4] = {tv.x, tv.y, tv.z, tv.w};
          for (int u = 0; u < PER && tid * PER + u < ixn; ++u) {
            Tix[g0 + tid * PER + u] = t4[u];
            Fix[g0 + tid * PER + u] = ixf[tid * PER + u];
          }
        }
      }
    };
    auto list_bucket = [&]() {
      if (src)
        for (int i = tid; i < S; i += kBktThreads) keys[lo + i] = rsrc(bk, lo)[i];
      if (tid == 0) blist[atomicAdd(nlist, 1u)] = uint32_t(bk);
      __syncthreads();
    };
    if (S <= 1) {
      if (ucnt && tid == 0) ucnt[bk] = uint32_t(S);
      if (src && S == 1 && tid == 0) keys[lo] = s[0];
      if (Tix) {  // the bucket's slice of the prefix index: at most one cell
        ix_zero();
        __syncthreads();
        if (S == 1 && tid == 0) ix_add(s[0]);
        __syncthreads();
        ix_write(bk, lo);
      }
      __syncthreads();
      continue;
    }
    if (S > CAP) {
      list_bucket();
      continue;
    }
    // ---- 1. bits that vary inside the bucket
    // the thread's keys (positions c * 256 + tid) stay in registers
    K kr[MAXC];
    uint64_t av[2] = {~0ull, ~0ull}, ov[2] = {0ull, 0ull};
    if (!PREF) {
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        const int i = c * kBktThreads + tid;
        kr[c] = rsrc(bk, lo)[i < S ? i : 0];
        if (i < S) s[i] = kr[c];
      }
    }
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int i = c * kBktThreads + tid;
      if (PREF) kr[c] = s[i < S ? i : 0];
      key_andor(kr[c], av, ov);
    }
#pragma unroll
    for (int w = 0; w < NW; ++w) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        av[w] &= __shfl_xor_sync(kFull, av[w], o);
        ov[w] |= __shfl_xor_sync(kFull, ov[w], o);
      }
    }
    if (lane == 0) {
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        s_red[0][wid][w] = av[w];
        s_red[1][wid][w] = ov[w];
      }
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) h[q * kBktThreads + tid] = 0u;
    if (tid == 0) s_nmany = s_eq = 0u;
    __syncthreads();
    uint64_t dif[2] = {0ull, 0ull};
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      uint64_t a = ~0ull, o = 0ull;
#pragma unroll
      for (int ww = 0; ww < kBktWarps; ++ww) {
        a &= s_red[0][ww][w];
        o |= s_red[1][ww][w];
      }
      dif[w] = a ^ o;
    }
    int f = 0;
    if (dif[0]) f = __clzll(dif[0]);
    else if (NW > 1 && dif[NW > 1 ? 1 : 0]) f = 64 + __clzll(dif[NW > 1 ? 1 : 0]);
    else f = -1;  // all keys equal
    if (f < 0) {
      if (ucnt) {
        if (tid == 0) {
          ucnt[bk] = 1u;
          keys[lo] = s[0];
        }
      } else {
        for (int i = tid; i < S; i += kBktThreads) keys[lo + i] = s[i];
      }
      if (Tix) {  // one distinct cell
        __syncthreads();
        ix_zero();
        __syncthreads();
        if (tid == 0) ix_add(s[0]);
        __syncthreads();
        ix_write(bk, lo);
      }
      __syncthreads();
      continue;
    }
    // ---- 2. counting pass on the digit at f
    uint32_t dg[MAXC], rk[MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int i = c * kBktThreads + tid;
      dg[c] = 0;
      rk[c] = 0;
      if (i < S) {
        dg[c] = uint32_t(key_bits_at(kr[c], f) >> (64 - kRankBits));
        rk[c] = atomicAdd(&h[hx(dg[c])], 1u);
      }
    }
    __syncthreads();
    uint32_t cl[kPer], loc = 0;
    int too_long = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      cl[q] = h[q * kBktThreads + tid];
      loc += cl[q];
      too_long |= cl[q] > uint32_t(kRankRun);
    }
    uint32_t all;
    uint32_t run = block_excl_scan(loc, s_scan, &all);
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      h[q * kBktThreads + tid] = run;
      run += cl[q];
    }
    if (tid == 0) h[kBins] = uint32_t(S);
    if (__syncthreads_or(too_long)) {
      list_bucket();
      continue;
    }
    // ---- 3. scatter, then rank inside the digit
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int i = c * kBktThreads + tid;
      if (i < S) nxt[h[hx(dg[c])] + rk[c]] = uint16_t(i);
    }
    __syncthreads();
    // digits of <= 2 keys (all but a few): one compare with the partner,
    // branch-free so the chains of the thread's keys overlap
    uint32_t bs[MAXC], ct[MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int i = c * kBktThreads + tid;
      bs[c] = h[hx(dg[c])];
      ct[c] = i < S ? h[hx(dg[c] + 1)] - bs[c] : 0u;
    }
    // keys of longer digits are listed and ranked afterwards by all threads
    // together (one list entry per thread: no lanes idle behind a long loop);
    // their positions come back through pos_of[]
    uint32_t ps[MAXC];
    int anyeq = 0;  // two equal keys seen (equal keys share a digit): the dedupe has work
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int i = c * kBktThreads + tid;
      const uint32_t pq = min(bs[c] + (rk[c] ^ 1u), uint32_t(CAP - 1));
      const int j = nxt[pq];
      ps[c] = bs[c];
      if (ct[c] == 2u) {
        const K kj = s[j];
        ps[c] += key_before(kj, j, kr[c], i);
        anyeq |= int(key_eq(kj, kr[c]));
      }
      if (ct[c] > 2u) {
        const uint32_t q = atomicAdd(&s_nmany, 1u);
        if (q < mcap) mlist[q] = uint32_t(i) | (dg[c] << 16);
      }
    }
    __syncthreads();
    const uint32_t nmany = s_nmany;
    if (nmany > mcap) {  // (skewed digits) the byte-pass kernel takes the bucket
      list_bucket();
      continue;
    }
    if (nmany) {
      for (uint32_t q = tid; q < nmany; q += kBktThreads) {
        const uint32_t e = mlist[q];
        const int i = int(e & 0xffffu);
        const uint32_t d = e >> 16, b0 = h[hx(d)], cn = h[hx(d + 1)] - b0;
        const K ki = s[i];
        uint32_t r = 0;
        uint32_t eq = 0;
        for (uint32_t m = 0; m < cn; ++m) {
          const int j = nxt[b0 + m];
          const K kj = s[j];
          r += (j != i) && key_before(kj, j, ki, i);
          eq |= uint32_t(j != i) & uint32_t(key_eq(kj, ki));
        }
        pos_of[i] = uint16_t(b0 + r);
        if (eq) s_eq = 1u;
      }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < MAXC; ++c)
        if (ct[c] > 2u) ps[c] = pos_of[c * kBktThreads + tid];
    }
    // ---- permute in place: every key is in a register, so after the
    // barrier each thread stores its keys at their sorted positions
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
      if (ct[c] != 0u) s[ps[c]] = kr[c];
    const bool nodup = !__syncthreads_or(anyeq) && s_eq == 0u;
    // ---- 4. write (deduplicated and compacted when ucnt is given); the
    // sorted keys are read contiguously.  No two keys compared equal (the
    // common case): every key is a cell, no dedupe pass over the buffer
    if (ucnt && nodup) {
      if (Tix) {
        ix_zero();
        __syncthreads();
      }
      for (int i = tid; i < S; i += kBktThreads) {
        const K k = s[i];
        keys[lo + i] = k;
        if (Tix) ix_add(k);
      }
      if (tid == 0) ucnt[bk] = uint32_t(S);
      if (Tix) {
        __syncthreads();
        ix_write(bk, lo);
      }
    } else if (!ucnt) {
      for (int i = tid; i < S; i += kBktThreads) keys[lo + i] = s[i];
    } else {
      uint32_t bl[MAXC];
      K sv[MAXC];
      if (Tix) ix_zero();  // (h is free after the permutation)
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        const int i = c * kBktThreads + tid;
        sv[c] = s[i < S ? i : 0];
        const bool fl = i < S && (i == 0 || !key_eq(s[i - 1], sv[c]));
        bl[c] = __ballot_sync(kFull, fl);
        if (lane == 0) s_wc[c * kBktWarps + wid] = __popc(bl[c]);
      }
      __syncthreads();
      if (Tix) {
#pragma unroll
        for (int c = 0; c < MAXC; ++c)
          if ((bl[c] >> lane) & 1u) ix_add(sv[c]);
      }
      if (tid < 32) {
        constexpr int NWC = MAXC * kBktWarps;
        constexpr int PER = (NWC + 31) / 32;
        uint32_t v[PER], sum = 0;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
          v[q] = (tid * PER + q < NWC) ? s_wc[tid * PER + q] : 0u;
          sum += v[q];
        }
        uint32_t inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, inc, o);
          if (tid >= o) inc += y;
        }
        uint32_t rr = inc - sum;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
          if (tid * PER + q < NWC) s_wc[tid * PER + q] = rr;
          rr += v[q];
        }
        if (tid == 31) ucnt[bk] = inc;
      }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        if ((bl[c] >> lane) & 1u)
          keys[lo + s_wc[c * kBktWarps + wid] + __popc(bl[c] & lt)] = sv[c];
      }
      if (Tix) ix_write(bk, lo);  // (the atomics above precede the last barrier)
    }
    __syncthreads();
  }
  cp_async_wait0();
}

// The region sweep as a persistent kernel (RS_PERSIST): two CTAs per SM walk
// the tiles with the next tile's rows already on their way -- one TMA bulk
// copy (cp.async.bulk global->shared, mbarrier completion) per tile issued a
// whole tile ahead -- so the loads overlap the ranking, the reservation
// atomics and the writes of the current tile; the tile's buffer is then
// reused for its own reorder.
#ifndef RS_PMINB
#define RS_PMINB 2  // persistent region sweep: CTAs per SM
#endif
template <class K, int B2T>
__global__ void __launch_bounds__(kSortThreads, RS_PMINB)
    k_region_sweep_p(const K* __restrict__ regions, uint32_t capr, const uint32_t* __restrict__ rcnt,
                     uint32_t tpr, K* __restrict__ slots, uint32_t cap16,
                     uint32_t* __restrict__ cnt16, uint32_t* __restrict__ ovf, int B2arg) {
  const int B2 = B2T ? B2T : B2arg;
  if (*ovf) return;  // a region overflowed in the pack: the caller re-runs the exact path
  constexpr int IPT = RsCfg<K>::IPT;
  constexpr int TILE = RsCfg<K>::TILE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* const buf0 = reinterpret_cast<K*>(smem_raw);
  K* const buf1 = buf0 + TILE;
  __shared__ uint32_t wcnt[kSortWarps][kRadix];
  __shared__ uint32_t s_dexcl[kRadix], s_lim[kRadix], s_gbase[kRadix];
  __shared__ uint32_t s_scan[33];
  __shared__ uint64_t s_bar[2];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t ntot = 256u * tpr;
  auto info = [&](uint32_t id, uint32_t& x, uint32_t& beg, int& nt) -> bool {
    x = id / tpr;
    const uint32_t cnt = min(rcnt[x], capr);
    beg = (id % tpr) * uint32_t(TILE);
    if (beg >= cnt) return false;
    nt = int(min(uint32_t(TILE), cnt - beg));
    return true;
  };
  auto next_tile = [&](uint32_t id) -> uint32_t {
    uint32_t x, b;
    int nt;
    for (; id < ntot; id += gridDim.x)
      if (info(id, x, b, nt)) return id;
    return ntot;
  };
  auto issue = [&](uint32_t id, K* dst, uint64_t* bar) {  // thread 0
    uint32_t x, beg;
    int nt;
    if (id < ntot && info(id, x, beg, nt)) {
      // bulk copies move multiples of 16 bytes from 16-byte aligned
      // addresses: 8-byte keys round up to an even count (capr is even and
      // the regions buffer has a 16-byte tail, so the extra key is readable)
      const uint32_t bytes = (uint32_t(nt) * uint32_t(sizeof(K)) + 15u) & ~15u;
      // the buffer was last written by the threads (generic proxy)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_expect_tx(bar, bytes);
      bulk_g2s(dst, regions + size_t(x) * capr + beg, bytes, bar);
    }
  };
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  uint32_t cur = next_tile(blockIdx.x);
  if (tid == 0) issue(cur, buf0, &s_bar[0]);
  for (int it = 0; cur < ntot; ++it) {
    K* const sb = (it & 1) ? buf1 : buf0;
    const uint32_t nxt = next_tile(cur + gridDim.x);
    if (tid == 0) issue(nxt, (it & 1) ? buf0 : buf1, &s_bar[(it + 1) & 1]);
    for (int i = tid; i < kSortWarps * kRadix; i += kSortThreads) (&wcnt[0][0])[i] = 0;
    uint32_t x, beg;
    int nt;
    info(cur, x, beg, nt);
    mbar_wait(&s_bar[it & 1], uint32_t(it >> 1) & 1u);
    __syncthreads();
    const int wb = w * 32 * IPT;
    K key[IPT];
    uint32_t rank[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int g = wb + i * 32 + lane;
      key[i] = g < nt ? sb[g] : K{};
    }
#pragma unroll
    for (int i = 0; i < IPT; ++i)
      if (wb + i * 32 + lane < nt) rank[i] = atomicAdd(&wcnt[w][rs_digit(key[i], B2)], 1u);
    __syncthreads();
    uint32_t total = 0;
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ++ww) {
      const uint32_t c = wcnt[ww][tid];
      wcnt[ww][tid] = total;
      total += c;
    }
    uint32_t tile_n;
    const uint32_t dex = block_excl_scan(total, s_scan, &tile_n);
    uint32_t base = 0;
    const uint32_t q = (x << B2) | uint32_t(tid);
    if (total) base = atomicAdd(&cnt16[q], total);
    s_dexcl[tid] = dex;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      if (wb + i * 32 + lane < nt) {
        const uint32_t d = rs_digit(key[i], B2);
        sb[s_dexcl[d] + wcnt[w][d] + rank[i]] = key[i];
      }
    }
    if (total && uint64_t(base) + total > cap16) atomicOr(ovf, 1u);
    s_gbase[tid] = q * cap16 + base - dex;
    s_lim[tid] = dex + (base < cap16 ? cap16 - base : 0u);
    __syncthreads();
    for (int j = tid; j < nt; j += kSortThreads) {
      const K k = sb[j];
      const uint32_t d = rs_digit(k, B2);
      if (uint32_t(j) < s_lim[d]) slots[s_gbase[d] + uint32_t(j)] = k;
    }
    __syncthreads();
    cur = nxt;
  }
}

// Index slices (see k_bucket_rank's fused prefix index) of the buckets listed
// to the byte-pass kernel, from their finished (deduplicated) rows.
template <class K>
__global__ void __launch_bounds__(256)
    k_bucket_slices(const K* __restrict__ keys, const uint32_t* __restrict__ off,
                    const uint32_t* __restrict__ ucnt, const uint32_t* __restrict__ blist,
                    const uint32_t* __restrict__ nlist, uint32_t* __restrict__ Tix,
                    uint32_t* __restrict__ Fix, int ib, int ibits,
                    const uint32_t* __restrict__ failed) {
  __shared__ uint32_t ixc[1024], ixf[1024], s_scan[33];
  const int tid = threadIdx.x, ixs = ib - ibits, ixn = 1 << ixs;
  // a bucket the byte-pass kernel could not finish has no ucnt: the whole
  // sort is redone by the caller, the index with it
  if (*failed) return;
  const uint32_t nl = *nlist;
  for (uint32_t q = blockIdx.x; q < nl; q += gridDim.x) {
    const uint32_t bk = blist[q], lo = off[bk], u = min(ucnt[bk], off[bk + 1] - lo);
    for (int r = tid; r < ixn; r += 256) ixc[r] = ixf[r] = 0u;
    __syncthreads();
    for (uint32_t i = tid; i < u; i += 256) {
      const uint64_t t = KT<K>::top(keys[lo + i]);
      const uint32_t x = uint32_t(t >> (64 - ib)) & uint32_t(ixn - 1);
      atomicAdd(&ixc[x], 1u);
      atomicOr(&ixf[x], 1u << (uint32_t(t >> (64 - ib - 5)) & 31u));
    }
    __syncthreads();
    uint32_t cv[4], loc = 0;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int r = tid * 4 + v;
      cv[v] = r < ixn ? ixc[r] : 0u;
      loc += cv[v];
    }
    uint32_t tot;
    uint32_t run = block_excl_scan(loc, s_scan, &tot);
    const size_t g0 = size_t(bk) << ixs;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int r = tid * 4 + v;
      if (r < ixn) {
        Tix[g0 + r] = lo + run;
        Fix[g0 + r] = ixf[r];
      }
      run += cv[v];
    }
    __syncthreads();
  }
}

// duplicates were dropped: the buckets moved from off[] to uoff[]
__global__ void k_fix_index(uint32_t* __restrict__ T, int ib, int ibits,
                            const uint32_t* __restrict__ off, const uint32_t* __restrict__ uoff) {
  const int64_t n = int64_t(1) << ib;
  for (int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < n;
       x += int64_t(gridDim.x) * blockDim.x) {
    const int64_t bk = x >> (ib - ibits);
    T[x] -= off[bk] - uoff[bk];
  }
}

__global__ void k_ix_end(uint32_t* p, uint32_t v) { *p = v; }

int grid_for(int64_t n, int threads, int per_sm = 8) {
  int64_t b = (n + threads - 1) / threads;
  int64_t cap = int64_t(num_sms()) * per_sm;
  return int(std::max<int64_t>(1, std::min(b, cap)));
}

// shared-memory capacity 2x the mean bucket (2048 or 4096 rows).  The rank
// pass handles the buckets it can; the ones it lists (skewed digits, or
// larger than its capacity) go through the stable byte-pass kernel.
template <class K>
void launch_bucket_sort(K* ko, const uint32_t* off, int64_t n, int64_t nb, int B, uint32_t* flag,
                        uint32_t* ucnt, cudaStream_t s, const K* src = nullptr,
                        uint32_t scap = 0, uint32_t* Tix = nullptr, uint32_t* Fix = nullptr,
                        int ib = 0, int ibits = 0, const uint32_t* abort_flag = nullptr) {
  const int64_t avg = (n + nb - 1) / nb;
  const int cap = avg <= 1024 ? 2048 : 4096;
  DevBuf<uint32_t> blist(size_t(nb), s), nlist(1, s);
  CG_CUDA(cudaMemsetAsync(nlist.p, 0, sizeof(uint32_t), s));
  {
    // rank pass: keys (double-buffered with PREF) + two u16 orders + the
    // long-digit list; 1.5x the mean bucket; larger buckets go to the byte passes
    const int rcap = avg <= 1024 ? BKT_RCAP : 2048;
    const size_t smem = size_t(rcap) * (2 * sizeof(K) + 8);
    const int per_sm = std::max(1, int((222 << 10) / (smem + 10 * 1024)));
    const int grid = int(std::min<int64_t>(nb, int64_t(num_sms()) * per_sm));
    auto go = [&](auto kern) {
      CG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      CG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      kern<<<grid, kBktThreads, smem, s>>>(ko, off, nb, rcap, ucnt, blist.p, nlist.p, src, scap, Tix,
                                           Fix, ib, ibits, abort_flag);
    };
    if (rcap <= 1280) go(k_bucket_rank<K, 5, true>);
    else if (rcap <= 1536) go(k_bucket_rank<K, 6, true>);
    else go(k_bucket_rank<K, 8, true>);
    CG_LAUNCH_CHECK();
  }
  const size_t smem = size_t(cap) * (sizeof(K) + 4);
  const int per_sm = std::max(1, int((200 << 10) / (smem + 12 * 1024)));
  const int grid = int(std::min<int64_t>(nb, int64_t(num_sms()) * per_sm));
  if (cap == 2048) {
    CG_CUDA(cudaFuncSetAttribute(k_bucket_sort<K, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    k_bucket_sort<K, 8><<<grid, kBktThreads, smem, s>>>(ko, off, nb, cap, B, flag, ucnt, blist.p, nlist.p);
  } else {
    CG_CUDA(cudaFuncSetAttribute(k_bucket_sort<K, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    k_bucket_sort<K, 16><<<grid, kBktThreads, smem, s>>>(ko, off, nb, cap, B, flag, ucnt, blist.p, nlist.p);
  }
  CG_LAUNCH_CHECK();
  if (Tix) {  // index slices of the buckets the byte-pass kernel finished
    k_bucket_slices<K><<<unsigned(num_sms() * 2), 256, 0, s>>>(ko, off, ucnt, blist.p, nlist.p,
                                                               Tix, Fix, ib, ibits, flag);
    CG_LAUNCH_CHECK();
  }
}

// bases[d][b] = exclusive scan of hist[d][0..256) (one block per digit)
__global__ void k_digit_bases(const uint32_t* __restrict__ hist, uint32_t* __restrict__ bases) {
  __shared__ uint32_t tmp[33];
  uint32_t total;
  const uint32_t v = hist[blockIdx.x * kRadix + threadIdx.x];
  bases[blockIdx.x * kRadix + threadIdx.x] = block_excl_scan(v, tmp, &total);
}

// tile_cnt[t][256] (per-tile digit counts) -> tile_pre[t][256] = exclusive
// prefix over tiles, per digit: chunk sums, a scan of the chunk sums, fill.
constexpr int kPreChunk = 64;
__global__ void k_tile_chunk_sum(const uint32_t* __restrict__ cnt, int64_t nt,
                                 uint32_t* __restrict__ csum) {
  const int64_t c = blockIdx.x, d = threadIdx.x;
  uint32_t t = 0;
  for (int64_t q = c * kPreChunk; q < min(nt, (c + 1) * kPreChunk); ++q) t += cnt[q * kRadix + d];
  csum[c * kRadix + d] = t;
}
// one warp per digit: exclusive scan of its nc chunk sums, 32 at a time
__global__ void k_tile_chunk_scan(uint32_t* __restrict__ csum, int64_t nc) {
  const int lane = threadIdx.x & 31;
  const int d = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (d >= kRadix) return;
  uint32_t run = 0;
  for (int64_t c0 = 0; c0 < nc; c0 += 32) {
    const int64_t c = c0 + lane;
    const uint32_t v = c < nc ? csum[c * kRadix + d] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (c < nc) csum[c * kRadix + d] = run + x - v;
    run += __shfl_sync(kFull, x, 31);
  }
}
__global__ void k_tile_fill(const uint32_t* __restrict__ cnt, int64_t nt,
                            const uint32_t* __restrict__ cpre, uint32_t* __restrict__ pre) {
  const int64_t c = blockIdx.x, d = threadIdx.x;
  uint32_t run = cpre[c * kRadix + d];
  for (int64_t q = c * kPreChunk; q < min(nt, (c + 1) * kPreChunk); ++q) {
    pre[q * kRadix + d] = run;
    run += cnt[q * kRadix + d];
  }
}

// Generic pass driver over digits [dlo, dhi) of the top word.
template <class K>
void radix_passes(K* keys, K* keys_alt, const uint32_t* vals_in, uint32_t* vals,
                  uint32_t* vals_alt, bool want_vals, int64_t n, int dlo, int dhi, K** keys_out,
                  uint32_t** vals_out, cudaStream_t s, SortStats* st,
                  const uint32_t* dev_hist = nullptr, const uint32_t* tile_hist = nullptr) {
  *keys_out = keys;
  if (vals_out) *vals_out = nullptr;
  auto identity_or_input = [&]() {
    if (!want_vals) return;
    if (vals_in) {
      *vals_out = const_cast<uint32_t*>(vals_in);
    } else {
      k_iota<<<grid_for(n, 256), 256, 0, s>>>(vals, n);
      CG_LAUNCH_CHECK();
      *vals_out = vals;
    }
  };
  if (n <= 1 || dhi <= dlo) {
    identity_or_input();
    return;
  }
  const int nd = dhi - dlo;
  DevBuf<uint32_t> hist(size_t(nd) * kRadix, s);
  const uint32_t* hsrc = dev_hist;
  if (!hsrc) {  // (the pack kernel may have counted these digits already)
    CG_CUDA(cudaMemsetAsync(hist.p, 0, hist.n * sizeof(uint32_t), s));
    k_digit_hist<K><<<grid_for(n, 256, 4), 256, 0, s>>>(keys, n, dlo, dhi, hist.p);
    CG_LAUNCH_CHECK();
    hsrc = hist.p;
  }
  std::vector<int> digits;
  std::vector<uint32_t> bases;
  DevBuf<uint32_t> dbases;
  if (dev_hist && !want_vals) {
    // (MSD partition, histogram counted by the pack kernel) no host round
    // trip: the digit bases are scanned on the device and every digit gets a
    // pass -- a constant digit only costs one extra copy-like pass
    for (int d = 0; d < nd; ++d) digits.push_back(d + dlo);
    dbases.alloc(size_t(nd) * kRadix, s);
    k_digit_bases<<<unsigned(nd), kRadix, 0, s>>>(dev_hist, dbases.p);
    CG_LAUNCH_CHECK();
  }
  uint32_t* hh = nullptr;
  if (digits.empty()) {
    hh = static_cast<uint32_t*>(host_stage(hist.n * sizeof(uint32_t)));
    CG_CUDA(cudaMemcpyAsync(hh, hsrc, hist.n * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaStreamSynchronize(s));
  }
  for (int d = 0; hh && d < nd; ++d) {
    const uint32_t* h = hh + d * kRadix;
    bool trivial = false;
    for (int b = 0; b < kRadix; ++b)
      if (int64_t(h[b]) == n) trivial = true;
    if (trivial) continue;
    digits.push_back(d + dlo);
    uint32_t run = 0;
    for (int b = 0; b < kRadix; ++b) {
      bases.push_back(run);
      run += h[b];
    }
  }
  if (st) st->passes += int(digits.size());
  if (digits.empty()) {
    identity_or_input();
    return;
  }
  const int P = int(digits.size());
  if (hh) {
    dbases.alloc(bases.size(), s);
    CG_CUDA(cudaMemcpyAsync(dbases.p, bases.data(), bases.size() * sizeof(uint32_t),
                            cudaMemcpyHostToDevice, s));
  }
  const bool V = want_vals;
  // as many resident tiles per SM as registers allow: prefer shared memory
  if (V) {
    CG_CUDA(cudaFuncSetAttribute(k_onesweep<K, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    CG_CUDA(cudaFuncSetAttribute(k_onesweep<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(TileCfg<K, true>::SMEM)));
  } else {
    CG_CUDA(cudaFuncSetAttribute(k_onesweep<K, false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    CG_CUDA(cudaFuncSetAttribute(k_onesweep<K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(TileCfg<K, false>::SMEM)));
  }
  const int TILE = V ? TileCfg<K, true>::TILE : TileCfg<K, false>::TILE;
  const int64_t tiles = (n + TILE - 1) / TILE;
  DevBuf<uint64_t> status(size_t(tiles) * kRadix, s);
  DevBuf<uint32_t> counters(size_t(P), s);
  CG_CUDA(cudaMemsetAsync(status.p, 0, status.n * sizeof(uint64_t), s));
  CG_CUDA(cudaMemsetAsync(counters.p, 0, counters.n * sizeof(uint32_t), s));
  // the first pass needs no look-back when the pack kernel counted its digit
  // per tile (same tiles: keys-only passes of the pack output)
  DevBuf<uint32_t> tpre(tile_hist && !V && digits[0] == dlo ? size_t(tiles) * kRadix : 0, s);
  if (tpre.n) {
    const int64_t nch = (tiles + kPreChunk - 1) / kPreChunk;
    DevBuf<uint32_t> csum(size_t(nch) * kRadix, s);
    k_tile_chunk_sum<<<unsigned(nch), kRadix, 0, s>>>(tile_hist, tiles, csum.p);
    CG_LAUNCH_CHECK();
    k_tile_chunk_scan<<<kRadix / 8, 256, 0, s>>>(csum.p, nch);
    CG_LAUNCH_CHECK();
    k_tile_fill<<<unsigned(nch), kRadix, 0, s>>>(tile_hist, tiles, csum.p, tpre.p);
    CG_LAUNCH_CHECK();
  }
  K* ck = keys;
  K* ak = keys_alt;
  const uint32_t* cv = vals_in;
  uint32_t* av = vals;
  uint32_t* spare_v = vals_alt;
  for (int p = 0; p < P; ++p) {
    const int shift = 8 * digits[p];
    if (V) {
      k_onesweep<K, true><<<unsigned(tiles), kSortThreads, TileCfg<K, true>::SMEM, s>>>(
          ck, ak, cv, av, n, shift, dbases.p + p * kRadix, status.p, counters.p + p,
          uint32_t(p + 1), nullptr);
    } else {
      k_onesweep<K, false><<<unsigned(tiles), kSortThreads, TileCfg<K, false>::SMEM, s>>>(
          ck, ak, nullptr, nullptr, n, shift, dbases.p + p * kRadix, status.p, counters.p + p,
          uint32_t(p + 1), (p == 0 && tpre.n) ? tpre.p : nullptr);
    }
    CG_LAUNCH_CHECK();
    std::swap(ck, ak);
    if (V) {
      // next pass reads what was just written; never writes into vals_in
      uint32_t* written = av;
      av = (cv == vals_in) ? spare_v : const_cast<uint32_t*>(cv);
      cv = written;
    }
  }
  *keys_out = ck;
  if (vals_out && V) *vals_out = const_cast<uint32_t*>(cv);
}

}  // namespace

template <class K>
void radix_sort(K* keys, K* keys_alt, const uint32_t* vals_in, uint32_t* vals, uint32_t* vals_alt,
                bool want_vals, int64_t n, int key_bits, K** keys_out, uint32_t** vals_out,
                cudaStream_t s, SortStats* st) {
  const int ndig = std::max(1, (key_bits + 7) / 8);
  radix_passes<K>(keys, keys_alt, vals_in, vals, vals_alt, want_vals, n, 0, ndig, keys_out,
                  vals_out, s, st);
}

template void radix_sort<uint32_t>(uint32_t*, uint32_t*, const uint32_t*, uint32_t*, uint32_t*,
                                   bool, int64_t, int, uint32_t**, uint32_t**, cudaStream_t,
                                   SortStats*);
template void radix_sort<uint64_t>(uint64_t*, uint64_t*, const uint32_t*, uint32_t*, uint32_t*,
                                   bool, int64_t, int, uint64_t**, uint32_t**, cudaStream_t,
                                   SortStats*);

namespace {
// Tie runs of the (word 0, index) order: rows whose word 0 is equal form
// contiguous runs; the thread at the head of a run (<= kTieRun rows)
// insertion-sorts the run's indices on the remaining words (stable: equal
// rows keep index order).  A longer run raises *long_run (then the caller
// sorts all words instead).
constexpr int kTieRun = 32;
__global__ void k_tie_fix(const uint64_t* __restrict__ keys, int W, const uint64_t* __restrict__ w0,
                          uint32_t* __restrict__ idx, int64_t n, uint32_t* __restrict__ long_run) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = w0[i];
    if (i > 0 && w0[i - 1] == k) continue;       // not a run head
    if (i + 1 >= n || w0[i + 1] != k) continue;  // run of one
    int64_t e = i + 2;
    while (e < n && w0[e] == k && e - i <= kTieRun) ++e;
    if (e - i > kTieRun) {
      atomicOr(long_run, 1u);
      continue;
    }
    for (int64_t a = i + 1; a < e; ++a) {
      const uint32_t v = idx[a];
      const uint64_t* rv = keys + int64_t(v) * W;
      int64_t z = a;
      while (z > i) {
        const uint32_t u = idx[z - 1];
        const uint64_t* ru = keys + int64_t(u) * W;
        int c = 0;
        for (int w = 1; w < W && c == 0; ++w) c = ru[w] < rv[w] ? -1 : (ru[w] > rv[w] ? 1 : 0);
        if (c < 0 || (c == 0 && u < v)) break;
        idx[z] = u;
        --z;
      }
      idx[z] = v;
    }
  }
}
}  // namespace

namespace {
// (top 32 bits of word 0) << 32 | row index: one u64 sort key per row
__global__ void k_prefix_idx(const uint64_t* __restrict__ keys, int W, int64_t n,
                             uint64_t* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = (keys[i * W] & 0xffffffff00000000ull) | uint64_t(i);
}

// pk sorted on the high halves (stable: equal prefixes in index order) ->
// the canonical order of the rows: positions outside runs of equal prefixes
// keep their index; the head of a run (<= kTieRun rows) insertion-sorts the
// run's indices on the full rows (equal rows keep index order).  A longer
// run raises *long_run (the caller then sorts every word).
__global__ void k_tie_fix_prefix(const uint64_t* __restrict__ keys, int W,
                                 const uint64_t* __restrict__ pk, int64_t n,
                                 uint32_t* __restrict__ order, uint32_t* __restrict__ long_run,
                                 int64_t run_cap, uint2* __restrict__ runs,
                                 uint32_t* __restrict__ nruns,
                                 const uint32_t* __restrict__ dup_hits) {
  if (dup_hits && *dup_hits >= 8u) {  // heavy duplication: the caller hashes first
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(long_run, 1u);
    return;
  }
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t k = uint32_t(pk[i] >> 32);
    const bool head = i == 0 || uint32_t(pk[i - 1] >> 32) != k;
    const bool tail = i + 1 >= n || uint32_t(pk[i + 1] >> 32) != k;
    if (head && tail) {
      order[i] = uint32_t(pk[i]);
      continue;
    }
    if (head) {
      // a short run (<= kTieRun rows): its head insertion-sorts it on the
      // full rows (equal rows keep index order)
      int64_t e = i + 2;
      while (e < n && uint32_t(pk[e] >> 32) == k && e - i <= kTieRun) ++e;
      if (e - i > kTieRun) continue;  // a long run: its tail lists it
      // a run beyond run_cap was found already: the caller discards this order
      if (*reinterpret_cast<volatile uint32_t*>(long_run) & 1u) continue;
      for (int64_t a = i; a < e; ++a) {
        const uint32_t v = uint32_t(pk[a]);
        const uint64_t* rv = keys + int64_t(v) * W;
        int64_t z = a;
        while (z > i) {
          const uint32_t u = order[z - 1];
          const uint64_t* ru = keys + int64_t(u) * W;
          int c = 0;
          for (int w = 0; w < W && c == 0; ++w) c = ru[w] < rv[w] ? -1 : (ru[w] > rv[w] ? 1 : 0);
          if (c == 0) atomicOr(long_run, 2u);  // equal rows: the dedupe has work
          if (c < 0 || (c == 0 && u < v)) break;
          order[z] = u;
          --z;
        }
        order[z] = v;
      }
      continue;
    }
    if (!tail) continue;
    // the tail of a run: its head by a binary search over the last run_cap + 1
    // positions (pk is sorted on the prefix); a run longer than kTieRun is
    // listed for k_run_sort, one longer than run_cap goes to the caller
    const int64_t lo0 = i - run_cap > 0 ? i - run_cap : 0;
    int64_t lo = lo0, len = i - lo0;
    while (len > 0) {
      const int64_t half = len >> 1;
      if (uint32_t(pk[lo + half] >> 32) < k) {
        lo += half + 1;
        len -= half + 1;
      } else {
        len = half;
      }
    }
    const int64_t rl = i - lo + 1;
    if (rl <= kTieRun) continue;  // its head sorted it
    if (lo == lo0 && lo0 > 0 && uint32_t(pk[lo0 - 1] >> 32) == k) {
      atomicOr(long_run, 1u);  // longer than run_cap
    } else {
      const uint32_t q = atomicAdd(nruns, 1u);
      runs[q] = make_uint2(uint32_t(lo), uint32_t(rl));
    }
  }
}

// A long run of equal 32-bit prefixes (arrangement signatures): one CTA
// loads its rows into shared memory and bitonic-sorts (row, index) pairs --
// rows compared word by word, equal rows by index -- then writes the run's
// part of the order.  Equal rows raise bit 2 of *flag (dedupe needed).
__global__ void __launch_bounds__(256)
    k_run_sort(const uint64_t* __restrict__ keys, int W, const uint64_t* __restrict__ pk,
               const uint2* __restrict__ runs, uint32_t* __restrict__ order,
               uint32_t* __restrict__ flag) {
  extern __shared__ __align__(16) uint64_t rsm[];
  const uint2 run = runs[blockIdx.x];
  const int len = int(run.y);
  int P = 1;
  while (P < len) P <<= 1;
  uint64_t* rw = rsm;                                    // [P][W]
  uint32_t* ix = reinterpret_cast<uint32_t*>(rsm + size_t(P) * W);  // [P]
  for (int t = threadIdx.x; t < P * W; t += blockDim.x) {
    const int r = t / W, w = t - r * W;
    rw[t] = r < len ? keys[int64_t(uint32_t(pk[run.x + r])) * W + w] : ~0ull;
  }
  for (int r = threadIdx.x; r < P; r += blockDim.x)
    ix[r] = r < len ? uint32_t(pk[run.x + r]) : 0xffffffffu;
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int o = i ^ j;
        if (o > i) {
          uint64_t* A = rw + size_t(i) * W;
          uint64_t* B = rw + size_t(o) * W;
          int c = 0;
          for (int w = 0; w < W && c == 0; ++w) c = A[w] < B[w] ? -1 : (A[w] > B[w] ? 1 : 0);
          if (c == 0) c = ix[i] < ix[o] ? -1 : (ix[i] > ix[o] ? 1 : 0);
          if ((i & k) == 0 ? c > 0 : c < 0) {
            for (int w = 0; w < W; ++w) {
              const uint64_t x = A[w];
              A[w] = B[w];
              B[w] = x;
            }
            const uint32_t y = ix[i];
            ix[i] = ix[o];
            ix[o] = y;
          }
        }
      }
      __syncthreads();
    }
  }
  bool dup = false;
  for (int r = threadIdx.x; r < len; r += blockDim.x) {
    order[run.x + r] = ix[r];
    if (r > 0) {
      bool eq = true;
      for (int w = 0; w < W && eq; ++w) eq = rw[size_t(r) * W + w] == rw[size_t(r - 1) * W + w];
      dup |= eq;
    }
  }
  if (dup) atomicOr(flag, 2u);
}
}  // namespace

bool sort_rows_multiword(const uint64_t* keys, int64_t n, int W, uint64_t* sorted,
                         cudaStream_t s, SortStats* st, uint32_t* order, bool* no_dups, int mode,
                         const uint32_t* dup_hits) {
  if (no_dups) *no_dups = false;
  auto finish = [&](const uint32_t* idx) {
    if (order) CG_CUDA(cudaMemcpyAsync(order, idx, size_t(n) * 4, cudaMemcpyDeviceToDevice, s));
    else launch_gather_rows(keys, idx, n, W, sorted, s);
  };
  bool tried = mode == 2;  // mode 2: every word, no prefix attempt
  if (order && MW_PREFIX32 && mode != 2) {
    // u64 keys (top 32 bits of word 0, row index): 4 stable keys-only passes
    // on the high half (digit bases scanned on the device: no host round
    // trip), then the runs of equal 32-bit prefixes are ordered on the full
    // rows -- planted/random rows leave runs of 1-2 rows
    DevBuf<uint64_t> pk(size_t(n), s), pk_alt(size_t(n), s);
    DevBuf<uint32_t> hist(4 * kRadix, s), flag(1, s);
    k_prefix_idx<<<grid_for(n, 256), 256, 0, s>>>(keys, W, n, pk.p);
    CG_LAUNCH_CHECK();
    CG_CUDA(cudaMemsetAsync(hist.p, 0, hist.n * sizeof(uint32_t), s));
    CG_CUDA(cudaMemsetAsync(flag.p, 0, 4, s));
    k_digit_hist<uint64_t><<<grid_for(n, 256, 4), 256, 0, s>>>(pk.p, n, 4, 8, hist.p);
    CG_LAUNCH_CHECK();
    uint64_t* ko = nullptr;
    radix_passes<uint64_t>(pk.p, pk_alt.p, nullptr, nullptr, nullptr, false, n, 4, 8, &ko, nullptr,
                           s, st, hist.p);
    // long tie runs up to run_cap rows are sorted by k_run_sort (96 KB of
    // shared memory per run at most)
    constexpr size_t kRunSmem = 96 * 1024;
    int64_t run_cap = 1;
    while ((run_cap * 2) * (int64_t(W) * 8 + 4) <= int64_t(kRunSmem)) run_cap *= 2;
    DevBuf<uint2> runs(size_t(n / (kTieRun + 1) + 1), s);
    DevBuf<uint32_t> nr(1, s);
    CG_CUDA(cudaMemsetAsync(nr.p, 0, 4, s));
    k_tie_fix_prefix<<<grid_for(n, 256), 256, 0, s>>>(keys, W, ko, n, order, flag.p, run_cap, runs.p,
                                                      nr.p, mode == 1 ? dup_hits : nullptr);
    CG_LAUNCH_CHECK();
    uint32_t* h = static_cast<uint32_t*>(host_stage(2 * sizeof(uint32_t)));
    CG_CUDA(cudaMemcpyAsync(h, flag.p, 4, cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaMemcpyAsync(h + 1, nr.p, 4, cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaStreamSynchronize(s));
    if ((h[0] & 1u) == 0 && h[1]) {
      CG_CUDA(cudaFuncSetAttribute(k_run_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kRunSmem)));
      k_run_sort<<<h[1], 256, size_t(run_cap) * (size_t(W) * 8 + 4), s>>>(keys, W, ko, runs.p, order,
                                                                           flag.p);
      CG_LAUNCH_CHECK();
      if (no_dups) *no_dups = false;  // (k_run_sort's duplicate bit is not read back)
      return true;
    }
    if ((h[0] & 1u) == 0) {
      if (no_dups) *no_dups = (h[0] & 2u) == 0;  // no two rows compared equal
      return true;
    }
    if (mode == 1) return false;  // long runs: the caller decides (dedupe first)
    tried = true;  // long runs of equal prefixes (arrangement data): every word
  }
  DevBuf<uint64_t> kw(size_t(n), s), kw_alt(size_t(n), s);
  DevBuf<uint32_t> ia(size_t(n), s), ib(size_t(n), s);
  if (!tried) {
    // word 0 decides most orders: sort (word 0, index), then order the runs
    // of equal word 0 on the remaining words; only if a run is long (heavy
    // word-0 ties, e.g. arrangement signatures) sort every word (LSD below)
    k_gather_word<<<grid_for(n, 256), 256, 0, s>>>(keys, W, 0, nullptr, n, kw.p);
    CG_LAUNCH_CHECK();
    uint64_t* ko = nullptr;
    uint32_t* vo = nullptr;
    radix_sort<uint64_t>(kw.p, kw_alt.p, nullptr, ia.p, ib.p, true, n, 64, &ko, &vo, s, st);
    DevBuf<uint32_t> flag(1, s);
    CG_CUDA(cudaMemsetAsync(flag.p, 0, 4, s));
    k_tie_fix<<<grid_for(n, 256), 256, 0, s>>>(keys, W, ko, vo, n, flag.p);
    CG_LAUNCH_CHECK();
    uint32_t* h = static_cast<uint32_t*>(host_stage(sizeof(uint32_t)));
    CG_CUDA(cudaMemcpyAsync(h, flag.p, 4, cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaStreamSynchronize(s));
    if (h[0] == 0) {
      finish(vo);
      return true;
    }
  }
  const uint32_t* idx = nullptr;  // identity before the first word pass
  for (int w = W - 1; w >= 0; --w) {
    k_gather_word<<<grid_for(n, 256), 256, 0, s>>>(keys, W, w, idx, n, kw.p);
    CG_LAUNCH_CHECK();
    uint32_t* vals = (idx == ia.p) ? ib.p : ia.p;
    uint32_t* vals_alt = (idx == ia.p) ? ia.p : ib.p;
    uint64_t* ko = nullptr;
    uint32_t* vo = nullptr;
    radix_sort<uint64_t>(kw.p, kw_alt.p, idx, vals, vals_alt, true, n, 64, &ko, &vo, s, st);
    idx = vo;
  }
  finish(idx);
  return true;
}

int msd_prefix_bits(int64_t n) {
  // B top bits (a multiple of 8) so buckets hold ~2^10 keys on average
  int B = 8;
  while (B < 24 && (n >> B) > 1024) B += 8;
  return B;
}

namespace {
template <class K>
bool msd_sort_impl(K* keys, K* alt, int64_t n, K** out, cudaStream_t s, SortStats* st,
                   const uint32_t* top_hist) {
  const int B = msd_prefix_bits(n);
  K* ko = nullptr;
  radix_passes<K>(keys, alt, nullptr, nullptr, nullptr, false, n, (64 - B) / 8, 8, &ko, nullptr,
                  s, st, top_hist);
  const int64_t nb = int64_t(1) << B;
  DevBuf<uint32_t> off(size_t(nb) + 1, s);
  DevBuf<uint32_t> flag(1, s);
  CG_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(uint32_t), s));
  k_bucket_bounds_search<K><<<unsigned((nb + 256) / 256), 256, 0, s>>>(ko, n, B, off.p);
  CG_LAUNCH_CHECK();
  launch_bucket_sort<K>(ko, off.p, n, nb, B, flag.p, nullptr, s);
  uint32_t* hf = static_cast<uint32_t*>(host_stage(sizeof(uint32_t)));
  CG_CUDA(cudaMemcpyAsync(hf, flag.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaStreamSynchronize(s));
  *out = ko;
  return hf[0] == 0;
}
}  // namespace

namespace {
// one warp per bucket: move its ucnt[b] unique rows from src + off[b] to
// dst + uoff[b] (only needed when duplicates were removed)
template <class K>
__global__ void k_compact_buckets(const K* __restrict__ src, const uint32_t* __restrict__ off,
                                  const uint32_t* __restrict__ ucnt, const uint32_t* __restrict__ uoff,
                                  int64_t nb, K* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t b = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; b < nb; b += nw) {
    const uint32_t c = ucnt[b], from = off[b], to = uoff[b];
    for (uint32_t q = lane; q < c; q += 32) dst[to + q] = src[from + q];
  }
}

template <class K>
bool sort_unique_impl(K* keys, K* alt, int64_t n, K** cells, int64_t* nc, cudaStream_t s,
                      SortStats* st, const uint32_t* top_hist, const uint32_t* pre_off = nullptr,
                      int pre_B = 0, const uint32_t* tile_hist = nullptr,
                      const uint32_t* side_dev = nullptr, uint32_t* side_host = nullptr,
                      int pre_skip = 0, const SweepIn* sw = nullptr) {
  // pre_off: keys are already grouped by their top pre_B bits (scatter pack),
  // pre_off[b] = first row of bucket b -- no global pass needed.
  // sw (the sweep path): the rows are in k_pack_sweep's 256 top-byte regions;
  // k_region_sweep splits them into the 2^16 bucket slots and the bucket
  // pass reads each slot and writes its bucket, sorted, to keys + off[b]
  const int B = sw ? 8 + sw->B2 : (pre_off ? pre_B : msd_prefix_bits(n));
  K* ko = keys;
  if (!pre_off && !sw)
    radix_passes<K>(keys, alt, nullptr, nullptr, nullptr, false, n, (64 - B) / 8, 8, &ko, nullptr,
                    s, st, top_hist, tile_hist);
  const int64_t nb = int64_t(1) << B;
  DevBuf<uint32_t> offb(pre_off ? 1 : size_t(nb) + 1, s);
  const uint32_t* offp = pre_off ? pre_off : offb.p;
  DevBuf<uint32_t> ucnt(size_t(nb), s), uoff(size_t(nb), s);
  DevBuf<uint32_t> flag(1, s);
  CG_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(uint32_t), s));
  DevBuf<K> slots;
  uint32_t cap16 = 0;
  if (sw) {
    // slot capacity: mean + max(mean / 4, 8 sigma) (uniform buckets of ~2^10
    // rows: 1312); a fuller bucket sets the overflow flag (caller re-runs)
    const int64_t mean = (n + nb - 1) / nb;
    int64_t sig8 = 8;
    while (sig8 * sig8 < 64 * mean) ++sig8;
    cap16 = uint32_t(mean + std::max(mean / 4, sig8) + 32);
    slots.alloc(size_t(nb) * cap16, s);
    DevBuf<uint32_t> cnt16(size_t(nb), s);
    CG_CUDA(cudaMemsetAsync(cnt16.p, 0, cnt16.n * 4, s));
    constexpr int TILE = RsCfg<K>::TILE;
    const uint32_t tpr = (sw->capr + TILE - 1) / TILE;
    auto go = [&](auto kern) {
      CG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      CG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(RsCfg<K>::SMEM)));
      kern<<<unsigned(256 * tpr), kSortThreads, RsCfg<K>::SMEM, s>>>(
          reinterpret_cast<const K*>(sw->regions), sw->capr, sw->rcnt, tpr, slots.p, cap16,
          cnt16.p, sw->ovf, sw->B2);
    };
    if (RS_PERSIST) {
      auto gop = [&](auto kern) {
        const size_t sm = 2 * RsCfg<K>::SMEM;
        CG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        CG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        const int grid = int(std::min<int64_t>(int64_t(256) * tpr, int64_t(num_sms()) * RS_PMINB));
        kern<<<unsigned(grid), kSortThreads, sm, s>>>(
            reinterpret_cast<const K*>(sw->regions), sw->capr, sw->rcnt, tpr, slots.p, cap16,
            cnt16.p, sw->ovf, sw->B2);
      };
      if (sw->B2 == 8) gop(k_region_sweep_p<K, 8>);
      else gop(k_region_sweep_p<K, 0>);
    } else if (sw->B2 == 8) {
      go(k_region_sweep<K, 8>);
    } else {
      go(k_region_sweep<K, 0>);
    }
    CG_LAUNCH_CHECK();
    k_clip_counts<<<grid_for(nb + 1, 256), 256, 0, s>>>(cnt16.p, nb, cap16, offb.p);
    CG_LAUNCH_CHECK();
    launch_scan_u32(offb.p, nb + 1, s);
    if (st) st->passes += 1;  // the region sweep (the first partition ran in the pack)
  } else if (!pre_off) {
    k_bucket_bounds_search<K><<<unsigned((nb + 256) / 256), 256, 0, s>>>(ko, n, B, offb.p);
    CG_LAUNCH_CHECK();
  }
  // the bucket kernels skip the key bytes every key of a bucket shares: the
  // top pre_skip + B bits
  uint32_t* Tix = sw ? sw->T : nullptr;
  launch_bucket_sort<K>(ko, offp, n, nb, B + pre_skip, flag.p, ucnt.p, s, sw ? slots.p : nullptr,
                        cap16, Tix, Tix ? sw->F : nullptr, Tix ? sw->b : 0, B,
                        sw ? sw->ovf : nullptr);
  CG_CUDA(cudaMemcpyAsync(uoff.p, ucnt.p, size_t(nb) * 4, cudaMemcpyDeviceToDevice, s));
  launch_scan_u32(uoff.p, nb, s);
  uint32_t* h = static_cast<uint32_t*>(host_stage(5 * sizeof(uint32_t)));
  h[4] = 0;
  if (sw) CG_CUDA(cudaMemcpyAsync(h + 4, sw->ovf, 4, cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaMemcpyAsync(h, flag.p, 4, cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaMemcpyAsync(h + 1, uoff.p + nb - 1, 4, cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaMemcpyAsync(h + 2, ucnt.p + nb - 1, 4, cudaMemcpyDeviceToHost, s));
  // the caller's input-error flag rides on the same round trip
  if (side_dev) CG_CUDA(cudaMemcpyAsync(h + 3, side_dev, 4, cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaStreamSynchronize(s));
  if (side_dev && side_host) *side_host = h[3];
  *cells = ko;
  if (h[0] || h[4]) return false;
  const int64_t total = int64_t(h[1]) + int64_t(h[2]);
  *nc = total;
  if (Tix) {  // the fused prefix index: final positions and the end sentinel
    if (total != n) {
      k_fix_index<<<grid_for(int64_t(1) << sw->b, 256), 256, 0, s>>>(Tix, sw->b, B, offp, uoff.p);
      CG_LAUNCH_CHECK();
    }
    k_ix_end<<<1, 1, 0, s>>>(Tix + (size_t(1) << sw->b), uint32_t(total));
    CG_LAUNCH_CHECK();
  }
  if (total != n) {  // duplicates removed: close the gaps between buckets
    K* dst = (ko == keys) ? alt : keys;
    const int64_t blocks = std::min<int64_t>((nb * 32 + 255) / 256, int64_t(num_sms()) * 16);
    k_compact_buckets<K><<<unsigned(std::max<int64_t>(1, blocks)), 256, 0, s>>>(ko, offp, ucnt.p,
                                                                                uoff.p, nb, dst);
    CG_LAUNCH_CHECK();
    *cells = dst;
  }
  return true;
}
}  // namespace

int msd_tile_rows(int W) {
  return W == 1 ? TileCfg<uint64_t, false>::TILE : TileCfg<ulonglong2, false>::TILE;
}

namespace {
template <class K>
bool merge_into_impl(K* gathered, const uint32_t* off, int64_t n, int B, int pre_skip, K* dst,
                     int64_t* nc, cudaStream_t s) {
  const int64_t nb = int64_t(1) << B;
  DevBuf<uint32_t> ucnt(size_t(nb), s), uoff(size_t(nb), s), flag(1, s);
  CG_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(uint32_t), s));
  launch_bucket_sort<K>(dst, off, n, nb, B + pre_skip, flag.p, ucnt.p, s, gathered, 0u);
  CG_CUDA(cudaMemcpyAsync(uoff.p, ucnt.p, size_t(nb) * 4, cudaMemcpyDeviceToDevice, s));
  launch_scan_u32(uoff.p, nb, s);
  uint32_t* h = static_cast<uint32_t*>(host_stage(3 * sizeof(uint32_t)));
  CG_CUDA(cudaMemcpyAsync(h, flag.p, 4, cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaMemcpyAsync(h + 1, uoff.p + nb - 1, 4, cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaMemcpyAsync(h + 2, ucnt.p + nb - 1, 4, cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaStreamSynchronize(s));
  if (h[0]) return false;
  const int64_t total = int64_t(h[1]) + int64_t(h[2]);
  if (total != n) {  // cross-run duplicates dropped: close the gaps (gathered is free now)
    const int64_t blocks = std::min<int64_t>((nb * 32 + 255) / 256, int64_t(num_sms()) * 16);
    k_compact_buckets<K><<<unsigned(std::max<int64_t>(1, blocks)), 256, 0, s>>>(dst, off, ucnt.p,
                                                                                uoff.p, nb, gathered);
    CG_LAUNCH_CHECK();
    CG_CUDA(cudaMemcpyAsync(dst, gathered, size_t(total) * sizeof(K), cudaMemcpyDeviceToDevice, s));
  }
  *nc = total;
  return true;
}
}  // namespace

bool merge_sorted_into(uint64_t* gathered, const uint32_t* off, int64_t n, int W, int B,
                       int pre_skip, uint64_t* dst, int64_t* nc, cudaStream_t s) {
  if (W == 1) return merge_into_impl<uint64_t>(gathered, off, n, B, pre_skip, dst, nc, s);
  if (W == 2)
    return merge_into_impl<ulonglong2>(reinterpret_cast<ulonglong2*>(gathered), off, n, B, pre_skip,
                                       reinterpret_cast<ulonglong2*>(dst), nc, s);
  return false;
}

bool sort_unique_msd(uint64_t* keys, uint64_t* alt, int64_t n, int W, uint64_t** cells,
                     int64_t* nc, cudaStream_t s, SortStats* st, const uint32_t* top_hist,
                     const uint32_t* pre_off, int pre_B, const uint32_t* tile_hist,
                     const uint32_t* side_dev, uint32_t* side_host, int pre_skip,
                     const SweepIn* sw) {
  if (W == 1) {
    uint64_t* o = nullptr;
    const bool ok = sort_unique_impl<uint64_t>(keys, alt, n, &o, nc, s, st, top_hist, pre_off,
                                               pre_B, tile_hist, side_dev, side_host, pre_skip, sw);
    *cells = o;
    return ok;
  }
  if (W == 2) {
    ulonglong2* o = nullptr;
    const bool ok = sort_unique_impl<ulonglong2>(reinterpret_cast<ulonglong2*>(keys),
                                                 reinterpret_cast<ulonglong2*>(alt), n, &o, nc, s,
                                                 st, top_hist, pre_off, pre_B, tile_hist, side_dev,
                                                 side_host, pre_skip, sw);
    *cells = reinterpret_cast<uint64_t*>(o);
    return ok;
  }
  return false;
}

// ---------------------------------------------------------------- merge of sorted runs
// (the distributed merge): G sorted runs are already
// ordered inside every top-B-bit bucket, so instead of re-sorting their
// concatenation the rows are gathered straight into the global buckets --
// per-run bucket bounds, global bucket offsets, one copy -- and the bucket
// pass (with its dedupe) does the rest.
namespace {
__global__ void k_set_u32(uint32_t* p, uint32_t v) { *p = v; }

__global__ void k_run_bucket_base(const uint32_t* __restrict__ offs, int G, int64_t nbk,
                                  uint32_t* __restrict__ size) {
  for (int64_t bk = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; bk < nbk;
       bk += int64_t(gridDim.x) * blockDim.x) {
    uint32_t t = 0;
    for (int g = 0; g < G; ++g) t += offs[g * (nbk + 1) + bk + 1] - offs[g * (nbk + 1) + bk];
    size[bk] = t;
  }
}

// base[g][bk] = start of run g's segment of bucket bk in the gathered array
__global__ void k_run_segment_base(const uint32_t* __restrict__ offs, const uint32_t* __restrict__ off,
                                   int G, int64_t nbk, uint32_t* __restrict__ base) {
  for (int64_t bk = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; bk < nbk;
       bk += int64_t(gridDim.x) * blockDim.x) {
    uint32_t t = off[bk];
    for (int g = 0; g < G; ++g) {
      base[g * nbk + bk] = t;
      t += offs[g * (nbk + 1) + bk + 1] - offs[g * (nbk + 1) + bk];
    }
  }
}

constexpr int kMaxRuns = 64;
struct RunCounts {
  int64_t c[kMaxRuns];
};

// bucket bounds of every run in one launch: thread (g, q) -> offs[g][q]
template <class K>
__global__ void k_runs_bounds(const K* __restrict__ runs, int64_t stride, RunCounts rc, int G,
                              int B, int skip, uint32_t* __restrict__ offs) {
  const int sh = 64 - B;
  const int64_t nq = (int64_t(1) << B) + 1;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < nq * G;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int g = int(t / nq);
    const int64_t q = t - int64_t(g) * nq;
    const K* keys = runs + int64_t(g) * stride;
    int64_t lo = 0, len = rc.c[g];
    while (len > 0) {
      const int64_t half = len >> 1;
      const uint64_t p = (KT<K>::top(__ldg(keys + lo + half)) << skip) >> sh;
      if (p < uint64_t(q)) {
        lo += half + 1;
        len -= half + 1;
      } else {
        len = half;
      }
    }
    offs[t] = uint32_t(lo);
  }
}

// every run's rows to their bucket segments, one launch over [G][stride]
template <class K>
__global__ void k_runs_gather(const K* __restrict__ runs, int64_t stride, RunCounts rc, int G,
                              int B, int skip, const uint32_t* __restrict__ offs,
                              const uint32_t* __restrict__ base, K* __restrict__ out) {
  const int64_t nbk = int64_t(1) << B;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < int64_t(G) * stride;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int g = int(t / stride);
    const int64_t e = t - int64_t(g) * stride;
    if (e >= rc.c[g]) continue;
    const K k = runs[t];
    const int64_t bk = int64_t((KT<K>::top(k) << skip) >> (64 - B));
    out[base[int64_t(g) * nbk + bk] + (e - offs[int64_t(g) * (nbk + 1) + bk])] = k;
  }
}

template <class K>
void gather_runs_impl(const K* runs, const int64_t* counts, int G, int64_t stride, int B, int skip,
                      K* out, uint32_t* off, cudaStream_t s) {
  if (G > kMaxRuns) throw CgError{CG_EINVAL, "more than 64 runs"};
  const int64_t nbk = int64_t(1) << B;
  DevBuf<uint32_t> offs(size_t(G) * (nbk + 1), s), base(size_t(G) * nbk, s);
  RunCounts rc{};
  int64_t total = 0;
  for (int g = 0; g < G; ++g) {
    rc.c[g] = counts[g];
    total += counts[g];
  }
  k_runs_bounds<K><<<grid_for((nbk + 1) * G, 256, 16), 256, 0, s>>>(runs, stride, rc, G, B, skip,
                                                                    offs.p);
  CG_LAUNCH_CHECK();
  k_run_bucket_base<<<grid_for(nbk, 256, 16), 256, 0, s>>>(offs.p, G, nbk, off);
  CG_LAUNCH_CHECK();
  launch_scan_u32(off, nbk, s);  // exclusive: bucket starts
  k_set_u32<<<1, 1, 0, s>>>(off + nbk, uint32_t(total));
  CG_LAUNCH_CHECK();
  k_run_segment_base<<<grid_for(nbk, 256, 16), 256, 0, s>>>(offs.p, off, G, nbk, base.p);
  CG_LAUNCH_CHECK();
  k_runs_gather<K><<<grid_for(int64_t(G) * stride, 256, 16), 256, 0, s>>>(runs, stride, rc, G, B,
                                                                          skip, offs.p, base.p, out);
  CG_LAUNCH_CHECK();
}
}  // namespace

void gather_runs_by_prefix(const uint64_t* runs, const int64_t* counts, int G, int64_t stride,
                           int W, int B, int skip, uint64_t* out, uint32_t* off, cudaStream_t s) {
  if (W == 1)
    gather_runs_impl<uint64_t>(runs, counts, G, stride, B, skip, out, off, s);
  else
    gather_runs_impl<ulonglong2>(reinterpret_cast<const ulonglong2*>(runs), counts, G, stride, B,
                                 skip, reinterpret_cast<ulonglong2*>(out), off, s);
}

void launch_prefix_bounds(const uint64_t* rows, int64_t n, int W, int B, uint32_t* off,
                          cudaStream_t s) {
  const int64_t nb = int64_t(1) << B;
  if (W == 1)
    k_bucket_bounds_search<uint64_t><<<unsigned((nb + 256) / 256), 256, 0, s>>>(rows, n, B, off);
  else if (W == 2)
    k_bucket_bounds_search<ulonglong2><<<unsigned((nb + 256) / 256), 256, 0, s>>>(
        reinterpret_cast<const ulonglong2*>(rows), n, B, off);
  else
    k_row_bounds_search<<<unsigned((nb + 256) / 256), 256, 0, s>>>(rows, n, W, B, off);
  CG_LAUNCH_CHECK();
}

bool sort_rows_msd(uint64_t* keys, uint64_t* alt, int64_t n, int W, uint64_t** sorted,
                   cudaStream_t s, SortStats* st, const uint32_t* top_hist) {
  if (W == 1) {
    uint64_t* o = nullptr;
    const bool ok = msd_sort_impl<uint64_t>(keys, alt, n, &o, s, st, top_hist);
    *sorted = o;
    return ok;
  }
  if (W == 2) {
    ulonglong2* o = nullptr;
    const bool ok = msd_sort_impl<ulonglong2>(reinterpret_cast<ulonglong2*>(keys),
                                              reinterpret_cast<ulonglong2*>(alt), n, &o, s, st,
                                              top_hist);
    *sorted = reinterpret_cast<uint64_t*>(o);
    return ok;
  }
  return false;
}

}  // namespace cgk
