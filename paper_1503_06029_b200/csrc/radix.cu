// radix.cu -- stable LSD radix sort engine (8-bit digits, one-sweep passes
// with decoupled look-back) used by the cell sort (a2), the popcount layering
// (a4) and the canonical edge sort (a7).
//
// "As these vectors are binary, the sorting can clearly be done in O(n*ell)
// time, using the radix sort algorithm".  The paper does not say
// which radix sort; this is a one-sweep LSD design for sm_100a:
//   * one histogram kernel reads the keys once and counts every digit
//     (run-length accumulated in registers so constant digits do not
//     serialise shared-memory atomics); digits whose histogram is a single
//     bucket are skipped (pad bits, small edge indices, narrow popcounts);
//   * each pass: a CTA takes a tile by atomic ticket, loads it warp-striped
//     (coalesced), ranks digits per warp with __match_any_sync, publishes
//     per-digit tile counts through a decoupled look-back, reorders the tile
//     in shared memory by digit and writes each digit run contiguously.
#include <algorithm>
#include <vector>

#include "kernels.cuh"

namespace cgk {
namespace {

constexpr int kRadix = 256;
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;

template <class K, bool V>
struct TileCfg {
  static constexpr int IPT = V ? 12 : 16;
  static constexpr int TILE = kSortThreads * IPT;
  static constexpr size_t SMEM = size_t(TILE) * (sizeof(K) + (V ? 4 : 0));
};

template <class K>
__global__ void __launch_bounds__(256) k_digit_hist(const K* __restrict__ keys, int64_t n,
                                                    int ndig, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[8][kRadix];
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
    const uint64_t k = uint64_t(keys[i]);
#pragma unroll
    for (int d = 0; d < 8; ++d) {
      if (d < ndig) {
        const uint32_t b = uint32_t(k >> (8 * d)) & 255u;
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
    if (d < ndig && cnt[d]) atomicAdd(&h[d][last[d]], cnt[d]);
  __syncthreads();
  for (int i = threadIdx.x; i < ndig * kRadix; i += blockDim.x) {
    const uint32_t v = (&h[0][0])[i];
    if (v) atomicAdd(&hist[i], v);
  }
}

template <class K, bool V>
__global__ void __launch_bounds__(kSortThreads)
    k_onesweep(const K* __restrict__ kin, K* __restrict__ kout, const uint32_t* __restrict__ vin,
               uint32_t* __restrict__ vout, int64_t n, int shift,
               const uint32_t* __restrict__ bucket_base, uint64_t* status,
               uint32_t* tile_counter, uint32_t epoch) {
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
      key[i] = 0;
      val[i] = 0;
    }
  }
  // warp-level stable ranking: items are visited in index order
  // (item i of every lane precedes item i+1; lanes in order within an item)
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const bool valid = wbase + i * 32 + lane < n;
    const uint32_t d = valid ? (uint32_t(uint64_t(key[i]) >> shift) & 255u) : 256u;
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
  const uint32_t excl_tiles = lookback(status, tile, kRadix, tid, total, epoch);
  uint32_t tile_n_u;
  const uint32_t dex = block_excl_scan(total, s_scan, &tile_n_u);
  s_dexcl[tid] = dex;
  s_gbase[tid] = bucket_base[tid] + excl_tiles - dex;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const bool valid = wbase + i * 32 + lane < n;
    if (valid) {
      const uint32_t d = uint32_t(uint64_t(key[i]) >> shift) & 255u;
      const uint32_t pos = s_dexcl[d] + wcnt[w][d] + rank[i];
      skeys[pos] = key[i];
      if (V) svals[pos] = val[i];
    }
  }
  __syncthreads();
  const int tile_n = int(tile_n_u);
  for (int j = tid; j < tile_n; j += kSortThreads) {
    const K k = skeys[j];
    const uint32_t d = uint32_t(uint64_t(k) >> shift) & 255u;
    const uint32_t gp = s_gbase[d] + uint32_t(j);
    kout[gp] = k;
    if (V) vout[gp] = svals[j];
  }
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

int grid_for(int64_t n, int threads, int per_sm = 8) {
  int64_t b = (n + threads - 1) / threads;
  int64_t cap = int64_t(num_sms()) * per_sm;
  return int(std::max<int64_t>(1, std::min(b, cap)));
}

}  // namespace

template <class K>
void radix_sort(K* keys, K* keys_alt, const uint32_t* vals_in, uint32_t* vals, uint32_t* vals_alt,
                bool want_vals, int64_t n, int key_bits, K** keys_out, uint32_t** vals_out,
                cudaStream_t s, SortStats* st) {
  const int ndig = std::max(1, (key_bits + 7) / 8);
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
  if (n <= 1) {
    identity_or_input();
    return;
  }
  DevBuf<uint32_t> hist(size_t(ndig) * kRadix, s);
  CG_CUDA(cudaMemsetAsync(hist.p, 0, hist.n * sizeof(uint32_t), s));
  k_digit_hist<K><<<grid_for(n, 256, 4), 256, 0, s>>>(keys, n, ndig, hist.p);
  CG_LAUNCH_CHECK();
  uint32_t* hh = static_cast<uint32_t*>(host_stage(hist.n * sizeof(uint32_t)));
  CG_CUDA(cudaMemcpyAsync(hh, hist.p, hist.n * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaStreamSynchronize(s));
  std::vector<int> digits;
  std::vector<uint32_t> bases;
  for (int d = 0; d < ndig; ++d) {
    const uint32_t* h = hh + d * kRadix;
    bool trivial = false;
    for (int b = 0; b < kRadix; ++b)
      if (int64_t(h[b]) == n) trivial = true;
    if (trivial) continue;
    digits.push_back(d);
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
  DevBuf<uint32_t> dbases(bases.size(), s);
  CG_CUDA(cudaMemcpyAsync(dbases.p, bases.data(), bases.size() * sizeof(uint32_t),
                          cudaMemcpyHostToDevice, s));
  const bool V = want_vals;
  const int TILE = V ? TileCfg<K, true>::TILE : TileCfg<K, false>::TILE;
  const int64_t tiles = (n + TILE - 1) / TILE;
  DevBuf<uint64_t> status(size_t(tiles) * kRadix, s);
  DevBuf<uint32_t> counters(size_t(P), s);
  CG_CUDA(cudaMemsetAsync(status.p, 0, status.n * sizeof(uint64_t), s));
  CG_CUDA(cudaMemsetAsync(counters.p, 0, counters.n * sizeof(uint32_t), s));
  // The host staging buffer is reused by later read-backs; bases were copied
  // from a std::vector, and the copy is ordered before those on the stream.
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
          uint32_t(p + 1));
    } else {
      k_onesweep<K, false><<<unsigned(tiles), kSortThreads, TileCfg<K, false>::SMEM, s>>>(
          ck, ak, nullptr, nullptr, n, shift, dbases.p + p * kRadix, status.p, counters.p + p,
          uint32_t(p + 1));
    }
    CG_LAUNCH_CHECK();
    std::swap(ck, ak);
    if (V) {
      // next pass reads av; writes into the other buffer (never into vals_in)
      uint32_t* written = av;
      av = (cv == vals_in) ? spare_v : const_cast<uint32_t*>(cv);
      cv = written;
    }
  }
  // The pass kernels must finish before the temporaries (status, bases) are
  // released: stream-ordered frees take care of that.
  *keys_out = ck;
  if (vals_out && V) *vals_out = const_cast<uint32_t*>(cv);
}

template void radix_sort<uint32_t>(uint32_t*, uint32_t*, const uint32_t*, uint32_t*, uint32_t*,
                                   bool, int64_t, int, uint32_t**, uint32_t**, cudaStream_t,
                                   SortStats*);
template void radix_sort<uint64_t>(uint64_t*, uint64_t*, const uint32_t*, uint32_t*, uint32_t*,
                                   bool, int64_t, int, uint64_t**, uint32_t**, cudaStream_t,
                                   SortStats*);

void sort_rows_multiword(const uint64_t* keys, int64_t n, int W, uint64_t* sorted,
                         cudaStream_t s, SortStats* st) {
  DevBuf<uint64_t> kw(size_t(n), s), kw_alt(size_t(n), s);
  DevBuf<uint32_t> ia(size_t(n), s), ib(size_t(n), s);
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
  launch_gather_rows(keys, idx, n, W, sorted, s);
}

}  // namespace cgk
