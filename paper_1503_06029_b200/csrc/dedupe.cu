// dedupe.cu -- a3: duplicate removal and compaction into the cell table.
//
// "During this step we also remove all duplicates in X"; X may be a
// multiset and only unique pairs may be output.  Over the
// canonically sorted rows, row g starts a new cell iff g == 0 or it differs
// from row g-1.  Flags are counted per warp with __ballot_sync/__popc,
// scanned per block, and the block's base is found by decoupled look-back,
// so cells are written in one pass straight to their final position.
// The same pass records per cell
//   popc[c] = popcount of the cell (its layer, a4) and
//   lcp[c]  = number of leading bits shared with the next cell (0xffff for
//             the last cell): the exact probe-pruning bound of a6.
#include "kernels.cuh"

namespace cgk {
namespace {

constexpr int kDedupThreads = 256;
constexpr int kDedupIPT = 8;  // rows per thread (contiguous run)

template <int WC>
struct Row {
  // compile-time W when WC > 0, else runtime
  __device__ static __forceinline__ bool equal(const uint64_t* a, const uint64_t* b, int W) {
    const int n = WC > 0 ? WC : W;
    for (int w = 0; w < n; ++w)
      if (a[w] != b[w]) return false;
    return true;
  }
  __device__ static __forceinline__ int lcp(const uint64_t* a, const uint64_t* b, int W) {
    const int n = WC > 0 ? WC : W;
    for (int w = 0; w < n; ++w) {
      const uint64_t x = a[w] ^ b[w];
      if (x) return 64 * w + __clzll(x);
    }
    return 64 * n;
  }
  __device__ static __forceinline__ uint32_t popc(const uint64_t* a, int W) {
    const int n = WC > 0 ? WC : W;
    uint32_t c = 0;
    for (int w = 0; w < n; ++w) c += __popcll(a[w]);
    return c;
  }
};

template <int WC>
__global__ void __launch_bounds__(kDedupThreads)
    k_dedupe(const uint64_t* __restrict__ sorted, int64_t n, int W, uint64_t* __restrict__ cells,
             uint32_t* __restrict__ popc, uint16_t* __restrict__ lcp_out, uint64_t* status,
             uint32_t* tile_counter, uint32_t* n_cells) {
  constexpr int TILE = kDedupThreads * kDedupIPT;
  constexpr int NWARP = kDedupThreads / 32;
  __shared__ uint32_t s_warp[NWARP];
  __shared__ uint32_t s_base;
  __shared__ uint32_t s_tile;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  // warp `wid` owns rows [wb, wb + 32*IPT): step i covers 32 consecutive rows
  const int64_t wb = tile * TILE + int64_t(wid) * 32 * kDedupIPT;
  using R = Row<WC>;
  uint32_t ball[kDedupIPT];
  uint32_t wcount = 0;
#pragma unroll
  for (int i = 0; i < kDedupIPT; ++i) {
    const int64_t g = wb + i * 32 + lane;
    bool f = false;
    if (g < n) f = (g == 0) || !R::equal(sorted + g * W, sorted + (g - 1) * W, W);
    ball[i] = __ballot_sync(kFull, f);
    wcount += __popc(ball[i]);
  }
  if (lane == 0) s_warp[wid] = wcount;
  __syncthreads();
  if (wid == 0) {
    uint32_t run = 0;
    uint32_t mine = 0;
    for (int w = 0; w < NWARP; ++w) {
      const uint32_t c = s_warp[w];
      if (lane == w) mine = run;
      run += c;
    }
    __syncwarp();
    if (lane < NWARP) s_warp[lane] = mine;
    const uint32_t base = lookback_warp(status, tile, run, 1);
    if (lane == 0) {
      s_base = base;
      if (tile * TILE < n && (tile + 1) * TILE >= n) *n_cells = base + run;
    }
  }
  __syncthreads();
  uint32_t c0 = s_base + s_warp[wid];  // first cell index of this warp's flags
  const uint32_t lt = lanemask_lt();
  const int nw = WC > 0 ? WC : W;
#pragma unroll
  for (int i = 0; i < kDedupIPT; ++i) {
    const int64_t g = wb + i * 32 + lane;
    const uint32_t b = ball[i];
    if (g < n) {
      const uint64_t* row = sorted + g * W;
      // cell of row g = (flags at rows <= g) - 1
      const uint32_t cell = c0 + __popc(b & lt) + ((b >> lane) & 1) - 1;
      if ((b >> lane) & 1) {
        for (int w = 0; w < nw; ++w) cells[int64_t(cell) * nw + w] = row[w];
        popc[cell] = R::popc(row, W);
      }
      // last row of its run: lcp with the next distinct row (a6 pruning bound)
      if (g + 1 >= n) {
        lcp_out[cell] = 0xffff;
      } else {
        const uint64_t* nxt = row + W;
        if (!R::equal(row, nxt, W)) lcp_out[cell] = uint16_t(R::lcp(row, nxt, W));
      }
    }
    c0 += __popc(b);
  }
}

// ---- W > 2: gather + dedupe in one warp-cooperative pass.  The multi-word
// sort returns the canonical order as row indices; this kernel moves the
// rows in that order and flags the first row of each run of equal rows
// in the same pass.  L lanes per row (W <= L <= 32), lane w moving
// word w, so a row is ONE contiguous access of the warp (the north star's
// warp-cooperative compares for long ell: with a thread per row every load
// instruction touched 32 different rows).  A warp owns 32 consecutive sorted
// positions, R = 32 / L rows per step; the previous row of a group is the
// group before it (or the last group of the previous step) by shuffle.
#ifndef GD_NOLB
#define GD_NOLB 0
#endif
template <int L>
__global__ void __launch_bounds__(256)
    k_gather_dedupe(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ order,
                    int64_t n, int W, uint64_t* __restrict__ cells, uint32_t* __restrict__ popc,
                    uint16_t* __restrict__ lcp_out, uint64_t* status, uint32_t* tile_counter,
                    uint32_t* n_cells) {
  constexpr int R = 32 / L;  // rows per warp step
  constexpr int S = 32 / R;  // steps per warp (32 rows)
  constexpr int NWARP = 8;
  constexpr int TILE = NWARP * 32;
  __shared__ uint32_t s_warp[NWARP];
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_pop[NWARP][32];
  __shared__ uint16_t s_lcp[NWARP][32];
  __shared__ uint32_t s_lb[97];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int q = lane / L, w = lane % L;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t wb = tile * TILE + int64_t(wid) * 32;
  uint64_t val[S];
  uint32_t flags = 0;  // bit r: sorted position wb + r starts a cell (all lanes)
  uint64_t xp = 0;     // previous step's word (group R-1 holds the row before group 0)
  {
    const int64_t g = wb - 1;  // the row before the warp's first position
    if (q == R - 1 && g >= 0 && g < n && w < W) xp = keys[(order ? int64_t(order[g]) : g) * W + w];
  }
  // all of the warp's rows in flight first, then the compares
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int64_t g = wb + s * R + q;
    const int64_t src = order ? int64_t(order[g < n ? g : 0]) : g;  // no order: rows already sorted
    val[s] = (g < n && w < W) ? keys[src * W + w] : 0ull;
  }
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int64_t g = wb + s * R + q;
    const bool ok = g < n;
    const uint64_t x = val[s];
    const uint64_t a = __shfl_sync(kFull, x, (lane + 32 - L) & 31);
    const uint64_t c = __shfl_sync(kFull, xp, (R - 1) * L + w);
    const uint64_t d = x ^ (q > 0 ? a : c);
    xp = x;
    const uint32_t gm = L == 32 ? kFull : (((1u << L) - 1u) << (q * L));
    const uint32_t gd = __ballot_sync(kFull, d != 0) & gm;
    const bool flag = ok && (g == 0 || gd != 0);
    const uint32_t fb = __ballot_sync(kFull, flag && w == 0);
#pragma unroll
    for (int qq = 0; qq < R; ++qq) flags |= ((fb >> (qq * L)) & 1u) << (s * R + qq);
    if (popc) {  // per-cell metadata for the layered dictionary (uniform branch)
      uint32_t pc = __popcll(x);
#pragma unroll
      for (int o = L / 2; o > 0; o >>= 1) pc += __shfl_xor_sync(kFull, pc, o);
      // lcp(previous row, this row): the first differing word of the group
      const int f = gd ? __ffs(gd) - 1 : lane;
      const uint64_t xd = __shfl_sync(kFull, d, f);
      if (w == 0 && ok) {
        s_pop[wid][s * R + q] = pc;
        s_lcp[wid][s * R + q] = gd ? uint16_t((f - q * L) * 64 + __clzll(xd)) : uint16_t(0xffff);
      }
    }
  }
  if (lane == 0) s_warp[wid] = __popc(flags);
  __syncthreads();
  uint32_t run = 0, mine = 0;
  for (int ww = 0; ww < NWARP; ++ww) {
    const uint32_t c = s_warp[ww];
    if (ww == wid) mine = run;
    run += c;
  }
  // the whole CTA looks back (256 predecessors per round)
#if GD_NOLB  // diagnostics only (wrong output): the kernel without its look-back
  const uint32_t base = uint32_t(tile) * TILE;
#else
  const uint32_t base = lookback_block(status, tile, run, 1, s_lb);
#endif
  if (tid == 0 && tile * TILE < n && (tile + 1) * TILE >= n) *n_cells = base + run;
  const uint32_t c0 = base + mine;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int r = s * R + q;
    const int64_t g = wb + r;
    if (g < n) {
      // cell of row g = (flags at rows <= g) - 1
      const uint32_t cell = c0 + __popc(flags & (0xffffffffu >> (31 - r))) - 1;
      if ((flags >> r) & 1u) {
        if (w < W) cells[int64_t(cell) * W + w] = val[s];
        if (popc && w == 0) {
          popc[cell] = s_pop[wid][r];
          if (g > 0) lcp_out[cell - 1] = s_lcp[wid][r];  // the previous cell vs this one
        }
      }
      if (popc && w == 0 && g + 1 == n) lcp_out[cell] = 0xffff;
    }
  }
}

template <int WC>
__global__ void k_cell_meta(const uint64_t* __restrict__ cells, int64_t nc, int W,
                            uint32_t* __restrict__ popc, uint16_t* __restrict__ lcp) {
  using R = Row<WC>;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nc;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t* row = cells + i * W;
    if (popc) popc[i] = R::popc(row, W);
    lcp[i] = (i + 1 < nc) ? uint16_t(R::lcp(row, row + W, W)) : uint16_t(0xffff);
  }
}

// ---- hash dedupe for skewed inputs (the MSD buckets overflowed: few
// distinct rows, heavy duplication): every row is inserted into an
// open-addressed table of row indices (load <= 1/2); the first row of each
// distinct value to claim a slot is kept, later equal rows are dropped.  The
// kept rows are then compacted (flags + scan) and only they are sorted.
__device__ __forceinline__ uint64_t row_hash64(const uint64_t* r, int W) {
  uint64_t h = 0x9E3779B97F4A7C15ull;
  for (int w = 0; w < W; ++w) {
    h ^= r[w] + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
    h *= 0xff51afd7ed558ccdull;
    h ^= h >> 33;
  }
  return h;
}

__global__ void k_hash_unique(const uint64_t* __restrict__ rows, int64_t n, int W,
                              uint32_t* __restrict__ table, uint64_t mask,
                              uint32_t* __restrict__ flag) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t* r = rows + i * W;
    uint64_t h = row_hash64(r, W) & mask;
    uint32_t keep = 0;
    while (true) {
      uint32_t v = table[h];
      if (v == 0xffffffffu) {
        v = atomicCAS(&table[h], 0xffffffffu, uint32_t(i));
        if (v == 0xffffffffu) {
          keep = 1;
          break;
        }
      }
      const uint64_t* o = rows + int64_t(v) * W;
      bool eq = true;
      for (int w = 0; w < W && eq; ++w) eq = o[w] == r[w];
      if (eq) break;  // a copy of a row already kept
      h = (h + 1) & mask;
    }
    flag[i] = keep;
  }
}

__global__ void k_hash_compact(const uint64_t* __restrict__ rows, int64_t n, int W,
                               const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                               uint64_t* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    if (flag[i])
      for (int w = 0; w < W; ++w) out[int64_t(pos[i]) * W + w] = rows[i * W + w];
}

// Duplication estimate: 1024 rows sampled at a fixed stride, their 64-bit
// row hashes inserted into a shared-memory table; *hits = sampled rows whose
// hash was already there (a repeated row, or a 2^-64-rare collision).
constexpr int kDupSample = 1024;
__global__ void __launch_bounds__(kDupSample)
    k_dup_sample(const uint64_t* __restrict__ rows, int64_t n, int W, uint32_t* hits) {
  __shared__ unsigned long long tab[2 * kDupSample];
  __shared__ uint32_t s_hits;
  for (int t = threadIdx.x; t < 2 * kDupSample; t += blockDim.x) tab[t] = 0ull;
  if (threadIdx.x == 0) s_hits = 0;
  __syncthreads();
  const int64_t stride = n / kDupSample > 0 ? n / kDupSample : 1;
  for (int q = threadIdx.x; q < kDupSample && int64_t(q) * stride < n; q += blockDim.x) {
    const uint64_t h = row_hash64(rows + int64_t(q) * stride * W, W) | 1ull;
    uint32_t b = uint32_t(h >> 53) & (2 * kDupSample - 1);
    while (true) {
      const unsigned long long o = atomicCAS(&tab[b], 0ull, h);
      if (o == 0ull) break;
      if (o == h) {
        atomicAdd(&s_hits, 1u);
        break;
      }
      b = (b + 1) & (2 * kDupSample - 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *hits = s_hits;
}

}  // namespace

// Top-byte histogram of up to kTopSample rows of a byte matrix at a fixed
// stride (the first 8 bytes of a row are the top byte of its packed key):
// the sweep path's region-skew estimate.
constexpr int kTopSample = 65536;
__global__ void __launch_bounds__(256) k_top_sample(const uint8_t* __restrict__ vecs, int64_t n,
                                                    int ell, int64_t stride, int S,
                                                    uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0u;
  __syncthreads();
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < S; q += gridDim.x * blockDim.x) {
    const uint64_t x = *reinterpret_cast<const uint64_t*>(vecs + int64_t(q) * stride * ell);
    atomicAdd(&h[uint32_t((x * 0x8040201008040201ull) >> 56)], 1u);
  }
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}

uint32_t sample_duplicates_and_top(const uint8_t* vecs, int64_t n, int ell, cudaStream_t s,
                                   double* max_top_share) {
  DevBuf<uint32_t> h(1 + 256, s);
  CG_CUDA(cudaMemsetAsync(h.p, 0, h.n * 4, s));
  k_dup_sample<<<1, kDupSample, 0, s>>>(reinterpret_cast<const uint64_t*>(vecs), n, ell / 8, h.p);
  CG_LAUNCH_CHECK();
  const int S = int(std::min<int64_t>(n, kTopSample));
  const int64_t stride = std::max<int64_t>(1, n / S);
  k_top_sample<<<64, 256, 0, s>>>(vecs, n, ell, stride, S, h.p + 1);
  CG_LAUNCH_CHECK();
  uint32_t* hh = static_cast<uint32_t*>(host_stage(257 * sizeof(uint32_t)));
  CG_CUDA(cudaMemcpyAsync(hh, h.p, 257 * 4, cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaStreamSynchronize(s));
  uint32_t mx = 0;
  for (int b = 0; b < 256; ++b) mx = std::max(mx, hh[1 + b]);
  *max_top_share = double(mx) / double(S);
  return hh[0];
}

uint32_t sample_duplicates(const uint64_t* rows, int64_t n, int W, cudaStream_t s) {
  DevBuf<uint32_t> h(1, s);
  k_dup_sample<<<1, kDupSample, 0, s>>>(rows, n, W, h.p);  // a thread per sampled row
  CG_LAUNCH_CHECK();
  uint32_t* hh = static_cast<uint32_t*>(host_stage(sizeof(uint32_t)));
  CG_CUDA(cudaMemcpyAsync(hh, h.p, 4, cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaStreamSynchronize(s));
  return hh[0];
}

int64_t hash_unique_rows(const uint64_t* rows, int64_t n, int W, uint64_t* out, cudaStream_t s) {
  uint64_t cap = 1;
  while (cap < 2 * uint64_t(n)) cap <<= 1;
  DevBuf<uint32_t> table(cap, s), flag(size_t(n), s), pos(size_t(n), s);
  CG_CUDA(cudaMemsetAsync(table.p, 0xff, cap * 4, s));
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 16);
  k_hash_unique<<<unsigned(std::max<int64_t>(1, blocks)), 256, 0, s>>>(rows, n, W, table.p, cap - 1,
                                                                       flag.p);
  CG_LAUNCH_CHECK();
  CG_CUDA(cudaMemcpyAsync(pos.p, flag.p, size_t(n) * 4, cudaMemcpyDeviceToDevice, s));
  launch_scan_u32(pos.p, n, s);
  uint32_t* h = static_cast<uint32_t*>(host_stage(2 * sizeof(uint32_t)));
  CG_CUDA(cudaMemcpyAsync(h, pos.p + n - 1, 4, cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaMemcpyAsync(h + 1, flag.p + n - 1, 4, cudaMemcpyDeviceToHost, s));
  k_hash_compact<<<unsigned(std::max<int64_t>(1, blocks)), 256, 0, s>>>(rows, n, W, flag.p, pos.p, out);
  CG_LAUNCH_CHECK();
  CG_CUDA(cudaStreamSynchronize(s));
  return int64_t(h[0]) + h[1];
}

void launch_cell_meta(const uint64_t* cells, int64_t nc, int W, uint32_t* popc, uint16_t* lcp,
                      cudaStream_t s) {
  if (nc <= 0) return;
  const int64_t blocks = std::min<int64_t>((nc + 255) / 256, int64_t(num_sms()) * 16);
  const unsigned g = unsigned(std::max<int64_t>(1, blocks));
  switch (W) {
    case 1: k_cell_meta<1><<<g, 256, 0, s>>>(cells, nc, W, popc, lcp); break;
    case 2: k_cell_meta<2><<<g, 256, 0, s>>>(cells, nc, W, popc, lcp); break;
    default: k_cell_meta<0><<<g, 256, 0, s>>>(cells, nc, W, popc, lcp); break;
  }
  CG_LAUNCH_CHECK();
}

bool gather_dedupe_ok(int W) { return W > 2 && W <= 32; }

void launch_gather_dedupe(const uint64_t* keys, const uint32_t* order, int64_t n, int W,
                          uint64_t* cells, uint32_t* popc, uint16_t* lcp, uint32_t* n_cells,
                          cudaStream_t s) {
  constexpr int TILE = 256;
  const int64_t tiles = (n + TILE - 1) / TILE;
  DevBuf<uint64_t> status(size_t(tiles), s);
  DevBuf<uint32_t> counter(1, s);
  CG_CUDA(cudaMemsetAsync(status.p, 0, status.n * sizeof(uint64_t), s));
  CG_CUDA(cudaMemsetAsync(counter.p, 0, sizeof(uint32_t), s));
  const unsigned g = unsigned(tiles);
#define CG_GD_ARGS keys, order, n, W, cells, popc, lcp, status.p, counter.p, n_cells
  if (W <= 4) k_gather_dedupe<4><<<g, 256, 0, s>>>(CG_GD_ARGS);
  else if (W <= 8) k_gather_dedupe<8><<<g, 256, 0, s>>>(CG_GD_ARGS);
  else if (W <= 16) k_gather_dedupe<16><<<g, 256, 0, s>>>(CG_GD_ARGS);
  else k_gather_dedupe<32><<<g, 256, 0, s>>>(CG_GD_ARGS);
#undef CG_GD_ARGS
  CG_LAUNCH_CHECK();
}

void launch_dedupe(const uint64_t* sorted, int64_t n, int W, uint64_t* cells, uint32_t* popc,
                   uint16_t* lcp, uint32_t* n_cells, cudaStream_t s) {
  constexpr int TILE = kDedupThreads * kDedupIPT;
  const int64_t tiles = (n + TILE - 1) / TILE;
  DevBuf<uint64_t> status(size_t(tiles), s);
  DevBuf<uint32_t> counter(1, s);
  CG_CUDA(cudaMemsetAsync(status.p, 0, status.n * sizeof(uint64_t), s));
  CG_CUDA(cudaMemsetAsync(counter.p, 0, sizeof(uint32_t), s));
  const unsigned g = unsigned(tiles);
  switch (W) {
    case 1: k_dedupe<1><<<g, kDedupThreads, 0, s>>>(sorted, n, W, cells, popc, lcp, status.p, counter.p, n_cells); break;
    case 2: k_dedupe<2><<<g, kDedupThreads, 0, s>>>(sorted, n, W, cells, popc, lcp, status.p, counter.p, n_cells); break;
    case 4: k_dedupe<4><<<g, kDedupThreads, 0, s>>>(sorted, n, W, cells, popc, lcp, status.p, counter.p, n_cells); break;
    default: k_dedupe<0><<<g, kDedupThreads, 0, s>>>(sorted, n, W, cells, popc, lcp, status.p, counter.p, n_cells); break;
  }
  CG_LAUNCH_CHECK();
}

}  // namespace cgk
