// edges.cu -- prefix sums used to place the canonical edge list (a7).
//
// The probe writes each 32-cell tile's hits as one sorted block of a scratch
// list and records the tile's hit count; the canonical position of a tile's
// block is the exclusive prefix sum of the counts of the tiles before it
// (tile order = canonical source order; DESIGN G4).  Edge totals can
// reach n*ell/2 >= 2^32, so those offsets are 64-bit
// (k_scan_u32_u64); k_scan_u32 serves totals bounded by a row count < 2^32.
#include "kernels.cuh"

namespace cgk {
namespace {

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

// Decoupled look-back over 64-bit status words [flag:2 | value:62] (the
// status array is zeroed before the launch, so no epoch is needed).
__device__ __forceinline__ uint64_t lookback_warp62(uint64_t* status, int64_t tile, uint64_t agg) {
  const int lane = threadIdx.x & 31;
  constexpr uint64_t kAgg = uint64_t(1) << 62, kInc = uint64_t(2) << 62, kVal = kAgg - 1;
  if (tile == 0) {
    if (lane == 0) st_relaxed_u64(status, kInc | agg);
    return 0;
  }
  if (lane == 0) st_relaxed_u64(status + tile, kAgg | agg);
  uint64_t excl = 0;
  int64_t j = tile - 1;
  while (true) {
    const int64_t jj = j - lane;
    const uint64_t s = jj >= 0 ? ld_relaxed_u64(status + jj) : kInc;
    const uint32_t flag = uint32_t(s >> 62);
    const uint32_t notready = __ballot_sync(kFull, flag == 0);
    const uint32_t incl = __ballot_sync(kFull, flag == 2);
    const int first_inc = incl ? __ffs(incl) - 1 : 32;
    const int first_nr = notready ? __ffs(notready) - 1 : 32;
    const int take = first_nr < first_inc ? first_nr : (first_inc < 32 ? first_inc + 1 : 32);
    uint64_t v = lane < take ? (s & kVal) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    excl += v;
    if (first_inc < 32 && first_inc < first_nr) break;
    j -= take;
  }
  if (lane == 0) st_relaxed_u64(status + tile, kInc | (excl + agg));
  return excl;
}

// out[i] = sum of in[0..i) as u64 (in: u32 counts); tiles by atomic ticket
__global__ void __launch_bounds__(kScanThreads)
    k_scan_u32_u64(const uint32_t* __restrict__ in, uint64_t* __restrict__ out, int64_t n,
                   uint64_t* status, uint32_t* ticket) {
  constexpr int TILE = kScanThreads * kScanIPT;
  __shared__ uint32_t s_scan[33];
  __shared__ uint64_t s_base;
  __shared__ uint32_t s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t g0 = tile * TILE + int64_t(threadIdx.x) * kScanIPT;
  uint32_t x[kScanIPT];
  uint32_t sum = 0;  // a tile's counts are per-tile hit counts (<= 2^17 each): no overflow
#pragma unroll
  for (int i = 0; i < kScanIPT; ++i) {
    x[i] = (g0 + i < n) ? in[g0 + i] : 0u;
    sum += x[i];
  }
  uint32_t total;
  const uint32_t excl = block_excl_scan(sum, s_scan, &total);
  if (threadIdx.x < 32) {
    const uint64_t b = lookback_warp62(status, tile, total);
    if (threadIdx.x == 0) s_base = b;
  }
  __syncthreads();
  uint64_t run = s_base + excl;
#pragma unroll
  for (int i = 0; i < kScanIPT; ++i) {
    if (g0 + i < n) out[g0 + i] = run;
    run += x[i];
  }
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

void launch_scan_u32_u64(const uint32_t* in, uint64_t* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  constexpr int TILE = kScanThreads * kScanIPT;
  const int64_t tiles = (n + TILE - 1) / TILE;
  DevBuf<uint64_t> status(size_t(tiles), s);
  DevBuf<uint32_t> ticket(1, s);
  CG_CUDA(cudaMemsetAsync(status.p, 0, size_t(tiles) * 8, s));
  CG_CUDA(cudaMemsetAsync(ticket.p, 0, 4, s));
  k_scan_u32_u64<<<unsigned(tiles), kScanThreads, 0, s>>>(in, out, n, status.p, ticket.p);
  CG_LAUNCH_CHECK();
}

}  // namespace cgk
