// common.cuh -- shared plumbing of the sm_100a cell-graph kernels (product path).
// Nothing here is shared with oracle/ (DESIGN "Oracle independence").
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "../../include/cg.h"

namespace cgk {

constexpr int kWarp = 32;
constexpr uint32_t kFull = 0xffffffffu;

// ---------------------------------------------------------------- errors
struct CgError {
  int code;
  std::string msg;
};
void set_last_error(const std::string& s);

#define CG_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      throw ::cgk::CgError{e_ == cudaErrorMemoryAllocation ? CG_ENOMEM : CG_ECUDA, \
                           std::string(#call) + ": " + cudaGetErrorString(e_)};    \
    }                                                                              \
  } while (0)

// every kernel launch is followed by CG_LAUNCH_CHECK(), which also counts it
// (cg_stats.kernel_launches: the bench's gpu_launches evidence)
void note_launch();
#define CG_LAUNCH_CHECK()          \
  do {                             \
    ::cgk::note_launch();          \
    CG_CUDA(cudaGetLastError());   \
  } while (0)

// ---------------------------------------------------------------- allocation
// Persistent allocations (outputs, index) go to the allocator hook / the
// device memory pool.  Workspace inside a build comes from a per-thread,
// per-device stack arena (one cudaMalloc, grown to the previous build's
// high-water mark), so a build makes no pool calls for its scratch buffers.
void* dev_alloc(size_t bytes, cudaStream_t s);  // throws CG_ENOMEM
void dev_free(void* p, cudaStream_t s);
void* ws_alloc(size_t bytes, cudaStream_t s, bool* from_arena);
void ws_free(void* p, cudaStream_t s, bool from_arena, size_t bytes);

// Marks one build: the arena is usable inside the scope; at the end it is
// sized for the next build.  All DevBufs of the build must die inside it.
struct WsScope {
  WsScope();
  ~WsScope();
};

enum class Mem { Scratch, Persist };

// RAII device buffer (scratch: arena stack; persist: pool), stream-ordered.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  bool arena = false;    // lives in the arena stack
  bool scratch = false;  // allocated as scratch (arena or overflow)
  DevBuf() = default;
  DevBuf(size_t count, cudaStream_t st, Mem m = Mem::Scratch) { alloc(count, st, m); }
  void alloc(size_t count, cudaStream_t st, Mem m = Mem::Scratch) {
    reset();
    s = st;
    n = count;
    const size_t bytes = count ? count * sizeof(T) : 16;
    if (m == Mem::Persist) {
      p = static_cast<T*>(dev_alloc(bytes, st));
      arena = scratch = false;
    } else {
      p = static_cast<T*>(ws_alloc(bytes, st, &arena));
      scratch = true;
    }
  }
  // take ownership of a persistent buffer released by another DevBuf
  void adopt(T* ptr, size_t count, cudaStream_t st) {
    reset();
    p = ptr;
    n = count;
    s = st;
    arena = scratch = false;
  }
  // hand a persistent buffer to the caller (never valid for scratch memory)
  T* release() {
    if (scratch) throw CgError{CG_ECUDA, "internal: release() of a scratch buffer"};
    T* r = p;
    p = nullptr;
    n = 0;
    return r;
  }
  void reset() {
    if (p) {
      if (scratch) ws_free(p, s, arena, n ? n * sizeof(T) : 16);
      else dev_free(p, s);
    }
    p = nullptr;
    n = 0;
    arena = scratch = false;
  }
  ~DevBuf() { reset(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// pinned host staging for small read-backs (per thread, grows)
void* host_stage(size_t bytes);

int num_sms();

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Decoupled look-back status word: [flag:2 | epoch:30 | value:32].
// flag 1 = tile aggregate only, 2 = inclusive prefix.  Epochs make a status
// buffer reusable across passes without clearing it (cleared once per sort).
__device__ __forceinline__ uint64_t lb_pack(uint32_t flag, uint32_t epoch, uint32_t value) {
  return (uint64_t(flag) << 62) | (uint64_t(epoch & 0x3fffffffu) << 32) | value;
}

// Publish `agg` for (tile, slot) and return the exclusive prefix over all
// earlier tiles of that slot.  Tiles are numbered in start order (atomic
// ticket), so every tile waited on has already published its aggregate.
__device__ __forceinline__ uint32_t lookback(uint64_t* status, int64_t tile, int nslots, int slot,
                                             uint32_t agg, uint32_t epoch) {
  uint64_t* me = status + tile * nslots + slot;
  if (tile == 0) {
    st_relaxed_u64(me, lb_pack(2, epoch, agg));
    return 0;
  }
  st_relaxed_u64(me, lb_pack(1, epoch, agg));
  uint32_t excl = 0;
  int64_t j = tile - 1;
  const uint32_t ep = epoch & 0x3fffffffu;
  // Walk back in windows of 8 predecessors whose statuses are loaded
  // independently (8 loads in flight), accumulating aggregates until an
  // inclusive prefix is found; an unpublished entry restarts the window there.
  constexpr int kWin = 8;
  while (true) {
    uint64_t s[kWin];
#pragma unroll
    for (int u = 0; u < kWin; ++u)
      s[u] = (j - u >= 0) ? ld_relaxed_u64(status + (j - u) * nslots + slot) : 0;
    bool done = false;
    int consumed = 0;
#pragma unroll
    for (int u = 0; u < kWin; ++u) {
      if (done || consumed < u) continue;  // stop at the first unusable entry
      const uint32_t flag = uint32_t(s[u] >> 62);
      const uint32_t sep = uint32_t(s[u] >> 32) & 0x3fffffffu;
      if (flag == 0 || sep != ep) continue;  // not yet published: reload from here
      excl += uint32_t(s[u]);
      consumed = u + 1;
      if (flag == 2) done = true;
    }
    if (done) break;
    j -= consumed;
  }
  st_relaxed_u64(me, lb_pack(2, epoch, excl + agg));
  return excl;
}

// Single-slot look-back run by ONE FULL WARP: each step loads the statuses of
// the 32 nearest unexamined predecessors at once (lane l -> tile j - l), so an
// inclusive prefix 32 tiles back costs one round trip instead of 32.
// Returns the exclusive prefix in every lane.
__device__ __forceinline__ uint32_t lookback_warp(uint64_t* status, int64_t tile, uint32_t agg,
                                                  uint32_t epoch) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_relaxed_u64(status, lb_pack(2, epoch, agg));
    return 0;
  }
  if (lane == 0) st_relaxed_u64(status + tile, lb_pack(1, epoch, agg));
  const uint32_t ep = epoch & 0x3fffffffu;
  uint32_t excl = 0;
  int64_t j = tile - 1;
  while (true) {
    const int64_t jj = j - lane;
    uint64_t s = jj >= 0 ? ld_relaxed_u64(status + jj) : lb_pack(2, epoch, 0);
    const uint32_t flag = uint32_t(s >> 62);
    const bool ready = flag != 0 && ((uint32_t(s >> 32) & 0x3fffffffu) == ep);
    const uint32_t notready = __ballot_sync(kFull, !ready);
    const uint32_t incl = __ballot_sync(kFull, ready && flag == 2);
    const int first_inc = incl ? __ffs(incl) - 1 : 32;
    const int first_nr = notready ? __ffs(notready) - 1 : 32;
    const int take = first_nr < first_inc ? first_nr : (first_inc < 32 ? first_inc + 1 : 32);
    uint32_t v = lane < take ? uint32_t(s) : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    excl += v;
    if (first_inc < 32 && first_inc < first_nr) break;
    j -= take;  // take == first_nr (spin there) or 32 (all aggregates)
  }
  if (lane == 0) st_relaxed_u64(status + tile, lb_pack(2, epoch, excl + agg));
  return excl;
}

// Single-slot look-back run by the WHOLE CTA (blockDim.x threads, a multiple
// of 32, <= 1024): each round loads the statuses of blockDim.x predecessors
// at once.  With short tiles the nearest inclusive prefix lies about as many
// tiles back as are in flight (hundreds); a warp needed one L2 round trip per
// 32 of them.  `tmp` needs 3 * 32 + 1 words of shared memory.  Every thread
// gets the exclusive prefix.
__device__ __forceinline__ uint32_t lookback_block(uint64_t* status, int64_t tile, uint32_t agg,
                                                   uint32_t epoch, uint32_t* tmp) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int nt = blockDim.x;
  if (tile == 0) {
    if (tid == 0) st_relaxed_u64(status, lb_pack(2, epoch, agg));
    return 0;
  }
  if (tid == 0) st_relaxed_u64(status + tile, lb_pack(1, epoch, agg));
  const uint32_t ep = epoch & 0x3fffffffu;
  uint32_t excl = 0;
  int64_t j = tile - 1;
  while (true) {
    const int64_t jj = j - tid;
    const uint64_t s = jj >= 0 ? ld_relaxed_u64(status + jj) : lb_pack(2, epoch, 0);
    const uint32_t flag = uint32_t(s >> 62);
    const bool ready = flag != 0 && ((uint32_t(s >> 32) & 0x3fffffffu) == ep);
    const uint32_t nr = __ballot_sync(kFull, !ready);
    const uint32_t inc = __ballot_sync(kFull, ready && flag == 2);
    if (lane == 0) {
      tmp[wid] = nr ? uint32_t(wid * 32 + __ffs(nr) - 1) : uint32_t(nt);
      tmp[32 + wid] = inc ? uint32_t(wid * 32 + __ffs(inc) - 1) : uint32_t(nt);
    }
    __syncthreads();
    int first_nr = nt, first_inc = nt;
    for (int w = 0; w < nw; ++w) {
      first_nr = min(first_nr, int(tmp[w]));
      first_inc = min(first_inc, int(tmp[32 + w]));
    }
    const int take = first_nr < first_inc ? first_nr : (first_inc < nt ? first_inc + 1 : nt);
    uint32_t v = tid < take ? uint32_t(s) : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    if (lane == 0) tmp[64 + wid] = v;
    __syncthreads();
    uint32_t sum = 0;
    for (int w = 0; w < nw; ++w) sum += tmp[64 + w];
    excl += sum;
    __syncthreads();  // tmp is rewritten by the next round
    if (first_inc < nt && first_inc < first_nr) break;
    j -= take;  // take == first_nr (spin there) or nt (all aggregates)
  }
  if (tid == 0) st_relaxed_u64(status + tile, lb_pack(2, epoch, excl + agg));
  return excl;
}

// Block-wide exclusive scan of one u32 per thread (blockDim.x multiple of 32,
// <= 1024).  `tmp` needs 33 words of shared memory.  Returns the total in *total.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* tmp, uint32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t t = lane < nw ? tmp[lane] : 0;
    uint32_t u = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(kFull, u, o);
      if (lane >= o) u += y;
    }
    if (lane < nw) tmp[lane] = u - t;
    if (lane == 31) tmp[32] = u;
  }
  __syncthreads();
  uint32_t r = tmp[wid] + x - v;
  *total = tmp[32];
  __syncthreads();
  return r;
}

}  // namespace cgk
