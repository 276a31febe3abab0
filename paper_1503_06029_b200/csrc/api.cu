// api.cu -- the C ABI (include/cg.h): argument checks, allocation, and the
// host pipeline that runs the hot path on one stream:
//   a1 pack -> a2 sort -> a3 dedupe (read back n_c) -> a4 layers (read back
//   layer offsets) -> a5 prefix index -> a6 probes + a7 append (read back m)
//   -> a7 canonical edge sort.
// See DESIGN.md for the data layout and the paper passages of each step.
#include <cuda_runtime.h>

#include <chrono>
#include <climits>
#include <new>
#include <atomic>
#include <cstdio>
#include <cstdlib>

#include <nvtx3/nvToolsExt.h>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "kernels.cuh"

struct cg_index {
  cgk::DictView view;
  // owned device buffers
  uint64_t* keys = nullptr;
  uint32_t* idx = nullptr;
  uint32_t* layer_off = nullptr;
  uint32_t* T = nullptr;
  uint64_t* tbase = nullptr;
  uint8_t* tbits = nullptr;
  uint32_t* F = nullptr;
  int device = 0;
  bool global = false;     // CG_DICT_GLOBAL index: gview over keys/T/F
  cgk::GlobalDict gview{};
};

namespace cgk {

// ---------------------------------------------------------------- errors
static thread_local std::string g_last_error;
void set_last_error(const std::string& s) { g_last_error = s; }
static thread_local int64_t g_launches = 0;
static std::atomic<int64_t> g_launches_total{0};  // process lifetime, all threads
void note_launch() {
  ++g_launches;
  g_launches_total.fetch_add(1, std::memory_order_relaxed);
}

// ---------------------------------------------------------------- allocator
static void* (*g_alloc)(size_t, cg_stream_t, void*) = nullptr;
static void (*g_dealloc)(void*, cg_stream_t, void*) = nullptr;
static void* g_alloc_ctx = nullptr;
static std::once_flag g_pool_once;

static void init_pool() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~uint64_t(0);  // keep freed blocks cached in the pool
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

static thread_local double g_alloc_us = 0;
static thread_local int64_t g_nallocs = 0;
static void reset_counters() {
  g_launches = 0;
  g_alloc_us = 0;
  g_nallocs = 0;
}
static void store_counters(cg_stats* st) {
  if (!st) return;
  st->kernel_launches = g_launches;
  st->us_host_alloc = g_alloc_us;
  st->n_allocs = g_nallocs;
}

struct AllocTimer {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  size_t bytes = 0;
  ~AllocTimer() {
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    g_alloc_us += us;
    ++g_nallocs;
  }
};

void* dev_alloc(size_t bytes, cudaStream_t s) {
  AllocTimer at;
  at.bytes = bytes;
  void* p = nullptr;
  if (g_alloc) {
    p = g_alloc(bytes, reinterpret_cast<cg_stream_t>(s), g_alloc_ctx);
    if (!p) throw CgError{CG_ENOMEM, "allocator hook returned NULL for " + std::to_string(bytes) + " bytes"};
    return p;
  }
  std::call_once(g_pool_once, init_pool);
  cudaError_t e = cudaMallocAsync(&p, bytes, s);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw CgError{CG_ENOMEM, "cudaMallocAsync(" + std::to_string(bytes) + "): " + cudaGetErrorString(e)};
  }
  return p;
}

void dev_free(void* p, cudaStream_t s) {
  if (!p) return;
  if (g_dealloc) {
    g_dealloc(p, reinterpret_cast<cg_stream_t>(s), g_alloc_ctx);
    return;
  }
  cudaFreeAsync(p, s);
}

// ---------------------------------------------------------------- workspace arena
namespace {
struct Arena {
  char* base = nullptr;
  size_t cap = 0;
  size_t top = 0;          // bytes in use at the top of the stack
  size_t overflow = 0;     // live scratch bytes that did not fit (pool-allocated)
  size_t peak = 0;         // high-water of top + overflow in this build
  size_t want = 0;         // capacity to provide at the next build
  int depth = 0;           // nested WsScope count
  struct Blk { size_t off, size; bool freed; };
  std::vector<Blk> stack;
};
constexpr int kMaxDev = 16;
thread_local Arena g_arena[kMaxDev];

Arena& cur_arena() {
  int dev = 0;
  cudaGetDevice(&dev);
  return g_arena[(dev >= 0 && dev < kMaxDev) ? dev : 0];
}
}  // namespace

WsScope::WsScope() {
  Arena& a = cur_arena();
  if (a.depth++ > 0) return;
  if (a.want > a.cap) {
    if (a.base) {
      cudaDeviceSynchronize();
      if (g_dealloc) g_dealloc(a.base, nullptr, g_alloc_ctx);
      else cudaFree(a.base);
    }
    a.base = nullptr;
    a.cap = 0;
    void* p = nullptr;
    if (g_alloc) {
      p = g_alloc(a.want, nullptr, g_alloc_ctx);
    } else if (cudaMalloc(&p, a.want) != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
    }
    if (p) {
      a.base = static_cast<char*>(p);
      a.cap = a.want;
    }
  }
  a.top = 0;
  a.overflow = 0;
  a.peak = 0;
  a.stack.clear();
}

WsScope::~WsScope() {
  Arena& a = cur_arena();
  if (--a.depth > 0) return;
  if (a.peak > a.cap) a.want = a.peak + a.peak / 4;  // grow once, with headroom
  a.stack.clear();
  a.top = 0;
}

void* ws_alloc(size_t bytes, cudaStream_t s, bool* from_arena) {
  Arena& a = cur_arena();
  const size_t sz = (bytes + 255) & ~size_t(255);
  if (a.depth > 0 && a.base && a.top + sz <= a.cap) {
    void* p = a.base + a.top;
    a.stack.push_back({a.top, sz, false});
    a.top += sz;
    a.peak = std::max(a.peak, a.top + a.overflow);
    *from_arena = true;
    return p;
  }
  *from_arena = false;
  if (a.depth > 0) {
    a.overflow += sz;
    a.peak = std::max(a.peak, a.top + a.overflow);
  }
  return dev_alloc(sz, s);
}

void ws_free(void* p, cudaStream_t s, bool from_arena, size_t bytes) {
  Arena& a = cur_arena();
  if (!from_arena) {
    const size_t sz = (bytes + 255) & ~size_t(255);
    if (a.depth > 0) a.overflow -= std::min(a.overflow, sz);
    dev_free(p, s);
    return;
  }
  const size_t off = static_cast<size_t>(static_cast<char*>(p) - a.base);
  for (size_t i = a.stack.size(); i-- > 0;) {
    if (a.stack[i].off == off) {
      a.stack[i].freed = true;
      break;
    }
  }
  while (!a.stack.empty() && a.stack.back().freed) {
    a.top = a.stack.back().off;
    a.stack.pop_back();
  }
}

void* host_stage(size_t bytes) {
  static thread_local void* buf = nullptr;
  static thread_local size_t cap = 0;
  if (bytes > cap) {
    if (buf) cudaFreeHost(buf);
    buf = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(bytes, 1 << 16);
    CG_CUDA(cudaMallocHost(&buf, want));
    cap = want;
  }
  return buf;
}

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 148;
  }
  return cached[dev];
}

// ---------------------------------------------------------------- pinned host pool (cg_build_host)
static std::mutex g_host_mu;
static std::multimap<size_t, void*> g_host_free;
static std::map<void*, size_t> g_host_size;

static void* host_pool_alloc(size_t bytes) {
  bytes = std::max<size_t>(bytes, 64);
  std::lock_guard<std::mutex> lk(g_host_mu);
  auto it = g_host_free.lower_bound(bytes);
  if (it != g_host_free.end() && it->first <= 2 * bytes) {
    void* p = it->second;
    g_host_free.erase(it);
    return p;
  }
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    throw CgError{CG_ENOMEM, "cudaHostAlloc(" + std::to_string(bytes) + ") failed"};
  }
  g_host_size[p] = bytes;
  return p;
}

static void host_pool_free(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_host_mu);
  auto it = g_host_size.find(p);
  if (it == g_host_size.end()) return;
  g_host_free.emplace(it->second, p);
}

// ---------------------------------------------------------------- stage timer
// Stage boundaries: CUDA events on the build stream (only with stats) and
// NVTX ranges "cg:<stage>" (always; no-ops unless a profiler is attached),
// so nsys/ncu timelines show the stages of every build.
struct StageTimer {
  bool on = false;
  cudaStream_t s = nullptr;
  std::vector<cudaEvent_t> ev;
  int nmark = 0;
  bool open = false;
  static const char* name(int k) {
    static const char* const n[] = {"cg:pack", "cg:sort", "cg:dedupe", "cg:layers",
                                    "cg:dict", "cg:probe", "cg:edges"};
    return k >= 0 && k < 7 ? n[k] : "cg:stage";
  }
  void start(bool enable, cudaStream_t st) {
    on = enable;
    s = st;
    mark();
  }
  void mark() {
    if (open) nvtxRangePop();
    open = false;
    if (nmark < 7) {
      nvtxRangePushA(name(nmark));
      open = true;
    }
    ++nmark;
    if (!on) return;
    cudaEvent_t e;
    CG_CUDA(cudaEventCreate(&e));
    CG_CUDA(cudaEventRecord(e, s));
    ev.push_back(e);
  }
  // drop every mark (a failed sweep attempt is re-run from the pack)
  void restart() {
    if (open) nvtxRangePop();
    open = false;
    for (auto e : ev) cudaEventDestroy(e);
    ev.clear();
    nmark = 0;
    mark();
  }
  double us(int a, int b) const {
    if (!on || b >= int(ev.size())) return 0.0;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev[a], ev[b]);
    return double(ms) * 1e3;
  }
  ~StageTimer() {
    if (open) nvtxRangePop();
    for (auto e : ev) cudaEventDestroy(e);
  }
};

static int bits_for(uint32_t v) {
  int b = 0;
  while ((uint64_t(1) << b) <= v) ++b;
  return std::max(b, 1);
}

static void check_device_ptr(const void* p, const char* what) {
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw CgError{CG_EINVAL, std::string(what) + ": not a CUDA pointer"};
  }
  if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged)
    throw CgError{CG_EINVAL, std::string(what) + ": host pointer where a device pointer is required"};
}

static void check_arch() {
  int dev = 0, major = 0;
  CG_CUDA(cudaGetDevice(&dev));
  CG_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major != 10) throw CgError{CG_EARCH, "cg is built for sm_100a (B200); device major = " + std::to_string(major)};
}

// Maps the exception in flight to a status code and records its detail: no
// exception (CgError, std::bad_alloc, anything else) crosses the C ABI.
static int current_error() {
  try {
    throw;
  } catch (const CgError& e) {
    set_last_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return CG_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return CG_ECUDA;
  } catch (...) {
    set_last_error("unknown exception");
    return CG_ECUDA;
  }
}

// ---------------------------------------------------------------- the pipeline
struct Built {
  uint64_t* cells = nullptr;
  int64_t n_cells = 0;
  uint32_t* edges = nullptr;  // (i, j) u32 pairs
  int64_t n_edges = 0;
  cg_index* index = nullptr;
};

// Distributed role of a build: cells only (phase 1 and the chunk merges of
// the distributed build return the sorted unique rows, no probe).
struct Shard {
  bool cells_only = false;
  int pre_skip = 0;  // pre_off buckets are bits [pre_skip, pre_skip + pre_B) (a prefix chunk)
};

// a5 + a6 + a7 over one prefix-indexed dictionary: T and F over the rows
// keys[0..nrows) (the canonical table, or a rank's subsequence U of it with
// canonical indices idx), probes of the sources (all rows, or the rows
// src_pos[0..n_src)), and the canonical edge list placed from the probe's
// sorted tile blocks.  Stage marks 4 (layers: implicit), 5 (dict), 6
// (probe), 7 (edges).  T/F are handed to *T_out/*F_out when requested.
struct GlobalOut {
  uint64_t* edges = nullptr;  // u32 pairs, dev_alloc'd
  int64_t m = 0;
  uint64_t issued = 0;
  int reruns = 0;
  int64_t dict_bytes = 0;
  int b = 0, fextra = 0;
  uint32_t* T = nullptr;  // when keep_index
  uint32_t* F = nullptr;
};

// PreIndex: T/F already written by the sweep path's bucket pass for b = pre_b
// (b + 5-bit filter); used when the dictionary here has that shape.
struct PreIndex {
  DevBuf<uint32_t>* T = nullptr;
  DevBuf<uint32_t>* F = nullptr;
  int b = -1;
};

static void global_probe(const uint64_t* keys, int64_t nrows, const uint32_t* src_pos,
                         const uint32_t* idx, int64_t n_src, int W, int ell, const cg_opts& o,
                         bool keep_index, StageTimer& tm, GlobalOut* go,
                         const PreIndex& pre = PreIndex()) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(o.stream);
  const int64_t nc = nrows;
  {
    tm.mark();  // 4: layers (implicit in the global dictionary)
    // ---- a5 one prefix index + filter over the canonical table
    // defaults measured on C5 (tools/tune_probe.sh): 1-2 cells per bucket and
    // a b+5-bit filter (probe 4.51 ms vs 5.00 ms at 4-8 cells / b+7 bits)
    const int target_log2 = o.bucket_log2 >= 0 ? o.bucket_log2 : 0;
    int b = 0;
    while (b < 28 && (uint64_t(nc) >> (b + 1)) >= (uint64_t(1) << target_log2)) ++b;
    int fextra = o.filter_extra >= 0 ? o.filter_extra : 5;
    fextra = std::min(fextra, 32 - b);  // filter prefix <= 32 bits
    const Mem gix = keep_index ? Mem::Persist : Mem::Scratch;  // T/F outlive the build
    // CG_DICT_HASH (the ncu A/B of SURVEY 8.a5): open-addressed buckets
    // instead of T/F, load 1/2 (2 slots per cell)
    const bool hash = o.dict_kind == CG_DICT_HASH;
    int lb = 0;
    while (hash && (int64_t(1) << lb) * 2 < nc) ++lb;
    const bool fused = pre.T && pre.T->p && !hash && b == pre.b && fextra == 5;
    DevBuf<uint32_t> T(hash || fused ? 1 : (size_t(1) << b) + 1, s, gix);
    DevBuf<uint32_t> F(hash || fused ? 1 : std::max<size_t>(1, (size_t(1) << (b + fextra)) / 32), s, gix);
    uint32_t* Tp = fused ? pre.T->p : T.p;
    uint32_t* Fp = fused ? pre.F->p : F.p;
    DevBuf<uint64_t> Z(hash ? size_t(ell) : 1, s), slots(hash ? (size_t(4) << lb) : 1, s),
        hv(hash ? size_t(nc) : 1, s);
    int64_t dict_bytes = 0;
    if (hash) {
      build_hash_dict(keys, nc, W, ell, lb, Z.p, slots.p, hv.p, s);
      dict_bytes = int64_t(slots.n + hv.n + Z.n) * 8;
    } else if (fused) {  // written by the bucket pass (sweep path)
      dict_bytes = int64_t(pre.T->n) * 4 + int64_t(pre.F->n) * 4;
    } else {
      CG_CUDA(cudaMemsetAsync(F.p, 0, F.n * 4, s));
      dict_bytes = int64_t(T.n) * 4 + int64_t(F.n) * 4;
      build_global_index(keys, nc, W, b, fextra, T.p, F.p, s);
    }
    tm.mark();  // 5: dict
    GlobalDict g{keys, nullptr, Tp, Fp, b, fextra, W, ell, nc};
    g.src_pos = src_pos;
    g.idx = idx;
    if (hash) {
      g.Z = Z.p;
      g.slots = slots.p;
      g.hv = hv.p;
      g.lb = lb;
    }
    // ---- a6 + a7: probes write the canonical edge list directly
    const int64_t i_lo = 0, i_hi = n_src;
    const int64_t ntiles = std::max<int64_t>(probe_global_tiles(i_hi - i_lo), 1);
    DevBuf<uint32_t> tcnt(size_t(ntiles), s);  // hits per tile
    DevBuf<uint64_t> tpos(size_t(ntiles), s);  // block position in the scratch list (~0: overflow)
    DevBuf<uint32_t> ticket(2, s);
    DevBuf<unsigned long long> ctr(6, s);
    DevBuf<uint4> ovf(size_t(ntiles), s);
    // scratch capacity: 4 hits per cell covers planted sets (m/n_c = 0.5) and
    // arrangement samples (degree ~ 2d, m/n_c <= 3 in R^3) in one probe pass;
    // a larger m (P:106 allows n_c*ell/2) costs one re-run at the exact size
    // (+ the warps' first chunk reservations: at least one tile cap each)
    uint64_t cap = std::max<uint64_t>(4 * uint64_t(i_hi - i_lo), 1 << 16) +
                   uint64_t(num_sms()) * 64 * uint64_t(probe_global_tile_edge_cap());
    if (o.edge_cap > 0) cap = uint64_t(o.edge_cap);
    DevBuf<uint64_t> hits(cap, s);  // tile blocks of sorted (i << 32 | j)
    unsigned long long* hc = static_cast<unsigned long long*>(host_stage(4 * sizeof(unsigned long long)));
    int reruns = 0;
    uint64_t m = 0, issued = 0, novf = 0;
    // ctr: [0] scratch slots reserved (warps reserve chunks), [1] hits placed,
    // [2] issued probes; [3] spill count, [4..5] the spill run's (unused) pair
    while (true) {
      CG_CUDA(cudaMemsetAsync(ticket.p, 0, 8, s));
      CG_CUDA(cudaMemsetAsync(ctr.p, 0, 6 * sizeof(unsigned long long), s));
      launch_probe_global(g, o.lcp_prune, i_lo, i_hi, hits.p, cap, tcnt.p, tpos.p, ticket.p, ctr.p,
                          ctr.p + 2, ovf.p, ticket.p + 1, nullptr, 0, nullptr, s);
      CG_CUDA(cudaMemcpyAsync(hc, ctr.p, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
      CG_CUDA(cudaMemcpyAsync(hc + 3, ticket.p + 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
      CG_CUDA(cudaStreamSynchronize(s));
      const uint64_t reserved = hc[0];
      m = hc[1];
      issued = hc[2];
      novf = uint32_t(hc[3] & 0xffffffffu);
      if (reserved <= cap) break;  // every block landed inside the scratch list
      // re-run with room for m plus the chunk tails: a closed chunk wastes
      // less than one block (<= tile cap), an open one less than a chunk
      const uint64_t nw = uint64_t(num_sms()) * 64, ch = probe_global_scratch_chunk(),
                     bc = uint64_t(probe_global_tile_edge_cap());
      cap = m + (m / (ch - bc) + nw + 1) * bc + nw * ch;
      hits.alloc(cap, s);
      ++reruns;
    }
    tm.mark();  // 6: probe
    // ---- canonical placement of the tile blocks: 64-bit offsets = exclusive
    // scan of the tile counts (overflow tiles included; m may exceed 2^32,
    // P:106), then one copy
    DevBuf<uint64_t> toff(size_t(ntiles), s);
    launch_scan_u32_u64(tcnt.p, toff.p, ntiles, s);
    uint64_t mt = m;  // total including overflow tiles
    if (novf) {
      std::vector<uint4> hv(novf);
      CG_CUDA(cudaMemcpyAsync(hv.data(), ovf.p, novf * sizeof(uint4), cudaMemcpyDeviceToHost, s));
      CG_CUDA(cudaStreamSynchronize(s));
      for (const uint4& t : hv) mt += t.z;
    }
    uint64_t* eout = static_cast<uint64_t*>(dev_alloc(std::max<uint64_t>(mt, 1) * 8, s));
    launch_tile_copy(hits.p, toff.p, tpos.p, tcnt.p, ntiles, eout, s);
    if (novf) {
      // tiles whose hits overflowed a warp buffer (dense graphs): re-run all
      // of them at once in spill mode, sort the spilled hits (tiles cover
      // disjoint source ranges, so the sorted list is the tiles' lists in
      // tile order) and drop each tile's part at its canonical offset
      const uint64_t ms = mt - m;
      if (ms >= (uint64_t(1) << 32))
        throw CgError{CG_ETOOBIG, ">= 2^32 edges from dense overflow tiles"};
      hits.reset();
      DevBuf<uint8_t> sel(size_t(ntiles), s);
      DevBuf<uint32_t> scnt(size_t(ntiles), s);
      DevBuf<uint64_t> sstart(size_t(ntiles), s);
      CG_CUDA(cudaMemsetAsync(sel.p, 0, size_t(ntiles), s));
      CG_CUDA(cudaMemsetAsync(scnt.p, 0, size_t(ntiles) * 4, s));
      launch_spill_select(ovf.p, uint32_t(novf), sel.p, scnt.p, s);
      launch_scan_u32_u64(scnt.p, sstart.p, ntiles, s);
      DevBuf<uint64_t> sp1(ms, s), sp2(ms, s);
      CG_CUDA(cudaMemsetAsync(ticket.p, 0, 4, s));
      CG_CUDA(cudaMemsetAsync(ctr.p + 3, 0, 3 * sizeof(unsigned long long), s));
      launch_probe_global(g, o.lcp_prune, i_lo, i_hi, nullptr, 0, tcnt.p, tpos.p, ticket.p,
                          ctr.p + 4, ctr.p + 4, ovf.p, ticket.p + 1, sp1.p, ms, ctr.p + 3, s, sel.p);
      uint64_t* so = sp1.p;
      if (ms > 1) radix_sort<uint64_t>(sp1.p, sp2.p, nullptr, nullptr, nullptr, false, int64_t(ms), 64, &so, nullptr, s, nullptr);
      launch_spill_place(g, so, int64_t(ms), i_lo, toff.p, sstart.p, eout, s);
    }
    m = mt;
    tm.mark();  // 7: edges (placement of the already sorted tile blocks)
    go->edges = eout;
    go->m = int64_t(m);
    go->issued = issued;
    go->reruns = reruns + int(novf);
    go->dict_bytes = dict_bytes;
    go->b = b;
    go->fextra = fextra;
    if (keep_index) {
      go->T = fused ? pre.T->release() : T.release();
      go->F = fused ? pre.F->release() : F.release();
    }
  }
}

// the dictionaries over the whole canonical table (no popcount layers)
static bool flat_dict(int k) { return k == CG_DICT_GLOBAL || k == CG_DICT_HASH || k == CG_DICT_AUTO; }

// Runs a2..a7 given packed keys (u64[n][W], consumed as scratch).
static void build_from_keys(DevBuf<uint64_t>& keys, int64_t n, int ell, const cg_opts& o,
                            uint32_t* d_flags, StageTimer& tm, cg_stats* st, Built* out,
                            const Shard& sh = Shard(), const uint32_t* top_hist = nullptr,
                            const uint32_t* pre_off = nullptr, int pre_B = 0,
                            const uint32_t* tile_hist = nullptr, const SweepIn* sw = nullptr,
                            bool* sweep_failed = nullptr, int dup_hint = -1) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(o.stream);
  const int W = (ell + 63) / 64;
  SortStats sst;
  // ---- a2 sort (+ a3 dedupe fused into the MSD bucket pass)
  const bool msd = W <= 2 && o.sort_kind != 1;
  // on the MSD path the result stays in keys or alt, which becomes the
  // output cell table: both are persistent allocations there
  DevBuf<uint64_t> alt(size_t(n) * W, s, (msd && !keys.scratch) ? Mem::Persist : Mem::Scratch);
  DevBuf<uint64_t> cellbuf;  // the output cell table
  DevBuf<uint32_t> popc(size_t(n), s);
  DevBuf<uint16_t> lcp(size_t(n), s);
  const uint64_t* sorted = nullptr;
  DevBuf<uint32_t> order;  // W > 2: canonical order of the rows (gather + dedupe fused)
  bool no_dups = false;    // W > 2: the sort saw no two equal rows
  bool done = false;
  int64_t nc = -1;
  uint32_t in_err = 0;
  bool in_err_read = false;  // the input-error flag already came back with the sort's counts
  // mid-size inputs with heavy duplication (arrangement samples, P:108;
  // C3: 54x) overflow the MSD buckets after two radix passes and the bucket
  // pass (~0.3 ms at 2^20 rows): a 1024-row duplication sample sends them to
  // the hash dedupe directly.  (Not at >= 2^24 rows, where the sample's
  // read-back would cost every distinct-input build.)
  const bool dupy_msd = msd && !sw && !sh.cells_only && pre_off == nullptr && n >= (int64_t(1) << 18) &&
                        n < (int64_t(1) << 24) &&
                        (dup_hint >= 0 ? dup_hint : int(sample_duplicates(keys.p, n, W, s))) >= 8;
  // the sweep path's bucket pass can write the global dictionary's index
  // (T, F) of the table it produces: shaped for b from n (= nc without
  // duplicates, the case it is for; global_probe falls back to the index
  // pass when b(nc) differs)
  DevBuf<uint32_t> preT, preF;
  PreIndex pre;
  SweepIn swx = sw ? *sw : SweepIn{};
  if (sw && !sh.cells_only && (o.dict_kind == CG_DICT_GLOBAL || o.dict_kind == CG_DICT_AUTO) &&
      (o.filter_extra < 0 || o.filter_extra == 5) && o.bucket_log2 <= 0) {
    int bp = 0;
    while (bp < 28 && (uint64_t(n) >> (bp + 1)) >= 1) ++bp;
    if (bp - (8 + swx.B2) >= 0 && bp - (8 + swx.B2) <= 10) {  // <= 1024 entries per bucket
      const Mem gix = o.index_out ? Mem::Persist : Mem::Scratch;
      preT.alloc((size_t(1) << bp) + 1, s, gix);
      preF.alloc(size_t(1) << bp, s, gix);
      pre = PreIndex{&preT, &preF, bp};
      swx.T = preT.p;
      swx.F = preF.p;
      swx.b = bp;
    }
  }
  if (msd && !dupy_msd) {
    uint64_t* ko = nullptr;
    int64_t ncu = 0;
    const bool fused = !keys.scratch && !alt.scratch;
    done = (fused || sw) ? sort_unique_msd(keys.p, alt.p, n, W, &ko, &ncu, s, &sst, top_hist, pre_off,
                                           pre_B, tile_hist, d_flags, &in_err, sh.pre_skip,
                                           sw ? &swx : nullptr)
                         : sort_rows_msd(keys.p, alt.p, n, W, &ko, s, &sst, top_hist);
    if (sw && !done) {  // a region or bucket slot overflowed: the caller re-packs
      *sweep_failed = true;
      return;
    }
    sorted = ko;
    if (done && fused) {
      nc = ncu;
      in_err_read = true;
      if (ko == keys.p) cellbuf.adopt(keys.release(), size_t(n) * W, s);
      else cellbuf.adopt(alt.release(), size_t(n) * W, s);
    }
    if (!done && ko != keys.p) {  // partially sorted data belongs in keys
      std::swap(keys.p, alt.p);
      std::swap(keys.arena, alt.arena);
      std::swap(keys.scratch, alt.scratch);
    }
  }
  int64_t ns = n;  // rows the full sort below orders
  if (!done) {
    if (msd && n >= (int64_t(1) << 18)) {
      // a bucket overflowed: skewed data, typically few distinct cells and
      // heavy duplication -- drop the copies by hashing first, then
      // sort only the distinct rows
      ns = hash_unique_rows(keys.p, n, W, alt.p, s);
      std::swap(keys.p, alt.p);
      std::swap(keys.arena, alt.arena);
      std::swap(keys.scratch, alt.scratch);
    }
    if (W == 1) {
      uint64_t* ko = nullptr;
      radix_sort<uint64_t>(keys.p, alt.p, nullptr, nullptr, nullptr, false, ns, 64, &ko, nullptr,
                           s, &sst);
      sorted = ko;
    } else if (gather_dedupe_ok(W)) {
      order.alloc(size_t(ns), s);  // canonical order; the rows move once, in the dedupe
      const bool big = ns >= (int64_t(1) << 15);
      // heavy duplication (sampled: >= 8 of 1024 rows repeat; arrangement
      // signatures) goes straight to the hash dedupe below (one
      // sampling kernel + read-back, ~20 us; the prefix attempt it saves on
      // such data costs ~100 us)
      const bool dupy = big && sample_duplicates(keys.p, ns, W, s) >= 8;
      if (dupy || !sort_rows_multiword(keys.p, ns, W, nullptr, s, &sst, order.p, &no_dups, big ? 1 : 0)) {
        // runs of equal 32-bit prefixes too long for the run sort
        // (arrangement signatures, which come with heavy duplication):
        // drop the copies by hashing, then sort the distinct rows
        ns = hash_unique_rows(keys.p, ns, W, alt.p, s);
        std::swap(keys.p, alt.p);
        std::swap(keys.arena, alt.arena);
        std::swap(keys.scratch, alt.scratch);
        order.alloc(size_t(ns), s);
        sort_rows_multiword(keys.p, ns, W, nullptr, s, &sst, order.p, &no_dups, 0);
        no_dups = true;  // every row is distinct now
      }
    } else {
      sort_rows_multiword(keys.p, ns, W, alt.p, s, &sst);
      sorted = alt.p;
    }
  }
  tm.mark();  // 2: sort
  if (nc < 0) {
    // ---- a3 dedupe + compaction (separate pass: LSD / multi-word paths)
    cellbuf.alloc(size_t(ns) * W, s, Mem::Persist);
    // (the global dictionary needs neither popcounts nor lcp: the probe
    // derives lcp from the next row)
    const bool meta = sh.cells_only || !flat_dict(o.dict_kind);
    if (order.p && no_dups) {
      // every row is a cell (the sort compared all ties): one gather, a
      // thread per word; n_c = n
      launch_gather_rows(keys.p, order.p, ns, W, cellbuf.p, s);
      nc = ns;
      if (meta) launch_cell_meta(cellbuf.p, nc, W, popc.p, lcp.p, s);
    } else if (order.p)
      launch_gather_dedupe(keys.p, order.p, ns, W, cellbuf.p, meta ? popc.p : nullptr,
                           meta ? lcp.p : nullptr, d_flags + 1, s);
    else launch_dedupe(sorted, ns, W, cellbuf.p, popc.p, lcp.p, d_flags + 1, s);
  } else if (!sh.cells_only && !flat_dict(o.dict_kind)) {
    // cells came out of the fused MSD pass: per-cell popcount and LCP for the
    // layered dictionary (the global-dictionary probe derives lcp itself)
    launch_cell_meta(cellbuf.p, nc, W, popc.p, lcp.p, s);
  }
  if (!in_err_read) {
    uint32_t* hf = static_cast<uint32_t*>(host_stage(2 * sizeof(uint32_t)));
    CG_CUDA(cudaMemcpyAsync(hf, d_flags, 2 * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaStreamSynchronize(s));
    in_err = hf[0];
    if (nc < 0) nc = hf[1];
  }
  if (in_err) throw CgError{CG_EINPUT, "input byte not in {0,1} (or pad bit set in packed input)"};
  tm.mark();  // 3: dedupe
  keys.reset();
  alt.reset();
  if (sh.cells_only) {  // distributed phase 1: the sorted unique run
    uint64_t* cout = nullptr;
    if (nc * 2 < n) {
      cout = static_cast<uint64_t*>(dev_alloc(size_t(nc) * W * 8, s));
      CG_CUDA(cudaMemcpyAsync(cout, cellbuf.p, size_t(nc) * W * 8, cudaMemcpyDeviceToDevice, s));
    } else {
      cout = cellbuf.release();
    }
    CG_CUDA(cudaStreamSynchronize(s));
    out->cells = cout;
    out->n_cells = nc;
    if (st) {
      st->n_cells = nc;
      st->sort_passes = sst.passes;
    }
    return;
  }
  if (flat_dict(o.dict_kind)) {
    // CG_DICT_AUTO: the hash dictionary for long rows with heavy duplication
    // (arrangement signatures: huge prefix buckets, DESIGN section 6 A/B --
    // C2 probe 267 -> 168 us), the prefix index otherwise
    cg_opts od = o;
    if (od.dict_kind == CG_DICT_AUTO)
      od.dict_kind = (W > 2 && !o.index_out && nc * 4 <= n) ? CG_DICT_HASH : CG_DICT_GLOBAL;
    GlobalOut go;
    global_probe(cellbuf.p, nc, nullptr, nullptr, nc, W, ell, od, o.index_out != nullptr, tm, &go,
                 pre);
    const uint64_t m = uint64_t(go.m);
    uint64_t* eout = go.edges;
    const int b = go.b, fextra = go.fextra;
    if (o.index_out) {
      // the index owns its own copy of the table plus T and F
      cg_index* ixp = new cg_index();
      ixp->global = true;
      ixp->keys = static_cast<uint64_t*>(dev_alloc(size_t(nc) * W * 8, s));
      CG_CUDA(cudaMemcpyAsync(ixp->keys, cellbuf.p, size_t(nc) * W * 8, cudaMemcpyDeviceToDevice, s));
      ixp->T = go.T;
      ixp->F = go.F;
      cudaGetDevice(&ixp->device);
      ixp->gview = GlobalDict{ixp->keys, nullptr, ixp->T, ixp->F, b, fextra, W, ell, nc};
      out->index = ixp;
    }
    uint64_t* cout = nullptr;
    if (nc * 2 < n) {
      cout = static_cast<uint64_t*>(dev_alloc(size_t(nc) * W * 8, s));
      CG_CUDA(cudaMemcpyAsync(cout, cellbuf.p, size_t(nc) * W * 8, cudaMemcpyDeviceToDevice, s));
    } else {
      cout = cellbuf.release();
    }
    CG_CUDA(cudaStreamSynchronize(s));
    out->cells = cout;
    out->n_cells = nc;
    out->edges = reinterpret_cast<uint32_t*>(eout);
    out->n_edges = int64_t(m);
    if (st) {
      st->n_cells = nc;
      st->n_edges = int64_t(m);
      st->logical_probes = nc * int64_t(ell);
      st->issued_probes = int64_t(go.issued);
      st->sort_passes = sst.passes;
      st->probe_reruns = go.reruns;
      st->dict_bytes = go.dict_bytes;
      st->dict_cells = nc;
    }
    return;
  }
  // ---- a4 popcount layering: stable sort of (popc, canonical index)
  // buffers that become the cg_index (when requested) outlive the build
  const Mem ix = o.index_out ? Mem::Persist : Mem::Scratch;
  DevBuf<uint32_t> popc_alt(size_t(nc), s), lidx(size_t(nc), s, ix), lidx_alt(size_t(nc), s, ix);
  uint32_t* sp = nullptr;
  uint32_t* li = nullptr;
  radix_sort<uint32_t>(popc.p, popc_alt.p, nullptr, lidx.p, lidx_alt.p, true, nc,
                       bits_for(uint32_t(ell)), &sp, &li, s, nullptr);
  DevBuf<uint32_t> loff(size_t(ell) + 2, s, ix);
  launch_layer_offsets(sp, nc, ell, loff.p, s);
  uint32_t* hoff = static_cast<uint32_t*>(host_stage((ell + 2) * sizeof(uint32_t)));
  CG_CUDA(cudaMemcpyAsync(hoff, loff.p, (ell + 2) * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaStreamSynchronize(s));
  std::vector<uint32_t> h_off(hoff, hoff + ell + 2);
  DevBuf<uint64_t> lkeys(size_t(nc) * W, s, ix);
  launch_gather_rows(cellbuf.p, li, nc, W, lkeys.p, s);
  DevBuf<uint16_t> llcp(size_t(nc), s);
  launch_gather_u16(lcp.p, li, nc, llcp.p, s);
  tm.mark();  // 4: layers
  // ---- a5 dictionary: per-layer prefix index sizes
  const int target_log2 = o.bucket_log2 >= 0 ? o.bucket_log2 : 2;
  std::vector<uint8_t> h_bits(ell + 1);
  std::vector<uint64_t> h_base(2 * (ell + 1));  // [tbase | fbase]
  uint64_t tot = 0, ftot = 0;
  // filter resolution (tuning knob, ncu-driven): b_p + fextra prefix bits
  const int fextra = o.filter_extra >= 0 ? o.filter_extra : kFilterExtra;
  for (int p = 0; p <= ell; ++p) {
    const uint64_t sz = h_off[p + 1] - h_off[p];
    int b = 0;
    if (o.dict_kind == CG_DICT_SORTED)
      while (b < 28 && (sz >> (b + 1)) >= (uint64_t(1) << target_log2)) ++b;
    h_bits[p] = uint8_t(b);
    h_base[p] = tot;
    tot += (uint64_t(1) << b) + 1;
    h_base[ell + 1 + p] = ftot;
    ftot += std::max<uint64_t>(1, (uint64_t(1) << (b + fextra)) / 32);
  }
  DevBuf<uint8_t> tbits(size_t(ell) + 1, s, ix);
  DevBuf<uint64_t> tbase(2 * (size_t(ell) + 1), s, ix);
  DevBuf<uint32_t> T(size_t(tot), s, ix);
  DevBuf<uint32_t> F(size_t(ftot), s, ix);
  CG_CUDA(cudaMemcpyAsync(tbits.p, h_bits.data(), h_bits.size(), cudaMemcpyHostToDevice, s));
  CG_CUDA(cudaMemcpyAsync(tbase.p, h_base.data(), h_base.size() * 8, cudaMemcpyHostToDevice, s));
  CG_CUDA(cudaMemsetAsync(F.p, 0, F.n * sizeof(uint32_t), s));
  DictView dv{lkeys.p, li, loff.p, T.p, tbase.p, tbits.p, F.p, tbase.p + ell + 1, W, ell, nc, fextra};
  launch_build_prefix_index(dv, sp, T.p, F.p, s);
  tm.mark();  // 5: dict
  const int64_t j_lo = 0, j_hi = nc;
  // ---- a6 probes + a7 warp-aggregated append
  DevBuf<unsigned long long> ctr(2, s);
  uint64_t cap = std::max<uint64_t>(4 * uint64_t(j_hi - j_lo), 1 << 16);
  DevBuf<uint64_t> eb(cap, s);
  unsigned long long* hc = static_cast<unsigned long long*>(host_stage(2 * sizeof(unsigned long long)));
  int reruns = 0;
  uint64_t m = 0, issued = 0;
  while (true) {
    CG_CUDA(cudaMemsetAsync(ctr.p, 0, 2 * sizeof(unsigned long long), s));
    launch_probe(dv, llcp.p, sp, o.lcp_prune, j_lo, j_hi, eb.p, cap, ctr.p, ctr.p + 1, s);
    CG_CUDA(cudaMemcpyAsync(hc, ctr.p, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaStreamSynchronize(s));
    m = hc[0];
    issued = hc[1];
    if (m <= cap) break;
    cap = m;
    eb.alloc(cap, s);
    ++reruns;
  }
  tm.mark();  // 6: probe
  // ---- a7 canonical order: radix sort of (i << 32 | j)
  if (m >= (uint64_t(1) << 32))
    throw CgError{CG_ETOOBIG, "layered dictionary: >= 2^32 edges (use CG_DICT_GLOBAL)"};
  uint64_t* eout = static_cast<uint64_t*>(dev_alloc(std::max<uint64_t>(m, 1) * 8, s));
  {
    uint64_t* eo = eb.p;
    DevBuf<uint64_t> eb_alt(std::max<uint64_t>(m, 1), s);
    if (m > 1) radix_sort<uint64_t>(eb.p, eb_alt.p, nullptr, nullptr, nullptr, false, int64_t(m), 64, &eo, nullptr, s, nullptr);
    launch_rotate_edges(eo, int64_t(m), eout, s);
  }
  tm.mark();  // 7: edges
  // ---- outputs
  uint64_t* cout = nullptr;
  if (nc * 2 < n) {
    cout = static_cast<uint64_t*>(dev_alloc(size_t(nc) * W * 8, s));
    CG_CUDA(cudaMemcpyAsync(cout, cellbuf.p, size_t(nc) * W * 8, cudaMemcpyDeviceToDevice, s));
  } else {
    cout = cellbuf.release();
  }
  if (o.index_out) {
    cg_index* ix = new cg_index();
    ix->keys = lkeys.release();
    if (li == lidx.p) ix->idx = lidx.release();
    else ix->idx = lidx_alt.release();
    ix->layer_off = loff.release();
    ix->T = T.release();
    ix->tbase = tbase.release();
    ix->tbits = tbits.release();
    ix->F = F.release();
    cudaGetDevice(&ix->device);
    ix->view = DictView{ix->keys, ix->idx, ix->layer_off, ix->T, ix->tbase, ix->tbits,
                        ix->F, ix->tbase + ell + 1, W, ell, nc, fextra};
    out->index = ix;
  }
  CG_CUDA(cudaStreamSynchronize(s));
  out->cells = cout;
  out->n_cells = nc;
  out->edges = reinterpret_cast<uint32_t*>(eout);
  out->n_edges = int64_t(m);
  if (st) {
    st->n_cells = nc;
    st->n_edges = int64_t(m);
    st->logical_probes = nc * int64_t(ell);
    st->issued_probes = int64_t(issued);
    st->sort_passes = sst.passes;
    st->probe_reruns = reruns;
  }
}

// The sweep path: pack + first MSD partition into top-byte
// regions, then build_from_keys with the region sweep.  Mid-size inputs
// (< 2^24 rows) first sample their duplication on the input bytes (1024
// rows): heavy duplication (arrangement samples) skews the top bytes
// and is left to the exact path's hash dedupe (*dup_hint carries the
// sample there).  false = not taken, or a region/slot overflowed (the stage
// timer and flags are reset; the caller packs again on the exact path).
static bool try_sweep(const uint8_t* vecs, int64_t n, int ell, const cg_opts& o,
                      DevBuf<uint64_t>& keys, uint32_t* flags, StageTimer& tm, cg_stats* st,
                      Built* b, const Shard& sh, int* dup_hint) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(o.stream);
  const int W = (ell + 63) / 64;
  const int B2 = sweep_bits(n);
  if (o.sort_kind == 1 || o.sort_kind == 3 || W > 2 || B2 == 0 || !pack_sweep_ok(vecs, n, ell))
    return false;
  const uint32_t capr = pack_sweep_capr(n);
  if (o.sort_kind != 4 && n < (int64_t(1) << 24)) {
    // the sample also estimates the fullest top-byte region: skewed bits
    // (arrangement signatures) would overflow the regions and waste a pack
    double top = 0.0;
    *dup_hint = int(sample_duplicates_and_top(vecs, n, ell, s, &top));
    if (*dup_hint >= 8 || top * double(n) > 0.85 * double(capr)) return false;
  }
  bool failed = false;
  {
    DevBuf<uint64_t> regions(size_t(256) * capr * W + 2, s);  // (+16 B: bulk-copy tail)
    DevBuf<uint32_t> rc(257, s);  // region counts, overflow flag
    CG_CUDA(cudaMemsetAsync(rc.p + 256, 0, 4, s));
    launch_pack_sweep(vecs, n, ell, regions.p, capr, rc.p, flags, rc.p + 256, s);
    tm.mark();  // 1: pack
    SweepIn sw{regions.p, capr, rc.p, rc.p + 256};
    sw.B2 = B2;
    build_from_keys(keys, n, ell, o, flags, tm, st, b, sh, nullptr, nullptr, 8 + B2, nullptr, &sw,
                    &failed);
  }
  if (failed) {  // skewed top bytes: the exact path from a fresh pack
    tm.restart();
    CG_CUDA(cudaMemsetAsync(flags, 0, 4 * sizeof(uint32_t), s));
  }
  return !failed;
}

static void fill_stats(const StageTimer& tm, int64_t n, cg_stats* st) {
  if (!st) return;
  st->n_in = n;
  st->us_pack = tm.us(0, 1);
  st->us_sort = tm.us(1, 2);
  st->us_dedupe = tm.us(2, 3);
  st->us_layers = tm.us(3, 4);
  st->us_dict = tm.us(4, 5);
  st->us_probe = tm.us(5, 6);
  st->us_edges = tm.us(6, 7);
  st->us_total = tm.us(0, 7);
}

static int finish(int rc, const Built& b, cg_cells* cells, cg_edges* edges, const cg_opts& o,
                  int ell) {
  if (rc == CG_OK) {
    cells->words = b.cells;
    cells->n_cells = b.n_cells;
    cells->ell = ell;
    cells->words_per_cell = (ell + 63) / 64;
    edges->ij = b.edges;
    edges->n_edges = b.n_edges;
    if (o.index_out) *o.index_out = b.index;
  }
  return rc;
}

static void validate_opts(const cg_opts& o) {
  if (o.dict_kind == CG_DICT_HASH && o.index_out)
    throw CgError{CG_EINVAL, "CG_DICT_HASH keeps no cg_index (use CG_DICT_GLOBAL for cg_query)"};
  if (o.dict_kind != CG_DICT_SORTED && o.dict_kind != CG_DICT_BSEARCH &&
      o.dict_kind != CG_DICT_GLOBAL && o.dict_kind != CG_DICT_HASH && o.dict_kind != CG_DICT_AUTO)
    throw CgError{CG_ENOTIMPL, "dict_kind not implemented"};
  if (o.filter_extra < -1 || o.filter_extra > 8) throw CgError{CG_EINVAL, "filter_extra must be in [-1, 8]"};
  if (o.edge_cap < 0) throw CgError{CG_EINVAL, "edge_cap must be >= 0"};
  if (o.sort_kind < 0 || o.sort_kind > 4) throw CgError{CG_EINVAL, "sort_kind must be in [0, 4]"};
  if (o.reserved0 != 0) throw CgError{CG_EINVAL, "reserved0 must be 0"};
}

static int validate_common(int64_t n, int32_t ell, const void* p, cg_cells* cells, cg_edges* edges) {
  if (!cells || !edges) throw CgError{CG_EINVAL, "cells/edges out-pointers must not be NULL"};
  if (!p) throw CgError{CG_EINVAL, "input pointer is NULL"};
  if (n < 1) throw CgError{CG_EINVAL, "n must be >= 1"};
  if (ell < 1 || ell > CG_MAX_ELL) throw CgError{CG_EINVAL, "ell must be in [1, 4096]"};
  if (n > int64_t(0xffffffffll)) throw CgError{CG_ETOOBIG, "n must be < 2^32"};
  return CG_OK;
}

// f1 input: sampled points + half-space constraints (signatures on device)
struct PointsIn {
  const double* points = nullptr;
  int dim = 0;
  const double* planes = nullptr;
};

static int build_entry(const uint8_t* vecs, const uint64_t* words, int64_t n, int32_t ell,
                       const cg_opts* o_in, cg_cells* cells, cg_edges* edges,
                       const PointsIn* pin = nullptr) {
  if (cells) std::memset(cells, 0, sizeof(*cells));
  if (edges) std::memset(edges, 0, sizeof(*edges));
  cg_opts o;
  cg_opts_init(&o);
  if (o_in) o = *o_in;
  if (o.index_out) *o.index_out = nullptr;
  Built b;
  const auto h0 = std::chrono::steady_clock::now();
  double setup_us = 0;
  try {
    const void* in0 = vecs ? static_cast<const void*>(vecs)
                           : (words ? static_cast<const void*>(words)
                                    : static_cast<const void*>(pin ? pin->points : nullptr));
    validate_common(n, ell, in0, cells, edges);
    if (pin) {
      if (pin->dim < 1 || pin->dim > signatures_max_dim())
        throw CgError{CG_EINVAL, "dim must be in [1, 16]"};
      if (!pin->planes) throw CgError{CG_EINVAL, "planes is NULL"};
    }
    validate_opts(o);
    check_arch();
    check_device_ptr(in0, "input");
    if (pin) check_device_ptr(pin->planes, "planes");
    reset_counters();
    cudaStream_t s = reinterpret_cast<cudaStream_t>(o.stream);
    const int W = (ell + 63) / 64;
    WsScope ws;
    StageTimer tm;
    tm.start(o.stats != nullptr, s);  // 0
    setup_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count();
    if (vecs && o.sort_kind == 0 && small_build_ok(n, ell) && !o.index_out && o.edge_cap == 0 &&
        flat_dict(o.dict_kind)) {
      // small input: the whole path in one CTA, one host read-back (small.cu)
      uint64_t* cw = static_cast<uint64_t*>(dev_alloc(size_t(n) * W * 8, s));
      b.cells = cw;
      // m <= n_c * ell / 2: the buffer can never overflow
      const uint64_t ecap = std::max<uint64_t>(1, uint64_t(n) * uint64_t(ell) / 2);
      uint64_t* ew = static_cast<uint64_t*>(dev_alloc(ecap * 8, s));
      b.edges = reinterpret_cast<uint32_t*>(ew);
      DevBuf<int64_t> res(8, s);  // n_c, m, error (+ 4 phase clocks with SMALL_CLK)
      launch_small_build(vecs, n, ell, o.lcp_prune, cw, ew, res.p, s);
      tm.mark();  // the whole build is one kernel: reported as the pack stage
      int64_t* hr = static_cast<int64_t*>(host_stage(3 * sizeof(int64_t)));
      CG_CUDA(cudaMemcpyAsync(hr, res.p, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      CG_CUDA(cudaStreamSynchronize(s));
      if (hr[2]) throw CgError{CG_EINPUT, "input byte not in {0,1}"};
      b.n_cells = hr[0];
      b.n_edges = hr[1];
      for (int q = 0; q < 6; ++q) tm.mark();
      fill_stats(tm, n, o.stats);
      if (o.stats) {
        o.stats->n_cells = b.n_cells;
        o.stats->n_edges = b.n_edges;
        o.stats->logical_probes = b.n_cells * int64_t(ell);
        o.stats->dict_cells = b.n_cells;
      }
      store_counters(o.stats);
    } else {
    DevBuf<uint32_t> flags(4, s);
    CG_CUDA(cudaMemsetAsync(flags.p, 0, 4 * sizeof(uint32_t), s));
    // the MSD sort's top-digit histogram, counted by the pack kernel; on the
    // MSD path the key buffer becomes the output cell table (persistent)
    const bool msd = W <= 2 && o.sort_kind != 1;
    DevBuf<uint64_t> keys(size_t(n) * W, s, msd ? Mem::Persist : Mem::Scratch);
    const int B = msd_prefix_bits(n);
    // the sweep path (64/128-bit rows, 2^18 < n <= 2^26): the pack kernel
    // does the MSD sort's first partition, the second needs no look-back
    //
    int dup_hint = -1;
    const bool swept = vecs && msd && try_sweep(vecs, n, ell, o, keys, flags.p, tm, o.stats, &b,
                                                Shard(), &dup_hint);
    if (swept) {
      fill_stats(tm, n, o.stats);
      store_counters(o.stats);
    } else {
    const int dlo = (64 - B) / 8;
    DevBuf<uint32_t> top_hist(size_t(8 - dlo) * 256, s);
    // the pack kernel's per-tile counts of the first sort pass's digit (that
    // pass then needs no look-back)
    DevBuf<uint32_t> tile_hist(msd ? size_t((n + msd_tile_rows(W) - 1) / msd_tile_rows(W)) * 256 : 1, s);
    if (vecs) {
      if (msd) CG_CUDA(cudaMemsetAsync(top_hist.p, 0, top_hist.n * 4, s));
      launch_pack(vecs, n, ell, keys.p, flags.p, s, msd ? top_hist.p : nullptr, dlo,
                  msd ? tile_hist.p : nullptr, msd_tile_rows(W));
    } else if (pin) {
      if (msd) CG_CUDA(cudaMemsetAsync(top_hist.p, 0, top_hist.n * 4, s));
      launch_signatures(pin->points, n, pin->dim, pin->planes, ell, keys.p, flags.p, s,
                        msd ? top_hist.p : nullptr, dlo);
    } else {
      CG_CUDA(cudaMemcpyAsync(keys.p, words, size_t(n) * W * 8, cudaMemcpyDeviceToDevice, s));
      launch_check_pad(keys.p, n, ell, flags.p, s);
    }
    tm.mark();  // 1: pack
    build_from_keys(keys, n, ell, o, flags.p, tm, o.stats, &b, Shard(),
                    ((vecs || pin) && msd) ? top_hist.p : nullptr, nullptr, B,
                    (vecs && msd) ? tile_hist.p : nullptr, nullptr, nullptr, dup_hint);
    fill_stats(tm, n, o.stats);
    store_counters(o.stats);
    }
    }
  } catch (...) {
    const int rc_ = current_error();
    if (b.cells) dev_free(b.cells, nullptr);
    if (b.edges) dev_free(b.edges, nullptr);
    if (b.index) cg_index_free(b.index);
    if (cells) std::memset(cells, 0, sizeof(*cells));
    if (edges) std::memset(edges, 0, sizeof(*edges));
    return rc_;
  }
  if (o.stats) {
    o.stats->us_host_setup = setup_us;
    o.stats->us_host_total =
        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count();
  }
  return finish(CG_OK, b, cells, edges, o, ell);
}

}  // namespace cgk

using namespace cgk;

extern "C" {

void cg_opts_init(cg_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->dict_kind = CG_DICT_AUTO;
  o->lcp_prune = 1;
  o->bucket_log2 = -1;
  o->filter_extra = -1;
}

int cg_build(const uint8_t* vecs, int64_t n, int32_t ell, cg_cells* cells, cg_edges* edges) {
  return build_entry(vecs, nullptr, n, ell, nullptr, cells, edges);
}

int cg_build_ex(const uint8_t* vecs, int64_t n, int32_t ell, const cg_opts* o, cg_cells* cells,
                cg_edges* edges) {
  return build_entry(vecs, nullptr, n, ell, o, cells, edges);
}

int cg_build_packed_ex(const uint64_t* words, int64_t n, int32_t ell, const cg_opts* o,
                       cg_cells* cells, cg_edges* edges) {
  return build_entry(nullptr, words, n, ell, o, cells, edges);
}

int cg_build_points(const double* points, int64_t n, int32_t dim, const double* planes,
                    int32_t ell, const cg_opts* o, cg_cells* cells, cg_edges* edges) {
  PointsIn pin;
  pin.points = points;
  pin.dim = dim;
  pin.planes = planes;
  return build_entry(nullptr, nullptr, n, ell, o, cells, edges, &pin);
}

int cg_insert(const uint64_t* cells, int64_t n_cells, const uint32_t* edges, int64_t n_edges,
              int32_t ell, const uint8_t* vecs, int64_t n_new, const cg_opts* o_in,
              cg_cells* cells_out, cg_edges* edges_out) {
  if (cells_out) std::memset(cells_out, 0, sizeof(*cells_out));
  if (edges_out) std::memset(edges_out, 0, sizeof(*edges_out));
  cg_opts o;
  cg_opts_init(&o);
  if (o_in) o = *o_in;
  cg_cells bc;
  cg_edges be;
  std::memset(&bc, 0, sizeof(bc));
  std::memset(&be, 0, sizeof(be));
  uint64_t* cout = nullptr;
  uint64_t* eout = nullptr;
  try {
    if (!cells || !vecs || !cells_out || !edges_out || (n_edges > 0 && !edges))
      throw CgError{CG_EINVAL, "NULL argument"};
    if (n_cells < 1 || n_edges < 0 || n_new < 1) throw CgError{CG_EINVAL, "n_cells >= 1, n_new >= 1"};
    if (ell < 1 || ell > CG_MAX_ELL) throw CgError{CG_EINVAL, "ell must be in [1, 4096]"};
    // self lookups into the existing table are int32 (-1 = absent)
    if (n_cells > int64_t(INT32_MAX)) throw CgError{CG_ETOOBIG, "n_cells >= 2^31"};
    if (n_edges >= (int64_t(1) << 32)) throw CgError{CG_ETOOBIG, "n_edges >= 2^32"};
    check_arch();
    check_device_ptr(cells, "cells");
    if (n_edges > 0) check_device_ptr(edges, "edges");
    check_device_ptr(vecs, "vecs");
    // 1. the batch alone: sorted unique cells + its internal edges
    cg_opts ob;
    cg_opts_init(&ob);
    ob.stream = o.stream;
    const int rc = build_entry(vecs, nullptr, n_new, ell, &ob, &bc, &be);
    if (rc != CG_OK) throw CgError{rc, std::string("batch build: ") + cg_last_error()};
    cudaStream_t s = reinterpret_cast<cudaStream_t>(o.stream);
    const int W = (ell + 63) / 64;
    WsScope ws;
    // 2. an index over the existing table; self + flip lookups of the batch
    int b = 0;
    while (b < 28 && (uint64_t(n_cells) >> (b + 1)) >= 1) ++b;
    const int fextra = std::min(5, 32 - b);
    DevBuf<uint32_t> T((size_t(1) << b) + 1, s);
    DevBuf<uint32_t> F(std::max<size_t>(1, (size_t(1) << (b + fextra)) / 32), s);
    CG_CUDA(cudaMemsetAsync(F.p, 0, F.n * 4, s));
    build_global_index(cells, n_cells, W, b, fextra, T.p, F.p, s);
    GlobalDict g{cells, nullptr, T.p, F.p, b, fextra, W, ell, n_cells};
    // 3-4. merge the tables, remap + extend the edges
    int64_t nc = 0, m = 0;
    insert_merge(cells, n_cells, edges, n_edges, bc.words, bc.n_cells, be.ij, be.n_edges, g, ell,
                 &cout, &nc, &eout, &m, s);
    CG_CUDA(cudaStreamSynchronize(s));
    cells_out->words = cout;
    cells_out->n_cells = nc;
    cells_out->ell = ell;
    cells_out->words_per_cell = W;
    edges_out->ij = reinterpret_cast<uint32_t*>(eout);
    edges_out->n_edges = m;
    cout = eout = nullptr;
  } catch (...) {
    const int rc_ = current_error();
    if (cout) dev_free(cout, nullptr);
    if (eout) dev_free(eout, nullptr);
    if (cells_out) std::memset(cells_out, 0, sizeof(*cells_out));
    if (edges_out) std::memset(edges_out, 0, sizeof(*edges_out));
    cg_cells_free(&bc);
    cg_edges_free(&be);
    return rc_;
  }
  cg_cells_free(&bc);
  cg_edges_free(&be);
  return CG_OK;
}

int cg_allpairs(const uint64_t* cells, int64_t n_cells, int32_t ell, int32_t anchors,
                cg_edges* edges, int64_t* pairs_compared, cg_stream_t stream) {
  if (edges) std::memset(edges, 0, sizeof(*edges));
  uint64_t* eout = nullptr;
  try {
    if (!cells || !edges) throw CgError{CG_EINVAL, "NULL argument"};
    if (n_cells < 1) throw CgError{CG_EINVAL, "n_cells must be >= 1"};
    if (n_cells > int64_t(0xffffffffll)) throw CgError{CG_ETOOBIG, "n_cells >= 2^32"};
    if (ell < 1 || ell > CG_MAX_ELL) throw CgError{CG_EINVAL, "ell must be in [1, 4096]"};
    if (anchors < 0 || anchors > allpairs_max_anchors() || anchors > n_cells)
      throw CgError{CG_EINVAL, "anchors must be in [0, min(8, n_cells)]"};
    check_arch();
    check_device_ptr(cells, "cells");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int W = (ell + 63) / 64;
    WsScope ws;
    uint64_t cap = std::max<uint64_t>(uint64_t(n_cells) * 2, 1 << 16);
    DevBuf<uint64_t> hits(cap, s);
    uint64_t cmp = 0;
    uint64_t m = launch_allpairs(cells, n_cells, W, anchors, hits.p, cap, &cmp, s);
    if (m > cap) {
      cap = m;
      hits.alloc(cap, s);
      m = launch_allpairs(cells, n_cells, W, anchors, hits.p, cap, &cmp, s);
    }
    DevBuf<uint64_t> alt(std::max<uint64_t>(m, 1), s);
    uint64_t* so = hits.p;
    if (m > 1)
      radix_sort<uint64_t>(hits.p, alt.p, nullptr, nullptr, nullptr, false, int64_t(m), 64, &so,
                           nullptr, s, nullptr);
    eout = static_cast<uint64_t*>(dev_alloc(std::max<uint64_t>(m, 1) * 8, s));
    if (m) launch_rotate_edges(so, int64_t(m), eout, s);
    CG_CUDA(cudaStreamSynchronize(s));
    edges->ij = reinterpret_cast<uint32_t*>(eout);
    edges->n_edges = int64_t(m);
    if (pairs_compared) *pairs_compared = int64_t(cmp);
  } catch (...) {
    const int rc_ = current_error();
    if (eout) dev_free(eout, nullptr);
    if (edges) std::memset(edges, 0, sizeof(*edges));
    return rc_;
  }
  return CG_OK;
}

int cg_csr(const uint32_t* edges, int64_t n_edges, int64_t n_cells, uint64_t* row_ptr,
           uint32_t* col, cg_stream_t stream) {
  try {
    if (!row_ptr || (n_edges > 0 && (!edges || !col))) throw CgError{CG_EINVAL, "NULL argument"};
    if (n_cells < 1 || n_edges < 0) throw CgError{CG_EINVAL, "n_cells >= 1, n_edges >= 0"};
    if (n_cells > int64_t(0xffffffffll)) throw CgError{CG_ETOOBIG, "n_cells >= 2^32"};
    check_arch();
    if (n_edges > 0) {
      check_device_ptr(edges, "edges");
      check_device_ptr(col, "col");
    }
    check_device_ptr(row_ptr, "row_ptr");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    WsScope ws;
    build_csr(edges, n_edges, n_cells, row_ptr, col, s);
    CG_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    const int rc_ = current_error();
    return rc_;
  }
  return CG_OK;
}

int cg_bfs(const uint64_t* row_ptr, const uint32_t* col, int64_t n_cells, int64_t source,
           int32_t* dist, int32_t* parent, int32_t* eccentricity, cg_stream_t stream) {
  try {
    if (!row_ptr || !col || !dist) throw CgError{CG_EINVAL, "NULL argument"};
    if (n_cells < 1 || source < 0 || source >= n_cells)
      throw CgError{CG_EINVAL, "source must be in [0, n_cells)"};
    if (n_cells > int64_t(0xffffffffll)) throw CgError{CG_ETOOBIG, "n_cells >= 2^32"};
    check_arch();
    check_device_ptr(row_ptr, "row_ptr");
    check_device_ptr(dist, "dist");
    if (parent) check_device_ptr(parent, "parent");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    WsScope ws;
    const int ecc = bfs(row_ptr, col, n_cells, source, dist, parent, s);
    CG_CUDA(cudaStreamSynchronize(s));
    if (eccentricity) *eccentricity = ecc;
  } catch (...) {
    const int rc_ = current_error();
    return rc_;
  }
  return CG_OK;
}

int cg_signatures(const double* points, int64_t n, int32_t dim, const double* planes,
                  int32_t ell, uint64_t* words, cg_stream_t stream) {
  try {
    if (!points || !planes || !words) throw CgError{CG_EINVAL, "NULL argument"};
    if (n < 1) throw CgError{CG_EINVAL, "n must be >= 1"};
    if (ell < 1 || ell > CG_MAX_ELL) throw CgError{CG_EINVAL, "ell must be in [1, 4096]"};
    if (dim < 1 || dim > signatures_max_dim()) throw CgError{CG_EINVAL, "dim must be in [1, 16]"};
    check_arch();
    check_device_ptr(points, "points");
    check_device_ptr(planes, "planes");
    check_device_ptr(words, "words");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    WsScope ws;
    DevBuf<uint32_t> flag(1, s);
    CG_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(uint32_t), s));
    launch_signatures(points, n, dim, planes, ell, words, flag.p, s);
    uint32_t* h = static_cast<uint32_t*>(host_stage(sizeof(uint32_t)));
    CG_CUDA(cudaMemcpyAsync(h, flag.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaStreamSynchronize(s));
    if (h[0]) throw CgError{CG_EINPUT, "non-finite constraint value (NaN/inf in points or planes)"};
  } catch (...) {
    const int rc_ = current_error();
    return rc_;
  }
  return CG_OK;
}

int cg_build_host(const uint8_t* h_vecs, int64_t n, int32_t ell, const cg_opts* o_in,
                  uint64_t** h_cells, int64_t* n_cells, uint32_t** h_edges, int64_t* n_edges) {
  if (h_cells) *h_cells = nullptr;
  if (h_edges) *h_edges = nullptr;
  if (n_cells) *n_cells = 0;
  if (n_edges) *n_edges = 0;
  cg_opts o;
  cg_opts_init(&o);
  if (o_in) o = *o_in;
  if (o.index_out) *o.index_out = nullptr;
  uint64_t* hc = nullptr;
  uint32_t* he = nullptr;
  Built b;
  try {
    if (!h_vecs || !h_cells || !h_edges || !n_cells || !n_edges)
      throw CgError{CG_EINVAL, "NULL pointer argument"};
    cg_cells dummy_c;
    cg_edges dummy_e;
    validate_common(n, ell, h_vecs, &dummy_c, &dummy_e);
    check_arch();
    reset_counters();
    cudaStream_t s = reinterpret_cast<cudaStream_t>(o.stream);
    const int W = (ell + 63) / 64;
    WsScope ws;
    StageTimer tm;
    tm.start(o.stats != nullptr, s);
    DevBuf<uint32_t> flags(4, s);
    CG_CUDA(cudaMemsetAsync(flags.p, 0, 4 * sizeof(uint32_t), s));
    DevBuf<uint64_t> keys(size_t(n) * W, s,
                          (W <= 2 && o.sort_kind != 1) ? Mem::Persist : Mem::Scratch);
    // H2D in row chunks, each packed as soon as it lands (copy/compute overlap
    // through two staging buffers and a copy stream).
    const int64_t row_bytes = ell;
    const int64_t chunk_rows = std::max<int64_t>(1, (int64_t(64) << 20) / row_bytes);
    DevBuf<uint8_t> stage[2];
    const int64_t nchunk_rows = std::min<int64_t>(chunk_rows, n);
    stage[0].alloc(size_t(nchunk_rows * row_bytes), s);
    stage[1].alloc(size_t(nchunk_rows * row_bytes), s);
    // copy stream and events are released on every exit path
    struct CopyCtx {
      cudaStream_t cs = nullptr;
      cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_packed[2] = {nullptr, nullptr};
      ~CopyCtx() {
        if (cs) cudaStreamSynchronize(cs);
        for (int i = 0; i < 2; ++i) {
          if (ev_copied[i]) cudaEventDestroy(ev_copied[i]);
          if (ev_packed[i]) cudaEventDestroy(ev_packed[i]);
        }
        if (cs) cudaStreamDestroy(cs);
      }
    } cc;
    CG_CUDA(cudaStreamCreateWithFlags(&cc.cs, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CG_CUDA(cudaEventCreateWithFlags(&cc.ev_copied[i], cudaEventDisableTiming));
      CG_CUDA(cudaEventCreateWithFlags(&cc.ev_packed[i], cudaEventDisableTiming));
    }
    cudaStream_t cs = cc.cs;
    cudaEvent_t* ev_copied = cc.ev_copied;
    cudaEvent_t* ev_packed = cc.ev_packed;
    // the stage buffers were allocated on s: make the copy stream wait for that
    CG_CUDA(cudaEventRecord(ev_packed[0], s));
    CG_CUDA(cudaEventRecord(ev_packed[1], s));
    int64_t r0 = 0;
    int k = 0;
    while (r0 < n) {
      const int64_t r1 = std::min<int64_t>(n, r0 + chunk_rows);
      const int sb = k & 1;
      CG_CUDA(cudaStreamWaitEvent(cs, ev_packed[sb], 0));
      CG_CUDA(cudaMemcpyAsync(stage[sb].p, h_vecs + r0 * row_bytes, size_t((r1 - r0) * row_bytes),
                              cudaMemcpyHostToDevice, cs));
      CG_CUDA(cudaEventRecord(ev_copied[sb], cs));
      CG_CUDA(cudaStreamWaitEvent(s, ev_copied[sb], 0));
      launch_pack(stage[sb].p, r1 - r0, ell, keys.p + r0 * W, flags.p, s);
      CG_CUDA(cudaEventRecord(ev_packed[sb], s));
      r0 = r1;
      ++k;
    }
    CG_CUDA(cudaStreamSynchronize(s));
    stage[0].reset();
    stage[1].reset();
    tm.mark();  // 1: H2D + pack
    build_from_keys(keys, n, ell, o, flags.p, tm, o.stats, &b);
    fill_stats(tm, n, o.stats);
    store_counters(o.stats);
    const size_t cb = size_t(b.n_cells) * W * 8, ebytes = size_t(b.n_edges) * 8;
    hc = static_cast<uint64_t*>(host_pool_alloc(cb));
    he = static_cast<uint32_t*>(host_pool_alloc(ebytes));
    CG_CUDA(cudaMemcpyAsync(hc, b.cells, cb, cudaMemcpyDeviceToHost, s));
    if (ebytes) CG_CUDA(cudaMemcpyAsync(he, b.edges, ebytes, cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaStreamSynchronize(s));
    dev_free(b.cells, s);
    dev_free(b.edges, s);
    b.cells = nullptr;
    b.edges = nullptr;
    *h_cells = hc;
    *h_edges = he;
    *n_cells = b.n_cells;
    *n_edges = b.n_edges;
    if (o.index_out) *o.index_out = b.index;
    else if (b.index) cg_index_free(b.index);
    return CG_OK;
  } catch (...) {
    const int rc_ = current_error();
    if (b.cells) dev_free(b.cells, nullptr);
    if (b.edges) dev_free(b.edges, nullptr);
    if (b.index) cg_index_free(b.index);
    host_pool_free(hc);
    host_pool_free(he);
    return rc_;
  }
}

void cg_host_free(void* p) { host_pool_free(p); }

int cg_query(const cg_index* idx, const uint64_t* q, int64_t nq, int32_t* self_idx,
             int32_t* nbr_idx, cg_stream_t s) {
  try {
    if (!idx) throw CgError{CG_EINVAL, "NULL index"};
    if (nq < 0) throw CgError{CG_EINVAL, "nq < 0"};
    if (nq == 0) return CG_OK;
    if (!q || !self_idx || !nbr_idx) throw CgError{CG_EINVAL, "NULL query/output pointer"};
    const int64_t ncx = idx->global ? idx->gview.n_cells : idx->view.n_cells;
    if (ncx > int64_t(INT32_MAX)) throw CgError{CG_ETOOBIG, "index has >= 2^31 cells (int32 outputs)"};
    if (idx->global)
      launch_query_global(idx->gview, q, nq, self_idx, nbr_idx, reinterpret_cast<cudaStream_t>(s));
    else
      launch_query(idx->view, q, nq, self_idx, nbr_idx, reinterpret_cast<cudaStream_t>(s));
    return CG_OK;
  } catch (...) {
    const int rc_ = current_error();
    return rc_;
  }
}

int cg_index_info(const cg_index* idx, int64_t* n_cells, int32_t* ell) {
  if (!idx) return CG_EINVAL;
  if (n_cells) *n_cells = idx->global ? idx->gview.n_cells : idx->view.n_cells;
  if (ell) *ell = idx->global ? idx->gview.ell : idx->view.ell;
  return CG_OK;
}

int cg_set_allocator(void* (*alloc)(size_t, cg_stream_t, void*),
                     void (*dealloc)(void*, cg_stream_t, void*), void* ctx) {
  if ((alloc == nullptr) != (dealloc == nullptr)) return CG_EINVAL;
  g_alloc = alloc;
  g_dealloc = dealloc;
  g_alloc_ctx = alloc ? ctx : nullptr;
  return CG_OK;
}

void cg_cells_free(cg_cells* c) {
  if (!c) return;
  if (c->words) dev_free(c->words, nullptr);
  std::memset(c, 0, sizeof(*c));
}

void cg_edges_free(cg_edges* e) {
  if (!e) return;
  if (e->ij) dev_free(e->ij, nullptr);
  std::memset(e, 0, sizeof(*e));
}

void cg_index_free(cg_index* idx) {
  if (!idx) return;
  dev_free(idx->keys, nullptr);
  dev_free(idx->idx, nullptr);
  dev_free(idx->layer_off, nullptr);
  dev_free(idx->T, nullptr);
  dev_free(idx->tbase, nullptr);
  dev_free(idx->tbits, nullptr);
  dev_free(idx->F, nullptr);
  delete idx;
}

const char* cg_strerror(int code) {
  switch (code) {
    case CG_OK: return "ok";
    case CG_EINVAL: return "invalid argument";
    case CG_EINPUT: return "input byte not in {0,1} / pad bit set";
    case CG_ENOMEM: return "out of memory";
    case CG_ECUDA: return "CUDA error";
    case CG_ETOOBIG: return "too many vectors (n >= 2^32)";
    case CG_EARCH: return "unsupported GPU architecture (need sm_100)";
    case CG_ENOTIMPL: return "not implemented";
    default: return "unknown error";
  }
}

const char* cg_last_error(void) { return g_last_error.c_str(); }

int64_t cg_kernel_launches(void) { return g_launches_total.load(std::memory_order_relaxed); }

int cg_version(void) { return (0 << 16) | 1; }

int cg_dist_local(const uint8_t* vecs, int64_t n_local, int32_t ell, const cg_opts* o_in,
                  int32_t chunk_bits, cg_cells* run, int64_t* chunk_off) {
  if (run) std::memset(run, 0, sizeof(*run));
  cg_opts o;
  cg_opts_init(&o);
  if (o_in) o = *o_in;
  Built b;
  try {
    cg_edges dummy;
    validate_common(n_local, ell, vecs, run, &dummy);
    validate_opts(o);
    if (chunk_bits < 0 || chunk_bits > 8) throw CgError{CG_EINVAL, "chunk_bits must be in [0, 8]"};
    if (!chunk_off) throw CgError{CG_EINVAL, "chunk_off is NULL"};
    check_arch();
    check_device_ptr(vecs, "vecs");
    reset_counters();
    cudaStream_t s = reinterpret_cast<cudaStream_t>(o.stream);
    const int W = (ell + 63) / 64;
    WsScope ws;
    StageTimer tm;
    tm.start(o.stats != nullptr, s);
    DevBuf<uint32_t> flags(4, s);
    CG_CUDA(cudaMemsetAsync(flags.p, 0, 4 * sizeof(uint32_t), s));
    const bool msd = W <= 2 && o.sort_kind != 1;
    DevBuf<uint64_t> keys(size_t(n_local) * W, s, msd ? Mem::Persist : Mem::Scratch);
    const int B = msd_prefix_bits(n_local);
    const int dlo = (64 - B) / 8;
    DevBuf<uint32_t> top_hist(size_t(8 - dlo) * 256, s);
    DevBuf<uint32_t> tile_hist(msd ? size_t((n_local + msd_tile_rows(W) - 1) / msd_tile_rows(W)) * 256 : 1, s);
    Shard sh;
    sh.cells_only = true;
    int dup_hint = -1;
    if (!(msd && try_sweep(vecs, n_local, ell, o, keys, flags.p, tm, o.stats, &b, sh, &dup_hint))) {
      if (msd) CG_CUDA(cudaMemsetAsync(top_hist.p, 0, top_hist.n * 4, s));
      launch_pack(vecs, n_local, ell, keys.p, flags.p, s, msd ? top_hist.p : nullptr, dlo,
                  msd ? tile_hist.p : nullptr, msd_tile_rows(W));
      tm.mark();
      build_from_keys(keys, n_local, ell, o, flags.p, tm, o.stats, &b, sh,
                      msd ? top_hist.p : nullptr, nullptr, B, msd ? tile_hist.p : nullptr, nullptr,
                      nullptr, dup_hint);
    }
    // the run's split into 2^chunk_bits prefix chunks (the pipelined exchange)
    const int C = 1 << chunk_bits;
    if (chunk_bits == 0) {
      chunk_off[0] = 0;
      chunk_off[1] = b.n_cells;
    } else {
      DevBuf<uint32_t> off(size_t(C) + 1, s);
      launch_prefix_bounds(b.cells, b.n_cells, W, chunk_bits, off.p, s);
      uint32_t* h = static_cast<uint32_t*>(host_stage(size_t(C + 1) * 4));
      CG_CUDA(cudaMemcpyAsync(h, off.p, size_t(C + 1) * 4, cudaMemcpyDeviceToHost, s));
      CG_CUDA(cudaStreamSynchronize(s));
      for (int c = 0; c <= C; ++c) chunk_off[c] = h[c];
    }
    store_counters(o.stats);
  } catch (...) {
    const int rc_ = current_error();
    if (b.cells) dev_free(b.cells, nullptr);
    return rc_;
  }
  run->words = b.cells;
  run->n_cells = b.n_cells;
  run->ell = ell;
  run->words_per_cell = (ell + 63) / 64;
  return CG_OK;
}

int cg_dist_merge_chunk(const uint64_t* pieces, const int64_t* counts, int32_t G, int64_t stride,
                        int32_t ell, int32_t chunk_bits, const cg_opts* o_in, uint64_t* table,
                        int64_t table_cap, int64_t* n_table) {
  cg_opts o;
  cg_opts_init(&o);
  if (o_in) o = *o_in;
  o.index_out = nullptr;
  Built b;
  try {
    if (!counts || !table || !n_table) throw CgError{CG_EINVAL, "NULL argument"};
    if (G < 1 || stride < 0) throw CgError{CG_EINVAL, "bad G/stride"};
    if (ell < 1 || ell > CG_MAX_ELL) throw CgError{CG_EINVAL, "ell must be in [1, 4096]"};
    if (chunk_bits < 0 || chunk_bits > 8) throw CgError{CG_EINVAL, "chunk_bits must be in [0, 8]"};
    validate_opts(o);
    int64_t total = 0;
    for (int g = 0; g < G; ++g) {
      if (counts[g] < 0 || counts[g] > stride) throw CgError{CG_EINVAL, "counts[g] out of range"};
      total += counts[g];
    }
    if (*n_table < 0 || total + *n_table > table_cap)
      throw CgError{CG_EINVAL, "table capacity exceeded"};
    if (total + *n_table > int64_t(0xffffffffll)) throw CgError{CG_ETOOBIG, "too many rows"};
    if (total == 0) return CG_OK;
    if (!pieces) throw CgError{CG_EINVAL, "pieces is NULL"};
    check_arch();
    check_device_ptr(pieces, "pieces");
    check_device_ptr(table, "table");
    reset_counters();
    cudaStream_t s = reinterpret_cast<cudaStream_t>(o.stream);
    const int W = (ell + 63) / 64;
    WsScope ws;
    StageTimer tm;
    tm.start(false, s);
    uint64_t* dst = table + *n_table * W;
    int nonempty = 0, last = 0;
    for (int g = 0; g < G; ++g)
      if (counts[g]) ++nonempty, last = g;
    if (nonempty == 1) {  // one sorted unique piece: it is the merge
      CG_CUDA(cudaMemcpyAsync(dst, pieces + int64_t(last) * stride * W, size_t(total) * W * 8,
                              cudaMemcpyDeviceToDevice, s));
      CG_CUDA(cudaStreamSynchronize(s));
      *n_table += total;
      return CG_OK;
    }
    DevBuf<uint32_t> flags(4, s);
    CG_CUDA(cudaMemsetAsync(flags.p, 0, 4 * sizeof(uint32_t), s));
    // the pieces are sorted: on the MSD path they are gathered straight into
    // the chunk's prefix buckets (bits after the chunk's common top bits; no
    // radix pass) and the bucket pass sorts each bucket's segments and drops
    // cross-rank duplicates; otherwise concatenated and sorted in full
    const bool msd = W <= 2 && o.sort_kind != 1;
    DevBuf<uint64_t> keys(size_t(total) * W, s, msd ? Mem::Persist : Mem::Scratch);
    // bucket bits after the chunk's common top bits: ~1024 rows per bucket
    // (no radix pass here, so any B works)
    int B = 1;
    while (B < 24 - chunk_bits && total > (int64_t(1024) << B)) ++B;
    DevBuf<uint32_t> boff(msd ? (size_t(1) << B) + 1 : 1, s);
    if (msd) {
      gather_runs_by_prefix(pieces, counts, G, stride, W, B, chunk_bits, keys.p, boff.p, s);
    } else {
      int64_t at = 0;
      for (int g = 0; g < G; ++g) {
        if (counts[g])
          CG_CUDA(cudaMemcpyAsync(keys.p + at * W, pieces + int64_t(g) * stride * W,
                                  size_t(counts[g]) * W * 8, cudaMemcpyDeviceToDevice, s));
        at += counts[g];
      }
    }
    // MSD: the bucket pass writes the merged chunk straight into the table
    // (no 1 GB copy of a staged result per rank at C5)
    if (msd) {
      int64_t ncm = 0;
      if (merge_sorted_into(keys.p, boff.p, total, W, B, chunk_bits, dst, &ncm, s)) {
        *n_table += ncm;
        return CG_OK;
      }
    }
    Shard sh;
    sh.cells_only = true;
    sh.pre_skip = chunk_bits;
    build_from_keys(keys, total, ell, o, flags.p, tm, nullptr, &b, sh, nullptr,
                    msd ? boff.p : nullptr, B);
    CG_CUDA(cudaMemcpyAsync(dst, b.cells, size_t(b.n_cells) * W * 8, cudaMemcpyDeviceToDevice, s));
    CG_CUDA(cudaStreamSynchronize(s));
    dev_free(b.cells, s);
    b.cells = nullptr;
    *n_table += b.n_cells;
  } catch (...) {
    const int rc_ = current_error();
    if (b.cells) dev_free(b.cells, nullptr);
    return rc_;
  }
  return CG_OK;
}

int cg_dist_probe(const uint64_t* table, int64_t n_cells, int32_t ell, int32_t G, int32_t rank,
                  const cg_opts* o_in, cg_edges* local_edges) {
  if (local_edges) std::memset(local_edges, 0, sizeof(*local_edges));
  cg_opts o;
  cg_opts_init(&o);
  if (o_in) o = *o_in;
  o.index_out = nullptr;
  GlobalOut go;
  try {
    if (!table || !local_edges) throw CgError{CG_EINVAL, "NULL argument"};
    if (G < 1 || G > 64 || rank < 0 || rank >= G) throw CgError{CG_EINVAL, "bad G/rank (1 <= G <= 64)"};
    if (n_cells < 1) throw CgError{CG_EINVAL, "n_cells must be >= 1"};
    if (n_cells > int64_t(0xffffffffll)) throw CgError{CG_ETOOBIG, "n_cells >= 2^32"};
    if (ell < 1 || ell > CG_MAX_ELL) throw CgError{CG_EINVAL, "ell must be in [1, 4096]"};
    validate_opts(o);
    if (o.dict_kind != CG_DICT_GLOBAL && o.dict_kind != CG_DICT_AUTO)
      throw CgError{CG_ENOTIMPL, "cg_dist_probe uses CG_DICT_GLOBAL"};
    o.dict_kind = CG_DICT_GLOBAL;
    check_arch();
    check_device_ptr(table, "table");
    reset_counters();
    cudaStream_t s = reinterpret_cast<cudaStream_t>(o.stream);
    const int W = (ell + 63) / 64;
    WsScope ws;
    StageTimer tm;
    tm.start(o.stats != nullptr, s);  // 0
    int64_t n_src = n_cells, n_keep = n_cells;
    if (G == 1) {
      tm.mark();  // 1 (layer split: none)
      tm.mark();  // 2
      tm.mark();  // 3
      global_probe(table, n_cells, nullptr, nullptr, n_cells, W, ell, o, false, tm, &go);
    } else {
      // ---- the rank's share of the (popcount layer, canonical block) order,
      // cut at equal probe weight; blocks of 2^16 canonical cells
      const int blk_log2 = 16;
      const int64_t nblk = (n_cells + (int64_t(1) << blk_log2) - 1) >> blk_log2;
      const int64_t nflat = int64_t(ell + 1) * nblk;
      DevBuf<uint32_t> hist(size_t(nflat), s);
      layer_block_weights(table, n_cells, W, ell, o.lcp_prune, blk_log2, hist.p, s);
      const uint32_t* hh = static_cast<uint32_t*>(host_stage(size_t(nflat) * 4));
      CG_CUDA(cudaMemcpyAsync(const_cast<uint32_t*>(hh), hist.p, size_t(nflat) * 4,
                              cudaMemcpyDeviceToHost, s));
      CG_CUDA(cudaStreamSynchronize(s));
      tm.mark();  // 1: weights
      uint64_t wtot = 0;
      for (int64_t f = 0; f < nflat; ++f) wtot += hh[f];
      auto cut = [&](int r) -> int64_t {  // first flat position where the prefix reaches r/G
        if (r <= 0) return 0;
        if (r >= G) return nflat;
        const uint64_t target = (wtot * uint64_t(r)) / uint64_t(G);
        uint64_t acc = 0;
        for (int64_t f = 0; f < nflat; ++f) {
          if (acc >= target) return f;
          acc += hh[f];
        }
        return nflat;
      };
      const int64_t c_lo = cut(rank), c_hi = cut(rank + 1);
      int t_lo = 1, t_hi = 0;  // target layers: one above the source layers
      if (c_hi > c_lo) {
        t_lo = int(c_lo / nblk) + 1;
        t_hi = int((c_hi - 1) / nblk) + 1;
      }
      DevBuf<uint64_t> U(size_t(n_cells) * W, s);
      DevBuf<uint32_t> idx(size_t(n_cells), s), src_pos(size_t(n_cells), s);
      select_rows(table, n_cells, W, blk_log2, c_lo, c_hi, t_lo, t_hi, U.p, idx.p, src_pos.p,
                  &n_keep, &n_src, s);
      tm.mark();  // 2: the rank's subsequence
      tm.mark();  // 3
      if (n_src == 0) {
        tm.mark();
        tm.mark();
        tm.mark();
        tm.mark();
        go.edges = static_cast<uint64_t*>(dev_alloc(8, s));
      } else {
        global_probe(U.p, n_keep, src_pos.p, idx.p, n_src, W, ell, o, false, tm, &go);
      }
    }
    CG_CUDA(cudaStreamSynchronize(s));
    if (o.stats) {
      cg_stats* st = o.stats;
      st->n_in = n_cells;
      st->us_sort = tm.us(0, 1);    // probe weights per (layer, block)
      st->us_layers = tm.us(1, 2);  // the rank's dictionary subsequence
      st->us_dict = tm.us(4, 5);
      st->us_probe = tm.us(5, 6);
      st->us_edges = tm.us(6, 7);
      st->us_total = tm.us(0, 7);
      st->n_cells = n_cells;
      st->n_edges = go.m;
      st->logical_probes = n_src * int64_t(ell);
      st->issued_probes = int64_t(go.issued);
      st->probe_reruns = go.reruns;
      st->dict_bytes = go.dict_bytes;
      st->dict_cells = n_keep;
      store_counters(st);
    }
  } catch (...) {
    const int rc_ = current_error();
    if (go.edges) dev_free(go.edges, nullptr);
    return rc_;
  }
  local_edges->ij = reinterpret_cast<uint32_t*>(go.edges);
  local_edges->n_edges = go.m;
  return CG_OK;
}

int cg_dist_finalize(const uint32_t* gathered, const int64_t* counts, int32_t G, int64_t stride,
                     const cg_opts* o_in, cg_edges* edges) {
  if (edges) std::memset(edges, 0, sizeof(*edges));
  cg_opts o;
  cg_opts_init(&o);
  if (o_in) o = *o_in;
  uint64_t* eout = nullptr;
  int64_t m = 0;
  try {
    if (!gathered || !counts || !edges) throw CgError{CG_EINVAL, "NULL argument"};
    if (G < 1 || G > 64 || stride < 0) throw CgError{CG_EINVAL, "bad G/stride (1 <= G <= 64)"};
    for (int g = 0; g < G; ++g) {
      if (counts[g] < 0 || counts[g] > stride) throw CgError{CG_EINVAL, "counts[g] out of range"};
      m += counts[g];
    }
    check_arch();
    if (m > 0) check_device_ptr(gathered, "gathered");
    reset_counters();
    cudaStream_t s = reinterpret_cast<cudaStream_t>(o.stream);
    WsScope ws;
    // the ranks' lists are canonical and disjoint (each edge is emitted by
    // the rank owning its source cell): a G-way merge gives the canonical list
    eout = static_cast<uint64_t*>(dev_alloc(size_t(std::max<int64_t>(m, 1)) * 8, s));
    if (m > 0)
      merge_edge_lists(reinterpret_cast<const uint64_t*>(gathered), counts, G, stride, eout, s);
    CG_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    const int rc_ = current_error();
    if (eout) dev_free(eout, nullptr);
    return rc_;
  }
  edges->ij = reinterpret_cast<uint32_t*>(eout);
  edges->n_edges = m;
  return CG_OK;
}

}  // extern "C"
