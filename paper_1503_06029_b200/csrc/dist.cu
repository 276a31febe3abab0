// dist.cu -- device steps of the multi-GPU build (row e):
// the popcount-layer query split, the rank's dictionary subsequence, and the
// merge of the ranks' edge lists.
//
// A 0->1 flip raises the popcount by exactly one (the two
// vectors differ in one bit), so the cells of popcount layer p have all their
// i < j neighbours in layer p+1.  Rank r probes the cells of a contiguous
// range of the (layer, canonical block) order, cut at equal probe weight, and
// its dictionary holds only the cells it probes plus the layers they can hit:
// about 1/G of the table plus one layer.
#include <vector>

#include "kernels.cuh"

namespace cgk {
namespace {

constexpr int kWeightStride = 8;  // cells sampled per weighted cell
#ifndef SEL_KB
#define SEL_KB 4  // rows in flight per lane (k_select_rows)
#endif
constexpr int kSelThreads = 256;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kSelPerWarp = 512;  // cells per warp and tile (16 rounds of 32)
constexpr int kSelTile = kSelWarps * kSelPerWarp;

__device__ __forceinline__ int row_popc(const uint64_t* r, int W) {
  int p = 0;
  for (int w = 0; w < W; ++w) p += __popcll(r[w]);
  return p;
}

// Probe weight of every kWeightStride-th cell (1 + candidate bits: zero bits k <= lcp with
// the next cell, as the probe issues them), summed per (popcount layer,
// block of 2^blk_log2 canonical cells): hist[p * nblk + blk].  One CTA per
// block; per-warp shared histograms (nh copies) keep atomics uncontended.
__global__ void __launch_bounds__(256)
    k_layer_weights(const uint64_t* __restrict__ cells, int64_t nc, int W, int ell, int lcp_prune,
                    int blk_log2, int64_t nblk, int nh, uint32_t* __restrict__ hist) {
  extern __shared__ uint32_t sh[];  // [nh][ell + 1]
  const int nb = ell + 1;
  for (int t = threadIdx.x; t < nh * nb; t += blockDim.x) sh[t] = 0;
  __syncthreads();
  uint32_t* my = sh + ((threadIdx.x >> 5) % nh) * nb;
  const int64_t blk = blockIdx.x;
  const int64_t i0 = blk << blk_log2;
  const int64_t i1 = min(nc, (blk + 1) << blk_log2);
  // a sample of every kWeightStride-th cell, weight scaled up: the cut only
  // balances work (the output does not depend on it), and the full pass cost
  // 0.46 ms of replicated work per rank at C5
  for (int64_t i = i0 + int64_t(threadIdx.x) * kWeightStride; i < i1;
       i += int64_t(blockDim.x) * kWeightStride) {
    const uint64_t* r = cells + i * W;
    int kmax = ell - 1;
    if (i + 1 >= nc) {
      kmax = -1;  // the last cell probes nothing
    } else if (lcp_prune) {
      const uint64_t* nx = r + W;
      int l = -1;
      for (int w = 0; w < W && l < 0; ++w) {
        const uint64_t x = __ldg(r + w) ^ __ldg(nx + w);
        if (x) l = 64 * w + __clzll(x);
      }
      if (l >= 0) kmax = min(kmax, l);
    }
    int cand = 0, p = 0;
    for (int w = 0; w < W; ++w) {
      const uint64_t x = __ldg(r + w);
      p += __popcll(x);
      if (64 * w <= kmax) {
        uint64_t z = ~x;
        const int hi = kmax - 64 * w;  // bits 0..hi of this word (MSB-first)
        if (hi < 63) z &= ~(~0ull >> (hi + 1));
        cand += __popcll(z);
      }
    }
    atomicAdd(&my[p], uint32_t(1 + cand) * uint32_t(kWeightStride));
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nb; t += blockDim.x) {
    uint32_t v = 0;
    for (int h = 0; h < nh; ++h) v += sh[h * nb + t];
    hist[int64_t(t) * nblk + blk] = v;
  }
}

// The rank's dictionary subsequence U (canonical order) and its sources S:
//   src(i)  = (popc_i * nblk + blk_i) in [c_lo, c_hi)   -- the rank's probes
//   keep(i) = src(i) or popc_i in [t_lo, t_hi]          -- plus their targets
// U[u] = cells[i], idx[u] = i for the kept cells; src_pos[s] = u for the
// sources.  Stable compaction: warp ballots + block scan + decoupled
// look-back (two counters); tiles of kSelTile cells by atomic ticket.
template <int WT>  // WT: words per row at compile time (1, 2), 0 = W
__global__ void __launch_bounds__(kSelThreads)
    k_select_rows(const uint64_t* __restrict__ cells, int64_t nc, int Wr, int blk_log2,
                  int64_t nblk, int64_t c_lo, int64_t c_hi, int t_lo, int t_hi,
                  uint64_t* __restrict__ U, uint32_t* __restrict__ idx,
                  uint32_t* __restrict__ src_pos, uint64_t* st_keep, uint64_t* st_src,
                  uint32_t* ticket, unsigned long long* totals) {
  __shared__ uint32_t s_bal[kSelWarps][kSelPerWarp / 32][2];
  __shared__ uint32_t s_wk[kSelWarps], s_ws[kSelWarps];
  __shared__ uint32_t s_tile;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int W = WT ? WT : Wr;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t w0 = tile * kSelTile + int64_t(wid) * kSelPerWarp;
  uint32_t ck = 0, cs = 0;
  constexpr int kB = SEL_KB;  // rows in flight per lane
  for (int it0 = 0; it0 < kSelPerWarp / 32; it0 += kB) {
    int pc[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int64_t i = w0 + (it0 + u) * 32 + lane;
      if (WT == 2) {
        const ulonglong2 r = i < nc ? reinterpret_cast<const ulonglong2*>(cells)[i] : ulonglong2{};
        pc[u] = i < nc ? __popcll(r.x) + __popcll(r.y) : -1;
      } else {
        pc[u] = i < nc ? row_popc(cells + i * W, W) : -1;
      }
    }
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int it = it0 + u;
      const int64_t i = w0 + it * 32 + lane;
      bool keep = false, src = false;
      if (pc[u] >= 0) {
        const int64_t flat = int64_t(pc[u]) * nblk + (i >> blk_log2);
        src = flat >= c_lo && flat < c_hi;
        keep = src || (pc[u] >= t_lo && pc[u] <= t_hi);
      }
      const uint32_t bk = __ballot_sync(kFull, keep), bs = __ballot_sync(kFull, src);
      if (lane == 0) {
        s_bal[wid][it][0] = bk;
        s_bal[wid][it][1] = bs;
      }
      ck += __popc(bk);
      cs += __popc(bs);
    }
  }
  if (lane == 0) {
    s_wk[wid] = ck;
    s_ws[wid] = cs;
  }
  __syncthreads();
  if (wid == 0) {
    uint32_t xk = lane < kSelWarps ? s_wk[lane] : 0u, xs = lane < kSelWarps ? s_ws[lane] : 0u;
    uint32_t ik = xk, is = xs;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t yk = __shfl_up_sync(kFull, ik, o), ys = __shfl_up_sync(kFull, is, o);
      if (lane >= o) {
        ik += yk;
        is += ys;
      }
    }
    const uint32_t tk = __shfl_sync(kFull, ik, kSelWarps - 1), ts = __shfl_sync(kFull, is, kSelWarps - 1);
    const uint32_t bk = lookback_warp(st_keep, tile, tk, 1);
    const uint32_t bs = lookback_warp(st_src, tile, ts, 1);
    if (lane < kSelWarps) {
      s_wk[lane] = bk + ik - xk;  // exclusive base of warp `lane`
      s_ws[lane] = bs + is - xs;
    }
    if (lane == 0) {
      if (tk) atomicAdd(totals, (unsigned long long)tk);
      if (ts) atomicAdd(totals + 1, (unsigned long long)ts);
    }
  }
  __syncthreads();
  uint32_t bk = s_wk[wid], bs = s_ws[wid];
  const uint32_t lt = lanemask_lt();
  for (int it = 0; it < kSelPerWarp / 32; ++it) {
    const int64_t i = w0 + it * 32 + lane;
    const uint32_t mk = s_bal[wid][it][0], ms = s_bal[wid][it][1];
    if ((mk >> lane) & 1u) {
      const uint32_t u = bk + __popc(mk & lt);
      if (WT == 2)
        reinterpret_cast<ulonglong2*>(U)[u] = reinterpret_cast<const ulonglong2*>(cells)[i];
      else
        for (int w = 0; w < W; ++w) U[int64_t(u) * W + w] = cells[i * W + w];
      idx[u] = uint32_t(i);
      if ((ms >> lane) & 1u) src_pos[bs + __popc(ms & lt)] = u;
    }
    bk += __popc(mk);
    bs += __popc(ms);
  }
}

__device__ __forceinline__ uint64_t edge_key(uint64_t pair) { return (pair << 32) | (pair >> 32); }

// ---- finalize: pairwise merge-path merges of the ranks' sorted lists (a
// tree of ceil(log2 G) levels, each one streaming pass over the edges)
constexpr int kMrgThreads = 256;
constexpr int kMrgPer = 8;                      // outputs per thread
constexpr int kMrgTile = kMrgThreads * kMrgPer;  // outputs per CTA

// split of output diagonal d between A and B: the number of A elements among
// the first d outputs (ties cannot occur: the lists are disjoint)
__device__ __forceinline__ int64_t diag_split(const uint64_t* A, int64_t na, const uint64_t* B,
                                              int64_t nb, int64_t d) {
  int64_t lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
  while (lo < hi) {
    const int64_t a = (lo + hi) >> 1;  // take a from A, d - a from B
    if (edge_key(__ldg(A + a)) < edge_key(__ldg(B + d - a - 1))) lo = a + 1;
    else hi = a;
  }
  return lo;
}

__global__ void k_merge_splits(const uint64_t* __restrict__ A, int64_t na,
                               const uint64_t* __restrict__ B, int64_t nb, int64_t ntiles,
                               int64_t* __restrict__ split) {
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t <= ntiles;
       t += int64_t(gridDim.x) * blockDim.x)
    split[t] = diag_split(A, na, B, nb, min(t * kMrgTile, na + nb));
}

__global__ void __launch_bounds__(kMrgThreads)
    k_merge_tiles(const uint64_t* __restrict__ A, int64_t na, const uint64_t* __restrict__ B,
                  int64_t nb, const int64_t* __restrict__ split, int64_t ntiles,
                  uint64_t* __restrict__ out) {
  __shared__ uint64_t sk[kMrgTile];  // the tile's A part then its B part, as keys
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t d0 = t * kMrgTile, d1 = min(d0 + kMrgTile, na + nb);
    const int64_t a0 = split[t], a1 = split[t + 1];
    const int la = int(a1 - a0), lb = int((d1 - d0) - la);
    const int64_t b0 = d0 - a0;
    __syncthreads();
    for (int q = threadIdx.x; q < la + lb; q += kMrgThreads)
      sk[q] = edge_key(q < la ? A[a0 + q] : B[b0 + (q - la)]);
    __syncthreads();
    // this thread's outputs: local diagonal [k0, k0 + kMrgPer)
    const int k0 = threadIdx.x * kMrgPer;
    if (k0 < la + lb) {
      int lo = k0 > lb ? k0 - lb : 0, hi = k0 < la ? k0 : la;
      while (lo < hi) {
        const int a = (lo + hi) >> 1;
        if (sk[a] < sk[la + k0 - a - 1]) lo = a + 1;
        else hi = a;
      }
      int ia = lo, ib = k0 - lo;
      const int kend = min(k0 + kMrgPer, la + lb);
      for (int k = k0; k < kend; ++k) {
        const bool takeA = ib >= lb || (ia < la && sk[ia] < sk[la + ib]);
        const uint64_t key = takeA ? sk[ia++] : sk[la + ib++];
        out[d0 + k] = edge_key(key);  // back to the (i, j) pair
      }
    }
  }
}

void merge_two(const uint64_t* A, int64_t na, const uint64_t* B, int64_t nb, uint64_t* out,
               cudaStream_t s) {
  const int64_t ntiles = (na + nb + kMrgTile - 1) / kMrgTile;
  if (ntiles == 0) return;
  DevBuf<int64_t> split(size_t(ntiles) + 1, s);
  k_merge_splits<<<unsigned((ntiles + 256) / 256), 256, 0, s>>>(A, na, B, nb, ntiles, split.p);
  CG_LAUNCH_CHECK();
  const int64_t grid = std::min<int64_t>(ntiles, int64_t(num_sms()) * 8);
  k_merge_tiles<<<unsigned(grid), kMrgThreads, 0, s>>>(A, na, B, nb, split.p, ntiles, out);
  CG_LAUNCH_CHECK();
}

}  // namespace

void layer_block_weights(const uint64_t* cells, int64_t nc, int W, int ell, int lcp_prune,
                         int blk_log2, uint32_t* hist, cudaStream_t s) {
  const int64_t nblk = (nc + (int64_t(1) << blk_log2) - 1) >> blk_log2;
  if (nblk <= 0) return;
  const int nh = (ell + 1) * 8 * 4 <= 48 * 1024 ? 8 : 1;  // per-warp copies when they fit
  k_layer_weights<<<unsigned(nblk), 256, size_t(nh) * (ell + 1) * 4, s>>>(
      cells, nc, W, ell, lcp_prune, blk_log2, nblk, nh, hist);
  CG_LAUNCH_CHECK();
}

void select_rows(const uint64_t* cells, int64_t nc, int W, int blk_log2, int64_t c_lo, int64_t c_hi,
                 int t_lo, int t_hi, uint64_t* U, uint32_t* idx, uint32_t* src_pos,
                 int64_t* n_keep, int64_t* n_src, cudaStream_t s) {
  const int64_t nblk = (nc + (int64_t(1) << blk_log2) - 1) >> blk_log2;
  const int64_t tiles = (nc + kSelTile - 1) / kSelTile;
  DevBuf<uint64_t> st(2 * size_t(tiles), s);
  DevBuf<uint32_t> ticket(1, s);
  DevBuf<unsigned long long> tot(2, s);
  CG_CUDA(cudaMemsetAsync(st.p, 0, st.n * 8, s));
  CG_CUDA(cudaMemsetAsync(ticket.p, 0, 4, s));
  CG_CUDA(cudaMemsetAsync(tot.p, 0, 16, s));
  auto sel = W == 2 ? k_select_rows<2> : (W == 1 ? k_select_rows<1> : k_select_rows<0>);
  sel<<<unsigned(tiles), kSelThreads, 0, s>>>(cells, nc, W, blk_log2, nblk, c_lo, c_hi,
                                                        t_lo, t_hi, U, idx, src_pos, st.p,
                                                        st.p + tiles, ticket.p, tot.p);
  CG_LAUNCH_CHECK();
  unsigned long long* h = static_cast<unsigned long long*>(host_stage(2 * sizeof(unsigned long long)));
  CG_CUDA(cudaMemcpyAsync(h, tot.p, 16, cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaStreamSynchronize(s));
  *n_keep = int64_t(h[0]);
  *n_src = int64_t(h[1]);
}

void merge_edge_lists(const uint64_t* lists, const int64_t* counts, int G, int64_t stride,
                      uint64_t* out, cudaStream_t s) {
  int64_t m = 0;
  for (int g = 0; g < G; ++g) m += counts[g];
  if (m == 0) return;
  // level 0: the gathered lists in place; each level merges neighbours into
  // a ping-pong buffer; the last level writes `out`
  struct L {
    const uint64_t* p;
    int64_t n;
  };
  std::vector<L> cur;
  for (int g = 0; g < G; ++g)
    if (counts[g]) cur.push_back({lists + int64_t(g) * stride, counts[g]});
  if (cur.size() == 1) {
    CG_CUDA(cudaMemcpyAsync(out, cur[0].p, size_t(m) * 8, cudaMemcpyDeviceToDevice, s));
    return;
  }
  DevBuf<uint64_t> buf[2];
  int pp = 0;
  while (cur.size() > 1) {
    const bool last = cur.size() <= 2;
    uint64_t* dst = out;
    if (!last) {
      if (!buf[pp].p) buf[pp].alloc(size_t(m), s);
      dst = buf[pp].p;
    }
    std::vector<L> nxt;
    int64_t at = 0;
    for (size_t k = 0; k < cur.size(); k += 2) {
      if (k + 1 < cur.size()) {
        merge_two(cur[k].p, cur[k].n, cur[k + 1].p, cur[k + 1].n, dst + at, s);
        nxt.push_back({dst + at, cur[k].n + cur[k + 1].n});
        at += cur[k].n + cur[k + 1].n;
      } else {  // odd one out: carried to the next level
        CG_CUDA(cudaMemcpyAsync(dst + at, cur[k].p, size_t(cur[k].n) * 8, cudaMemcpyDeviceToDevice, s));
        nxt.push_back({dst + at, cur[k].n});
        at += cur[k].n;
      }
    }
    cur.swap(nxt);
    pp ^= 1;
  }
}

}  // namespace cgk
