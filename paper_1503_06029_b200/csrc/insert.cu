// insert.cu -- f2: incremental insertion of a new batch of samples.
//
// The sample generator "generates (and possibly accumulates)" points;
// this row extends an existing cell graph (table V, canonical edges E) by a
// new batch X' without rebuilding it:
//   1. the batch alone goes through the normal build -> sorted unique B and
//      its internal edges;
//   2. cg_query's kernel on an index over V gives, for every b in B, whether
//      b is already a cell of V and the indices in V of all its Hamming-1
//      neighbours (both flip directions);
//   3. B' = the cells of B not in V; the merged table V u B' is a merge of a
//      small and a large sorted, disjoint table: the small one's rows find
//      their positions by binary search in the large one; the large one is
//      streamed once, each 256-row tile counting the few small rows that
//      fall inside its key range;
//   4. edges of the merged graph = old edges (remapped through the index
//      map, still ascending), new-old edges (from the queries of B') and
//      new-new edges (the batch's edges between cells of B'), each found
//      exactly once; the new ones are sorted and merged into the old ones
//      the same way as the tables.
#include "kernels.cuh"

namespace cgk {
namespace {

__global__ void k_mark_new(const int32_t* __restrict__ self_idx, int64_t nb, uint32_t* __restrict__ flag) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < nb;
       j += int64_t(gridDim.x) * blockDim.x)
    flag[j] = self_idx[j] < 0 ? 1u : 0u;
}

// flag (0/1) and its exclusive scan -> compacted B' rows and map B -> B'
__global__ void k_compact_new(const uint64_t* __restrict__ cb, const int32_t* __restrict__ self_idx,
                              const uint32_t* __restrict__ pos, int64_t nb, int W,
                              uint64_t* __restrict__ bp, uint32_t* __restrict__ map) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < nb;
       j += int64_t(gridDim.x) * blockDim.x) {
    if (self_idx[j] < 0) {
      const uint32_t p = pos[j];
      for (int w = 0; w < W; ++w) bp[int64_t(p) * W + w] = cb[j * W + w];
      map[j] = p;
    } else {
      map[j] = 0xffffffffu;
    }
  }
}

// less[i] = number of rows of the sorted table B that are < row i of A
__global__ void k_count_less(const uint64_t* __restrict__ A, int64_t na,
                             const uint64_t* __restrict__ B, int64_t nb, int W,
                             uint32_t* __restrict__ less) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < na;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t* a = A + i * W;
    int64_t lo = 0, len = nb;
    while (len > 0) {
      const int64_t half = len >> 1;
      const uint64_t* b = B + (lo + half) * W;
      int c = 0;
      for (int w = 0; w < W && c == 0; ++w) c = b[w] < a[w] ? -1 : (b[w] > a[w] ? 1 : 0);
      if (c < 0) {
        lo += half + 1;
        len -= half + 1;
      } else {
        len = half;
      }
    }
    less[i] = uint32_t(lo);
  }
}

__global__ void k_count_less_u64(const uint64_t* __restrict__ A, int64_t na,
                                 const uint64_t* __restrict__ B, int64_t nb, uint32_t* __restrict__ less) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < na;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t a = A[i];
    int64_t lo = 0, len = nb;
    while (len > 0) {
      const int64_t half = len >> 1;
      if (B[lo + half] < a) {
        lo += half + 1;
        len -= half + 1;
      } else {
        len = half;
      }
    }
    less[i] = uint32_t(lo);
  }
}

// Large-table side of the merge without flags or per-row searches over L:
// with pos[j] = #(L rows < S_j) (ascending), L row i moves to
// i + c_i, c_i = #{j : pos[j] <= i}.  tilec[t] = c at the first row of the
// 256-row tile t (one binary search over pos per tile), so a row only
// counts the few pos values inside its tile's window.
constexpr int kMergeTile = 256;

// c_i = #{j : pos[j] <= i}: tilec gives the window [tilec[t], tilec[t+1]) of
// S rows that can fall inside tile t; the threads count within it
__device__ __forceinline__ int64_t merged_shift(int64_t i, const uint32_t* __restrict__ pos,
                                                uint32_t c0, uint32_t c1) {
  int64_t c = c0;
  if (c1 - c0 <= 16) {
    while (c < c1 && int64_t(pos[c]) <= i) ++c;
  } else {
    int64_t len = c1 - c0;
    while (len > 0) {
      const int64_t half = len >> 1;
      if (int64_t(pos[c + half]) <= i) {
        c += half + 1;
        len -= half + 1;
      } else {
        len = half;
      }
    }
  }
  return c;
}

__global__ void k_merge_large_rows(const uint64_t* __restrict__ L, int64_t nl,
                                   const uint32_t* __restrict__ pos, const uint32_t* __restrict__ tilec,
                                   int W, uint64_t* __restrict__ out, uint32_t* __restrict__ newidx) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nl;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i / kMergeTile;
    const int64_t p = i + merged_shift(i, pos, tilec[t], tilec[t + 1]);
    for (int w = 0; w < W; ++w) out[p * W + w] = L[i * W + w];
    if (newidx) newidx[i] = uint32_t(p);
  }
}

__global__ void k_merge_large_keys(const uint64_t* __restrict__ L, int64_t nl,
                                   const uint32_t* __restrict__ pos, const uint32_t* __restrict__ tilec,
                                   uint64_t* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nl;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i / kMergeTile;
    const uint64_t k = L[i];
    out[i + merged_shift(i, pos, tilec[t], tilec[t + 1])] = (k >> 32) | (k << 32);
  }
}

// small-table side: out[j + less[j]] = S_j
__global__ void k_merge_small_rows(const uint64_t* __restrict__ S, int64_t ns,
                                   const uint32_t* __restrict__ less, int W, bool rotate,
                                   uint64_t* __restrict__ out) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < ns;
       j += int64_t(gridDim.x) * blockDim.x) {
    const int64_t p = j + less[j];
    for (int w = 0; w < W; ++w) {
      const uint64_t k = S[j * W + w];
      out[p * W + w] = rotate ? ((k >> 32) | (k << 32)) : k;
    }
  }
}

// old edges (i, j) -> keys (newidx[i] << 32 | newidx[j]), still ascending
__global__ void k_edges_remap(const uint32_t* __restrict__ e, int64_t m,
                              const uint32_t* __restrict__ newidx, uint64_t* __restrict__ out) {
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < m;
       q += int64_t(gridDim.x) * blockDim.x)
    out[q] = (uint64_t(newidx[e[2 * q]]) << 32) | newidx[e[2 * q + 1]];
}

// index of row (q with bit (fw, bm) flipped; bm = 0: q itself) in the table
// of g, or -1: prefix filter, then a lower bound in the row's b-prefix bucket
__device__ __forceinline__ int64_t gd_lookup(const GlobalDict& g, const uint64_t* q, int fw,
                                             uint64_t bm) {
  const int W = g.W, b = g.b, fb = g.b + g.fextra;
  auto tw = [&](int w) -> uint64_t { return q[w] ^ (w == fw ? bm : 0ull); };
  const uint64_t t0 = tw(0);
  const uint64_t y = fb ? (t0 >> (64 - fb)) : 0ull;
  if (!((g.F[y >> 5] >> (y & 31)) & 1u)) return -1;
  const int64_t x = b ? int64_t(t0 >> (64 - b)) : 0;
  uint32_t lo = g.T[x];
  const uint32_t hi = g.T[x + 1];
  uint32_t len = hi - lo;
  while (len > 0) {
    const uint32_t half = len >> 1;
    const uint64_t* R = g.keys + int64_t(lo + half) * W;
    int c = 0;
    for (int w = 0; w < W && c == 0; ++w) {
      const uint64_t a = R[w], v = tw(w);
      c = a < v ? -1 : (a > v ? 1 : 0);
    }
    if (c < 0) {
      lo += half + 1;
      len -= half + 1;
    } else {
      len = half;
    }
  }
  if (lo >= hi) return -1;
  const uint64_t* R = g.keys + int64_t(lo) * W;
  for (int w = 0; w < W; ++w)
    if (R[w] != tw(w)) return -1;
  return int64_t(lo);
}

__global__ void k_self_lookup(GlobalDict g, const uint64_t* __restrict__ rows, int64_t n,
                              int32_t* __restrict__ self_idx) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
       j += int64_t(gridDim.x) * blockDim.x)
    self_idx[j] = int32_t(gd_lookup(g, rows + j * g.W, -1, 0ull));
}

// new-old edges: one warp per new cell B'_j (merged position j + cbl[j]),
// lanes over its ell single-bit flips looked up in the old table
__global__ void k_emit_newold(GlobalDict g, const uint64_t* __restrict__ bp, int64_t n2,
                              const uint32_t* __restrict__ cbl, const uint32_t* __restrict__ newidx,
                              uint64_t* __restrict__ out, uint64_t cap,
                              unsigned long long* __restrict__ ctr) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; j < n2; j += nw) {
    const uint64_t* q = bp + j * g.W;
    const uint64_t p = uint64_t(j) + cbl[j];
    for (int k0 = 0; k0 < g.ell; k0 += 32) {
      const int k = k0 + lane;
      int64_t v = -1;
      if (k < g.ell) v = gd_lookup(g, q, k >> 6, 1ull << (63 - (k & 63)));
      const bool hit = v >= 0;
      const uint32_t bal = __ballot_sync(kFull, hit);
      if (bal) {
        unsigned long long base = 0;
        if (lane == __ffs(bal) - 1) base = atomicAdd(ctr, (unsigned long long)__popc(bal));
        base = __shfl_sync(kFull, base, __ffs(bal) - 1);
        if (hit) {
          const uint64_t qq = newidx[v];
          const uint64_t pos = base + __popc(bal & lt);
          if (pos < cap) out[pos] = p < qq ? ((p << 32) | qq) : ((qq << 32) | p);
        }
      }
    }
  }
}

// tilec[t] = #{j : pos[j] <= kMergeTile * t} for t in [0, ntiles]; pos ascending
__global__ void k_tile_counts(const uint32_t* __restrict__ pos, int64_t ns, int64_t ntiles,
                              uint32_t* __restrict__ tilec) {
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t <= ntiles;
       t += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t key = uint64_t(t) * kMergeTile;
    int64_t lo = 0, len = ns;
    while (len > 0) {
      const int64_t half = len >> 1;
      if (uint64_t(pos[lo + half]) <= key) {
        lo += half + 1;
        len -= half + 1;
      } else {
        len = half;
      }
    }
    tilec[t] = uint32_t(lo);
  }
}

// new-new edges: the batch's edges whose two ends are both new cells
__global__ void k_edges_newnew(const uint32_t* __restrict__ eb, int64_t mb,
                               const uint32_t* __restrict__ map, const uint32_t* __restrict__ cbp,
                               uint64_t* __restrict__ out, unsigned long long* __restrict__ ctr) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t t0 = int64_t(blockIdx.x) * blockDim.x; t0 < mb; t0 += stride) {
    const int64_t t = t0 + threadIdx.x;
    bool hit = false;
    uint64_t e = 0;
    if (t < mb) {
      const uint32_t mu = map[eb[2 * t]], mv = map[eb[2 * t + 1]];
      if (mu != 0xffffffffu && mv != 0xffffffffu) {
        hit = true;
        e = ((uint64_t(mu) + cbp[mu]) << 32) | (uint64_t(mv) + cbp[mv]);
      }
    }
    const uint32_t bal = __ballot_sync(kFull, hit);
    if (bal) {
      unsigned long long base = 0;
      if (lane == __ffs(bal) - 1) base = atomicAdd(ctr, (unsigned long long)__popc(bal));
      base = __shfl_sync(kFull, base, __ffs(bal) - 1);
      if (hit && out) out[base + __popc(bal & lt)] = e;
    }
  }
}

int gridn(int64_t n) {
  return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 16)));
}

}  // namespace

void insert_merge(const uint64_t* cv_rows, int64_t nv, const uint32_t* ev, int64_t mv,
                  const uint64_t* cb_rows, int64_t nb, const uint32_t* eb, int64_t mb,
                  const GlobalDict& g, int ell, uint64_t** cells_out, int64_t* nc_out,
                  uint64_t** edges_out, int64_t* m_out, cudaStream_t s) {
  const int W = (ell + 63) / 64;
  // B' = batch cells not in V (self lookups into the old table)
  DevBuf<int32_t> self_idx(size_t(nb), s);
  k_self_lookup<<<gridn(nb), 256, 0, s>>>(g, cb_rows, nb, self_idx.p);
  CG_LAUNCH_CHECK();
  DevBuf<uint32_t> pos(size_t(nb), s), map(size_t(nb), s);
  k_mark_new<<<gridn(nb), 256, 0, s>>>(self_idx.p, nb, pos.p);
  CG_LAUNCH_CHECK();
  DevBuf<uint32_t> flag_last(1, s);
  CG_CUDA(cudaMemcpyAsync(flag_last.p, pos.p + nb - 1, 4, cudaMemcpyDeviceToDevice, s));
  launch_scan_u32(pos.p, nb, s);
  uint32_t* h = static_cast<uint32_t*>(host_stage(2 * sizeof(uint32_t)));
  CG_CUDA(cudaMemcpyAsync(h, pos.p + nb - 1, 4, cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaMemcpyAsync(h + 1, flag_last.p, 4, cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaStreamSynchronize(s));
  const int64_t n2 = int64_t(h[0]) + h[1];
  DevBuf<uint64_t> bp(std::max<size_t>(1, size_t(n2) * W), s);
  k_compact_new<<<gridn(nb), 256, 0, s>>>(cb_rows, self_idx.p, pos.p, nb, W, bp.p, map.p);
  CG_LAUNCH_CHECK();
  // merged table: B' (small) placed by binary search in V; V streamed once
  const int64_t nc = nv + n2;
  if (nc >= (int64_t(1) << 32)) throw CgError{CG_ETOOBIG, "merged table has >= 2^32 cells"};
  DevBuf<uint32_t> cbl(std::max<size_t>(1, size_t(n2)), s);
  if (n2) {
    k_count_less<<<gridn(n2), 256, 0, s>>>(bp.p, n2, cv_rows, nv, W, cbl.p);
    CG_LAUNCH_CHECK();
  }
  const int64_t vt = (nv + kMergeTile - 1) / kMergeTile;
  DevBuf<uint32_t> vtc(size_t(vt) + 1, s), newidx(size_t(nv), s);
  k_tile_counts<<<gridn(vt + 1), 256, 0, s>>>(cbl.p, n2, vt, vtc.p);
  CG_LAUNCH_CHECK();
  uint64_t* cout = static_cast<uint64_t*>(dev_alloc(size_t(nc) * W * 8, s));
  k_merge_large_rows<<<gridn(nv), 256, 0, s>>>(cv_rows, nv, cbl.p, vtc.p, W, cout, newidx.p);
  CG_LAUNCH_CHECK();
  if (n2) {
    k_merge_small_rows<<<gridn(n2), 256, 0, s>>>(bp.p, n2, cbl.p, W, false, cout);
    CG_LAUNCH_CHECK();
  }
  // new edges: new-old (flip lookups of the new cells, warp per cell) into a
  // buffer of 4 per new cell (rerun at the exact size if denser), then the
  // batch's new-new edges; sorted
  DevBuf<unsigned long long> ctr(2, s);
  unsigned long long* hc = static_cast<unsigned long long*>(host_stage(2 * sizeof(unsigned long long)));
  uint64_t cap = std::max<uint64_t>(uint64_t(4) * uint64_t(n2) + uint64_t(mb), 1024);
  DevBuf<uint64_t> nk(cap, s);
  for (int pass = 0; pass < 2; ++pass) {
    CG_CUDA(cudaMemsetAsync(ctr.p, 0, 2 * sizeof(unsigned long long), s));
    if (n2) {
      const int64_t blocks = std::min<int64_t>((n2 * 32 + 255) / 256, int64_t(num_sms()) * 16);
      k_emit_newold<<<unsigned(std::max<int64_t>(1, blocks)), 256, 0, s>>>(g, bp.p, n2, cbl.p,
                                                                         newidx.p, nk.p, cap, ctr.p);
      CG_LAUNCH_CHECK();
    }
    CG_CUDA(cudaMemcpyAsync(hc, ctr.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaStreamSynchronize(s));
    if (hc[0] + uint64_t(mb) <= cap) break;
    cap = hc[0] + uint64_t(mb);
    nk.alloc(cap, s);
  }
  if (mb) {
    k_edges_newnew<<<gridn(mb), 256, 0, s>>>(eb, mb, map.p, cbl.p, nk.p + hc[0], ctr.p + 1);
    CG_LAUNCH_CHECK();
  }
  CG_CUDA(cudaMemcpyAsync(hc + 1, ctr.p + 1, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaStreamSynchronize(s));
  const int64_t mn = int64_t(hc[0]) + int64_t(hc[1]);
  const int64_t m = mv + mn;
  // the merge ranks new edge keys among the old ones in 32 bits
  if (m >= (int64_t(1) << 32)) throw CgError{CG_ETOOBIG, "merged edge list has >= 2^32 edges"};
  DevBuf<uint64_t> nk_alt(std::max<size_t>(1, size_t(mn)), s);
  uint64_t* ns = nk.p;
  if (mn > 1) radix_sort<uint64_t>(nk.p, nk_alt.p, nullptr, nullptr, nullptr, false, mn, 64, &ns, nullptr, s, nullptr);
  // old edges remapped (order preserved: the index map is increasing)
  DevBuf<uint64_t> ok(std::max<size_t>(1, size_t(mv)), s);
  if (mv) {
    k_edges_remap<<<gridn(mv), 256, 0, s>>>(ev, mv, newidx.p, ok.p);
    CG_LAUNCH_CHECK();
  }
  // merge the new keys (small) into the old keys (large), rotate to pairs
  uint64_t* eout = static_cast<uint64_t*>(dev_alloc(size_t(std::max<int64_t>(m, 1)) * 8, s));
  DevBuf<uint32_t> el(std::max<size_t>(1, size_t(mn)), s);
  if (mn) {
    k_count_less_u64<<<gridn(mn), 256, 0, s>>>(ns, mn, ok.p, mv, el.p);
    CG_LAUNCH_CHECK();
  }
  if (mv) {
    const int64_t et = (mv + kMergeTile - 1) / kMergeTile;
    DevBuf<uint32_t> etc(size_t(et) + 1, s);
    k_tile_counts<<<gridn(et + 1), 256, 0, s>>>(el.p, mn, et, etc.p);
    CG_LAUNCH_CHECK();
    k_merge_large_keys<<<gridn(mv), 256, 0, s>>>(ok.p, mv, el.p, etc.p, eout);
    CG_LAUNCH_CHECK();
  }
  if (mn) {
    k_merge_small_rows<<<gridn(mn), 256, 0, s>>>(ns, mn, el.p, 1, true, eout);
    CG_LAUNCH_CHECK();
  }
  *cells_out = cout;
  *nc_out = nc;
  *edges_out = eout;
  *m_out = m;
}

}  // namespace cgk
