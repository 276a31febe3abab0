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
//   3. B' = the cells of B not in V; the merged table V u B' is a merge of
//      two sorted, disjoint tables: every row's new index = its old index +
//      the number of rows of the other table that are smaller (binary
//      search), then one scatter;
//   4. edges of the merged graph = old edges (remapped), new-old edges (from
//      the queries of B'), new-new edges (the batch's edges between cells of
//      B'), each found exactly once; a u64 radix sort makes them canonical.
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

__global__ void k_merge_scatter(const uint64_t* __restrict__ A, int64_t na,
                                const uint32_t* __restrict__ less, int W, uint64_t* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < na;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t p = i + less[i];
    for (int w = 0; w < W; ++w) out[p * W + w] = A[i * W + w];
  }
}

__global__ void k_edges_old(const uint32_t* __restrict__ e, int64_t m, const uint32_t* __restrict__ cv,
                            uint64_t* __restrict__ out) {
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < m;
       q += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t i = e[2 * q], j = e[2 * q + 1];
    out[q] = (uint64_t(i + cv[i]) << 32) | uint64_t(j + cv[j]);
  }
}

// new-old edges: count (out == nullptr) or write, appended at *ctr
__global__ void k_edges_newold(const int32_t* __restrict__ nbr, int ell, int64_t nb,
                               const uint32_t* __restrict__ map, const uint32_t* __restrict__ cbp,
                               const uint32_t* __restrict__ cv, uint64_t* __restrict__ out,
                               unsigned long long* __restrict__ ctr) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  const int64_t total = nb * ell;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t t0 = int64_t(blockIdx.x) * blockDim.x; t0 < total; t0 += stride) {
    const int64_t t = t0 + threadIdx.x;
    bool hit = false;
    uint64_t e = 0;
    if (t < total) {
      const int64_t j = t / ell;
      const int32_t v = nbr[t];
      const uint32_t mj = map[j];
      if (v >= 0 && mj != 0xffffffffu) {
        const uint64_t p = uint64_t(mj) + cbp[mj], q = uint64_t(uint32_t(v)) + cv[v];
        hit = true;
        e = p < q ? ((p << 32) | q) : ((q << 32) | p);
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
                  const int32_t* self_idx, const int32_t* nbr, int ell, uint64_t** cells_out,
                  int64_t* nc_out, uint64_t** edges_out, int64_t* m_out, cudaStream_t s) {
  const int W = (ell + 63) / 64;
  // B' = batch cells not in V
  DevBuf<uint32_t> pos(size_t(nb), s), map(size_t(nb), s);
  k_mark_new<<<gridn(nb), 256, 0, s>>>(self_idx, nb, pos.p);
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
  k_compact_new<<<gridn(nb), 256, 0, s>>>(cb_rows, self_idx, pos.p, nb, W, bp.p, map.p);
  CG_LAUNCH_CHECK();
  // merged table
  const int64_t nc = nv + n2;
  if (nc >= (int64_t(1) << 32)) throw CgError{CG_ETOOBIG, "merged table has >= 2^32 cells"};
  DevBuf<uint32_t> cvl(size_t(nv), s), cbl(std::max<size_t>(1, size_t(n2)), s);
  k_count_less<<<gridn(nv), 256, 0, s>>>(cv_rows, nv, bp.p, n2, W, cvl.p);
  CG_LAUNCH_CHECK();
  if (n2) {
    k_count_less<<<gridn(n2), 256, 0, s>>>(bp.p, n2, cv_rows, nv, W, cbl.p);
    CG_LAUNCH_CHECK();
  }
  uint64_t* cout = static_cast<uint64_t*>(dev_alloc(size_t(nc) * W * 8, s));
  k_merge_scatter<<<gridn(nv), 256, 0, s>>>(cv_rows, nv, cvl.p, W, cout);
  CG_LAUNCH_CHECK();
  if (n2) {
    k_merge_scatter<<<gridn(n2), 256, 0, s>>>(bp.p, n2, cbl.p, W, cout);
    CG_LAUNCH_CHECK();
  }
  // edges: count the new ones, then write old + new-old + new-new, sort
  DevBuf<unsigned long long> ctr(2, s);
  CG_CUDA(cudaMemsetAsync(ctr.p, 0, 2 * sizeof(unsigned long long), s));
  k_edges_newold<<<gridn(nb * ell), 256, 0, s>>>(nbr, ell, nb, map.p, cbl.p, cvl.p, nullptr, ctr.p);
  CG_LAUNCH_CHECK();
  if (mb) {
    k_edges_newnew<<<gridn(mb), 256, 0, s>>>(eb, mb, map.p, cbl.p, nullptr, ctr.p + 1);
    CG_LAUNCH_CHECK();
  }
  unsigned long long* hc = static_cast<unsigned long long*>(host_stage(2 * sizeof(unsigned long long)));
  CG_CUDA(cudaMemcpyAsync(hc, ctr.p, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaStreamSynchronize(s));
  const int64_t m = mv + int64_t(hc[0]) + int64_t(hc[1]);
  DevBuf<uint64_t> keys(std::max<size_t>(1, size_t(m)), s), alt(std::max<size_t>(1, size_t(m)), s);
  if (mv) {
    k_edges_old<<<gridn(mv), 256, 0, s>>>(ev, mv, cvl.p, keys.p);
    CG_LAUNCH_CHECK();
  }
  CG_CUDA(cudaMemsetAsync(ctr.p, 0, 2 * sizeof(unsigned long long), s));
  k_edges_newold<<<gridn(nb * ell), 256, 0, s>>>(nbr, ell, nb, map.p, cbl.p, cvl.p, keys.p + mv, ctr.p);
  CG_LAUNCH_CHECK();
  if (mb) {
    k_edges_newnew<<<gridn(mb), 256, 0, s>>>(eb, mb, map.p, cbl.p, keys.p + mv + hc[0], ctr.p + 1);
    CG_LAUNCH_CHECK();
  }
  uint64_t* so = keys.p;
  if (m > 1) radix_sort<uint64_t>(keys.p, alt.p, nullptr, nullptr, nullptr, false, m, 64, &so, nullptr, s, nullptr);
  uint64_t* eout = static_cast<uint64_t*>(dev_alloc(size_t(std::max<int64_t>(m, 1)) * 8, s));
  if (m) launch_rotate_edges(so, m, eout, s);
  *cells_out = cout;
  *nc_out = nc;
  *edges_out = eout;
  *m_out = m;
}

}  // namespace cgk
