// probe.cu -- a6 single-bit-flip probes, a7 warp-aggregated edge append,
// and the cg_query kernel.
//
// a6 follows Alg. 4 (ParallelTreeBased): for every cell x and
// every bit k, x' = x with bit k negated is looked up in the dictionary, and
// (x, x') is output when found.  Differences from the paper's kernel
// (DESIGN "What differs"):
//   * only 0->1 flips are issued: x < x' iff x(k) = 0, so each edge is
//     emitted once, from its smaller endpoint (DESIGN G3), into layer p+1;
//   * exact LCP pruning: if x | e_k = V_j exists then V_i < V_{i+1} <= V_j and
//     all three share bits 0..k-1 (sorted prefix ranges are contiguous),
//     so only k <= lcp(V_i, V_{i+1}) can hit;
//   * x' is never materialised ("we do not have to keep the vector x'
//     explicitly"): word w of x' is x_w | (w == k/64 ? bit : 0);
//   * near / far split on the target layer's prefix width b:
//       near (k >= b): x' has x's b-bit prefix, so all near probes of a cell
//         fall in ONE prefix bucket of layer p+1; they are resolved by a
//         single merge walk over that bucket (x' ascends as k descends);
//       far (k < b): each x' has its own bucket; a 1-bit-per-(b+4)-bit-prefix
//         filter rejects most misses with one load before the bucket search;
//   * one thread per cell; the warp advances in lock-step rounds so each
//     round's hits are appended with ONE atomicAdd per warp (ballot + popc).
#include "kernels.cuh"

namespace cgk {
namespace {

// Lower-bound search of the implicit key t (word accessor tw) in layer q of
// the dictionary; returns the layer-major row or -1.  (cg_query path.)
template <class TW>
__device__ __forceinline__ int64_t dict_find(const DictView& d, int q, uint64_t t0, TW tw) {
  const uint32_t* Tq = d.T + d.tbase[q];
  const int b = d.tbits[q];
  const int64_t x = b ? int64_t(t0 >> (64 - b)) : 0;
  uint32_t lo = Tq[x], hi = Tq[x + 1];
  const int W = d.W;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    const uint64_t* r = d.keys + int64_t(mid) * W;
    bool less = false;
    const uint64_t a = r[0];
    if (a != t0) {
      less = a < t0;
    } else {
      for (int w = 1; w < W; ++w) {
        const uint64_t aw = r[w], bw = tw(w);
        if (aw != bw) {
          less = aw < bw;
          break;
        }
      }
    }
    if (less) lo = mid + 1;
    else hi = mid;
  }
  if (lo >= d.layer_off[q + 1]) return -1;
  const uint64_t* r = d.keys + int64_t(lo) * W;
  if (r[0] != t0) return -1;
  for (int w = 1; w < W; ++w)
    if (r[w] != tw(w)) return -1;
  return lo;
}

// Cell words: registers for W <= 2, global memory otherwise.
template <int WC>
struct CellWords {
  uint64_t r[WC > 0 ? WC : 1];
  const uint64_t* g;
  __device__ __forceinline__ void load(const uint64_t* p) {
    g = p;
    if (WC > 0) {
#pragma unroll
      for (int w = 0; w < (WC > 0 ? WC : 1); ++w) r[w] = p[w];
    }
  }
  __device__ __forceinline__ uint64_t operator()(int w) const {
    if (WC > 0) {
      uint64_t v = r[0];
#pragma unroll
      for (int u = 1; u < (WC > 0 ? WC : 1); ++u)
        if (u == w) v = r[u];
      return v;
    }
    return g[w];
  }
};

// row < t, where t = V with bit mask bm set in word fw (rows share nothing
// assumed); compares word 0 first (nearly always decisive).
template <int WC>
__device__ __forceinline__ int cmp_row(const uint64_t* row, const CellWords<WC>& V, int W, int fw,
                                       uint64_t bm, uint64_t t0) {
  const uint64_t a0 = row[0];
  if (a0 != t0) return a0 < t0 ? -1 : 1;
  const int n = WC > 0 ? WC : W;
  for (int w = 1; w < n; ++w) {
    const uint64_t a = row[w], b = V(w) | (w == fw ? bm : 0ull);
    if (a != b) return a < b ? -1 : 1;
  }
  return 0;
}

template <int WC>
__global__ void __launch_bounds__(256)
    k_probe(DictView d, const uint16_t* __restrict__ llcp, const uint32_t* __restrict__ sp,
            int lcp_prune, int64_t j_lo, int64_t j_hi, uint64_t* __restrict__ edges, uint64_t cap,
            unsigned long long* count, unsigned long long* issued) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  const int W = WC > 0 ? WC : d.W;
  const int ell = d.ell;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  unsigned long long my_issued = 0;

  // Per-warp staging buffer in shared memory: each round's hits are ranked
  // with a ballot and appended locally; when the buffer fills up (and at the
  // end) the warp reserves space with ONE atomicAdd and copies the staged
  // edges out coalesced.  (One global counter hit by every round made the
  // atomic's return latency the kernel's top stall.)
  constexpr int kStage = 256;
  __shared__ uint64_t stage[256 / 32][kStage];
  uint64_t* my_stage = stage[threadIdx.x >> 5];
  int fill = 0;  // warp-uniform
  auto flush = [&]() {
    if (fill == 0) return;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(count, (unsigned long long)fill);
    base = __shfl_sync(kFull, base, 0);
    __syncwarp();
    for (int i = lane; i < fill; i += 32)
      if (base + i < cap) edges[base + i] = my_stage[i];
    __syncwarp();
    fill = 0;
  };
  auto emit = [&](bool hit, uint64_t e) {
    const uint32_t hb = __ballot_sync(kFull, hit);
    if (hb) {
      if (hit) my_stage[fill + __popc(hb & lt)] = e;
      fill += __popc(hb);
      if (fill > kStage - 32) flush();
    }
  };

  for (int64_t jb = j_lo + int64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31); jb < j_hi;
       jb += stride) {
    const int64_t j = jb + lane;
    const bool valid = j < j_hi;
    CellWords<WC> V;
    V.load(d.keys + (valid ? j : 0) * W);
    int kmax = -1, q = 0;
    if (valid) {
      const int p = int(sp[j]);
      q = p + 1;
      if (p < ell && d.layer_off[q] != d.layer_off[q + 1]) {
        if (lcp_prune) {
          const int l = llcp[j];
          kmax = (l == 0xffff) ? -1 : min(l, ell - 1);
        } else {
          kmax = ell - 1;
        }
      }
    }
    const uint64_t ci = valid ? (uint64_t(d.idx[valid ? j : 0]) << 32) : 0;
    int b = 0;
    const uint32_t* Tq = d.T;
    const uint32_t* Fq = d.F;
    uint32_t qend = 0;
    if (kmax >= 0) {
      b = d.tbits[q];
      Tq = d.T + d.tbase[q];
      Fq = d.F + d.fbase[q];
      qend = d.layer_off[q + 1];
    }
    const uint64_t v0 = V(0);
    // ---------------- near candidates: zero bits k in [b, kmax], taken in
    // descending k (ascending target) against the one bucket of V's prefix
    int nw_hi = -1, nw = -1;  // current word and last word (descending)
    uint64_t nz = 0;          // remaining near candidate bits of word nw
    uint32_t r = 0, rhi = 0;  // merge cursor in the bucket
    if (kmax >= b) {
      const int64_t x = b ? int64_t(v0 >> (64 - b)) : 0;
      r = Tq[x];
      rhi = Tq[x + 1];
      if (r < rhi) {
        nw_hi = kmax >> 6;
        nw = nw_hi;
      }
    }
    const int nw_lo = b >> 6;  // b <= 28: always word 0
    auto near_mask = [&](int w) -> uint64_t {
      uint64_t m = ~V(w);
      if (w == nw_hi) m &= ~0ull << (63 - (kmax & 63));  // k <= kmax
      if (w == nw_lo && b > 0) m &= ~0ull >> b;          // k >= b (b < 64)
      return m;
    };
    if (nw >= 0) nz = near_mask(nw);
    auto near_next = [&]() -> bool {
      while (nz == 0 && nw > nw_lo) {
        --nw;
        nz = near_mask(nw);
      }
      return nz != 0;
    };
    // Small bucket (the common case): scan its rows instead of iterating the
    // candidates.  A row R of layer p+1 with V's b-bit prefix equals V | e_k
    // for some k >= b iff R contains every bit of V (popc(R) = popc(V) + 1),
    // and any such k is <= lcp (the LCP argument above), so the subset test
    // finds exactly the near edges.
    const bool scan = (nw >= 0) && (rhi - r <= 16);
    bool has = scan ? true : ((nw >= 0) && near_next());
    while (__any_sync(kFull, scan && r < rhi)) {
      // four rows per round, loaded independently (16-byte loads for W = 2)
      bool sub[4] = {false, false, false, false};
      if (scan && r < rhi) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t rr = r + u;
          if (rr < rhi) {
            const uint64_t* R = d.keys + int64_t(rr) * W;
            if (WC == 2) {
              const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(R);
              sub[u] = ((v0 & ~v.x) | (V(1) & ~v.y)) == 0;
            } else {
              bool sb = (v0 & ~R[0]) == 0;
              const int n = WC > 0 ? WC : W;
              for (int w = 1; w < n && sb; ++w) sb = (V(w) & ~R[w]) == 0;
              sub[u] = sb;
            }
            ++my_issued;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) emit(sub[u], sub[u] ? (ci | d.idx[r + u]) : 0ull);
      if (scan) r += 4;  // non-scan lanes keep their merge cursor
    }
    if (scan) has = false;
    while (__any_sync(kFull, has)) {
      bool hit = false;
      uint64_t e = 0;
      if (has) {
        const uint64_t bm = nz & (~nz + 1);  // lowest set bit = largest k
        nz ^= bm;
        const uint64_t t0 = v0 | (nw == 0 ? bm : 0ull);
        ++my_issued;
        if (rhi - r > 32) {
          // big bucket (skewed data): binary search instead of a long walk
          uint32_t lo = r, len = rhi - r;
          while (len > 0) {
            const uint32_t half = len >> 1;
            if (cmp_row<WC>(d.keys + int64_t(lo + half) * W, V, W, nw, bm, t0) < 0) {
              lo += half + 1;
              len -= half + 1;
            } else {
              len = half;
            }
          }
          r = lo;
        } else {
          while (r < rhi && cmp_row<WC>(d.keys + int64_t(r) * W, V, W, nw, bm, t0) < 0) ++r;
        }
        if (r < rhi && cmp_row<WC>(d.keys + int64_t(r) * W, V, W, nw, bm, t0) == 0) {
          hit = true;
          e = ci | d.idx[r];
          ++r;
        }
        if (r >= rhi) nz = 0, nw = nw_lo;  // bucket exhausted: no more near hits
        has = near_next();
      }
      emit(hit, e);
    }
    // ---------------- far candidates: zero bits k < min(b, kmax + 1), all in
    // word 0 (b <= 28); filter first, then search the surviving ones
    uint32_t surv = 0;  // bit k set = candidate k passed the filter
    const int kfar = min(b - 1, kmax);
    if (kfar >= 0) {
      const int fbits = b + d.fextra;
      const uint64_t y0 = v0 >> (64 - fbits);
      uint64_t z = ~v0 & (~0ull << (63 - kfar));  // zero bits with k <= kfar
      while (z) {
        // four independent filter loads in flight per thread
        int ks[4];
        uint32_t fw[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          ks[u] = -1;
          fw[u] = 0;
          if (z) {
            const int c = __clzll(z);  // k
            z &= ~(1ull << (63 - c));
            ks[u] = c;
            fw[u] = __ldg(Fq + ((y0 | (1ull << (fbits - 1 - c))) >> 5));
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (ks[u] >= 0) {
            const uint64_t y = y0 | (1ull << (fbits - 1 - ks[u]));
            ++my_issued;
            if ((fw[u] >> (y & 31)) & 1u) surv |= 1u << ks[u];
          }
        }
      }
    }
    // Flatten the warp's surviving far probes (a few per cell, unevenly
    // spread) so every lane works in every round: survivor g of the warp is
    // the m-th set bit of the mask of lane `owner`, whose cell data arrive by
    // shuffles.
    const uint32_t nsv = __popc(surv);
    uint32_t incl = nsv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t total_sv = __shfl_sync(kFull, incl, 31);
    const uint32_t tq_off = uint32_t(Tq - d.T);
    const uint64_t my_v1 = (WC == 2) ? V(1) : 0ull;
    for (uint32_t gb = 0; gb < total_sv; gb += 32) {
      const uint32_t g = gb + lane;
      int owner = 0;
#pragma unroll
      for (int s2 = 16; s2 >= 1; s2 >>= 1) {
        const uint32_t ic = __shfl_sync(kFull, incl, owner + s2 - 1);
        if (ic <= g) owner += s2;
      }
      owner = min(owner, 31);
      const uint32_t o_incl = __shfl_sync(kFull, incl, owner);
      const uint32_t o_cnt = __shfl_sync(kFull, nsv, owner);
      const uint32_t o_surv = __shfl_sync(kFull, surv, owner);
      const uint64_t o_v0 = __shfl_sync(kFull, v0, owner);
      const uint64_t o_v1 = __shfl_sync(kFull, my_v1, owner);
      const int o_b = __shfl_sync(kFull, b, owner);
      const uint32_t o_tq = __shfl_sync(kFull, tq_off, owner);
      const uint32_t o_qend = __shfl_sync(kFull, qend, owner);
      const uint64_t o_ci = __shfl_sync(kFull, ci, owner);
      const int64_t o_j = __shfl_sync(kFull, j, owner);
      bool hit = false;
      uint64_t e = 0;
      if (g < total_sv) {
        // m-th set bit (from the least significant end) of the owner's mask
        int m = int(g - (o_incl - o_cnt));
        int k = 0;
#pragma unroll
        for (int s2 = 16; s2 >= 1; s2 >>= 1) {
          const int c = __popc((o_surv >> k) & ((1u << s2) - 1u));
          if (m >= c) {
            m -= c;
            k += s2;
          }
        }
        CellWords<WC> OV;
        if (WC == 2) {
          OV.r[0] = o_v0;
          OV.r[WC > 1 ? 1 : 0] = o_v1;
        } else {
          OV.load(d.keys + o_j * W);
        }
        const uint64_t bm = 1ull << (63 - k);
        const uint64_t t0 = o_v0 | bm;
        const uint32_t* To = d.T + o_tq;
        const int64_t x = int64_t(t0 >> (64 - o_b));
        uint32_t lo = To[x];
        const uint32_t hi = To[x + 1];
        const uint32_t qend_ = o_qend;
        int64_t found = -1;
        auto V = OV;  // the owner's cell from here on
        const uint32_t qend = qend_;
        if (hi - lo <= 12) {
          // small bucket: compare up to four rows per step, loads independent
          for (uint32_t rr = lo; rr < hi && found < 0; rr += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const uint32_t ru = rr + u;
              if (ru < hi) {
                const uint64_t* R = d.keys + int64_t(ru) * W;
                bool eq;
                if (WC == 2) {
                  const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(R);
                  eq = v.x == t0 && v.y == V(1);
                } else {
                  eq = R[0] == t0;
                  const int n = WC > 0 ? WC : W;
                  for (int w = 1; w < n && eq; ++w) eq = R[w] == V(w);
                }
                if (eq) found = ru;
              }
            }
          }
        } else {
          uint32_t len = hi - lo;
          while (len > 0) {
            const uint32_t half = len >> 1;
            if (cmp_row<WC>(d.keys + int64_t(lo + half) * W, V, W, 0, bm, t0) < 0) {
              lo += half + 1;
              len -= half + 1;
            } else {
              len = half;
            }
          }
          if (lo < qend && cmp_row<WC>(d.keys + int64_t(lo) * W, V, W, 0, bm, t0) == 0) found = lo;
        }
        if (found >= 0) {
          hit = true;
          e = o_ci | d.idx[found];
        }
      }
      emit(hit, e);
    }
  }
  flush();
  // warp-reduce the issued-probe counter
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) my_issued += __shfl_xor_sync(kFull, my_issued, o);
  if (lane == 0 && my_issued) atomicAdd(issued, my_issued);
}


__global__ void k_rotate(const uint64_t* __restrict__ in, int64_t m, uint64_t* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t v = in[i];
    out[i] = (v >> 32) | (v << 32);
  }
}

// cg_query: one thread per (query r, slot s), s < ell: flip bit s; s == ell: self.
__global__ void __launch_bounds__(256)
    k_query(DictView d, const uint64_t* __restrict__ qv, int64_t nq, int32_t* __restrict__ self_idx,
            int32_t* __restrict__ nbr) {
  const int ell = d.ell, W = d.W;
  const int64_t total = nq * (ell + 1);
  const uint64_t lastmask = (ell % 64) ? ~(~0ull >> (ell % 64)) : ~0ull;
  for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < total;
       g += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = g / (ell + 1);
    const int s = int(g - r * (ell + 1));
    const uint64_t* Q = qv + r * W;
    auto qw = [&](int w) -> uint64_t { return w == W - 1 ? (Q[w] & lastmask) : Q[w]; };
    int pc = 0;
    for (int w = 0; w < W; ++w) pc += __popcll(qw(w));
    int fw = -1;
    uint64_t bm = 0;
    int layer = pc;
    if (s < ell) {
      fw = s >> 6;
      bm = 1ull << (63 - (s & 63));
      layer = (qw(fw) & bm) ? pc - 1 : pc + 1;
    }
    int64_t found = -1;
    if (layer >= 0 && layer <= ell && d.layer_off[layer] != d.layer_off[layer + 1]) {
      auto tw = [&](int w) -> uint64_t { return qw(w) ^ (w == fw ? bm : 0ull); };
      const int64_t row = dict_find(d, layer, tw(0), tw);
      if (row >= 0) found = d.idx[row];
    }
    if (s < ell) nbr[r * ell + s] = int32_t(found);
    else self_idx[r] = int32_t(found);
  }
}

int blocks_for(int64_t n, int threads, int per_sm) {
  int64_t b = (n + threads - 1) / threads;
  return int(std::max<int64_t>(1, std::min<int64_t>(b, int64_t(num_sms()) * per_sm)));
}

}  // namespace

void launch_probe(const DictView& d, const uint16_t* layer_lcp, const uint32_t* sorted_popc,
                  int lcp_prune, int64_t j_lo, int64_t j_hi, uint64_t* edges, uint64_t cap,
                  unsigned long long* count, unsigned long long* issued, cudaStream_t s) {
  if (j_hi <= j_lo) return;
  const int g = blocks_for(j_hi - j_lo, 256, 8);
  switch (d.W) {
    case 1: k_probe<1><<<g, 256, 0, s>>>(d, layer_lcp, sorted_popc, lcp_prune, j_lo, j_hi, edges, cap, count, issued); break;
    case 2: k_probe<2><<<g, 256, 0, s>>>(d, layer_lcp, sorted_popc, lcp_prune, j_lo, j_hi, edges, cap, count, issued); break;
    default: k_probe<0><<<g, 256, 0, s>>>(d, layer_lcp, sorted_popc, lcp_prune, j_lo, j_hi, edges, cap, count, issued); break;
  }
  CG_LAUNCH_CHECK();
}

void launch_rotate_edges(const uint64_t* in, int64_t m, uint64_t* out, cudaStream_t s) {
  if (m <= 0) return;
  k_rotate<<<blocks_for(m, 256, 16), 256, 0, s>>>(in, m, out);
  CG_LAUNCH_CHECK();
}

void launch_query(const DictView& d, const uint64_t* q, int64_t nq, int32_t* self_idx,
                  int32_t* nbr_idx, cudaStream_t s) {
  if (nq <= 0) return;
  k_query<<<blocks_for(nq * (d.ell + 1), 256, 16), 256, 0, s>>>(d, q, nq, self_idx, nbr_idx);
  CG_LAUNCH_CHECK();
}

}  // namespace cgk
