// probe_global.cu -- a5/a6/a7 over ONE prefix-indexed dictionary on the
// canonical cell table, with the edge list produced in canonical order by
// the probe itself (no edge sort).
//
// Dictionary (a5): the canonical table V (sorted, unique) with a 2^b prefix
// index T (T[x] = first cell whose top b bits are >= x; 1-2 cells per
// bucket at the defaults) and a prefix filter F of 2^(b+E) bits.  The popcount layering of
// the north star is implicit: a hit R of cell V must satisfy R ⊇ V and
// popc(R) = popc(V) + 1 (the adjacent layer), which the subset/equality tests
// enforce; the layered dictionary remains available (CG_DICT_SORTED).
//
// Probes (a6), one thread per canonical cell V_i, candidate bits = zero bits
// k <= lcp(V_i, V_{i+1}) (exact LCP pruning, see probe.cu):
//   near (k >= b): every target shares V_i's b-prefix and is > V_i, so it is
//     one of the cells right after i in the same bucket -- the next rows of
//     the table, already in L1 for the warp.  Row R is a hit iff R ⊇ V_i and
//     popc(R ^ V_i) = 1.
//   far (k < b): filter bit of the target's (b+E)-prefix, then the bucket
//     T[x]..T[x+1] of the survivors is compared (warp-flattened rounds).
// Output (a7): a warp owns a contiguous tile of 32 cells (per-warp ticket;
// the warps of a CTA never wait for each other); its hits go to its
// shared-memory buffer and the warp orders them by (i, j).  The tile
// reserves one block of a scratch list with a single atomicAdd and records
// (count, position); a scan of the counts + k_tile_copy then place the
// blocks in tile order, so the concatenation IS the canonical edge list (no
// global sort).
// Tiles whose hits overflow a warp buffer (dense graphs) are re-run together
// in spill mode; their hits are sorted and dropped into their ranges.
#include "kernels.cuh"

namespace cgk {
namespace {

// Work unit ("tile"): 32 consecutive canonical cells = one warp, taken by a
// per-warp atomic ticket; the 8 warps of a CTA never synchronise with each
// other (no barrier stalls behind the slowest warp of a CTA).
constexpr int kTileCells = 32;      // cells per tile = lanes per warp
constexpr int kProbeWarps = 8;      // warps per CTA (independent)
constexpr int kWarpEdgeCap = 512;   // shared-memory edge buffer per warp
constexpr int kTileEdgeCap = kWarpEdgeCap;
constexpr uint32_t kScratchChunk = 4096;  // scratch slots a warp reserves at once (>= kWarpEdgeCap)
#ifndef PROBE_TB
#define PROBE_TB 4  // tiles a warp takes per ticket
#endif
#ifndef PROBE_MIN_BLOCKS
#define PROBE_MIN_BLOCKS 6  // 40 registers, 6 CTAs (48 warps) per SM
#endif
#ifndef PROBE_FR
#define PROBE_FR 5  // filter loads in flight per round
#endif
#ifndef PROBE_UNI
#define PROBE_UNI 1  // far filter rounds over the warp's union of candidate bits
#endif
#ifndef PROBE_FRU
#define PROBE_FRU 5  // filter loads in flight per warp-uniform round
#endif
#ifndef PROBE_STG
#define PROBE_STG 1  // W in (2, 16]: tile rows staged in shared memory
#endif
#ifndef PROBE_ND
#define PROBE_ND 3  // near window: rows i+1..i+ND taken from the warp's registers (W <= 2)
#endif

template <int WC>
struct GRow {
  uint64_t w[WC > 0 ? WC : 1];
};

__global__ void k_global_index(const uint64_t* __restrict__ cells, int64_t nc, int W, int b,
                               int fb, uint32_t* __restrict__ T, uint32_t* __restrict__ F) {
  const int64_t top = int64_t(1) << b;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nc;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t w0 = cells[i * W];
    const int64_t x = b ? int64_t(w0 >> (64 - b)) : 0;
    const int64_t xp = i == 0 ? -1 : (b ? int64_t(cells[(i - 1) * W] >> (64 - b)) : 0);
    for (int64_t q = xp + 1; q <= x; ++q) T[q] = uint32_t(i);
    if (i == nc - 1)
      for (int64_t q = x + 1; q <= top; ++q) T[q] = uint32_t(nc);
    const uint64_t y = w0 >> (64 - fb);
    atomicOr(F + (y >> 5), 1u << (y & 31));
  }
}

// ---------------------------------------------------------------- tile output
// Shared by the prefix-dictionary and the hash-dictionary probes.  A warp
// owns a tile of 32 consecutive source cells; its hits are appended to its
// shared-memory buffer (one ballot per round) and, at the end of the tile,
// ordered by (i, j) and written as one block of the scratch list.
struct TileOut {
  uint64_t* wbuf;       // the warp's buffer [kWarpEdgeCap]
  uint32_t wfill;       // warp-uniform fill
  uint32_t lt;          // lanemask_lt
  uint64_t* spill;      // spill mode (overflow re-run): unordered global list
  uint64_t spill_cap;
  unsigned long long* spill_n;
  // lane 0: the warp's current reservation of the scratch list (chunks of
  // kScratchChunk slots, one atomic per chunk instead of one per tile: the
  // per-tile atomic on a single counter was 38 % of the stall samples) and
  // the warp's total hits (one atomic at the end of the kernel)
  // (kept in shared memory, [0] chunk position, [1] slots left, [2] hits:
  // registers are the probe's occupancy limit)
  unsigned long long* st;
  uint32_t chunk;  // slots per reservation: up to kScratchChunk, at most a quarter
                   // of the scratch list spread over all warps (small inputs)

  __device__ __forceinline__ void emit(bool hit, uint64_t e) {
    const int lane = threadIdx.x & 31;
    const uint32_t hb = __ballot_sync(kFull, hit);
    if (hb) {
      const int leader = __ffs(hb) - 1;
      if (spill) {
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(spill_n, (unsigned long long)__popc(hb));
        base = __shfl_sync(kFull, base, leader);
        if (hit) {
          const unsigned long long pos = base + __popc(hb & lt);
          if (pos < spill_cap) spill[pos] = e;
        }
        return;
      }
      // per-warp buffer: the warp owns 32 consecutive cells, so its list
      // sorted on its own is a contiguous piece of the tile's sorted list
      if (hit) {
        const uint32_t pos = wfill + __popc(hb & lt);
        if (pos < kWarpEdgeCap) wbuf[pos] = e;
      }
      wfill += __popc(hb);
    }
  }

  // The warp orders its own list: short lists (<= 32, the common case) by
  // rank counting, <= 64 on 64-bit keys, longer ones by a warp-synchronous
  // bitonic network in the buffer; one atomicAdd reserves the tile's block of
  // the scratch list.  tcnt / tpos let a scan + copy place the blocks in
  // canonical order afterwards (a look-back would make each tile wait for its
  // predecessor).  i0 = the tile's first source sequence number.
  // at the end of the kernel: the warp's hits into total[1]
  __device__ __forceinline__ void finish(unsigned long long* total) {
    if ((threadIdx.x & 31) == 0 && st[2]) atomicAdd(total + 1, st[2]);
  }

  template <class Canon>
  __device__ __forceinline__ void flush(int64_t tile, int64_t i0, uint64_t* __restrict__ out,
                                        uint64_t cap, uint32_t* __restrict__ tcnt,
                                        uint64_t* __restrict__ tpos, unsigned long long* total,
                                        uint4* __restrict__ ovf, uint32_t* ovf_n, Canon canon) {
    const int lane = threadIdx.x & 31;
    const uint32_t wn = min(wfill, uint32_t(kWarpEdgeCap));
    __syncwarp();
    if (wn > 64) {
      int P = 1;
      while (P < int(wn)) P <<= 1;
      for (int q = int(wn) + lane; q < P; q += 32) wbuf[q] = ~0ull;
      __syncwarp();
      for (int kk = 2; kk <= P; kk <<= 1) {
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
          const int lg = __ffs(jj) - 1;
          for (int p = lane; p < (P >> 1); p += 32) {
            const int a = ((p >> lg) << (lg + 1)) | (p & (jj - 1));
            const int c = a + jj;
            const bool up = (a & kk) == 0;
            const uint64_t x = wbuf[a], y = wbuf[c];
            if ((y < x) == up) {
              wbuf[a] = y;
              wbuf[c] = x;
            }
          }
          __syncwarp();
        }
      }
    }
    // block positions are 64-bit: m may exceed 2^32 (m <= n_c*ell/2)
    uint64_t bs = 0;
    if (lane == 0) {
      tcnt[tile] = wfill;
      if (wfill <= uint32_t(kWarpEdgeCap)) st[2] += wfill;  // hits placed in the scratch list
      if (wfill > uint32_t(kWarpEdgeCap)) {
        // rare: hits beyond the warp buffer were dropped; the host re-runs
        // this tile in spill mode and writes its range directly
        const uint32_t k = atomicAdd(ovf_n, 1u);
        ovf[k] = make_uint4(uint32_t(tile), 0u, wfill, 0u);
        bs = ~0ull;
      } else if (wfill) {
        if (st[1] < wfill) {  // a fresh chunk (the rest of the old one stays unused)
          st[0] = atomicAdd(total, (unsigned long long)chunk);
          st[1] = chunk;
        }
        bs = st[0];
        st[0] += wfill;
        st[1] -= wfill;
      }
      tpos[tile] = bs;  // position of the tile's block in the scratch list
    }
    const uint64_t wpos = __shfl_sync(kFull, bs, 0);
    if (wpos != ~0ull && wn > 0) {
      if (wn <= 32) {
        // one hit per lane.  Every path emits a source cell's hits in
        // ascending j, so the rank of a hit is #(hits of lower source lanes)
        // + #(earlier hits of its own source): a 5-bit radix rank of the
        // source lane from five ballots
        const bool h0 = lane < int(wn);
        const uint64_t e0 = h0 ? wbuf[lane] : 0ull;
        const uint32_t src = h0 ? uint32_t(e0 >> 32) - uint32_t(i0) : 0u;
        uint32_t same = __ballot_sync(kFull, h0), less = 0;
#pragma unroll
        for (int k = 4; k >= 0; --k) {
          const uint32_t bk = __ballot_sync(kFull, (src >> k) & 1u);
          const uint32_t sb = 0u - ((src >> k) & 1u);  // all ones iff bit k set
          less |= same & ~bk & sb;
          same &= bk ^ ~sb;
        }
        const uint32_t r0 = __popc(less) + __popc(same & lt);
        if (h0 && wpos + r0 < cap) out[wpos + r0] = canon(e0);
      } else if (wn <= 64) {
        // rank = number of smaller keys (the (i, j) keys are distinct);
        // every lane reads the same word per step (broadcast)
        const bool h0 = lane < int(wn), h1 = lane + 32 < int(wn);
        const uint64_t e0 = h0 ? wbuf[lane] : 0ull, e1 = h1 ? wbuf[lane + 32] : 0ull;
        uint32_t r0 = 0, r1 = 0;
        for (uint32_t p = 0; p < wn; ++p) {
          const uint64_t x = wbuf[p];
          r0 += x < e0;
          r1 += x < e1;
        }
        if (h0 && wpos + r0 < cap) out[wpos + r0] = canon(e0);
        if (h1 && wpos + r1 < cap) out[wpos + r1] = canon(e1);
      } else {
        for (uint32_t q = lane; q < wn; q += 32)
          if (wpos + q < cap) out[wpos + q] = canon(wbuf[q]);  // sorted (i << 32 | j) keys
      }
    }
  }
};

// FR: filter loads in flight per lane and round; NR / SR: near rows and
// survivor-bucket rows compared per round (A/B at C5: FR 3-6, NR/SR 1, 2, 4)
// SUB: the dictionary is a subsequence U of the canonical table (a rank's
// popcount layers): source q is dictionary row
// g.src_pos[q], and rows map to canonical indices through g.idx.  Hits are
// keyed (q << 32 | dictionary row) inside the kernel and converted to
// canonical (i << 32 | j) when written (idx is increasing, so the order is
// the same).  Without SUB, q = row = canonical index.
// STG (2 < W <= kStgMaxW, full dictionary): the warp first copies its tile's
// 32 rows and the kStgExtra rows after it into shared memory with coalesced
// loads (a row is W contiguous words, lanes over words); the cells' own
// words, lcp(V_i, V_{i+1}), the near-bucket compares and the survivors'
// owner words are then read from there.  With a thread per cell straight
// from global memory every load instruction touched 32 different rows (the
// north star's warp-cooperative handling of long ell).
constexpr int kStgMaxW = 16;
constexpr int kStgExtra = 4;
constexpr int kStgRows = kTileCells + kStgExtra;
size_t probe_stg_smem(int W) { return size_t(kProbeWarps) * kStgRows * (W + 1) * 8; }

template <int WC, bool SUB = false, int FR = PROBE_FR, int NR = 2, int SR = 2, bool STG = false,
          int FRU = PROBE_FRU>
__global__ void __launch_bounds__(32 * kProbeWarps, STG ? 3 : PROBE_MIN_BLOCKS)
    k_probe_global(GlobalDict g, int lcp_prune, int64_t i_lo, int64_t i_hi, int64_t ntiles,
                   uint64_t* __restrict__ out, uint64_t cap, uint32_t* __restrict__ tcnt,
                   uint64_t* __restrict__ tpos, uint32_t* ticket,
                   unsigned long long* total, unsigned long long* issued,
                   uint64_t* __restrict__ spill, uint64_t spill_cap, unsigned long long* spill_n,
                   uint4* __restrict__ ovf, uint32_t* ovf_n,
                   const uint8_t* __restrict__ tile_sel) {
  __shared__ uint64_t ebuf[kProbeWarps][kWarpEdgeCap];
  extern __shared__ __align__(16) uint64_t stg_raw[];  // STG: [warp][kStgRows][W + 1]
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t lt = lanemask_lt();
  const int W = WC > 0 ? WC : g.W;
  const int b = g.b;
  const int fb = g.b + g.fextra;
  uint32_t my_issued = 0;  // per thread (< 2^32); summed as 64-bit at the end
  uint64_t* wbuf = ebuf[tid >> 5];
  __shared__ unsigned long long s_to[kProbeWarps][3];
  if (lane == 0) s_to[tid >> 5][0] = s_to[tid >> 5][1] = s_to[tid >> 5][2] = 0;
  __syncwarp();
  uint32_t chunk = kScratchChunk;
  while (chunk > uint32_t(kWarpEdgeCap) &&
         uint64_t(chunk) * 4ull * gridDim.x * kProbeWarps > cap)
    chunk >>= 1;
  TileOut to{wbuf, 0u, lt, spill, spill_cap, spill_n, s_to[tid >> 5], chunk};
  uint32_t tb_left = 0, tb_next = 0;
  // PROBE_TB tiles per ticket only when every warp gets many tickets (small
  // inputs: one tile per ticket, or a few warps would take all the work)
  const uint32_t tb =
      ntiles >= int64_t(64) * gridDim.x * kProbeWarps ? uint32_t(PROBE_TB) : 1u;

  while (true) {
    if (tb_left == 0) {  // tb consecutive tiles per ticket
      uint32_t tk = 0;
      if (lane == 0) tk = atomicAdd(ticket, tb);
      tb_next = __shfl_sync(kFull, tk, 0);
      tb_left = tb;
    }
    const int64_t tile = int64_t(tb_next++);
    --tb_left;
    if (tile >= ntiles) break;
    if (tile_sel && !tile_sel[tile]) continue;  // spill re-run: only the overflow tiles
    const int64_t i = i_lo + tile * kTileCells + lane;  // source sequence number q
    const bool valid = i < i_hi;           // this lane probes
    int64_t row = i;                       // its dictionary row
    if (SUB) row = valid ? int64_t(g.src_pos[i]) : -1;
    const bool row_ok = SUB ? valid : (i < g.n_cells);  // row exists (a shuffle source past i_hi)
    // ---- the cell
    const uint64_t* Vp = g.keys + (row_ok ? row : 0) * W;
    const int SW = W + 1;  // STG row stride in words (odd: lanes hit different banks)
    uint64_t* srw = nullptr;
    int64_t stg_r0 = 0, stg_n = 0;  // STG: first staged row, staged rows
    if (STG) {
      srw = stg_raw + (tid >> 5) * (kStgRows * SW);
      stg_r0 = i - lane;
      stg_n = min(int64_t(kStgRows), g.n_cells - stg_r0);
      // lanes over words: Wp = pow2 >= W lanes per row, 32 / Wp rows per step
      const int lw = W <= 4 ? 2 : (W <= 8 ? 3 : 4);
      const int wq = lane & ((1 << lw) - 1), rq = lane >> lw;
      const int per = 32 >> lw;
      __syncwarp();  // the previous tile's reads of the buffer are done
      // asynchronous copies (cp.async, no register round trip): all of the
      // lane's words are in flight at once
      if (wq < W)
        for (int rr = rq; rr < int(stg_n); rr += per) {
          const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(srw + rr * SW + wq));
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d),
                       "l"(g.keys + (stg_r0 + rr) * W + wq)
                       : "memory");
        }
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncwarp();
      if (row_ok) Vp = srw + lane * SW;
    }
    uint64_t v[WC > 0 ? WC : 1];
    if (WC > 0) {
#pragma unroll
      for (int w = 0; w < (WC > 0 ? WC : 1); ++w) v[w] = row_ok ? Vp[w] : 0ull;
    }
    auto V = [&](int w) -> uint64_t {
      if (WC > 0) {
        uint64_t r = v[0];
#pragma unroll
        for (int u = 1; u < (WC > 0 ? WC : 1); ++u)
          if (u == w) r = v[u];
        return r;
      }
      return Vp[w];
    };
    int kmax = -1;
    // Near window (W <= 2, full dictionary): rows i+1..i+ND are the cells of
    // lanes lane+1..lane+ND, or of the ND rows after the tile (loaded once by
    // lanes 0..ND-1); taken by shuffle, they give lcp(V_i, V_{i+1}) and the
    // near-bit hits without a T load or a row load
    constexpr bool WIN = (WC == 1 || WC == 2) && !SUB && PROBE_ND > 0;
    constexpr int ND = WIN ? PROBE_ND : 1;
    constexpr int WW = WC > 0 ? WC : 1;
    uint64_t rw[ND][WW];
    bool rin[ND];
    if (WIN) {
      const int64_t er = i - lane + kTileCells + lane;  // row after the tile
      uint64_t e[WW];
#pragma unroll
      for (int w = 0; w < WW; ++w) e[w] = 0ull;
      if (lane < ND && er < g.n_cells) {
        if (WC == 2) {
          const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(g.keys + er * 2);
          e[0] = x.x;
          e[WW - 1] = x.y;
        } else {
          e[0] = g.keys[er];
        }
      }
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        const int src = (lane + d + 1) & 31;
        const bool inw = lane + d + 1 < 32;
#pragma unroll
        for (int w = 0; w < WW; ++w) {
          const uint64_t a = __shfl_sync(kFull, v[w], src);
          const uint64_t c = __shfl_sync(kFull, e[w], src);
          rw[d][w] = inw ? a : c;
        }
        rin[d] = row_ok && i + d + 1 < g.n_cells;
      }
      if (valid) {
        if (lcp_prune) {
          if (rin[0]) {
            const uint64_t x0 = rw[0][0] ^ v[0];
            int l;
            if (WC == 2) {
              const uint64_t x1 = rw[0][WW - 1] ^ v[WW - 1];
              l = x0 ? __clzll(x0) : 64 + __clzll(x1);  // rows differ: x1 != 0 if x0 == 0
            } else {
              l = __clzll(x0);
            }
            kmax = min(l, g.ell - 1);
          }
        } else {
          kmax = g.ell - 1;
        }
      }
    } else {
    // the next row is the neighbouring lane's cell: take it by shuffle
    // (lane 31 and the end of the range load it)
    const bool nx_ok = row_ok && row + 1 < g.n_cells;  // the row has a successor row
    uint64_t nxt[WC > 0 ? WC : 1];
    if (WC > 0) {
#pragma unroll
      for (int w = 0; w < (WC > 0 ? WC : 1); ++w) nxt[w] = __shfl_down_sync(kFull, v[w], 1);
      bool nx_shfl = lane < 31;
      if (SUB) {
        const int64_t rn = __shfl_down_sync(kFull, row, 1);  // every lane shuffles
        nx_shfl = nx_shfl && rn == row + 1;
      }
      if (!nx_shfl && nx_ok) {
#pragma unroll
        for (int w = 0; w < (WC > 0 ? WC : 1); ++w) nxt[w] = Vp[W + w];
      }
    }
    if (valid) {
      if (lcp_prune) {
        // lcp(V_i, V_{i+1}); the last cell has no successor and probes nothing
        if (nx_ok) {
          const uint64_t* Np = (STG && lane + 1 < stg_n) ? Vp + SW : g.keys + (row + 1) * W;
          const bool shfl = WC > 0;
          int l = -1;
          const int n = WC > 0 ? WC : W;
          for (int w = 0; w < n && l < 0; ++w) {
            uint64_t nw = 0;
            if (WC > 0) {
#pragma unroll
              for (int u = 0; u < (WC > 0 ? WC : 1); ++u)
                if (u == w) nw = nxt[u];
            }
            const uint64_t x = (shfl ? nw : Np[w]) ^ V(w);
            if (x) l = 64 * w + __clzll(x);
          }
          kmax = (l < 0) ? g.ell - 1 : min(l, g.ell - 1);
        }
      } else {
        kmax = g.ell - 1;
      }
    }
    }
    const uint64_t v0 = V(0);
    const uint64_t ci = uint64_t(i) << 32;
    // in-kernel hit key (q << 32 | row) -> canonical (i << 32 | j)
    auto canon = [&](uint64_t e) -> uint64_t {
      if (!SUB) return e;
      return (uint64_t(g.idx[g.src_pos[uint32_t(e >> 32)]]) << 32) | g.idx[uint32_t(e)];
    };

    to.wfill = 0;
    auto emit = [&](bool hit, uint64_t e) { to.emit(hit, e); };

    // ---- near: rows i+1.. in V's own b-prefix bucket.  Every such row R is
    // > V and shares V's first b bits, so it is a hit iff R ^ V is one bit
    // (R = V | e_k, k >= b); the rows stay in the bucket up to its end.
    const uint64_t pv = b ? (v0 >> (64 - b)) : 0ull;
    // row indices fit in 32 bits (T is u32): 32-bit index arithmetic
    const uint32_t i32 = uint32_t(row);
    bool near_on = kmax >= b;
    uint32_t r = i32 + 1;  // first row the scan below compares
    if (WIN) {
      // the window: rows i+1..i+ND from registers
      bool inb = valid && near_on;
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        const uint64_t x0 = rw[d][0] ^ v0;
        inb = inb && rin[d] && (b == 0 || (x0 >> (64 - b)) == 0);
        int diff = __popcll(x0);
        if (WC == 2) diff += __popcll(rw[d][WW - 1] ^ v[WW - 1]);
        my_issued += inb;
        emit(inb && diff == 1, ci | uint64_t(i32 + uint32_t(d) + 1u));
      }
      near_on = inb;  // row i+ND is still in the bucket: scan on from i+ND+1
      r = i32 + uint32_t(ND) + 1u;
    }
    const uint32_t r0 = r;
    uint32_t bucket_end = r0;
    if (near_on) bucket_end = g.T[pv + 1];
    const bool near_scan = near_on && (bucket_end - r0 <= 16u);
    while (__any_sync(kFull, near_scan && r < bucket_end)) {
      bool hit[NR] = {};
      if (near_scan && r < bucket_end) {
#pragma unroll
        for (int u = 0; u < NR; ++u) {
          const uint32_t rr = r + u;
          if (rr < bucket_end) {
            const int64_t so = int64_t(rr) - stg_r0;
            const uint64_t* R = (STG && so < stg_n) ? srw + so * SW : g.keys + size_t(rr) * W;
            uint64_t miss = 0;
            int diff = 0;
            if (WC == 2) {
              const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(R);
              miss = (v0 & ~x.x) | (V(1) & ~x.y);
              diff = __popcll(x.x ^ v0) + __popcll(x.y ^ V(1));
            } else {
              const int n = WC > 0 ? WC : W;
              for (int w = 0; w < n; ++w) {
                const uint64_t x = R[w];
                miss |= V(w) & ~x;
                diff += __popcll(x ^ V(w));
              }
            }
            hit[u] = (miss == 0) && (diff == 1);
            ++my_issued;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < NR; ++u) emit(hit[u], ci | uint64_t(r + uint32_t(u)));
      if (near_scan) r += NR;
    }
    // big bucket (skewed data): per candidate binary search in (i, bucket_end)
    {
      bool has = near_on && !near_scan;
      int cw = has ? (kmax >> 6) : 0;
      const int cw_lo = b >> 6;
      auto nmask = [&](int w) -> uint64_t {
        uint64_t m = ~V(w);
        if (w == (kmax >> 6)) m &= ~0ull << (63 - (kmax & 63));
        if (w == cw_lo && b > 0) m &= ~0ull >> b;
        return m;
      };
      uint64_t z = has ? nmask(cw) : 0ull;
      auto next = [&]() -> bool {
        while (z == 0 && cw > cw_lo) {
          --cw;
          z = nmask(cw);
        }
        return z != 0;
      };
      has = has && next();
      while (__any_sync(kFull, has)) {
        bool hit = false;
        uint64_t e = 0;
        if (has) {
          const uint64_t bm = z & (~z + 1);
          z ^= bm;
          const int fw = cw;
          ++my_issued;
          int64_t lo = r0, len = int64_t(bucket_end) - r0;  // rows before r0 were compared
          while (len > 0) {
            const int64_t half = len >> 1;
            const uint64_t* R = g.keys + (lo + half) * W;
            int c = 0;
            const int n = WC > 0 ? WC : W;
            for (int w = 0; w < n && c == 0; ++w) {
              const uint64_t a = R[w], tv = V(w) | (w == fw ? bm : 0ull);
              c = a < tv ? -1 : (a > tv ? 1 : 0);
            }
            if (c < 0) {
              lo += half + 1;
              len -= half + 1;
            } else {
              len = half;
            }
          }
          if (lo < bucket_end) {
            const uint64_t* R = g.keys + lo * W;
            bool eq = true;
            const int n = WC > 0 ? WC : W;
            for (int w = 0; w < n && eq; ++w) eq = R[w] == (V(w) | (w == fw ? bm : 0ull));
            if (eq) {
              hit = true;
              e = ci | uint64_t(lo);
            }
          }
          has = next();
        }
        emit(hit, e);
      }
    }
    // ---- far: zero bits k < min(b, kmax + 1) (word 0, b <= 28): filter.
    // 32-bit arithmetic: bit k of the key is bit 31 - k of its top word, the
    // filter prefix (fb <= 32 bits) fits in a u32; surv marks the survivors
    // in the same top-word bit positions.
    uint32_t surv = 0;
    const int kfar = min(b - 1, kmax);
    // With fextra >= 5 a far flip (key bit k < b) lands on prefix bit
    // fb - 1 - k >= 5: it changes the filter WORD only, the bit within the
    // word is the cell's own (y0 & 31), so the test is two shifts.
    // Warp-uniform rounds (PROBE_UNI): the 32 cells of a tile are consecutive
    // in canonical order and share their top ~log2(n/32) bits, so their
    // candidate far bits are mostly the same positions; the warp walks the
    // union of its lanes' candidate bits once (the loop counter, the bit
    // extraction and the filter word offset are warp-uniform) and each lane
    // keeps the bits it needs.  A lane whose bit k is 1 loads its own word
    // (OR with the flip) and masks it out.  Per-lane rounds ran as many
    // rounds as the lane with the most zero bits, ~11 instructions per slot.
    if (PROBE_UNI && g.fextra >= 5 && b > 0) {
      const uint32_t y0 = uint32_t(v0 >> (64 - fb));
      const uint32_t zl = kfar >= 0 ? ~uint32_t(v0 >> 32) & (0xffffffffu << (31 - kfar)) : 0u;
      my_issued += __popc(zl);
      uint32_t uz = __reduce_or_sync(kFull, zl);
      const uint32_t wy = y0 >> 5;
      const int sh5 = 32 - fb + 5;
      const uint32_t sc = 31u - (y0 & 31u);
      while (uz) {
        uint32_t bm[FRU], fw[FRU];
#pragma unroll
        for (int u = 0; u < FRU; ++u) {
          bm[u] = uz & (0u - uz);
          uz ^= bm[u];
          fw[u] = __ldg(g.F + (wy | (bm[u] >> sh5)));
        }
#pragma unroll
        for (int u = 0; u < FRU; ++u) surv |= bm[u] & uint32_t(int32_t(fw[u] << sc) >> 31);
      }
      surv &= zl;
    } else if (kfar >= 0) {
      const uint32_t y0 = uint32_t(v0 >> (64 - fb));
      const int fsh = 32 - fb;
      uint32_t z = ~uint32_t(v0 >> 32) & (0xffffffffu << (31 - kfar));
      my_issued += __popc(z);
      // branch-free rounds of FR filter loads in flight; an exhausted slot
      // (bm = 0) re-reads the cell's own filter word and is masked out.
      if (g.fextra >= 5) {
        const uint32_t wy = y0 >> 5;
        const int sh5 = fsh + 5;
        const uint32_t sc = 31u - (y0 & 31u);
        while (z) {
          uint32_t bm[FR], fw[FR];
#pragma unroll
          for (int u = 0; u < FR; ++u) {
            bm[u] = z & (0u - z);
            z ^= bm[u];
            fw[u] = __ldg(g.F + (wy | (bm[u] >> sh5)));
          }
#pragma unroll
          for (int u = 0; u < FR; ++u) surv |= bm[u] & uint32_t(int32_t(fw[u] << sc) >> 31);
        }
      }
      while (z) {
        uint32_t bm[FR], fa[FR], fw[FR];
#pragma unroll
        for (int u = 0; u < FR; ++u) {
          bm[u] = z & (0u - z);
          z ^= bm[u];
          fa[u] = y0 | (bm[u] >> fsh);
          fw[u] = __ldg(g.F + (fa[u] >> 5));
        }
#pragma unroll
        for (int u = 0; u < FR; ++u) surv |= bm[u] & (0u - (__funnelshift_r(fw[u], fw[u], fa[u]) & 1u));  // shift mod 32
      }
    }
    // ---- far survivors, flattened over the warp
    const uint32_t nsv = __popc(surv);
    uint32_t incl = nsv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t total_sv = __shfl_sync(kFull, incl, 31);
    const uint64_t my_v1 = (WC == 2) ? V(1) : 0ull;
    // (owner lane, bit) of every survivor in flattened order, as a u16 table
    // at the tail of the warp's edge buffer when it fits beside the hits the
    // rounds can still append (at most one per survivor); else both are
    // found per round by a search over the prefix sums
    const bool use_tab = to.wfill + total_sv + (total_sv + 3) / 4 <= uint32_t(kWarpEdgeCap);
    uint16_t* stab = reinterpret_cast<uint16_t*>(wbuf + kWarpEdgeCap) - total_sv;
    if (use_tab) {
      uint32_t sv = surv, pos = incl - nsv;
      while (sv) {
        const uint32_t k = __ffs(sv) - 1;  // least significant bit first: ascending j
        sv &= sv - 1;
        stab[pos++] = uint16_t((uint32_t(lane) << 8) | k);
      }
      __syncwarp();
    }
    for (uint32_t gb = 0; gb < total_sv; gb += 32) {
      const uint32_t gg = gb + lane;
      int owner = 31, k = 0;
      if (use_tab) {
        if (gg < total_sv) {
          const uint32_t en = stab[gg];
          owner = int(en >> 8);
          k = int(en & 255u);
        }
      } else {
        owner = 0;
#pragma unroll
        for (int s2 = 16; s2 >= 1; s2 >>= 1) {
          const uint32_t ic = __shfl_sync(kFull, incl, owner + s2 - 1);
          if (ic <= gg) owner += s2;
        }
        owner = min(owner, 31);
        const uint32_t o_incl = __shfl_sync(kFull, incl, owner);
        const uint32_t o_cnt = __shfl_sync(kFull, nsv, owner);
        const uint32_t o_surv = __shfl_sync(kFull, surv, owner);
        if (gg < total_sv) {
          int m = int(gg - (o_incl - o_cnt));
#pragma unroll
          for (int s2 = 16; s2 >= 1; s2 >>= 1) {
            const int c = __popc((o_surv >> k) & ((1u << s2) - 1u));
            if (m >= c) {
              m -= c;
              k += s2;
            }
          }
        }
      }
      const uint64_t o_v0 = __shfl_sync(kFull, v0, owner);
      const uint64_t o_v1 = __shfl_sync(kFull, my_v1, owner);
      const uint32_t o_i = __shfl_sync(kFull, i32, owner);  // owner's row
      const uint32_t o_q = SUB ? __shfl_sync(kFull, uint32_t(i), owner) : o_i;
      bool hit = false;
      uint64_t e = 0;
      if (gg < total_sv) {
        const uint64_t bm = 1ull << (32 + k);  // top-word bit k = key bit 31 - k
        const uint64_t t0 = o_v0 | bm;
        const int64_t x = int64_t(t0 >> (64 - b));
        const uint32_t lo = g.T[x], hi = g.T[x + 1];
        // owner's row (W > 2 path; STG: the owner's staged row)
        const uint64_t* OV = STG ? srw + owner * SW : g.keys + size_t(o_i) * W;
        int64_t found = -1;
        if (hi - lo <= 12) {
          for (uint32_t rr = lo; rr < hi && found < 0; rr += SR) {
#pragma unroll
            for (int u = 0; u < SR; ++u) {
              const uint32_t ru = rr + u;
              if (ru < hi) {
                const uint64_t* R = g.keys + int64_t(ru) * W;
                bool eq;
                if (WC == 2) {
                  const ulonglong2 xv = *reinterpret_cast<const ulonglong2*>(R);
                  eq = xv.x == t0 && xv.y == o_v1;
                } else {
                  eq = R[0] == t0;
                  const int n = WC > 0 ? WC : W;
                  for (int w = 1; w < n && eq; ++w) eq = R[w] == OV[w];
                }
                if (eq) found = ru;
              }
            }
          }
        } else {
          int64_t lo2 = lo, len = int64_t(hi) - lo;
          while (len > 0) {
            const int64_t half = len >> 1;
            const uint64_t* R = g.keys + (lo2 + half) * W;
            int c = R[0] < t0 ? -1 : (R[0] > t0 ? 1 : 0);
            const int n = WC > 0 ? WC : W;
            for (int w = 1; w < n && c == 0; ++w) {
              const uint64_t ow = (WC == 2) ? o_v1 : OV[w];
              c = R[w] < ow ? -1 : (R[w] > ow ? 1 : 0);
            }
            if (c < 0) {
              lo2 += half + 1;
              len -= half + 1;
            } else {
              len = half;
            }
          }
          if (lo2 < int64_t(hi)) {
            const uint64_t* R = g.keys + lo2 * W;
            bool eq = R[0] == t0;
            const int n = WC > 0 ? WC : W;
            for (int w = 1; w < n && eq; ++w) eq = R[w] == ((WC == 2) ? o_v1 : OV[w]);
            if (eq) found = lo2;
          }
        }
        if (found >= 0) {
          hit = true;
          e = (uint64_t(o_q) << 32) | uint64_t(found);
        }
      }
      emit(hit, e);
    }
    if (spill) continue;  // spill mode: no ordered output
    to.flush(tile, i - lane, out, cap, tcnt, tpos, total, ovf, ovf_n, canon);
    __syncwarp();
  }
  to.finish(total);
  unsigned long long wsum = my_issued;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(kFull, wsum, o);
  if (lane == 0 && wsum) atomicAdd(issued, wsum);
}

// ---------------------------------------------------------------- hash dictionary
// The north star's alternative dictionary (a5, "an open-addressed table
// keyed on a word hash"), kept for the ncu A/B against the prefix index
// (DESIGN section 6):
//   h(x) = XOR of Z[k] over the set bits k of x, Z[k] = splitmix64(k):
//   GF(2)-linear, so the flipped key's hash is h(x) ^ Z[k] -- the probe never
//   materialises x ^ e_k;
//   buckets of 4 slots (32 B = one sector), slot = tag32 << 32 | row, tag =
//   low 32 bits of h | 1 (0 = empty), bucket = the top lb bits of h, linear
//   probing over buckets; every tag hit is verified on the full row, so a
//   hash collision costs time, never correctness.
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void k_hash_z(uint64_t* __restrict__ Z, int ell) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < ell; k += gridDim.x * blockDim.x)
    Z[k] = splitmix64(uint64_t(k));
}

__global__ void k_hash_build(const uint64_t* __restrict__ cells, int64_t nc, int W,
                             const uint64_t* __restrict__ Z, int lb,
                             unsigned long long* __restrict__ slots, uint64_t* __restrict__ hv) {
  const uint64_t nb = uint64_t(1) << lb;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nc;
       i += int64_t(gridDim.x) * blockDim.x) {
    uint64_t h = 0;
    for (int w = 0; w < W; ++w) {
      uint64_t x = cells[i * W + w];
      while (x) {  // bit k of the key = bit 63 - (k & 63) of word k >> 6
        const int t = __clzll(x);
        h ^= __ldg(Z + 64 * w + t);
        x &= ~(0x8000000000000000ull >> t);
      }
    }
    hv[i] = h;
    const unsigned long long e = (uint64_t(uint32_t(h) | 1u) << 32) | uint64_t(i);
    uint64_t b = lb ? (h >> (64 - lb)) : 0;
    while (true) {
      bool done = false;
      for (int q = 0; q < 4 && !done; ++q)
        done = atomicCAS(slots + b * 4 + q, 0ull, e) == 0ull;
      if (done) break;
      b = (b + 1) & (nb - 1);
    }
  }
}

// One thread per canonical cell (tiles of 32 per warp, as k_probe_global):
// every zero bit k <= lcp(V_i, V_{i+1}) is looked up -- FR lookups in flight
// per round, from the least significant candidate up (ascending targets)
#ifndef HASH_FR
#define HASH_FR 3
#endif
template <int WC, int FR = HASH_FR>
__global__ void __launch_bounds__(32 * kProbeWarps, 4)
    k_probe_hash(GlobalDict g, int lcp_prune, int64_t i_lo, int64_t i_hi, int64_t ntiles,
                 uint64_t* __restrict__ out, uint64_t cap, uint32_t* __restrict__ tcnt,
                 uint64_t* __restrict__ tpos, uint32_t* ticket, unsigned long long* total,
                 unsigned long long* issued, uint64_t* __restrict__ spill, uint64_t spill_cap,
                 unsigned long long* spill_n, uint4* __restrict__ ovf, uint32_t* ovf_n,
                 const uint8_t* __restrict__ tile_sel) {
  __shared__ uint64_t ebuf[kProbeWarps][kWarpEdgeCap];
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t lt = lanemask_lt();
  const int W = WC > 0 ? WC : g.W;
  const int lb = g.lb;
  const uint64_t bmask = (uint64_t(1) << lb) - 1;
  uint32_t my_issued = 0;
  uint64_t* wbuf = ebuf[tid >> 5];
  __shared__ unsigned long long s_to[kProbeWarps][3];
  if (lane == 0) s_to[tid >> 5][0] = s_to[tid >> 5][1] = s_to[tid >> 5][2] = 0;
  __syncwarp();
  uint32_t chunk = kScratchChunk;
  while (chunk > uint32_t(kWarpEdgeCap) &&
         uint64_t(chunk) * 4ull * gridDim.x * kProbeWarps > cap)
    chunk >>= 1;
  TileOut to{wbuf, 0u, lt, spill, spill_cap, spill_n, s_to[tid >> 5], chunk};
  uint32_t tb_left = 0, tb_next = 0;
  // PROBE_TB tiles per ticket only when every warp gets many tickets (small
  // inputs: one tile per ticket, or a few warps would take all the work)
  const uint32_t tb =
      ntiles >= int64_t(64) * gridDim.x * kProbeWarps ? uint32_t(PROBE_TB) : 1u;
  while (true) {
    if (tb_left == 0) {  // tb consecutive tiles per ticket
      uint32_t tk = 0;
      if (lane == 0) tk = atomicAdd(ticket, tb);
      tb_next = __shfl_sync(kFull, tk, 0);
      tb_left = tb;
    }
    const int64_t tile = int64_t(tb_next++);
    --tb_left;
    if (tile >= ntiles) break;
    if (tile_sel && !tile_sel[tile]) continue;
    const int64_t i = i_lo + tile * kTileCells + lane;
    const bool valid = i < i_hi;
    const uint64_t* Vp = g.keys + (valid ? i : 0) * W;
    int kmax = -1;
    if (valid) {
      if (!lcp_prune) {
        kmax = g.ell - 1;
      } else if (i + 1 < g.n_cells) {
        int l = -1;
        for (int w = 0; w < W && l < 0; ++w) {
          const uint64_t x = Vp[w] ^ Vp[W + w];
          if (x) l = 64 * w + __clzll(x);
        }
        kmax = l < 0 ? g.ell - 1 : min(l, g.ell - 1);
      }
    }
    const uint64_t h = valid ? g.hv[i] : 0ull;
    to.wfill = 0;
    // candidate bits: zero bits k <= kmax, word by word from the last
    int cw = kmax >= 0 ? (kmax >> 6) : -1;
    auto cmask = [&](int w) -> uint64_t {
      uint64_t m = ~Vp[w];
      if (w == (kmax >> 6)) m &= ~0ull << (63 - (kmax & 63));
      return m;
    };
    uint64_t z = cw >= 0 ? cmask(cw) : 0ull;
    auto next_bit = [&](int* k) -> bool {
      while (z == 0 && cw > 0) {
        --cw;
        z = cmask(cw);
      }
      if (z == 0) return false;
      const int t = 63 - (__ffsll(z) - 1);  // least significant candidate first
      z &= z - 1;
      *k = 64 * cw + t;
      return true;
    };
    bool more = true;
    while (__any_sync(kFull, more)) {
      int k[FR];
      bool on[FR];
      ulonglong2 s0[FR], s1[FR];
      uint64_t hh[FR];
#pragma unroll
      for (int u = 0; u < FR; ++u) {
        on[u] = more && next_bit(&k[u]);
        more = on[u];
        hh[u] = on[u] ? (h ^ __ldg(g.Z + k[u])) : 0ull;
        const uint64_t b = lb ? (hh[u] >> (64 - lb)) : 0ull;
        const ulonglong2* bp = reinterpret_cast<const ulonglong2*>(g.slots + b * 4);
        if (on[u]) {
          s0[u] = bp[0];
          s1[u] = bp[1];
          ++my_issued;
        }
      }
#pragma unroll
      for (int u = 0; u < FR; ++u) {
        bool hit = false;
        uint64_t e = 0;
        if (on[u]) {
          const uint32_t tag = uint32_t(hh[u]) | 1u;
          uint64_t b = lb ? (hh[u] >> (64 - lb)) : 0ull;
          ulonglong2 a = s0[u], c = s1[u];
          const int fw = k[u] >> 6;
          const uint64_t fb = 0x8000000000000000ull >> (k[u] & 63);
          while (true) {
            const uint64_t sl[4] = {a.x, a.y, c.x, c.y};
            bool empty = false;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (sl[q] == 0ull) empty = true;
              if (!hit && uint32_t(sl[q] >> 32) == tag) {
                const int64_t j = int64_t(uint32_t(sl[q]));
                const uint64_t* R = g.keys + j * W;
                bool eq = true;
                for (int w = 0; w < W && eq; ++w) eq = R[w] == (Vp[w] ^ (w == fw ? fb : 0ull));
                if (eq) {
                  hit = true;
                  e = (uint64_t(i) << 32) | uint64_t(j);
                }
              }
            }
            if (hit || empty) break;
            b = (b + 1) & bmask;  // a full bucket: the key may sit further on
            const ulonglong2* bp = reinterpret_cast<const ulonglong2*>(g.slots + b * 4);
            a = bp[0];
            c = bp[1];
          }
        }
        to.emit(hit, e);
      }
    }
    if (spill) continue;
    to.flush(tile, i - lane, out, cap, tcnt, tpos, total, ovf, ovf_n,
             [](uint64_t e) { return e; });
    __syncwarp();
  }
  to.finish(total);
  unsigned long long wsum = my_issued;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(kFull, wsum, o);
  if (lane == 0 && wsum) atomicAdd(issued, wsum);
}

}  // namespace

void build_hash_dict(const uint64_t* cells, int64_t nc, int W, int ell, int lb, uint64_t* Z,
                     uint64_t* slots, uint64_t* hv, cudaStream_t s) {
  k_hash_z<<<std::max(1, (ell + 255) / 256), 256, 0, s>>>(Z, ell);
  CG_LAUNCH_CHECK();
  CG_CUDA(cudaMemsetAsync(slots, 0, (size_t(4) << lb) * 8, s));
  const int64_t blocks = std::min<int64_t>((nc + 255) / 256, int64_t(num_sms()) * 16);
  k_hash_build<<<unsigned(std::max<int64_t>(1, blocks)), 256, 0, s>>>(
      cells, nc, W, Z, lb, reinterpret_cast<unsigned long long*>(slots), hv);
  CG_LAUNCH_CHECK();
}

void build_global_index(const uint64_t* cells, int64_t nc, int W, int b, int fextra, uint32_t* T,
                        uint32_t* F, cudaStream_t s) {
  int64_t blocks = std::min<int64_t>((nc + 255) / 256, int64_t(num_sms()) * 16);
  k_global_index<<<unsigned(std::max<int64_t>(1, blocks)), 256, 0, s>>>(cells, nc, W, b, b + fextra, T, F);
  CG_LAUNCH_CHECK();
}

void launch_probe_global(const GlobalDict& g, int lcp_prune, int64_t i_lo, int64_t i_hi,
                         uint64_t* out, uint64_t cap, uint32_t* tcnt, uint64_t* tpos, uint32_t* ticket,
                         unsigned long long* total, unsigned long long* issued, uint4* ovf,
                         uint32_t* ovf_n, uint64_t* spill, uint64_t spill_cap,
                         unsigned long long* spill_n, cudaStream_t s, const uint8_t* tile_sel) {
  const int64_t ntiles = (i_hi - i_lo + kTileCells - 1) / kTileCells;
  if (ntiles <= 0) return;
  const int grid = int(std::min<int64_t>((ntiles + kProbeWarps - 1) / kProbeWarps, int64_t(num_sms()) * 8));
#define CG_PROBE_ARGS                                                                         \
  g, lcp_prune, i_lo, i_hi, ntiles, out, cap, tcnt, tpos, ticket, total, issued, spill, spill_cap, \
      spill_n, ovf, ovf_n, tile_sel
  const bool sub = g.src_pos != nullptr;
  if (g.slots) {  // hash dictionary (full table only)
    if (g.W == 1) k_probe_hash<1><<<grid, 32 * kProbeWarps, 0, s>>>(CG_PROBE_ARGS);
    else if (g.W == 2) k_probe_hash<2><<<grid, 32 * kProbeWarps, 0, s>>>(CG_PROBE_ARGS);
    else k_probe_hash<0><<<grid, 32 * kProbeWarps, 0, s>>>(CG_PROBE_ARGS);
    CG_LAUNCH_CHECK();
    return;
  }
  switch (g.W) {
    case 1:
      if (sub) k_probe_global<1, true><<<grid, 32 * kProbeWarps, 0, s>>>(CG_PROBE_ARGS);
      else k_probe_global<1><<<grid, 32 * kProbeWarps, 0, s>>>(CG_PROBE_ARGS);
      break;
    case 2:
      if (sub) k_probe_global<2, true><<<grid, 32 * kProbeWarps, 0, s>>>(CG_PROBE_ARGS);
      else k_probe_global<2><<<grid, 32 * kProbeWarps, 0, s>>>(CG_PROBE_ARGS);
      break;
    default:
      if (sub) {
        k_probe_global<0, true><<<grid, 32 * kProbeWarps, 0, s>>>(CG_PROBE_ARGS);
      } else if (g.W <= kStgMaxW && PROBE_STG) {
        auto kern = k_probe_global<0, false, PROBE_FR, 2, 2, true>;
        const size_t sm = probe_stg_smem(g.W);
        CG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        const int gs = int(std::min<int64_t>((ntiles + kProbeWarps - 1) / kProbeWarps, int64_t(num_sms()) * 3));
        kern<<<gs, 32 * kProbeWarps, sm, s>>>(CG_PROBE_ARGS);
      } else {
        k_probe_global<0><<<grid, 32 * kProbeWarps, 0, s>>>(CG_PROBE_ARGS);
      }
      break;
  }
#undef CG_PROBE_ARGS
  CG_LAUNCH_CHECK();
}

// overflow tiles: sel[t] = 1, scnt[t] = their hit count (0 elsewhere)
__global__ void k_spill_select(const uint4* __restrict__ ovf, uint32_t novf, uint8_t* __restrict__ sel,
                               uint32_t* __restrict__ scnt) {
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < novf; q += gridDim.x * blockDim.x) {
    sel[ovf[q].x] = 1;
    scnt[ovf[q].x] = ovf[q].z;
  }
}

// sorted spilled hits -> their tiles' canonical ranges:
// dst = toff[t] + (q - sstart[t]) with t the tile of the hit's source cell
__global__ void k_spill_place(const uint64_t* __restrict__ sorted, int64_t m, int64_t i_lo,
                              const uint64_t* __restrict__ toff, const uint64_t* __restrict__ sstart,
                              const uint32_t* __restrict__ src_pos, const uint32_t* __restrict__ idx,
                              uint64_t* __restrict__ out) {
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < m;
       q += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = sorted[q];
    const int64_t t = (int64_t(k >> 32) - i_lo) / kTileCells;
    uint32_t ci = uint32_t(k >> 32), cj = uint32_t(k);
    if (src_pos) {  // subsequence dictionary: (source seq, row) -> canonical
      ci = idx[src_pos[ci]];
      cj = idx[cj];
    }
    out[toff[t] + (q - sstart[t])] = uint64_t(ci) | (uint64_t(cj) << 32);
  }
}

void launch_spill_select(const uint4* ovf, uint32_t novf, uint8_t* sel, uint32_t* scnt,
                         cudaStream_t s) {
  k_spill_select<<<std::max(1u, std::min((novf + 255) / 256, 1024u)), 256, 0, s>>>(ovf, novf, sel, scnt);
  CG_LAUNCH_CHECK();
}

void launch_spill_place(const GlobalDict& g, const uint64_t* sorted, int64_t m, int64_t i_lo,
                        const uint64_t* toff, const uint64_t* sstart, uint64_t* out, cudaStream_t s) {
  if (m <= 0) return;
  const int64_t blocks = std::min<int64_t>((m + 255) / 256, int64_t(num_sms()) * 16);
  k_spill_place<<<unsigned(blocks), 256, 0, s>>>(sorted, m, i_lo, toff, sstart, g.src_pos, g.idx, out);
  CG_LAUNCH_CHECK();
}

// Tile blocks -> canonical positions.  A CTA takes 256 consecutive tiles:
// their destination ranges are contiguous (off = exclusive scan of the
// counts, 64-bit), so the CTA flattens them -- thread per destination
// element, its tile found by a binary search over the tiles' prefix in shared
// memory -- and writes one contiguous run as (i, j) u32 pairs.  Overflow
// tiles (pos = ~0) are written by the spill path and skipped here.
constexpr int kCopyTiles = 256;
constexpr int kCopyMap = 16384;  // (bytes of shared memory for the element -> tile map)

__global__ void __launch_bounds__(256)
    k_tile_copy(const uint64_t* __restrict__ scratch, const uint64_t* __restrict__ off,
                const uint64_t* __restrict__ pos, const uint32_t* __restrict__ cntv, int64_t ntiles,
                uint64_t* __restrict__ out) {
  __shared__ uint32_t s_pre[kCopyTiles + 1];
  __shared__ uint64_t s_pos[kCopyTiles];
  __shared__ uint8_t s_tile[kCopyMap];  // destination element -> its tile (E <= kCopyMap)
  for (int64_t t0 = int64_t(blockIdx.x) * kCopyTiles; t0 < ntiles;
       t0 += int64_t(gridDim.x) * kCopyTiles) {
    const int nt = int(ntiles - t0 < kCopyTiles ? ntiles - t0 : int64_t(kCopyTiles));
    __syncthreads();
    const uint64_t base = off[t0];
    // within 256 tiles the relative offsets fit 32 bits (<= 256 * 32 * ell hits)
    for (int q = threadIdx.x; q < nt; q += blockDim.x) {
      s_pre[q] = uint32_t(off[t0 + q] - base);
      s_pos[q] = pos[t0 + q];
    }
    if (threadIdx.x == 0) s_pre[nt] = uint32_t(off[t0 + nt - 1] - base) + cntv[t0 + nt - 1];
    __syncthreads();
    const uint32_t E = s_pre[nt];
    // each tile marks its destination elements (one shared byte each, no
    // per-element binary search) when the 256 tiles hold <= kCopyMap edges
    const bool map = E <= uint32_t(kCopyMap);
    if (map) {
      for (int q = threadIdx.x; q < nt; q += blockDim.x)
        for (uint32_t e = s_pre[q]; e < s_pre[q + 1]; ++e) s_tile[e] = uint8_t(q);
      __syncthreads();
    }
    // 4 edges per thread and step: all four loads in flight before the stores
    constexpr int U = 4;
    for (uint32_t e0 = threadIdx.x; e0 < E; e0 += U * blockDim.x) {
      uint64_t src[U];
      uint64_t k[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t e = e0 + u * blockDim.x;
        src[u] = ~0ull;
        if (e < E) {
          int lo = 0, hi = nt - 1;  // last tile with s_pre <= e
          if (map) lo = s_tile[e];
          else
            while (lo < hi) {
              const int mid = (lo + hi + 1) >> 1;
              if (s_pre[mid] <= e) lo = mid;
              else hi = mid - 1;
            }
          const uint64_t p = s_pos[lo];
          if (p != ~0ull) src[u] = p + (e - s_pre[lo]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) k[u] = src[u] != ~0ull ? __ldcs(scratch + src[u]) : 0ull;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (src[u] != ~0ull) out[base + e0 + u * blockDim.x] = (k[u] >> 32) | (k[u] << 32);
    }
  }
}

void launch_tile_copy(const uint64_t* scratch, const uint64_t* off, const uint64_t* pos,
                      const uint32_t* cnt, int64_t ntiles, uint64_t* out, cudaStream_t s) {
  if (ntiles <= 0) return;
  const int64_t blocks = std::min<int64_t>((ntiles + kCopyTiles - 1) / kCopyTiles, int64_t(num_sms()) * 8);
  k_tile_copy<<<unsigned(std::max<int64_t>(1, blocks)), 256, 0, s>>>(scratch, off, pos, cnt, ntiles, out);
  CG_LAUNCH_CHECK();
}

// cg_query on the global dictionary: one thread per (query r, slot s),
// s < ell: the query with bit s negated, s == ell: the query itself; the
// target's b-prefix bucket of the canonical table is searched (the row index
// IS the canonical index)
__global__ void __launch_bounds__(256)
    k_query_global(GlobalDict g, const uint64_t* __restrict__ qv, int64_t nq,
                   int32_t* __restrict__ self_idx, int32_t* __restrict__ nbr) {
  const int ell = g.ell, W = g.W, b = g.b;
  const int64_t total = nq * (ell + 1);
  const uint64_t lastmask = (ell % 64) ? ~(~0ull >> (ell % 64)) : ~0ull;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = t / (ell + 1);
    const int s = int(t - r * (ell + 1));
    const uint64_t* Q = qv + r * W;
    const int fw = s < ell ? (s >> 6) : -1;
    const uint64_t bm = s < ell ? (1ull << (63 - (s & 63))) : 0ull;
    auto tw = [&](int w) -> uint64_t {
      const uint64_t x = (w == W - 1) ? (Q[w] & lastmask) : Q[w];
      return x ^ (w == fw ? bm : 0ull);
    };
    const uint64_t t0 = tw(0);
    const int64_t x = b ? int64_t(t0 >> (64 - b)) : 0;
    // prefix filter first: most flipped targets are absent
    const int fb = b + g.fextra;
    const uint64_t y = fb ? (t0 >> (64 - fb)) : 0ull;
    const bool maybe = (g.F[y >> 5] >> (y & 31)) & 1u;
    uint32_t lo = maybe ? g.T[x] : 0u;
    uint32_t len = maybe ? g.T[x + 1] - lo : 0u;
    while (len > 0) {  // lower bound of t in the bucket
      const uint32_t half = len >> 1;
      const uint64_t* R = g.keys + int64_t(lo + half) * W;
      int c = 0;
      for (int w = 0; w < W && c == 0; ++w) {
        const uint64_t a = R[w], tv = tw(w);
        c = a < tv ? -1 : (a > tv ? 1 : 0);
      }
      if (c < 0) {
        lo += half + 1;
        len -= half + 1;
      } else {
        len = half;
      }
    }
    int32_t found = -1;
    if (maybe && lo < g.T[x + 1]) {
      const uint64_t* R = g.keys + int64_t(lo) * W;
      bool eq = true;
      for (int w = 0; w < W && eq; ++w) eq = R[w] == tw(w);
      if (eq) found = int32_t(lo);
    }
    if (s < ell) nbr[r * ell + s] = found;
    else self_idx[r] = found;
  }
}

void launch_query_global(const GlobalDict& g, const uint64_t* q, int64_t nq, int32_t* self_idx,
                         int32_t* nbr_idx, cudaStream_t s) {
  if (nq <= 0) return;
  const int64_t blocks = std::min<int64_t>((nq * (g.ell + 1) + 255) / 256, int64_t(num_sms()) * 16);
  k_query_global<<<unsigned(std::max<int64_t>(1, blocks)), 256, 0, s>>>(g, q, nq, self_idx, nbr_idx);
  CG_LAUNCH_CHECK();
}

int64_t probe_global_tiles(int64_t n) { return (n + kTileCells - 1) / kTileCells; }
int probe_global_tile_edge_cap() { return kTileEdgeCap; }
uint64_t probe_global_scratch_chunk() { return kScratchChunk; }
int probe_global_tile_cells() { return kTileCells; }

}  // namespace cgk
