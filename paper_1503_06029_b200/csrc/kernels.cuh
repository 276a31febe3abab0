// kernels.cuh -- host-side launchers of the cell-graph kernels (internal API).
#pragma once

#include "common.cuh"

namespace cgk {

// ---------------------------------------------------------------- a1 pack
// uint8[n][ell] (0/1 bytes) -> u64[n][W] MSB-first; *err |= 1 on a byte > 1.
// hist (optional, zeroed, u32[(8 - dlo) * 256]): counts of the 8-bit digits
// dlo..7 of word 0, for the MSD sort (dlo in 5..7).
// tile_hist (optional, with hist): u32[ceil(n / tile_rows)][256] counts of
// digit dlo per tile of tile_rows rows (the first one-sweep pass's tiles).
// The sweep path's input to sort_unique_msd (sw): launch_pack_sweep's regions
// (u64[256][capr][W]), their row counts rcnt[256] and the overflow flag.
// T/F (optional, b in [16, 26]): the bucket pass also writes the prefix index
// T[2^b + 1] and the b + 5-bit filter F[2^b] of the sorted unique table
// (the global dictionary of probe_global.cu) -- no separate index pass.
struct SweepIn {
  const uint64_t* regions;
  uint32_t capr;
  const uint32_t* rcnt;
  uint32_t* ovf;
  uint32_t* T = nullptr;
  uint32_t* F = nullptr;
  int b = 0;
  int B2 = 8;  // the region sweep's digit: buckets are the top 8 + B2 bits
};
// B2 for n rows (~2^10 rows per top-(8 + B2)-bit bucket), 0 = no sweep path
// (n <= 2^18 or n > 2^26)
int sweep_bits(int64_t n);
// Pack + the MSD sort's first partition (the "sweep" path, ell = 64 W,
// W <= 2): rows go to 256 regions of capr rows by the top byte of word 0,
// region d = regions[d * capr * W ..), rcnt[d] rows (unordered inside a
// region); *ovf != 0 if some region overflowed (the result is then invalid).
// ell = 64 or 128, 16-byte aligned rows (the size rule is sweep_bits)
bool pack_sweep_ok(const uint8_t* vecs, int64_t n, int ell);
uint32_t pack_sweep_capr(int64_t n);
void launch_pack_sweep(const uint8_t* vecs, int64_t n, int ell, uint64_t* regions, uint32_t capr,
                       uint32_t* rcnt, uint32_t* err, uint32_t* ovf, cudaStream_t s);
void launch_pack(const uint8_t* vecs, int64_t n, int ell, uint64_t* keys, uint32_t* err,
                 cudaStream_t s, uint32_t* hist = nullptr, int dlo = 8,
                 uint32_t* tile_hist = nullptr, int tile_rows = 0);
// packed input: copy + check pad bits (err |= 1 if a pad bit is set)
void launch_check_pad(const uint64_t* words, int64_t n, int ell, uint32_t* err, cudaStream_t s);

// ---------------------------------------------------------------- small inputs (small.cu)
// n <= 2048 rows, ell <= 256: pack, sort, dedupe, probe and the canonical
// edge list in one CTA.  cells u64[n][W], edges u64[n * ell / 2] as (i, j)
// u32 pairs (capacity: the P:106 bound), res[3] = n_c, m, input error.
bool small_build_ok(int64_t n, int ell);
void launch_small_build(const uint8_t* vecs, int64_t n, int ell, int lcp_prune, uint64_t* cells,
                        uint64_t* edges, int64_t* res, cudaStream_t s);

// ---------------------------------------------------------------- f1 signatures
// points f64[n][dim], planes f64[ell][dim+1] (a_0..a_{dim-1}, b) -> packed
// keys u64[n][W]: bit k = [fma chain b + sum a_t p_t >= 0] (sign.cu);
// *err |= 1 on a non-finite value; optional top-digit histogram as k_pack.
int signatures_max_dim();
void launch_signatures(const double* pts, int64_t n, int dim, const double* planes, int ell,
                       uint64_t* keys, uint32_t* err, cudaStream_t s, uint32_t* hist = nullptr,
                       int dlo = 8);

// ---------------------------------------------------------------- f4 CSR + BFS (graph.cu)
// canonical edge list (u32 (i, j), i < j, ascending) -> CSR with sorted
// adjacency: row_ptr u64[nv + 1], col u32[2m]
void build_csr(const uint32_t* edges, int64_t m, int64_t nv, uint64_t* row_ptr, uint32_t* col,
               cudaStream_t s);
// level-synchronous BFS from src: dist i32[nv] (-1 unreachable), optional
// canonical parent i32[nv] (smallest neighbour one level closer, -1 for the
// source / unreachable).  Returns the source's eccentricity.  Host-synchronising.
int bfs(const uint64_t* row_ptr, const uint32_t* col, int64_t nv, int64_t src, int32_t* dist,
        int32_t* parent, cudaStream_t s);

// ---------------------------------------------------------------- f3 all-pairs (allpairs.cu)
// distance-1 pairs of a cell table by the naive / anchor method (Alg. 1-2):
// unsorted (i << 32 | j) into out[0..cap); returns the total (rerun if > cap)
int allpairs_max_anchors();
uint64_t launch_allpairs(const uint64_t* cells, int64_t n, int W, int h, uint64_t* out,
                         uint64_t cap, uint64_t* n_compared, cudaStream_t s);

// ---------------------------------------------------------------- f2 insertion (insert.cu)
// V (nv sorted unique rows, canonical edges ev[mv], index g over it) +
// batch B (nb sorted unique rows, its canonical edges eb[mb]) -> the merged
// table and its canonical edge list (allocated with dev_alloc, u32 pairs).
struct GlobalDict;
void insert_merge(const uint64_t* cv_rows, int64_t nv, const uint32_t* ev, int64_t mv,
                  const uint64_t* cb_rows, int64_t nb, const uint32_t* eb, int64_t mb,
                  const GlobalDict& g, int ell, uint64_t** cells_out, int64_t* nc_out,
                  uint64_t** edges_out, int64_t* m_out, cudaStream_t s);

// ---------------------------------------------------------------- radix engine (a2, a4, a7)
struct SortStats {
  int passes = 0;
};

// Stable LSD sort of n keys (K = uint32_t or uint64_t) on bits [0, key_bits),
// 8-bit digits, constant digits skipped.  Optional u32 payload: vals_in ==
// nullptr with want_vals means "payload = original index".  Buffers are
// ping-ponged; on return *keys_out / *vals_out point to the sorted data
// (one of the given buffers).  Host-synchronising (digit histogram read-back).
template <class K>
void radix_sort(K* keys, K* keys_alt, const uint32_t* vals_in, uint32_t* vals, uint32_t* vals_alt,
                bool want_vals, int64_t n, int key_bits, K** keys_out, uint32_t** vals_out,
                cudaStream_t s, SortStats* st);

// Canonical sort of packed rows u64[n][W] (W >= 2): LSD over words W-1..0
// on (word, u32 index) pairs, then a row gather into `sorted` (u64[n][W]);
// with `order` given, the canonical order (row indices) goes there instead
// and no rows move.
// *no_dups (optional) = true when the order is known to hold no two equal
// rows (the 32-bit-prefix path compared every tie and found none).
// mode: 0 = 32-bit-prefix sort, per-word LSD if long prefix-tie runs; 1 =
// prefix sort only (returns false on long runs: nothing sorted); 2 = per-word
// LSD only.  Returns true when the order is complete.
// dup_hits (device, mode 1): a duplication sample; >= 8 makes the prefix
// sort give up at once (the caller then dedupes by hashing first).
bool sort_rows_multiword(const uint64_t* keys, int64_t n, int W, uint64_t* sorted,
                         cudaStream_t s, SortStats* st, uint32_t* order = nullptr,
                         bool* no_dups = nullptr, int mode = 0,
                         const uint32_t* dup_hits = nullptr);

// MSD fast path for W in {1, 2}: LSD passes over the top B bits only (whole
// keys move), then a shared-memory bitonic sort of each 2^B prefix bucket.
// keys/alt are ping-ponged; *sorted points at the result.  Returns false if
// a bucket exceeded the shared-memory capacity: *sorted is then only
// bucket-ordered and the caller must finish with a full sort.
bool sort_rows_msd(uint64_t* keys, uint64_t* alt, int64_t n, int W, uint64_t** sorted,
                   cudaStream_t s, SortStats* st, const uint32_t* top_hist = nullptr);
// G sorted runs (rows u64[G][stride][W], stride in rows, W <= 2, counts on the host) ->
// their rows grouped by the top B bits into out (u64[total][W]; each bucket
// holds its runs' segments one after the other) and off[2^B + 1] = bucket
// starts -- the input of sort_unique_msd(..., pre_off = off, pre_B = B).
// skip: the top `skip` bits are common to every row (a prefix chunk); the
// buckets are then bits [skip, skip + B).
void gather_runs_by_prefix(const uint64_t* runs, const int64_t* counts, int G, int64_t stride,
                           int W, int B, int skip, uint64_t* out, uint32_t* off, cudaStream_t s);
// off[q] = first row of sorted rows u64[n][W] whose top B bits are >= q, q in [0, 2^B]
void launch_prefix_bounds(const uint64_t* rows, int64_t n, int W, int B, uint32_t* off,
                          cudaStream_t s);
// prefix bits B (8, 16 or 24) the MSD path uses for n keys; digit dlo = (64-B)/8
int msd_prefix_bits(int64_t n);
// MSD sort with dedupe fused into the bucket pass: the sorted unique cells
// end up in keys or alt (*cells), *nc of them.  false = a bucket overflowed
// (keys/alt then hold the same SET of keys, bucket-ordered; run the full
// sort + dedupe instead).
// pre_off (device, 2^pre_B + 1 entries): keys already grouped by their top
// pre_B bits (launch_pack_scatter) -> no global radix pass.
// tile_hist (optional): per-tile counts of the first pass's digit from the
// pack kernel, tiles of msd_tile_rows(W) rows: the first pass skips its
// look-back.
bool sort_unique_msd(uint64_t* keys, uint64_t* alt, int64_t n, int W, uint64_t** cells,
                     int64_t* nc, cudaStream_t s, SortStats* st, const uint32_t* top_hist,
                     const uint32_t* pre_off = nullptr, int pre_B = 0,
                     const uint32_t* tile_hist = nullptr, const uint32_t* side_dev = nullptr,
                     uint32_t* side_host = nullptr, int pre_skip = 0,
                     const struct SweepIn* sw = nullptr);
// The distributed merge's bucket pass writing straight into the table: rows
// gathered[0..n) grouped into 2^B buckets (off[2^B + 1], the common top
// pre_skip bits skipped), each bucket sorted and deduplicated into
// dst + off[b], then compacted in dst; *nc distinct rows.  false = a bucket
// the shared-memory passes could not take (gathered is left intact).
bool merge_sorted_into(uint64_t* gathered, const uint32_t* off, int64_t n, int W, int B,
                       int pre_skip, uint64_t* dst, int64_t* nc, cudaStream_t s);
int msd_tile_rows(int W);
// popcount (optional) and lcp with the next cell, for a canonical table
void launch_cell_meta(const uint64_t* cells, int64_t nc, int W, uint32_t* popc, uint16_t* lcp,
                      cudaStream_t s);

// ---------------------------------------------------------------- a3 dedupe + compaction
// Distinct rows of rows u64[n][W] (first occurrences, input order) into out
// (u64[n][W] capacity) by an open-addressed hash set; returns their count.
// Used when skew overflows the MSD buckets.  Host-synchronising.
int64_t hash_unique_rows(const uint64_t* rows, int64_t n, int W, uint64_t* out, cudaStream_t s);
// repeated rows among 1024 rows sampled at a fixed stride (0 for distinct
// inputs); host-synchronising
uint32_t sample_duplicates(const uint64_t* rows, int64_t n, int W, cudaStream_t s);
// the same duplication sample on a byte matrix (ell = 64/128, 8-byte aligned
// rows), plus the largest top-byte share among up to 65536 sampled rows
uint32_t sample_duplicates_and_top(const uint8_t* vecs, int64_t n, int ell, cudaStream_t s,
                                   double* max_top_share);
// sorted rows u64[n][W] -> cells u64[n_c][W] (strictly increasing), popc[n_c],
// lcp[n_c] (leading equal bits with the next cell; 0xffff for the last),
// *n_cells (device u32).
void launch_dedupe(const uint64_t* sorted, int64_t n, int W, uint64_t* cells, uint32_t* popc,
                   uint16_t* lcp, uint32_t* n_cells, cudaStream_t s);
// 2 < W <= 32: the same from the UNSORTED rows keys[.][W] and the canonical
// order (row indices): gather + dedupe in one warp-cooperative pass.
bool gather_dedupe_ok(int W);
void launch_gather_dedupe(const uint64_t* keys, const uint32_t* order, int64_t n, int W,
                          uint64_t* cells, uint32_t* popc, uint16_t* lcp, uint32_t* n_cells,
                          cudaStream_t s);

// ---------------------------------------------------------------- a4/a5 layers + dictionary
// Prefix filter: per layer p a bitmap over the top (b_p + kFilterExtra) bits
// of its cells; a probe whose target prefix bit is clear cannot hit.
// default 7 (C5 probe: E=4 12.6 ms, 5 10.5, 6 8.9, 7 8.1, 8 7.9 ms on B200;
// the bitmap costs 2^(b+E) bits per layer, ~16-32 bits per cell at E=7);
// DictView.fextra holds the value in use (env CG_FILTER_EXTRA overrides).
constexpr int kFilterExtra = 7;

struct DictView {
  const uint64_t* keys;       // layer-major cell rows u64[n_c][W]
  const uint32_t* idx;        // canonical index of each layer-major row
  const uint32_t* layer_off;  // [ell + 2]
  const uint32_t* T;          // prefix index entries
  const uint64_t* tbase;      // [ell + 1] offset of layer p's prefix table in T
  const uint8_t* tbits;       // [ell + 1] prefix bits b_p (0 = no prefix index)
  const uint32_t* F;          // prefix filter bitmaps (u32 words)
  const uint64_t* fbase;      // [ell + 1] offset (in u32 words) of layer p's bitmap in F
  int W;
  int ell;
  int64_t n_cells;
  int fextra;                 // filter prefix = b_p + fextra bits
};

// layer_off[p] = first position of popcount p in sorted_popc (p in [0, ell+1]).
void launch_layer_offsets(const uint32_t* sorted_popc, int64_t nc, int ell, uint32_t* layer_off,
                          cudaStream_t s);
// out rows[j] = in rows[idx[j]] (W words per row); lcp_out[j] = lcp_in[idx[j]].
void launch_gather_rows(const uint64_t* in, const uint32_t* idx, int64_t n, int W, uint64_t* out,
                        cudaStream_t s);
void launch_gather_u16(const uint16_t* in, const uint32_t* idx, int64_t n, uint16_t* out,
                       cudaStream_t s);
// T entries and filter bits of every layer (sizes precomputed in
// tbase/tbits/fbase; F must be zeroed by the caller).
void launch_build_prefix_index(const DictView& d, const uint32_t* sorted_popc, uint32_t* T,
                               uint32_t* F, cudaStream_t s);

// ---------------------------------------------------------------- a6/a7 probes + edges
// For each layer-major cell j (popcount p), each bit k (<= lcp if lcp_prune)
// with V(k) = 0: look up V | e_k in layer p+1.  Hits are appended with
// warp-aggregated atomics as u64 (i << 32 | j) into edges[0..cap); *count
// gets the total (may exceed cap -> rerun with a bigger buffer).
void launch_probe(const DictView& d, const uint16_t* layer_lcp, const uint32_t* sorted_popc,
                  int lcp_prune, int64_t j_lo, int64_t j_hi, uint64_t* edges, uint64_t cap,
                  unsigned long long* count, unsigned long long* issued, cudaStream_t s);
// (i << 32 | j) -> u32 pair (i, j) little-endian.
void launch_rotate_edges(const uint64_t* in, int64_t m, uint64_t* out, cudaStream_t s);

// ---------------------------------------------------------------- global dictionary
// (probe_global.cu): one prefix index + filter over the canonical table; the
// probe writes the canonical edge list directly (tile order + look-back).
struct GlobalDict {
  const uint64_t* keys;  // canonical cells u64[n_c][W] (or a subsequence U of them)
  const uint16_t* lcp;   // unused (the probe derives lcp from the next row)
  const uint32_t* T;     // [2^b + 1]
  const uint32_t* F;     // 2^(b + fextra) bits
  int b;
  int fextra;
  int W;
  int ell;
  int64_t n_cells;             // rows of keys
  const uint32_t* src_pos = nullptr;  // subsequence mode: dictionary row of source q
  const uint32_t* idx = nullptr;      // subsequence mode: canonical index of each row
  // hash dictionary (CG_DICT_HASH; T/F unused): Z[ell] bit hashes, 2^lb
  // buckets of 4 (tag32 << 32 | row) slots, hv[n_cells] = h(cell)
  const uint64_t* Z = nullptr;
  const uint64_t* slots = nullptr;
  const uint64_t* hv = nullptr;
  int lb = 0;
};
// hash dictionary over a canonical table: Z u64[ell], slots u64[4 << lb]
// (zeroed here), hv u64[nc]
void build_hash_dict(const uint64_t* cells, int64_t nc, int W, int ell, int lb, uint64_t* Z,
                     uint64_t* slots, uint64_t* hv, cudaStream_t s);
void build_global_index(const uint64_t* cells, int64_t nc, int W, int b, int fextra, uint32_t* T,
                        uint32_t* F, cudaStream_t s);
// Each tile of 32 cells writes its sorted hits (i << 32 | j) as one block of
// out[0..cap) (reserved by atomicAdd on *total) and records tcnt[t] = count,
// tpos[t] = block position (~0 for an overflow tile).  Tiles whose hits
// overflow the warp buffer are listed in ovf (tile, -, count) and must be
// re-run in spill mode (spill != nullptr: unordered append to
// spill[0..spill_cap), *spill_n).
void launch_probe_global(const GlobalDict& g, int lcp_prune, int64_t i_lo, int64_t i_hi,
                         uint64_t* out, uint64_t cap, uint32_t* tcnt, uint64_t* tpos,
                         uint32_t* ticket, unsigned long long* total, unsigned long long* issued,
                         uint4* ovf, uint32_t* ovf_n, uint64_t* spill, uint64_t spill_cap,
                         unsigned long long* spill_n, cudaStream_t s,
                         const uint8_t* tile_sel = nullptr);
// overflow tiles (batched spill path): selection mask + per-tile counts
void launch_spill_select(const uint4* ovf, uint32_t novf, uint8_t* sel, uint32_t* scnt,
                         cudaStream_t s);
// sorted spilled hits -> out[toff[t] + q - sstart[t]] as (i, j) pairs
void launch_spill_place(const GlobalDict& g, const uint64_t* sorted, int64_t m, int64_t i_lo,
                        const uint64_t* toff, const uint64_t* sstart, uint64_t* out, cudaStream_t s);
// place every tile block at its canonical offset off[t] as (i, j) pairs
void launch_tile_copy(const uint64_t* scratch, const uint64_t* off, const uint64_t* pos,
                      const uint32_t* cnt, int64_t ntiles, uint64_t* out, cudaStream_t s);
int64_t probe_global_tiles(int64_t n);
int probe_global_tile_cells();
uint64_t probe_global_scratch_chunk();
int probe_global_tile_edge_cap();
// exclusive prefix sum of u32 in place (total < 2^32); edges.cu
void launch_scan_u32(uint32_t* v, int64_t n, cudaStream_t s);
// out[i] = sum of in[0..i) in 64 bits (edge offsets: m may exceed 2^32)
void launch_scan_u32_u64(const uint32_t* in, uint64_t* out, int64_t n, cudaStream_t s);

// ---------------------------------------------------------------- multi-GPU (dist.cu)
// hist[p * nblk + blk] = probe weight (1 + candidate bits) of the cells of
// popcount layer p in canonical block blk (2^blk_log2 cells); u32[(ell+1) * nblk]
void layer_block_weights(const uint64_t* cells, int64_t nc, int W, int ell, int lcp_prune,
                         int blk_log2, uint32_t* hist, cudaStream_t s);
// a rank's dictionary subsequence: sources = cells with p * nblk + blk in
// [c_lo, c_hi), kept = sources + layers [t_lo, t_hi]; U/idx (kept rows and
// their canonical indices), src_pos (row in U of each source).  Host-synchronising.
void select_rows(const uint64_t* cells, int64_t nc, int W, int blk_log2, int64_t c_lo, int64_t c_hi,
                 int t_lo, int t_hi, uint64_t* U, uint32_t* idx, uint32_t* src_pos,
                 int64_t* n_keep, int64_t* n_src, cudaStream_t s);
// G sorted, disjoint canonical edge lists (u32 pairs, list g at lists + g *
// stride, counts on the host) -> their merge into out
void merge_edge_lists(const uint64_t* lists, const int64_t* counts, int G, int64_t stride,
                      uint64_t* out, cudaStream_t s);

// ---------------------------------------------------------------- cg_query
void launch_query(const DictView& d, const uint64_t* q, int64_t nq, int32_t* self_idx,
                  int32_t* nbr_idx, cudaStream_t s);
void launch_query_global(const GlobalDict& g, const uint64_t* q, int64_t nq, int32_t* self_idx,
                         int32_t* nbr_idx, cudaStream_t s);

}  // namespace cgk
