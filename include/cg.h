/*
 * cg.h -- C ABI of the B200-native cell-graph builder (arXiv 1503.06029).
 *
 * Citations "P:n" are lines of the paper's text (reference PAPER.md); "G.."
 * are the readings listed in DESIGN.md.  No torch or CUDA-runtime types appear
 * in these signatures: pointers are plain (device unless stated), sizes are
 * int64, streams are passed as the opaque cudaStream_t handle value.
 *
 * The problem.  X = {x_0..x_{n-1}} is a multiset of n binary
 * vectors of length ell (a cell signature: bit i = 1 iff the sampled point
 * satisfies constraint c_i).  The cell graph G_X has the distinct
 * vectors as vertices and an edge between every pair at Hamming distance
 * exactly 1.  cg_build returns
 *   cells: the distinct vectors in canonical order -- lexicographic, bit 0
 *          first, 0 < 1 (the order "sort X" gives; pinned by
 *          Fig. 2; G1) -- and
 *   edges: every pair (i, j), i < j, of canonical indices with
 *          dist(cells[i], cells[j]) = 1, each pair once, ascending by (i, j)
 *          (G3, G4).
 *
 * Packed word format (cells, cg_query inputs): W = ceil(ell/64) u64 words per
 * vector, bit k in word k/64 at bit position 63-(k%64) (MSB-first), so that
 * comparing rows word by word as unsigned integers IS the canonical order.
 * The unused low bits of the last word are zero (G6).
 *
 * Errors: every entry point returns CG_OK (0) or a negative code; details
 * for the calling thread are in cg_last_error().  On error all output structs
 * are zeroed and nothing is leaked.
 */
#ifndef CG_H_
#define CG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* cg_stream_t; /* == cudaStream_t; NULL = legacy default stream */

enum {
  CG_OK = 0,
  CG_EINVAL = -1,   /* bad argument: n < 1, ell not in [1, CG_MAX_ELL], NULL or host pointer where a device pointer is required */
  CG_EINPUT = -2,   /* an input byte is not 0 or 1 (G5), or set pad bits in packed input */
  CG_ENOMEM = -3,   /* device (or pinned host) allocation failed */
  CG_ECUDA = -4,    /* a CUDA runtime error (kernel launch, sticky error) */
  CG_ETOOBIG = -5,  /* n >= 2^32 (cell indices are u32, G11); int32 index outputs with >= 2^31 cells */
  CG_EARCH = -6,    /* the current device is not sm_100 (B200) */
  CG_ENOTIMPL = -7  /* option not implemented */
};

#define CG_MAX_ELL 4096

/* Cell table: words[n_cells][words_per_cell] (device, owned by the caller,
 * release with cg_cells_free).  Rows strictly increasing. */
typedef struct {
  uint64_t* words;
  int64_t n_cells;
  int32_t ell;
  int32_t words_per_cell;
} cg_cells;

/* Edge list: ij[n_edges][2] u32 (device, owned by the caller, release with
 * cg_edges_free).  ij[2e] < ij[2e+1]; ascending by (i, j); each pair once. */
typedef struct {
  uint32_t* ij;
  int64_t n_edges;
} cg_edges;

/* Opaque, immutable dictionary over a cell table, built by cg_build_ex when
 * cg_opts.index_out is set: with CG_DICT_GLOBAL (or AUTO) a copy of the
 * canonical table plus its 2^b prefix index and prefix filter; with
 * CG_DICT_SORTED / CG_DICT_BSEARCH the popcount-layered arrays (DESIGN.md
 * a4-a5).  The dictionary replaces the paper's search tree (P:205-212,
 * P:276-281). */
typedef struct cg_index cg_index;

/* Per-stage device times (CUDA events on the build stream, microseconds)
 * and counters; filled when cg_opts.stats != NULL. */
typedef struct {
  double us_total, us_pack, us_sort, us_dedupe, us_layers, us_dict, us_probe, us_edges;
  int64_t n_in, n_cells, n_edges;
  int64_t logical_probes; /* n_cells * ell: the paper's one probe per (cell, bit) */
  int64_t issued_probes;  /* lookups actually issued (0->1 flips, <= lcp when pruning) */
  int32_t sort_passes;    /* radix passes executed by the cell sort */
  int32_t probe_reruns;   /* probe stage reruns because the edge buffer was too small */
  int64_t kernel_launches; /* CUDA kernels this library launched for the call */
  double us_host_alloc;    /* host time spent inside device allocation calls */
  int64_t n_allocs;        /* device allocations made for the call */
  double us_host_total;    /* host wall time of the whole call */
  double us_host_setup;    /* host wall time before the first stage event */
  int64_t dict_bytes;      /* device bytes of the dictionary's index structures (prefix
                              index T + filter F; the cell table itself not counted) */
  int64_t dict_cells;      /* cells the dictionary holds (n_cells, or a rank's share) */
} cg_stats;

enum {
  CG_DICT_SORTED = 0,  /* popcount layers: per-layer sorted array + 2^b prefix index + filter */
  CG_DICT_BSEARCH = 1, /* popcount layers, plain per-layer binary search (no prefix index) */
  CG_DICT_GLOBAL = 2,  /* one prefix index + filter over the canonical table; the probe
                          writes the edge list in canonical order (no edge sort); its
                          cg_index holds a copy of the table. */
  CG_DICT_HASH = 3,    /* open-addressed hash table over the canonical table (h = XOR of
                          per-bit 64-bit keys, so a flip is h ^ Z[k]; 4-slot 32-byte
                          buckets, load 1/2, every tag hit verified on the full row):
                          the north star's alternative dictionary (P:205 / P:276-281
                          replace the paper's tree), kept for the ncu A/B.  Same
                          output as CG_DICT_GLOBAL; keeps no cg_index (index_out with
                          it is CG_EINVAL). */
  CG_DICT_AUTO = 4     /* default of cg_opts_init: CG_DICT_HASH when the rows are long
                          (ell > 128) and heavily duplicated (n >= 4 n_c, arrangement
                          signatures) and no index is requested, else
                          CG_DICT_GLOBAL (DESIGN.md section 6 A/B) */
};

typedef struct {
  cg_stream_t stream;   /* stream all work is ordered on (NULL = legacy default) */
  int32_t dict_kind;    /* CG_DICT_* */
  int32_t lcp_prune;    /* 1: probe bit k only if k <= lcp(V_i, V_{i+1}) (exact, DESIGN a6) */
  int32_t bucket_log2;  /* prefix index: target log2(cells per bucket); -1 = default (2) */
  int32_t sort_kind;    /* 0 = auto (n <= 2048 and ell <= 256: the whole build in one CTA;
                           else MSD prefix buckets + shared-memory sort for ell <= 128,
                           prefix/LSD sorts beyond, full LSD fallback; 2^18 < n <= 2^26
                           rows of ell = 64 or 128 bytes: the sweep path, the pack kernel
                           doing the first MSD partition -- below 2^24 rows unless a
                           1024-row sample shows heavy duplication), 1 = full LSD only,
                           2 = auto without the one-CTA small path, 3 = auto without the
                           sweep path, 4 = auto with the sweep path whatever the sample */
  cg_index** index_out; /* if non-NULL, receives the dictionary (release with cg_index_free) */
  cg_stats* stats;      /* if non-NULL, stage times and counters */
  int32_t filter_extra; /* prefix filter resolution: b + filter_extra prefix bits per filter
                           slot, in [0, 8]; -1 = default (5 global, 7 layered).  Changes
                           only how many probes reach a bucket search, never the result */
  int32_t reserved0;    /* must be 0 */
  int64_t edge_cap;     /* initial capacity (edges) of the probe's hit buffer; 0 = default
                           (4 per probed cell).  A larger m re-runs the probe at the exact
                           size; only speed depends on it */
} cg_opts;

/* Fill *o with defaults: stream NULL, CG_DICT_AUTO, lcp_prune 1,
 * bucket_log2 -1, no index, no stats, filter_extra -1, edge_cap 0. */
void cg_opts_init(cg_opts* o);

/* Build the cell graph of vecs = uint8[n][ell] (device, row-major,
 * contiguous; byte k of row r is bit k of x_r and must be 0 or 1, G5).
 * Input is borrowed read-only.  Blocks until cells/edges are complete (it
 * must learn n_cells and n_edges).  Errors: CG_EINVAL (n < 1, ell out of
 * range, NULL/host vecs), CG_ETOOBIG (n >= 2^32), CG_EINPUT (a byte > 1),
 * CG_ENOMEM, CG_ECUDA. */
int cg_build(const uint8_t* vecs, int64_t n, int32_t ell, cg_cells* cells, cg_edges* edges);

/* As cg_build with options (stream, dictionary kind, index and stats out). */
int cg_build_ex(const uint8_t* vecs, int64_t n, int32_t ell, const cg_opts* o, cg_cells* cells,
                cg_edges* edges);

/* As cg_build_ex from already packed vectors words = u64[n][ceil(ell/64)]
 * (device) in the packed word format; set pad bits -> CG_EINPUT. */
int cg_build_packed_ex(const uint64_t* words, int64_t n, int32_t ell, const cg_opts* o,
                       cg_cells* cells, cg_edges* edges);

/* ---- f1: cell signatures computed on the device ----
 * "the i-th bit of v_P is 1 iff P satisfies the inequality c_i" for
 * sampled points P.  Constraint c_k is the half-space
 * a_k . p + b_k >= 0 in R^dim (a tie counts as satisfied, DESIGN G12).
 *   points = f64[n][dim] (device, row-major), dim in [1, 16];
 *   planes = f64[ell][dim + 1] (device), row k = (a_k0 .. a_k(dim-1), b_k).
 * The value is evaluated in one fixed IEEE-754 order, v = b_k;
 * v = fma(a_kt, p_t, v) for t = 0 .. dim-1 (round to nearest, DESIGN G21),
 * so results are bit-reproducible on any IEEE machine.  Inputs are borrowed.
 * Every coordinate and coefficient must be finite with |x| <= 2^60 (then no
 * value can overflow).  Errors: CG_EINVAL (NULL/host pointers, n < 1, ell or
 * dim out of range), CG_EINPUT (an input NaN, infinite or above 2^60). */

/* Signatures only: words = u64[n][ceil(ell/64)] (device, caller-allocated),
 * the packed format of cg_cells.  Blocks until done (the error flag). */
int cg_signatures(const double* points, int64_t n, int32_t dim, const double* planes,
                  int32_t ell, uint64_t* words, cg_stream_t stream);

/* As cg_build_ex, with the signatures computed on the device and packed in
 * the same kernel (the n*ell-byte signature matrix is never formed). */
int cg_build_points(const double* points, int64_t n, int32_t dim, const double* planes,
                    int32_t ell, const cg_opts* o, cg_cells* cells, cg_edges* edges);

/* ---- f2: incremental insertion ----------------------
 * The generator "generates (and possibly accumulates)" samples: extend
 * the cell graph of an accumulated input (its canonical table cells =
 * u64[n_cells][W] and edge list edges = u32[n_edges][2], device, e.g. the
 * outputs of cg_build) by new samples vecs = uint8[n_new][ell] (device, 0/1
 * bytes).  *cells_out / *edges_out receive the cell graph of the union of
 * both multisets -- byte-identical to cg_build on the concatenated input --
 * computed from the batch alone plus flip lookups into the existing table
 * (free with cg_cells_free / cg_edges_free).  Blocks.  Errors: as cg_build
 * (the batch), CG_EINVAL (NULL/host pointers, sizes), CG_ETOOBIG.  The
 * existing table and edges must be canonical (unchecked). */
int cg_insert(const uint64_t* cells, int64_t n_cells, const uint32_t* edges, int64_t n_edges,
              int32_t ell, const uint8_t* vecs, int64_t n_new, const cg_opts* o,
              cg_cells* cells_out, cg_edges* edges_out);

/* ---- f3: the all-pairs methods ----------------------
 * Distance-1 pairs of a cell table by comparing pairs: the naive method
 * with `anchors` = 0, Alg. 1-2 with `anchors` = h in
 * [1, 8]: d(x_a, x_j) precomputed for the first h cells, a pair skipped when
 * |d(x_a, x_i) - d(x_a, x_j)| > 1 for some anchor (the triangle inequality,
 * P:46; the sound form of the guard, DESIGN G15).  cells = u64[n_cells][W]
 * (device, distinct rows, e.g. cg_build's table); *edges receives the
 * canonical list (i < j, ascending; free with cg_edges_free) -- equal to
 * cg_build's edge list for a canonical table, hence an independent in-GPU
 * cross-check.  *pairs_compared (optional) = pairs that passed the anchor
 * test.  O(n^2) work: meant for n up to ~10^6.  Blocks.  Errors: CG_EINVAL,
 * CG_ETOOBIG, CG_ENOMEM. */
int cg_allpairs(const uint64_t* cells, int64_t n_cells, int32_t ell, int32_t anchors,
                cg_edges* edges, int64_t* pairs_compared, cg_stream_t stream);

/* ---- f4: path queries on G_X ----------------------
 * The graph is built so that one can "find a path in such a graph" (P:20,
 * P:57); GPU graph traversal is the paper's stated next step. */

/* CSR of the undirected cell graph from the canonical edge list of
 * cg_build (edges = u32[n_edges][2], (i, j) with i < j, ascending; device).
 * Outputs (device, caller-allocated): row_ptr = u64[n_cells + 1], col =
 * u32[2 * n_edges]; the neighbours of v are col[row_ptr[v] .. row_ptr[v+1])
 * in ascending order.  Blocks until done.  Errors: CG_EINVAL (NULL/host
 * pointers, n_cells < 1, n_edges < 0), CG_ETOOBIG (n_cells >= 2^32).  The
 * edge list must be canonical with indices < n_cells (unchecked). */
int cg_csr(const uint32_t* edges, int64_t n_edges, int64_t n_cells, uint64_t* row_ptr,
           uint32_t* col, cg_stream_t stream);

/* Breadth-first search from `source` over a CSR of cg_csr: dist = i32[n_cells]
 * (device) receives the number of edges on a shortest path (-1: not
 * reachable); parent (optional, i32[n_cells]) the canonical BFS tree: the
 * smallest neighbour one step closer to the source (-1 for the source and
 * unreachable cells), so a path to any cell is read back by following it.
 * *eccentricity (optional, host) = the largest finite distance.  Blocks
 * (one host synchronisation per level).  Errors: CG_EINVAL (NULL/host
 * pointers, source out of range), CG_ETOOBIG. */
int cg_bfs(const uint64_t* row_ptr, const uint32_t* col, int64_t n_cells, int64_t source,
           int32_t* dist, int32_t* parent, int32_t* eccentricity, cg_stream_t stream);

/* End-to-end entry with HOST buffers.  h_vecs = uint8[n][ell] in host memory
 * (pinned for full PCIe speed, pageable accepted).  The library copies it to
 * the device (chunked, overlapped with the pack kernel), builds, and copies
 * the results back into host arrays it allocates (pinned; release with
 * cg_host_free).  *h_cells = u64[*n_cells][W], *h_edges = u32[*n_edges][2].
 * Same error codes as cg_build_ex (CG_EINVAL for a NULL host pointer). */
int cg_build_host(const uint8_t* h_vecs, int64_t n, int32_t ell, const cg_opts* o,
                  uint64_t** h_cells, int64_t* n_cells, uint32_t** h_edges, int64_t* n_edges);
void cg_host_free(void* p);

/* Streaming query against a built index: Alg. 4's lookups for
 * a batch of vectors -- the vector itself and each of its ell single-bit
 * flips x XOR e_k are searched in the dictionary.
 * q = u64[nq][W] packed cells (device; pad bits ignored, G19).  Writes
 * (device, caller-allocated)
 *   self_idx[r]        = canonical index of q_r, or -1 if q_r is not a cell;
 *   nbr_idx[r*ell + k] = canonical index of q_r with bit k negated, or -1.
 * Asynchronous on stream s (no host sync); nq == 0 is a no-op.
 * Errors: CG_EINVAL (NULL index, NULL pointers with nq > 0, nq < 0),
 * CG_ETOOBIG (the index holds >= 2^31 cells: indices would not fit int32). */
int cg_query(const cg_index* idx, const uint64_t* q, int64_t nq, int32_t* self_idx,
             int32_t* nbr_idx, cg_stream_t s);

/* Index metadata (host). */
int cg_index_info(const cg_index* idx, int64_t* n_cells, int32_t* ell);

/* Allocator hook for every device allocation the library makes (outputs and
 * workspace).  alloc(bytes, stream, ctx) returns a device pointer or NULL;
 * dealloc(ptr, stream, ctx).  Passing NULLs restores the default
 * (cudaMallocAsync / cudaFreeAsync on the stream's device memory pool).
 * Must not be changed while outputs allocated by the previous allocator are
 * alive. */
int cg_set_allocator(void* (*alloc)(size_t, cg_stream_t, void*),
                     void (*dealloc)(void*, cg_stream_t, void*), void* ctx);

void cg_cells_free(cg_cells* c); /* frees c->words, zeroes *c; NULL-safe */
void cg_edges_free(cg_edges* e); /* frees e->ij, zeroes *e; NULL-safe */
void cg_index_free(cg_index* idx);

const char* cg_strerror(int code);
const char* cg_last_error(void); /* thread-local detail of the last failure */
int cg_version(void);            /* (major << 16) | minor */
/* CUDA kernels this library has launched in the process so far (all calls,
 * all threads); the difference across a region counts its launches. */
int64_t cg_kernel_launches(void);

/* ---- distributed phases (row e; one process per GPU, the caller runs the
 * NCCL collectives between them) --------------------
 * The paper builds on one GPU; the multi-GPU split follows from the
 * structure of the problem: a 0->1 flip raises the popcount by one (P:93,
 * P:103), so the cells of popcount layer p have all their i < j neighbours in
 * layer p+1, and the flip queries are sharded by popcount layer.
 *   1. cg_dist_local: each rank's rows -> its sorted unique run, split into
 *      2^chunk_bits prefix chunks;
 *   2. per chunk (in prefix order): all-gather of the ranks' pieces, then
 *      cg_dist_merge_chunk appends their merge to the replicated table (the
 *      all-gather of chunk c+1 overlaps the merge of chunk c);
 *   3. cg_dist_probe: the rank probes its share of the (layer, block) order
 *      with a dictionary over its cells and their target layer only;
 *   4. all-gather of the edge lists, cg_dist_finalize merges them. */

/* Phase 1: pack + sort + dedupe this rank's rows (vecs = uint8[n_local][ell],
 * device, n_local >= 1): *run = its sorted unique rows (cg_cells; free with
 * cg_cells_free).  chunk_off = host int64[2^chunk_bits + 1] receives the row
 * offsets of the prefix chunks: chunk c = the rows whose top chunk_bits bits
 * equal c (chunk_bits in [0, 8]).  Errors as cg_build, CG_EINVAL for a bad
 * chunk_bits / NULL chunk_off. */
int cg_dist_local(const uint8_t* vecs, int64_t n_local, int32_t ell, const cg_opts* o,
                  int32_t chunk_bits, cg_cells* run, int64_t* chunk_off);

/* Phase 2: merge chunk c of every rank's run -- G sorted unique pieces in the
 * device buffer pieces = u64[G][stride][W], piece g holding counts[g] (host)
 * rows, all with the same top chunk_bits bits and above every row already in
 * the table -- and append the sorted unique union at table + (*n_table)*W;
 * *n_table (host) is advanced.  table = u64[table_cap][W], caller-allocated
 * (device).  Called once per chunk in prefix order, the result is the
 * canonical table (G1), identical on every rank.  Errors: CG_EINVAL (NULL,
 * counts > stride, capacity), CG_ETOOBIG (>= 2^32 rows). */
int cg_dist_merge_chunk(const uint64_t* pieces, const int64_t* counts, int32_t G, int64_t stride,
                        int32_t ell, int32_t chunk_bits, const cg_opts* o, uint64_t* table,
                        int64_t table_cap, int64_t* n_table);

/* Phase 3: rank `rank` of G probes its share of the flip queries over the
 * canonical table (device u64[n_cells][W]): the cells of a contiguous range of
 * the (popcount layer, block of 2^16 canonical cells) order cut at equal probe
 * weight (1 + candidate bits per cell).  Its dictionary (prefix index +
 * filter, CG_DICT_GLOBAL) holds only those cells and the layers one above
 * them (cg_stats.dict_cells / dict_bytes report its size).  *local_edges =
 * this rank's edges (canonical indices, i < j, ascending; free with
 * cg_edges_free); the ranks' lists are disjoint and cover E.  G = 1 probes
 * everything.  Errors: CG_EINVAL (NULL, G not in [1, 64], rank), CG_ETOOBIG. */
int cg_dist_probe(const uint64_t* table, int64_t n_cells, int32_t ell, int32_t G, int32_t rank,
                  const cg_opts* o, cg_edges* local_edges);

/* Phase 4: merge G gathered canonical, disjoint edge lists (device buffer
 * u32[G][stride][2], list g holding counts[g] (host) pairs) into the
 * canonical edge list (G-way merge, G <= 64). */
int cg_dist_finalize(const uint32_t* gathered, const int64_t* counts, int32_t G, int64_t stride,
                     const cg_opts* o, cg_edges* edges);

#ifdef __cplusplus
}
#endif
#endif /* CG_H_ */
