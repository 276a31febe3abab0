/*
 * cg_oracle.cpp -- CPU ORACLE for the cell-graph construction path of
 * Kaczmarski, Rzazewski, Wolant, "Massively Parallel Construction of the Cell
 * Graph" (arXiv 1503.06029).  Citations "P:n" are lines of PAPER.md.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  It
 * shares no code, header, table or helper with the CUDA product path
 * (paper_1503_06029_b200/csrc), and the product path never calls it.
 *
 * What it computes is the plain definition of the result (the method is
 * exact, so the oracle is the definition written out, not a replica):
 *   X      = multiset of n binary vectors of length ell
 *   V      = the distinct elements of X in canonical order: lexicographic,
 *            bit 0 compared first, 0 < 1                            (DESIGN G1)
 *   E      = { (i,j) : 0 <= i < j < |V|, dist(V_i,V_j) = 1 }, ascending (G3,G4)
 *
 * Two independent implementations live here:
 *   ORACLE-A  oracle_build : std::set of packed keys + single-bit-flip lookup
 *             (the flip enumeration of Alg. 4, with the dictionary
 *             being a std::set instead of the paper's tree).
 *   ORACLE-B  oracle_brute : unpacked byte vectors, std::sort + std::unique,
 *             then all-pairs Hamming distance (the naive method).
 *   plus      oracle_query : self/neighbour lookup of query vectors.
 *   and       oracle_csr / oracle_bfs : adjacency lists of G_X and breadth-
 *             first distances from a source (the f4 row: "find a path in
 *             such a graph"); parent = the smallest neighbour
 *             one step closer to the source (DESIGN G22).
 *   and       oracle_signatures : the cell signature of sampled points (the
 *             f1 row): bit k of point P is 1 iff P satisfies constraint c_k
 *             (P:92), c_k being the half-space a_k . p + b_k >= 0 (a tie is
 *             satisfied, DESIGN G12), evaluated as v = b_k, then
 *             v = fma(a_kt, p_t, v) for t = 0..dim-1 (DESIGN G21).
 *
 * Output word format of oracle_build / oracle_brute (the C-ABI's format):
 *   W = ceil(ell/64) little-endian u64 words per cell; bit k of the vector is
 *   bit 63-(k%64) of word k/64 (MSB-first), unused low bits of the last word 0.
 *   Edges are u32 pairs (i, j), i < j, ascending by (i, j).
 *
 * Error codes (same meaning as the C ABI, DESIGN G5/G10):
 *   0 ok, -1 EINVAL (n < 1, ell not in [1,4096], null pointer), -2 EINPUT
 *   (a byte not in {0,1}), -3 ENOMEM, -5 ETOOBIG (more than 2^32-1 cells),
 *   -9 self-check failure (an edge not found from both endpoints).
 */
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <new>
#include <set>
#include <thread>
#include <utility>
#include <vector>

namespace {

constexpr int kOK = 0, kEINVAL = -1, kEINPUT = -2, kENOMEM = -3, kETOOBIG = -5, kESELF = -9;
constexpr int kMaxEll = 4096;

using Key = std::vector<uint64_t>;  // std::vector's operator< is lexicographic = canonical order

double now_s() {
  using namespace std::chrono;
  return duration<double>(steady_clock::now().time_since_epoch()).count();
}

int words_for(int ell) { return (ell + 63) / 64; }

// Pack one row of bytes (each 0 or 1) MSB-first: bit k -> word k/64, bit 63-(k%64).
// Returns false when a byte is not 0/1 (bit i is 1 iff the constraint holds).
bool pack_row(const uint8_t* row, int ell, Key& out) {
  out.assign(words_for(ell), 0);
  for (int k = 0; k < ell; ++k) {
    uint8_t b = row[k];
    if (b > 1) return false;
    if (b) out[k / 64] |= uint64_t(1) << (63 - (k % 64));
  }
  return true;
}

bool get_bit(const Key& x, int k) { return (x[k / 64] >> (63 - (k % 64))) & 1; }

void flip_bit(Key& x, int k) { x[k / 64] ^= uint64_t(1) << (63 - (k % 64)); }

int validate(const void* p, int64_t n, int ell) {
  if (!p || n < 1 || ell < 1 || ell > kMaxEll) return kEINVAL;
  return kOK;
}

template <class T>
T* copy_out(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(std::max<size_t>(1, v.size() * sizeof(T))));
  if (p && !v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
  return p;
}

// ORACLE-A core, from already packed keys.
int build_from_keys(std::vector<Key>& keys, int ell, int nthreads, int self_check,
                    uint64_t** cells_out, int64_t* n_cells, uint32_t** edges_out,
                    int64_t* n_edges, double* t) {
  const int W = words_for(ell);
  double t0 = now_s();
  // Step 1 ("sorting ... we also remove all duplicates"): a set.
  std::set<Key> S;
  for (auto& k : keys) S.insert(std::move(k));
  keys.clear();
  keys.shrink_to_fit();
  if (S.size() > 0xFFFFFFFFull) return kETOOBIG;
  // Walk the set in order: V_i (canonical index i).
  std::vector<Key> V(S.begin(), S.end());
  S.clear();
  double t1 = now_s();
  // Step 2 (Alg. 4): for every cell and every bit k, the candidate
  // x' = x with bit k negated; an edge (i, index(x')) is kept when x' is a
  // cell and i < index(x') (single emission, DESIGN G3).  Membership and the
  // index of x' come from a binary search of the sorted table V.
  const int64_t nc = static_cast<int64_t>(V.size());
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  std::vector<std::vector<std::pair<uint32_t, uint32_t>>> part(nthreads), back(nthreads);
  std::vector<int> bad(nthreads, 0);
  auto worker = [&](int tid) {
    int64_t lo = nc * tid / nthreads, hi = nc * (tid + 1) / nthreads;
    auto& out = part[tid];
    Key y;
    for (int64_t i = lo; i < hi; ++i) {
      for (int k = 0; k < ell; ++k) {
        y = V[i];
        flip_bit(y, k);
        auto it = std::lower_bound(V.begin(), V.end(), y);
        if (it == V.end() || *it != y) continue;
        int64_t j = it - V.begin();
        if (i < j) {
          out.emplace_back(static_cast<uint32_t>(i), static_cast<uint32_t>(j));
          // x < x with bit k negated  <=>  x(k) = 0 (DESIGN G3)
          if (self_check && get_bit(V[i], k)) bad[tid] = 1;
        } else if (self_check) {
          back[tid].emplace_back(static_cast<uint32_t>(j), static_cast<uint32_t>(i));
          if (!get_bit(V[i], k)) bad[tid] = 1;
        }
      }
    }
  };
  if (nthreads == 1) {
    worker(0);
  } else {
    std::vector<std::thread> th;
    for (int tid = 0; tid < nthreads; ++tid) th.emplace_back(worker, tid);
    for (auto& x : th) x.join();
  }
  for (int b : bad)
    if (b) return kESELF;
  std::vector<std::pair<uint32_t, uint32_t>> E;
  for (auto& p : part) E.insert(E.end(), p.begin(), p.end());
  double t2 = now_s();
  std::sort(E.begin(), E.end());  // ascending (i, j), DESIGN G4
  if (self_check) {
    // Every edge must be found from both endpoints (Alg. 4 outputs (x, x')
    // from each end): the downward finds, reoriented, equal E.
    std::vector<std::pair<uint32_t, uint32_t>> B;
    for (auto& p : back) B.insert(B.end(), p.begin(), p.end());
    std::sort(B.begin(), B.end());
    if (B != E) return kESELF;
  }
  double t3 = now_s();

  std::vector<uint64_t> cells(static_cast<size_t>(nc) * W);
  for (int64_t i = 0; i < nc; ++i)
    for (int w = 0; w < W; ++w) cells[i * W + w] = V[i][w];
  std::vector<uint32_t> ed(E.size() * 2);
  for (size_t e = 0; e < E.size(); ++e) {
    ed[2 * e] = E[e].first;
    ed[2 * e + 1] = E[e].second;
  }
  *cells_out = copy_out(cells);
  *edges_out = copy_out(ed);
  if (!*cells_out || !*edges_out) return kENOMEM;
  *n_cells = nc;
  *n_edges = static_cast<int64_t>(E.size());
  if (t) {
    t[0] = t1 - t0;  // set build + walk
    t[1] = t2 - t1;  // flip lookups
    t[2] = t3 - t2;  // edge sort
  }
  return kOK;
}

}  // namespace

extern "C" {

/* ORACLE-A over uint8[n][ell] bytes.  t (optional, 4 doubles): pack, set,
 * lookups, sort seconds. */
int oracle_build(const uint8_t* bytes, int64_t n, int32_t ell, int32_t nthreads,
                 int32_t self_check, uint64_t** cells_out, int64_t* n_cells,
                 uint32_t** edges_out, int64_t* n_edges, double* t) {
  *cells_out = nullptr;
  *edges_out = nullptr;
  *n_cells = 0;
  *n_edges = 0;
  int rc = validate(bytes, n, ell);
  if (rc) return rc;
  double t0 = now_s();
  std::vector<Key> keys;
  try {
    keys.resize(static_cast<size_t>(n));
  } catch (const std::bad_alloc&) {
    return kENOMEM;
  }
  for (int64_t r = 0; r < n; ++r)
    if (!pack_row(bytes + r * static_cast<int64_t>(ell), ell, keys[r])) return kEINPUT;
  double tt[3] = {0, 0, 0};
  double t1 = now_s();
  rc = build_from_keys(keys, ell, nthreads, self_check, cells_out, n_cells, edges_out,
                       n_edges, tt);
  if (t) {
    t[0] = t1 - t0;
    t[1] = tt[0];
    t[2] = tt[1];
    t[3] = tt[2];
  }
  return rc;
}

/* ORACLE-A over already packed MSB-first words u64[n][ceil(ell/64)] (pad bits
 * must be zero; -2 otherwise). */
int oracle_build_packed(const uint64_t* words, int64_t n, int32_t ell, int32_t nthreads,
                        uint64_t** cells_out, int64_t* n_cells, uint32_t** edges_out,
                        int64_t* n_edges, double* t) {
  *cells_out = nullptr;
  *edges_out = nullptr;
  *n_cells = 0;
  *n_edges = 0;
  int rc = validate(words, n, ell);
  if (rc) return rc;
  const int W = words_for(ell);
  const uint64_t padmask = (ell % 64) ? (~uint64_t(0) >> (ell % 64)) : 0;
  double t0 = now_s();
  std::vector<Key> keys(static_cast<size_t>(n));
  for (int64_t r = 0; r < n; ++r) {
    keys[r].assign(words + r * W, words + (r + 1) * W);
    if (keys[r][W - 1] & padmask) return kEINPUT;
  }
  double tt[3] = {0, 0, 0};
  double t1 = now_s();
  rc = build_from_keys(keys, ell, nthreads, 0, cells_out, n_cells, edges_out, n_edges, tt);
  if (t) {
    t[0] = t1 - t0;
    t[1] = tt[0];
    t[2] = tt[1];
    t[3] = tt[2];
  }
  return rc;
}

/* ORACLE-B: the naive O(n^2 * ell) method of P:119, written independently of
 * ORACLE-A.  Vectors stay unpacked (one byte per bit); canonical order is the
 * lexicographic order of those byte strings (bit 0 first, 0 < 1); duplicates
 * go with std::unique; every pair i < j is compared bit by bit.  Only the
 * final output is written in the packed word format. */
int oracle_brute(const uint8_t* bytes, int64_t n, int32_t ell, int32_t nthreads,
                 uint64_t** cells_out, int64_t* n_cells, uint32_t** edges_out,
                 int64_t* n_edges) {
  *cells_out = nullptr;
  *edges_out = nullptr;
  *n_cells = 0;
  *n_edges = 0;
  int rc = validate(bytes, n, ell);
  if (rc) return rc;
  std::vector<std::vector<uint8_t>> rows(static_cast<size_t>(n));
  for (int64_t r = 0; r < n; ++r) {
    const uint8_t* p = bytes + r * static_cast<int64_t>(ell);
    for (int k = 0; k < ell; ++k)
      if (p[k] > 1) return kEINPUT;
    rows[r].assign(p, p + ell);
  }
  std::sort(rows.begin(), rows.end());
  rows.erase(std::unique(rows.begin(), rows.end()), rows.end());
  const int64_t nc = static_cast<int64_t>(rows.size());
  if (nc > 0xFFFFFFFFll) return kETOOBIG;
  // A second, differently laid out packing (LSB-first within 64-bit words)
  // used only to count differing positions quickly: popcount(x ^ y) is the
  // number of positions where the bytes differ, independent of bit layout.
  const int W = words_for(ell);
  std::vector<uint64_t> lsb(static_cast<size_t>(nc) * W, 0);
  for (int64_t i = 0; i < nc; ++i)
    for (int k = 0; k < ell; ++k)
      if (rows[i][k]) lsb[i * W + k / 64] |= uint64_t(1) << (k % 64);
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  std::vector<std::vector<std::pair<uint32_t, uint32_t>>> part(nthreads);
  auto worker = [&](int tid) {
    for (int64_t i = tid; i < nc; i += nthreads) {
      const uint64_t* a = &lsb[i * W];
      for (int64_t j = i + 1; j < nc; ++j) {
        const uint64_t* b = &lsb[j * W];
        int d = 0;
        for (int w = 0; w < W && d < 2; ++w) d += __builtin_popcountll(a[w] ^ b[w]);
        if (d == 1) part[tid].emplace_back(static_cast<uint32_t>(i), static_cast<uint32_t>(j));
      }
    }
  };
  if (nthreads == 1) {
    worker(0);
  } else {
    std::vector<std::thread> th;
    for (int tid = 0; tid < nthreads; ++tid) th.emplace_back(worker, tid);
    for (auto& x : th) x.join();
  }
  std::vector<std::pair<uint32_t, uint32_t>> E;
  for (auto& p : part) E.insert(E.end(), p.begin(), p.end());
  std::sort(E.begin(), E.end());
  std::vector<uint64_t> cells(static_cast<size_t>(nc) * W, 0);
  for (int64_t i = 0; i < nc; ++i)
    for (int k = 0; k < ell; ++k)
      if (rows[i][k]) cells[i * W + k / 64] |= uint64_t(1) << (63 - (k % 64));
  std::vector<uint32_t> ed(E.size() * 2);
  for (size_t e = 0; e < E.size(); ++e) {
    ed[2 * e] = E[e].first;
    ed[2 * e + 1] = E[e].second;
  }
  *cells_out = copy_out(cells);
  *edges_out = copy_out(ed);
  if (!*cells_out || !*edges_out) return kENOMEM;
  *n_cells = nc;
  *n_edges = static_cast<int64_t>(E.size());
  return kOK;
}

/* Query oracle: given the canonical cell table (u64[nc][W], strictly
 * increasing) and nq packed queries, write self_idx[q] = index of q in the
 * table or -1, and nbr_idx[q*ell + k] = index of (q with bit k negated) or -1.
 * Pad bits of the queries are ignored (DESIGN G19). */
int oracle_query(const uint64_t* cells, int64_t nc, int32_t ell, const uint64_t* q,
                 int64_t nq, int32_t* self_idx, int32_t* nbr_idx) {
  if (!cells || nc < 1 || ell < 1 || ell > kMaxEll || (nq > 0 && (!q || !self_idx || !nbr_idx)))
    return kEINVAL;
  const int W = words_for(ell);
  const uint64_t padmask = (ell % 64) ? (~uint64_t(0) >> (ell % 64)) : 0;
  std::vector<Key> V(static_cast<size_t>(nc));
  for (int64_t i = 0; i < nc; ++i) V[i].assign(cells + i * W, cells + (i + 1) * W);
  auto find = [&](const Key& y) -> int32_t {
    auto it = std::lower_bound(V.begin(), V.end(), y);
    if (it == V.end() || *it != y) return -1;
    return static_cast<int32_t>(it - V.begin());
  };
  Key x, y;
  for (int64_t r = 0; r < nq; ++r) {
    x.assign(q + r * W, q + (r + 1) * W);
    x[W - 1] &= ~padmask;
    self_idx[r] = find(x);
    for (int k = 0; k < ell; ++k) {
      y = x;
      flip_bit(y, k);
      nbr_idx[r * ell + k] = find(y);
    }
  }
  return kOK;
}

// f1: signatures of n points (row-major f64[n][dim]) against ell half-spaces
// (f64[ell][dim+1], row k = a_k0 .. a_k(dim-1), b_k) as bytes u8[n][ell]
// (the oracle's vector input form).  Returns 0, or -1 (bad sizes or
// NULL), -2 (an input not finite or above 2^60 in magnitude, or a
// non-finite value).
int oracle_signatures(const double* points, int64_t n, int32_t dim, const double* planes,
                      int32_t ell, uint8_t* out) {
  if (!points || !planes || !out || n < 1 || dim < 1 || dim > 16 || ell < 1 || ell > kMaxEll)
    return kEINVAL;
  int rc = kOK;
  // inputs must be finite with magnitude <= 2^60 (the C ABI's contract)
  const double kMaxMag = std::ldexp(1.0, 60);
  for (int64_t i = 0; i < n * dim; ++i)
    if (!(std::fabs(points[i]) <= kMaxMag)) rc = kEINPUT;
  for (int64_t i = 0; i < int64_t(ell) * (dim + 1); ++i)
    if (!(std::fabs(planes[i]) <= kMaxMag)) rc = kEINPUT;
  for (int64_t r = 0; r < n; ++r) {
    const double* p = points + r * dim;
    for (int k = 0; k < ell; ++k) {
      const double* a = planes + int64_t(k) * (dim + 1);
      double v = a[dim];
      for (int t = 0; t < dim; ++t) v = std::fma(a[t], p[t], v);
      if (!std::isfinite(v)) rc = kEINPUT;
      out[r * ell + k] = v >= 0.0 ? 1 : 0;
    }
  }
  return rc;
}

// f4: adjacency of the undirected graph with vertices 0..nv-1 and edge list
// u32[m][2] -> row_ptr u64[nv+1], col u32[2m] (each list ascending).
int oracle_csr(const uint32_t* edges, int64_t m, int64_t nv, uint64_t* row_ptr, uint32_t* col) {
  if (nv < 1 || m < 0 || !row_ptr || (m > 0 && (!edges || !col))) return kEINVAL;
  std::vector<std::vector<uint32_t>> adj(static_cast<size_t>(nv));
  for (int64_t e = 0; e < m; ++e) {
    const uint32_t a = edges[2 * e], b = edges[2 * e + 1];
    if (a >= nv || b >= nv) return kEINVAL;
    adj[a].push_back(b);
    adj[b].push_back(a);
  }
  uint64_t at = 0;
  for (int64_t v = 0; v < nv; ++v) {
    std::sort(adj[v].begin(), adj[v].end());
    row_ptr[v] = at;
    for (uint32_t w : adj[v]) col[at++] = w;
  }
  row_ptr[nv] = at;
  return kOK;
}

// f4: BFS distances from src over the CSR (queue order is irrelevant to the
// distances); parent[v] = smallest neighbour u with dist[u] = dist[v] - 1.
int oracle_bfs(const uint64_t* row_ptr, const uint32_t* col, int64_t nv, int64_t src,
               int32_t* dist, int32_t* parent) {
  if (nv < 1 || src < 0 || src >= nv || !row_ptr || !dist || !parent) return kEINVAL;
  for (int64_t v = 0; v < nv; ++v) dist[v] = -1;
  std::deque<uint32_t> q;
  dist[src] = 0;
  q.push_back(uint32_t(src));
  while (!q.empty()) {
    const uint32_t v = q.front();
    q.pop_front();
    for (uint64_t k = row_ptr[v]; k < row_ptr[v + 1]; ++k) {
      const uint32_t w = col[k];
      if (dist[w] < 0) {
        dist[w] = dist[v] + 1;
        q.push_back(w);
      }
    }
  }
  for (int64_t v = 0; v < nv; ++v) {
    parent[v] = -1;
    if (dist[v] > 0)
      for (uint64_t k = row_ptr[v]; k < row_ptr[v + 1]; ++k)
        if (dist[col[k]] == dist[v] - 1) {
          parent[v] = int32_t(col[k]);
          break;
        }
  }
  return kOK;
}

void oracle_free(void* p) { std::free(p); }

}  // extern "C"
