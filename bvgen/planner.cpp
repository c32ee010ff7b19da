/* =============================================================================
 * bvgen/planner.cpp — seeded plan construction (the INPUTS of the hot path).
 *
 * Part of the input generator shared by both sides (tests feed its output to
 * the oracle and to the CUDA path).  It holds none of the likelihood's
 * arithmetic: no covariance function, no factorisation.  It implements the
 * paper's preprocessing (Alg. 1 l.4-9), which the paper
 * runs once per fit and excludes from timing:
 *   pl_kmeans    K-means clustering g (Alg. 1 l.5), Lloyd
 *                iterations with exact grid-accelerated nearest-centroid
 *                search (ties → lower centroid id), empty-cluster repair by
 *                the farthest point (ties → lowest id), centroids summed in
 *                ascending point id.  Pinned against the oracle's brute-force
 *                assignment (tests/test_planner.py).
 *   pl_block_nn  mNearestNeighborsForBlock (Alg. 1 l.7-9): for position k, the
 *                m_k = min(m, #earlier points) points of earlier blocks nearest
 *                the block centroid, key (d², id), emitted
 *                ascending.  Exact grid ring search; pinned bit-exact against
 *                the oracle's O(n²) brute force for n ≤ 500.
 * Build: g++ -O2 -std=c++17 -ffp-contract=off -fopenmp -shared -fPIC
 * ========================================================================== */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <queue>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

inline double sqdist(const double* a, const double* b, int d) {
  double s = 0;
  for (int q = 0; q < d; ++q) {
    double t = a[q] - b[q];
    s += t * t;
  }
  return s;
}

/* Uniform grid over a point set: CSR of point ids per cell, ids ascending. */
struct Grid {
  int d = 2;
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0}, h[3] = {1, 1, 1};
  int64_t nc[3] = {1, 1, 1};
  std::vector<int64_t> ptr;
  std::vector<int32_t> ids;

  void build(const double* pts, int64_t np, int dim, double per_cell) {
    d = dim;
    for (int q = 0; q < 3; ++q) { lo[q] = 0; hi[q] = 0; nc[q] = 1; h[q] = 1; }
    for (int q = 0; q < d; ++q) {
      lo[q] = INFINITY;
      hi[q] = -INFINITY;
    }
    for (int64_t i = 0; i < np; ++i)
      for (int q = 0; q < d; ++q) {
        lo[q] = std::min(lo[q], pts[i * d + q]);
        hi[q] = std::max(hi[q], pts[i * d + q]);
      }
    // number of cells ≈ np / per_cell, split by extent
    double ext[3] = {1, 1, 1}, vol = 1;
    int nz = 0;
    for (int q = 0; q < d; ++q) {
      ext[q] = hi[q] - lo[q];
      if (ext[q] > 0) { vol *= ext[q]; ++nz; }
    }
    double cells = std::max(1.0, (double)np / per_cell);
    double side = nz ? std::pow(vol / cells, 1.0 / nz) : 1.0;
    int64_t total = 1;
    for (int q = 0; q < d; ++q) {
      if (ext[q] > 0 && side > 0) nc[q] = std::max<int64_t>(1, std::min<int64_t>(4096, (int64_t)std::ceil(ext[q] / side)));
      else nc[q] = 1;
      h[q] = ext[q] > 0 ? ext[q] / (double)nc[q] : 1.0;
      total *= nc[q];
    }
    ptr.assign((size_t)total + 1, 0);
    std::vector<int64_t> cell(np);
    for (int64_t i = 0; i < np; ++i) {
      cell[i] = cell_of(pts + i * d);
      ptr[(size_t)cell[i] + 1]++;
    }
    for (int64_t c = 0; c < total; ++c) ptr[c + 1] += ptr[c];
    ids.assign(np, 0);
    std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
    for (int64_t i = 0; i < np; ++i) ids[fill[cell[i]]++] = (int32_t)i;
  }
  void coord(const double* p, int64_t* c) const {
    for (int q = 0; q < 3; ++q) c[q] = 0;
    for (int q = 0; q < d; ++q) {
      int64_t v = (int64_t)std::floor((p[q] - lo[q]) / h[q]);
      c[q] = std::min<int64_t>(nc[q] - 1, std::max<int64_t>(0, v));
    }
  }
  int64_t cell_of(const double* p) const {
    int64_t c[3];
    coord(p, c);
    return (c[2] * nc[1] + c[1]) * nc[0] + c[0];
  }
  /* Lower bound on the distance from p to any point in a cell at Chebyshev
   * ring > r around p's cell (conservative). */
  double ring_lb(const double* p, const int64_t* c, int64_t r) const {
    double lb = INFINITY;
    for (int q = 0; q < d; ++q) {
      if (nc[q] == 1) continue;
      // the box of rings ≤ r spans cells [c-r, c+r]; outside it in dim q
      double lo_edge = lo[q] + (double)(c[q] - r) * h[q];
      double hi_edge = lo[q] + (double)(c[q] + r + 1) * h[q];
      double dl = (c[q] - r > 0) ? p[q] - lo_edge : INFINITY;
      double dh = (c[q] + r + 1 < nc[q]) ? hi_edge - p[q] : INFINITY;
      lb = std::min(lb, std::min(dl, dh));
    }
    lb = lb * (1.0 - 1e-9) - 1e-12;  // conservative against cell-index rounding
    return lb < 0 ? 0.0 : lb;
  }
  int64_t max_ring() const { return std::max(nc[0], std::max(nc[1], nc[2])); }
  /* visit every cell at Chebyshev ring exactly r around c */
  template <class F> void for_ring(const int64_t* c, int64_t r, F&& f) const {
    int64_t lo3[3], hi3[3];
    for (int q = 0; q < 3; ++q) {
      lo3[q] = std::max<int64_t>(0, c[q] - r);
      hi3[q] = std::min<int64_t>(nc[q] - 1, c[q] + r);
    }
    for (int64_t z = lo3[2]; z <= hi3[2]; ++z)
      for (int64_t y = lo3[1]; y <= hi3[1]; ++y) {
        const bool shell = std::llabs(z - c[2]) == r || std::llabs(y - c[1]) == r;
        const int64_t row = (z * nc[1] + y) * nc[0];
        if (shell) {
          for (int64_t x = lo3[0]; x <= hi3[0]; ++x) f(row + x);
        } else {
          if (c[0] - r >= 0) f(row + c[0] - r);
          if (r > 0 && c[0] + r < nc[0]) f(row + c[0] + r);
        }
      }
  }
};

}  // namespace

extern "C" {

/* Lloyd K-means.  init_idx: k distinct point ids used as
 * initial centroids (the caller draws them with its seeded RNG).  Returns the
 * number of iterations run; writes assign[n] and cent[k*d] (final centroids =
 * member means). */
int pl_kmeans(int64_t n, int d, const double* locs, int32_t k, const int32_t* init_idx, int max_iter,
              int32_t* assign, double* cent, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  for (int32_t c = 0; c < k; ++c)
    for (int q = 0; q < d; ++q) cent[(size_t)c * d + q] = locs[(size_t)init_idx[c] * d + q];
  std::vector<int32_t> prev(n, -1);
  std::vector<double> dist2(n);
  int it = 0;
  for (; it < max_iter; ++it) {
    Grid g;
    g.build(cent, k, d, 2.0);
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 4096)
#endif
    for (int64_t i = 0; i < n; ++i) {
      const double* p = locs + i * d;
      int64_t c[3];
      g.coord(p, c);
      double best = INFINITY;
      int32_t bi = INT32_MAX;
      for (int64_t r = 0; r <= g.max_ring(); ++r) {
        g.for_ring(c, r, [&](int64_t cell) {
          for (int64_t q = g.ptr[cell]; q < g.ptr[cell + 1]; ++q) {
            int32_t cid = g.ids[q];
            double s = sqdist(p, cent + (size_t)cid * d, d);
            if (s < best || (s == best && cid < bi)) {
              best = s;
              bi = cid;
            }
          }
        });
        if (bi != INT32_MAX) {
          double lb = g.ring_lb(p, c, r);
          if (best < lb * lb) break;
        }
      }
      assign[i] = bi;
      dist2[i] = best;
    }
    // empty-cluster repair: farthest point (ties → lowest id) moves in
    std::vector<int64_t> cnt(k, 0);
    for (int64_t i = 0; i < n; ++i) cnt[assign[i]]++;
    for (int32_t c = 0; c < k; ++c) {
      if (cnt[c] > 0) continue;
      int64_t far = -1;
      for (int64_t i = 0; i < n; ++i)
        if (cnt[assign[i]] > 1 && (far < 0 || dist2[i] > dist2[far])) far = i;
      if (far < 0) break;
      cnt[assign[far]]--;
      assign[far] = c;
      cnt[c] = 1;
      dist2[far] = 0;
    }
    // centroid update: member means summed in ascending point id
    std::vector<double> acc((size_t)k * d, 0.0);
    for (int64_t i = 0; i < n; ++i)
      for (int q = 0; q < d; ++q) acc[(size_t)assign[i] * d + q] += locs[i * d + q];
    for (int32_t c = 0; c < k; ++c)
      for (int q = 0; q < d; ++q) cent[(size_t)c * d + q] = acc[(size_t)c * d + q] / (double)cnt[c];
    bool same = std::equal(prev.begin(), prev.end(), assign);
    std::copy(assign, assign + n, prev.begin());
    if (same) {
      ++it;
      break;
    }
  }
  return it;
}

/* Block nearest neighbours (Alg. 1 l.7-9).  nbr_ptr[bc+1]; nbr_idx room for
 * bc*m ids.  Deterministic for any thread count. */
int pl_block_nn(int64_t n, int d, const double* locs, int32_t bc, const int32_t* block_id, const int32_t* order,
                int32_t m, int64_t* nbr_ptr, int32_t* nbr_idx, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  std::vector<int32_t> pos_of_block(bc);
  for (int32_t k = 0; k < bc; ++k) pos_of_block[order[k]] = k;
  std::vector<int32_t> ppos(n);
  for (int64_t i = 0; i < n; ++i) ppos[i] = pos_of_block[block_id[i]];
  // centroids by block id, summed in ascending point id
  std::vector<double> cent((size_t)bc * d, 0.0);
  std::vector<int64_t> cnt(bc, 0);
  for (int64_t i = 0; i < n; ++i) {
    for (int q = 0; q < d; ++q) cent[(size_t)block_id[i] * d + q] += locs[i * d + q];
    cnt[block_id[i]]++;
  }
  for (int32_t b = 0; b < bc; ++b)
    for (int q = 0; q < d; ++q) cent[(size_t)b * d + q] /= (double)cnt[b];
  // number of earlier points per position
  std::vector<int64_t> before(bc + 1, 0);
  for (int32_t k = 0; k < bc; ++k) before[k + 1] = before[k] + cnt[order[k]];
  std::vector<int32_t> mk(bc);
  for (int32_t k = 0; k < bc; ++k) mk[k] = (int32_t)std::min<int64_t>(m, before[k]);
  nbr_ptr[0] = 0;
  for (int32_t k = 0; k < bc; ++k) nbr_ptr[k + 1] = nbr_ptr[k] + mk[k];
  Grid g;
  g.build(locs, n, d, 4.0);
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (int32_t k = 1; k < bc; ++k) {
    const int32_t want = mk[k];
    if (want == 0) continue;
    const double* c0 = cent.data() + (size_t)order[k] * d;
    int64_t cc[3];
    g.coord(c0, cc);
    // max-heap of (d², id) holding the best `want` keys
    std::priority_queue<std::pair<double, int32_t>> heap;
    for (int64_t r = 0; r <= g.max_ring(); ++r) {
      g.for_ring(cc, r, [&](int64_t cell) {
        for (int64_t q = g.ptr[cell]; q < g.ptr[cell + 1]; ++q) {
          int32_t id = g.ids[q];
          if (ppos[id] >= k) continue;
          std::pair<double, int32_t> key(sqdist(locs + (size_t)id * d, c0, d), id);
          if ((int32_t)heap.size() < want) heap.push(key);
          else if (key < heap.top()) {
            heap.pop();
            heap.push(key);
          }
        }
      });
      if ((int32_t)heap.size() == want) {
        double lb = g.ring_lb(c0, cc, r);
        if (heap.top().first < lb * lb) break;
      }
    }
    std::vector<std::pair<double, int32_t>> out;
    out.reserve(want);
    while (!heap.empty()) {
      out.push_back(heap.top());
      heap.pop();
    }
    std::sort(out.begin(), out.end());
    for (int32_t q = 0; q < want; ++q) nbr_idx[nbr_ptr[k] + q] = out[q].second;
  }
  return 0;
}

}  // extern "C"
