// bv_plan.cu — GPU plan construction: the preprocessing of
// Alg. 1 l.4-9 that the paper runs once per fit on the host
// and excludes from time-to-solution:
//   * K-means clustering g (Alg. 1 l.5): Lloyd iterations —
//     every point to its nearest centroid (squared distance summed in x, y, z
//     order with no FMA contraction; ties → lower centroid id), empty clusters
//     repaired with the farthest point of a cluster that keeps ≥ 1 member (ties
//     → lowest point id), centroids = member means summed in ascending point id;
//     stop when the assignment repeats or after max_iter;
//   * mNearestNeighborsForBlock (Alg. 1 l.7-9): for position k, the m_k =
//     min(m, #earlier points) points of blocks at positions < k nearest the
//     block centroid, key (d², id), emitted ascending.
// Both are exact selections with total orders, so the output is bit-identical
// to any other exact implementation (tests compare with the CPU planner
// bvgen/planner.cpp, an independent grid/heap implementation).
//
// Device design: a uniform grid (counting sort into cells; order inside a cell
// is irrelevant because every selection breaks ties by id) and per-query ring
// searches with a conservative distance bound; one thread per point for the
// assignment, one warp per position for the NN lists (a sorted top-m list in
// shared memory, merged with 32 candidates at a time); stable radix sort (CUB)
// + one thread per cluster for the deterministic centroid sums.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

namespace bv {
namespace plan {

// exact squared distance in x, y(, z) order: no contraction (matches a
// -ffp-contract=off host loop s = 0; s += t·t)
__device__ __forceinline__ double sqd(const double* a, const double* b, int d) {
  double s = 0.0;
  for (int q = 0; q < d; ++q) {
    const double t = __dsub_rn(a[q], b[q]);
    s = __dadd_rn(s, __dmul_rn(t, t));
  }
  return s;
}

struct GridDesc {
  int d;
  double lo[3], h[3];
  int nc[3];
};

__device__ __forceinline__ void cell_coord(const GridDesc& g, const double* p, int* c) {
  c[0] = c[1] = c[2] = 0;
  for (int q = 0; q < g.d; ++q) {
    double v = floor((p[q] - g.lo[q]) / g.h[q]);
    v = fmin(fmax(v, 0.0), (double)(g.nc[q] - 1));
    c[q] = (int)v;
  }
}
__device__ __forceinline__ int cell_index(const GridDesc& g, const int* c) { return (c[2] * g.nc[1] + c[1]) * g.nc[0] + c[0]; }

// lower bound on the distance from p to any point outside the cells of
// Chebyshev ring ≤ r around c (conservative against rounding)
__device__ __forceinline__ double ring_lb(const GridDesc& g, const double* p, const int* c, int r) {
  double lb = 1e300;
  for (int q = 0; q < g.d; ++q) {
    if (g.nc[q] == 1) continue;
    const double dl = (c[q] - r > 0) ? p[q] - (g.lo[q] + (double)(c[q] - r) * g.h[q]) : 1e300;
    const double dh = (c[q] + r + 1 < g.nc[q]) ? (g.lo[q] + (double)(c[q] + r + 1) * g.h[q]) - p[q] : 1e300;
    lb = fmin(lb, fmin(dl, dh));
  }
  lb = lb * (1.0 - 1e-9) - 1e-12;
  return lb < 0.0 ? 0.0 : lb;
}

__global__ void cell_count(const double* __restrict__ pts, int np, GridDesc g, int* __restrict__ cell_of,
                           int* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= np) return;
  int c[3];
  cell_coord(g, pts + (size_t)i * g.d, c);
  const int ci = cell_index(g, c);
  cell_of[i] = ci;
  atomicAdd(&cnt[ci], 1);
}

__global__ void cell_fill(int np, const int* __restrict__ cell_of, int* __restrict__ cursor, int* __restrict__ ids) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= np) return;
  ids[atomicAdd(&cursor[cell_of[i]], 1)] = i;
}

// ------------------------------------------------------------------ K-means
__global__ void kmeans_assign(const double* __restrict__ locs, int64_t n, const double* __restrict__ cent, GridDesc g,
                              const int* __restrict__ cptr, const int* __restrict__ cids, int32_t* __restrict__ assign,
                              double* __restrict__ dist2) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int d = g.d;
  double p[3] = {0, 0, 0};
  for (int q = 0; q < d; ++q) p[q] = locs[i * d + q];
  int c[3];
  cell_coord(g, p, c);
  double best = 1e308;
  int bi = 0x7fffffff;
  const int maxr = max(g.nc[0], max(g.nc[1], g.nc[2]));
  for (int r = 0; r <= maxr; ++r) {
    const int z0 = max(0, c[2] - r), z1 = min(g.nc[2] - 1, c[2] + r);
    const int y0 = max(0, c[1] - r), y1 = min(g.nc[1] - 1, c[1] + r);
    const int x0 = max(0, c[0] - r), x1 = min(g.nc[0] - 1, c[0] + r);
    for (int z = z0; z <= z1; ++z)
      for (int y = y0; y <= y1; ++y) {
        const bool shell = abs(z - c[2]) == r || abs(y - c[1]) == r;
        const int xs = (shell || r == 0) ? 1 : 2 * r;  // inside the ring's box only its two x faces
        for (int x = shell ? x0 : c[0] - r; x <= x1; x += xs) {
          if (x < x0) continue;
          const int cell = (z * g.nc[1] + y) * g.nc[0] + x;
          for (int e = cptr[cell]; e < cptr[cell + 1]; ++e) {
            const int cid = cids[e];
            const double s = sqd(p, cent + (size_t)cid * d, d);
            if (s < best || (s == best && cid < bi)) {
              best = s;
              bi = cid;
            }
          }
        }
      }
    if (bi != 0x7fffffff) {
      const double lb = ring_lb(g, p, c, r);
      if (best < lb * lb) break;
    }
  }
  assign[i] = bi;
  dist2[i] = best;
}

__global__ void histogram(const int32_t* __restrict__ key, int64_t n, int* __restrict__ cnt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(&cnt[key[i]], 1);
}

// member means in ascending point id: `ids` is the point list stably sorted by cluster
__global__ void segment_means(const double* __restrict__ locs, int d, int k, const int* __restrict__ off,
                              const int* __restrict__ cnt, const int32_t* __restrict__ ids, double* __restrict__ cent) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= k) return;
  double a[3] = {0, 0, 0};
  for (int e = off[c]; e < off[c] + cnt[c]; ++e)
    for (int q = 0; q < d; ++q) a[q] = __dadd_rn(a[q], locs[(size_t)ids[e] * d + q]);
  for (int q = 0; q < d; ++q) cent[(size_t)c * d + q] = __ddiv_rn(a[q], (double)cnt[c]);
}

// farthest point among clusters keeping ≥ 2 members (ties → lowest id): block-wide argmax, one block
__global__ void farthest(const double* __restrict__ dist2, const int32_t* __restrict__ assign, const int* __restrict__ cnt,
                         int64_t n, int64_t* __restrict__ out) {
  __shared__ double bv[1024];
  __shared__ int64_t bi[1024];
  double best = -1.0;
  int64_t idx = -1;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    if (cnt[assign[i]] > 1 && (idx < 0 || dist2[i] > best)) {  // i ascending per thread: first max kept
      best = dist2[i];
      idx = i;
    }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = idx;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double ob = bv[threadIdx.x + s];
      const int64_t oi = bi[threadIdx.x + s];
      const bool take = oi >= 0 && (bi[threadIdx.x] < 0 || ob > bv[threadIdx.x] ||
                                    (ob == bv[threadIdx.x] && oi < bi[threadIdx.x]));
      if (take) {
        bv[threadIdx.x] = ob;
        bi[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = bi[0];
}

__global__ void move_point(int64_t* __restrict__ far, int32_t c, int32_t* __restrict__ assign, int* __restrict__ cnt,
                           double* __restrict__ dist2) {
  const int64_t f = *far;
  if (f < 0) return;
  cnt[assign[f]]--;
  assign[f] = c;
  cnt[c] = 1;
  dist2[f] = 0.0;
}

__global__ void count_changed(const int32_t* __restrict__ a, const int32_t* __restrict__ b, int64_t n,
                              unsigned long long* __restrict__ changed) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && a[i] != b[i]) atomicAdd(changed, 1ull);
}

// ------------------------------------------------------------------ block NN
constexpr int kNnWarps = 4;
constexpr int kNnMax = 256;  // largest m this kernel takes

struct Key {
  double d2;
  int32_t id;
};
__device__ __forceinline__ bool key_less(double a2, int32_t ai, double b2, int32_t bi) {
  return a2 < b2 || (a2 == b2 && ai < bi);
}

// merge up to 32 candidate keys (one per lane, `valid` flag) into the sorted list
// L[0..len) of capacity `want`; C (32 slots) and T (want slots) are scratch
__device__ void merge_keys(Key* L, Key* C, Key* T, int& len, int want, double kd, int32_t kid, bool valid, int lane) {
  if (len == want && valid) valid = key_less(kd, kid, L[want - 1].d2, L[want - 1].id);
  const unsigned vm = __ballot_sync(0xffffffffu, valid);
  if (!vm) return;
  int rk = 0;  // rank among the valid candidates (keys are distinct: ids differ)
  for (int o = 0; o < 32; ++o) {
    const double od = __shfl_sync(0xffffffffu, kd, o);
    const int32_t oi = __shfl_sync(0xffffffffu, kid, o);
    if (((vm >> o) & 1u) && key_less(od, oi, kd, kid)) ++rk;
  }
  const int nv = __popc(vm);
  if (valid) C[rk] = Key{kd, kid};
  __syncwarp();
  const int newlen = min(want, len + nv);
  for (int i = lane; i < len; i += 32) {  // old entry i moves up by #candidates below it
    const Key e = L[i];
    int lo = 0, hi = nv;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (key_less(C[mid].d2, C[mid].id, e.d2, e.id)) lo = mid + 1;
      else hi = mid;
    }
    if (i + lo < newlen) T[i + lo] = e;
  }
  if (lane < nv) {  // candidate `lane` moves up by #old entries below it
    const Key e = C[lane];
    int lo = 0, hi = len;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (key_less(L[mid].d2, L[mid].id, e.d2, e.id)) lo = mid + 1;
      else hi = mid;
    }
    if (lane + lo < newlen) T[lane + lo] = e;
  }
  __syncwarp();
  for (int i = lane; i < newlen; i += 32) L[i] = T[i];
  len = newlen;
  __syncwarp();
}

__global__ void __launch_bounds__(kNnWarps * 32) block_nn(const double* __restrict__ locs, int d,
                                                           const int32_t* __restrict__ ppos,
                                                           const double* __restrict__ bcent,
                                                           const int32_t* __restrict__ order, int32_t bc,
                                                           const int64_t* __restrict__ nbr_ptr, GridDesc g,
                                                           const int* __restrict__ gptr, const int* __restrict__ gids,
                                                           int32_t* __restrict__ nbr_idx) {
  __shared__ Key Ls[kNnWarps][kNnMax];
  __shared__ Key Ts[kNnWarps][kNnMax];
  __shared__ Key Cs[kNnWarps][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int k = blockIdx.x * kNnWarps + w;
  if (k >= bc) return;
  const int want = (int)(nbr_ptr[k + 1] - nbr_ptr[k]);
  if (want == 0) return;
  Key* L = Ls[w];
  Key* T = Ts[w];
  double c0[3] = {0, 0, 0};
  for (int q = 0; q < d; ++q) c0[q] = bcent[(size_t)order[k] * d + q];
  int cc[3];
  cell_coord(g, c0, cc);
  int len = 0;
  const int maxr = max(g.nc[0], max(g.nc[1], g.nc[2]));
  for (int r = 0; r <= maxr; ++r) {
    const int z0 = max(0, cc[2] - r), z1 = min(g.nc[2] - 1, cc[2] + r);
    const int y0 = max(0, cc[1] - r), y1 = min(g.nc[1] - 1, cc[1] + r);
    const int x0 = max(0, cc[0] - r), x1 = min(g.nc[0] - 1, cc[0] + r);
    for (int z = z0; z <= z1; ++z)
      for (int y = y0; y <= y1; ++y) {
        const bool shell = abs(z - cc[2]) == r || abs(y - cc[1]) == r;
        const int xs = (shell || r == 0) ? 1 : 2 * r;
        for (int x = shell ? x0 : cc[0] - r; x <= x1; x += xs) {
          if (x < x0) continue;
          const int cell = (z * g.nc[1] + y) * g.nc[0] + x;
          for (int e0 = gptr[cell]; e0 < gptr[cell + 1]; e0 += 32) {
            const int e = e0 + lane;
            bool valid = e < gptr[cell + 1];
            double kd = 0.0;
            int32_t kid = 0x7fffffff;
            if (valid) {
              kid = gids[e];
              valid = ppos[kid] < k;  // earlier blocks only
              if (valid) kd = sqd(locs + (size_t)kid * d, c0, d);
            }
            merge_keys(L, Cs[w], T, len, want, kd, kid, valid, lane);
          }
        }
      }
    if (len == want) {
      const double lb = ring_lb(g, c0, cc, r);
      if (L[want - 1].d2 < lb * lb) break;
    }
  }
  for (int i = lane; i < len; i += 32) nbr_idx[nbr_ptr[k] + i] = L[i].id;
}

__global__ void point_pos(const int32_t* __restrict__ block_id, const int32_t* __restrict__ pos_of_block, int64_t n,
                          int32_t* __restrict__ ppos) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) ppos[i] = pos_of_block[block_id[i]];
}

__global__ void iota(int32_t* __restrict__ a, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = (int32_t)i;
}

}  // namespace plan
}  // namespace bv

// =============================================================== host side (C ABI)
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "bv.h"

namespace {
using bv::plan::GridDesc;

thread_local std::string g_plan_err;

GridDesc grid_for(const std::vector<double>& lo, const std::vector<double>& hi, int d, double np, double per_cell) {
  GridDesc g{};
  g.d = d;
  double vol = 1.0;
  int nz = 0;
  for (int q = 0; q < 3; ++q) {
    g.lo[q] = 0.0;
    g.h[q] = 1.0;
    g.nc[q] = 1;
  }
  for (int q = 0; q < d; ++q) {
    const double ext = hi[q] - lo[q];
    g.lo[q] = lo[q];
    if (ext > 0) {
      vol *= ext;
      ++nz;
    }
  }
  const double cells = std::max(1.0, np / per_cell);
  const double side = nz ? std::pow(vol / cells, 1.0 / nz) : 1.0;
  for (int q = 0; q < d; ++q) {
    const double ext = hi[q] - lo[q];
    g.nc[q] = (ext > 0 && side > 0) ? (int)std::max(1.0, std::min(2048.0, std::ceil(ext / side))) : 1;
    g.h[q] = ext > 0 ? ext / (double)g.nc[q] : 1.0;
  }
  return g;
}

struct DevGrid {
  int cells = 0;
  int *ptr = nullptr, *ids = nullptr, *cell_of = nullptr, *cursor = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  void release() {
    cudaFree(ptr);
    cudaFree(ids);
    cudaFree(cell_of);
    cudaFree(cursor);
    cudaFree(tmp);
    ptr = ids = cell_of = cursor = nullptr;
    tmp = nullptr;
  }
  // counting sort of np points into g's cells (allocates on first use)
  cudaError_t build(const double* pts, int np, const GridDesc& g, cudaStream_t s) {
    const int c = g.nc[0] * g.nc[1] * g.nc[2];
    cudaError_t e = cudaSuccess;
    if (!ptr) {
      cells = c;
      if ((e = cudaMalloc(&ptr, sizeof(int) * (c + 1))) != cudaSuccess) return e;
      if ((e = cudaMalloc(&cursor, sizeof(int) * (c + 1))) != cudaSuccess) return e;
      if ((e = cudaMalloc(&ids, sizeof(int) * std::max(np, 1))) != cudaSuccess) return e;
      if ((e = cudaMalloc(&cell_of, sizeof(int) * std::max(np, 1))) != cudaSuccess) return e;
      cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cursor, ptr, c + 1, s);
      if ((e = cudaMalloc(&tmp, tmp_bytes)) != cudaSuccess) return e;
    }
    if ((e = cudaMemsetAsync(cursor, 0, sizeof(int) * (c + 1), s)) != cudaSuccess) return e;
    const int T = 256;
    bv::plan::cell_count<<<(np + T - 1) / T, T, 0, s>>>(pts, np, g, cell_of, cursor);
    if ((e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cursor, ptr, c + 1, s)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(cursor, ptr, sizeof(int) * c, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) return e;
    bv::plan::cell_fill<<<(np + T - 1) / T, T, 0, s>>>(np, cell_of, cursor, ids);
    return cudaGetLastError();
  }
};

struct Bufs {
  std::vector<void*> p;
  template <class T> cudaError_t alloc(T** out, size_t count) {
    void* v = nullptr;
    cudaError_t e = cudaMalloc(&v, sizeof(T) * std::max<size_t>(count, 1));
    if (e == cudaSuccess) p.push_back(v);
    *out = (T*)v;
    return e;
  }
  ~Bufs() {
    for (void* v : p) cudaFree(v);
  }
};

void bbox(const double* locs, int64_t n, int d, std::vector<double>& lo, std::vector<double>& hi) {
  lo.assign(d, INFINITY);
  hi.assign(d, -INFINITY);
  for (int64_t i = 0; i < n; ++i)
    for (int q = 0; q < d; ++q) {
      lo[q] = std::min(lo[q], locs[i * d + q]);
      hi[q] = std::max(hi[q], locs[i * d + q]);
    }
}

// stable sort of point ids by key (keys < k), then per-segment means
cudaError_t segment_mean_pass(const double* d_locs, int64_t n, int d, int k, const int32_t* d_key, const int32_t* d_iota,
                              int* d_cnt, int* d_off, uint32_t* d_ks, int32_t* d_ids, void* tmp, size_t tmp_bytes,
                              void* stmp, size_t stmp_bytes, double* d_out, cudaStream_t s) {
  cudaError_t e;
  int bits = 1;
  while ((1ll << bits) < (long long)k) ++bits;
  if ((e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, reinterpret_cast<const uint32_t*>(d_key), d_ks, d_iota,
                                            d_ids, (int)n, 0, bits, s)) != cudaSuccess)
    return e;
  if ((e = cub::DeviceScan::ExclusiveSum(stmp, stmp_bytes, d_cnt, d_off, k, s)) != cudaSuccess) return e;
  bv::plan::segment_means<<<(k + 127) / 128, 128, 0, s>>>(d_locs, d, k, d_off, d_cnt, d_ids, d_out);
  return cudaGetLastError();
}

}  // namespace

#define PL_CUDA(call)                                                 \
  do {                                                                \
    cudaError_t e_ = (call);                                          \
    if (e_ != cudaSuccess) {                                          \
      g_plan_err = std::string(#call) + ": " + cudaGetErrorString(e_); \
      grid.release();                                                 \
      return e_ == cudaErrorMemoryAllocation ? BV_ENOMEM : BV_ECUDA;  \
    }                                                                 \
  } while (0)

extern "C" {

const char* bv_plan_last_error(void) { return g_plan_err.c_str(); }

bv_status bv_plan_kmeans(int32_t device, int64_t n, int32_t d, const double* locs, int32_t k, const int32_t* init_idx,
                         int32_t max_iter, int32_t* assign, double* cent, int32_t* iters) {
  g_plan_err.clear();
  if (n < 1 || n > INT32_MAX || (d != 2 && d != 3) || k < 1 || k > n || !locs || !init_idx || !assign || !cent ||
      max_iter < 1) {
    g_plan_err = "invalid argument";
    return BV_EINVAL;
  }
  for (int32_t c = 0; c < k; ++c)
    if (init_idx[c] < 0 || init_idx[c] >= n) {
      g_plan_err = "init_idx out of range";
      return BV_EINVAL;
    }
  DevGrid grid;
  PL_CUDA(cudaSetDevice(device));
  cudaStream_t s = 0;
  Bufs B;
  double *d_locs, *d_cent, *d_dist2;
  int32_t *d_assign, *d_prev, *d_iota, *d_ids;
  uint32_t* d_ks;
  int *d_cnt, *d_off;
  int64_t* d_far;
  unsigned long long* d_changed;
  PL_CUDA(B.alloc(&d_locs, (size_t)n * d));
  PL_CUDA(B.alloc(&d_cent, (size_t)k * d));
  PL_CUDA(B.alloc(&d_dist2, (size_t)n));
  PL_CUDA(B.alloc(&d_assign, (size_t)n));
  PL_CUDA(B.alloc(&d_prev, (size_t)n));
  PL_CUDA(B.alloc(&d_iota, (size_t)n));
  PL_CUDA(B.alloc(&d_ids, (size_t)n));
  PL_CUDA(B.alloc(&d_ks, (size_t)n));
  PL_CUDA(B.alloc(&d_cnt, (size_t)k));
  PL_CUDA(B.alloc(&d_off, (size_t)k + 1));
  PL_CUDA(B.alloc(&d_far, 1));
  PL_CUDA(B.alloc(&d_changed, 1));
  PL_CUDA(cudaMemcpy(d_locs, locs, sizeof(double) * n * d, cudaMemcpyHostToDevice));
  {
    std::vector<double> c0((size_t)k * d);
    for (int32_t c = 0; c < k; ++c)
      for (int q = 0; q < d; ++q) c0[(size_t)c * d + q] = locs[(size_t)init_idx[c] * d + q];
    PL_CUDA(cudaMemcpy(d_cent, c0.data(), sizeof(double) * k * d, cudaMemcpyHostToDevice));
  }
  PL_CUDA(cudaMemset(d_prev, 0xff, sizeof(int32_t) * n));
  const int T = 256;
  const int nb = (int)((n + T - 1) / T);
  bv::plan::iota<<<nb, T>>>(d_iota, n);
  size_t sort_bytes = 0, scan_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const uint32_t*)d_assign, d_ks, d_iota, d_ids, (int)n, 0, 32);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, d_cnt, d_off, k);
  void *sort_tmp, *scan_tmp;
  PL_CUDA(B.alloc((char**)&sort_tmp, sort_bytes));
  PL_CUDA(B.alloc((char**)&scan_tmp, scan_bytes));
  std::vector<double> lo, hi;
  bbox(locs, n, d, lo, hi);  // centroids stay inside the points' box
  const GridDesc g = grid_for(lo, hi, d, (double)k, 2.0);
  std::vector<int> hcnt(k);
  int it = 0;
  for (; it < max_iter; ++it) {
    PL_CUDA(grid.build(d_cent, k, g, s));
    bv::plan::kmeans_assign<<<nb, T, 0, s>>>(d_locs, n, d_cent, g, grid.ptr, grid.ids, d_assign, d_dist2);
    PL_CUDA(cudaGetLastError());
    PL_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(int) * k, s));
    bv::plan::histogram<<<nb, T, 0, s>>>(d_assign, n, d_cnt);
    PL_CUDA(cudaMemcpy(hcnt.data(), d_cnt, sizeof(int) * k, cudaMemcpyDeviceToHost));
    for (int32_t c = 0; c < k; ++c) {  // empty-cluster repair, clusters in ascending id
      if (hcnt[c] > 0) continue;
      bv::plan::farthest<<<1, 1024, 0, s>>>(d_dist2, d_assign, d_cnt, n, d_far);
      bv::plan::move_point<<<1, 1, 0, s>>>(d_far, c, d_assign, d_cnt, d_dist2);
      int64_t f = -1;
      PL_CUDA(cudaMemcpy(&f, d_far, sizeof(int64_t), cudaMemcpyDeviceToHost));
      if (f < 0) break;
    }
    PL_CUDA(segment_mean_pass(d_locs, n, d, k, d_assign, d_iota, d_cnt, d_off, d_ks, d_ids, sort_tmp, sort_bytes,
                              scan_tmp, scan_bytes, d_cent, s));
    PL_CUDA(cudaMemsetAsync(d_changed, 0, sizeof(unsigned long long), s));
    bv::plan::count_changed<<<nb, T, 0, s>>>(d_assign, d_prev, n, d_changed);
    unsigned long long changed = 0;
    PL_CUDA(cudaMemcpy(&changed, d_changed, sizeof(changed), cudaMemcpyDeviceToHost));
    PL_CUDA(cudaMemcpyAsync(d_prev, d_assign, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
    if (changed == 0) {
      ++it;
      break;
    }
  }
  PL_CUDA(cudaMemcpy(assign, d_assign, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  PL_CUDA(cudaMemcpy(cent, d_cent, sizeof(double) * k * d, cudaMemcpyDeviceToHost));
  grid.release();
  if (iters) *iters = it;
  return BV_OK;
}

bv_status bv_plan_block_nn(int32_t device, int64_t n, int32_t d, const double* locs, int32_t bc, const int32_t* block_id,
                           const int32_t* order, int32_t m, int64_t* nbr_ptr, int32_t* nbr_idx) {
  g_plan_err.clear();
  if (n < 1 || n > INT32_MAX || (d != 2 && d != 3) || bc < 1 || bc > n || !locs || !block_id || !order || !nbr_ptr ||
      m < 0 || m > bv::plan::kNnMax) {
    g_plan_err = "invalid argument (m must be in [0, 256])";
    return BV_EINVAL;
  }
  std::vector<int32_t> pos_of_block(bc, -1);
  for (int32_t k = 0; k < bc; ++k) {
    if (order[k] < 0 || order[k] >= bc || pos_of_block[order[k]] >= 0) {
      g_plan_err = "order is not a permutation";
      return BV_EINVAL;
    }
    pos_of_block[order[k]] = k;
  }
  std::vector<int64_t> cnt(bc, 0);
  for (int64_t i = 0; i < n; ++i) {
    if (block_id[i] < 0 || block_id[i] >= bc) {
      g_plan_err = "block_id out of range";
      return BV_EINVAL;
    }
    cnt[block_id[i]]++;
  }
  for (int32_t b = 0; b < bc; ++b)
    if (cnt[b] == 0) {
      g_plan_err = "empty block";
      return BV_EINVAL;
    }
  int64_t before = 0;
  nbr_ptr[0] = 0;
  for (int32_t k = 0; k < bc; ++k) {  // m_k = min(m, #earlier points) (reading G6)
    nbr_ptr[k + 1] = nbr_ptr[k] + std::min<int64_t>(m, before);
    before += cnt[order[k]];
  }
  if (!nbr_idx && nbr_ptr[bc] > 0) {
    g_plan_err = "nbr_idx is NULL";
    return BV_EINVAL;
  }
  DevGrid grid;
  PL_CUDA(cudaSetDevice(device));
  cudaStream_t s = 0;
  Bufs B;
  double *d_locs, *d_bcent;
  int32_t *d_bid, *d_pob, *d_ppos, *d_order, *d_iota, *d_ids, *d_nbr;
  uint32_t* d_ks;
  int *d_cnt, *d_off;
  int64_t* d_ptr;
  PL_CUDA(B.alloc(&d_locs, (size_t)n * d));
  PL_CUDA(B.alloc(&d_bcent, (size_t)bc * d));
  PL_CUDA(B.alloc(&d_bid, (size_t)n));
  PL_CUDA(B.alloc(&d_pob, (size_t)bc));
  PL_CUDA(B.alloc(&d_ppos, (size_t)n));
  PL_CUDA(B.alloc(&d_order, (size_t)bc));
  PL_CUDA(B.alloc(&d_iota, (size_t)n));
  PL_CUDA(B.alloc(&d_ids, (size_t)n));
  PL_CUDA(B.alloc(&d_ks, (size_t)n));
  PL_CUDA(B.alloc(&d_cnt, (size_t)bc));
  PL_CUDA(B.alloc(&d_off, (size_t)bc + 1));
  PL_CUDA(B.alloc(&d_ptr, (size_t)bc + 1));
  PL_CUDA(B.alloc(&d_nbr, (size_t)std::max<int64_t>(nbr_ptr[bc], 1)));
  PL_CUDA(cudaMemcpy(d_locs, locs, sizeof(double) * n * d, cudaMemcpyHostToDevice));
  PL_CUDA(cudaMemcpy(d_bid, block_id, sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  PL_CUDA(cudaMemcpy(d_pob, pos_of_block.data(), sizeof(int32_t) * bc, cudaMemcpyHostToDevice));
  PL_CUDA(cudaMemcpy(d_order, order, sizeof(int32_t) * bc, cudaMemcpyHostToDevice));
  PL_CUDA(cudaMemcpy(d_ptr, nbr_ptr, sizeof(int64_t) * (bc + 1), cudaMemcpyHostToDevice));
  const int T = 256;
  const int nb = (int)((n + T - 1) / T);
  bv::plan::iota<<<nb, T>>>(d_iota, n);
  bv::plan::point_pos<<<nb, T>>>(d_bid, d_pob, n, d_ppos);
  PL_CUDA(cudaMemset(d_cnt, 0, sizeof(int) * bc));
  bv::plan::histogram<<<nb, T>>>(d_bid, n, d_cnt);
  size_t sort_bytes = 0, scan_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const uint32_t*)d_bid, d_ks, d_iota, d_ids, (int)n, 0, 32);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, d_cnt, d_off, bc);
  void *sort_tmp, *scan_tmp;
  PL_CUDA(B.alloc((char**)&sort_tmp, sort_bytes));
  PL_CUDA(B.alloc((char**)&scan_tmp, scan_bytes));
  // block centroids: member means in ascending point id
  PL_CUDA(segment_mean_pass(d_locs, n, d, bc, d_bid, d_iota, d_cnt, d_off, d_ks, d_ids, sort_tmp, sort_bytes, scan_tmp,
                            scan_bytes, d_bcent, s));
  std::vector<double> lo, hi;
  bbox(locs, n, d, lo, hi);
  const GridDesc g = grid_for(lo, hi, d, (double)n, 4.0);
  PL_CUDA(grid.build(d_locs, (int)n, g, s));
  bv::plan::block_nn<<<(bc + bv::plan::kNnWarps - 1) / bv::plan::kNnWarps, bv::plan::kNnWarps * 32, 0, s>>>(
      d_locs, d, d_ppos, d_bcent, d_order, bc, d_ptr, g, grid.ptr, grid.ids, d_nbr);
  PL_CUDA(cudaGetLastError());
  if (nbr_ptr[bc] > 0)
    PL_CUDA(cudaMemcpy(nbr_idx, d_nbr, sizeof(int32_t) * nbr_ptr[bc], cudaMemcpyDeviceToHost));
  PL_CUDA(cudaDeviceSynchronize());
  grid.release();
  return BV_OK;
}

}  // extern "C"
