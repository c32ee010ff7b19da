// bv_host.cpp — host runtime behind include/bv.h.
//
// bv_setup: validates the frozen plan (Alg. 1 l.4-9 output),
// lays it out on the device (block-contiguous 32-byte point records, neighbour
// lists remapped to permuted indices), splits positions across ranks by
// estimated cost, groups this rank's blocks into size buckets, creates the
// NCCL communicator and captures one CUDA graph per Matérn kind:
//   memcpy θ → zero accumulator → bucket kernels on concurrent branches
//   (Alg. 1 l.10-29 fused per block, each block adding its exact fixed-point
//   term atomically: l.28-30) → [ncclAllReduce of 7 uint64] → memcpy result.
// bv_loglik: fills θ (and ν-only constants) into pinned memory, replays the
// graph, decodes the exact fixed-point sum.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/bv.h"
#include "bv_common.cuh"

namespace bv {
cudaError_t launch_cv(int kind, int count, cudaStream_t s, const PointRec* pts, const int32_t* nbr,
                      const BlockDesc* desc, const int32_t* list, const Theta* th, const double* etab, double* u,
                      double* d, unsigned long long* acc, int k_begin);
size_t predict_smem_bytes(int N);
cudaError_t prepare_predict(size_t smem);
cudaError_t launch_predict(int nblocks, size_t smem, cudaStream_t s, const PointRec* train, const PointRec* newp,
                           const int32_t* nbr, const BlockDesc* desc, const Theta* th, const int64_t* cov_off,
                           double* mean, double* var, double* cov, int32_t* status);
cudaError_t launch_scatter_y(const double* y, const int32_t* perm_of_id, int64_t n, PointRec* pts, cudaStream_t s);
int v3_maxt_for(int TI);
size_t v3_smem_bytes(int TImax, int cap);
cudaError_t prepare_block_v3(size_t max_smem);
cudaError_t launch_block_v3(int kind, int nblocks, int TImax, int cap, cudaStream_t s, const PointRec* pts,
                            const int32_t* nbr, const BlockDesc* desc, const int32_t* list, const Theta* th,
                            const int16_t* tabs, const int32_t* tab_off, const double* etab, double* u, double* d,
                            unsigned long long* acc, int k_begin, double* gslots, int gs_grid, const double* pre,
                            const int64_t* pre_off, double jit);
cudaError_t launch_pregen(int nblocks, int chunks, cudaStream_t s, const PointRec* pts, const int32_t* nbr,
                          const BlockDesc* desc, const Theta* th, const double* etab, const int64_t* pre_off,
                          double* pre);
bool v3_global_slots(int TI);
int debug_v3_cycles(unsigned long long* out, int reset);
int w_max_ti();
cudaError_t prepare_block_w();
cudaError_t launch_block_w(int kind, int nblocks, int TI, cudaStream_t s, const PointRec* pts, const int32_t* nbr,
                           const BlockDesc* desc, const int32_t* list, const Theta* th, const double* etab, double* u,
                           double* d, unsigned long long* acc, int k_begin, const double* pre, const int64_t* pre_off,
                           double jit);
}  // namespace bv

namespace {
constexpr size_t kSmemOptin = 232448;  // B200 per-block opt-in shared memory

// The block kernels.  Positions are grouped into buckets by kernel and tile
// rows TI = ⌈(N+1)/8⌉ (N = m + l, the y row appended).
enum KernelKind : int { kKernCV = 0, kKernW = 1, kKernV3 = 2 };
struct Bucket {
  int TI, count, offset;  // TI = 0 for the classic-Vecchia kernel
  int cap;                // v3: tile slots for this TI
  size_t gs_off = 0;      // v3 with global slots (TI > 37): this bucket's scratch offset (doubles)
  int kern = kKernV3;
};

// Slot tables of the large-block kernel (bv_block_v3.cu).  Every tile of column
// K lives in one shared-memory slot from its generation (C, row-major) through
// its in-place triangular solve (L, fragment order) until its last use; diagonal
// tiles never occupy a slot.  Column 0 (I ≥ 1) first; iteration J frees row J's
// tiles except L(J,J−1), plus L(J−1,J−2), then generates column J+1's tiles
// I ≥ J+2.  A LIFO free list replays that schedule; slot[I·TI + K] is the slot
// of tile (I,K).  off[2·TI + (TI−TJ)] indexes the table of each (TI, TJ) pair
// (TI − TJ ∈ {0, 1}); cap[TI] = the most slots live at once.
struct SlotTables {
  std::vector<int16_t> tabs;
  std::vector<int32_t> off;
  std::vector<int> cap;
  void build(int TImax) {
    off.assign(2 * (size_t)(TImax + 1), 0);
    cap.assign((size_t)TImax + 1, 0);
    tabs.clear();
    for (int TI = 1; TI <= TImax; ++TI)
      for (int e = 0; e < 2; ++e) {
        const int TJ = TI - e;
        off[2 * TI + e] = (int32_t)tabs.size();
        std::vector<int16_t> t((size_t)TI * TI, 0);
        std::vector<int16_t> freel;
        int next = 0, live = 0, most = 0;
        auto alloc = [&]() -> int16_t {
          ++live;
          most = std::max(most, live);
          if (!freel.empty()) {
            int16_t v = freel.back();
            freel.pop_back();
            return v;
          }
          return (int16_t)next++;
        };
        auto release = [&](int16_t v) {
          --live;
          freel.push_back(v);
        };
        for (int I = 1; I < TI; ++I) t[(size_t)I * TI + 0] = alloc();
        for (int J = 0; J + 1 < TJ; ++J) {
          // L(J,J−1) is the b operand of iteration J−1's final term, which a slow
          // update warp may still be reading while a fast one generates column J+1:
          // it is released one iteration later (after iteration J's U barrier)
          for (int K = 0; K + 1 < J; ++K) release(t[(size_t)J * TI + K]);
          if (J >= 2) release(t[(size_t)(J - 1) * TI + J - 2]);
          for (int I = J + 2; I < TI; ++I) t[(size_t)I * TI + J + 1] = alloc();
        }
        tabs.insert(tabs.end(), t.begin(), t.end());
        cap[TI] = std::max(cap[TI], std::max(most, 1));
      }
  }
};
}  // namespace

struct bv_handle {
  int device = 0, rank = 0, world = 1;
  int64_t n = 0;
  int d = 2;
  int32_t bc = 0, kb = 0, ke = 0, nq = 0;
  cudaStream_t stream = nullptr;
  cudaGraph_t graph[4] = {nullptr, nullptr, nullptr, nullptr};      // one per MaternKind
  cudaGraphExec_t exec[4] = {nullptr, nullptr, nullptr, nullptr};
  ncclComm_t comm = nullptr;
  bv::PointRec* d_pts = nullptr;
  int32_t* d_nbr = nullptr;
  bv::BlockDesc* d_desc = nullptr;
  int32_t* d_list = nullptr;
  bv::Theta* d_theta = nullptr;
  double* d_u = nullptr;
  double* d_d = nullptr;
  unsigned long long* d_acc = nullptr;
  unsigned long long* d_min = nullptr;
  int32_t* d_perm_of_id = nullptr;
  std::vector<int32_t> h_perm_of_id;       // global id → permuted record (host copy, for bv_predict)
  double* d_y_stage = nullptr;
  int16_t* d_tabs = nullptr;
  double* d_exptab = nullptr;
  double* d_gslots = nullptr;  // tile-slot scratch of the global-slot buckets (joint sizes > 295)
  int gs_grid = 0;             // persistent CTAs per global-slot bucket launch
  int32_t* d_tab_off = nullptr;
  bool local = false;                      // test-only rank-local handle (bv_setup_rank_local): no communicator
  int wmax = 0;                            // largest TI run by the warp-per-block kernel
  std::vector<int> cap_of;                 // v3 slot capacity by TI
  std::vector<int> kern_of;                // kernel of each TI's bucket (jitter retries use the same)
  std::vector<size_t> gsoff_of;            // v3 global-slot scratch offset by TI (TI > 37)
  bv::Theta* h_theta = nullptr;            // pinned
  unsigned long long* h_acc = nullptr;     // pinned
  cudaEvent_t ev_k0 = nullptr, ev_k1 = nullptr;  // around the block kernels (graph event nodes)
  static constexpr int kBranches = 4;             // concurrent bucket streams inside the graph
  cudaStream_t side[kBranches] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t fork_ev = nullptr, join_ev[kBranches] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<Bucket> buckets;
  std::string err;
  int32_t failed_pos = -1;
  // optional jitter retry (reading G15b; off the hot path, never captured)
  bool jitter = false;
  int64_t jitter_events = 0;
  std::vector<int32_t> h_N;                  // joint size N_q = l + m per local position
  int32_t* d_jlist = nullptr;                // failed positions being retried
  unsigned long long* d_jacc = nullptr;      // the retry's own accumulator (kAccSlots) + 3 allreduce slots
  // general-ν pre-generation (small plans): packed Σ triangles, offsets per local position
  double* d_pre = nullptr;
  int64_t* d_pre_off = nullptr;
  int pre_chunks = 0;
  int last_kind = -1;  // MaternKind of the most recent evaluation
  std::vector<int64_t> pred_stamp;  // bv_predict's duplicate-neighbour table (n entries)
  int64_t pred_epoch = 0;
};

namespace {

bv_status fail(bv_handle* h, bv_status st, const std::string& msg) {
  if (h) h->err = msg;
  return st;
}

#define BV_CUDA(h, call)                                                                              \
  do {                                                                                                \
    cudaError_t e_ = (call);                                                                          \
    if (e_ != cudaSuccess)                                                                            \
      return fail(h, e_ == cudaErrorMemoryAllocation ? BV_ENOMEM : BV_ECUDA,                          \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                                \
  } while (0)

#define BV_NCCL(h, call)                                                                              \
  do {                                                                                                \
    ncclResult_t r_ = (call);                                                                         \
    if (r_ != ncclSuccess) return fail(h, BV_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

thread_local std::string g_setup_err;

// ν-only constants of the general-ν K_ν evaluator (bessel_k.cuh), computed in
// long double once per evaluation.
void fill_general_nu(bv::Theta& t, double nu) {
  const long double ln = (long double)nu;
  const long double nl = std::floor(ln + 0.5L);
  const long double mu = ln - nl;
  const long double gampl = 1.0L / std::tgamma(1.0L + mu);
  const long double gammi = 1.0L / std::tgamma(1.0L - mu);
  long double gam1;
  if (std::fabs(mu) >= 1e-3L) {
    gam1 = (gammi - gampl) / (2.0L * mu);
  } else {
    // 1/Γ(1+z) = 1 + γz + c3 z² + c4 z³ + … (Abramowitz–Stegun 6.1.34):
    // γ1(z) = −(γ + c4 z² + c6 z⁴ + …)
    const long double g = 0.5772156649015328606065120900824024L;
    const long double c4 = -0.0420026350340952355290039348754298L;
    const long double c6 = -0.0421977345555443367482083012891874L;
    const long double z2 = mu * mu;
    gam1 = -(g + c4 * z2 + c6 * z2 * z2);
  }
  const long double gam2 = 0.5L * (gammi + gampl);
  const long double pimu = 3.14159265358979323846264338327950288L * mu;
  const long double fact = (std::fabs(pimu) < 1e-18L) ? 1.0L : pimu / std::sin(pimu);
  for (double& g : t.gen) g = 0.0;
  t.gen[0] = (double)mu;
  t.gen[1] = (double)nl;
  t.gen[2] = (double)gam1;
  t.gen[3] = (double)gam2;
  t.gen[4] = (double)gampl;
  t.gen[5] = (double)gammi;
  t.gen[6] = (double)fact;
}

// σ², β finite and > 0; ν ∈ {½, 3/2, 5/2} (closed forms) or ν ∈ [0.2, 3], the range the
// device K_ν evaluator is validated on (bessel_k.cuh; the MLE box of SURVEY §8d).
bool theta_valid(const double* th) {
  for (int i = 0; i < 3; ++i)
    if (!(th[i] > 0.0) || !std::isfinite(th[i])) return false;
  const double nu = th[2];
  return nu == 0.5 || nu == 1.5 || nu == 2.5 || (nu >= 0.2 && nu <= 3.0);
}

// ν-only table of the x > 2 K_ν evaluators (bessel_k.cuh), long double:
//   [0, 28):  cosh(t_k) − 1,  [28, 56): cosh(ν t_k)      (t_k = 0.15 k, trapezoid)
//   [56, 76): a_j = Π_{i≤j} (4ν² − (2i−1)²) / (8i)        (asymptotic series in 1/x)
void fill_nu_table(double* tab, double nu) {
  const long double ln = (long double)nu;
  for (int k = 1; k <= bv::kNuTrapNodes; ++k) {
    const long double t = 0.15L * (long double)k;
    tab[k - 1] = (double)(std::cosh(t) - 1.0L);
    tab[bv::kNuTrapNodes + k - 1] = (double)std::cosh(ln * t);
  }
  long double a = 1.0L;
  for (int j = 1; j <= bv::kNuAsymTerms; ++j) {
    const long double o = 2.0L * j - 1.0L;
    a *= (4.0L * ln * ln - o * o) / (8.0L * j);
    tab[2 * bv::kNuTrapNodes + j - 1] = (double)a;
  }
}

void fill_theta(bv::Theta& t, const double* th) {
  std::memset(&t, 0, sizeof(t));
  t.sigma2 = th[0];
  t.inv_beta = 1.0 / th[1];
  t.nu = th[2];
  if (th[2] == 0.5) t.kind = bv::kNuHalf;
  else if (th[2] == 1.5) t.kind = bv::kNu3Half;
  else if (th[2] == 2.5) t.kind = bv::kNu5Half;
  else {
    t.kind = bv::kNuGeneral;
    const long double ln = (long double)th[2];
    t.c_nu = (double)((long double)th[0] * std::pow(2.0L, 1.0L - ln) / std::tgamma(ln));
    fill_general_nu(t, th[2]);
  }
}

// θ into the pinned slot buffer: Theta in slot 0, the ν table right after it; `dev` = the
// device copy's base (the table's device address goes into Theta::nutab)
void fill_theta_buf(bv::Theta* host, const bv::Theta* dev, const double* th) {
  fill_theta(*host, th);
  double* tab = reinterpret_cast<double*>(host + 1);
  host->nutab = reinterpret_cast<const double*>(dev + 1);
  if (host->kind == bv::kNuGeneral) fill_nu_table(tab, th[2]);
}

void release(bv_handle* h) {
  if (!h) return;
  if (h->device >= 0) cudaSetDevice(h->device);
  for (int k = 0; k < 4; ++k) {
    if (h->exec[k]) cudaGraphExecDestroy(h->exec[k]);
    if (h->graph[k]) cudaGraphDestroy(h->graph[k]);
    h->exec[k] = nullptr;
    h->graph[k] = nullptr;
  }
  if (h->comm) ncclCommDestroy(h->comm);
  void* dev[] = {h->d_gslots, h->d_pts, h->d_nbr, h->d_desc, h->d_list, h->d_theta, h->d_u, h->d_d,
                 h->d_jlist, h->d_jacc, h->d_pre, h->d_pre_off, h->d_acc, h->d_min, h->d_perm_of_id, h->d_y_stage, h->d_tabs, h->d_tab_off, h->d_exptab};
  for (void* p : dev)
    if (p) cudaFree(p);
  if (h->h_theta) cudaFreeHost(h->h_theta);
  if (h->h_acc) cudaFreeHost(h->h_acc);
  for (int b = 0; b < bv_handle::kBranches; ++b) {
    if (h->side[b]) cudaStreamDestroy(h->side[b]);
    if (h->join_ev[b]) cudaEventDestroy(h->join_ev[b]);
  }
  if (h->fork_ev) cudaEventDestroy(h->fork_ev);
  if (h->ev_k0) cudaEventDestroy(h->ev_k0);
  if (h->ev_k1) cudaEventDestroy(h->ev_k1);
  if (h->stream) cudaStreamDestroy(h->stream);
  h->comm = nullptr;
}

template <class T>
bv_status upload(bv_handle* h, T** dst, const T* src, size_t count) {
  if (count == 0) count = 1;
  BV_CUDA(h, cudaMalloc((void**)dst, count * sizeof(T)));
  if (src) BV_CUDA(h, cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice));
  return BV_OK;
}

// One bucket (or a retry group) of positions through its kernel family.
cudaError_t launch_bucket(bv_handle* h, const Bucket& b, int kind, cudaStream_t st, const int32_t* list, int count,
                          unsigned long long* acc, double jit) {
  switch (b.kern) {
    case kKernCV:
      return bv::launch_cv(kind == 4 ? bv::kNuGeneral : kind, count, st, h->d_pts, h->d_nbr, h->d_desc, list,
                           h->d_theta, h->d_exptab, h->d_u, h->d_d, acc, h->kb);
    case kKernW:
      return bv::launch_block_w(kind, count, b.TI, st, h->d_pts, h->d_nbr, h->d_desc, list, h->d_theta, h->d_exptab,
                                h->d_u, h->d_d, acc, h->kb, h->d_pre, h->d_pre_off, jit);
    default:
      return bv::launch_block_v3(kind, count, b.TI, b.cap, st, h->d_pts, h->d_nbr, h->d_desc, list, h->d_theta,
                                 h->d_tabs, h->d_tab_off, h->d_exptab, h->d_u, h->d_d, acc, h->kb,
                                 h->d_gslots ? h->d_gslots + b.gs_off : nullptr, h->gs_grid, h->d_pre, h->d_pre_off,
                                 jit);
  }
}

}  // namespace

extern "C" {

const char* bv_version(void) { return "bvecchia-b200 0.1 (sm_100a, FP64)"; }

bv_status bv_nccl_unique_id(void* out128) {
  if (!out128) return BV_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return BV_ENCCL;
  std::memcpy(out128, &id, sizeof(id));
  return BV_OK;
}

bv_status bv_partition(int32_t bc, const int32_t* l, const int32_t* m, int32_t world, int32_t* cuts) {
  if (bc < 1 || world < 1 || !l || !m || !cuts) return BV_EINVAL;
  std::vector<double> prefix((size_t)bc + 1, 0.0);
  for (int32_t k = 0; k < bc; ++k) {
    const double N = (double)l[k] + (double)m[k];
    const double cost = N * N * N / 3.0 + 40.0 * (N * (N + 1.0) / 2.0);
    prefix[(size_t)k + 1] = prefix[k] + cost;
  }
  const double total = prefix[bc];
  cuts[0] = 0;
  int32_t k = 0;
  for (int32_t g = 1; g < world; ++g) {
    const double target = (double)g * total / (double)world;
    while (k < bc && prefix[k] < target) ++k;
    cuts[g] = k;
  }
  cuts[world] = bc;
  return BV_OK;
}

bv_status bv_fixed_encode(double t, uint32_t chunks[6]) {
  if (!chunks) return BV_EINVAL;
  return bv::fixed_encode(t, chunks) ? BV_EINVAL : BV_OK;
}

double bv_fixed_decode(const uint64_t acc[6]) {
  // Σ acc[c]·2^(32c) mod 2^192, as signed, times 2⁻⁶⁴
  unsigned __int128 carry = 0;
  uint64_t L[3];
  for (int w = 0; w < 3; ++w) {
    unsigned __int128 s = carry + (unsigned __int128)acc[2 * w] + ((unsigned __int128)acc[2 * w + 1] << 32);
    L[w] = (uint64_t)s;
    carry = s >> 64;
  }
  const bool neg = (L[2] >> 63) != 0;
  if (neg) {
    L[0] = ~L[0]; L[1] = ~L[1]; L[2] = ~L[2];
    L[0] += 1;
    if (L[0] == 0) { L[1] += 1; if (L[1] == 0) L[2] += 1; }
  }
  // correctly rounded: keep the top 63 significant bits with a sticky bit
  // (round-to-odd), then one rounding to double
  int top = -1;
  for (int w = 2; w >= 0 && top < 0; --w)
    if (L[w]) top = 64 * w + 63 - __builtin_clzll(L[w]);
  if (top < 0) return 0.0;
  auto bit_range = [&](int lo, int nbits) -> uint64_t {  // bits [lo, lo+nbits) of the 192-bit value
    uint64_t v = 0;
    for (int b = 0; b < nbits; ++b) {
      const int p = lo + b;
      if (p >= 0 && p < 192 && ((L[p >> 6] >> (p & 63)) & 1ull)) v |= (1ull << b);
    }
    return v;
  };
  const int lo = top - 62;  // 63 bits [lo, top]
  uint64_t mant = bit_range(lo, 63);
  if (lo > 0) {
    bool sticky = false;
    for (int p = 0; p < lo && !sticky; ++p) sticky = (L[p >> 6] >> (p & 63)) & 1ull;
    if (sticky) mant |= 1ull;
  }
  const double r = std::ldexp((double)mant, lo - 64);  // (double)mant rounds once (63 → 53 bits)
  return neg ? -r : r;
}

// Shared by bv_setup and the test-only bv_setup_rank_local (local = true: the
// rank's partition is laid out exactly as under NCCL, but no communicator is
// created and nothing is reduced across ranks).
static bv_status setup_impl(const bv_plan* plan, int device, int rank, int world, const void* nid, bool local,
                            bv_handle** out) {
  if (!out) return BV_EINVAL;
  *out = nullptr;
  bv_handle* h = nullptr;
  if (!plan) {
    g_setup_err = "plan is NULL";
    return BV_EINVAL;
  }
  const int64_t n = plan->n;
  const int d = plan->d;
  const int32_t bc = plan->bc;
  auto bad = [&](const std::string& m) {
    g_setup_err = m;
    return BV_EINVAL;
  };
  if (n < 1 || n > INT32_MAX) return bad("n must be in [1, 2^31)");
  if (d != 2 && d != 3) return bad("d must be 2 or 3");
  if (bc < 1 || (int64_t)bc > n) return bad("bc must be in [1, n]");
  if (!plan->locs || !plan->y || !plan->block_id || !plan->order || !plan->nbr_ptr)
    return bad("NULL plan array");
  for (int64_t i = 0; i < n * d; ++i)
    if (!std::isfinite(plan->locs[i])) return bad("locs[" + std::to_string(i) + "] is not finite");
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(plan->y[i])) return bad("y[" + std::to_string(i) + "] is not finite");
  std::vector<int64_t> bptr((size_t)bc + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    const int32_t b = plan->block_id[i];
    if (b < 0 || b >= bc) return bad("block_id[" + std::to_string(i) + "] out of range");
    bptr[(size_t)b + 1]++;
  }
  for (int32_t b = 0; b < bc; ++b)
    if (bptr[(size_t)b + 1] == 0) return bad("block " + std::to_string(b) + " is empty");
  for (int32_t b = 0; b < bc; ++b) bptr[(size_t)b + 1] += bptr[b];
  std::vector<int32_t> pos_of_block(bc, -1);
  for (int32_t k = 0; k < bc; ++k) {
    const int32_t b = plan->order[k];
    if (b < 0 || b >= bc || pos_of_block[b] >= 0) return bad("order is not a permutation (position " + std::to_string(k) + ")");
    pos_of_block[b] = k;
  }
  if (plan->nbr_ptr[0] != 0) return bad("nbr_ptr[0] != 0");
  for (int32_t k = 0; k < bc; ++k)
    if (plan->nbr_ptr[k + 1] < plan->nbr_ptr[k]) return bad("nbr_ptr decreases at " + std::to_string(k));
  const int64_t nnz = plan->nbr_ptr[bc];
  if (nnz > INT32_MAX) return bad("too many neighbour entries (> 2^31)");
  if (nnz > 0 && !plan->nbr_idx) return bad("nbr_idx is NULL");
  {
    std::vector<int32_t> stamp(n, -1);
    for (int32_t k = 0; k < bc; ++k)
      for (int64_t q = plan->nbr_ptr[k]; q < plan->nbr_ptr[k + 1]; ++q) {
        const int32_t id = plan->nbr_idx[q];
        if (id < 0 || id >= n) return bad("nbr_idx[" + std::to_string(q) + "] out of range");
        if (pos_of_block[plan->block_id[id]] >= k)
          return bad("neighbour " + std::to_string(id) + " of position " + std::to_string(k) +
                     " is not in an earlier block");
        if (stamp[id] == k) return bad("duplicate neighbour in position " + std::to_string(k));
        stamp[id] = k;
      }
  }
  // sizes per position
  std::vector<int32_t> L(bc), M(bc);
  for (int32_t k = 0; k < bc; ++k) {
    L[k] = (int32_t)(bptr[(size_t)plan->order[k] + 1] - bptr[plan->order[k]]);
    M[k] = (int32_t)(plan->nbr_ptr[k + 1] - plan->nbr_ptr[k]);
  }
  // kernel choice: classic-Vecchia positions (block size 1, m ≤ 31) → warp per position
  // (bv_cv.cu); joint sizes N ≤ 8·wmax − 1 → warp per block (bv_block_w.cu); larger →
  // the warp-specialised CTA kernel (bv_block_v3.cu).  BV_KERNEL=v3 / BV_NO_CV=1 /
  // BV_WMAX=t are A/B switches only.
  const char* kenv = std::getenv("BV_KERNEL");
  const bool force_v3 = kenv && std::string(kenv) == "v3";
  // Up to wmax (10) tile rows every bucket goes to the warp-per-block kernel; up to wbig only the
  // buckets with at least wbig_min blocks in the whole plan (one warp per block: a small
  // bucket of large blocks would leave its last blocks' single warps as the tail — measured
  // c5 m = 60: its 1,175 TI = 13 blocks 306 → 291 evals/s on the warp kernel; c4: its 21,460
  // TI = 15 and 19,044 TI = 16 blocks 229 → 247 → 252 on it; TI 17 neutral, TI 18 slower).
  const char* wenv = std::getenv("BV_WMAX");
  const char* wbenv = std::getenv("BV_WBIG");
  const char* wmenv = std::getenv("BV_WBIG_MIN");
  const int wmax = force_v3 ? 0 : std::max(0, std::min(bv::w_max_ti(), wenv ? std::atoi(wenv) : 10));
  const int wbig = force_v3 ? 0 : std::max(wmax, std::min(bv::w_max_ti(), wbenv ? std::atoi(wbenv) : 16));
  const int wbig_min = wmenv ? std::atoi(wmenv) : 2048;
  const int Nlimit = [&] {
    int N = 8;
    SlotTables st;
    st.build(64);
    while (N + 1 < 8 * 64) {
      const int TI = (N + 1 + 8) >> 3;
      if (bv::v3_smem_bytes(TI, st.cap[TI]) > kSmemOptin || bv::v3_maxt_for(TI) < 0) break;
      ++N;
    }
    return N;
  }();
  for (int32_t k = 0; k < bc; ++k)
    if (L[k] + M[k] > Nlimit)
      return bad("position " + std::to_string(k) + " has m+l = " + std::to_string(L[k] + M[k]) +
                 " > " + std::to_string(Nlimit) + " (largest joint size this build supports)");

  if (world < 1 || rank < 0 || rank >= world) return bad("invalid rank/world");
  if (world > 1 && !nid && !local) return bad("world > 1 needs an nccl_id");

  h = new bv_handle();
  h->device = device;
  h->rank = rank;
  h->world = world;
  h->local = local;
  h->n = n;
  h->d = d;
  h->bc = bc;
  h->wmax = wmax;
  auto bail = [&](bv_status st) {
    g_setup_err = h->err;
    release(h);
    delete h;
    return st;
  };
#define TRY(x)                         \
  do {                                 \
    bv_status s_ = (x);                \
    if (s_ != BV_OK) return bail(s_);  \
  } while (0)
#define TRYC(call)                                                                                   \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess) {                                                                         \
      h->err = std::string(#call) + ": " + cudaGetErrorString(e_);                                   \
      return bail(e_ == cudaErrorMemoryAllocation ? BV_ENOMEM : BV_ECUDA);                           \
    }                                                                                                \
  } while (0)

  TRYC(cudaSetDevice(device));
  TRYC(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));

  // partition (contiguous, cost-balanced)
  std::vector<int32_t> cuts((size_t)world + 1);
  bv_partition(bc, L.data(), M.data(), world, cuts.data());
  h->kb = cuts[rank];
  h->ke = cuts[(size_t)rank + 1];
  h->nq = h->ke - h->kb;

  // permuted point records: positions in order, block points in ascending id
  std::vector<int32_t> bidx(n);
  {
    std::vector<int64_t> fill(bptr.begin(), bptr.end() - 1);
    for (int64_t i = 0; i < n; ++i) bidx[fill[plan->block_id[i]]++] = (int32_t)i;
  }
  std::vector<int32_t> pstart((size_t)bc + 1, 0);
  for (int32_t k = 0; k < bc; ++k) pstart[(size_t)k + 1] = pstart[k] + L[k];
  std::vector<int32_t> perm_of_id(n);
  std::vector<bv::PointRec> pts(n);
  for (int32_t k = 0; k < bc; ++k) {
    const int32_t b = plan->order[k];
    for (int32_t a = 0; a < L[k]; ++a) {
      const int32_t id = bidx[bptr[b] + a];
      const int32_t p = pstart[k] + a;
      perm_of_id[id] = p;
      const double* s = plan->locs + (size_t)id * d;
      pts[p] = bv::PointRec{s[0], s[1], d == 3 ? s[2] : 0.0, plan->y[id]};
    }
  }
  // this rank's descriptors and remapped neighbour lists
  const int64_t nb0 = plan->nbr_ptr[h->kb], nb1 = plan->nbr_ptr[h->ke];
  std::vector<int32_t> nbr((size_t)(nb1 - nb0));
  for (int64_t q = nb0; q < nb1; ++q) nbr[(size_t)(q - nb0)] = perm_of_id[plan->nbr_idx[q]];
  std::vector<bv::BlockDesc> desc((size_t)h->nq);
  for (int32_t q = 0; q < h->nq; ++q) {
    const int32_t k = h->kb + q;
    desc[q] = bv::BlockDesc{pstart[k], L[k], M[k], (int32_t)(plan->nbr_ptr[k] - nb0)};
  }
  // buckets: key = TI = ⌈(N+1)/8⌉ (0 for classic-Vecchia positions, launched last);
  // largest first, inside a bucket N descending, then position
  std::vector<int32_t> list((size_t)h->nq);
  for (int32_t q = 0; q < h->nq; ++q) list[q] = q;
  auto Nq = [&](int32_t q) { return desc[q].l + desc[q].m; };
  const char* nocv = std::getenv("BV_NO_CV");
  const bool cv_ok = !(nocv && nocv[0] == '1');
  auto is_cv = [&](int32_t q) { return cv_ok && desc[q].l == 1 && desc[q].m <= 31; };
  auto bkey = [&](int32_t q) { return is_cv(q) ? 0 : (Nq(q) + 8) >> 3; };
  std::stable_sort(list.begin(), list.end(), [&](int32_t a, int32_t b) {
    if (bkey(a) != bkey(b)) return bkey(a) > bkey(b);
    if (Nq(a) != Nq(b)) return Nq(a) > Nq(b);
    return a < b;
  });
  // bucket sizes over the WHOLE plan (not this rank's range): the kernel of a tile-row count
  // is a property of the plan, so every world size runs every block on the same kernel and
  // ℓ is bitwise the same for any G (§6)
  std::vector<int64_t> glob_count(64 + 2, 0);
  for (int32_t k = 0; k < bc; ++k) {
    const bool cv = cv_ok && L[k] == 1 && M[k] <= 31;
    const int TI = (L[k] + M[k] + 8) >> 3;
    if (!cv && TI < (int)glob_count.size()) ++glob_count[(size_t)TI];
  }
  SlotTables slot_tables;
  int TImax_all = 1;
  for (int32_t q = 0; q < h->nq; ++q) TImax_all = std::max(TImax_all, (Nq(q) + 8) >> 3);
  slot_tables.build(TImax_all);
  h->cap_of = slot_tables.cap;
  h->gsoff_of.assign((size_t)TImax_all + 1, 0);
  bool any_w = false;
  size_t max_smem = 0, gs_total = 0;
  {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
    h->gs_grid = 2 * sms;
  }
  for (int32_t i = 0; i < h->nq;) {
    int32_t j = i;
    while (j < h->nq && bkey(list[j]) == bkey(list[i])) ++j;
    const int TI = bkey(list[i]);
    Bucket bk{TI, j - i, i, TI ? slot_tables.cap[TI] : 0};
    if (TI == 0) {
      bk.kern = kKernCV;
    } else if (TI <= wmax || (TI <= wbig && glob_count[(size_t)TI] >= wbig_min)) {
      bk.kern = kKernW;
      any_w = true;
    } else {
      bk.kern = kKernV3;
      if (bv::v3_global_slots(TI)) {
        bk.gs_off = gs_total;
        h->gsoff_of[TI] = gs_total;
        gs_total += (size_t)std::min(j - i, h->gs_grid) * slot_tables.cap[TI] * 64;
      }
      max_smem = std::max(max_smem, bv::v3_smem_bytes(TI, slot_tables.cap[TI]));
    }
    h->buckets.push_back(bk);
    if (TI > 0) {
      if ((int)h->kern_of.size() <= TI) h->kern_of.resize((size_t)TI + 1, -1);
      h->kern_of[(size_t)TI] = bk.kern;
    }
    i = j;
  }

  if (gs_total > 0) TRY(upload<double>(h, &h->d_gslots, nullptr, gs_total));
  TRY(upload(h, &h->d_pts, pts.data(), pts.size()));
  TRY(upload(h, &h->d_nbr, nbr.data(), nbr.size()));
  TRY(upload(h, &h->d_desc, desc.data(), desc.size()));
  h->h_N.resize((size_t)h->nq);
  for (int32_t q = 0; q < h->nq; ++q) h->h_N[q] = Nq(q);
  {
    // General-ν pre-generation (bv_block_v3.cu, bv_pregen_kernel): when every block's
    // packed Σ fits a small L2-resident buffer (≤ 64 MB: c1, c2), the K_ν entries are
    // evaluated by one all-SM kernel instead of inside the block kernels.
    // BV_NO_PREGEN=1 disables it (A/B and the bitwise-equality test).
    const char* npg = std::getenv("BV_NO_PREGEN");
    std::vector<int64_t> off((size_t)h->nq + 1, 0);
    for (int32_t q = 0; q < h->nq; ++q) off[(size_t)q + 1] = off[q] + (int64_t)Nq(q) * (Nq(q) + 1) / 2;
    constexpr int64_t kPreMaxBytes = 64ll << 20;
    if (!(npg && npg[0] == '1') && h->nq > 0 && off[(size_t)h->nq] * 8 <= kPreMaxBytes) {
      TRY(upload<double>(h, &h->d_pre, nullptr, (size_t)std::max<int64_t>(1, off[(size_t)h->nq])));
      TRY(upload(h, &h->d_pre_off, off.data(), (size_t)h->nq));
      h->pre_chunks = std::max(1, std::min(64, (16 * 148 + h->nq - 1) / h->nq));
    }
  }
  TRY(upload(h, &h->d_list, list.data(), list.size()));
  TRY(upload(h, &h->d_perm_of_id, perm_of_id.data(), perm_of_id.size()));
  h->h_perm_of_id = perm_of_id;
  TRY(upload<double>(h, &h->d_y_stage, nullptr, (size_t)n));
  TRY(upload<bv::Theta>(h, &h->d_theta, nullptr, bv::kThetaSlots));
  TRY(upload<double>(h, &h->d_u, nullptr, (size_t)h->nq));
  TRY(upload<double>(h, &h->d_d, nullptr, (size_t)h->nq));
  TRY(upload<unsigned long long>(h, &h->d_acc, nullptr, bv::kAccSlots));
  TRY(upload<unsigned long long>(h, &h->d_min, nullptr, 1));
  TRYC(cudaMallocHost((void**)&h->h_theta, sizeof(bv::Theta) * bv::kThetaSlots));
  TRYC(cudaMallocHost((void**)&h->h_acc, sizeof(unsigned long long) * bv::kAccSlots));
  std::memset(h->h_theta, 0, sizeof(bv::Theta) * bv::kThetaSlots);
  TRY(upload(h, &h->d_tabs, slot_tables.tabs.data(), slot_tables.tabs.size()));
  TRY(upload(h, &h->d_tab_off, slot_tables.off.data(), slot_tables.off.size()));
  {
    double et[64];  // 2^{−j/64}, correctly rounded via long double (exp_neg in matern.cuh)
    for (int j = 0; j < 64; ++j) et[j] = (double)std::exp2(-(long double)j / 64.0L);
    TRY(upload(h, &h->d_exptab, et, 64));
  }
  TRYC(bv::prepare_block_v3(std::max<size_t>(max_smem, 1024)));
  if (any_w || wmax > 0) TRYC(bv::prepare_block_w());

  if (world > 1 && !local) {
    ncclUniqueId id;
    std::memcpy(&id, nid, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&h->comm, world, id, rank);
    if (r != ncclSuccess) {
      h->err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
      return bail(BV_ENCCL);
    }
  }

  TRYC(cudaEventCreate(&h->ev_k0));
  TRYC(cudaEventCreate(&h->ev_k1));
  TRYC(cudaEventCreateWithFlags(&h->fork_ev, cudaEventDisableTiming));
  for (int b = 0; b < bv_handle::kBranches; ++b) {
    TRYC(cudaStreamCreateWithFlags(&h->side[b], cudaStreamNonBlocking));
    TRYC(cudaEventCreateWithFlags(&h->join_ev[b], cudaEventDisableTiming));
  }
  // Capture the per-evaluation graph, one per Matérn kind (the block kernels are
  // specialised on it; the kind is chosen from ν at each evaluation):
  //   θ upload → zero the accumulator → bucket kernels (largest first, spread
  //   over kBranches concurrent graph branches so small buckets overlap big
  //   ones instead of draining the GPU between launches; each block adds its
  //   exact term atomically) → [ncclAllReduce] → result to the host.
  for (int kind = 0; kind < 4; ++kind) {
    TRYC(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    cudaError_t e = cudaMemcpyAsync(h->d_theta, h->h_theta, sizeof(bv::Theta) * bv::kThetaSlots,
                                    cudaMemcpyHostToDevice, h->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(h->d_acc, 0, sizeof(unsigned long long) * 7, h->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(h->d_acc + 7, 0xff, sizeof(unsigned long long), h->stream);
    if (e == cudaSuccess) e = cudaEventRecordWithFlags(h->ev_k0, h->stream, cudaEventRecordExternal);
    const bool pre = kind == bv::kNuGeneral && h->d_pre != nullptr;
    if (e == cudaSuccess && pre)
      e = bv::launch_pregen(h->nq, h->pre_chunks, h->stream, h->d_pts, h->d_nbr, h->d_desc, h->d_theta, h->d_exptab,
                            h->d_pre_off, h->d_pre);
    if (e == cudaSuccess) e = cudaEventRecord(h->fork_ev, h->stream);
    const int nbr_streams = std::min<int>(bv_handle::kBranches, std::max<int>(1, (int)h->buckets.size()));
    for (int b = 0; b < nbr_streams && e == cudaSuccess; ++b) e = cudaStreamWaitEvent(h->side[b], h->fork_ev, 0);
    for (size_t bi = 0; bi < h->buckets.size() && e == cudaSuccess; ++bi) {
      const Bucket& b = h->buckets[bi];
      e = launch_bucket(h, b, pre ? 4 : kind, h->side[bi % nbr_streams], h->d_list + b.offset, b.count, h->d_acc, 0.0);
    }
    for (int b = 0; b < nbr_streams && e == cudaSuccess; ++b) {
      e = cudaEventRecord(h->join_ev[b], h->side[b]);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(h->stream, h->join_ev[b], 0);
    }
    if (e == cudaSuccess) e = cudaEventRecordWithFlags(h->ev_k1, h->stream, cudaEventRecordExternal);
    ncclResult_t r = ncclSuccess;
    if (e == cudaSuccess && h->comm)
      r = ncclAllReduce(h->d_acc, h->d_acc, 7, ncclUint64, ncclSum, h->comm, h->stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(h->h_acc, h->d_acc, sizeof(unsigned long long) * bv::kAccSlots, cudaMemcpyDeviceToHost,
                          h->stream);
    cudaError_t e2 = cudaStreamEndCapture(h->stream, &h->graph[kind]);
    if (e != cudaSuccess || e2 != cudaSuccess) {
      h->err = std::string("graph capture: ") + cudaGetErrorString(e != cudaSuccess ? e : e2);
      return bail(BV_ECUDA);
    }
    if (r != ncclSuccess) {
      h->err = std::string("ncclAllReduce (capture): ") + ncclGetErrorString(r);
      return bail(BV_ENCCL);
    }
    TRYC(cudaGraphInstantiate(&h->exec[kind], h->graph[kind], 0));
  }
  *out = h;
  g_setup_err.clear();
#undef TRY
#undef TRYC
  return BV_OK;
}

bv_status bv_setup(const bv_plan* plan, const bv_dist* dist, bv_handle** out) {
  int device = 0, rank = 0, world = 1;
  const void* nid = nullptr;
  if (dist) {
    device = dist->device;
    rank = dist->rank;
    world = dist->world;
    nid = dist->nccl_id;
  }
  return setup_impl(plan, device, rank, world, nid, false, out);
}

bv_status bv_setup_rank_local(const bv_plan* plan, int32_t device, int32_t rank, int32_t world, bv_handle** out) {
  return setup_impl(plan, device, rank, world, nullptr, true, out);
}

// Optional jitter mode (reading G15b; SPEC.md:197, :238 schedule with
// base_scale = σ²): after an evaluation in which some block failed, every
// failed position (d_k = NaN) is recomputed from scratch by the same block
// kernels with ε·σ² added to every diagonal entry of its joint matrix, ε = 1e-10,
// 1e-8, 1e-6, the first success kept — any joint size the evaluation supports.
// The retry's exact terms go to their own accumulator and are added slot-wise
// to the evaluation's (integer sums: still order-independent).  Collective when
// world > 1 (every rank sees the same global failure count and enters).
constexpr bv_status kJitterDefer = (bv_status)-1;
static bv_status jitter_retry(bv_handle* h, const unsigned long long* acc, double* loglik) {
  static const double kSched[3] = {1e-10, 1e-8, 1e-6};
  std::vector<double> dh((size_t)h->nq);
  if (h->nq > 0) BV_CUDA(h, cudaMemcpy(dh.data(), h->d_d, sizeof(double) * h->nq, cudaMemcpyDeviceToHost));
  std::vector<int32_t> F;
  for (int32_t q = 0; q < h->nq; ++q)
    if (std::isnan(dh[(size_t)q])) F.push_back(q);
  const uint64_t nan_local = F.size();
  uint64_t sums[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};  // [0..5] retry chunk sums, [6] still failed, [7] events, [8] NaN
  if (!F.empty()) {
    if (!h->d_jlist) BV_CUDA(h, cudaMalloc(&h->d_jlist, sizeof(int32_t) * (size_t)h->nq));
    if (!h->d_jacc) BV_CUDA(h, cudaMalloc(&h->d_jacc, sizeof(unsigned long long) * 9));
    const double s2 = h->h_theta->sigma2;
    const int kind = (h->h_theta->kind == bv::kNuGeneral && h->d_pre) ? 4 : h->h_theta->kind;
    std::vector<int32_t> R = F;
    for (int e = 0; e < 3 && !R.empty(); ++e) {
      // group by tile rows (the kernel family follows from TI exactly as in the evaluation)
      auto ti = [&](int32_t q) { return (h->h_N[(size_t)q] + 8) >> 3; };
      std::stable_sort(R.begin(), R.end(), [&](int32_t a, int32_t b) { return ti(a) < ti(b); });
      unsigned long long a0[bv::kAccSlots] = {0, 0, 0, 0, 0, 0, 0, ~0ull};
      BV_CUDA(h, cudaMemcpyAsync(h->d_jacc, a0, sizeof(a0), cudaMemcpyHostToDevice, h->stream));
      BV_CUDA(h, cudaMemcpyAsync(h->d_jlist, R.data(), sizeof(int32_t) * R.size(), cudaMemcpyHostToDevice,
                                 h->stream));
      for (size_t i = 0; i < R.size();) {
        size_t j = i;
        while (j < R.size() && ti(R[j]) == ti(R[i])) ++j;
        const int TI = ti(R[i]);
        Bucket b{TI, (int)(j - i), 0, h->cap_of[(size_t)TI]};
        // the kernel this TI's bucket runs in the evaluation (classic-Vecchia positions, which
        // have no block-kernel bucket, by the size rule alone)
        b.kern = (size_t)TI < h->kern_of.size() && h->kern_of[(size_t)TI] >= 0 ? h->kern_of[(size_t)TI]
                 : TI <= h->wmax                                            ? kKernW
                                                                            : kKernV3;
        b.gs_off = h->gsoff_of[(size_t)TI];
        BV_CUDA(h, launch_bucket(h, b, kind, h->stream, h->d_jlist + i, b.count, h->d_jacc, kSched[e] * s2));
        i = j;
      }
      BV_CUDA(h, cudaMemcpyAsync(a0, h->d_jacc, sizeof(a0), cudaMemcpyDeviceToHost, h->stream));
      BV_CUDA(h, cudaMemcpyAsync(dh.data(), h->d_d, sizeof(double) * h->nq, cudaMemcpyDeviceToHost, h->stream));
      BV_CUDA(h, cudaStreamSynchronize(h->stream));
      std::vector<int32_t> R2;
      for (int32_t q : R)
        if (std::isnan(dh[(size_t)q])) R2.push_back(q);
      if (a0[6] > R2.size()) {  // a retried block became PD but its term is out of the exact range
        h->failed_pos = (int32_t)(a0[7] >> 8);
        *loglik = -INFINITY;
        return fail(h, BV_EINVAL, "block term at position " + std::to_string(h->failed_pos) + " exceeds 2^96");
      }
      for (int i = 0; i < 6; ++i) sums[i] += a0[i];
      sums[7] += R.size() - R2.size();
      R.swap(R2);
    }
    F.swap(R);
    sums[6] = F.size();
  }
  sums[8] = nan_local;
  if (h->comm) {
    if (!h->d_jacc) BV_CUDA(h, cudaMalloc(&h->d_jacc, sizeof(unsigned long long) * 9));
    BV_CUDA(h, cudaMemcpyAsync(h->d_jacc, sums, sizeof(sums), cudaMemcpyHostToDevice, h->stream));
    BV_NCCL(h, ncclAllReduce(h->d_jacc, h->d_jacc, 9, ncclUint64, ncclSum, h->comm, h->stream));
    BV_CUDA(h, cudaMemcpyAsync(sums, h->d_jacc, sizeof(sums), cudaMemcpyDeviceToHost, h->stream));
    BV_CUDA(h, cudaStreamSynchronize(h->stream));
  }
  if (sums[8] != acc[6]) return kJitterDefer;  // a non-NaN failure (term range): caller reports it
  h->jitter_events = (int64_t)sums[7];
  if (sums[6] != 0) {
    unsigned long long mn = F.empty() ? ~0ull : ((unsigned long long)(h->kb + *std::min_element(F.begin(), F.end())));
    if (h->comm) {
      BV_CUDA(h, cudaMemcpyAsync(h->d_min, &mn, 8, cudaMemcpyHostToDevice, h->stream));
      BV_NCCL(h, ncclAllReduce(h->d_min, h->d_min, 1, ncclUint64, ncclMin, h->comm, h->stream));
      BV_CUDA(h, cudaMemcpyAsync(&mn, h->d_min, 8, cudaMemcpyDeviceToHost, h->stream));
      BV_CUDA(h, cudaStreamSynchronize(h->stream));
    }
    h->failed_pos = (int32_t)mn;
    *loglik = -INFINITY;
    return fail(h, BV_ENOTPD, "block at position " + std::to_string(h->failed_pos) +
                                  " is not positive definite after the jitter schedule");
  }
  uint64_t a6[6];
  for (int i = 0; i < 6; ++i) a6[i] = acc[i] + sums[i];
  for (int i = 0; i < 6; ++i) h->h_acc[i] = a6[i];  // bv_loglik_acc reports the jittered sum
  h->h_acc[6] = 0;
  h->h_acc[7] = ~0ull;
  *loglik = bv_fixed_decode(a6);
  return BV_OK;
}

static bv_status run_eval(bv_handle* h, const double theta[3], double* loglik) {
  h->failed_pos = -1;
  h->jitter_events = 0;
  h->err.clear();
  if (!theta || !loglik) return fail(h, BV_EINVAL, "NULL argument");
  if (!theta_valid(theta)) return fail(h, BV_EINVAL, "theta: sigma2, beta must be finite and > 0; nu in {0.5, 1.5, 2.5} or [0.2, 3]");
  BV_CUDA(h, cudaSetDevice(h->device));
  fill_theta_buf(h->h_theta, h->d_theta, theta);
  h->last_kind = h->h_theta->kind;
  BV_CUDA(h, cudaGraphLaunch(h->exec[h->h_theta->kind], h->stream));
  BV_CUDA(h, cudaStreamSynchronize(h->stream));
  const unsigned long long* acc = h->h_acc;
  if (acc[6] != 0 && h->jitter) {
    const bv_status js = jitter_retry(h, acc, loglik);
    if (js != kJitterDefer) return js;
  }
  if (acc[6] != 0) {
    unsigned long long mn = acc[7];
    if (h->comm) {
      BV_CUDA(h, cudaMemcpyAsync(h->d_min, &mn, 8, cudaMemcpyHostToDevice, h->stream));
      BV_NCCL(h, ncclAllReduce(h->d_min, h->d_min, 1, ncclUint64, ncclMin, h->comm, h->stream));
      BV_CUDA(h, cudaMemcpyAsync(&mn, h->d_min, 8, cudaMemcpyDeviceToHost, h->stream));
      BV_CUDA(h, cudaStreamSynchronize(h->stream));
    }
    h->failed_pos = (int32_t)(mn >> 8);
    *loglik = -INFINITY;
    if ((mn & 0xff) == bv::kNotPD)
      return fail(h, BV_ENOTPD, "block at position " + std::to_string(h->failed_pos) + " is not positive definite");
    return fail(h, BV_EINVAL, "block term at position " + std::to_string(h->failed_pos) + " exceeds 2^96");
  }
  uint64_t a6[6];
  for (int i = 0; i < 6; ++i) a6[i] = acc[i];
  *loglik = bv_fixed_decode(a6);
  return BV_OK;
}

bv_status bv_loglik(bv_handle* h, const double theta[3], double* loglik) {
  if (!h) return BV_EINVAL;
  return run_eval(h, theta, loglik);
}

bv_status bv_loglik_terms(bv_handle* h, const double theta[3], double* loglik, double* logdet, double* quad) {
  if (!h) return BV_EINVAL;
  bv_status st = run_eval(h, theta, loglik);
  if (st != BV_OK && st != BV_ENOTPD) return st;
  if (h->nq > 0) {
    if (logdet) BV_CUDA(h, cudaMemcpy(logdet, h->d_d, sizeof(double) * h->nq, cudaMemcpyDeviceToHost));
    if (quad) BV_CUDA(h, cudaMemcpy(quad, h->d_u, sizeof(double) * h->nq, cudaMemcpyDeviceToHost));
  }
  return st;
}

bv_status bv_loglik_acc(bv_handle* h, const double theta[3], uint64_t acc_out[8]) {
  if (!h || !acc_out) return BV_EINVAL;
  double ll = 0.0;
  const bv_status st = run_eval(h, theta, &ll);
  if (st != BV_OK && st != BV_ENOTPD) return st;
  for (int i = 0; i < bv::kAccSlots; ++i) acc_out[i] = h->h_acc[i];
  return st;
}

// y is validated only when the evaluation fails: a non-finite y_i reaches the y row of its own
// block (u = Σ L_Nj² becomes inf/NaN, the term's encoding reports it), so a successful
// evaluation proves y finite and the host never scans 8n bytes on the hot path (a single-core
// scan of c4's 8 MB is ~0.5 ms per call, a tenth of the evaluation).
bv_status bv_loglik_host_y(bv_handle* h, const double* y, const double theta[3], double* loglik) {
  if (!h || !y) return BV_EINVAL;
  BV_CUDA(h, cudaSetDevice(h->device));
  BV_CUDA(h, cudaMemcpyAsync(h->d_y_stage, y, sizeof(double) * h->n, cudaMemcpyHostToDevice, h->stream));
  BV_CUDA(h, bv::launch_scatter_y(h->d_y_stage, h->d_perm_of_id, h->n, h->d_pts, h->stream));
  const bv_status st = run_eval(h, theta, loglik);
  if (st != BV_OK && st != BV_ECUDA) {
    for (int64_t i = 0; i < h->n; ++i)
      if (!std::isfinite(y[i])) {
        if (loglik) *loglik = -INFINITY;
        h->failed_pos = -1;
        return fail(h, BV_EINVAL, "y[" + std::to_string(i) + "] is not finite");
      }
  }
  return st;
}

bv_status bv_set_jitter(bv_handle* h, int32_t enable) {
  if (!h) return BV_EINVAL;
  h->jitter = enable != 0;
  return BV_OK;
}

bv_status bv_jitter_events(const bv_handle* h, int64_t* events) {
  if (!h || !events) return BV_EINVAL;
  *events = h->jitter_events;
  return BV_OK;
}

bv_status bv_owned_range(const bv_handle* h, int32_t* k_begin, int32_t* k_end) {
  if (!h || !k_begin || !k_end) return BV_EINVAL;
  *k_begin = h->kb;
  *k_end = h->ke;
  return BV_OK;
}

bv_status bv_last_error(const bv_handle* h, int32_t* failed_position, const char** msg) {
  if (!h) {
    if (msg) *msg = g_setup_err.c_str();
    if (failed_position) *failed_position = -1;
    return BV_OK;
  }
  if (failed_position) *failed_position = h->failed_pos;
  if (msg) *msg = h->err.c_str();
  return BV_OK;
}

void* bv_stream(const bv_handle* h) { return h ? (void*)h->stream : nullptr; }

// Debug builds only (-DBV_PROFILE_PHASES, libbv_prof.so): per-phase cycle sums.
int bv_debug_v3_cycles(unsigned long long* out16, int reset) { return bv::debug_v3_cycles(out16, reset); }

bv_status bv_last_kernel_ms(const bv_handle* h, float* ms) {
  if (!h || !ms) return BV_EINVAL;
  cudaError_t e = cudaEventElapsedTime(ms, h->ev_k0, h->ev_k1);
  return e == cudaSuccess ? BV_OK : BV_ECUDA;
}

int32_t bv_launches_per_eval(const bv_handle* h) {
  if (!h) return 0;
  int32_t c = 0;  // one kernel per non-empty bucket (the reduction is fused into them)
  for (const Bucket& b : h->buckets)
    if (b.count > 0) ++c;
  if (h->last_kind == bv::kNuGeneral && h->d_pre) ++c;  // the general-ν pre-generation kernel
  return c;
}

void bv_destroy(bv_handle* h) {
  if (!h) return;
  release(h);
  delete h;
}

}  // extern "C"

// ---------------------------------------------------------------- prediction (Alg. 2)
bv_status bv_predict(bv_handle* h, const double theta[3], const bv_pred_plan* pp, double* mean, double* var,
                     double* cov) {
  if (!h) return BV_EINVAL;
  h->failed_pos = -1;
  h->err.clear();
  if (!theta || !pp || !mean) return fail(h, BV_EINVAL, "NULL argument");
  if (!theta_valid(theta)) return fail(h, BV_EINVAL, "theta: sigma2, beta must be finite and > 0; nu in {0.5, 1.5, 2.5} or [0.2, 3]");
  const int64_t nn = pp->n_new;
  const int32_t bc = pp->bc_new;
  const int d = h->d;
  if (nn < 1 || nn > INT32_MAX) return fail(h, BV_EINVAL, "n_new must be in [1, 2^31)");
  if (bc < 1 || (int64_t)bc > nn) return fail(h, BV_EINVAL, "bc_new must be in [1, n_new]");
  if (!pp->locs_new || !pp->block_id || !pp->nbr_ptr) return fail(h, BV_EINVAL, "NULL pred plan array");
  for (int64_t i = 0; i < nn * d; ++i)
    if (!std::isfinite(pp->locs_new[i])) return fail(h, BV_EINVAL, "locs_new[" + std::to_string(i) + "] is not finite");
  std::vector<int64_t> bptr((size_t)bc + 1, 0);
  for (int64_t i = 0; i < nn; ++i) {
    const int32_t b = pp->block_id[i];
    if (b < 0 || b >= bc) return fail(h, BV_EINVAL, "block_id[" + std::to_string(i) + "] out of range");
    bptr[(size_t)b + 1]++;
  }
  for (int32_t b = 0; b < bc; ++b)
    if (bptr[(size_t)b + 1] == 0) return fail(h, BV_EINVAL, "prediction block " + std::to_string(b) + " is empty");
  for (int32_t b = 0; b < bc; ++b) bptr[(size_t)b + 1] += bptr[b];
  if (pp->nbr_ptr[0] != 0) return fail(h, BV_EINVAL, "nbr_ptr[0] != 0");
  for (int32_t b = 0; b < bc; ++b)
    if (pp->nbr_ptr[b + 1] < pp->nbr_ptr[b]) return fail(h, BV_EINVAL, "nbr_ptr decreases at " + std::to_string(b));
  const int64_t nnz = pp->nbr_ptr[bc];
  if (nnz > INT32_MAX) return fail(h, BV_EINVAL, "too many neighbour entries (> 2^31)");
  if (nnz > 0 && !pp->nbr_idx) return fail(h, BV_EINVAL, "nbr_idx is NULL");
  constexpr int kPredNmax = 235;  // predict_smem_bytes(235) ≤ 232448
  size_t smax = 0;
  {
    // duplicate check: h->pred_stamp[id] holds the last (call epoch, block) that used id, so the
    // n-sized table is allocated once per handle instead of once per call
    if (h->pred_stamp.size() != (size_t)h->n) h->pred_stamp.assign((size_t)h->n, -1);
    std::vector<int64_t>& stamp = h->pred_stamp;
    const int64_t base = h->pred_epoch;
    h->pred_epoch += bc;
    for (int32_t b = 0; b < bc; ++b) {
      for (int64_t q = pp->nbr_ptr[b]; q < pp->nbr_ptr[b + 1]; ++q) {
        const int32_t id = pp->nbr_idx[q];
        if (id < 0 || id >= h->n) return fail(h, BV_EINVAL, "nbr_idx[" + std::to_string(q) + "] out of range");
        if (stamp[id] == base + b)
          return fail(h, BV_EINVAL, "duplicate neighbour in prediction block " + std::to_string(b));
        stamp[id] = base + b;
      }
      const int N = (int)(pp->nbr_ptr[b + 1] - pp->nbr_ptr[b] + bptr[(size_t)b + 1] - bptr[b]);
      if (N > kPredNmax)
        return fail(h, BV_EINVAL, "prediction block " + std::to_string(b) + " has m+l = " + std::to_string(N) +
                                      " > " + std::to_string(kPredNmax));
      smax = std::max(smax, bv::predict_smem_bytes(N));
    }
  }
  // block-contiguous new-point records (ascending id inside a block), descriptors, remapped neighbours
  std::vector<bv::PointRec> np((size_t)nn);
  std::vector<int32_t> order_new((size_t)nn);
  {
    std::vector<int64_t> fill(bptr.begin(), bptr.end() - 1);
    for (int64_t i = 0; i < nn; ++i) order_new[(size_t)fill[pp->block_id[i]]++] = (int32_t)i;
  }
  for (int64_t p = 0; p < nn; ++p) {
    const double* s = pp->locs_new + (size_t)order_new[p] * d;
    np[p] = bv::PointRec{s[0], s[1], d == 3 ? s[2] : 0.0, 0.0};
  }
  std::vector<bv::BlockDesc> desc((size_t)bc);
  std::vector<int64_t> coff((size_t)bc + 1, 0);
  for (int32_t b = 0; b < bc; ++b) {
    const int64_t l = bptr[(size_t)b + 1] - bptr[b];
    desc[b] = bv::BlockDesc{(int32_t)bptr[b], (int32_t)l, (int32_t)(pp->nbr_ptr[b + 1] - pp->nbr_ptr[b]),
                            (int32_t)pp->nbr_ptr[b]};
    coff[(size_t)b + 1] = coff[b] + l * l;
  }
  std::vector<int32_t> nbr((size_t)std::max<int64_t>(nnz, 1), 0);
  for (int64_t q = 0; q < nnz; ++q) nbr[(size_t)q] = h->h_perm_of_id[pp->nbr_idx[q]];

  BV_CUDA(h, cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  bv::PointRec* d_np = nullptr;
  int32_t *d_nbr = nullptr, *d_status = nullptr;
  bv::BlockDesc* d_desc = nullptr;
  int64_t* d_coff = nullptr;
  double *d_mean = nullptr, *d_var = nullptr, *d_cov = nullptr;
  auto release = [&]() {
    cudaFreeAsync(d_np, st);
    cudaFreeAsync(d_nbr, st);
    cudaFreeAsync(d_status, st);
    cudaFreeAsync(d_desc, st);
    cudaFreeAsync(d_coff, st);
    cudaFreeAsync(d_mean, st);
    cudaFreeAsync(d_var, st);
    cudaFreeAsync(d_cov, st);
    cudaStreamSynchronize(st);
  };
#define PCALL(call)                                                                                     \
  do {                                                                                                  \
    cudaError_t e_ = (call);                                                                            \
    if (e_ != cudaSuccess) {                                                                            \
      release();                                                                                        \
      return fail(h, e_ == cudaErrorMemoryAllocation ? BV_ENOMEM : BV_ECUDA,                            \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                                  \
    }                                                                                                   \
  } while (0)
  PCALL(cudaMallocAsync((void**)&d_np, sizeof(bv::PointRec) * np.size(), st));
  PCALL(cudaMallocAsync((void**)&d_nbr, sizeof(int32_t) * nbr.size(), st));
  PCALL(cudaMallocAsync((void**)&d_status, sizeof(int32_t) * bc, st));
  PCALL(cudaMallocAsync((void**)&d_desc, sizeof(bv::BlockDesc) * bc, st));
  PCALL(cudaMallocAsync((void**)&d_coff, sizeof(int64_t) * coff.size(), st));
  PCALL(cudaMallocAsync((void**)&d_mean, sizeof(double) * nn, st));
  PCALL(cudaMallocAsync((void**)&d_var, sizeof(double) * nn, st));
  if (cov) PCALL(cudaMallocAsync((void**)&d_cov, sizeof(double) * std::max<int64_t>(coff[bc], 1), st));
  PCALL(cudaMemcpyAsync(d_np, np.data(), sizeof(bv::PointRec) * np.size(), cudaMemcpyHostToDevice, st));
  PCALL(cudaMemcpyAsync(d_nbr, nbr.data(), sizeof(int32_t) * nbr.size(), cudaMemcpyHostToDevice, st));
  PCALL(cudaMemcpyAsync(d_desc, desc.data(), sizeof(bv::BlockDesc) * bc, cudaMemcpyHostToDevice, st));
  PCALL(cudaMemcpyAsync(d_coff, coff.data(), sizeof(int64_t) * coff.size(), cudaMemcpyHostToDevice, st));
  fill_theta_buf(h->h_theta, h->d_theta, theta);
  PCALL(cudaMemcpyAsync(h->d_theta, h->h_theta, sizeof(bv::Theta) * bv::kThetaSlots, cudaMemcpyHostToDevice, st));
  PCALL(bv::prepare_predict(std::max<size_t>(smax, 1024)));
  PCALL(cudaEventRecord(h->ev_k0, st));  // bv_last_kernel_ms then reports the prediction kernel
  PCALL(bv::launch_predict(bc, smax, st, h->d_pts, d_np, d_nbr, d_desc, h->d_theta, d_coff, d_mean, d_var, d_cov,
                           d_status));
  PCALL(cudaEventRecord(h->ev_k1, st));
  std::vector<double> hm((size_t)nn), hv((size_t)nn);
  std::vector<int32_t> hs((size_t)bc);
  PCALL(cudaMemcpyAsync(hm.data(), d_mean, sizeof(double) * nn, cudaMemcpyDeviceToHost, st));
  PCALL(cudaMemcpyAsync(hv.data(), d_var, sizeof(double) * nn, cudaMemcpyDeviceToHost, st));
  PCALL(cudaMemcpyAsync(hs.data(), d_status, sizeof(int32_t) * bc, cudaMemcpyDeviceToHost, st));
  if (cov) PCALL(cudaMemcpyAsync(cov, d_cov, sizeof(double) * coff[bc], cudaMemcpyDeviceToHost, st));
  PCALL(cudaStreamSynchronize(st));
#undef PCALL
  release();
  for (int32_t b = 0; b < bc; ++b)
    if (hs[b] != bv::kOk) {
      h->failed_pos = b;
      return fail(h, BV_ENOTPD, "prediction block " + std::to_string(b) + ": Sigma_con is not positive definite");
    }
  for (int64_t p = 0; p < nn; ++p) {
    mean[order_new[p]] = hm[p];
    if (var) var[order_new[p]] = hv[p];
  }
  return BV_OK;
}
