/* =============================================================================
 * bv.h — C ABI of the B200-native block-Vecchia log-likelihood library.
 *
 * The library evaluates, for a frozen plan (blocks, block order ζ, neighbour
 * lists), the block-Vecchia log-likelihood of arXiv 2410.04477:
 *
 *   ℓ(θ) = Σ_k −½ (u_k + d_k + l_k log 2π)                 (Alg. 1 l.28-30,
 *                                                            PAPER.md:631-633)
 *   u_k = v_kᵀv_k,  d_k = 2 log det L'_k                    (l.26-27, :627-629)
 *   L'_k L'_kᵀ = Σlk − Σcrossᵀ Σcon⁻¹ Σcross,
 *   v_k = L'_k⁻¹ (y_B − Σcrossᵀ Σcon⁻¹ y_NN)                (l.16-25, :602-625)
 *
 * with Σlk = K(s_B, s_B), Σcon = K(s_NN, s_NN), Σcross = K(s_NN, s_B)
 * (l.10-15, :593-599) and K the isotropic Matérn of Eq. (7):
 * C(r) = σ² 2^{1−ν}/Γ(ν) (r/β)^ν K_ν(r/β), θ = (σ², β, ν).  Eq. (4)
 * is the approximation this evaluates.  Everything runs in
 * FP64 on the GPU; nothing falls back to the CPU.
 *
 * Conventions:
 *  - every call returns bv_status; no exception crosses the ABI;
 *  - inputs are borrowed for the duration of the call: bv_setup copies the
 *    plan to the device and keeps no caller pointer; outputs are caller-owned
 *    host memory;
 *  - a handle is not thread-safe; one evaluation runs at a time; bv_loglik is
 *    synchronous (ℓ is on the host when it returns);
 *  - canonical order (part of the contract): the points of a block are taken
 *    in ascending global id; a neighbour set in the order given (the planner
 *    emits ascending (distance to centroid, id)).  The joint matrix of block
 *    k is [NN_k ; B_k] in that order.
 * ========================================================================== */
#ifndef BV_H_
#define BV_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BV_OK = 0,
  BV_EINVAL = 2,   /* invalid plan, θ or argument; bv_last_error names the first violation */
  BV_ENOTPD = 3,   /* a block's joint covariance is not positive definite (Alg. 1 l.17/l.24 POTRF
                      fails); *loglik = -INFINITY and bv_last_error gives the smallest failing
                      permuted position k */
  BV_EIO = 4,
  BV_ECUDA = 5,    /* CUDA runtime error (message in bv_last_error) */
  BV_ENCCL = 6,    /* NCCL error */
  BV_ENOMEM = 7    /* device allocation failed */
} bv_status;

typedef struct bv_handle bv_handle; /* opaque; owns all device state, stream, CUDA graph, NCCL comm */

/* The frozen plan (Alg. 1 l.4-9 output).  All pointers are
 * HOST memory, borrowed for the duration of bv_setup. */
typedef struct {
  int64_t n;               /* number of points, n ≥ 1 */
  int32_t d;               /* dimension, 2 or 3 */
  const double* locs;      /* n*d row-major coordinates, finite */
  const double* y;         /* n observations, finite, zero-mean model */
  int32_t bc;              /* block count, 1 ≤ bc ≤ n */
  const int32_t* block_id; /* n entries in [0, bc); every block non-empty (partition B, Eq. 2) */
  const int32_t* order;    /* bc entries, a permutation: order[k] = block at position k (ζ, Eq. 3) */
  const int64_t* nbr_ptr;  /* bc+1 CSR offsets by POSITION k, nbr_ptr[0] = 0, non-decreasing */
  const int32_t* nbr_idx;  /* global point ids; set k lies in blocks order[0..k-1] only
                              (PAPER.md:165), no duplicates; may be empty (position 0) */
} bv_plan;

/* Distribution (optional).  NULL or world == 1 → single GPU `device`.
 * world > 1: every rank passes the SAME full plan, its own rank, and the same
 * 128-byte ncclUniqueId (from bv_nccl_unique_id on rank 0, broadcast by the
 * caller, e.g. through torch.distributed).  Positions are split into
 * contiguous, cost-balanced ranges; ℓ is reduced with exactly
 * one ncclAllReduce per evaluation and is bitwise identical on every rank and
 * for every world size. */
typedef struct {
  int32_t device;
  int32_t rank;
  int32_t world;
  const void* nccl_id; /* 128 bytes (ncclUniqueId) or NULL when world == 1 */
} bv_dist;

/* Library version string (static storage). */
const char* bv_version(void);

/* Rank 0 creates the NCCL unique id; out128 must hold 128 bytes. */
bv_status bv_nccl_unique_id(void* out128);

/* Validate the plan, build the device layout (block-contiguous 32-byte point
 * records, neighbour lists remapped to permuted indices, size buckets, this
 * rank's position range), upload it, create the NCCL communicator (world > 1)
 * and capture the per-evaluation CUDA graph.  *out is NULL on failure.
 * Errors: BV_EINVAL (plan violation, message names the first one in index
 * order), BV_ECUDA, BV_ENOMEM, BV_ENCCL.  Runs once per plan; not timed
 * (PAPER.md:411). */
bv_status bv_setup(const bv_plan* plan, const bv_dist* dist, bv_handle** out);

/* TEST-ONLY rank emulation (no communicator).  Builds exactly the device layout
 * rank `rank` of `world` would get from bv_setup (the same contiguous,
 * cost-balanced position range, rank-local neighbour slice and rebased
 * offsets — DESIGN.md §6, "independent of each other"), but
 * creates no NCCL communicator and reduces nothing across ranks: bv_loglik on
 * such a handle returns this rank's PARTIAL sum, and bv_loglik_acc its exact
 * fixed-point accumulator, so the G partial accumulators can be summed by the
 * caller and compared with the single-rank one.  Lets one GPU evaluate the
 * ranks of a world > 1 partition one after another (no rank waits on another).
 * Failing positions are reported as GLOBAL permuted positions k.  Errors as
 * bv_setup. */
bv_status bv_setup_rank_local(const bv_plan* plan, int32_t device, int32_t rank, int32_t world, bv_handle** out);

/* ℓ(θ) for θ = (σ², β, ν) (host array of 3 doubles): σ², β finite and > 0;
 * ν exactly 0.5, 1.5 or 2.5 (closed forms) or any ν in [0.2, 3] (the general
 * K_ν path, validated on that range; the MLE box of SURVEY §8d).  Collective when world > 1 (all ranks, identical θ).
 * Errors: BV_EINVAL (bad θ), BV_ENOTPD (*loglik = -INFINITY), BV_ECUDA,
 * BV_ENCCL. */
bv_status bv_loglik(bv_handle* h, const double theta[3], double* loglik);

/* As bv_loglik, and also the per-block log-determinants d_k and quadratic
 * forms u_k (Alg. 1 l.26-27) for this rank's positions [k_begin, k_end)
 * (bv_owned_range), written to logdet[k - k_begin] / quad[k - k_begin]
 * (host arrays of k_end - k_begin doubles; either may be NULL). */
bv_status bv_loglik_terms(bv_handle* h, const double theta[3], double* loglik, double* logdet, double* quad);

/* One evaluation, returning the exact fixed-point accumulator instead of ℓ:
 * acc_out[0..5] = the six 32-bit chunk sums of round(t_k·2⁶⁴) (
 * ℓ = bv_fixed_decode(acc_out)), acc_out[6] = failed-block count,
 * acc_out[7] = (smallest failing global position << 8 | status) or UINT64_MAX.
 * After a world > 1 bv_setup the chunks are already all-reduced; after
 * bv_setup_rank_local they are this rank's partial.  Returns BV_OK or
 * BV_ENOTPD like bv_loglik (acc_out is filled either way), or an error. */
bv_status bv_loglik_acc(bv_handle* h, const double theta[3], uint64_t acc_out[8]);

/* Optional jitter mode (off by default; reading G15b, SPEC.md:197,
 * :238).  When enabled, a bv_loglik* evaluation in which some block is not
 * positive definite recomputes each failed block with ε·σ² added to every
 * diagonal entry of its joint matrix (the diagonals of Σcon and Σlk),
 * ε = 1e-10, 1e-8, 1e-6 in turn, keeping the first that succeeds; only if
 * one still fails does the call return BV_ENOTPD.  The retry runs off the
 * captured graph and only after a failure, so evaluations without failures
 * cost the same.  Every joint size the evaluation supports is retried, with
 * the same kernels and ε·σ² added to the diagonal inside the factorisation.
 * Collective when world > 1: set it identically on every rank.  Errors: BV_EINVAL (NULL). */
bv_status bv_set_jitter(bv_handle* h, int32_t enable);

/* Blocks (over all ranks) that needed jitter in the most recent evaluation
 * (SPEC.md:269 jitter_events); 0 when the mode is off. */
bv_status bv_jitter_events(const bv_handle* h, int64_t* events);

/* This rank's contiguous range of permuted positions. */
bv_status bv_owned_range(const bv_handle* h, int32_t* k_begin, int32_t* k_end);

/* End-to-end variant (host observations in, ℓ out): copies y (n host
 * doubles, in global point-id order, all finite — else BV_EINVAL naming the
 * first non-finite entry, *loglik = −∞) to the device inside the call, then
 * evaluates.  A non-finite y_i always makes its own block's term non-finite, so
 * y is scanned on the host only when the evaluation fails (the precise error
 * then replaces the block-level one); the success path never reads y on the
 * host.  Used to time the whole path with host↔device traffic. */
bv_status bv_loglik_host_y(bv_handle* h, const double* y, const double theta[3], double* loglik);

/* ---- block-Vecchia prediction (Alg. 2; §2.3 :194-240) ----
 *
 * New locations S* are clustered into prediction blocks B*_1..B*_bc (l.4) and
 * every block conditions on m_i training points (l.6, any training point —
 * "m nearest neighbor observations from y").  For each block:
 *   μ_B* = Σcrossᵀ Σcon⁻¹ y_NN,   Σ_B* = Σlk − Σcrossᵀ Σcon⁻¹ Σcross      (l.10-11)
 * with Σcon = K(s_NN, s_NN), Σcross = K(s_NN, s_B*) (m×l, reading G8),
 * Σlk = K(s_B*, s_B*) and K the Matérn of Eq. (7).  y is the handle's current
 * y (the plan's, or the last bv_loglik_host_y's).  All pointers HOST memory,
 * borrowed for the call. */
typedef struct {
  int64_t n_new;            /* number of new locations, ≥ 1 */
  const double* locs_new;   /* n_new*d row-major (d of the handle's plan), finite */
  int32_t bc_new;           /* number of prediction blocks, ≥ 1 */
  const int32_t* block_id;  /* n_new, in [0, bc_new), every block non-empty; a block's points are
                               taken in ascending new-point id */
  const int64_t* nbr_ptr;   /* bc_new+1 CSR offsets by prediction block id, nbr_ptr[0] = 0 */
  const int32_t* nbr_idx;   /* training point ids in [0, n), no duplicate within a block, in the
                               order given (the planner emits ascending (distance to centroid, id)) */
} bv_pred_plan;

/* Prediction at θ.  mean[n_new] = μ (the predicted values y*, l.12), indexed
 * by new-point id; var[n_new] (or NULL) = diag Σ_B* (PAPER.md:242); cov (or
 * NULL) = every block's l_b×l_b Σ_B* row-major, blocks in id order at offset
 * Σ_{b'<b} l_b'² (l.15, "for conditional simulations").  Requires
 * m_b + l_b ≤ 235 (the joint triangle lives in shared memory).  Errors:
 * BV_EINVAL (invalid pred plan / θ; message names the first violation),
 * BV_ENOTPD (Σcon of a block not positive definite; bv_last_error's
 * failed_position = the smallest such block id).  Prediction never jitters
 * (bv_set_jitter applies to bv_loglik* only): Alg. 2 has no fallback and a
 * singular Σcon means duplicated training locations in a conditioning set.
 * Not collective: under multi-GPU any rank may call it alone (the point
 * records are replicated). */
bv_status bv_predict(bv_handle* h, const double theta[3], const bv_pred_plan* pp, double* mean, double* var,
                     double* cov);

/* ---- GPU plan construction (Alg. 1 l.4-9) ----
 * The preprocessing the paper runs once per fit and excludes from timing
 * (PAPER.md:411).  Exact selections with total orders, so the results are
 * bit-identical to any exact implementation (tests: the CPU planner in
 * bvgen/).  Host pointers in and out; device = CUDA ordinal.  Not collective. */

/* Lloyd K-means (Alg. 1 l.5).  locs n*d row-major; init_idx:
 * k distinct point ids, the initial centroids (drawn by the caller's seeded
 * RNG).  Each iteration: every point to the nearest centroid (squared distance
 * summed in x, y, z order, no FMA contraction; ties → lower id); empty
 * clusters (ascending id) take the farthest point of a cluster with ≥ 2
 * members (ties → lowest id); centroids = member means summed in ascending
 * point id.  Stops when the assignment repeats or after max_iter iterations.
 * Outputs assign[n], cent[k*d], *iters (may be NULL).  BV_EINVAL on bad
 * arguments (1 ≤ k ≤ n < 2^31, d ∈ {2,3}). */
bv_status bv_plan_kmeans(int32_t device, int64_t n, int32_t d, const double* locs, int32_t k, const int32_t* init_idx,
                         int32_t max_iter, int32_t* assign, double* cent, int32_t* iters);

/* mNearestNeighborsForBlock (Alg. 1 l.7-9): for every position k of the order
 * ζ (order[k] = block id), the m_k = min(m, #points in earlier blocks) points
 * of blocks at positions < k nearest the block centroid (mean of
 * its points), ascending (d², id).  nbr_ptr[bc+1] is written
 * (CSR by position); nbr_idx needs room for nbr_ptr[bc] ≤ bc*m ids.  m ≤ 256.
 * BV_EINVAL: bad block ids / order / empty block / m. */
bv_status bv_plan_block_nn(int32_t device, int64_t n, int32_t d, const double* locs, int32_t bc, const int32_t* block_id,
                           const int32_t* order, int32_t m, int64_t* nbr_ptr, int32_t* nbr_idx);

/* Message of the last failed bv_plan_* call on this thread ("" after success). */
const char* bv_plan_last_error(void);

/* Last error message and (after BV_ENOTPD) the smallest failing position, or
 * -1.  *msg points into the handle and is valid until the next call. */
bv_status bv_last_error(const bv_handle* h, int32_t* failed_position, const char** msg);

/* The handle's CUDA stream (a cudaStream_t), so a caller can record timing
 * events on the stream the library's kernels run on. */
void* bv_stream(const bv_handle* h);

/* Device time (ms) of the block kernels (all size buckets, gather through
 * per-block terms; excludes θ upload, reduction and allreduce) in the most
 * recent evaluation, from CUDA events captured inside the graph.  After a
 * bv_predict it is the device time of the prediction kernel instead. */
bv_status bv_last_kernel_ms(const bv_handle* h, float* ms);

/* Kernel launches per evaluation on this rank (for the bench's gpu_launches), for
 * the Matérn kind of the most recent evaluation: after a general-ν evaluation of
 * a small plan (Σ ≤ 64 MB) it includes the one pre-generation launch. */
int32_t bv_launches_per_eval(const bv_handle* h);

/* Free everything the handle owns.  NULL is a no-op. */
void bv_destroy(bv_handle* h);

/* ---- host-side twins, callable without a GPU (tests / multi-rank logic) ---- */

/* Cost-balanced contiguous partition of positions 0..bc-1 over `world`
 * ranks: cost_k = N_k³/3 + 40·E_k with N_k = m_k + l_k and
 * E_k = N_k(N_k+1)/2; cut g is the first k with prefix(k) ≥ g·total/world.
 * l, m: bc entries each.  cuts: world+1 entries (cuts[0] = 0, cuts[world] = bc). */
bv_status bv_partition(int32_t bc, const int32_t* l, const int32_t* m, int32_t world, int32_t* cuts);

/* Exact fixed-point encoding of a block term t: round(t·2⁶⁴) as
 * a 192-bit two's-complement integer split into six 32-bit chunks (chunk 0
 * least significant).  Returns BV_EINVAL for non-finite t or |t| ≥ 2⁹⁶ (so that
 * up to 2³¹ terms sum without overflowing 192 bits). */
bv_status bv_fixed_encode(double t, uint32_t chunks[6]);

/* Decode six chunk SUMS (each the sum of up to 2³¹ chunks) to the double
 * nearest Σ round(t_k·2⁶⁴)·2⁻⁶⁴. */
double bv_fixed_decode(const uint64_t acc[6]);

#ifdef __cplusplus
}
#endif

#endif /* BV_H_ */
