// bv_common.cuh — types and host/device helpers shared by the library's host
// runtime (bv_host.cpp) and its kernels (bv_kernels.cu).  Product code only:
// nothing here is shared with oracle/ (the oracle has its own everything).
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>

namespace bv {

// θ as the kernels see it (written once per evaluation by a graph memcpy node).
// Eq. (7): C(r) = σ² 2^{1−ν}/Γ(ν) (r/β)^ν K_ν(r/β).
enum MaternKind : int32_t { kNuHalf = 0, kNu3Half = 1, kNu5Half = 2, kNuGeneral = 3 };

struct alignas(16) Theta {
  double sigma2;    // σ²
  double inv_beta;  // 1/β
  double nu;        // ν
  double c_nu;      // σ²·2^{1−ν}/Γ(ν)  (general ν only)
  int32_t kind;     // MaternKind; closed forms iff ν ∈ {0.5, 1.5, 2.5} exactly
  int32_t pad0;
  double gen[10];   // ν-only constants of the general-ν K_ν evaluator (host-computed)
  const double* nutab;  // device address of the ν-only node/coefficient table (bessel_k.cuh)
};
// The θ buffer on the device (and its pinned host twin) is kThetaSlots Theta-sized
// slots: slot 0 = Theta, slots 1.. = the kNuTab doubles of the general-ν table.
constexpr int kNuTrapNodes = 28;   // trapezoid nodes t_k = k·h, k = 1..28, h = 0.15 (2 < x ≤ 22)
constexpr int kNuAsymTerms = 20;   // asymptotic-series coefficients (x > 22)
constexpr int kNuTab = 2 * kNuTrapNodes + kNuAsymTerms;
constexpr int kThetaSlots = 1 + (kNuTab * 8 + (int)sizeof(double) * 16 - 1) / ((int)sizeof(double) * 16);

// Per permuted position k (local index q = k − k_begin): where the block's
// points and neighbour list live.  Points of position k are the contiguous
// records pts[pstart .. pstart+l); neighbours are nbr[nbr_off .. nbr_off+m)
// (indices into pts).  Joint order: neighbours first, then block points.
struct alignas(16) BlockDesc {
  int32_t pstart;
  int32_t l;
  int32_t m;
  int32_t nbr_off;
};

// 32-byte AoS point record {x, y, z|0, observation} — one 256-bit load.
struct alignas(32) PointRec {
  double x, y, z, v;
};

// ln(2π) rounded to nearest double (0x3FFD67F1C864BEB5), for l_k log 2π
// (Alg. 1 l.29).
constexpr double kLn2Pi = 0x1.d67f1c864beb5p+0;

// Non-PD rule (reading G15): a Cholesky pivot must exceed
// kPivotFloor·σ² (σ² = every diagonal entry of Σθ); below it the block is
// FP64-singular (e.g. a repeated location) whatever the rounding order.
constexpr double kPivotFloor = 1e-14;

// Block status codes written by the kernels.
enum BlockStatus : int32_t { kOk = 0, kNotPD = 1, kTermRange = 2 };
// A block that failed with kNotPD writes d_k = NaN (a valid d_k is finite), so the
// host's optional jitter retry (reading G15b) can list the failed positions.
#ifdef __CUDACC__
__device__ __forceinline__ double failed_d() { return __longlong_as_double(0x7ff8000000000000ll); }
#endif

// ---------------------------------------------------------------------------
// Exact fixed-point block terms.  T = round(t·2⁶⁴) as a 192-bit
// two's-complement integer, split into six 32-bit chunks.  Integer sums are
// associative, so ℓ is bitwise independent of summation order, bucket
// schedule and GPU count.  |t| < 2⁹⁶ required.
__host__ __device__ inline int fixed_encode(double t, uint32_t c[6]) {
  uint64_t bits;
#ifdef __CUDA_ARCH__
  bits = (uint64_t)__double_as_longlong(t);
#else
  __builtin_memcpy(&bits, &t, 8);
#endif
  const int neg = (int)(bits >> 63);
  int E = (int)((bits >> 52) & 0x7ff);
  uint64_t mant = bits & ((1ull << 52) - 1);
  for (int i = 0; i < 6; ++i) c[i] = 0;
  if (E == 0x7ff) return 1;
  if (E >= 1023 + 96) return 1;
  if (E == 0) {
    if (mant == 0) return 0;
    E = 1;  // subnormal: mant·2^(1−1075)
  } else {
    mant |= (1ull << 52);
  }
  uint64_t L0 = 0, L1 = 0, L2 = 0;
  const int s = E - 1011;  // t·2⁶⁴ = mant·2^s
  if (s >= 0) {
    const int w = s >> 6, b = s & 63;
    const uint64_t lo = mant << b;
    const uint64_t hi = b ? (mant >> (64 - b)) : 0ull;
    if (w == 0) { L0 = lo; L1 = hi; }
    else if (w == 1) { L1 = lo; L2 = hi; }
    else { L2 = lo; }
  } else {
    const int r = -s;
    if (r <= 53) {  // round half to even
      uint64_t q = mant >> r;
      const uint64_t rem = mant & ((1ull << r) - 1);
      const uint64_t half = 1ull << (r - 1);
      if (rem > half || (rem == half && (q & 1ull))) ++q;
      L0 = q;
    }
  }
  if (neg) {  // two's complement over 192 bits
    L0 = ~L0; L1 = ~L1; L2 = ~L2;
    L0 += 1ull;
    if (L0 == 0) { L1 += 1ull; if (L1 == 0) L2 += 1ull; }
  }
  c[0] = (uint32_t)L0; c[1] = (uint32_t)(L0 >> 32);
  c[2] = (uint32_t)L1; c[3] = (uint32_t)(L1 >> 32);
  c[4] = (uint32_t)L2; c[5] = (uint32_t)(L2 >> 32);
  return 0;
}

// Reduction result slots (uint64): [0..5] chunk sums, [6] failed-block count,
// [7] local smallest failing (position << 8 | status), UINT64_MAX if none.
constexpr int kAccSlots = 8;

#ifdef __CUDACC__
// a9: add one block's exact term to the evaluation's accumulator.  Integer
// atomics are associative, so the sum is independent of the order blocks
// finish in (and of bucket schedule and GPU count).  Each slot receives < 2³²
// additions of < 2³² → no uint64 overflow.
__device__ __forceinline__ void accumulate_term(unsigned long long* acc, const uint32_t c[6], int st, int k) {
#pragma unroll
  for (int i = 0; i < 6; ++i)
    if (c[i]) atomicAdd(acc + i, (unsigned long long)c[i]);
  if (st != kOk) {
    atomicAdd(acc + 6, 1ull);
    atomicMin(acc + 7, ((unsigned long long)k << 8) | (unsigned long long)st);
  }
}
#endif

}  // namespace bv
