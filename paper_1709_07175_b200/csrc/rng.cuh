// Counter-based random streams, restated for the device from the reference's
// proj/core/include/lazypca/rng.hpp:15-97 (splitmix64 seeding, xoshiro256**,
// per-(seed, column) streams, Acklam inverse normal CDF).
//
// Bit parity with the reference: every floating-point step of normal_icdf is an
// explicit round-to-nearest intrinsic in the reference's evaluation order (no
// FMA contraction), matching the reference compiled with -ffp-contract=off.
// The two tail branches (p < 0.02425 or p > 0.97575, ~4.85% of draws) call
// log(); CUDA's log is within 1 ulp of glibc's, so tail entries may differ by
// an ulp or two — tests/test_gpu_parity.py::test_omega_matches_reference_bits
// measures and bounds that.
#pragma once
#include <cstdint>

namespace lpca {

__host__ __device__ __forceinline__ std::uint64_t splitmix64(std::uint64_t& state) {
  std::uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ std::uint64_t mix64(std::uint64_t z) { return splitmix64(z); }

struct Xoshiro {
  std::uint64_t s0, s1, s2, s3;
  __host__ __device__ __forceinline__ explicit Xoshiro(std::uint64_t seed) {
    std::uint64_t sm = seed;
    s0 = splitmix64(sm);
    s1 = splitmix64(sm);
    s2 = splitmix64(sm);
    s3 = splitmix64(sm);
  }
  __host__ __device__ __forceinline__ static std::uint64_t rotl(std::uint64_t x, int k) {
    return (x << k) | (x >> (64 - k));
  }
  __host__ __device__ __forceinline__ std::uint64_t next() {
    const std::uint64_t result = rotl(s1 * 5, 7) * 9;
    const std::uint64_t t = s1 << 17;
    s2 ^= s0;
    s3 ^= s1;
    s1 ^= s2;
    s0 ^= s3;
    s2 ^= t;
    s3 = rotl(s3, 45);
    return result;
  }
};

// column_stream(seed, col) (rng.hpp:61-65)
__host__ __device__ __forceinline__ Xoshiro column_stream(std::uint64_t seed, std::uint64_t col) {
  return Xoshiro(mix64(mix64(seed) ^ (0x9e3779b97f4a7c15ULL * (col + 1))));
}

#if defined(__CUDA_ARCH__)
#define LPCA_ADD(a, b) __dadd_rn((a), (b))
#define LPCA_SUB(a, b) __dsub_rn((a), (b))
#define LPCA_MUL(a, b) __dmul_rn((a), (b))
#define LPCA_DIV(a, b) __ddiv_rn((a), (b))
#define LPCA_SQRT(a) __dsqrt_rn((a))
#else
#define LPCA_ADD(a, b) ((a) + (b))
#define LPCA_SUB(a, b) ((a) - (b))
#define LPCA_MUL(a, b) ((a) * (b))
#define LPCA_DIV(a, b) ((a) / (b))
#define LPCA_SQRT(a) sqrt((a))
#endif

// Xoshiro256::uniform (rng.hpp:49-51): ((next >> 11) + 0.5) * 2^-53.
__host__ __device__ __forceinline__ double u64_to_uniform(std::uint64_t bits) {
  return LPCA_MUL(LPCA_ADD(static_cast<double>(bits >> 11), 0.5), 0x1.0p-53);
}

// normal_icdf (rng.hpp:69-97), Acklam's rational approximation.
__host__ __device__ __forceinline__ double normal_icdf(double p) {
  const double a0 = -3.969683028665376e+01, a1 = 2.209460984245205e+02, a2 = -2.759285104469687e+02,
               a3 = 1.383577518672690e+02, a4 = -3.066479806614716e+01, a5 = 2.506628277459239e+00;
  const double b0 = -5.447609879822406e+01, b1 = 1.615858368580409e+02, b2 = -1.556989798598866e+02,
               b3 = 6.680131188771972e+01, b4 = -1.328068155288572e+01;
  const double c0 = -7.784894002430293e-03, c1 = -3.223964580411365e-01, c2 = -2.400758277161838e+00,
               c3 = -2.549732539343734e+00, c4 = 4.374664141464968e+00, c5 = 2.938163982698783e+00;
  const double d0 = 7.784695709041462e-03, d1 = 3.224671290700398e-01, d2 = 2.445134137142996e+00,
               d3 = 3.754408661907416e+00;
  const double p_low = 0.02425;
  if (p < p_low || p > LPCA_SUB(1.0, p_low)) {
    const bool upper = !(p < p_low);
    const double arg = upper ? LPCA_SUB(1.0, p) : p;
    const double q = LPCA_SQRT(LPCA_MUL(-2.0, log(arg)));
    double num = LPCA_ADD(LPCA_MUL(c0, q), c1);
    num = LPCA_ADD(LPCA_MUL(num, q), c2);
    num = LPCA_ADD(LPCA_MUL(num, q), c3);
    num = LPCA_ADD(LPCA_MUL(num, q), c4);
    num = LPCA_ADD(LPCA_MUL(num, q), c5);
    double den = LPCA_ADD(LPCA_MUL(d0, q), d1);
    den = LPCA_ADD(LPCA_MUL(den, q), d2);
    den = LPCA_ADD(LPCA_MUL(den, q), d3);
    den = LPCA_ADD(LPCA_MUL(den, q), 1.0);
    return upper ? LPCA_DIV(-num, den) : LPCA_DIV(num, den);
  }
  const double q = LPCA_SUB(p, 0.5);
  const double r = LPCA_MUL(q, q);
  double num = LPCA_ADD(LPCA_MUL(a0, r), a1);
  num = LPCA_ADD(LPCA_MUL(num, r), a2);
  num = LPCA_ADD(LPCA_MUL(num, r), a3);
  num = LPCA_ADD(LPCA_MUL(num, r), a4);
  num = LPCA_ADD(LPCA_MUL(num, r), a5);
  num = LPCA_MUL(num, q);
  double den = LPCA_ADD(LPCA_MUL(b0, r), b1);
  den = LPCA_ADD(LPCA_MUL(den, r), b2);
  den = LPCA_ADD(LPCA_MUL(den, r), b3);
  den = LPCA_ADD(LPCA_MUL(den, r), b4);
  den = LPCA_ADD(LPCA_MUL(den, r), 1.0);
  return LPCA_DIV(num, den);
}

// Counter-based N(0,1) for the synthetic data generator (not in the reference;
// BASELINE's dense low-rank workloads). Any element can be produced on any GPU.
__host__ __device__ __forceinline__ double counter_normal(std::uint64_t seed, std::uint64_t idx) {
  return normal_icdf(u64_to_uniform(mix64(seed ^ (idx * 0x9e3779b97f4a7c15ULL))));
}

}  // namespace lpca
