// Shared device structures and the exact RNS base-conversion helpers.
//
// Ciphertext tensors are limb-major u32: [ct][part][limb][N].
//
// Exact base conversion.  The reference lifts every ciphertext part to its
// canonical integer in [0, q) (ring.py:286-295, bfv.py:321-333) and rounds
// t*d/q exactly (bfv.py:229-236, 325-328).  On the device a canonical value
// x = sum_i xt_i (q/q_i) - v q  (xt_i = x_i (q/q_i)^-1 mod q_i) is moved to
// another prime p with the CRT matrix; the overflow count v is estimated in
// 60-bit fixed point and, only when that estimate lies within its error bound
// of an integer, decided exactly with multiword arithmetic.  Nothing is
// approximate: every output residue equals the reference's.
#pragma once
#include <cuda_runtime.h>

#include "modarith.cuh"

namespace hcnn {

constexpr int KMAX = 16;   // primes of q
constexpr int KPMAX = 19;  // primes of the auxiliary base P (K+2 or K+3)
constexpr int WMAX = 17;   // 32-bit words of (K+1) q
constexpr int DMAX = 64;   // relinearisation digits

// Exact base-conversion and scaling constants; passed by value (param space,
// served from the constant bank with static indices).
struct ConvTabs {
  int K, KP, W, D, digit_bits;
  uint32_t q[KMAX];
  uint64_t qmu[KMAX];
  uint32_t p[KPMAX];
  uint64_t pmu[KPMAX];
  // Q -> P of a canonical [0, q) value
  uint32_t qhi[KMAX], qhis[KMAX];  // (q/q_i)^-1 mod q_i and its Shoup word
  uint64_t qG[KMAX];               // floor(2^(60+qb) / q_i)
  uint32_t qb[KMAX];               // bit length of q_i
  uint32_t qhat_p[KMAX][KPMAX];    // (q/q_i) mod p_j
  uint32_t negq_p[KPMAX];          // -q mod p_j
  uint32_t qhat_w[KMAX][WMAX];     // q/q_i, 32-bit words
  uint32_t q_w[WMAX];              // q, 32-bit words
  // P -> Q of a centred (-P/2, P/2) value
  uint64_t pG[KPMAX];
  uint32_t pb[KPMAX];
  uint32_t phat_q[KPMAX][KMAX];  // (P/p_j) mod q_i
  uint32_t negp_q[KMAX];         // -P mod q_i
  // scale-and-round: r~_i = d_i A_i + B_i  (mod q_i)
  //                  y~_j = d_j C_j + (p_j - r_j) E_j + F_j  (mod p_j)
  uint32_t A[KMAX], As[KMAX], B[KMAX];
  uint32_t C[KPMAX], Cs[KPMAX], Ej[KPMAX], Ejs[KPMAX], F[KPMAX];
};

// Device pointers of the per-context NTT tables (all primes, Q first, then P).
struct NttTabs {
  const uint32_t* prime;  // [K+KP]
  const uint64_t* mu;     // [K+KP] floor(2^64/p)
  const uint2* tw;        // [(K+KP) * N]  psi^brv(i), Shoup
  const uint2* itw;       // [(K+KP) * N]  psi^-brv(i), Shoup
  const uint2* ninv;      // [K+KP]        N^-1, Shoup
  const uint32_t* pinv;   // [K+KP]        -p^-1 mod 2^32 (Montgomery)
};

constexpr uint64_t FRAC_ONE = 1ull << 60;
constexpr uint64_t FRAC_MASK = FRAC_ONE - 1;

// words needed for (K+1) q with K primes below 2^30, plus one
__host__ __device__ constexpr int words_for(int k) { return (30 * k + 5 + 31) / 32 + 1; }

// floor(x * 2^60 / m) - e, e in [0, 2), from G = floor(2^(60+b)/m), b = bitlen(m)
DI uint64_t frac60(uint32_t x, uint64_t G, uint32_t b) {
  const uint64_t lo = (uint64_t)x * G;
  const uint64_t hi = __umul64hi((uint64_t)x, G);
  return (hi << (64 - b)) | (lo >> b);
}

// S = sum_i xt_i * (q/q_i) as words, exact (column sums of 32-bit halves).
template <int K>
DI void mw_lift(const uint32_t (&xt)[K], const ConvTabs& tb, uint32_t (&S)[words_for(K)]) {
  uint64_t carry = 0, hiprev = 0;
#pragma unroll
  for (int w = 0; w < words_for(K); ++w) {
    uint64_t lo = 0, hi = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const uint64_t pr = (uint64_t)xt[i] * tb.qhat_w[i][w];
      lo += (uint32_t)pr;
      hi += pr >> 32;
    }
    const uint64_t s = lo + hiprev + carry;
    S[w] = (uint32_t)s;
    carry = s >> 32;
    hiprev = hi;
  }
}

// S - m*q in place; returns the final borrow (1 if S < m*q).
template <int K>
DI uint32_t mw_sub_mq(uint32_t (&S)[words_for(K)], uint32_t m, const ConvTabs& tb) {
  uint64_t carry = 0;
  uint32_t borrow = 0;
#pragma unroll
  for (int w = 0; w < words_for(K); ++w) {
    const uint64_t mq = (uint64_t)tb.q_w[w] * m + carry;
    carry = mq >> 32;
    const uint64_t d = (uint64_t)S[w] - (uint32_t)mq - borrow;
    S[w] = (uint32_t)d;
    borrow = (uint32_t)(d >> 63);
  }
  return borrow;
}

// Exact v = floor(sum_i xt_i / q_i) for a canonical lift: 60-bit fixed point
// (error in (-2K, 0] units of 2^-60), with an exact multiword decision when the
// estimate is within that error of an integer (lifted value within ~2^-56 q of
// q; astronomically rare for ciphertext data, but handled).
template <int K>
DI uint32_t exact_v(const uint32_t (&xt)[K], const ConvTabs& tb) {
  uint64_t F = 0;
#pragma unroll
  for (int i = 0; i < K; ++i) F += frac60(xt[i], tb.qG[i], tb.qb[i]);
  uint32_t V = (uint32_t)(F >> 60);
  if ((F & FRAC_MASK) >= FRAC_ONE - 2 * (uint64_t)K - 2) {
    uint32_t S[words_for(K)];
    mw_lift<K>(xt, tb, S);
    if (!mw_sub_mq<K>(S, V + 1, tb)) V += 1;
  }
  return V;
}

// x_j = (sum_i xt_i (q/q_i) - v q) mod p_j
template <int K>
DI uint32_t q_to_p(const uint32_t (&xt)[K], uint32_t v, int j, const ConvTabs& tb) {
  uint64_t acc = (uint64_t)v * tb.negq_p[j];
#pragma unroll
  for (int i = 0; i < K; ++i) acc += (uint64_t)xt[i] * tb.qhat_p[i][j];
  return reduce64(acc, tb.p[j], tb.pmu[j]);
}

}  // namespace hcnn
