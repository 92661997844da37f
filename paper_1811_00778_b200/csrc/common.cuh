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

DI uint32_t umin_u32(uint32_t a, uint32_t b) { return a < b ? a : b; }

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
  uint32_t qg[KMAX], qk[KMAX];     // fixed point: x/q_i ~ (x * qg_i << qk_i) / 2^59
  uint32_t qpinv[KMAX];            // -q_i^-1 mod 2^32
  uint32_t qhat_p[KMAX][KPMAX];    // (q/q_i) 2^32 mod p_j (Montgomery form)
  uint32_t negq_p[KPMAX];          // -q 2^32 mod p_j (Montgomery form)
  uint32_t qhat_w[KMAX][WMAX];     // q/q_i, 32-bit words
  uint32_t q_w[WMAX];              // q, 32-bit words
  // P -> Q of a centred (-P/2, P/2) value
  uint32_t pg[KPMAX], pk[KPMAX];
  uint32_t ppinv[KPMAX];         // -p_j^-1 mod 2^32
  uint32_t phat_q[KPMAX][KMAX];  // (P/p_j) 2^32 mod q_i (Montgomery form)
  uint32_t negp_q[KMAX];         // -P 2^32 mod q_i (Montgomery form)
  // scale-and-round: r~_i = d_i A_i + B_i  (mod q_i)
  //                  y~_j = d_j C_j + (p_j - r_j) E_j + F_j  (mod p_j)
  uint32_t A[KMAX], As[KMAX], B[KMAX];
  uint32_t C[KPMAX], Cs[KPMAX], Ej[KPMAX], Ejs[KPMAX], F[KPMAX];
  // decryption rounding m = round(t x / q) mod t (bfv.py:229-250), t < 2^48:
  // t = dec_a_i q_i + dec_f_i, H = floor((q-1)/2 * 2^59 / q), h_w = words of (q-1)/2
  uint64_t t, tmu;
  uint64_t dec_a[KMAX];
  uint32_t dec_f[KMAX];
  uint64_t H;
  uint32_t h_w[WMAX];
};

// Device pointers of the per-context NTT tables (all primes, Q first, then P).
struct NttTabs {
  const uint32_t* prime;  // [K+KP]
  const uint64_t* mu;     // [K+KP] floor(2^64/p)
  const uint2* tw;        // [(K+KP) * N]  psi^brv(i), Shoup
  const uint2* itw;       // [(K+KP) * N]  psi^-brv(i), Shoup
  const uint2* ninv;      // [K+KP]        N^-1, Shoup
  const uint32_t* pinv;   // [K+KP]        -p^-1 mod 2^32 (Montgomery)
  const uint2* ninv_m;    // [K+KP]        N^-1 2^32 mod p, Shoup: undoes the 2^-32
                          //               of Montgomery pointwise products
  const uint2* ninv_w;    // [K+KP]        psi^-N/2 N^-1: the last inverse stage's twiddle, scaled
  const uint2* ninv_mw;   // [K+KP]        psi^-N/2 N^-1 2^32
};

// Relinearisation through a shared three-prime basis R = r0 r1 r2
// (flag RELIN_RBASIS).  The key-switching sums Z = sum_i d_i k_i over
// Z[X]/(X^N+1), with digits d_i in [0, w) and key rows k_i centred mod q_j,
// satisfy |Z| < D N w q_j / 2 < R / 2, so the NTTs of the digits are taken
// once over R (3 per digit instead of K) and Z mod q_j is recovered exactly
// from Z mod r0, r1, r2 (Garner, centred).  Table index of r_a: roff + a.
constexpr int RB_A = 3;
struct RbTabs {
  int roff;
  uint32_t r[RB_A];
  uint2 t32[RB_A];     // 2^32 mod r_a (Shoup): folds the high word of a 64-bit sum
  uint32_t one[RB_A];  // floor(2^32 / r_a): the Shoup word of 1 (low word)
  uint32_t rpinv[RB_A];  // -r_a^-1 mod 2^32 (REDC of the tensor-core MAC)
  uint2 isc_n[RB_A], isc_nw[RB_A];  // inverse scaling N^-1 g_a, psi^-N/2 N^-1 g_a with
                                    // g_a = (R/r_a)^-1 mod r_a: the inverse leaves x~_a
  float rinv[RB_A];    // 1 / r_a: v = rint(sum_a x~_a / r_a) (|Z| / R < 2^-25)
  uint32_t crt_q[KMAX][RB_A];  // (R/r_a) 2^32 mod q_j (Montgomery form)
  uint32_t negR_q[KMAX];       // -R 2^32 mod q_j (Montgomery form)
};

// Output scaling of an inverse transform, folded into its last stage (whose
// butterflies all share the twiddle psi^-N/2): n for the sum, nw for the
// difference.
struct InvScale {
  uint2 n, nw;
};

DI InvScale inv_scale(const NttTabs& nt, int j, bool mont) {
  return mont ? InvScale{nt.ninv_m[j], nt.ninv_mw[j]} : InvScale{nt.ninv[j], nt.ninv_w[j]};
}

// fixed point of the CRT overflow estimates: 59 fractional bits
constexpr int FRAC_BITS = 59;
constexpr uint64_t FRAC_ONE = 1ull << FRAC_BITS;
constexpr uint64_t FRAC_MASK = FRAC_ONE - 1;
// per-term error bound of frac59 (units of 2^-59): below 2^30
constexpr uint64_t FRAC_ERR = 1ull << 30;

// words needed for (K+1) q with K primes below 2^30, plus one
__host__ __device__ constexpr int words_for(int k) { return (30 * k + 5 + 31) / 32 + 1; }

// x * 2^59 / m - e with 0 <= e < 2^30, for x < m: g = floor(2^(59-k)/m) < 2^32
// (k = 0 for primes above 2^27), one 32x32->64 multiply
DI uint64_t frac59(uint32_t x, uint32_t g, uint32_t k) { return ((uint64_t)x * g) << k; }

// Montgomery reduction of a 64-bit sum: acc * 2^-32 mod p for acc < 3 * 2^62,
// result fully reduced.  With constants pre-multiplied by 2^32 the sum of
// products reduces to the plain value.
DI uint32_t redc(uint64_t acc, uint32_t p, uint32_t pinv) {
  const uint32_t m = (uint32_t)acc * pinv;
  uint32_t r = (uint32_t)((acc + (uint64_t)m * p) >> 32);  // < acc/2^32 + p < 4p
  r = umin_u32(r, r - 2 * p);
  return umin_u32(r, r - p);
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

// Exact v = floor(sum_i xt_i / q_i) for a canonical lift: 59-bit fixed point
// (error in (-K 2^30, 0] units of 2^-59), with an exact multiword decision when
// the estimate is within that error of an integer (lifted value within
// ~K 2^-29 q of q: about one coefficient in 2^25, handled exactly).
template <int K>
DI uint32_t exact_v(const uint32_t (&xt)[K], const ConvTabs& tb) {
  uint64_t F = 0;
#pragma unroll
  for (int i = 0; i < K; ++i) F += frac59(xt[i], tb.qg[i], tb.qk[i]);
  uint32_t V = (uint32_t)(F >> FRAC_BITS);
  if ((F & FRAC_MASK) >= FRAC_ONE - K * FRAC_ERR) {
    uint32_t S[words_for(K)];
    mw_lift<K>(xt, tb, S);
    if (!mw_sub_mq<K>(S, V + 1, tb)) V += 1;
  }
  return V;
}

// Montgomery reduction by subtraction: acc * 2^-32 mod m for any acc < 2^64
// with (acc >> 32) < 4m.  mpos = m^-1 mod 2^32 (minus the REDC constant):
// u = lo(acc) mpos makes acc - u m a multiple of 2^32, so
// (acc - u m) / 2^32 = hi(acc) - umulhi(u, m) exactly, in (-m, 4m).
DI uint32_t redc_sub(uint64_t acc, uint32_t m, uint32_t minv) {
  const uint32_t u = (uint32_t)acc * (0u - minv);
  const uint32_t ah = (uint32_t)(acc >> 32), mh = __umulhi(u, m);
  uint32_t r = ah - mh;
  if (ah < mh) r += m;
  r = umin_u32(r, r - 2 * m);
  return umin_u32(r, r - m);
}

// sum_{i<K} x_i c_i (+ v c_v), x_i < 2^30, c's in Montgomery form mod m (< m),
// v c_v < 2^60, reduced.  Up to 11 products: one REDC (3 * 2^62 headroom).
// 12-15 products: the sum still stays below 2^64 with its high word below
// 16 * 2^30 m / 2^32 = 4m, so one subtractive REDC (measured cheaper than two
// REDCs; the additive one stays cheaper where it suffices).  Larger K: two
// halves of <= 11.
template <int K, class Getc>
DI uint32_t mont_dot(const uint32_t* x, Getc c, uint32_t v, uint32_t cv, uint32_t m, uint32_t minv) {
  constexpr int H = K <= 15 ? K : (K + 1) / 2;
  uint64_t a0 = (uint64_t)v * cv, a1 = 0;
#pragma unroll
  for (int i = 0; i < H; ++i) a0 += (uint64_t)x[i] * c(i);
#pragma unroll
  for (int i = H; i < K; ++i) a1 += (uint64_t)x[i] * c(i);
  if constexpr (K <= 11) {
    return redc(a0, m, minv);
  } else if constexpr (K <= 15) {
    return redc_sub(a0, m, minv);
  } else {
    return add_mod(redc(a0, m, minv), redc(a1, m, minv), m);
  }
}

// x_j = (sum_i xt_i (q/q_i) - v q) mod p_j
template <int K>
DI uint32_t q_to_p(const uint32_t (&xt)[K], uint32_t v, int j, const ConvTabs& tb) {
  return mont_dot<K>(xt, [&](int i) { return tb.qhat_p[i][j]; }, v, tb.negq_p[j], tb.p[j], tb.ppinv[j]);
}

}  // namespace hcnn
