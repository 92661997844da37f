// Exact RNS base-conversion kernels of the multiplication path, templated on
// the number of primes of q (K) and of the auxiliary base (KP = K+2 or K+3),
// one translation unit per K (conv_inst.cu).
//
//   k_extend  Q -> P extension of canonical lifts            (ring.py:286-295)
//   k_scale   exact round(t d / q) mod q of the 3-part tensor (bfv.py:325-328)
//             + base-w digits of the canonical c2           (bfv.py:350-365)
//   k_digits  base-w digits of part 2 of a 3-part ct         (bfv.py:350-365)
#pragma once
#include <cstdlib>
#include "common.cuh"

namespace hcnn {

struct TcTabs;

struct ConvLaunch {
  cudaStream_t stream;
  dim3 grid, block;
  const uint32_t* in;
  uint32_t* out;
  uint32_t* dig;
  int N;
  const TcTabs* tc;  // ops 4 / 5: the tensor-core conversion matrices (tc_bconv.cuh)
  size_t tiles;      // ops 4 / 5: 128-coefficient tiles
};

// write the D base-2^db digits of the canonical value held in S
template <int K>
DI void store_digits(const uint32_t (&S)[words_for(K)], uint32_t* __restrict__ dd, int N,
                     const ConvTabs& tb) {
  const int db = tb.digit_bits;
  const uint32_t mask = db == 32 ? 0xffffffffu : ((1u << db) - 1);
  if (db == 16) {
#pragma unroll
    for (int w = 0; w < words_for(K); ++w) {
      if (2 * w < tb.D) dd[(size_t)(2 * w) * N] = S[w] & 0xffffu;
      if (2 * w + 1 < tb.D) dd[(size_t)(2 * w + 1) * N] = S[w] >> 16;
    }
    return;
  }
#pragma unroll
  for (int w = 0; w < words_for(K); ++w) {
    const int per = 32 / db;
#pragma unroll 4
    for (int k = 0; k < per; ++k) {
      const int d = w * per + k;
      if (d < tb.D) dd[(size_t)d * N] = (S[w] >> (k * db)) & mask;
    }
  }
}

// in: [B][2][K][N] canonical residues; ext: [B][2][KP][N]
template <int K, int KP>
__global__ void __launch_bounds__(128)
    k_extend(const uint32_t* __restrict__ in, uint32_t* __restrict__ ext, int N,
             const __grid_constant__ ConvTabs tb) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const size_t poly = blockIdx.y;  // ct * 2 + part
  const uint32_t* src = in + poly * K * N + n;
  uint32_t x[K];
#pragma unroll
  for (int i = 0; i < K; ++i) x[i] = src[(size_t)i * N];
  uint32_t xt[K];
#pragma unroll
  for (int i = 0; i < K; ++i) xt[i] = mul_shoup(x[i], tb.qhi[i], tb.qhis[i], tb.q[i]);
  const uint32_t v = exact_v<K>(xt, tb);
  uint32_t* dst = ext + poly * KP * N + n;
#pragma unroll
  for (int j = 0; j < KP; ++j) dst[(size_t)j * N] = q_to_p<K>(xt, v, j, tb);
}

// d: [B][3][K+KP][N] exact tensor residues (coefficient domain).
// y3: [B][3][K][N] = round(t d / q) mod q per part; dig (optional): [B][D][N].
// Each thread handles V coefficients (n, n + blockDim, ...): the constant-bank
// operands are loaded once for all V and the V chains interleave.
template <int K, int KP, int V>
__global__ void __launch_bounds__(128)
    k_scale(const uint32_t* __restrict__ d, uint32_t* __restrict__ y3, uint32_t* __restrict__ dig,
            int N, const __grid_constant__ ConvTabs tb) {
  const int n0 = blockIdx.x * blockDim.x * V + threadIdx.x;
  if (n0 >= N) return;
  const int part = blockIdx.y % 3;
  const size_t ct = blockIdx.y / 3;
  const uint32_t* src = d + (size_t)blockIdx.y * (K + KP) * N + n0;

  // r = (t d + h) mod q, h = (q-1)/2, held as r~_i = r_i (q/q_i)^-1 mod q_i
  uint32_t rt[V][K];
  uint32_t dp[V][KP];
#pragma unroll
  for (int v = 0; v < V; ++v) {
#pragma unroll
    for (int i = 0; i < K; ++i)
      rt[v][i] = add_mod(mul_shoup(src[(size_t)i * N + v * blockDim.x], tb.A[i], tb.As[i], tb.q[i]), tb.B[i], tb.q[i]);
#pragma unroll
    for (int j = 0; j < KP; ++j) dp[v][j] = src[(size_t)(K + j) * N + v * blockDim.x];
  }
  uint32_t vq[V];
#pragma unroll
  for (int v = 0; v < V; ++v) vq[v] = exact_v<K>(rt[v], tb);

  // y = (t d + h - r) / q exactly, in P (centred, |y| < P/4): y~_j = y_j (P/p_j)^-1
  uint32_t yt[V][KP];
  uint64_t F[V];
#pragma unroll
  for (int v = 0; v < V; ++v) F[v] = 0;
#pragma unroll
  for (int j = 0; j < KP; ++j) {
    const uint32_t pj = tb.p[j];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const uint32_t rj = q_to_p<K>(rt[v], vq[v], j, tb);
      uint32_t acc = add_mod(mul_shoup(dp[v][j], tb.C[j], tb.Cs[j], pj), mul_shoup(pj - rj, tb.Ej[j], tb.Ejs[j], pj), pj);
      acc = add_mod(acc, tb.F[j], pj);
      yt[v][j] = acc;
      F[v] += frac59(acc, tb.pg[j], tb.pk[j]);
    }
  }
  uint32_t vp[V];
#pragma unroll
  for (int v = 0; v < V; ++v) vp[v] = (uint32_t)((F[v] + (FRAC_ONE >> 1)) >> FRAC_BITS);

  // back to Q: y_i = (sum_j y~_j (P/p_j) - vp P) mod q_i
  uint32_t yq[V][K];
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int v = 0; v < V; ++v)
      yq[v][i] = mont_dot<KP>(yt[v], [&](int j) { return tb.phat_q[j][i]; }, vp[v], tb.negp_q[i], tb.q[i], tb.qpinv[i]);
  uint32_t* dst = y3 + (size_t)blockIdx.y * K * N + n0;
#pragma unroll
  for (int v = 0; v < V; ++v)
#pragma unroll
    for (int i = 0; i < K; ++i) dst[(size_t)i * N + v * blockDim.x] = yq[v][i];

  if (part != 2 || dig == nullptr) return;
  // canonical binary of y_2 mod q, then base-w digits
#pragma unroll
  for (int v = 0; v < V; ++v) {
    uint32_t xt[K];
#pragma unroll
    for (int i = 0; i < K; ++i) xt[i] = mul_shoup(yq[v][i], tb.qhi[i], tb.qhis[i], tb.q[i]);
    uint64_t Fq = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) Fq += frac59(xt[i], tb.qg[i], tb.qk[i]);
    uint32_t S[words_for(K)];
    mw_lift<K>(xt, tb, S);
    mw_sub_mq<K>(S, (uint32_t)(Fq >> FRAC_BITS), tb);  // S - V q >= 0 with V in {v-1, v}
    {
      uint32_t Tq[words_for(K)];
#pragma unroll
      for (int w = 0; w < words_for(K); ++w) Tq[w] = S[w];
      if (!mw_sub_mq<K>(Tq, 1, tb)) {
#pragma unroll
        for (int w = 0; w < words_for(K); ++w) S[w] = Tq[w];
      }
    }
    store_digits<K>(S, dig + ct * tb.D * N + n0 + v * blockDim.x, N, tb);
  }
}

// digits of part 2 of a 3-part tensor in3: [B][3][K][N] -> dig [B][D][N]
template <int K>
__global__ void __launch_bounds__(128)
    k_digits(const uint32_t* __restrict__ in3, uint32_t* __restrict__ dig, int N,
             const __grid_constant__ ConvTabs tb) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const size_t ct = blockIdx.y;
  const uint32_t* src = in3 + (ct * 3 + 2) * K * N + n;
  uint32_t xt[K];
#pragma unroll
  for (int i = 0; i < K; ++i) xt[i] = mul_shoup(src[(size_t)i * N], tb.qhi[i], tb.qhis[i], tb.q[i]);
  const uint32_t v = exact_v<K>(xt, tb);
  uint32_t S[words_for(K)];
  mw_lift<K>(xt, tb, S);
  mw_sub_mq<K>(S, v, tb);
  store_digits<K>(S, dig + ct * tb.D * N + n, N, tb);
}

// Exact decryption rounding (bfv.py:229-250): phase residues [B][K][N]
// (canonical, coefficient domain) -> m = round(t x / q) mod t as u64 [B][N].
// With x = sum xt_i (q/q_i) - v q:  t x / q + h/q = sum_i t xt_i / q_i + h/q - v t,
// t xt_i = c_i q_i + rho_i, so m = (sum c_i + floor(sum rho_i/q_i + h/q)) mod t;
// the floor is a fixed-point estimate with an exact multiword decision near
// integers, like exact_v.
template <int K>
__global__ void __launch_bounds__(128)
    k_decrypt_round(const uint32_t* __restrict__ ph, uint64_t* __restrict__ m, int N,
                    const __grid_constant__ ConvTabs tb) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const size_t ct = blockIdx.y;
  const uint32_t* src = ph + ct * K * N + n;
  uint32_t rho[K];
  uint64_t csum = 0, F = tb.H;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const uint32_t xt = mul_shoup(src[(size_t)i * N], tb.qhi[i], tb.qhis[i], tb.q[i]);
    const uint64_t u = (uint64_t)xt * tb.dec_f[i];          // < q_i^2
    uint64_t qh = __umul64hi(u, tb.qmu[i]);                 // floor(u/q_i) or one less
    uint64_t r = u - qh * tb.q[i];
    if (r >= tb.q[i]) {
      r -= tb.q[i];
      ++qh;
    }
    rho[i] = (uint32_t)r;
    csum += tb.dec_a[i] * xt + qh;  // < K * 2^49: no overflow for t < 2^48
    F += frac59(rho[i], tb.qg[i], tb.qk[i]);
  }
  uint32_t V = (uint32_t)(F >> FRAC_BITS);
  if ((F & FRAC_MASK) >= FRAC_ONE - (K + 1) * FRAC_ERR) {
    // exact: is sum rho_i (q/q_i) + h >= (V+1) q ?
    uint32_t S[words_for(K)];
    mw_lift<K>(rho, tb, S);
    uint64_t carry = 0;
#pragma unroll
    for (int w = 0; w < words_for(K); ++w) {
      const uint64_t s = (uint64_t)S[w] + tb.h_w[w] + carry;
      S[w] = (uint32_t)s;
      carry = s >> 32;
    }
    if (!mw_sub_mq<K>(S, V + 1, tb)) V += 1;
  }
  uint64_t total = csum + V;
  const uint64_t qh = __umul64hi(total, tb.tmu);
  uint64_t r = total - qh * tb.t;
  while (r >= tb.t) r -= tb.t;
  m[ct * N + n] = r;
}

}  // namespace hcnn

#include "tc_bconv.cuh"

namespace hcnn {

// resident CTAs per SM of the tensor-core conversions (TMEM: 64 columns each,
// at most 8; registers: 7 at __launch_bounds__(128, 7))
constexpr int TC_CTAS_PER_SM = 7;

// op: 0 extend, 1 scale, 2 digits, 3 decrypt rounding,
//     4 extend / 5 scale on the tensor cores (K, KP <= 15, N % 128 == 0)
template <int K, int KP>
cudaError_t conv_launch(int op, const ConvLaunch& a, const ConvTabs& tb) {
  switch (op) {
    case 4:
    case 5: {
      if constexpr (K <= 15 && KP <= 15) {
        static_assert(sizeof(TcSmem) <= 48 * 1024, "no opt-in needed");
        // resident CTAs per SM, per device and kernel (the occupancy query
        // costs host time: once per device)
        static int slots[2][2][64];
        static const bool wide = [] {  // tuning probe (tools/tc_sweep.sh): 128 TMEM columns, 4 CTAs per SM
          const char* ce = getenv("HCNN_TC_COLS");
          return ce && atoi(ce) == 128;
        }();
        int dev = 0;
        cudaGetDevice(&dev);
        int& per = slots[op - 4][wide][dev & 63];
        if (per == 0) {
          // __launch_bounds__(128, 7) caps the registers at 72: 7 CTAs fit by
          // registers, shared memory (17 KB each) and TMEM (64 columns each;
          // 4 CTAs with 128)
          int sms = 0;
          cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
          int occ = wide ? 4 : TC_CTAS_PER_SM;
          if (const char* e = getenv("HCNN_TC_CTAS")) {  // tuning probe
            const int c = atoi(e);
            if (c > 0 && c < occ) occ = c;
          }
          per = sms * occ;
        }
        const size_t cap = (size_t)per;
        const unsigned grid = (unsigned)(a.tiles < cap ? a.tiles : cap);
        if (grid == 0) return cudaSuccess;
        if (op == 4) {
          if (wide)
            k_extend_tc<K, KP, 128><<<grid, TC_M, sizeof(TcSmem), a.stream>>>(a.in, a.out, a.N, a.tiles, tb, *a.tc);
          else
            k_extend_tc<K, KP, 64><<<grid, TC_M, sizeof(TcSmem), a.stream>>>(a.in, a.out, a.N, a.tiles, tb, *a.tc);
        } else {
          if (wide)
            k_scale_tc<K, KP, 128><<<grid, TC_M, sizeof(TcSmem), a.stream>>>(a.in, a.out, a.dig, a.N, a.tiles, tb,
                                                                              *a.tc);
          else
            k_scale_tc<K, KP, 64><<<grid, TC_M, sizeof(TcSmem), a.stream>>>(a.in, a.out, a.dig, a.N, a.tiles, tb,
                                                                             *a.tc);
        }
        break;
      } else {
        return cudaErrorInvalidValue;
      }
    }
    case 0:
      k_extend<K, KP><<<a.grid, a.block, 0, a.stream>>>(a.in, a.out, a.N, tb);
      break;
    case 1: {
      // V = 2 coefficients per thread: faster up to K = 7 (K = 6: 0.95 vs
      // 1.01 us per ciphertext), level at 8, slower above (K = 10: 1.96 vs
      // 1.88; K = 11: 2.47 vs 2.19 us: registers); the kernel is
      // fmaheavy-bound (profiles/r1_micro_scale_v2.jsonl)
      if (K <= 7 && a.N % (2 * a.block.x) == 0) {
        dim3 g2(a.grid.x / 2 > 0 ? a.grid.x / 2 : 1, a.grid.y);
        k_scale<K, KP, 2><<<g2, a.block, 0, a.stream>>>(a.in, a.out, a.dig, a.N, tb);
      } else {
        k_scale<K, KP, 1><<<a.grid, a.block, 0, a.stream>>>(a.in, a.out, a.dig, a.N, tb);
      }
      break;
    }
    case 2:
      k_digits<K><<<a.grid, a.block, 0, a.stream>>>(a.in, a.dig, a.N, tb);
      break;
    case 3:
      k_decrypt_round<K><<<a.grid, a.block, 0, a.stream>>>(a.in, reinterpret_cast<uint64_t*>(a.out), a.N, tb);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace hcnn

#define HCNN_K_LIST(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)
#define HCNN_DECLARE_CONV(K) \
  cudaError_t hcnn_conv_launch_##K(int op, int kp, const hcnn::ConvLaunch& a, const hcnn::ConvTabs& tb);
HCNN_K_LIST(HCNN_DECLARE_CONV)
