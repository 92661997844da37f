// Relinearisation over the shared basis R (RbTabs, common.cuh): step 2 (the
// key-switching multiply-accumulate) and the key preparation.  Steps 1 and 3
// (forward / inverse NTTs mod r_a, the exact CRT back to q_j) are per ring
// degree in ntt_kernels.cuh (k_rb_fwd, k_rb_inv).
//
// The reference (bfv.py:368-404) multiplies the NTTs of the D digits of c2 by
// the key rows mod every q_j: D K forward transforms.  Here the integer sums
// Z_{j,part} = sum_i d_i k_{i,j,part} (key rows centred mod q_j) are formed
// mod r0, r1, r2 instead: 3 D forward and 6 K inverse transforms (63 + 66 at
// set 1 against 231 + 22), with 3 x the multiply-accumulates.  The result mod
// q_j is the same residue the reference computes, bit for bit.
#pragma once
#include "common.cuh"

namespace hcnn {

constexpr int RB_MAC_C = 32;                     // coefficients per CTA tile
constexpr int RB_MAC_QD = RB_MAC_C / 4;          // 16-byte quads per tile
constexpr int RB_MAC_T = 256;                    // threads
constexpr int RB_MAC_CS = RB_MAC_T / RB_MAC_QD;  // ciphertexts in flight per CTA
constexpr int RB_DMAX = 23;                      // D (r_a - 1)^2 < 2^64 without folds

// s mod r in [0, 2r) for any 64-bit s and r < 2^30: hi 2^32 + lo with the
// high word through Shoup's 2^32 mod r and the low word through Shoup's 1
// (five 32-bit multiplies; a 64-bit Barrett step costs about twice that)
DI uint32_t fold64(uint64_t s, uint2 t32, uint32_t one, uint32_t r) {
  const uint32_t hi = (uint32_t)(s >> 32), lo = (uint32_t)s;
  const uint32_t u = mul_shoup_lazy(hi, t32.x, t32.y, r) + (lo - __umulhi(lo, one) * r);  // < 4r
  return umin_u32(u, u - 2 * r);
}

// Step 2.  Grid (N / 32, RB_A, ct ranges); each CTA stages the key tile
// kx[a][i][jp][c0 .. c0+32) (jp = 2 j + part) in shared memory once, then each
// thread takes one 4-coefficient quad of a ciphertext: its DD digit spectra
// stay in registers, and for every (j, part) 4 lazy 64-bit dot products of
// length DD (< 2^64: r_a < 2^32 / sqrt(23)) are reduced mod r_a.  A warp is
// 8 quads x 4 ciphertexts: key reads are 128-byte broadcasts, digit and
// output rows 4 x 128 contiguous bytes.
// dspec: [B][RB_A][DD][N]; kx: [RB_A][DD][2K][N]; zspec: [B][K][RB_A][2][N]
// (all rows in the tiled layout of the transforms, which the products keep).
template <int DD>
__global__ void __launch_bounds__(RB_MAC_T, 2)
    k_rb_mac(const uint32_t* __restrict__ dspec, const uint32_t* __restrict__ kx, uint32_t* __restrict__ zspec,
             int nct, int K, int N, int cts_per_cta, RbTabs rb) {
  extern __shared__ uint4 ks[];  // [DD][2K][QD]
  const int a = blockIdx.y;
  const int c0 = blockIdx.x * RB_MAC_C;
  const int K2 = 2 * K;
  const uint32_t p = rb.r[a];
  const uint2 t32 = rb.t32[a];
  const uint32_t one = rb.one[a];
  const size_t rowq = (size_t)N / 4;  // uint4 per row
  {
    const uint4* src = reinterpret_cast<const uint4*>(kx + (size_t)a * DD * K2 * N + c0);
    for (int idx = threadIdx.x; idx < DD * K2 * RB_MAC_QD; idx += RB_MAC_T)
      ks[idx] = __ldg(src + (size_t)(idx / RB_MAC_QD) * rowq + idx % RB_MAC_QD);
  }
  __syncthreads();
  const int q = threadIdx.x % RB_MAC_QD;
  const int cs = threadIdx.x / RB_MAC_QD;
  const size_t ct0 = (size_t)blockIdx.z * cts_per_cta;
  size_t ct1 = ct0 + cts_per_cta;
  if (ct1 > (size_t)nct) ct1 = nct;
  for (size_t ct = ct0 + cs; ct < ct1; ct += RB_MAC_CS) {
    uint4 d[DD];
    const uint4* dp = reinterpret_cast<const uint4*>(dspec + (ct * RB_A + a) * (size_t)DD * N + c0) + q;
#pragma unroll
    for (int i = 0; i < DD; ++i) d[i] = __ldg(dp + i * rowq);
    uint4* zp = reinterpret_cast<uint4*>(zspec + ct * (size_t)K * RB_A * 2 * N + (size_t)a * 2 * N + c0) + q;
    for (int j = 0; j < K; ++j) {  // both parts of q_j: 8 independent chains
      uint64_t s0 = 0, s1 = 0, s2 = 0, s3 = 0, u0 = 0, u1 = 0, u2 = 0, u3 = 0;
      const uint4* kp = ks + 2 * j * RB_MAC_QD + q;
#pragma unroll
      for (int i = 0; i < DD; ++i) {
        const uint4 k = kp[i * K2 * RB_MAC_QD];
        const uint4 l = kp[i * K2 * RB_MAC_QD + RB_MAC_QD];
        s0 += (uint64_t)d[i].x * k.x;
        s1 += (uint64_t)d[i].y * k.y;
        s2 += (uint64_t)d[i].z * k.z;
        s3 += (uint64_t)d[i].w * k.w;
        u0 += (uint64_t)d[i].x * l.x;
        u1 += (uint64_t)d[i].y * l.y;
        u2 += (uint64_t)d[i].z * l.z;
        u3 += (uint64_t)d[i].w * l.w;
      }
      // rows (ct, j, a, part 0 / 1); values in [0, 2 r_a)
      zp[(size_t)j * RB_A * 2 * rowq] = make_uint4(fold64(s0, t32, one, p), fold64(s1, t32, one, p),
                                                   fold64(s2, t32, one, p), fold64(s3, t32, one, p));
      zp[((size_t)j * RB_A * 2 + 1) * rowq] = make_uint4(fold64(u0, t32, one, p), fold64(u1, t32, one, p),
                                                         fold64(u2, t32, one, p), fold64(u3, t32, one, p));
    }
  }
}

// reference-order NTT rows -> device spectral positions (dst[i] = src[brv(i)])
__global__ void k_ref_to_spectral(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, int logn) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = 1 << logn;
  if (i >= n) return;
  const size_t row = blockIdx.y;
  dst[row * n + i] = src[row * n + (int)(__brev((unsigned)i) >> (32 - logn))];
}

// coefficient-domain key rows [D][2][K][N] (canonical mod q_j) -> rows
// [RB_A][D][2K][N] of the centred values mod r_a (coefficient domain)
__global__ void k_rb_key_rows(const uint32_t* __restrict__ coef, uint32_t* __restrict__ out, int D, int K,
                              int N, const uint32_t* __restrict__ primes, RbTabs rb) {
  const size_t total = (size_t)D * 2 * K * N;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int n = (int)(idx % N);
  const size_t row = idx / N;  // (i, part, j)
  const int j = (int)(row % K);
  const int part = (int)((row / K) % 2);
  const size_t i = row / (2 * K);
  const uint32_t qj = primes[j];
  const uint32_t v = coef[idx];
  const bool neg = v > (qj - 1) / 2;  // centred value v - q_j
  const uint32_t mag = neg ? qj - v : v;
#pragma unroll
  for (int a = 0; a < RB_A; ++a) {
    const uint32_t r = rb.r[a];
    const uint32_t m = mag % r;
    const uint32_t val = (neg && m) ? r - m : m;
    out[(((size_t)a * D + i) * 2 * K + 2 * j + part) * N + n] = val;
  }
}

}  // namespace hcnn
