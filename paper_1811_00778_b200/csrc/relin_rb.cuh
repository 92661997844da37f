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
#include "tc_bconv.cuh"

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

// ---------------------------------------------------------------------------
// Step 2 on the tensor cores (flag RB_MAC_TC).  For one r_a and one
// coefficient n, Z[ct][jp] = sum_i D[ct][i] K[i][jp] is a (ciphertexts x D) x
// (D x 2K) product with a key matrix that changes with n; byte-split like
// tc_bconv.cuh: A[ct][4i+b] = byte b of D[ct][i], B_n[4jp+e][4i+b] = byte e
// of (2^8b K[i][jp] 2^32 mod r_a) (built once per key by k_rb_key_tc), four
// s32 columns per output (< 92 * 255^2 < 2^23), one REDC.  A CTA takes four
// consecutive positions n (16-byte loads and stores of the tiled rows) and
// walks the ciphertexts in tiles of 128; two positions per MMA batch (TMEM
// 256 columns, two CTAs per SM).  Exact, but off by default: at set 1 it
// moves the algorithmic bytes (ncu: 1.72 GB read, 1.52 GB written per launch)
// at 0.8 TB/s, latency-bound with 8 warps per SM (3.6 vs 1.39 ms per launch
// for k_rb_mac); a deeper pipeline (asynchronous copies into a staging tile,
// more warps for the REDC epilogue) is what it needs.
constexpr int RBT_KB = 96;                   // K bytes: 4 D <= 92
constexpr int RBT_SBO = RBT_KB / 16 * 128;   // 768: next 8 rows
constexpr int RBT_N = 96;                    // columns: 4 x 2K <= 88
constexpr int RBT_TILE = TC_M * RBT_KB;      // 12 KB (A, 128 ciphertexts)
constexpr int RBT_BT = RBT_N * RBT_KB;       // 9 KB (B, one position)
constexpr int RBT_NB = 4;                    // positions per CTA

__host__ __device__ constexpr int rbt_off(int row, int k) {
  return (row >> 3) * RBT_SBO + (k >> 4) * 128 + (row & 7) * 16 + (k & 15);
}

DI uint64_t rbt_desc(const void* smem) {
  const uint32_t a = smem_u32(smem);
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(RBT_SBO >> 4) << 32) |
         (1ull << 46);
}

// D[tmem] = A x B^T over 96 K-bytes (three k32 steps)
DI void rbt_mma(uint32_t tmem, const uint8_t* a, const uint8_t* b) {
  const uint64_t da = rbt_desc(a), db = rbt_desc(b);
  constexpr uint32_t id = (2u << 4) | ((uint32_t)(RBT_N >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);
#pragma unroll
  for (int k = 0; k < RBT_KB / 32; ++k) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
        "l"(da + 16 * k), "l"(db + 16 * k), "r"(id), "r"(k)
        : "memory");
  }
}

// kx: [RB_A][D][2K][N] key spectra mod r_a -> kt: [RB_A][N][RBT_BT] bytes
// (zero-filled beforehand)
__global__ void k_rb_key_tc(const uint32_t* __restrict__ kx, uint8_t* __restrict__ kt, int D, int K2, int N,
                            RbTabs rb) {
  const size_t total = (size_t)RB_A * D * K2 * N;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int n = (int)(idx % N);
  const size_t row = idx / N;  // (a, i, jp)
  const int jp = (int)(row % K2);
  const int i = (int)((row / K2) % D);
  const int a = (int)(row / ((size_t)K2 * D));
  const uint64_t r = rb.r[a];
  const uint64_t k = kx[idx] % r;
  uint8_t* dst = kt + ((size_t)a * N + n) * RBT_BT;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const uint64_t g = ((uint64_t)1 << (8 * b + 32)) % r;  // 2^(8b+32) mod r
    const uint32_t c = (uint32_t)(k * g % r);
#pragma unroll
    for (int e = 0; e < 4; ++e) dst[rbt_off(4 * jp + e, 4 * i + b)] = (uint8_t)(c >> (8 * e));
  }
}

struct RbtSmem {
  uint8_t a[RBT_NB][RBT_TILE];
  uint8_t b[RBT_NB][RBT_BT];
  uint64_t bar;
  uint32_t tmem;
};

// dspec: [B][RB_A][D][N]; kt: [RB_A][N][RBT_BT]; zspec: [B][K][RB_A][2][N]
template <int DD>
__global__ void __launch_bounds__(TC_M, 2)
    k_rb_mac_tc(const uint32_t* __restrict__ dspec, const uint8_t* __restrict__ kt, uint32_t* __restrict__ zspec,
                int nct, int K, int N, RbTabs rb) {
  static_assert(4 * DD <= RBT_KB, "digits exceed the 96-byte row");
  extern __shared__ __align__(1024) uint8_t smraw[];
  RbtSmem& sm = *reinterpret_cast<RbtSmem*>(smraw);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int a = blockIdx.y;
  const int n0 = blockIdx.x * RBT_NB;
  const int K2 = 2 * K;
  const uint32_t r = rb.r[a], rinv = rb.rpinv[a];
  {  // the key matrices of the four positions (contiguous)
    const uint4* src = reinterpret_cast<const uint4*>(kt + ((size_t)a * N + n0) * RBT_BT);
    uint4* dst = reinterpret_cast<uint4*>(&sm.b[0][0]);
    for (int i = tid; i < RBT_NB * RBT_BT / 16; i += TC_M) dst[i] = __ldg(src + i);
  }
  if (tid == 0) {
    mbar_init(&sm.bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&sm.tmem))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = sm.tmem;
  const uint32_t tlane = tbase + ((uint32_t)(warp * 32) << 16);
  uint32_t phase = 0;
  for (int c0 = 0; c0 < nct; c0 += TC_M) {
    const int ct = c0 + tid;
    const bool live = ct < nct;
    {  // this thread's row of the four A tiles: 16-byte loads of its digit rows
      uint4 d[DD];
      const uint4* dp = reinterpret_cast<const uint4*>(dspec + ((size_t)ct * RB_A + a) * DD * N + n0);
#pragma unroll
      for (int i = 0; i < DD; ++i) d[i] = live ? __ldg(dp + (size_t)i * (N / 4)) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int c = 0; c < RBT_KB / 16; ++c) {
        uint32_t w[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = 4 * c + u;
          const uint4 v = i < DD ? d[i] : make_uint4(0, 0, 0, 0);
          w[0][u] = v.x;
          w[1][u] = v.y;
          w[2][u] = v.z;
          w[3][u] = v.w;
        }
#pragma unroll
        for (int k = 0; k < RBT_NB; ++k)
          *reinterpret_cast<uint4*>(&sm.a[k][rbt_off(tid, 16 * c)]) = make_uint4(w[k][0], w[k][1], w[k][2], w[k][3]);
      }
    }
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      fence_proxy_async();
      tc_fence_before();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        rbt_mma(tbase, sm.a[2 * half], sm.b[2 * half]);
        rbt_mma(tbase + 128, sm.a[2 * half + 1], sm.b[2 * half + 1]);
        tc_commit(&sm.bar);
      }
      mbar_wait(&sm.bar, phase);
      phase ^= 1;
      tc_fence_after();
      uint32_t out[2][RBT_N / 4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int g = 0; g < RBT_N / 16; ++g) {
          uint32_t v[16];
          tc_ld16(tlane + 128 * h + 16 * g, v);
          tc_wait_ld();
#pragma unroll
          for (int u = 0; u < 4; ++u) out[h][4 * g + u] = tc_redc(&v[4 * u], r, rinv);
        }
      }
      tc_fence_before();
      if (live) {  // positions n0 + 2 half, + 1 of every (j, part) row
        uint32_t* zp = zspec + (size_t)ct * K * RB_A * 2 * N + (size_t)a * 2 * N + n0 + 2 * half;
#pragma unroll
        for (int jp = 0; jp < RBT_N / 4; ++jp) {
          if (jp < K2)
            *reinterpret_cast<uint2*>(zp + ((size_t)(jp >> 1) * RB_A * 2 + (jp & 1)) * N) =
                make_uint2(out[0][jp], out[1][jp]);
        }
      }
    }
    __syncthreads();  // A tiles and the accumulators are free for the next tile
  }
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase) : "memory");
}

}  // namespace hcnn
