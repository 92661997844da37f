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
// walks the ciphertexts in tiles of 128 (see k_rb_mac_tc below).  Exact and
// opt-in: 3.97 ms per MNIST step against 2.79 ms for k_rb_mac (DESIGN.md
// section 9, item 0).
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

constexpr int RBT_T = 256;                   // threads: two warps per TMEM lane quadrant
constexpr int RBT_SROW = 25 * 16;            // staging bytes per ciphertext: 24 digit rows x 4 positions,
                                             // padded so 8 consecutive rows hit distinct banks

struct RbtSmem {
  uint8_t a[RBT_NB][RBT_TILE];               // A tiles; after the MMAs the output staging
  uint8_t b[RBT_NB][RBT_BT];                 // key matrices of the four positions
  uint8_t stg[2][TC_M * RBT_SROW];           // digit rows as loaded, double-buffered
  uint64_t bar;
  uint32_t tmem;
};

DI void cp_async16(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes)
               : "memory");
}
DI void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
DI void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// dspec: [B][RB_A][D][N]; kt: [RB_A][N][RBT_BT]; zspec: [B][K][RB_A][2][N]
// One CTA per (four positions, r_a), walking the ciphertexts in tiles of
// 128: the next tile's digit rows stream into a staging buffer by
// asynchronous copies while the current one is transposed into the A tiles,
// multiplied (four MMAs, 512 TMEM columns) and reduced.
template <int DD>
__global__ void __launch_bounds__(RBT_T, 1)
    k_rb_mac_tc(const uint32_t* __restrict__ dspec, const uint8_t* __restrict__ kt, uint32_t* __restrict__ zspec,
                int nct, int K, int N, RbTabs rb) {
  static_assert(4 * DD <= RBT_KB, "digits exceed the 96-byte row");
  extern __shared__ __align__(1024) uint8_t smraw[];
  RbtSmem& sm = *reinterpret_cast<RbtSmem*>(smraw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int a = blockIdx.y;
  const int n0 = blockIdx.x * RBT_NB;
  const int K2 = 2 * K;
  const uint32_t r = rb.r[a], rinv = rb.rpinv[a];
  auto fetch = [&](int c0, int buf) {  // digit rows of ciphertexts c0 .. c0 + 127
    for (int task = tid; task < TC_M * DD; task += RBT_T) {
      const int row = task / DD, i = task % DD;
      const int ct = c0 + row;
      const uint32_t* src = ct < nct ? dspec + (((size_t)ct * RB_A + a) * DD + i) * N + n0 : dspec;
      cp_async16(&sm.stg[buf][row * RBT_SROW + i * 16], src, ct < nct ? 16u : 0u);
    }
    cp_async_commit();
  };
  {  // the key matrices of the four positions (contiguous), asynchronously
     // with the first tile's rows (same commit group)
    const uint8_t* src = kt + ((size_t)a * N + n0) * RBT_BT;
    for (int i = tid; i < RBT_NB * RBT_BT / 16; i += RBT_T) cp_async16(&sm.b[0][16 * i], src + 16 * i, 16u);
  }
  if (tid == 0) {
    mbar_init(&sm.bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&sm.tmem))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fetch(0, 0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = sm.tmem;
  const int quad = warp & 3, pp = warp >> 2;  // TMEM lane quadrant; positions 2 pp, 2 pp + 1
  const uint32_t tlane = tbase + ((uint32_t)(quad * 32) << 16);
  uint32_t phase = 0;
  int buf = 0;
  for (int c0 = 0; c0 < nct; c0 += TC_M, buf ^= 1) {
    if (c0 + TC_M < nct) fetch(c0 + TC_M, buf ^ 1);
    else cp_async_commit();  // an empty group keeps the wait count uniform
    cp_async_wait1();
    __syncthreads();  // this tile's rows have landed (every thread's copies)
    // transpose: staging [row][digit][4 positions] -> A tile k [row][4 digits]
    for (int task = tid; task < TC_M * (RBT_KB / 16); task += RBT_T) {
      const int row = task % TC_M, c = task / TC_M;  // rows fastest: conflict-free
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        v[u] = *reinterpret_cast<const uint4*>(&sm.stg[buf][row * RBT_SROW + (4 * c + u) * 16]);
      *reinterpret_cast<uint4*>(&sm.a[0][rbt_off(row, 16 * c)]) = make_uint4(v[0].x, v[1].x, v[2].x, v[3].x);
      *reinterpret_cast<uint4*>(&sm.a[1][rbt_off(row, 16 * c)]) = make_uint4(v[0].y, v[1].y, v[2].y, v[3].y);
      *reinterpret_cast<uint4*>(&sm.a[2][rbt_off(row, 16 * c)]) = make_uint4(v[0].z, v[1].z, v[2].z, v[3].z);
      *reinterpret_cast<uint4*>(&sm.a[3][rbt_off(row, 16 * c)]) = make_uint4(v[0].w, v[1].w, v[2].w, v[3].w);
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int k = 0; k < RBT_NB; ++k) rbt_mma(tbase + 128 * k, sm.a[k], sm.b[k]);
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
        tc_ld16(tlane + 128 * (2 * pp + h) + 16 * g, v);
        tc_wait_ld();
#pragma unroll
        for (int u = 0; u < 4; ++u) out[h][4 * g + u] = tc_redc(&v[4 * u], r, rinv);
      }
    }
    tc_fence_before();
    // the MMAs have read A: stage the sums there as [jp][row][4 positions]
    {
      const int row = quad * 32 + lane;
      uint8_t* ost = &sm.a[0][0];
#pragma unroll
      for (int jp = 0; jp < RBT_N / 4; ++jp)
        *reinterpret_cast<uint2*>(ost + (jp * TC_M + row) * 16 + pp * 8) = make_uint2(out[0][jp], out[1][jp]);
    }
    __syncthreads();
    for (int task = tid; task < TC_M * K2; task += RBT_T) {
      const int row = task % TC_M, jp = task / TC_M;
      const int ct = c0 + row;
      if (ct < nct)
        *reinterpret_cast<uint4*>(zspec + (size_t)ct * K * RB_A * 2 * N +
                                  ((size_t)(jp >> 1) * RB_A * 2 + (size_t)a * 2 + (jp & 1)) * N + n0) =
            *reinterpret_cast<const uint4*>(&sm.a[0][(jp * TC_M + row) * 16]);
    }
    __syncthreads();  // the staging reads are done before the next transpose
  }
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
}

}  // namespace hcnn
