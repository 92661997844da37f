// Exact RNS base conversion on the tensor cores (tcgen05.mma kind::i8).
//
// A base conversion x_j = (sum_i xt_i c_ij + v c_vj) mod m_j (ring.py:286-302;
// the Q -> P extension of k_extend and both conversions of k_scale) is, per
// coefficient, a dot product against a constant matrix: a GEMM with the
// coefficients as M.  The 30-bit operands are split into bytes so that the
// products are exact u8 x u8 -> s32 tensor-core work:
//
//   xt_i c_ij = sum_b byte_b(xt_i) 2^8b c_ij
//            == sum_b byte_b(xt_i) c'_ijb              (mod m_j),
//   c'_ijb    = 2^8b c_ij 2^32 mod m_j  (Montgomery form, < 2^30)
//            = sum_e byte_e(c'_ijb) 2^8e,
//
// so with A[n][4i+b] = byte_b(xt_i) (the residue words themselves, little
// endian) and B[4j+e][4i+b] = byte_e(c'_ijb), the four accumulator columns
// acc_{j,e} = sum_{i,b} A B (< (4K+1) 255^2 < 2^22) give
// S_j = sum_e acc_{j,e} 2^8e < 2^46.1 == x_j 2^32 (mod m_j), and one REDC
// returns x_j fully reduced.  The overflow count v (< 256) is one more A byte
// whose B column holds the bytes of -q (or -P).  Every output residue equals
// the integer path's (q_to_p / mont_dot), bit for bit.
//
// Tile: 128 coefficients (TMEM lanes) x 64 K-bytes (two k32 MMAs) x 64
// columns (4 per output prime, up to 16 primes).  Operands in shared memory
// use the canonical K-major no-swizzle layout: 8-row x 16-byte core matrices,
// LBO (next 16 K-bytes) = 128 B, SBO (next 8 rows) = 512 B.
#pragma once
#include "common.cuh"
#include "tma.cuh"

namespace hcnn {

constexpr int TC_M = 128;        // coefficients per tile
constexpr int TC_KB = 64;        // K bytes per row
constexpr int TC_N = 64;         // accumulator columns per conversion
constexpr int TC_TILE_BYTES = TC_M * TC_KB;  // 8 KB (A); B is TC_N x TC_KB = 4 KB
constexpr int TC_LBO = 128, TC_SBO = 512;

// Device byte matrices of the two conversions (core-matrix layout, 4 KB each).
struct TcTabs {
  const uint32_t* bqp;  // Q -> P: rows 4j+e (j < KP), K bytes 4i+b (i < K), 4K = v
  const uint32_t* bpq;  // P -> Q: rows 4i+e (i < K), K bytes 4j+b (j < KP), 4KP = v
  const uint32_t* bsc;  // scale, Q -> P with -E_j folded in: byte e of 2^8b (-E_j c_ij) 2^32 mod p_j
  const uint32_t* bdg;  // canonical lift for the digits: row s (byte s of the
                        // lift), K byte 4i+b: byte s-b of q/q_i; 4K: byte s of
                        // 2^(32 W) - q
};

// byte offset of (row, k) in a core-matrix tile
__host__ __device__ constexpr int tc_off(int row, int k) {
  return (row >> 3) * TC_SBO + (k >> 4) * TC_LBO + (row & 7) * 16 + (k & 15);
}

DI uint64_t tc_sdesc(const void* smem) {
  const uint32_t a = smem_u32(smem);
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(TC_LBO >> 4) << 16) | ((uint64_t)(TC_SBO >> 4) << 32) |
         (1ull << 46);  // version 1 (sm_100), base offset 0, SWIZZLE_NONE
}

// kind::i8 instruction descriptor: u8 x u8 -> s32, both K-major, M = 128
__host__ __device__ constexpr uint32_t tc_idesc(int n) {
  return (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);
}

// COLS TMEM columns per CTA (64: one conversion's accumulator)
template <int COLS>
DI void tc_alloc(uint32_t* slot, int warp) {
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
                 "n"(COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
}
template <int COLS>
DI void tc_dealloc(uint32_t base, int warp) {
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(COLS) : "memory");
}
DI void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
DI void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] = A x B^T over 64 K-bytes (two k32 steps), one thread issues
DI void tc_mma64(uint32_t tmem, const uint8_t* a, const uint8_t* b) {
  const uint64_t da = tc_sdesc(a), db = tc_sdesc(b);
  constexpr uint32_t id = tc_idesc(TC_N);
  // k32 step = 2 core matrices along K = 256 B = 16 in descriptor units
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, 0, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(id)
      : "memory");
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, 1, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
      "l"(da + 16), "l"(db + 16), "r"(id)
      : "memory");
}

DI void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// 16 consecutive accumulator columns of this thread's lane
DI void tc_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
DI void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// this thread's A row (16 words: the residues, then v, then zeros)
template <int NW>
DI void tc_put_row(uint8_t* a, int row, const uint32_t (&w)[NW], uint32_t v) {
  static_assert(NW <= 15, "4 NW + 1 bytes must fit the 64-byte row");
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = 4 * c + u;
      q[u] = i < NW ? w[i] : i == NW ? v : 0u;
    }
    *reinterpret_cast<uint4*>(a + tc_off(row, 16 * c)) = make_uint4(q[0], q[1], q[2], q[3]);
  }
}

// S = sum_e acc_e 2^8e (< 2^46.1) -> S 2^-32 mod m, fully reduced
DI uint32_t tc_redc(const uint32_t* acc, uint32_t m, uint32_t minv) {
  const uint64_t S = (uint64_t)acc[0] + ((uint64_t)acc[1] << 8) + ((uint64_t)acc[2] << 16) +
                     ((uint64_t)acc[3] << 24);
  const uint32_t u = (uint32_t)S * minv;
  const uint32_t r = (uint32_t)((S + (uint64_t)u * m) >> 32);  // < 2^14.1 + m
  return umin_u32(r, r - m);
}

// Columns [0, 4 NOUT) of the accumulator at taddr -> NOUT residues
template <int NOUT, class Fn>
DI void tc_drain(uint32_t taddr, Fn fn) {
#pragma unroll
  for (int g = 0; g < (4 * NOUT + 15) / 16; ++g) {
    uint32_t v[16];
    tc_ld16(taddr + 16 * g, v);
    tc_wait_ld();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = 4 * g + u;
      if (j < NOUT) fn(j, &v[4 * u]);
    }
  }
}

// Shared layout of the tensor-core conversion kernels
struct TcSmem {
  uint8_t a[TC_TILE_BYTES];
  uint8_t bqp[TC_N * TC_KB];
  uint8_t bpq[TC_N * TC_KB];
  uint8_t bdg[TC_N * TC_KB];
  uint64_t bar;
  uint32_t tmem;
};

DI void tc_load_b(uint8_t* dst, const uint32_t* __restrict__ src) {
  for (int i = threadIdx.x; i < TC_N * TC_KB / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(dst)[i] = __ldg(reinterpret_cast<const uint4*>(src) + i);
}

// k_extend on the tensor cores.  in: [B][2][K][N]; ext: [B][2][KP][N].
// Persistent: CTA walks 128-coefficient tiles (poly, n0).
template <int K, int KP, int COLS>
__global__ void __launch_bounds__(TC_M, 7)
    k_extend_tc(const uint32_t* __restrict__ in, uint32_t* __restrict__ ext, int N, size_t tiles,
                const __grid_constant__ ConvTabs tb, const __grid_constant__ TcTabs tc) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  TcSmem& sm = *reinterpret_cast<TcSmem*>(smraw);
  const int tid = threadIdx.x, warp = tid >> 5;
  tc_load_b(sm.bqp, tc.bqp);
  if (tid == 0) {
    mbar_init(&sm.bar, 1);
    fence_mbar_init();
  }
  tc_alloc<COLS>(&sm.tmem, warp);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = sm.tmem;
  const uint32_t tlane = tbase + ((uint32_t)(warp * 32) << 16);
  const int per = N / TC_M;
  uint32_t phase = 0;
  // the next tile's residues load while this tile's MMA runs
  uint32_t x[K];
  auto load = [&](size_t t) {
    if (t >= tiles) return;
    const uint32_t* src = in + (t / per) * K * N + (int)(t % per) * TC_M + tid;
#pragma unroll
    for (int i = 0; i < K; ++i) x[i] = src[(size_t)i * N];
  };
  load(blockIdx.x);
  for (size_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const size_t poly = t / per;
    const int n = (int)(t % per) * TC_M + tid;
    {
      uint32_t xt[K];
#pragma unroll
      for (int i = 0; i < K; ++i) xt[i] = mul_shoup(x[i], tb.qhi[i], tb.qhis[i], tb.q[i]);
      const uint32_t v = exact_v<K>(xt, tb);
      tc_put_row<K>(sm.a, tid, xt, v);
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      tc_mma64(tbase, sm.a, sm.bqp);
      tc_commit(&sm.bar);
    }
    load(t + gridDim.x);
    mbar_wait(&sm.bar, phase);
    phase ^= 1;
    tc_fence_after();
    uint32_t* dst = ext + poly * KP * N + n;
    tc_drain<KP>(tlane, [&](int j, const uint32_t* acc) { dst[(size_t)j * N] = tc_redc(acc, tb.p[j], tb.ppinv[j]); });
    tc_fence_before();
    __syncthreads();  // A and the accumulator are free for the next tile
  }
  tc_fence_after();
  tc_dealloc<COLS>(tbase, warp);
}

// k_scale on the tensor cores (same outputs as k_scale<K, KP, 1>).
// d: [B][3][K+KP][N]; y3: [B][3][K][N]; dig (optional): [B][D][N].
template <int K, int KP, int COLS>
__global__ void __launch_bounds__(TC_M, 7)
    k_scale_tc(const uint32_t* __restrict__ d, uint32_t* __restrict__ y3, uint32_t* __restrict__ dig, int N,
               size_t tiles, const __grid_constant__ ConvTabs tb, const __grid_constant__ TcTabs tc) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  TcSmem& sm = *reinterpret_cast<TcSmem*>(smraw);
  const int tid = threadIdx.x, warp = tid >> 5;
  tc_load_b(sm.bqp, tc.bsc);  // the scale's Q -> P matrix (-E_j folded in)
  tc_load_b(sm.bpq, tc.bpq);
  if (dig != nullptr) tc_load_b(sm.bdg, tc.bdg);
  if (tid == 0) {
    mbar_init(&sm.bar, 1);
    fence_mbar_init();
  }
  tc_alloc<COLS>(&sm.tmem, warp);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = sm.tmem;
  const uint32_t tlane = tbase + ((uint32_t)(warp * 32) << 16);
  const int per = N / TC_M;
  uint32_t phase = 0;
  for (size_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const size_t row = t / per;  // ct * 3 + part
    const int part = (int)(row % 3);
    const size_t ct = row / 3;
    const int n = (int)(t % per) * TC_M + tid;
    const uint32_t* src = d + row * (K + KP) * N + n;
    // r = (t d + h) mod q as r~_i = r_i (q/q_i)^-1 mod q_i
    {
      uint32_t rt[K];
#pragma unroll
      for (int i = 0; i < K; ++i)
        rt[i] = add_mod(mul_shoup(src[(size_t)i * N], tb.A[i], tb.As[i], tb.q[i]), tb.B[i], tb.q[i]);
      const uint32_t vq = exact_v<K>(rt, tb);
      tc_put_row<K>(sm.a, tid, rt, vq);
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      tc_mma64(tbase, sm.a, sm.bqp);
      tc_commit(&sm.bar);
    }
    // the P residues of d load while the MMA runs
    uint32_t dp[KP];
#pragma unroll
    for (int j = 0; j < KP; ++j) dp[j] = src[(size_t)(K + j) * N];
    mbar_wait(&sm.bar, phase);
    phase ^= 1;
    tc_fence_after();
    // y = (t d + h - r) / q exactly, in P: y~_j
    uint32_t yt[KP];
    uint64_t F = 0;
    tc_drain<KP>(tlane, [&](int j, const uint32_t* acc) {
      const uint32_t pj = tb.p[j];
      const uint32_t er = tc_redc(acc, pj, tb.ppinv[j]);  // (p_j - r_j) E_j mod p_j
      uint32_t a = add_mod(mul_shoup(dp[j], tb.C[j], tb.Cs[j], pj), er, pj);
      a = add_mod(a, tb.F[j], pj);
      yt[j] = a;
      F += frac59(a, tb.pg[j], tb.pk[j]);
    });
    const uint32_t vp = (uint32_t)((F + (FRAC_ONE >> 1)) >> FRAC_BITS);
    // the MMA has read A (its commit arrived) and every lane has drained the
    // accumulator (barrier below): A takes the P row, the columns the sums
    tc_put_row<KP>(sm.a, tid, yt, vp);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      tc_mma64(tbase + (COLS >= 128 ? TC_N : 0), sm.a, sm.bpq);
      tc_commit(&sm.bar);
    }
    mbar_wait(&sm.bar, phase);
    phase ^= 1;
    tc_fence_after();
    uint32_t yq[K];
    tc_drain<K>(tlane + (COLS >= 128 ? TC_N : 0), [&](int i, const uint32_t* acc) { yq[i] = tc_redc(acc, tb.q[i], tb.qpinv[i]); });
    uint32_t* dst = y3 + row * K * N + n;
#pragma unroll
    for (int i = 0; i < K; ++i) dst[(size_t)i * N] = yq[i];
    if (part == 2 && dig != nullptr) {  // uniform over the tile
      // canonical binary of y_2 mod q: sum_i xt_i (q/q_i) - V q as bytes on
      // the tensor cores (exact mod 2^(32 W), the value lies in [0, 2q)),
      // words by one carry pass, then at most one more q off
      uint32_t S[words_for(K)];
      {
        uint32_t xt[K];
        uint64_t Fq = 0;
#pragma unroll
        for (int i = 0; i < K; ++i) {
          xt[i] = mul_shoup(yq[i], tb.qhi[i], tb.qhis[i], tb.q[i]);
          Fq += frac59(xt[i], tb.qg[i], tb.qk[i]);
        }
        tc_put_row<K>(sm.a, tid, xt, (uint32_t)(Fq >> FRAC_BITS));
      }
      fence_proxy_async();
      tc_fence_before();
      __syncthreads();  // every lane has drained the P -> Q sums
      if (tid == 0) {
        tc_fence_after();
        tc_mma64(tbase, sm.a, sm.bdg);
        tc_commit(&sm.bar);
      }
      mbar_wait(&sm.bar, phase);
      phase ^= 1;
      tc_fence_after();
      {
        uint64_t carry = 0;
#pragma unroll
        for (int g = 0; g < (words_for(K) + 3) / 4; ++g) {
          uint32_t v[16];
          tc_ld16(tlane + 16 * g, v);
          tc_wait_ld();
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int w = 4 * g + u;
            if (w < words_for(K)) {
              const uint64_t x = carry + v[4 * u] + ((uint64_t)v[4 * u + 1] << 8) +
                                 ((uint64_t)v[4 * u + 2] << 16) + ((uint64_t)v[4 * u + 3] << 24);
              S[w] = (uint32_t)x;
              carry = x >> 32;
            }
          }
        }
      }
      {
        uint32_t Tq[words_for(K)];
        uint32_t borrow = 0;
#pragma unroll
        for (int w = 0; w < words_for(K); ++w) {
          const uint64_t d = (uint64_t)S[w] - tb.q_w[w] - borrow;
          Tq[w] = (uint32_t)d;
          borrow = (uint32_t)(d >> 63);
        }
        if (!borrow) {
#pragma unroll
          for (int w = 0; w < words_for(K); ++w) S[w] = Tq[w];
        }
      }
      store_digits<K>(S, dig + ct * tb.D * N + n, N, tb);
    }
    tc_fence_before();
    __syncthreads();
  }
  tc_fence_after();
  tc_dealloc<COLS>(tbase, warp);
}

}  // namespace hcnn
