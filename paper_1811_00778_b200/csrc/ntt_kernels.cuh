// NTT-based kernels, templated on the NTT geometry G = NttGeom<LOGN, LOGE>
// (ntt.cuh); one translation unit per ring degree (ntt_inst.cu, compiled with
// -DHCNN_LOGN=L) keeps the build parallel.
//
//   k_ntt_rows      standalone forward / inverse NTT of RNS rows (ring.py:147-163)
//   k_tensor        ct x ct tensor over Q u P: NTT, pointwise, INTT (bfv.py:331-347)
//   k_relin         digit NTT x rlk MAC, INTT, + (y0, y1)          (bfv.py:368-404)
//   k_encrypt       public-key encryption from host randomness     (bfv.py:201-216)
//   k_ref_to_tiled  reference-order NTT keys -> device tiled layout
#pragma once
#include <type_traits>

#include "common.cuh"
#include "ntt.cuh"
#include "tma.cuh"

namespace hcnn {

struct NttLaunch {
  cudaStream_t stream;
  dim3 grid;
  NttTabs nt;
  int variant;  // radix of the fused kernels: 0 = default, 4 or 5 = log2 E
  // rows
  uint32_t* rows;
  int limbs, prime_off, inverse;
  // tensor
  const uint32_t *a, *ae, *b, *be;
  uint32_t* d;
  int K, KP, square;
  // relin
  const uint32_t *dig, *y3, *rlk;
  uint32_t* out;
  int D, reduce_digits, rlk_mont;
  // encrypt
  const int8_t *u, *e1, *e2;
  const int64_t* msg;
  const uint32_t* pk;
  const uint2* delta;
};

// Montgomery product x * k' * 2^-32 mod p in [0, 2p) for x, k' < p < 2^30;
// pinv = -p^-1 mod 2^32.  With k' = k 2^32 mod p this is x * k mod p.
DI uint32_t mont_mul(uint32_t x, uint32_t kp, uint32_t p, uint32_t pinv) {
  const uint64_t z = (uint64_t)x * kp;
  const uint32_t m = (uint32_t)z * pinv;
  return (uint32_t)((z + (uint64_t)m * p) >> 32);
}

template <class G>
DI void load_natural(uint32_t* x, const uint32_t* __restrict__ row, int tid) {
#pragma unroll
  for (int e = 0; e < G::E; ++e) x[e] = row[natural_index<G>(tid, e)];
}

template <class G>
DI void inv_store(uint32_t* x, uint32_t* s, const uint2* itw, uint32_t p, uint2 ninv, int tid,
                  uint32_t* __restrict__ row) {
  ntt_inv<G>(x, s, itw, p, ninv, tid);
#pragma unroll
  for (int e = 0; e < G::E; ++e) row[natural_index<G>(tid, e)] = x[e];
}

// in place on [rows][N]; row r uses prime prime_off + r % limbs.
// inverse: 0 forward (spectral positions), 1 inverse, 2 forward to tiled layout
template <class G>
__global__ void __launch_bounds__(G::T, (G::T <= 256 ? 2 : 1))
    k_ntt_rows(uint32_t* __restrict__ data, int limbs, int prime_off, int inverse, NttTabs nt) {
  extern __shared__ uint32_t s[];
  const int tid = threadIdx.x;
  const int row = blockIdx.x;
  const int j = prime_off + row % limbs;
  uint32_t* r = data + (size_t)row * G::N;
  const uint32_t p = nt.prime[j];
  uint32_t x[G::E];
  if (inverse == 1) {
#pragma unroll
    for (int e = 0; e < G::E; ++e) x[e] = r[spectral_index<G>(tid, e)];
    ntt_inv<G>(x, s, nt.itw + (size_t)j * G::N, p, nt.ninv[j], tid);
#pragma unroll
    for (int e = 0; e < G::E; ++e) r[natural_index<G>(tid, e)] = x[e];
    return;
  }
  load_natural<G>(x, r, tid);
  ntt_fwd<G>(x, s, nt.tw + (size_t)j * G::N, p, tid);
  if (inverse == 2) {
    __syncthreads();
    store_tiled<G>(x, r, tid);
  } else {
#pragma unroll
    for (int e = 0; e < G::E; ++e) r[spectral_index<G>(tid, e)] = x[e];
  }
}

// One CTA per (ct, prime of Q u P).  a/b: [B][2][K][N]; ae/be: [B][2][KP][N]
// (exact extensions); d: [B][3][K+KP][N] exact tensor parts, coefficient domain.
template <class G>
__global__ void __launch_bounds__(G::T, (G::T <= 256 ? 2 : 1))
    k_tensor(const uint32_t* __restrict__ a, const uint32_t* __restrict__ a_ext,
             const uint32_t* __restrict__ b, const uint32_t* __restrict__ b_ext,
             uint32_t* __restrict__ d, int K, int KP, int square, NttTabs nt) {
  extern __shared__ uint32_t s[];
  const int tid = threadIdx.x;
  const int j = blockIdx.x;
  const size_t ct = blockIdx.y;
  const int L = K + KP;
  const uint32_t p = nt.prime[j];
  const uint64_t mu = nt.mu[j];
  const uint2* tw = nt.tw + (size_t)j * G::N;
  const uint2* itw = nt.itw + (size_t)j * G::N;
  const uint2 ninv = nt.ninv[j];
  auto row_of = [&](const uint32_t* base, const uint32_t* ext, int part) -> const uint32_t* {
    return j < K ? base + ((ct * 2 + part) * K + j) * G::N
                 : ext + ((ct * 2 + part) * KP + (j - K)) * G::N;
  };
  uint32_t* o0 = d + ((ct * 3 + 0) * L + j) * G::N;
  uint32_t* o1 = d + ((ct * 3 + 1) * L + j) * G::N;
  uint32_t* o2 = d + ((ct * 3 + 2) * L + j) * G::N;
  uint32_t x0[G::E], x1[G::E], t[G::E];
  load_natural<G>(x0, row_of(a, a_ext, 0), tid);
  ntt_fwd<G>(x0, s, tw, p, tid);
  if (square) {
    load_natural<G>(x1, row_of(a, a_ext, 1), tid);
    ntt_fwd<G>(x1, s, tw, p, tid);
#pragma unroll
    for (int e = 0; e < G::E; ++e) t[e] = mul_mod(x0[e], x0[e], p, mu);
    inv_store<G>(t, s, itw, p, ninv, tid, o0);
#pragma unroll
    for (int e = 0; e < G::E; ++e) {
      const uint32_t c = mul_mod(x0[e], x1[e], p, mu);
      t[e] = add_mod(c, c, p);
    }
    inv_store<G>(t, s, itw, p, ninv, tid, o1);
#pragma unroll
    for (int e = 0; e < G::E; ++e) t[e] = mul_mod(x1[e], x1[e], p, mu);
    inv_store<G>(t, s, itw, p, ninv, tid, o2);
  } else {
    // x0 = A0, x1 = B0 -> d0; then A1 into t; x1 := A1 B0 (part of d1)
    load_natural<G>(x1, row_of(b, b_ext, 0), tid);
    ntt_fwd<G>(x1, s, tw, p, tid);
#pragma unroll
    for (int e = 0; e < G::E; ++e) t[e] = mul_mod(x0[e], x1[e], p, mu);
    inv_store<G>(t, s, itw, p, ninv, tid, o0);
    load_natural<G>(t, row_of(a, a_ext, 1), tid);
    ntt_fwd<G>(t, s, tw, p, tid);
#pragma unroll
    for (int e = 0; e < G::E; ++e) x1[e] = mul_mod(t[e], x1[e], p, mu);
    uint32_t y1[G::E];
    load_natural<G>(y1, row_of(b, b_ext, 1), tid);
    ntt_fwd<G>(y1, s, tw, p, tid);
#pragma unroll
    for (int e = 0; e < G::E; ++e) {
      x1[e] = add_mod(x1[e], mul_mod(x0[e], y1[e], p, mu), p);  // d1
      t[e] = mul_mod(t[e], y1[e], p, mu);                       // d2
    }
    inv_store<G>(x1, s, itw, p, ninv, tid, o1);
    inv_store<G>(t, s, itw, p, ninv, tid, o2);
  }
}

// Shared-memory plan of k_relin: STAGES buffers, each holding one digit row
// (padded, doubling as the NTT exchange buffer once its residues are in
// registers) and the two rlk rows of that digit, streamed in by TMA bulk
// copies one digit ahead of the compute.
template <class G>
struct RelinSmem {
  // [two NTT exchange buffers][STAGES digit rows streamed by TMA][mbarriers]
  static constexpr int STAGE_WORDS = G::N;
  static constexpr int LIMIT = 220 * 1024;
  static constexpr int BASE = G::NTT_SMEM_WORDS;
  static constexpr int STAGES = (BASE + 2 * G::N) * 4 <= LIMIT ? 2 : ((BASE + G::N) * 4 <= LIMIT ? 1 : 0);
  static constexpr int BYTES = (BASE + STAGES * G::N) * 4 + 16 * 2;
};

// One CTA per (ct, prime of q).  dig: [B][D][N] base-w digits of c2;
// y3: [B][3][K][N] scaled parts (0 and 1 used); rlk: [D][2][K][N] NTT domain,
// tiled layout (ntt.cuh), Montgomery form unless ACC64;
// out: [B][2][K][N] = (y0 + sum_i D_i k0_i, y1 + sum_i D_i k1_i).
// ACC64: lazy 64-bit accumulators (one reduction per 15 digits); otherwise
// u32 accumulators in [0, 2p) fed by Montgomery products (half the registers).
template <class G, bool ACC64>
__global__ void __launch_bounds__(G::T, (G::T <= 256 ? 2 : 1))
    k_relin(const uint32_t* __restrict__ dig, const uint32_t* __restrict__ y3,
            const uint32_t* __restrict__ rlk, uint32_t* __restrict__ out, int K, int D,
            int reduce_digits, NttTabs nt) {
  using SM = RelinSmem<G>;
  extern __shared__ __align__(16) uint32_t s[];
  const int tid = threadIdx.x;
  const int j = blockIdx.x;
  const size_t ct = blockIdx.y;
  const uint32_t p = nt.prime[j];
  const uint64_t mu = nt.mu[j];
  const uint32_t pinv = nt.pinv[j];
  const uint32_t p2 = 2 * p;
  const uint2* tw = nt.tw + (size_t)j * G::N;
  using Acc = typename std::conditional<ACC64, uint64_t, uint32_t>::type;
  Acc acc0[G::E], acc1[G::E];
#pragma unroll
  for (int e = 0; e < G::E; ++e) acc0[e] = acc1[e] = 0;

  const uint32_t* dig_ct = dig + ct * D * G::N;
  auto krow = [&](int i, int part) { return rlk + ((size_t)(i * 2 + part) * K + j) * G::N; };
  uint32_t* stage0 = s + SM::BASE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stage0 + SM::STAGES * G::N);
  auto issue = [&](int i) {  // elected thread: digit row i into its stage
    uint64_t* bar = &bars[i % SM::STAGES];
    fence_proxy_async();
    mbar_expect_tx(bar, G::N * 4);
    bulk_g2s(stage0 + (i % SM::STAGES) * G::N, dig_ct + (size_t)i * G::N, G::N * 4, bar);
  };
  if constexpr (SM::STAGES > 0) {
    if (tid == 0) {
      for (int st = 0; st < SM::STAGES; ++st) mbar_init(&bars[st], 1);
      fence_mbar_init();
      issue(0);
    }
    __syncthreads();
  }

  for (int i = 0; i < D; ++i) {
    uint32_t x[G::E];
    if constexpr (SM::STAGES > 0) {
      // with two stages, digit i+1 streams in while digit i is transformed;
      // its buffer was last read before this thread's previous-digit barriers
      if constexpr (SM::STAGES == 2) {
        if (tid == 0 && i + 1 < D) issue(i + 1);
      }
      const uint32_t* row = stage0 + (i % SM::STAGES) * G::N;
      mbar_wait(&bars[i % SM::STAGES], (uint32_t)(i / SM::STAGES) & 1);
#pragma unroll
      for (int e = 0; e < G::E; ++e) x[e] = row[natural_index<G>(tid, e)];
      if constexpr (SM::STAGES == 1) {
        __syncthreads();
        if (tid == 0 && i + 1 < D) issue(i + 1);
      }
    } else {
      load_natural<G>(x, dig_ct + (size_t)i * G::N, tid);
    }
    if (reduce_digits) {
#pragma unroll
      for (int e = 0; e < G::E; ++e) x[e] = reduce64(x[e], p, mu);
    }
    ntt_fwd<G>(x, s, tw, p, tid);
#pragma unroll
    for (int part = 0; part < 2; ++part) {
      Acc* acc = part ? acc1 : acc0;
      uint32_t k[G::E];
      load_tiled<G>(k, krow(i, part), tid);
#pragma unroll
      for (int e = 0; e < G::E; ++e) {
        if constexpr (ACC64) {
          acc[e] += (uint64_t)x[e] * k[e];
        } else {
          const uint32_t v = acc[e] + mont_mul(x[e], k[e], p, pinv);
          acc[e] = umin32(v, v - p2);
        }
      }
    }
    if constexpr (ACC64) {
      // at most 16 products of (p-1)^2 on top of a reduced value stay < 2^64
      if ((i & 15) == 14) {
#pragma unroll
        for (int e = 0; e < G::E; ++e) {
          acc0[e] = reduce64(acc0[e], p, mu);
          acc1[e] = reduce64(acc1[e], p, mu);
        }
      }
    }
  }
  const uint2* itw = nt.itw + (size_t)j * G::N;
  const uint2 ninv = nt.ninv[j];
#pragma unroll
  for (int part = 0; part < 2; ++part) {
    uint32_t x[G::E];
#pragma unroll
    for (int e = 0; e < G::E; ++e) {
      if constexpr (ACC64) x[e] = reduce64(part ? acc1[e] : acc0[e], p, mu);
      else x[e] = part ? acc1[e] : acc0[e];  // in [0, 2p): valid inverse input
    }
    ntt_inv<G>(x, s, itw, p, ninv, tid);
    const uint32_t* yr = y3 + ((ct * 3 + part) * K + j) * G::N;
    uint32_t* o = out + ((ct * 2 + part) * K + j) * G::N;
#pragma unroll
    for (int e = 0; e < G::E; ++e) {
      const int idx = natural_index<G>(tid, e);
      o[idx] = add_mod(x[e], yr[idx], p);
    }
  }
}

// Public-key encryption from host-drawn randomness (bfv.py:201-216).  One CTA
// per (ct, prime of q): c0 = INTT(b * NTT(u)) + e1 + Delta m, c1 = INTT(a *
// NTT(u)) + e2.  u: [P][N] in {0,1}; e1, e2: [P][N] small signed; msg: [P][N]
// in [0, t); pk: [2][K][N] NTT domain, tiled layout; delta: [K] (Delta mod q_i,
// Shoup); out: [P][2][K][N].
template <class G>
__global__ void __launch_bounds__(G::T, (G::T <= 256 ? 2 : 1))
    k_encrypt(const int8_t* __restrict__ u, const int8_t* __restrict__ e1,
              const int8_t* __restrict__ e2, const int64_t* __restrict__ msg,
              const uint32_t* __restrict__ pk, const uint2* __restrict__ delta,
              uint32_t* __restrict__ out, int K, NttTabs nt) {
  extern __shared__ uint32_t s[];
  const int tid = threadIdx.x;
  const int j = blockIdx.x;
  const size_t ct = blockIdx.y;
  const uint32_t p = nt.prime[j];
  const uint64_t mu = nt.mu[j];
  uint32_t x[G::E];
#pragma unroll
  for (int e = 0; e < G::E; ++e) x[e] = (uint32_t)u[ct * G::N + natural_index<G>(tid, e)];
  ntt_fwd<G>(x, s, nt.tw + (size_t)j * G::N, p, tid);
  const uint2 dl = delta[j];
#pragma unroll
  for (int part = 0; part < 2; ++part) {
    uint32_t y[G::E];
    load_tiled<G>(y, pk + ((size_t)part * K + j) * G::N, tid);
#pragma unroll
    for (int e = 0; e < G::E; ++e) y[e] = mul_mod(x[e], y[e], p, mu);
    ntt_inv<G>(y, s, nt.itw + (size_t)j * G::N, p, nt.ninv[j], tid);
    const int8_t* er = (part ? e2 : e1) + ct * G::N;
    uint32_t* o = out + ((ct * 2 + part) * K + j) * G::N;
#pragma unroll
    for (int e = 0; e < G::E; ++e) {
      const int idx = natural_index<G>(tid, e);
      const int ev = er[idx];
      uint32_t v = add_mod(y[e], ev < 0 ? p - (uint32_t)(-ev) : (uint32_t)ev, p);
      if (part == 0) {
        const uint32_t m = reduce64((uint64_t)msg[ct * G::N + idx], p, mu);
        v = add_mod(v, mul_shoup(m, dl.x, dl.y, p), p);
      }
      o[idx] = v;
    }
  }
}

// reference-order NTT rows (natural order, ref[k] = a(psi^(2k+1))) -> tiled
// device layout: dst[tid*E + e] = src[brv(spectral_index(tid, e))], times
// 2^32 mod p (Montgomery form) when mont; row r uses prime r % limbs.
template <class G>
__global__ void k_ref_to_tiled(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                               int limbs, int mont, NttTabs nt) {
  const int tid = threadIdx.x;
  const size_t row = blockIdx.x;
  const int j = (int)(row % limbs);
  const uint32_t p = nt.prime[j];
  const uint32_t r32 = (uint32_t)((1ull << 32) % p);
#pragma unroll
  for (int e = 0; e < G::E; ++e) {
    const int i = spectral_index<G>(tid, e);
    const int r = (int)(__brev((unsigned)i) >> (32 - G::LOGN));
    uint32_t v = src[row * G::N + r];
    if (mont) v = mul_mod(v, r32, p, nt.mu[j]);
    dst[row * G::N + tiled_index<G>(tid, e)] = v;
  }
}

// tiled key rows (plain) -> Montgomery form in place
template <class G>
__global__ void k_to_mont(uint32_t* __restrict__ rows, int limbs, NttTabs nt) {
  const int tid = threadIdx.x;
  const size_t row = blockIdx.x;
  const int j = (int)(row % limbs);
  const uint32_t p = nt.prime[j];
  const uint32_t r32 = (uint32_t)((1ull << 32) % p);
#pragma unroll
  for (int e = 0; e < G::E; ++e) {
    uint32_t* v = rows + row * G::N + tiled_index<G>(tid, e);
    *v = mul_mod(*v, r32, p, nt.mu[j]);
  }
}

template <class G>
void configure_smem() {
  const int smem = G::NTT_SMEM_WORDS * sizeof(uint32_t);
  cudaFuncSetAttribute(k_ntt_rows<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_tensor<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_relin<G, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, RelinSmem<G>::BYTES);
  cudaFuncSetAttribute(k_relin<G, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, RelinSmem<G>::BYTES);
  cudaFuncSetAttribute(k_encrypt<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

// relin accumulators: u64 when the registers allow (<= 16 per thread and at
// most 512 threads), Montgomery u32 otherwise (rlk uploaded in that form)
template <class G>
constexpr bool relin_acc64() { return G::E <= 16 && G::T <= 512; }

template <class G>
cudaError_t launch_with(int op, const NttLaunch& a) {
  static bool configured = false;
  if (!configured) {
    configure_smem<G>();
    configured = true;
  }
  const size_t smem = G::NTT_SMEM_WORDS * sizeof(uint32_t);
  switch (op) {
    case 0:
      k_ntt_rows<G><<<a.grid, G::T, smem, a.stream>>>(a.rows, a.limbs, a.prime_off, a.inverse, a.nt);
      break;
    case 1:
      k_tensor<G><<<a.grid, G::T, smem, a.stream>>>(a.a, a.ae, a.b, a.be, a.d, a.K, a.KP, a.square, a.nt);
      break;
    case 2:
      if (a.rlk_mont != (relin_acc64<G>() ? 0 : 1)) return cudaErrorInvalidValue;
      if constexpr (relin_acc64<G>())
        k_relin<G, true><<<a.grid, G::T, RelinSmem<G>::BYTES, a.stream>>>(a.dig, a.y3, a.rlk, a.out, a.K, a.D, a.reduce_digits, a.nt);
      else
        k_relin<G, false><<<a.grid, G::T, RelinSmem<G>::BYTES, a.stream>>>(a.dig, a.y3, a.rlk, a.out, a.K, a.D, a.reduce_digits, a.nt);
      break;
    case 3:
      k_encrypt<G><<<a.grid, G::T, smem, a.stream>>>(a.u, a.e1, a.e2, a.msg, a.pk, a.delta, a.out, a.K, a.nt);
      break;
    case 4:
      k_ref_to_tiled<G><<<a.grid, G::T, 0, a.stream>>>(a.a, a.out, a.limbs, a.rlk_mont, a.nt);
      break;
    case 5:
      k_to_mont<G><<<a.grid, G::T, 0, a.stream>>>(a.rows, a.limbs, a.nt);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// variant: log2 E of the fused kernels (0 = default geometry); the key layout
// (tiled, Montgomery) follows the geometry, so keys are uploaded per variant.
template <int LOGN>
cudaError_t ntt_launch(int op, const NttLaunch& a) {
  if constexpr (LOGN >= 10 && LOGN <= 13 && pick_loge(LOGN) != 3) {
    if (a.variant == 3) return launch_with<NttGeom<LOGN, 3>>(op, a);
  }
  if constexpr (LOGN >= 10 && pick_loge(LOGN) != 5) {
    if (a.variant == 5) return launch_with<NttGeom<LOGN, 5>>(op, a);
  }
  if constexpr (LOGN >= 10 && pick_loge(LOGN) != 4) {
    if (a.variant == 4) return launch_with<NttGeom<LOGN, 4>>(op, a);
  }
  return launch_with<NttGeom<LOGN>>(op, a);
}

// does variant v use Montgomery-form rlk?
template <int LOGN>
int ntt_variant_mont(int v) {
  if constexpr (LOGN >= 10 && LOGN <= 13) {
    if (v == 3) return relin_acc64<NttGeom<LOGN, 3>>() ? 0 : 1;
  }
  if constexpr (LOGN >= 10) {
    if (v == 5) return relin_acc64<NttGeom<LOGN, 5>>() ? 0 : 1;
    if (v == 4) return relin_acc64<NttGeom<LOGN, 4>>() ? 0 : 1;
  }
  return relin_acc64<NttGeom<LOGN>>() ? 0 : 1;
}

}  // namespace hcnn

#define HCNN_LOGN_LIST(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15)
#define HCNN_DECLARE_LAUNCH(L)                                       \
  cudaError_t hcnn_ntt_launch_##L(int op, const hcnn::NttLaunch& a); \
  int hcnn_ntt_mont_##L(int variant);
HCNN_LOGN_LIST(HCNN_DECLARE_LAUNCH)
