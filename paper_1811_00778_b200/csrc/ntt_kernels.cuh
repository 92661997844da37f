// NTT-based kernels (templated on log2 N); one translation unit per ring
// degree (ntt_inst.cu, compiled with -DHCNN_LOGN=L) keeps the build parallel.
//
//   k_ntt_rows  standalone forward / inverse NTT of RNS rows (ring.py:147-163)
//   k_tensor    ct x ct tensor over Q u P: NTT, pointwise, INTT   (bfv.py:331-347)
//   k_relin     digit NTT x rlk MAC, INTT, + (y0, y1)            (bfv.py:368-404)
#pragma once
#include "common.cuh"
#include "ntt.cuh"

#include <type_traits>

namespace hcnn {

struct NttLaunch {
  cudaStream_t stream;
  dim3 grid;
  NttTabs nt;
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
  int D, reduce_digits;
  // encrypt
  const int8_t *u, *e1, *e2;
  const int64_t* msg;
  const uint32_t* pk;
  const uint2* delta;
};

template <int LOGN>
__global__ void __launch_bounds__(NttGeom<LOGN>::T)
    k_ntt_rows(uint32_t* __restrict__ data, int limbs, int prime_off, int inverse, NttTabs nt) {
  using G = NttGeom<LOGN>;
  extern __shared__ uint32_t s[];
  const int tid = threadIdx.x;
  const int row = blockIdx.x;
  const int j = prime_off + row % limbs;
  uint32_t* r = data + (size_t)row * G::N;
  const uint32_t p = nt.prime[j];
  uint32_t x[G::E];
  if (!inverse) {
#pragma unroll
    for (int e = 0; e < G::E; ++e) x[e] = r[natural_index<LOGN>(tid, e)];
    ntt_fwd<LOGN>(x, s, nt.tw + (size_t)j * G::N, p, tid);
#pragma unroll
    for (int e = 0; e < G::E; ++e) r[spectral_index<LOGN>(tid, e)] = x[e];
  } else {
#pragma unroll
    for (int e = 0; e < G::E; ++e) x[e] = r[spectral_index<LOGN>(tid, e)];
    ntt_inv<LOGN>(x, s, nt.itw + (size_t)j * G::N, p, nt.ninv[j], tid);
#pragma unroll
    for (int e = 0; e < G::E; ++e) r[natural_index<LOGN>(tid, e)] = x[e];
  }
}

template <int LOGN>
DI void load_natural(uint32_t* x, const uint32_t* __restrict__ row, int tid) {
#pragma unroll
  for (int e = 0; e < NttGeom<LOGN>::E; ++e) x[e] = row[natural_index<LOGN>(tid, e)];
}

template <int LOGN>
DI void inv_store(uint32_t* x, uint32_t* s, const uint2* itw, uint32_t p, uint2 ninv, int tid,
                  uint32_t* __restrict__ row) {
  ntt_inv<LOGN>(x, s, itw, p, ninv, tid);
#pragma unroll
  for (int e = 0; e < NttGeom<LOGN>::E; ++e) row[natural_index<LOGN>(tid, e)] = x[e];
}

// One CTA per (ct, prime of Q u P).  a/b: [B][2][K][N]; ae/be: [B][2][KP][N]
// (exact extensions); d: [B][3][K+KP][N] exact tensor parts, coefficient domain.
template <int LOGN>
__global__ void __launch_bounds__(NttGeom<LOGN>::T)
    k_tensor(const uint32_t* __restrict__ a, const uint32_t* __restrict__ a_ext,
             const uint32_t* __restrict__ b, const uint32_t* __restrict__ b_ext,
             uint32_t* __restrict__ d, int K, int KP, int square, NttTabs nt) {
  using G = NttGeom<LOGN>;
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
  load_natural<LOGN>(x0, row_of(a, a_ext, 0), tid);
  ntt_fwd<LOGN>(x0, s, tw, p, tid);
  if (square) {
    load_natural<LOGN>(x1, row_of(a, a_ext, 1), tid);
    ntt_fwd<LOGN>(x1, s, tw, p, tid);
#pragma unroll
    for (int e = 0; e < G::E; ++e) t[e] = mul_mod(x0[e], x0[e], p, mu);
    inv_store<LOGN>(t, s, itw, p, ninv, tid, o0);
#pragma unroll
    for (int e = 0; e < G::E; ++e) {
      const uint32_t c = mul_mod(x0[e], x1[e], p, mu);
      t[e] = add_mod(c, c, p);
    }
    inv_store<LOGN>(t, s, itw, p, ninv, tid, o1);
#pragma unroll
    for (int e = 0; e < G::E; ++e) t[e] = mul_mod(x1[e], x1[e], p, mu);
    inv_store<LOGN>(t, s, itw, p, ninv, tid, o2);
  } else {
    // x0 = A0, x1 = B0 -> d0; then A1 (t), B1 (x1 reused after d1 partial)
    load_natural<LOGN>(x1, row_of(b, b_ext, 0), tid);
    ntt_fwd<LOGN>(x1, s, tw, p, tid);
#pragma unroll
    for (int e = 0; e < G::E; ++e) t[e] = mul_mod(x0[e], x1[e], p, mu);
    inv_store<LOGN>(t, s, itw, p, ninv, tid, o0);
    // A1 into t
    load_natural<LOGN>(t, row_of(a, a_ext, 1), tid);
    ntt_fwd<LOGN>(t, s, tw, p, tid);
    // x1 := A1*B0 (partial d1), keep A0 (x0) and A1 (t)
#pragma unroll
    for (int e = 0; e < G::E; ++e) x1[e] = mul_mod(t[e], x1[e], p, mu);
    uint32_t y1[G::E];
    load_natural<LOGN>(y1, row_of(b, b_ext, 1), tid);
    ntt_fwd<LOGN>(y1, s, tw, p, tid);
#pragma unroll
    for (int e = 0; e < G::E; ++e) {
      x1[e] = add_mod(x1[e], mul_mod(x0[e], y1[e], p, mu), p);  // d1
      t[e] = mul_mod(t[e], y1[e], p, mu);                       // d2
    }
    inv_store<LOGN>(x1, s, itw, p, ninv, tid, o1);
    inv_store<LOGN>(t, s, itw, p, ninv, tid, o2);
  }
}

// One CTA per (ct, prime of q).  dig: [B][D][N] base-w digits of c2;
// y3: [B][3][K][N] scaled parts (0 and 1 used); rlk: [D][2][K][N] in device
// spectral order; out: [B][2][K][N] = (y0 + sum_i D_i k0_i, y1 + sum_i D_i k1_i).
template <int LOGN>
__global__ void __launch_bounds__(NttGeom<LOGN>::T)
    k_relin(const uint32_t* __restrict__ dig, const uint32_t* __restrict__ y3,
            const uint32_t* __restrict__ rlk, uint32_t* __restrict__ out, int K, int D,
            int reduce_digits, NttTabs nt) {
  using G = NttGeom<LOGN>;
  extern __shared__ uint32_t s[];
  const int tid = threadIdx.x;
  const int j = blockIdx.x;
  const size_t ct = blockIdx.y;
  const uint32_t p = nt.prime[j];
  const uint64_t mu = nt.mu[j];
  const uint2* tw = nt.tw + (size_t)j * G::N;
  // 1024-thread CTAs (N >= 2^14) have 64 registers per thread: accumulate
  // reduced u32 there, lazy u64 (one reduction per 15 digits) otherwise.
  constexpr bool kWide = G::T < 1024;
  using Acc = typename std::conditional<kWide, uint64_t, uint32_t>::type;
  Acc acc0[G::E], acc1[G::E];
#pragma unroll
  for (int e = 0; e < G::E; ++e) acc0[e] = acc1[e] = 0;
  for (int i = 0; i < D; ++i) {
    uint32_t x[G::E];
    load_natural<LOGN>(x, dig + (ct * D + i) * G::N, tid);
    if (reduce_digits) {
#pragma unroll
      for (int e = 0; e < G::E; ++e) x[e] = reduce64(x[e], p, mu);
    }
    ntt_fwd<LOGN>(x, s, tw, p, tid);
    const uint32_t* k0 = rlk + ((size_t)(i * 2 + 0) * K + j) * G::N;
    const uint32_t* k1 = rlk + ((size_t)(i * 2 + 1) * K + j) * G::N;
#pragma unroll
    for (int e = 0; e < G::E; ++e) {
      const int idx = spectral_index<LOGN>(tid, e);
      if constexpr (kWide) {
        acc0[e] += (uint64_t)x[e] * __ldg(&k0[idx]);
        acc1[e] += (uint64_t)x[e] * __ldg(&k1[idx]);
      } else {
        acc0[e] = add_mod(acc0[e], mul_mod(x[e], __ldg(&k0[idx]), p, mu), p);
        acc1[e] = add_mod(acc1[e], mul_mod(x[e], __ldg(&k1[idx]), p, mu), p);
      }
    }
    // at most 16 products of (p-1)^2 on top of a reduced value stay < 2^64
    if (kWide && (i & 15) == 14) {
#pragma unroll
      for (int e = 0; e < G::E; ++e) {
        acc0[e] = reduce64(acc0[e], p, mu);
        acc1[e] = reduce64(acc1[e], p, mu);
      }
    }
  }
  const uint2* itw = nt.itw + (size_t)j * G::N;
  const uint2 ninv = nt.ninv[j];
#pragma unroll
  for (int part = 0; part < 2; ++part) {
    uint32_t x[G::E];
#pragma unroll
    for (int e = 0; e < G::E; ++e) x[e] = reduce64(part ? acc1[e] : acc0[e], p, mu);
    ntt_inv<LOGN>(x, s, itw, p, ninv, tid);
    const uint32_t* yr = y3 + ((ct * 3 + part) * K + j) * G::N;
    uint32_t* o = out + ((ct * 2 + part) * K + j) * G::N;
#pragma unroll
    for (int e = 0; e < G::E; ++e) {
      const int idx = natural_index<LOGN>(tid, e);
      o[idx] = add_mod(x[e], yr[idx], p);
    }
  }
}

// Public-key encryption from host-drawn randomness (bfv.py:201-216).  One CTA
// per (ct, prime of q): c0 = INTT(b * NTT(u)) + e1 + Delta m, c1 = INTT(a *
// NTT(u)) + e2.  u: [P][N] in {0,1}; e1, e2: [P][N] small signed; msg: [P][N]
// in [0, t); pk: [2][K][N] device spectral order; delta: [K] (Delta mod q_i,
// Shoup); out: [P][2][K][N].
template <int LOGN>
__global__ void __launch_bounds__(NttGeom<LOGN>::T)
    k_encrypt(const int8_t* __restrict__ u, const int8_t* __restrict__ e1,
              const int8_t* __restrict__ e2, const int64_t* __restrict__ msg,
              const uint32_t* __restrict__ pk, const uint2* __restrict__ delta,
              uint32_t* __restrict__ out, int K, NttTabs nt) {
  using G = NttGeom<LOGN>;
  extern __shared__ uint32_t s[];
  const int tid = threadIdx.x;
  const int j = blockIdx.x;
  const size_t ct = blockIdx.y;
  const uint32_t p = nt.prime[j];
  const uint64_t mu = nt.mu[j];
  uint32_t x[G::E];
#pragma unroll
  for (int e = 0; e < G::E; ++e) x[e] = (uint32_t)u[ct * G::N + natural_index<LOGN>(tid, e)];
  ntt_fwd<LOGN>(x, s, nt.tw + (size_t)j * G::N, p, tid);
  const uint2 dl = delta[j];
#pragma unroll
  for (int part = 0; part < 2; ++part) {
    const uint32_t* key = pk + ((size_t)part * K + j) * G::N;
    uint32_t y[G::E];
#pragma unroll
    for (int e = 0; e < G::E; ++e) y[e] = mul_mod(x[e], __ldg(&key[spectral_index<LOGN>(tid, e)]), p, mu);
    ntt_inv<LOGN>(y, s, nt.itw + (size_t)j * G::N, p, nt.ninv[j], tid);
    const int8_t* er = (part ? e2 : e1) + ct * G::N;
    uint32_t* o = out + ((ct * 2 + part) * K + j) * G::N;
#pragma unroll
    for (int e = 0; e < G::E; ++e) {
      const int idx = natural_index<LOGN>(tid, e);
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

// op: 0 rows, 1 tensor, 2 relin, 3 encrypt
template <int LOGN>
cudaError_t ntt_launch(int op, const NttLaunch& a) {
  using G = NttGeom<LOGN>;
  const size_t smem = G::SMEM_WORDS * sizeof(uint32_t);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_ntt_rows<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_tensor<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_relin<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_encrypt<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  switch (op) {
    case 0:
      k_ntt_rows<LOGN><<<a.grid, G::T, smem, a.stream>>>(a.rows, a.limbs, a.prime_off, a.inverse, a.nt);
      break;
    case 1:
      k_tensor<LOGN><<<a.grid, G::T, smem, a.stream>>>(a.a, a.ae, a.b, a.be, a.d, a.K, a.KP, a.square, a.nt);
      break;
    case 2:
      k_relin<LOGN><<<a.grid, G::T, smem, a.stream>>>(a.dig, a.y3, a.rlk, a.out, a.K, a.D, a.reduce_digits, a.nt);
      break;
    case 3:
      k_encrypt<LOGN><<<a.grid, G::T, smem, a.stream>>>(a.u, a.e1, a.e2, a.msg, a.pk, a.delta, a.out, a.K, a.nt);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace hcnn

#define HCNN_LOGN_LIST(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15)
#define HCNN_DECLARE_LAUNCH(L) cudaError_t hcnn_ntt_launch_##L(int op, const hcnn::NttLaunch& a);
HCNN_LOGN_LIST(HCNN_DECLARE_LAUNCH)
