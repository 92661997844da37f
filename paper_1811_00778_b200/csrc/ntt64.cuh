// 64-bit modular negacyclic NTT (moduli below 2^62; ring.py:45-46 admits
// primes to 62 bits, ntt.py:113-154 transforms them) for the plaintext side:
// SIMD slot encoding / decoding over Z_t (batching.py:41-95) where t is the
// 43-bit MNIST modulus (presets.py:25), and the u64 rows of the kernel
// microbench (hcnn_ntt64).
//
// Same convention as the u32 path: Cooley-Tukey forward with the psi^brv
// twiddles folded in (natural in, bit-reversed out), Gentleman-Sande inverse
// with N^-1 folded into its last stage.  Layout: the row sits in padded
// shared memory (one pad word per 16) of one CTA, or of a 2-CTA cluster at
// N = 2^15 (2^15 u64 do not fit one CTA); passes of up to 4 butterfly bits
// run in registers, 16 residues per thread, Harvey lazy butterflies with
// Shoup twiddle pairs (w, floor(w 2^64 / p)) read through L1.  At 2^15 the
// top bit is one butterfly stage across the pair through distributed shared
// memory; everything below it is local to each CTA.
#pragma once
#include <cooperative_groups.h>

#include <cstdint>

#include "modarith.cuh"

namespace hcnn {

DI uint64_t mul_shoup64_lazy(uint64_t x, uint64_t w, uint64_t ws, uint64_t p) {
  const uint64_t q = __umul64hi(x, ws);
  return x * w - q * p;  // in [0, 2p) for x < 2^64, w < p
}

DI uint64_t csub64(uint64_t x, uint64_t p) { return x >= p ? x - p : x; }

template <int LOGN_>
struct N64Geom {
  static constexpr int LOGN = LOGN_;
  static constexpr int CL = LOGN >= 15 ? 2 : 1;  // CTAs per row
  static constexpr int LOGNL = LOGN - (CL == 2 ? 1 : 0);
  static constexpr int NL = 1 << LOGNL;          // residues per CTA
  static constexpr int T = NL >= 512 ? NL / 16 : 32;
  static constexpr int NP = (LOGNL + 3) / 4;     // register passes
  // width of pass P (from the top bits): spread evenly, wider ones first
  __host__ __device__ static constexpr int kb(int P) { return LOGNL / NP + (P < LOGNL % NP ? 1 : 0); }
  __host__ __device__ static constexpr int lo(int P) { return P < 0 ? LOGNL : lo(P - 1) - kb(P); }
  static constexpr int SMEM_BYTES = (NL + NL / 16 + 16) * 8;
  // resident CTAs per SM asked of the register allocator (two up to 2^13:
  // one row's load / store overlaps the other's butterflies)
  static constexpr int MINB = NL <= 8192 ? 2 : 1;
};

DI int sp64(int i) { return i + (i >> 4); }  // padded slot

// One register pass over local bits [LO, LO+KB): every group of 2^KB
// residues that differ only in those bits, 16 / 2^KB groups per thread.
// gbase: global index of this CTA's first residue (twiddle indices are global).
template <class GM, int P, bool INV>
DI void pass64(uint64_t* s, uint32_t gbase, const ulonglong2* __restrict__ tw, uint64_t p, int tid,
               ulonglong2 nsc, ulonglong2 nwsc) {
  constexpr int KB = GM::kb(P), LO = GM::lo(P), E = 1 << KB;
  constexpr int GROUPS = GM::NL >> KB;
  const uint64_t p2 = 2 * p;
#pragma unroll
  for (int k = 0; k < 16 / E; ++k) {
    const int g = tid + k * GM::T;
    if (g >= GROUPS) break;
    const int base = ((g >> LO) << (LO + KB)) | (g & ((1 << LO) - 1));
    uint64_t v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = s[sp64(base + (e << LO))];
    const uint32_t jg = gbase + (uint32_t)base;
#pragma unroll
    for (int t = 0; t < KB; ++t) {
      const int ss = INV ? KB - 1 - t : t;  // inverse: bits ascending
      const int bit = LO + KB - 1 - ss;
      const int sg = GM::LOGN - 1 - bit;     // global stage
      const int half = 1 << (KB - 1 - ss);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if (e & half) continue;
        const uint32_t j = jg | ((uint32_t)e << LO);
        const ulonglong2 w = __ldg(&tw[(1u << sg) + (j >> (bit + 1))]);
        uint64_t& a = v[e];
        uint64_t& b = v[e | half];
        if (!INV) {
          const uint64_t X = csub64(a, p2);
          const uint64_t Tt = mul_shoup64_lazy(b, w.x, w.y, p);
          a = X + Tt;
          b = X - Tt + p2;
        } else if (sg == 0) {  // last inverse stage: N^-1 folded in, fully reduced
          const uint64_t X = a, Y = b;
          a = csub64(mul_shoup64_lazy(X + Y, nsc.x, nsc.y, p), p);
          b = csub64(mul_shoup64_lazy(X - Y + p2, nwsc.x, nwsc.y, p), p);
        } else {
          const uint64_t X = a, Y = b;
          a = csub64(X + Y, p2);
          b = mul_shoup64_lazy(X - Y + p2, w.x, w.y, p);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) s[sp64(base + (e << LO))] = v[e];
  }
  __syncthreads();
}

template <class GM, int P, bool INV>
DI void passes64(uint64_t* s, uint32_t gbase, const ulonglong2* tw, uint64_t p, int tid, ulonglong2 nsc,
                 ulonglong2 nwsc) {
  if constexpr (P >= 0 && P < GM::NP) {
    if constexpr (!INV) {
      pass64<GM, P, false>(s, gbase, tw, p, tid, nsc, nwsc);
      passes64<GM, P + 1, false>(s, gbase, tw, p, tid, nsc, nwsc);
    } else {
      pass64<GM, P, true>(s, gbase, tw, p, tid, nsc, nwsc);
      passes64<GM, P - 1, true>(s, gbase, tw, p, tid, nsc, nwsc);
    }
  }
}

// The top butterfly bit of a 2^15 row across the CTA pair (DSMEM): pairs
// (j, j + N/2), j < N/2, residue j in CTA 0 and j + N/2 in CTA 1 at the same
// local slot; each CTA does half of them.  Inverse: N^-1 folded in.
template <class GM, bool INV>
DI void cross_stage64(uint64_t* s, const ulonglong2* __restrict__ tw, uint64_t p, int tid, ulonglong2 nsc,
                      ulonglong2 nwsc) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned r = cl.block_rank();
  uint64_t* s0 = cl.map_shared_rank(s, 0);
  uint64_t* s1 = cl.map_shared_rank(s, 1);
  const uint64_t p2 = 2 * p;
  const ulonglong2 w = __ldg(&tw[1]);
  cl.sync();
  for (int j = (int)r * (GM::NL / 2) + tid; j < ((int)r + 1) * (GM::NL / 2); j += GM::T) {
    const int sj = sp64(j);
    const uint64_t X = s0[sj], Y = s1[sj];
    if (!INV) {
      const uint64_t Xr = csub64(X, p2);
      const uint64_t Tt = mul_shoup64_lazy(Y, w.x, w.y, p);
      s0[sj] = Xr + Tt;
      s1[sj] = Xr - Tt + p2;
    } else {
      s0[sj] = csub64(mul_shoup64_lazy(X + Y, nsc.x, nsc.y, p), p);
      s1[sj] = csub64(mul_shoup64_lazy(X - Y + p2, nwsc.x, nwsc.y, p), p);
    }
  }
  cl.sync();
}

// rows [n_rows][N] u64 in place (values < p in; forward out in bit-reversed
// positions, inverse out natural, both fully reduced).  nsc = N^-1 and
// nwsc = psi^-N/2 N^-1 (Shoup pairs); tw / itw: psi^brv / psi^-brv pairs.
template <int LOGN, bool INV>
__global__ void __launch_bounds__(N64Geom<LOGN>::T, N64Geom<LOGN>::MINB) k_ntt64(uint64_t* __restrict__ rows, uint64_t p,
                                                            const ulonglong2* __restrict__ tw, ulonglong2 nsc,
                                                            ulonglong2 nwsc) {
  using GM = N64Geom<LOGN>;
  static_assert(GM::CL == 1, "one CTA per row");
  extern __shared__ uint64_t s64[];
  const int tid = threadIdx.x;
  uint64_t* r = rows + (size_t)blockIdx.x * GM::NL;
#pragma unroll
  for (int i = tid; i < GM::NL; i += GM::T) s64[sp64(i)] = r[i];
  __syncthreads();
  passes64<GM, INV ? GM::NP - 1 : 0, INV>(s64, 0, tw, p, tid, nsc, nwsc);
  const uint64_t p2 = 2 * p;
#pragma unroll
  for (int i = tid; i < GM::NL; i += GM::T) r[i] = INV ? s64[sp64(i)] : csub64(csub64(s64[sp64(i)], p2), p);
}

// N = 2^15: one 2-CTA cluster per row (CTA r holds residues [r N/2, (r+1) N/2))
template <bool INV>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(N64Geom<15>::T)
    k_ntt64_cl(uint64_t* __restrict__ rows, uint64_t p, const ulonglong2* __restrict__ tw, ulonglong2 nsc,
               ulonglong2 nwsc) {
  using GM = N64Geom<15>;
  extern __shared__ uint64_t s64[];
  const int tid = threadIdx.x;
  const unsigned r = blockIdx.x & 1;
  uint64_t* row = rows + (size_t)(blockIdx.x >> 1) * (2 * GM::NL) + r * GM::NL;
#pragma unroll
  for (int i = tid; i < GM::NL; i += GM::T) s64[sp64(i)] = row[i];
  if (!INV) {
    cross_stage64<GM, false>(s64, tw, p, tid, nsc, nwsc);
    passes64<GM, 0, false>(s64, r * GM::NL, tw, p, tid, nsc, nwsc);
  } else {
    __syncthreads();
    passes64<GM, GM::NP - 1, true>(s64, r * GM::NL, tw, p, tid, nsc, nwsc);
    cross_stage64<GM, true>(s64, tw, p, tid, nsc, nwsc);
  }
  const uint64_t p2 = 2 * p;
#pragma unroll
  for (int i = tid; i < GM::NL; i += GM::T) row[i] = INV ? s64[sp64(i)] : csub64(csub64(s64[sp64(i)], p2), p);
}

// natural-order slot vector <-> device (bit-reversed) spectral order
__global__ void k_permute_brv64(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst,
                                int logn) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = 1 << logn;
  if (i >= n) return;
  const size_t row = blockIdx.y;
  dst[row * n + i] = src[row * n + (int)(__brev((unsigned)i) >> (32 - logn))];
}

// host dispatch over the ring degree (1 <= logn <= 15)
template <bool INV>
inline cudaError_t launch_ntt64(uint64_t* rows, size_t n_rows, int logn, uint64_t p, const ulonglong2* tw,
                                ulonglong2 nsc, ulonglong2 nwsc, cudaStream_t st) {
  if (!n_rows) return cudaSuccess;
  switch (logn) {
#define X(L)                                                                                              \
  case L: {                                                                                               \
    using GM = N64Geom<L>;                                                                                \
    if constexpr (GM::CL == 1) {                                                                          \
      cudaFuncSetAttribute(k_ntt64<L, INV>, cudaFuncAttributeMaxDynamicSharedMemorySize, GM::SMEM_BYTES); \
      k_ntt64<L, INV><<<(unsigned)n_rows, GM::T, GM::SMEM_BYTES, st>>>(rows, p, tw, nsc, nwsc);           \
    } else {                                                                                              \
      cudaFuncSetAttribute(k_ntt64_cl<INV>, cudaFuncAttributeMaxDynamicSharedMemorySize, GM::SMEM_BYTES); \
      k_ntt64_cl<INV><<<(unsigned)(2 * n_rows), GM::T, GM::SMEM_BYTES, st>>>(rows, p, tw, nsc, nwsc);     \
    }                                                                                                     \
    break;                                                                                                \
  }
    X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15)
#undef X
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace hcnn
