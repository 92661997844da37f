// 64-bit modular negacyclic NTT (moduli below 2^62) for the plaintext side:
// SIMD slot encoding / decoding over Z_t (batching.py:41-95) where t is the
// 43-bit MNIST modulus (presets.py:25), and any wide-prime microbench.
//
// Same convention as the u32 path: Cooley-Tukey forward with the psi^brv
// twiddles folded in (natural in, bit-reversed out), Gentleman-Sande inverse
// with N^-1; twiddles are Shoup pairs (w, floor(w 2^64 / p)) staged in shared
// memory, residues live in shared memory, one CTA per row.
#pragma once
#include <cstdint>

#include "modarith.cuh"

namespace hcnn {

DI uint64_t mul_shoup64_lazy(uint64_t x, uint64_t w, uint64_t ws, uint64_t p) {
  const uint64_t q = __umul64hi(x, ws);
  return x * w - q * p;  // in [0, 2p) for x < 2^64, w < p
}

DI uint64_t csub64(uint64_t x, uint64_t p) { return x >= p ? x - p : x; }

// rows [n_rows][N] u64 in place; tw/itw: [N] (w, w') pairs as ulonglong2 in
// psi^brv order (read through L1); smem: N u64
template <bool INVERSE>
__global__ void k_ntt64(uint64_t* __restrict__ rows, int logn, uint64_t p,
                        const ulonglong2* __restrict__ tw, ulonglong2 ninv) {
  extern __shared__ uint64_t s64[];
  const int n = 1 << logn;
  uint64_t* a = s64;
  const ulonglong2* __restrict__ w = tw;
  uint64_t* r = rows + (size_t)blockIdx.x * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = r[i];
  __syncthreads();
  const uint64_t p2 = 2 * p;
  if (!INVERSE) {
    for (int s = 0; s < logn; ++s) {
      const int m = 1 << s, t = n >> (s + 1);
      for (int b = threadIdx.x; b < n / 2; b += blockDim.x) {
        const int grp = b / t, k = b % t;
        const int j = 2 * grp * t + k;
        const ulonglong2 ww = __ldg(&w[m + grp]);
        uint64_t X = csub64(a[j], p2);
        const uint64_t T = mul_shoup64_lazy(a[j + t], ww.x, ww.y, p);
        a[j] = X + T;
        a[j + t] = X - T + p2;
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) r[i] = csub64(csub64(a[i], p2), p);
  } else {
    for (int s = logn - 1; s >= 0; --s) {
      const int m = 1 << s, t = n >> (s + 1);
      for (int b = threadIdx.x; b < n / 2; b += blockDim.x) {
        const int grp = b / t, k = b % t;
        const int j = 2 * grp * t + k;
        const ulonglong2 ww = __ldg(&w[m + grp]);
        const uint64_t X = a[j], Y = a[j + t];
        a[j] = csub64(X + Y, p2);
        a[j + t] = mul_shoup64_lazy(X - Y + p2, ww.x, ww.y, p);
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      r[i] = csub64(mul_shoup64_lazy(a[i], ninv.x, ninv.y, p), p);
  }
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

}  // namespace hcnn
