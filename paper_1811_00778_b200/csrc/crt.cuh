// Plaintext-CRT recombination of decrypted logits on the GPU
// (engine.reconstruct_logits, engine.py:494-506; CrtSystem.reconstruct_centered,
// codec.py:79-89; ring.crt_combine, ring.py:276-283).
//
// Every value m has one residue per channel t_i (pairwise coprime, < 2^62).
// Garner's mixed-radix form gives the unique X in [0, T), T = prod t_i,
// exactly, with single-word arithmetic per channel:
//   v_0 = r_0,  v_i = (...((r_i - v_0) c_0i - v_1) c_1i ... - v_{i-1}) c_{i-1,i}  mod t_i,
//   c_ji = t_j^-1 mod t_i,   X = v_0 + t_0 (v_1 + t_1 (v_2 + ...)),
// then the centred value X - T if X > floor(T/2) (from_modular), written as W
// little-endian 32-bit words of two's complement.  One thread per value.
#pragma once
#include <cstdint>

namespace hcnn {

constexpr int CRT_MAXC = 16;
constexpr int CRT_MAXW = 34;  // 16 x 62 bits + sign + carry, in 32-bit words

struct CrtTabs {
  int C, W;
  uint64_t t[CRT_MAXC];
  uint64_t inv[CRT_MAXC][CRT_MAXC];  // inv[j][i] = t_j^-1 mod t_i (j < i)
  uint32_t T[CRT_MAXW];              // prod t_i
  uint32_t half[CRT_MAXW];           // floor(T / 2)
};

__device__ __forceinline__ uint64_t crt_mulmod(uint64_t a, uint64_t b, uint64_t m) {
  return (uint64_t)(((unsigned __int128)a * b) % m);
}

__global__ void k_crt_combine(const uint64_t* __restrict__ res, size_t M, const CrtTabs tb,
                              uint32_t* __restrict__ out, int* __restrict__ bad) {
  const size_t m = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  uint64_t v[CRT_MAXC];
  const int C = tb.C, W = tb.W;
  for (int i = 0; i < C; ++i) {
    const uint64_t ti = tb.t[i];
    uint64_t x = res[(size_t)i * M + m];
    if (x >= ti) atomicOr(bad, 1);  // CrtSystem.reconstruct: residue outside [0, t_i)
    x %= ti;
    for (int j = 0; j < i; ++j) {
      const uint64_t vj = v[j] % ti;
      x = crt_mulmod(x >= vj ? x - vj : x + ti - vj, tb.inv[j][i], ti);
    }
    v[i] = x;
  }
  uint32_t X[CRT_MAXW];
  for (int k = 0; k < W; ++k) X[k] = 0;
  for (int i = C - 1; i >= 0; --i) {
    // X = X * t_i + v_i
    unsigned __int128 carry = v[i];
    for (int k = 0; k < W; ++k) {
      const unsigned __int128 acc = (unsigned __int128)X[k] * tb.t[i] + carry;
      X[k] = (uint32_t)acc;
      carry = acc >> 32;
    }
  }
  // X > floor(T/2)  ->  X - T (negative, two's complement over W words)
  int gt = 0;
  for (int k = W - 1; k >= 0; --k) {
    if (X[k] != tb.half[k]) {
      gt = X[k] > tb.half[k];
      break;
    }
  }
  if (gt) {
    uint64_t borrow = 0;
    for (int k = 0; k < W; ++k) {
      const uint64_t d = (uint64_t)X[k] - tb.T[k] - borrow;
      X[k] = (uint32_t)d;
      borrow = (d >> 63) & 1;
    }
  }
  uint32_t* o = out + m * (size_t)W;
  for (int k = 0; k < W; ++k) o[k] = X[k];
}

}  // namespace hcnn
