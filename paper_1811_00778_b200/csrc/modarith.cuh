// Word-size modular arithmetic for the RNS limbs (primes < 2^30, u32 lanes).
//
// Residues of the reference are canonical [0, p) int64 (ring.py:98-112); the
// device keeps them as u32.  Fixed operands (twiddles, rlk, CRT constants) use
// Shoup's precomputed quotient (3 integer multiplies, result in [0, 2p));
// variable x variable products go through a 64-bit Barrett reduction.
#pragma once
#include <cstdint>

#define HD __host__ __device__ __forceinline__
#define DI __device__ __forceinline__

namespace hcnn {

// floor(w * 2^32 / p): Shoup companion of a fixed multiplicand w < p.
HD uint32_t shoup_of(uint32_t w, uint32_t p) {
  return (uint32_t)(((uint64_t)w << 32) / p);
}

// x * w mod p in [0, 2p) for any x < 2^32 and w < p.
DI uint32_t mul_shoup_lazy(uint32_t x, uint32_t w, uint32_t ws, uint32_t p) {
  uint32_t qh = __umulhi(x, ws);
  return x * w - qh * p;
}

DI uint32_t csub(uint32_t x, uint32_t p) { return x >= p ? x - p : x; }

DI uint32_t mul_shoup(uint32_t x, uint32_t w, uint32_t ws, uint32_t p) {
  return csub(mul_shoup_lazy(x, w, ws, p), p);
}

DI uint32_t add_mod(uint32_t a, uint32_t b, uint32_t p) { return csub(a + b, p); }
DI uint32_t sub_mod(uint32_t a, uint32_t b, uint32_t p) { return a >= b ? a - b : a + p - b; }

// x mod p for any 64-bit x; mu = floor(2^64 / p).
DI uint32_t reduce64(uint64_t x, uint32_t p, uint64_t mu) {
  uint64_t qh = __umul64hi(x, mu);
  uint32_t r = (uint32_t)(x - qh * (uint64_t)p);  // in [0, 2p)
  return csub(r, p);
}

DI uint32_t mul_mod(uint32_t a, uint32_t b, uint32_t p, uint64_t mu) {
  return reduce64((uint64_t)a * b, p, mu);
}

// Montgomery reduction z 2^-32 mod p in [0, 2p) for z < 2^32 p;
// pinv = -p^-1 mod 2^32.
DI uint32_t redc64(uint64_t z, uint32_t p, uint32_t pinv) {
  const uint32_t m = (uint32_t)z * pinv;
  return (uint32_t)((z + (uint64_t)m * p) >> 32);
}

// Montgomery product x k 2^-32 mod p in [0, 2p) for x, k < p < 2^30.  With
// k = k' 2^32 mod p (Montgomery form) this is x k' mod p.
DI uint32_t mont_mul(uint32_t x, uint32_t k, uint32_t p, uint32_t pinv) {
  return redc64((uint64_t)x * k, p, pinv);
}

}  // namespace hcnn
