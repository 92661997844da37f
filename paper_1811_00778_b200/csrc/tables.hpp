// Host-side precomputation for one BFV context: primes of the auxiliary base
// P, NTT twiddles, exact CRT / base-conversion constants.  Pure C++ (no CUDA).
//
// Reference counterparts: RnsContext tables and CRT weights (ring.py:51-95),
// NttPlan / find_primitive_2n_root / stage twiddles (ntt.py:50-108),
// BfvParams' l and Delta (bfv.py:45-91).
#pragma once
#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace hcnn {

using u32 = uint32_t;
using u64 = uint64_t;
using u128 = unsigned __int128;

// ----------------------------------------------------------------- modular u64
inline u64 mulmod64(u64 a, u64 b, u64 m) { return (u64)((u128)a * b % m); }
inline u64 powmod64(u64 b, u64 e, u64 m) {
  u64 r = 1 % m;
  b %= m;
  while (e) {
    if (e & 1) r = mulmod64(r, b, m);
    b = mulmod64(b, b, m);
    e >>= 1;
  }
  return r;
}
inline u64 invmod64(u64 a, u64 m) {  // m prime
  return powmod64(a % m, m - 2, m);
}

// deterministic Miller-Rabin for n < 3.3e24 (same bases as ntt.py:25-47)
inline bool is_prime64(u64 n) {
  if (n < 2) return false;
  static const u64 bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  for (u64 b : bases)
    if (n % b == 0) return n == b;
  u64 d = n - 1;
  int r = 0;
  while ((d & 1) == 0) {
    d >>= 1;
    ++r;
  }
  for (u64 a : bases) {
    u64 x = powmod64(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int i = 0; i < r - 1; ++i) {
      x = mulmod64(x, x, n);
      if (x == n - 1) {
        comp = false;
        break;
      }
    }
    if (comp) return false;
  }
  return true;
}

// The reference's root: first g^((p-1)/2N), g = 2, 3, ..., whose N-th power is
// -1 (ntt.py:50-60).  NTT-domain keys depend on this exact choice.
inline u64 primitive_2n_root(u64 p, u64 n) {
  if ((p - 1) % (2 * n)) throw std::invalid_argument("prime is not 1 mod 2N");
  const u64 e = (p - 1) / (2 * n);
  for (u64 g = 2; g < p; ++g) {
    u64 c = powmod64(g, e, p);
    if (powmod64(c, n, p) == p - 1) return c;
  }
  throw std::invalid_argument("no primitive 2N-th root");
}

inline u32 bitrev(u32 x, int bits) {
  u32 r = 0;
  for (int i = 0; i < bits; ++i) {
    r = (r << 1) | (x & 1);
    x >>= 1;
  }
  return r;
}

// ------------------------------------------------------------ small bigint
// little-endian base-2^32 magnitude
struct Big {
  std::vector<u32> w;
  Big() {}
  explicit Big(u64 v) {
    if (v) w.push_back((u32)v);
    if (v >> 32) w.push_back((u32)(v >> 32));
  }
  void trim() {
    while (!w.empty() && w.back() == 0) w.pop_back();
  }
  bool is_zero() const { return w.empty(); }
  int bits() const {
    if (w.empty()) return 0;
    int b = 32 * (int)(w.size() - 1);
    u32 top = w.back();
    while (top) {
      ++b;
      top >>= 1;
    }
    return b;
  }
  u32 word(size_t i) const { return i < w.size() ? w[i] : 0; }
};

inline Big mul_small(const Big& a, u64 m) {
  Big r;
  u128 carry = 0;
  for (size_t i = 0; i < a.w.size(); ++i) {
    u128 cur = (u128)a.w[i] * m + carry;
    r.w.push_back((u32)cur);
    carry = cur >> 32;
  }
  while (carry) {
    r.w.push_back((u32)carry);
    carry >>= 32;
  }
  r.trim();
  return r;
}

inline Big add(const Big& a, const Big& b) {
  Big r;
  u64 carry = 0;
  size_t n = std::max(a.w.size(), b.w.size());
  for (size_t i = 0; i < n; ++i) {
    u64 s = (u64)a.word(i) + b.word(i) + carry;
    r.w.push_back((u32)s);
    carry = s >> 32;
  }
  if (carry) r.w.push_back((u32)carry);
  r.trim();
  return r;
}

inline int cmp(const Big& a, const Big& b) {
  if (a.w.size() != b.w.size()) return a.w.size() < b.w.size() ? -1 : 1;
  for (size_t i = a.w.size(); i-- > 0;)
    if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
  return 0;
}

inline Big sub(const Big& a, const Big& b) {  // a >= b
  Big r;
  int64_t borrow = 0;
  for (size_t i = 0; i < a.w.size(); ++i) {
    int64_t d = (int64_t)a.w[i] - b.word(i) - borrow;
    borrow = d < 0;
    r.w.push_back((u32)(d + (borrow << 32)));
  }
  r.trim();
  return r;
}

inline u64 mod_small(const Big& a, u64 m) {
  u128 r = 0;
  for (size_t i = a.w.size(); i-- > 0;) r = ((r << 32) | a.w[i]) % m;
  return (u64)r;
}

inline Big div_small(const Big& a, u64 m) {
  Big q;
  q.w.assign(a.w.size(), 0);
  u128 r = 0;
  for (size_t i = a.w.size(); i-- > 0;) {
    r = (r << 32) | a.w[i];
    q.w[i] = (u32)(r / m);
    r %= m;
  }
  q.trim();
  return q;
}

inline Big shr1(const Big& a) {
  Big r;
  r.w.assign(a.w.size(), 0);
  for (size_t i = 0; i < a.w.size(); ++i) {
    r.w[i] = (a.w[i] >> 1) | (i + 1 < a.w.size() ? (a.w[i + 1] << 31) : 0);
  }
  r.trim();
  return r;
}

inline Big product(const std::vector<u64>& ps) {
  Big r(1);
  for (u64 p : ps) r = mul_small(r, p);
  return r;
}

// Auxiliary-base primes: largest p < 2^30 with p = 1 mod 2^17 (every ring
// degree up to 2^16), skipping the primes of q.
inline std::vector<u64> aux_primes(const std::vector<u64>& avoid, size_t count) {
  std::vector<u64> out;
  const u64 step = 1ull << 17;
  for (u64 k = 1; out.size() < count; ++k) {
    u64 p = (1ull << 30) - k * step + 1;
    if (p < (1ull << 28)) throw std::runtime_error("ran out of auxiliary primes");
    if (std::find(avoid.begin(), avoid.end(), p) != avoid.end()) continue;
    if (is_prime64(p)) out.push_back(p);
  }
  return out;
}

}  // namespace hcnn
