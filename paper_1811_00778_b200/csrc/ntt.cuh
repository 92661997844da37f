// CTA-level negacyclic NTT over RNS limbs (u32 residues, p < 2^30).
//
// What it computes.  The reference transforms with a psi-twist followed by a
// bit-reverse + radix-2 Cooley-Tukey pass and keeps natural order
// (ring.py:147-163, ntt.py:113-139): ref[k] = a(psi^(2k+1)).  On the device
// the twist is merged into the twiddles (negacyclic Cooley-Tukey, natural
// input, bit-reversed output; Gentleman-Sande inverse with N^-1 folded in at
// the end), so that
//     dev[i] = a(psi^(2*brv(i)+1)),  i.e.  ref[k] = dev[brv(k)],
// with the same psi (the reference's primitive root search, ntt.py:50-60).
// Only pointwise products and sums happen in the NTT domain, so results in the
// coefficient domain are bit-identical to the reference's; reference-order
// NTT-domain keys are permuted once at upload.
//
// How.  One CTA transforms NR rows of N residues of the same prime in lockstep
// (NR = 1 or 2: the rows share every twiddle load, barrier and exchange).  T =
// N/E threads each keep E = 2^LOGE residues of every row in registers.  The
// top LOGN - REM butterfly bits are done in radix-E passes (LOGE stages in
// registers, then an exchange through padded shared memory, alternating
// between two buffers so that each exchange needs one barrier); the REM =
// LOGN mod LOGE lowest bits are done with warp shuffles (radix-16 geometry) or
// in registers after one more exchange (radix-32 geometry).  Butterflies are
// Harvey's lazy ones: forward values in [0, 4p), inverse values in [0, 2p).
// Twiddles are Shoup pairs (w, floor(w 2^32/p)) indexed like SEAL's psi^brv
// table; each thread loads the 2^ss twiddles of stage ss as one contiguous
// vector (15 per radix-16 pass in 8 loads).
#pragma once
#include "modarith.cuh"

namespace hcnn {

__host__ __device__ constexpr int pick_loge(int logn) {
  return logn >= 15 ? 5 : logn >= 9 ? 4 : logn >= 6 ? logn - 5 : 1;
}

// MIXED geometries cover the LOGN butterfly bits with passes of unequal
// width and no tail: the first pass takes LOGE bits (natural layout in), the
// remaining bits are split evenly over the other passes; a pass narrower than
// LOGE works on E / 2^kb independent groups per thread.  They use one
// exchange buffer at radix 32 (so that two CTAs fit one SM).
template <int LOGN_, int LOGE_ = pick_loge(LOGN_), bool SHFL_TAIL_ = (LOGE_ <= 4), bool MIXED_ = false>
struct NttGeom {
  static constexpr int LOGN = LOGN_;
  static constexpr int N = 1 << LOGN;
  static constexpr int LOGE = LOGE_;
  static constexpr int E = 1 << LOGE;
  static constexpr int LOGT = LOGN - LOGE;
  static constexpr int T = 1 << LOGT;
  static constexpr bool MIXED = MIXED_;
  static constexpr int REST = LOGN - LOGE;
  static constexpr int NFULL = MIXED ? 1 + (REST + LOGE - 1) / LOGE : LOGN / LOGE;  // passes
  static constexpr int REM = MIXED ? 0 : LOGN % LOGE;  // low bits of the tail
  static constexpr bool SHFL_TAIL = !MIXED && SHFL_TAIL_ && REM > 0;
  // a one-bit shuffle tail (N = 2^13, 2^9) swaps register halves between the
  // lane pair once instead of exchanging every butterfly's operands and
  // results (fwd_swap / inv_swap); the spectral layout keeps the swap
  static constexpr bool SWAP_TAIL = SHFL_TAIL && REM == 1;
  static constexpr bool REG_TAIL = !MIXED && !SHFL_TAIL_ && REM > 0;
  static_assert(!SHFL_TAIL || T >= 32, "shuffle stages need full warps");
  // shared-memory words for one padded row; an NR-row NTT uses
  // ntt_smem_words(NR) (two alternating buffers of NR rows)
  static constexpr int SMEM_WORDS = N + 2 * (N >> 5) + 2;
  static constexpr int XW = (SMEM_WORDS + 3) & ~3;
  // two alternating exchange buffers (one barrier per exchange) when they fit
  // in LIMIT_WORDS, else one buffer and two barriers per exchange
  static constexpr int LIMIT_WORDS = (MIXED && LOGE >= 5 ? 40 : 200) * 1024 / 4;
  __host__ __device__ static constexpr bool dbl(int nr) { return 2 * nr * XW <= LIMIT_WORDS; }
  __host__ __device__ static constexpr int ntt_smem_words(int nr) { return (dbl(nr) ? 2 : 1) * nr * XW; }
  __host__ __device__ static constexpr bool fits(int nr) { return ntt_smem_words(nr) <= 227 * 1024 / 4; }
  static constexpr int FWD_EXCHANGES = NFULL - 1 + (REG_TAIL ? 1 : 0);
  // width of pass P (from the top bits)
  __host__ __device__ static constexpr int kb(int P) {
    return !MIXED ? LOGE : P == 0 ? LOGE : REST / (NFULL - 1) + ((P - 1) < REST % (NFULL - 1) ? 1 : 0);
  }
  // pass P covers butterfly bits [lo(P), lo(P) + kb(P)), from the top
  __host__ __device__ static constexpr int lo(int P) { return P < 0 ? LOGN : lo(P - 1) - kb(P); }
};

// padded shared-memory slot of element idx (2 words every 32)
DI int sidx(int idx) { return idx + ((idx >> 5) << 1); }

// Element index held in register e of thread tid during a pass covering
// butterfly bits [LO, LO+KB): e supplies those bits, tid the others.
template <int LO, int KB>
DI int pass_index(int tid, int e) {
  return ((tid >> LO) << (LO + KB)) | (e << LO) | (tid & ((1 << LO) - 1));
}

// Element index of register e in a pass of KB <= LOGE bits at [LO, LO+KB):
// e = (g, el), el supplies the butterfly bits and o = (g, tid) the others.
template <class G, int LO, int KB>
DI int gpass_index(int tid, int e) {
  if constexpr (KB == G::LOGE) {
    return pass_index<LO, KB>(tid, e);
  } else {
    const int o = ((e >> KB) << G::LOGT) | tid;
    return ((o >> LO) << (LO + KB)) | ((e & ((1 << KB) - 1)) << LO) | (o & ((1 << LO) - 1));
  }
}

DI uint32_t umin32(uint32_t a, uint32_t b) { return a < b ? a : b; }

// Twiddle loads are volatile non-coherent loads: kernels that run several
// transforms with the same table must not keep one transform's twiddles live
// into the next (the compiler would CSE __ldg loads and pin registers).
DI uint4 ldg_tw4(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

DI uint2 ldg_tw2(const uint2* p) {
  uint2 r;
  asm volatile("ld.global.nc.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

// register-tail mapping: bits [0, REM) from e's low bits, group e >> REM and
// tid fill the rest
template <class G>
DI int tail_index(int tid, int e) {
  return ((((e >> G::REM) * G::T) + tid) << G::REM) | (e & ((1 << G::REM) - 1));
}

// COUNT consecutive twiddles starting at an index aligned to COUNT
template <int COUNT>
DI void load_tw(uint2* w, const uint2* __restrict__ tw, int base) {
  if constexpr (COUNT == 1) {
    w[0] = ldg_tw2(&tw[base]);
  } else {
    const uint4* v = reinterpret_cast<const uint4*>(tw + base);
#pragma unroll
    for (int k = 0; k < COUNT / 2; ++k) {
      const uint4 q = ldg_tw4(&v[k]);
      w[2 * k] = make_uint2(q.x, q.y);
      w[2 * k + 1] = make_uint2(q.z, q.w);
    }
  }
}

DI void bfly_fwd(uint32_t& a, uint32_t& b, uint2 w, uint32_t p, uint32_t p2) {
  uint32_t X = umin32(a, a - p2);
  const uint32_t Tt = mul_shoup_lazy(b, w.x, w.y, p);
  a = X + Tt;
  b = X - Tt + p2;
}

DI void bfly_inv(uint32_t& a, uint32_t& b, uint2 w, uint32_t p, uint32_t p2) {
  const uint32_t X = a, Y = b;
  const uint32_t U = X + Y;
  a = umin32(U, U - p2);
  b = mul_shoup_lazy(X - Y + p2, w.x, w.y, p);
}

// twiddle pairs live at once per stage (bounds register pressure at radix 32)
constexpr int TW_CHUNK = 4;

// forward (CT) stage SS of a pass at bits [LO, LO+KB); values in [0, 4p)
template <class G, int LO, int KB, int SS, int NR>
DI void fwd_stage(uint32_t* x, const uint2* __restrict__ tw, uint32_t p, int tid) {
  if constexpr (SS < KB) {
    constexpr int bpos = LO + KB - 1 - SS;
    constexpr int s = G::LOGN - 1 - bpos;
    constexpr int half = 1 << (KB - 1 - SS);
    const uint32_t p2 = 2 * p;
#pragma unroll
    for (int g = 0; g < (G::E >> KB); ++g) {
      const int o = (g << G::LOGT) | tid;
      // twiddles in chunks of TWC pairs, loaded just before their butterflies
      constexpr int TWC = (1 << SS) < TW_CHUNK ? (1 << SS) : TW_CHUNK;
#pragma unroll
      for (int tc = 0; tc < (1 << SS); tc += TWC) {
        uint2 w[TWC];
        load_tw<TWC>(w, tw, (1 << s) + ((o >> LO) << SS) + tc);
#pragma unroll
        for (int el = tc << (KB - SS); el < (tc + TWC) << (KB - SS); ++el) {
          if (el & half) continue;
          const int e = (g << KB) | el;
#pragma unroll
          for (int r = 0; r < NR; ++r) bfly_fwd(x[r * G::E + e], x[r * G::E + (e | half)], w[(el >> (KB - SS)) - tc], p, p2);
        }
      }
    }
    fwd_stage<G, LO, KB, SS + 1, NR>(x, tw, p, tid);
  }
}

// inverse (GS) stage SS of a pass (SS descending = bits ascending); values
// in [0, 2p).  The last stage (s = 0, one twiddle psi^-N/2 for every
// butterfly) also applies the output scaling: sum * n, difference * nw, both
// fully reduced.
template <class G, int LO, int KB, int SS, int NR>
DI void inv_stage(uint32_t* x, const uint2* __restrict__ itw, uint32_t p, int tid, const InvScale& sc) {
  if constexpr (SS >= 0) {
    constexpr int bpos = LO + KB - 1 - SS;
    constexpr int s = G::LOGN - 1 - bpos;
    constexpr int half = 1 << (KB - 1 - SS);
    const uint32_t p2 = 2 * p;
    if constexpr (s == 0) {
#pragma unroll
      for (int e = 0; e < G::E; ++e) {
        if (e & half) continue;
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          const uint32_t X = x[r * G::E + e], Y = x[r * G::E + (e | half)];
          x[r * G::E + e] = mul_shoup(X + Y, sc.n.x, sc.n.y, p);
          x[r * G::E + (e | half)] = mul_shoup(X - Y + p2, sc.nw.x, sc.nw.y, p);
        }
      }
    } else {
#pragma unroll
      for (int g = 0; g < (G::E >> KB); ++g) {
        const int o = (g << G::LOGT) | tid;
        // twiddles in chunks of TWC pairs, loaded just before their butterflies
        constexpr int TWC = (1 << SS) < TW_CHUNK ? (1 << SS) : TW_CHUNK;
#pragma unroll
        for (int tc = 0; tc < (1 << SS); tc += TWC) {
          uint2 w[TWC];
          load_tw<TWC>(w, itw, (1 << s) + ((o >> LO) << SS) + tc);
#pragma unroll
          for (int el = tc << (KB - SS); el < (tc + TWC) << (KB - SS); ++el) {
            if (el & half) continue;
            const int e = (g << KB) | el;
#pragma unroll
            for (int r = 0; r < NR; ++r) bfly_inv(x[r * G::E + e], x[r * G::E + (e | half)], w[(el >> (KB - SS)) - tc], p, p2);
          }
        }
      }
    }
    inv_stage<G, LO, KB, SS - 1, NR>(x, itw, p, tid, sc);
  }
}

// register tail, forward stage SS (bits REM-1-SS), all E/2^REM groups
template <class G, int SS, int NR>
DI void fwd_tail(uint32_t* x, const uint2* __restrict__ tw, uint32_t p, int tid) {
  if constexpr (SS < G::REM) {
    constexpr int R = G::REM;
    constexpr int bpos = R - 1 - SS;
    constexpr int s = G::LOGN - 1 - bpos;
    constexpr int half = 1 << (R - 1 - SS);
    const uint32_t p2 = 2 * p;
#pragma unroll
    for (int grp = 0; grp < (G::E >> R); ++grp) {
      uint2 w[1 << SS];
      load_tw<(1 << SS)>(w, tw, (1 << s) + ((grp * G::T + tid) << SS));
#pragma unroll
      for (int el = 0; el < (1 << R); ++el) {
        if (el & half) continue;
        const int e = (grp << R) | el;
#pragma unroll
        for (int r = 0; r < NR; ++r) bfly_fwd(x[r * G::E + e], x[r * G::E + (e | half)], w[el >> (R - SS)], p, p2);
      }
    }
    fwd_tail<G, SS + 1, NR>(x, tw, p, tid);
  }
}

template <class G, int SS, int NR>
DI void inv_tail(uint32_t* x, const uint2* __restrict__ itw, uint32_t p, int tid) {
  if constexpr (SS >= 0) {
    constexpr int R = G::REM;
    constexpr int bpos = R - 1 - SS;
    constexpr int s = G::LOGN - 1 - bpos;
    constexpr int half = 1 << (R - 1 - SS);
    const uint32_t p2 = 2 * p;
#pragma unroll
    for (int grp = 0; grp < (G::E >> R); ++grp) {
      uint2 w[1 << SS];
      load_tw<(1 << SS)>(w, itw, (1 << s) + ((grp * G::T + tid) << SS));
#pragma unroll
      for (int el = 0; el < (1 << R); ++el) {
        if (el & half) continue;
        const int e = (grp << R) | el;
#pragma unroll
        for (int r = 0; r < NR; ++r) bfly_inv(x[r * G::E + e], x[r * G::E + (e | half)], w[el >> (R - SS)], p, p2);
      }
    }
    inv_tail<G, SS - 1, NR>(x, itw, p, tid);
  }
}

// twiddle index of the shuffle stage at butterfly bit b < REM for register e,
// in the spectral layout (last pass LO = REM): (1 << s) + (j >> (b + 1))
template <class G>
DI int shfl_tw_index(int tid, int e, int b) {
  const int j = pass_index<G::REM, G::LOGE>(tid, e);
  return (1 << (G::LOGN - 1 - b)) + (j >> (b + 1));
}

// Twiddles of the shuffle stage at bit B for registers [e0, e0 + CNT) of
// this lane (every lane loads only the half it multiplies with).
template <class G, int B, int CNT>
DI void load_shfl_tw(uint2* w, const uint2* __restrict__ tw, int tid, int e0) {
  if constexpr (B == G::REM - 1) {
    // consecutive in e: aligned vectors
    load_tw<CNT>(w, tw, shfl_tw_index<G>(tid, 0, B) + e0);
  } else {
#pragma unroll
    for (int k = 0; k < CNT; ++k) w[k] = __ldg(&tw[shfl_tw_index<G>(tid, e0 + k, B)]);
  }
}

// Butterflies on the REM lowest bits through warp shuffles.  Lanes L and U =
// L ^ 2^B hold the two operands of every butterfly in the same register e;
// L computes the butterflies of e < E/2 and U those of e >= E/2 (one shuffle
// brings the partner operand, one returns the partner result), so every
// modular product is computed once.
template <class G, int B, int NR>
DI void fwd_shfl(uint32_t* x, const uint2* __restrict__ tw, uint32_t p, int tid) {
  if constexpr (B >= 0) {
    constexpr int H = G::E / 2;
    constexpr int C = H < TW_CHUNK ? H : TW_CHUNK;
    const uint32_t p2 = 2 * p;
    const bool upper = (tid >> B) & 1;
    const int off = upper ? H : 0;
#pragma unroll
    for (int c0 = 0; c0 < H; c0 += C) {
      uint2 w[C];
      load_shfl_tw<G, B, C>(w, tw, tid, c0 + off);
#pragma unroll
      for (int k = 0; k < C; ++k) {
        const int e = c0 + k;
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          uint32_t& lo = x[r * G::E + e];
          uint32_t& hi = x[r * G::E + e + H];
          const uint32_t got = __shfl_xor_sync(0xffffffffu, upper ? lo : hi, 1 << B);
          uint32_t X = upper ? got : lo;   // L: own e, U: L's e+H
          const uint32_t Y = upper ? hi : got;
          X = umin32(X, X - p2);
          const uint32_t Tt = mul_shoup_lazy(Y, w[k].x, w[k].y, p);
          const uint32_t A = X + Tt, Bv = X - Tt + p2;  // results for L, U
          const uint32_t back = __shfl_xor_sync(0xffffffffu, upper ? A : Bv, 1 << B);
          lo = upper ? back : A;
          hi = upper ? Bv : back;
        }
      }
    }
    fwd_shfl<G, B - 1, NR>(x, tw, p, tid);
  }
}

template <class G, int B, int NR>
DI void inv_shfl(uint32_t* x, const uint2* __restrict__ itw, uint32_t p, int tid) {
  if constexpr (B < G::REM) {
    constexpr int H = G::E / 2;
    constexpr int C = H < TW_CHUNK ? H : TW_CHUNK;
    const uint32_t p2 = 2 * p;
    const bool upper = (tid >> B) & 1;
    const int off = upper ? H : 0;
#pragma unroll
    for (int c0 = 0; c0 < H; c0 += C) {
      uint2 w[C];
      load_shfl_tw<G, B, C>(w, itw, tid, c0 + off);
#pragma unroll
      for (int k = 0; k < C; ++k) {
        const int e = c0 + k;
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          uint32_t& lo = x[r * G::E + e];
          uint32_t& hi = x[r * G::E + e + H];
          const uint32_t got = __shfl_xor_sync(0xffffffffu, upper ? lo : hi, 1 << B);
          const uint32_t X = upper ? got : lo;
          const uint32_t Y = upper ? hi : got;
          const uint32_t U = X + Y;
          const uint32_t A = umin32(U, U - p2);
          const uint32_t Bv = mul_shoup_lazy(X - Y + p2, w[k].x, w[k].y, p);
          const uint32_t back = __shfl_xor_sync(0xffffffffu, upper ? A : Bv, 1 << B);
          lo = upper ? back : A;
          hi = upper ? Bv : back;
        }
      }
    }
    inv_shfl<G, B + 1, NR>(x, itw, p, tid);
  }
}

// One-bit shuffle tail by a register-half swap.  Lane L (bit 0 of tid clear)
// and U = L ^ 1 hold the two operands of every butterfly in the same register
// e.  swap_halves: L sends x[e + E/2] and receives U's x[e] into it, U sends
// x[e] and receives L's x[e + E/2] into it; afterwards every butterfly is
// local: L owns the pairs e < E/2, U the pairs e + E/2, both on registers
// (e, e + E/2).  The forward ends swapped (spectral_index absorbs it), the
// inverse starts there and swaps back after its first stage.  One SHFL and
// three SELs per register pair instead of two SHFLs and ~six SELs per
// butterfly.
template <class G, int NR>
DI void swap_halves(uint32_t* x, int tid) {
  constexpr int H = G::E / 2;
  const bool upper = tid & 1;
#pragma unroll
  for (int e = 0; e < H; ++e)
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      uint32_t& lo = x[r * G::E + e];
      uint32_t& hi = x[r * G::E + e + H];
      const uint32_t got = __shfl_xor_sync(0xffffffffu, upper ? lo : hi, 1);
      lo = upper ? got : lo;
      hi = upper ? hi : got;
    }
}

template <class G, int NR>
DI void fwd_swap(uint32_t* x, const uint2* __restrict__ tw, uint32_t p, int tid) {
  constexpr int H = G::E / 2;
  constexpr int C = H < TW_CHUNK ? H : TW_CHUNK;
  const uint32_t p2 = 2 * p;
  const int off = (tid & 1) ? H : 0;
  swap_halves<G, NR>(x, tid);
#pragma unroll
  for (int c0 = 0; c0 < H; c0 += C) {
    uint2 w[C];
    load_shfl_tw<G, 0, C>(w, tw, tid, c0 + off);
#pragma unroll
    for (int k = 0; k < C; ++k)
#pragma unroll
      for (int r = 0; r < NR; ++r) bfly_fwd(x[r * G::E + c0 + k], x[r * G::E + c0 + k + H], w[k], p, p2);
  }
}

template <class G, int NR>
DI void inv_swap(uint32_t* x, const uint2* __restrict__ itw, uint32_t p, int tid) {
  constexpr int H = G::E / 2;
  constexpr int C = H < TW_CHUNK ? H : TW_CHUNK;
  const uint32_t p2 = 2 * p;
  const int off = (tid & 1) ? H : 0;
#pragma unroll
  for (int c0 = 0; c0 < H; c0 += C) {
    uint2 w[C];
    load_shfl_tw<G, 0, C>(w, itw, tid, c0 + off);
#pragma unroll
    for (int k = 0; k < C; ++k)
#pragma unroll
      for (int r = 0; r < NR; ++r) bfly_inv(x[r * G::E + c0 + k], x[r * G::E + c0 + k + H], w[k], p, p2);
  }
  swap_halves<G, NR>(x, tid);
}

// exchange buffer XI of an NR-row transform
template <class G, int NR>
DI uint32_t* xbuf(uint32_t* s, int xi) {
  if constexpr (G::dbl(NR)) return s + (xi & 1) * NR * G::XW;
  else return s;
}

// before writing an exchange buffer: with a single buffer, wait until every
// thread has read the previous exchange
template <class G, int NR>
DI void pre_exchange() {
  if constexpr (!G::dbl(NR)) __syncthreads();
}

// after a transform: with two buffers the next transform's first exchange
// writes buffer 0, which was read by this one's last exchange when the count
// is odd; with one buffer it is always the same buffer
template <class G, int NR>
DI void post_transform() {
  if constexpr (G::FWD_EXCHANGES > 0 && (!G::dbl(NR) || (G::FWD_EXCHANGES & 1))) __syncthreads();
}

// The pass maps are bit permutations of (e, tid), so an element's padded slot
// splits into a per-thread base plus a compile-time offset per register:
// sidx(A | C) = sidx(A) + sidx(C) for disjoint bit sets A, C.
template <class G, int P, int NR>
DI void regs_to_smem(const uint32_t* x, uint32_t* b, int tid) {
  uint32_t* bt = b + sidx(gpass_index<G, G::lo(P), G::kb(P)>(tid, 0));
#pragma unroll
  for (int r = 0; r < NR; ++r)
#pragma unroll
    for (int e = 0; e < G::E; ++e) bt[r * G::XW + sidx(gpass_index<G, G::lo(P), G::kb(P)>(0, e))] = x[r * G::E + e];
}

template <class G, int P, int NR>
DI void smem_to_regs(uint32_t* x, const uint32_t* b, int tid) {
  const uint32_t* bt = b + sidx(gpass_index<G, G::lo(P), G::kb(P)>(tid, 0));
#pragma unroll
  for (int r = 0; r < NR; ++r)
#pragma unroll
    for (int e = 0; e < G::E; ++e) x[r * G::E + e] = bt[r * G::XW + sidx(gpass_index<G, G::lo(P), G::kb(P)>(0, e))];
}

template <class G, int P, int NR>
DI void fwd_from(uint32_t* x, uint32_t* s, const uint2* __restrict__ tw, uint32_t p, int tid) {
  if constexpr (P < G::NFULL) {
    if constexpr (P > 0) {
      uint32_t* b = xbuf<G, NR>(s, P - 1);  // exchange P-1
      pre_exchange<G, NR>();
      regs_to_smem<G, P - 1, NR>(x, b, tid);
      __syncthreads();
      smem_to_regs<G, P, NR>(x, b, tid);
    }
    fwd_stage<G, G::lo(P), G::kb(P), 0, NR>(x, tw, p, tid);
    fwd_from<G, P + 1, NR>(x, s, tw, p, tid);
  }
}

template <class G, int P, int NR>
DI void inv_from(uint32_t* x, uint32_t* s, const uint2* __restrict__ itw, uint32_t p, int tid, const InvScale& sc) {
  if constexpr (P >= 0) {
    if constexpr (P < G::NFULL - 1) {
      // exchange index continues after the register-tail exchange (if any)
      constexpr int XI = (G::REG_TAIL ? 1 : 0) + (G::NFULL - 2 - P);
      uint32_t* b = xbuf<G, NR>(s, XI);
      pre_exchange<G, NR>();
      regs_to_smem<G, P + 1, NR>(x, b, tid);
      __syncthreads();
      smem_to_regs<G, P, NR>(x, b, tid);
    }
    inv_stage<G, G::lo(P), G::kb(P), G::kb(P) - 1, NR>(x, itw, p, tid, sc);
    inv_from<G, P - 1, NR>(x, s, itw, p, tid, sc);
  }
}

// Register layouts at the boundaries:
//   natural  : x[e] = a[e * T + tid]                     (coalesced global access)
//   spectral : x[e] = A[spectral_index(tid, e)]          (what the forward leaves)
//   tiled    : spectral values in 16-byte groups (device key layout, below)
template <class G>
DI int natural_index(int tid, int e) { return e * G::T + tid; }

template <class G>
DI int spectral_index(int tid, int e) {
  if constexpr (G::MIXED) return gpass_index<G, 0, G::kb(G::NFULL - 1)>(tid, e);
  else if constexpr (G::REG_TAIL) return tail_index<G>(tid, e);
  else if constexpr (G::SWAP_TAIL) {
    // register bit LOGE-1 and lane bit 0 exchanged (fwd_swap)
    constexpr int H = G::E / 2;
    const int lane = (tid & ~1) | (e >= H ? 1 : 0);
    const int ee = (e & (H - 1)) | ((tid & 1) ? H : 0);
    return pass_index<G::REM, G::LOGE>(lane, ee);
  } else return pass_index<G::REM, G::LOGE>(tid, e);
}

// tiled: groups of 4 spectral values, group-major then thread:
//   element e of thread tid at ((e/4) * T + tid) * 4 + e%4
// so each thread moves 16-byte vectors and a warp's vectors are contiguous
// (coalesced in global memory, conflict-free in shared memory).
template <class G>
DI int tiled_index(int tid, int e) {
  if constexpr (G::E >= 4) return (((e >> 2) * G::T + tid) << 2) | (e & 3);
  else return e * G::T + tid;
}

template <class G>
DI void load_tiled(uint32_t* x, const uint32_t* __restrict__ row, int tid) {
  if constexpr (G::E >= 4) {
    const uint4* v = reinterpret_cast<const uint4*>(row) + tid;
#pragma unroll
    for (int k = 0; k < G::E / 4; ++k) {
      const uint4 q = __ldg(&v[k * G::T]);
      x[4 * k] = q.x;
      x[4 * k + 1] = q.y;
      x[4 * k + 2] = q.z;
      x[4 * k + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int e = 0; e < G::E; ++e) x[e] = __ldg(&row[tiled_index<G>(tid, e)]);
  }
}

template <class G>
DI void store_tiled(const uint32_t* x, uint32_t* __restrict__ row, int tid) {
  if constexpr (G::E >= 4) {
    uint4* v = reinterpret_cast<uint4*>(row) + tid;
#pragma unroll
    for (int k = 0; k < G::E / 4; ++k)
      v[k * G::T] = make_uint4(x[4 * k], x[4 * k + 1], x[4 * k + 2], x[4 * k + 3]);
  } else {
#pragma unroll
    for (int e = 0; e < G::E; ++e) row[tiled_index<G>(tid, e)] = x[e];
  }
}

// Forward negacyclic NTT of NR rows of one prime: natural layout in (values
// < 4p), spectral layout out, fully reduced to [0, p) (FULL) or to [0, 2p)
// when the result only feeds Montgomery products.  `s`:
// G::ntt_smem_words(NR) words of shared memory.
template <class G, int NR = 1, bool FULL = true>
DI void ntt_fwd(uint32_t* x, uint32_t* s, const uint2* __restrict__ tw, uint32_t p, int tid) {
  fwd_from<G, 0, NR>(x, s, tw, p, tid);
  if constexpr (G::SWAP_TAIL) {
    fwd_swap<G, NR>(x, tw, p, tid);
  } else if constexpr (G::SHFL_TAIL) {
    fwd_shfl<G, G::REM - 1, NR>(x, tw, p, tid);
  } else if constexpr (G::REG_TAIL) {
    uint32_t* b = xbuf<G, NR>(s, G::NFULL - 1);
    pre_exchange<G, NR>();
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
      for (int e = 0; e < G::E; ++e) b[r * G::XW + sidx(pass_index<G::REM, G::LOGE>(tid, e))] = x[r * G::E + e];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
      for (int e = 0; e < G::E; ++e) x[r * G::E + e] = b[r * G::XW + sidx(tail_index<G>(tid, e))];
    fwd_tail<G, 0, NR>(x, tw, p, tid);
  }
  post_transform<G, NR>();
  const uint32_t p2 = 2 * p;
#pragma unroll
  for (int e = 0; e < NR * G::E; ++e) {
    const uint32_t v = umin32(x[e], x[e] - p2);
    x[e] = FULL ? umin32(v, v - p) : v;
  }
}

// Inverse negacyclic NTT of NR rows: spectral layout in (values < 2p),
// natural layout out, scaled by sc (N^-1, folded into the last stage),
// reduced to [0, p).
template <class G, int NR = 1>
DI void ntt_inv(uint32_t* x, uint32_t* s, const uint2* __restrict__ itw, uint32_t p, const InvScale& sc,
                int tid) {
  if constexpr (G::SWAP_TAIL) {
    inv_swap<G, NR>(x, itw, p, tid);
  } else if constexpr (G::SHFL_TAIL) {
    inv_shfl<G, 0, NR>(x, itw, p, tid);
  } else if constexpr (G::REG_TAIL) {
    inv_tail<G, G::REM - 1, NR>(x, itw, p, tid);
    uint32_t* b = xbuf<G, NR>(s, 0);
    pre_exchange<G, NR>();
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
      for (int e = 0; e < G::E; ++e) b[r * G::XW + sidx(tail_index<G>(tid, e))] = x[r * G::E + e];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
      for (int e = 0; e < G::E; ++e) x[r * G::E + e] = b[r * G::XW + sidx(pass_index<G::REM, G::LOGE>(tid, e))];
  }
  inv_from<G, G::NFULL - 1, NR>(x, s, itw, p, tid, sc);
  post_transform<G, NR>();
}

}  // namespace hcnn
