// CTA-level negacyclic NTT over one RNS limb (u32 residues, p < 2^30).
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
// How.  One CTA owns one row of N residues: T = N/E threads each keep E = 2^LOGE
// residues in registers, run LOGE butterfly stages locally, and exchange
// through padded shared memory between passes.  Butterflies are Harvey's lazy
// ones: forward values live in [0, 4p), inverse values in [0, 2p), Shoup
// twiddles (w, floor(w 2^32 / p)) are read through the read-only path.
#pragma once
#include "modarith.cuh"

namespace hcnn {

__host__ __device__ constexpr int pick_loge(int logn) {
  return logn >= 15 ? 5 : logn >= 9 ? 4 : logn >= 6 ? logn - 5 : 1;
}

template <int LOGN>
struct NttGeom {
  static constexpr int N = 1 << LOGN;
  static constexpr int LOGE = pick_loge(LOGN);
  static constexpr int E = 1 << LOGE;
  static constexpr int LOGT = LOGN - LOGE;
  static constexpr int T = 1 << LOGT;
  static constexpr int NFULL = LOGN / LOGE;
  static constexpr int REM = LOGN % LOGE;
  static constexpr int NPASS = NFULL + (REM ? 1 : 0);
  // shared-memory words for one padded row
  static constexpr int SMEM_WORDS = N + 2 * (N >> 5) + 2;
  // forward pass P covers butterfly bits [lo(P), lo(P) + kb(P))
  __host__ __device__ static constexpr int lo(int P) { return P < NFULL ? LOGN - (P + 1) * LOGE : 0; }
  __host__ __device__ static constexpr int kb(int P) { return P < NFULL ? LOGE : REM; }
};

// padded shared-memory slot of element idx (2 words every 32: no bank conflicts
// for the pass layouts used here except a 2-way one in the radix-2 tail pass)
DI int sidx(int idx) { return idx + ((idx >> 5) << 1); }

// Element index held in register e of thread tid during a pass covering
// butterfly bits [LO, LO+KB).  The low KB bits of e select the butterfly
// position, the rest of e and tid fill the other bits, tid lowest.
template <int LOGN, int LO, int KB>
DI int pass_index(int tid, int e) {
  constexpr int T = NttGeom<LOGN>::T;
  const int elo = e & ((1 << KB) - 1);
  const int o = (e >> KB) * T + tid;
  return ((o >> LO) << (LO + KB)) | (elo << LO) | (o & ((1 << LO) - 1));
}

// forward (CT) butterfly stages of one pass; values in [0, 4p)
template <int LOGN, int LO, int KB>
DI void fwd_pass(uint32_t* x, const uint2* __restrict__ tw, uint32_t p, int tid) {
  constexpr int E = NttGeom<LOGN>::E;
  const uint32_t p2 = 2 * p;
#pragma unroll
  for (int ss = 0; ss < KB; ++ss) {
    const int bpos = LO + KB - 1 - ss;
    const int s = LOGN - 1 - bpos;
    const int half = 1 << (KB - 1 - ss);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (e & half) continue;
      const int j = pass_index<LOGN, LO, KB>(tid, e);
      const uint2 w = __ldg(&tw[(1 << s) + (j >> (bpos + 1))]);
      uint32_t X = x[e];
      X = X >= p2 ? X - p2 : X;
      const uint32_t Tt = mul_shoup_lazy(x[e | half], w.x, w.y, p);
      x[e] = X + Tt;
      x[e | half] = X - Tt + p2;
    }
  }
}

// inverse (GS) butterfly stages of one pass, bits ascending; values in [0, 2p)
template <int LOGN, int LO, int KB>
DI void inv_pass(uint32_t* x, const uint2* __restrict__ itw, uint32_t p, int tid) {
  constexpr int E = NttGeom<LOGN>::E;
  const uint32_t p2 = 2 * p;
#pragma unroll
  for (int ss = 0; ss < KB; ++ss) {
    const int bpos = LO + ss;
    const int s = LOGN - 1 - bpos;
    const int half = 1 << ss;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (e & half) continue;
      const int j = pass_index<LOGN, LO, KB>(tid, e);
      const uint2 w = __ldg(&itw[(1 << s) + (j >> (bpos + 1))]);
      const uint32_t X = x[e], Y = x[e | half];
      uint32_t U = X + Y;
      U = U >= p2 ? U - p2 : U;
      x[e] = U;
      x[e | half] = mul_shoup_lazy(X - Y + p2, w.x, w.y, p);
    }
  }
}

template <int LOGN, int LO, int KB>
DI void regs_to_smem(const uint32_t* x, uint32_t* s, int tid) {
#pragma unroll
  for (int e = 0; e < NttGeom<LOGN>::E; ++e) s[sidx(pass_index<LOGN, LO, KB>(tid, e))] = x[e];
}

template <int LOGN, int LO, int KB>
DI void smem_to_regs(uint32_t* x, const uint32_t* s, int tid) {
#pragma unroll
  for (int e = 0; e < NttGeom<LOGN>::E; ++e) x[e] = s[sidx(pass_index<LOGN, LO, KB>(tid, e))];
}

template <int LOGN, int P>
DI void fwd_from(uint32_t* x, uint32_t* s, const uint2* __restrict__ tw, uint32_t p, int tid) {
  using G = NttGeom<LOGN>;
  if constexpr (P < G::NPASS) {
    if constexpr (P > 0) {
      regs_to_smem<LOGN, G::lo(P - 1), G::kb(P - 1)>(x, s, tid);
      __syncthreads();
      smem_to_regs<LOGN, G::lo(P), G::kb(P)>(x, s, tid);
      __syncthreads();
    }
    fwd_pass<LOGN, G::lo(P), G::kb(P)>(x, tw, p, tid);
    fwd_from<LOGN, P + 1>(x, s, tw, p, tid);
  }
}

template <int LOGN, int P>
DI void inv_from(uint32_t* x, uint32_t* s, const uint2* __restrict__ itw, uint32_t p, int tid) {
  using G = NttGeom<LOGN>;
  if constexpr (P >= 0) {
    if constexpr (P < G::NPASS - 1) {
      regs_to_smem<LOGN, G::lo(P + 1), G::kb(P + 1)>(x, s, tid);
      __syncthreads();
      smem_to_regs<LOGN, G::lo(P), G::kb(P)>(x, s, tid);
      __syncthreads();
    }
    inv_pass<LOGN, G::lo(P), G::kb(P)>(x, itw, p, tid);
    inv_from<LOGN, P - 1>(x, s, itw, p, tid);
  }
}

// Register layouts at the boundaries:
//   natural layout  : x[e] = a[e * T + tid]            (coalesced global access)
//   spectral layout : x[e] = A[pass_index<last pass>]  (what the forward leaves)
template <int LOGN>
DI int natural_index(int tid, int e) { return e * NttGeom<LOGN>::T + tid; }

template <int LOGN>
DI int spectral_index(int tid, int e) {
  using G = NttGeom<LOGN>;
  return pass_index<LOGN, G::lo(G::NPASS - 1), G::kb(G::NPASS - 1)>(tid, e);
}

// Forward negacyclic NTT: natural layout in (any values < 4p), spectral layout
// out, fully reduced to [0, p).
template <int LOGN>
DI void ntt_fwd(uint32_t* x, uint32_t* s, const uint2* __restrict__ tw, uint32_t p, int tid) {
  fwd_from<LOGN, 0>(x, s, tw, p, tid);
  const uint32_t p2 = 2 * p;
#pragma unroll
  for (int e = 0; e < NttGeom<LOGN>::E; ++e) {
    uint32_t v = x[e];
    v = v >= p2 ? v - p2 : v;
    x[e] = v >= p ? v - p : v;
  }
}

// Inverse negacyclic NTT: spectral layout in (values < 2p), natural layout out,
// times N^-1, reduced to [0, p).
template <int LOGN>
DI void ntt_inv(uint32_t* x, uint32_t* s, const uint2* __restrict__ itw, uint32_t p, uint2 ninv,
                int tid) {
  inv_from<LOGN, NttGeom<LOGN>::NPASS - 1>(x, s, itw, p, tid);
#pragma unroll
  for (int e = 0; e < NttGeom<LOGN>::E; ++e) x[e] = mul_shoup(x[e], ninv.x, ninv.y, p);
}

}  // namespace hcnn
