// NTT-based kernels, templated on the NTT geometry G = NttGeom<LOGN, LOGE>
// (ntt.cuh); one translation unit per ring degree (ntt_inst.cu, compiled with
// -DHCNN_LOGN=L) keeps the build parallel.
//
//   k_ntt_rows      standalone forward / inverse NTT of RNS rows (ring.py:147-163)
//   k_tensor        ct x ct tensor over Q u P: NTT, pointwise, INTT (bfv.py:331-347)
//   k_relin         digit NTT x rlk MAC, INTT, + (y0, y1)          (bfv.py:368-404)
//   k_encrypt       public-key encryption from host randomness     (bfv.py:201-216)
//   k_mul_plain     ct x plaintext polynomial, NTT path           (bfv.py:301-318)
//   k_ref_to_tiled  reference-order NTT keys -> device tiled layout
#pragma once
#include <atomic>
#include <type_traits>

#include "common.cuh"
#include "ntt.cuh"
#include "ntt_cluster.cuh"
#include "tma.cuh"

namespace hcnn {

struct NttLaunch {
  cudaStream_t stream;
  dim3 grid;
  NttTabs nt;
  int variant;  // geometry flags of the fused kernels (RELIN_SINGLE, TENSOR_MIXED, MIXED_PASSES)
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
  // relinearisation over R
  RbTabs rb;
};

template <class G>
DI void load_natural(uint32_t* x, const uint32_t* __restrict__ row, int tid) {
#pragma unroll
  for (int e = 0; e < G::E; ++e) x[e] = row[natural_index<G>(tid, e)];
}

template <class G>
DI void inv_store(uint32_t* x, uint32_t* s, const uint2* itw, uint32_t p, const InvScale& ninv, int tid,
                  uint32_t* __restrict__ row) {
  ntt_inv<G>(x, s, itw, p, ninv, tid);
#pragma unroll
  for (int e = 0; e < G::E; ++e) row[natural_index<G>(tid, e)] = x[e];
}

// in place on [rows][N]; row r uses prime prime_off + r % limbs.
// inverse: 0 forward (spectral positions), 1 inverse, 2 forward to tiled layout
// The spectral positions a thread holds are scattered (pairs of words 128 B
// apart), so spectral rows cross shared memory once: read or written there
// in the spectral pattern, moved to / from global memory in natural
// (coalesced) order.  Up to 512 threads two CTAs share an SM (one row's
// loads and stores overlap the other's butterflies).
template <class G>
__global__ void __launch_bounds__(G::T, (G::T <= 512 ? 2 : 1))
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
    for (int e = 0; e < G::E; ++e) s[sidx(natural_index<G>(tid, e))] = r[natural_index<G>(tid, e)];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < G::E; ++e) x[e] = s[sidx(spectral_index<G>(tid, e))];
    __syncthreads();
    ntt_inv<G>(x, s, nt.itw + (size_t)j * G::N, p, inv_scale(nt, j, false), tid);
#pragma unroll
    for (int e = 0; e < G::E; ++e) r[natural_index<G>(tid, e)] = x[e];
    return;
  }
  load_natural<G>(x, r, tid);
  ntt_fwd<G>(x, s, nt.tw + (size_t)j * G::N, p, tid);
  __syncthreads();
  if (inverse == 2) {
    store_tiled<G>(x, r, tid);
  } else {
#pragma unroll
    for (int e = 0; e < G::E; ++e) s[sidx(spectral_index<G>(tid, e))] = x[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < G::E; ++e) r[natural_index<G>(tid, e)] = s[sidx(natural_index<G>(tid, e))];
  }
}

// Persistent rows (forward and inverse): each CTA walks rows r = blockIdx.x,
// + gridDim.x, ...; the next row streams into a shared-memory stage by one TMA
// bulk copy while the current one is transformed, so no row starts with an
// exposed HBM load.  Spectral rows cross the padded exchange buffer once
// (scattered pairs of words would conflict in the raw stage / uncoalesce in
// HBM).  Same results as k_ntt_rows.
template <class G>
constexpr int rows_pf_smem_words() { return G::ntt_smem_words(1) + G::N; }

template <class G>
__global__ void __launch_bounds__(G::T, 1)
    k_ntt_rows_pf(uint32_t* __restrict__ data, int n_rows, int limbs, int prime_off, int inverse, NttTabs nt) {
  extern __shared__ __align__(16) uint32_t s[];
  __shared__ __align__(8) uint64_t bar;
  constexpr int E = G::E;
  const int tid = threadIdx.x;
  uint32_t* stage = s + G::ntt_smem_words(1);
  auto fetch = [&](int r) {
    fence_proxy_async();
    mbar_expect_tx(&bar, G::N * 4);
    bulk_g2s(stage, data + (size_t)r * G::N, G::N * 4, &bar);
  };
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  int row = blockIdx.x;
  if (tid == 0 && row < n_rows) fetch(row);
  uint32_t phase = 0;
#pragma unroll 1
  for (; row < n_rows; row += gridDim.x) {
    const int j = prime_off + row % limbs;
    const uint32_t p = nt.prime[j];
    uint32_t* r = data + (size_t)row * G::N;
    uint32_t x[E];
    mbar_wait(&bar, phase);
    phase ^= 1;
    if (inverse) {
#pragma unroll
      for (int e = 0; e < E; ++e) s[sidx(natural_index<G>(tid, e))] = stage[natural_index<G>(tid, e)];
      __syncthreads();
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = s[sidx(spectral_index<G>(tid, e))];
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = stage[natural_index<G>(tid, e)];
    }
    __syncthreads();  // the stage and the exchange buffers are free
    if (tid == 0 && row + (int)gridDim.x < n_rows) fetch(row + gridDim.x);
    if (inverse) {
      ntt_inv<G>(x, s, nt.itw + (size_t)j * G::N, p, inv_scale(nt, j, false), tid);
#pragma unroll
      for (int e = 0; e < E; ++e) r[natural_index<G>(tid, e)] = x[e];
    } else {
      ntt_fwd<G>(x, s, nt.tw + (size_t)j * G::N, p, tid);
      __syncthreads();
#pragma unroll
      for (int e = 0; e < E; ++e) s[sidx(spectral_index<G>(tid, e))] = x[e];
      __syncthreads();
#pragma unroll
      for (int e = 0; e < E; ++e) r[natural_index<G>(tid, e)] = s[sidx(natural_index<G>(tid, e))];
    }
  }
}

// Transforms of two rows x[0, E) and x[E, 2E): in lockstep when the
// geometry's shared memory allows, else one after the other.
template <class G>
__host__ __device__ constexpr int pair_nr() { return G::E < 32 && G::fits(2) ? 2 : 1; }

template <class G, bool FULL = true>
DI void ntt_fwd_pair(uint32_t* x, uint32_t* s, const uint2* tw, uint32_t p, int tid) {
  if constexpr (pair_nr<G>() == 2) {
    ntt_fwd<G, 2, FULL>(x, s, tw, p, tid);
  } else {
    ntt_fwd<G, 1, FULL>(x, s, tw, p, tid);
    ntt_fwd<G, 1, FULL>(x + G::E, s, tw, p, tid);
  }
}

template <class G>
DI void ntt_inv_pair(uint32_t* x, uint32_t* s, const uint2* itw, uint32_t p, const InvScale& ninv, int tid) {
  if constexpr (pair_nr<G>() == 2) {
    ntt_inv<G, 2>(x, s, itw, p, ninv, tid);
  } else {
    ntt_inv<G>(x, s, itw, p, ninv, tid);
    ntt_inv<G>(x + G::E, s, itw, p, ninv, tid);
  }
}

// TMEM as per-thread stash (no tensor-core use): warp w owns lanes
// 32 (w % 4) + [0, 32) and columns W (w / 4) + [0, W) of the CTA's allocation
// (W = 2E for the relinearisation sums, E for the tensor's parked row).
template <class G, int W>
__host__ __device__ constexpr uint32_t tmem_stash_cols() {
  return W * (G::T / 128) <= 128 ? 128 : W * (G::T / 128) <= 256 ? 256 : 512;
}

DI void tmem_alloc_cols(uint32_t* slot, uint32_t cols) {
  if (cols == 128)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(slot)) : "memory");
  else if (cols == 256)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(slot)) : "memory");
  else
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

DI void tmem_dealloc_cols(uint32_t base, uint32_t cols) {
  if (cols == 128) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(base) : "memory");
  else if (cols == 256) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(base) : "memory");
  else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base) : "memory");
}

template <int E>
DI void tmem_st_row(uint32_t taddr, const uint32_t* v) {
#pragma unroll
  for (int c = 0; c < E / 16; ++c) tmem_st16(taddr + 16 * c, v + 16 * c);
}

template <int E>
DI void tmem_ld_row(uint32_t taddr, uint32_t* v) {
#pragma unroll
  for (int c = 0; c < E / 16; ++c) tmem_ld16(taddr + 16 * c, v + 16 * c);
}

DI uint32_t tmem_stash_alloc(uint32_t* slot, uint32_t cols, int tid, int width) {
  const int warp = tid >> 5;
  if (warp == 0) tmem_alloc_cols(slot, cols);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  return *slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(warp >> 2) * width;
}

DI void tmem_stash_free(uint32_t base, uint32_t cols, int tid) {
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if ((tid >> 5) == 0) tmem_dealloc_cols(base, cols);
}

// One CTA per (ct, prime of Q u P).  a/b: [B][2][K][N]; ae/be: [B][2][KP][N]
// (exact extensions); d: [B][3][K+KP][N] exact tensor parts, coefficient domain.
// The four (two for a square) forward transforms run as row pairs and the
// inverse of d0, d1 as a pair, sharing twiddle loads and barriers.
// TM (E = 16, squares only): one row in registers at a time, A0 and then
// d1, d2 parked in TMEM (flag TENSOR_TMEM).
template <class G, int TM = 0>
__global__ void __launch_bounds__(G::T, (G::T <= 256 ? 2 : 1))
    k_tensor(const uint32_t* __restrict__ a, const uint32_t* __restrict__ a_ext,
             const uint32_t* __restrict__ b, const uint32_t* __restrict__ b_ext,
             uint32_t* __restrict__ d, int K, int KP, int square, NttTabs nt) {
  extern __shared__ uint32_t s[];
  constexpr int E = G::E;
  static_assert(TM == 0 || E % 16 == 0, "TMEM stash: rows of 16-column chunks");
  const int tid = threadIdx.x;
  const int j = blockIdx.x;
  const size_t ct = blockIdx.y;
  const int L = K + KP;
  const uint32_t p = nt.prime[j];
  const uint2* tw = nt.tw + (size_t)j * G::N;
  const uint2* itw = nt.itw + (size_t)j * G::N;
  auto row_of = [&](const uint32_t* base, const uint32_t* ext, int part) -> const uint32_t* {
    return j < K ? base + ((ct * 2 + part) * K + j) * G::N
                 : ext + ((ct * 2 + part) * KP + (j - K)) * G::N;
  };
  uint32_t* o0 = d + ((ct * 3 + 0) * L + j) * G::N;
  uint32_t* o1 = d + ((ct * 3 + 1) * L + j) * G::N;
  uint32_t* o2 = d + ((ct * 3 + 2) * L + j) * G::N;
  // pointwise products are Montgomery products (x y 2^-32, in [0, 2p)); the
  // inverse transforms multiply by N^-1 2^32 instead of N^-1
  const uint32_t pinv = nt.pinv[j];
  const uint32_t p2 = 2 * p;
  const InvScale ninv = inv_scale(nt, j, true);
  if constexpr (TM == 2) {
    // square only: A0, A1 transformed as a pair, d2 parked in TMEM while d0,
    // d1 go through their inverse pair
    __shared__ uint32_t tmem_slot2;
    constexpr uint32_t COLS = tmem_stash_cols<G, E>();
    const uint32_t tp = tmem_stash_alloc(&tmem_slot2, COLS, tid, E);
    uint32_t x[2 * E];
    load_natural<G>(x, row_of(a, a_ext, 0), tid);
    load_natural<G>(x + E, row_of(a, a_ext, 1), tid);
    ntt_fwd_pair<G, false>(x, s, tw, p, tid);
    {
      uint32_t t[E];
#pragma unroll
      for (int e = 0; e < E; ++e) t[e] = mont_mul(x[E + e], x[E + e], p, pinv);
      tmem_st_row<E>(tp, t);  // d2
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t a0 = x[e], a1 = x[E + e];
      const uint32_t c = mont_mul(a0, a1, p, pinv);
      x[e] = mont_mul(a0, a0, p, pinv);
      x[E + e] = umin32(2 * c, 2 * c - p2);
    }
    ntt_inv_pair<G>(x, s, itw, p, ninv, tid);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      o0[natural_index<G>(tid, e)] = x[e];
      o1[natural_index<G>(tid, e)] = x[E + e];
    }
    tmem_ld_row<E>(tp, x);
    tmem_stash_free(tmem_slot2, COLS, tid);
    inv_store<G>(x, s, itw, p, ninv, tid, o2);
  } else if constexpr (TM == 1) {
    // square only (the dispatch sends general products to TM = 0): the
    // transforms run one row at a time and the waiting rows sit in TMEM
    __shared__ uint32_t tmem_slot;
    constexpr uint32_t COLS = tmem_stash_cols<G, 2 * E>();
    const uint32_t tp = tmem_stash_alloc(&tmem_slot, COLS, tid, 2 * E);
    uint32_t x[E];
    // rolled loops: one copy of each transform's code (five inlined
    // transforms would hoist enough addressing to spill at 64 registers)
#pragma unroll 1
    for (int r = 0; r < 2; ++r) {
      load_natural<G>(x, row_of(a, a_ext, r), tid);
      ntt_fwd<G, 1, false>(x, s, tw, p, tid);
      if (r == 0) tmem_st_row<E>(tp, x);  // A0
    }
    {  // x = A1
      uint32_t a0[E], t[E];
      tmem_ld_row<E>(tp, a0);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint32_t c = mont_mul(a0[e], x[e], p, pinv);
        t[e] = umin32(2 * c, 2 * c - p2);
      }
      tmem_st_row<E>(tp, t);  // d1
#pragma unroll
      for (int e = 0; e < E; ++e) t[e] = mont_mul(x[e], x[e], p, pinv);
      tmem_st_row<E>(tp + E, t);  // d2
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = mont_mul(a0[e], a0[e], p, pinv);  // d0
    }
#pragma unroll 1
    for (int r = 0; r < 3; ++r) {
      if (r > 0) tmem_ld_row<E>(tp + (r - 1) * E, x);
      inv_store<G>(x, s, itw, p, ninv, tid, r == 0 ? o0 : r == 1 ? o1 : o2);
    }
    tmem_stash_free(tmem_slot, COLS, tid);
  } else {
  uint32_t x[2 * E], y[2 * E];
  if (square) {
    // x = (A0 | A1)
    load_natural<G>(x, row_of(a, a_ext, 0), tid);
    load_natural<G>(x + E, row_of(a, a_ext, 1), tid);
    ntt_fwd_pair<G, false>(x, s, tw, p, tid);  // [0, 2p): products < 4p^2 < 2^32 p
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t a0 = x[e], a1 = x[E + e];
      const uint32_t c = mont_mul(a0, a1, p, pinv);
      x[e] = mont_mul(a0, a0, p, pinv);
      x[E + e] = umin32(2 * c, 2 * c - p2);
      y[e] = mont_mul(a1, a1, p, pinv);
    }
  } else {
    // x = (A0 | B0), y = (A1 | B1)
    load_natural<G>(x, row_of(a, a_ext, 0), tid);
    load_natural<G>(x + E, row_of(b, b_ext, 0), tid);
    ntt_fwd_pair<G>(x, s, tw, p, tid);
    load_natural<G>(y, row_of(a, a_ext, 1), tid);
    load_natural<G>(y + E, row_of(b, b_ext, 1), tid);
    ntt_fwd_pair<G>(y, s, tw, p, tid);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t a0 = x[e], b0 = x[E + e], a1 = y[e], b1 = y[E + e];
      x[e] = mont_mul(a0, b0, p, pinv);
      // a0 b1 + a1 b0 < 2 p^2 < 2^32 p: one reduction
      x[E + e] = redc64((uint64_t)a0 * b1 + (uint64_t)a1 * b0, p, pinv);
      y[e] = mont_mul(a1, b1, p, pinv);
    }
  }
  ntt_inv_pair<G>(x, s, itw, p, ninv, tid);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    o0[natural_index<G>(tid, e)] = x[e];
    o1[natural_index<G>(tid, e)] = x[E + e];
  }
  inv_store<G>(y, s, itw, p, ninv, tid, o2);
  }  // !TM
}

// Persistent square tensor (flag TENSOR_PERSIST): one CTA per SM walks the
// (ct, prime) items; the two input rows of the NEXT item stream into shared
// memory by TMA bulk copies while the current item computes, so no CTA starts
// with an exposed HBM load.  Same arithmetic as k_tensor's square path.
template <class G>
constexpr int tensor_pf_smem_words() { return G::ntt_smem_words(pair_nr<G>()) + 2 * G::N; }

// the persistent square tensor's three inverses as one lockstep transform
// (its exchange buffers fit inside the pair transform's)
template <class G>
__host__ __device__ constexpr bool tensor_nr3() {
  return G::E == 16 && !G::MIXED && G::ntt_smem_words(3) <= G::ntt_smem_words(pair_nr<G>());
}

template <class G>
__global__ void __launch_bounds__(G::T, 1)
    k_tensor_sq_pf(const uint32_t* __restrict__ a, const uint32_t* __restrict__ a_ext,
                   uint32_t* __restrict__ d, int K, int KP, int n_items, NttTabs nt) {
  extern __shared__ __align__(16) uint32_t s[];
  __shared__ __align__(8) uint64_t bar;
  constexpr int E = G::E;
  const int tid = threadIdx.x;
  const int L = K + KP;
  uint32_t* stage = s + G::ntt_smem_words(pair_nr<G>());
  auto row_of = [&](int item, int part) -> const uint32_t* {
    const size_t ct = item / L;
    const int j = item % L;
    return j < K ? a + ((ct * 2 + part) * K + j) * G::N : a_ext + ((ct * 2 + part) * KP + (j - K)) * G::N;
  };
  auto fetch = [&](int item) {
    fence_proxy_async();
    mbar_expect_tx(&bar, 2 * G::N * 4);
    bulk_g2s(stage, row_of(item, 0), G::N * 4, &bar);
    bulk_g2s(stage + G::N, row_of(item, 1), G::N * 4, &bar);
  };
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  int item = blockIdx.x;
  if (tid == 0 && item < n_items) fetch(item);
  uint32_t phase = 0;
#pragma unroll 1
  for (; item < n_items; item += gridDim.x) {
    const size_t ct = item / L;
    const int j = item % L;
    const uint32_t p = nt.prime[j];
    const uint32_t pinv = nt.pinv[j];
    const uint32_t p2 = 2 * p;
    const uint2* tw = nt.tw + (size_t)j * G::N;
    const uint2* itw = nt.itw + (size_t)j * G::N;
    const InvScale ninv = inv_scale(nt, j, true);
    mbar_wait(&bar, phase);
    phase ^= 1;
    uint32_t x[2 * E], y[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      x[e] = stage[natural_index<G>(tid, e)];
      x[E + e] = stage[G::N + natural_index<G>(tid, e)];
    }
    __syncthreads();  // every thread has read the stage
    if (tid == 0 && item + (int)gridDim.x < n_items) fetch(item + gridDim.x);
    ntt_fwd_pair<G, false>(x, s, tw, p, tid);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t a0 = x[e], a1 = x[E + e];
      const uint32_t c = mont_mul(a0, a1, p, pinv);
      x[e] = mont_mul(a0, a0, p, pinv);
      x[E + e] = umin32(2 * c, 2 * c - p2);
      y[e] = mont_mul(a1, a1, p, pinv);
    }
    if constexpr (tensor_nr3<G>()) {
    // the three inverses in lockstep (shared twiddle loads and barriers,
    // single-buffered exchanges; at 2^13 this also removes the pair version's
    // 192-byte register spill)
    uint32_t z[3 * E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      z[e] = x[e];
      z[E + e] = x[E + e];
      z[2 * E + e] = y[e];
    }
    ntt_inv<G, 3>(z, s, itw, p, ninv, tid);
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      uint32_t* o = d + ((ct * 3 + r) * L + j) * G::N;
#pragma unroll
      for (int e = 0; e < E; ++e) o[natural_index<G>(tid, e)] = z[r * E + e];
    }
    } else {
    ntt_inv_pair<G>(x, s, itw, p, ninv, tid);
    uint32_t* o0 = d + ((ct * 3 + 0) * L + j) * G::N;
    uint32_t* o1 = d + ((ct * 3 + 1) * L + j) * G::N;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      o0[natural_index<G>(tid, e)] = x[e];
      o1[natural_index<G>(tid, e)] = x[E + e];
    }
    inv_store<G>(y, s, itw, p, ninv, tid, d + ((ct * 3 + 2) * L + j) * G::N);
    }
  }
}

// Plaintext-polynomial product (bfv.py:301-318, NTT path): one CTA per (ct,
// prime of q); a: [B][2][K][N]; pt: [K][N] NTT domain, tiled layout (plain
// form; the Montgomery 2^-32 is undone by the N^-1 2^32 of the inverse).
template <class G>
__global__ void __launch_bounds__(G::T, (G::T <= 256 ? 2 : 1))
    k_mul_plain(const uint32_t* __restrict__ a, const uint32_t* __restrict__ pt,
                uint32_t* __restrict__ out, int K, NttTabs nt) {
  extern __shared__ uint32_t s[];
  constexpr int E = G::E;
  const int tid = threadIdx.x;
  const int j = blockIdx.x;
  const size_t ct = blockIdx.y;
  const uint32_t p = nt.prime[j];
  const uint32_t pinv = nt.pinv[j];
  uint32_t x[2 * E];
  load_natural<G>(x, a + ((ct * 2 + 0) * K + j) * G::N, tid);
  load_natural<G>(x + E, a + ((ct * 2 + 1) * K + j) * G::N, tid);
  ntt_fwd_pair<G, false>(x, s, nt.tw + (size_t)j * G::N, p, tid);  // [0, 2p) feeds Montgomery products
  {
    uint32_t k[E];
    load_tiled<G>(k, pt + (size_t)j * G::N, tid);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      x[e] = mont_mul(x[e], k[e], p, pinv);
      x[E + e] = mont_mul(x[E + e], k[e], p, pinv);
    }
  }
  ntt_inv_pair<G>(x, s, nt.itw + (size_t)j * G::N, p, inv_scale(nt, j, true), tid);
#pragma unroll
  for (int part = 0; part < 2; ++part) {
    uint32_t* o = out + ((ct * 2 + part) * K + j) * G::N;
#pragma unroll
    for (int e = 0; e < E; ++e) o[natural_index<G>(tid, e)] = x[part * E + e];
  }
}

// Square tensor for MIXED geometries (T = N/32 threads; two CTAs per SM up to
// N = 8192, 128 registers per thread above): one
// row in registers at a time; A0 and then d0, d1 wait in shared memory
// (thread-owned slots e*T + tid) behind the single exchange buffer.
template <class G>
constexpr int tensor_sq_smem_words() { return G::ntt_smem_words(1) + 2 * G::N; }

template <class G>
__global__ void __launch_bounds__(G::T, (G::T <= 256 ? 2 : 1))
    k_tensor_sq(const uint32_t* __restrict__ a, const uint32_t* __restrict__ a_ext,
                uint32_t* __restrict__ d, int K, int KP, NttTabs nt) {
  extern __shared__ __align__(16) uint32_t s[];
  constexpr int E = G::E;
  const int tid = threadIdx.x;
  const int j = blockIdx.x;
  const size_t ct = blockIdx.y;
  const int L = K + KP;
  const uint32_t p = nt.prime[j];
  const uint32_t pinv = nt.pinv[j];
  const uint32_t p2 = 2 * p;
  const uint2* tw = nt.tw + (size_t)j * G::N;
  const uint2* itw = nt.itw + (size_t)j * G::N;
  const InvScale ninv = inv_scale(nt, j, true);
  uint32_t* st0 = s + G::ntt_smem_words(1);
  uint32_t* st1 = st0 + G::N;
  auto row_of = [&](int part) -> const uint32_t* {
    return j < K ? a + ((ct * 2 + part) * K + j) * G::N : a_ext + ((ct * 2 + part) * KP + (j - K)) * G::N;
  };
  uint32_t x[E];
  load_natural<G>(x, row_of(0), tid);
  ntt_fwd<G>(x, s, tw, p, tid);
#pragma unroll
  for (int e = 0; e < E; ++e) st0[e * G::T + tid] = x[e];
  load_natural<G>(x, row_of(1), tid);
  ntt_fwd<G>(x, s, tw, p, tid);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t a0 = st0[e * G::T + tid], a1 = x[e];
    const uint32_t c = mont_mul(a0, a1, p, pinv);
    st0[e * G::T + tid] = mont_mul(a0, a0, p, pinv);
    st1[e * G::T + tid] = umin32(2 * c, 2 * c - p2);
    x[e] = mont_mul(a1, a1, p, pinv);
  }
  inv_store<G>(x, s, itw, p, ninv, tid, d + ((ct * 3 + 2) * L + j) * G::N);
#pragma unroll
  for (int e = 0; e < E; ++e) x[e] = st0[e * G::T + tid];
  inv_store<G>(x, s, itw, p, ninv, tid, d + ((ct * 3 + 0) * L + j) * G::N);
#pragma unroll
  for (int e = 0; e < E; ++e) x[e] = st1[e * G::T + tid];
  inv_store<G>(x, s, itw, p, ninv, tid, d + ((ct * 3 + 1) * L + j) * G::N);
}

// Relinearisation configuration of a geometry: NR digit rows transformed in
// lockstep, and the accumulator form: lazy u64 (plain keys) while the
// registers allow, else u32 fed by Montgomery products (keys uploaded in
// Montgomery form).  single selects the one-row kernel (variant flag).
template <class G>
__host__ __device__ constexpr int relin_nr(bool single) { return single ? 1 : pair_nr<G>(); }

template <class G>
__host__ __device__ constexpr bool relin_acc64(bool single) { return relin_nr<G>(single) * G::E <= 16 && G::T <= 512; }

// Shared-memory plan of k_relin: [NTT exchange buffers][STAGES groups of NR
// digit rows streamed in by TMA bulk copies one group ahead][mbarriers]
template <class G, int NR>
struct RelinSmem {
  static constexpr int LIMIT = 220 * 1024;
  static constexpr int BASE = G::ntt_smem_words(NR);
  static constexpr int STAGE_WORDS = NR * G::N;
  static constexpr int STAGES = (BASE + 2 * STAGE_WORDS) * 4 <= LIMIT ? 2
                                : ((BASE + STAGE_WORDS) * 4 <= LIMIT ? 1 : 0);
  static constexpr int BYTES = (BASE + STAGES * STAGE_WORDS) * 4 + 16 * 2;
};

// One CTA per (ct, prime of q).  dig: [B][D][N] base-w digits of c2;
// y3: [B][3][K][N] scaled parts (0 and 1 used); rlk: [D][2][K][N] NTT domain,
// tiled layout (ntt.cuh), Montgomery form unless ACC64;
// out: [B][2][K][N] = (y0 + sum_i D_i k0_i, y1 + sum_i D_i k1_i).
// Digits go through the forward NTT NR at a time (a single one first when the
// count is odd); ACC64: lazy 64-bit accumulators (reduced before 16 products
// pile up); otherwise u32 accumulators in [0, 2p) fed by Montgomery products.
// TM: the running sums live in TMEM instead of registers (E = 16: one
// 32x32b.x16 load / store per part and digit group; warp w uses lanes
// 32 (w % 4) + lane and columns 2E (w / 4) + [0, 2E)).
template <class G, bool ACC64, int NR, bool TM = false>
__global__ void __launch_bounds__(G::T, (G::T <= 256 ? 2 : 1))
    k_relin(const uint32_t* __restrict__ dig, const uint32_t* __restrict__ y3,
            const uint32_t* __restrict__ rlk, uint32_t* __restrict__ out, int K, int D,
            int reduce_digits, NttTabs nt) {
  using SM = RelinSmem<G, NR>;
  constexpr int E = G::E;
  static_assert(!TM || (E == 16 && !ACC64), "TMEM running sums: E = 16, Montgomery accumulators");
  extern __shared__ __align__(16) uint32_t s[];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x;
  const int j = blockIdx.x;
  const size_t ct = blockIdx.y;
  const uint32_t p = nt.prime[j];
  const uint64_t mu = nt.mu[j];
  const uint32_t pinv = nt.pinv[j];
  const uint32_t p2 = 2 * p;
  const uint2* tw = nt.tw + (size_t)j * G::N;
  using Acc = typename std::conditional<ACC64, uint64_t, uint32_t>::type;
  Acc acc0[TM ? 1 : E], acc1[TM ? 1 : E];
  uint32_t tacc = 0;
  if constexpr (TM) {
    tacc = tmem_stash_alloc(&tmem_slot, tmem_stash_cols<G, 2 * G::E>(), tid, 2 * E);
    uint32_t z[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) z[e] = 0;
    tmem_st16(tacc, z);
    tmem_st16(tacc + E, z);
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) acc0[e] = acc1[e] = 0;
  }

  const uint32_t* dig_ct = dig + ct * D * G::N;
  auto krow = [&](int i, int part) { return rlk + ((size_t)(i * 2 + part) * K + j) * G::N; };
  // rows in the group starting at digit i
  auto group_rows = [&](int i) { return (NR == 2 && ((D - i) & 1)) ? 1 : NR; };
  uint32_t* stage0 = s + SM::BASE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stage0 + SM::STAGES * SM::STAGE_WORDS);
  auto issue = [&](int i, int g) {  // elected thread: group g (from digit i) into its stage
    constexpr int NS = SM::STAGES > 0 ? SM::STAGES : 1;
    uint64_t* bar = &bars[g % NS];
    const uint32_t bytes = (uint32_t)group_rows(i) * G::N * 4;
    fence_proxy_async();
    mbar_expect_tx(bar, bytes);
    bulk_g2s(stage0 + (g % NS) * SM::STAGE_WORDS, dig_ct + (size_t)i * G::N, bytes, bar);
  };
  // y0, y1 (added after the inverse) follow the last digit group into the
  // stage it frees, so the epilogue does not wait on HBM
  constexpr bool Y3PF = SM::STAGES == 2 && NR == 2;
  auto issue_y3 = [&](int g) {
    uint64_t* bar = &bars[g % 2];
    uint32_t* dst = stage0 + (g % 2) * SM::STAGE_WORDS;
    fence_proxy_async();
    mbar_expect_tx(bar, 2 * G::N * 4);
    bulk_g2s(dst, y3 + ((ct * 3 + 0) * K + j) * G::N, G::N * 4, bar);
    bulk_g2s(dst + G::N, y3 + ((ct * 3 + 1) * K + j) * G::N, G::N * 4, bar);
  };
  if constexpr (SM::STAGES > 0) {
    if (tid == 0) {
      for (int st = 0; st < SM::STAGES; ++st) mbar_init(&bars[st], 1);
      fence_mbar_init();
      issue(0, 0);
    }
    __syncthreads();
  }

  int pending = 0;  // ACC64: products accumulated since the last reduction
  auto step = [&](auto rows_c, int i, int g) {
    constexpr int R = decltype(rows_c)::value;
    uint32_t x[R * E];
    if constexpr (SM::STAGES > 0) {
      // with two stages, group g+1 streams in while group g is transformed;
      // its buffer was last read before this thread's previous-group barriers
      if constexpr (SM::STAGES == 2) {
        if (tid == 0) {
          if (i + R < D) issue(i + R, g + 1);
          else if constexpr (Y3PF) issue_y3(g + 1);  // the free stage takes y0, y1
        }
      }
      const uint32_t* row = stage0 + (g % SM::STAGES) * SM::STAGE_WORDS;
      mbar_wait(&bars[g % SM::STAGES], (uint32_t)(g / SM::STAGES) & 1);
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int e = 0; e < E; ++e) x[r * E + e] = row[r * G::N + natural_index<G>(tid, e)];
      if constexpr (SM::STAGES == 1) {
        __syncthreads();
        if (tid == 0 && i + R < D) issue(i + R, g + 1);
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) load_natural<G>(x + r * E, dig_ct + (size_t)(i + r) * G::N, tid);
    }
    if (reduce_digits) {
#pragma unroll
      for (int e = 0; e < R * E; ++e) x[e] = reduce64(x[e], p, mu);
    }
    // Montgomery MACs take the digit spectra in [0, 2p) (paired sums < 4p^2 < 2^32 p)
    ntt_fwd<G, R, ACC64>(x, s, tw, p, tid);
    if constexpr (!ACC64 && R == 2) {
      // both digits' products summed in 64 bits (< 2 p^2 < 2^32 p), one
      // Montgomery reduction per pair; keys streamed 16 bytes at a time
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        uint32_t ta[TM ? E : 1];
        if constexpr (TM) tmem_ld16(tacc + part * E, ta);
        const uint4* k0 = reinterpret_cast<const uint4*>(krow(i, part)) + tid;
        const uint4* k1 = reinterpret_cast<const uint4*>(krow(i + 1, part)) + tid;
#pragma unroll
        for (int c = 0; c < E / 4; ++c) {
          const uint4 u = __ldg(&k0[c * G::T]);
          const uint4 v = __ldg(&k1[c * G::T]);
          const uint32_t ku[4] = {u.x, u.y, u.z, u.w}, kv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int l = 0; l < 4; ++l) {
            const int e = 4 * c + l;
            const uint32_t m = redc64((uint64_t)x[e] * ku[l] + (uint64_t)x[E + e] * kv[l], p, pinv);
            if constexpr (TM) {
              const uint32_t sum = ta[e] + m;
              ta[e] = umin32(sum, sum - p2);
            } else {
              Acc* acc = part ? acc1 : acc0;
              const uint32_t sum = (uint32_t)acc[e] + m;
              acc[e] = umin32(sum, sum - p2);
            }
          }
        }
        if constexpr (TM) tmem_st16(tacc + part * E, ta);
      }
    } else {
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        uint32_t k[E];
        load_tiled<G>(k, krow(i + r, part), tid);
        if constexpr (TM) {
          uint32_t ta[E];
          tmem_ld16(tacc + part * E, ta);
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const uint32_t v = ta[e] + mont_mul(x[r * E + e], k[e], p, pinv);
            ta[e] = umin32(v, v - p2);
          }
          tmem_st16(tacc + part * E, ta);
        } else {
          Acc* acc = part ? acc1 : acc0;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            if constexpr (ACC64) {
              acc[e] += (uint64_t)x[r * E + e] * k[e];
            } else {
              const uint32_t v = acc[e] + mont_mul(x[r * E + e], k[e], p, pinv);
              acc[e] = umin32(v, v - p2);
            }
          }
        }
      }
    }
    }
    if constexpr (ACC64) {
      // a reduced value plus 16 products of (p-1)^2 stays below 2^64
      pending += R;
      if (pending + NR > 16) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          acc0[e] = reduce64(acc0[e], p, mu);
          acc1[e] = reduce64(acc1[e], p, mu);
        }
        pending = 0;
      }
    }
  };
  int ngroups = 0;
  for (int i = 0; i < D; ++ngroups) {
    const int R = group_rows(i);
    if (NR == 2 && R == 2) {
      step(std::integral_constant<int, NR>(), i, ngroups);
    } else {
      step(std::integral_constant<int, 1>(), i, ngroups);
      // a one-row transform's last exchange buffer overlaps the two-row one's first
      if constexpr (NR == 2) __syncthreads();
    }
    i += R;
  }
  const uint2* itw = nt.itw + (size_t)j * G::N;
  const InvScale ninv = inv_scale(nt, j, false);
  // both parts through the inverse (in lockstep when NR = 2)
  uint32_t x[2 * E];
  if constexpr (TM) {
    tmem_ld16(tacc, x);
    tmem_ld16(tacc + E, x + E);
    tmem_stash_free(tmem_slot, tmem_stash_cols<G, 2 * G::E>(), tid);
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if constexpr (ACC64) {
        x[e] = reduce64(acc0[e], p, mu);
        x[E + e] = reduce64(acc1[e], p, mu);
      } else {  // in [0, 2p): valid inverse input
        x[e] = acc0[e];
        x[E + e] = acc1[e];
      }
    }
  }
  if constexpr (NR == 2) {
    ntt_inv<G, 2>(x, s, itw, p, ninv, tid);
  } else {
    ntt_inv<G>(x, s, itw, p, ninv, tid);
    ntt_inv<G>(x + E, s, itw, p, ninv, tid);
  }
  if constexpr (Y3PF) {
    if (ngroups > 0) {
      mbar_wait(&bars[ngroups % 2], (uint32_t)(ngroups / 2) & 1);
      const uint32_t* yst = stage0 + (ngroups % 2) * SM::STAGE_WORDS;
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        uint32_t* o = out + ((ct * 2 + part) * K + j) * G::N;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int idx = natural_index<G>(tid, e);
          o[idx] = add_mod(x[part * E + e], yst[part * G::N + idx], p);
        }
      }
      return;
    }
  }
#pragma unroll
  for (int part = 0; part < 2; ++part) {
    const uint32_t* yr = y3 + ((ct * 3 + part) * K + j) * G::N;
    uint32_t* o = out + ((ct * 2 + part) * K + j) * G::N;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int idx = natural_index<G>(tid, e);
      o[idx] = add_mod(x[part * E + e], yr[idx], p);
    }
  }
}

// ------------------------------------------- relinearisation over R (RbTabs)
// geometries with the R kernels: radix-16 shuffle tail, 256-512 threads
template <class G>
__host__ __device__ constexpr bool rb_geom() {
  return G::E == 16 && !G::MIXED && G::LOGN >= 12 && G::LOGN <= 13 && G::fits(2);
}
// 1024-thread geometries (N = 2^14, 64 registers): one-row variants
template <class G>
__host__ __device__ constexpr bool rb_geom1() {
  return G::E == 16 && G::T == 1024 && G::LOGN == 14 && (G::ntt_smem_words(1) + G::N) * 4 <= 220 * 1024;
}

// Step 1 of 3 (bfv.py:368-404 restated over the basis R, common.cuh).  One
// CTA per (r_a, ct): the D digit rows of c2 through the forward NTT mod r_a,
// two at a time (the next pair's loads issued before the current pair's
// transform), spectra fully reduced, stored in the tiled layout.
// dig: [B][D][N]; dspec: [B][RB_A][D][N].
template <class G>
__global__ void __launch_bounds__(G::T, 1)
    k_rb_fwd(const uint32_t* __restrict__ dig, uint32_t* __restrict__ dspec, int D, int reduce_digits,
             RbTabs rb, NttTabs nt) {
  extern __shared__ __align__(16) uint32_t s[];
  constexpr int E = G::E;
  const int tid = threadIdx.x;
  const int a = blockIdx.x;
  const size_t ct = blockIdx.y;
  const int jj = rb.roff + a;
  const uint32_t p = nt.prime[jj];
  const uint64_t mu = nt.mu[jj];
  const uint2* tw = nt.tw + (size_t)jj * G::N;
  const uint32_t* drow = dig + ct * D * G::N;
  uint32_t* orow = dspec + (ct * RB_A + a) * (size_t)D * G::N;
  // digits [i0, i1) of this CTA (blockIdx.z: an even-sized share, so that
  // small batches still fill the SMs)
  const int share = ((D + gridDim.z - 1) / gridDim.z + 1) & ~1;
  const int i0 = blockIdx.z * share;
  const int i1 = min(D, i0 + share);
  if (i0 >= i1) return;
  uint32_t x[2 * E];
  auto load_pair = [&](uint32_t* v, int i) {
    load_natural<G>(v, drow + (size_t)i * G::N, tid);
    if (i + 1 < i1) load_natural<G>(v + E, drow + (size_t)(i + 1) * G::N, tid);
  };
  load_pair(x, i0);
  int i = i0;
  for (; i + 1 < i1; i += 2) {
    uint32_t nx[2 * E];
    if (i + 2 < i1) load_pair(nx, i + 2);
    if (reduce_digits) {
#pragma unroll
      for (int e = 0; e < 2 * E; ++e) x[e] = reduce64(x[e], p, mu);
    }
    ntt_fwd<G, 2, true>(x, s, tw, p, tid);
    store_tiled<G>(x, orow + (size_t)i * G::N, tid);
    store_tiled<G>(x + E, orow + (size_t)(i + 1) * G::N, tid);
#pragma unroll
    for (int e = 0; e < 2 * E; ++e) x[e] = nx[e];
  }
  if (i < i1) {  // odd count: one row left (its loads were issued above)
    __syncthreads();  // the one-row exchange buffers overlap the pair's
    if (reduce_digits) {
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = reduce64(x[e], p, mu);
    }
    ntt_fwd<G, 1, true>(x, s, tw, p, tid);
    store_tiled<G>(x, orow + (size_t)i * G::N, tid);
  }
}

// Step 1 at 1024 threads (64 registers): one digit row at a time; the next
// row streams into a shared-memory stage by one TMA bulk copy (a register
// prefetch would not fit the 64-register budget).
template <class G>
constexpr int rb1_smem_words() { return G::ntt_smem_words(1) + G::N; }

template <class G>
__global__ void __launch_bounds__(G::T, 1)
    k_rb_fwd1(const uint32_t* __restrict__ dig, uint32_t* __restrict__ dspec, int D, int reduce_digits,
              RbTabs rb, NttTabs nt) {
  extern __shared__ __align__(16) uint32_t s[];
  __shared__ __align__(8) uint64_t bar;
  constexpr int E = G::E;
  const int tid = threadIdx.x;
  const int a = blockIdx.x;
  const size_t ct = blockIdx.y;
  const int jj = rb.roff + a;
  const uint32_t p = nt.prime[jj];
  const uint64_t mu = nt.mu[jj];
  const uint2* tw = nt.tw + (size_t)jj * G::N;
  const uint32_t* drow = dig + ct * D * G::N;
  uint32_t* orow = dspec + (ct * RB_A + a) * (size_t)D * G::N;
  const int share = (D + gridDim.z - 1) / gridDim.z;
  const int i0 = blockIdx.z * share;
  const int i1 = min(D, i0 + share);
  if (i0 >= i1) return;
  uint32_t* stage = s + G::ntt_smem_words(1);
  auto fetch = [&](int i) {
    fence_proxy_async();
    mbar_expect_tx(&bar, G::N * 4);
    bulk_g2s(stage, drow + (size_t)i * G::N, G::N * 4, &bar);
  };
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    fetch(i0);
  }
  __syncthreads();
  uint32_t phase = 0;
  for (int i = i0; i < i1; ++i) {
    uint32_t x[E];
    mbar_wait(&bar, phase);
    phase ^= 1;
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = stage[natural_index<G>(tid, e)];
    __syncthreads();  // every thread has read the stage
    if (tid == 0 && i + 1 < i1) fetch(i + 1);
    if (reduce_digits) {
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = reduce64(x[e], p, mu);
    }
    ntt_fwd<G, 1, true>(x, s, tw, p, tid);
    store_tiled<G>(x, orow + (size_t)i * G::N, tid);
  }
}

// Step 3 at 1024 threads: per part, the three one-row inverses mod r0, r1, r2
// (each next row staged by TMA; the first two results parked in TMEM), then
// that part's CRT and store.
template <class G>
__global__ void __launch_bounds__(G::T, 1)
    k_rb_inv1(const uint32_t* __restrict__ zspec, const uint32_t* __restrict__ y3, uint32_t* __restrict__ out,
              int K, RbTabs rb, NttTabs nt) {
  extern __shared__ __align__(16) uint32_t s[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar;
  constexpr int E = G::E;
  static_assert(E == 16, "TMEM parking in 16-column chunks");
  const int tid = threadIdx.x;
  const int j = blockIdx.x;
  const size_t ct = blockIdx.y;
  const uint32_t* zr = zspec + (ct * K + j) * (size_t)RB_A * 2 * G::N;
  constexpr uint32_t COLS = tmem_stash_cols<G, 2 * E>();
  uint32_t* stage = s + G::ntt_smem_words(1);
  auto fetch = [&](int row) {  // row (a, part) = 2 a + part
    fence_proxy_async();
    mbar_expect_tx(&bar, G::N * 4);
    bulk_g2s(stage, zr + (size_t)row * G::N, G::N * 4, &bar);
  };
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    fetch(0);  // (a = 0, part 0)
  }
  const uint32_t tbase = tmem_stash_alloc(&tmem_slot, COLS, tid, 2 * E);  // (synchronises the CTA)
  const uint32_t q = nt.prime[j];
  const uint32_t qinv = nt.pinv[j];
  const uint32_t c0 = rb.crt_q[j][0], c1 = rb.crt_q[j][1], c2 = rb.crt_q[j][2];
  const uint32_t cR = rb.negR_q[j];
  uint32_t phase = 0;
#pragma unroll 1
  for (int part = 0; part < 2; ++part) {
#pragma unroll
    for (int a = 0; a < RB_A; ++a) {
      uint32_t x[E];
      mbar_wait(&bar, phase);
      phase ^= 1;
      {
        const uint4* v = reinterpret_cast<const uint4*>(stage) + tid;
#pragma unroll
        for (int k = 0; k < E / 4; ++k) {
          const uint4 w4 = v[k * G::T];
          x[4 * k] = w4.x, x[4 * k + 1] = w4.y, x[4 * k + 2] = w4.z, x[4 * k + 3] = w4.w;
        }
      }
      __syncthreads();  // every thread has read the stage
      const int nxt = a + 1 < RB_A ? 2 * (a + 1) + part : (part == 0 ? 1 : -1);  // next (a, part) row
      if (tid == 0 && nxt >= 0) fetch(nxt);
      const int jj = rb.roff + a;
      ntt_inv<G, 1>(x, s, nt.itw + (size_t)jj * G::N, nt.prime[jj], InvScale{rb.isc_n[a], rb.isc_nw[a]}, tid);
      if (a + 1 < RB_A) {
        tmem_st16(tbase + (uint32_t)a * E, x);
      } else {
        uint32_t z0[E], z1[E];
        tmem_ld16(tbase, z0);
        tmem_ld16(tbase + E, z1);
        const uint32_t* yr = y3 + ((ct * 3 + part) * K + j) * G::N;
        uint32_t* o = out + ((ct * 2 + part) * K + j) * G::N;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const float f = __fmaf_rn((float)z0[e], rb.rinv[0], __fmaf_rn((float)z1[e], rb.rinv[1], (float)x[e] * rb.rinv[2]));
          const uint32_t v = (uint32_t)__float2int_rn(f);
          const uint64_t acc = (uint64_t)z0[e] * c0 + (uint64_t)z1[e] * c1 + (uint64_t)x[e] * c2 + (uint64_t)v * cR;
          const int idx = natural_index<G>(tid, e);
          o[idx] = add_mod(redc(acc, q, qinv), yr[idx], q);
        }
      }
    }
  }
  tmem_stash_free(tmem_slot, COLS, tid);
}

// Step 3 of 3.  One CTA per (q_j, ct): for each r_a the pair (Z_0, Z_1) mod
// r_a through the inverse NTT (two rows in lockstep; the next pair's loads
// issued first) with (R/r_a)^-1 folded into its scaling, the first two
// results parked in TMEM, then the exact centred CRT
//   Z = sum_a x~_a (R/r_a) - v R,  v = rint(sum_a x~_a / r_a)
// (|Z| / R < 2^-25, so an fp32 estimate decides v) reduced mod q_j with one
// Montgomery dot product, plus (y0, y1).
// zspec: [B][K][RB_A][2][N] tiled; y3: [B][3][K][N]; out: [B][2][K][N].
template <class G>
__global__ void __launch_bounds__(G::T, 1)
    k_rb_inv(const uint32_t* __restrict__ zspec, const uint32_t* __restrict__ y3, uint32_t* __restrict__ out,
             int K, RbTabs rb, NttTabs nt) {
  extern __shared__ __align__(16) uint32_t s[];
  __shared__ uint32_t tmem_slot;
  constexpr int E = G::E;
  static_assert(E == 16, "TMEM parking in 16-column chunks");
  const int tid = threadIdx.x;
  const int j = blockIdx.x;
  const size_t ct = blockIdx.y;
  const uint32_t* zr = zspec + (ct * K + j) * (size_t)RB_A * 2 * G::N;
  constexpr uint32_t COLS = tmem_stash_cols<G, 4 * E>();
  const uint32_t tbase = tmem_stash_alloc(&tmem_slot, COLS, tid, 4 * E);
  uint32_t x[2 * E];
  load_tiled<G>(x, zr, tid);
  load_tiled<G>(x + E, zr + G::N, tid);
#pragma unroll
  for (int a = 0; a < RB_A; ++a) {
    uint32_t nx[2 * E];
    if (a + 1 < RB_A) {
      load_tiled<G>(nx, zr + (size_t)(2 * a + 2) * G::N, tid);
      load_tiled<G>(nx + E, zr + (size_t)(2 * a + 3) * G::N, tid);
    }
    const int jj = rb.roff + a;
    ntt_inv<G, 2>(x, s, nt.itw + (size_t)jj * G::N, nt.prime[jj], InvScale{rb.isc_n[a], rb.isc_nw[a]}, tid);
    if (a + 1 < RB_A) {
      tmem_st16(tbase + (uint32_t)(2 * a) * E, x);
      tmem_st16(tbase + (uint32_t)(2 * a + 1) * E, x + E);
#pragma unroll
      for (int e = 0; e < 2 * E; ++e) x[e] = nx[e];
    }
  }
  const uint32_t q = nt.prime[j];
  const uint32_t qinv = nt.pinv[j];
  const uint32_t c0 = rb.crt_q[j][0], c1 = rb.crt_q[j][1], c2 = rb.crt_q[j][2];
  const uint32_t cR = rb.negR_q[j];
#pragma unroll
  for (int part = 0; part < 2; ++part) {
    uint32_t z0[E], z1[E];
    tmem_ld16(tbase + (uint32_t)part * E, z0);
    tmem_ld16(tbase + (uint32_t)(2 + part) * E, z1);
    const uint32_t* yr = y3 + ((ct * 3 + part) * K + j) * G::N;
    uint32_t* o = out + ((ct * 2 + part) * K + j) * G::N;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t x2 = x[part * E + e];
      const float f = __fmaf_rn((float)z0[e], rb.rinv[0],
                                __fmaf_rn((float)z1[e], rb.rinv[1], (float)x2 * rb.rinv[2]));
      const uint32_t v = (uint32_t)__float2int_rn(f);
      const uint64_t acc = (uint64_t)z0[e] * c0 + (uint64_t)z1[e] * c1 + (uint64_t)x2 * c2 + (uint64_t)v * cR;
      const int idx = natural_index<G>(tid, e);
      o[idx] = add_mod(redc(acc, q, qinv), yr[idx], q);
    }
  }
  tmem_stash_free(tmem_slot, COLS, tid);
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
    ntt_inv<G>(y, s, nt.itw + (size_t)j * G::N, p, inv_scale(nt, j, false), tid);
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

// Kernel attributes (dynamic smem opt-in) are per device: run `fn` once per
// device the process launches on (a 64-bit mask of device ordinals).
template <class Fn>
inline void per_device_once(std::atomic<uint64_t>& done, Fn fn) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  fn();
  done.fetch_or(bit, std::memory_order_release);
}

template <class G>
void configure_smem() {
  const int smem = G::ntt_smem_words(1) * sizeof(uint32_t);
  cudaFuncSetAttribute(k_ntt_rows<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_tensor<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       G::ntt_smem_words(pair_nr<G>()) * sizeof(uint32_t));
  if constexpr (G::E % 16 == 0 && G::E * (G::T / 128) <= 256) {
    cudaFuncSetAttribute(k_tensor<G, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         G::ntt_smem_words(pair_nr<G>()) * sizeof(uint32_t));
    cudaFuncSetAttribute(k_tensor<G, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         G::ntt_smem_words(pair_nr<G>()) * sizeof(uint32_t));
  }
  cudaFuncSetAttribute(k_relin<G, relin_acc64<G>(false), relin_nr<G>(false)>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, RelinSmem<G, relin_nr<G>(false)>::BYTES);
  cudaFuncSetAttribute(k_relin<G, relin_acc64<G>(true), 1>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, RelinSmem<G, 1>::BYTES);
  cudaFuncSetAttribute(k_encrypt<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if constexpr (rb_geom1<G>()) {
    cudaFuncSetAttribute(k_rb_fwd1<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         rb1_smem_words<G>() * sizeof(uint32_t));
    cudaFuncSetAttribute(k_rb_inv1<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         rb1_smem_words<G>() * sizeof(uint32_t));
  }
  if constexpr (rb_geom<G>()) {
    cudaFuncSetAttribute(k_rb_fwd<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         G::ntt_smem_words(2) * sizeof(uint32_t));
    cudaFuncSetAttribute(k_rb_inv<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         G::ntt_smem_words(2) * sizeof(uint32_t));
  }
  cudaFuncSetAttribute(k_mul_plain<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       G::ntt_smem_words(pair_nr<G>()) * sizeof(uint32_t));
}

// variant: bits 0-3 = log2 E of the fused kernels (0 = default geometry);
// RELIN_SINGLE = one-row relinearisation transforms
constexpr int RELIN_SINGLE = 16;
// relinearisation running sums in TMEM instead of registers
constexpr int RELIN_TMEM = 1024;
// square tensor with one row in registers and the others parked in TMEM
constexpr int TENSOR_TMEM = 2048;
// square tensor with the pair transforms kept and only d2 parked in TMEM
constexpr int TENSOR_TMEM_PAIR = 4096;
// persistent square tensor with TMA prefetch of the next item's rows
constexpr int TENSOR_PERSIST = 8192;

template <class G, bool SINGLE>
cudaError_t launch_relin(const NttLaunch& a) {
  constexpr int NR = relin_nr<G>(SINGLE);
  constexpr bool ACC64 = relin_acc64<G>(SINGLE);
  if (a.rlk_mont != (ACC64 ? 0 : 1)) return cudaErrorInvalidValue;
  if constexpr (!ACC64 && G::E == 16) {
    if (a.variant & RELIN_TMEM) {
      static std::atomic<uint64_t> cfg{0};
      per_device_once(cfg, [] {
        cudaFuncSetAttribute(k_relin<G, false, NR, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             RelinSmem<G, NR>::BYTES);
      });
      k_relin<G, false, NR, true><<<a.grid, G::T, RelinSmem<G, NR>::BYTES, a.stream>>>(
          a.dig, a.y3, a.rlk, a.out, a.K, a.D, a.reduce_digits, a.nt);
      return cudaSuccess;
    }
  }
  k_relin<G, ACC64, NR><<<a.grid, G::T, RelinSmem<G, NR>::BYTES, a.stream>>>(
      a.dig, a.y3, a.rlk, a.out, a.K, a.D, a.reduce_digits, a.nt);
  return cudaSuccess;
}

template <class G>
cudaError_t launch_with(int op, const NttLaunch& a) {
  static std::atomic<uint64_t> configured{0};
  per_device_once(configured, [] { configure_smem<G>(); });
  const size_t smem = G::ntt_smem_words(1) * sizeof(uint32_t);
  switch (op) {
    case 0:
      // one CTA per SM (1024 threads): the persistent prefetching kernel
      // (measured: 1.17 -> 1.70 T butterflies/s at 2^14; with two CTAs per
      // SM the plain kernel overlaps its loads itself and is faster)
      if constexpr (rows_pf_smem_words<G>() * 4 <= 220 * 1024 && G::T > 512) {
        if (a.inverse != 2) {
          static std::atomic<uint64_t> cfg{0};
          static int slots = 0;
          per_device_once(cfg, [] {
            cudaFuncSetAttribute(k_ntt_rows_pf<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 rows_pf_smem_words<G>() * 4);
            int dev = 0, sms = 0, per = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_ntt_rows_pf<G>, G::T,
                                                          rows_pf_smem_words<G>() * 4);
            slots = sms * (per > 0 ? per : 1);
          });
          const int n = (int)a.grid.x;
          k_ntt_rows_pf<G><<<n < slots ? n : slots, G::T, rows_pf_smem_words<G>() * 4, a.stream>>>(
              a.rows, n, a.limbs, a.prime_off, a.inverse, a.nt);
          break;
        }
      }
      k_ntt_rows<G><<<a.grid, G::T, smem, a.stream>>>(a.rows, a.limbs, a.prime_off, a.inverse, a.nt);
      break;
    case 1:
      if constexpr (tensor_pf_smem_words<G>() * 4 <= 220 * 1024 && G::N >= 1024) {
        if ((a.variant & TENSOR_PERSIST) && a.square) {
          static std::atomic<uint64_t> cfg{0};
          static int sms = 0;
          per_device_once(cfg, [] {
            cudaFuncSetAttribute(k_tensor_sq_pf<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 tensor_pf_smem_words<G>() * 4);
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
          });
          const int n = (int)(a.grid.x * a.grid.y);
          const int blocks = n < sms ? n : sms;
          if (n > 0)
            k_tensor_sq_pf<G><<<blocks, G::T, tensor_pf_smem_words<G>() * 4, a.stream>>>(a.a, a.ae, a.d, a.K, a.KP,
                                                                                         n, a.nt);
          break;
        }
      }
      if constexpr (G::E % 16 == 0 && G::E * (G::T / 128) <= 256) {
        if ((a.variant & TENSOR_TMEM_PAIR) && a.square) {
          k_tensor<G, 2><<<a.grid, G::T, G::ntt_smem_words(pair_nr<G>()) * sizeof(uint32_t), a.stream>>>(
              a.a, a.ae, a.b, a.be, a.d, a.K, a.KP, a.square, a.nt);
          break;
        }
        if ((a.variant & TENSOR_TMEM) && a.square) {
          k_tensor<G, 1><<<a.grid, G::T, G::ntt_smem_words(pair_nr<G>()) * sizeof(uint32_t), a.stream>>>(
              a.a, a.ae, a.b, a.be, a.d, a.K, a.KP, a.square, a.nt);
          break;
        }
      }
      k_tensor<G><<<a.grid, G::T, G::ntt_smem_words(pair_nr<G>()) * sizeof(uint32_t), a.stream>>>(
          a.a, a.ae, a.b, a.be, a.d, a.K, a.KP, a.square, a.nt);
      break;
    case 2: {
      const cudaError_t e = (a.variant & RELIN_SINGLE) ? launch_relin<G, true>(a) : launch_relin<G, false>(a);
      if (e != cudaSuccess) return e;
      break;
    }
    case 3:
      k_encrypt<G><<<a.grid, G::T, smem, a.stream>>>(a.u, a.e1, a.e2, a.msg, a.pk, a.delta, a.out, a.K, a.nt);
      break;
    case 4:
      k_ref_to_tiled<G><<<a.grid, G::T, 0, a.stream>>>(a.a, a.out, a.limbs, a.rlk_mont, a.nt);
      break;
    case 5:
      k_to_mont<G><<<a.grid, G::T, 0, a.stream>>>(a.rows, a.limbs, a.nt);
      break;
    case 6:
      k_mul_plain<G><<<a.grid, G::T, G::ntt_smem_words(pair_nr<G>()) * sizeof(uint32_t), a.stream>>>(
          a.a, a.b, a.out, a.K, a.nt);
      break;
    case 7:  // relinearisation over R, step 1: digit spectra mod r_a
    case 8:  // step 3: inverse mod r_a, exact CRT to q_j, + (y0, y1)
      if constexpr (rb_geom1<G>()) {
        if (op == 7)
          k_rb_fwd1<G><<<a.grid, G::T, rb1_smem_words<G>() * sizeof(uint32_t), a.stream>>>(
              a.dig, a.out, a.D, a.reduce_digits, a.rb, a.nt);
        else
          k_rb_inv1<G><<<a.grid, G::T, rb1_smem_words<G>() * sizeof(uint32_t), a.stream>>>(
              a.a, a.y3, a.out, a.K, a.rb, a.nt);
      } else if constexpr (rb_geom<G>()) {
        if (op == 7)
          k_rb_fwd<G><<<a.grid, G::T, G::ntt_smem_words(2) * sizeof(uint32_t), a.stream>>>(
              a.dig, a.out, a.D, a.reduce_digits, a.rb, a.nt);
        else
          k_rb_inv<G><<<a.grid, G::T, G::ntt_smem_words(2) * sizeof(uint32_t), a.stream>>>(
              a.a, a.y3, a.out, a.K, a.rb, a.nt);
      } else {
        return cudaErrorInvalidValue;
      }
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// variant bit: square tensors through k_tensor_sq on the MIXED radix-32
// geometry (two CTAs per SM); independent of the relinearisation key layout
constexpr int TENSOR_MIXED = 32;
// variant bit: every fused kernel on the MIXED geometry of the default radix
// (passes of unequal width instead of a warp-shuffle tail)
constexpr int MIXED_PASSES = 64;

template <class G>
cudaError_t launch_tensor_sq(const NttLaunch& a) {
  static std::atomic<uint64_t> configured{0};
  constexpr int smem = tensor_sq_smem_words<G>() * sizeof(uint32_t);
  per_device_once(configured, [] {
    cudaFuncSetAttribute(k_tensor_sq<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  k_tensor_sq<G><<<a.grid, G::T, smem, a.stream>>>(a.a, a.ae, a.d, a.K, a.KP, a.nt);
  return cudaGetLastError();
}

// The key layout (tiled, Montgomery or not) follows the geometry and the
// relinearisation kernel, so keys are laid out per variant.
// variant bit (default at N = 2^15): relinearisation on 2-CTA clusters
// (ntt_cluster.cuh) with keys in the radix-32 mixed layout
constexpr int CLUSTER_ROWS = 512;

template <int LOGN>
cudaError_t ntt_launch(int op, const NttLaunch& a) {
  if constexpr (LOGN == 15 || LOGN == 14) {
    if (a.variant & CLUSTER_ROWS) {
      // rows and relinearisation on 2-CTA clusters; the key-layout kernels on
      // the same (radix-32 mixed) geometry; the tensor keeps the one-CTA one
      using GC = NttGeom<LOGN, 5, false, true>;
      constexpr int smem = ClusterGeom<GC>::smem_words(1) * sizeof(uint32_t);
      static std::atomic<uint64_t> cfg{0};
      per_device_once(cfg, [] {
        cudaFuncSetAttribute(k_ntt_rows_cl<GC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_relin_cl<GC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if constexpr (LOGN == 15) {
          cudaFuncSetAttribute(k_rb_fwd_cl<GC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
          cudaFuncSetAttribute(k_rb_inv_cl<GC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        }
      });
      if constexpr (LOGN == 15) {
        if (op == 7) {  // relinearisation over R, cluster kernels
          k_rb_fwd_cl<GC><<<dim3(2 * a.grid.x, a.grid.y, a.grid.z), GC::T / 2, smem, a.stream>>>(
              a.dig, a.out, a.D, a.reduce_digits, a.rb, a.nt);
          return cudaGetLastError();
        }
        if (op == 8) {
          k_rb_inv_cl<GC><<<dim3(2 * a.grid.x, a.grid.y), GC::T / 2, smem, a.stream>>>(
              a.a, a.y3, a.out, a.K, a.rb, a.nt);
          return cudaGetLastError();
        }
      }
      if (op == 0 && a.inverse == 2) {  // forward to the tiled key layout of GC
        k_ntt_rows_cl<GC><<<dim3(2 * a.grid.x), GC::T / 2, smem, a.stream>>>(a.rows, a.limbs, a.prime_off,
                                                                             a.inverse, a.nt);
        return cudaGetLastError();
      }
      if (op == 2) {
        if (a.rlk_mont != 1) return cudaErrorInvalidValue;
        k_relin_cl<GC><<<dim3(2 * a.grid.x, a.grid.y), GC::T / 2, smem, a.stream>>>(
            a.dig, a.y3, a.rlk, a.out, a.K, a.D, a.reduce_digits, a.nt);
        return cudaGetLastError();
      }
      // everything that reads tiled keys: GC; rows in the spectral / natural
      // layouts and the tensor: the one-CTA dispatch below (faster there)
      if (op != 0 && op != 1) return launch_with<GC>(op, a);
    }
  }
  if constexpr (LOGN >= 10) {
    if (op == 1 && a.square && (a.variant & TENSOR_MIXED)) return launch_tensor_sq<NttGeom<LOGN, 5, false, true>>(a);
    if (a.variant & MIXED_PASSES) return launch_with<NttGeom<LOGN, pick_loge(LOGN), false, true>>(op, a);
  }
  return launch_with<NttGeom<LOGN>>(op, a);
}

template <class G>
int mont_of(int v) { return relin_acc64<G>((v & RELIN_SINGLE) != 0) ? 0 : 1; }


// does variant v use Montgomery-form rlk?
template <int LOGN>
int ntt_variant_mont(int v) {
  if constexpr (LOGN == 15 || LOGN == 14) {
    if (v & CLUSTER_ROWS) return 1;  // k_relin_cl: Montgomery-form keys
  }
  if constexpr (LOGN >= 10) {
    if (v & MIXED_PASSES) return mont_of<NttGeom<LOGN, pick_loge(LOGN), false, true>>(v);
  }
  return mont_of<NttGeom<LOGN>>(v);
}

}  // namespace hcnn

#define HCNN_LOGN_LIST(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15)
#define HCNN_DECLARE_LAUNCH(L)                                       \
  cudaError_t hcnn_ntt_launch_##L(int op, const hcnn::NttLaunch& a); \
  int hcnn_ntt_mont_##L(int variant);
HCNN_LOGN_LIST(HCNN_DECLARE_LAUNCH)
