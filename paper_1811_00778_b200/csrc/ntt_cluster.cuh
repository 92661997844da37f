// NTT of one row split over a CLUSTER of two CTAs (N = 2^15): each CTA holds
// half of the row in registers (512 threads x 32 residues, 128 registers per
// thread, where one 1024-thread CTA would have only 64 and spill), and the
// exchange between the two halves goes through distributed shared memory.
//
// Geometry: the radix-32 MIXED geometry (passes of 5 + 5 + 5 bits, no tail)
// over T = 1024 VIRTUAL threads, vtid = rank * 512 + tid.  With those pass
// maps the forward's first exchange sends half of every thread's residues to
// the other CTA (the rank bit of the element index comes from the register
// index) and the second exchange is CTA-local; the inverse mirrors that.
// Each CTA's exchange buffer is COMPACT: the element index with the exchange's
// rank bit squeezed out (2^14 words + padding), so two rows fit in 227 KB.
// Barriers are cluster barriers (arrive.release / wait.acquire), one per
// exchange with two alternating buffers.
#pragma once
#include "common.cuh"
#include "ntt.cuh"
#include "tma.cuh"

namespace hcnn {

DI uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

DI void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// shared::cluster address of `local` (a shared::cta address) in CTA `rank`
DI uint32_t map_rank(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}

DI void st_cluster(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// element index with bit RB removed
template <int RB>
DI int squeeze(int idx) {
  return ((idx >> (RB + 1)) << RB) | (idx & ((1 << RB) - 1));
}

template <class G>
struct ClusterGeom {
  static_assert(G::MIXED && G::LOGE == 5 && (G::LOGN == 15 || G::LOGN == 14),
                "cluster NTT: 2^14 / 2^15 on the radix-32 mixed geometry");
  static_assert(G::NFULL == 3, "cluster NTT: three register passes, two exchanges");
  static constexpr int TC = G::T / 2;                  // threads per CTA
  static constexpr int HALF = G::N / 2;                // residues per CTA
  static constexpr int XW = (HALF + 2 * (HALF >> 5) + 2 + 3) & ~3;  // padded compact row
  __host__ __device__ static constexpr int smem_words(int nr) { return 2 * nr * XW; }
};

// Exchange between pass P_OUT (registers now) and P_IN (registers after): the
// CTA that reads element idx in pass P_IN is bit RB of idx.  Writes go to that
// CTA's buffer (through DSMEM when it is the other one), reads are local.
template <class G, int P_OUT, int P_IN, int RB, int NR>
DI void cluster_exchange(uint32_t* x, uint32_t* buf, int vtid, uint32_t rank) {
  using C = ClusterGeom<G>;
  const uint32_t base_local = smem_u32(buf);
  const uint32_t base_other = map_rank(base_local, rank ^ 1u);
  const uint32_t base_self = map_rank(base_local, rank);
#pragma unroll
  for (int r = 0; r < NR; ++r)
#pragma unroll
    for (int e = 0; e < G::E; ++e) {
      const int idx = gpass_index<G, G::lo(P_OUT), G::kb(P_OUT)>(vtid, e);
      const uint32_t dst = (uint32_t)((idx >> RB) & 1);
      const uint32_t off = (uint32_t)(r * C::XW + sidx(squeeze<RB>(idx))) * 4u;
      st_cluster((dst == rank ? base_self : base_other) + off, x[r * G::E + e]);
    }
  cluster_sync_all();
#pragma unroll
  for (int r = 0; r < NR; ++r)
#pragma unroll
    for (int e = 0; e < G::E; ++e)
      x[r * G::E + e] = buf[r * C::XW + sidx(squeeze<RB>(gpass_index<G, G::lo(P_IN), G::kb(P_IN)>(vtid, e)))];
}

// rank bit of the element index in pass P's map: the top virtual-thread bit
// lands at bit LOGT - 1 below lo(P), else LOGT - 1 + kb(P)
template <class G, int P>
__host__ __device__ constexpr int rank_bit() {
  return (G::LOGT - 1) < G::lo(P) ? (G::LOGT - 1) : (G::LOGT - 1 + G::kb(P));
}

// Forward: natural layout in (values < 4p), spectral layout out, reduced to
// [0, p) (FULL) or [0, 2p).  s: ClusterGeom::smem_words(NR) words.
template <class G, int NR = 1, bool FULL = true>
DI void ntt_fwd_cl(uint32_t* x, uint32_t* s, const uint2* __restrict__ tw, uint32_t p, int vtid,
                   uint32_t rank) {
  using C = ClusterGeom<G>;
  fwd_stage<G, G::lo(0), G::kb(0), 0, NR>(x, tw, p, vtid);
  cluster_exchange<G, 0, 1, rank_bit<G, 1>(), NR>(x, s, vtid, rank);
  fwd_stage<G, G::lo(1), G::kb(1), 0, NR>(x, tw, p, vtid);
  cluster_exchange<G, 1, 2, rank_bit<G, 2>(), NR>(x, s + NR * C::XW, vtid, rank);
  fwd_stage<G, G::lo(2), G::kb(2), 0, NR>(x, tw, p, vtid);
  const uint32_t p2 = 2 * p;
#pragma unroll
  for (int e = 0; e < NR * G::E; ++e) {
    const uint32_t v = umin32(x[e], x[e] - p2);
    x[e] = FULL ? umin32(v, v - p) : v;
  }
}

// Inverse: spectral layout in (values < 2p), natural layout out, scaled by
// sc (folded into the last stage), reduced to [0, p).
template <class G, int NR = 1>
DI void ntt_inv_cl(uint32_t* x, uint32_t* s, const uint2* __restrict__ itw, uint32_t p, const InvScale& sc,
                   int vtid, uint32_t rank) {
  using C = ClusterGeom<G>;
  inv_stage<G, G::lo(2), G::kb(2), G::kb(2) - 1, NR>(x, itw, p, vtid, sc);
  cluster_exchange<G, 2, 1, rank_bit<G, 1>(), NR>(x, s, vtid, rank);
  inv_stage<G, G::lo(1), G::kb(1), G::kb(1) - 1, NR>(x, itw, p, vtid, sc);
  cluster_exchange<G, 1, 0, rank_bit<G, 0>(), NR>(x, s + NR * C::XW, vtid, rank);
  inv_stage<G, G::lo(0), G::kb(0), G::kb(0) - 1, NR>(x, itw, p, vtid, sc);
}

// Rows of N = 2^15 residues, one cluster of two CTAs per row (grid.x = 2 rows):
// like k_ntt_rows (inverse: 0 forward to spectral positions, 1 inverse, 2
// forward to the tiled layout).
template <class G>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(G::T / 2, (G::T / 2 <= 256 ? 2 : 1))
    k_ntt_rows_cl(uint32_t* __restrict__ data, int limbs, int prime_off, int inverse, NttTabs nt) {
  extern __shared__ __align__(16) uint32_t s[];
  const uint32_t rank = cluster_rank();
  const int vtid = (int)rank * ClusterGeom<G>::TC + threadIdx.x;
  const int row = blockIdx.x / 2;
  const int j = prime_off + row % limbs;
  uint32_t* r = data + (size_t)row * G::N;
  const uint32_t p = nt.prime[j];
  uint32_t x[G::E];
  cluster_sync_all();  // both CTAs running before any DSMEM store
  if (inverse == 1) {
#pragma unroll
    for (int e = 0; e < G::E; ++e) x[e] = r[spectral_index<G>(vtid, e)];
    ntt_inv_cl<G>(x, s, nt.itw + (size_t)j * G::N, p, inv_scale(nt, j, false), vtid, rank);
#pragma unroll
    for (int e = 0; e < G::E; ++e) r[natural_index<G>(vtid, e)] = x[e];
  } else {
#pragma unroll
    for (int e = 0; e < G::E; ++e) x[e] = r[natural_index<G>(vtid, e)];
    ntt_fwd_cl<G>(x, s, nt.tw + (size_t)j * G::N, p, vtid, rank);
    if (inverse == 2) {
#pragma unroll
      for (int e = 0; e < G::E; ++e) r[tiled_index<G>(vtid, e)] = x[e];
    } else {
#pragma unroll
      for (int e = 0; e < G::E; ++e) r[spectral_index<G>(vtid, e)] = x[e];
    }
  }
  // (every DSMEM store precedes a cluster barrier both CTAs pass: no exit sync)
}

// ---- TMEM as accumulator storage (the relinearisation's 2 x 32 running sums
// per thread would not fit beside a 32-residue row in 128 registers).  One
// warp allocates 256 columns; warp w uses lanes 32 (w % 4) + lane and columns
// 64 (w / 4) + [0, 64): part 0 in the first 32, part 1 in the next 32.
DI void tmem_alloc256(uint32_t* slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(slot)) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

DI void tmem_dealloc256(uint32_t base) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(base) : "memory");
}

DI void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
DI void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

DI void tmem_ld16(uint32_t addr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

DI void tmem_st16(uint32_t addr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16};" ::"r"(addr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Relinearisation (bfv.py:368-404) at N = 2^15 on 2-CTA clusters: one cluster
// per (ct, prime of q); each digit row goes through the cluster forward NTT
// and is multiply-accumulated with the key (tiled layout of G, Montgomery
// form) into u32 accumulators in [0, 2p) held in TMEM; the two parts then go
// through the cluster inverse and are added to (y0, y1).  Digits are read
// straight from global memory.  grid: (2 K, B).
template <class G>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(G::T / 2, (G::T / 2 <= 256 ? 2 : 1))
    k_relin_cl(const uint32_t* __restrict__ dig, const uint32_t* __restrict__ y3,
               const uint32_t* __restrict__ rlk, uint32_t* __restrict__ out, int K, int D,
               int reduce_digits, NttTabs nt) {
  extern __shared__ __align__(16) uint32_t s[];
  __shared__ uint32_t tmem_slot;
  constexpr int E = G::E;
  static_assert(E == 32 && (G::T / 2 == 512 || G::T / 2 == 256), "TMEM plan: 8 or 16 warps x 32 lanes x 64 columns");
  const uint32_t rank = cluster_rank();
  const int vtid = (int)rank * ClusterGeom<G>::TC + threadIdx.x;
  const int j = blockIdx.x / 2;
  const size_t ct = blockIdx.y;
  const uint32_t p = nt.prime[j];
  const uint64_t mu = nt.mu[j];
  const uint32_t pinv = nt.pinv[j];
  const uint32_t p2 = 2 * p;
  const uint2* tw = nt.tw + (size_t)j * G::N;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc256(&tmem_slot);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tacc = tmem_slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(warp >> 2) * 64;
  {
    uint32_t z[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) z[e] = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_st16(tacc + 16 * c, z);
  }
  const uint32_t* dig_ct = dig + ct * D * G::N;
  cluster_sync_all();  // both CTAs running before any DSMEM store
  for (int i = 0; i < D; ++i) {
    uint32_t x[E];
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = dig_ct[(size_t)i * G::N + natural_index<G>(vtid, e)];
    if (reduce_digits) {
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = reduce64(x[e], p, mu);
    }
    ntt_fwd_cl<G, 1, false>(x, s, tw, p, vtid, rank);  // [0, 2p): x k < 2 p^2 < 2^32 p
#pragma unroll
    for (int part = 0; part < 2; ++part) {
      const uint4* kr = reinterpret_cast<const uint4*>(rlk + ((size_t)(i * 2 + part) * K + j) * G::N) + vtid;
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // 16 accumulators at a time
        uint32_t a[16];
        tmem_ld16(tacc + part * 32 + h * 16, a);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint4 kv = __ldg(&kr[(h * 4 + c) * G::T]);
          const uint32_t k4[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
          for (int l = 0; l < 4; ++l) {
            const uint32_t v = a[4 * c + l] + mont_mul(x[16 * h + 4 * c + l], k4[l], p, pinv);
            a[4 * c + l] = umin32(v, v - p2);
          }
        }
        tmem_st16(tacc + part * 32 + h * 16, a);
      }
    }
  }
  const uint2* itw = nt.itw + (size_t)j * G::N;
  const InvScale ninv = inv_scale(nt, j, false);
#pragma unroll 1
  for (int part = 0; part < 2; ++part) {
    uint32_t x[E];
    tmem_ld16(tacc + part * 32, x);
    tmem_ld16(tacc + part * 32 + 16, x + 16);
    ntt_inv_cl<G>(x, s, itw, p, ninv, vtid, rank);
    const uint32_t* yr = y3 + ((ct * 3 + part) * K + j) * G::N;
    uint32_t* o = out + ((ct * 2 + part) * K + j) * G::N;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int idx = natural_index<G>(vtid, e);
      o[idx] = add_mod(x[e], yr[idx], p);
    }
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc256(tmem_slot);
}

// Relinearisation over R (RbTabs, common.cuh) at N = 2^15 on 2-CTA clusters.
// Step 1: one cluster per (r_a, ct, digit share) — every digit row through
// the cluster forward NTT mod r_a (the next row's loads issued first),
// spectra fully reduced, stored in the tiled layout of G.  grid (2 RB_A, B, split).
// Every CTA of a 2^15 cluster holds 16 warps, so the row loads overlap
// the other CTAs' transforms.
template <class G>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(G::T / 2, 1)
    k_rb_fwd_cl(const uint32_t* __restrict__ dig, uint32_t* __restrict__ dspec, int D, int reduce_digits,
                RbTabs rb, NttTabs nt) {
  extern __shared__ __align__(16) uint32_t s[];
  constexpr int E = G::E;
  const uint32_t rank = cluster_rank();
  const int vtid = (int)rank * ClusterGeom<G>::TC + threadIdx.x;
  const int a = blockIdx.x / 2;
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
  if (i0 >= i1) return;  // (both CTAs of the cluster take the same branch)
  cluster_sync_all();  // both CTAs running before any DSMEM store
  for (int i = i0; i < i1; ++i) {
    uint32_t x[E];  // (no register prefetch: 32 more live residues would spill)
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = drow[(size_t)i * G::N + natural_index<G>(vtid, e)];
    if (reduce_digits) {
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = reduce64(x[e], p, mu);
    }
    ntt_fwd_cl<G, 1, true>(x, s, tw, p, vtid, rank);
#pragma unroll
    for (int e = 0; e < E; ++e) orow[(size_t)i * G::N + tiled_index<G>(vtid, e)] = x[e];
  }
}

// Step 3: one cluster per (q_j, ct); per part the three inverses mod r0, r1,
// r2 (first two results parked in TMEM), then the exact centred CRT to q_j
// (k_rb_inv in ntt_kernels.cuh) + (y0, y1).  grid (2 K, B).
template <class G>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(G::T / 2, 1)
    k_rb_inv_cl(const uint32_t* __restrict__ zspec, const uint32_t* __restrict__ y3, uint32_t* __restrict__ out,
                int K, RbTabs rb, NttTabs nt) {
  extern __shared__ __align__(16) uint32_t s[];
  __shared__ uint32_t tmem_slot;
  constexpr int E = G::E;
  static_assert(E == 32 && G::T / 2 == 512, "TMEM plan: 16 warps x 32 lanes x 64 columns");
  const uint32_t rank = cluster_rank();
  const int vtid = (int)rank * ClusterGeom<G>::TC + threadIdx.x;
  const int j = blockIdx.x / 2;
  const size_t ct = blockIdx.y;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc256(&tmem_slot);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tz = tmem_slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(warp >> 2) * 64;
  const uint32_t* zr = zspec + (ct * K + j) * (size_t)RB_A * 2 * G::N;
  const uint32_t q = nt.prime[j];
  const uint32_t qinv = nt.pinv[j];
  const uint32_t c0 = rb.crt_q[j][0], c1 = rb.crt_q[j][1], c2 = rb.crt_q[j][2];
  const uint32_t cR = rb.negR_q[j];
  cluster_sync_all();  // both CTAs running before any DSMEM store
#pragma unroll 1
  for (int part = 0; part < 2; ++part) {
    uint32_t x[E];
#pragma unroll 1
    for (int a = 0; a < RB_A; ++a) {
      const uint32_t* row = zr + (size_t)(2 * a + part) * G::N;
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = row[tiled_index<G>(vtid, e)];
      const int jj = rb.roff + a;
      ntt_inv_cl<G>(x, s, nt.itw + (size_t)jj * G::N, nt.prime[jj], InvScale{rb.isc_n[a], rb.isc_nw[a]}, vtid,
                    rank);
      if (a + 1 < RB_A) {
        tmem_st16(tz + a * 32, x);
        tmem_st16(tz + a * 32 + 16, x + 16);
      }
    }
    const uint32_t* yr = y3 + ((ct * 3 + part) * K + j) * G::N;
    uint32_t* o = out + ((ct * 2 + part) * K + j) * G::N;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t z0[16], z1[16];
      tmem_ld16(tz + h * 16, z0);
      tmem_ld16(tz + 32 + h * 16, z1);
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const uint32_t x2 = x[16 * h + e];
        const float f = __fmaf_rn((float)z0[e], rb.rinv[0], __fmaf_rn((float)z1[e], rb.rinv[1], (float)x2 * rb.rinv[2]));
        const uint32_t v = (uint32_t)__float2int_rn(f);
        const uint64_t acc = (uint64_t)z0[e] * c0 + (uint64_t)z1[e] * c1 + (uint64_t)x2 * c2 + (uint64_t)v * cR;
        const int idx = natural_index<G>(vtid, 16 * h + e);
        o[idx] = add_mod(redc(acc, q, qinv), yr[idx], q);
      }
    }
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc256(tmem_slot);
}

}  // namespace hcnn
