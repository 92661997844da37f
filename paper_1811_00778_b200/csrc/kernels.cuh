// Non-NTT kernels of the hot path (included by hcnn.cu only).
#pragma once
#include "common.cuh"

namespace hcnn {

// ------------------------------------------------ plaintext-weight MAC
// Residues < 2^30 and weights reduced mod p_i < 2^30: 15 lazy 64-bit products
// fit before a reduction (15 * (2^30-1)^2 + 2^30 < 2^64).
struct ConvGeom {
  int h, w, c, f, kh, kw, cg, sh, sw, ph, pw, oh, ow, per_group;
  int z0;  // first output block of this launch (launches are tiled by 65535 blocks in z)
};

DI void mac4(uint64_t* a, uint32_t wv, uint4 x) {
  a[0] += (uint64_t)wv * x.x;
  a[1] += (uint64_t)wv * x.y;
  a[2] += (uint64_t)wv * x.z;
  a[3] += (uint64_t)wv * x.w;
}

// grid: x = coefficient quads, y = part*K + limb, z = out position * nfb + filter block
// wred: [F][kh][kw][cg][K] weights mod p_i.
template <int FB>
__global__ void k_conv(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                       const uint32_t* __restrict__ wred, ConvGeom g, int K, int N,
                       const uint32_t* __restrict__ primes, const uint64_t* __restrict__ mus) {
  const int quad = blockIdx.x * blockDim.x + threadIdx.x;
  if (quad * 4 >= N) return;
  const int limb = blockIdx.y % K, part = blockIdx.y / K;
  const int nfb = g.f / FB;
  const int zb = blockIdx.z + g.z0;
  const int pos = zb / nfb, fbk = zb % nfb;
  const int oy = pos / g.ow, ox = pos % g.ow;
  const int f0 = fbk * FB;
  const int grp = f0 / g.per_group;
  const uint32_t p = primes[limb];
  const uint64_t mu = mus[limb];
  uint64_t acc[FB][4];
#pragma unroll
  for (int f = 0; f < FB; ++f) acc[f][0] = acc[f][1] = acc[f][2] = acc[f][3] = 0;
  int cnt = 0;
  for (int ky = 0; ky < g.kh; ++ky) {
    const int iy = oy * g.sh + ky - g.ph;
    if (iy < 0 || iy >= g.h) continue;
    for (int kx = 0; kx < g.kw; ++kx) {
      const int ix = ox * g.sw + kx - g.pw;
      if (ix < 0 || ix >= g.w) continue;
      for (int ci = 0; ci < g.cg; ++ci) {
        const size_t in_ct = ((size_t)iy * g.w + ix) * g.c + grp * g.cg + ci;
        const uint4 xv = *reinterpret_cast<const uint4*>(in + ((in_ct * 2 + part) * K + limb) * N + quad * 4);
        const size_t wbase = (((size_t)f0 * g.kh + ky) * g.kw + kx) * g.cg + ci;
        const size_t fstride = (size_t)g.kh * g.kw * g.cg;
#pragma unroll
        for (int f = 0; f < FB; ++f) mac4(acc[f], __ldg(&wred[(wbase + f * fstride) * K + limb]), xv);
        if (++cnt == 15) {
          cnt = 0;
#pragma unroll
          for (int f = 0; f < FB; ++f)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[f][v] = reduce64(acc[f][v], p, mu);
        }
      }
    }
  }
#pragma unroll
  for (int f = 0; f < FB; ++f) {
    const size_t out_ct = (size_t)pos * g.f + f0 + f;
    uint4 r;
    r.x = reduce64(acc[f][0], p, mu);
    r.y = reduce64(acc[f][1], p, mu);
    r.z = reduce64(acc[f][2], p, mu);
    r.w = reduce64(acc[f][3], p, mu);
    *reinterpret_cast<uint4*>(out + ((out_ct * 2 + part) * K + limb) * N + quad * 4) = r;
  }
}

// dense: out[o] = sum_i W[o][i] in[i]; wred: [O][I][K]; grid z = output block
template <int OB>
__global__ void k_fc(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                     const uint32_t* __restrict__ wred, int n_in, int n_out, int K, int N,
                     const uint32_t* __restrict__ primes, const uint64_t* __restrict__ mus) {
  const int quad = blockIdx.x * blockDim.x + threadIdx.x;
  if (quad * 4 >= N) return;
  const int limb = blockIdx.y % K, part = blockIdx.y / K;
  const int o0 = blockIdx.z * OB;
  const uint32_t p = primes[limb];
  const uint64_t mu = mus[limb];
  uint64_t acc[OB][4];
#pragma unroll
  for (int o = 0; o < OB; ++o) acc[o][0] = acc[o][1] = acc[o][2] = acc[o][3] = 0;
  int cnt = 0;
  for (int i = 0; i < n_in; ++i) {
    const uint4 xv = *reinterpret_cast<const uint4*>(in + (((size_t)i * 2 + part) * K + limb) * N + quad * 4);
#pragma unroll
    for (int o = 0; o < OB; ++o)
      if (o0 + o < n_out) mac4(acc[o], __ldg(&wred[((size_t)(o0 + o) * n_in + i) * K + limb]), xv);
    if (++cnt == 15) {
      cnt = 0;
#pragma unroll
      for (int o = 0; o < OB; ++o)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[o][v] = reduce64(acc[o][v], p, mu);
    }
  }
#pragma unroll
  for (int o = 0; o < OB; ++o) {
    if (o0 + o >= n_out) break;
    uint4 r;
    r.x = reduce64(acc[o][0], p, mu);
    r.y = reduce64(acc[o][1], p, mu);
    r.z = reduce64(acc[o][2], p, mu);
    r.w = reduce64(acc[o][3], p, mu);
    *reinterpret_cast<uint4*>(out + (((size_t)(o0 + o) * 2 + part) * K + limb) * N + quad * 4) = r;
  }
}

// ---- small-weight MAC: |w| < 2^15.  Weights enter biased, wb = w + 2^15 in
// [0, 2^16), so every product wb * x < 2^46 is non-negative and 2^18 of them
// fit a u64 with no intermediate reduction; out = (sum wb x - 2^15 sum x) mod p.
constexpr uint32_t WBIAS = 1u << 15;

DI uint32_t unbias(uint64_t acc, uint64_t xsum, uint32_t p, uint64_t mu) {
  return sub_mod(reduce64(acc, p, mu), reduce64(xsum << 15, p, mu), p);
}

// grid: x = coefficient quads, y = part*K + limb, z = out position * nfb + filter block;
// wb: [F][kh][kw][cg] biased u16; smem: FB * taps u16
template <int FB>
__global__ void __launch_bounds__(128)
    k_conv_sw(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
              const uint16_t* __restrict__ wb, ConvGeom g, int K, int N,
              const uint32_t* __restrict__ primes, const uint64_t* __restrict__ mus) {
  extern __shared__ uint16_t wsm[];
  const int taps = g.kh * g.kw * g.cg;
  const int nfb = g.f / FB;
  const int zb = blockIdx.z + g.z0;
  const int pos = zb / nfb, fbk = zb % nfb;
  const int f0 = fbk * FB;
  for (int idx = threadIdx.x; idx < FB * taps; idx += blockDim.x) wsm[idx] = wb[(size_t)f0 * taps + idx];
  __syncthreads();
  const int quad = blockIdx.x * blockDim.x + threadIdx.x;
  if (quad * 4 >= N) return;
  const int limb = blockIdx.y % K, part = blockIdx.y / K;
  const int oy = pos / g.ow, ox = pos % g.ow;
  const int grp = f0 / g.per_group;
  uint64_t acc[FB][4], xs[4] = {0, 0, 0, 0};
#pragma unroll
  for (int f = 0; f < FB; ++f) acc[f][0] = acc[f][1] = acc[f][2] = acc[f][3] = 0;
  for (int ky = 0; ky < g.kh; ++ky) {
    const int iy = oy * g.sh + ky - g.ph;
    if (iy < 0 || iy >= g.h) continue;
    for (int kx = 0; kx < g.kw; ++kx) {
      const int ix = ox * g.sw + kx - g.pw;
      if (ix < 0 || ix >= g.w) continue;
      const size_t in_ct0 = ((size_t)iy * g.w + ix) * g.c + grp * g.cg;
      const int tap0 = (ky * g.kw + kx) * g.cg;
      for (int ci = 0; ci < g.cg; ++ci) {
        const uint4 xv = __ldg(reinterpret_cast<const uint4*>(in + (((in_ct0 + ci) * 2 + part) * K + limb) * N) + quad);
        xs[0] += xv.x;
        xs[1] += xv.y;
        xs[2] += xv.z;
        xs[3] += xv.w;
#pragma unroll
        for (int f = 0; f < FB; ++f) mac4(acc[f], wsm[f * taps + tap0 + ci], xv);
      }
    }
  }
  const uint32_t p = primes[limb];
  const uint64_t mu = mus[limb];
#pragma unroll
  for (int f = 0; f < FB; ++f) {
    const size_t out_ct = (size_t)pos * g.f + f0 + f;
    uint4 r;
    r.x = unbias(acc[f][0], xs[0], p, mu);
    r.y = unbias(acc[f][1], xs[1], p, mu);
    r.z = unbias(acc[f][2], xs[2], p, mu);
    r.w = unbias(acc[f][3], xs[3], p, mu);
    *(reinterpret_cast<uint4*>(out + ((out_ct * 2 + part) * K + limb) * N) + quad) = r;
  }
}

// dense, small weights: wb [n_out][n_in] biased u16; smem OB * n_in u16
template <int OB>
__global__ void __launch_bounds__(128)
    k_fc_sw(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
            const uint16_t* __restrict__ wb, int n_in, int n_out, int K, int N,
            const uint32_t* __restrict__ primes, const uint64_t* __restrict__ mus) {
  extern __shared__ uint16_t wsm[];
  const int o0 = blockIdx.z * OB;
  const int nob = min(OB, n_out - o0);
  for (int idx = threadIdx.x; idx < nob * n_in; idx += blockDim.x) wsm[idx] = wb[(size_t)o0 * n_in + idx];
  __syncthreads();
  const int quad = blockIdx.x * blockDim.x + threadIdx.x;
  if (quad * 4 >= N) return;
  const int limb = blockIdx.y % K, part = blockIdx.y / K;
  uint64_t acc[OB][4], xs[4] = {0, 0, 0, 0};
#pragma unroll
  for (int o = 0; o < OB; ++o) acc[o][0] = acc[o][1] = acc[o][2] = acc[o][3] = 0;
  for (int i = 0; i < n_in; ++i) {
    const uint4 xv = __ldg(reinterpret_cast<const uint4*>(in + (((size_t)i * 2 + part) * K + limb) * N) + quad);
    xs[0] += xv.x;
    xs[1] += xv.y;
    xs[2] += xv.z;
    xs[3] += xv.w;
#pragma unroll
    for (int o = 0; o < OB; ++o)
      if (o < nob) mac4(acc[o], wsm[o * n_in + i], xv);
  }
  const uint32_t p = primes[limb];
  const uint64_t mu = mus[limb];
#pragma unroll
  for (int o = 0; o < OB; ++o) {
    if (o >= nob) break;
    uint4 r;
    r.x = unbias(acc[o][0], xs[0], p, mu);
    r.y = unbias(acc[o][1], xs[1], p, mu);
    r.z = unbias(acc[o][2], xs[2], p, mu);
    r.w = unbias(acc[o][3], xs[3], p, mu);
    *(reinterpret_cast<uint4*>(out + (((size_t)(o0 + o) * 2 + part) * K + limb) * N) + quad) = r;
  }
}

// ---- FP64 MAC for small integer weights (|w| < 2^22).  Residues x < 2^30
// and weights are exact doubles; a product is below 2^52, and `flush` taps of
// them stay below 2^53, so DFMA accumulates the exact integer sum (on the FP64
// pipe, twice the rate of 64-bit integer multiply-adds).  Every `flush` taps
// the accumulator is reduced mod p exactly (|acc| < p afterwards).
DI double u32_to_f64(uint32_t x) {  // exact, without a conversion instruction
  return __hiloint2double(0x43300000, (int)x) - 4503599627370496.0;
}

// CNT consecutive doubles from 16-byte aligned shared memory (CNT even)
template <int CNT>
DI void lds_pairs(double* w, const double* src) {
#pragma unroll
  for (int k = 0; k < CNT / 2; ++k) {
    const double2 v = reinterpret_cast<const double2*>(src)[k];
    w[2 * k] = v.x;
    w[2 * k + 1] = v.y;
  }
}

DI double fold_mod(double acc, double p, double pinv) {
  const double qd = floor(acc * pinv);
  return fma(-qd, p, acc);  // exact: |result| < 2p
}

DI uint32_t f64_mod(double acc, double p, double pinv) {
  double r = fold_mod(acc, p, pinv);
  if (r < 0) r += p;
  if (r >= p) r -= p;
  return (uint32_t)__double2uint_rn(r);
}

// grid: x = out position * nfb + filter block, y = part, z = coefficient
// quads.  Blocks launch x-fastest, so the resident blocks sweep the output
// positions of ONE coefficient slice: the input rows their windows share
// (a 1/16 slice of each ciphertext) stay in L2 between neighbouring
// positions and each input slice crosses HBM about once.
// The block loops over the K limbs, reusing its staged weights (doubles, one
// copy for all limbs) and tap table (input ciphertext per tap, -1 when the tap
// falls in the padding).  smem: FB * taps doubles + taps ints.
template <int FB>
__global__ void __launch_bounds__(128)
    k_conv_f64(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
               const double* __restrict__ wd, ConvGeom g, int K, int N, int flush,
               const uint32_t* __restrict__ primes) {
  extern __shared__ double wsd[];
  const int taps = g.kh * g.kw * g.cg;
  int* tct = reinterpret_cast<int*>(wsd + FB * taps);
  const int nfb = g.f / FB;
  const int zb = blockIdx.x + g.z0;  // output position x filter block: the fastest grid index
  const int pos = zb / nfb, fbk = zb % nfb;
  const int f0 = fbk * FB;
  const int oy = pos / g.ow, ox = pos % g.ow;
  const int grp = f0 / g.per_group;
  for (int idx = threadIdx.x; idx < FB * taps; idx += blockDim.x) wsd[idx] = wd[(size_t)f0 * taps + idx];
  for (int t = threadIdx.x; t < taps; t += blockDim.x) {
    const int ci = t % g.cg, kk = t / g.cg;
    const int ky = kk / g.kw, kx = kk % g.kw;
    const int iy = oy * g.sh + ky - g.ph, ix = ox * g.sw + kx - g.pw;
    tct[t] = (iy < 0 || iy >= g.h || ix < 0 || ix >= g.w) ? -1 : (iy * g.w + ix) * g.c + grp * g.cg + ci;
  }
  __syncthreads();
  const int quad = blockIdx.z * blockDim.x + threadIdx.x;
  if (quad * 4 >= N) return;
  const int part = blockIdx.y;
  const size_t ct_stride = (size_t)2 * K * N / 4;  // uint4 per ciphertext
  for (int limb = 0; limb < K; ++limb) {
    const double p = (double)primes[limb];
    const double pinv = 1.0 / p;
    const uint4* base = reinterpret_cast<const uint4*>(in + ((size_t)part * K + limb) * N) + quad;
    double acc[FB][4];
#pragma unroll
    for (int f = 0; f < FB; ++f) acc[f][0] = acc[f][1] = acc[f][2] = acc[f][3] = 0.0;
    int since = 0;
    constexpr int U = 8;
    for (int t = 0; t < taps; t += U) {
      uint4 xv[U];
      int ok[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int ct = t + u < taps ? tct[t + u] : -1;
        ok[u] = ct >= 0;
        xv[u] = ok[u] ? __ldg(base + (size_t)ct * ct_stride) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!ok[u]) continue;
        const double x0 = u32_to_f64(xv[u].x), x1 = u32_to_f64(xv[u].y);
        const double x2 = u32_to_f64(xv[u].z), x3 = u32_to_f64(xv[u].w);
#pragma unroll
        for (int f = 0; f < FB; ++f) {
          const double w = wsd[f * taps + t + u];
          acc[f][0] = fma(w, x0, acc[f][0]);
          acc[f][1] = fma(w, x1, acc[f][1]);
          acc[f][2] = fma(w, x2, acc[f][2]);
          acc[f][3] = fma(w, x3, acc[f][3]);
        }
      }
      since += U;
      if (since >= flush - U) {
        since = 0;
#pragma unroll
        for (int f = 0; f < FB; ++f)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[f][v] = fold_mod(acc[f][v], p, pinv);
      }
    }
#pragma unroll
    for (int f = 0; f < FB; ++f) {
      const size_t out_ct = (size_t)pos * g.f + f0 + f;
      uint4 r;
      r.x = f64_mod(acc[f][0], p, pinv);
      r.y = f64_mod(acc[f][1], p, pinv);
      r.z = f64_mod(acc[f][2], p, pinv);
      r.w = f64_mod(acc[f][3], p, pinv);
      *(reinterpret_cast<uint4*>(out + ((out_ct * 2 + part) * K + limb) * N) + quad) = r;
    }
  }
}

// dense: wd [n_out][n_in] doubles staged CH inputs at a time (smem OB * CH doubles)
template <int OB, int CH>
__global__ void __launch_bounds__(128)
    k_fc_f64(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
             const double* __restrict__ wd, int n_in, int n_out, int K, int N, int flush,
             const uint32_t* __restrict__ primes) {
  __shared__ double wsd[OB * CH];
  const int o0 = blockIdx.z * OB;
  const int nob = min(OB, n_out - o0);
  const int quad = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = quad * 4 < N;
  const int limb = blockIdx.y % K, part = blockIdx.y / K;
  const double p = (double)primes[limb];
  const double pinv = 1.0 / p;
  double acc[OB][4];
#pragma unroll
  for (int o = 0; o < OB; ++o) acc[o][0] = acc[o][1] = acc[o][2] = acc[o][3] = 0.0;
  int cnt = 0;
  for (int c0 = 0; c0 < n_in; c0 += CH) {
    const int len = min(CH, n_in - c0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < OB * CH; idx += blockDim.x) {
      const int o = idx / CH, i = idx % CH;
      wsd[idx] = (o < nob && i < len) ? wd[(size_t)(o0 + o) * n_in + c0 + i] : 0.0;
    }
    __syncthreads();
    if (!active) continue;
    const size_t ct_stride = (size_t)2 * K * N / 4;
    const uint4* base = reinterpret_cast<const uint4*>(in + ((size_t)part * K + limb) * N) + quad;
    constexpr int U = 4;
    for (int i = 0; i < len; i += U) {
      uint4 xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = __ldg(base + (size_t)(c0 + min(i + u, len - 1)) * ct_stride);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (i + u >= len) break;
        const double x0 = u32_to_f64(xv[u].x), x1 = u32_to_f64(xv[u].y);
        const double x2 = u32_to_f64(xv[u].z), x3 = u32_to_f64(xv[u].w);
#pragma unroll
        for (int o = 0; o < OB; ++o) {
          const double w = wsd[o * CH + i + u];
          acc[o][0] = fma(w, x0, acc[o][0]);
          acc[o][1] = fma(w, x1, acc[o][1]);
          acc[o][2] = fma(w, x2, acc[o][2]);
          acc[o][3] = fma(w, x3, acc[o][3]);
        }
      }
      cnt += U;
      if (cnt >= flush - U) {
        cnt = 0;
#pragma unroll
        for (int o = 0; o < OB; ++o)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[o][v] = fold_mod(acc[o][v], p, pinv);
      }
    }
  }
  if (!active) return;
#pragma unroll
  for (int o = 0; o < OB; ++o) {
    if (o >= nob) break;
    uint4 r;
    r.x = f64_mod(acc[o][0], p, pinv);
    r.y = f64_mod(acc[o][1], p, pinv);
    r.z = f64_mod(acc[o][2], p, pinv);
    r.w = f64_mod(acc[o][3], p, pinv);
    *(reinterpret_cast<uint4*>(out + (((size_t)(o0 + o) * 2 + part) * K + limb) * N) + quad) = r;
  }
}

// Split-K dense layer: blockIdx.x = (output block, input split), z = slab.  Each block
// sums inputs [split*chunk, +chunk) for OB outputs of one (part, limb) over a
// slab of 2 * blockDim coefficients (2 per thread, 8-byte loads) and writes
// the reduced partial sum; k_fc_reduce adds the S partials mod p.  The block's
// OB x chunk weights are staged in shared memory once.  Every input ciphertext
// is read once per output block.  ws: [S][n_out][2][K][N] u32.
template <int OB>
__global__ void __launch_bounds__(128)
    k_fc_f64_split(const uint32_t* __restrict__ in, uint32_t* __restrict__ ws,
                   const double* __restrict__ wd, int n_in, int n_out, int K, int N, int flush,
                   int chunk, int nob_blocks, const uint32_t* __restrict__ primes) {
  extern __shared__ double wsd[];  // [chunk][OBP]: an input's OB weights are one run of 16-byte loads
  constexpr int OBP = OB + (OB & 1);
  // output block fastest in the launch order: the blocks sharing one input
  // slab run together and read it from L2, not DRAM, after the first
  const int ob = blockIdx.x % nob_blocks, split = blockIdx.x / nob_blocks;
  const int o0 = ob * OB;
  const int i0 = split * chunk, len = min(n_in, i0 + chunk) - i0;
  for (int idx = threadIdx.x; idx < OBP * chunk; idx += blockDim.x) {
    const int i = idx / OBP, o = idx % OBP;
    wsd[idx] = (i < len && o < OB) ? wd[(size_t)(o0 + o) * n_in + i0 + i] : 0.0;
  }
  __syncthreads();
  const int pair = blockIdx.z * blockDim.x + threadIdx.x;
  if (pair * 2 >= N) return;
  const int limb = blockIdx.y % K, part = blockIdx.y / K;
  const double p = (double)primes[limb];
  const double pinv = 1.0 / p;
  double acc[OB][2];
#pragma unroll
  for (int o = 0; o < OB; ++o) acc[o][0] = acc[o][1] = 0.0;
  const size_t ct_stride = (size_t)K * N;  // uint2 per ciphertext
  const uint2* base = reinterpret_cast<const uint2*>(in + ((size_t)part * K + limb) * N) + pair +
                      (size_t)i0 * ct_stride;
  int cnt = 0;
  constexpr int U = 8;
  // software-pipelined: the next U inputs are in flight while these are summed
  uint2 nxt[U];
#pragma unroll
  for (int u = 0; u < U; ++u) nxt[u] = __ldg(base + (size_t)min(u, len - 1) * ct_stride);
  for (int i = 0; i < len; i += U) {
    uint2 xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = nxt[u];
    if (i + U < len) {
#pragma unroll
      for (int u = 0; u < U; ++u) nxt[u] = __ldg(base + (size_t)min(i + U + u, len - 1) * ct_stride);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i + u >= len) break;
      const double x0 = u32_to_f64(xv[u].x), x1 = u32_to_f64(xv[u].y);
      double wv[OBP];
      lds_pairs<OBP>(wv, wsd + (i + u) * OBP);
#pragma unroll
      for (int o = 0; o < OB; ++o) {
        acc[o][0] = fma(wv[o], x0, acc[o][0]);
        acc[o][1] = fma(wv[o], x1, acc[o][1]);
      }
    }
    cnt += U;
    if (cnt >= flush - U) {
      cnt = 0;
#pragma unroll
      for (int o = 0; o < OB; ++o) {
        acc[o][0] = fold_mod(acc[o][0], p, pinv);
        acc[o][1] = fold_mod(acc[o][1], p, pinv);
      }
    }
  }
#pragma unroll
  for (int o = 0; o < OB; ++o) {
    const uint2 r = make_uint2(f64_mod(acc[o][0], p, pinv), f64_mod(acc[o][1], p, pinv));
    *(reinterpret_cast<uint2*>(ws + ((((size_t)split * n_out + o0 + o) * 2 + part) * K + limb) * N) + pair) = r;
  }
}

// out = sum over S partial sums mod p; ws [S][rows][N], rows = n_out * 2 * K
__global__ void k_fc_reduce(const uint32_t* __restrict__ ws, uint32_t* __restrict__ out, int S, size_t rows,
                            int K, int N, const uint32_t* __restrict__ primes) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;  // uint4 index
  const size_t quads = rows * N / 4;
  if (i >= quads) return;
  const uint32_t p = primes[(i * 4 / N) % K];
  const uint4* src = reinterpret_cast<const uint4*>(ws) + i;
  uint4 a = src[0];
  for (int s = 1; s < S; ++s) {
    const uint4 b = src[(size_t)s * quads];
    a.x = add_mod(a.x, b.x, p);
    a.y = add_mod(a.y, b.y, p);
    a.z = add_mod(a.z, b.z, p);
    a.w = add_mod(a.w, b.w, p);
  }
  reinterpret_cast<uint4*>(out)[i] = a;
}

__global__ void k_weights_f64(const int64_t* __restrict__ w, size_t n, double* __restrict__ out) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) out[t] = (double)w[t];
}

__global__ void k_bias_weights(const int64_t* __restrict__ w, size_t n, uint16_t* __restrict__ out) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) out[t] = (uint16_t)(w[t] + (int64_t)WBIAS);
}

// sum-pool: grid x = quads, y = part*K + limb, z = output ct - o0
__global__ void k_pool(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, int h, int w,
                       int c, int e, int sh, int sw, int ow, int K, int N,
                       const uint32_t* __restrict__ primes, const uint64_t* __restrict__ mus, int o0) {
  const int quad = blockIdx.x * blockDim.x + threadIdx.x;
  if (quad * 4 >= N) return;
  const int limb = blockIdx.y % K, part = blockIdx.y / K;
  const int o = blockIdx.z + o0;
  const int ch = o % c, pos = o / c;
  const int oy = pos / ow, ox = pos % ow;
  uint64_t a[4] = {0, 0, 0, 0};
  for (int dy = 0; dy < e; ++dy)
    for (int dx = 0; dx < e; ++dx) {
      const size_t ict = ((size_t)(oy * sh + dy) * w + (ox * sw + dx)) * c + ch;
      const uint4 x = *reinterpret_cast<const uint4*>(in + ((ict * 2 + part) * K + limb) * N + quad * 4);
      a[0] += x.x;
      a[1] += x.y;
      a[2] += x.z;
      a[3] += x.w;
    }
  const uint32_t p = primes[limb];
  const uint64_t mu = mus[limb];
  uint4 r;
  r.x = reduce64(a[0], p, mu);
  r.y = reduce64(a[1], p, mu);
  r.z = reduce64(a[2], p, mu);
  r.w = reduce64(a[3], p, mu);
  *reinterpret_cast<uint4*>(out + (((size_t)o * 2 + part) * K + limb) * N + quad * 4) = r;
}

// weights (int64, any sign) -> [n][K] residues mod q_i
__global__ void k_reduce_weights(const int64_t* __restrict__ w, size_t n, uint32_t* __restrict__ out,
                                 const uint32_t* __restrict__ primes, int K) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int64_t v = w[t];
  for (int i = 0; i < K; ++i) {
    int64_t r = v % (int64_t)primes[i];
    if (r < 0) r += primes[i];
    out[t * K + i] = (uint32_t)r;
  }
}

// device rows [r][K][N] u32 <-> HFIR element bodies [r][N][K] u64 (serial.py:87-97)
__global__ void k_hfir_pack(const uint32_t* __restrict__ in, uint64_t* __restrict__ out, int K, int N,
                            size_t rows) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;  // (row, n)
  if (i >= rows * N) return;
  const size_t r = i / N, n = i % N;
  const uint32_t* src = in + r * K * N + n;
  uint64_t* dst = out + i * K;
  for (int k = 0; k < K; ++k) dst[k] = src[(size_t)k * N];
}

__global__ void k_hfir_unpack(const uint64_t* __restrict__ in, uint32_t* __restrict__ out, int K, int N,
                              size_t rows, const uint32_t* __restrict__ primes, int* __restrict__ bad) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * N) return;
  const size_t r = i / N, n = i % N;
  const uint64_t* src = in + i * K;
  uint32_t* dst = out + r * K * N + n;
  for (int k = 0; k < K; ++k) {
    const uint64_t v = src[k];
    if (v >= primes[k]) atomicOr(bad, 1);
    dst[(size_t)k * N] = (uint32_t)v;
  }
}

// centred plaintext coefficients (int64) -> [K][N] residues mod q_i
__global__ void k_lift_plain(const int64_t* __restrict__ pt, uint32_t* __restrict__ rows, int N, int K,
                             const uint32_t* __restrict__ primes) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const int64_t v = pt[n];
  for (int i = 0; i < K; ++i) {
    int64_t r = v % (int64_t)primes[i];
    if (r < 0) r += primes[i];
    rows[(size_t)i * N + n] = (uint32_t)r;
  }
}

// out = in * (s mod q_i): the scalar path of hmult_plain (bfv.py:311-314,
// ring.py:193-196); sres: [K] residues of the scalar
__global__ void k_mul_scalar(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                             const uint32_t* __restrict__ sres, int K, int N, size_t total,
                             const uint32_t* __restrict__ primes, const uint64_t* __restrict__ mus) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int limb = (int)((i / N) % K);
  out[i] = mul_mod(in[i], sres[limb], primes[limb], mus[limb]);
}

// small signed coefficients (int8 [R][N]) -> residues [R][K][N]
__global__ void k_embed_small(const int8_t* __restrict__ e, uint32_t* __restrict__ rows, int R, int K, int N,
                              const uint32_t* __restrict__ primes) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;  // (r, n)
  if (i >= (size_t)R * N) return;
  const size_t r = i / N, n = i % N;
  const int v = e[i];
  for (int k = 0; k < K; ++k) rows[(r * K + k) * N + n] = v < 0 ? primes[k] - (uint32_t)(-v) : (uint32_t)v;
}

// key rows in the NTT domain (bfv.py:164-188), R = 1 + D rows [R][K][N]:
// row 0 = b = e - a s, row 1+i = k0_i = w^i s^2 - (a_i s + e_i); wres [R][K]
__global__ void k_keygen_combine(const uint32_t* __restrict__ a, const uint32_t* __restrict__ e,
                                 const uint32_t* __restrict__ s, const uint32_t* __restrict__ wres,
                                 uint32_t* __restrict__ out, int R, int K, int N,
                                 const uint32_t* __restrict__ primes, const uint64_t* __restrict__ mus) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)R * K * N) return;
  const size_t row = i / N, n = i % N;
  const int r = (int)(row / K), k = (int)(row % K);
  const uint32_t p = primes[k];
  const uint64_t mu = mus[k];
  const uint32_t sv = s[(size_t)k * N + n];
  const uint32_t as = mul_mod(a[i], sv, p, mu);
  if (r == 0) {
    out[i] = sub_mod(e[i], as, p);
  } else {
    const uint32_t s2w = mul_mod(mul_mod(sv, sv, p, mu), wres[r * K + k], p, mu);
    out[i] = sub_mod(s2w, add_mod(as, e[i], p), p);
  }
}

// reference-order NTT (natural, a(psi^(2k+1))) -> device spectral order
// in place on [rows][N] via a temp: dst[i] = src[brv(i)]
__global__ void k_bitrev_rows(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, int N,
                              int logn) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const size_t row = blockIdx.y;
  const int r = __brev(i) >> (32 - logn);
  dst[row * N + i] = src[row * N + r];
}

// u64 residues -> u32
__global__ void k_narrow(const uint64_t* __restrict__ src, uint32_t* __restrict__ dst, size_t n) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = (uint32_t)src[i];
}
__global__ void k_widen(const uint32_t* __restrict__ src, uint64_t* __restrict__ dst, size_t n) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[i];
}

}  // namespace hcnn
