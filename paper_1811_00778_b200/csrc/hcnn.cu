// Context, dispatch and the exported C ABI (include/hcnn_b200.h).
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <condition_variable>
#include <functional>

#include <immintrin.h>
#include <string>
#include <vector>

#include "../../include/hcnn_b200.h"
#include "conv_kernels.cuh"
#include "crt.cuh"
#include "kernels.cuh"
#include "ntt_kernels.cuh"
#include "ntt64.cuh"
#include "relin_rb.cuh"
#include "tables.hpp"

using namespace hcnn;

namespace {

thread_local std::string g_err;

struct Error {
  int code;
  std::string msg;
};

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error{HCNN_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}
#define CK(x) check_cuda((x), #x)

template <class F>
int guarded(F&& f) {
  try {
    f();
    return HCNN_OK;
  } catch (const Error& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HCNN_ERR_UNSUPPORTED;
  }
}

void fail(int code, const std::string& m) { throw Error{code, m}; }

// The library's own stream-ordered memory pool per device: workspaces and
// temporaries stay pooled across synchronisations (release threshold = max)
// without changing the device's default pool, which other cudaMallocAsync
// users in the process (e.g. PyTorch's async allocator) share.
std::mutex g_pool_mu;
cudaMemPool_t g_pools[64] = {};

cudaMemPool_t lib_pool(int device) {
  if (device < 0 || device >= 64) fail(HCNN_ERR_PARAM, "device index out of range");
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_pools[device]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool;
    CK(cudaMemPoolCreate(&pool, &props));
    uint64_t keep = ~0ull;
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    g_pools[device] = pool;
  }
  return g_pools[device];
}

// cudaMallocAsync from the library pool of `device`
template <class T>
void pool_malloc(T** ptr, size_t bytes, cudaStream_t stream, int device) {
  CK(cudaMallocFromPoolAsync((void**)ptr, bytes, lib_pool(device), stream));
}

}  // namespace

// Slot codec over Z_t (batching.py:41-95): u64 negacyclic NTT tables.
struct hcnn_codec {
  int device = 0;
  uint32_t n = 0, logn = 0;
  uint64_t t = 0, zeta = 0;
  ulonglong2* d_tw = nullptr;
  ulonglong2* d_itw = nullptr;
  ulonglong2 ninv{}, ninv_w{};  // N^-1 and psi^-N/2 N^-1 (the last inverse stage), Shoup
};

struct hcnn_weights {
  size_t count = 0;
  double* wd = nullptr;   // |w| < 2^22: exact FP64 MAC path
  int flush = 0;          // taps between exact mod-p folds on that path
  int small = 0;          // all |w| < 2^15: biased u16 path
  uint16_t* wb = nullptr; // [count] biased (small)
  uint32_t* wred = nullptr;  // [count][K] residues mod q_i (general)
};

struct hcnn_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  uint32_t N = 0, logN = 0, K = 0, KP = 0, D = 0, log2w = 0;
  uint64_t t = 0;
  std::vector<u64> primes;  // Q then P
  std::vector<u64> psi;
  ConvTabs tabs{};
  NttTabs nt{};
  uint32_t* d_prime = nullptr;
  uint64_t* d_mu = nullptr;
  uint2* d_tw = nullptr;
  uint2* d_itw = nullptr;
  uint2* d_ninv = nullptr;
  uint32_t* d_pinv = nullptr;
  uint32_t* d_rlk = nullptr;      // NTT domain, tiled layout of `keys_variant`
  uint32_t* d_rlk_raw = nullptr;  // as uploaded (domain rlk_domain)
  int rlk_domain = 0;
  uint32_t* d_pk = nullptr;
  uint32_t* d_pk_raw = nullptr;
  uint32_t* d_sk = nullptr;  // secret key s, NTT domain (spectral positions), [K][N]
  int pk_domain = 0;
  int variant = 0;       // NTT radix variant of the fused kernels (0 = default)
  int keys_variant = -1; // variant the tiled keys were laid out for
  // relinearisation over R (RELIN_RBASIS): usable when D <= RB_DMAX and
  // R > 2 (D N (w-1) max q_j / 2 + r0 r1)
  bool rb_ok = false;
  RbTabs rb{};
  uint32_t* d_rlk_rb = nullptr;  // [RB_A][D][2K][N] NTT domain mod r_a, tiled
  bool rb_keys = false;
  uint8_t* d_rlk_tc = nullptr;  // [RB_A][N][RBT_BT] byte-split key matrices (RB_MAC_TC)
  bool rb_tc_keys = false;
  // base conversions on the tensor cores (TC_BCONV, tc_bconv.cuh): usable
  // when K, KP <= 15 and 128 | N
  bool tc_ok = false;
  uint32_t* d_tcb = nullptr;  // the two 4 KB byte matrices
  TcTabs tc{};
  uint2* d_delta = nullptr;
  bool rlk_reduce = false;
  uint8_t* ws = nullptr;
  size_t ws_bytes = 0;
  // memory for the multiply / relinearisation scratch (the workspace plus the
  // R-basis spectra): whole MNIST layers (800 cts at set 1) in one chunk
  size_t ws_limit = size_t(12) << 30;
  size_t ts_sub = 0;  // ciphertexts per extend/tensor/scale sub-chunk (0: whole chunk)
  // smallest batch relinearised over R (below it the per-prime kernel is
  // faster: set 1, 8 cts 20.2 vs 23.6 us, 16 cts 18.5 vs 16.8 us per ct)
  size_t rb_min_batch = 12;
  int64_t launches = 0;
  cudaEvent_t switch_ev = nullptr;  // orders the old stream before the new one (hcnn_ctx_set_stream)

  uint8_t* workspace(size_t bytes) {
    if (bytes > ws_bytes) {
      if (ws) CK(cudaFreeAsync(ws, stream));
      ws = nullptr;
      ws_bytes = 0;
      pool_malloc(&ws, bytes, stream, device);
      ws_bytes = bytes;
    }
    return ws;
  }
  // per-launch CUDA events on the launching stream (hcnn_profile): kernel i
  // spans [event after launch i-1 (or the call's mark), event after launch i]
  struct ProfRec {
    const char* name;
    cudaEvent_t a, b;
  };
  bool prof = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> ev_pool, ev_used;
  cudaEvent_t last_ev = nullptr;
  cudaEvent_t new_event() {
    cudaEvent_t e;
    if (ev_pool.empty()) {
      CK(cudaEventCreate(&e));
    } else {
      e = ev_pool.back();
      ev_pool.pop_back();
    }
    ev_used.push_back(e);
    return e;
  }
  void mark() {
    if (!prof) return;
    last_ev = new_event();
    CK(cudaEventRecord(last_ev, stream));
  }
  void launched(const char* what) {
    ++launches;
    check_cuda(cudaGetLastError(), what);
    if (prof) {
      if (!last_ev) mark();
      cudaEvent_t e = new_event();
      CK(cudaEventRecord(e, stream));
      recs.push_back({what, last_ev, e});
      last_ev = e;
    }
  }
  void prof_reset() {
    for (auto e : ev_used) ev_pool.push_back(e);
    ev_used.clear();
    recs.clear();
    last_ev = nullptr;
  }
};

namespace {

// fixed point x/m ~ (x * g << k) / 2^59 with g = floor(2^(59-k)/m) < 2^32
void fixed59(u64 m, uint32_t* g, uint32_t* k) {
  uint32_t kk = 0;
  while ((((u128)1 << (59 - kk)) / m) >> 32) ++kk;
  *g = (uint32_t)(((u128)1 << (59 - kk)) / m);
  *k = kk;
}

uint32_t neg_inv32(uint32_t p) {
  uint32_t inv = 1;  // Newton: p^-1 mod 2^32
  for (int it = 0; it < 5; ++it) inv *= 2u - p * inv;
  return 0u - inv;
}

u64 mont_form(u64 x, u64 p) { return (u64)(((u128)x << 32) % p); }

void build_tables(hcnn_ctx* c, const std::vector<u64>& q, uint64_t t) {
  const uint32_t N = c->N;
  // q, h = (q-1)/2, relin digit count l+1 (bfv.py:68-76)
  Big Q = product(q);
  {
    Big acc(1);
    for (uint32_t i = 0; i < c->log2w; ++i) acc = mul_small(acc, 2);
    Big wpow = acc;
    uint32_t l = 0;
    while (cmp(wpow, Q) <= 0) {
      for (uint32_t i = 0; i < c->log2w; ++i) wpow = mul_small(wpow, 2);
      ++l;
    }
    c->D = l + 1;
  }
  if (c->D > (uint32_t)DMAX) fail(HCNN_ERR_UNSUPPORTED, "too many relinearisation digits");
  // auxiliary base: P > 8 t N q + 4 so that round(t d / q) is centred in P
  // with |y| < P/4 (exact rounding, no ambiguity).  KP = K+2 covers t below
  // ~2^45 with 30-bit primes; K+3 is always enough (t < 2^64, N <= 2^15).
  Big bound = mul_small(mul_small(mul_small(Q, t), N), 8);
  bound = add(bound, Big(4));
  std::vector<u64> P;
  Big Pp(1);
  {
    std::vector<u64> cand = aux_primes(q, c->K + 3);
    for (u64 p : cand) {
      if (P.size() >= c->K + 2 && cmp(Pp, bound) > 0) break;
      P.push_back(p);
      Pp = mul_small(Pp, p);
    }
    if (cmp(Pp, bound) <= 0 || P.size() > (size_t)KPMAX)
      fail(HCNN_ERR_UNSUPPORTED, "auxiliary base too small for this t");
  }
  c->KP = (uint32_t)P.size();
  c->primes = q;
  c->primes.insert(c->primes.end(), P.begin(), P.end());
  // R: three primes = 1 mod 2^17 with D (r - 1)^2 < 2^64 for D <= RB_DMAX
  std::vector<u64> R;
  {
    const u64 rmax = 895562590ull;  // 23 (rmax - 1)^2 < 2^64
    for (u64 k = rmax >> 17; R.size() < (size_t)RB_A && k > 1; --k) {
      const u64 r = (k << 17) + 1;
      if (r > rmax || std::find(c->primes.begin(), c->primes.end(), r) != c->primes.end()) continue;
      if (is_prime64(r)) R.push_back(r);
    }
    c->primes.insert(c->primes.end(), R.begin(), R.end());
  }
  const uint32_t L = c->K + c->KP + RB_A;

  // NTT tables
  std::vector<uint32_t> hp(L);
  std::vector<uint64_t> hmu(L);
  std::vector<uint2> htw((size_t)L * N), hitw((size_t)L * N), hninv(4 * L);
  std::vector<uint32_t> hpinv(L);
  c->psi.resize(L);
  for (uint32_t j = 0; j < L; ++j) {
    const u64 p = c->primes[j];
    const u64 psi = primitive_2n_root(p, N);
    const u64 ipsi = invmod64(psi, p);
    c->psi[j] = psi;
    hp[j] = (uint32_t)p;
    hmu[j] = (uint64_t)(((u128)1 << 64) / p);
    {
      uint32_t inv = 1;  // Newton iteration for p^-1 mod 2^32
      for (int it = 0; it < 5; ++it) inv *= 2u - (uint32_t)p * inv;
      hpinv[j] = (uint32_t)(0u - inv);
    }
    std::vector<u64> pw(N), ipw(N);
    pw[0] = ipw[0] = 1;
    for (uint32_t i = 1; i < N; ++i) {
      pw[i] = mulmod64(pw[i - 1], psi, p);
      ipw[i] = mulmod64(ipw[i - 1], ipsi, p);
    }
    for (uint32_t i = 0; i < N; ++i) {
      const uint32_t r = bitrev(i, c->logN);
      htw[(size_t)j * N + i] = make_uint2((uint32_t)pw[r], shoup_of((uint32_t)pw[r], (uint32_t)p));
      hitw[(size_t)j * N + i] = make_uint2((uint32_t)ipw[r], shoup_of((uint32_t)ipw[r], (uint32_t)p));
    }
    const uint32_t ninv = (uint32_t)invmod64(N % p, p);
    hninv[j] = make_uint2(ninv, shoup_of(ninv, (uint32_t)p));
    const uint32_t ninv_m = (uint32_t)mont_form(ninv, p);
    hninv[L + j] = make_uint2(ninv_m, shoup_of(ninv_m, (uint32_t)p));
    const uint32_t wl = (uint32_t)ipw[N / 2];  // twiddle of the last inverse stage (itw[1])
    const uint32_t nw = (uint32_t)mulmod64(wl, ninv, p), nmw = (uint32_t)mulmod64(wl, ninv_m, p);
    hninv[2 * L + j] = make_uint2(nw, shoup_of(nw, (uint32_t)p));
    hninv[3 * L + j] = make_uint2(nmw, shoup_of(nmw, (uint32_t)p));
  }

  // relinearisation over R: CRT constants and the exactness bound
  {
    RbTabs& rb = c->rb;
    std::memset(&rb, 0, sizeof(rb));
    rb.roff = (int)(c->K + c->KP);
    auto shp = [](u64 w, u64 m) { return make_uint2((uint32_t)w, shoup_of((uint32_t)w, (uint32_t)m)); };
    u128 Rp = 1;
    for (int a = 0; a < RB_A; ++a) Rp *= R[a];
    for (int a = 0; a < RB_A; ++a) {
      const u64 r = R[a];
      rb.r[a] = (uint32_t)r;
      rb.t32[a] = shp(((u64)1 << 32) % r, r);
      rb.one[a] = shoup_of(1, (uint32_t)r);
      rb.rpinv[a] = neg_inv32((uint32_t)r);
      const u64 g = invmod64((u64)((Rp / r) % r), r);  // (R/r_a)^-1 mod r_a
      const uint32_t jj = (uint32_t)rb.roff + a;
      rb.isc_n[a] = shp(mulmod64(hninv[jj].x, g, r), r);
      rb.isc_nw[a] = shp(mulmod64(hninv[2 * L + jj].x, g, r), r);
      rb.rinv[a] = (float)(1.0 / (double)r);
    }
    u64 qmax = 0;
    for (uint32_t j = 0; j < c->K; ++j) {
      const u64 qj = q[j];
      qmax = qj > qmax ? qj : qmax;
      for (int a = 0; a < RB_A; ++a) rb.crt_q[j][a] = (uint32_t)mont_form((u64)((Rp / R[a]) % qj), qj);
      rb.negR_q[j] = (uint32_t)mont_form((qj - (u64)(Rp % qj)) % qj, qj);
    }
    // |Z| <= D N (w - 1) floor(q_j / 2) must stay below R/4: then
    // sum_a x~_a / r_a lies within 1/4 of the integer v and the fp32 estimate
    // (error below 2^-20) rounds to it
    const u128 zmax = (u128)c->D * N * (((u128)1 << c->log2w) - 1) * (qmax / 2);
    c->rb_ok = R.size() == (size_t)RB_A && c->D <= (uint32_t)RB_DMAX && zmax < (Rp >> 2);
  }

  // exact base conversion and scaling constants
  ConvTabs& tb = c->tabs;
  std::memset(&tb, 0, sizeof(tb));
  tb.K = (int)c->K;
  tb.KP = (int)c->KP;
  tb.D = (int)c->D;
  tb.digit_bits = (int)c->log2w;
  const Big Kq = mul_small(Q, c->K + 1);
  tb.W = (Kq.bits() + 31) / 32 + 1;
  if (tb.W > WMAX) fail(HCNN_ERR_UNSUPPORTED, "q too large");
  for (int w2 = 0; w2 < WMAX; ++w2) tb.q_w[w2] = Q.word(w2);
  const Big h = shr1(Q);  // (q-1)/2, q odd
  for (uint32_t i = 0; i < c->K; ++i) {
    const u64 qi = q[i];
    tb.q[i] = (uint32_t)qi;
    tb.qmu[i] = (uint64_t)(((u128)1 << 64) / qi);
    const Big qhat = div_small(Q, qi);
    const u64 qhi = invmod64(mod_small(qhat, qi), qi);
    tb.qhi[i] = (uint32_t)qhi;
    tb.qhis[i] = shoup_of((uint32_t)qhi, (uint32_t)qi);
    fixed59(qi, &tb.qg[i], &tb.qk[i]);
    tb.qpinv[i] = neg_inv32((uint32_t)qi);
    for (int w2 = 0; w2 < WMAX; ++w2) tb.qhat_w[i][w2] = qhat.word(w2);
    for (uint32_t j = 0; j < c->KP; ++j) tb.qhat_p[i][j] = (uint32_t)mont_form(mod_small(qhat, P[j]), P[j]);
    // scale: r~_i = (t d + h) qhi = d (t qhi) + h qhi
    const u64 A = mulmod64(t % qi, qhi, qi);
    tb.A[i] = (uint32_t)A;
    tb.As[i] = shoup_of((uint32_t)A, (uint32_t)qi);
    tb.B[i] = (uint32_t)mulmod64(mod_small(h, qi), qhi, qi);
  }
  for (uint32_t j = 0; j < c->KP; ++j) {
    const u64 pj = P[j];
    tb.p[j] = (uint32_t)pj;
    tb.pmu[j] = (uint64_t)(((u128)1 << 64) / pj);
    tb.negq_p[j] = (uint32_t)mont_form((pj - mod_small(Q, pj)) % pj, pj);
    tb.ppinv[j] = neg_inv32((uint32_t)pj);
    const Big phat = div_small(Pp, pj);
    const u64 phi = invmod64(mod_small(phat, pj), pj);
    fixed59(pj, &tb.pg[j], &tb.pk[j]);
    for (uint32_t i = 0; i < c->K; ++i) tb.phat_q[j][i] = (uint32_t)mont_form(mod_small(phat, q[i]), q[i]);
    // y~_j = (t d + h - r) q^-1 phi = d C + (p - r) E + F
    const u64 E = mulmod64(invmod64(mod_small(Q, pj), pj), phi, pj);
    const u64 C = mulmod64(t % pj, E, pj);
    tb.C[j] = (uint32_t)C;
    tb.Cs[j] = shoup_of((uint32_t)C, (uint32_t)pj);
    tb.Ej[j] = (uint32_t)E;
    tb.Ejs[j] = shoup_of((uint32_t)E, (uint32_t)pj);
    tb.F[j] = (uint32_t)mulmod64(mod_small(h, pj), E, pj);
  }
  for (uint32_t i = 0; i < c->K; ++i)
    tb.negp_q[i] = (uint32_t)mont_form((q[i] - mod_small(Pp, q[i])) % q[i], q[i]);
  // decryption rounding constants (usable when t < 2^48)
  tb.t = t;
  tb.tmu = (uint64_t)(((u128)1 << 64) / t);
  for (uint32_t i = 0; i < c->K; ++i) {
    tb.dec_a[i] = t / q[i];
    tb.dec_f[i] = (uint32_t)(t % q[i]);
  }
  {
    // H = floor(h 2^59 / q) from the top words of h and q
    Big h59 = h;
    for (int b = 0; b < 59; ++b) h59 = mul_small(h59, 2);
    // long division h59 / Q by repeated subtraction of shifted Q is costly;
    // h/q = 1/2 - 1/(2q), so H = 2^58 - 1 exactly for q > 2^60
    if (Q.bits() > 61) {
      tb.H = (1ull << 58) - 1;  // h/q = 1/2 - 1/(2q), q > 2^61
    } else {
      u128 hq = 0, qq = 0;
      for (int w2 = 3; w2 >= 0; --w2) {
        hq = (hq << 32) | h.word(w2);
        qq = (qq << 32) | Q.word(w2);
      }
      tb.H = (uint64_t)((hq << 59) / qq);
    }
    (void)h59;
  }
  for (int w2 = 0; w2 < WMAX; ++w2) tb.h_w[w2] = h.word(w2);

  // tensor-core conversion matrices (tc_bconv.cuh): B[4o+e][4i+b] =
  // byte e of (2^8b c_io 2^32 mod m_o); input i = nin is the overflow count v
  c->tc_ok = c->K <= 15 && c->KP <= 15 && N % TC_M == 0;
  if (c->tc_ok) {
    std::vector<uint8_t> hb(4 * TC_N * TC_KB, 0);
    auto fill = [&](uint8_t* B, uint32_t nin, uint32_t nout, auto cin, auto cv, auto mod) {
      for (uint32_t o = 0; o < nout; ++o) {
        const u64 m = mod(o);
        for (uint32_t i = 0; i <= nin; ++i) {
          const u64 cc = i < nin ? cin(i, o) : cv(o);
          for (int b = 0; b < (i < nin ? 4 : 1); ++b) {
            const u64 cp = mont_form(mulmod64(cc, ((u64)1 << (8 * b)) % m, m), m);
            for (int e = 0; e < 4; ++e) B[tc_off(4 * (int)o + e, 4 * (int)i + b)] = (uint8_t)(cp >> (8 * e));
          }
        }
      }
    };
    fill(hb.data(), c->K, c->KP, [&](uint32_t i, uint32_t j) { return mod_small(div_small(Q, q[i]), P[j]); },
         [&](uint32_t j) { return (P[j] - mod_small(Q, P[j])) % P[j]; }, [&](uint32_t j) { return P[j]; });
    // the scale's Q -> P conversion with -E_j folded in: (p_j - r_j) E_j directly
    fill(hb.data() + 3 * TC_N * TC_KB, c->K, c->KP,
         [&](uint32_t i, uint32_t j) {
           return mulmod64(mod_small(div_small(Q, q[i]), P[j]), (P[j] - tb.Ej[j]) % P[j], P[j]);
         },
         [&](uint32_t j) { return mulmod64((P[j] - mod_small(Q, P[j])) % P[j], (P[j] - tb.Ej[j]) % P[j], P[j]); },
         [&](uint32_t j) { return P[j]; });
    fill(hb.data() + TC_N * TC_KB, c->KP, c->K,
         [&](uint32_t j, uint32_t i) { return mod_small(div_small(Pp, P[j]), q[i]); },
         [&](uint32_t i) { return (q[i] - mod_small(Pp, q[i])) % q[i]; }, [&](uint32_t i) { return q[i]; });
    // the digits' canonical lift: row s = byte s of sum_i xt_i (q/q_i) + V (2^(32 W) - q),
    // W = words_for(K) (the words the kernel carries; the lift is < 2q there)
    {
      uint8_t* B = hb.data() + 2 * TC_N * TC_KB;
      const int W = words_for((int)c->K);
      auto byte_of = [](const Big& x, int k) { return (uint8_t)(x.word(k / 4) >> (8 * (k % 4))); };
      for (uint32_t i = 0; i < c->K; ++i) {
        const Big qh = div_small(Q, q[i]);
        for (int b = 0; b < 4; ++b)
          for (int sb = b; sb < 4 * W; ++sb) B[tc_off(sb, 4 * (int)i + b)] = byte_of(qh, sb - b);
      }
      uint64_t cy = 1;
      for (int w2 = 0; w2 < W; ++w2) {  // two's complement words of q
        const uint64_t x = (uint64_t)(~Q.word(w2) & 0xffffffffu) + cy;
        cy = x >> 32;
        for (int u = 0; u < 4; ++u) B[tc_off(4 * w2 + u, 4 * (int)c->K)] = (uint8_t)(x >> (8 * u));
      }
    }
    CK(cudaMalloc(&c->d_tcb, hb.size()));
    CK(cudaMemcpy(c->d_tcb, hb.data(), hb.size(), cudaMemcpyHostToDevice));
    c->tc = TcTabs{c->d_tcb, c->d_tcb + TC_N * TC_KB / 4, c->d_tcb + 3 * TC_N * TC_KB / 4,
                   c->d_tcb + 2 * TC_N * TC_KB / 4};
  }

  // upload
  CK(cudaMalloc(&c->d_prime, L * sizeof(uint32_t)));
  CK(cudaMalloc(&c->d_mu, L * sizeof(uint64_t)));
  CK(cudaMalloc(&c->d_tw, (size_t)L * N * sizeof(uint2)));
  CK(cudaMalloc(&c->d_itw, (size_t)L * N * sizeof(uint2)));
  CK(cudaMalloc(&c->d_ninv, 4 * L * sizeof(uint2)));
  CK(cudaMalloc(&c->d_pinv, L * sizeof(uint32_t)));
  CK(cudaMemcpy(c->d_pinv, hpinv.data(), L * sizeof(uint32_t), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_prime, hp.data(), L * sizeof(uint32_t), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_mu, hmu.data(), L * sizeof(uint64_t), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_tw, htw.data(), (size_t)L * N * sizeof(uint2), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_itw, hitw.data(), (size_t)L * N * sizeof(uint2), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_ninv, hninv.data(), 4 * L * sizeof(uint2), cudaMemcpyHostToDevice));
  c->nt = NttTabs{c->d_prime, c->d_mu, c->d_tw, c->d_itw, c->d_ninv, c->d_pinv, c->d_ninv + L, c->d_ninv + 2 * L,
                 c->d_ninv + 3 * L};
}

// ---------------------------------------------------------------- dispatch
int variant_mont(hcnn_ctx* c, int v) {
  switch (c->logN) {
#define X(L) \
  case L:    \
    return hcnn_ntt_mont_##L(v);
    HCNN_LOGN_LIST(X)
#undef X
  }
  return 0;
}

void ntt_dispatch(hcnn_ctx* c, int op, NttLaunch& a, const char* what) {
  a.stream = c->stream;
  a.nt = c->nt;
  a.variant = c->variant;
  cudaError_t e;
  switch (c->logN) {
#define X(L)                              \
  case L:                                 \
    e = hcnn_ntt_launch_##L(op, a);       \
    break;
    HCNN_LOGN_LIST(X)
#undef X
    default:
      fail(HCNN_ERR_UNSUPPORTED, "ring degree");
  }
  c->launched(what);
  check_cuda(e, what);
}

void launch_ntt_rows(hcnn_ctx* c, uint32_t* rows, size_t n_rows, int limbs, int off, int inverse) {
  if (n_rows == 0) return;
  NttLaunch a{};
  a.grid = dim3((unsigned)n_rows);
  a.rows = rows;
  a.limbs = limbs;
  a.prime_off = off;
  a.inverse = inverse;
  ntt_dispatch(c, 0, a, "k_ntt_rows");
}

void launch_tensor(hcnn_ctx* c, const uint32_t* a_, const uint32_t* ae, const uint32_t* b,
                   const uint32_t* be, uint32_t* d, size_t nct, int square) {
  NttLaunch a{};
  a.grid = dim3(c->K + c->KP, (unsigned)nct);
  a.a = a_;
  a.ae = ae;
  a.b = b;
  a.be = be;
  a.d = d;
  a.K = (int)c->K;
  a.KP = (int)c->KP;
  a.square = square;
  ntt_dispatch(c, 1, a, "k_tensor");
}

void prepare_keys(hcnn_ctx* c);

unsigned cdiv(size_t a, size_t b) { return (unsigned)((a + b - 1) / b); }

// variant bit: relinearisation over the shared basis R (relin_rb.cuh)
constexpr int RELIN_RBASIS = 16384;
constexpr int TC_BCONV = 32768;  // k_extend / k_scale on the tensor cores (tc_bconv.cuh)

bool tc_active(const hcnn_ctx* c) { return (c->variant & TC_BCONV) && c->tc_ok; }
constexpr size_t TC_MIN_BATCH = 12;  // ciphertexts per multiply chunk for the tensor-core conversions

bool rb_active(const hcnn_ctx* c) {
  if (!(c->variant & RELIN_RBASIS) || !c->rb_ok) return false;
  // 3 D + 6 K transforms and 3x the products against D K + 2 K transforms:
  // below ~8 primes the per-prime path is as fast or faster (measured at
  // 2^15: K = 6 17.0 vs 14.7 us, K = 11 32.2 vs 43.2 us per ciphertext)
  if (c->K < 8) return false;
  if (c->logN == 12 || c->logN == 13) return !(c->variant & 64);  // radix-16 shuffle-tail kernels
  if (c->logN == 14) return !(c->variant & 512);                   // one-row kernels (not the 2^14 cluster)
  if (c->logN == 15) return (c->variant & 512) != 0;               // 2-CTA cluster kernels
  return false;
}

// key rows mod r_a in the NTT domain (tiled layout of the R kernels' geometry)
void prepare_rb_keys(hcnn_ctx* c) {
  if (c->rb_keys || !c->d_rlk_raw) return;
  const size_t N = c->N, K = c->K, D = c->D, rows = D * 2 * K;
  uint32_t* coef = nullptr;
  pool_malloc(&coef, rows * N * sizeof(uint32_t), c->stream, c->device);
  if (c->rlk_domain == HCNN_DOMAIN_REF_NTT) {
    k_ref_to_spectral<<<dim3(cdiv(N, 256), (unsigned)rows), 256, 0, c->stream>>>(c->d_rlk_raw, coef, (int)c->logN);
    c->launched("k_ref_to_spectral");
    launch_ntt_rows(c, coef, rows, (int)K, 0, 1);  // back to the coefficient domain mod q_j
  } else {
    CK(cudaMemcpyAsync(coef, c->d_rlk_raw, rows * N * sizeof(uint32_t), cudaMemcpyDeviceToDevice, c->stream));
  }
  if (!c->d_rlk_rb) CK(cudaMalloc((void**)&c->d_rlk_rb, RB_A * rows * N * sizeof(uint32_t)));
  k_rb_key_rows<<<cdiv(rows * N, 256), 256, 0, c->stream>>>(coef, c->d_rlk_rb, (int)D, (int)K, (int)N, c->d_prime,
                                                           c->rb);
  c->launched("k_rb_key_rows");
  for (int a = 0; a < RB_A; ++a)
    launch_ntt_rows(c, c->d_rlk_rb + a * rows * N, rows, 1, c->rb.roff + a, 2);
  CK(cudaFreeAsync(coef, c->stream));
  c->rb_keys = true;
  c->rb_tc_keys = false;
}

// variant bit: the relinearisation multiply-accumulate on the tensor cores
constexpr int RB_MAC_TC = 65536;

bool rb_mac_tc(const hcnn_ctx* c) {
  return (c->variant & RB_MAC_TC) && c->D <= 23 && 2 * c->K <= RBT_N / 4 && c->N % (4 * RBT_NB) == 0;
}

void prepare_rb_tc_keys(hcnn_ctx* c) {
  if (c->rb_tc_keys) return;
  const size_t N = c->N, K = c->K, D = c->D;
  const size_t bytes = (size_t)RB_A * N * RBT_BT;
  if (!c->d_rlk_tc) CK(cudaMalloc((void**)&c->d_rlk_tc, bytes));
  CK(cudaMemsetAsync(c->d_rlk_tc, 0, bytes, c->stream));
  const size_t total = (size_t)RB_A * D * 2 * K * N;
  k_rb_key_tc<<<cdiv(total, 256), 256, 0, c->stream>>>(c->d_rlk_rb, c->d_rlk_tc, (int)D, (int)(2 * K), (int)N,
                                                      c->rb);
  c->launched("k_rb_key_tc");
  c->rb_tc_keys = true;
}

template <int DD>
void rb_mac_launch(hcnn_ctx* c, const uint32_t* ds, uint32_t* zs, size_t nct) {
  if (rb_mac_tc(c)) {
    static std::atomic<uint64_t> cfg_tc{0};
    per_device_once(cfg_tc, [] {
      cudaFuncSetAttribute(k_rb_mac_tc<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(RbtSmem));
    });
    prepare_rb_tc_keys(c);
    k_rb_mac_tc<DD><<<dim3(c->N / RBT_NB, RB_A), RBT_T, sizeof(RbtSmem), c->stream>>>(
        ds, c->d_rlk_tc, zs, (int)nct, (int)c->K, (int)c->N, c->rb);
    return;
  }
  static std::atomic<uint64_t> cfg{0};
  per_device_once(cfg, [] {
    cudaFuncSetAttribute(k_rb_mac<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
  });
  const size_t smem = (size_t)DD * 2 * c->K * RB_MAC_QD * sizeof(uint4);
  const int cpc = 256;  // ciphertexts per CTA (measured 32-512: 256 best, 1.82 vs 1.87 us at 128)
  k_rb_mac<DD><<<dim3(c->N / RB_MAC_C, RB_A, cdiv(nct, cpc)), RB_MAC_T, smem, c->stream>>>(
      ds, c->d_rlk_rb, zs, (int)nct, (int)c->K, (int)c->N, cpc, c->rb);
}

void launch_rb_mac(hcnn_ctx* c, const uint32_t* ds, uint32_t* zs, size_t nct) {
  switch (c->D) {
#define X(DD)                            \
  case DD:                               \
    rb_mac_launch<DD>(c, ds, zs, nct);   \
    break;
    X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12)
    X(13) X(14) X(15) X(16) X(17) X(18) X(19) X(20) X(21) X(22) X(23)
#undef X
    default:
      fail(HCNN_ERR_UNSUPPORTED, "relinearisation over R: digit count");
  }
  c->launched(rb_mac_tc(c) ? "k_rb_mac_tc" : "k_rb_mac");
}

// relinearisation over R: digit spectra mod r_a, multiply-accumulate with
// the key, inverse + exact CRT to q_j + (y0, y1)
void launch_relin_rb(hcnn_ctx* c, const uint32_t* dig, const uint32_t* y3, uint32_t* out, size_t nct) {
  prepare_rb_keys(c);
  const size_t N = c->N, K = c->K, D = c->D;
  uint32_t *ds = nullptr, *zs = nullptr;
  pool_malloc(&ds, nct * RB_A * D * N * sizeof(uint32_t), c->stream, c->device);
  pool_malloc(&zs, nct * K * RB_A * 2 * N * sizeof(uint32_t), c->stream, c->device);
  NttLaunch f{};
  // digits split over up to 4 CTAs per (r_a, ct) when the batch alone would
  // give fewer than 6 waves of one CTA per SM
  unsigned split = 1;
  while (split < 4 && (size_t)RB_A * nct * split < 6 * 148) split *= 2;
  f.grid = dim3(RB_A, (unsigned)nct, split);
  f.dig = dig;
  f.out = ds;
  f.D = (int)D;
  f.reduce_digits = c->log2w >= 30 ? 1 : 0;
  f.rb = c->rb;
  ntt_dispatch(c, 7, f, "k_rb_fwd");
  launch_rb_mac(c, ds, zs, nct);
  NttLaunch b{};
  b.grid = dim3((unsigned)K, (unsigned)nct);
  b.a = zs;
  b.y3 = y3;
  b.out = out;
  b.K = (int)K;
  b.rb = c->rb;
  ntt_dispatch(c, 8, b, "k_rb_inv");
  CK(cudaFreeAsync(ds, c->stream));
  CK(cudaFreeAsync(zs, c->stream));
}

void launch_relin(hcnn_ctx* c, const uint32_t* dig, const uint32_t* y3, uint32_t* out, size_t nct) {
  if (rb_active(c) && c->d_rlk_raw && nct >= c->rb_min_batch) {
    launch_relin_rb(c, dig, y3, out, nct);
    return;
  }
  prepare_keys(c);
  NttLaunch a{};
  a.rlk_mont = variant_mont(c, c->variant);
  a.grid = dim3(c->K, (unsigned)nct);
  a.dig = dig;
  a.y3 = y3;
  a.rlk = c->d_rlk;
  a.out = out;
  a.K = (int)c->K;
  a.D = (int)c->D;
  a.reduce_digits = c->rlk_reduce ? 1 : 0;
  ntt_dispatch(c, 2, a, "k_relin");
}

// scratch of the relinearisation over R per ciphertext (digit spectra and
// the multiply-accumulate output; allocated from the library pool per call)
size_t rb_bytes_per_ct(const hcnn_ctx* c) {
  return rb_active(c) ? ((size_t)RB_A * c->D + (size_t)c->K * RB_A * 2) * c->N * sizeof(uint32_t) : 0;
}

// bytes of workspace per ciphertext of a multiply chunk
size_t mul_ws_per_ct(hcnn_ctx* c, bool general) {
  const size_t N = c->N, K = c->K, KP = c->KP;
  size_t b = (general ? 2 : 1) * 2 * KP * N;  // extensions
  b += 3 * (K + KP) * N;                      // tensor
  b += 3 * K * N;                             // scaled 3-part
  b += (size_t)c->D * N;                      // digits
  return b * sizeof(uint32_t);
}

size_t chunk_cts(hcnn_ctx* c, size_t n, bool general, bool relin) {
  const size_t per = mul_ws_per_ct(c, general) + (relin ? rb_bytes_per_ct(c) : 0);
  size_t ch = c->ws_limit / per;
  if (ch < 1) ch = 1;
  if (ch > 16384) ch = 16384;
  return ch < n ? ch : n;
}

void conv_dispatch(hcnn_ctx* c, int op, ConvLaunch& a, const char* what) {
  a.stream = c->stream;
  a.N = (int)c->N;
  cudaError_t e = cudaErrorInvalidValue;
  switch (c->K) {
#define X(KK)                                                \
  case KK:                                                   \
    e = hcnn_conv_launch_##KK(op, (int)c->KP, a, c->tabs);   \
    break;
    HCNN_K_LIST(X)
#undef X
    default:
      fail(HCNN_ERR_UNSUPPORTED, "prime count");
  }
  c->launched(what);
  check_cuda(e, what);
}

// a (and b) -> out3 (3-part scaled) and, if dig, the digits of part 2
void mul_chunk(hcnn_ctx* c, const uint32_t* a, const uint32_t* b, size_t nct, uint32_t* y3,
               uint32_t* dig, uint8_t* ws) {
  const size_t N = c->N, K = c->K, KP = c->KP;
  const bool square = (a == b);
  uint32_t* ae = (uint32_t*)ws;
  uint32_t* be = square ? ae : ae + nct * 2 * KP * N;
  uint32_t* d = be + nct * 2 * KP * N;
  const unsigned tpb = 128;
  ConvLaunch ca{};
  ca.block = dim3(tpb);
  ca.grid = dim3(cdiv(N, tpb), (unsigned)(nct * 2));
  // a handful of ciphertexts: the integer kernels' shorter latency wins
  // (set 1, one HSquare 0.119 vs 0.123 ms; 8 cts 20.5 vs 20.8 us each)
  const bool tc = tc_active(c) && nct >= TC_MIN_BATCH;
  ca.tc = &c->tc;
  ca.tiles = nct * 2 * (N / TC_M);
  ca.in = a;
  ca.out = ae;
  conv_dispatch(c, tc ? 4 : 0, ca, tc ? "k_extend_tc" : "k_extend");
  if (!square) {
    ca.in = b;
    ca.out = be;
    conv_dispatch(c, tc ? 4 : 0, ca, tc ? "k_extend_tc" : "k_extend");
  }
  launch_tensor(c, a, ae, b, be, d, nct, square ? 1 : 0);
  ca.grid = dim3(cdiv(N, tpb), (unsigned)(nct * 3));
  ca.tiles = nct * 3 * (N / TC_M);
  ca.in = d;
  ca.out = y3;
  ca.dig = dig;
  conv_dispatch(c, tc ? 5 : 1, ca, tc ? "k_scale_tc" : "k_scale");
  (void)K;
}

void require_rlk(hcnn_ctx* c) {
  if (!c->d_rlk) fail(HCNN_ERR_MISSING_KEY, "relinearization key required");
}

// y3 = hmult_raw(a, b); optionally relinearised into out
void multiply(hcnn_ctx* c, const uint32_t* a, const uint32_t* b, size_t n, uint32_t* out3,
              uint32_t* out2) {
  if (n == 0) return;
  const size_t N = c->N, K = c->K;
  const bool general = a != b;
  const size_t ch = chunk_cts(c, n, general, out2 != nullptr);
  const size_t per = mul_ws_per_ct(c, general);
  uint8_t* ws = c->workspace(per * ch);
  const size_t ext_bytes = ((general ? 2 : 1) * 2 * c->KP + 3 * (K + c->KP)) * N * sizeof(uint32_t);
  for (size_t s = 0; s < n; s += ch) {
    const size_t m = (n - s < ch) ? n - s : ch;
    const uint32_t* ac = a + s * 2 * K * N;
    const uint32_t* bc = b + s * 2 * K * N;
    uint32_t* y3 = out3 ? out3 + s * 3 * K * N : (uint32_t*)(ws + ext_bytes * ch);
    uint32_t* dig = out2 ? (uint32_t*)(ws + ext_bytes * ch + 3 * K * N * sizeof(uint32_t) * ch) : nullptr;
    // extend / tensor / scale in sub-chunks whose tensor output can stay in
    // L2 for k_scale (ts_sub; 0 = the whole chunk at once)
    const size_t sub = (c->ts_sub && c->ts_sub < m) ? c->ts_sub : m;
    for (size_t u = 0; u < m; u += sub) {
      const size_t mu = (m - u < sub) ? m - u : sub;
      mul_chunk(c, ac + u * 2 * K * N, (general ? bc : ac) + u * 2 * K * N, mu, y3 + u * 3 * K * N,
                dig ? dig + u * c->D * N : nullptr, ws);
    }
    if (out2) launch_relin(c, dig, y3, out2 + s * 2 * K * N, m);
  }
}

__global__ void k_sk_rows(const uint8_t* __restrict__ s, uint32_t* __restrict__ rows, int K, int N) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  for (int i = 0; i < K; ++i) rows[(size_t)i * N + n] = s[n];
}

// tmp[ct][i][:] = tmp * s_ntt[i] (NTT domain, same positions) mod q_i
__global__ void k_mul_sk(uint32_t* __restrict__ tmp, const uint32_t* __restrict__ sk, int K, int N,
                         size_t total, const uint32_t* __restrict__ primes, const uint64_t* __restrict__ mus) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int limb = (int)((i / N) % K);
  const size_t n = i % N;
  tmp[i] = mul_mod(tmp[i], sk[(size_t)limb * N + n], primes[limb], mus[limb]);
}

// tmp[ct][i][n] += c0[ct][i][n]; cts: [ct][2][K][N]
__global__ void k_add_c0(uint32_t* __restrict__ tmp, const uint32_t* __restrict__ cts, int K, int N,
                         size_t total, const uint32_t* __restrict__ primes) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const size_t kn = (size_t)K * N;
  const size_t ct = i / kn, r = i % kn;
  const int limb = (int)(r / N);
  tmp[i] = add_mod(tmp[i], cts[ct * 2 * kn + r], primes[limb]);
}

__global__ void k_hadd(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                       uint32_t* __restrict__ out, int K, int N, size_t total,
                       const uint32_t* __restrict__ primes) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int limb = (int)((i / N) % K);
  out[i] = add_mod(a[i], b[i], primes[limb]);
}

// FP64 FMA probe (kind 6): 8 independent chains per thread
__global__ void k_dfma_peak(uint32_t* out, double a, double b, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 7 + i + blockIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += x[i];
  if (acc == 1.2345) out[0] = 1;
}

// Harvey forward butterflies in registers (kind 8), 8 independent pairs per
// thread, fixed Shoup twiddle: the attainable butterfly rate of the integer
// pipes for the NTT kernels' instruction mix; counts butterflies
__global__ void k_bfly_peak(uint32_t* out, uint32_t w, uint32_t ws, uint32_t p, int iters) {
  uint32_t a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = (threadIdx.x * 7 + i + blockIdx.x) % p;
    b[i] = (threadIdx.x * 13 + 3 * i + blockIdx.x) % p;
  }
  const uint32_t p2 = 2 * p;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t X = a[i] < a[i] - p2 ? a[i] : a[i] - p2;
      const uint32_t T = b[i] * w - __umulhi(b[i], ws) * p;
      a[i] = X + T;
      b[i] = X - T + p2;
    }
#pragma unroll
    for (int i = 0; i < 8; i += 2) {  // mix the pairs like the next NTT stage
      const uint32_t t = a[i + 1];
      a[i + 1] = b[i];
      b[i] = t;
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc ^= a[i] ^ b[i];
  if (acc == 0x9e3779b9u) out[0] = acc;
}

// The u64 counterpart (kind 16): Harvey forward butterflies on 62-bit
// residues (mul_shoup64_lazy: one 64x64 high product, two 64-bit low
// products), the attainable rate of the u64 NTT's instruction mix
__global__ void k_bfly64_peak(uint32_t* out, uint64_t w, uint64_t ws, uint64_t p, int iters) {
  uint64_t a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = ((uint64_t)threadIdx.x * 7919 + i + blockIdx.x) % p;
    b[i] = ((uint64_t)threadIdx.x * 104729 + 3 * i + blockIdx.x) % p;
  }
  const uint64_t p2 = 2 * p;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint64_t X = csub64(a[i], p2);
      const uint64_t T = mul_shoup64_lazy(b[i], w, ws, p);
      a[i] = X + T;
      b[i] = X - T + p2;
    }
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      const uint64_t t = a[i + 1];
      a[i + 1] = b[i];
      b[i] = t;
    }
  }
  uint64_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc ^= a[i] ^ b[i];
  if (acc == 0x9e3779b97f4a7c15ull) out[0] = (uint32_t)acc;
}

// Butterfly cost decomposition probes (kinds 10-12), same chain structure as
// k_bfly_peak.  10: the quotient of b w / p from the fp64 pipe (exact to +-1:
// b -> double by the 2^52 trick, one DFMA with the magic 1.5 2^52 rounds it to
// an integer in the low mantissa word), 2 IMAD for the lazy remainder;
// 11: only the integer multiplies of a Shoup butterfly; 12: only its adds.
template <int KIND>
__global__ void k_bfly_probe(uint32_t* out, uint32_t w, uint32_t ws, uint32_t p, double wd, int iters) {
  uint32_t a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = (threadIdx.x * 7 + i + blockIdx.x) % p;
    b[i] = (threadIdx.x * 13 + 3 * i + blockIdx.x) % p;
  }
  const uint32_t p2 = 2 * p;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 10) {
        const uint32_t X = umin_u32(a[i], a[i] - p2);
        const double bd = __hiloint2double(0x43300000, (int)b[i]) - 4503599627370496.0;
        const double qd = fma(bd, wd, 6755399441055744.0);
        const uint32_t q = (uint32_t)__double2loint(qd);
        const uint32_t T = b[i] * w - q * p;  // in [-p, p)
        a[i] = X + T + p;
        b[i] = X - T + p;
      } else if (KIND == 11) {
        const uint32_t T = b[i] * w - __umulhi(b[i], ws) * p;
        b[i] = T ^ a[i];
        a[i] = T;
      } else {
        const uint32_t X = umin_u32(a[i], a[i] - p2);
        a[i] = X + b[i];
        b[i] = X - b[i] + p2;
      }
    }
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      const uint32_t t = a[i + 1];
      a[i + 1] = b[i];
      b[i] = t;
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc ^= a[i] ^ b[i];
  if (acc == 0x9e3779b9u) out[0] = acc;
}

// Base-conversion dot products (kinds 13-15): per output j, sum_{i<11} x_i
// c_ij mod p for 13 outputs, as in k_scale / k_extend.  13: lazy 64-bit
// integer sums (IMAD.WIDE) + Montgomery REDC; 14: exact FP64 (c split into
// 15-bit halves, two DFMA per term, fp64 reduction); 15: outputs alternate
// between the two.  Counts dot products (of 11 terms).
DI uint32_t dot_int(const uint32_t* x, const uint32_t* c, uint32_t p, uint32_t pinv) {
  uint64_t a = 0;
#pragma unroll
  for (int i = 0; i < 11; ++i) a += (uint64_t)x[i] * c[i];
  const uint32_t m = (uint32_t)a * pinv;
  return (uint32_t)((a + (uint64_t)m * p) >> 32);
}

DI uint32_t dot_f64(const double* xd, const double* ch, const double* cl, double p, double pinv) {
  double h = 0, l = 0;
#pragma unroll
  for (int i = 0; i < 11; ++i) {
    h = fma(xd[i], ch[i], h);
    l = fma(xd[i], cl[i], l);
  }
  const double qh = rint(h * pinv);
  const double rh = fma(-qh, p, h);  // |rh| <= p
  const double t = fma(rh, 32768.0, l);
  const double q2 = rint(t * pinv);
  double r = fma(-q2, p, t);
  r = r < 0 ? r + p : r;
  return (uint32_t)__double2loint(r + 4503599627370496.0);
}

template <int KIND>
__global__ void k_dot_probe(uint32_t* out, uint32_t seed, int iters) {
  const uint32_t p = 1073643521u, pinv = 0x3fff7fffu;
  uint32_t x[11];
  double xd[11];
#pragma unroll
  for (int i = 0; i < 11; ++i) x[i] = (seed * (threadIdx.x + 3 * i + 1) + blockIdx.x) & 0x3fffffff;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 11; ++i) xd[i] = __hiloint2double(0x43300000, (int)x[i]) - 4503599627370496.0;
#pragma unroll
    for (int j = 0; j < 13; ++j) {
      uint32_t c[11];
      double ch[11], cl[11];
#pragma unroll
      for (int i = 0; i < 11; ++i) {
        c[i] = (0x9e3779b9u * (i + 1) + 0x7f4a7c15u * j) & 0x3fffffff;
        ch[i] = (double)(c[i] >> 15);
        cl[i] = (double)(c[i] & 0x7fff);
      }
      const bool use_f = KIND == 14 || (KIND == 15 && (j & 1));
      acc += use_f ? dot_f64(xd, ch, cl, (double)p, 1.0 / p) : dot_int(x, c, p, pinv);
    }
    x[it % 11] ^= acc;
  }
  if (acc == 0x12345u) out[0] = acc;
}

// IMAD.WIDE and DFMA interleaved (kind 7): whether the fp64 pipe runs beside
// the integer multiplier; counts both kinds of operation
__global__ void k_mix_peak(uint32_t* out, uint32_t a, double da, double db, int iters) {
  uint64_t x[4];
  double y[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    x[i] = threadIdx.x * 7 + i + blockIdx.x;
    y[i] = x[i];
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      x[i] = (uint64_t)(uint32_t)x[i] * a + x[i];
      y[i] = fma(y[i], da, db);
    }
  }
  uint64_t acc = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) acc ^= x[i] ^ (uint64_t)y[i];
  if (acc == 0x9e3779b9u) out[0] = (uint32_t)acc;
}

// integer-pipe throughput probe: 8 independent chains per thread
template <int KIND>
__global__ void k_int_peak(uint32_t* out, uint32_t a, uint32_t b, int iters) {
  uint32_t x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 7 + i + blockIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) {
        x[i] = x[i] * a + b;
      } else if (KIND == 1) {
        x[i] = __umulhi(x[i], a) + b;
      } else if (KIND == 2) {
        const uint64_t w = (uint64_t)x[i] * a + b;
        x[i] = (uint32_t)(w >> 32) + (uint32_t)w;
      } else if (KIND == 3) {  // add + unsigned min (VIADDMNMX)
        const uint32_t y = x[i] - a;
        x[i] = (y < x[i] ? y : x[i]) + b;
      } else if (KIND == 4) {  // conditional subtract via sign mask
        const uint32_t y = x[i] - a;
        x[i] = y + (a & (uint32_t)((int32_t)y >> 31)) + b;
      } else {  // plain IADD3 chain
        x[i] = x[i] + a + b;
      }
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc ^= x[i];
  if (acc == 0x9e3779b9u) out[0] = acc;
}

// host u64 key rows -> device raw u32 copy (kept so the tiled layout can be
// rebuilt for another NTT variant)
void upload_raw_key(hcnn_ctx* c, const uint64_t* host, size_t rows, uint32_t** raw) {
  const size_t count = rows * c->N;
  uint64_t* stage = nullptr;
  pool_malloc(&stage, count * sizeof(uint64_t), c->stream, c->device);
  if (!*raw) CK(cudaMalloc((void**)raw, count * sizeof(uint32_t)));
  CK(cudaMemcpyAsync(stage, host, count * sizeof(uint64_t), cudaMemcpyHostToDevice, c->stream));
  k_narrow<<<cdiv(count, 256), 256, 0, c->stream>>>(stage, *raw, count);
  c->launched("k_narrow");
  CK(cudaFreeAsync(stage, c->stream));
}

// raw key rows -> NTT domain, tiled layout of the current variant (Montgomery
// form for the relinearisation key when the variant accumulates in u32)
void layout_key(hcnn_ctx* c, const uint32_t* raw, int domain, size_t rows, uint32_t** dst, int mont) {
  const size_t count = rows * c->N;
  if (!*dst) CK(cudaMalloc((void**)dst, count * sizeof(uint32_t)));
  if (domain == HCNN_DOMAIN_REF_NTT) {
    NttLaunch a{};
    a.grid = dim3((unsigned)rows);
    a.a = raw;
    a.out = *dst;
    a.limbs = (int)c->K;
    a.rlk_mont = mont;
    ntt_dispatch(c, 4, a, "k_ref_to_tiled");
  } else if (domain == HCNN_DOMAIN_COEFF) {
    CK(cudaMemcpyAsync(*dst, raw, count * sizeof(uint32_t), cudaMemcpyDeviceToDevice, c->stream));
    NttLaunch a{};
    a.grid = dim3((unsigned)rows);
    a.rows = *dst;
    a.limbs = (int)c->K;
    a.prime_off = 0;
    a.inverse = 2;
    ntt_dispatch(c, 0, a, "k_ntt_rows");
    if (mont) {
      NttLaunch m{};
      m.grid = dim3((unsigned)rows);
      m.rows = *dst;
      m.limbs = (int)c->K;
      ntt_dispatch(c, 5, m, "k_to_mont");
    }
  } else {
    fail(HCNN_ERR_DOMAIN, "unknown key domain");
  }
}

void prepare_keys(hcnn_ctx* c) {
  if (rb_active(c)) prepare_rb_keys(c);
  if (c->keys_variant == (c->variant & ~(32 | 1024 | 2048 | 4096 | 8192 | RELIN_RBASIS | TC_BCONV | RB_MAC_TC))) return;
  if (c->d_rlk_raw)
    layout_key(c, c->d_rlk_raw, c->rlk_domain, (size_t)c->D * 2 * c->K, &c->d_rlk, variant_mont(c, c->variant));
  if (c->d_pk_raw) layout_key(c, c->d_pk_raw, c->pk_domain, 2 * (size_t)c->K, &c->d_pk, 0);
  c->keys_variant = c->variant & ~(32 | 1024 | 2048 | 4096 | 8192 | RELIN_RBASIS | TC_BCONV | RB_MAC_TC);
}

}  // namespace

// =================================================================== C ABI
extern "C" {

const char* hcnn_last_error(void) { return g_err.c_str(); }
namespace {
// one thread's share of hcnn_host_narrow; returns the OR of all inputs' high
// words (non-zero: a value outside [0, 2^32))
// Persistent host worker threads for the drop-in staging (hcnn_host_narrow
// runs once per row band; spawning its threads every call cost ~0.3 ms).
// run(n, fn) calls fn(k) for k in [0, n), k = 0 on the caller; one job at a
// time.  The pool is never destroyed (its idle threads wait on a condition).
class HostPool {
 public:
  static HostPool& get() {
    static HostPool* p = new HostPool;
    return *p;
  }
  void run(size_t n, const std::function<void(size_t)>& fn) {
    std::lock_guard<std::mutex> one(run_m_);
    {
      std::lock_guard<std::mutex> g(m_);
      while (nthreads_ + 1 < n) {
        const size_t id = ++nthreads_;
        std::thread([this, id] { loop(id); }).detach();
      }
      fn_ = &fn;
      jobs_ = n - 1;
      pending_ = n - 1;
      ++gen_;
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> l(m_);
    done_.wait(l, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  void loop(size_t id) {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> l(m_);
    for (;;) {
      cv_.wait(l, [&] { return gen_ != seen; });
      seen = gen_;
      if (id > jobs_) continue;
      const std::function<void(size_t)>* f = fn_;
      l.unlock();
      (*f)(id);
      l.lock();
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::mutex run_m_, m_;
  std::condition_variable cv_, done_;
  const std::function<void(size_t)>* fn_ = nullptr;
  size_t nthreads_ = 0, jobs_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
};

// AVX2 with streaming stores: the pinned destination is written without
// being read first (a plain store reads each line for ownership, a third of
// the host memory traffic of the narrowing, which is memory-bound while the
// uploads run)
__attribute__((target("avx2"))) uint64_t narrow_rows_avx2(const int64_t* const* src, size_t a, size_t b,
                                                          size_t len, uint32_t* dst) {
  const __m256i perm = _mm256_setr_epi32(0, 2, 4, 6, 1, 3, 5, 7);
  __m256i hiv = _mm256_setzero_si256();
  uint64_t hi = 0;
  for (size_t i = a; i < b; ++i) {
    const int64_t* s = src[i];
    uint32_t* d = dst + i * len;
    size_t j = 0;
    if ((reinterpret_cast<uintptr_t>(d) & 31) == 0) {
      for (; j + 8 <= len; j += 8) {
        const __m256i x = _mm256_permutevar8x32_epi32(_mm256_loadu_si256((const __m256i*)(s + j)), perm);
        const __m256i y = _mm256_permutevar8x32_epi32(_mm256_loadu_si256((const __m256i*)(s + j + 4)), perm);
        _mm256_stream_si256((__m256i*)(d + j), _mm256_permute2x128_si256(x, y, 0x20));
        hiv = _mm256_or_si256(hiv, _mm256_permute2x128_si256(x, y, 0x31));
      }
    }
    for (; j < len; ++j) {
      const uint64_t v = (uint64_t)s[j];
      hi |= v >> 32;
      d[j] = (uint32_t)v;
    }
  }
  _mm_sfence();
  alignas(32) uint32_t h8[8];
  _mm256_store_si256((__m256i*)h8, hiv);
  for (int k = 0; k < 8; ++k) hi |= h8[k];
  return hi;
}

__attribute__((optimize("O3"))) uint64_t narrow_rows(const int64_t* const* src, size_t a, size_t b,
                                                      size_t len, uint32_t* dst) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (avx2) return narrow_rows_avx2(src, a, b, len, dst);
  uint64_t hi = 0;
  for (size_t i = a; i < b; ++i) {
    const uint64_t* __restrict__ s = reinterpret_cast<const uint64_t*>(src[i]);
    uint32_t* __restrict__ d = dst + i * len;
    for (size_t j = 0; j < len; ++j) {
      const uint64_t v = s[j];
      hi |= v;
      d[j] = (uint32_t)v;
    }
  }
  return hi >> 32;
}
}  // namespace

int hcnn_host_narrow(const int64_t* const* src, size_t count, size_t len, uint32_t* dst, int threads) {
  return guarded([&] {
    if (!count || !len) return;
    if (!src || !dst) fail(HCNN_ERR_PARAM, "null argument");
    for (size_t i = 0; i < count; ++i)
      if (!src[i]) fail(HCNN_ERR_PARAM, "null source array");
    size_t nt = threads > 0 ? (size_t)threads : (size_t)std::thread::hardware_concurrency();
    if (nt < 1) nt = 1;
    if (nt > 64) nt = 64;
    if (nt > count) nt = count;
    std::vector<uint64_t> bad(nt, 0);
    HostPool::get().run(nt, [&](size_t k) { bad[k] = narrow_rows(src, count * k / nt, count * (k + 1) / nt, len, dst); });
    for (uint64_t b : bad)
      if (b) fail(HCNN_ERR_PARAM, "residue outside [0, 2^32): not a canonical RNS residue");
  });
}

int hcnn_host_widen(const uint32_t* src, size_t count, size_t len, int64_t* const* dst, int threads) {
  return guarded([&] {
    if (!count || !len) return;
    if (!src || !dst) fail(HCNN_ERR_PARAM, "null argument");
    for (size_t i = 0; i < count; ++i)
      if (!dst[i]) fail(HCNN_ERR_PARAM, "null destination array");
    size_t nt = threads > 0 ? (size_t)threads : (size_t)std::thread::hardware_concurrency();
    nt = nt < 1 ? 1 : nt > 64 ? 64 : nt;
    if (nt > count) nt = count;
    HostPool::get().run(nt, [&](size_t k) {
      for (size_t i = count * k / nt; i < count * (k + 1) / nt; ++i) {
        const uint32_t* __restrict__ s = src + i * len;
        int64_t* __restrict__ d = dst[i];
        for (size_t j = 0; j < len; ++j) d[j] = (int64_t)s[j];
      }
    });
  });
}

namespace {
uint64_t inv_mod_u64(uint64_t a, uint64_t m) {  // a^-1 mod m (gcd 1), extended Euclid in signed 128-bit
  __int128 t0 = 0, t1 = 1, r0 = m, r1 = a % m;
  while (r1) {
    const __int128 q = r0 / r1, r2 = r0 - q * r1, t2 = t0 - q * t1;
    r0 = r1;
    r1 = r2;
    t0 = t1;
    t1 = t2;
  }
  if (r0 != 1) fail(HCNN_ERR_PARAM, "CRT moduli are not pairwise coprime");
  if (t0 < 0) t0 += m;
  return (uint64_t)t0;
}
}  // namespace

int hcnn_release_memory(int device) {
  return guarded([&] {
    CK(cudaSetDevice(device));
    CK(cudaDeviceSynchronize());
    CK(cudaMemPoolTrimTo(lib_pool(device), 0));
  });
}

int hcnn_crt_combine(const uint64_t* res, const uint64_t* moduli, int n_moduli, size_t count, uint32_t* out,
                     int words, int* flag, int device, void* stream) {
  return guarded([&] {
    if (!moduli || n_moduli < 1 || n_moduli > CRT_MAXC) fail(HCNN_ERR_PARAM, "1..16 CRT moduli supported");
    if (words < 1 || words > CRT_MAXW) fail(HCNN_ERR_PARAM, "output words out of range");
    CrtTabs tb{};
    tb.C = n_moduli;
    tb.W = words;
    std::vector<uint32_t> T(CRT_MAXW + 4, 0);
    T[0] = 1;
    for (int i = 0; i < n_moduli; ++i) {
      if (moduli[i] < 2 || moduli[i] >= (1ull << 62)) fail(HCNN_ERR_PARAM, "CRT moduli must lie in [2, 2^62)");
      tb.t[i] = moduli[i];
      unsigned __int128 carry = 0;
      for (auto& w : T) {
        const unsigned __int128 acc = (unsigned __int128)w * moduli[i] + carry;
        w = (uint32_t)acc;
        carry = acc >> 32;
      }
      for (int j = 0; j < i; ++j) tb.inv[j][i] = inv_mod_u64(moduli[j], moduli[i]);
    }
    int used = (int)T.size();
    while (used > 0 && T[used - 1] == 0) --used;
    if (used + 1 > words) fail(HCNN_ERR_PARAM, "output words too few for the product of the moduli plus a sign");
    for (int k = 0; k < words; ++k) {
      tb.T[k] = T[k];
      tb.half[k] = (T[k] >> 1) | (k + 1 < (int)T.size() ? T[k + 1] << 31 : 0u);
    }
    if (!count) return;
    if (!res || !out) fail(HCNN_ERR_PARAM, "null argument");
    CK(cudaSetDevice(device));
    cudaStream_t st = (cudaStream_t)stream;
    int* bad = flag;
    if (!bad) {
      pool_malloc(&bad, sizeof(int), st, device);
      CK(cudaMemsetAsync(bad, 0, sizeof(int), st));
    }
    k_crt_combine<<<(unsigned)((count + 127) / 128), 128, 0, st>>>(res, count, tb, out, bad);
    CK(cudaGetLastError());
    if (!flag) {  // checked here: synchronous
      int h_bad = 0;
      CK(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaFreeAsync(bad, st));
      CK(cudaStreamSynchronize(st));
      if (h_bad) fail(HCNN_ERR_PARAM, "CRT residue outside [0, t_i)");
    }
  });
}

int hcnn_int_peak(int device, int kind, double* ops_per_s) {
  return guarded([&] {
    CK(cudaSetDevice(device));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    uint32_t* out = nullptr;
    CK(cudaMalloc(&out, 4));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int iters = 4096, tpb = 256, blocks = sms * 8;
    auto run = [&] {
      switch (kind) {
        case 0: k_int_peak<0><<<blocks, tpb>>>(out, 0x9e3779b1u, 12345u, iters); break;
        case 1: k_int_peak<1><<<blocks, tpb>>>(out, 0x9e3779b1u, 12345u, iters); break;
        case 2: k_int_peak<2><<<blocks, tpb>>>(out, 0x9e3779b1u, 12345u, iters); break;
        case 3: k_int_peak<3><<<blocks, tpb>>>(out, 0x3e3779b1u, 12345u, iters); break;
        case 4: k_int_peak<4><<<blocks, tpb>>>(out, 0x3e3779b1u, 12345u, iters); break;
        case 6: k_dfma_peak<<<blocks, tpb>>>(out, 0.999999, 1e-9, iters); break;
        case 7: k_mix_peak<<<blocks, tpb>>>(out, 0x9e3779b1u, 0.999999, 1e-9, iters); break;
        case 8: k_bfly_peak<<<blocks, tpb>>>(out, 123456789u, 493942125u, 1073643521u, iters); break;
        case 9: k_bfly_peak<<<blocks / 4, tpb>>>(out, 123456789u, 493942125u, 1073643521u, iters); break;
        case 10: k_bfly_probe<10><<<blocks, tpb>>>(out, 123456789u, 493942125u, 1073643521u, 123456789.0 / 1073643521.0, iters); break;
        case 11: k_bfly_probe<11><<<blocks, tpb>>>(out, 123456789u, 493942125u, 1073643521u, 0.0, iters); break;
        case 13: k_dot_probe<13><<<blocks, tpb>>>(out, 12345u, iters / 16); break;
        case 14: k_dot_probe<14><<<blocks, tpb>>>(out, 12345u, iters / 16); break;
        case 15: k_dot_probe<15><<<blocks, tpb>>>(out, 12345u, iters / 16); break;
        case 12: k_bfly_probe<12><<<blocks, tpb>>>(out, 123456789u, 493942125u, 1073643521u, 0.0, iters); break;
        case 16: {
          const uint64_t p = 4611686018427322369ull, w = 1234567890123456789ull;
          k_bfly64_peak<<<blocks, tpb>>>(out, w, (uint64_t)(((u128)w << 64) / p), p, iters / 4);
          break;
        }
        default: k_int_peak<5><<<blocks, tpb>>>(out, 0x3e3779b1u, 12345u, iters); break;
      }
    };
    run();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) run();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    *ops_per_s = 5.0 * (kind == 9 ? blocks / 4 : blocks) * tpb * (double)iters * 8 / (ms * 1e-3);
    if (kind >= 13 && kind <= 15) *ops_per_s = 5.0 * blocks * tpb * (double)(iters / 16) * 13 / (ms * 1e-3);
    if (kind == 16) *ops_per_s = 5.0 * blocks * tpb * (double)(iters / 4) * 8 / (ms * 1e-3);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
  });
}

const char* hcnn_version(void) { return "hcnn_b200 0.1 (sm_100a)"; }

int hcnn_ctx_create(hcnn_ctx** out, uint32_t n, uint32_t k, const uint64_t* primes, uint64_t t,
                    uint32_t log2w, int device) {
  return guarded([&] {
    if (!out || !primes) fail(HCNN_ERR_PARAM, "null argument");
    *out = nullptr;
    if (n < 4 || (n & (n - 1)) || n > (1u << 15)) fail(HCNN_ERR_UNSUPPORTED, "ring degree must be a power of two in [4, 2^15]");
    if (k < 1 || k > (uint32_t)KMAX) fail(HCNN_ERR_UNSUPPORTED, "1..16 primes supported");
    if (log2w != 8 && log2w != 16 && log2w != 32) fail(HCNN_ERR_PARAM, "relin base must be 2^8, 2^16 or 2^32");
    std::vector<u64> q(primes, primes + k);
    for (uint32_t i = 0; i < k; ++i) {
      if (q[i] >= (1ull << 30) || q[i] < 3) fail(HCNN_ERR_UNSUPPORTED, "RNS primes must be below 2^30 on the u32 path");
      if (!is_prime64(q[i])) fail(HCNN_ERR_UNSUPPORTED, std::to_string(q[i]) + " is not prime");
      if (q[i] % (2ull * n) != 1) fail(HCNN_ERR_UNSUPPORTED, std::to_string(q[i]) + " is not 1 mod 2N");
      for (uint32_t j = 0; j < i; ++j)
        if (q[j] == q[i]) fail(HCNN_ERR_PARAM, "primes must be pairwise distinct");
    }
    if (t < 2) fail(HCNN_ERR_PARAM, "plaintext modulus must be >= 2");
    {
      Big Q = product(q);
      if (cmp(Big(t), Q) >= 0) fail(HCNN_ERR_PARAM, "plaintext modulus must be below q");
    }
    auto c = std::make_unique<hcnn_ctx>();
    c->device = device;
    CK(cudaSetDevice(device));
    lib_pool(device);  // the library's own pool (stream-ordered workspace and temporaries)
    CK(cudaEventCreateWithFlags(&c->switch_ev, cudaEventDisableTiming));
    CK(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    c->stream = c->own_stream;
    c->N = n;
    c->logN = 0;
    while ((1u << c->logN) < n) ++c->logN;
    c->K = k;
    c->t = t;
    c->log2w = log2w;
    // default geometry per ring degree (profiles/r1_micro_sweep.jsonl): the
    // shuffle-tail radix-16 kernels up to 2^13 (persistent square tensor and
    // relinearisation over R at 2^13: profiles/r2/micro_rbasis.jsonl),
    // mixed-width passes at 2^14, 2-CTA cluster relinearisation at 2^15
    // base conversions on the tensor cores from K = 8 primes (MNIST set 1
    // 17.58 -> 16.46 ms, set 3 38.3 -> 36.4 ms, CIFAR set 5 -4 %; HSquare at
    // K = 11-12 -5..-9 %, at K = 6 +2..3 %: tools/tc_sweep.sh, tools/tc_ab.sh,
    // profiles/r2/micro_sweep_v4.jsonl)
    c->variant = (k >= 8 ? TC_BCONV : 0) | (c->logN == 13   ? (8192 | RELIN_RBASIS)
                             : c->logN == 14 ? (64 | 1024 | 4096 | RELIN_RBASIS)
                             : c->logN == 15 ? (512 | 2048 | RELIN_RBASIS)
                                             : 0);
    build_tables(c.get(), q, t);
    *out = c.release();
  });
}

int hcnn_ctx_destroy(hcnn_ctx* c) {
  return guarded([&] {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    if (c->ws) cudaFree(c->ws);
    cudaFree(c->d_prime);
    cudaFree(c->d_mu);
    cudaFree(c->d_tw);
    cudaFree(c->d_itw);
    cudaFree(c->d_ninv);
    if (c->d_rlk) cudaFree(c->d_rlk);
    if (c->d_rlk_raw) cudaFree(c->d_rlk_raw);
    if (c->d_rlk_rb) cudaFree(c->d_rlk_rb);
    if (c->d_rlk_tc) cudaFree(c->d_rlk_tc);
    if (c->d_tcb) cudaFree(c->d_tcb);
    if (c->d_pk_raw) cudaFree(c->d_pk_raw);
    cudaFree(c->d_pinv);
    if (c->d_pk) cudaFree(c->d_pk);
    if (c->d_sk) cudaFree(c->d_sk);
    if (c->d_delta) cudaFree(c->d_delta);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    if (c->switch_ev) cudaEventDestroy(c->switch_ev);
    delete c;
  });
}

int hcnn_profile(hcnn_ctx* c, int enable) {
  return guarded([&] {
    CK(cudaStreamSynchronize(c->stream));
    c->prof_reset();
    c->prof = enable != 0;
  });
}

int64_t hcnn_profile_dump(hcnn_ctx* c, char* buf, size_t len) {
  std::string out;
  int rc = guarded([&] {
    CK(cudaStreamSynchronize(c->stream));
    std::vector<std::pair<std::string, std::pair<int64_t, double>>> agg;
    for (auto& r : c->recs) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, r.a, r.b));
      bool found = false;
      for (auto& a : agg)
        if (a.first == r.name) {
          a.second.first += 1;
          a.second.second += ms;
          found = true;
        }
      if (!found) agg.push_back({r.name, {1, (double)ms}});
    }
    for (auto& a : agg) {
      char line[256];
      snprintf(line, sizeof line, "%s %lld %.6f\n", a.first.c_str(), (long long)a.second.first, a.second.second);
      out += line;
    }
  });
  if (rc != HCNN_OK) return -rc;
  if (buf && len) {
    size_t n = out.size() < len - 1 ? out.size() : len - 1;
    memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return (int64_t)out.size();
}

int hcnn_ctx_set_stream(hcnn_ctx* c, void* stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    if (s == c->stream) return;
    // everything already queued for this context (including the workspace
    // it shares across calls, and any stream-ordered free of it) is ordered
    // before the new stream's work
    CK(cudaEventRecord(c->switch_ev, c->stream));
    CK(cudaStreamWaitEvent(s, c->switch_ev, 0));
    c->stream = s;
  });
}

int hcnn_ctx_set_option(hcnn_ctx* c, int key, int64_t value) {
  return guarded([&] {
    if (key == HCNN_OPT_NTT_VARIANT) {
      // geometry flags of the fused kernels (ntt_kernels.cuh): +16 one-row
      // relinearisation transforms, +32 square tensors on the radix-32 mixed
      // geometry, +64 mixed-width passes instead of a warp-shuffle tail
      if (value & ~(int64_t)(16 | 32 | 64 | 512 | 1024 | 2048 | 4096 | 8192 | RELIN_RBASIS | TC_BCONV | RB_MAC_TC))
        fail(HCNN_ERR_PARAM, "NTT variant flags are 16, 32, 64, 512, 1024, 2048, 4096, 8192, 16384, 32768 and 65536");
      if ((value & (32 | 64)) && c->logN < 10) fail(HCNN_ERR_UNSUPPORTED, "mixed geometries need N >= 1024");
      if ((value & 512) && c->logN != 15 && c->logN != 14)
        fail(HCNN_ERR_UNSUPPORTED, "cluster kernels are for N = 2^14 and 2^15");
      c->variant = (int)value;
    } else if (key == HCNN_OPT_RB_MIN_BATCH) {
      if (value < 1) fail(HCNN_ERR_PARAM, "minimum batch must be >= 1");
      c->rb_min_batch = (size_t)value;
    } else if (key == HCNN_OPT_TS_CHUNK) {
      if (value < 0) fail(HCNN_ERR_PARAM, "sub-chunk size must be >= 0");
      c->ts_sub = (size_t)value;
    } else {
      fail(HCNN_ERR_PARAM, "unknown option");
    }
  });
}

int hcnn_ctx_set_workspace_limit(hcnn_ctx* c, size_t bytes) {
  return guarded([&] { c->ws_limit = bytes; });
}

int64_t hcnn_ctx_query(hcnn_ctx* c, int what) {
  switch (what) {
    case HCNN_Q_N: return c->N;
    case HCNN_Q_K: return c->K;
    case HCNN_Q_KP: return c->KP;
    case HCNN_Q_DIGITS: return c->D;
    case HCNN_Q_LOG2W: return c->log2w;
    case HCNN_Q_WS_BYTES: return (int64_t)c->ws_bytes;
    case HCNN_Q_KERNELS: return c->launches;
    case HCNN_Q_NTT_VARIANT: return c->variant;
    case HCNN_Q_RELIN_RBASIS: return rb_active(c) ? 1 : 0;
    case HCNN_Q_TC_BCONV: return tc_active(c) ? 1 : 0;
    default: return -1;
  }
}

uint64_t hcnn_ctx_prime(hcnn_ctx* c, int i, uint64_t* psi) {
  if (i < 0 || (size_t)i >= c->primes.size()) return 0;
  if (psi) *psi = c->psi[i];
  return c->primes[i];
}

int hcnn_set_relin_key(hcnn_ctx* c, const uint64_t* rlk, int domain) {
  return guarded([&] {
    if (!rlk) fail(HCNN_ERR_MISSING_KEY, "relinearization key required");
    if (domain != HCNN_DOMAIN_REF_NTT && domain != HCNN_DOMAIN_COEFF) fail(HCNN_ERR_DOMAIN, "unknown key domain");
    CK(cudaSetDevice(c->device));
    upload_raw_key(c, rlk, (size_t)c->D * 2 * c->K, &c->d_rlk_raw);
    c->rlk_domain = domain;
    c->keys_variant = -1;
    c->rb_keys = false;
    prepare_keys(c);
    // digits of w = 2^32 may exceed a prime; 2^8 / 2^16 digits never do here
    c->rlk_reduce = false;
    for (uint32_t i = 0; i < c->K; ++i)
      if ((c->log2w >= 32) || ((1ull << c->log2w) > c->primes[i])) c->rlk_reduce = true;
    CK(cudaStreamSynchronize(c->stream));
  });
}

int hcnn_set_public_key(hcnn_ctx* c, const uint64_t* pk, int domain) {
  return guarded([&] {
    if (!pk) fail(HCNN_ERR_MISSING_KEY, "public key required");
    if (domain != HCNN_DOMAIN_REF_NTT && domain != HCNN_DOMAIN_COEFF) fail(HCNN_ERR_DOMAIN, "unknown key domain");
    CK(cudaSetDevice(c->device));
    upload_raw_key(c, pk, 2 * (size_t)c->K, &c->d_pk_raw);
    c->pk_domain = domain;
    c->keys_variant = -1;
    prepare_keys(c);
    // Delta = floor(q / t) mod q_i (bfv.py:77)
    if (!c->d_delta) {
      Big Q = product(std::vector<u64>(c->primes.begin(), c->primes.begin() + c->K));
      // floor(Q / t) with t up to 64 bits: long division by a u64
      Big D;
      D.w.assign(Q.w.size(), 0);
      u128 r = 0;
      for (size_t i = Q.w.size(); i-- > 0;) {
        r = (r << 32) | Q.w[i];
        D.w[i] = (u32)(r / c->t);
        r %= c->t;
      }
      D.trim();
      std::vector<uint2> hd(c->K);
      for (uint32_t i = 0; i < c->K; ++i) {
        const uint32_t v = (uint32_t)mod_small(D, c->primes[i]);
        hd[i] = make_uint2(v, shoup_of(v, (uint32_t)c->primes[i]));
      }
      CK(cudaMalloc((void**)&c->d_delta, c->K * sizeof(uint2)));
      CK(cudaMemcpy(c->d_delta, hd.data(), c->K * sizeof(uint2), cudaMemcpyHostToDevice));
    }
    CK(cudaStreamSynchronize(c->stream));
  });
}

static int hcnn_encrypt_impl(hcnn_ctx* c, const int8_t* u, const int8_t* e1, const int8_t* e2,
                             const int64_t* msg, int msg_on_device, uint32_t* out, size_t n);

int hcnn_encrypt(hcnn_ctx* c, const int8_t* u, const int8_t* e1, const int8_t* e2, const int64_t* msg,
                 uint32_t* out, size_t n) {
  return hcnn_encrypt_impl(c, u, e1, e2, msg, 0, out, n);
}

int hcnn_encrypt_device_msg(hcnn_ctx* c, const int8_t* u, const int8_t* e1, const int8_t* e2,
                            const int64_t* msg_dev, uint32_t* out, size_t n) {
  return hcnn_encrypt_impl(c, u, e1, e2, msg_dev, 1, out, n);
}

static int hcnn_encrypt_impl(hcnn_ctx* c, const int8_t* u, const int8_t* e1, const int8_t* e2,
                             const int64_t* msg, int msg_on_device, uint32_t* out, size_t n) {
  return guarded([&] {
    if (!c->d_pk_raw) fail(HCNN_ERR_MISSING_KEY, "public key required");
    CK(cudaSetDevice(c->device));
    if (n == 0) return;
    prepare_keys(c);
    c->mark();
    const size_t N = c->N;
    const size_t ch = n < 4096 ? n : 4096;
    uint8_t* stage = nullptr;
    const size_t bytes = ch * N * (3 + sizeof(int64_t));
    pool_malloc(&stage, bytes, c->stream, c->device);
    for (size_t s0 = 0; s0 < n; s0 += ch) {
      const size_t m = n - s0 < ch ? n - s0 : ch;
      int8_t* du = (int8_t*)stage;
      int8_t* d1 = du + ch * N;
      int8_t* d2 = d1 + ch * N;
      int64_t* dm = (int64_t*)(d2 + ch * N);
      CK(cudaMemcpyAsync(du, u + s0 * N, m * N, cudaMemcpyHostToDevice, c->stream));
      CK(cudaMemcpyAsync(d1, e1 + s0 * N, m * N, cudaMemcpyHostToDevice, c->stream));
      CK(cudaMemcpyAsync(d2, e2 + s0 * N, m * N, cudaMemcpyHostToDevice, c->stream));
      if (msg_on_device)
        CK(cudaMemcpyAsync(dm, msg + s0 * N, m * N * sizeof(int64_t), cudaMemcpyDeviceToDevice, c->stream));
      else
        CK(cudaMemcpyAsync(dm, msg + s0 * N, m * N * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
      NttLaunch a{};
      a.grid = dim3(c->K, (unsigned)m);
      a.u = du;
      a.e1 = d1;
      a.e2 = d2;
      a.msg = dm;
      a.pk = c->d_pk;
      a.delta = c->d_delta;
      a.out = out + s0 * 2 * c->K * N;
      a.K = (int)c->K;
      ntt_dispatch(c, 3, a, "k_encrypt");
    }
    CK(cudaFreeAsync(stage, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int hcnn_codec_create(uint64_t t, uint32_t n, int device, hcnn_codec** out) {
  return guarded([&] {
    if (!out) fail(HCNN_ERR_PARAM, "null argument");
    if (n < 2 || (n & (n - 1)) || n > (1u << 15)) fail(HCNN_ERR_UNSUPPORTED, "ring degree must be a power of two in [2, 2^15]");
    if (t >= (1ull << 62) || !is_prime64(t)) fail(HCNN_ERR_UNSUPPORTED, "t must be a prime below 2^62");
    if ((t - 1) % (2ull * n)) fail(HCNN_ERR_UNSUPPORTED, "2N does not divide t-1");
    CK(cudaSetDevice(device));
    auto c = std::make_unique<hcnn_codec>();
    c->device = device;
    c->n = n;
    while ((1u << c->logn) < n) ++c->logn;
    c->t = t;
    c->zeta = primitive_2n_root(t, n);
    const u64 iz = invmod64(c->zeta, t);
    std::vector<ulonglong2> tw(n), itw(n);
    std::vector<u64> pw(n), ipw(n);
    pw[0] = ipw[0] = 1;
    for (uint32_t i = 1; i < n; ++i) {
      pw[i] = mulmod64(pw[i - 1], c->zeta, t);
      ipw[i] = mulmod64(ipw[i - 1], iz, t);
    }
    auto shoup64 = [&](u64 w) { return (u64)(((u128)w << 64) / t); };
    for (uint32_t i = 0; i < n; ++i) {
      const u64 a = pw[bitrev(i, c->logn)], b = ipw[bitrev(i, c->logn)];
      tw[i] = make_ulonglong2(a, shoup64(a));
      itw[i] = make_ulonglong2(b, shoup64(b));
    }
    const u64 ni = invmod64(n % t, t);
    c->ninv = make_ulonglong2(ni, shoup64(ni));
    const u64 nw = mulmod64(ipw[n / 2], ni, t);
    c->ninv_w = make_ulonglong2(nw, shoup64(nw));
    CK(cudaMalloc(&c->d_tw, n * sizeof(ulonglong2)));
    CK(cudaMalloc(&c->d_itw, n * sizeof(ulonglong2)));
    CK(cudaMemcpy(c->d_tw, tw.data(), n * sizeof(ulonglong2), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_itw, itw.data(), n * sizeof(ulonglong2), cudaMemcpyHostToDevice));
    *out = c.release();
  });
}

int hcnn_codec_destroy(hcnn_codec* c) {
  return guarded([&] {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaFree(c->d_tw);
    cudaFree(c->d_itw);
    delete c;
  });
}

// slots (natural order, values < t) -> plaintext polys: batching.encode
int hcnn_codec_encode(hcnn_codec* c, const uint64_t* slots, uint64_t* polys, size_t rows, void* stream) {
  return guarded([&] {
    if (!rows) return;
    CK(cudaSetDevice(c->device));
    cudaStream_t st = (cudaStream_t)stream;
    k_permute_brv64<<<dim3(cdiv(c->n, 256), (unsigned)rows), 256, 0, st>>>(slots, polys, (int)c->logn);
    CK(cudaGetLastError());
    CK(launch_ntt64<true>(polys, rows, (int)c->logn, c->t, c->d_itw, c->ninv, c->ninv_w, st));
  });
}

// in-place u64 negacyclic NTT rows over the codec's prime (ntt.py:113-154
// for primes up to 62 bits): forward natural -> bit-reversed positions,
// inverse back, fully reduced
int hcnn_ntt64(hcnn_codec* c, uint64_t* rows, size_t n_rows, int inverse, void* stream) {
  return guarded([&] {
    if (!n_rows) return;
    if (!rows) fail(HCNN_ERR_PARAM, "null argument");
    CK(cudaSetDevice(c->device));
    cudaStream_t st = (cudaStream_t)stream;
    if (inverse)
      CK(launch_ntt64<true>(rows, n_rows, (int)c->logn, c->t, c->d_itw, c->ninv, c->ninv_w, st));
    else
      CK(launch_ntt64<false>(rows, n_rows, (int)c->logn, c->t, c->d_tw, c->ninv, c->ninv_w, st));
  });
}

// plaintext polys -> slots (natural order): batching.decode
int hcnn_codec_decode(hcnn_codec* c, const uint64_t* polys, uint64_t* slots, size_t rows, void* stream) {
  return guarded([&] {
    if (!rows) return;
    CK(cudaSetDevice(c->device));
    cudaStream_t st = (cudaStream_t)stream;
    uint64_t* tmp = nullptr;
    pool_malloc(&tmp, rows * c->n * sizeof(uint64_t), st, c->device);
    CK(cudaMemcpyAsync(tmp, polys, rows * c->n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
    CK(launch_ntt64<false>(tmp, rows, (int)c->logn, c->t, c->d_tw, c->ninv, c->ninv_w, st));
    k_permute_brv64<<<dim3(cdiv(c->n, 256), (unsigned)rows), 256, 0, st>>>(tmp, slots, (int)c->logn);
    CK(cudaGetLastError());
    CK(cudaFreeAsync(tmp, st));
  });
}

int hcnn_set_secret_key(hcnn_ctx* c, const uint8_t* s_bits) {
  return guarded([&] {
    if (!s_bits) fail(HCNN_ERR_MISSING_KEY, "secret key required");
    CK(cudaSetDevice(c->device));
    const size_t N = c->N, K = c->K;
    uint8_t* ds = nullptr;
    pool_malloc(&ds, N, c->stream, c->device);
    CK(cudaMemcpyAsync(ds, s_bits, N, cudaMemcpyHostToDevice, c->stream));
    if (!c->d_sk) CK(cudaMalloc((void**)&c->d_sk, K * N * sizeof(uint32_t)));
    k_sk_rows<<<cdiv(N, 256), 256, 0, c->stream>>>(ds, c->d_sk, (int)K, (int)N);
    c->launched("k_sk_rows");
    launch_ntt_rows(c, c->d_sk, K, (int)K, 0, 0);
    CK(cudaFreeAsync(ds, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int hcnn_keygen(hcnn_ctx* c, const uint8_t* s_bits, const uint64_t* a_ref, const int8_t* e, uint64_t* pk_out,
                uint64_t* rlk_out) {
  const int st = guarded([&] {
    if (!s_bits || !a_ref || !e || !pk_out || !rlk_out) fail(HCNN_ERR_PARAM, "keygen: null buffer");
    CK(cudaSetDevice(c->device));
    const size_t N = c->N, K = c->K, D = c->D, R = 1 + D;
    const unsigned logn = c->logN;
    // secret key rows in the device NTT order (also the decryption key)
    uint8_t* ds = nullptr;
    pool_malloc(&ds, N, c->stream, c->device);
    CK(cudaMemcpyAsync(ds, s_bits, N, cudaMemcpyHostToDevice, c->stream));
    if (!c->d_sk) CK(cudaMalloc((void**)&c->d_sk, K * N * sizeof(uint32_t)));
    k_sk_rows<<<cdiv(N, 256), 256, 0, c->stream>>>(ds, c->d_sk, (int)K, (int)N);
    c->launched("k_sk_rows");
    launch_ntt_rows(c, c->d_sk, K, (int)K, 0, 0);
    // a (reference NTT order) -> device order; e -> NTT
    const size_t rows = R * K, count = rows * N;
    uint64_t* stage = nullptr;
    uint32_t *da = nullptr, *adev = nullptr, *erow = nullptr, *out = nullptr, *dw = nullptr;
    int8_t* de = nullptr;
    pool_malloc(&stage, count * sizeof(uint64_t), c->stream, c->device);
    pool_malloc(&da, count * sizeof(uint32_t), c->stream, c->device);
    pool_malloc(&adev, count * sizeof(uint32_t), c->stream, c->device);
    pool_malloc(&erow, count * sizeof(uint32_t), c->stream, c->device);
    pool_malloc(&out, count * sizeof(uint32_t), c->stream, c->device);
    pool_malloc(&de, R * N, c->stream, c->device);
    pool_malloc(&dw, rows * sizeof(uint32_t), c->stream, c->device);
    CK(cudaMemcpyAsync(stage, a_ref, count * sizeof(uint64_t), cudaMemcpyHostToDevice, c->stream));
    k_narrow<<<cdiv(count, 256), 256, 0, c->stream>>>(stage, da, count);
    c->launched("k_narrow");
    k_bitrev_rows<<<dim3(cdiv(N, 256), (unsigned)rows), 256, 0, c->stream>>>(da, adev, (int)N, (int)logn);
    c->launched("k_bitrev_rows");
    CK(cudaMemcpyAsync(de, e, R * N, cudaMemcpyHostToDevice, c->stream));
    k_embed_small<<<cdiv(R * N, 256), 256, 0, c->stream>>>(de, erow, (int)R, (int)K, (int)N, c->d_prime);
    c->launched("k_embed_small");
    launch_ntt_rows(c, erow, rows, (int)K, 0, 0);
    // w^i mod q_k (row 0, the public key, takes no s^2 term)
    std::vector<uint32_t> wres(rows, 0);
    for (size_t k = 0; k < K; ++k) {
      u64 wp = 1 % c->primes[k];
      const u64 w = (u64)(((u128)1 << c->log2w) % c->primes[k]);
      for (size_t r = 1; r < R; ++r) {
        wres[r * K + k] = (uint32_t)wp;
        wp = mulmod64(wp, w, c->primes[k]);
      }
    }
    CK(cudaMemcpyAsync(dw, wres.data(), rows * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
    k_keygen_combine<<<cdiv(count, 256), 256, 0, c->stream>>>(adev, erow, c->d_sk, dw, out, (int)R, (int)K,
                                                             (int)N, c->d_prime, c->d_mu);
    c->launched("k_keygen_combine");
    // back to the reference order, widened to u64
    k_bitrev_rows<<<dim3(cdiv(N, 256), (unsigned)rows), 256, 0, c->stream>>>(out, da, (int)N, (int)logn);
    c->launched("k_bitrev_rows");
    k_widen<<<cdiv(count, 256), 256, 0, c->stream>>>(da, stage, count);
    c->launched("k_widen");
    std::vector<uint64_t> host(count);
    CK(cudaMemcpyAsync(host.data(), stage, count * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
    for (void* ptr : {(void*)stage, (void*)da, (void*)adev, (void*)erow, (void*)out, (void*)de, (void*)dw, (void*)ds})
      CK(cudaFreeAsync(ptr, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    const size_t row_n = K * N;
    std::memcpy(pk_out, host.data(), row_n * sizeof(uint64_t));
    std::memcpy(pk_out + row_n, a_ref, row_n * sizeof(uint64_t));
    for (size_t i = 0; i < D; ++i) {
      std::memcpy(rlk_out + (2 * i) * row_n, host.data() + (1 + i) * row_n, row_n * sizeof(uint64_t));
      std::memcpy(rlk_out + (2 * i + 1) * row_n, a_ref + (1 + i) * row_n, row_n * sizeof(uint64_t));
    }
  });
  if (st) return st;
  // install the new keys in the context
  const int s1 = hcnn_set_public_key(c, pk_out, HCNN_DOMAIN_REF_NTT);
  return s1 ? s1 : hcnn_set_relin_key(c, rlk_out, HCNN_DOMAIN_REF_NTT);
}

int hcnn_decrypt(hcnn_ctx* c, const uint32_t* cts, uint64_t* m, size_t n) {
  return guarded([&] {
    if (!c->d_sk) fail(HCNN_ERR_MISSING_KEY, "secret key required");
    if (c->t >= (1ull << 48)) fail(HCNN_ERR_UNSUPPORTED, "GPU decryption needs t < 2^48");
    CK(cudaSetDevice(c->device));
    if (!n) return;
    c->mark();
    const size_t N = c->N, K = c->K, kn = K * N;
    uint32_t* tmp = nullptr;
    pool_malloc(&tmp, n * kn * sizeof(uint32_t), c->stream, c->device);
    // c1 of every ciphertext -> tmp, then c1 * s in the NTT domain
    CK(cudaMemcpy2DAsync(tmp, kn * sizeof(uint32_t), cts + kn, 2 * kn * sizeof(uint32_t),
                         kn * sizeof(uint32_t), n, cudaMemcpyDeviceToDevice, c->stream));
    launch_ntt_rows(c, tmp, n * K, (int)K, 0, 0);
    const size_t total = n * kn;
    k_mul_sk<<<cdiv(total, 256), 256, 0, c->stream>>>(tmp, c->d_sk, (int)K, (int)N, total, c->d_prime, c->d_mu);
    c->launched("k_mul_sk");
    launch_ntt_rows(c, tmp, n * K, (int)K, 0, 1);
    k_add_c0<<<cdiv(total, 256), 256, 0, c->stream>>>(tmp, cts, (int)K, (int)N, total, c->d_prime);
    c->launched("k_add_c0");
    ConvLaunch ca{};
    ca.block = dim3(128);
    ca.grid = dim3(cdiv(N, 128), (unsigned)n);
    ca.in = tmp;
    ca.out = reinterpret_cast<uint32_t*>(m);
    conv_dispatch(c, 3, ca, "k_decrypt_round");
    CK(cudaFreeAsync(tmp, c->stream));
  });
}

int hcnn_alloc(hcnn_ctx* c, size_t bytes, void** out) {
  return guarded([&] {
    CK(cudaSetDevice(c->device));
    pool_malloc(out, bytes, c->stream, c->device);
  });
}

int hcnn_free(hcnn_ctx* c, void* ptr) {
  return guarded([&] {
    CK(cudaSetDevice(c->device));
    CK(cudaFreeAsync(ptr, c->stream));
  });
}

int hcnn_upload_u64(hcnn_ctx* c, uint32_t* dst, const uint64_t* src, size_t count) {
  return guarded([&] {
    CK(cudaSetDevice(c->device));
    uint64_t* stage = nullptr;
    pool_malloc(&stage, count * sizeof(uint64_t), c->stream, c->device);
    CK(cudaMemcpyAsync(stage, src, count * sizeof(uint64_t), cudaMemcpyHostToDevice, c->stream));
    k_narrow<<<cdiv(count, 256), 256, 0, c->stream>>>(stage, dst, count);
    c->launched("k_narrow");
    CK(cudaFreeAsync(stage, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int hcnn_download_u64(hcnn_ctx* c, uint64_t* dst, const uint32_t* src, size_t count) {
  return guarded([&] {
    CK(cudaSetDevice(c->device));
    uint64_t* stage = nullptr;
    pool_malloc(&stage, count * sizeof(uint64_t), c->stream, c->device);
    k_widen<<<cdiv(count, 256), 256, 0, c->stream>>>(src, stage, count);
    c->launched("k_widen");
    CK(cudaMemcpyAsync(dst, stage, count * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaFreeAsync(stage, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int hcnn_sync(hcnn_ctx* c) {
  return guarded([&] {
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int hcnn_weights_create(hcnn_ctx* c, const int64_t* w, size_t count, hcnn_weights** out) {
  return guarded([&] {
    if (!out || (!w && count)) fail(HCNN_ERR_PARAM, "null argument");
    CK(cudaSetDevice(c->device));
    auto h = std::make_unique<hcnn_weights>();
    h->count = count;
    int64_t big = 0;
    for (size_t i = 0; i < count; ++i) {
      const int64_t a = w[i] < 0 ? -w[i] : w[i];
      if (w[i] == INT64_MIN) big = INT64_MAX;
      else if (a > big) big = a;
    }
    h->small = big < (int64_t)WBIAS;
    const bool f64 = big < (int64_t(1) << 22);
    if (f64) {
      // after a fold |acc| < 2^31; keep |acc| + flush * big * 2^30 < 2^53
      const double room = 9007199254740992.0 - 4294967296.0;
      const double per = (double)(big > 0 ? big : 1) * 1073741824.0;
      double fl = room / per;
      h->flush = fl > (double)(1 << 20) ? (1 << 20) : (int)fl;
    }
    if (count) {
      int64_t* stage = nullptr;
      pool_malloc(&stage, count * sizeof(int64_t), c->stream, c->device);
      CK(cudaMemcpyAsync(stage, w, count * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
      if (h->small) {
        CK(cudaMalloc((void**)&h->wb, count * sizeof(uint16_t)));
        k_bias_weights<<<cdiv(count, 256), 256, 0, c->stream>>>(stage, count, h->wb);
        c->launched("k_bias_weights");
      }
      if (f64) {
        CK(cudaMalloc((void**)&h->wd, count * sizeof(double)));
        k_weights_f64<<<cdiv(count, 256), 256, 0, c->stream>>>(stage, count, h->wd);
        c->launched("k_weights_f64");
      }
      // residues mod q_i: the general path (and the fallback when a layer's
      // small weights exceed the shared-memory stage)
      CK(cudaMalloc((void**)&h->wred, count * c->K * sizeof(uint32_t)));
      k_reduce_weights<<<cdiv(count, 256), 256, 0, c->stream>>>(stage, count, h->wred, c->d_prime, (int)c->K);
      c->launched("k_reduce_weights");
      CK(cudaFreeAsync(stage, c->stream));
      CK(cudaStreamSynchronize(c->stream));
    }
    *out = h.release();
  });
}

int hcnn_weights_destroy(hcnn_ctx* c, hcnn_weights* h) {
  return guarded([&] {
    if (!h) return;
    cudaSetDevice(c->device);
    if (h->wb) cudaFree(h->wb);
    if (h->wd) cudaFree(h->wd);
    if (h->wred) cudaFree(h->wred);
    delete h;
  });
}

int hcnn_conv(hcnn_ctx* c, const uint32_t* in, uint32_t* out, int h, int w, int ch,
              const hcnn_weights* wt, int f, int kh, int kw, int sh, int sw, int padded, int groups) {
  return guarded([&] {
    c->mark();
    if (groups < 1 || ch % groups || f % groups) fail(HCNN_ERR_PARAM, "conv: channel mismatch");
    if (!wt || wt->count != (size_t)f * kh * kw * (ch / groups)) fail(HCNN_ERR_PARAM, "conv: weight count");
    ConvGeom g;
    g.h = h;
    g.w = w;
    g.c = ch;
    g.f = f;
    g.kh = kh;
    g.kw = kw;
    g.cg = ch / groups;
    g.sh = sh;
    g.sw = sw;
    g.ph = padded ? (kh - 1) / 2 : 0;
    g.pw = padded ? (kw - 1) / 2 : 0;
    g.oh = (h + 2 * g.ph - kh) / sh + 1;
    g.ow = (w + 2 * g.pw - kw) / sw + 1;
    g.per_group = f / groups;
    if (g.oh <= 0 || g.ow <= 0) fail(HCNN_ERR_PARAM, "conv: empty output");
    CK(cudaSetDevice(c->device));
    const unsigned tpb = c->N >= 512 ? 128 : (c->N / 4 >= 32 ? c->N / 4 : 32);
    int fb = 1;
    for (int cand : {8, 5, 4, 2, 1})
      if (g.per_group % cand == 0) {
        fb = cand;
        break;
      }
    size_t smem_d = (size_t)fb * kh * kw * g.cg * sizeof(double) + (size_t)kh * kw * g.cg * sizeof(int);
    const size_t smem = (size_t)fb * kh * kw * g.cg * sizeof(uint16_t);
    const int path = (wt->wd && wt->flush >= 16 && smem_d <= 96 * 1024) ? 0 : (wt->small && smem <= 48 * 1024) ? 1 : 2;
    // FP64 path: ten filters per block when the group allows (MNIST conv2:
    // every loaded input feeds 40 DFMAs instead of 20)
    if (path == 0 && g.per_group % 10 == 0 && fb < 10) {
      const size_t s10 = (size_t)10 * kh * kw * g.cg * sizeof(double) + (size_t)kh * kw * g.cg * sizeof(int);
      if (s10 <= 96 * 1024) {
        fb = 10;
        smem_d = s10;
      }
    }
    const size_t zdim = (size_t)g.oh * g.ow * (f / fb);
    if (zdim > (size_t)INT32_MAX) fail(HCNN_ERR_CAPACITY, "conv: output too large");
    if (path == 2 && !wt->wred) fail(HCNN_ERR_CAPACITY, "conv: filter too large for the small-weight kernel");
    // grid z holds at most 65535 blocks: tile the output blocks over launches
    for (size_t z0 = 0; z0 < zdim; z0 += 65535) {
      const unsigned zn = (unsigned)(zdim - z0 < 65535 ? zdim - z0 : 65535);
      g.z0 = (int)z0;
      const dim3 grid(cdiv(c->N / 4, tpb), 2 * c->K, zn);
      if (path == 0) {
        const dim3 gridp(zn, 2, cdiv(c->N / 4, tpb));
        switch (fb) {
#define X(FB)                                                                                           \
  case FB: {                                                                                            \
    static std::atomic<uint64_t> cfg{0};                                                                \
    per_device_once(cfg, [] {                                                                           \
      cudaFuncSetAttribute(k_conv_f64<FB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);     \
    });                                                                                                 \
    k_conv_f64<FB><<<gridp, tpb, smem_d, c->stream>>>(in, out, wt->wd, g, (int)c->K, (int)c->N, wt->flush, c->d_prime); \
    break;                                                                                              \
  }
          X(1) X(2) X(4) X(5) X(8) X(10)
#undef X
        }
      } else if (path == 1) {
        switch (fb) {
#define X(FB)                                                                                          \
  case FB:                                                                                             \
    k_conv_sw<FB><<<grid, tpb, smem, c->stream>>>(in, out, wt->wb, g, (int)c->K, (int)c->N, c->d_prime, c->d_mu); \
    break;
          X(1) X(2) X(4) X(5) X(8)
#undef X
        }
      } else {
        switch (fb) {
#define X(FB)                                                                                       \
  case FB:                                                                                          \
    k_conv<FB><<<grid, tpb, 0, c->stream>>>(in, out, wt->wred, g, (int)c->K, (int)c->N, c->d_prime, c->d_mu); \
    break;
          X(1) X(2) X(4) X(5) X(8)
#undef X
        }
      }
      c->launched("k_conv");
    }
  });
}

int hcnn_fc(hcnn_ctx* c, const uint32_t* in, uint32_t* out, int n_in, int n_out, const hcnn_weights* wt) {
  return guarded([&] {
    c->mark();
    if (!wt || wt->count != (size_t)n_in * n_out) fail(HCNN_ERR_PARAM, "fc: weight count");
    CK(cudaSetDevice(c->device));
    const unsigned tpb = c->N >= 512 ? 128 : (c->N / 4 >= 32 ? c->N / 4 : 32);
    constexpr int OB = 8;
    dim3 grid(cdiv(c->N / 4, tpb), 2 * c->K, cdiv(n_out, OB));
    int obs = 0;  // outputs per block of the split-K kernel: a divisor of n_out
    for (int cand : {16, 10, 8, 5, 4, 2, 1})
      if (n_out % cand == 0) {
        obs = cand;
        break;
      }
    if (wt->wd && wt->flush >= 16 && c->N >= 256) {
      // split the inputs so that the grid covers the GPU ~8 times over; the
      // block's weights (OB x chunk doubles) are staged in shared memory
      const int nob = n_out / obs;
      const unsigned bx = cdiv(c->N / 2, tpb);
      const size_t base_blocks = (size_t)bx * 2 * c->K * nob;
      int S = (int)std::min<size_t>(64, std::max<size_t>(1, (8 * 148 + base_blocks - 1) / base_blocks));
      S = std::min(S, std::max(1, n_in / 32));
      int chunk = (n_in + S - 1) / S;
      const int obp = obs + (obs & 1);
      while ((size_t)obp * chunk * sizeof(double) > 64 * 1024) chunk = (chunk + 1) / 2;
      S = (n_in + chunk - 1) / chunk;
      const size_t rows = (size_t)n_out * 2 * c->K;
      uint32_t* ws = S > 1 ? (uint32_t*)c->workspace((size_t)S * rows * c->N * sizeof(uint32_t)) : out;
      const dim3 gs((unsigned)(nob * S), 2 * c->K, bx);  // output blocks fastest (L2 reuse of input slabs)
      const size_t smem = (size_t)obp * chunk * sizeof(double);
      switch (obs) {
#define X(OBS)                                                                                             \
  case OBS: {                                                                                              \
    static std::atomic<uint64_t> cfg{0};                                                                   \
    per_device_once(cfg, [] {                                                                              \
      cudaFuncSetAttribute(k_fc_f64_split<OBS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);   \
    });                                                                                                    \
    k_fc_f64_split<OBS><<<gs, tpb, smem, c->stream>>>(in, ws, wt->wd, n_in, n_out, (int)c->K, (int)c->N,   \
                                                      wt->flush, chunk, nob, c->d_prime);                  \
    break;                                                                                                 \
  }
        X(16) X(10) X(8) X(5) X(4) X(2) X(1)
#undef X
      }
      c->launched("k_fc");
      if (S > 1) {
        const size_t quads = rows * c->N / 4;
        k_fc_reduce<<<cdiv(quads, 256), 256, 0, c->stream>>>(ws, out, S, rows, (int)c->K, (int)c->N, c->d_prime);
        c->launched("k_fc_reduce");
      }
      return;
    }
    if (wt->wd && wt->flush >= 8) {
      k_fc_f64<OB, 256><<<grid, tpb, 0, c->stream>>>(in, out, wt->wd, n_in, n_out, (int)c->K, (int)c->N, wt->flush, c->d_prime);
      c->launched("k_fc");
      return;
    }
    const size_t smem = (size_t)OB * n_in * sizeof(uint16_t);
    if (wt->small && smem <= 48 * 1024) {
      k_fc_sw<OB><<<grid, tpb, smem, c->stream>>>(in, out, wt->wb, n_in, n_out, (int)c->K, (int)c->N, c->d_prime, c->d_mu);
      c->launched("k_fc");
      return;
    }
    if (!wt->wred) fail(HCNN_ERR_CAPACITY, "fc: layer too wide for the small-weight kernel");
    k_fc<OB><<<grid, tpb, 0, c->stream>>>(in, out, wt->wred, n_in, n_out, (int)c->K, (int)c->N, c->d_prime, c->d_mu);
    c->launched("k_fc");
  });
}

int hcnn_pool(hcnn_ctx* c, const uint32_t* in, uint32_t* out, int h, int w, int ch, int e, int sh, int sw) {
  return guarded([&] {
    c->mark();
    CK(cudaSetDevice(c->device));
    const int oh = (h - e) / sh + 1, ow = (w - e) / sw + 1;
    if (oh <= 0 || ow <= 0) fail(HCNN_ERR_PARAM, "pool: empty output");
    const size_t nout = (size_t)oh * ow * ch;
    if (nout > (size_t)INT32_MAX) fail(HCNN_ERR_CAPACITY, "pool: output too large");
    const unsigned tpb = c->N >= 512 ? 128 : (c->N / 4 >= 32 ? c->N / 4 : 32);
    for (size_t o0 = 0; o0 < nout; o0 += 65535) {  // grid z <= 65535 blocks per launch
      const unsigned zn = (unsigned)(nout - o0 < 65535 ? nout - o0 : 65535);
      dim3 grid(cdiv(c->N / 4, tpb), 2 * c->K, zn);
      k_pool<<<grid, tpb, 0, c->stream>>>(in, out, h, w, ch, e, sh, sw, ow, (int)c->K, (int)c->N, c->d_prime,
                                          c->d_mu, (int)o0);
      c->launched("k_pool");
    }
  });
}

int hcnn_square(hcnn_ctx* c, const uint32_t* in, uint32_t* out, size_t n) {
  return guarded([&] {
    c->mark();
    require_rlk(c);
    CK(cudaSetDevice(c->device));
    multiply(c, in, in, n, nullptr, out);
  });
}

int hcnn_hmult_raw(hcnn_ctx* c, const uint32_t* a, const uint32_t* b, uint32_t* out3, size_t n) {
  return guarded([&] {
    c->mark();
    CK(cudaSetDevice(c->device));
    multiply(c, a, b, n, out3, nullptr);
  });
}

int hcnn_hmult(hcnn_ctx* c, const uint32_t* a, const uint32_t* b, uint32_t* out, size_t n) {
  return guarded([&] {
    c->mark();
    require_rlk(c);
    CK(cudaSetDevice(c->device));
    multiply(c, a, b, n, nullptr, out);
  });
}

int hcnn_relinearize(hcnn_ctx* c, const uint32_t* in3, uint32_t* out, size_t n) {
  return guarded([&] {
    c->mark();
    require_rlk(c);
    CK(cudaSetDevice(c->device));
    if (n == 0) return;
    const size_t per = (size_t)c->D * c->N * sizeof(uint32_t);
    size_t ch = c->ws_limit / (per + rb_bytes_per_ct(c));
    if (ch < 1) ch = 1;
    if (ch > 65535) ch = 65535;
    if (ch > n) ch = n;
    uint32_t* dig = (uint32_t*)c->workspace(per * ch);
    const size_t K = c->K, N = c->N;
    for (size_t s = 0; s < n; s += ch) {
      const size_t m = (n - s < ch) ? n - s : ch;
      ConvLaunch ca{};
      ca.block = dim3(128);
      ca.grid = dim3(cdiv(N, 128), (unsigned)m);
      ca.in = in3 + s * 3 * K * N;
      ca.dig = dig;
      conv_dispatch(c, 2, ca, "k_digits");
      launch_relin(c, dig, in3 + s * 3 * K * N, out + s * 2 * K * N, m);
    }
  });
}

int hcnn_hfir_pack(hcnn_ctx* c, const uint32_t* rows_in, size_t rows, uint64_t* hfir) {
  return guarded([&] {
    c->mark();
    CK(cudaSetDevice(c->device));
    const size_t total = rows * c->N;
    if (!total) return;
    k_hfir_pack<<<cdiv(total, 256), 256, 0, c->stream>>>(rows_in, hfir, (int)c->K, (int)c->N, rows);
    c->launched("k_hfir_pack");
  });
}

int hcnn_hfir_unpack(hcnn_ctx* c, const uint64_t* hfir, size_t rows, uint32_t* rows_out) {
  return guarded([&] {
    c->mark();
    CK(cudaSetDevice(c->device));
    const size_t total = rows * c->N;
    if (!total) return;
    int* bad = nullptr;
    pool_malloc(&bad, sizeof(int), c->stream, c->device);
    CK(cudaMemsetAsync(bad, 0, sizeof(int), c->stream));
    k_hfir_unpack<<<cdiv(total, 256), 256, 0, c->stream>>>(hfir, rows_out, (int)c->K, (int)c->N, rows,
                                                            c->d_prime, bad);
    c->launched("k_hfir_unpack");
    int h = 0;
    CK(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaFreeAsync(bad, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (h) fail(HCNN_ERR_FORMAT, "residue not reduced modulo its prime");
  });
}

int hcnn_mul_plain(hcnn_ctx* c, const uint32_t* cts, const int64_t* pt, uint32_t* out, size_t n) {
  return guarded([&] {
    c->mark();
    CK(cudaSetDevice(c->device));
    if (!n) return;
    const size_t N = c->N, K = c->K;
    bool constant = true;
    for (size_t i = 1; i < N && constant; ++i) constant = pt[i] == 0;
    if (constant) {  // scalar fast path (bfv.py:311-314)
      std::vector<uint32_t> sres(K);
      for (size_t i = 0; i < K; ++i) {
        const int64_t p = (int64_t)c->primes[i];
        int64_t r = pt[0] % p;
        sres[i] = (uint32_t)(r < 0 ? r + p : r);
      }
      uint32_t* d_s = nullptr;
      pool_malloc(&d_s, K * sizeof(uint32_t), c->stream, c->device);
      CK(cudaMemcpyAsync(d_s, sres.data(), K * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
      const size_t total = n * 2 * K * N;
      k_mul_scalar<<<cdiv(total, 256), 256, 0, c->stream>>>(cts, out, d_s, (int)K, (int)N, total, c->d_prime,
                                                             c->d_mu);
      c->launched("k_mul_scalar");
      CK(cudaFreeAsync(d_s, c->stream));  // sres (pageable) was consumed by the copy call
      return;
    }
    int64_t* d_pt = nullptr;
    uint32_t* rows = nullptr;
    pool_malloc(&d_pt, N * sizeof(int64_t), c->stream, c->device);
    pool_malloc(&rows, K * N * sizeof(uint32_t), c->stream, c->device);
    const std::vector<int64_t> hpt(pt, pt + N);  // pageable copy: staged before the call returns
    CK(cudaMemcpyAsync(d_pt, hpt.data(), N * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    k_lift_plain<<<cdiv(N, 256), 256, 0, c->stream>>>(d_pt, rows, (int)N, (int)K, c->d_prime);
    c->launched("k_lift_plain");
    launch_ntt_rows(c, rows, K, (int)K, 0, 2);  // NTT domain, tiled layout
    NttLaunch a{};
    a.grid = dim3((unsigned)K, (unsigned)n);
    a.a = cts;
    a.b = rows;
    a.out = out;
    a.K = (int)K;
    ntt_dispatch(c, 6, a, "k_mul_plain");
    CK(cudaFreeAsync(d_pt, c->stream));
    CK(cudaFreeAsync(rows, c->stream));
  });
}

int hcnn_hadd(hcnn_ctx* c, const uint32_t* a, const uint32_t* b, uint32_t* out, size_t n) {
  return guarded([&] {
    c->mark();
    CK(cudaSetDevice(c->device));
    const size_t total = n * 2 * c->K * c->N;
    if (!total) return;
    k_hadd<<<cdiv(total, 256), 256, 0, c->stream>>>(a, b, out, (int)c->K, (int)c->N, total, c->d_prime);
    c->launched("k_hadd");
  });
}

int hcnn_ntt(hcnn_ctx* c, uint32_t* rows, size_t n_rows, uint32_t limbs, uint32_t off, int inverse) {
  return guarded([&] {
    c->mark();
    if (limbs == 0 || off + limbs > c->K + c->KP) fail(HCNN_ERR_PARAM, "ntt: prime range");
    CK(cudaSetDevice(c->device));
    launch_ntt_rows(c, rows, n_rows, (int)limbs, (int)off, inverse);
  });
}

}  // extern "C"
