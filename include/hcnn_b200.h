/* hcnn_b200.h — C ABI of the B200 backend for HCNN's homomorphic-evaluation
 * hot path (RNS-BFV over Z_q[X]/(X^N+1), exact FV scaling, base-w relin).
 *
 * The reference (hefir, pure Python) has no FFI; its seam is the Python layer
 * API of engine.py / bfv.py.  Each entry point below replaces one reference
 * function; the Python mirror (paper_1811_00778_b200/engine.py) binds them
 * with ctypes behind the reference's own signatures.
 *
 * Conventions
 *   - Ciphertext tensors live in device memory as u32 residues, limb-major:
 *     [ct][part][limb][N] (parts = 2, or 3 for a raw product).  Residues are
 *     canonical [0, p_i), coefficient domain, exactly the reference's
 *     RingElem.residues (ring.py:98-112) narrowed from int64.
 *   - Device pointers are plain pointers (the caller may allocate them with
 *     hcnn_alloc or with any CUDA allocator, e.g. torch's).  All work is
 *     enqueued on the context's stream; call hcnn_sync to wait.
 *   - Every function returns 0 on success or an HCNN_ERR_* code;
 *     hcnn_last_error() gives the message (thread-local).  The codes map onto
 *     the reference's exception hierarchy (errors.py:4-54).
 */
#ifndef HCNN_B200_H
#define HCNN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  HCNN_OK = 0,
  HCNN_ERR_PARAM = 1,       /* ParameterMismatchError (bfv.py:146-148, engine.py:248-251) */
  HCNN_ERR_MISSING_KEY = 2, /* MissingKeyError (bfv.py:370-371, 437-438) */
  HCNN_ERR_CAPACITY = 3,    /* CapacityError (engine.py:109-112) */
  HCNN_ERR_UNSUPPORTED = 4, /* UnsupportedParametersError (presets.py:72-88) */
  HCNN_ERR_CUDA = 5,        /* device / runtime failure */
  HCNN_ERR_DOMAIN = 6,      /* DomainError (ring.py:147-163) */
  HCNN_ERR_FORMAT = 7       /* FormatError (serial.py:53-72) */
};

enum { HCNN_DOMAIN_COEFF = 0, HCNN_DOMAIN_REF_NTT = 1 };

typedef struct hcnn_ctx hcnn_ctx;

/* Context for one BFV parameter set (one plaintext-CRT channel t).
 * Replaces RnsContext + NttPlan + BfvParams construction
 * (ring.py:51-95, ntt.py:88-108, bfv.py:45-91, presets.py:145-162).
 * primes: k RNS primes of q (< 2^30, = 1 mod 2n); log2w in {8, 16, 32}. */
int hcnn_ctx_create(hcnn_ctx** out, uint32_t n, uint32_t k, const uint64_t* primes, uint64_t t,
                    uint32_t log2w, int device);
int hcnn_ctx_destroy(hcnn_ctx* ctx);
/* stream: a cudaStream_t to enqueue on (NULL = the legacy default stream);
 * until this is called the context uses a private non-blocking stream. */
int hcnn_ctx_set_stream(hcnn_ctx* ctx, void* stream);
/* HCNN_Q_*: query context properties */
enum {
  HCNN_Q_N = 0,
  HCNN_Q_K = 1,
  HCNN_Q_KP = 2,       /* primes of the auxiliary base P */
  HCNN_Q_DIGITS = 3,   /* l + 1 relinearisation digits (bfv.py:70-76) */
  HCNN_Q_LOG2W = 4,
  HCNN_Q_WS_BYTES = 5, /* workspace currently held */
  HCNN_Q_KERNELS = 6,  /* kernels launched since creation */
  HCNN_Q_NTT_VARIANT = 7,
  HCNN_Q_RELIN_RBASIS = 8, /* 1 when relinearisations of at least HCNN_OPT_RB_MIN_BATCH ciphertexts take
                              the shared-basis R path (flag + parameters) */
  HCNN_Q_TC_BCONV = 9      /* 1 when the multiply's base conversions of chunks of at least 12
                              ciphertexts run on the tensor cores (flag 32768 + parameters) */
};
/* Tuning options.  HCNN_OPT_NTT_VARIANT: geometry flags of the fused NTT
 * kernels: 16 one-row relinearisation, 32 radix-32 square tensor, 64
 * mixed-width passes, 512 two-CTA cluster rows (N = 2^14, 2^15), 1024
 * relinearisation sums in TMEM, 2048 square tensor with one-row transforms
 * and rows parked in TMEM, 4096 square tensor with pair transforms and d2
 * parked in TMEM, 8192 persistent square tensor (one CTA per SM, TMA
 * prefetch of the next item's rows), 16384 relinearisation over a shared
 * three-prime basis R (digit NTTs mod 3 primes instead of mod every q_j, exact
 * CRT back; N = 2^12 to 2^15 (2-CTA clusters at 2^15), at most 23 digits,
 * at least 8 primes), 32768 the multiply's exact base conversions (k_extend,
 * k_scale) as u8 x u8 -> s32 tcgen05 MMAs (at most 15 primes in Q and P,
 * N >= 128), 65536 the relinearisation multiply-accumulate over R on the
 * tensor cores (k_rb_mac_tc; exact, opt-in: slower than the integer kernel at
 * every measured size).  Default: 32768 from K = 8 primes, plus per N 8192|16384 at 2^13,
 * 64|1024|4096|16384 at 2^14, 512|2048|16384 at 2^15.
 * Results are identical for every setting. */
/* HCNN_OPT_TS_CHUNK: ciphertexts per extend/tensor/scale sub-chunk of a
 * multiply (the tensor's output of one sub-chunk stays in L2 for the scale
 * kernel); 0 = the whole chunk at once. */
/* HCNN_OPT_RB_MIN_BATCH: smallest number of ciphertexts relinearised over R
 * (flag 16384) in one call; smaller batches take the per-prime kernel, which
 * is faster there (default 12). */
enum { HCNN_OPT_NTT_VARIANT = 1, HCNN_OPT_TS_CHUNK = 2, HCNN_OPT_RB_MIN_BATCH = 3 };
int hcnn_ctx_set_option(hcnn_ctx* ctx, int key, int64_t value);
int64_t hcnn_ctx_query(hcnn_ctx* ctx, int what);
/* psi (primitive 2N-th root) of prime i, i < K + KP (ntt.py:50-60) */
uint64_t hcnn_ctx_prime(hcnn_ctx* ctx, int i, uint64_t* psi);
/* upper bound on the multiply / relinearisation scratch the context may hold
 * per call: the workspace plus the relinearisation-over-R spectra (default
 * 12 GiB; batches are chunked to fit) */
int hcnn_ctx_set_workspace_limit(hcnn_ctx* ctx, size_t bytes);

/* Relinearisation key, host u64 [digits][2][K][N] (RelinKey.components,
 * bfv.py:129-133, 177-187).  domain: HCNN_DOMAIN_REF_NTT for the in-memory
 * reference keys (natural-order NTT), HCNN_DOMAIN_COEFF for serialised ones
 * (serial.py:87-90, 171-187). */
int hcnn_set_relin_key(hcnn_ctx* ctx, const uint64_t* rlk, int domain);

/* Public key, host u64 [2][K][N] (PublicKey b_ntt, a_ntt; bfv.py:122-126). */
int hcnn_set_public_key(hcnn_ctx* ctx, const uint64_t* pk, int domain);
/* Client-side encryption of n plaintext polys with host-drawn randomness
 * (bfv.py:201-216): u [n][N] in {0,1}, e1/e2 [n][N] in [-19,19], msg [n][N]
 * in [0,t) (all host), out: device [n][2][K][N]. */
int hcnn_encrypt(hcnn_ctx* ctx, const int8_t* u, const int8_t* e1, const int8_t* e2,
                 const int64_t* msg, uint32_t* out, size_t n);

/* Same, with the plaintext polys already on the device (e.g. hcnn_codec_encode). */
int hcnn_encrypt_device_msg(hcnn_ctx* ctx, const int8_t* u, const int8_t* e1, const int8_t* e2,
                            const int64_t* msg_dev, uint32_t* out, size_t n);

/* Client-side decryption (bfv.py:219-250): secret key bits s (N bytes, 0/1),
 * then m = round(t (c0 + c1 s) / q) mod t for n 2-part ciphertexts (device
 * [n][2][K][N] u32) into device u64 [n][N].  Exact (multiword decision near
 * rounding boundaries); needs t < 2^48. */
int hcnn_set_secret_key(hcnn_ctx* ctx, const uint8_t* s_bits);
int hcnn_decrypt(hcnn_ctx* ctx, const uint32_t* cts, uint64_t* m, size_t n);

/* SIMD slot codec over Z_t (batching.py:41-95) on the u64 NTT: slot i is the
 * evaluation at zeta^(2i+1), zeta the reference's root (ntt.py:50-60).  t: a
 * prime below 2^62 with 2N | t-1.  rows of N u64 on the device. */
typedef struct hcnn_codec hcnn_codec;
int hcnn_codec_create(uint64_t t, uint32_t n, int device, hcnn_codec** out);
int hcnn_codec_destroy(hcnn_codec* codec);
int hcnn_codec_encode(hcnn_codec* codec, const uint64_t* slots, uint64_t* polys, size_t rows, void* stream);
int hcnn_codec_decode(hcnn_codec* codec, const uint64_t* polys, uint64_t* slots, size_t rows, void* stream);
/* The u64 negacyclic NTT itself (ntt.py:113-154 for primes up to 62 bits;
 * replaces transform_rows on wide primes), in place on n_rows device rows of
 * N u64 over the codec's prime: forward (inverse = 0) natural order in,
 * bit-reversed positions out (out[i] = a(zeta^(2 brv(i) + 1))); inverse = 1
 * the way back.  Canonical residues in and out.  One CTA per row up to 2^14,
 * a 2-CTA cluster at 2^15. */
int hcnn_ntt64(hcnn_codec* codec, uint64_t* rows, size_t n_rows, int inverse, void* stream);

/* Device memory helpers (stream-ordered). */
int hcnn_alloc(hcnn_ctx* ctx, size_t bytes, void** out);
int hcnn_free(hcnn_ctx* ctx, void* ptr);
/* host int64/u64 residues -> device u32 (count residues), and back */
int hcnn_upload_u64(hcnn_ctx* ctx, uint32_t* dst, const uint64_t* src, size_t count);
int hcnn_download_u64(hcnn_ctx* ctx, uint64_t* dst, const uint32_t* src, size_t count);
int hcnn_sync(hcnn_ctx* ctx);

/* Layer weights (host int64, any sign) uploaded once.  Each weight w acts
 * as w mod q_i on limb i, exactly like ring.accumulate_scaled (ring.py:199-207,
 * RnsContext.reduce_scalar ring.py:91-95); weights below 2^15 in magnitude
 * additionally get the lazy biased-u16 kernels. */
typedef struct hcnn_weights hcnn_weights;
int hcnn_weights_create(hcnn_ctx* ctx, const int64_t* w, size_t count, hcnn_weights** out);
int hcnn_weights_destroy(hcnn_ctx* ctx, hcnn_weights* w);

/* Convolution layer: engine.eval_conv (engine.py:237-303).
 * in: h*w*c cts, (y,x,c) row-major; weights [f][kh][kw][c/groups]. */
int hcnn_conv(hcnn_ctx* ctx, const uint32_t* in, uint32_t* out, int h, int w, int c,
              const hcnn_weights* wt, int f, int kh, int kw, int sh, int sw, int padded,
              int groups);
/* Dense layer: engine.eval_fc (engine.py:306-334); weights [n_out][n_in]. */
int hcnn_fc(hcnn_ctx* ctx, const uint32_t* in, uint32_t* out, int n_in, int n_out,
            const hcnn_weights* wt);
/* Sum-pool layer: engine.eval_pool (engine.py:367-397). */
int hcnn_pool(hcnn_ctx* ctx, const uint32_t* in, uint32_t* out, int h, int w, int c, int extent,
              int sh, int sw);
/* Square activation over n cts: engine.eval_square / bfv.hsquare
 * (engine.py:337-364, bfv.py:435-443). */
int hcnn_square(hcnn_ctx* ctx, const uint32_t* in, uint32_t* out, size_t n);
/* 3-part scaled tensor: bfv.hmult_raw (bfv.py:407-416); b may equal a. */
int hcnn_hmult_raw(hcnn_ctx* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out3, size_t n);
/* ct x ct multiply + relinearise: bfv.hmult (bfv.py:419-432). */
int hcnn_hmult(hcnn_ctx* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out, size_t n);
/* 3-part -> 2-part key switch: bfv.relinearize (bfv.py:368-404). */
int hcnn_relinearize(hcnn_ctx* ctx, const uint32_t* in3, uint32_t* out, size_t n);
/* HFIR element bodies (serial.py:87-97: u64 LE, position-major then prime)
 * <-> device ciphertext rows.  rows = ciphertexts x parts; `hfir` is a DEVICE
 * buffer of rows * N * K u64.  unpack returns HCNN_ERR_FORMAT if a residue is
 * not below its prime (the device store keeps canonical residues only). */
int hcnn_hfir_pack(hcnn_ctx* ctx, const uint32_t* rows_in, size_t rows, uint64_t* hfir);
int hcnn_hfir_unpack(hcnn_ctx* ctx, const uint64_t* hfir, size_t rows, uint32_t* rows_out);
/* Key generation from host-drawn randomness (bfv.keygen, bfv.py:164-188): the
 * NTT-domain arithmetic on the device, bit-identical keys.  s_bits: N binary
 * coefficients; a_ref: [1+D][K][N] uniform residues in the reference NTT order
 * (row 0 for pk, row 1+i for rlk component i); e: [1+D][N] Gaussian noise.
 * Outputs (HOST, reference NTT order): pk_out [2][K][N] = (b, a), rlk_out
 * [D][2][K][N] = (k0_i, a_i).  The keys are also installed in the context
 * (public, relinearisation and decryption key). */
int hcnn_keygen(hcnn_ctx* ctx, const uint8_t* s_bits, const uint64_t* a_ref, const int8_t* e,
                uint64_t* pk_out, uint64_t* rlk_out);
/* ct x plaintext polynomial for n cts: bfv.hmult_plain (bfv.py:301-318).
 * pt: HOST pointer to the N centred plaintext coefficients (Plaintext.centered()).
 * A constant plaintext takes the scalar path (poly_mul_scalar, ring.py:193-196),
 * any other the NTT path; both equal the reference bit for bit. */
int hcnn_mul_plain(hcnn_ctx* ctx, const uint32_t* cts, const int64_t* pt, uint32_t* out, size_t n);
/* Elementwise add of two ct tensors: bfv.hadd (bfv.py:264-274). */
int hcnn_hadd(hcnn_ctx* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out, size_t n);
/* In-place NTT of n_rows rows of N residues; row r uses prime
 * prime_offset + r % limbs (indices over Q then P).  inverse = 0 forward.
 * Device spectral order: dev[i] = ref[brv(i)] (ring.py:147-163). */
int hcnn_ntt(hcnn_ctx* ctx, uint32_t* rows, size_t n_rows, uint32_t limbs, uint32_t prime_offset,
             int inverse);

/* Host-side staging of the reference's residue arrays (no device work):
 * dst[i * len + j] = (uint32_t)src[i][j] for count HOST int64 arrays of len
 * residues each (RingElem.residues, ring.py:98-112: canonical [0, p), p <
 * 2^30) into one HOST buffer (normally pinned, for the upload), split over
 * `threads` host threads (<= 0: all cores).  HCNN_ERR_PARAM if a value lies
 * outside [0, 2^32).  This is what engine.upload / eval_network do to a
 * host CipherTensor before it crosses PCIe (engine.py:42-58 objects in). */
int hcnn_host_narrow(const int64_t* const* src, size_t count, size_t len, uint32_t* dst, int threads);

/* The way back (no device work): dst[i][j] = src[i * len + j] for count HOST
 * int64 arrays of len residues (the caller's freshly allocated
 * RingElem.residues) from one HOST u32 buffer (normally the pinned download
 * of a result tensor), split over `threads` host threads (<= 0: all cores).
 * What engine.eval_network does to hand a host CipherTensor back
 * (engine.py:42-58 objects out). */
int hcnn_host_widen(const uint32_t* src, size_t count, size_t len, int64_t* const* dst, int threads);

/* Return the library pool's free memory on `device` to the driver (the pool
 * keeps freed blocks across synchronisations otherwise).  Synchronises the
 * device; workspaces owned by live contexts are not freed. */
int hcnn_release_memory(int device);

/* Plaintext-CRT recombination on the device (engine.reconstruct_logits,
 * engine.py:494-506 / CrtSystem.reconstruct_centered, codec.py:79-89):
 * res: DEVICE u64 [n_moduli][count], residue of value m mod moduli[i] at
 * [i][m], each in [0, moduli[i]); moduli: HOST, pairwise coprime, in
 * [2, 2^62), at most 16.  out: DEVICE u32 [count][words], the centred value
 * (X - T when X > floor(T/2), T = prod moduli) as little-endian two's
 * complement words; words must exceed the word length of T.  Runs on
 * `stream` of `device`.  flag: NULL = the range check is done here (the
 * call synchronises the stream and returns HCNN_ERR_PARAM for a residue
 * outside its range, which the reference raises as HefirError); else a
 * DEVICE int (zeroed by the caller) that the kernel sets non-zero on a bad
 * residue, and the call stays asynchronous. */
int hcnn_crt_combine(const uint64_t* res, const uint64_t* moduli, int n_moduli, size_t count, uint32_t* out,
                     int words, int* flag, int device, void* stream);

/* Per-kernel CUDA-event timing on the context's stream.  hcnn_profile(ctx, 1)
 * resets and starts recording; hcnn_profile_dump writes "name count total_ms"
 * lines (returns the text length, or -status). */
int hcnn_profile(hcnn_ctx* ctx, int enable);
int64_t hcnn_profile_dump(hcnn_ctx* ctx, char* buf, size_t len);

/* Integer-pipe probe (roofline denominator): kind 0 = 32-bit IMAD,
 * 1 = IMAD.HI (umulhi), 2 = IMAD.WIDE (32x32->64), 8 = register-resident
 * Harvey butterflies on u32 residues (the NTT kernels' attainable rate),
 * 16 = the same on 62-bit u64 residues (the u64 NTT's); ops per second. */
int hcnn_int_peak(int device, int kind, double* ops_per_s);

const char* hcnn_last_error(void);
const char* hcnn_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HCNN_B200_H */
