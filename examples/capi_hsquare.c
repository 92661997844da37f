/* Plain C caller of libhcnn_b200.so (no Python, no torch): the C-ABI
 * counterpart of bfv.hsquare (bfv.py:435-443) over a batch of ciphertexts.
 *
 *   capi_hsquare <in.bin> <out.bin>
 *
 * in.bin (little endian):  u32 n, u32 k, u32 count, u64 t, u32 log2w,
 *                          u64 primes[k],
 *                          u64 rlk[D][2][k][n]   (reference NTT order, D = digits),
 *                          u64 cts[count][2][k][n]
 * out.bin:                 u64 out[count][2][k][n]
 * Exit status: 0, or the HCNN_ERR_* code of the failing call.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "../include/hcnn_b200.h"

static int check(int st, const char* what) {
  if (st) fprintf(stderr, "%s: %s\n", what, hcnn_last_error());
  return st;
}

static void* read_exact(FILE* f, size_t bytes) {
  void* p = malloc(bytes ? bytes : 1);
  if (!p || fread(p, 1, bytes, f) != bytes) {
    fprintf(stderr, "short input\n");
    exit(7);
  }
  return p;
}

int main(int argc, char** argv) {
  if (argc != 3) {
    fprintf(stderr, "usage: %s in.bin out.bin\n", argv[0]);
    return 1;
  }
  FILE* f = fopen(argv[1], "rb");
  if (!f) return 1;
  uint32_t hdr[3];
  uint64_t t;
  uint32_t log2w;
  if (fread(hdr, 4, 3, f) != 3 || fread(&t, 8, 1, f) != 1 || fread(&log2w, 4, 1, f) != 1) return 7;
  const uint32_t n = hdr[0], k = hdr[1], count = hdr[2];
  uint64_t* primes = (uint64_t*)read_exact(f, (size_t)k * 8);

  hcnn_ctx* ctx = NULL;
  int st = check(hcnn_ctx_create(&ctx, n, k, primes, t, log2w, 0), "hcnn_ctx_create");
  if (st) return st;
  const size_t digits = (size_t)hcnn_ctx_query(ctx, HCNN_Q_DIGITS);
  const size_t ct_words = (size_t)2 * k * n;
  uint64_t* rlk = (uint64_t*)read_exact(f, digits * ct_words * 8);
  uint64_t* cts = (uint64_t*)read_exact(f, count * ct_words * 8);
  fclose(f);

  if ((st = check(hcnn_set_relin_key(ctx, rlk, HCNN_DOMAIN_REF_NTT), "hcnn_set_relin_key"))) return st;
  void *d_in = NULL, *d_out = NULL;
  if ((st = check(hcnn_alloc(ctx, count * ct_words * 4, &d_in), "hcnn_alloc"))) return st;
  if ((st = check(hcnn_alloc(ctx, count * ct_words * 4, &d_out), "hcnn_alloc"))) return st;
  if ((st = check(hcnn_upload_u64(ctx, (uint32_t*)d_in, cts, count * ct_words), "hcnn_upload_u64"))) return st;
  if ((st = check(hcnn_square(ctx, (const uint32_t*)d_in, (uint32_t*)d_out, count), "hcnn_square"))) return st;
  uint64_t* out = (uint64_t*)malloc(count * ct_words * 8);
  if ((st = check(hcnn_download_u64(ctx, out, (const uint32_t*)d_out, count * ct_words), "hcnn_download_u64")))
    return st;
  if ((st = check(hcnn_sync(ctx), "hcnn_sync"))) return st;

  FILE* g = fopen(argv[2], "wb");
  if (!g || fwrite(out, 8, count * ct_words, g) != count * ct_words) return 1;
  fclose(g);
  hcnn_free(ctx, d_in);
  hcnn_free(ctx, d_out);
  hcnn_ctx_destroy(ctx);
  printf("hsquare of %u ciphertexts (N=%u, %u primes, %zu digits) through the C ABI\n", count, n, k, digits);
  return 0;
}
