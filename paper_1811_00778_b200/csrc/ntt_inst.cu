// One ring degree's NTT-based kernels; built once per HCNN_LOGN in parallel.
#include "ntt_kernels.cuh"

#ifndef HCNN_LOGN
#error "compile with -DHCNN_LOGN=<log2 N>"
#endif

#define HCNN_CAT2(a, b) a##b
#define HCNN_CAT(a, b) HCNN_CAT2(a, b)

cudaError_t HCNN_CAT(hcnn_ntt_launch_, HCNN_LOGN)(int op, const hcnn::NttLaunch& a) {
  return hcnn::ntt_launch<HCNN_LOGN>(op, a);
}

int HCNN_CAT(hcnn_ntt_mont_, HCNN_LOGN)(int variant) { return hcnn::ntt_variant_mont<HCNN_LOGN>(variant); }
