// Base-conversion kernels for one prime count K of q (-DHCNN_K=K); the
// auxiliary base has KP = K+2 or K+3 primes (tables.hpp / hcnn.cu).
#include "conv_kernels.cuh"

#ifndef HCNN_K
#error "compile with -DHCNN_K=<primes of q>"
#endif

#define HCNN_CAT2(a, b) a##b
#define HCNN_CAT(a, b) HCNN_CAT2(a, b)

cudaError_t HCNN_CAT(hcnn_conv_launch_, HCNN_K)(int op, int kp, const hcnn::ConvLaunch& a,
                                               const hcnn::ConvTabs& tb) {
  if (kp == HCNN_K + 2) return hcnn::conv_launch<HCNN_K, HCNN_K + 2>(op, a, tb);
  if (kp == HCNN_K + 3) return hcnn::conv_launch<HCNN_K, HCNN_K + 3>(op, a, tb);
  return cudaErrorInvalidValue;
}
