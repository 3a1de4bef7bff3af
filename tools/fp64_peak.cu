// tools/fp64_peak.cu — measured FP64 pipe throughput on this B200 (the
// roofline denominator for the fp64 Q-network forward):
// separately rounded DMUL/DADD (what the bit-exact engine issues under
// -fmad=false) and DFMA, 8 independent chains per thread, all SMs busy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) x[j] = __dadd_rn(__dmul_rn(x[j], a), b);  // 2 FLOP, 2 instructions
      else x[j] = __fma_rn(x[j], a, b);                          // 2 FLOP, 1 instruction
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000, threads = 512, blocks = sms * 4;
  const char* names[2] = {"dmul+dadd (separately rounded)", "dfma"};
  double best[2] = {0, 0};
  for (int rep = 0; rep < 5; ++rep) {
    for (int mode = 0; mode < 2; ++mode) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
      else k<1><<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flop = 2.0 * 8 * (double)iters * threads * blocks;
      const double tf = flop / (ms * 1e-3) / 1e12;
      if (tf > best[mode]) best[mode] = tf;
    }
  }
  printf("{\"fp64_tflops_mul_add\": %.3f, \"fp64_tflops_fma\": %.3f, \"sms\": %d, \"how\": \"%s vs %s, 8 chains/thread, %d blocks x %d threads, best of 5\"}\n",
         best[0], best[1], sms, names[0], names[1], blocks, threads);
  return 0;
}
