// FP64 (non-tensor) DFMA peak of this GPU: the roofline denominator for the assembly kernels
// ("FP64 non-tensor peak is not in MEASURED_PEAKS.json; it must be measured
// with a DFMA microbenchmark").  Independent FMA chains per thread, all SMs, CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cuda_runtime.h>
#include <stdio.h>

template <int CH>
__global__ void k_dfma(double *out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 1.2345) out[threadIdx.x] = s;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, iters = 1 << 16;
  for (int per_sm : {4, 8}) {
    const int blocks = sms * per_sm;
    k_dfma<8><<<blocks, threads>>>(out, 1024, 0.999999, 1e-7);
    cudaEventRecord(e0);
    k_dfma<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * (double)iters * threads * blocks;
    printf("{\"kind\": \"dfma\", \"blocks_per_sm\": %d, \"tflops\": %.2f, \"ms\": %.3f, \"err\": \"%s\"}\n", per_sm,
           flops / ms / 1e9, ms, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
