// Probe: shared-memory ingest rate of cp.async.bulk (TMA) vs LDG on B200, for L2-resident and
// HBM-resident sources, as a function of copy size and bytes in flight per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_probe tools/tma_probe.cu
//   tools/tma_probe
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t ph) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(b)), "r"(ph) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void mbar_wait_test(uint64_t *b, uint32_t ph) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(b)), "r"(ph) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// Each CTA walks `iters` stages; a stage = `ncopy` bulk copies of `csize` bytes from src (wrapping
// within `span` bytes, CTA-interleaved).  One thread issues, waits; nstages in flight.
__global__ void k_tma(const uint8_t *src, uint64_t span, int csize, int ncopy, int nstages, int iters, int lanes, int test) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + (size_t)nstages * csize * ncopy);
  const int lane = threadIdx.x;
  if (lane == 0)
    for (int s = 0; s < nstages; ++s) mbar_init(bar + s, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const uint64_t stage_bytes = (uint64_t)csize * ncopy;
  for (int it = 0; it < iters + nstages; ++it) {
    const int s = it % nstages;
    if (it >= nstages) {  // wait for the stage issued nstages ago
      if (test) mbar_wait_test(bar + s, ((it - nstages) / nstages) & 1);
      else mbar_wait(bar + s, ((it - nstages) / nstages) & 1);
    }
    __syncwarp();
    if (it < iters) {
      const uint64_t base = (((uint64_t)it * gridDim.x + blockIdx.x) % (span / stage_bytes)) * stage_bytes;
      if (lane == 0) mbar_expect_tx(bar + s, (uint32_t)stage_bytes);
      __syncwarp();
      if (lane < lanes)
        for (int q = lane; q < ncopy; q += lanes)
        bulk(sm + (size_t)s * stage_bytes + (size_t)q * csize, src + base + (uint64_t)q * csize, csize, bar + s);
    }
  }
}

// LDG ingest: every thread loads 16-byte vectors (L1-bypassing .cg) and accumulates.
__global__ void k_ldg(const double2 *src, uint64_t n2, int iters, double *sink) {
  double acc = 0.0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + (i + u * stride) % n2);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y;
    i += 8 * stride;
  }
  if (acc == 12345.678) *sink = acc;
}

int main() {
  const uint64_t big = 4ull << 30;
  uint8_t *buf;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 1, big);
  double *sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  struct Cfg { uint64_t span; int csize, ncopy, nstages, lanes; };
  const Cfg cfgs[] = {
      {big, 65536, 1, 3, 1},       {big, 2304, 28, 3, 32},     {big, 2304, 28, 3, 1},
      {16u << 20, 65536, 1, 3, 1}, {16u << 20, 2304, 28, 3, 32}, {16u << 20, 2304, 28, 3, 1},
      {16u << 20, 32768, 1, 6, 1}, {16u << 20, 16384, 1, 12, 1}, {16u << 20, 8192, 1, 24, 1},
      {big, 32768, 1, 6, 1},       {big, 16384, 1, 12, 1},     {big, 8192, 4, 6, 4},
      {16u << 20, 2304, 14, 6, 32}, {big, 2304, 14, 6, 32},    {64u << 20, 2304, 28, 3, 32},
  };
  for (int test = 0; test < 2; ++test)
  for (const Cfg &c : cfgs) {
    const uint64_t stage = (uint64_t)c.csize * c.ncopy;
    const int iters = (int)std::min<uint64_t>(4000, (8ull << 30) / (stage * sms));
    const size_t smem = stage * c.nstages + 8 * c.nstages;
    k_tma<<<sms, 32, smem>>>(buf, c.span, c.csize, c.ncopy, c.nstages, 10, c.lanes, test);
    cudaEventRecord(e0);
    k_tma<<<sms, 32, smem>>>(buf, c.span, c.csize, c.ncopy, c.nstages, iters, c.lanes, test);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)stage * iters * sms;
    printf("{\"kind\": \"tma\", \"test_wait\": %d, \"span_MB\": %llu, \"copy_B\": %d, \"copies\": %d, \"stages\": %d, \"issuing_lanes\": %d, "
           "\"inflight_KB\": %.0f, \"GBs\": %.1f, \"GBs_per_SM\": %.2f, \"err\": \"%s\"}\n",
           test, (unsigned long long)(c.span >> 20), c.csize, c.ncopy, c.nstages, c.lanes, stage * c.nstages / 1024.0,
           bytes / ms / 1e6, bytes / ms / 1e6 / sms, cudaGetErrorString(cudaGetLastError()));
  }
  const uint64_t spans[] = {16u << 20, 64u << 20, big};
  for (uint64_t span : spans) {
    for (int threads : {256, 512, 1024}) {
      const uint64_t n2 = span / 16;
      const int iters = 200;
      k_ldg<<<sms, threads>>>((const double2 *)buf, n2, 10, sink);
      cudaEventRecord(e0);
      k_ldg<<<sms, threads>>>((const double2 *)buf, n2, iters, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = 16.0 * 8 * iters * (double)sms * threads;
      printf("{\"kind\": \"ldg\", \"span_MB\": %llu, \"threads\": %d, \"GBs\": %.1f, \"GBs_per_SM\": %.2f}\n",
             (unsigned long long)(span >> 20), threads, bytes / ms / 1e6, bytes / ms / 1e6 / sms);
    }
  }
  return 0;
}
