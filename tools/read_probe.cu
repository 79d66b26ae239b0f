// Read-bandwidth ceiling for the GRID3 matvec (config 3: 2,571,353 nodes, 14 x 9 value
// streams tiled by 32 nodes, 2.59 GB of values): how fast can the value bytes alone be read
// with (a) a linear grid-stride double2 read, (b) the matvec's own pattern (warp per 32-node
// chunk, thread per node, 126 coalesced 256-byte loads per chunk, 1 CTA of 8 warps per SM),
// (c) the same with 2 / 4 CTAs per SM.  The matvec's time over these is what any restructuring
// of its loads could still gain.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/read_probe.cu -o /tmp/read_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_linear(const double2 *__restrict__ a, long n2, double *out) {
  double acc = 0.0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) {
    const double2 v = __ldg(a + i);
    acc += v.x + v.y;
  }
  if (acc == 12345.678) *out = acc;
}

template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_tiles(const double *__restrict__ g, int nch, double *out) {
  const int lane = threadIdx.x & 31;
  const int warp0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (int c = warp0; c < nch; c += nwarps) {
#pragma unroll
    for (int q = 0; q < 14; ++q) {
      const double *B = g + ((long)q * nch + c) * 288 + lane;
#pragma unroll
      for (int e = 0; e < 9; ++e) acc += __ldg(B + 32 * e);
    }
  }
  if (acc == 12345.678) *out = acc;
}

// (d) the matvec's full value pattern: + the 13 lower blocks of node a read at node a - off_q
// (L2 re-reads, two tiles per warp load); (e) + the 27 x gathers (3 doubles per neighbour).
__constant__ int c_off[14];
template <bool X, bool SOA = false>
__global__ void __launch_bounds__(256, 1) k_full(const double *__restrict__ g, const double *__restrict__ x, int nch,
                                                 int nn, double *out) {
  const int lane = threadIdx.x & 31;
  const int warp0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (int c = warp0; c < nch; c += nwarps) {
    const int node = c * 32 + lane;
#pragma unroll
    for (int q = 0; q < 14; ++q) {
      const double *B = g + ((long)q * nch + c) * 288 + lane;
      const int m = min(node + c_off[q], nn - 1);
#pragma unroll
      for (int e = 0; e < 9; ++e) acc += __ldg(B + 32 * e);
      if (X)
#pragma unroll
        for (int t = 0; t < 3; ++t) acc += __ldg(SOA ? x + (long)t * nn + m : x + 3L * m + t);
    }
#pragma unroll
    for (int q = 1; q < 14; ++q) {
      const int m = max(node - c_off[q], 0);
      const double *B = g + ((long)q * nch + (m >> 5)) * 288 + (m & 31);
#pragma unroll
      for (int e = 0; e < 9; ++e) acc += __ldg(B + 32 * e);
      if (X)
#pragma unroll
        for (int t = 0; t < 3; ++t) acc += __ldg(SOA ? x + (long)t * nn + m : x + 3L * m + t);
    }
  }
  if (acc == 12345.678) *out = acc;
}

template <class F>
static float time_ms(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  const long nodes = 137L * 137 * 137, npad = (nodes + 31) / 32 * 32, nch = npad / 32;
  const long nvals = 14 * 9 * npad;
  double *g, *out;
  cudaMalloc(&g, nvals * sizeof(double));
  cudaMalloc(&out, sizeof(double));
  cudaMemset(g, 0, nvals * sizeof(double));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double gb = nvals * 8.0 / 1e9;
  const float t_lin = time_ms([&] { k_linear<<<sms * 8, 256>>>((const double2 *)g, nvals / 2, out); }, 20);
  const float t1 = time_ms([&] { k_tiles<1><<<sms, 256>>>(g, (int)nch, out); }, 20);
  const float t2 = time_ms([&] { k_tiles<2><<<2 * sms, 256>>>(g, (int)nch, out); }, 20);
  const float t4 = time_ms([&] { k_tiles<4><<<4 * sms, 256>>>(g, (int)nch, out); }, 20);
  const int nx = 137, nxy = 137 * 137;
  int off[14];
  int k = 0;
  off[k++] = 0;
  for (int dk = 0; dk <= 1; ++dk)
    for (int dj = -1; dj <= 1; ++dj)
      for (int di = -1; di <= 1; ++di) {
        const int o = di + dj * nx + dk * nxy;
        if (o > 0 && k < 14) off[k++] = o;
      }
  cudaMemcpyToSymbol(c_off, off, sizeof(off));
  double *x;
  cudaMalloc(&x, 3 * nodes * sizeof(double));
  cudaMemset(x, 0, 3 * nodes * sizeof(double));
  const float tf = time_ms([&] { k_full<false><<<sms, 256>>>(g, x, (int)nch, (int)nodes, out); }, 20);
  const float tx = time_ms([&] { k_full<true><<<sms, 256>>>(g, x, (int)nch, (int)nodes, out); }, 20);
  const float ts = time_ms([&] { k_full<true, true><<<sms, 256>>>(g, x, (int)nch, (int)nodes, out); }, 20);
  printf("{\"upper_lower_us\": %.1f, \"upper_lower_x_us\": %.1f, \"upper_lower_x_soa_us\": %.1f}\n", tf * 1e3,
         tx * 1e3, ts * 1e3);
  printf("{\"value_gb\": %.4f, \"linear_us\": %.1f, \"linear_gbs\": %.1f, \"tiles_1cta_us\": %.1f, \"tiles_1cta_gbs\": %.1f, "
         "\"tiles_2cta_us\": %.1f, \"tiles_2cta_gbs\": %.1f, \"tiles_4cta_us\": %.1f, \"tiles_4cta_gbs\": %.1f, \"err\": \"%s\"}\n",
         gb, t_lin * 1e3, gb / t_lin * 1e3, t1 * 1e3, gb / t1 * 1e3, t2 * 1e3, gb / t2 * 1e3, t4 * 1e3, gb / t4 * 1e3,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
