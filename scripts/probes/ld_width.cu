// Streaming-read bandwidth vs per-thread load width (4 / 8 / 16 B) and loads
// in flight per thread, on B200: is a 4-byte-per-lane slot stream (fp32 RgCSR:
// one 128 B line per warp request) request-rate bound below the copy peak?
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a ld_width.cu -o ld_width
#include <cstdio>
#include <cuda_runtime.h>

template <class V, int U>
__global__ void __launch_bounds__(256) rd(const V* __restrict__ p, size_t n, float* out) {
  float acc = 0.f;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    V v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float* f = reinterpret_cast<const float*>(&v[u]);
#pragma unroll
      for (int k = 0; k < (int)(sizeof(V) / 4); ++k) acc += f[k];
    }
  }
  for (; i < n; i += stride) {
    V v = __ldcs(p + i);
    acc += reinterpret_cast<const float*>(&v)[0];
  }
  if (acc == 12345.f) *out = acc;
}

template <class V, int U>
void run(const char* name, void* buf, size_t bytes, float* out, int blocks_per_sm) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t n = bytes / sizeof(V);
  dim3 grid(sms * blocks_per_sm);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) rd<V, U><<<grid, 256>>>((const V*)buf, n, out);
  cudaEventRecord(a);
  const int reps = 20;
  for (int r = 0; r < reps; ++r) rd<V, U><<<grid, 256>>>((const V*)buf, n, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("%-8s U=%d blocks/SM=%d  %.1f GB/s\n", name, U, blocks_per_sm, bytes * reps / (ms * 1e-3) / 1e9);
}

int main() {
  const size_t bytes = 1ull << 30;
  void* buf;
  float* out;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&out, 4);
  cudaMemset(buf, 0, bytes);
  for (int bps : {4, 8}) {
    run<float, 4>("float", buf, bytes, out, bps);
    run<float, 8>("float", buf, bytes, out, bps);
    run<float2, 4>("float2", buf, bytes, out, bps);
    run<float2, 8>("float2", buf, bytes, out, bps);
    run<float4, 2>("float4", buf, bytes, out, bps);
    run<float4, 4>("float4", buf, bytes, out, bps);
  }
  return 0;
}
