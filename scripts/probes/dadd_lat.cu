// Dependent-chain latency of DADD / FADD / DFMA on one thread (cycles per op),
// plus the LDS->DADD chain as ordered_sum runs it.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double* out, long long* cyc, double a, double b, int n) {
  __shared__ double sh[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sh[i] = a * i;
  __syncthreads();
  if (threadIdx.x) return;
  double acc = b;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, a);
  long long t1 = clock64();
  float f = (float)b;
  for (int i = 0; i < n; ++i) f = __fadd_rn(f, (float)a);
  long long t2 = clock64();
  double s = 0;
  for (int k = 0; k < n / 1024; ++k)
    for (int i = 0; i < 1024; ++i) s = __dadd_rn(s, sh[i]);
  long long t3 = clock64();
  out[0] = acc + f + s;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 64);
  int n = 1 << 16;
  for (int rep = 0; rep < 2; ++rep) chain<<<1, 32>>>(o, c, 1e-3, 1.0, n);
  long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("dadd %.2f cyc/op, fadd %.2f cyc/op, lds+dadd %.2f cyc/op\n", h[0] / (double)n,
         h[1] / (double)n, h[2] / (double)n);
  return 0;
}
