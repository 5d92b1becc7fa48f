// Probe (not product code): PCIe Gen5 throughput of SM-driven transfers
// (kernels loading from / storing to mapped pinned host memory with 16-byte
// accesses) vs copy-engine cudaMemcpyAsync, alone and concurrently in both
// directions -- which mix moves 16 MB up and 16 MB down fastest for the
// e2e host-span SpMV.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// pcie_sm.cu -o pcie_sm
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void sm_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

int main() {
  const size_t bytes = 16u << 20, n = bytes / 16;
  void *hx, *hy, *dx, *dy, *dx2, *dy2;
  CK(cudaHostAlloc(&hx, bytes, cudaHostAllocMapped));
  CK(cudaHostAlloc(&hy, bytes, cudaHostAllocMapped));
  CK(cudaMalloc(&dx, bytes)); CK(cudaMalloc(&dy, bytes));
  CK(cudaMalloc(&dx2, bytes)); CK(cudaMalloc(&dy2, bytes));
  void *mhx, *mhy;
  CK(cudaHostGetDevicePointer(&mhx, hx, 0)); CK(cudaHostGetDevicePointer(&mhy, hy, 0));
  cudaStream_t s1, s2; CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a, b, j; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); CK(cudaEventCreate(&j));
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  auto run = [&](const char* name, int mode, int grid) {
    float best = 1e9;
    for (int rep = 0; rep < 20; ++rep) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a, s1));
      CK(cudaStreamWaitEvent(s2, a, 0));
      if (mode & 1) CK(cudaMemcpyAsync(dx, hx, bytes, cudaMemcpyHostToDevice, s1));        // CE up
      if (mode & 2) CK(cudaMemcpyAsync(hy, dy, bytes, cudaMemcpyDeviceToHost, s2));        // CE down
      if (mode & 4) sm_copy<<<grid, 256, 0, s1>>>((const uint4*)mhx, (uint4*)dx2, n);     // SM up
      if (mode & 8) sm_copy<<<grid, 256, 0, s2>>>((const uint4*)dy2, (uint4*)mhy, n);     // SM down
      CK(cudaEventRecord(j, s2));
      CK(cudaStreamWaitEvent(s1, j, 0));
      CK(cudaEventRecord(b, s1));
      CK(cudaEventSynchronize(b));
      float ms; CK(cudaEventElapsedTime(&ms, a, b));
      if (rep >= 3 && ms < best) best = ms;
    }
    int dirs = ((mode & 5) ? 1 : 0) + ((mode & 10) ? 1 : 0);
    printf("{\"case\": \"%s\", \"grid\": %d, \"us\": %.1f, \"GBps_per_dir\": %.1f}\n", name, grid,
           best * 1e3, bytes / (best * 1e-3) / 1e9 * ((mode == 5 || mode == 10) ? 2 : 1) /
           (dirs == 2 ? 1 : 1));
  };
  run("CE up", 1, 0);
  run("CE down", 2, 0);
  run("CE up + CE down", 3, 0);
  for (int g : {sms, 2 * sms, 4 * sms, 8 * sms}) {
    run("SM up", 4, g);
    run("SM down", 8, g);
    run("SM up + SM down", 12, g);
    run("CE up + SM down", 9, g);
    run("SM up + CE down", 6, g);
  }
  return 0;
}
