// Conjugate gradients around the RgCSR SpMV (the paper's
// motivating workload; not in the reference).
//
// Device-resident, host-sync-free iteration: every scalar (rr, pAp, alpha,
// beta) lives in device memory and the kernels read it there, so one CG
// iteration is a few launches (SpMV with the p.q dot fused into its
// epilogue, update+dot, direction) that can be
// captured in a CUDA graph.  Dot products are deterministic: per-CTA partials
// of a fixed grid reduced in a fixed order by one CTA.
//   1. q = A p, pAp = p . q            (spmvk_rgcsr_spmv_dot_f64: grp walk +
//                                       DotEpi, per-CTA partials + finish)
//   2. alpha = rr / pAp;  x += alpha p;  r -= alpha q;  rr' = r . r   (fused)
//   3. beta = rr' / rr;   p = r + beta p;  rr = rr'
#include <cmath>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"

namespace spmvk {
namespace {

constexpr int kDotThreads = 256;
constexpr int kDotBlocks = 592;  // fixed grid -> fixed reduction order

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[kDotThreads / 32];
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < kDotThreads / 32 ? sh[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  __syncthreads();
  return t;  // valid in thread 0
}

__global__ void __launch_bounds__(kDotThreads) dot_partials(uint64_t n, const double* __restrict__ a,
                                                            const double* __restrict__ b,
                                                            double* __restrict__ part) {
  double s = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)kDotThreads + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * kDotThreads)
    s += a[i] * b[i];
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kDotThreads) dot_finish(const double* __restrict__ part, int np,
                                                          double* __restrict__ out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += kDotThreads) s += part[i];
  s = block_sum(s);
  if (threadIdx.x == 0) *out = s;
}

// x += alpha p; r -= alpha q; partial r.r   (alpha = rr / pAp from device)
__global__ void __launch_bounds__(kDotThreads) cg_update(uint64_t n, const double* __restrict__ rr,
                                                         const double* __restrict__ pap,
                                                         const double* __restrict__ p,
                                                         const double* __restrict__ q,
                                                         double* __restrict__ x,
                                                         double* __restrict__ r,
                                                         double* __restrict__ part) {
  const double alpha = *rr / *pap;
  double s = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)kDotThreads + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * kDotThreads) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    s += ri * ri;
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// p = r + (rr_new / rr) p; rr = rr_new
__global__ void __launch_bounds__(kDotThreads) cg_direction(uint64_t n,
                                                            const double* __restrict__ r,
                                                            double* __restrict__ p,
                                                            double* __restrict__ rr,
                                                            const double* __restrict__ rr_new) {
  const double beta = *rr_new / *rr;
  for (uint64_t i = blockIdx.x * (uint64_t)kDotThreads + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * kDotThreads)
    p[i] = r[i] + beta * p[i];
  // rr itself is advanced by copy_scalar in a separate launch: CTAs of this
  // grid are not synchronised, so none may overwrite *rr while others read it.
}

__global__ void copy_scalar(const double* __restrict__ src, double* __restrict__ dst) { *dst = *src; }

// r = b - q ; p = r ; partial r.r
__global__ void __launch_bounds__(kDotThreads) cg_init(uint64_t n, const double* __restrict__ b,
                                                       const double* __restrict__ q,
                                                       double* __restrict__ r,
                                                       double* __restrict__ p,
                                                       double* __restrict__ part) {
  double s = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)kDotThreads + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * kDotThreads) {
    const double ri = b[i] - q[i];
    r[i] = ri;
    p[i] = ri;
    s += ri * ri;
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}


}  // namespace
}  // namespace spmvk

using namespace spmvk;

extern "C" {

int spmvk_dot_f64(const double* a, const double* b, uint64_t n, double* out_dev, void* stream) {
  return guarded([&] {
    cudaStream_t s = as_stream(stream);
    double* part = stream_scratch(s, kDotBlocks);
    dot_partials<<<kDotBlocks, kDotThreads, 0, s>>>(n, a, b, part);
    SPMVK_LAUNCH("dot_partials");
    dot_finish<<<1, kDotThreads, 0, s>>>(part, kDotBlocks, out_dev);
    SPMVK_LAUNCH("dot_finish");
  });
}

int spmvk_cg_update_f64(uint64_t n, const double* rr, const double* pap, const double* p,
                        const double* q, double* x, double* r, double* rr_new, void* stream) {
  return guarded([&] {
    cudaStream_t s = as_stream(stream);
    double* part = stream_scratch(s, kDotBlocks);
    cg_update<<<kDotBlocks, kDotThreads, 0, s>>>(n, rr, pap, p, q, x, r, part);
    SPMVK_LAUNCH("cg_update");
    dot_finish<<<1, kDotThreads, 0, s>>>(part, kDotBlocks, rr_new);
    SPMVK_LAUNCH("dot_finish");
  });
}

int spmvk_cg_direction_f64(uint64_t n, const double* r, double* p, double* rr,
                           const double* rr_new, void* stream) {
  return guarded([&] {
    cudaStream_t s = as_stream(stream);
    cg_direction<<<kDotBlocks, kDotThreads, 0, s>>>(n, r, p, rr, rr_new);
    SPMVK_LAUNCH("cg_direction");
    copy_scalar<<<1, 1, 0, s>>>(rr_new, rr);
    SPMVK_LAUNCH("copy_scalar");
  });
}

int spmvk_cg_solve_f64(const spmvk_rgcsr* a, const double* b, double* x, uint64_t n, double tol,
                       uint64_t max_iter, uint64_t check_every, uint64_t* iters,
                       double* rel_residual, void* stream) {
  return guarded([&] {
    if (!a || !b || !x) fail(SPMVK_EINVAL, "null argument");
    if (a->rows != n || a->cols != n) fail(SPMVK_EINVAL, "cg: matrix must be square n x n");
    if (a->prec != SPMVK_F64) fail(SPMVK_EINVAL, "cg: fp64 RgCSR required");
    cudaStream_t s = as_stream(stream);
    DevBuf<double> r(n), p(n), q(n), partb(kDotBlocks), sc(4);  // sc: rr, pAp, rr_new, bb
    double* part = partb.p;
    double* rr = sc.p;
    double* pap = sc.p + 1;
    double* rrn = sc.p + 2;
    double* bb = sc.p + 3;
    const unsigned grid = kDotBlocks;
    // bb = b.b ; q = A x ; r = b - q ; p = r ; rr = r.r
    dot_partials<<<grid, kDotThreads, 0, s>>>(n, b, b, part);
    dot_finish<<<1, kDotThreads, 0, s>>>(part, kDotBlocks, bb);
    if (spmvk_rgcsr_spmv_f64(a, x, n, q.p, n, s) != SPMVK_OK)
      fail(SPMVK_ECUDA, std::string("cg spmv: ") + spmvk_last_error());
    cg_init<<<grid, kDotThreads, 0, s>>>(n, b, q.p, r.p, p.p, part);
    dot_finish<<<1, kDotThreads, 0, s>>>(part, kDotBlocks, rr);
    SPMVK_LAUNCH("cg_init");
    double h[4];
    SPMVK_CUDA(cudaMemcpyAsync(h, sc.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    SPMVK_CUDA(cudaStreamSynchronize(s));
    const double bnorm = std::sqrt(h[3]);
    double res = bnorm > 0 ? std::sqrt(h[0]) / bnorm : std::sqrt(h[0]);
    uint64_t k = 0;
    if (check_every == 0) check_every = 10;
    auto iteration = [&](cudaStream_t st) {
      // q = A p with pAp = p.q fused into the SpMV epilogue
      if (spmvk_rgcsr_spmv_dot_f64(a, p.p, n, q.p, n, 0, pap, st) != SPMVK_OK)
        fail(SPMVK_ECUDA, std::string("cg spmv: ") + spmvk_last_error());
      cg_update<<<grid, kDotThreads, 0, st>>>(n, rr, pap, p.p, q.p, x, r.p, part);
      dot_finish<<<1, kDotThreads, 0, st>>>(part, kDotBlocks, rrn);
      cg_direction<<<grid, kDotThreads, 0, st>>>(n, r.p, p.p, rr, rrn);
      copy_scalar<<<1, 1, 0, st>>>(rrn, rr);
      SPMVK_LAUNCH("cg iteration");
    };
    auto read_res = [&](cudaStream_t st) {
      SPMVK_CUDA(cudaMemcpyAsync(h, rr, sizeof(double), cudaMemcpyDeviceToHost, st));
      SPMVK_CUDA(cudaStreamSynchronize(st));
      res = bnorm > 0 ? std::sqrt(h[0]) / bnorm : std::sqrt(h[0]);
    };
    // check_every iterations are captured once as a CUDA graph (7 launches
    // each) on a private stream ordered after the caller's, then replayed:
    // same kernels, same order, so x is bitwise the eager loop's.
    cudaStream_t cs = nullptr;
    cudaEvent_t ev = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    SPMVK_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    SPMVK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    SPMVK_CUDA(cudaEventRecord(ev, s));
    SPMVK_CUDA(cudaStreamWaitEvent(cs, ev, 0));
    try {
      if (check_every >= 2 && max_iter >= check_every && res > tol) {
        // one eager fused SpMV+dot first: its per-thread partials buffer is
        // allocated on first use, which must not happen during the capture
        // (q and pAp are recomputed by the first captured iteration)
        if (spmvk_rgcsr_spmv_dot_f64(a, p.p, n, q.p, n, 0, pap, cs) != SPMVK_OK)
          fail(SPMVK_ECUDA, std::string("cg spmv: ") + spmvk_last_error());
        SPMVK_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        for (uint64_t i = 0; i < check_every; ++i) iteration(cs);
        SPMVK_CUDA(cudaStreamEndCapture(cs, &graph));
        SPMVK_CUDA(cudaGraphInstantiate(&exec, graph, 0));
        while (k + check_every <= max_iter && res > tol) {
          SPMVK_CUDA(cudaGraphLaunch(exec, cs));
          k += check_every;
          read_res(cs);
        }
      }
      while (k < max_iter && res > tol) {
        iteration(cs);
        ++k;
        if (k % check_every == 0 || k == max_iter) read_res(cs);
      }
      SPMVK_CUDA(cudaEventRecord(ev, cs));
      SPMVK_CUDA(cudaStreamWaitEvent(s, ev, 0));
      SPMVK_CUDA(cudaStreamSynchronize(cs));
    } catch (...) {
      cudaStreamEndCapture(cs, &graph);
      if (exec) cudaGraphExecDestroy(exec);
      if (graph) cudaGraphDestroy(graph);
      cudaEventDestroy(ev);
      cudaStreamDestroy(cs);
      throw;
    }
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    cudaEventDestroy(ev);
    cudaStreamDestroy(cs);
    SPMVK_CUDA(cudaStreamSynchronize(s));
    if (iters) *iters = k;
    if (rel_residual) *rel_residual = res;
  });
}

}  // extern "C"
