// nlfem_cg.cu -- conjugate gradients on the assembled system, on the device.
//
// The reference's solver is unpreconditioned CG from x = 0, stopping at the
// first iteration with ||r|| <= tol ||b|| or when p.Ap loses positivity
// (reference proj/src/solver.cpp:26-66).  Here every vector and scalar stays
// in HBM: the SpMV (warp per row) is fused with the block partials of p.Ap,
// the x / r update with the partials of r.r, and each kernel's prologue
// finishes the previous dot product from the block partials in a fixed order,
// so results are deterministic run to run.  Scalars live in a device state
// block; once converged (or broken down) every kernel is a no-op, so the host
// launches a CUDA graph of kGraphIters iterations and looks at the state only
// between graph launches.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>
#include <algorithm>

#include "nlfem_gpu.h"

namespace {

#define CKC(x)                                                                          \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      throw std::runtime_error(std::string(#x) + ": " + cudaGetErrorString(e_));        \
  } while (0)

constexpr unsigned FULL = 0xffffffffu;
constexpr int kThreads = 256;
constexpr int kMaxBlocks = 148 * 4;  // fixed partition of every dot product
constexpr int kGraphIters = 16;

struct CgState {
  double rr;      // r.r of the current residual (read by every block of k_update_xr)
  double rr_new;  // published by k_update_p, promoted to rr by the next k_spmv_dot
  double alpha, beta;
  double bnorm;   // ||b||
  double tol;
  int iters, done, converged, pad;
};

__device__ __forceinline__ double warp_sum(double v) {
  for (int sh = 16; sh > 0; sh >>= 1) v += __shfl_xor_sync(FULL, v, sh);
  return v;
}

// block sum in a fixed tree; the result is valid in thread 0
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double ws[kThreads / 32];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < kThreads / 32 ? ws[threadIdx.x] : 0.0;
    t = warp_sum(t);
  }
  __syncthreads();
  return t;
}

// sum of the G block partials in a fixed order (every block computes the same)
__device__ __forceinline__ double sum_partials(const double* part, int G) {
  double v = 0;
  for (int i = threadIdx.x; i < G; i += kThreads) v += part[i];
  __shared__ double tot;
  const double t = block_sum(v);
  if (threadIdx.x == 0) tot = t;
  __syncthreads();
  return tot;
}

__global__ void k_init(int n, const double* b, double* x, double* r, double* p, double* part,
                       int G) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    x[i] = 0.0;
    r[i] = b[i];
    p[i] = b[i];
  }
  double v = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    v += b[i] * b[i];
  const double t = block_sum(v);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

__global__ void k_init_state(CgState* s, const double* part, int G, double tol, int max_iter) {
  const double bb = sum_partials(part, G);
  if (threadIdx.x == 0) {
    s->rr = bb;
    s->rr_new = bb;
    s->bnorm = sqrt(bb);
    s->tol = tol;
    s->iters = 0;
    s->converged = bb == 0.0;
    s->done = bb == 0.0 || max_iter <= 0;
  }
}

// Ap = A p (warp per row) and the block partials of p.Ap
__global__ void __launch_bounds__(kThreads) k_spmv_dot(int n, const int64_t* rowp, const int* col,
                                                       const double* val, const double* p,
                                                       double* Ap, double* part,
                                                       CgState* s) {
  if (s->done) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) s->rr = s->rr_new;  // k_update_xr reads it next
  const int lane = threadIdx.x & 31;
  const int wpb = kThreads / 32;
  double acc_dot = 0;
  for (int row = blockIdx.x * wpb + (threadIdx.x >> 5); row < n; row += gridDim.x * wpb) {
    double acc = 0;
    for (int64_t k = rowp[row] + lane; k < rowp[row + 1]; k += 32) acc += val[k] * p[col[k]];
    acc = warp_sum(acc);
    if (lane == 0) {
      Ap[row] = acc;
      acc_dot += p[row] * acc;
    }
  }
  const double t = block_sum(acc_dot);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// alpha = rr / pAp (breakdown stops), x += alpha p, r -= alpha Ap, partials of r.r
__global__ void __launch_bounds__(kThreads) k_update_xr(int n, double* x, double* r,
                                                        const double* p, const double* Ap,
                                                        const double* part_in, double* part_out,
                                                        int G, CgState* s) {
  if (s->done) return;
  const double pAp = sum_partials(part_in, G);
  if (!(pAp > 0)) {  // lost positive definiteness in finite precision
    if (blockIdx.x == 0 && threadIdx.x == 0) s->done = 1;
    return;
  }
  const double alpha = s->rr / pAp;
  if (blockIdx.x == 0 && threadIdx.x == 0) s->alpha = alpha;
  double v = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * Ap[i];
    r[i] = ri;
    v += ri * ri;
  }
  const double t = block_sum(v);
  if (threadIdx.x == 0) part_out[blockIdx.x] = t;
}

// rr_next, the stopping test, beta, p = r + beta p
__global__ void __launch_bounds__(kThreads) k_update_p(int n, const double* r, double* p,
                                                       const double* part, int G, CgState* s) {
  if (s->done) return;
  const double rr_next = sum_partials(part, G);
  const bool conv = sqrt(rr_next) <= s->tol * s->bnorm;
  const double beta = rr_next / s->rr;  // s->rr is not written during this kernel
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    s->iters += 1;
    s->rr_new = rr_next;
    s->beta = beta;
    if (conv) {  // the reference keeps rr = rr_next for the reported residual
      s->converged = 1;
      s->done = 1;
    }
  }
  if (conv) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p[i] = r[i] + beta * p[i];
}

// iteration cap: the last kernel of an iteration also checks max_iter
__global__ void k_cap(CgState* s, int max_iter) {
  if (threadIdx.x == 0 && !s->done && s->iters >= max_iter) s->done = 1;
}

struct Work {
  double *x = nullptr, *r = nullptr, *p = nullptr, *Ap = nullptr, *part = nullptr,
         *part2 = nullptr;
  CgState* s = nullptr;
  ~Work() {
    cudaFree(x);
    cudaFree(r);
    cudaFree(p);
    cudaFree(Ap);
    cudaFree(part);
    cudaFree(part2);
    cudaFree(s);
  }
};

}  // namespace

extern "C" {

int nlfem_gpu_cg_device(int32_t rows, const int64_t* row_off, const int32_t* col_idx,
                        const double* values, const double* b, double tol, int32_t max_iter,
                        double* x_out, void* stream, nlfem_gpu_solve_report* report, char* err,
                        size_t errlen) {
  try {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int n = rows;
    const int G = std::max(1, std::min(kMaxBlocks, (n + kThreads - 1) / kThreads));
    const int Gs = std::max(1, std::min(kMaxBlocks, (n + kThreads / 32 - 1) / (kThreads / 32)));
    Work w;
    const size_t vb = sizeof(double) * std::max(n, 1);
    CKC(cudaMalloc(&w.x, vb));
    CKC(cudaMalloc(&w.r, vb));
    CKC(cudaMalloc(&w.p, vb));
    CKC(cudaMalloc(&w.Ap, vb));
    CKC(cudaMalloc(&w.part, sizeof(double) * kMaxBlocks));
    CKC(cudaMalloc(&w.part2, sizeof(double) * kMaxBlocks));
    CKC(cudaMalloc(&w.s, sizeof(CgState)));
    k_init<<<G, kThreads, 0, st>>>(n, b, w.x, w.r, w.p, w.part, G);
    k_init_state<<<1, kThreads, 0, st>>>(w.s, w.part, G, tol, max_iter);
    // a graph of kGraphIters iterations, replayed until the state says done
    cudaGraph_t graph;
    cudaGraphExec_t exec;
    cudaStream_t cap;
    CKC(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    CKC(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    for (int it = 0; it < kGraphIters; ++it) {
      k_spmv_dot<<<Gs, kThreads, 0, cap>>>(n, row_off, col_idx, values, w.p, w.Ap, w.part2, w.s);
      k_update_xr<<<G, kThreads, 0, cap>>>(n, w.x, w.r, w.p, w.Ap, w.part2, w.part, Gs, w.s);
      k_update_p<<<G, kThreads, 0, cap>>>(n, w.r, w.p, w.part, G, w.s);
      k_cap<<<1, 32, 0, cap>>>(w.s, max_iter);
    }
    CKC(cudaStreamEndCapture(cap, &graph));
    CKC(cudaGraphInstantiate(&exec, graph, 0));
    CgState h{};
    CKC(cudaMemcpyAsync(&h, w.s, sizeof(h), cudaMemcpyDeviceToHost, st));
    CKC(cudaStreamSynchronize(st));
    while (!h.done) {
      CKC(cudaGraphLaunch(exec, st));
      CKC(cudaMemcpyAsync(&h, w.s, sizeof(h), cudaMemcpyDeviceToHost, st));
      CKC(cudaStreamSynchronize(st));
    }
    CKC(cudaGraphExecDestroy(exec));
    CKC(cudaGraphDestroy(graph));
    CKC(cudaStreamDestroy(cap));
    if (n) CKC(cudaMemcpyAsync(x_out, w.x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    CKC(cudaStreamSynchronize(st));
    if (report) {
      // rr of the last completed iteration (rr_new); rr itself lags by one
      const double rr = h.iters > 0 ? h.rr_new : h.rr;
      report->iterations = h.iters;
      report->converged = h.converged;
      report->relative_residual = h.bnorm > 0 ? std::sqrt(rr) / h.bnorm : 0.0;
    }
    return 0;
  } catch (const std::exception& e) {
    if (err && errlen) std::snprintf(err, errlen, "%s", e.what());
    return NLFEM_GPU_ENODEVICE;
  }
}

int nlfem_gpu_cg(const nlfem_gpu_csr* sys, const double* b, double tol, int32_t max_iter,
                 int32_t device, double* x, nlfem_gpu_solve_report* report, char* err,
                 size_t errlen) {
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0) {
    if (err && errlen)
      std::snprintf(err, errlen, "no CUDA device available (the GPU path has no CPU fallback)");
    return NLFEM_GPU_ENODEVICE;
  }
  int64_t* rp = nullptr;
  int32_t* ci = nullptr;
  double *va = nullptr, *bd = nullptr, *xd = nullptr;
  int rc = 0;
  try {
    if (device >= 0) CKC(cudaSetDevice(device));
    const int n = sys->rows;
    const long long nnz = sys->nnz;
    std::vector<int64_t> rp64(sys->row_ptr, sys->row_ptr + n + 1);
    CKC(cudaMalloc(&rp, sizeof(int64_t) * (n + 1)));
    CKC(cudaMalloc(&ci, sizeof(int32_t) * std::max<long long>(nnz, 1)));
    CKC(cudaMalloc(&va, sizeof(double) * std::max<long long>(nnz, 1)));
    CKC(cudaMalloc(&bd, sizeof(double) * std::max(n, 1)));
    CKC(cudaMalloc(&xd, sizeof(double) * std::max(n, 1)));
    CKC(cudaMemcpy(rp, rp64.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice));
    if (nnz) {
      CKC(cudaMemcpy(ci, sys->col_idx, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice));
      CKC(cudaMemcpy(va, sys->values, sizeof(double) * nnz, cudaMemcpyHostToDevice));
    }
    if (n) CKC(cudaMemcpy(bd, b, sizeof(double) * n, cudaMemcpyHostToDevice));
    rc = nlfem_gpu_cg_device(n, rp, ci, va, bd, tol, max_iter, xd, nullptr, report, err, errlen);
    if (!rc && n) CKC(cudaMemcpy(x, xd, sizeof(double) * n, cudaMemcpyDeviceToHost));
  } catch (const std::exception& e) {
    if (err && errlen) std::snprintf(err, errlen, "%s", e.what());
    rc = NLFEM_GPU_ENODEVICE;
  }
  cudaFree(rp);
  cudaFree(ci);
  cudaFree(va);
  cudaFree(bd);
  cudaFree(xd);
  return rc;
}

}  // extern "C"
