// Microbenchmark for the sweep design: cost of one grid barrier (cooperative
// groups, 1 CTA per SM) against a cluster barrier (one cluster of 8/16 CTAs),
// alone and with a batch-like body (n_orb orbits of 8 random L2-resident
// amplitudes each: load, rotate, store) between barriers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier_probe barrier_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>
namespace cg = cooperative_groups;

__device__ __forceinline__ void body(double2* psi, const uint32_t* rows, int n_orb, int it,
                                     int64_t gt, int64_t nt, uint32_t nrows) {
  for (int64_t o = gt; o < n_orb; o += nt) {
    uint32_t r[8];
    double2 v[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) r[t] = (rows[(o * 8 + t) % (1 << 20)] + it * 7919u) % nrows;
#pragma unroll
    for (int t = 0; t < 8; ++t) v[t] = psi[r[t]];
#pragma unroll
    for (int t = 0; t < 8; t += 2) {
      double2 a = v[t], b = v[t + 1];
      v[t] = make_double2(0.8 * a.x - 0.6 * b.x, 0.8 * a.y - 0.6 * b.y);
      v[t + 1] = make_double2(0.8 * b.x + 0.6 * a.x, 0.8 * b.y + 0.6 * a.y);
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) psi[r[t]] = v[t];
  }
}

__global__ void k_grid(double2* psi, const uint32_t* rows, int n_orb, int iters, uint32_t nrows,
                       int spread) {
  // spread: consecutive warps of work go to different CTAs (SMs)
  const int wpb = blockDim.x >> 5;
  const int64_t lw = spread ? (int64_t)(threadIdx.x >> 5) * gridDim.x + blockIdx.x
                            : (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5);
  const int64_t gt = lw * 32 + (threadIdx.x & 31);
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  for (int i = 0; i < iters; ++i) {
    body(psi, rows, n_orb, i, gt, nt, nrows);
    cg::this_grid().sync();
  }
}

__global__ void k_cluster(double2* psi, const uint32_t* rows, int n_orb, int iters, uint32_t nrows) {
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  for (int i = 0; i < iters; ++i) {
    body(psi, rows, n_orb, i, gt, nt, nrows);
    __threadfence();
    cg::this_cluster().sync();
  }
}

int main() {
  const uint32_t nrows = 853776;
  double2* psi;
  uint32_t* rows;
  cudaMalloc(&psi, nrows * sizeof(double2));
  cudaMemset(psi, 0, nrows * sizeof(double2));
  cudaMalloc(&rows, (1 << 20) * 4);
  std::vector<uint32_t> h(1 << 20);
  uint64_t s = 1;
  for (auto& x : h) { s = s * 6364136223846793005ull + 1442695040888963407ull; x = (uint32_t)(s >> 33) % nrows; }
  cudaMemcpy(rows, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2000;
  for (int n_orb : {0, 2000, 5000, 20000}) {
    for (int grid : {148, 74}) {
      for (int threads : {128, 256, 512}) {
       for (int spread : {0, 1}) {
        int it = iters;
        void* args[] = {&psi, &rows, &n_orb, &it, (void*)&nrows, &spread};
        cudaLaunchCooperativeKernel((void*)k_grid, grid, threads, args, 0, 0);
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)k_grid, grid, threads, args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t err = cudaGetLastError();
        printf("grid    n_orb %6d ctas %3d thr %4d spread %d: %.3f us/iter %s\n", n_orb, grid, threads,
               spread, ms * 1e3 / iters, err ? cudaGetErrorString(err) : "");
       }
      }
    }
    cudaFuncSetAttribute((void*)k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cl : {8, 16}) {
      for (int threads : {256, 512}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cl); cfg.blockDim = dim3(threads);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k_cluster, psi, (const uint32_t*)rows, n_orb, iters, nrows);
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, k_cluster, psi, (const uint32_t*)rows, n_orb, iters, nrows);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t err = cudaGetLastError();
        printf("cluster n_orb %6d ctas %3d thr %4d: %.3f us/iter %s\n", n_orb, cl, threads, ms * 1e3 / iters,
               err ? cudaGetErrorString(err) : "");
      }
    }
  }
  return 0;
}
