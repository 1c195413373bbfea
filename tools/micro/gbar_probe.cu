// Grid barrier variants for the batched sweeps (1 CTA per SM, 148 CTAs):
//   0 cooperative_groups grid.sync()
//   1 centralised counter: atom.add.release + ld.acquire spin on a generation word
//   2 flag array: every CTA st.release's its epoch to its own word, warp 0 of
//     every CTA polls all words with ld.acquire (no atomics, no serialisation)
// each alone and with a dependent L2 round trip (load, store) between barriers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gbar_probe gbar_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

template <int MODE>
__device__ __forceinline__ void gbar(unsigned* ctr, unsigned* flags, unsigned epoch) {
  if (MODE == 0) {
    cg::this_grid().sync();
    return;
  }
  __syncthreads();
  if (MODE == 1) {
    if (threadIdx.x == 0) {
      // ctr[0]: arrivals (monotone), target = epoch * gridDim.x
      atom_add_rel(ctr, 1u);
      const unsigned target = epoch * gridDim.x;
      while ((int)(ld_acq(ctr) - target) < 0) {}
    }
  } else {
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0) st_rel(flags + blockIdx.x * 32, epoch);   // own 128-B line
      for (unsigned b = threadIdx.x; b < gridDim.x; b += 32)
        while ((int)(ld_acq(flags + b * 32) - epoch) < 0) {}
      __syncwarp();
    }
  }
  __syncthreads();
}

template <int MODE>
__global__ void k_bar(double* buf, unsigned* ctr, unsigned* flags, int iters, int work) {
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double v = 0.0;
  for (int i = 1; i <= iters; ++i) {
    if (work && threadIdx.x < 32) {   // one dependent L2 round trip per warp 0 lane
      const int64_t idx = (gt * 7919 + i * 104729) & ((1 << 20) - 1);
      v = buf[idx] + 1.0;
      buf[(idx + 4096) & ((1 << 20) - 1)] = v;
    }
    gbar<MODE>(ctr, flags, (unsigned)i);
  }
  if (v == -1.0) buf[0] = v;
}

int main() {
  double* buf;
  unsigned *ctr, *flags;
  cudaMalloc(&buf, (1 << 20) * sizeof(double));
  cudaMalloc(&ctr, 64);
  cudaMalloc(&flags, 148 * 128 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000;
  for (int work : {0, 1})
    for (int grid : {148, 74}) {
      for (int mode = 0; mode < 3; ++mode) {
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
          cudaMemset(ctr, 0, 64);
          cudaMemset(flags, 0, 148 * 128 * 4);
          int it = iters;
          void* args[] = {&buf, &ctr, &flags, &it, &work};
          const void* fn = mode == 0 ? (const void*)k_bar<0> : mode == 1 ? (const void*)k_bar<1> : (const void*)k_bar<2>;
          cudaEventRecord(e0);
          cudaLaunchCooperativeKernel(fn, grid, 256, args, 0, 0);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms; cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) best = ms;
        }
        cudaError_t err = cudaGetLastError();
        printf("work %d ctas %3d mode %d: %.3f us/barrier %s\n", work, grid, mode, best * 1e3 / iters,
               err ? cudaGetErrorString(err) : "");
      }
    }
  return 0;
}
