// Latency tail of small device->host readbacks (the library's count / result
// reads): pageable cudaMemcpyAsync vs pinned cudaMemcpyAsync vs a kernel
// storing into mapped pinned memory, each after a short kernel, for ~S s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o d2h_probe d2h_probe.cu
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

__global__ void k_work(double* d, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[i] = d[i] * 1.0000001 + 1.0;
}
__global__ void k_store(volatile double* h, const double* d) { h[0] = d[0]; h[1] = d[1]; }

int main(int argc, char** argv) {
  const double secs = argc > 1 ? atof(argv[1]) : 10.0;
  const int n = 1 << 22;
  double* d;
  cudaMalloc(&d, n * sizeof(double));
  cudaMemset(d, 0, n * sizeof(double));
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  std::vector<double> pageable(2);
  double* pinned;
  cudaMallocHost(&pinned, 64);
  double *mapped, *mapped_d;
  cudaHostAlloc(&mapped, 64, cudaHostAllocMapped);
  cudaHostGetDevicePointer(&mapped_d, mapped, 0);
  const char* names[] = {"pageable", "pinned", "mapped", "none", "fresh", "freshbig"};
  for (int round = 0; round < 2; ++round)
  for (int mode = 0; mode < 6; ++mode) {
    std::vector<double> lat;
    auto t_end = std::chrono::steady_clock::now() + std::chrono::duration<double>(secs);
    while (std::chrono::steady_clock::now() < t_end) {
      auto t0 = std::chrono::steady_clock::now();
      k_work<<<(n + 255) / 256, 256, 0, st>>>(d, n);
      if (mode == 0) cudaMemcpyAsync(pageable.data(), d, 16, cudaMemcpyDeviceToHost, st);
      if (mode == 1) cudaMemcpyAsync(pinned, d, 16, cudaMemcpyDeviceToHost, st);
      if (mode == 2) k_store<<<1, 1, 0, st>>>(mapped_d, d);
      double* fresh = nullptr;
      if (mode >= 4) {   // a newly allocated pageable buffer every call (numpy's np.empty)
        const size_t nb = mode == 4 ? 3200 : (1 << 20);
        fresh = (double*)malloc(nb);
        cudaMemcpyAsync(fresh, d, mode == 4 ? 3200 : 16, cudaMemcpyDeviceToHost, st);
      }
      cudaStreamSynchronize(st);
      if (fresh) free(fresh);
      lat.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
    std::sort(lat.begin(), lat.end());
    int over = 0;
    for (double v : lat) over += v > 5.0;
    printf("%-8s n %7zu p50 %.3f p99 %.3f p999 %.3f max %.1f ms  >5ms: %d\n", names[mode], lat.size(),
           lat[lat.size() / 2], lat[lat.size() * 99 / 100], lat[lat.size() * 999 / 1000], lat.back(), over);
    fflush(stdout);
  }
  return 0;
}
