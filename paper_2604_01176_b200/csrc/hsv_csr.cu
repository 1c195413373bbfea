// K1b: generic CSR x sparse vector (spmspv on an arbitrary CsrMatrix,
// sparse.py:163-201).  The input vector is scattered to dense once (the
// reference's replicated view), one warp reduces one row in a fixed lane
// order, and the output support is compacted in ascending row order with the
// reference's drop rule (y != 0, or |y| >= prune).
#include <cub/cub.cuh>

#include <algorithm>

#include "hsv_common.cuh"
#include "hsv_kernels.cuh"

namespace hsv {

__global__ void k_scatter_x(const int64_t* __restrict__ idx, const double* __restrict__ val,
                            int64_t n, double* __restrict__ x) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) x[idx[i]] = val[i];
}

__global__ void k_csr_rows_mv(const int64_t* __restrict__ ro, const int64_t* __restrict__ cols,
                              const double* __restrict__ vals, const double* __restrict__ x,
                              int64_t n_rows, double prune, double* __restrict__ y,
                              int32_t* __restrict__ flag) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  const int64_t a = ro[row], b = ro[row + 1];
  double acc = 0.0;
  for (int64_t i = a + lane; i < b; i += 32) acc += vals[i] * x[cols[i]];
  acc = warp_sum(acc);
  if (lane == 0) {
    const bool keep = prune > 0.0 ? fabs(acc) >= prune : acc != 0.0;
    y[row] = acc;
    flag[row] = keep ? 1 : 0;
  }
}

__global__ void k_compact_f64(const double* __restrict__ y, const int32_t* __restrict__ flag,
                              const int64_t* __restrict__ off, int64_t n,
                              int64_t* __restrict__ oi, double* __restrict__ ov) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n || !flag[r]) return;
  oi[off[r]] = r;
  ov[off[r]] = y[r];
}


// ---- generic sparse vectors (SparseVector dot / axpy / scale, sparse.py:210-245)
__global__ void k_vec_dot(const int64_t* __restrict__ ui, const double* __restrict__ uv, int64_t nu,
                          const int64_t* __restrict__ vi, const double* __restrict__ vv, int64_t nv,
                          double* __restrict__ part) {
  double acc = 0.0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nv;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t key = vi[j];
    int64_t lo = 0, hi = nu;   // lower_bound in the ascending u indices
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ui[mid] < key) lo = mid + 1; else hi = mid;
    }
    if (lo < nu && ui[lo] == key) acc += uv[lo] * vv[j];
  }
  __shared__ double sh[32];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double x = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    x = warp_sum(x);
    if (threadIdx.x == 0) part[blockIdx.x] = x;
  }
}
__global__ void k_vec_scatter_axpy(const int64_t* __restrict__ idx, const double* __restrict__ val,
                                   int64_t n, double a, int add, double* __restrict__ d) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (add) d[idx[i]] = __dadd_rn(d[idx[i]], val[i]);
  else d[idx[i]] = __dmul_rn(a, val[i]);
}
__global__ void k_vec_flag(const double* __restrict__ d, int64_t n, double prune,
                           int32_t* __restrict__ flag) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) flag[i] = (prune > 0.0 ? fabs(d[i]) >= prune : d[i] != 0.0) ? 1 : 0;
}
__global__ void k_vec_scale(const double* __restrict__ x, int64_t n, double a, int divide,
                            double* __restrict__ y) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = divide ? __ddiv_rn(x[i], a) : __dmul_rn(a, x[i]);
}

template <typename T>
static int upload(const T* h, int64_t n, T** d) {
  HSV_TRY(dalloc(d, n));
  if (n) HSV_TRY_CUDA(cudaMemcpyAsync(*d, h, n * sizeof(T), cudaMemcpyHostToDevice, stream()));
  return HSV_OK;
}

}  // namespace hsv

using namespace hsv;

extern "C" {

int hsv_csr_spmspv(int64_t n_rows, int64_t n_cols, const int64_t* row_offsets, const int64_t* cols,
                   const double* vals, int64_t nnz, const int64_t* x_idx, const double* x_val,
                   int64_t x_nnz, double prune, int64_t* y_idx, double* y_val, int64_t* y_nnz) {
  HSV_TRY(ensure_init());
  HSV_REQUIRE(n_rows >= 0 && n_cols >= 0 && row_offsets && y_nnz, HSV_ERR_INVALID, "bad argument");
  HSV_REQUIRE(row_offsets[0] == 0 && row_offsets[n_rows] == nnz, HSV_ERR_INVALID,
              "row offsets are not a valid non-decreasing prefix");
  *y_nnz = 0;
  if (n_rows == 0 || x_nnz == 0) return HSV_OK;
  for (int64_t i = 0; i < x_nnz; ++i)
    HSV_REQUIRE(x_idx[i] >= 0 && x_idx[i] < n_cols, HSV_ERR_INVALID, "vector index out of range");
  cudaStream_t st = stream();
  int64_t *d_ro, *d_cols, *d_xi, *d_off, *d_oi;
  double *d_vals, *d_xv, *d_x, *d_y, *d_ov;
  int32_t* d_flag;
  HSV_TRY(dalloc(&d_ro, n_rows + 1));
  HSV_TRY(dalloc(&d_cols, nnz));
  HSV_TRY(dalloc(&d_vals, nnz));
  HSV_TRY(dalloc(&d_xi, x_nnz));
  HSV_TRY(dalloc(&d_xv, x_nnz));
  HSV_TRY(dalloc(&d_x, n_cols));
  HSV_TRY(dalloc(&d_y, n_rows));
  HSV_TRY(dalloc(&d_flag, n_rows));
  HSV_TRY(dalloc(&d_off, n_rows));
  HSV_TRY_CUDA(cudaMemcpyAsync(d_ro, row_offsets, (n_rows + 1) * 8, cudaMemcpyHostToDevice, st));
  if (nnz) {
    HSV_TRY_CUDA(cudaMemcpyAsync(d_cols, cols, nnz * 8, cudaMemcpyHostToDevice, st));
    HSV_TRY_CUDA(cudaMemcpyAsync(d_vals, vals, nnz * 8, cudaMemcpyHostToDevice, st));
  }
  HSV_TRY_CUDA(cudaMemcpyAsync(d_xi, x_idx, x_nnz * 8, cudaMemcpyHostToDevice, st));
  HSV_TRY_CUDA(cudaMemcpyAsync(d_xv, x_val, x_nnz * 8, cudaMemcpyHostToDevice, st));
  HSV_TRY_CUDA(cudaMemsetAsync(d_x, 0, std::max<int64_t>(n_cols, 1) * 8, st));
  k_scatter_x<<<(unsigned)((x_nnz + 255) / 256), 256, 0, st>>>(d_xi, d_xv, x_nnz, d_x);
  count_launch();
  k_csr_rows_mv<<<(unsigned)((n_rows * 32 + 255) / 256), 256, 0, st>>>(d_ro, d_cols, d_vals, d_x,
                                                                       n_rows, prune, d_y, d_flag);
  count_launch();
  HSV_CHECK_LAUNCH();
  size_t tb = 0;
  HSV_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, d_flag, d_off, n_rows, st));
  char* d_tmp = nullptr;
  HSV_TRY(dalloc(&d_tmp, tb));
  HSV_TRY_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tb, d_flag, d_off, n_rows, st));
  count_launch();
  int64_t last_off = 0;
  int32_t last_flag = 0;
  HSV_TRY_CUDA(cudaMemcpyAsync(&last_off, d_off + n_rows - 1, 8, cudaMemcpyDeviceToHost, st));
  HSV_TRY_CUDA(cudaMemcpyAsync(&last_flag, d_flag + n_rows - 1, 4, cudaMemcpyDeviceToHost, st));
  HSV_TRY(stream_sync());
  const int64_t cnt = last_off + last_flag;
  HSV_TRY(dalloc(&d_oi, cnt));
  HSV_TRY(dalloc(&d_ov, cnt));
  k_compact_f64<<<(unsigned)((n_rows + 255) / 256), 256, 0, st>>>(d_y, d_flag, d_off, n_rows, d_oi, d_ov);
  count_launch();
  HSV_CHECK_LAUNCH();
  if (cnt) {
    HSV_TRY_CUDA(cudaMemcpyAsync(y_idx, d_oi, cnt * 8, cudaMemcpyDeviceToHost, st));
    HSV_TRY_CUDA(cudaMemcpyAsync(y_val, d_ov, cnt * 8, cudaMemcpyDeviceToHost, st));
  }
  HSV_TRY(stream_sync());
  *y_nnz = cnt;
  dfree(d_ro); dfree(d_cols); dfree(d_vals); dfree(d_xi); dfree(d_xv); dfree(d_x);
  dfree(d_y); dfree(d_flag); dfree(d_off); dfree(d_tmp); dfree(d_oi); dfree(d_ov);
  return HSV_OK;
}

// Compact a dense device vector (support by the reference drop rule) to host.
static int compact_dense_to_host(const double* d_y, int64_t n, double prune, int64_t* out_idx,
                                 double* out_val, int64_t* n_out) {
  cudaStream_t st = stream();
  int32_t* d_flag;
  int64_t *d_off, *d_oi;
  double* d_ov;
  HSV_TRY(dalloc(&d_flag, n));
  HSV_TRY(dalloc(&d_off, n));
  k_vec_flag<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d_y, n, prune, d_flag);
  count_launch();
  HSV_CHECK_LAUNCH();
  size_t tb = 0;
  HSV_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, d_flag, d_off, n, st));
  char* d_tmp = nullptr;
  HSV_TRY(dalloc(&d_tmp, tb));
  HSV_TRY_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tb, d_flag, d_off, n, st));
  count_launch();
  int64_t last_off = 0;
  int32_t last_flag = 0;
  HSV_TRY_CUDA(cudaMemcpyAsync(&last_off, d_off + n - 1, 8, cudaMemcpyDeviceToHost, st));
  HSV_TRY_CUDA(cudaMemcpyAsync(&last_flag, d_flag + n - 1, 4, cudaMemcpyDeviceToHost, st));
  HSV_TRY(stream_sync());
  const int64_t cnt = last_off + last_flag;
  HSV_TRY(dalloc(&d_oi, cnt));
  HSV_TRY(dalloc(&d_ov, cnt));
  k_compact_f64<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d_y, d_flag, d_off, n, d_oi, d_ov);
  count_launch();
  HSV_CHECK_LAUNCH();
  if (cnt) {
    HSV_TRY_CUDA(cudaMemcpyAsync(out_idx, d_oi, cnt * 8, cudaMemcpyDeviceToHost, st));
    HSV_TRY_CUDA(cudaMemcpyAsync(out_val, d_ov, cnt * 8, cudaMemcpyDeviceToHost, st));
  }
  HSV_TRY(stream_sync());
  *n_out = cnt;
  dfree(d_flag); dfree(d_off); dfree(d_tmp); dfree(d_oi); dfree(d_ov);
  return HSV_OK;
}


int hsv_vec_dot(const int64_t* u_idx, const double* u_val, int64_t nu, const int64_t* v_idx,
                const double* v_val, int64_t nv, double* out) {
  HSV_TRY(ensure_init());
  HSV_REQUIRE(out, HSV_ERR_INVALID, "null output");
  *out = 0.0;
  if (nu == 0 || nv == 0) return HSV_OK;
  int64_t *d_ui, *d_vi;
  double *d_uv, *d_vv, *part, *d_r;
  HSV_TRY(upload(u_idx, nu, &d_ui));
  HSV_TRY(upload(u_val, nu, &d_uv));
  HSV_TRY(upload(v_idx, nv, &d_vi));
  HSV_TRY(upload(v_val, nv, &d_vv));
  const int grid = grid_for(nv, 256);
  HSV_TRY(dalloc(&part, grid));
  HSV_TRY(dalloc(&d_r, 1));
  k_vec_dot<<<grid, 256, 0, stream()>>>(d_ui, d_uv, nu, d_vi, d_vv, nv, part);
  count_launch();
  HSV_CHECK_LAUNCH();
  HSV_TRY(reduce_sum_f64(part, grid, 1, 1, d_r));
  HSV_TRY_CUDA(cudaMemcpyAsync(out, d_r, 8, cudaMemcpyDeviceToHost, stream()));
  HSV_TRY(stream_sync());
  dfree(d_ui); dfree(d_uv); dfree(d_vi); dfree(d_vv); dfree(part); dfree(d_r);
  return HSV_OK;
}

int hsv_vec_axpy(int64_t dim, double a, const int64_t* x_idx, const double* x_val, int64_t nx,
                 const int64_t* y_idx, const double* y_val, int64_t ny, double prune,
                 int64_t* out_idx, double* out_val, int64_t* n_out) {
  HSV_TRY(ensure_init());
  HSV_REQUIRE(n_out && dim >= 0, HSV_ERR_INVALID, "bad argument");
  *n_out = 0;
  if (dim == 0 || nx + ny == 0) return HSV_OK;
  int64_t *d_xi, *d_yi;
  double *d_xv, *d_yv, *d;
  HSV_TRY(upload(x_idx, nx, &d_xi));
  HSV_TRY(upload(x_val, nx, &d_xv));
  HSV_TRY(upload(y_idx, ny, &d_yi));
  HSV_TRY(upload(y_val, ny, &d_yv));
  HSV_TRY(dalloc(&d, dim));
  HSV_TRY_CUDA(cudaMemsetAsync(d, 0, dim * 8, stream()));
  if (nx) k_vec_scatter_axpy<<<(unsigned)((nx + 255) / 256), 256, 0, stream()>>>(d_xi, d_xv, nx, a, 0, d);
  if (ny) k_vec_scatter_axpy<<<(unsigned)((ny + 255) / 256), 256, 0, stream()>>>(d_yi, d_yv, ny, a, 1, d);
  count_launch(2);
  HSV_CHECK_LAUNCH();
  HSV_TRY(compact_dense_to_host(d, dim, prune, out_idx, out_val, n_out));
  dfree(d_xi); dfree(d_xv); dfree(d_yi); dfree(d_yv); dfree(d);
  return HSV_OK;
}

int hsv_vec_scale(const double* x, int64_t n, double a, int divide, double* y) {
  HSV_TRY(ensure_init());
  if (n == 0) return HSV_OK;
  double *d_x, *d_y;
  HSV_TRY(upload(x, n, &d_x));
  HSV_TRY(dalloc(&d_y, n));
  k_vec_scale<<<(unsigned)((n + 255) / 256), 256, 0, stream()>>>(d_x, n, a, divide, d_y);
  count_launch();
  HSV_CHECK_LAUNCH();
  HSV_TRY_CUDA(cudaMemcpyAsync(y, d_y, n * 8, cudaMemcpyDeviceToHost, stream()));
  HSV_TRY(stream_sync());
  dfree(d_x); dfree(d_y);
  return HSV_OK;
}

}  // extern "C"
