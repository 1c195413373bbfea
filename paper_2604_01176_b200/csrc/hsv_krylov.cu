// Block operations on a Krylov basis of device states (the FCI reference,
// fci.py: thick-restart Lanczos replacing scipy eigsh in oracle.py:99-142):
//   project:  c_j = <q_j|w> for all j in ONE launch (+ a fixed-order reduce),
//             then optionally w -= sum_j c_j q_j in one pass over the basis;
//   combine:  out = sum_j c_j q_j (Ritz vectors at a restart).
// Every reduction is in a fixed order, so repeated solves are bit-identical;
// no host round trip between the dot products and the update.
#include <algorithm>
#include <vector>

#include "hsv_common.cuh"
#include "hsv_kernels.cuh"

namespace hsv {

namespace {

constexpr int kKChunk = 8192;   // rows per partial dot block

// block (chunk x, vector j): partial <q_j|w> over the chunk
__global__ void __launch_bounds__(256) k_kdot(const double2* const* __restrict__ q,
                                              const double2* __restrict__ w, int64_t dim,
                                              double* __restrict__ part, int n_chunks) {
  const int j = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * kKChunk;
  const int64_t r1 = min(dim, r0 + kKChunk);
  const double2* qj = q[j];
  double re = 0.0, im = 0.0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    const double2 a = qj[i], b = w[i];
    re += a.x * b.x + a.y * b.y;
    im += a.x * b.y - a.y * b.x;
  }
  __shared__ double sh[2][8];
  re = warp_sum(re);
  im = warp_sum(im);
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  if (lane == 0) { sh[0][wp] = re; sh[1][wp] = im; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int k = 0; k < 8; ++k) { x += sh[0][k]; y += sh[1][k]; }
    part[((int64_t)j * n_chunks + blockIdx.x) * 2] = x;
    part[((int64_t)j * n_chunks + blockIdx.x) * 2 + 1] = y;
  }
}

// one block per vector: c_j = sum over chunks, fixed order
__global__ void k_kdot_reduce(const double* __restrict__ part, int n_chunks,
                              double* __restrict__ c) {
  const int j = blockIdx.x;
  double re = 0.0, im = 0.0;
  for (int k = threadIdx.x; k < n_chunks; k += blockDim.x) {
    re += part[((int64_t)j * n_chunks + k) * 2];
    im += part[((int64_t)j * n_chunks + k) * 2 + 1];
  }
  __shared__ double sh[2][8];
  re = warp_sum(re);
  im = warp_sum(im);
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  if (lane == 0) { sh[0][wp] = re; sh[1][wp] = im; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int k = 0; k < 8; ++k) { x += sh[0][k]; y += sh[1][k]; }
    c[2 * j] = x;
    c[2 * j + 1] = y;
  }
}

// out[i] = (accumulate ? out[i] : 0) + sign * sum_j c_j q_j[i]   (complex c, j ascending)
__global__ void k_kaxpy(const double2* const* __restrict__ q, const double* __restrict__ c, int m,
                        double2* __restrict__ out, int64_t dim, int accumulate, double sign) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < dim; i += stride) {
    double2 s = make_double2(0.0, 0.0);
    for (int j = 0; j < m; ++j) {
      const double2 a = q[j][i];
      const double cr = c[2 * j], ci = c[2 * j + 1];
      s.x += cr * a.x - ci * a.y;
      s.y += cr * a.y + ci * a.x;
    }
    double2 o = accumulate ? out[i] : make_double2(0.0, 0.0);
    o.x += sign * s.x;
    o.y += sign * s.y;
    out[i] = o;
  }
}

int basis_ptrs(const hsv_state* q, int64_t m, const hsv_sector_s* sec, double2*** d_out) {
  std::vector<double2*> h(m);
  for (int64_t j = 0; j < m; ++j) {
    HSV_REQUIRE(q[j] && q[j]->sec == sec, HSV_ERR_INVALID, "basis state %lld: bad sector",
                (long long)j);
    h[j] = q[j]->d_amp;
  }
  HSV_TRY(dalloc(d_out, std::max<int64_t>(m, 1)));
  HSV_TRY_CUDA(cudaMemcpyAsync(*d_out, h.data(), m * sizeof(double2*), cudaMemcpyHostToDevice,
                               stream()));
  return HSV_OK;
}

}  // namespace

}  // namespace hsv

using namespace hsv;

extern "C" {

int hsv_krylov_project(const hsv_state* q, int64_t m, hsv_state w, int subtract, double* c_out) {
  HSV_REQUIRE(q && w && m >= 0 && m <= 65535, HSV_ERR_INVALID, "bad argument");
  if (m == 0) return HSV_OK;
  const hsv_sector_s* sec = w->sec;
  const int64_t dim = sec->dim;
  const int n_chunks = (int)std::max<int64_t>(1, (dim + kKChunk - 1) / kKChunk);
  double2** d_q = nullptr;
  double *part = nullptr, *c = nullptr;
  HSV_TRY(basis_ptrs(q, m, sec, &d_q));
  HSV_TRY(dalloc(&part, 2 * m * (int64_t)n_chunks));
  HSV_TRY(dalloc(&c, 2 * m));
  {
    ProfScope prof("krylov");
    k_kdot<<<dim3((unsigned)n_chunks, (unsigned)m), 256, 0, stream()>>>(d_q, w->d_amp, dim, part,
                                                                          n_chunks);
    k_kdot_reduce<<<(unsigned)m, 256, 0, stream()>>>(part, n_chunks, c);
    count_launch(2);
    if (subtract) {
      k_kaxpy<<<grid_for(dim, 256), 256, 0, stream()>>>(d_q, c, (int)m, w->d_amp, dim, 1, -1.0);
      count_launch();
      w->norm2_valid = w->arow_valid = w->smap_valid = false;
      w->dense_hint = false;
    }
  }
  HSV_CHECK_LAUNCH();
  if (c_out)
    HSV_TRY_CUDA(cudaMemcpyAsync(c_out, c, 2 * m * sizeof(double), cudaMemcpyDeviceToHost,
                                 stream()));
  dfree(d_q);
  dfree(part);
  dfree(c);
  return stream_sync();
}

int hsv_krylov_combine(const hsv_state* q, int64_t m, const double* coeff, hsv_state out) {
  HSV_REQUIRE(q && out && coeff && m >= 0 && m <= 65535, HSV_ERR_INVALID, "bad argument");
  const hsv_sector_s* sec = out->sec;
  double2** d_q = nullptr;
  double* c = nullptr;
  HSV_TRY(basis_ptrs(q, m, sec, &d_q));
  HSV_TRY(dalloc(&c, 2 * std::max<int64_t>(m, 1)));
  std::vector<double> h(2 * m, 0.0);
  for (int64_t j = 0; j < m; ++j) h[2 * j] = coeff[j];
  HSV_TRY_CUDA(cudaMemcpyAsync(c, h.data(), 2 * m * sizeof(double), cudaMemcpyHostToDevice,
                               stream()));
  {
    ProfScope prof("krylov");
    k_kaxpy<<<grid_for(sec->dim, 256), 256, 0, stream()>>>(d_q, c, (int)m, out->d_amp, sec->dim, 0,
                                                          1.0);
    count_launch();
  }
  HSV_CHECK_LAUNCH();
  out->norm2_valid = out->arow_valid = out->smap_valid = false;
  out->dense_hint = false;
  dfree(d_q);
  dfree(c);
  return stream_sync();
}

}  // extern "C"
