// States: dense complex128 amplitudes over a sector in alpha-major internal
// order.  Support == exactly-nonzero amplitudes, which mirrors the reference
// SparseVector invariant (sparse.py:33-47 drops `values == 0.0`).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "hsv_common.cuh"

namespace hsv {

__device__ __forceinline__ bool is_nz(double2 v) { return v.x != 0.0 || v.y != 0.0; }

__global__ void k_fill_zero(double2* __restrict__ a, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) a[i] = make_double2(0.0, 0.0);
}

int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  int64_t cap = (int64_t)ctx().num_sms * 16;
  return (int)std::max<int64_t>(1, std::min(g, cap));
}

int state_fill_zero_async(hsv_state st) {
  HSV_TRY_CUDA(cudaMemsetAsync(st->d_amp, 0, st->sec->dim * sizeof(double2), stream()));
  HSV_TRY_CUDA(cudaMemsetAsync(st->d_norm2, 0, sizeof(double), stream()));
  HSV_TRY_CUDA(cudaMemsetAsync(st->d_arow, 0, st->sec->Na * sizeof(uint32_t), stream()));
  st->norm2_valid = true;
  st->arow_valid = true;
  st->smap_valid = false;
  st->dense_hint = false;
  return HSV_OK;
}

// One warp per alpha row: flag = any nonzero amplitude in the row.
__global__ void k_arow_flags(const double2* __restrict__ amp, int64_t Na, int64_t Nb,
                             uint32_t* __restrict__ flags) {
  const int64_t ra = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (ra >= Na) return;
  const double2* row = amp + ra * Nb;
  bool nz = false;
  for (int64_t j = lane; j < Nb && !nz; j += 32) {
    const double2 v = row[j];
    nz = v.x != 0.0 || v.y != 0.0;
  }
  nz = __any_sync(0xffffffffu, nz);
  if (lane == 0) flags[ra] = nz ? 1u : 0u;
}

int arow_flags_async(const double2* amp, int64_t Na, int64_t Nb, uint32_t* flags) {
  if (Na == 0) return HSV_OK;
  k_arow_flags<<<(unsigned)((Na * 32 + 255) / 256), 256, 0, stream()>>>(amp, Na, Nb, flags);
  count_launch();
  HSV_CHECK_LAUNCH();
  return HSV_OK;
}

int state_arow_async(hsv_state st) {
  if (st->arow_valid) return HSV_OK;
  HSV_TRY(arow_flags_async(st->d_amp, st->sec->Na, st->sec->Nb, st->d_arow));
  st->arow_valid = true;
  return HSV_OK;
}

// Per-block partial sums, fixed order; final pass in reduce_sum_f64.
template <int NV>
__device__ __forceinline__ void block_store(double (&v)[NV], double* __restrict__ out) {
  __shared__ double sh[NV][32];
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    double s = warp_sum(v[j]);
    if (l == 0) sh[j][w] = s;
  }
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      double s = (l < (int)(blockDim.x >> 5)) ? sh[j][l] : 0.0;
      s = warp_sum(s);
      if (l == 0) out[blockIdx.x * (int64_t)NV + j] = s;
    }
  }
}

__global__ void k_norm2(const double2* __restrict__ a, int64_t n, double* __restrict__ part) {
  double v[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double2 x = a[i];
    v[0] += x.x * x.x + x.y * x.y;
  }
  block_store<1>(v, part);
}

__global__ void k_dot(const double2* __restrict__ a, const double2* __restrict__ b, int64_t n,
                      double* __restrict__ part) {
  double v[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double2 x = a[i], y = b[i];
    v[0] += x.x * y.x + x.y * y.y;   // Re conj(x) y
    v[1] += x.x * y.y - x.y * y.x;   // Im conj(x) y
  }
  block_store<2>(v, part);
}

__global__ void k_count_nz(const double2* __restrict__ a, int64_t n,
                           unsigned long long* __restrict__ cnt) {
  int64_t c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    c += is_nz(a[i]) ? 1 : 0;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, (unsigned long long)c);
}

int state_norm2_async(hsv_state st) {
  const int64_t n = st->sec->dim;
  const int grid = grid_for(n, 256);
  double* part = nullptr;
  HSV_TRY(dalloc(&part, grid));
  k_norm2<<<grid, 256, 0, stream()>>>(st->d_amp, n, part);
  count_launch();
  HSV_CHECK_LAUNCH();
  HSV_TRY(reduce_sum_f64(part, grid, 1, 1, st->d_norm2));
  dfree(part);
  st->norm2_valid = true;
  return HSV_OK;
}

// scatter (ref positions -> internal rows)
__global__ void k_scatter_pos(const int64_t* __restrict__ pos, const double* __restrict__ re,
                              const double* __restrict__ im, int64_t n, int64_t dim,
                              const int64_t* __restrict__ iperm, double2* __restrict__ a,
                              int* __restrict__ bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t p = pos[i];
  if (p < 0 || p >= dim) { *bad = 1; return; }
  a[iperm[p]] = make_double2(re[i], im ? im[i] : 0.0);
}
// dense input: internal row j takes reference position perm[j] (coalesced stores)
__global__ void k_gather_dense(const double* __restrict__ re, const double* __restrict__ im,
                               int64_t dim, const int64_t* __restrict__ perm,
                               double2* __restrict__ a) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= dim) return;
  const int64_t p = perm[j];
  a[j] = make_double2(re[p], im ? im[p] : 0.0);
}
__global__ void k_scatter_idx(const int64_t* __restrict__ idx, const double2* __restrict__ v,
                              int64_t n, double2* __restrict__ a) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[idx[i]] = v[i];
}

// gather into reference order + support flags
__global__ void k_gather_ref(const double2* __restrict__ a, const int64_t* __restrict__ iperm,
                             int64_t n, double prune, double2* __restrict__ out,
                             int32_t* __restrict__ flag) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  double2 v = a[iperm[p]];
  bool keep = prune > 0.0 ? (sqrt(v.x * v.x + v.y * v.y) >= prune) : is_nz(v);
  out[p] = v;
  flag[p] = keep ? 1 : 0;
}
__global__ void k_compact(const double2* __restrict__ v, const int32_t* __restrict__ flag,
                          const int64_t* __restrict__ off, int64_t n, int64_t* __restrict__ pos,
                          double* __restrict__ re, double* __restrict__ im) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n || !flag[p]) return;
  int64_t o = off[p];
  pos[o] = p;
  re[o] = v[p].x;
  im[o] = v[p].y;
}

__global__ void k_axpy(double ar, double ai, const double2* __restrict__ x,
                       double2* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double2 a = x[i], b = y[i];
    double2 r;
    if (ai == 0.0) {   // real scale: a*x + y with separate roundings (sparse.py:226-228)
      r.x = __dadd_rn(__dmul_rn(ar, a.x), b.x);
      r.y = __dadd_rn(__dmul_rn(ar, a.y), b.y);
    } else {
      r.x = __dadd_rn(__dsub_rn(__dmul_rn(ar, a.x), __dmul_rn(ai, a.y)), b.x);
      r.y = __dadd_rn(__dadd_rn(__dmul_rn(ar, a.y), __dmul_rn(ai, a.x)), b.y);
    }
    y[i] = r;
  }
}
__global__ void k_scale(double ar, double ai, double2* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double2 a = y[i];
    if (ai == 0.0) y[i] = make_double2(__dmul_rn(ar, a.x), __dmul_rn(ar, a.y));
    else y[i] = make_double2(__dsub_rn(__dmul_rn(ar, a.x), __dmul_rn(ai, a.y)),
                             __dadd_rn(__dmul_rn(ar, a.y), __dmul_rn(ai, a.x)));
  }
}
__global__ void k_gather_i64(const int64_t* __restrict__ tab, const int64_t* __restrict__ idx,
                             int64_t n, int64_t* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = idx[i] < 0 ? -1 : tab[idx[i]];
}

__global__ void k_gather_amp(const double2* __restrict__ a, const int64_t* __restrict__ idx,
                             int64_t n, double2* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[idx[i]];
}

int upload_amps(const double* re, const double* im, int64_t n, double2** d_out) {
  std::vector<double2> h(n);
  for (int64_t i = 0; i < n; ++i) h[i] = make_double2(re[i], im ? im[i] : 0.0);
  HSV_TRY(dalloc(d_out, n));
  HSV_TRY_CUDA(cudaMemcpyAsync(*d_out, h.data(), n * sizeof(double2), cudaMemcpyHostToDevice,
                               stream()));
  // the host staging buffer must outlive the async copy
  return stream_sync();
}

// <a|b> into d_r[0..1] (re, im), stream-ordered
// <a|b> -> d_r[0..1] and <b|b> -> b's cached norm in one pass over both
// (the adjoint evaluation needs both; each sum is the one the separate
// kernels form: same grid, same per-thread order, same block reduction)
__global__ void k_dot_norm2(const double2* __restrict__ a, const double2* __restrict__ b,
                            int64_t n, double* __restrict__ part) {
  double v[3] = {0.0, 0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double2 x = a[i], y = b[i];
    v[0] += x.x * y.x + x.y * y.y;
    v[1] += x.x * y.y - x.y * y.x;
    v[2] += y.x * y.x + y.y * y.y;
  }
  block_store<3>(v, part);
}

int state_dot_norm2_async(hsv_state a, hsv_state b, double* d_r) {
  const int64_t n = a->sec->dim;
  const int grid = grid_for(n, 256);
  double* part = nullptr;
  HSV_TRY(dalloc(&part, 3 * (int64_t)grid));
  k_dot_norm2<<<grid, 256, 0, stream()>>>(a->d_amp, b->d_amp, n, part);
  count_launch();
  HSV_CHECK_LAUNCH();
  HSV_TRY(reduce_sum_f64(part, grid, 3, 2, d_r));
  HSV_TRY(reduce_sum_f64(part + 2, grid, 3, 1, b->d_norm2));
  dfree(part);
  b->norm2_valid = true;
  return HSV_OK;
}

int state_dot_async(hsv_state a, hsv_state b, double* d_r) {
  const int64_t n = a->sec->dim;
  const int grid = grid_for(n, 256);
  double* part = nullptr;
  HSV_TRY(dalloc(&part, 2 * (int64_t)grid));
  k_dot<<<grid, 256, 0, stream()>>>(a->d_amp, b->d_amp, n, part);
  count_launch();
  HSV_CHECK_LAUNCH();
  HSV_TRY(reduce_sum_f64(part, grid, 2, 2, d_r));
  dfree(part);
  return HSV_OK;
}
}  // namespace hsv

using namespace hsv;

extern "C" {

int hsv_state_create(hsv_sector s, hsv_state* out) {
  HSV_TRY(ensure_init());
  HSV_REQUIRE(s && out, HSV_ERR_INVALID, "null argument");
  auto* st = new hsv_state_s();
  st->sec = s;
  int rc = dalloc(&st->d_amp, s->dim);
  if (!rc) rc = dalloc(&st->d_norm2, 1);
  if (!rc) rc = dalloc(&st->d_arow, std::max<int64_t>(s->Na, 1));
  if (!rc) rc = state_fill_zero_async(st);
  if (!rc) rc = stream_sync();
  if (rc) { hsv_state_destroy(st); return rc; }
  *out = st;
  return HSV_OK;
}

int hsv_state_destroy(hsv_state st) {
  if (!st) return HSV_OK;
  dfree(st->d_amp);
  dfree(st->d_norm2);
  dfree(st->d_arow);
  dfree(st->d_pend_err);
  dfree(st->d_pend_val);
  dfree(st->d_smap);
  delete st;
  return HSV_OK;
}

int hsv_state_copy(hsv_state dst, hsv_state src) {
  HSV_REQUIRE(dst && src && dst->sec == src->sec, HSV_ERR_INVALID,
              "dimension mismatch: states belong to different sectors");
  if (dst == src) return HSV_OK;
  HSV_TRY_CUDA(cudaMemcpyAsync(dst->d_amp, src->d_amp, src->sec->dim * sizeof(double2),
                               cudaMemcpyDeviceToDevice, stream()));
  HSV_TRY_CUDA(cudaMemcpyAsync(dst->d_norm2, src->d_norm2, sizeof(double),
                               cudaMemcpyDeviceToDevice, stream()));
  HSV_TRY_CUDA(cudaMemcpyAsync(dst->d_arow, src->d_arow, src->sec->Na * sizeof(uint32_t),
                               cudaMemcpyDeviceToDevice, stream()));
  dst->norm2_valid = src->norm2_valid;
  dst->arow_valid = src->arow_valid;
  dst->smap_valid = false;
  dst->dense_hint = src->dense_hint;
  return stream_sync();
}

int hsv_state_zero(hsv_state st) {
  HSV_REQUIRE(st, HSV_ERR_INVALID, "null state");
  HSV_TRY(state_fill_zero_async(st));
  return stream_sync();
}

int hsv_state_set_basis(hsv_state st, uint64_t key, double re, double im) {
  HSV_REQUIRE(st, HSV_ERR_INVALID, "null state");
  hsv_sector s = st->sec;
  uint32_t sa = s->compress_a(key), sb = s->compress_b(key);
  bool ok = (s->n_qubits >= 64 || (key >> s->n_qubits) == 0) && s->Ra[sa] != ~0u &&
            s->Rb[sb] != ~0u;
  HSV_REQUIRE(ok, HSV_ERR_SECTOR, "configuration %#llx is outside the basis sector",
              (unsigned long long)key);
  int64_t idx = (int64_t)s->Ra[sa] * s->Nb + s->Rb[sb];
  HSV_TRY(state_fill_zero_async(st));
  static thread_local double2 v;
  static thread_local double n2;
  v = make_double2(re, im);
  n2 = re * re + im * im;
  HSV_TRY_CUDA(cudaMemcpyAsync(st->d_amp + idx, &v, sizeof(double2), cudaMemcpyHostToDevice,
                               stream()));
  HSV_TRY_CUDA(cudaMemcpyAsync(st->d_norm2, &n2, sizeof(double), cudaMemcpyHostToDevice,
                               stream()));
  st->arow_valid = false;
  st->smap_valid = false;
  st->dense_hint = false;
  return stream_sync();
}

int hsv_state_set_sparse(hsv_state st, const int64_t* pos, const double* re, const double* im,
                         int64_t n) {
  HSV_REQUIRE(st && (n == 0 || (pos && re)), HSV_ERR_INVALID, "null argument");
  // Host buffers go straight to the device (pinned buffers copy asynchronously);
  // positions are range-checked by the scatter kernel.
  HSV_TRY(state_fill_zero_async(st));
  int h_bad = 0;
  if (n > 0) {
    double *d_re = nullptr, *d_im = nullptr;
    int64_t* d_p = nullptr;
    int* d_bad = nullptr;
    HSV_TRY(dalloc(&d_p, n));
    HSV_TRY(dalloc(&d_re, n));
    if (im) HSV_TRY(dalloc(&d_im, n));
    HSV_TRY(dalloc(&d_bad, 1));
    HSV_TRY_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int), stream()));
    HSV_TRY_CUDA(cudaMemcpyAsync(d_p, pos, n * 8, cudaMemcpyHostToDevice, stream()));
    HSV_TRY_CUDA(cudaMemcpyAsync(d_re, re, n * 8, cudaMemcpyHostToDevice, stream()));
    if (im) HSV_TRY_CUDA(cudaMemcpyAsync(d_im, im, n * 8, cudaMemcpyHostToDevice, stream()));
    k_scatter_pos<<<(unsigned)((n + 255) / 256), 256, 0, stream()>>>(
        d_p, d_re, d_im, n, st->sec->dim, st->sec->d_iperm, st->d_amp, d_bad);
    count_launch();
    HSV_CHECK_LAUNCH();
    HSV_TRY_CUDA(cudaMemcpyAsync(&h_bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, stream()));
    dfree(d_re);
    dfree(d_im);
    dfree(d_p);
    dfree(d_bad);
  }
  st->arow_valid = false;
  st->smap_valid = false;
  // more than dim/8 entries is always past the push path's budget: skip its probe
  st->dense_hint = n > st->sec->dim / 8;
  HSV_TRY(state_norm2_async(st));
  HSV_TRY(stream_sync());
  HSV_REQUIRE(!h_bad, HSV_ERR_INVALID, "position out of range for dimension %lld",
              (long long)st->sec->dim);
  return HSV_OK;
}

int hsv_state_set_dense(hsv_state st, const double* re, const double* im) {
  HSV_REQUIRE(st && re, HSV_ERR_INVALID, "null argument");
  const int64_t dim = st->sec->dim;
  // every amplitude in reference position order: no positions to move or check,
  // no zero fill (every row is written)
  double *d_re = nullptr, *d_im = nullptr;
  HSV_TRY(dalloc(&d_re, dim));
  if (im) HSV_TRY(dalloc(&d_im, dim));
  HSV_TRY_CUDA(cudaMemcpyAsync(d_re, re, dim * 8, cudaMemcpyHostToDevice, stream()));
  if (im) HSV_TRY_CUDA(cudaMemcpyAsync(d_im, im, dim * 8, cudaMemcpyHostToDevice, stream()));
  k_gather_dense<<<(unsigned)((dim + 255) / 256), 256, 0, stream()>>>(d_re, d_im, dim,
                                                                       st->sec->d_perm, st->d_amp);
  count_launch();
  HSV_CHECK_LAUNCH();
  dfree(d_re);
  dfree(d_im);
  st->arow_valid = false;
  st->smap_valid = false;
  st->dense_hint = true;
  HSV_TRY(state_norm2_async(st));
  HSV_TRY(stream_sync());   // host buffers may be reused on return
  return HSV_OK;
}

int hsv_state_set_keys(hsv_state st, const uint64_t* keys, const double* re, const double* im,
                       int64_t n) {
  HSV_REQUIRE(st && (n == 0 || (keys && re)), HSV_ERR_INVALID, "null argument");
  hsv_sector s = st->sec;
  std::vector<int64_t> idx(n);
  for (int64_t i = 0; i < n; ++i) {
    uint64_t k = keys[i];
    uint32_t sa = s->compress_a(k), sb = s->compress_b(k);
    bool ok = (s->n_qubits >= 64 || (k >> s->n_qubits) == 0) && s->Ra[sa] != ~0u &&
              s->Rb[sb] != ~0u;
    HSV_REQUIRE(ok, HSV_ERR_SECTOR, "configuration %#llx is outside the ci sector",
                (unsigned long long)k);
    idx[i] = (int64_t)s->Ra[sa] * s->Nb + s->Rb[sb];
  }
  HSV_TRY(state_fill_zero_async(st));
  if (n > 0) {
    double2* d_v = nullptr;
    int64_t* d_i = nullptr;
    HSV_TRY(upload_amps(re, im, n, &d_v));
    HSV_TRY(dalloc(&d_i, n));
    HSV_TRY_CUDA(cudaMemcpyAsync(d_i, idx.data(), n * 8, cudaMemcpyHostToDevice, stream()));
    k_scatter_idx<<<(unsigned)((n + 255) / 256), 256, 0, stream()>>>(d_i, d_v, n, st->d_amp);
    count_launch();
    HSV_CHECK_LAUNCH();
    HSV_TRY(stream_sync());
    dfree(d_v);
    dfree(d_i);
  }
  st->arow_valid = false;
  st->smap_valid = false;
  st->dense_hint = n > st->sec->dim / 8;
  HSV_TRY(state_norm2_async(st));
  return stream_sync();
}

int hsv_state_nnz(hsv_state st, int64_t* nnz) {
  HSV_REQUIRE(st && nnz, HSV_ERR_INVALID, "null argument");
  unsigned long long* d_c = nullptr;
  HSV_TRY(dalloc(&d_c, 1));
  HSV_TRY_CUDA(cudaMemsetAsync(d_c, 0, 8, stream()));
  int grid = grid_for(st->sec->dim, 256);
  k_count_nz<<<grid, 256, 0, stream()>>>(st->d_amp, st->sec->dim, d_c);
  count_launch();
  HSV_CHECK_LAUNCH();
  unsigned long long h = 0;
  HSV_TRY_CUDA(cudaMemcpyAsync(&h, d_c, 8, cudaMemcpyDeviceToHost, stream()));
  HSV_TRY(stream_sync());
  dfree(d_c);
  *nnz = (int64_t)h;
  return HSV_OK;
}

int hsv_state_get_sparse(hsv_state st, double prune, int64_t* pos, double* re, double* im,
                         int64_t cap, int64_t* n_out) {
  HSV_REQUIRE(st && n_out, HSV_ERR_INVALID, "null argument");
  const int64_t n = st->sec->dim;
  double2* d_ref = nullptr;
  int32_t* d_flag = nullptr;
  int64_t* d_off = nullptr;
  HSV_TRY(dalloc(&d_ref, n));
  HSV_TRY(dalloc(&d_flag, n));
  HSV_TRY(dalloc(&d_off, n));
  const unsigned g = (unsigned)((n + 255) / 256);
  k_gather_ref<<<g, 256, 0, stream()>>>(st->d_amp, st->sec->d_iperm, n, prune, d_ref, d_flag);
  count_launch();
  HSV_CHECK_LAUNCH();
  size_t tmp_bytes = 0;
  HSV_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_flag, d_off, n, stream()));
  void* d_tmp = nullptr;
  HSV_TRY(dalloc(reinterpret_cast<char**>(&d_tmp), tmp_bytes));
  HSV_TRY_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_flag, d_off, n, stream()));
  count_launch();
  int64_t last_off = 0;
  int32_t last_flag = 0;
  if (n > 0) {
    HSV_TRY_CUDA(cudaMemcpyAsync(&last_off, d_off + n - 1, 8, cudaMemcpyDeviceToHost, stream()));
    HSV_TRY_CUDA(cudaMemcpyAsync(&last_flag, d_flag + n - 1, 4, cudaMemcpyDeviceToHost, stream()));
  }
  HSV_TRY(stream_sync());
  const int64_t cnt = last_off + last_flag;
  *n_out = cnt;
  if (pos && cnt > 0) {
    HSV_REQUIRE(cap >= cnt, HSV_ERR_INVALID, "output capacity %lld < support size %lld",
                (long long)cap, (long long)cnt);
    int64_t* d_pos = nullptr;
    double *d_re = nullptr, *d_im = nullptr;
    HSV_TRY(dalloc(&d_pos, cnt));
    HSV_TRY(dalloc(&d_re, cnt));
    HSV_TRY(dalloc(&d_im, cnt));
    k_compact<<<g, 256, 0, stream()>>>(d_ref, d_flag, d_off, n, d_pos, d_re, d_im);
    count_launch();
    HSV_CHECK_LAUNCH();
    HSV_TRY_CUDA(cudaMemcpyAsync(pos, d_pos, cnt * 8, cudaMemcpyDeviceToHost, stream()));
    if (re) HSV_TRY_CUDA(cudaMemcpyAsync(re, d_re, cnt * 8, cudaMemcpyDeviceToHost, stream()));
    if (im) HSV_TRY_CUDA(cudaMemcpyAsync(im, d_im, cnt * 8, cudaMemcpyDeviceToHost, stream()));
    HSV_TRY(stream_sync());
    dfree(d_pos); dfree(d_re); dfree(d_im);
  }
  dfree(d_ref); dfree(d_flag); dfree(d_off); dfree(reinterpret_cast<char*>(d_tmp));
  return HSV_OK;
}

int hsv_state_get_positions(hsv_state st, const int64_t* pos, int64_t n, double* re, double* im) {
  HSV_REQUIRE(st && (n == 0 || (pos && re)), HSV_ERR_INVALID, "null argument");
  if (n == 0) return HSV_OK;
  for (int64_t i = 0; i < n; ++i)
    HSV_REQUIRE(pos[i] >= 0 && pos[i] < st->sec->dim, HSV_ERR_INVALID,
                "position %lld out of range", (long long)pos[i]);
  int64_t *d_p = nullptr, *d_i = nullptr;
  double2* d_v = nullptr;
  HSV_TRY(dalloc(&d_p, n));
  HSV_TRY(dalloc(&d_i, n));
  HSV_TRY(dalloc(&d_v, n));
  HSV_TRY_CUDA(cudaMemcpyAsync(d_p, pos, n * 8, cudaMemcpyHostToDevice, stream()));
  const unsigned g = (unsigned)((n + 255) / 256);
  k_gather_i64<<<g, 256, 0, stream()>>>(st->sec->d_iperm, d_p, n, d_i);
  k_gather_amp<<<g, 256, 0, stream()>>>(st->d_amp, d_i, n, d_v);
  count_launch(2);
  HSV_CHECK_LAUNCH();
  std::vector<double2> h(n);
  HSV_TRY_CUDA(cudaMemcpyAsync(h.data(), d_v, n * sizeof(double2), cudaMemcpyDeviceToHost, stream()));
  HSV_TRY(stream_sync());
  dfree(d_p); dfree(d_i); dfree(d_v);
  for (int64_t i = 0; i < n; ++i) {
    re[i] = h[i].x;
    if (im) im[i] = h[i].y;
  }
  return HSV_OK;
}


int hsv_state_dot(hsv_state a, hsv_state b, double* re, double* im) {
  HSV_REQUIRE(a && b, HSV_ERR_INVALID, "null state");
  HSV_REQUIRE(a->sec == b->sec, HSV_ERR_INVALID, "dimension mismatch in dot");
  double* d_r = nullptr;
  HSV_TRY(dalloc(&d_r, 2));
  HSV_TRY(state_dot_async(a, b, d_r));
  double h[2];
  HSV_TRY_CUDA(cudaMemcpyAsync(h, d_r, 16, cudaMemcpyDeviceToHost, stream()));
  HSV_TRY(stream_sync());
  dfree(d_r);
  if (re) *re = h[0];
  if (im) *im = h[1];
  return HSV_OK;
}

int hsv_state_norm(hsv_state st, double* norm) {
  HSV_REQUIRE(st && norm, HSV_ERR_INVALID, "null argument");
  HSV_TRY(state_norm2_async(st));
  double h = 0;
  HSV_TRY_CUDA(cudaMemcpyAsync(&h, st->d_norm2, 8, cudaMemcpyDeviceToHost, stream()));
  HSV_TRY(stream_sync());
  *norm = std::sqrt(h);
  return HSV_OK;
}

int hsv_state_axpy(double ar, double ai, hsv_state x, hsv_state y) {
  HSV_REQUIRE(x && y && x->sec == y->sec, HSV_ERR_INVALID, "dimension mismatch in axpy");
  const int64_t n = x->sec->dim;
  k_axpy<<<grid_for(n, 256), 256, 0, stream()>>>(ar, ai, x->d_amp, y->d_amp, n);
  count_launch();
  HSV_CHECK_LAUNCH();
  y->norm2_valid = false;
  y->arow_valid = false;
  y->smap_valid = false;
  y->dense_hint = false;
  return stream_sync();
}

int hsv_state_scale(hsv_state st, double ar, double ai) {
  HSV_REQUIRE(st, HSV_ERR_INVALID, "null state");
  const int64_t n = st->sec->dim;
  k_scale<<<grid_for(n, 256), 256, 0, stream()>>>(ar, ai, st->d_amp, n);
  count_launch();
  HSV_CHECK_LAUNCH();
  st->norm2_valid = false;
  st->arow_valid = false;
  st->smap_valid = false;
  st->dense_hint = false;
  return stream_sync();
}

int hsv_state_device_ptr(hsv_state st, void** ptr, int64_t* n) {
  HSV_REQUIRE(st, HSV_ERR_INVALID, "null state");
  if (ptr) *ptr = st->d_amp;
  if (n) *n = st->sec->dim;
  st->norm2_valid = false;   // caller may write through the pointer
  st->arow_valid = false;
  st->smap_valid = false;
  st->dense_hint = false;
  return HSV_OK;
}

int hsv_sector_positions(hsv_sector s, const uint64_t* keys, int64_t n, int64_t* pos) {
  HSV_REQUIRE(s && (n == 0 || (keys && pos)), HSV_ERR_INVALID, "null argument");
  if (n == 0) return HSV_OK;
  std::vector<int64_t> internal(n);
  for (int64_t i = 0; i < n; ++i) {
    uint64_t k = keys[i];
    bool ok = s->n_qubits >= 64 || (k >> s->n_qubits) == 0;
    uint32_t sa = s->compress_a(k), sb = s->compress_b(k);
    ok = ok && s->Ra[sa] != ~0u && s->Rb[sb] != ~0u;
    internal[i] = ok ? (int64_t)s->Ra[sa] * s->Nb + s->Rb[sb] : -1;
  }
  int64_t *d_i = nullptr, *d_o = nullptr;
  HSV_TRY(dalloc(&d_i, n));
  HSV_TRY(dalloc(&d_o, n));
  HSV_TRY_CUDA(cudaMemcpyAsync(d_i, internal.data(), n * 8, cudaMemcpyHostToDevice, stream()));
  k_gather_i64<<<(unsigned)((n + 255) / 256), 256, 0, stream()>>>(s->d_perm, d_i, n, d_o);
  count_launch();
  HSV_CHECK_LAUNCH();
  HSV_TRY_CUDA(cudaMemcpyAsync(pos, d_o, n * 8, cudaMemcpyDeviceToHost, stream()));
  HSV_TRY(stream_sync());
  dfree(d_i);
  dfree(d_o);
  return HSV_OK;
}

int hsv_sector_keys(hsv_sector s, const int64_t* pos, int64_t n, uint64_t* keys) {
  HSV_REQUIRE(s && (n == 0 || (keys && pos)), HSV_ERR_INVALID, "null argument");
  if (n == 0) return HSV_OK;
  for (int64_t i = 0; i < n; ++i)
    HSV_REQUIRE(pos[i] >= 0 && pos[i] < s->dim, HSV_ERR_INVALID, "position %lld out of range",
                (long long)pos[i]);
  std::vector<int64_t> internal(n);
  int64_t *d_i = nullptr, *d_o = nullptr;
  HSV_TRY(dalloc(&d_i, n));
  HSV_TRY(dalloc(&d_o, n));
  HSV_TRY_CUDA(cudaMemcpyAsync(d_i, pos, n * 8, cudaMemcpyHostToDevice, stream()));
  k_gather_i64<<<(unsigned)((n + 255) / 256), 256, 0, stream()>>>(s->d_iperm, d_i, n, d_o);
  count_launch();
  HSV_CHECK_LAUNCH();
  HSV_TRY_CUDA(cudaMemcpyAsync(internal.data(), d_o, n * 8, cudaMemcpyDeviceToHost, stream()));
  HSV_TRY(stream_sync());
  dfree(d_i);
  dfree(d_o);
  for (int64_t i = 0; i < n; ++i) {
    int64_t ra = internal[i] / s->Nb, rb = internal[i] % s->Nb;
    keys[i] = s->expand(s->Sa[ra], s->Sb[rb]);
  }
  return HSV_OK;
}

}  // extern "C"
