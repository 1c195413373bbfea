// K4: batched pool gradients g_k = 2 Re <H psi | T_k psi> for every pool
// operator in one pass (replaces the per-operator Python loop of
// SvAdaptEngine.screen, adapt.py:212-214, and pool_gradients, svengine.py:253-257).
//
// Row formulation (owner computes): for an owned row b,
//   (T_k psi)_b = +psi_{b^f}  if b is in target pattern (V set, O clear),
//               = -psi_{b^f}  if b is in source pattern (O set, V clear),
// so only w_b = (H psi)_b of owned rows is needed and psi (replicated) is
// gathered at the partner.  Each CTA owns a contiguous, equal share of rows,
// stages them in shared memory in chunks, and each warp owns a fixed subset
// of operators; per-operator sums are reduced in a fixed order.
#include <algorithm>
#include <cmath>

#include "hsv_common.cuh"
#include "hsv_kernels.cuh"

namespace hsv {

constexpr int kScreenRows = 1024;
constexpr int kScreenBlock = 256;

struct ScreenArgs {
  const uint32_t* Sa;
  const uint32_t* Sb;
  const uint32_t* Ra;
  const uint32_t* Rb;
  const int4* ops;     // {oa, va, ob, vb}
  int n_ops;
  const double2* psi;
  const double2* w;
  int64_t Nb;
  int64_t row_lo, row_hi;
  double* part;        // [gridDim.x][n_ops]
};

__global__ void __launch_bounds__(kScreenBlock) k_screen(const ScreenArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  double2* s_w = reinterpret_cast<double2*>(smem);
  uint32_t* s_sb = reinterpret_cast<uint32_t*>(s_w + kScreenRows);
  double* acc = reinterpret_cast<double*>(s_sb + kScreenRows);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kScreenBlock / 32;
  const int64_t nrows = a.row_hi - a.row_lo;
  const int64_t r0 = a.row_lo + nrows * blockIdx.x / gridDim.x;
  const int64_t r1 = a.row_lo + nrows * (blockIdx.x + 1) / gridDim.x;
  for (int q = threadIdx.x; q < a.n_ops; q += kScreenBlock) acc[q] = 0.0;
  for (int64_t c0 = r0; c0 < r1; c0 += kScreenRows) {
    const int n = (int)imin64(kScreenRows, r1 - c0);
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += kScreenBlock) {
      const int64_t idx = c0 + i;
      const int64_t rb = idx % a.Nb;
      s_sb[i] = __ldg(a.Sb + rb);
      s_w[i] = a.w[idx];
    }
    __syncthreads();
    const int64_t ra_first = c0 / a.Nb;
    for (int op = warp; op < a.n_ops; op += nw) {
      const int4 O = __ldg(a.ops + op);
      const uint32_t oa = (uint32_t)O.x, va = (uint32_t)O.y, ob = (uint32_t)O.z, vb = (uint32_t)O.w;
      const uint32_t fa = oa | va, fb = ob | vb;
      double g = 0.0;
      // alpha-uniform segments of the chunk
      int lo = 0;
      for (int64_t ra = ra_first; lo < n; ++ra) {
        const int hi = (int)imin64(n, (ra + 1) * a.Nb - c0);
        const uint32_t sa = __ldg(a.Sa + ra);
        const bool as = (sa & oa) == oa && (sa & va) == 0;
        const bool at = (sa & va) == va && (sa & oa) == 0;
        if (as || at) {
          const double2* __restrict__ prow = a.psi + (int64_t)__ldg(a.Ra + (sa ^ fa)) * a.Nb;
          for (int r = lo + lane; r < hi; r += 32) {
            const uint32_t sb = s_sb[r];
            const bool bs = (sb & ob) == ob && (sb & vb) == 0;
            const bool bt = (sb & vb) == vb && (sb & ob) == 0;
            const bool tgt = at && bt, src = as && bs;
            if (tgt || src) {
              const double2 p = prow[__ldg(a.Rb + (sb ^ fb))];
              const double2 wv = s_w[r];
              const double x = wv.x * p.x + wv.y * p.y;   // Re conj(w_b) psi_{b^f}
              g += tgt ? x : -x;
            }
          }
        }
        lo = hi;
      }
      g = warp_sum(g);
      if (lane == 0) acc[op] += g;
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < a.n_ops; q += kScreenBlock)
    a.part[(int64_t)blockIdx.x * a.n_ops + q] = 2.0 * acc[q];
}

int launch_screen(const hsv_op_s* op, const double2* psi, const double2* w, const int4* d_ops,
                  int n_ops, int64_t row_lo, int64_t row_hi, double* d_grads) {
  const hsv_sector_s* s = op->sec;
  if (n_ops <= 0) return HSV_OK;
  const size_t smem = kScreenRows * (sizeof(double2) + sizeof(uint32_t)) + n_ops * sizeof(double);
  HSV_REQUIRE(smem <= 227 * 1024, HSV_ERR_UNSUPPORTED, "operator pool too large (%d)", n_ops);
  HSV_TRY_CUDA(cudaFuncSetAttribute(k_screen, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  HSV_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_screen, kScreenBlock, smem));
  occ = std::max(occ, 1);
  const int64_t nrows = row_hi - row_lo;
  int64_t grid = (int64_t)ctx().num_sms * occ;
  grid = std::max<int64_t>(1, std::min(grid, (nrows + 255) / 256));
  double* part = nullptr;
  HSV_TRY(dalloc(&part, grid * n_ops));
  ScreenArgs a{};
  a.Sa = s->d_Sa; a.Sb = s->d_Sb; a.Ra = s->d_Ra; a.Rb = s->d_Rb;
  a.ops = d_ops; a.n_ops = n_ops; a.psi = psi; a.w = w; a.Nb = s->Nb;
  a.row_lo = row_lo; a.row_hi = row_hi; a.part = part;
  if (nrows > 0) {
    {
      ProfScope prof("screen");
      k_screen<<<(unsigned)grid, kScreenBlock, smem, stream()>>>(a);
    }
    count_launch();
    HSV_CHECK_LAUNCH();
    HSV_TRY(reduce_sum_f64(part, grid, n_ops, n_ops, d_grads));
  } else {
    HSV_TRY_CUDA(cudaMemsetAsync(d_grads, 0, n_ops * sizeof(double), stream()));
  }
  dfree(part);
  return HSV_OK;
}

static int upload_ops(const hsv_sector_s* s, const uint64_t* occ, const uint64_t* virt, int64_t n,
                      int4** d_ops) {
  std::vector<int4> h(n);
  for (int64_t i = 0; i < n; ++i) {
    HSV_REQUIRE((occ[i] & virt[i]) == 0 && occ[i] && virt[i], HSV_ERR_INVALID,
                "excitation indices must be distinct");
    OpMasks m = compress_op(s, occ[i], virt[i]);
    h[i] = make_int4((int)m.oa, (int)m.va, (int)m.ob, (int)m.vb);
  }
  HSV_TRY(dalloc(d_ops, n));
  if (n) HSV_TRY_CUDA(cudaMemcpyAsync(*d_ops, h.data(), n * sizeof(int4), cudaMemcpyHostToDevice, stream()));
  return stream_sync();
}

}  // namespace hsv

using namespace hsv;

extern "C" {

static int energy_screen_dev(hsv_op op, hsv_state psi, const int4* d_ops, int64_t n_ops,
                             int64_t a_lo, int64_t a_hi, double* d_out) {
  const hsv_sector_s* s = op->sec;
  double2* w = nullptr;
  HSV_TRY(dalloc(&w, s->dim));
  const int nw = apply_warps(op);
  double* epart = nullptr;
  HSV_TRY(dalloc(&epart, 2 * (int64_t)nw));
  HSV_TRY_CUDA(cudaMemsetAsync(epart, 0, 2 * sizeof(double) * nw, stream()));
  int64_t used = 0;
  HSV_TRY(launch_apply(op, psi->d_amp, w, epart, a_lo, a_hi, 0.0, 0, &used));
  HSV_TRY(reduce_sum_f64(epart, used, 2, 2, d_out));
  HSV_TRY(launch_screen(op, psi->d_amp, w, d_ops, (int)n_ops, a_lo * s->Nb, a_hi * s->Nb, d_out + 2));
  dfree(w);
  dfree(epart);
  return HSV_OK;
}

static int check_es_args(hsv_op op, hsv_state psi, int64_t a_lo, int64_t a_hi) {
  HSV_REQUIRE(op && psi, HSV_ERR_INVALID, "null argument");
  HSV_REQUIRE(psi->sec == op->sec, HSV_ERR_INVALID, "dimension mismatch");
  HSV_REQUIRE(0 <= a_lo && a_lo <= a_hi && a_hi <= op->sec->Na, HSV_ERR_INVALID,
              "bad alpha-row range");
  return HSV_OK;
}

int hsv_energy_screen_partial_async(hsv_op op, hsv_state psi, const uint64_t* occ,
                                    const uint64_t* virt, int64_t n_ops, int64_t a_lo,
                                    int64_t a_hi, double* d_out) {
  HSV_TRY(check_es_args(op, psi, a_lo, a_hi));
  HSV_REQUIRE(d_out && (n_ops == 0 || (occ && virt)), HSV_ERR_INVALID, "null argument");
  int4* d_ops = nullptr;
  HSV_TRY(upload_ops(op->sec, occ, virt, n_ops, &d_ops));
  HSV_TRY(energy_screen_dev(op, psi, d_ops, n_ops, a_lo, a_hi, d_out));
  dfree(d_ops);
  return HSV_OK;
}

int hsv_energy_screen_pool_async(hsv_op op, hsv_state psi, hsv_pool pool, int64_t a_lo,
                                 int64_t a_hi, double* d_out) {
  HSV_TRY(check_es_args(op, psi, a_lo, a_hi));
  HSV_REQUIRE(pool && d_out && pool->sec == op->sec, HSV_ERR_INVALID, "bad pool argument");
  return energy_screen_dev(op, psi, pool->d, pool->n, a_lo, a_hi, d_out);
}

int hsv_energy_screen_pool(hsv_op op, hsv_state psi, hsv_pool pool, double* energy, double* grads) {
  HSV_REQUIRE(op && pool && (pool->n == 0 || grads), HSV_ERR_INVALID, "null argument");
  const int64_t n_ops = pool->n;
  double* d_out = nullptr;
  HSV_TRY(dalloc(&d_out, 2 + n_ops));
  HSV_TRY(hsv_energy_screen_pool_async(op, psi, pool, 0, op->sec->Na, d_out));
  static thread_local std::vector<double> h;
  h.resize(2 + n_ops);
  HSV_TRY_CUDA(cudaMemcpyAsync(h.data(), d_out, (2 + n_ops) * sizeof(double), cudaMemcpyDeviceToHost, stream()));
  HSV_TRY(stream_sync());
  dfree(d_out);
  if (energy) *energy = h[0];
  for (int64_t i = 0; i < n_ops; ++i) grads[i] = h[2 + i];
  return HSV_OK;
}

int hsv_energy_screen(hsv_op op, hsv_state psi, const uint64_t* occ, const uint64_t* virt,
                      int64_t n_ops, double* energy, double* grads) {
  HSV_REQUIRE(op && psi && (n_ops == 0 || (occ && virt && grads)), HSV_ERR_INVALID, "null argument");
  double* d_out = nullptr;
  HSV_TRY(dalloc(&d_out, 2 + n_ops));
  HSV_TRY(hsv_energy_screen_partial_async(op, psi, occ, virt, n_ops, 0, op->sec->Na, d_out));
  std::vector<double> h(2 + n_ops);
  HSV_TRY_CUDA(cudaMemcpyAsync(h.data(), d_out, (2 + n_ops) * sizeof(double), cudaMemcpyDeviceToHost, stream()));
  HSV_TRY(stream_sync());
  dfree(d_out);
  if (energy) *energy = h[0];
  for (int64_t i = 0; i < n_ops; ++i) grads[i] = h[2 + i];
  return HSV_OK;
}

}  // extern "C"
