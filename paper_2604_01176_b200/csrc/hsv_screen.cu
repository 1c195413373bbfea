// K4: batched pool gradients g_k = 2 Re <H psi | T_k psi> for every pool
// operator in one pass (replaces the per-operator Python loop of
// SvAdaptEngine.screen, adapt.py:212-214, and pool_gradients, svengine.py:253-257).
//
// Row formulation (owner computes): for an owned row b,
//   (T_k psi)_b = +psi_{b^f}  if b is in target pattern (V set, O clear),
//               = -psi_{b^f}  if b is in source pattern (O set, V clear),
// so only w = H psi on owned rows is needed and psi (replicated) is gathered
// at the partner b^f.
//
// A CTA owns one alpha row and a slice of the operators; a warp owns one
// operator at a time.  If the alpha half of the row is in source (target)
// pattern, the matching beta strings are exactly the operator's precomputed
// beta source list (its partners), so the warp walks that list -- no per-row
// tests, work proportional to the matches.  Operators are processed in
// alpha-part order so the warps of a CTA share partner rows in L1.  Each
// (alpha row, operator) partial is written once and reduced over alpha rows
// in a fixed order: bitwise deterministic.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <map>

#include "hsv_common.cuh"
#include "hsv_kernels.cuh"

namespace hsv {

constexpr int kScreenBlock = 256;
constexpr int kScreenWarps = kScreenBlock / 32;

struct ScreenArgs {
  const uint32_t* Sa;
  const uint32_t* Ra;
  const int4* ops;       // {oa, va, ob, vb} (compressed)
  const int* order;      // operator indices in alpha-part order
  const int4* qa;        // per slot: {oa, va, op, beta list offset}
  const int* qn;         // per slot: beta list length (-1: empty beta half)
  const int2* opl;       // per operator: {beta list offset, length}; length < 0: empty beta half
  const int2* blist;     // beta source lists: {rb_src, rb_tgt}
  int n_ops;
  const double2* psi;
  const double2* w;
  const uint32_t* psi_arow;  // alpha-row occupancy of psi (or nullptr)
  const uint32_t* w_arow;    // alpha-row occupancy of w on owned rows (or nullptr)
  int64_t Nb;
  int64_t a_lo, a_hi;
  int slices;
  double* part;          // [alpha rows][n_ops]
};

__device__ __forceinline__ double re_conj_mul(double2 a, double2 b) {
  return a.x * b.x + a.y * b.y;   // Re(conj(a) b)
}

// D list entries per lane in flight: 2 (44 registers) while psi sits in L2, 4
// (54 registers, fewer resident warps) once the gathers go to DRAM: H12 0.72 vs
// 0.77 ms with 2, H16 0.68 vs 0.59 s with 4; 8 spills.
//
// PIVOT (sparse psi): a CTA owns one alpha row rp of psi instead of one owned
// row of w, and each operator pairs it with the w row Ra[s_p ^ f_a] (skipped
// outside [a_lo, a_hi) or where w is zero).  The same (w row, psi row, beta
// list) triples are summed, grouped by psi row: CTAs of empty psi rows write
// zeros and leave, so the cost follows the support of psi.
template <int D, bool PIVOT>
__global__ void __launch_bounds__(kScreenBlock) k_screen(const ScreenArgs a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t rloc = blockIdx.y;
  const int64_t rc = PIVOT ? rloc : a.a_lo + rloc;   // the CTA's row: w (own) or psi
  const uint32_t sc = __ldg(a.Sa + rc);
  const double2* __restrict__ crow = (PIVOT ? a.psi : a.w) + rc * a.Nb;
  const int stride = a.slices * kScreenWarps;
  const bool c_zero = PIVOT ? (a.psi_arow && !__ldg(a.psi_arow + rc))
                            : (a.w_arow && !__ldg(a.w_arow + rc));
  int q = blockIdx.x * kScreenWarps + warp;
  if (PIVOT && c_zero) {   // empty psi row: its partials are zero
    if (lane == 0)
      for (; q < a.n_ops; q += stride) a.part[rloc * a.n_ops + __ldg(a.qa + q).z] = 0.0;
    return;
  }
  // per-slot records in screen order, the next one loaded while the current
  // operator's list is walked (the per-operator setup was a chain of dependent
  // loads: order -> masks -> partner rank -> flag -> list)
  int4 Qn = q < a.n_ops ? __ldg(a.qa + q) : make_int4(0, 0, 0, 0);
  int Ln = q < a.n_ops ? __ldg(a.qn + q) : 0;
  for (; q < a.n_ops; q += stride) {
    const int4 Q = Qn;
    const int Ly = Ln;
    if (q + stride < a.n_ops) {
      Qn = __ldg(a.qa + q + stride);
      Ln = __ldg(a.qn + q + stride);
    }
    const int op = Q.z;
    const uint32_t oa = (uint32_t)Q.x, va = (uint32_t)Q.y;
    const uint32_t fa = oa | va;
    const uint32_t m = sc & fa;
    // as / at: the w row in source / target pattern (both for an empty alpha half);
    // when pivoting the CTA row is the psi partner, whose pattern is the reverse
    const bool as = PIVOT ? m == va : m == oa, at = PIVOT ? m == oa : m == va;
    double g = 0.0;
    const uint32_t r2 = (as || at) ? __ldg(a.Ra + (sc ^ fa)) : 0u;
    bool ok = (as || at) && !c_zero;
    if (PIVOT)
      ok = ok && r2 >= (uint32_t)a.a_lo && r2 < (uint32_t)a.a_hi &&
           !(a.w_arow && !__ldg(a.w_arow + r2));
    else
      ok = ok && !(a.psi_arow && !__ldg(a.psi_arow + r2));
    if (ok) {
      // 32-bit row offsets (dim < 2^32, checked by K1) and D list entries per
      // lane in flight: independent gathers instead of one latency per entry
      // (0.87 -> 0.72 ms at H12)
      const double2* __restrict__ wrow = PIVOT ? a.w + r2 * (uint32_t)a.Nb : crow;
      const double2* __restrict__ prow = PIVOT ? crow : a.psi + r2 * (uint32_t)a.Nb;
      const int2 L = make_int2(Q.w, Ly);
      if (L.y < 0) {
        // empty beta half: every beta string is both source and target (alpha decides)
        for (int64_t j = lane; j < a.Nb; j += 32) g += re_conj_mul(wrow[j], prow[j]);
        if (!at) g = -g;
      } else {
        const int2* __restrict__ lst = a.blist + L.x;
        // own rows in source pattern: (T psi)_b = -psi_p; in target pattern: +psi_p
#pragma unroll
        for (int side = 0; side < 2; ++side) {
          if (!(side == 0 ? as : at)) continue;
          double g4[4] = {0.0, 0.0, 0.0, 0.0};
          int j = lane;
          for (; j + 32 * (D - 1) < L.y; j += 32 * D) {
            int2 e[D];
#pragma unroll
            for (int q = 0; q < D; ++q) e[q] = __ldg(lst + j + 32 * q);
            double2 wv[D], pv[D];
#pragma unroll
            for (int q = 0; q < D; ++q) {
              wv[q] = wrow[side == 0 ? e[q].x : e[q].y];
              pv[q] = prow[side == 0 ? e[q].y : e[q].x];
            }
#pragma unroll
            for (int q = 0; q < D; ++q) g4[q] += re_conj_mul(wv[q], pv[q]);
          }
          for (; j < L.y; j += 32) {
            const int2 e = __ldg(lst + j);
            g4[0] += re_conj_mul(wrow[side == 0 ? e.x : e.y], prow[side == 0 ? e.y : e.x]);
          }
          const double s4 = (g4[0] + g4[1]) + (g4[2] + g4[3]);
          g = side == 0 ? g - s4 : g + s4;
        }
      }
    }
    g = warp_sum(g);
    if (lane == 0) a.part[rloc * a.n_ops + op] = 2.0 * g;
  }
}

// One block per beta pattern: rank-ascending source strings and partners.
__global__ void __launch_bounds__(1024) k_beta_lists(const uint32_t* __restrict__ Sb,
                                                     const uint32_t* __restrict__ Rb, int64_t Nb,
                                                     const int4* __restrict__ pats,
                                                     int2* __restrict__ out) {
  using Scan = cub::BlockScan<int, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  const int4 P = pats[blockIdx.x];   // {ob, vb, offset, count}
  const uint32_t ob = (uint32_t)P.x, vb = (uint32_t)P.y, fb = ob | vb;
  int base = P.z;
  for (int64_t c0 = 0; c0 < Nb; c0 += 1024) {
    const int64_t i = c0 + threadIdx.x;
    uint32_t s = 0;
    int f = 0;
    if (i < Nb) {
      s = Sb[i];
      f = (s & fb) == ob ? 1 : 0;
    }
    int off, tot;
    Scan(tmp).ExclusiveSum(f, off, tot);
    if (f) out[base + off] = make_int2((int)i, (int)Rb[s ^ fb]);
    base += tot;
    __syncthreads();
  }
}

int pool_prepare(hsv_pool_s* p) {
  const hsv_sector_s* s = p->sec;
  const int64_t n = p->n;
  std::map<std::pair<uint32_t, uint32_t>, int> pid;
  std::vector<int4> pats;
  std::vector<int2> opl(n);
  int64_t total = 0;
  for (int64_t i = 0; i < n; ++i) {
    const uint32_t ob = (uint32_t)p->h[i].z, vb = (uint32_t)p->h[i].w;
    if ((ob | vb) == 0) { opl[i] = make_int2(0, -1); continue; }
    auto key = std::make_pair(ob, vb);
    auto it = pid.find(key);
    if (it == pid.end()) {
      const int64_t cnt = src_count(s->norb, s->n_beta, ob, vb);
      pats.push_back(make_int4((int)ob, (int)vb, (int)total, (int)cnt));
      it = pid.emplace(key, (int)pats.size() - 1).first;
      total += cnt;
    }
    opl[i] = make_int2(pats[it->second].z, pats[it->second].w);
  }
  HSV_REQUIRE(total < INT32_MAX, HSV_ERR_UNSUPPORTED, "beta pattern lists too large");
  std::vector<int> order(n);
  for (int64_t i = 0; i < n; ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
    const uint32_t fx = (uint32_t)(p->h[x].x | p->h[x].y), fy = (uint32_t)(p->h[y].x | p->h[y].y);
    return fx != fy ? fx < fy : (uint32_t)p->h[x].x < (uint32_t)p->h[y].x;
  });
  // per-slot records in screen order: no dependent order -> op -> masks chain
  std::vector<int4> qa(n);
  std::vector<int> qn(n);
  for (int64_t q = 0; q < n; ++q) {
    const int op = order[q];
    qa[q] = make_int4(p->h[op].x, p->h[op].y, op, opl[op].x);
    qn[q] = opl[op].y;
  }
  HSV_TRY(dalloc(&p->d_order, n));
  HSV_TRY(dalloc(&p->d_opl, n));
  HSV_TRY(dalloc(&p->d_qa, n));
  HSV_TRY(dalloc(&p->d_qn, n));
  HSV_TRY(dalloc(&p->d_blist, total));
  int4* d_pats = nullptr;
  HSV_TRY(dalloc(&d_pats, pats.size()));
  cudaStream_t st = stream();
  if (n) {
    HSV_TRY_CUDA(cudaMemcpyAsync(p->d_order, order.data(), n * sizeof(int), cudaMemcpyHostToDevice, st));
    HSV_TRY_CUDA(cudaMemcpyAsync(p->d_opl, opl.data(), n * sizeof(int2), cudaMemcpyHostToDevice, st));
    HSV_TRY_CUDA(cudaMemcpyAsync(p->d_qa, qa.data(), n * sizeof(int4), cudaMemcpyHostToDevice, st));
    HSV_TRY_CUDA(cudaMemcpyAsync(p->d_qn, qn.data(), n * sizeof(int), cudaMemcpyHostToDevice, st));
  }
  if (!pats.empty()) {
    HSV_TRY_CUDA(cudaMemcpyAsync(d_pats, pats.data(), pats.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
    k_beta_lists<<<(unsigned)pats.size(), 1024, 0, st>>>(s->d_Sb, s->d_Rb, s->Nb, d_pats, p->d_blist);
    count_launch();
    HSV_CHECK_LAUNCH();
  }
  HSV_TRY(stream_sync());
  dfree(d_pats);
  return HSV_OK;
}

// K4 partials of owned alpha rows [r0, r1) (no pivot) into part rows
// [r0 - part_row0, r1 - part_row0) on stream st.
static int launch_screen_rows(const hsv_op_s* op, const double2* psi, const double2* w,
                              const hsv_pool_s* pool, int64_t r0, int64_t r1, double* part,
                              const uint32_t* psi_arow, cudaStream_t st) {
  const hsv_sector_s* s = op->sec;
  const int n_ops = (int)pool->n;
  const int64_t rows = r1 - r0;
  if (n_ops <= 0 || rows <= 0) return HSV_OK;
  HSV_REQUIRE(rows <= 65535, HSV_ERR_UNSUPPORTED, "too many alpha rows for one launch");
  const int64_t want = (int64_t)ctx().num_sms * 8 * 4;
  int slices = (int)std::min<int64_t>((want + rows - 1) / rows,
                                      (n_ops + kScreenWarps - 1) / kScreenWarps);
  slices = std::max(slices, 1);
  ScreenArgs a{};
  a.Sa = s->d_Sa; a.Ra = s->d_Ra;
  a.ops = pool->d; a.order = pool->d_order; a.opl = pool->d_opl; a.blist = pool->d_blist;
  a.qa = pool->d_qa; a.qn = pool->d_qn;
  a.n_ops = n_ops; a.psi = psi; a.w = w; a.Nb = s->Nb; a.a_lo = r0; a.a_hi = r1;
  a.slices = slices;
  a.part = part;
  a.psi_arow = psi_arow;
  a.w_arow = nullptr;
  const dim3 grid((unsigned)slices, (unsigned)rows);
  const bool big = 2 * s->dim * (int64_t)sizeof(double2) > ctx().l2_bytes;
  big ? k_screen<4, false><<<grid, kScreenBlock, 0, st>>>(a)
      : k_screen<2, false><<<grid, kScreenBlock, 0, st>>>(a);
  count_launch();
  HSV_CHECK_LAUNCH();
  return HSV_OK;
}

int launch_screen(const hsv_op_s* op, const double2* psi, const double2* w,
                  const hsv_pool_s* pool, int64_t a_lo, int64_t a_hi, double* d_grads,
                  const uint32_t* psi_arow, const uint32_t* w_arow, bool sparse_psi) {
  const hsv_sector_s* s = op->sec;
  const int n_ops = (int)pool->n;
  if (n_ops <= 0) return HSV_OK;
  const int pv = tuning().screen_pivot;
  const bool pivot = a_hi > a_lo && psi_arow && (pv > 0 || (pv < 0 && sparse_psi));
  const int64_t rows = pivot ? s->Na : a_hi - a_lo;
  if (a_hi <= a_lo) {
    HSV_TRY_CUDA(cudaMemsetAsync(d_grads, 0, n_ops * sizeof(double), stream()));
    return HSV_OK;
  }
  HSV_REQUIRE(rows <= 65535, HSV_ERR_UNSUPPORTED, "too many alpha rows for one launch");
  // enough CTAs to fill the machine several times over
  const int64_t want = (int64_t)ctx().num_sms * 8 * 4;
  int slices = (int)std::min<int64_t>((want + rows - 1) / rows,
                                      (n_ops + kScreenWarps - 1) / kScreenWarps);
  slices = std::max(slices, 1);
  double* part = nullptr;
  HSV_TRY(dalloc(&part, rows * n_ops));
  ScreenArgs a{};
  a.Sa = s->d_Sa; a.Ra = s->d_Ra;
  a.ops = pool->d; a.order = pool->d_order; a.opl = pool->d_opl; a.blist = pool->d_blist;
  a.qa = pool->d_qa; a.qn = pool->d_qn;
  a.n_ops = n_ops; a.psi = psi; a.w = w; a.Nb = s->Nb; a.a_lo = a_lo; a.a_hi = a_hi;
  a.slices = slices;
  a.part = part;
  a.psi_arow = psi_arow;
  a.w_arow = w_arow;
  {
    ProfScope prof("screen");
    const dim3 grid((unsigned)slices, (unsigned)rows);
    const bool big = 2 * s->dim * (int64_t)sizeof(double2) > ctx().l2_bytes;
    if (pivot)
      big ? k_screen<4, true><<<grid, kScreenBlock, 0, stream()>>>(a)
          : k_screen<2, true><<<grid, kScreenBlock, 0, stream()>>>(a);
    else
      big ? k_screen<4, false><<<grid, kScreenBlock, 0, stream()>>>(a)
          : k_screen<2, false><<<grid, kScreenBlock, 0, stream()>>>(a);
  }
  count_launch();
  HSV_CHECK_LAUNCH();
  HSV_TRY(reduce_sum_f64(part, rows, n_ops, n_ops, d_grads));
  dfree(part);
  return HSV_OK;
}

}  // namespace hsv

using namespace hsv;

extern "C" {

// Energy + screen with the assembled rows, overlapped: K1a runs phase after
// phase (alpha-row ranges, chunk-aligned) on the library stream, and K4 works on
// each finished range on a second stream while K1a streams the next one (K1a
// is HBM-bound, K4 L1-bound on L2-resident data).  The K4 partials and the K1a
// energy partials are reduced once, in the serial path's order: bitwise equal.
static int energy_screen_overlap(hsv_op op, hsv_state psi, const hsv_pool_s* pool, int64_t a_lo,
                                 int64_t a_hi, double* d_out, bool* done) {
  *done = false;
  const int P = tuning().screen_overlap;
  if (P <= 1 || !psi->dense_hint || pool->n <= 0 || a_hi - a_lo < 2 * P) return HSV_OK;
  int64_t nc = 0;
  HSV_TRY(sell_chunks(op, a_lo, a_hi, &nc));
  if (nc == 0) return HSV_OK;
  const hsv_sector_s* s = op->sec;
  Context& C = ctx();
  if (!C.aux) HSV_TRY_CUDA(cudaStreamCreateWithFlags(&C.aux, cudaStreamNonBlocking));
  while ((int)C.aux_ev.size() < P + 1) {
    cudaEvent_t e;
    HSV_TRY_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    C.aux_ev.push_back(e);
  }
  const int n_ops = (int)pool->n;
  const int64_t rows = a_hi - a_lo;
  double2* w = nullptr;
  double *cpart = nullptr, *part = nullptr;
  HSV_TRY(dalloc(&w, s->dim));
  HSV_TRY(dalloc(&cpart, 2 * nc));
  HSV_TRY(dalloc(&part, rows * n_ops));
  HSV_TRY(state_arow_async(psi));
  const int64_t Nb = s->Nb;
  int64_t c_prev = 0, done_rows = a_lo;
  for (int r = 0; r < P; ++r) {
    // phase r: chunks up to the one holding the end of alpha row ra1 - 1 ...
    const int64_t ra1 = a_lo + rows * (r + 1) / P;
    const int64_t c1 = r == P - 1 ? nc : ((ra1 - a_lo) * Nb) / 32;
    HSV_TRY(sell_apply_chunks(op, psi->d_amp, w, a_lo, a_hi, c_prev, c1, cpart));
    HSV_TRY_CUDA(cudaEventRecord(C.aux_ev[r], stream()));
    // ... and K4 on the alpha rows those chunks completed
    const int64_t ra_done = r == P - 1 ? a_hi : a_lo + (c1 * 32) / Nb;
    if (ra_done > done_rows) {
      HSV_TRY_CUDA(cudaStreamWaitEvent(C.aux, C.aux_ev[r], 0));
      ProfScope prof("screen", C.aux);
      HSV_TRY(launch_screen_rows(op, psi->d_amp, w, pool, done_rows, ra_done,
                                 part + (done_rows - a_lo) * n_ops, psi->d_arow, C.aux));
      done_rows = ra_done;
    }
    c_prev = c1;
  }
  HSV_TRY_CUDA(cudaEventRecord(C.aux_ev[P], C.aux));
  HSV_TRY_CUDA(cudaStreamWaitEvent(stream(), C.aux_ev[P], 0));
  HSV_TRY(reduce_sum_f64(cpart, nc, 2, 2, d_out));
  HSV_TRY(reduce_sum_f64(part, rows, n_ops, n_ops, d_out + 2));
  dfree(part);
  dfree(cpart);
  dfree(w);
  *done = true;
  return HSV_OK;
}

static int energy_screen_dev(hsv_op op, hsv_state psi, const hsv_pool_s* pool, int64_t a_lo,
                             int64_t a_hi, double* d_out) {
  const hsv_sector_s* s = op->sec;
  {
    bool done = false;
    HSV_TRY(energy_screen_overlap(op, psi, pool, a_lo, a_hi, d_out, &done));
    if (done) return HSV_OK;
  }
  ProfScope prof_all("es_all");
  double2* w = nullptr;
  HSV_TRY(dalloc(&w, s->dim));
  const int nw = apply_warps(op);
  double* epart = nullptr;
  HSV_TRY(dalloc(&epart, 2 * (int64_t)nw));
  HSV_TRY_CUDA(cudaMemsetAsync(epart, 0, 2 * sizeof(double) * nw, stream()));
  int64_t used = 0;
  {
    ProfScope prof("es_arow");
    HSV_TRY(state_arow_async(psi));
  }
  {
    ProfScope prof("es_k1");
    HSV_TRY(launch_apply(op, psi->d_amp, w, epart, a_lo, a_hi, 0.0, 0, &used, psi->d_arow,
                         &psi->dense_hint));
  }
  if (used == 1)   // already reduced to one (re, im) pair (dynamic schedule, push path)
    HSV_TRY_CUDA(cudaMemcpyAsync(d_out, epart, 2 * sizeof(double), cudaMemcpyDeviceToDevice,
                                 stream()));
  else
    HSV_TRY(reduce_sum_f64(epart, used, 2, 2, d_out));
  // occupancy of the owned rows of w (other rows of w are never read), which
  // only lets K4 skip empty rows: not computed for a dense psi
  uint32_t* wrow = nullptr;
  if (!psi->dense_hint) {
    HSV_TRY(dalloc(&wrow, std::max<int64_t>(s->Na, 1)));
    HSV_TRY(arow_flags_async(w + a_lo * s->Nb, a_hi - a_lo, s->Nb, wrow + a_lo));
  }
  // psi found sparse by K1 (push path taken, dense_hint still clear): pivot on psi rows
  ProfScope prof_k4("es_k4");
  HSV_TRY(launch_screen(op, psi->d_amp, w, pool, a_lo, a_hi, d_out + 2, psi->d_arow, wrow,
                        !psi->dense_hint));
  dfree(wrow);
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
  hsv_pool pool = nullptr;
  HSV_TRY(hsv_pool_create(op->sec, occ, virt, n_ops, &pool));
  const int rc = energy_screen_dev(op, psi, pool, a_lo, a_hi, d_out);
  hsv_pool_destroy(pool);
  return rc;
}

int hsv_energy_screen_pool_async(hsv_op op, hsv_state psi, hsv_pool pool, int64_t a_lo,
                                 int64_t a_hi, double* d_out) {
  HSV_TRY(check_es_args(op, psi, a_lo, a_hi));
  HSV_REQUIRE(pool && d_out && pool->sec == op->sec, HSV_ERR_INVALID, "bad pool argument");
  return energy_screen_dev(op, psi, pool, a_lo, a_hi, d_out);
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
