// K3b / K5b: batched forward and adjoint sweeps (ansatz_energy_gradient,
// svengine.py:260-281), one grid barrier per BATCH of up to kBatch
// consecutive rotations instead of one per rotation.
//
// Why it is exact.  The flip masks f_1..f_m of a batch (linearly independent
// over GF(2), enforced when batches are formed) generate a group of 2^m key
// translations; its orbits {b ^ XOR_{j in S} f_j} are closed under every
// rotation of the batch (a rotation pairs b with b ^ f_j).  A thread that owns
// one orbit can therefore apply rotation 1, then 2, ..., then m to the orbit's
// amplitudes in registers and reproduce, amplitude for amplitude, the
// sequential result: every amplitude sees the same Givens products, in the
// same order, with the same non-FMA roundings (svengine.py:219-233).
//
// Work items.  Only orbits that contain a source row of some rotation matter.
// They are enumerated once per operator list (the plan, cached across the
// L-BFGS evaluations and ADAPT iterations: an appended operator only changes
// the last batch): every (op j, source row b) pair is unranked directly and
// kept iff (b, j) is the smallest (key, op) source pair of its orbit; a
// stable compaction (cub::DeviceSelect) lists the kept orbits in enumeration
// order, so the plan and every reduction over it are deterministic.
//
// Support.  The forward sweep maintains the structural support map of psi
// (hsv_state_s::d_smap; a rotation with s != 0 marks both rows of a pair if
// either is marked).  Orbits with no marked row hold only exact zeros: the
// forward sweep skips them, and so does the adjoint sweep (it reads w = H psi
// only on the support, see K1r).
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "hsv_common.cuh"
#include "hsv_kernels.cuh"

namespace hsv {

namespace {

constexpr int kBatch = 3;               // rotations per batch (orbits of 2^kBatch rows)
constexpr int kOrb = 1 << kBatch;
enum { kFwd = 0, kAdj = 1 };

struct BatchDev {
  uint32_t oa[kBatch], va[kBatch], ob[kBatch], vb[kBatch];
  double c[kBatch], s[kBatch];
  int n;                 // rotations in the batch
  int op0;               // index (in sweep-list order) of the batch's first rotation
  const uint2* items;    // orbit representatives (sa, sb)
  const uint32_t* count; // number of items (device)
};

struct BSweepArgs {
  const BatchDev* batches;
  int n_batches;          // in processing order (adjoint: reversed)
  int n_ops;
  int n_alpha, n_beta;
  int64_t Nb;
  const uint32_t* Ra;
  const uint32_t* Rb;
  double2* psi;
  double2* lam;
  uint8_t* smap;          // forward: maintained; adjoint: read (support of the final psi)
  double* part;           // [batch][block][kBatch][NV]
  double* red;            // [op][NV] per-rotation totals, sweep-list order
  double* norm2;
  double* grads;          // adjoint: gradient of list op i at grads[i]
  int* err;
  double* err_val;
  unsigned long long* stats;   // pairs processed (kStatPairsFwd / kStatPairsAdj)
};

__device__ __forceinline__ void rot(double2 vb, double2 vp, double c, double s, double2& nb,
                                    double2& np) {
  nb.x = __dadd_rn(__dmul_rn(c, vb.x), __dmul_rn(-s, vp.x));
  nb.y = __dadd_rn(__dmul_rn(c, vb.y), __dmul_rn(-s, vp.y));
  np.x = __dadd_rn(__dmul_rn(c, vp.x), __dmul_rn(s, vb.x));
  np.y = __dadd_rn(__dmul_rn(c, vp.y), __dmul_rn(s, vb.y));
}

__device__ __forceinline__ double n2(double2 v) { return v.x * v.x + v.y * v.y; }

__device__ __forceinline__ bool is_src(uint32_t sa, uint32_t sb, uint32_t oa, uint32_t va,
                                       uint32_t ob, uint32_t vb) {
  return (sa & oa) == oa && (sa & va) == 0u && (sb & ob) == ob && (sb & vb) == 0u;
}

__device__ __forceinline__ void grid_sync() { cooperative_groups::this_grid().sync(); }

// i-th string (ascending) with occ set, virt clear and `ones` electrons on the
// remaining orbitals of nmask (binomials bt[n * 32 + k]).
__device__ __forceinline__ uint32_t unrank(int64_t i, uint32_t occ, uint32_t virt, uint32_t nmask,
                                           int ones, const int64_t* bt) {
  uint32_t fm = nmask & ~(occ | virt);
  uint32_t s = occ;
  for (int p = __popc(fm) - 1; p >= 0 && ones > 0; --p) {
    const int pos = 31 - __clz(fm);
    fm &= ~(1u << pos);
    const int64_t c = ones <= p ? bt[p * kBinomN + ones] : 0;
    if (i >= c) {
      s |= 1u << pos;
      i -= c;
      --ones;
    }
  }
  return s;
}

// Plan build: candidate orbit representatives of one batch.  Thread t covers
// source pair t of the batch (op j = the op whose range holds t).
struct BuildArgs {
  uint32_t oa[kBatch], va[kBatch], ob[kBatch], vb[kBatch];
  int64_t ca[kBatch], cb[kBatch], off[kBatch + 1];
  int n, norb, n_alpha, n_beta;
  const int64_t* binom;
  uint2* cand;
  uint8_t* flag;
};

__global__ void k_plan_candidates(const BuildArgs a) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= a.off[a.n]) return;
  int j = 0;
  while (t >= a.off[j + 1]) ++j;
  const int64_t r = t - a.off[j];
  const int64_t ia = r / a.cb[j], ib = r - ia * a.cb[j];
  const uint32_t nmask = a.norb >= 32 ? 0xffffffffu : ((1u << a.norb) - 1u);
  const uint32_t sa = unrank(ia, a.oa[j], a.va[j], nmask, a.n_alpha - __popc(a.oa[j]), a.binom);
  const uint32_t sb = unrank(ib, a.ob[j], a.vb[j], nmask, a.n_beta - __popc(a.ob[j]), a.binom);
  const uint64_t key = (uint64_t)sb << 32 | sa;
  bool keep = true;
  for (int S = 1; S < (1 << a.n) && keep; ++S) {   // S = 0 is b itself
    uint32_t ea = sa, eb = sb;
    for (int i = 0; i < a.n; ++i)
      if ((S >> i) & 1) { ea ^= a.oa[i] | a.va[i]; eb ^= a.ob[i] | a.vb[i]; }
    if (__popc(ea) != a.n_alpha || __popc(eb) != a.n_beta) continue;
    const uint64_t ek = (uint64_t)eb << 32 | ea;
    for (int i = 0; i < a.n; ++i)
      if (is_src(ea, eb, a.oa[i], a.va[i], a.ob[i], a.vb[i]) && (ek < key || (ek == key && i < j)))
        keep = false;
  }
  // b itself as a source of an earlier op of the batch
  for (int i = 0; i < j; ++i)
    if (is_src(sa, sb, a.oa[i], a.va[i], a.ob[i], a.vb[i])) keep = false;
  a.cand[t] = make_uint2(sa, sb);
  a.flag[t] = keep ? 1 : 0;
}

// One orbit of a batch: forward rotations (MODE kFwd) or, in reverse order,
// gradient partial + adjoint rotation + uncompute (kAdj).
template <int MODE>
__device__ __forceinline__ void do_orbit(const BSweepArgs& a, const BatchDev& B, uint2 rep,
                                         double (&acc)[kBatch][3], unsigned& npairs) {
  uint32_t ea[kOrb], eb[kOrb];
  unsigned touched = 0u, srcm[kBatch];
#pragma unroll
  for (int j = 0; j < kBatch; ++j) srcm[j] = 0u;
#pragma unroll
  for (int t = 0; t < kOrb; ++t) {
    uint32_t x = rep.x, y = rep.y;
#pragma unroll
    for (int j = 0; j < kBatch; ++j)
      if (((t >> j) & 1) && j < B.n) { x ^= B.oa[j] | B.va[j]; y ^= B.ob[j] | B.vb[j]; }
    ea[t] = x;
    eb[t] = y;
    if (t >= (1 << B.n) || __popc(x) != a.n_alpha || __popc(y) != a.n_beta) continue;
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      if (j >= B.n) continue;
      if (is_src(x, y, B.oa[j], B.va[j], B.ob[j], B.vb[j])) {
        srcm[j] |= 1u << t;
        touched |= (1u << t) | (1u << (t ^ (1 << j)));
      }
    }
  }
  uint32_t row[kOrb];
  unsigned marked = 0u;
#pragma unroll
  for (int t = 0; t < kOrb; ++t) {
    row[t] = 0u;
    if ((touched >> t) & 1u) {
      row[t] = __ldg(a.Ra + ea[t]) * (uint32_t)a.Nb + __ldg(a.Rb + eb[t]);
      if (!a.smap || a.smap[row[t]]) marked |= 1u << t;
    }
  }
  if (!marked) return;               // exact zeros only (or outside the support)
#pragma unroll
  for (int j = 0; j < kBatch; ++j) npairs += __popc(srcm[j]);
  double2 v[kOrb];
  double2 l[kOrb];
#pragma unroll
  for (int t = 0; t < kOrb; ++t) {
    v[t] = make_double2(0.0, 0.0);
    l[t] = make_double2(0.0, 0.0);
    if ((touched >> t) & 1u) {
      v[t] = a.psi[row[t]];
      if (MODE == kAdj) l[t] = a.lam[row[t]];
    }
  }
  if (MODE == kFwd) {
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      if (j >= B.n || (B.c[j] == 1.0 && B.s[j] == 0.0)) continue;   // theta == 0: skipped
#pragma unroll
      for (int t = 0; t < kOrb; ++t) {
        if (!((srcm[j] >> t) & 1u)) continue;
        const int p = t ^ (1 << j);
        double2 nb, np;
        rot(v[t], v[p], B.c[j], B.s[j], nb, np);
        acc[j][0] += n2(v[t]) + n2(v[p]);
        acc[j][1] += n2(nb) + n2(np);
        v[t] = nb;
        v[p] = np;
        if ((marked >> t | marked >> p) & 1u) marked |= (1u << t) | (1u << p);
      }
    }
#pragma unroll
    for (int t = 0; t < kOrb; ++t) {
      if (!((touched >> t) & 1u)) continue;
      a.psi[row[t]] = v[t];
      if (a.smap && ((marked >> t) & 1u)) a.smap[row[t]] = 1;
    }
  } else {
#pragma unroll
    for (int jj = kBatch - 1; jj >= 0; --jj) {
      if (jj >= B.n) continue;
      const bool unc = B.op0 + jj > 0;   // psi of the first rotation is never read again
#pragma unroll
      for (int t = 0; t < kOrb; ++t) {
        if (!((srcm[jj] >> t) & 1u)) continue;
        const int p = t ^ (1 << jj);
        const double2 pb = v[t], pp = v[p], lb = l[t], lp = l[p];
        acc[jj][0] += (lp.x * pb.x + lp.y * pb.y) - (lb.x * pp.x + lb.y * pp.y);
        double2 nb, np;
        rot(lb, lp, B.c[jj], -B.s[jj], nb, np);
        acc[jj][1] += n2(lb) + n2(lp);
        acc[jj][2] += n2(nb) + n2(np);
        l[t] = nb;
        l[p] = np;
        if (unc) {
          double2 qb, qp;
          rot(pb, pp, B.c[jj], -B.s[jj], qb, qp);
          v[t] = qb;
          v[p] = qp;
        }
      }
    }
#pragma unroll
    for (int t = 0; t < kOrb; ++t) {
      if (!((touched >> t) & 1u)) continue;
      a.lam[row[t]] = l[t];
      a.psi[row[t]] = v[t];
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) k_bsweep(const BSweepArgs a) {
  constexpr int NV = MODE == kAdj ? 3 : 2;
  __shared__ double sh[8][kBatch][NV];
  __shared__ BatchDev B;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  for (int bi = 0; bi < a.n_batches; ++bi) {
    if (threadIdx.x == 0) B = a.batches[bi];
    __syncthreads();
    const uint32_t n_items = __ldg(B.count);
    double acc[kBatch][3];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) acc[j][0] = acc[j][1] = acc[j][2] = 0.0;
    unsigned npairs = 0u;
    for (int64_t it = gt; it < n_items; it += nt)
      do_orbit<MODE>(a, B, __ldg(B.items + it), acc, npairs);
    if (a.stats) {
      const unsigned tot = __reduce_add_sync(0xffffffffu, npairs);
      if (lane == 0 && tot) atomicAdd(a.stats + (MODE == kFwd ? kStatPairsFwd : kStatPairsAdj),
                                      (unsigned long long)tot);
    }
    // block partials per rotation (fixed shuffle tree and warp order)
#pragma unroll
    for (int j = 0; j < kBatch; ++j)
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const double x = warp_sum(acc[j][q]);
        if (lane == 0) sh[w][j][q] = x;
      }
    __syncthreads();
    if (threadIdx.x < kBatch * NV) {
      const int j = threadIdx.x / NV, q = threadIdx.x - j * NV;
      double x = 0.0;
      for (int k = 0; k < 8; ++k) x += sh[k][j][q];
      a.part[(((int64_t)bi * gridDim.x + blockIdx.x) * kBatch + j) * NV + q] = x;
    }
    __syncthreads();
    grid_sync();   // batch bi+1 reads rows batch bi wrote
  }
  // per-rotation totals: one rotation per warp, blocks summed in a fixed order
  const int64_t gw = gt >> 5, nw = nt >> 5;
  for (int64_t oi = gw; oi < (int64_t)a.n_batches * kBatch; oi += nw) {
    const int bi = (int)(oi / kBatch), j = (int)(oi - (int64_t)bi * kBatch);
    const BatchDev& B = a.batches[bi];
    if (j >= B.n) continue;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double x = 0.0;
      for (int k = lane; k < (int)gridDim.x; k += 32)
        x += __ldcg(a.part + (((int64_t)bi * gridDim.x + k) * kBatch + j) * NV + q);
      x = warp_sum(x);
      if (lane == 0) a.red[(int64_t)(B.op0 + j) * NV + q] = x;
    }
  }
  grid_sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {   // norm chain in sweep order (svengine.py:234-236)
    double nn = *a.norm2;
    for (int o = 0; o < a.n_ops; ++o) {
      const int op = MODE == kFwd ? o : a.n_ops - 1 - o;
      const double* tot = a.red + (int64_t)op * NV;
      const double dold = MODE == kAdj ? __ldcg(tot + 1) : __ldcg(tot);
      const double dnew = MODE == kAdj ? __ldcg(tot + 2) : __ldcg(tot + 1);
      const double nnew = nn - dold + dnew;
      const double nrm = sqrt(fmax(nn, 0.0));
      const double drift = fabs(sqrt(fmax(nnew, 0.0)) - nrm);
      if (drift > kNormDriftTol * fmax(1.0, nrm)) {
        if (atomicExch(a.err, 1) == 0) *a.err_val = drift;
      }
      nn = nnew;
      if (MODE == kAdj) a.grads[op] = 2.0 * __ldcg(tot);
    }
    *a.norm2 = nn;
  }
}

// ----------------------------------------------------------------- plans
struct PlanBatch {
  std::vector<OpMasks> m;
  int64_t n_cand = 0;
  uint2* items = nullptr;
  uint32_t* count = nullptr;
};

struct Plan {
  const hsv_sector_s* sec = nullptr;
  std::vector<PlanBatch> b;
  void clear() {
    for (auto& x : b) { dfree(x.items); dfree(x.count); }
    b.clear();
  }
};

Plan& plan() {
  static Plan p;
  return p;
}

bool same(const OpMasks& x, const OpMasks& y) {
  return x.oa == y.oa && x.va == y.va && x.ob == y.ob && x.vb == y.vb;
}

// Greedy batches of consecutive rotations with independent flip masks.
std::vector<std::vector<int>> partition(const std::vector<OpMasks>& ops) {
  std::vector<std::vector<int>> out;
  std::vector<uint64_t> span;   // span of the current batch's flips (all subset XORs)
  for (int i = 0; i < (int)ops.size(); ++i) {
    const uint64_t f = (uint64_t)(ops[i].ob | ops[i].vb) << 32 | (ops[i].oa | ops[i].va);
    bool dep = false;
    for (uint64_t x : span) dep |= x == f;
    if (out.empty() || (int)out.back().size() == kBatch || dep) {
      out.push_back({});
      span.assign(1, 0ull);
    }
    out.back().push_back(i);
    const size_t n = span.size();
    for (size_t q = 0; q < n; ++q) span.push_back(span[q] ^ f);
  }
  return out;
}

int build_batch(const hsv_sector_s* sec, PlanBatch& pb) {
  BuildArgs a{};
  a.n = (int)pb.m.size();
  a.norb = sec->norb; a.n_alpha = sec->n_alpha; a.n_beta = sec->n_beta;
  a.binom = sec->d_binom;
  a.off[0] = 0;
  for (int j = 0; j < a.n; ++j) {
    const OpMasks& m = pb.m[j];
    a.oa[j] = m.oa; a.va[j] = m.va; a.ob[j] = m.ob; a.vb[j] = m.vb;
    a.ca[j] = src_count(sec->norb, sec->n_alpha, m.oa, m.va);
    a.cb[j] = src_count(sec->norb, sec->n_beta, m.ob, m.vb);
    if (a.ca[j] == 0 || a.cb[j] == 0) a.ca[j] = a.cb[j] = 0;
    a.off[j + 1] = a.off[j] + a.ca[j] * a.cb[j];
  }
  if (a.cb[0] == 0) a.cb[0] = 1;   // guard the division of an empty range
  for (int j = 1; j < a.n; ++j)
    if (a.cb[j] == 0) a.cb[j] = 1;
  const int64_t T = a.off[a.n];
  pb.n_cand = T;
  HSV_TRY(dalloc(&pb.items, std::max<int64_t>(T, 1)));
  HSV_TRY(dalloc(&pb.count, 1));
  HSV_TRY_CUDA(cudaMemsetAsync(pb.count, 0, sizeof(uint32_t), stream()));
  if (T == 0) return HSV_OK;
  HSV_REQUIRE(T < (int64_t)UINT32_MAX, HSV_ERR_UNSUPPORTED, "batch plan too large");
  uint2* cand = nullptr;
  uint8_t* flag = nullptr;
  HSV_TRY(dalloc(&cand, T));
  HSV_TRY(dalloc(&flag, T));
  a.cand = cand;
  a.flag = flag;
  k_plan_candidates<<<(unsigned)((T + 255) / 256), 256, 0, stream()>>>(a);
  count_launch();
  HSV_CHECK_LAUNCH();
  size_t tb = 0;
  HSV_TRY_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, cand, flag, pb.items, pb.count, (int)T,
                                          stream()));
  void* tmp = nullptr;
  HSV_TRY(dalloc(reinterpret_cast<char**>(&tmp), tb));
  HSV_TRY_CUDA(cub::DeviceSelect::Flagged(tmp, tb, cand, flag, pb.items, pb.count, (int)T,
                                          stream()));
  count_launch();
  dfree(reinterpret_cast<char*>(tmp));
  dfree(cand);
  dfree(flag);
  return HSV_OK;
}

// Plan for the operator list `ops`; batches equal to the cached ones at the
// same position are reused.
int get_plan(const hsv_sector_s* sec, const std::vector<OpMasks>& ops,
             std::vector<std::vector<int>>& parts) {
  Plan& P = plan();
  if (P.sec != sec) {
    P.clear();
    P.sec = sec;
  }
  parts = partition(ops);
  size_t keep = 0;
  while (keep < parts.size() && keep < P.b.size()) {
    const auto& idx = parts[keep];
    const auto& pb = P.b[keep];
    bool eq = pb.m.size() == idx.size();
    for (size_t q = 0; eq && q < idx.size(); ++q) eq = same(pb.m[q], ops[idx[q]]);
    if (!eq) break;
    ++keep;
  }
  for (size_t q = keep; q < P.b.size(); ++q) { dfree(P.b[q].items); dfree(P.b[q].count); }
  P.b.resize(keep);
  for (size_t q = keep; q < parts.size(); ++q) {
    PlanBatch pb;
    for (int i : parts[q]) pb.m.push_back(ops[i]);
    HSV_TRY(build_batch(sec, pb));
    P.b.push_back(pb);
  }
  return HSV_OK;
}

}  // namespace

// Batched sweep over the rotation list (ops[i], cs[i], sn[i]) in list order:
// MODE 0 forward (psi rotated, smap maintained), 1 adjoint (reverse order;
// gradients into d_grads[i]; psi uncomputed, lam = w rotated).
int launch_bsweep(const hsv_sector_s* sec, int mode, const std::vector<OpMasks>& ops,
                  const double* cs, const double* sn, double2* psi, double2* lam, uint8_t* smap,
                  double* norm2, double* d_grads, int* err, double* err_val) {
  const int k = (int)ops.size();
  if (k == 0) return HSV_OK;
  std::vector<std::vector<int>> parts;
  HSV_TRY(get_plan(sec, ops, parts));
  Plan& P = plan();
  const int nb = (int)parts.size();
  static thread_local std::vector<BatchDev> hb;
  hb.assign(nb, BatchDev{});
  for (int q = 0; q < nb; ++q) {
    const int bq = mode == kFwd ? q : nb - 1 - q;
    BatchDev& d = hb[q];
    d.n = (int)parts[bq].size();
    d.op0 = parts[bq][0];
    for (int j = 0; j < d.n; ++j) {
      const int i = parts[bq][j];
      d.oa[j] = ops[i].oa; d.va[j] = ops[i].va; d.ob[j] = ops[i].ob; d.vb[j] = ops[i].vb;
      d.c[j] = cs[i];
      d.s[j] = sn[i];
    }
    d.items = P.b[bq].items;
    d.count = P.b[bq].count;
  }
  BatchDev* d_b = nullptr;
  HSV_TRY(dalloc(&d_b, nb));
  HSV_TRY_CUDA(cudaMemcpyAsync(d_b, hb.data(), nb * sizeof(BatchDev), cudaMemcpyHostToDevice,
                               stream()));
  static int occ[2] = {0, 0};
  if (!occ[mode]) {
    HSV_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &occ[mode], mode == kFwd ? (const void*)k_bsweep<kFwd> : (const void*)k_bsweep<kAdj>, 256,
        0));
    occ[mode] = std::max(occ[mode], 1);
  }
  int64_t max_items = 1;
  for (int q = 0; q < nb; ++q) max_items = std::max(max_items, P.b[q].n_cand);
  const int64_t resident = (int64_t)ctx().num_sms * occ[mode];
  const int64_t want = tuning().sweep_grid > 0 ? tuning().sweep_grid
                       : std::min<int64_t>(resident, (max_items + 255) / 256);
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(resident, want));
  const int NV = mode == kAdj ? 3 : 2;
  double *part = nullptr, *red = nullptr;
  HSV_TRY(dalloc(&part, (int64_t)nb * grid * kBatch * NV));
  HSV_TRY(dalloc(&red, (int64_t)k * NV));
  BSweepArgs a{};
  a.batches = d_b; a.n_batches = nb; a.n_ops = k;
  a.n_alpha = sec->n_alpha; a.n_beta = sec->n_beta; a.Nb = sec->Nb;
  a.Ra = sec->d_Ra; a.Rb = sec->d_Rb;
  a.psi = psi; a.lam = lam; a.smap = smap; a.part = part; a.red = red;
  a.norm2 = norm2; a.grads = d_grads; a.err = err; a.err_val = err_val;
  a.stats = ctx().d_stats;
  void* params[] = {&a};
  {
    ProfScope prof(mode == kFwd ? "qeb" : "adjoint");
    HSV_TRY_CUDA(cudaLaunchCooperativeKernel(
        mode == kFwd ? (const void*)k_bsweep<kFwd> : (const void*)k_bsweep<kAdj>,
        dim3((unsigned)grid), dim3(256), params, 0, stream()));
  }
  count_launch();
  dfree(d_b);
  dfree(part);
  dfree(red);
  return HSV_OK;
}

void release_sweep_plans() { plan().clear(); }

// Alpha-row occupancy flags from the structural support map (a superset of
// the nonzeros, which is all the flags promise): one warp per alpha row.
__global__ void k_smap_arow(const uint8_t* __restrict__ smap, int64_t Na, int64_t Nb,
                            uint32_t* __restrict__ flags) {
  const int64_t ra = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (ra >= Na) return;
  bool f = false;
  for (int64_t j = lane; j < Nb && !f; j += 32) f = smap[ra * Nb + j] != 0;
  f = __any_sync(0xffffffffu, f);
  if (lane == 0) flags[ra] = f ? 1u : 0u;
}

int smap_arow_async(const hsv_sector_s* sec, const uint8_t* smap, uint32_t* flags) {
  if (sec->Na == 0) return HSV_OK;
  k_smap_arow<<<(unsigned)((sec->Na * 32 + 255) / 256), 256, 0, stream()>>>(smap, sec->Na,
                                                                             sec->Nb, flags);
  count_launch();
  HSV_CHECK_LAUNCH();
  return HSV_OK;
}

}  // namespace hsv
