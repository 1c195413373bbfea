// K3 / K5: qubit-excitation (QEB) rotations, generator application and the
// fused adjoint energy+gradient sweep (svengine.py:179-281).
//
// A QEB generator T with occupied set O and virtual set V couples a source
// row b (O set, V clear) with its partner p = b ^ (O|V) (V set, O clear):
//   T|b> = +|p>,  T|p> = -|b>;  exp(theta T) is a Givens rotation per pair.
// Source rows are enumerated without scanning the sector: the alpha and beta
// halves of a source row are independent, so the pair set is the product of
// an alpha list (ranks of matching alpha strings and their partners) and a
// beta list.  One thread handles one pair and touches only 2 rows.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "hsv_common.cuh"
#include "hsv_kernels.cuh"

namespace hsv {

OpMasks compress_op(const hsv_sector_s* s, uint64_t occ, uint64_t virt) {
  return OpMasks{s->compress_a(occ), s->compress_a(virt), s->compress_b(occ),
                 s->compress_b(virt)};
}

int64_t src_count(int norb, int n, uint32_t occ, uint32_t virt) {
  const int po = __builtin_popcount(occ), pv = __builtin_popcount(virt);
  const int free_pos = norb - po - pv, ones = n - po;
  if (free_pos < 0 || ones < 0 || ones > free_pos) return 0;
  return binom_host().c[free_pos][ones];
}

// One block per spin: deterministic (rank-ascending) compaction of the
// strings in source pattern, paired with their partner ranks.
__global__ void __launch_bounds__(1024) k_pair_list(const uint32_t* __restrict__ Sa,
                                                    const uint32_t* __restrict__ Sb,
                                                    const uint32_t* __restrict__ Ra,
                                                    const uint32_t* __restrict__ Rb, int64_t Na,
                                                    int64_t Nb, OpMasks m, int2* __restrict__ la,
                                                    int2* __restrict__ lb) {
  using Scan = cub::BlockScan<int, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int base_sh;
  const bool alpha = blockIdx.x == 0;
  const uint32_t* S = alpha ? Sa : Sb;
  const uint32_t* R = alpha ? Ra : Rb;
  const int64_t N = alpha ? Na : Nb;
  const uint32_t occ = alpha ? m.oa : m.ob, virt = alpha ? m.va : m.vb;
  const uint32_t flip = occ | virt;
  int2* out = alpha ? la : lb;
  int base = 0;
  for (int64_t c0 = 0; c0 < N; c0 += 1024) {
    const int64_t i = c0 + threadIdx.x;
    uint32_t s = 0;
    int f = 0;
    if (i < N) {
      s = S[i];
      f = ((s & occ) == occ && (s & virt) == 0) ? 1 : 0;
    }
    int off, tot;
    Scan(tmp).ExclusiveSum(f, off, tot);
    if (f) out[base + off] = make_int2((int)i, (int)R[s ^ flip]);
    base += tot;
    __syncthreads();
  }
  (void)base_sh;
}

int build_pair_lists_async(const hsv_sector_s* s, const OpMasks& m, PairLists& pl) {
  pl.ca = src_count(s->norb, s->n_alpha, m.oa, m.va);
  pl.cb = src_count(s->norb, s->n_beta, m.ob, m.vb);
  if (!pl.la) HSV_TRY(dalloc(&pl.la, s->Na));
  if (!pl.lb) HSV_TRY(dalloc(&pl.lb, s->Nb));
  if (pl.ca == 0 || pl.cb == 0) return HSV_OK;
  k_pair_list<<<2, 1024, 0, stream()>>>(s->d_Sa, s->d_Sb, s->d_Ra, s->d_Rb, s->Na, s->Nb, m,
                                        pl.la, pl.lb);
  count_launch();
  HSV_CHECK_LAUNCH();
  return HSV_OK;
}

// ------------------------------------------------------------ pair kernels
enum PairMode { kRotate = 0, kGenerator = 1, kAdjoint = 2 };

struct PairArgs {
  const int2* la;
  const int2* lb;
  int64_t cb, Nb;
  double2* psi;          // rotated in place (kRotate / kAdjoint uncompute)
  double2* lam;          // kAdjoint: adjoint state (rotated in place); kGenerator: output
  const double2* src;    // kGenerator: input state
  double c, s;           // rotation (already -theta for the adjoint sweep)
  double* part;          // per-block partials
  unsigned int* counter; // last-block detection (zero on entry, reset on exit)
  double* norm2;         // kRotate: <psi|psi>; kAdjoint: <lam|lam> (in/out)
  double* result;        // kAdjoint: gradient slot
  int* err;              // set to 1 on norm drift
  double* err_val;
  int uncompute;
  uint32_t* fpsi;        // alpha-row occupancy of psi (maintained), or nullptr
  uint32_t* flam;        // alpha-row occupancy of lam (kAdjoint), or nullptr
};

__device__ __forceinline__ void givens(double2 vb, double2 vp, double c, double s, double2& nb,
                                       double2& np) {
  // exact two-term sums with separate roundings, as SparseVector.from_entries
  // merges (c*v_own) with (+-sin*v_partner) (svengine.py:219-233)
  nb.x = __dadd_rn(__dmul_rn(c, vb.x), __dmul_rn(-s, vp.x));
  nb.y = __dadd_rn(__dmul_rn(c, vb.y), __dmul_rn(-s, vp.y));
  np.x = __dadd_rn(__dmul_rn(c, vp.x), __dmul_rn(s, vb.x));
  np.y = __dadd_rn(__dmul_rn(c, vp.y), __dmul_rn(s, vb.y));
}

// Block partials then a deterministic last-block reduction (fixed order).
template <int NV>
__device__ bool last_block_sum(double (&v)[NV], double* __restrict__ part,
                               unsigned int* counter, double (&tot)[NV]) {
  __shared__ double sh[NV][32];
  __shared__ bool amlast;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  const unsigned nblocks = gridDim.x * gridDim.y;
  const unsigned bid = blockIdx.y * gridDim.x + blockIdx.x;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    double x = warp_sum(v[j]);
    if (l == 0) sh[j][w] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      double x = 0.0;
      for (int q = 0; q < nw; ++q) x += sh[j][q];
      part[(int64_t)bid * NV + j] = x;
    }
    __threadfence();
    amlast = atomicAdd(counter, 1u) == nblocks - 1;
  }
  __syncthreads();
  if (!amlast) return false;
  __threadfence();
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    double x = 0.0;
    for (unsigned i = threadIdx.x; i < nblocks; i += blockDim.x) x += __ldcg(part + (int64_t)i * NV + j);
    x = warp_sum(x);
    __syncthreads();
    if (l == 0) sh[j][w] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int q = 0; q < nw; ++q) t += sh[j][q];
      tot[j] = t;
    }
  }
  if (threadIdx.x == 0) *counter = 0u;
  return true;
}

template <int MODE>
__global__ void __launch_bounds__(256) k_pairs(const PairArgs a) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int2 A = a.la[blockIdx.y];
  double v[MODE == kAdjoint ? 3 : 2];
#pragma unroll
  for (int q = 0; q < (MODE == kAdjoint ? 3 : 2); ++q) v[q] = 0.0;
  // Skip alpha-row pairs that are entirely zero (results unchanged: all terms
  // would be exact zeros); a nonzero row makes both rows of the pair nonzero.
  bool active = true;
  if (MODE != kGenerator) {
    const bool ap = !a.fpsi || a.fpsi[A.x] || a.fpsi[A.y];
    const bool al = MODE == kAdjoint && (!a.flam || a.flam[A.x] || a.flam[A.y]);
    active = ap || al;
    __syncthreads();   // every thread has read the flags before thread 0 updates them
    if (threadIdx.x == 0 && blockIdx.x == 0) {
      if (a.fpsi && ap && (MODE == kRotate || a.uncompute)) { a.fpsi[A.x] = 1u; a.fpsi[A.y] = 1u; }
      if (MODE == kAdjoint && a.flam && al) { a.flam[A.x] = 1u; a.flam[A.y] = 1u; }
    }
  }
  if (j < a.cb && active) {
    const int2 B = a.lb[j];
    const int64_t ib = (int64_t)A.x * a.Nb + B.x;   // source row
    const int64_t ip = (int64_t)A.y * a.Nb + B.y;   // partner (target pattern)
    if (MODE == kRotate) {
      const double2 vb = a.psi[ib], vp = a.psi[ip];
      double2 nb, np;
      givens(vb, vp, a.c, a.s, nb, np);
      a.psi[ib] = nb;
      a.psi[ip] = np;
      v[0] = vb.x * vb.x + vb.y * vb.y + vp.x * vp.x + vp.y * vp.y;
      v[1] = nb.x * nb.x + nb.y * nb.y + np.x * np.x + np.y * np.y;
    } else if (MODE == kGenerator) {
      // source b -> +v_b at p; target p -> -v_p at b (svengine.py:196-203)
      const double2 vb = a.src[ib], vp = a.src[ip];
      a.lam[ip] = vb;
      a.lam[ib] = make_double2(-vp.x, -vp.y);
    } else {
      const double2 pb = a.psi[ib], pp = a.psi[ip];
      const double2 lb = a.lam[ib], lp = a.lam[ip];
      // <lam| T psi>: (T psi)_b = -psi_p, (T psi)_p = +psi_b
      v[0] = (lp.x * pb.x + lp.y * pb.y) - (lb.x * pp.x + lb.y * pp.y);
      double2 nb, np;
      givens(lb, lp, a.c, a.s, nb, np);
      a.lam[ib] = nb;
      a.lam[ip] = np;
      v[1] = lb.x * lb.x + lb.y * lb.y + lp.x * lp.x + lp.y * lp.y;
      v[2] = nb.x * nb.x + nb.y * nb.y + np.x * np.x + np.y * np.y;
      if (a.uncompute) {
        double2 qb, qp;
        givens(pb, pp, a.c, a.s, qb, qp);
        a.psi[ib] = qb;
        a.psi[ip] = qp;
      }
    }
  }
  if (MODE == kGenerator) return;
  constexpr int NV = MODE == kAdjoint ? 3 : 2;
  double tot[NV];
  if (last_block_sum<NV>(v, a.part, a.counter, tot) && threadIdx.x == 0) {
    const double dold = MODE == kAdjoint ? tot[1] : tot[0];
    const double dnew = MODE == kAdjoint ? tot[2] : tot[1];
    const double n2 = *a.norm2;
    const double n2new = n2 - dold + dnew;
    const double nrm = sqrt(fmax(n2, 0.0));
    const double drift = fabs(sqrt(fmax(n2new, 0.0)) - nrm);
    if (drift > kNormDriftTol * fmax(1.0, nrm)) {   // svengine.py:234-236
      if (atomicExch(a.err, 1) == 0) *a.err_val = drift;
    }
    *a.norm2 = n2new;
    if (MODE == kAdjoint) *a.result = 2.0 * tot[0];
  }
}

template <int MODE>
static int launch_pairs(const PairLists& pl, PairArgs a, int64_t* nblocks_out = nullptr) {
  if (pl.ca == 0 || pl.cb == 0) {
    if (nblocks_out) *nblocks_out = 0;
    return HSV_OK;
  }
  a.la = pl.la;
  a.lb = pl.lb;
  a.cb = pl.cb;
  dim3 grid((unsigned)((pl.cb + 255) / 256), (unsigned)pl.ca);
  HSV_REQUIRE(pl.ca <= 65535, HSV_ERR_UNSUPPORTED, "alpha pair list too long (%lld)",
              (long long)pl.ca);
  if (nblocks_out) *nblocks_out = (int64_t)grid.x * grid.y;
  ProfScope prof(MODE == kRotate ? "qeb" : MODE == kAdjoint ? "adjoint" : "generator");
  k_pairs<MODE><<<grid, 256, 0, stream()>>>(a);
  count_launch();
  HSV_CHECK_LAUNCH();
  return HSV_OK;
}

static int64_t max_pair_blocks(const hsv_sector_s* s) {
  return ((s->Nb + 255) / 256) * std::max<int64_t>(1, s->Na);
}

// Scratch shared by the pair launches of one API call.
struct PairScratch {
  double* part = nullptr;
  unsigned int* counter = nullptr;
  int* err = nullptr;
  double* err_val = nullptr;
  int init(const hsv_sector_s* s, int nv) {
    HSV_TRY(dalloc(&part, max_pair_blocks(s) * nv));
    HSV_TRY(dalloc(&counter, 1));
    HSV_TRY(dalloc(&err, 1));
    HSV_TRY(dalloc(&err_val, 1));
    HSV_TRY_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned), stream()));
    HSV_TRY_CUDA(cudaMemsetAsync(err, 0, sizeof(int), stream()));
    HSV_TRY_CUDA(cudaMemsetAsync(err_val, 0, sizeof(double), stream()));
    return HSV_OK;
  }
  void release() { dfree(part); dfree(counter); dfree(err); dfree(err_val); }
  int check() {
    int h_err = 0;
    double h_val = 0.0;
    HSV_TRY_CUDA(cudaMemcpyAsync(&h_err, err, sizeof(int), cudaMemcpyDeviceToHost, stream()));
    HSV_TRY_CUDA(cudaMemcpyAsync(&h_val, err_val, sizeof(double), cudaMemcpyDeviceToHost, stream()));
    HSV_TRY(stream_sync());
    HSV_REQUIRE(!h_err, HSV_ERR_NORM_DRIFT, "norm drift %.3e in qeb exponential", h_val);
    return HSV_OK;
  }
};

// ------------------------------------------------------------- fused sweep
// All k rotations of a forward (kRotate) or adjoint (kAdjoint) sweep in ONE
// cooperative launch: a persistent grid walks op after op, separated by a
// grid barrier, instead of 2k launches (pair-list build + pair kernel per op)
// whose host cost dominates at ADAPT sizes.
//   phase 0: the pair lists of every op, built in parallel: the i-th source
//            string of an op's alpha (beta) half is unranked directly
//            (combinatorial number system over the free orbitals; ascending
//            order = the rank order k_pair_list produces);
//   phase 1: per op, work item = (alpha pair y, 256-wide beta chunk x) =
//            block (x, y) of k_pairs; grid barrier between ops;
//   phase 2: per-op totals (one op per block) and the norm chain.
// Every reduction replays last_block_sum's order, so results are
// bit-identical to the per-op launch path (tests/test_gpu_sweep.py).
struct SweepOp {
  uint32_t oa, va, ob, vb;
  int32_t ca, cb, nx, la_off;   // la_off / lb_off: offsets of the op's lists
  int32_t lb_off, pad;
  double c, s;
};

struct SweepArgs {
  const SweepOp* ops;
  int n_ops;
  int norb, n_alpha, n_beta;
  int64_t Nb;
  const uint32_t* Ra;
  const uint32_t* Rb;
  const int64_t* binom;
  int2* lists;           // phase-0 pair lists {rank, partner rank}
  double2* psi;
  double2* lam;
  uint32_t* fpsi;
  uint32_t* flam;
  double* part;          // [chunk][max_items][NV] per-op block partials
  int64_t part_stride;   // max_items * NV
  int chunk;             // ops per reduction chunk
  double* red;           // [n_ops][NV] per-op totals
  double* norm2;
  double* grads;         // kAdjoint: gradient of op i at grads[i]
  int* err;
  double* err_val;
  uint8_t* smap;         // kRotate: structural support map (see hsv_state_s), or nullptr
};

// Grid-wide barrier of the cooperative launch (measured 1.2 us at 2 blocks/SM,
// 2.0 us at 6 blocks/SM; a hand-rolled atomic/spin barrier was 1.7x slower).
__device__ __forceinline__ void grid_barrier() { cooperative_groups::this_grid().sync(); }

// i-th string (ascending) with `occ` set, `virt` clear and `ones` electrons on
// the remaining orbitals of `nmask`; binomials from a 32-bit table bt[n*32+k].
__device__ __forceinline__ uint32_t unrank_string(int i, uint32_t occ, uint32_t virt,
                                                  uint32_t nmask, int ones, const int* bt) {
  uint32_t fm = nmask & ~(occ | virt);
  uint32_t s = occ;
  for (int p = __popc(fm) - 1; p >= 0 && ones > 0; --p) {
    const int pos = 31 - __clz(fm);
    fm &= ~(1u << pos);
    const int c = ones <= p ? bt[p * 32 + ones] : 0;   // strings with this orbital empty first
    if (i >= c) {
      s |= 1u << pos;
      i -= c;
      --ones;
    }
  }
  return s;
}

template <int MODE>
__global__ void __launch_bounds__(256) k_sweep(const SweepArgs a) {
  constexpr int NV = MODE == kAdjoint ? 3 : 2;
  __shared__ double sh[NV][8];
  __shared__ int bt[33 * 32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const uint32_t nmask = a.norb >= 32 ? 0xffffffffu : ((1u << a.norb) - 1u);
  for (int i = threadIdx.x; i < 33 * 32; i += blockDim.x) {
    const int n = i >> 5, k = i & 31;
    bt[i] = (int)dbinom(a.binom, n, k);
  }
  __syncthreads();
  // phase 0: pair lists of all ops
  {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    for (int oi = 0; oi < a.n_ops; ++oi) {
      const SweepOp o = a.ops[oi];
      const int ones_a = a.n_alpha - __popc(o.oa), ones_b = a.n_beta - __popc(o.ob);
      for (int e = tid; e < o.ca + o.cb; e += nth) {
        const bool al = e < o.ca;
        const uint32_t oc = al ? o.oa : o.ob, vi = al ? o.va : o.vb;
        const uint32_t s = unrank_string(al ? e : e - o.ca, oc, vi, nmask, al ? ones_a : ones_b, bt);
        const uint32_t* R = al ? a.Ra : a.Rb;
        a.lists[(al ? o.la_off : o.lb_off - o.ca) + e] =
            make_int2((int)__ldg(R + s), (int)__ldg(R + (s ^ (oc | vi))));
      }
    }
  }
  grid_barrier();
  for (int c0 = 0; c0 < a.n_ops; c0 += a.chunk) {
  const int c1 = min(a.n_ops, c0 + a.chunk);
  for (int op = c0; op < c1; ++op) {
    const int oi = MODE == kRotate ? op : a.n_ops - 1 - op;
    const SweepOp o = a.ops[oi];
    const int uncompute = MODE == kAdjoint && oi > 0;
    double* part = a.part + (op - c0) * a.part_stride;
    const int items = o.ca * o.nx;
    const int2* la = a.lists + o.la_off;
    const int2* lb = a.lists + o.lb_off;
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      const int y = it / o.nx;
      const int xc = it - y * o.nx;
      const int j = xc * 256 + threadIdx.x;
      const int2 A = la[y];
      const int2 B = j < o.cb ? lb[j] : make_int2(0, 0);
      const bool ap = !a.fpsi || a.fpsi[A.x] || a.fpsi[A.y];
      const bool al = MODE == kAdjoint && (!a.flam || a.flam[A.x] || a.flam[A.y]);
      __syncthreads();   // flags read by every thread before thread 0 updates them
      if (threadIdx.x == 0 && xc == 0) {
        if (a.fpsi && ap && (MODE == kRotate || uncompute)) { a.fpsi[A.x] = 1u; a.fpsi[A.y] = 1u; }
        if (MODE == kAdjoint && a.flam && al) { a.flam[A.x] = 1u; a.flam[A.y] = 1u; }
      }
      if (!(ap || al)) {   // whole item inactive: its partials are exact zeros
        if (threadIdx.x == 0)
          for (int q = 0; q < NV; ++q) part[(int64_t)it * NV + q] = 0.0;
        continue;
      }
      double v[NV];
#pragma unroll
      for (int q = 0; q < NV; ++q) v[q] = 0.0;
      if (j < o.cb) {
        const int64_t ib = (int64_t)A.x * a.Nb + B.x;   // source row
        const int64_t ip = (int64_t)A.y * a.Nb + B.y;   // partner
        if (MODE == kRotate) {
          const double2 vb = a.psi[ib], vp = a.psi[ip];
          double2 nb, np;
          givens(vb, vp, o.c, o.s, nb, np);
          a.psi[ib] = nb;
          a.psi[ip] = np;
          if (a.smap) {   // structural support: either side marked -> both marked
            if (a.smap[ib] | a.smap[ip]) { a.smap[ib] = 1; a.smap[ip] = 1; }
          }
          v[0] = vb.x * vb.x + vb.y * vb.y + vp.x * vp.x + vp.y * vp.y;
          v[1] = nb.x * nb.x + nb.y * nb.y + np.x * np.x + np.y * np.y;
        } else {
          const double2 pb = a.psi[ib], pp = a.psi[ip];
          const double2 lb2 = a.lam[ib], lp = a.lam[ip];
          v[0] = (lp.x * pb.x + lp.y * pb.y) - (lb2.x * pp.x + lb2.y * pp.y);
          double2 nb, np;
          givens(lb2, lp, o.c, -o.s, nb, np);
          a.lam[ib] = nb;
          a.lam[ip] = np;
          v[1] = lb2.x * lb2.x + lb2.y * lb2.y + lp.x * lp.x + lp.y * lp.y;
          v[NV - 1] = nb.x * nb.x + nb.y * nb.y + np.x * np.x + np.y * np.y;
          if (uncompute) {
            double2 qb, qp;
            givens(pb, pp, o.c, -o.s, qb, qp);
            a.psi[ib] = qb;
            a.psi[ip] = qp;
          }
        }
      }
#pragma unroll
      for (int q = 0; q < NV; ++q) {   // block partial, last_block_sum order
        const double x = warp_sum(v[q]);
        if (l == 0) sh[q][w] = x;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          double x = 0.0;
          for (int k = 0; k < 8; ++k) x += sh[q][k];
          part[(int64_t)it * NV + q] = x;
        }
      }
    }
    grid_barrier();   // op i+1 reads rows and flags op i wrote
  }
  // phase 2: per-op totals of the chunk, one op per block (last_block_sum order)
  for (int op = c0 + blockIdx.x; op < c1; op += gridDim.x) {
    const int oi = MODE == kRotate ? op : a.n_ops - 1 - op;
    const int items = a.ops[oi].ca * a.ops[oi].nx;
    const double* part = a.part + (op - c0) * a.part_stride;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double x = 0.0;
      for (int i = threadIdx.x; i < items; i += blockDim.x) x += __ldcg(part + (int64_t)i * NV + q);
      x = warp_sum(x);
      __syncthreads();
      if (l == 0) sh[q][w] = x;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += sh[q][k];
        a.red[(int64_t)op * NV + q] = t;
      }
    }
  }
  grid_barrier();   // totals visible; partial buffers free for the next chunk
  if (blockIdx.x == 0 && threadIdx.x == 0) {   // norm chain in sweep order
    double n2 = *a.norm2;
    for (int op = c0; op < c1; ++op) {
      const int oi = MODE == kRotate ? op : a.n_ops - 1 - op;
      const double* tot = a.red + (int64_t)op * NV;
      const double dold = MODE == kAdjoint ? __ldcg(tot + 1) : __ldcg(tot);
      const double dnew = MODE == kAdjoint ? __ldcg(tot + 2) : __ldcg(tot + 1);
      const double n2new = n2 - dold + dnew;
      const double nrm = sqrt(fmax(n2, 0.0));
      const double drift = fabs(sqrt(fmax(n2new, 0.0)) - nrm);
      if (drift > kNormDriftTol * fmax(1.0, nrm)) {   // svengine.py:234-236
        if (atomicExch(a.err, 1) == 0) *a.err_val = drift;
      }
      n2 = n2new;
      if (MODE == kAdjoint)
        a.grads[oi] = a.ops[oi].ca > 0 ? 2.0 * __ldcg(tot) : 0.0;
    }
    *a.norm2 = n2;
  }
  }
}

// Launch one fused sweep over host op descriptors (MODE kRotate: forward order,
// kAdjoint: reverse order, gradients to d_grads).
template <int MODE>
static int launch_sweep(const hsv_sector_s* sec, const std::vector<SweepOp>& ops_in, double2* psi,
                        uint32_t* fpsi, double2* lam, uint32_t* flam, double* norm2,
                        double* d_grads, PairScratch& sc, uint8_t* smap = nullptr) {
  if (ops_in.empty()) return HSV_OK;
  constexpr int NV = MODE == kAdjoint ? 3 : 2;
  static thread_local std::vector<SweepOp> ops;
  ops = ops_in;
  int64_t max_items = 1, n_list = 0;
  for (SweepOp& o : ops) {
    max_items = std::max<int64_t>(max_items, (int64_t)o.ca * o.nx);
    o.la_off = (int32_t)n_list;
    o.lb_off = (int32_t)(n_list + o.ca);
    n_list += (int64_t)o.ca + o.cb;
  }
  HSV_REQUIRE(n_list < INT32_MAX && max_items < INT32_MAX, HSV_ERR_UNSUPPORTED,
              "sweep pair lists too long");
  int2* lists = nullptr;
  HSV_TRY(dalloc(&lists, std::max<int64_t>(n_list, 1)));
  // ops per reduction chunk: partials of a chunk stay within 64 MB
  const int64_t chunk = std::max<int64_t>(
      1, std::min<int64_t>((int64_t)ops.size(), ((int64_t)8 << 20) / (max_items * NV)));
  SweepOp* d_ops = nullptr;
  double *part = nullptr, *red = nullptr;
  HSV_TRY(dalloc(&d_ops, ops.size()));
  HSV_TRY(dalloc(&part, chunk * max_items * NV));
  HSV_TRY(dalloc(&red, (int64_t)ops.size() * NV));
  HSV_TRY_CUDA(cudaMemcpyAsync(d_ops, ops.data(), ops.size() * sizeof(SweepOp),
                               cudaMemcpyHostToDevice, stream()));
  SweepArgs a{};
  a.ops = d_ops; a.n_ops = (int)ops.size();
  a.norb = sec->norb; a.n_alpha = sec->n_alpha; a.n_beta = sec->n_beta;
  a.Nb = sec->Nb; a.Ra = sec->d_Ra; a.Rb = sec->d_Rb; a.binom = sec->d_binom; a.lists = lists;
  a.psi = psi; a.lam = lam; a.fpsi = fpsi; a.flam = flam;
  a.part = part; a.part_stride = max_items * NV; a.chunk = (int)chunk; a.red = red;
  a.norm2 = norm2; a.grads = d_grads; a.err = sc.err; a.err_val = sc.err_val;
  a.smap = smap;
  static int occ[3] = {0, 0, 0};
  if (!occ[MODE]) {
    HSV_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[MODE], k_sweep<MODE>, 256, 0));
    occ[MODE] = std::max(occ[MODE], 1);
  }
  // Full residency only when the ops carry enough rows to need the memory
  // parallelism; small sweeps are barrier bound (cheaper with fewer blocks).
  const int64_t resident = (int64_t)ctx().num_sms * occ[MODE];
  const int64_t want = tuning().sweep_grid > 0 ? tuning().sweep_grid
                       : max_items >= 8 * resident ? resident
                                                   : std::min<int64_t>(max_items, 2 * ctx().num_sms);
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(resident, want));
  void* params[] = {&a};
  {
    ProfScope prof(MODE == kRotate ? "qeb" : "adjoint");
    HSV_TRY_CUDA(cudaLaunchCooperativeKernel((const void*)k_sweep<MODE>, dim3((unsigned)grid),
                                             dim3(256), params, 0, stream()));
  }
  count_launch();
  dfree(d_ops);
  dfree(part);
  dfree(red);
  dfree(lists);
  return HSV_OK;
}

static SweepOp sweep_op(const hsv_sector_s* sec, uint64_t occ, uint64_t virt, double c, double s) {
  const OpMasks m = compress_op(sec, occ, virt);
  SweepOp o{};
  o.oa = m.oa; o.va = m.va; o.ob = m.ob; o.vb = m.vb;
  o.ca = (int32_t)src_count(sec->norb, sec->n_alpha, m.oa, m.va);
  o.cb = (int32_t)src_count(sec->norb, sec->n_beta, m.ob, m.vb);
  o.nx = (int32_t)((o.cb + 255) / 256);
  if (o.ca == 0 || o.cb == 0) o.ca = o.cb = o.nx = 0;
  o.c = c; o.s = s;
  return o;
}

}  // namespace hsv

using namespace hsv;

extern "C" {

int hsv_apply_qeb(hsv_state in, hsv_state out, uint64_t occ, uint64_t virt, double c, double s) {
  HSV_REQUIRE(in && out && in->sec == out->sec, HSV_ERR_INVALID, "dimension mismatch");
  HSV_REQUIRE((occ & virt) == 0 && occ && virt, HSV_ERR_INVALID, "excitation indices must be distinct");
  if (out != in) {
    HSV_TRY_CUDA(cudaMemcpyAsync(out->d_amp, in->d_amp, in->sec->dim * sizeof(double2),
                                 cudaMemcpyDeviceToDevice, stream()));
    HSV_TRY_CUDA(cudaMemcpyAsync(out->d_norm2, in->d_norm2, sizeof(double),
                                 cudaMemcpyDeviceToDevice, stream()));
    out->norm2_valid = in->norm2_valid;
    HSV_TRY_CUDA(cudaMemcpyAsync(out->d_arow, in->d_arow, in->sec->Na * sizeof(uint32_t),
                                 cudaMemcpyDeviceToDevice, stream()));
    out->arow_valid = in->arow_valid;
    out->dense_hint = in->dense_hint;
  }
  if (c == 1.0 && s == 0.0) return stream_sync();   // theta == 0 returns the input (svengine.py:212)
  if (!out->norm2_valid) HSV_TRY(state_norm2_async(out));
  const hsv_sector_s* sec = out->sec;
  PairLists pl;
  PairScratch sc;
  HSV_TRY(sc.init(sec, 2));
  HSV_TRY(build_pair_lists_async(sec, compress_op(sec, occ, virt), pl));
  PairArgs a{};
  a.Nb = sec->Nb; a.psi = out->d_amp; a.c = c; a.s = s;
  a.part = sc.part; a.counter = sc.counter; a.norm2 = out->d_norm2;
  a.err = sc.err; a.err_val = sc.err_val;
  HSV_TRY(state_arow_async(out));
  a.fpsi = out->d_arow;                      // maintained by the kernel
  HSV_TRY(launch_pairs<kRotate>(pl, a));
  int rc = sc.check();
  dfree(pl.la); dfree(pl.lb);
  sc.release();
  out->norm2_valid = true;
  out->smap_valid = false;
  out->dense_hint = false;
  return rc;
}

int hsv_apply_generator(hsv_state in, hsv_state out, uint64_t occ, uint64_t virt) {
  HSV_REQUIRE(in && out && in->sec == out->sec, HSV_ERR_INVALID, "dimension mismatch");
  HSV_REQUIRE(in != out, HSV_ERR_INVALID, "hsv_apply_generator: output must not alias input");
  HSV_REQUIRE((occ & virt) == 0 && occ && virt, HSV_ERR_INVALID, "excitation indices must be distinct");
  const hsv_sector_s* sec = in->sec;
  HSV_TRY(state_fill_zero_async(out));
  PairLists pl;
  HSV_TRY(build_pair_lists_async(sec, compress_op(sec, occ, virt), pl));
  PairArgs a{};
  a.Nb = sec->Nb; a.src = in->d_amp; a.lam = out->d_amp;
  HSV_TRY(launch_pairs<kGenerator>(pl, a));
  dfree(pl.la); dfree(pl.lb);
  out->norm2_valid = false;
  out->arow_valid = false;
  out->smap_valid = false;
  out->dense_hint = false;
  return stream_sync();
}

static int check_eg_args(hsv_op op, const uint64_t* occ, const uint64_t* virt, const double* cs,
                         const double* sn, int64_t k) {
  HSV_REQUIRE(op && (k == 0 || (occ && virt && cs && sn)), HSV_ERR_INVALID, "null argument");
  for (int64_t i = 0; i < k; ++i)
    HSV_REQUIRE((occ[i] & virt[i]) == 0 && occ[i] && virt[i], HSV_ERR_INVALID,
                "excitation indices must be distinct");
  return HSV_OK;
}

// psi <- prod_i exp(theta_i T_i)|hf> on all rows, occupancy flags and norm
// maintained (fused sweep, or one launch per rotation); drift errors are left
// in `sc` for the caller's sc.check().
static int forward_psi(const hsv_sector_s* sec, uint64_t hf_key, const uint64_t* occ,
                       const uint64_t* virt, const double* cs, const double* sn, int64_t k,
                       hsv_state psi, PairScratch& sc, PairLists& pl, bool want_smap = false) {
  const uint32_t sa = sec->compress_a(hf_key), sb = sec->compress_b(hf_key);
  HSV_REQUIRE((sec->n_qubits >= 64 || (hf_key >> sec->n_qubits) == 0) && sec->Ra[sa] != ~0u &&
                  sec->Rb[sb] != ~0u,
              HSV_ERR_SECTOR, "configuration %#llx is outside the basis sector",
              (unsigned long long)hf_key);
  // psi <- |hf>, flags = HF alpha row only
  HSV_TRY(state_fill_zero_async(psi));
  static thread_local double2 one;
  static thread_local double n2one;
  static thread_local uint32_t one_flag;
  one = make_double2(1.0, 0.0);
  n2one = 1.0;
  one_flag = 1u;
  const int64_t hidx = (int64_t)sec->Ra[sa] * sec->Nb + sec->Rb[sb];
  HSV_TRY_CUDA(cudaMemcpyAsync(psi->d_amp + hidx, &one, sizeof(double2), cudaMemcpyHostToDevice,
                               stream()));
  HSV_TRY_CUDA(cudaMemcpyAsync(psi->d_norm2, &n2one, sizeof(double), cudaMemcpyHostToDevice,
                               stream()));
  HSV_TRY_CUDA(cudaMemcpyAsync(psi->d_arow + sec->Ra[sa], &one_flag, sizeof(uint32_t),
                               cudaMemcpyHostToDevice, stream()));
  if (tuning().sweep == 2) {   // batched sweep (hsv_sweep.cu) + the plan's support map
    if (!psi->d_smap) HSV_TRY(dalloc(&psi->d_smap, sec->dim));
    static thread_local std::vector<OpMasks> ops;
    ops.clear();
    for (int64_t i = 0; i < k; ++i) ops.push_back(compress_op(sec, occ[i], virt[i]));
    bool used = false;
    HSV_TRY(launch_bsweep(sec, 0, hidx, ops, cs, sn, psi->d_amp, nullptr, psi->d_smap,
                          psi->d_norm2, nullptr, sc.err, sc.err_val, &used));
    HSV_TRY(smap_arow_async(sec, psi->d_smap, psi->d_arow));
    psi->norm2_valid = psi->arow_valid = psi->smap_valid = true;
    psi->dense_hint = false;
    (void)want_smap;
    return HSV_OK;
  }
  // structural support map: HF row only, grown by every rotation of the sweep
  uint8_t* smap = nullptr;
  if (want_smap && tuning().sweep) {
    if (!psi->d_smap) HSV_TRY(dalloc(&psi->d_smap, sec->dim));
    smap = psi->d_smap;
    static thread_local uint8_t one_b;
    one_b = 1;
    HSV_TRY_CUDA(cudaMemsetAsync(smap, 0, sec->dim, stream()));
    HSV_TRY_CUDA(cudaMemcpyAsync(smap + hidx, &one_b, 1, cudaMemcpyHostToDevice, stream()));
  }
  if (tuning().sweep) {
    static thread_local std::vector<SweepOp> ops;
    ops.clear();
    for (int64_t i = 0; i < k; ++i)
      if (!(cs[i] == 1.0 && sn[i] == 0.0)) ops.push_back(sweep_op(sec, occ[i], virt[i], cs[i], sn[i]));
    HSV_TRY(launch_sweep<kRotate>(sec, ops, psi->d_amp, psi->d_arow, nullptr, nullptr,
                                  psi->d_norm2, nullptr, sc, smap));
  } else {
    for (int64_t i = 0; i < k; ++i) {
      if (cs[i] == 1.0 && sn[i] == 0.0) continue;
      HSV_TRY(build_pair_lists_async(sec, compress_op(sec, occ[i], virt[i]), pl));
      PairArgs a{};
      a.Nb = sec->Nb; a.psi = psi->d_amp; a.c = cs[i]; a.s = sn[i];
      a.part = sc.part; a.counter = sc.counter; a.norm2 = psi->d_norm2;
      a.err = sc.err; a.err_val = sc.err_val; a.fpsi = psi->d_arow;
      HSV_TRY(launch_pairs<kRotate>(pl, a));
    }
  }
  psi->norm2_valid = psi->arow_valid = true;
  psi->smap_valid = smap != nullptr;
  psi->dense_hint = false;
  return HSV_OK;
}

// Reads (synchronously) and clears the forward sweep's drift flags left on psi.
static int take_pending_drift(hsv_state psi) {
  int h_err = 0;
  double h_val = 0.0;
  HSV_TRY_CUDA(cudaMemcpyAsync(&h_err, psi->d_pend_err, sizeof(int), cudaMemcpyDeviceToHost,
                               stream()));
  HSV_TRY_CUDA(cudaMemcpyAsync(&h_val, psi->d_pend_val, sizeof(double), cudaMemcpyDeviceToHost,
                               stream()));
  HSV_TRY(stream_sync());
  dfree(psi->d_pend_err);
  dfree(psi->d_pend_val);
  psi->d_pend_err = nullptr;
  psi->d_pend_val = nullptr;
  HSV_REQUIRE(!h_err, HSV_ERR_NORM_DRIFT, "norm drift %.3e in qeb exponential", h_val);
  return HSV_OK;
}

// Phase 1 of the adjoint sweep: psi <- prod_i exp(theta_i T_i)|hf> (all rows;
// occupancy flags and norm maintained), w rows [a_lo, a_hi) <- (H psi) rows.
int hsv_eg_forward_async(hsv_op op, uint64_t hf_key, const uint64_t* occ, const uint64_t* virt,
                         const double* cs, const double* sn, int64_t k, int64_t a_lo,
                         int64_t a_hi, hsv_state psi, hsv_state w) {
  HostProf hp("eg_fwd");
  HSV_TRY(check_eg_args(op, occ, virt, cs, sn, k));
  HSV_REQUIRE(psi && w && psi != w && psi->sec == op->sec && w->sec == op->sec,
              HSV_ERR_INVALID, "bad state argument");
  const hsv_sector_s* sec = op->sec;
  HSV_REQUIRE(0 <= a_lo && a_lo <= a_hi && a_hi <= sec->Na, HSV_ERR_INVALID, "bad alpha-row range");
  PairScratch sc;
  HSV_TRY(sc.init(sec, 2));
  PairLists pl;
  // K1r: the adjoint sweep reads w = H psi only on the structural support of
  // psi (rotation pairs never straddle it), so w is computed there
  // (the support map closes over every rotation, theta = 0 included, in the
  // batched sweep only)
  const bool rows_only = tuning().restrict_rows != 0 && tuning().sweep == 2;
  {
    HostProf hf("fwd_psi");
    HSV_TRY(forward_psi(sec, hf_key, occ, virt, cs, sn, k, psi, sc, pl, rows_only));
  }
  int64_t used = 0;
  HostProf hk("k1r_launch");
  if (rows_only && psi->smap_valid)
    HSV_TRY(launch_apply_rows(op, psi->d_amp, w->d_amp, a_lo, a_hi, psi->d_arow, psi->d_smap,
                              sweep_plan_support(sec), sweep_plan_version(sec)));
  else
    HSV_TRY(launch_apply(op, psi->d_amp, w->d_amp, nullptr, a_lo, a_hi, 0.0, 0, &used,
                         psi->d_arow, &psi->dense_hint));
  w->norm2_valid = w->arow_valid = false;
  w->dense_hint = false;
  // drift errors are read by hsv_eg_backward (no host sync here); an unread
  // earlier report on psi is checked first
  int rc = HSV_OK;
  if (psi->d_pend_err) rc = take_pending_drift(psi);
  psi->d_pend_err = sc.err;
  psi->d_pend_val = sc.err_val;
  sc.err = nullptr;
  sc.err_val = nullptr;
  dfree(pl.la); dfree(pl.lb);
  sc.release();
  return rc;
}

// The ansatz state alone (apply_ansatz, svengine.py:240-244): one fused sweep
// instead of one rotation call (and host sync) per operator.
int hsv_ansatz_state(hsv_sector s, uint64_t hf_key, const uint64_t* occ, const uint64_t* virt,
                     const double* cs, const double* sn, int64_t k, hsv_state psi) {
  HSV_REQUIRE(s && psi && psi->sec == s, HSV_ERR_INVALID, "bad state argument");
  HSV_REQUIRE(k == 0 || (occ && virt && cs && sn), HSV_ERR_INVALID, "null argument");
  for (int64_t i = 0; i < k; ++i)
    HSV_REQUIRE((occ[i] & virt[i]) == 0 && occ[i] && virt[i], HSV_ERR_INVALID,
                "excitation indices must be distinct");
  PairScratch sc;
  HSV_TRY(sc.init(s, 2));
  PairLists pl;
  HSV_TRY(forward_psi(s, hf_key, occ, virt, cs, sn, k, psi, sc, pl));
  // a support far past the push path's source budget: the next H application
  // goes straight to the pull / assembled path (and the overlapped screen)
  // instead of first counting sources to find out
  if (psi->smap_valid && sweep_plan_support(s) > 65536) psi->dense_hint = true;
  const int rc = sc.check();   // synchronizes; drift errors surface here
  dfree(pl.la); dfree(pl.lb);
  sc.release();
  return rc;
}

// Phase 2: E = Re <psi|w> (w complete on every row) and the backward sweep
// (svengine.py:276-280), uncomputing psi instead of storing k+1 states.
// psi and w are consumed (rotated in place).
int hsv_eg_backward(hsv_op op, hsv_state psi, hsv_state w, const uint64_t* occ,
                    const uint64_t* virt, const double* cs, const double* sn, int64_t k,
                    double* energy, double* grads) {
  HostProf hp("eg_bwd");
  HSV_TRY(check_eg_args(op, occ, virt, cs, sn, k));
  HSV_REQUIRE(energy && (k == 0 || grads), HSV_ERR_INVALID, "null output");
  HSV_REQUIRE(psi && w && psi != w && psi->sec == op->sec && w->sec == op->sec,
              HSV_ERR_INVALID, "bad state argument");
  const hsv_sector_s* sec = op->sec;
  // [0, k): gradients, [k, k + 2): <psi|w>; one copy back at the end (no sync here)
  double* d_grad = nullptr;
  HSV_TRY(dalloc(&d_grad, k + 2));
  // E = <psi|w>, and <lam|lam> (lam = w) for the drift checks: one pass
  if (k > 0) HSV_TRY(state_dot_norm2_async(psi, w, d_grad + k));
  else HSV_TRY(state_dot_async(psi, w, d_grad + k));
  if (tuning().sweep == 0) {   // flags of the per-rotation launches
    HSV_TRY(state_arow_async(psi));
    HSV_TRY(state_arow_async(w));
  }
  PairScratch sc;
  HSV_TRY(sc.init(sec, 3));
  PairLists pl;
  bool batched = false;
  if (tuning().sweep == 2 && psi->smap_valid) {   // psi came from the batched forward sweep
    static thread_local std::vector<OpMasks> bops;
    bops.clear();
    for (int64_t i = 0; i < k; ++i) bops.push_back(compress_op(sec, occ[i], virt[i]));
    HSV_TRY(launch_bsweep(sec, 1, -1, bops, cs, sn, psi->d_amp, w->d_amp, nullptr, w->d_norm2,
                          d_grad, sc.err, sc.err_val, &batched));
  }
  if (!batched && tuning().sweep) {
    HSV_TRY(state_arow_async(psi));
    HSV_TRY(state_arow_async(w));
    static thread_local std::vector<SweepOp> ops;
    ops.clear();
    for (int64_t i = 0; i < k; ++i) ops.push_back(sweep_op(sec, occ[i], virt[i], cs[i], sn[i]));
    HSV_TRY(launch_sweep<kAdjoint>(sec, ops, psi->d_amp, psi->d_arow, w->d_amp, w->d_arow,
                                   w->d_norm2, d_grad, sc));
  }
  for (int64_t i = tuning().sweep ? -1 : k - 1; i >= 0; --i) {   // per-op launches
    HSV_TRY(build_pair_lists_async(sec, compress_op(sec, occ[i], virt[i]), pl));
    if (pl.ca == 0 || pl.cb == 0) {
      HSV_TRY_CUDA(cudaMemsetAsync(d_grad + i, 0, sizeof(double), stream()));
      continue;
    }
    PairArgs a{};
    a.Nb = sec->Nb; a.psi = psi->d_amp; a.lam = w->d_amp; a.c = cs[i]; a.s = -sn[i];
    a.part = sc.part; a.counter = sc.counter; a.norm2 = w->d_norm2; a.result = d_grad + i;
    a.err = sc.err; a.err_val = sc.err_val; a.uncompute = i > 0;
    a.fpsi = psi->d_arow; a.flam = w->d_arow;
    HSV_TRY(launch_pairs<kAdjoint>(pl, a));
  }
  static thread_local std::vector<double> h;
  h.resize(k + 2);
  {
    HostWatch hw("gradients D2H");
    HostProf hs("bwd_wait");
    HSV_TRY_CUDA(cudaMemcpyAsync(h.data(), d_grad, (k + 2) * sizeof(double),
                                 cudaMemcpyDeviceToHost, stream()));
  }
  const int rc = sc.check();
  dfree(pl.la); dfree(pl.lb);
  sc.release();
  dfree(d_grad);
  psi->norm2_valid = false;
  psi->arow_valid = psi->arow_valid && tuning().sweep != 2;   // batched sweep keeps no flags
  w->arow_valid = w->arow_valid && tuning().sweep != 2;
  psi->smap_valid = w->smap_valid = false;
  psi->dense_hint = w->dense_hint = false;
  HSV_TRY(stream_sync());
  for (int64_t i = 0; i < k; ++i) grads[i] = h[i];
  *energy = h[k];
  if (psi->d_pend_err) {   // the forward sweep's drift report comes first
    const int rf = take_pending_drift(psi);
    if (rf) return rf;
  }
  return rc;
}

int hsv_energy_gradient(hsv_op op, uint64_t hf_key, const uint64_t* occ, const uint64_t* virt,
                        const double* cs, const double* sn, int64_t k, double* energy,
                        double* grads) {
  HSV_TRY(check_eg_args(op, occ, virt, cs, sn, k));
  HSV_REQUIRE(energy && (k == 0 || grads), HSV_ERR_INVALID, "null output");
  hsv_state psi = nullptr, w = nullptr;
  HSV_TRY(hsv_state_create(op->sec, &psi));
  int rc = hsv_state_create(op->sec, &w);
  if (!rc) rc = hsv_eg_forward_async(op, hf_key, occ, virt, cs, sn, k, 0, op->sec->Na, psi, w);
  if (!rc) rc = hsv_eg_backward(op, psi, w, occ, virt, cs, sn, k, energy, grads);
  hsv_state_destroy(psi);
  hsv_state_destroy(w);
  return rc;
}

}  // extern "C"
