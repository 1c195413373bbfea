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
// (hsv_state_s::d_smap; every rotation -- also one at theta = 0, whose
// gradient reads w on T psi -- marks both rows of a pair if either is
// marked).  Orbits with no marked row hold only exact zeros: the
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

constexpr int kBatch = 3;   // rotations per batch (orbits of 2^kBatch rows); 4 measured slower (H12 depth 400: 0.79 vs 0.60 ms forward)
constexpr int kOrb = 1 << kBatch;
constexpr int kRW = kOrb / 4;           // uint4 words of an orbit's rows
static_assert(kBatch <= 7 && kOrb <= 16, "orbit masks are 16-bit fields of one uint4");

// 16-bit field f of an orbit's masks: f = 0 touched elements, f = j + 1 the
// elements that are sources of rotation j
__host__ __device__ __forceinline__ unsigned mfield(const uint4& mk, int f) {
  const unsigned w = f < 2 ? mk.x : f < 4 ? mk.y : f < 6 ? mk.z : mk.w;
  return (f & 1) ? (w >> 16) : (w & 0xffffu);
}
enum { kFwd = 0, kAdj = 1 };

struct __align__(16) BatchDev {
  double c[kBatch], s[kBatch];
  const uint32_t* rows;  // live orbits: kOrb rows each (plan)
  const uint4* masks;    // live orbits: 16-bit fields touched, srcm_0 .. (mfield)
  const uint32_t* ranks; // live orbits: per element, write rank | row writers << 16
  int n;                 // rotations in the batch
  int op0;               // index (in sweep-list order) of the batch's first rotation
  uint32_t count;        // live orbits of the batch
};
constexpr int kBChunk = 96;   // batch descriptors staged in shared memory at a time
static_assert(sizeof(BatchDev) % 16 == 0, "BatchDev is copied as 16-byte words");

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
  uint32_t* ver;               // barrier-free sweep: writes completed per row (zeroed)
  unsigned* bar;               // barrier sweep: counting-barrier word (zeroed), nullptr: grid.sync
  // barrier-free sweep: the plan's global (padded) orbit arrays, chunk maps
  const uint32_t* rows;
  const uint4* masks;
  const uint32_t* ranks;
  int64_t n_chunks;
  const int* chunk_batch;       // physical chunk -> batch (plan order)
  const uint32_t* chunk_order;  // sweep order -> physical chunk (nullptr: identity)
  const int64_t* chunk_off;     // batch -> first chunk (n_batches + 1)
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

// Counting grid barrier for the batched sweep (co-residency from the
// cooperative launch): arrivals on one monotone counter, zeroed before the
// launch; barrier e completes when e * gridDim.x blocks have arrived.  The
// release add / acquire poll pair replaces grid.sync()'s fence + atomic + fence
// (microbenchmark, 148 blocks with an L2 round trip between barriers: 1.73 vs
// 2.07 us, tools/micro/gbar_probe.cu).
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void count_barrier(unsigned* ctr, unsigned& epoch) {
  ++epoch;
  if (!ctr) {
    grid_sync();
    return;
  }
  __syncthreads();   // the block's writes are ordered before thread 0's release
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    const unsigned target = epoch * gridDim.x;
    while ((int)(ld_acquire_u32(ctr) - target) < 0) {}
  }
  __syncthreads();
}

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

// Geometry of one orbit: its rows, the rows a rotation of the batch touches
// and, per rotation j, the orbit elements that are its sources (partner of
// element t is t ^ (1 << j)).
struct BatchMasks {
  uint32_t oa[kBatch], va[kBatch], ob[kBatch], vb[kBatch];
  int n;
};

__device__ __forceinline__ void orbit_geom(uint2 rep, const BatchMasks& B, int n_alpha,
                                           int n_beta, const uint32_t* __restrict__ Ra,
                                           const uint32_t* __restrict__ Rb, uint32_t Nb,
                                           uint32_t (&row)[kOrb], unsigned& touched,
                                           unsigned (&srcm)[kBatch]) {
  touched = 0u;
#pragma unroll
  for (int j = 0; j < kBatch; ++j) srcm[j] = 0u;
#pragma unroll
  for (int t = 0; t < kOrb; ++t) {
    uint32_t x = rep.x, y = rep.y;
#pragma unroll
    for (int j = 0; j < kBatch; ++j)
      if (((t >> j) & 1) && j < B.n) { x ^= B.oa[j] | B.va[j]; y ^= B.ob[j] | B.vb[j]; }
    row[t] = 0u;
    if (t >= (1 << B.n) || __popc(x) != n_alpha || __popc(y) != n_beta) continue;
    row[t] = __ldg(Ra + x) * Nb + __ldg(Rb + y);
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      if (j >= B.n) continue;
      if (is_src(x, y, B.oa[j], B.va[j], B.ob[j], B.vb[j])) {
        srcm[j] |= 1u << t;
        touched |= (1u << t) | (1u << (t ^ (1 << j)));
      }
    }
  }
}

// Plan filter (cooperative, once per operator list): the structural support
// closure of the HF row under every rotation, batch by batch, and for every
// candidate orbit whether it holds a supported row when its batch runs (the
// orbit is closed under the batch, so that is also whether it holds one after
// it).  Only those "live" orbits are ever rotated, forward or adjoint.
struct FilterArgs {
  const BatchMasks* bm;
  const uint2* const* cand;
  const uint32_t* const* cand_count;
  const int64_t* flag_off;
  int n_batches;
  uint8_t* flags;
  uint8_t* smap;
  int n_alpha, n_beta;
  uint32_t Nb;
  const uint32_t* Ra;
  const uint32_t* Rb;
  uint32_t* live_count;
  uint32_t* wcount;       // per row: live orbits (so far, in batch order) that touch it
  uint16_t* wrank;        // per candidate and orbit element: the orbit's rank among them
  unsigned long long* n_marked;   // rows added to the support map (running count)
  uint32_t* added;                // ... and the rows, in batch order (unmarked on a replan)
  uint32_t* batch_new;            // per batch: rows it added (zeroed)
};

__global__ void __launch_bounds__(256) k_plan_filter(const FilterArgs a) {
  __shared__ BatchMasks B;
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (int bi = 0; bi < a.n_batches; ++bi) {
    if (threadIdx.x == 0) B = a.bm[bi];
    __syncthreads();
    const uint32_t n = __ldg(a.cand_count[bi]);
    unsigned live_n = 0u, new_n = 0u;
    for (int64_t it = gt; it < n; it += nt) {
      uint32_t row[kOrb];
      unsigned touched, srcm[kBatch];
      orbit_geom(__ldg(a.cand[bi] + it), B, a.n_alpha, a.n_beta, a.Ra, a.Rb, a.Nb, row, touched,
                 srcm);
      unsigned marked = 0u;
#pragma unroll
      for (int t = 0; t < kOrb; ++t)
        if (((touched >> t) & 1u) && a.smap[row[t]]) marked |= 1u << t;
      const bool live = marked != 0u;
      a.flags[a.flag_off[bi] + it] = live ? 1 : 0;
      if (!live) continue;
      ++live_n;
#pragma unroll
      for (int j = 0; j < kBatch; ++j)
#pragma unroll
        for (int t = 0; t < kOrb; ++t) {
          if (!((srcm[j] >> t) & 1u)) continue;
          const int p = t ^ (1 << j);
          if ((marked >> t | marked >> p) & 1u) marked |= (1u << t) | (1u << p);
        }
#pragma unroll
      for (int t = 0; t < kOrb; ++t)
        if ((marked >> t) & 1u) {
          if (!a.smap[row[t]]) {
            const unsigned long long pos = atomicAdd(a.n_marked, 1ull);
            if (a.added) a.added[pos] = row[t];
            ++new_n;
          }
          a.smap[row[t]] = 1;
        }
      // write ranks for the barrier-free sweep: orbits of one batch are
      // disjoint, and the grid barrier orders batches, so a plain increment
      // gives every row's writers their batch order
#pragma unroll
      for (int t = 0; t < kOrb; ++t)
        if (a.wcount && ((touched >> t) & 1u)) {
          const uint32_t r = a.wcount[row[t]];
          a.wcount[row[t]] = r + 1;
          a.wrank[(a.flag_off[bi] + it) * kOrb + t] = (uint16_t)min(r, 65535u);
        }
    }
    const unsigned tot = __reduce_add_sync(0xffffffffu, live_n);
    if (lane == 0 && tot) atomicAdd(a.live_count + bi, tot);
    const unsigned totn = __reduce_add_sync(0xffffffffu, new_n);
    if (lane == 0 && totn && a.batch_new) atomicAdd(a.batch_new + bi, totn);
    __syncthreads();
    grid_sync();   // batch bi + 1 sees the marks of batch bi
  }
}

// Live orbit i (global order = batch order, then candidate order): its touched
// rows and masks (touched | srcm_j << 8 (j + 1)), precomputed once per plan.
struct GatherArgs {
  const BatchMasks* bm;
  const uint2* const* cand;
  const int64_t* flag_off;
  int n_batches;
  const int* sel;
  const int* n_sel;
  int n_alpha, n_beta;
  uint32_t Nb;
  const uint32_t* Ra;
  const uint32_t* Rb;
  uint32_t* rows;
  uint4* masks;
  const uint16_t* wrank;
  const uint32_t* wcount;
  uint32_t* ranks;        // per live orbit element: rank | (writers of the row) << 16
  const int64_t* loff_cmp;  // live orbits before batch b (compact) ...
  const int64_t* loff_pad;  // ... and in the padded layout (whole 32-orbit chunks per batch)
};

__global__ void k_plan_gather(const GatherArgs a) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= *a.n_sel) return;
  const int64_t g = a.sel[i];
  int lo = 0, hi = a.n_batches;   // last batch with flag_off <= g
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    if (a.flag_off[mid] <= g) lo = mid; else hi = mid;
  }
  const BatchMasks B = a.bm[lo];
  uint32_t row[kOrb];
  unsigned touched, srcm[kBatch];
  orbit_geom(a.cand[lo][g - a.flag_off[lo]], B, a.n_alpha, a.n_beta, a.Ra, a.Rb, a.Nb, row,
             touched, srcm);
  const int64_t si = i;   // compact index (selection order)
  const int64_t pi = a.loff_pad[lo] + (si - a.loff_cmp[lo]);   // padded slot
  unsigned f[8] = {touched, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
  for (int j = 0; j < kBatch; ++j) f[j + 1] = srcm[j];
  a.masks[pi] = make_uint4(f[0] | f[1] << 16, f[2] | f[3] << 16, f[4] | f[5] << 16,
                           f[6] | f[7] << 16);
  uint4* r = reinterpret_cast<uint4*>(a.rows + pi * kOrb);
#pragma unroll
  for (int q = 0; q < kRW; ++q)
    r[q] = make_uint4(row[4 * q], row[4 * q + 1], row[4 * q + 2], row[4 * q + 3]);
  if (a.ranks) {
    uint32_t k[kOrb];
#pragma unroll
    for (int t = 0; t < kOrb; ++t)
      k[t] = ((touched >> t) & 1u)
                 ? (uint32_t)a.wrank[g * kOrb + t] | (min(a.wcount[row[t]], 65535u) << 16)
                 : 0u;
    uint4* kr = reinterpret_cast<uint4*>(a.ranks + pi * kOrb);
#pragma unroll
    for (int q = 0; q < kRW; ++q) kr[q] = make_uint4(k[4 * q], k[4 * q + 1], k[4 * q + 2], k[4 * q + 3]);
  }
}

// Norm-drift chain in sweep order (svengine.py:234-236) and, adjoint, the
// gradients: block 0, after the per-rotation totals are complete.
template <int MODE, int NV>
__device__ __forceinline__ void norm_chain(const BSweepArgs& a) {
  if (blockIdx.x == 0) {   // norm chain in sweep order (svengine.py:234-236)
    // the totals are staged in shared memory by the whole block first, so the
    // sequential chain runs on on-chip loads (400 dependent L2 loads cost
    // ~0.3 ms at k = 400)
    constexpr int kChunk = 1024;
    __shared__ double tsh[kChunk * NV];
    double nn = 0.0;
    if (threadIdx.x == 0) nn = *a.norm2;
    for (int o0 = 0; o0 < a.n_ops; o0 += kChunk) {
      const int n = min(kChunk, a.n_ops - o0);
      __syncthreads();
      for (int i = threadIdx.x; i < n * NV; i += blockDim.x) {
        const int o = o0 + i / NV;
        const int op = MODE == kFwd ? o : a.n_ops - 1 - o;
        tsh[i] = __ldcg(a.red + (int64_t)op * NV + i % NV);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int i = 0; i < n; ++i) {
          const double* tot = tsh + i * NV;
          const double dold = MODE == kAdj ? tot[1] : tot[0];
          const double dnew = MODE == kAdj ? tot[2] : tot[1];
          const double nnew = nn - dold + dnew;
          const double nrm = sqrt(fmax(nn, 0.0));
          const double drift = fabs(sqrt(fmax(nnew, 0.0)) - nrm);
          if (drift > kNormDriftTol * fmax(1.0, nrm)) {
            if (atomicExch(a.err, 1) == 0) *a.err_val = drift;
          }
          nn = nnew;
        }
      }
      if (MODE == kAdj)
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
          const int o = o0 + i;
          a.grads[a.n_ops - 1 - o] = 2.0 * tsh[i * NV];
        }
    }
    if (threadIdx.x == 0) *a.norm2 = nn;
  }
}

// One live orbit of a batch: forward rotations (MODE kFwd) or, in reverse
// order, gradient partial + adjoint rotation + uncompute (kAdj).
struct OrbitRec {
  uint4 mk;
  uint4 r[kRW];
};

template <int MODE>
__device__ __forceinline__ void do_orbit(const BSweepArgs& a, const BatchDev& B, const OrbitRec& o,
                                         double (&acc)[kBatch][3], unsigned& npairs) {
  const unsigned touched = mfield(o.mk, 0);
  uint32_t row[kOrb];
#pragma unroll
  for (int q = 0; q < kRW; ++q) {
    row[4 * q] = o.r[q].x; row[4 * q + 1] = o.r[q].y;
    row[4 * q + 2] = o.r[q].z; row[4 * q + 3] = o.r[q].w;
  }
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
      const unsigned sj = mfield(o.mk, j + 1);
      npairs += __popc(sj);
      if (j >= B.n || (B.c[j] == 1.0 && B.s[j] == 0.0)) continue;   // theta == 0: identity
#pragma unroll
      for (int t = 0; t < kOrb; ++t) {
        if (!((sj >> t) & 1u)) continue;
        const int p = t ^ (1 << j);
        double2 nb, np;
        rot(v[t], v[p], B.c[j], B.s[j], nb, np);
        acc[j][0] += n2(v[t]) + n2(v[p]);
        acc[j][1] += n2(nb) + n2(np);
        v[t] = nb;
        v[p] = np;
      }
    }
#pragma unroll
    for (int t = 0; t < kOrb; ++t)
      if ((touched >> t) & 1u) a.psi[row[t]] = v[t];
  } else {
#pragma unroll
    for (int jj = kBatch - 1; jj >= 0; --jj) {
      if (jj >= B.n) continue;
      const unsigned sj = mfield(o.mk, jj + 1);
      npairs += __popc(sj);
      const bool unc = B.op0 + jj > 0;   // psi of the first rotation is never read again
#pragma unroll
      for (int t = 0; t < kOrb; ++t) {
        if (!((sj >> t) & 1u)) continue;
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

// An orbit's plan record (masks + 8 rows): loaded before the grid barrier that
// precedes its batch -- it does not depend on amplitudes -- so after the
// barrier only the amplitude loads remain on the critical path.
__device__ __forceinline__ OrbitRec load_orbit(const BatchDev& B, int64_t it) {
  OrbitRec o;
  o.mk = __ldg(B.masks + it);
  const uint4* rp = reinterpret_cast<const uint4*>(B.rows + it * kOrb);
#pragma unroll
  for (int q = 0; q < kRW; ++q) o.r[q] = __ldg(rp + q);
  return o;
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) k_bsweep(const BSweepArgs a) {   // <= one block per SM (launch_bsweep)
  constexpr int NV = MODE == kAdj ? 3 : 2;
  // batch descriptors staged in shared memory kBChunk at a time by the whole
  // block: no serial descriptor load between a grid barrier and the next batch
  __shared__ __align__(16) BatchDev sB[kBChunk];
  const int lane = threadIdx.x & 31;
  // logical warp gw: consecutive warps of a batch's orbit list sit on
  // different SMs (a batch of a few thousand orbits would otherwise load all
  // its amplitudes through the first ~20 SMs' LSUs)
  const int64_t gw = (int64_t)(threadIdx.x >> 5) * gridDim.x + blockIdx.x;
  const int64_t gt = gw * 32 + lane;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  const int64_t nw = nt >> 5;
  OrbitRec next{};
  bool have_next = false;
  unsigned epoch = 0;
  for (int bi = 0; bi < a.n_batches; ++bi) {
    if (bi % kBChunk == 0) {
      __syncthreads();
      const int n = min(kBChunk, a.n_batches - bi);
      constexpr int W4 = sizeof(BatchDev) / 16;
      const uint4* src = reinterpret_cast<const uint4*>(a.batches + bi);
      uint4* dst = reinterpret_cast<uint4*>(sB);
      for (int i = threadIdx.x; i < n * W4; i += blockDim.x) dst[i] = __ldg(src + i);
      __syncthreads();
    }
    const BatchDev& B = sB[bi % kBChunk];
    const uint32_t n_items = B.count;
    double acc[kBatch][3];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) acc[j][0] = acc[j][1] = acc[j][2] = 0.0;
    unsigned npairs = 0u;
    for (int64_t it = gt; it < n_items; it += nt) {
      const OrbitRec o = (it == gt && have_next) ? next : load_orbit(B, it);
      do_orbit<MODE>(a, B, o, acc, npairs);
    }
    if (a.stats) {
      const unsigned tot = __reduce_add_sync(0xffffffffu, npairs);
      if (lane == 0 && tot) atomicAdd(a.stats + (MODE == kFwd ? kStatPairsFwd : kStatPairsAdj),
                                      (unsigned long long)tot);
    }
    // warp partials per rotation (fixed shuffle tree; no block barrier)
    if (gw * 32 < (int64_t)n_items) {
#pragma unroll
      for (int j = 0; j < kBatch; ++j)
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          const double x = warp_sum(acc[j][q]);
          if (lane == 0) a.part[(((int64_t)bi * nw + gw) * kBatch + j) * NV + q] = x;
        }
    }
    // prefetch this thread's first orbit of the next batch
    have_next = false;
    if (bi + 1 < a.n_batches) {
      const BatchDev& Bn = ((bi + 1) % kBChunk) ? sB[(bi + 1) % kBChunk] : a.batches[bi + 1];
      if (gt < (int64_t)Bn.count) {
        next = load_orbit(Bn, gt);
        have_next = true;
      }
    }
    count_barrier(a.bar, epoch);   // batch bi+1 reads rows batch bi wrote
  }
  // per-rotation totals: one rotation per warp, warps summed in a fixed order
  // (warps whose first orbit index is past the batch wrote nothing: skipped)
  for (int64_t oi = gw; oi < (int64_t)a.n_batches * kBatch; oi += nw) {
    const int bi = (int)(oi / kBatch), j = (int)(oi - (int64_t)bi * kBatch);
    const BatchDev& B = a.batches[bi];
    if (j >= B.n) continue;
    const int64_t used = min((int64_t)nw, ((int64_t)B.count + 31) / 32);
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double x = 0.0;
      for (int64_t k = lane; k < used; k += 32)
        x += __ldcg(a.part + (((int64_t)bi * nw + k) * kBatch + j) * NV + q);
      x = warp_sum(x);
      if (lane == 0) a.red[(int64_t)(B.op0 + j) * NV + q] = x;
    }
  }
  count_barrier(a.bar, epoch);
  norm_chain<MODE, NV>(a);
}

// ------------------------------------------------- barrier-free variant
// The same orbit work without grid barriers between batches: every row
// carries a version (writes completed in this sweep); an orbit of batch b
// waits, per touched row, until the orbits of earlier batches (forward order;
// later ones in the adjoint) that touch it have written it -- its rank among
// the row's writers, from the plan -- then rotates and publishes version + 1
// with a release store.  Orbits of one batch are disjoint, so each row's
// writers are totally ordered and the amplitudes are exactly the sequential
// ones; warps run ahead into later batches wherever the rows allow, instead
// of the whole grid waiting for the slowest block of every batch (67% of the
// barrier sweep's stall samples were grid/block barriers, ncu).
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int MODE>
__device__ __forceinline__ void do_orbit_p2p(const BSweepArgs& a, const BatchDev& B, int64_t it,
                                             double (&acc)[kBatch][3], unsigned& npairs) {
  // it: global (padded) orbit index of the plan; padding orbits have masks 0
  const uint4 mk = __ldg(a.masks + it);
  const unsigned touched = mfield(mk, 0);
  if (!touched) return;
  uint32_t row[kOrb], rk[kOrb];
  const uint4* rp = reinterpret_cast<const uint4*>(a.rows + it * kOrb);
  const uint4* kp = reinterpret_cast<const uint4*>(a.ranks + it * kOrb);
#pragma unroll
  for (int q = 0; q < kRW; ++q) {
    const uint4 r = __ldg(rp + q), k = __ldg(kp + q);
    row[4 * q] = r.x; row[4 * q + 1] = r.y; row[4 * q + 2] = r.z; row[4 * q + 3] = r.w;
    rk[4 * q] = k.x; rk[4 * q + 1] = k.y; rk[4 * q + 2] = k.z; rk[4 * q + 3] = k.w;
  }
  uint32_t need[kOrb];
#pragma unroll
  for (int t = 0; t < kOrb; ++t) {
    const uint32_t r = rk[t] & 0xffffu, n = rk[t] >> 16;
    need[t] = MODE == kFwd ? r : n - 1u - r;
  }
#pragma unroll
  for (int t = 0; t < kOrb; ++t) {
    if (!((touched >> t) & 1u)) continue;
    unsigned ns = 32;
    while (ld_acquire(a.ver + row[t]) != need[t]) {   // backoff: hot rows have many waiters
      __nanosleep(ns);
      ns = min(ns * 2, 1024u);
    }
  }
  double2 v[kOrb];
  double2 l[kOrb];
#pragma unroll
  for (int t = 0; t < kOrb; ++t) {
    v[t] = make_double2(0.0, 0.0);
    l[t] = make_double2(0.0, 0.0);
    if ((touched >> t) & 1u) {
      v[t] = __ldcg(a.psi + row[t]);
      if (MODE == kAdj) l[t] = __ldcg(a.lam + row[t]);
    }
  }
  if (MODE == kFwd) {
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const unsigned sj = mfield(mk, j + 1);
      npairs += __popc(sj);
      if (j >= B.n || (B.c[j] == 1.0 && B.s[j] == 0.0)) continue;
#pragma unroll
      for (int t = 0; t < kOrb; ++t) {
        if (!((sj >> t) & 1u)) continue;
        const int p = t ^ (1 << j);
        double2 nb, np;
        rot(v[t], v[p], B.c[j], B.s[j], nb, np);
        acc[j][0] += n2(v[t]) + n2(v[p]);
        acc[j][1] += n2(nb) + n2(np);
        v[t] = nb;
        v[p] = np;
      }
    }
#pragma unroll
    for (int t = 0; t < kOrb; ++t)
      if ((touched >> t) & 1u) __stcg(a.psi + row[t], v[t]);
  } else {
#pragma unroll
    for (int jj = kBatch - 1; jj >= 0; --jj) {
      if (jj >= B.n) continue;
      const unsigned sj = mfield(mk, jj + 1);
      npairs += __popc(sj);
      const bool unc = B.op0 + jj > 0;
#pragma unroll
      for (int t = 0; t < kOrb; ++t) {
        if (!((sj >> t) & 1u)) continue;
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
      __stcg(a.lam + row[t], l[t]);
      __stcg(a.psi + row[t], v[t]);
    }
  }
#pragma unroll
  for (int t = 0; t < kOrb; ++t)
    if ((touched >> t) & 1u) st_release(a.ver + row[t], need[t] + 1u);
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) k_psweep(const BSweepArgs a) {
  constexpr int NV = MODE == kAdj ? 3 : 2;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // Live orbits are laid out batch after batch, each batch padded to whole
  // 32-orbit chunks; warps take chunks round robin in sweep order (adjoint:
  // batches reversed), so consecutive batches run on different warps at the
  // same time, ordered only by the rows they share.
  for (int64_t L = gw; L < a.n_chunks; L += nw) {
    const int64_t c = a.chunk_order ? (int64_t)__ldg(a.chunk_order + L) : L;
    const int bi = __ldg(a.chunk_batch + c);
    const BatchDev& B = a.batches[bi];
    double acc[kBatch][3];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) acc[j][0] = acc[j][1] = acc[j][2] = 0.0;
    unsigned npairs = 0u;
    do_orbit_p2p<MODE>(a, B, c * 32 + lane, acc, npairs);
    if (a.stats) {
      const unsigned tot = __reduce_add_sync(0xffffffffu, npairs);
      if (lane == 0 && tot) atomicAdd(a.stats + (MODE == kFwd ? kStatPairsFwd : kStatPairsAdj),
                                      (unsigned long long)tot);
    }
#pragma unroll
    for (int j = 0; j < kBatch; ++j)
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const double x = warp_sum(acc[j][q]);
        if (lane == 0) a.part[(c * kBatch + j) * NV + q] = x;
      }
  }
  grid_sync();   // every chunk partial written
  // per-rotation totals: one rotation per warp, the batch's chunks in order
  for (int64_t oi = gw; oi < (int64_t)a.n_batches * kBatch; oi += nw) {
    const int bi = (int)(oi / kBatch), j = (int)(oi - (int64_t)bi * kBatch);
    const BatchDev& B = a.batches[bi];
    if (j >= B.n) continue;
    const int64_t c0 = __ldg(a.chunk_off + bi), c1 = __ldg(a.chunk_off + bi + 1);
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double x = 0.0;
      for (int64_t k = c0 + lane; k < c1; k += 32) x += __ldcg(a.part + (k * kBatch + j) * NV + q);
      x = warp_sum(x);
      if (lane == 0) a.red[(int64_t)(B.op0 + j) * NV + q] = x;
    }
  }
  grid_sync();
  norm_chain<MODE, NV>(a);
}

// ----------------------------------------------------------------- plans
struct PlanBatch {
  std::vector<OpMasks> m;
  int64_t n_cand = 0;             // upper bound of the candidate count
  uint2* cand = nullptr;          // canonical orbit representatives
  uint32_t* cand_count = nullptr; // device count
};

// Cached per (sector, HF row, operator list): batches with their candidate
// orbits (reused by prefix: an appended operator changes the last batch only),
// and -- after the filter -- the live orbits with precomputed rows and the
// structural support closure of HF (the K1r rows).
struct Plan {
  const hsv_sector_s* sec = nullptr;
  int64_t hf_row = -1;
  std::vector<PlanBatch> b;
  bool filtered = false;
  uint8_t* smap = nullptr;
  uint32_t* rows = nullptr;
  uint4* masks = nullptr;
  uint32_t* ranks = nullptr;   // barrier-free sweep: per element write rank | writers << 16
  uint32_t* ver = nullptr;     // per-row versions (dim), zeroed before each barrier-free sweep
  unsigned* bar = nullptr;     // counting-barrier word of the barrier sweep
  int* chunk_batch = nullptr;  // physical 32-orbit chunk -> batch
  uint32_t* chunk_rev = nullptr;   // adjoint order: chunks of the batches in reverse
  int64_t* chunk_off = nullptr;    // batch -> first chunk
  int64_t n_chunks = 0;
  int64_t support_rows = 0;    // rows of the support map (HF closure)
  uint64_t version = 0;        // changes whenever the support map does (K1s caches on it)
  uint32_t* added = nullptr;   // rows each batch added to the map, batch after batch (dim)
  std::vector<int64_t> added_end;   // per batch: rows added by batches <= it
  bool has_ranks = false;
  std::vector<int64_t> live_off, live_cnt;
  int64_t max_live = 0;
  void drop_live() {
    dfree(rows); dfree(masks); dfree(ranks);
    dfree(chunk_batch); dfree(chunk_rev); dfree(chunk_off);
    rows = ranks = chunk_rev = nullptr;
    masks = nullptr;
    chunk_batch = nullptr;
    chunk_off = nullptr;
    n_chunks = 0;
    filtered = false;
  }
  void clear() {
    for (auto& x : b) { dfree(x.cand); dfree(x.cand_count); }
    b.clear();
    drop_live();
    dfree(smap);
    dfree(ver);
    dfree(added);
    dfree(bar);
    smap = nullptr;
    ver = nullptr;
    bar = nullptr;
    added = nullptr;
    hf_row = -1;
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

BatchMasks batch_masks(const PlanBatch& pb) {
  BatchMasks m{};
  m.n = (int)pb.m.size();
  for (int j = 0; j < m.n; ++j) {
    m.oa[j] = pb.m[j].oa; m.va[j] = pb.m[j].va; m.ob[j] = pb.m[j].ob; m.vb[j] = pb.m[j].vb;
  }
  return m;
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
  for (int j = 0; j < a.n; ++j)   // guard the division of an empty range
    if (a.cb[j] == 0) a.cb[j] = 1;
  const int64_t T = a.off[a.n];
  pb.n_cand = T;
  HSV_TRY(dalloc(&pb.cand, std::max<int64_t>(T, 1)));
  HSV_TRY(dalloc(&pb.cand_count, 1));
  HSV_TRY_CUDA(cudaMemsetAsync(pb.cand_count, 0, sizeof(uint32_t), stream()));
  if (T == 0) return HSV_OK;
  HSV_REQUIRE(T < (int64_t)INT32_MAX, HSV_ERR_UNSUPPORTED, "batch plan too large");
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
  HSV_TRY_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, cand, flag, pb.cand, pb.cand_count, (int)T,
                                          stream()));
  char* tmp = nullptr;
  HSV_TRY(dalloc(&tmp, tb));
  HSV_TRY_CUDA(cub::DeviceSelect::Flagged(tmp, tb, cand, flag, pb.cand, pb.cand_count, (int)T,
                                          stream()));
  count_launch();
  dfree(tmp);
  dfree(cand);
  dfree(flag);
  return HSV_OK;
}

int coop_grid(const void* fn, int64_t want, int threads = 256) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, 0) != cudaSuccess) {
    cudaGetLastError();
    occ = 1;
  }
  const int64_t resident = (int64_t)ctx().num_sms * std::max(occ, 1);
  return (int)std::max<int64_t>(1, std::min<int64_t>(resident, want));
}

int64_t ops_total(const Plan& P) {
  int64_t n = 0;
  for (const auto& b : P.b) n += (int64_t)b.m.size();
  return n;
}

__global__ void k_unmark(const uint32_t* __restrict__ rows, int64_t n, uint8_t* __restrict__ smap) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) smap[rows[i]] = 0;
}

// The filter + gather of batches [first, nb) of a plan whose batches are built
// (k_plan_filter).  first == 0: from scratch (support map = HF).  first > 0:
// incremental -- batches [0, first) and their live orbits are kept, the
// support map holds exactly their closure (get_plan unmarked the rows later
// batches had added), and only the new batches are filtered and appended.
// The barrier-free sweep's per-row write ranks need every batch: built (and
// only then) from scratch when that sweep is enabled.
int filter_plan(Plan& P, int first) {
  const hsv_sector_s* sec = P.sec;
  const int nb = (int)P.b.size();
  const bool ranks = tuning().sweep_p2p != 0 && (int64_t)ops_total(P) < 65535;
  if (ranks || !P.filtered || P.has_ranks) first = 0;
  if (!P.smap) HSV_TRY(dalloc(&P.smap, sec->dim));
  if (!P.added) HSV_TRY(dalloc(&P.added, sec->dim));
  int64_t added0 = 0;
  if (first == 0) {
    P.drop_live();
    static thread_local uint8_t one;
    one = 1;
    HSV_TRY_CUDA(cudaMemsetAsync(P.smap, 0, sec->dim, stream()));
    HSV_TRY_CUDA(cudaMemcpyAsync(P.smap + P.hf_row, &one, 1, cudaMemcpyHostToDevice, stream()));
    P.live_off.assign(1, 0);
    P.live_cnt.clear();
    P.added_end.clear();
    P.max_live = 0;
  } else {
    added0 = P.added_end[first - 1];
    P.live_off.resize(first + 1);
    P.live_cnt.resize(first);
    P.added_end.resize(first);
    P.max_live = 0;
    for (int q = 0; q < first; ++q) P.max_live = std::max(P.max_live, P.live_cnt[q]);
  }
  P.has_ranks = ranks;
  const int nn = nb - first;   // batches to filter
  P.support_rows = 1 + added0;
  if (nn == 0) {
    P.filtered = true;
    return stream_sync();
  }
  std::vector<BatchMasks> hm(nn);
  std::vector<const uint2*> hc(nn);
  std::vector<const uint32_t*> hn(nn);
  std::vector<int64_t> off(nn + 1, 0);
  int64_t max_cand = 1;
  for (int q = 0; q < nn; ++q) {
    const PlanBatch& pb = P.b[first + q];
    hm[q] = batch_masks(pb);
    hc[q] = pb.cand;
    hn[q] = pb.cand_count;
    off[q + 1] = off[q] + pb.n_cand;
    max_cand = std::max(max_cand, pb.n_cand);
  }
  const int64_t total = off[nn];
  HSV_REQUIRE(total < (int64_t)INT32_MAX, HSV_ERR_UNSUPPORTED, "sweep plan too large");
  BatchMasks* d_m = nullptr;
  const uint2** d_c = nullptr;
  const uint32_t** d_n = nullptr;
  int64_t* d_off = nullptr;
  uint8_t* flags = nullptr;
  uint32_t* live = nullptr;
  int *sel = nullptr, *n_sel = nullptr;
  uint32_t* wcount = nullptr;
  uint16_t* wrank = nullptr;
  unsigned long long* n_marked = nullptr;
  uint32_t* d_bnew = nullptr;
  if (ranks) {
    HSV_TRY(dalloc(&wcount, sec->dim));
    HSV_TRY(dalloc(&wrank, std::max<int64_t>(total, 1) * kOrb));
    HSV_TRY_CUDA(cudaMemsetAsync(wcount, 0, sec->dim * sizeof(uint32_t), stream()));
  }
  static thread_local unsigned long long a0;
  a0 = (unsigned long long)added0;
  HSV_TRY(dalloc(&n_marked, 1));
  HSV_TRY_CUDA(cudaMemcpyAsync(n_marked, &a0, sizeof(a0), cudaMemcpyHostToDevice, stream()));
  HSV_TRY(dalloc(&d_bnew, nn));
  HSV_TRY_CUDA(cudaMemsetAsync(d_bnew, 0, nn * sizeof(uint32_t), stream()));
  HSV_TRY(dalloc(&d_m, nn));
  HSV_TRY(dalloc(&d_c, nn));
  HSV_TRY(dalloc(&d_n, nn));
  HSV_TRY(dalloc(&d_off, nn + 1));
  HSV_TRY(dalloc(&flags, std::max<int64_t>(total, 1)));
  HSV_TRY(dalloc(&live, nn));
  HSV_TRY(dalloc(&sel, std::max<int64_t>(total, 1)));
  HSV_TRY(dalloc(&n_sel, 1));
  HSV_TRY_CUDA(cudaMemcpyAsync(d_m, hm.data(), nn * sizeof(BatchMasks), cudaMemcpyHostToDevice,
                               stream()));
  HSV_TRY_CUDA(cudaMemcpyAsync(d_c, hc.data(), nn * sizeof(void*), cudaMemcpyHostToDevice,
                               stream()));
  HSV_TRY_CUDA(cudaMemcpyAsync(d_n, hn.data(), nn * sizeof(void*), cudaMemcpyHostToDevice,
                               stream()));
  HSV_TRY_CUDA(cudaMemcpyAsync(d_off, off.data(), (nn + 1) * sizeof(int64_t),
                               cudaMemcpyHostToDevice, stream()));
  HSV_TRY_CUDA(cudaMemsetAsync(flags, 0, std::max<int64_t>(total, 1), stream()));
  HSV_TRY_CUDA(cudaMemsetAsync(live, 0, nn * sizeof(uint32_t), stream()));
  FilterArgs fa{};
  fa.bm = d_m; fa.cand = d_c; fa.cand_count = d_n; fa.flag_off = d_off; fa.n_batches = nn;
  fa.flags = flags; fa.smap = P.smap; fa.n_alpha = sec->n_alpha; fa.n_beta = sec->n_beta;
  fa.Nb = (uint32_t)sec->Nb; fa.Ra = sec->d_Ra; fa.Rb = sec->d_Rb; fa.live_count = live;
  fa.wcount = wcount; fa.wrank = wrank; fa.n_marked = n_marked;
  fa.added = P.added; fa.batch_new = d_bnew;
  {
    ProfScope prof("sweep_plan");
    const int grid = coop_grid((const void*)k_plan_filter, (max_cand + 255) / 256);
    void* params[] = {&fa};
    HSV_TRY_CUDA(cudaLaunchCooperativeKernel((const void*)k_plan_filter, dim3(grid), dim3(256),
                                             params, 0, stream()));
    count_launch();
    size_t tb = 0;
    cub::CountingInputIterator<int> idx(0);
    HSV_TRY_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, idx, flags, sel, n_sel, (int)total,
                                            stream()));
    char* tmp = nullptr;
    HSV_TRY(dalloc(&tmp, tb));
    HSV_TRY_CUDA(cub::DeviceSelect::Flagged(tmp, tb, idx, flags, sel, n_sel, (int)total,
                                            stream()));
    count_launch();
    dfree(tmp);
  }
  std::vector<uint32_t> hl(nn);
  std::vector<uint32_t> hbn(nn);
  HSV_TRY_CUDA(cudaMemcpyAsync(hl.data(), live, nn * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                               stream()));
  HSV_TRY_CUDA(cudaMemcpyAsync(hbn.data(), d_bnew, nn * sizeof(uint32_t),
                               cudaMemcpyDeviceToHost, stream()));
  HSV_TRY(stream_sync());
  std::vector<int64_t> cmp(nn + 1, 0);
  for (int q = 0; q < nn; ++q) {
    P.live_cnt.push_back(hl[q]);
    P.added_end.push_back((P.added_end.empty() ? 0 : P.added_end.back()) + (int64_t)hbn[q]);
    cmp[q + 1] = cmp[q] + hl[q];
    P.live_off.push_back(P.live_off.back() + ((int64_t)hl[q] + 31) / 32 * 32);   // whole chunks
    P.max_live = std::max<int64_t>(P.max_live, hl[q]);
  }
  P.support_rows = 1 + P.added_end.back();   // HF + the rows the batches added
  const int64_t n_live = cmp[nn];
  const int64_t keep_slots = P.live_off[first];
  const int64_t n_slots = P.live_off[nb];
  {   // live-orbit arrays: keep the first batches' slots, append the new ones
    uint32_t* rows = nullptr;
    uint4* masks = nullptr;
    HSV_TRY(dalloc(&rows, std::max<int64_t>(n_slots, 1) * kOrb));
    HSV_TRY(dalloc(&masks, std::max<int64_t>(n_slots, 1)));
    if (keep_slots > 0) {
      HSV_TRY_CUDA(cudaMemcpyAsync(rows, P.rows, keep_slots * kOrb * sizeof(uint32_t),
                                   cudaMemcpyDeviceToDevice, stream()));
      HSV_TRY_CUDA(cudaMemcpyAsync(masks, P.masks, keep_slots * sizeof(uint4),
                                   cudaMemcpyDeviceToDevice, stream()));
    }
    HSV_TRY_CUDA(cudaMemsetAsync(masks + keep_slots, 0,
                                 std::max<int64_t>(n_slots - keep_slots, 0) * sizeof(uint4),
                                 stream()));
    dfree(P.rows);
    dfree(P.masks);
    P.rows = rows;
    P.masks = masks;
  }
  dfree(P.ranks);
  P.ranks = nullptr;
  if (ranks) HSV_TRY(dalloc(&P.ranks, std::max<int64_t>(n_slots, 1) * kOrb));
  P.n_chunks = n_slots / 32;
  dfree(P.chunk_batch); dfree(P.chunk_rev); dfree(P.chunk_off);
  P.chunk_batch = nullptr; P.chunk_rev = nullptr; P.chunk_off = nullptr;
  if (ranks) {   // chunk maps of the barrier-free sweep
    std::vector<int> cb(std::max<int64_t>(P.n_chunks, 1));
    std::vector<uint32_t> rev;
    std::vector<int64_t> choff(nb + 1);
    rev.reserve(P.n_chunks);
    for (int q = 0; q < nb; ++q) {
      choff[q] = P.live_off[q] / 32;
      for (int64_t c = P.live_off[q] / 32; c < P.live_off[q + 1] / 32; ++c) cb[c] = q;
    }
    choff[nb] = P.n_chunks;
    for (int q = nb - 1; q >= 0; --q)
      for (int64_t c = P.live_off[q] / 32; c < P.live_off[q + 1] / 32; ++c) rev.push_back((uint32_t)c);
    HSV_TRY(dalloc(&P.chunk_batch, cb.size()));
    HSV_TRY(dalloc(&P.chunk_rev, std::max<size_t>(rev.size(), 1)));
    HSV_TRY(dalloc(&P.chunk_off, nb + 1));
    HSV_TRY_CUDA(cudaMemcpyAsync(P.chunk_batch, cb.data(), cb.size() * sizeof(int),
                                 cudaMemcpyHostToDevice, stream()));
    if (!rev.empty())
      HSV_TRY_CUDA(cudaMemcpyAsync(P.chunk_rev, rev.data(), rev.size() * sizeof(uint32_t),
                                   cudaMemcpyHostToDevice, stream()));
    HSV_TRY_CUDA(cudaMemcpyAsync(P.chunk_off, choff.data(), (nb + 1) * sizeof(int64_t),
                                 cudaMemcpyHostToDevice, stream()));
    HSV_TRY(stream_sync());   // host vectors die here
  }
  int64_t *d_cmp = nullptr, *d_pad = nullptr;
  HSV_TRY(dalloc(&d_cmp, nn + 1));
  HSV_TRY(dalloc(&d_pad, nn + 1));
  HSV_TRY_CUDA(cudaMemcpyAsync(d_cmp, cmp.data(), (nn + 1) * sizeof(int64_t),
                               cudaMemcpyHostToDevice, stream()));
  HSV_TRY_CUDA(cudaMemcpyAsync(d_pad, P.live_off.data() + first, (nn + 1) * sizeof(int64_t),
                               cudaMemcpyHostToDevice, stream()));
  if (n_live > 0) {
    GatherArgs ga{};
    ga.bm = d_m; ga.cand = d_c; ga.flag_off = d_off; ga.n_batches = nn; ga.sel = sel;
    ga.n_sel = n_sel; ga.n_alpha = sec->n_alpha; ga.n_beta = sec->n_beta;
    ga.Nb = (uint32_t)sec->Nb; ga.Ra = sec->d_Ra; ga.Rb = sec->d_Rb;
    ga.rows = P.rows; ga.masks = P.masks;
    ga.wrank = wrank; ga.wcount = wcount; ga.ranks = P.ranks;
    ga.loff_cmp = d_cmp; ga.loff_pad = d_pad;
    ProfScope prof("sweep_plan");
    k_plan_gather<<<(unsigned)((n_live + 255) / 256), 256, 0, stream()>>>(ga);
    count_launch();
    HSV_CHECK_LAUNCH();
  }
  dfree(d_m); dfree(d_c); dfree(d_n); dfree(d_off); dfree(flags); dfree(live); dfree(sel);
  dfree(n_sel); dfree(wcount); dfree(wrank); dfree(d_cmp); dfree(d_pad); dfree(n_marked);
  dfree(d_bnew);
  HSV_TRY(stream_sync());   // the host offset vectors above must outlive their copies
  P.filtered = true;
  return HSV_OK;
}

// Plan for (hf_row, ops): cached batches equal to the requested ones at the
// same position are reused; the live lists are refiltered whenever anything
// changed.  hf_row < 0: the caller (the adjoint sweep) needs the current plan
// as it is; *ok = false when it does not match.
int get_plan(const hsv_sector_s* sec, int64_t hf_row, const std::vector<OpMasks>& ops,
             std::vector<std::vector<int>>& parts, bool* ok) {
  Plan& P = plan();
  *ok = true;
  parts = partition(ops);
  if (P.sec != sec) {
    if (hf_row < 0) { *ok = false; return HSV_OK; }
    P.clear();
    P.sec = sec;
  }
  size_t keep = 0;
  while (keep < parts.size() && keep < P.b.size()) {
    const auto& idx = parts[keep];
    const auto& pb = P.b[keep];
    bool eq = pb.m.size() == idx.size();
    for (size_t q = 0; eq && q < idx.size(); ++q) eq = same(pb.m[q], ops[idx[q]]);
    if (!eq) break;
    ++keep;
  }
  const bool unchanged = keep == parts.size() && keep == P.b.size() &&
                         (hf_row < 0 || hf_row == P.hf_row) && P.filtered;
  if (unchanged) return HSV_OK;
  if (hf_row < 0) { *ok = false; return HSV_OK; }
  // the new list extends the old one (ADAPT appends): its support map contains
  // the old map, so an unchanged row count means an unchanged map and the
  // map's version (K1s caches on it) stays
  bool extends = P.filtered && hf_row == P.hf_row;
  size_t pos = 0;
  for (const auto& pb : P.b)
    for (const auto& m : pb.m) {
      extends = extends && pos < ops.size() && same(m, ops[pos]);
      ++pos;
    }
  const int64_t old_rows = P.support_rows;
  // incremental replan (the common ADAPT case: an appended operator changes the
  // last batch or adds one): drop the support rows the replaced batches added,
  // keep the prefix's live orbits, filter only the new batches
  int first = 0;
  if (tuning().sweep_incr != 0 && P.filtered && hf_row == P.hf_row && keep > 0 && !P.has_ranks &&
      (int)P.added_end.size() == (int)P.b.size()) {
    first = (int)keep;
    const int64_t a0 = P.added_end[keep - 1], a1 = P.added_end.back();
    if (a1 > a0) {
      k_unmark<<<(unsigned)((a1 - a0 + 255) / 256), 256, 0, stream()>>>(P.added + a0, a1 - a0,
                                                                        P.smap);
      count_launch();
      HSV_CHECK_LAUNCH();
    }
  }
  for (size_t q = keep; q < P.b.size(); ++q) { dfree(P.b[q].cand); dfree(P.b[q].cand_count); }
  P.b.resize(keep);
  for (size_t q = keep; q < parts.size(); ++q) {
    PlanBatch pb;
    for (int i : parts[q]) pb.m.push_back(ops[i]);
    HSV_TRY(build_batch(sec, pb));
    P.b.push_back(pb);
  }
  P.hf_row = hf_row;
  HSV_TRY(filter_plan(P, first));
  static uint64_t g_version = 0;
  if (!(extends && P.support_rows == old_rows && P.version)) P.version = ++g_version;
  return HSV_OK;
}

}  // namespace

// Batched sweep over the rotation list (ops[i], cs[i], sn[i]) in list order:
// mode 0 forward from |hf_row> (psi rotated; the plan's support map copied to
// smap_out), 1 adjoint (reverse order; gradients into d_grads[i]; psi
// uncomputed, lam = w rotated; hf_row ignored, the forward's plan is reused).
// *used = false: no matching plan (the caller runs the per-rotation sweep).
int launch_bsweep(const hsv_sector_s* sec, int mode, int64_t hf_row,
                  const std::vector<OpMasks>& ops, const double* cs, const double* sn,
                  double2* psi, double2* lam, uint8_t* smap_out, double* norm2, double* d_grads,
                  int* err, double* err_val, bool* used) {
  *used = true;
  const int k = (int)ops.size();
  std::vector<std::vector<int>> parts;
  bool ok = true;
  {
    HostProf hp("get_plan");
    HSV_TRY(get_plan(sec, mode == kFwd ? hf_row : -1, ops, parts, &ok));
  }
  if (!ok) {
    *used = false;
    return HSV_OK;
  }
  Plan& P = plan();
  if (smap_out)
    HSV_TRY_CUDA(cudaMemcpyAsync(smap_out, P.smap, sec->dim, cudaMemcpyDeviceToDevice, stream()));
  if (k == 0) return HSV_OK;
  const int nb = (int)parts.size();
  const bool p2p = P.ranks && tuning().sweep_p2p != 0;
  static thread_local std::vector<BatchDev> hb;
  hb.assign(nb, BatchDev{});
  for (int q = 0; q < nb; ++q) {
    // barrier version: descriptors in processing order; barrier-free: plan order
    const int bq = (mode == kFwd || p2p) ? q : nb - 1 - q;
    BatchDev& d = hb[q];
    d.n = (int)parts[bq].size();
    d.op0 = parts[bq][0];
    for (int j = 0; j < d.n; ++j) {
      const int i = parts[bq][j];
      d.c[j] = cs[i];
      d.s[j] = sn[i];
    }
    d.rows = P.rows + P.live_off[bq] * kOrb;
    d.masks = P.masks + P.live_off[bq];
    d.ranks = P.ranks ? P.ranks + P.live_off[bq] * kOrb : nullptr;
    d.count = (uint32_t)P.live_cnt[bq];
  }
  BatchDev* d_b = nullptr;
  HSV_TRY(dalloc(&d_b, nb));
  HSV_TRY_CUDA(cudaMemcpyAsync(d_b, hb.data(), nb * sizeof(BatchDev), cudaMemcpyHostToDevice,
                               stream()));
  const void* fn = p2p ? (mode == kFwd ? (const void*)k_psweep<kFwd> : (const void*)k_psweep<kAdj>)
                       : (mode == kFwd ? (const void*)k_bsweep<kFwd> : (const void*)k_bsweep<kAdj>);
  // barrier version: one block per SM at most -- a cheaper grid barrier beats more
  // resident warps (H12 depth 400: 0.67 vs 0.89 ms forward, 0.84 vs 0.98 adjoint;
  // equal at depth 100/200, profiles/r02/sweep_probe_grid.txt)
  const int64_t want = tuning().sweep_grid > 0 ? tuning().sweep_grid
                       : p2p ? (int64_t)ctx().num_sms
                             : std::min<int64_t>(ctx().num_sms, (P.max_live + 255) / 256);
  const int threads = p2p ? 256 : tuning().sweep_threads;
  const int grid = coop_grid(fn, std::max<int64_t>(want * 256 / threads, 1), threads);
  const int NV = mode == kAdj ? 3 : 2;
  double *part = nullptr, *red = nullptr;
  // barrier version: [batch][block][rotation][NV]; barrier-free: [batch][warp][...]
  HSV_TRY(dalloc(&part, (p2p ? std::max<int64_t>(P.n_chunks, 1)
                              : (int64_t)nb * grid * (threads / 32)) * kBatch * NV));
  if (!p2p && tuning().sweep_bar == 1) {
    if (!P.bar) HSV_TRY(dalloc(&P.bar, 1));
    HSV_TRY_CUDA(cudaMemsetAsync(P.bar, 0, sizeof(unsigned), stream()));
  }
  if (p2p) {
    if (!P.ver) HSV_TRY(dalloc(&P.ver, sec->dim));
    HSV_TRY_CUDA(cudaMemsetAsync(P.ver, 0, sec->dim * sizeof(uint32_t), stream()));
  }
  HSV_TRY(dalloc(&red, (int64_t)k * NV));
  HSV_TRY_CUDA(cudaMemsetAsync(red, 0, (int64_t)k * NV * sizeof(double), stream()));
  BSweepArgs a{};
  a.batches = d_b; a.n_batches = nb; a.n_ops = k;
  a.n_alpha = sec->n_alpha; a.n_beta = sec->n_beta; a.Nb = sec->Nb;
  a.Ra = sec->d_Ra; a.Rb = sec->d_Rb;
  a.psi = psi; a.lam = lam; a.smap = nullptr; a.part = part; a.red = red;
  a.norm2 = norm2; a.grads = d_grads; a.err = err; a.err_val = err_val;
  a.stats = ctx().d_stats;
  a.ver = P.ver;
  a.bar = (!p2p && tuning().sweep_bar == 1) ? P.bar : nullptr;
  a.rows = P.rows; a.masks = P.masks; a.ranks = P.ranks;
  a.n_chunks = P.n_chunks; a.chunk_batch = P.chunk_batch; a.chunk_off = P.chunk_off;
  a.chunk_order = mode == kFwd ? nullptr : P.chunk_rev;
  void* params[] = {&a};
  {
    ProfScope prof(mode == kFwd ? "qeb" : "adjoint");
    HostWatch hw("k_bsweep cooperative launch");
    HSV_TRY_CUDA(cudaLaunchCooperativeKernel(fn, dim3((unsigned)grid), dim3((unsigned)threads),
                                             params, 0, stream()));
  }
  count_launch();
  dfree(d_b);
  dfree(part);
  dfree(red);
  return HSV_OK;
}

int64_t sweep_plan_support(const hsv_sector_s* s) {
  const Plan& P = plan();
  return P.sec == s && P.filtered ? P.support_rows : -1;
}

uint64_t sweep_plan_version(const hsv_sector_s* s) {
  const Plan& P = plan();
  return P.sec == s && P.filtered ? P.version : 0;
}

void release_sweep_plans(const hsv_sector_s* s) {
  Plan& P = plan();
  if (!s || P.sec == s) {
    P.clear();
    P.sec = nullptr;
  }
}

// Alpha-row occupancy flags from the structural support map (a superset of
// the nonzeros, which is all the flags promise): one warp per alpha row.
__global__ void k_smap_arow(const uint8_t* __restrict__ smap, int64_t Na, int64_t Nb,
                            uint32_t* __restrict__ flags) {
  const int64_t ra = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (ra >= Na) return;
  // no early exit: the loads are independent and stay in flight together (the
  // exit test made them a chain of ~Nb / 32 L2 round trips, 13 us at H12)
  unsigned f = 0;
  const uint8_t* __restrict__ r = smap + ra * Nb;
#pragma unroll 8
  for (int64_t j = lane; j < Nb; j += 32) f |= r[j];
  f = __any_sync(0xffffffffu, f != 0);
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
