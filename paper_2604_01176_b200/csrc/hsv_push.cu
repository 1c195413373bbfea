// K1 push path for sparse psi: scatter + radix sort + segmented reduce.
//
// The pull kernel (hsv_apply.cu) visits every row of the range, so its cost
// does not fall with the support of psi: an ADAPT state with 150 nonzeros
// costs 75% of a dense one.  Here every nonzero source row b emits one key per
// in-sector neighbour t = b ^ x_g,
//     key = (t - lo) << gbits | (g + 1)        (g + 1 = 0: the diagonal),
// the keys are radix-sorted (keys are unique: the group fixes the source) and
// one thread per target row walks its run in ascending group order,
// recomputing amp_g(t) exactly as the pull kernel does and accumulating
// fma(amp, psi[t ^ x_g], acc) in the pull kernel's own order (diagonal, then
// groups by index).  Rows never reached are exactly zero.  No atomics touch
// floating point; the key order, hence every sum, is independent of
// scheduling, so results are deterministic (and bit-identical to the
// unsplit pull kernel for the rows).
//
// Replaces spmspv over the CSR rows (sparse.py:163-219) when nnz(psi) is small;
// the SURVEY.md 8(a) "segmented sort-reduce" formulation of H|psi>.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>

#include "hsv_common.cuh"
#include "hsv_kernels.cuh"

namespace hsv {

struct PushArgs {
  ApplyArgs a;
  const int64_t* src;              // nonzero source rows (any order)
  int64_t n_src;
  uint64_t* keys;
  unsigned long long cap_keys;
  unsigned long long* n_keys;
  int gbits;
  int64_t lo;                      // first row of the range (a_lo * Nb)
  // device-sized launch (one host sync per call): the source count is read
  // from here; more than n_src sources means the keys buffer is too small and
  // the kernel writes nothing (the host re-runs it at the exact size)
  const unsigned long long* n_src_dev;
  int64_t target_items;
};

// Nonzero rows of psi, compacted in any order (the sort fixes the order).
// Stops early once more than `cap` rows were found (dense psi: use pull).
__global__ void k_push_collect(const double2* __restrict__ psi, int64_t n, int64_t cap,
                               unsigned long long* __restrict__ cnt, int64_t* __restrict__ src) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    unsigned long long seen = 0;
    if (lane == 0) seen = *reinterpret_cast<volatile unsigned long long*>(cnt);
    if (__shfl_sync(0xffffffffu, seen, 0) > (unsigned long long)cap) return;   // warp-uniform
    const int64_t i = base + threadIdx.x;
    bool nz = false;
    if (i < n) {
      const double2 v = psi[i];
      nz = v.x != 0.0 || v.y != 0.0;
    }
    const unsigned m = __ballot_sync(0xffffffffu, nz);
    unsigned long long b = 0;
    if (lane == 0 && m) b = atomicAdd(cnt, (unsigned long long)__popc(m));
    b = __shfl_sync(0xffffffffu, b, 0);
    if (nz) {
      const unsigned long long j = b + __popc(m & ((1u << lane) - 1u));
      if (j < (unsigned long long)cap) src[j] = i;
    }
  }
}

// One warp per work item = (source row, chunk of `bchunk` buckets): count its
// keys (pass 0), reserve a slot range with one atomic, write them (pass 1).
// Lanes run over the groups of a bucket.  Slot order is scheduling dependent,
// but keys are unique, so the sorted sequence is not.
template <typename W, int SH>
__global__ void __launch_bounds__(256) k_push_keys(const PushArgs p, int bchunk, int64_t n_items) {
  const ApplyArgs& a = p.a;
  if (p.n_src_dev) {   // same sizing rule as the host path, from the device count
    const int64_t n_src = (int64_t)*p.n_src_dev;
    if (n_src > p.n_src) return;
    const int64_t nbk = a.n_buckets > 1 ? a.n_buckets : 1;
    int64_t bc = (n_src * nbk + p.target_items - 1) / p.target_items;
    bc = bc < 1 ? 1 : bc > nbk ? nbk : bc;
    bchunk = (int)bc;
    n_items = n_src * ((nbk + bchunk - 1) / bchunk);
  }
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t tw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int n_chunks = (a.n_buckets + bchunk - 1) / bchunk;
  for (int64_t it = gw; it < n_items; it += tw) {
    const int64_t j = it / n_chunks;
    const int c = (int)(it - j * n_chunks);
    const int bk0 = c * bchunk, bk1 = min(a.n_buckets, bk0 + bchunk);
    const int64_t i = p.src[j];
    const int64_t ra = i / a.Nb, rb = i - ra * a.Nb;
    const uint32_t sa = __ldg(a.Sa + ra), sb = __ldg(a.Sb + rb);
    unsigned long long base = 0;
    for (int pass = 0; pass < 2; ++pass) {
      unsigned long long cnt = 0;
      if (c == 0 && a.diag && ra >= a.a_lo && ra < a.a_hi) {
        if (pass == 1 && lane == 0) p.keys[base] = (uint64_t)(i - p.lo) << p.gbits;
        ++cnt;
      }
      for (int bk = bk0; bk < bk1; ++bk) {
        const int4 B = __ldg(a.buckets + bk);
        if (__popc(sa & (uint32_t)B.x) != B.y) continue;
        const int64_t ra2 = __ldg(a.Ra + (sa ^ (uint32_t)B.x));
        if (ra2 < a.a_lo || ra2 >= a.a_hi) continue;
        for (int g0 = B.z; g0 < B.w; g0 += 32) {
          const int g = g0 + lane;
          bool v = false;
          int64_t t = 0;
          if (g < B.w) {
            const int4 G = __ldg(a.groups + g);
            if (__popc(sb & (uint32_t)G.x) == G.y) {
              t = ra2 * a.Nb + __ldg(a.Rb + (sb ^ (uint32_t)G.x));
              if (a.energy_only) {
                const double2 pt = a.psi[t];
                v = pt.x != 0.0 || pt.y != 0.0;
              } else {
                v = true;
              }
            }
          }
          const unsigned m = __ballot_sync(0xffffffffu, v);
          if (pass == 1 && v)
            p.keys[base + cnt + __popc(m & lt)] =
                ((uint64_t)(t - p.lo) << p.gbits) | (uint64_t)(g + 1);
          cnt += __popc(m);
        }
      }
      if (pass == 0) {
        if (cnt == 0) break;
        if (lane == 0) base = atomicAdd(p.n_keys, cnt);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base + cnt > p.cap_keys) break;   // host sees the overflow and falls back
      }
    }
  }
}

// One thread per sorted key; the first key of each target row sums the run.
template <typename W, int SH>
__global__ void __launch_bounds__(256) k_push_reduce(const PushArgs p,
                                                     const uint64_t* __restrict__ keys, int64_t n,
                                                     double* __restrict__ eblk) {
  const ApplyArgs& a = p.a;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double er = 0.0, ei = 0.0;
  if (i < n) {
    const uint64_t t = keys[i] >> p.gbits;
    if (i == 0 || (keys[i - 1] >> p.gbits) != t) {
      const int64_t row = p.lo + (int64_t)t;
      const int64_t ra = row / a.Nb, rb = row - ra * a.Nb;
      const uint32_t sa = __ldg(a.Sa + ra), sb = __ldg(a.Sb + rb);
      const W s = (W)sa | ((W)sb << SH);
      const uint64_t gmask = (1ull << p.gbits) - 1ull;
      const Rec<W>* __restrict__ recs = reinterpret_cast<const Rec<W>*>(a.recs);
      double2 acc = make_double2(0.0, 0.0);
      for (int64_t j = i; j < n; ++j) {
        const uint64_t k = keys[j];
        if ((k >> p.gbits) != t) break;
        const int g1 = (int)(k & gmask);
        if (g1 == 0) {   // diagonal: first in the run, as in the pull kernel
          const double d = a.diag[row];
          const double2 pv = a.psi[row];
          acc = make_double2(d * pv.x, d * pv.y);
          continue;
        }
        const int g = g1 - 1;
        const uint32_t xa = __ldg(a.gxa + g);   // alpha flip part of group g
        const int4 G = __ldg(a.groups + g);
        double amp;
        if (g < a.g_hashed) {
          amp = rec_amp<W>(ldrec(recs + g), s, a.tabs);
        } else {
          amp = 0.0;
          const uint64_t gz = __ldg(a.gsz + g);
          if (gz >> 63) {   // single-Z group, as in the pull kernel (exact)
            const SzTerm* __restrict__ sz = reinterpret_cast<const SzTerm*>(a.szt);
            for (int tt = G.z; tt < G.w; ++tt) {
              const uint4 q = __ldg(reinterpret_cast<const uint4*>(sz + tt));
              const uint32_t sb31 = SH == 16 ? ((uint32_t)s << q.z) & q.w
                                             : ((uint32_t)(s >> q.z) << 31) & q.w;
              amp += __hiloint2double((int)q.y ^ (int)sb31, (int)q.x);
            }
            const int sgn = popc(s & (W)gz) << 31;
            amp = __hiloint2double(__double2hiint(amp) ^ sgn, __double2loint(amp));
          } else {
            for (int tt = G.z; tt < G.w; ++tt) {
              const double c = __ldg(&a.terms[tt].c);
              const W z = (W)__ldg(&a.terms[tt].z);
              const int sgn = popc(s & z) << 31;
              amp += __hiloint2double(__double2hiint(c) ^ sgn, __double2loint(c));
            }
          }
        }
        const int64_t src = (int64_t)__ldg(a.Ra + (sa ^ xa)) * a.Nb +
                            __ldg(a.Rb + (sb ^ (uint32_t)G.x));
        const double2 pv = a.psi[src];
        acc.x = fma(amp, pv.x, acc.x);
        acc.y = fma(amp, pv.y, acc.y);
      }
      if (a.out) {
        double2 y = acc;
        if (a.prune > 0.0 && sqrt(y.x * y.x + y.y * y.y) < a.prune) y = make_double2(0.0, 0.0);
        put_row(a.out, a.peer_rows, a.n_peer_rows, row, y);
      }
      if (eblk) {
        const double2 pv = a.psi[row];
        er = pv.x * acc.x + pv.y * acc.y;
        ei = pv.x * acc.y - pv.y * acc.x;
      }
    }
  }
  if (eblk) {   // fixed-order block reduction
    __shared__ double sh[2][8];
    er = warp_sum(er);
    ei = warp_sum(ei);
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { sh[0][w] = er; sh[1][w] = ei; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double r = 0.0, m = 0.0;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { r += sh[0][k]; m += sh[1][k]; }
      eblk[2 * blockIdx.x] = r;
      eblk[2 * blockIdx.x + 1] = m;
    }
  }
}

static int bits_for(uint64_t n) {   // bits to hold values in [0, n)
  int b = 0;
  while (b < 64 && (n - 1) >> b) ++b;
  return n <= 1 ? 1 : b;
}

template <typename W, int SH>
static int push_t(const hsv_op_s* op, const ApplyArgs& a0, bool* done, int64_t* n_warps,
                  bool* dense_hint) {
  const hsv_sector_s* s = op->sec;
  const int mode = tuning().push;
  const int64_t rows = (a0.a_hi - a0.a_lo) * s->Nb;
  const int64_t per_src = 1 + op->n_active;
  const int gbits = bits_for((uint64_t)per_src);
  if (rows <= 0 || gbits + bits_for((uint64_t)rows) > 64) return HSV_OK;
  // Measured on H10/H12 (tools/sparse_probe.py): pull costs ~3-4 ns per row,
  // push ~0.1 ms fixed (two host syncs, sort launches) + ~0.1 ns per bound key
  // (bound = nnz * (1 + groups), about 3x the emitted keys).
  const int64_t budget = mode == 1 ? ((int64_t)1 << 27)
                                   : rows * tuning().push_keys - ((int64_t)1 << 20);
  const int64_t cap_src = budget / per_src;
  if (cap_src < 1) return HSV_OK;
  if (dense_hint && *dense_hint && mode != 1) return HSV_OK;

  PushArgs p{};
  p.a = a0;
  p.gbits = gbits;
  p.lo = a0.a_lo * s->Nb;
  p.target_items = (int64_t)ctx().num_sms * 32;   // about 32 warps' worth of items per SM
  int64_t* src = nullptr;
  unsigned long long* cnt = nullptr;
  HSV_TRY(dalloc(&src, cap_src));
  HSV_TRY(dalloc(&cnt, 2));
  HSV_TRY_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), stream()));
  unsigned long long h[2] = {0, 0};
  {
    ProfScope prof("push_collect");
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((s->dim + 255) / 256,
                                                                (int64_t)ctx().num_sms * 8));
    k_push_collect<<<(unsigned)grid, 256, 0, stream()>>>(a0.psi, s->dim, cap_src, cnt, src);
  }
  count_launch();
  HSV_CHECK_LAUNCH();
  p.src = src;
  p.n_keys = cnt + 1;
  const int nbk = (int)std::max<int64_t>(op->n_buckets, 1);
  auto launch_keys = [&](bool device_sized) -> int {
    ProfScope prof("push");
    int bchunk = 1;
    int64_t n_items = 0, grid = (int64_t)ctx().num_sms * 8;
    if (!device_sized) {
      if (p.n_src == 0) return HSV_OK;
      bchunk = (int)std::min<int64_t>(
          nbk, std::max<int64_t>(1, (p.n_src * nbk + p.target_items - 1) / p.target_items));
      n_items = p.n_src * ((nbk + bchunk - 1) / bchunk);
      grid = std::min<int64_t>((n_items + 7) / 8, grid);
    }
    k_push_keys<W, SH><<<(unsigned)std::max<int64_t>(grid, 1), 256, 0, stream()>>>(p, bchunk,
                                                                                   n_items);
    count_launch();
    HSV_CHECK_LAUNCH();
    return HSV_OK;
  };
  // Source count of the previous call (ADAPT evaluations come in runs of
  // similar supports): size the keys buffer for 4x that and let the keys kernel
  // read the real count on the device -- one host sync instead of two.
  static int64_t last_nsrc = -1;
  uint64_t *keys = nullptr, *keys2 = nullptr;
  void* tmp = nullptr;
  bool sized = false;
  // an allocation the push path cannot get is not an error: free what it holds
  // and let launch_apply run the pull kernel, which needs no scratch keys
#define HSV_PUSH_ALLOC(ptr, n)                                                   \
  do {                                                                           \
    if (dalloc((ptr), (n)) != HSV_OK) {                                          \
      dfree(keys); dfree(keys2); dfree(reinterpret_cast<char*>(tmp));            \
      dfree(src); dfree(cnt);                                                    \
      return HSV_OK;                                                             \
    }                                                                            \
  } while (0)
  if (last_nsrc >= 0) {
    const int64_t guess = std::min<int64_t>(cap_src, std::max<int64_t>(4 * last_nsrc, 64));
    p.n_src = guess;
    p.n_src_dev = cnt;
    p.cap_keys = (unsigned long long)(guess * per_src);
    HSV_PUSH_ALLOC(&keys, guess * per_src);
    p.keys = keys;
    HSV_TRY(launch_keys(true));
    HostWatch hw("push count D2H");
    HSV_TRY_CUDA(cudaMemcpyAsync(h, cnt, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                 stream()));
    HSV_TRY(stream_sync());
    sized = h[0] <= (unsigned long long)guess;
    if (!sized) {
      dfree(keys);
      keys = nullptr;
    }
  } else {
    HSV_TRY_CUDA(cudaMemcpyAsync(h, cnt, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                 stream()));
    HSV_TRY(stream_sync());
  }
  last_nsrc = (int64_t)std::min<unsigned long long>(h[0], (unsigned long long)cap_src + 1);
  if (h[0] > (unsigned long long)cap_src) {   // dense psi
    if (dense_hint) *dense_hint = true;
    dfree(keys);
    dfree(src);
    dfree(cnt);
    return HSV_OK;
  }
  if (!sized) {   // exact size: the second sync of the first call (or of a larger support)
    p.n_src = (int64_t)h[0];
    p.n_src_dev = nullptr;
    p.cap_keys = (unsigned long long)(p.n_src * per_src);
    HSV_PUSH_ALLOC(&keys, std::max<int64_t>(1, p.n_src * per_src));
    p.keys = keys;
    HSV_TRY_CUDA(cudaMemsetAsync(cnt + 1, 0, sizeof(unsigned long long), stream()));
    HSV_TRY(launch_keys(false));
    HSV_TRY_CUDA(cudaMemcpyAsync(h + 1, cnt + 1, sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, stream()));
    HSV_TRY(stream_sync());
  }
  const int64_t nk = (int64_t)h[1];
  // h[1] > cap_keys cannot happen (per-source bound); more than INT_MAX keys
  // would truncate CUB's int item count: both go to the pull kernel
  if (h[1] > p.cap_keys || nk > (int64_t)INT32_MAX) {
    dfree(keys); dfree(src); dfree(cnt);
    return HSV_OK;
  }
  {
    ProfScope prof("push");
    if (a0.out)
      HSV_TRY_CUDA(cudaMemsetAsync(a0.out + p.lo, 0, rows * sizeof(double2), stream()));
    const int end_bit = gbits + bits_for((uint64_t)rows);
    const uint64_t* sorted = keys;
    if (nk > 1) {
      HSV_PUSH_ALLOC(&keys2, nk);
      size_t tmp_bytes = 0;
      cub::DoubleBuffer<uint64_t> db(keys, keys2);
      HSV_TRY_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, db, (int)nk, 0, end_bit,
                                                  stream()));
      HSV_PUSH_ALLOC(reinterpret_cast<char**>(&tmp), tmp_bytes);
      HSV_TRY_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, db, (int)nk, 0, end_bit,
                                                  stream()));
      sorted = db.Current();
    }
    const int64_t nblk = (nk + 255) / 256;
    double* eblk = nullptr;
    if (a0.epart) HSV_TRY(dalloc(&eblk, 2 * std::max<int64_t>(nblk, 1)));
    if (nk > 0) {
      k_push_reduce<W, SH><<<(unsigned)nblk, 256, 0, stream()>>>(p, sorted, nk, eblk);
      count_launch();
      HSV_CHECK_LAUNCH();
    }
    if (a0.epart) HSV_TRY(reduce_sum_f64(eblk, nblk, 2, 2, a0.epart));
    dfree(eblk);
  }
#undef HSV_PUSH_ALLOC
  dfree(reinterpret_cast<char*>(tmp));
  dfree(keys2);
  dfree(keys);
  dfree(src);
  dfree(cnt);
  if (n_warps) *n_warps = 1;
  *done = true;
  return HSV_OK;
}

int launch_push(const hsv_op_s* op, const ApplyArgs& a, bool* done, int64_t* n_warps,
                bool* dense_hint) {
  *done = false;
  if (tuning().push == 0) return HSV_OK;
  // rows the push path never reaches are zeroed locally only; with peer sinks
  // (fused all-gather) every row must be stored, which the pull kernel does
  if (a.n_peer_rows > 0) return HSV_OK;
  if (op->sec->wide) return push_t<uint64_t, 32>(op, a, done, n_warps, dense_hint);
  return push_t<uint32_t, 16>(op, a, done, n_warps, dense_hint);
}

}  // namespace hsv
