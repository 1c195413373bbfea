// Matrix-free Pauli operator: upload/validation (replaces the CSR assembly of
// svengine.py:115-171) and the K1 pull kernel computing H|psi> and
// <psi|H|psi> (replaces spmspv + dot, sparse.py:163-219).
//
// Row b of H|psi> is   y_b = D_b psi_b + sum_{groups g, b^x_g in sector} amp_g(b) psi_{b^x_g}
// with amp_g(b) = sum_{t in g, ascending z} c_t (-1)^{popcount(b & z_t)}, the
// same sequential sum the reference forms per x-group (svengine.py:137-146),
// so every matrix element is bit-identical to the reference CSR value.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>

#include <cub/cub.cuh>

#include "hsv_common.cuh"
#include "hsv_kernels.cuh"

namespace hsv {

// --------------------------------------------------------- leak + diagonal
// For every off-diagonal x-group, max |amp_g(b)| over sector rows b whose
// image b^x leaves the sector (svengine.py:153-160).
template <typename W, int SH>
__global__ void k_leak(const uint32_t* __restrict__ Sa, const uint32_t* __restrict__ Sb,
                       int64_t Na, int64_t Nb, const uint32_t* __restrict__ gxa,
                       const uint32_t* __restrict__ gxb, const int32_t* __restrict__ gha,
                       const int32_t* __restrict__ ghb, const int32_t* __restrict__ gt0,
                       const int32_t* __restrict__ gt1, int n_groups,
                       const Term* __restrict__ terms, unsigned long long* __restrict__ leak) {
  const int64_t ra = blockIdx.y;
  const int64_t rb = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool live = rb < Nb;
  const uint32_t sa = Sa[ra];
  const uint32_t sb = live ? Sb[rb] : 0u;
  const W s = (W)sa | ((W)sb << SH);
  for (int g = 0; g < n_groups; ++g) {
    const bool aok = __popc(sa & gxa[g]) == gha[g];
    const bool inval = live && !(aok && __popc(sb & gxb[g]) == ghb[g]);
    double m = 0.0;
    if (inval) {
      double amp = 0.0;
      for (int t = gt0[g]; t < gt1[g]; ++t) {
        const Term T = terms[t];
        amp += (popc(s & (W)T.z) & 1) ? -T.c : T.c;
      }
      m = fabs(amp);
    }
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0 && m > 0.0)
      atomicMax(&leak[g], (unsigned long long)__double_as_longlong(m));
  }
}

template <typename W, int SH>
__global__ void k_diag(const uint32_t* __restrict__ Sa, const uint32_t* __restrict__ Sb,
                       int64_t Na, int64_t Nb, const Term* __restrict__ terms, int t0, int t1,
                       double* __restrict__ diag) {
  // the diagonal terms staged in shared memory (H16: 529 terms, 8.5 KB); the
  // sum stays sequential in term order (svengine.py:137-146)
  extern __shared__ Term tsh[];
  const int nt = t1 - t0;
  for (int i = threadIdx.x; i < nt; i += blockDim.x) tsh[i] = terms[t0 + i];
  __syncthreads();
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= Na * Nb) return;
  const int64_t ra = idx / Nb, rb = idx - ra * Nb;
  const W s = (W)Sa[ra] | ((W)Sb[rb] << SH);
  double amp = 0.0;
#pragma unroll 4
  for (int t = 0; t < nt; ++t) {
    const Term T = tsh[t];
    const int sgn = popc(s & (W)T.z) << 31;   // exact +-c: flip the sign bit
    amp += __hiloint2double(__double2hiint(T.c) ^ sgn, __double2loint(T.c));
  }
  diag[idx] = amp;
}

// Structural nonzeros per row (== reference CSR row lengths) and, in a second
// pass, the (column, value) pairs of each row.
template <typename W, int SH>
__global__ void k_csr_rows(const uint32_t* __restrict__ Sa, const uint32_t* __restrict__ Sb,
                           const uint32_t* __restrict__ Ra, const uint32_t* __restrict__ Rb,
                           int64_t Na, int64_t Nb, const int4* __restrict__ buckets, int n_buckets,
                           const int4* __restrict__ groups, const Term* __restrict__ terms,
                           const double* __restrict__ diag, const int64_t* __restrict__ perm,
                           int64_t* __restrict__ counts, const int64_t* __restrict__ offsets,
                           int64_t* __restrict__ cols, double* __restrict__ vals) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= Na * Nb) return;
  const int64_t ra = idx / Nb, rb = idx - ra * Nb;
  const uint32_t sa = Sa[ra], sb = Sb[rb];
  const W s = (W)sa | ((W)sb << SH);
  const int64_t row = perm[idx];
  int64_t n = 0, o = offsets ? offsets[row] : 0;
  if (diag && diag[idx] != 0.0) {
    if (offsets) { cols[o + n] = row; vals[o + n] = diag[idx]; }
    ++n;
  }
  for (int bk = 0; bk < n_buckets; ++bk) {
    const int4 B = buckets[bk];
    if (__popc(sa & (uint32_t)B.x) != B.y) continue;
    const int64_t base = (int64_t)Ra[sa ^ (uint32_t)B.x] * Nb;
    for (int g = B.z; g < B.w; ++g) {
      const int4 G = groups[g];
      if (__popc(sb & (uint32_t)G.x) != G.y) continue;
      double amp = 0.0;
      for (int t = G.z; t < G.w; ++t) {
        const Term T = terms[t];
        amp += (popc(s & (W)T.z) & 1) ? -T.c : T.c;
      }
      if (amp == 0.0) continue;
      if (offsets) {
        cols[o + n] = perm[base + Rb[sb ^ (uint32_t)G.x]];
        vals[o + n] = amp;
      }
      ++n;
    }
  }
  if (!offsets) counts[row] = n;
}

// --------------------------------------------------------------- K1 apply
// Warp-granular static schedule: a unit is 32*R consecutive beta rows of one
// alpha row, so the alpha half of every sector test is warp-uniform and whole
// buckets are skipped without divergence.  Each lane owns R rows.
//
// Matrix element of an x-local group (every z_t ^ z_0 inside the flip mask x):
//   amp(b) = (-1)^popcount(b & z_0) * A_g[h(b & x)],
// A_g precomputed on the host in the reference's sequential term order (exact:
// IEEE rounding is symmetric under negation) and h a per-group perfect
// multiply-shift hash of the in-sector patterns of b on x.  Other groups
// (singles carrying number-operator Z's) run the sequential term loop.
template <typename W, int SH, int R, int MINB, int RM, int LM, int EM = 0>
__global__ void __launch_bounds__(256, MINB) k_apply(const ApplyArgs a) {
  // EM (SELL build): 0 accumulate; 1 count the (row, split) entries with a
  // nonzero matrix element; 2 write them -- (partner row, element) in exactly
  // the order the accumulation adds them
  static_assert(EM == 0 || LM == 0, "the SELL build runs over the full row range");
  constexpr bool RS = RM == 1;
  static_assert(!(LM && RM == 2), "row-list mode reads partner ranks from Rb0");
  const int lane = threadIdx.x & 31;
  // Pass-1 partner beta rank rank(Sb[rb] ^ xb), by RM:
  //   0: Rb0[Sb[rb] ^ xb]        (random 4-byte gather over the 2^norb table)
  //   2: bperm[slot(xb) + rb]    (per-xb rank permutation, one coalesced 128-byte
  //                               line per warp: fewer L1 wavefronts per pair)
  // RM 1 (RS): the pass-1 beta rank table Rb0 (2^norb words) is copied to shared
  // memory once per CTA, so the per-(row, group) rank lookup is an LDS with a
  // 32-bit address instead of a 64-bit-addressed LDG
  extern __shared__ uint32_t rb0_sh[];
  if (RS) {
    for (uint32_t i = threadIdx.x; i < (uint32_t)a.rb0_n; i += blockDim.x) rb0_sh[i] = __ldg(a.Rb0 + i);
    __syncthreads();
  }
  // 32-bit indices throughout (dim < 2^32 is checked at launch): fewer
  // registers and integer instructions than 64-bit row arithmetic
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t tw = (gridDim.x * blockDim.x) >> 5;
  // LM (K1r): the unit count comes from the device-built list (no host sync)
  const uint32_t units = LM ? __ldg(a.d_units) * (uint32_t)a.nsplit : (uint32_t)a.units;
  const uint32_t Nb = (uint32_t)a.Nb;
  // energy partials live in shared memory, not in registers across the group loop
  __shared__ double esh[8][2];
  if (lane == 0) { esh[threadIdx.x >> 5][0] = 0.0; esh[threadIdx.x >> 5][1] = 0.0; }
  // Static schedule.  Interleaved (default): warp gw takes work units gw,
  // gw + tw, ..., so the warps of an SM work on neighbouring row units of one
  // alpha row and the same bucket range at the same time and share the partner
  // rows they gather in L1 (and in L2 when psi is far larger than L2).
  // Contiguous unit blocks per warp remain as a tuning alternative.
  // Dynamic (default, interleave == 2): a warp takes the next work unit from
  // a global counter when it finishes one.  Units are still handed out in
  // order, so the warps of an SM stay on neighbouring units, but a slow unit no
  // longer holds up a fixed share of later ones (H12 2.71 -> 2.39 ms, H14 -11%).
  const bool dyn = a.interleave == 2;
  auto grab = [&]() -> uint32_t {
    uint32_t v = 0;
    if (lane == 0) v = atomicAdd(a.ucounter, 1u);
    return __shfl_sync(0xffffffffu, v, 0);
  };
  const uint32_t u_begin = dyn ? grab() : a.interleave ? gw : (uint32_t)((uint64_t)gw * units / tw);
  const uint32_t u_end = a.interleave ? units : (uint32_t)((uint64_t)(gw + 1) * units / tw);
  const uint32_t u_step = a.interleave ? tw : 1u;
  for (uint32_t uw = u_begin; uw < u_end; uw = dyn ? grab() : uw + u_step) {
    // a work unit = (row unit, bucket split), split-major: neighbouring work
    // units are neighbouring row units with the same bucket range (measured
    // -6% at H12 against unit-major)
    const uint32_t units1 = units / (uint32_t)a.nsplit;
    const int sp = (int)(uw / units1);
    const uint32_t u = uw - (uint32_t)sp * units1;
    const int bk0 = a.split_bk ? __ldg(a.split_bk + sp) : 0;
    const int bk1 = a.split_bk ? __ldg(a.split_bk + sp + 1) : a.n_buckets;
    uint32_t ra, rb0, lcnt = 0u;
    const uint32_t* lrow = nullptr;
    if (LM) {   // K1r: the lane's rows are list entries rb0, rb0 + 32, ... of alpha row ra
      const uint2 ut = __ldg(a.utab + u);
      ra = (uint32_t)a.a_lo + ut.x;
      rb0 = ut.y * (32 * R) + lane;
      lcnt = __ldg(a.rcnt + ut.x);
      lrow = a.rlist + (size_t)ut.x * Nb;
    } else {
      const uint32_t ur = u / (uint32_t)a.upr;
      ra = (uint32_t)a.a_lo + ur;
      rb0 = (u - ur * (uint32_t)a.upr) * (32 * R) + lane;
    }
    const uint32_t sa = __ldg(a.Sa + ra);
    const uint32_t rowbase = ra * Nb;
    W s[R];
    uint32_t sb[R];
    double2 acc[R];
    uint64_t epos[R];   // EM: entry count (1) or next slot (2) of the lane's (row, split)
    unsigned live = 0u, inrm = 0u;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const uint32_t rb = LM ? (rb0 + k * 32 < lcnt ? __ldg(lrow + rb0 + k * 32) : Nb) : rb0 + k * 32;
      const bool inr = rb < Nb;
      if (LM) inrm |= inr ? (1u << k) : 0u;
      sb[k] = inr ? __ldg(a.Sb + rb) : 0u;
      s[k] = (W)sa | ((W)sb[k] << SH);
      if (EM) {
        live |= inr ? (1u << k) : 0u;
        const uint64_t rl = (uint64_t)(rowbase + rb - (uint32_t)a.a_lo * Nb);
        epos[k] = EM == 1 ? 0ull
                          : (inr ? __ldg(a.sell_off + (rl >> 5) * (uint64_t)a.nsplit + sp) + (rl & 31u)
                                 : 0ull);
        continue;
      }
      const double2 pv = inr ? a.psi[rowbase + rb] : make_double2(0.0, 0.0);
      const bool lv = inr && (!a.energy_only || pv.x != 0.0 || pv.y != 0.0);
      const double d = (a.diag && lv && sp == 0) ? a.diag[rowbase + rb] : 0.0;
      acc[k] = make_double2(d * pv.x, d * pv.y);
      live |= lv ? (1u << k) : 0u;
    }
    if (__any_sync(0xffffffffu, live != 0u)) {
      // pass 1: x-local groups, amp = sign * table[hash(pattern)]
      for (int bk = bk0; bk < min(bk1, a.n_buckets_h); ++bk) {
        const int4 B = __ldg(a.buckets + bk);
        if (__popc(sa & (uint32_t)B.x) != B.y) continue;
        const uint32_t ra2 = __ldg(a.Ra + (sa ^ (uint32_t)B.x));
        if (a.arow && !__ldg(a.arow + ra2)) continue;   // partner alpha row all zero
        // 32-bit row offsets (dim < 2^32, checked at launch) and no record
        // prefetch: both free registers the compiler otherwise spends on
        // re-deriving addresses (measured -6.6% at H12)
        const uint32_t rowoff = ra2 * (uint32_t)a.Nb;
        const Rec<W>* __restrict__ rp = reinterpret_cast<const Rec<W>*>(a.recs);
        for (int g = B.z; g < B.w; ++g) {
          const Rec<W> cur = ldrec(rp + g);
          const uint32_t xb = cur.xb;
          // No per-lane sector test: the table holds 0 for out-of-sector beta
          // patterns and Rb0 maps out-of-sector strings to rank 0 (a harmless
          // in-row gather), so such rows add exactly +-0 (H14 -7%, H12 -1%).
          const int shift = (int)((cur.meta >> 8) & 0xffu);
#pragma unroll
          for (int k = 0; k < R; ++k) {
            const uint32_t h = cur.tab + (uint32_t)((W)((s[k] & cur.xm) * cur.mul) >> shift);
            const double A = __ldg(a.tabs + h);
            const int sgn = popc(s[k] & cur.z0) << 31;
            const double amp = __hiloint2double(__double2hiint(A) ^ sgn, __double2loint(A));
            const uint32_t rk = RM == 2 ? __ldg(a.bperm + (cur.pad0 + rb0 + k * 32))
                                : RS ? rb0_sh[sb[k] ^ xb] : __ldg(a.Rb0 + (uint32_t)(sb[k] ^ xb));
            if (EM) {   // out-of-sector partners and cancelled sums hold A = 0: no entry
              if (A != 0.0 && ((live >> k) & 1u)) {
                if (EM == 2) {
                  a.sell_cols[epos[k]] = rowoff + rk;
                  a.sell_amps[epos[k]] = amp;
                  epos[k] += 32;
                } else {
                  ++epos[k];
                }
              }
              continue;
            }
            const double2 p = a.psi[rowoff + rk];
            acc[k].x = fma(amp, p.x, acc[k].x);
            acc[k].y = fma(amp, p.y, acc[k].y);
          }
        }
      }
      // pass 2: remaining groups, sequential term loop in reference order
      for (int bk = max(bk0, a.n_buckets_h); bk < bk1; ++bk) {
        const int4 B = __ldg(a.buckets + bk);
        if (__popc(sa & (uint32_t)B.x) != B.y) continue;
        const uint32_t ra2 = __ldg(a.Ra + (sa ^ (uint32_t)B.x));
        if (a.arow && !__ldg(a.arow + ra2)) continue;
        const uint32_t rowoff = ra2 * (uint32_t)a.Nb;
        for (int g = B.z; g < B.w; ++g) {
          const int4 G = __ldg(a.groups + g);
          const uint32_t xb = (uint32_t)G.x;
          unsigned v = 0u;
#pragma unroll
          for (int k = 0; k < R; ++k)
            v |= ((live >> k) & 1u) && __popc(sb[k] & xb) == G.y ? (1u << k) : 0u;
          if (!__any_sync(0xffffffffu, v != 0u)) continue;
          double amp[R];
#pragma unroll
          for (int k = 0; k < R; ++k) amp[k] = 0.0;
          const uint64_t gz = __ldg(a.gsz + g);
          if (gz >> 63) {   // single-Z group: one shift + one LOP per term and row
            const SzTerm* __restrict__ sz = reinterpret_cast<const SzTerm*>(a.szt);
            for (int t = G.z; t < G.w; ++t) {
              const uint4 q = __ldg(reinterpret_cast<const uint4*>(sz + t));
              const int chi = (int)q.y;
#pragma unroll
              for (int k = 0; k < R; ++k) {
                const uint32_t sb31 = SH == 16 ? ((uint32_t)s[k] << q.z) & q.w
                                               : ((uint32_t)(s[k] >> q.z) << 31) & q.w;
                amp[k] += __hiloint2double(chi ^ (int)sb31, (int)q.x);
              }
            }
#pragma unroll
            for (int k = 0; k < R; ++k) {   // common sign (-1)^popc(s & z0): exact
              const int sgn = popc(s[k] & (W)gz) << 31;
              amp[k] = __hiloint2double(__double2hiint(amp[k]) ^ sgn, __double2loint(amp[k]));
            }
          } else {
            for (int t = G.z; t < G.w; ++t) {
              const double c = __ldg(&a.terms[t].c);
              const W z = (W)__ldg(&a.terms[t].z);
#pragma unroll
              for (int k = 0; k < R; ++k) {
                const int sgn = popc(s[k] & z) << 31;   // exact +-c: flip the sign bit
                amp[k] += __hiloint2double(__double2hiint(c) ^ sgn, __double2loint(c));
              }
            }
          }
#pragma unroll
          for (int k = 0; k < R; ++k) {
            if ((v >> k) & 1u) {
              if (EM) {
                if (amp[k] != 0.0) {
                  if (EM == 2) {
                    a.sell_cols[epos[k]] = rowoff + __ldg(a.Rb + (sb[k] ^ xb));
                    a.sell_amps[epos[k]] = amp[k];
                    epos[k] += 32;
                  } else {
                    ++epos[k];
                  }
                }
                continue;
              }
              const double2 p = a.psi[rowoff + __ldg(a.Rb + (sb[k] ^ xb))];
              acc[k].x = fma(amp[k], p.x, acc[k].x);
              acc[k].y = fma(amp[k], p.y, acc[k].y);
            }
          }
        }
      }
    }
    if (EM == 1) {
#pragma unroll
      for (int k = 0; k < R; ++k)
        if (rb0 + k * 32 < Nb)
          a.sell_cnt[(uint64_t)(rowbase + rb0 + k * 32 - (uint32_t)a.a_lo * Nb) * a.nsplit + sp] =
              (uint32_t)epos[k];
    }
    if (EM) continue;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (LM ? !((inrm >> k) & 1u) : rb0 + k * 32 >= Nb) continue;
      const uint32_t rb = LM ? __ldg(a.Rb + sb[k]) : rb0 + k * 32;
      if (a.out) {
        if (a.nsplit > 1) {   // partial row, combined in split order by k_combine_splits
          a.ypart[(int64_t)sp * a.part_stride + (rowbase + rb - (uint32_t)a.a_lo * Nb)] = acc[k];
        } else {
          double2 y = acc[k];
          if (a.prune > 0.0 && sqrt(y.x * y.x + y.y * y.y) < a.prune) y = make_double2(0.0, 0.0);
          put_row(a.out, a.peer_rows, a.n_peer_rows, rowbase + rb, y);
        }
      }
    }
    if (a.epart) {   // this unit's <psi|H psi> share, added in unit order (fixed)
      double er = 0.0, ei = 0.0;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if ((LM ? (inrm >> k) & 1u : rb0 + k * 32 < Nb) && ((live >> k) & 1u)) {
          const uint32_t rb = LM ? __ldg(a.Rb + sb[k]) : rb0 + k * 32;
          const double2 pv = a.psi[rowbase + rb];
          er += pv.x * acc[k].x + pv.y * acc[k].y;
          ei += pv.x * acc[k].y - pv.y * acc[k].x;
        }
      }
      er = warp_sum(er);
      ei = warp_sum(ei);
      if (dyn) {   // which warp ran a unit varies: per-unit partials, summed in unit order
        if (lane == 0) { a.upart[2 * uw] = er; a.upart[2 * uw + 1] = ei; }
      } else if (lane == 0) {
        esh[threadIdx.x >> 5][0] += er;
        esh[threadIdx.x >> 5][1] += ei;
      }
    }
  }
  if (a.epart && lane == 0 && !dyn) {
    a.epart[2 * gw] = esh[threadIdx.x >> 5][0];
    a.epart[2 * gw + 1] = esh[threadIdx.x >> 5][1];
  }
}

// Sum the per-split partial rows in split order (fixed), then the drop rule.
// Rows go to out[off + i] (and to the peer buffers, see put_row).
__global__ void k_combine_splits(const double2* __restrict__ part, int S, int64_t rows,
                                 double2* __restrict__ out, int64_t off, double prune,
                                 double2* const* peers, int n_peers) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows) return;
  double2 y = part[i];
  for (int s = 1; s < S; ++s) {
    const double2 p = part[s * rows + i];
    y.x += p.x;
    y.y += p.y;
  }
  if (prune > 0.0 && sqrt(y.x * y.x + y.y * y.y) < prune) y = make_double2(0.0, 0.0);
  put_row(out, peers, n_peers, off + i, y);
}

void launch_combine_splits(const double2* part, int S, int64_t rows, double2* out, int64_t off,
                           double prune, double2* const* peers, int n_peers) {
  k_combine_splits<<<(unsigned)((rows + 255) / 256), 256, 0, stream()>>>(part, S, rows, out, off,
                                                                           prune, peers, n_peers);
}

// K1r: rows marked in smap get the sum of their split partials (split order,
// as k_combine_splits), every other row an exact zero.
__global__ void k_combine_splits_map(const double2* __restrict__ part, int S, int64_t rows,
                                     double2* __restrict__ out, int64_t off,
                                     const uint8_t* __restrict__ smap, double2* const* peers,
                                     int n_peers) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows) return;
  double2 y = make_double2(0.0, 0.0);
  if (smap[off + i]) {
    y = part[i];
    for (int s = 1; s < S; ++s) {
      const double2 p = part[s * rows + i];
      y.x += p.x;
      y.y += p.y;
    }
  }
  put_row(out, peers, n_peers, off + i, y);
}

void launch_combine_splits_map(const double2* part, int S, int64_t rows, double2* out,
                               int64_t off, const uint8_t* smap, double2* const* peers,
                               int n_peers) {
  k_combine_splits_map<<<(unsigned)((rows + 255) / 256), 256, 0, stream()>>>(
      part, S, rows, out, off, smap, peers, n_peers);
}

// Point a launch at the split table for S parts (virtual buckets + cuts).
void use_split_table(const hsv_op_s* op, int St, ApplyArgs& a) {
  if (St <= 1) {
    a.split_bk = nullptr;
    return;
  }
  const SplitTable& T = op->split[__builtin_ctz((unsigned)St) - 1];
  a.buckets = op->d_vbuckets + T.vb_off;
  a.n_buckets = T.nb;
  a.n_buckets_h = T.nbh;
  a.split_bk = op->d_splits + T.cut_off;
}

template <typename W, int SH, int R, int MINB, int RM = 0, int LM = 0, int EM = 0>
static int launch_apply_t(const hsv_op_s* op, const ApplyArgs& a0, int64_t* n_warps_out,
                          const uint8_t* smap = nullptr, int64_t list_units = 0) {
  ApplyArgs a = a0;
  a.upr = (int)((a.Nb + 32 * R - 1) / (32 * R));
  // units of the full row range: the split count S below depends on it only, so
  // the row-list launch (LM) picks the same S as the full one and its rows are
  // bit-identical to the full kernel's
  const int64_t units1_full = (a.a_hi - a.a_lo) * a.upr;
  const int64_t units1 = LM ? list_units : units1_full;
  const size_t smem = RM == 1 ? (size_t)a.rb0_n * sizeof(uint32_t) : 0;
  int occ = 0;
  {
    HostWatch hw("k_apply attributes");
    if (smem > 48 * 1024)
      HSV_TRY_CUDA(cudaFuncSetAttribute(k_apply<W, SH, R, MINB, RM, LM, EM>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    HSV_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_apply<W, SH, R, MINB, RM, LM, EM>, 256, smem));
  }
  occ = std::max(occ, 1);
  const int64_t max_warps = (int64_t)ctx().num_sms * occ * 8;
  // Split the bucket range of each row unit.  Split-major unit order keeps the
  // warps of the machine on one bucket range at a time (tables and partner rows
  // shared in L1/L2), so 8 parts win even when row units are plentiful (H14
  // 57.3 against 57.9 ms unsplit, H16 1.40 against 1.43 s); more parts, up to
  // 32, while that leaves fewer than 8 units per warp (rank shards: H12 / 8
  // 0.354 against 0.42 ms with the earlier at-most-8 rule).  Capped so the
  // partial rows stay under 32 GB.
  int S = a0.nsplit > 0 ? a0.nsplit : tuning().apply_split;
  if (S <= 0) {
    S = 8;
    while (S < 32 && units1_full * S < 8 * max_warps) S *= 2;
    const int64_t rows_all = (a.a_hi - a.a_lo) * a.Nb;
    while (S > 1 && a.out && S * rows_all * (int64_t)sizeof(double2) > (32ll << 30)) S /= 2;
  }
  if (!a0.split_bk) S = 1;
  // K1r with peer stores: the combine pass must write (zero) every row to the peers
  if (LM && S == 1 && a.n_peer_rows > 0 && a0.split_bk) S = 2;
  a.nsplit = S;
  use_split_table(op, S, a);
  // interleaved unless forced off (measured best at H12 and H14)
  const int il = tuning().apply_interleave;   // -1 auto (= 2), 0 contiguous, 1 interleaved, 2 dynamic
  a.interleave = LM || il < 0 ? 2 : il;       // the list mode's unit count is on the device
  a.units = units1 * S;
  int64_t grid = max_warps / 8;
  const int64_t need = (a.units + 7) / 8;
  grid = std::max<int64_t>(1, std::min(grid, need));
  if (n_warps_out) *n_warps_out = grid * 8;
  if (a.units == 0) return HSV_OK;
  unsigned int* ucounter = nullptr;
  double* upart = nullptr;
  if (a.interleave == 2) {
    HSV_TRY(dalloc(&ucounter, 1));
    HSV_TRY_CUDA(cudaMemsetAsync(ucounter, 0, sizeof(unsigned), stream()));
    a.ucounter = ucounter;
    if (a.epart) {
      HSV_TRY(dalloc(&upart, 2 * a.units));
      if (LM)   // units past the device count leave their partials untouched
        HSV_TRY_CUDA(cudaMemsetAsync(upart, 0, 2 * a.units * sizeof(double), stream()));
      a.upart = upart;
    }
    if (n_warps_out) *n_warps_out = 1;   // the unit partials are reduced into epart[0..1] below
  }
  const int64_t rows = (a.a_hi - a.a_lo) * a.Nb;
  double2* ypart = nullptr;
  if (S > 1 && a.out) {
    HSV_TRY(dalloc(&ypart, S * rows));
    a.ypart = ypart;
    a.part_stride = rows;
  }
  if (LM && a.out && !ypart)   // rows outside the list are exact zeros
    HSV_TRY_CUDA(cudaMemsetAsync(a.out + a.a_lo * a.Nb, 0, rows * sizeof(double2), stream()));
  {
    ProfScope prof(EM ? "sell_build" : LM ? "apply_rows" : "apply");
    HostWatch hw("k_apply launch");
    k_apply<W, SH, R, MINB, RM, LM, EM><<<(unsigned)grid, 256, smem, stream()>>>(a);
    if (ypart && LM)
      launch_combine_splits_map(ypart, S, rows, a.out, a.a_lo * a.Nb, smap, a.peer_rows,
                                a.n_peer_rows);
    else if (ypart)
      launch_combine_splits(ypart, S, rows, a.out, a.a_lo * a.Nb, a.prune, a.peer_rows,
                            a.n_peer_rows);
  }
  count_launch(ypart ? 2 : 1);
  HSV_CHECK_LAUNCH();
  if (upart) HSV_TRY(reduce_sum_f64(upart, a.units, 2, 2, a.epart));
  dfree(upart);
  dfree(ucounter);
  dfree(ypart);
  return HSV_OK;
}

// Rows per lane of the register-row K1 (launch_apply's automatic choice).
static int k1_auto_r(const hsv_sector_s* s, int64_t a_lo, int64_t a_hi) {
  const int64_t units8 = (a_hi - a_lo) * ((s->Nb + 255) / 256);
  const int64_t warps8 = (int64_t)ctx().num_sms * 2 * 8;
  const int64_t units4 = (a_hi - a_lo) * ((s->Nb + 127) / 128);
  const int64_t warps4 = (int64_t)ctx().num_sms * 3 * 8;
  const bool dyn = tuning().apply_interleave < 0 || tuning().apply_interleave == 2;
  return (dyn ? 32 * units8 >= warps8 : 4 * units8 >= 3 * warps8) ? 8 : units4 >= warps4 ? 4 : 2;
}

// The bucket split count the default register-row K1 uses for rows
// [a_lo, a_hi) (launch_apply_t's rule; its occupancy is the launch-bounds
// minimum: R = 8 -> 2, 4 -> 3, 2 -> 4 blocks of 256 per SM).  Every kernel that
// must reproduce K1's rows bit for bit (K1r, K1v) uses this S.
int k1_default_split(const hsv_op_s* op, int64_t a_lo, int64_t a_hi, bool has_out) {
  if (!op->d_splits) return 1;
  if (tuning().apply_split > 0) return tuning().apply_split;
  const hsv_sector_s* s = op->sec;
  const int R = tuning().apply_r > 0 ? tuning().apply_r : k1_auto_r(s, a_lo, a_hi);
  const int occ = R == 8 ? 2 : R == 4 ? 3 : 4;
  const int64_t units1 = (a_hi - a_lo) * ((s->Nb + 32 * R - 1) / (32 * R));
  const int64_t max_warps = (int64_t)ctx().num_sms * occ * 8;
  int S = 8;
  while (S < 32 && units1 * S < 8 * max_warps) S *= 2;
  const int64_t rows_all = (a_hi - a_lo) * s->Nb;
  while (S > 1 && has_out && S * rows_all * (int64_t)sizeof(double2) > (32ll << 30)) S /= 2;
  return S;
}

// ------------------------------------------------------ K1a (assembled rows)
// The matrix-free K1 recomputes every element each launch: x-local hash,
// sign, partner rank, out-of-sector partners adding exact zeros (issue-bound,
// 1,455 instructions per row at H12).  Where the rows fit in HBM, they are
// enumerated ONCE by K1 itself (EM count and emit modes: same buckets, same
// groups, same order) into a sliced ELL matrix, and every later H application
// streams it: 12 B per stored element, coalesced, plus the psi gather.  Each
// lane replays K1's per-split FMA chain (diagonal first in split 0, elements
// in K1's order, exact zeros dropped -- adding +-0 changes nothing but the
// sign of a zero) and sums the split partials in split order, so rows are
// bit-identical to K1's.
__global__ void k_sell_len(const uint32_t* __restrict__ cnt, int64_t rows, int S, int64_t n_chunks,
                           uint32_t* __restrict__ len, uint64_t* __restrict__ sz) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;   // (chunk, split)
  if (i >= n_chunks * S) return;
  const int64_t c = i / S;
  const int sp = (int)(i - c * S);
  uint32_t m = 0;
  for (int l = 0; l < 32; ++l) {
    const int64_t r = c * 32 + l;
    if (r < rows) m = max(m, __ldg(cnt + r * S + sp));
  }
  len[i] = m;
  sz[i] = 32ull * m;
}

struct SellArgs {
  const uint32_t* cols;
  const double* amps;
  const uint64_t* off;
  const uint32_t* len;
  int64_t n_chunks, rows, row0;   // rows of the range (K1s: of the list), first internal row
  int64_t chunk_lo, chunk_hi;      // chunks this launch processes
  const uint32_t* rlist;          // K1s: local rows of the list (nullptr: rows in order)
  unsigned long long* stats;      // K1s: rows computed -> the K1r row counter (hsv_stats)
  int S;
  const double2* psi;
  const double* diag;
  double2* out;
  double prune;
  int energy_only;
  double* cpart;                  // [chunk][2] energy partials or nullptr
  double2* const* peer_rows;
  int n_peer_rows;
};

template <int U, int MINB>
__global__ void __launch_bounds__(256, MINB) k_apply_sell(const SellArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = a.chunk_lo + gw; c < a.chunk_hi; c += nw) {
    const int64_t li = c * 32 + lane;
    const bool inr = li < a.rows;
    const int64_t row = a.row0 + (a.rlist ? (inr ? (int64_t)__ldg(a.rlist + li) : 0) : li);
    const double2 pv = inr ? a.psi[row] : make_double2(0.0, 0.0);
    if (a.energy_only && !__any_sync(0xffffffffu, pv.x != 0.0 || pv.y != 0.0)) {
      if (lane == 0 && a.cpart) { a.cpart[2 * c] = 0.0; a.cpart[2 * c + 1] = 0.0; }
      continue;
    }
    const double d = (a.diag && inr) ? a.diag[row] : 0.0;
    double2 y = make_double2(0.0, 0.0);
    for (int sp = 0; sp < a.S; ++sp) {
      const double ds = sp == 0 ? d : 0.0;
      double2 acc = make_double2(ds * pv.x, ds * pv.y);
      const uint32_t L = __ldg(a.len + c * a.S + sp);
      const uint64_t base = __ldg(a.off + c * a.S + sp) + lane;
      const uint32_t* __restrict__ cp = a.cols + base;
      const double* __restrict__ ap = a.amps + base;
      // software pipeline: the next U slots' (column, element) loads are in
      // flight while this group's psi gathers return (the stream and the
      // gathers would otherwise serialize: ncu, 91 % of cycles without an
      // eligible warp at U = 4 unpipelined).  12 B per slot: an 8 B form
      // (column + code into a value table) read 8.0 instead of 10.1 GB but was
      // slower (1.69 vs 1.58 ms): the extra gather made it L1-bound (91 %).
      const uint32_t Lu = L / U * U;
      uint32_t q[U];
      double m[U];
      if (Lu > 0) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          q[u] = __ldcs(cp + (uint64_t)u * 32);
          m[u] = __ldcs(ap + (uint64_t)u * 32);
        }
      }
      for (uint32_t j = 0; j < Lu; j += U) {
        double2 p[U];
#pragma unroll
        for (int u = 0; u < U; ++u) p[u] = a.psi[q[u]];
        uint32_t qn[U];
        double mn[U];
        const bool more = j + U < Lu;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          qn[u] = more ? __ldcs(cp + (uint64_t)(j + U + u) * 32) : 0u;
          mn[u] = more ? __ldcs(ap + (uint64_t)(j + U + u) * 32) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          acc.x = fma(m[u], p[u].x, acc.x);
          acc.y = fma(m[u], p[u].y, acc.y);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) { q[u] = qn[u]; m[u] = mn[u]; }
      }
      for (uint32_t j = Lu; j < L; ++j) {
        const uint32_t qq = __ldcs(cp + (uint64_t)j * 32);
        const double mm = __ldcs(ap + (uint64_t)j * 32);
        const double2 pp = a.psi[qq];
        acc.x = fma(mm, pp.x, acc.x);
        acc.y = fma(mm, pp.y, acc.y);
      }
      if (sp == 0) {
        y = acc;
      } else {
        y.x += acc.x;
        y.y += acc.y;
      }
    }
    if (inr && a.out && !a.energy_only) {
      double2 v = y;
      if (a.prune > 0.0 && sqrt(v.x * v.x + v.y * v.y) < a.prune) v = make_double2(0.0, 0.0);
      put_row(a.out, a.peer_rows, a.n_peer_rows, row, v);
    }
    if (a.stats) {
      const unsigned nr = __popc(__ballot_sync(0xffffffffu, inr));
      if (lane == 0 && nr) atomicAdd(a.stats + kStatRowsK1r, (unsigned long long)nr);
    }
    if (a.cpart) {   // this chunk's <psi|H psi> share, summed in chunk order
      double er = 0.0, ei = 0.0;
      if (inr) {
        er = pv.x * y.x + pv.y * y.y;
        ei = pv.x * y.y - pv.y * y.x;
      }
      er = warp_sum(er);
      ei = warp_sum(ei);
      if (lane == 0) { a.cpart[2 * c] = er; a.cpart[2 * c + 1] = ei; }
    }
  }
}

// Split-parallel K1a: a work unit is one (chunk, bucket split) segment, so a
// rank's shard (6.7 k chunks at H12 / 4 against ~4.7 k resident warps) still
// gives every warp ~11 units instead of 1-2 (0.55 vs 0.41 ms ideal).  Each lane
// writes its split partial; k_sell_combine sums them in split order, exactly
// as the chunk-per-warp kernel does in registers.
template <int U, int MINB>
__global__ void __launch_bounds__(256, MINB) k_apply_sell_sp(const SellArgs a, double2* ypart,
                                                             int64_t pstride) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nch = a.chunk_hi - a.chunk_lo;
  for (int64_t u = gw; u < nch * a.S; u += nw) {
    const int sp = (int)(u / nch);                  // split-major: one bucket range at a time
    const int64_t c = a.chunk_lo + (u - (int64_t)sp * nch);
    const int64_t li = c * 32 + lane;
    const bool inr = li < a.rows;
    const int64_t row = a.row0 + li;
    const double2 pv = inr ? a.psi[row] : make_double2(0.0, 0.0);
    if (a.energy_only && !__any_sync(0xffffffffu, pv.x != 0.0 || pv.y != 0.0)) {
      if (inr) ypart[sp * pstride + li] = make_double2(0.0, 0.0);
      continue;
    }
    const double ds = (sp == 0 && a.diag && inr) ? a.diag[row] : 0.0;
    double2 acc = make_double2(ds * pv.x, ds * pv.y);
    const uint32_t L = __ldg(a.len + c * a.S + sp);
    const uint64_t base = __ldg(a.off + c * a.S + sp) + lane;
    const uint32_t* __restrict__ cp = a.cols + base;
    const double* __restrict__ ap = a.amps + base;
    const uint32_t Lu = L / U * U;
    uint32_t q[U];
    double m[U];
    if (Lu > 0) {
#pragma unroll
      for (int k = 0; k < U; ++k) {
        q[k] = __ldcs(cp + (uint64_t)k * 32);
        m[k] = __ldcs(ap + (uint64_t)k * 32);
      }
    }
    for (uint32_t j = 0; j < Lu; j += U) {
      double2 p[U];
#pragma unroll
      for (int k = 0; k < U; ++k) p[k] = a.psi[q[k]];
      uint32_t qn[U];
      double mn[U];
      const bool more = j + U < Lu;
#pragma unroll
      for (int k = 0; k < U; ++k) {
        qn[k] = more ? __ldcs(cp + (uint64_t)(j + U + k) * 32) : 0u;
        mn[k] = more ? __ldcs(ap + (uint64_t)(j + U + k) * 32) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        acc.x = fma(m[k], p[k].x, acc.x);
        acc.y = fma(m[k], p[k].y, acc.y);
      }
#pragma unroll
      for (int k = 0; k < U; ++k) { q[k] = qn[k]; m[k] = mn[k]; }
    }
    for (uint32_t j = Lu; j < L; ++j) {
      const uint32_t qq = __ldcs(cp + (uint64_t)j * 32);
      const double mm = __ldcs(ap + (uint64_t)j * 32);
      const double2 pp = a.psi[qq];
      acc.x = fma(mm, pp.x, acc.x);
      acc.y = fma(mm, pp.y, acc.y);
    }
    if (inr) ypart[sp * pstride + li] = acc;
  }
}

// rows of chunks [chunk_lo, chunk_hi): y = part_0 + part_1 + ... (split order),
// the drop rule, the stores (and peer stores), and each chunk's energy share
// summed over its 32 rows in lane order (the chunk-per-warp kernel's cpart)
__global__ void k_sell_combine(const SellArgs a, const double2* __restrict__ ypart,
                               int64_t pstride) {
  const int lane = threadIdx.x & 31;
  const int64_t c = a.chunk_lo + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (c >= a.chunk_hi) return;
  const int64_t li = c * 32 + lane;
  const bool inr = li < a.rows;
  const int64_t row = a.row0 + li;
  double2 y = make_double2(0.0, 0.0);
  double2 pv = make_double2(0.0, 0.0);
  if (inr) {
    pv = a.psi[row];
    y = ypart[li];
    for (int sp = 1; sp < a.S; ++sp) {
      const double2 p = ypart[sp * pstride + li];
      y.x += p.x;
      y.y += p.y;
    }
    if (a.out && !a.energy_only) {
      double2 v = y;
      if (a.prune > 0.0 && sqrt(v.x * v.x + v.y * v.y) < a.prune) v = make_double2(0.0, 0.0);
      put_row(a.out, a.peer_rows, a.n_peer_rows, row, v);
    }
  }
  if (a.cpart) {
    double er = 0.0, ei = 0.0;
    if (inr) {
      er = pv.x * y.x + pv.y * y.y;
      ei = pv.x * y.y - pv.y * y.x;
    }
    er = warp_sum(er);
    ei = warp_sum(ei);
    if (lane == 0) { a.cpart[2 * c] = er; a.cpart[2 * c + 1] = ei; }
  }
}

static void free_sell(hsv_op_s::Sell& m) {
  dfree(m.cols); dfree(m.amps); dfree(m.rcnt); dfree(m.off); dfree(m.len);
  m.cols = nullptr; m.amps = nullptr; m.rcnt = nullptr; m.off = nullptr; m.len = nullptr;
}

static void drop_sells(hsv_op_s* op) {
  for (auto& m : op->sells) free_sell(m);
  op->sells.clear();
  op->sell_declined.clear();
  free_sell(op->sup);
  dfree(op->sup_rows);
  op->sup_rows = nullptr;
  op->sup_version = 0;
}

// Enumerate rows [a0.a_lo, a0.a_hi) with K1's EM modes into m (m.cols == nullptr:
// declined, over the budget left after `held` bytes of other ranges).
template <typename W, int SH>
static int build_sell_t(hsv_op_s* op, const ApplyArgs& a0, int S, int64_t held,
                        hsv_op_s::Sell& m) {
  const hsv_sector_s* s = op->sec;
  const int64_t rows = (a0.a_hi - a0.a_lo) * s->Nb;
  const int64_t n_chunks = (rows + 31) / 32;
  const int64_t nl = n_chunks * S;
  uint32_t* cnt = nullptr;
  uint64_t* sz = nullptr;
  HSV_TRY(dalloc(&cnt, rows * S));
  HSV_TRY(dalloc(&m.len, nl));
  HSV_TRY(dalloc(&m.off, nl + 1));
  HSV_TRY(dalloc(&sz, nl + 1));
  ApplyArgs a = a0;
  a.psi = nullptr; a.out = nullptr; a.epart = nullptr; a.arow = nullptr; a.diag = nullptr;
  a.peer_rows = nullptr; a.n_peer_rows = 0; a.prune = 0.0; a.energy_only = 0;
  a.nsplit = S;
  a.sell_cnt = cnt;
  const bool bp = op->d_bperm && tuning().bperm != 0 && !s->wide;
  a.bperm = op->d_bperm;   // (launch_apply sets it only on its own K1 branch)
  a.rb0_n = 0;
  if (bp) HSV_TRY((launch_apply_t<W, SH, 8, 2, 2, 0, 1>(op, a, nullptr)));
  else HSV_TRY((launch_apply_t<W, SH, 8, 2, 0, 0, 1>(op, a, nullptr)));
  k_sell_len<<<(unsigned)((nl + 255) / 256), 256, 0, stream()>>>(cnt, rows, S, n_chunks, m.len, sz);
  HSV_TRY_CUDA(cudaMemsetAsync(sz + nl, 0, sizeof(uint64_t), stream()));
  count_launch();
  size_t tb = 0;
  HSV_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, sz, m.off, nl + 1, stream()));
  unsigned char* tmp = nullptr;
  HSV_TRY(dalloc(&tmp, std::max<size_t>(tb, 1)));
  HSV_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, sz, m.off, nl + 1, stream()));
  uint64_t total = 0;
  HSV_TRY_CUDA(cudaMemcpyAsync(&total, m.off + nl, sizeof(uint64_t), cudaMemcpyDeviceToHost,
                               stream()));
  HSV_TRY(stream_sync());
  dfree(tmp); dfree(sz);
  m.rcnt = cnt;   // kept: the K1s build skips the padding by it
  const int64_t bytes = (int64_t)total * 12;
  if (held + bytes > tuning().sell_budget_mb * (1ll << 20) ||
      dalloc(&m.cols, std::max<uint64_t>(total, 1)) != HSV_OK ||
      dalloc(&m.amps, std::max<uint64_t>(total, 1)) != HSV_OK) {
    free_sell(m);
    return HSV_OK;
  }
  // padding slots: column 0, element 0.0 (fma(0, psi, acc) == acc up to the sign of a zero)
  HSV_TRY_CUDA(cudaMemsetAsync(m.cols, 0, total * sizeof(uint32_t), stream()));
  HSV_TRY_CUDA(cudaMemsetAsync(m.amps, 0, total * sizeof(double), stream()));
  a.sell_cnt = nullptr;
  a.sell_off = m.off;
  a.sell_cols = m.cols;
  a.sell_amps = m.amps;
  if (bp) HSV_TRY((launch_apply_t<W, SH, 8, 2, 2, 0, 2>(op, a, nullptr)));
  else HSV_TRY((launch_apply_t<W, SH, 8, 2, 0, 0, 2>(op, a, nullptr)));
  m.lo = a0.a_lo;
  m.hi = a0.a_hi;
  m.chunks = n_chunks;
  m.entries = (int64_t)total;
  m.S = S;
  return HSV_OK;
}

// The range's assembled rows, built on first use when they fit (nullptr: not
// assembled -- over the budget, declined before, or K1a off).
static int get_sell(hsv_op_s* op, const ApplyArgs& a, int S, hsv_op_s::Sell** out) {
  *out = nullptr;
  if (tuning().sell == 0 || a.a_hi <= a.a_lo) return HSV_OK;
  const hsv_sector_s* s = op->sec;
  for (const int4& d : op->sell_declined)
    if (d.x == (int)a.a_lo && d.y == (int)a.a_hi && d.z == S) return HSV_OK;
  for (auto& x : op->sells)
    if (x.lo == a.a_lo && x.hi == a.a_hi && x.S == S) {
      *out = &x;
      return HSV_OK;
    }
  const int64_t rows = (a.a_hi - a.a_lo) * s->Nb;
  const double budget = (double)tuning().sell_budget_mb * (double)(1ll << 20);
  // cheap bound first (every (row, active group) pair stored), then the exact count
  if ((double)rows * (double)op->n_active * 12.0 > 4.0 * budget) {
    op->sell_declined.push_back(make_int4((int)a.a_lo, (int)a.a_hi, S, 0));
    return HSV_OK;
  }
  while (op->sells.size() >= 2) {   // keep at most two ranges: drop the oldest
    free_sell(op->sells.front());
    op->sells.erase(op->sells.begin());
  }
  int64_t held = 0;
  for (auto& x : op->sells) held += x.entries * 12;
  hsv_op_s::Sell nm;
  if (s->wide) HSV_TRY((build_sell_t<uint64_t, 32>(op, a, S, held, nm)));
  else HSV_TRY((build_sell_t<uint32_t, 16>(op, a, S, held, nm)));
  if (!nm.cols) {
    op->sell_declined.push_back(make_int4((int)a.a_lo, (int)a.a_hi, S, 0));
    return HSV_OK;
  }
  op->sells.push_back(nm);
  *out = &op->sells.back();
  return HSV_OK;
}

static int run_sell(const hsv_op_s* op, const hsv_op_s::Sell& m, const ApplyArgs& a, int S,
                    const uint32_t* rlist, int64_t list_n, const char* scope,
                    int64_t c0 = 0, int64_t c1 = -1, double* cpart_ext = nullptr) {
  SellArgs g{};
  g.cols = m.cols; g.amps = m.amps; g.off = m.off; g.len = m.len;
  g.n_chunks = m.chunks;
  g.chunk_lo = c0;
  g.chunk_hi = c1 < 0 ? m.chunks : c1;
  g.rows = rlist ? list_n : (a.a_hi - a.a_lo) * op->sec->Nb;
  g.row0 = a.a_lo * op->sec->Nb;
  g.rlist = rlist;
  g.stats = rlist ? ctx().d_stats : nullptr;
  g.S = S;
  g.psi = a.psi; g.diag = a.diag; g.out = a.out; g.prune = a.prune; g.energy_only = a.energy_only;
  g.peer_rows = a.peer_rows; g.n_peer_rows = a.n_peer_rows;
  const int64_t nch = g.chunk_hi - g.chunk_lo;
  if (nch <= 0) {
    if (a.epart && !cpart_ext) HSV_TRY_CUDA(cudaMemsetAsync(a.epart, 0, 2 * sizeof(double), stream()));
    return HSV_OK;
  }
  double* cpart = nullptr;
  if (cpart_ext) {
    g.cpart = cpart_ext;
  } else if (a.epart) {
    HSV_TRY(dalloc(&cpart, 2 * std::max<int64_t>(g.n_chunks, 1)));
    g.cpart = cpart;
  }
  // auto: split-parallel while the launch has fewer than ~2 chunks per resident
  // warp (rank shards: H12 / 4 0.514 vs 0.551 ms, / 8 0.269 vs 0.288); the whole
  // H12 range keeps a chunk per warp (1.639 vs 1.666 ms)
  const bool sp_auto = nch < 2ll * ctx().num_sms * 32;
  if (!rlist && S > 1 && (tuning().sell_sp > 0 || (tuning().sell_sp < 0 && sp_auto))) {
    // split-parallel units + an in-order combine (bitwise the same rows/energy)
    const int64_t rows_l = g.rows;
    double2* ypart = nullptr;
    HSV_TRY(dalloc(&ypart, (int64_t)S * std::max<int64_t>(rows_l, 1)));
    const int64_t units = nch * S;
    const int64_t grid_sp = std::max<int64_t>(1, std::min<int64_t>((units + 7) / 8,
                                                                   (int64_t)ctx().num_sms * 4));
    {
      ProfScope prof(scope);
      k_apply_sell_sp<8, 4><<<(unsigned)grid_sp, 256, 0, stream()>>>(g, ypart, rows_l);
      k_sell_combine<<<(unsigned)((nch * 32 + 255) / 256), 256, 0, stream()>>>(g, ypart, rows_l);
    }
    count_launch(2);
    HSV_CHECK_LAUNCH();
    dfree(ypart);
    if (cpart) HSV_TRY(reduce_sum_f64(cpart, g.n_chunks, 2, 2, a.epart));
    dfree(cpart);
    return HSV_OK;
  }
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((nch + 7) / 8,
                                                              (int64_t)ctx().num_sms * 16));
  {
    ProfScope prof(scope);
    switch (tuning().sell_kernel) {   // (elements per pipeline stage, blocks per SM)
      case 1: k_apply_sell<4, 6><<<(unsigned)grid, 256, 0, stream()>>>(g); break;
      case 2: k_apply_sell<8, 3><<<(unsigned)grid, 256, 0, stream()>>>(g); break;
      case 3: k_apply_sell<8, 4><<<(unsigned)grid, 256, 0, stream()>>>(g); break;
      case 4: k_apply_sell<2, 8><<<(unsigned)grid, 256, 0, stream()>>>(g); break;
      default: k_apply_sell<4, 4><<<(unsigned)grid, 256, 0, stream()>>>(g); break;
    }
  }
  count_launch();
  HSV_CHECK_LAUNCH();
  if (cpart) HSV_TRY(reduce_sum_f64(cpart, g.n_chunks, 2, 2, a.epart));
  dfree(cpart);
  return HSV_OK;
}

// K1a: run the assembled rows when they exist (or can be built) for this row
// range and split count; *done = false leaves the launch to K1.
static int launch_apply_sell(const hsv_op_s* cop, const ApplyArgs& a, int S, int64_t* n_warps,
                             bool* done) {
  *done = false;
  if (!a.out && !a.epart) return HSV_OK;
  hsv_op_s* op = const_cast<hsv_op_s*>(cop);
  hsv_op_s::Sell* m = nullptr;
  HSV_TRY(get_sell(op, a, S, &m));
  if (!m) return HSV_OK;
  HSV_TRY(run_sell(op, *m, a, S, nullptr, 0, "apply"));
  if (n_warps) *n_warps = 1;   // epart[0..1] holds the total
  *done = true;
  return HSV_OK;
}

static ApplyArgs sell_args(const hsv_op_s* op, const double2* psi, double2* out, int64_t a_lo,
                           int64_t a_hi) {
  const hsv_sector_s* s = op->sec;
  ApplyArgs a{};
  a.split_bk = op->d_splits;
  a.dim_bytes = s->dim * (int64_t)sizeof(double2);
  a.Sa = s->d_Sa; a.Sb = s->d_Sb; a.Ra = s->d_Ra; a.Rb = s->d_Rb; a.Rb0 = s->d_Rb0;
  a.buckets = op->d_buckets; a.n_buckets = (int)op->n_buckets;
  a.groups = op->d_groups; a.terms = op->d_terms; a.diag = op->d_diag;
  a.tabs = op->d_tabs; a.recs = op->d_recs; a.n_buckets_h = (int)op->n_buckets_h;
  a.gsz = op->d_gsz; a.szt = op->d_szt; a.gxa = op->d_gxa; a.g_hashed = (int)op->g_hashed;
  a.peer_rows = out ? ctx().peer_rows : nullptr;
  a.n_peer_rows = out ? ctx().n_peer_rows : 0;
  a.psi = psi; a.out = out;
  a.Nb = s->Nb; a.a_lo = a_lo; a.a_hi = a_hi;
  return a;
}

int sell_chunks(const hsv_op_s* cop, int64_t a_lo, int64_t a_hi, int64_t* chunks) {
  *chunks = 0;
  if (tuning().sell == 0 || a_hi <= a_lo) return HSV_OK;
  hsv_op_s* op = const_cast<hsv_op_s*>(cop);
  const int S = k1_default_split(op, a_lo, a_hi, true);
  hsv_op_s::Sell* m = nullptr;
  HSV_TRY(get_sell(op, sell_args(op, nullptr, nullptr, a_lo, a_hi), S, &m));
  if (m) *chunks = m->chunks;
  return HSV_OK;
}

int sell_apply_chunks(const hsv_op_s* cop, const double2* psi, double2* out, int64_t a_lo,
                      int64_t a_hi, int64_t c0, int64_t c1, double* cpart) {
  hsv_op_s* op = const_cast<hsv_op_s*>(cop);
  const int S = k1_default_split(op, a_lo, a_hi, true);
  hsv_op_s::Sell* m = nullptr;
  const ApplyArgs a = sell_args(op, psi, out, a_lo, a_hi);
  HSV_TRY(get_sell(op, a, S, &m));
  HSV_REQUIRE(m, HSV_ERR_INVALID, "assembled rows missing for the range");
  return run_sell(op, *m, a, S, nullptr, 0, "apply", c0, c1, cpart);
}

// ------------------------------------------------------ K1s (support rows)
// Warp per 32-row chunk of the range's assembled rows (coalesced): the rows in
// the support map keep, split by split and in order, the elements whose partner
// is in the map (psi is exactly zero elsewhere).  Pass 1 lists the support rows
// and counts; pass 2 copies into the compacted sliced-ELL rows (list order, so
// a chunk's rows land in one or two compacted chunks).
__global__ void k_sup_chunk_count(const uint8_t* __restrict__ smap, int64_t row0, int64_t rows,
                                  int64_t n_chunks, uint32_t* __restrict__ ccount) {
  const int lane = threadIdx.x & 31;
  const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (c >= n_chunks) return;
  const int64_t rl = c * 32 + lane;
  const unsigned b = __ballot_sync(0xffffffffu, rl < rows && smap[row0 + rl] != 0);
  if (lane == 0) ccount[c] = __popc(b);
}

template <bool EMIT>
__global__ void __launch_bounds__(256) k_sup_pass(
    const uint8_t* __restrict__ smap, int64_t row0, int64_t rows, int64_t n_chunks, int S,
    const uint32_t* __restrict__ cprefix, const uint32_t* __restrict__ cols,
    const double* __restrict__ amps, const uint32_t* __restrict__ rcnt,
    const uint64_t* __restrict__ off, const uint32_t* __restrict__ len,
    uint32_t* __restrict__ list, uint32_t* __restrict__ cnt2, const uint64_t* __restrict__ off2,
    uint32_t* __restrict__ cols2, double* __restrict__ amps2) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = gw; c < n_chunks; c += nw) {
    const int64_t rl = c * 32 + lane;
    const bool act = rl < rows && smap[row0 + rl] != 0;
    const unsigned b = __ballot_sync(0xffffffffu, act);
    if (!b) continue;
    const uint32_t lidx = __ldg(cprefix + c) + __popc(b & ((1u << lane) - 1u));
    if (!EMIT && act) list[lidx] = (uint32_t)rl;
    for (int sp = 0; sp < S; ++sp) {
      const uint32_t L = __ldg(len + c * S + sp);
      const uint64_t base = __ldg(off + c * S + sp) + lane;
      const uint32_t rc = act ? __ldg(rcnt + (uint64_t)rl * S + sp) : 0u;
      uint64_t o = EMIT && act ? __ldg(off2 + (uint64_t)(lidx >> 5) * S + sp) + (lidx & 31u) : 0;
      uint32_t n = 0;
      // groups of 8 slots: the column loads, then the map gathers, are
      // independent within a group (8 round trips in flight, not 1)
      for (uint32_t j0 = 0; j0 < L; j0 += 8) {
        uint32_t q[8];
        double v[8];
        bool ok[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          ok[u] = j0 + u < rc;
          const uint64_t idx = base + (uint64_t)(j0 + u) * 32;
          q[u] = ok[u] ? __ldcs(cols + idx) : 0u;
          v[u] = (EMIT && ok[u]) ? __ldcs(amps + idx) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) ok[u] = ok[u] && __ldg(smap + q[u]) != 0;   // partner in the map
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (!ok[u]) continue;
          if (EMIT) {
            cols2[o] = q[u];
            amps2[o] = v[u];
            o += 32;
          } else {
            ++n;
          }
        }
      }
      if (!EMIT && act) cnt2[(uint64_t)lidx * S + sp] = n;
    }
  }
}

static int build_sup(hsv_op_s* op, const hsv_op_s::Sell& m, const ApplyArgs& a, int S,
                     const uint8_t* smap, uint64_t version, int64_t held) {
  hsv_op_s::Sell& u = op->sup;
  free_sell(u);
  dfree(op->sup_rows);
  op->sup_rows = nullptr;
  op->sup_version = 0;
  const int64_t Nb = op->sec->Nb;
  const int64_t rows = (a.a_hi - a.a_lo) * Nb;
  const int64_t row0 = a.a_lo * Nb;
  const int64_t nc = m.chunks;
  ProfScope pa("sup_list");
  uint32_t *ccount = nullptr, *cprefix = nullptr;
  HSV_TRY(dalloc(&ccount, nc + 1));
  HSV_TRY(dalloc(&cprefix, nc + 1));
  HSV_TRY_CUDA(cudaMemsetAsync(ccount + nc, 0, sizeof(uint32_t), stream()));
  k_sup_chunk_count<<<(unsigned)((nc * 32 + 255) / 256), 256, 0, stream()>>>(smap, row0, rows, nc,
                                                                            ccount);
  size_t tb = 0;
  HSV_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, ccount, cprefix, nc + 1, stream()));
  unsigned char* tmp = nullptr;
  HSV_TRY(dalloc(&tmp, std::max<size_t>(tb, 1)));
  HSV_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, ccount, cprefix, nc + 1, stream()));
  uint32_t n_s = 0;
  HSV_TRY_CUDA(cudaMemcpyAsync(&n_s, cprefix + nc, sizeof(uint32_t), cudaMemcpyDeviceToHost,
                               stream()));
  HSV_TRY(stream_sync());
  dfree(tmp);
  const int64_t chunks = ((int64_t)n_s + 31) / 32;
  const int64_t nl = chunks * S;
  uint32_t* cnt = nullptr;
  uint64_t* sz = nullptr;
  HSV_TRY(dalloc(&op->sup_rows, std::max<int64_t>(n_s, 1)));
  HSV_TRY(dalloc(&cnt, std::max<int64_t>((int64_t)n_s * S, 1)));
  HSV_TRY(dalloc(&u.len, std::max<int64_t>(nl, 1)));
  HSV_TRY(dalloc(&u.off, nl + 1));
  HSV_TRY(dalloc(&sz, nl + 1));
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((nc + 7) / 8,
                                                              (int64_t)ctx().num_sms * 16));
  ProfScope pb("sup_count");
  k_sup_pass<false><<<(unsigned)grid, 256, 0, stream()>>>(
      smap, row0, rows, nc, S, cprefix, m.cols, m.amps, m.rcnt, m.off, m.len, op->sup_rows, cnt,
      nullptr, nullptr, nullptr);
  if (nl)
    k_sell_len<<<(unsigned)((nl + 255) / 256), 256, 0, stream()>>>(cnt, n_s, S, chunks, u.len, sz);
  HSV_TRY_CUDA(cudaMemsetAsync(sz + nl, 0, sizeof(uint64_t), stream()));
  tb = 0;
  HSV_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, sz, u.off, nl + 1, stream()));
  HSV_TRY(dalloc(&tmp, std::max<size_t>(tb, 1)));
  HSV_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, sz, u.off, nl + 1, stream()));
  uint64_t total = 0;
  HSV_TRY_CUDA(cudaMemcpyAsync(&total, u.off + nl, sizeof(uint64_t), cudaMemcpyDeviceToHost,
                               stream()));
  HSV_TRY(stream_sync());
  dfree(tmp); dfree(sz); dfree(cnt);
  if (held + (int64_t)total * 12 > tuning().sell_budget_mb * (1ll << 20) ||
      dalloc(&u.cols, std::max<uint64_t>(total, 1)) != HSV_OK ||
      dalloc(&u.amps, std::max<uint64_t>(total, 1)) != HSV_OK) {
    free_sell(u);
    dfree(ccount); dfree(cprefix);
    return HSV_OK;
  }
  {
    ProfScope pc("sup_memset");
    HSV_TRY_CUDA(cudaMemsetAsync(u.cols, 0, total * sizeof(uint32_t), stream()));
    HSV_TRY_CUDA(cudaMemsetAsync(u.amps, 0, total * sizeof(double), stream()));
  }
  ProfScope pd("sup_emit");
  k_sup_pass<true><<<(unsigned)grid, 256, 0, stream()>>>(
      smap, row0, rows, nc, S, cprefix, m.cols, m.amps, m.rcnt, m.off, m.len, nullptr, nullptr,
      u.off, u.cols, u.amps);
  count_launch(4);
  HSV_CHECK_LAUNCH();
  dfree(ccount); dfree(cprefix);
  u.lo = a.a_lo; u.hi = a.a_hi; u.S = S; u.chunks = chunks; u.entries = (int64_t)total;
  op->sup_n = n_s;
  op->sup_version = version;
  return HSV_OK;
}

// K1s: K1r from the support-compacted assembled rows; *done = false leaves the
// launch to the matrix-free K1r.
static int launch_apply_sup(const hsv_op_s* cop, const ApplyArgs& a, int S, const uint8_t* smap,
                            uint64_t version, int64_t support_rows, bool* done) {
  *done = false;
  hsv_op_s* op = const_cast<hsv_op_s*>(cop);
  if (!smap || !version || !a.out || a.n_peer_rows > 0 || tuning().sup == 0) return HSV_OK;
  // auto: only for a map that outlives its iteration.  While the support grows
  // the map changes with nearly every appended operator and a rebuild per
  // iteration costs more than its ~7 evaluations save; on a plateau (H12 free
  // run: 213,744 rows from depth ~200 to ~325) one build serves every later
  // evaluation.  A map seen by more than 10 evaluations (about 1.5 iterations)
  // is taken to be on a plateau; the rows are bitwise K1r's either way.
  if (tuning().sup < 0) {
    if (op->sup_seen != version) {
      op->sup_seen = version;
      op->sup_seen_evals = 0;
    }
    if (++op->sup_seen_evals <= 10 && op->sup_version != version) return HSV_OK;
  }
  hsv_op_s::Sell* m = nullptr;
  HSV_TRY(get_sell(op, a, S, &m));
  if (!m) return HSV_OK;
  hsv_op_s::Sell& u = op->sup;
  if (op->sup_version != version || u.lo != a.a_lo || u.hi != a.a_hi || u.S != S || !u.cols) {
    ProfScope prof("sup_build");
    int64_t held = 0;
    for (auto& x : op->sells) held += x.entries * 12;
    HSV_TRY(build_sup(op, *m, a, S, smap, version, held));
    if (!u.cols) return HSV_OK;
  }
  const int64_t rows = (a.a_hi - a.a_lo) * op->sec->Nb;
  // rows outside the support are exact zeros (K1r's contract)
  HSV_TRY_CUDA(cudaMemsetAsync(a.out + a.a_lo * op->sec->Nb, 0, rows * sizeof(double2), stream()));
  ApplyArgs b = a;
  b.epart = nullptr;
  HSV_TRY(run_sell(op, u, b, S, op->sup_rows, op->sup_n, "apply_rows"));
  *done = true;
  return HSV_OK;
}

int apply_warps(const hsv_op_s* op) {
  // upper bound on the warps the apply kernel uses (energy-partial sizing):
  // 256-thread blocks, at most 8 resident per SM
  (void)op;
  return ctx().num_sms * 64;
}

int launch_apply(const hsv_op_s* op, const double2* psi, double2* out, double* epart,
                 int64_t a_lo, int64_t a_hi, double prune, int energy_only, int64_t* n_warps,
                 const uint32_t* arow, bool* dense_hint) {
  const hsv_sector_s* s = op->sec;
  ApplyArgs a{};
  a.arow = arow;
  a.split_bk = op->d_splits;
  a.dim_bytes = s->dim * (int64_t)sizeof(double2);
  a.Sa = s->d_Sa; a.Sb = s->d_Sb; a.Ra = s->d_Ra; a.Rb = s->d_Rb; a.Rb0 = s->d_Rb0;
  a.buckets = op->d_buckets; a.n_buckets = (int)op->n_buckets;
  a.groups = op->d_groups; a.terms = op->d_terms; a.diag = op->d_diag;
  a.tabs = op->d_tabs; a.recs = op->d_recs; a.n_buckets_h = (int)op->n_buckets_h;
  a.gsz = op->d_gsz; a.szt = op->d_szt; a.gxa = op->d_gxa; a.g_hashed = (int)op->g_hashed;
  a.peer_rows = out ? ctx().peer_rows : nullptr;
  a.n_peer_rows = out ? ctx().n_peer_rows : 0;
  a.psi = psi; a.out = out; a.epart = epart;
  a.Nb = s->Nb; a.a_lo = a_lo; a.a_hi = a_hi; a.prune = prune; a.energy_only = energy_only;
  HSV_REQUIRE(s->dim < ((int64_t)1 << 32), HSV_ERR_UNSUPPORTED,
              "sector dimension %lld exceeds the 32-bit row index of the apply kernel",
              (long long)s->dim);
  if (tuning().push != 0) {   // sparse psi: scatter + sort-reduce (hsv_push.cu)
    bool done = false;
    HSV_TRY(launch_push(op, a, &done, n_warps, dense_hint));
    if (done) return HSV_OK;
  }
  {   // K1a: assembled rows (built on first use where they fit)
    bool done = false;
    HSV_TRY(launch_apply_sell(op, a, k1_default_split(op, a_lo, a_hi, true), n_warps, &done));
    if (done) return HSV_OK;
  }
  if (tuning().staged != 1) {   // K1t: alpha tiles (hsv_apply_t.cu)
    bool done = false;
    HSV_TRY(launch_apply_t(op, a, k1_default_split(op, a_lo, a_hi, out != nullptr), &done));
    if (done) {
      if (n_warps) *n_warps = 1;   // epart[0..1] holds the total
      return HSV_OK;
    }
  }
  if (out && tuning().staged != 1) {   // K1v: valid beta lists (hsv_apply_v.cu)
    bool done = false;
    HSV_TRY(launch_apply_v(op, a, k1_default_split(op, a_lo, a_hi, true), &done));
    if (done) {
      if (n_warps) *n_warps = 1;   // epart[0..1] holds the total
      return HSV_OK;
    }
  }
  {   // small beta rows: partner rows staged on chip by TMA (hsv_apply_staged.cu)
    bool done = false;
    HSV_TRY(launch_apply_staged(op, a, n_warps, &done));
    if (done) return HSV_OK;
  }
  int R = tuning().apply_r;
  const int M = tuning().apply_minb;
  if (R == 0) {
    // auto: more rows per lane amortize the per-group overhead and keep more
    // independent gathers in flight; with the dynamic schedule and up to 32
    // bucket splits 8 rows win whenever there is a unit per warp (H12 sixteenth
    // shard 0.207 against 0.215 ms with 2, H10 0.126 against 0.14 ms)
    const int64_t units8 = (a_hi - a_lo) * ((s->Nb + 255) / 256);
    const int64_t warps8 = (int64_t)ctx().num_sms * 2 * 8;
    const int64_t units4 = (a_hi - a_lo) * ((s->Nb + 127) / 128);
    const int64_t warps4 = (int64_t)ctx().num_sms * 3 * 8;
    const bool dyn = tuning().apply_interleave < 0 || tuning().apply_interleave == 2;
    R = (dyn ? 32 * units8 >= warps8 : 4 * units8 >= 3 * warps8) ? 8 : units4 >= warps4 ? 4 : 2;
  }
  // Rb0 in shared memory (opt-in; 2^norb words, H12 16 KB, H14 64 KB): measured
  // slower, H12 2.415 vs 2.394 ms, H14 58.8 vs 57.3 ms -- K1 is issue-bound and
  // the LDS saves no issue slot over the L1-resident LDG
  const bool rs = !s->wide && tuning().rb0_smem == 1 && s->norb <= 15;
  a.rb0_n = rs ? (1 << s->norb) : 0;
  // per-xb beta rank permutations (built at upload for 32-bit words when small)
  // on wherever built (16-bit rows): H10 0.130 -> 0.125 ms, H12 2.386 -> 2.385,
  // H14 57.3 -> 56.4, H16 1404 -> 1359 ms (32-bit rows lost at H12, 2.415)
  const bool bp = !rs && op->d_bperm && tuning().bperm != 0;
  a.bperm = op->d_bperm;
#define HSV_APPLY_CASES(W, SH)                                              \
  if (R == 1) return launch_apply_t<W, SH, 1, 6>(op, a, n_warps);              \
  if (R == 4 && M == 2) return launch_apply_t<W, SH, 4, 2>(op, a, n_warps);    \
  if (R == 8 && rs) return launch_apply_t<W, SH, 8, 2, 1>(op, a, n_warps);     \
  if (R == 8 && bp) return launch_apply_t<W, SH, 8, 2, 2>(op, a, n_warps);     \
  if (R == 8) return launch_apply_t<W, SH, 8, 2>(op, a, n_warps);              \
  if (R == 4) return launch_apply_t<W, SH, 4, 3>(op, a, n_warps);              \
  if (M == 3) return launch_apply_t<W, SH, 2, 3>(op, a, n_warps);              \
  if (M == 5) return launch_apply_t<W, SH, 2, 5>(op, a, n_warps);              \
  if (M == 6) return launch_apply_t<W, SH, 2, 6>(op, a, n_warps);              \
  return launch_apply_t<W, SH, 2, 4>(op, a, n_warps);
  if (s->wide) { HSV_APPLY_CASES(uint64_t, 32) }
  HSV_APPLY_CASES(uint32_t, 16)
#undef HSV_APPLY_CASES
}

// ------------------------------------------------------ K1r (row lists)
// One block per alpha row: the marked beta ranks of the row in ascending order
// (ballot + popc compaction), and their count.
__global__ void k_rowlist(const uint8_t* __restrict__ smap, const double2* __restrict__ amp,
                          int64_t a_lo, int64_t Nb, uint32_t* __restrict__ rlist,
                          uint32_t* __restrict__ rcnt, unsigned long long* stats) {
  __shared__ uint32_t wsum[8];
  __shared__ uint32_t base;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t row0 = (a_lo + blockIdx.x) * Nb;
  uint32_t* out = rlist + (int64_t)blockIdx.x * Nb;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int64_t j0 = 0; j0 < Nb; j0 += 256) {
    const int64_t j = j0 + threadIdx.x;
    bool f = false;
    if (j < Nb) {
      if (smap) {
        f = smap[row0 + j] != 0;
      } else {
        const double2 v = amp[row0 + j];
        f = v.x != 0.0 || v.y != 0.0;
      }
    }
    const unsigned b = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wsum[w] = __popc(b);
    __syncthreads();
    uint32_t off = base;
    for (int q = 0; q < w; ++q) off += wsum[q];
    if (f) out[off + __popc(b & ((1u << lane) - 1u))] = (uint32_t)j;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t t = 0;
      for (int q = 0; q < 8; ++q) t += wsum[q];
      base += t;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    rcnt[blockIdx.x] = base;
    if (stats && base) atomicAdd(stats + kStatRowsK1r, (unsigned long long)base);
  }
}

// Single block: unit table (alpha row, chunk) in alpha-row order, and the count.
__global__ void __launch_bounds__(1024) k_unit_table(const uint32_t* __restrict__ rcnt,
                                                     int64_t n_rows, uint32_t rpu,
                                                     uint2* __restrict__ utab,
                                                     uint32_t* __restrict__ d_units) {
  typedef cub::BlockScan<uint32_t, 1024> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t c0 = 0; c0 < n_rows; c0 += 1024) {
    const int64_t i = c0 + threadIdx.x;
    const uint32_t nu = i < n_rows ? (__ldg(rcnt + i) + rpu - 1) / rpu : 0u;
    uint32_t ex, tot;
    Scan(tmp).ExclusiveSum(nu, ex, tot);
    const uint32_t off = carry + ex;
    for (uint32_t q = 0; q < nu; ++q) utab[off + q] = make_uint2((uint32_t)i, q);
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *d_units = carry;
}

int RowList::build(const hsv_sector_s* s, const uint8_t* smap, const double2* amp, int64_t a_lo,
                   int64_t a_hi, int rpu) {
  const int64_t na = a_hi - a_lo;
  max_units = na * ((s->Nb + rpu - 1) / rpu);
  HSV_TRY(dalloc(&rlist, std::max<int64_t>(na * s->Nb, 1)));
  HSV_TRY(dalloc(&rcnt, std::max<int64_t>(na, 1)));
  HSV_TRY(dalloc(&utab, std::max<int64_t>(max_units, 1)));
  HSV_TRY(dalloc(&d_units, 1));
  if (na == 0) {
    HSV_TRY_CUDA(cudaMemsetAsync(d_units, 0, sizeof(uint32_t), stream()));
    return HSV_OK;
  }
  k_rowlist<<<(unsigned)na, 256, 0, stream()>>>(smap, amp, a_lo, s->Nb, rlist, rcnt,
                                                 ctx().d_stats);
  k_unit_table<<<1, 1024, 0, stream()>>>(rcnt, na, (uint32_t)rpu, utab, d_units);
  count_launch(2);
  HSV_CHECK_LAUNCH();
  return HSV_OK;
}

void RowList::release() {
  dfree(rlist);
  dfree(rcnt);
  dfree(utab);
  dfree(d_units);
  rlist = rcnt = d_units = nullptr;
  utab = nullptr;
}

int launch_apply_rows(const hsv_op_s* op, const double2* psi, double2* out, int64_t a_lo,
                      int64_t a_hi, const uint32_t* arow, const uint8_t* smap,
                      int64_t support_rows, uint64_t smap_version) {
  const hsv_sector_s* s = op->sec;
  HSV_REQUIRE(s->dim < ((int64_t)1 << 32), HSV_ERR_UNSUPPORTED,
              "sector dimension %lld exceeds the 32-bit row index of the apply kernel",
              (long long)s->dim);
  ApplyArgs a{};
  a.arow = arow;
  a.split_bk = op->d_splits;
  a.dim_bytes = s->dim * (int64_t)sizeof(double2);
  a.Sa = s->d_Sa; a.Sb = s->d_Sb; a.Ra = s->d_Ra; a.Rb = s->d_Rb; a.Rb0 = s->d_Rb0;
  a.buckets = op->d_buckets; a.n_buckets = (int)op->n_buckets;
  a.groups = op->d_groups; a.terms = op->d_terms; a.diag = op->d_diag;
  a.tabs = op->d_tabs; a.recs = op->d_recs; a.n_buckets_h = (int)op->n_buckets_h;
  a.gsz = op->d_gsz; a.szt = op->d_szt; a.gxa = op->d_gxa; a.g_hashed = (int)op->g_hashed;
  a.peer_rows = ctx().peer_rows;
  a.n_peer_rows = ctx().n_peer_rows;
  a.psi = psi; a.out = out; a.epart = nullptr;
  a.Nb = s->Nb; a.a_lo = a_lo; a.a_hi = a_hi; a.prune = 0.0; a.energy_only = 0;
  // rows per lane: 8 while the full row range gives a 256-row unit to every
  // resident warp (the full kernel's rule), else 4
  const int S = k1_default_split(op, a_lo, a_hi, true);
  {   // K1s: the support-compacted assembled rows (built once per support map)
    bool done = false;
    HSV_TRY(launch_apply_sup(op, a, S, smap, smap_version, support_rows, &done));
    if (done) return HSV_OK;
  }
  {   // K1v over the support rows (hsv_apply_v.cu)
    bool done = false;
    ApplyArgs av = a;
    av.smap = smap;
    HSV_TRY(launch_apply_v(op, av, S, &done));
    if (done) return HSV_OK;
  }
  a.nsplit = S;
  // rows per lane: a lane's R rows are consecutive list entries of one alpha
  // row, and the group loop runs for all R whether the entries exist or not, so
  // R follows the support's rows per alpha row (H12 depth 100: 24 of 924)
  const int64_t units8 = (a_hi - a_lo) * ((s->Nb + 255) / 256);
  int R = 32 * units8 >= (int64_t)ctx().num_sms * 2 * 8 ? 8 : 4;
  if (support_rows > 0 && tuning().apply_r == 0) {
    const double per_row = (double)support_rows * s->Nb / (double)s->dim;   // per alpha row
    const int Rs = per_row >= 192 ? 8 : per_row >= 96 ? 4 : per_row >= 48 ? 2 : 1;
    R = std::min(R, Rs);
  }
  RowList rl;
  int rc = rl.build(s, smap, nullptr, a_lo, a_hi, 32 * R);
  if (rc == HSV_OK) {
    a.rlist = rl.rlist; a.rcnt = rl.rcnt; a.utab = rl.utab; a.d_units = rl.d_units;
#define HSV_ROWS_CASES(W, SH)                                                               \
  rc = R == 8   ? launch_apply_t<W, SH, 8, 2, 0, 1>(op, a, nullptr, smap, rl.max_units)       \
       : R == 4 ? launch_apply_t<W, SH, 4, 3, 0, 1>(op, a, nullptr, smap, rl.max_units)       \
       : R == 2 ? launch_apply_t<W, SH, 2, 4, 0, 1>(op, a, nullptr, smap, rl.max_units)       \
                : launch_apply_t<W, SH, 1, 4, 0, 1>(op, a, nullptr, smap, rl.max_units);
    if (s->wide) {
      HSV_ROWS_CASES(uint64_t, 32)
    } else {
      HSV_ROWS_CASES(uint32_t, 16)
    }
#undef HSV_ROWS_CASES
  }
  rl.release();
  return rc;
}

// Host: does group [t0, t1) admit amp(b) = (-1)^popc(b&z0) * A[h(b & x)]?  If
// so, fill a perfect multiply-shift hash over the in-sector patterns of b on
// x (ha of the alpha bits, hb of the beta bits set) and append A, summed in
// the reference's term order, to `tabs`.
static uint64_t splitmix(uint64_t& st) {
  uint64_t z = (st += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

bool build_group_hash(const std::vector<Term>& terms, int t0, int t1, uint64_t xp, int ha,
                      int hb, int SH, GroupHash& gh, std::vector<double>& tabs) {
  gh = GroupHash{0, 0, 0, 0, -1};
  if (t1 <= t0) return false;
  const uint64_t z0 = terms[t0].z;
  for (int t = t0; t < t1; ++t)
    if ((terms[t].z ^ z0) & ~xp) return false;          // not x-local
  std::vector<int> bits;
  for (int q = 0; q < 64; ++q)
    if ((xp >> q) & 1ull) bits.push_back(q);
  if (bits.size() > 12) return false;
  const uint64_t amask = SH == 16 ? 0xffffull : 0xffffffffull;
  std::vector<uint64_t> pats;
  std::vector<double> vals;
  for (uint32_t m = 0; m < (1u << bits.size()); ++m) {
    uint64_t t = 0;
    for (size_t i = 0; i < bits.size(); ++i)
      if ((m >> i) & 1u) t |= 1ull << bits[i];
    // every pattern with an in-sector alpha part (K1 tests alpha per warp);
    // out-of-sector beta patterns get A = 0, so K1 needs no per-lane beta test
    if (__builtin_popcountll(t & amask) != ha) continue;
    const bool bvalid = __builtin_popcountll(t & ~amask) == hb;
    double A = 0.0;
    if (bvalid)
      for (int q = t0; q < t1; ++q)
        A += (__builtin_popcountll(t & (terms[q].z ^ z0)) & 1) ? -terms[q].c : terms[q].c;
    pats.push_back(t);
    vals.push_back(A);
  }
  if (pats.empty()) return false;
  const int wbits = SH == 16 ? 32 : 64;
  int b0 = 0;
  while ((1u << b0) < pats.size()) ++b0;
  uint64_t seed = xp * 0x2545f4914f6cdd1dull + 1;
  for (int B = std::max(b0, 1); B <= b0 + 3 && B <= 8; ++B) {
    for (int tries = 0; tries < 20000; ++tries) {
      const uint64_t mul = splitmix(seed) | 1ull;
      uint64_t used[4] = {0, 0, 0, 0};
      bool ok = true;
      for (uint64_t t : pats) {
        const uint64_t prod = wbits == 32 ? (uint64_t)(uint32_t)((uint32_t)t * (uint32_t)mul)
                                          : t * mul;
        const unsigned h = (unsigned)(prod >> (wbits - B));
        if ((used[h >> 6] >> (h & 63)) & 1ull) { ok = false; break; }
        used[h >> 6] |= 1ull << (h & 63);
      }
      if (!ok) continue;
      gh.z0 = z0;
      gh.xm = xp;
      gh.mul = wbits == 32 ? (uint64_t)(uint32_t)mul : mul;
      gh.shift = wbits - B;
      gh.tab = (int32_t)tabs.size();
      tabs.resize(tabs.size() + (1u << B), 0.0);
      for (size_t i = 0; i < pats.size(); ++i) {
        const uint64_t prod = wbits == 32 ? (uint64_t)(uint32_t)((uint32_t)pats[i] * (uint32_t)mul)
                                          : pats[i] * mul;
        tabs[gh.tab + (prod >> (wbits - B))] = vals[i];
      }
      return true;
    }
  }
  return false;
}

}  // namespace hsv

using namespace hsv;

extern "C" {

int hsv_op_create(hsv_sector s, int n_qubits, const int64_t* xs, const int64_t* zs,
                  const double* coeffs, int64_t n_terms, hsv_op* out) {
  HSV_TRY(ensure_init());
  HSV_REQUIRE(s && out && (n_terms == 0 || (xs && zs && coeffs)), HSV_ERR_INVALID,
              "null argument");
  HSV_REQUIRE(n_qubits == s->n_qubits, HSV_ERR_INVALID,
              "Pauli sum and basis disagree on qubit count");
  const int SH = s->wide ? 32 : 16;
  // HSV_TIMING=1: host wall time of each setup phase on stderr
  static const bool timing = getenv("HSV_TIMING") && getenv("HSV_TIMING")[0] == '1';
  auto t_last = std::chrono::steady_clock::now();
  auto op_phase = [&](const char* name) {
    if (!timing) return;
    cudaStreamSynchronize(stream());
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "hsv_op_create %-14s %8.2f ms\n", name,
            std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  const uint64_t qmask = n_qubits >= 64 ? ~0ull : ((1ull << n_qubits) - 1);
  for (int64_t t = 0; t < n_terms; ++t)
    HSV_REQUIRE(((uint64_t)xs[t] & ~qmask) == 0 && ((uint64_t)zs[t] & ~qmask) == 0,
                HSV_ERR_INVALID, "Pauli mask exceeds %d qubits", n_qubits);
  // PauliSum order: ascending (x, z) (pauli.py:175-187); stable for duplicates.
  std::vector<int64_t> ord(n_terms);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int64_t i, int64_t j) {
    return xs[i] != xs[j] ? xs[i] < xs[j] : zs[i] < zs[j];
  });
  struct HGroup {
    int64_t x;
    uint32_t xa, xb;
    int pa, pb;
    bool nonreal, possible;
    int t0, t1;
  };
  std::vector<HGroup> hg;
  std::vector<Term> all_terms;
  all_terms.reserve(n_terms);
  auto fits = [](int p, int n, int norb) {   // can some n-of-norb string hit p/2 of p bits
    return p % 2 == 0 && p / 2 <= n && n - p / 2 <= norb - p;
  };
  for (int64_t i = 0; i < n_terms;) {
    const int64_t x = xs[ord[i]];
    HGroup g{};
    g.x = x;
    g.xa = s->compress_a((uint64_t)x);
    g.xb = s->compress_b((uint64_t)x);
    g.pa = __builtin_popcount(g.xa);
    g.pb = __builtin_popcount(g.xb);
    g.possible = fits(g.pa, s->n_alpha, s->norb) && fits(g.pb, s->n_beta, s->norb);
    g.t0 = (int)all_terms.size();
    for (; i < n_terms && xs[ord[i]] == x; ++i) {
      const int64_t t = ord[i];
      const int ny = __builtin_popcountll((uint64_t)(x & zs[t]));
      if (ny % 2) g.nonreal = true;
      const double sign_y = (ny % 4 == 2) ? -1.0 : 1.0;   // svengine.py:144
      Term T;
      T.c = coeffs[t] * sign_y;
      const uint64_t z = (uint64_t)zs[t];
      T.z = (uint64_t)s->compress_a(z) | ((uint64_t)s->compress_b(z) << SH);
      all_terms.push_back(T);
    }
    g.t1 = (int)all_terms.size();
    hg.push_back(g);
  }
  auto* op = new hsv_op_s();
  op->sec = s;
  op->n_terms = n_terms;
  op->n_groups = (int64_t)hg.size();
  int rc = HSV_OK;
  auto fail = [&](int code) { hsv_op_destroy(op); return code; };

  op_phase("grouping");
  // ---- device validation: sector leak per off-diagonal group ----
  Term* d_all = nullptr;
  if ((rc = dalloc(&d_all, all_terms.size()))) return fail(rc);
  if (!all_terms.empty())
    HSV_TRY_CUDA(cudaMemcpyAsync(d_all, all_terms.data(), all_terms.size() * sizeof(Term),
                                 cudaMemcpyHostToDevice, stream()));
  // Leak of an x-local group (every z_t ^ z_0 inside the flip mask x) depends
  // on the pattern p = b & x only: |amp(b)| = |sum_t c_t (-1)^popc(p & (z_t ^ z_0))|
  // summed in the reference's term order (the common sign (-1)^popc(b & z_0)
  // flips every term, and IEEE rounding is symmetric under negation, so the
  // magnitude is bit-identical to svengine.py:137-146).  So the check is a
  // host loop over the <= 2^|x| patterns that some sector row realizes and
  // whose image b ^ x leaves the sector; only the other groups (singles
  // carrying number-operator Z's) need the per-row device kernel.  H12:
  // 13.6 ms -> ~0.3 ms; H16: O(groups x rows) -> O(60-odd groups x rows).
  std::vector<int> offd;
  for (int g = 0; g < (int)hg.size(); ++g)
    if (hg[g].x != 0) offd.push_back(g);
  const int n_off = (int)offd.size();
  std::vector<unsigned long long> leak(n_off, 0ull);
  std::vector<int> on_dev;   // indices j into offd still checked row by row on the device
  for (int j = 0; j < n_off; ++j) {
    const HGroup& g = hg[offd[j]];
    const uint64_t xp = (uint64_t)g.xa | ((uint64_t)g.xb << SH);
    const uint64_t z0 = all_terms[g.t0].z;
    bool local = true;
    for (int t = g.t0; t < g.t1; ++t) local = local && ((all_terms[t].z ^ z0) & ~xp) == 0;
    // single-Z form: a reference term zr (the one without an extra number-operator
    // Z) every term differs from by <= 1 bit off the flip mask
    uint64_t zr = z0;
    bool single_z = false;
    if (!local)
      for (int r = g.t0; r < g.t1 && !single_z; ++r) {
        bool fits = true;
        for (int t = g.t0; t < g.t1 && fits; ++t)
          fits = __builtin_popcountll((all_terms[t].z ^ all_terms[r].z) & ~xp) <= 1;
        if (fits) { zr = all_terms[r].z; single_z = true; }
      }
    if (__builtin_popcountll(xp) > 16 || !(local || single_z)) {
      on_dev.push_back(j);
      continue;
    }
    if (!local) {
      // single-Z group (a single excitation with its number-operator Z's): per
      // out-of-sector pattern p of b on x, amp(b) = +-(C0 + sum_r C_r (-1)^{b_r})
      // (terms grouped by their one extra Z bit r), so |amp| <= |C0| + sum |C_r|,
      // and the reference's sequential sum adds at most gamma * sum |c_t| of
      // rounding.  A group whose bound is below the tolerance cannot leak; any
      // other goes to the exact per-row device check.
      double worst = 0.0, abs_sum = 0.0;
      const int nt = g.t1 - g.t0;
      for (int t = g.t0; t < g.t1; ++t) abs_sum += std::fabs(all_terms[t].c);
      const double eps = std::numeric_limits<double>::epsilon();
      const double gamma = nt * eps / (1.0 - nt * eps);
      const uint64_t amask = (SH == 16 ? 0xffffull : 0xffffffffull);
      std::vector<std::pair<uint64_t, double>> cr;
      for (uint64_t p = xp;; p = (p - 1) & xp) {
        const int na_p = __builtin_popcountll(p & amask), nb_p = __builtin_popcountll(p >> SH);
        const bool real_a = s->n_alpha - na_p >= 0 && s->n_alpha - na_p <= s->norb - g.pa;
        const bool real_b = s->n_beta - nb_p >= 0 && s->n_beta - nb_p <= s->norb - g.pb;
        const bool stays = 2 * na_p == g.pa && 2 * nb_p == g.pb;
        if (real_a && real_b && !stays) {
          double c0 = 0.0;
          cr.clear();
          for (int t = g.t0; t < g.t1; ++t) {
            const Term& T = all_terms[t];
            const double c = (__builtin_popcountll(p & (T.z ^ zr) & xp) & 1) ? -T.c : T.c;
            const uint64_t out = (T.z ^ zr) & ~xp;
            if (!out) { c0 += c; continue; }
            bool found = false;
            for (auto& e : cr)
              if (e.first == out) { e.second += c; found = true; break; }
            if (!found) cr.push_back({out, c});
          }
          double bound = std::fabs(c0);
          for (const auto& e : cr) bound += std::fabs(e.second);
          worst = std::max(worst, bound + 2.0 * gamma * abs_sum);
        }
        if (p == 0) break;
      }
      if (worst > kSectorLeakTol) {   // possibly leaking: exact device check
        on_dev.push_back(j);
        continue;
      }
      memcpy(&leak[j], &worst, 8);   // a bound below the tolerance
      continue;
    }
    double worst = 0.0;
    const uint64_t amask = (SH == 16 ? 0xffffull : 0xffffffffull);
    for (uint64_t p = xp;; p = (p - 1) & xp) {   // every sub-pattern of x
      const int na_p = __builtin_popcountll(p & amask), nb_p = __builtin_popcountll(p >> SH);
      const bool real_a = s->n_alpha - na_p >= 0 && s->n_alpha - na_p <= s->norb - g.pa;
      const bool real_b = s->n_beta - nb_p >= 0 && s->n_beta - nb_p <= s->norb - g.pb;
      const bool stays = 2 * na_p == g.pa && 2 * nb_p == g.pb;
      if (real_a && real_b && !stays) {
        double amp = 0.0;
        for (int t = g.t0; t < g.t1; ++t) {
          const Term& T = all_terms[t];
          amp += (__builtin_popcountll(p & (T.z ^ z0)) & 1) ? -T.c : T.c;
        }
        worst = std::max(worst, std::fabs(amp));
      }
      if (p == 0) break;
    }
    memcpy(&leak[j], &worst, 8);
  }
  if (timing) fprintf(stderr, "hsv_op_create leak: %d of %d groups on the device\n",
                      (int)on_dev.size(), n_off);
  if (!on_dev.empty() && s->dim > 0) {
    const int n_dev = (int)on_dev.size();
    std::vector<uint32_t> gxa(n_dev), gxb(n_dev);
    std::vector<int32_t> gha(n_dev), ghb(n_dev), gt0(n_dev), gt1(n_dev);
    for (int j = 0; j < n_dev; ++j) {
      const HGroup& g = hg[offd[on_dev[j]]];
      gxa[j] = g.xa; gxb[j] = g.xb;
      // odd popcount can never match: use an impossible target count
      gha[j] = g.pa % 2 ? -1 : g.pa / 2;
      ghb[j] = g.pb % 2 ? -1 : g.pb / 2;
      gt0[j] = g.t0; gt1[j] = g.t1;
    }
    uint32_t *d_gxa, *d_gxb;
    int32_t *d_gha, *d_ghb, *d_gt0, *d_gt1;
    unsigned long long* d_leak;
    if ((rc = dalloc(&d_gxa, n_dev)) || (rc = dalloc(&d_gxb, n_dev)) ||
        (rc = dalloc(&d_gha, n_dev)) || (rc = dalloc(&d_ghb, n_dev)) ||
        (rc = dalloc(&d_gt0, n_dev)) || (rc = dalloc(&d_gt1, n_dev)) ||
        (rc = dalloc(&d_leak, n_dev)))
      return fail(rc);
    cudaStream_t st = stream();
    HSV_TRY_CUDA(cudaMemcpyAsync(d_gxa, gxa.data(), n_dev * 4, cudaMemcpyHostToDevice, st));
    HSV_TRY_CUDA(cudaMemcpyAsync(d_gxb, gxb.data(), n_dev * 4, cudaMemcpyHostToDevice, st));
    HSV_TRY_CUDA(cudaMemcpyAsync(d_gha, gha.data(), n_dev * 4, cudaMemcpyHostToDevice, st));
    HSV_TRY_CUDA(cudaMemcpyAsync(d_ghb, ghb.data(), n_dev * 4, cudaMemcpyHostToDevice, st));
    HSV_TRY_CUDA(cudaMemcpyAsync(d_gt0, gt0.data(), n_dev * 4, cudaMemcpyHostToDevice, st));
    HSV_TRY_CUDA(cudaMemcpyAsync(d_gt1, gt1.data(), n_dev * 4, cudaMemcpyHostToDevice, st));
    HSV_TRY_CUDA(cudaMemsetAsync(d_leak, 0, n_dev * 8, st));
    dim3 grid((unsigned)((s->Nb + 127) / 128), (unsigned)s->Na);
    if (s->wide)
      k_leak<uint64_t, 32><<<grid, 128, 0, st>>>(s->d_Sa, s->d_Sb, s->Na, s->Nb, d_gxa, d_gxb,
                                                 d_gha, d_ghb, d_gt0, d_gt1, n_dev, d_all, d_leak);
    else
      k_leak<uint32_t, 16><<<grid, 128, 0, st>>>(s->d_Sa, s->d_Sb, s->Na, s->Nb, d_gxa, d_gxb,
                                                 d_gha, d_ghb, d_gt0, d_gt1, n_dev, d_all, d_leak);
    count_launch();
    HSV_CHECK_LAUNCH();
    std::vector<unsigned long long> dl(n_dev);
    HSV_TRY_CUDA(cudaMemcpyAsync(dl.data(), d_leak, n_dev * 8, cudaMemcpyDeviceToHost, st));
    if ((rc = stream_sync())) return fail(rc);
    for (int j = 0; j < n_dev; ++j) leak[on_dev[j]] = dl[j];
    dfree(d_gxa); dfree(d_gxb); dfree(d_gha); dfree(d_ghb); dfree(d_gt0); dfree(d_gt1);
    dfree(d_leak);
  }
  // errors in ascending-x order, odd-Y before leak within a group (svengine.py:135-160)
  {
    int j = 0;
    for (int g = 0; g < (int)hg.size(); ++g) {
      if (hg[g].nonreal) {
        dfree(d_all);
        set_error(HSV_ERR_NONREAL,
                  "odd-Y Pauli term has imaginary matrix elements; Hamiltonian is not real");
        return fail(HSV_ERR_NONREAL);
      }
      if (hg[g].x == 0) continue;
      double lk;
      unsigned long long bits = leak[j++];
      memcpy(&lk, &bits, 8);
      if (lk > kSectorLeakTol) {
        dfree(d_all);
        set_error(HSV_ERR_LEAK,
                  "Pauli terms with flip mask %#llx leak amplitude %.3e outside the sector; "
                  "Hamiltonian is not spin-conserving",
                  (unsigned long long)hg[g].x, lk);
        return fail(HSV_ERR_LEAK);
      }
    }
  }
  op_phase("leak");
  // ---- diagonal table ----
  for (const HGroup& g : hg) {
    if (g.x != 0 || s->dim == 0) continue;
    if ((rc = dalloc(&op->d_diag, s->dim))) return fail(rc);
    const unsigned nb = (unsigned)((s->dim + 255) / 256);
    const size_t tsm = (size_t)(g.t1 - g.t0) * sizeof(Term);
    if (tsm > 48 * 1024) {
      HSV_TRY_CUDA(cudaFuncSetAttribute(k_diag<uint64_t, 32>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
      HSV_TRY_CUDA(cudaFuncSetAttribute(k_diag<uint32_t, 16>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
    }
    if (s->wide)
      k_diag<uint64_t, 32><<<nb, 256, tsm, stream()>>>(s->d_Sa, s->d_Sb, s->Na, s->Nb, d_all,
                                                       g.t0, g.t1, op->d_diag);
    else
      k_diag<uint32_t, 16><<<nb, 256, tsm, stream()>>>(s->d_Sa, s->d_Sb, s->Na, s->Nb, d_all,
                                                       g.t0, g.t1, op->d_diag);
    count_launch();
    HSV_CHECK_LAUNCH();
  }
  op_phase("diag");
  // ---- active groups, bucketed by alpha flip part ----
  std::vector<int> act;
  for (int g = 0; g < (int)hg.size(); ++g)
    if (hg[g].x != 0 && hg[g].possible) act.push_back(g);
  std::stable_sort(act.begin(), act.end(), [&](int i, int j) {
    return hg[i].xa != hg[j].xa ? hg[i].xa < hg[j].xa : hg[i].xb < hg[j].xb;
  });
  for (size_t q = 0; q < act.size(); ++q) {
    const HGroup& g = hg[act[q]];
    if (op->buckets.empty() || (uint32_t)op->buckets.back().x != g.xa)
      op->buckets.push_back(make_int4((int)g.xa, g.pa / 2, (int)q, (int)q));
    op->buckets.back().w = (int)q + 1;
    const int t0 = (int)op->terms.size();
    for (int t = g.t0; t < g.t1; ++t) op->terms.push_back(all_terms[t]);
    op->groups.push_back(make_int4((int)g.xb, g.pb / 2, t0, (int)op->terms.size()));
  }
  op->n_active = (int64_t)act.size();
  op->n_buckets = (int64_t)op->buckets.size();
  op_phase("buckets");
  // ---- pattern tables for x-local groups ----
  std::vector<GroupHash> ghash(op->groups.size());
  std::vector<double> tabs;
  for (size_t q = 0; q < op->groups.size(); ++q) {
    const HGroup& g = hg[act[q]];
    const uint64_t xp = (uint64_t)g.xa | ((uint64_t)g.xb << SH);
    if (build_group_hash(op->terms, op->groups[q].z, op->groups[q].w, xp, g.pa / 2, g.pb / 2,
                         SH, ghash[q], tabs))
      ++op->n_hashed;
  }
  // Kernel layout: hashed groups first, then term-loop groups, each bucketed by
  // alpha flip part (the order of groups only changes the summation order of
  // distinct matrix elements, never an element's value).
  {
    std::vector<int4> nb, ng;
    std::vector<GroupHash> nh;
    const std::vector<int4> ob = op->buckets, og = op->groups;
    for (int pass = 0; pass < 2; ++pass) {
      for (const int4& B : ob) {
        bool opened = false;
        for (int q = B.z; q < B.w; ++q) {
          const bool hashed = ghash[q].tab >= 0;
          if (hashed != (pass == 0)) continue;
          if (!opened) {
            nb.push_back(make_int4(B.x, B.y, (int)ng.size(), (int)ng.size()));
            opened = true;
          }
          ng.push_back(og[q]);
          nh.push_back(ghash[q]);
          nb.back().w = (int)ng.size();
        }
      }
      if (pass == 0) op->n_buckets_h = (int64_t)nb.size();
    }
    op->buckets = nb;
    op->groups = ng;
    ghash = nh;
    op->n_buckets = (int64_t)nb.size();
  }
  // per-group alpha flip part and the hashed/term-loop boundary (push path)
  std::vector<uint32_t> gxa(op->groups.size(), 0u);
  for (const int4& B : op->buckets)
    for (int q = B.z; q < B.w; ++q) gxa[q] = (uint32_t)B.x;
  op->g_hashed = op->n_buckets_h < op->n_buckets ? op->buckets[op->n_buckets_h].z
                                                  : (int64_t)op->groups.size();
  // single-Z form of the term-loop groups (see SzTerm)
  std::vector<uint64_t> gsz(op->groups.size(), 0ull);
  std::vector<SzTerm> szt(op->terms.size(), SzTerm{0.0, 0u, 0u});
  for (const int4& B : op->buckets) {
    for (int q = B.z; q < B.w; ++q) {
      if (ghash[q].tab >= 0) continue;
      const int4 G = op->groups[q];
      const uint64_t xp = (uint64_t)(uint32_t)B.x | ((uint64_t)(uint32_t)G.x << SH);
      const int fixed = (B.y + G.y) & 1;   // parity(s & xp) on in-sector rows
      // reference z: a term every other term differs from by <= 1 bit off the
      // flip mask (the term without an extra number-operator Z)
      auto fits = [&](uint64_t zr) {
        for (int t = G.z; t < G.w; ++t) {
          const uint64_t d = op->terms[t].z ^ zr, dx = d & xp;
          if (!(dx == 0 || dx == xp) || __builtin_popcountll(d & ~xp) > 1) return false;
        }
        return true;
      };
      uint64_t z0 = 0;
      bool ok = false;
      for (int t = G.z; !ok && t < G.w; ++t)
        if (fits(op->terms[t].z)) { z0 = op->terms[t].z; ok = true; }
      ok = ok && (z0 >> 63) == 0;
      for (int t = G.z; ok && t < G.w; ++t) {
        const uint64_t d = op->terms[t].z ^ z0, dx = d & xp, dout = d & ~xp;
        ok = (dx == 0 || dx == xp) && __builtin_popcountll(dout) <= 1;
        if (!ok) break;
        const int r = dout ? __builtin_ctzll(dout) : 0;
        const double c = (dx == xp && fixed) ? -op->terms[t].c : op->terms[t].c;
        szt[t] = SzTerm{c, (uint32_t)(SH == 16 ? 31 - r : r), dout ? 0x80000000u : 0u};
      }
      if (ok) {
        gsz[q] = (1ull << 63) | z0;
        ++op->n_single_z;
      }
    }
  }
  // Split tables (S = 2, 4, 8, 16, 32) cutting the group range at equal
  // estimated cost, inside buckets where needed: a bucket cut in two becomes two
  // "virtual" buckets with the same alpha flip and disjoint group ranges, so the
  // kernel loops stay bucket-granular.  Cost per group: 1 (hashed) or
  // 1 + terms / 8, times the fraction of alpha strings for which the bucket's
  // alpha flip stays in the sector (C(k, y) C(norb - k, na - y) / C(norb, na)
  // for a flip of k orbitals needing y occupied).  Unweighted bucket cuts left
  // the parts of an 8-way bucket split 1.5x apart in time (H12).
  std::vector<int4> vbk;
  std::vector<int> cuts;
  {
    auto binom = [](int n, int k) -> double {
      if (k < 0 || k > n) return 0.0;
      double r = 1.0;
      for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
      return r;
    };
    const int na = s->n_alpha, no = s->norb;
    const double call = binom(no, na);
    const int nb = (int)op->buckets.size();
    const int ng = nb ? op->buckets[nb - 1].w : 0;
    std::vector<int> gb(ng, 0);   // bucket of each group (buckets own consecutive ranges)
    std::vector<double> cum(ng + 1, 0.0), cum0(ng + 1, 0.0);
    for (int b = 0; b < nb; ++b) {
      const int4 B = op->buckets[b];
      const int k = __builtin_popcount((uint32_t)B.x);
      const double frac = binom(k, B.y) * binom(no - k, na - B.y) / call;
      for (int q = B.z; q < B.w; ++q) {
        gb[q] = b;
        const double c = ghash[q].tab >= 0 ? 1.0 : 1.0 + (op->groups[q].w - op->groups[q].z) / 8.0;
        cum[q + 1] = cum[q] + frac * c + (q == B.z ? 0.01 : 0.0);
        cum0[q + 1] = cum0[q] + c;
      }
    }
    for (int li = 0; li < kSplitTables; ++li) {
      const int S = 2 << li;
      std::vector<int> cut(S + 1, ng);
      cut[0] = 0;
      if (S <= 8) {
        // up to 8 parts: bucket boundaries by unweighted group cost, the cut
        // measured best at full size (H12 2.39 against 2.42 ms weighted)
        for (int k = 1, b = 0; k < S; ++k) {
          const double target = cum0[ng] * k / S;
          while (b < nb && cum0[op->buckets[b].z] < target) ++b;
          cut[k] = b < nb ? op->buckets[b].z : ng;
        }
      } else {
        for (int k = 1, g = 0; k < S; ++k) {
          const double target = cum[ng] * k / S;
          while (g < ng && cum[g] < target) ++g;
          cut[k] = g;
        }
      }
      SplitTable& T = op->split[li];
      T.vb_off = (int)vbk.size();
      T.cut_off = (int)cuts.size();
      T.nbh = 0;
      for (int k = 0; k < S; ++k) {
        cuts.push_back((int)vbk.size() - T.vb_off);
        for (int g0 = cut[k]; g0 < cut[k + 1];) {   // pieces of buckets inside [cut k, cut k+1)
          const int4 B = op->buckets[gb[g0]];
          const int g1 = std::min(B.w, cut[k + 1]);
          vbk.push_back(make_int4(B.x, B.y, g0, g1));
          if (gb[g0] < op->n_buckets_h) ++T.nbh;
          g0 = g1;
        }
      }
      T.nb = (int)vbk.size() - T.vb_off;
      cuts.push_back(T.nb);
    }
  }
  op_phase("tables+splits");
  std::vector<unsigned char> recs;
  // K1 pass-1 beta rank permutations: for each distinct beta flip xb of a hashed
  // group, bperm[slot + rb] = rank(Sb[rb] ^ xb) (0 out of sector, as Rb0), rows
  // padded to a multiple of 256 so a unit's tail lanes stay inside the slot.
  // 16-bit ranks (Nb <= 65536): 64 bytes per warp row.  Rec.pad0 holds the slot
  // offset.  Skipped above 256 MB.
  std::vector<uint16_t> bperm;
  std::vector<uint32_t> bslot(ghash.size(), 0u);
  if (SH == 16) {
    const int64_t NbP = (s->Nb + 255) / 256 * 256;
    std::vector<uint32_t> xbs;
    for (size_t q = 0; q < ghash.size(); ++q)
      if (ghash[q].tab >= 0) xbs.push_back((uint32_t)op->groups[q].x);
    std::sort(xbs.begin(), xbs.end());
    xbs.erase(std::unique(xbs.begin(), xbs.end()), xbs.end());
    const int64_t entries = (int64_t)xbs.size() * NbP + 256;
    if (!xbs.empty() && s->Nb <= 65536 && entries * 2 <= (256ll << 20)) {
      bperm.assign((size_t)entries, 0u);
      for (size_t i = 0; i < xbs.size(); ++i)
        for (int64_t rb = 0; rb < s->Nb; ++rb) {
          const uint32_t r = s->Rb[s->Sb[rb] ^ xbs[i]];
          bperm[i * NbP + rb] = (uint16_t)(r == ~0u ? 0u : r);
        }
      for (size_t q = 0; q < ghash.size(); ++q)
        if (ghash[q].tab >= 0)
          bslot[q] = (uint32_t)((std::lower_bound(xbs.begin(), xbs.end(),
                                                  (uint32_t)op->groups[q].x) - xbs.begin()) * NbP);
    }
  }
  // K1v valid lists: per distinct beta flip xb of a hashed group, the beta
  // strings whose partner stays in the sector, rank-ascending, with chunk
  // offsets (Rec.pad1 = list * (nchunks + 1)).  Nb <= 65535 (16-bit ranks).
  std::vector<uint2> vl;
  std::vector<int> vloff;
  std::vector<uint32_t> vslot(ghash.size(), 0u);
  const int vchunk = 1024;
  const int vnch = (int)((s->Nb + vchunk - 1) / vchunk);
  if (SH == 16 && s->Nb <= 65535 && tuning().apply_v == 1) {   // only for the opt-in K1v
    std::vector<uint32_t> xbs;
    for (size_t q = 0; q < ghash.size(); ++q)
      if (ghash[q].tab >= 0) xbs.push_back((uint32_t)op->groups[q].x);
    std::sort(xbs.begin(), xbs.end());
    xbs.erase(std::unique(xbs.begin(), xbs.end()), xbs.end());
    for (size_t i = 0; i < xbs.size(); ++i) {
      const uint32_t xb = xbs[i];
      const int need = __builtin_popcount(xb) / 2;
      int c = 0;
      for (int64_t rb = 0; rb < s->Nb; ++rb) {
        while (c <= vnch && rb >= (int64_t)c * vchunk) { vloff.push_back((int)vl.size()); ++c; }
        const uint32_t sb = s->Sb[rb];
        if (__builtin_popcount(sb & xb) != need) continue;
        const uint32_t rp = s->Rb[sb ^ xb];
        if (rp == ~0u) continue;
        vl.push_back(make_uint2((uint32_t)rb | (rp << 16), sb));
      }
      while (c <= vnch) { vloff.push_back((int)vl.size()); ++c; }
    }
    for (size_t q = 0; q < ghash.size(); ++q)
      if (ghash[q].tab >= 0)
        vslot[q] = (uint32_t)((std::lower_bound(xbs.begin(), xbs.end(),
                                                (uint32_t)op->groups[q].x) - xbs.begin()) *
                              (vnch + 1));
  }
  if (SH == 16) {
    recs.resize(ghash.size() * 32);
    for (size_t q = 0; q < ghash.size(); ++q) {
      const GroupHash& h = ghash[q];
      uint32_t r[8] = {(uint32_t)op->groups[q].x,
                       (uint32_t)op->groups[q].y | ((uint32_t)h.shift << 8), (uint32_t)h.xm,
                       (uint32_t)h.z0, (uint32_t)h.mul, (uint32_t)std::max(h.tab, 0), bslot[q],
                       0u};
      memcpy(&recs[q * 32], r, 32);
    }
  } else {
    recs.resize(ghash.size() * 48);
    for (size_t q = 0; q < ghash.size(); ++q) {
      const GroupHash& h = ghash[q];
      uint32_t r[4] = {(uint32_t)op->groups[q].x,
                       (uint32_t)op->groups[q].y | ((uint32_t)h.shift << 8),
                       (uint32_t)std::max(h.tab, 0), 0u};
      uint64_t r2[4] = {h.xm, h.z0, h.mul, 0ull};
      memcpy(&recs[q * 48], r, 16);
      memcpy(&recs[q * 48 + 16], r2, 32);
    }
  }
  op_phase("bperm+recs");
  if ((rc = dalloc(&op->d_buckets, op->buckets.size())) ||
      (rc = dalloc(&op->d_groups, op->groups.size())) ||
      (rc = dalloc(&op->d_terms, op->terms.size())) ||
      (rc = dalloc(&op->d_ghash, ghash.size())) || (rc = dalloc(&op->d_tabs, tabs.size())) ||
      (rc = dalloc(reinterpret_cast<unsigned char**>(&op->d_recs), recs.size())) ||
      (rc = dalloc(&op->d_splits, cuts.size())) || (rc = dalloc(&op->d_vbuckets, vbk.size())) || (rc = dalloc(&op->d_gsz, gsz.size())) ||
      (rc = dalloc(reinterpret_cast<SzTerm**>(&op->d_szt), szt.size())) ||
      (rc = dalloc(&op->d_gxa, gxa.size())))
    return fail(rc);
  cudaStream_t st = stream();
  if (!gxa.empty())
    HSV_TRY_CUDA(cudaMemcpyAsync(op->d_gxa, gxa.data(), gxa.size() * sizeof(uint32_t),
                                 cudaMemcpyHostToDevice, st));
  if (!gsz.empty())
    HSV_TRY_CUDA(cudaMemcpyAsync(op->d_gsz, gsz.data(), gsz.size() * sizeof(uint64_t),
                                 cudaMemcpyHostToDevice, st));
  if (!szt.empty())
    HSV_TRY_CUDA(cudaMemcpyAsync(op->d_szt, szt.data(), szt.size() * sizeof(SzTerm),
                                 cudaMemcpyHostToDevice, st));
  HSV_TRY_CUDA(cudaMemcpyAsync(op->d_vbuckets, vbk.data(), vbk.size() * sizeof(int4),
                               cudaMemcpyHostToDevice, stream()));
  HSV_TRY_CUDA(cudaMemcpyAsync(op->d_splits, cuts.data(), cuts.size() * sizeof(int),
                               cudaMemcpyHostToDevice, st));
  if (!recs.empty())
    HSV_TRY_CUDA(cudaMemcpyAsync(op->d_recs, recs.data(), recs.size(), cudaMemcpyHostToDevice, st));
  if (!bperm.empty()) {
    if ((rc = dalloc(&op->d_bperm, bperm.size()))) return fail(rc);
    HSV_TRY_CUDA(cudaMemcpyAsync(op->d_bperm, bperm.data(), bperm.size() * sizeof(uint16_t),
                                 cudaMemcpyHostToDevice, st));
  }
  if (!vl.empty()) {
    if ((rc = dalloc(&op->d_vl, vl.size())) || (rc = dalloc(&op->d_vloff, vloff.size())) ||
        (rc = dalloc(&op->d_vgslot, vslot.size())))
      return fail(rc);
    HSV_TRY_CUDA(cudaMemcpyAsync(op->d_vgslot, vslot.data(), vslot.size() * sizeof(uint32_t),
                                 cudaMemcpyHostToDevice, st));
    HSV_TRY_CUDA(cudaMemcpyAsync(op->d_vl, vl.data(), vl.size() * sizeof(uint2),
                                 cudaMemcpyHostToDevice, st));
    HSV_TRY_CUDA(cudaMemcpyAsync(op->d_vloff, vloff.data(), vloff.size() * sizeof(int),
                                 cudaMemcpyHostToDevice, st));
    op->vl_chunk = vchunk;
    op->vl_nchunks = vnch;
  }
  if (!ghash.empty())
    HSV_TRY_CUDA(cudaMemcpyAsync(op->d_ghash, ghash.data(), ghash.size() * sizeof(GroupHash),
                                 cudaMemcpyHostToDevice, st));
  if (!tabs.empty())
    HSV_TRY_CUDA(cudaMemcpyAsync(op->d_tabs, tabs.data(), tabs.size() * sizeof(double),
                                 cudaMemcpyHostToDevice, st));
  if (!op->buckets.empty())
    HSV_TRY_CUDA(cudaMemcpyAsync(op->d_buckets, op->buckets.data(),
                                 op->buckets.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
  if (!op->groups.empty())
    HSV_TRY_CUDA(cudaMemcpyAsync(op->d_groups, op->groups.data(),
                                 op->groups.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
  if (!op->terms.empty())
    HSV_TRY_CUDA(cudaMemcpyAsync(op->d_terms, op->terms.data(), op->terms.size() * sizeof(Term),
                                 cudaMemcpyHostToDevice, st));
  if ((rc = stream_sync())) return fail(rc);
  op_phase("upload");
  dfree(d_all);
  *out = op;
  return HSV_OK;
}

int hsv_op_destroy(hsv_op op) {
  if (!op) return HSV_OK;
  dfree(op->d_buckets);
  dfree(op->d_groups);
  dfree(op->d_terms);
  dfree(op->d_diag);
  dfree(op->d_ghash);
  dfree(op->d_tabs);
  dfree(reinterpret_cast<unsigned char*>(op->d_recs));
  dfree(op->d_splits);
  dfree(op->d_vbuckets);
  dfree(op->d_gsz);
  dfree(reinterpret_cast<SzTerm*>(op->d_szt));
  dfree(op->d_gxa);
  dfree(op->d_bperm);
  dfree(op->d_vl);
  dfree(op->d_vloff);
  dfree(op->d_vgslot);
  drop_sells(op);
  delete op;
  return HSV_OK;
}

int hsv_op_sell_info(hsv_op op, int64_t a_lo, int64_t a_hi, int64_t* slots, int64_t* splits) {
  HSV_REQUIRE(op, HSV_ERR_INVALID, "null operator");
  int64_t n = 0, S = 0;
  for (const auto& m : op->sells)
    if (m.lo == a_lo && m.hi == a_hi) { n = m.entries; S = m.S; }
  if (slots) *slots = n;
  if (splits) *splits = S;
  return HSV_OK;
}

int hsv_op_info(hsv_op op, int64_t* n_terms, int64_t* n_groups, int64_t* n_active) {
  HSV_REQUIRE(op, HSV_ERR_INVALID, "null operator");
  if (n_terms) *n_terms = op->n_terms;
  if (n_groups) *n_groups = op->n_groups;
  if (n_active) *n_active = op->n_active;
  return HSV_OK;
}

static int csr_pass(hsv_op op, int64_t* d_counts, const int64_t* d_offsets, int64_t* d_cols,
                    double* d_vals) {
  hsv_sector s = op->sec;
  if (s->dim == 0) return HSV_OK;
  const unsigned nb = (unsigned)((s->dim + 127) / 128);
  if (s->wide)
    k_csr_rows<uint64_t, 32><<<nb, 128, 0, stream()>>>(
        s->d_Sa, s->d_Sb, s->d_Ra, s->d_Rb, s->Na, s->Nb, op->d_buckets, (int)op->n_buckets,
        op->d_groups, op->d_terms, op->d_diag, s->d_perm, d_counts, d_offsets, d_cols, d_vals);
  else
    k_csr_rows<uint32_t, 16><<<nb, 128, 0, stream()>>>(
        s->d_Sa, s->d_Sb, s->d_Ra, s->d_Rb, s->Na, s->Nb, op->d_buckets, (int)op->n_buckets,
        op->d_groups, op->d_terms, op->d_diag, s->d_perm, d_counts, d_offsets, d_cols, d_vals);
  count_launch();
  HSV_CHECK_LAUNCH();
  return HSV_OK;
}

int hsv_op_count_nnz(hsv_op op, int64_t* nnz) {
  HSV_REQUIRE(op && nnz, HSV_ERR_INVALID, "null argument");
  const int64_t dim = op->sec->dim;
  int64_t* d_counts = nullptr;
  HSV_TRY(dalloc(&d_counts, dim));
  HSV_TRY(csr_pass(op, d_counts, nullptr, nullptr, nullptr));
  std::vector<int64_t> h(dim);
  if (dim) HSV_TRY_CUDA(cudaMemcpyAsync(h.data(), d_counts, dim * 8, cudaMemcpyDeviceToHost, stream()));
  HSV_TRY(stream_sync());
  dfree(d_counts);
  int64_t t = 0;
  for (int64_t v : h) t += v;
  *nnz = t;
  return HSV_OK;
}

int hsv_op_to_csr(hsv_op op, int64_t* row_offsets, int64_t* cols, double* vals, int64_t cap) {
  HSV_REQUIRE(op && row_offsets, HSV_ERR_INVALID, "null argument");
  const int64_t dim = op->sec->dim;
  int64_t* d_counts = nullptr;
  HSV_TRY(dalloc(&d_counts, dim));
  HSV_TRY(csr_pass(op, d_counts, nullptr, nullptr, nullptr));
  std::vector<int64_t> cnt(dim);
  if (dim) HSV_TRY_CUDA(cudaMemcpyAsync(cnt.data(), d_counts, dim * 8, cudaMemcpyDeviceToHost, stream()));
  HSV_TRY(stream_sync());
  row_offsets[0] = 0;
  for (int64_t r = 0; r < dim; ++r) row_offsets[r + 1] = row_offsets[r] + cnt[r];
  const int64_t nnz = row_offsets[dim];
  HSV_REQUIRE(cap >= nnz && (nnz == 0 || (cols && vals)), HSV_ERR_INVALID,
              "CSR capacity %lld < nnz %lld", (long long)cap, (long long)nnz);
  int64_t *d_off = nullptr, *d_cols = nullptr;
  double* d_vals = nullptr;
  HSV_TRY(dalloc(&d_off, dim + 1));
  HSV_TRY(dalloc(&d_cols, nnz));
  HSV_TRY(dalloc(&d_vals, nnz));
  HSV_TRY_CUDA(cudaMemcpyAsync(d_off, row_offsets, (dim + 1) * 8, cudaMemcpyHostToDevice, stream()));
  HSV_TRY(csr_pass(op, nullptr, d_off, d_cols, d_vals));
  if (nnz) {
    HSV_TRY_CUDA(cudaMemcpyAsync(cols, d_cols, nnz * 8, cudaMemcpyDeviceToHost, stream()));
    HSV_TRY_CUDA(cudaMemcpyAsync(vals, d_vals, nnz * 8, cudaMemcpyDeviceToHost, stream()));
  }
  HSV_TRY(stream_sync());
  dfree(d_counts); dfree(d_off); dfree(d_cols); dfree(d_vals);
  // ascending columns within each row (CsrMatrix.from_coo lexsort, sparse.py:90-95)
  std::vector<std::pair<int64_t, double>> tmp;
  for (int64_t r = 0; r < dim; ++r) {
    const int64_t a = row_offsets[r], b = row_offsets[r + 1];
    tmp.clear();
    for (int64_t i = a; i < b; ++i) tmp.emplace_back(cols[i], vals[i]);
    std::sort(tmp.begin(), tmp.end(),
              [](const auto& p, const auto& q) { return p.first < q.first; });
    for (int64_t i = a; i < b; ++i) { cols[i] = tmp[i - a].first; vals[i] = tmp[i - a].second; }
  }
  return HSV_OK;
}

int hsv_apply_h(hsv_op op, hsv_state in, hsv_state out, double prune) {
  HSV_REQUIRE(op && in && out, HSV_ERR_INVALID, "null argument");
  HSV_REQUIRE(in->sec == op->sec && out->sec == op->sec, HSV_ERR_INVALID,
              "dimension mismatch: operator and vector belong to different sectors");
  HSV_REQUIRE(in != out, HSV_ERR_INVALID, "hsv_apply_h: output must not alias input");
  HSV_TRY(state_arow_async(in));
  HSV_TRY(launch_apply(op, in->d_amp, out->d_amp, nullptr, 0, op->sec->Na, prune, 0, nullptr,
                       in->d_arow, &in->dense_hint));
  out->norm2_valid = false;
  out->arow_valid = false;
  out->smap_valid = false;
  out->dense_hint = false;
  return stream_sync();
}

int hsv_apply_h_rows_async(hsv_op op, hsv_state in, hsv_state out, int64_t a_lo, int64_t a_hi,
                           double prune) {
  HSV_REQUIRE(op && in && out && in != out, HSV_ERR_INVALID, "bad argument");
  HSV_REQUIRE(in->sec == op->sec && out->sec == op->sec, HSV_ERR_INVALID, "dimension mismatch");
  HSV_REQUIRE(0 <= a_lo && a_lo <= a_hi && a_hi <= op->sec->Na, HSV_ERR_INVALID,
              "bad alpha-row range");
  HSV_TRY(state_arow_async(in));
  HSV_TRY(launch_apply(op, in->d_amp, out->d_amp, nullptr, a_lo, a_hi, prune, 0, nullptr,
                       in->d_arow, &in->dense_hint));
  out->norm2_valid = false;
  out->arow_valid = false;
  out->smap_valid = false;
  out->dense_hint = false;
  return HSV_OK;
}

int hsv_expect_h(hsv_op op, hsv_state psi, double* e_re, double* e_im) {
  HSV_REQUIRE(op && psi, HSV_ERR_INVALID, "null argument");
  HSV_REQUIRE(psi->sec == op->sec, HSV_ERR_INVALID, "dimension mismatch");
  const int nw = apply_warps(op);
  double *part = nullptr, *d_e = nullptr;
  HSV_TRY(dalloc(&part, 2 * (int64_t)nw));
  HSV_TRY(dalloc(&d_e, 2));
  HSV_TRY_CUDA(cudaMemsetAsync(part, 0, 2 * sizeof(double) * nw, stream()));
  int64_t used = 0;
  HSV_TRY(state_arow_async(psi));
  HSV_TRY(launch_apply(op, psi->d_amp, nullptr, part, 0, op->sec->Na, 0.0, 1, &used, psi->d_arow,
                       &psi->dense_hint));
  HSV_TRY(reduce_sum_f64(part, used, 2, 2, d_e));
  double h[2];
  HSV_TRY_CUDA(cudaMemcpyAsync(h, d_e, 16, cudaMemcpyDeviceToHost, stream()));
  HSV_TRY(stream_sync());
  dfree(part);
  dfree(d_e);
  if (e_re) *e_re = h[0];
  if (e_im) *e_im = h[1];
  return HSV_OK;
}

}  // extern "C"
