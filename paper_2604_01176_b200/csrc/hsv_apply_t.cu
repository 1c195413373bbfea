// K1t: H|psi> with alpha tiles -- the register-row K1 (hsv_apply.cu k_apply)
// gives each lane 8 rows of ONE alpha string (8 different beta strings), so
// every (row, group) pays the whole matrix-element pipeline: beta partner
// rank, hash of the pattern, table load, sign popcount, gather.
//
// Here a lane's 8 rows are 8 consecutive alpha strings with the SAME beta
// string (a work unit = 8 alpha rows x 32 beta ranks).  Per group and lane
// the beta half is computed once: the partner beta rank (one permutation-row
// load instead of 8), the beta sign parity, the beta bits of the hash input.
// Per alpha row only the alpha half remains, and that half is warp-uniform:
// for a bucket (fixed alpha flip xa) the alpha pattern sa & xa takes at most
// two values over the tile when |xa| = 2 (all alpha-beta doubles and alpha
// singles: the patterns 01 and 10), so the hash + table load run once per
// pattern, not once per row.  The gather of psi and the two FMAs stay per
// row.  Alpha validity per bucket is a warp-uniform mask over the 8 rows.
//
// Every row still sums its elements in the same group order with the same
// table values, signs and FMAs as K1 (diagonal first; pass-1 groups; then the
// term-loop groups; per bucket split), so the rows are bit-identical to K1's.
#include <algorithm>

#include "hsv_common.cuh"
#include "hsv_kernels.cuh"

namespace hsv {

namespace {

constexpr int kTA = 8;   // alpha rows per tile (rows per lane)

template <int RM>
__global__ void __launch_bounds__(256, 2) k_apply_t(const ApplyArgs a) {
  const int lane = threadIdx.x & 31;
  const uint32_t Nb = (uint32_t)a.Nb;
  const uint32_t nbc = (Nb + 31) / 32;                       // 32-rank beta chunks
  const uint32_t nt = (uint32_t)((a.a_hi - a.a_lo + kTA - 1) / kTA);
  const uint32_t units1 = nt * nbc;
  const uint32_t units = units1 * (uint32_t)a.nsplit;
  const Rec<uint32_t>* __restrict__ rp = reinterpret_cast<const Rec<uint32_t>*>(a.recs);
  auto grab = [&]() -> uint32_t {
    uint32_t v = 0;
    if (lane == 0) v = atomicAdd(a.ucounter, 1u);
    return __shfl_sync(0xffffffffu, v, 0);
  };
  for (uint32_t uw = grab(); uw < units; uw = grab()) {
    const int sp = (int)(uw / units1);                       // split-major, as K1
    const uint32_t u = uw - (uint32_t)sp * units1;
    const uint32_t tile = u / nbc, bc = u - tile * nbc;
    const int bk0 = a.split_bk ? __ldg(a.split_bk + sp) : 0;
    const int bk1 = a.split_bk ? __ldg(a.split_bk + sp + 1) : a.n_buckets;
    const uint32_t ra0 = (uint32_t)a.a_lo + tile * kTA;
    const uint32_t rb = bc * 32 + lane;
    const bool inr = rb < Nb;
    const uint32_t sb = inr ? __ldg(a.Sb + rb) : 0u;
    uint32_t sa[kTA];
    unsigned kval = 0u;                                       // alpha rows of the tile (uniform)
#pragma unroll
    for (int k = 0; k < kTA; ++k) {
      const bool ok = (int64_t)ra0 + k < a.a_hi;
      sa[k] = ok ? __ldg(a.Sa + ra0 + k) : 0u;
      kval |= ok ? (1u << k) : 0u;
    }
    double2 acc[kTA];
    unsigned live = 0u;                                       // per lane
#pragma unroll
    for (int k = 0; k < kTA; ++k) {
      acc[k] = make_double2(0.0, 0.0);
      if (((kval >> k) & 1u) && inr) {
        const uint32_t row = (ra0 + k) * Nb + rb;
        const double2 pv = a.psi[row];
        const bool lv = !a.energy_only || pv.x != 0.0 || pv.y != 0.0;
        const double d = (a.diag && lv && sp == 0) ? a.diag[row] : 0.0;
        acc[k] = make_double2(d * pv.x, d * pv.y);
        live |= lv ? (1u << k) : 0u;
      }
    }
    if (__any_sync(0xffffffffu, live != 0u)) {
      // pass 1: x-local groups
      for (int bk = bk0; bk < min(bk1, a.n_buckets_h); ++bk) {
        const int4 B = __ldg(a.buckets + bk);
        const uint32_t xa = (uint32_t)B.x;
        unsigned vm = 0u;                                     // warp-uniform
        uint32_t roff[kTA];
#pragma unroll
        for (int k = 0; k < kTA; ++k) {
          roff[k] = 0u;
          if (!((kval >> k) & 1u) || __popc(sa[k] & xa) != B.y) continue;
          const uint32_t ra2 = __ldg(a.Ra + (sa[k] ^ xa));
          if (a.arow && !__ldg(a.arow + ra2)) continue;
          roff[k] = ra2 * Nb;
          vm |= 1u << k;
        }
        if (!vm) continue;
        // the tile's alpha patterns on xa: two values cover it in the common case
        uint32_t p0 = 0u, p1 = 0u;
        bool have0 = false, have1 = false, two = true;
#pragma unroll
        for (int k = 0; k < kTA; ++k) {   // (no dynamic register indexing)
          if (!((vm >> k) & 1u)) continue;
          const uint32_t pk = sa[k] & xa;
          if (!have0) { p0 = pk; have0 = true; }
          else if (pk != p0) {
            if (!have1) { p1 = pk; have1 = true; }
            else if (pk != p1) two = false;
          }
        }
        if (!have1) p1 = p0;
        for (int g = B.z; g < B.w; ++g) {
          const Rec<uint32_t> cur = ldrec(rp + g);
          const int shift = (int)((cur.meta >> 8) & 0xffu);
          const double* __restrict__ tab = a.tabs + cur.tab;
          // beta half, once per lane: partner rank, hash bits, sign parity
          const uint32_t rk = RM == 2 ? __ldg(a.bperm + (cur.pad0 + rb))
                                      : __ldg(a.Rb0 + (sb ^ cur.xb));
          const uint32_t sbm = (sb << 16) & cur.xm;
          const int sgb = __popc(sb & (cur.z0 >> 16)) & 1;
          double A0 = 0.0, A1 = 0.0;
          if (two) {
            A0 = __ldg(tab + ((uint32_t)((p0 | sbm) * cur.mul) >> shift));
            A1 = __ldg(tab + ((uint32_t)((p1 | sbm) * cur.mul) >> shift));
          }
#pragma unroll
          for (int k = 0; k < kTA; ++k) {
            if (!((vm >> k) & 1u)) continue;
            const uint32_t pk = sa[k] & xa;
            const double A = two ? (pk == p0 ? A0 : A1)
                                 : __ldg(tab + ((uint32_t)((pk | sbm) * cur.mul) >> shift));
            const int sgn = ((__popc(sa[k] & cur.z0 & 0xffffu) & 1) ^ sgb) << 31;
            const double amp = __hiloint2double(__double2hiint(A) ^ sgn, __double2loint(A));
            const double2 p = a.psi[roff[k] + rk];
            acc[k].x = fma(amp, p.x, acc[k].x);
            acc[k].y = fma(amp, p.y, acc[k].y);
          }
        }
      }
      // pass 2: term-loop groups (K1's arithmetic, per row)
      for (int bk = max(bk0, a.n_buckets_h); bk < bk1; ++bk) {
        const int4 B = __ldg(a.buckets + bk);
        const uint32_t xa = (uint32_t)B.x;
        unsigned vm = 0u;
        uint32_t roff[kTA];
#pragma unroll
        for (int k = 0; k < kTA; ++k) {
          roff[k] = 0u;
          if (!((kval >> k) & 1u) || __popc(sa[k] & xa) != B.y) continue;
          const uint32_t ra2 = __ldg(a.Ra + (sa[k] ^ xa));
          if (a.arow && !__ldg(a.arow + ra2)) continue;
          roff[k] = ra2 * Nb;
          vm |= 1u << k;
        }
        if (!vm) continue;
        for (int g = B.z; g < B.w; ++g) {
          const int4 G = __ldg(a.groups + g);
          const uint32_t xb = (uint32_t)G.x;
          const bool bok = inr && __popc(sb & xb) == G.y;
          if (!__any_sync(0xffffffffu, bok && (live & vm))) continue;
          const uint64_t gz = __ldg(a.gsz + g);
          const uint32_t rk = bok ? __ldg(a.Rb + (sb ^ xb)) : 0u;
#pragma unroll
          for (int k = 0; k < kTA; ++k) {
            if (!((vm >> k) & 1u)) continue;
            const uint32_t s = sa[k] | (sb << 16);
            double amp = 0.0;
            if (gz >> 63) {
              const SzTerm* __restrict__ sz = reinterpret_cast<const SzTerm*>(a.szt);
              for (int t = G.z; t < G.w; ++t) {
                const uint4 q = __ldg(reinterpret_cast<const uint4*>(sz + t));
                const uint32_t sb31 = (s << q.z) & q.w;
                amp += __hiloint2double((int)q.y ^ (int)sb31, (int)q.x);
              }
              const int sgn = __popc(s & (uint32_t)gz) << 31;
              amp = __hiloint2double(__double2hiint(amp) ^ sgn, __double2loint(amp));
            } else {
              for (int t = G.z; t < G.w; ++t) {
                const double c = __ldg(&a.terms[t].c);
                const uint32_t z = (uint32_t)__ldg(&a.terms[t].z);
                const int sgn = __popc(s & z) << 31;
                amp += __hiloint2double(__double2hiint(c) ^ sgn, __double2loint(c));
              }
            }
            if (bok && ((live >> k) & 1u)) {
              const double2 p = a.psi[roff[k] + rk];
              acc[k].x = fma(amp, p.x, acc[k].x);
              acc[k].y = fma(amp, p.y, acc[k].y);
            }
          }
        }
      }
    }
    // output rows (+ this unit's <psi|H psi> share, added in unit order)
    double er = 0.0, ei = 0.0;
#pragma unroll
    for (int k = 0; k < kTA; ++k) {
      if (!((kval >> k) & 1u) || !inr) continue;
      const uint32_t row = (ra0 + k) * Nb + rb;
      if (a.out) {
        if (a.nsplit > 1) {
          a.ypart[(int64_t)sp * a.part_stride + (row - (uint32_t)a.a_lo * Nb)] = acc[k];
        } else {
          double2 y = acc[k];
          if (a.prune > 0.0 && sqrt(y.x * y.x + y.y * y.y) < a.prune) y = make_double2(0.0, 0.0);
          put_row(a.out, a.peer_rows, a.n_peer_rows, row, y);
        }
      }
      if (a.upart && ((live >> k) & 1u)) {
        const double2 pv = a.psi[row];
        er += pv.x * acc[k].x + pv.y * acc[k].y;
        ei += pv.x * acc[k].y - pv.y * acc[k].x;
      }
    }
    if (a.upart) {
      er = warp_sum(er);
      ei = warp_sum(ei);
      if (lane == 0) { a.upart[2 * uw] = er; a.upart[2 * uw + 1] = ei; }
    }
  }
}

}  // namespace

int launch_apply_t(const hsv_op_s* op, const ApplyArgs& a0, int S, bool* done) {
  *done = false;
  if (op->sec->wide || tuning().apply_t != 1) return HSV_OK;
  ApplyArgs a = a0;
  a.nsplit = S;
  use_split_table(op, S, a);
  if (S <= 1) {
    a.split_bk = nullptr;
    a.buckets = op->d_buckets;
    a.n_buckets = (int)op->n_buckets;
    a.n_buckets_h = (int)op->n_buckets_h;
  }
  const bool bp = op->d_bperm && tuning().bperm != 0;
  a.bperm = op->d_bperm;
  const int64_t nt = (a.a_hi - a.a_lo + kTA - 1) / kTA;
  const int64_t units1 = nt * ((a.Nb + 31) / 32);
  a.units = units1 * S;
  if (a.units == 0) { *done = true; return HSV_OK; }
  const void* fn = bp ? (const void*)k_apply_t<2> : (const void*)k_apply_t<0>;
  int occ = 0;
  HSV_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, 0));
  occ = std::max(occ, 1);
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx().num_sms * occ,
                                                              (a.units + 7) / 8));
  unsigned int* ucounter = nullptr;
  double* upart = nullptr;
  HSV_TRY(dalloc(&ucounter, 1));
  HSV_TRY_CUDA(cudaMemsetAsync(ucounter, 0, sizeof(unsigned), stream()));
  a.ucounter = ucounter;
  a.upart = nullptr;
  if (a.epart) {
    HSV_TRY(dalloc(&upart, 2 * a.units));
    a.upart = upart;
  }
  const int64_t rows = (a.a_hi - a.a_lo) * a.Nb;
  double2* ypart = nullptr;
  if (S > 1 && a.out) {
    HSV_TRY(dalloc(&ypart, S * rows));
    a.ypart = ypart;
    a.part_stride = rows;
  }
  {
    ProfScope prof("apply");
    void* params[] = {&a};
    HSV_TRY_CUDA(cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(256), params, 0, stream()));
    if (ypart)
      launch_combine_splits(ypart, S, rows, a.out, a.a_lo * a.Nb, a.prune, a.peer_rows,
                            a.n_peer_rows);
  }
  count_launch(ypart ? 2 : 1);
  HSV_CHECK_LAUNCH();
  if (upart) HSV_TRY(reduce_sum_f64(upart, a.units, 2, 2, a.epart));
  dfree(upart);
  dfree(ucounter);
  dfree(ypart);
  *done = true;
  return HSV_OK;
}

}  // namespace hsv
