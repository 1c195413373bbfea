// K1v: H|psi> with per-group valid beta lists and shared-memory row
// accumulators -- the register-row K1 (hsv_apply.cu k_apply) spends ~43% of
// its (row, group) iterations at H12 on rows whose partner b ^ x leaves the
// sector (adding an exact +-0 from a zero table entry), because its lanes own
// fixed rows and the beta validity of a group varies from lane to lane.
//
// Here a warp owns a work unit = (alpha row, 1024-row beta chunk, bucket
// split) whose row accumulators live in shared memory (16 KB).  For every
// x-local group the lanes walk the group's VALID list -- the beta strings of
// the chunk whose partner stays in the sector, precomputed per distinct beta
// flip xb at upload ({rb | partner rank << 16, sb}) -- so every iteration is a
// nonzero matrix element: amp = (-1)^popc(s & z0) A[h(s & x)] (the same
// table and sign as K1), gather psi[a ^ xa, partner], y[rb] += amp * p.  A
// __syncwarp between groups orders the updates of a row, so each row still
// sums its elements in the reference's group order (diagonal first, pass-1
// groups, then the term-loop groups, per bucket split): the rows are
// bit-identical to K1's (up to the sign of an exact zero).  Term-loop groups
// (pass 2) keep K1's per-lane row ownership over the chunk.
//
// Row-restricted mode (K1r, smap != nullptr): entries whose row is outside
// the structural support are skipped (a per-chunk bitmask in shared memory).
#include <algorithm>

#include "hsv_common.cuh"
#include "hsv_kernels.cuh"

namespace hsv {

namespace {

constexpr int kVWarps = 4;   // warps (units in flight) per block
constexpr int kVChunk = 1024;

template <int LM>
__global__ void __launch_bounds__(32 * kVWarps) k_apply_v(const ApplyArgs a) {
  extern __shared__ double2 vsh[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double2* y = vsh + wib * kVChunk;
  uint32_t* bits = reinterpret_cast<uint32_t*>(vsh + kVWarps * kVChunk) + wib * (kVChunk / 32);
  const uint32_t Nb = (uint32_t)a.Nb;
  const uint32_t nch = (uint32_t)a.vl_nchunks;
  const uint32_t units1 = (uint32_t)((a.a_hi - a.a_lo) * nch);
  const uint32_t units = units1 * (uint32_t)a.nsplit;
  const Rec<uint32_t>* __restrict__ rp = reinterpret_cast<const Rec<uint32_t>*>(a.recs);
  auto grab = [&]() -> uint32_t {
    uint32_t v = 0;
    if (lane == 0) v = atomicAdd(a.ucounter, 1u);
    return __shfl_sync(0xffffffffu, v, 0);
  };
  for (uint32_t uw = grab(); uw < units; uw = grab()) {
    const int sp = (int)(uw / units1);           // split-major, as K1
    const uint32_t u = uw - (uint32_t)sp * units1;
    const uint32_t ur = u / nch, ch = u - ur * nch;
    const int bk0 = a.split_bk ? __ldg(a.split_bk + sp) : 0;
    const int bk1 = a.split_bk ? __ldg(a.split_bk + sp + 1) : a.n_buckets;
    const uint32_t ra = (uint32_t)a.a_lo + ur;
    const uint32_t sa = __ldg(a.Sa + ra);
    const uint32_t rowbase = ra * Nb;
    const uint32_t c0 = ch * kVChunk;
    const uint32_t cn = min((uint32_t)kVChunk, Nb - c0);
    if (LM) {   // support bits of the chunk
      bool any = false;
      for (uint32_t i0 = 0; i0 < cn; i0 += 32) {
        const uint32_t i = i0 + lane;
        const bool f = i < cn && a.smap[rowbase + c0 + i] != 0;
        const unsigned b = __ballot_sync(0xffffffffu, f);
        if (lane == 0) bits[i0 >> 5] = b;
        any |= b != 0u;
      }
      __syncwarp();
      if (!any) continue;   // no supported row in the chunk (the output pass zeroes them)
    }
    // y <- diagonal part (split 0 only), as K1
    for (uint32_t i = lane; i < cn; i += 32) {
      const uint32_t row = rowbase + c0 + i;
      const double2 pv = a.psi[row];
      const double d = (a.diag && sp == 0) ? a.diag[row] : 0.0;
      y[i] = make_double2(d * pv.x, d * pv.y);
    }
    __syncwarp();
    // pass 1: x-local groups over their valid lists
    for (int bk = bk0; bk < min(bk1, a.n_buckets_h); ++bk) {
      const int4 B = __ldg(a.buckets + bk);
      if (__popc(sa & (uint32_t)B.x) != B.y) continue;
      const uint32_t ra2 = __ldg(a.Ra + (sa ^ (uint32_t)B.x));
      if (a.arow && !__ldg(a.arow + ra2)) continue;
      const double2* __restrict__ prow = a.psi + (size_t)ra2 * Nb;
      for (int g = B.z; g < B.w; ++g) {
        const Rec<uint32_t> cur = ldrec(rp + g);
        const uint32_t vs = __ldg(a.vgslot + g);
        const int lo = __ldg(a.vloff + vs + ch), hi = __ldg(a.vloff + vs + ch + 1);
        const int shift = (int)((cur.meta >> 8) & 0xffu);
        const double* __restrict__ tab = a.tabs + cur.tab;
        // four entries per lane in flight: their list loads, table loads and
        // psi gathers issue before the shared-memory updates
        for (int i0 = lo; i0 < hi; i0 += 128) {
          uint2 e[4];
          bool ok[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int i = i0 + q * 32 + lane;
            ok[q] = i < hi;
            e[q] = ok[q] ? __ldg(a.vl + i) : make_uint2(0u, 0u);
            if (LM && ok[q]) {
              const uint32_t li = (e[q].x & 0xffffu) - c0;
              ok[q] = (bits[li >> 5] >> (li & 31)) & 1u;
            }
          }
          double amp[4];
          double2 p[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            amp[q] = 0.0;
            p[q] = make_double2(0.0, 0.0);
            if (ok[q]) {
              const uint32_t s = sa | (e[q].y << 16);
              const uint32_t h = (uint32_t)((s & cur.xm) * cur.mul) >> shift;
              const double A = __ldg(tab + h);
              const int sgn = __popc(s & cur.z0) << 31;
              amp[q] = __hiloint2double(__double2hiint(A) ^ sgn, __double2loint(A));
              p[q] = prow[e[q].x >> 16];
            }
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (!ok[q]) continue;
            const uint32_t li = (e[q].x & 0xffffu) - c0;
            double2 yv = y[li];
            yv.x = fma(amp[q], p[q].x, yv.x);
            yv.y = fma(amp[q], p[q].y, yv.y);
            y[li] = yv;
          }
        }
        __syncwarp();   // the next group's updates of a row come after this group's
      }
    }
    // pass 2: term-loop groups, each lane owning rows i = lane (mod 32) of the chunk
    for (int bk = max(bk0, a.n_buckets_h); bk < bk1; ++bk) {
      const int4 B = __ldg(a.buckets + bk);
      if (__popc(sa & (uint32_t)B.x) != B.y) continue;
      const uint32_t ra2 = __ldg(a.Ra + (sa ^ (uint32_t)B.x));
      if (a.arow && !__ldg(a.arow + ra2)) continue;
      const double2* __restrict__ prow = a.psi + (size_t)ra2 * Nb;
      for (int g = B.z; g < B.w; ++g) {
        const int4 G = __ldg(a.groups + g);
        const uint32_t xb = (uint32_t)G.x;
        const uint64_t gz = __ldg(a.gsz + g);
        for (uint32_t i = lane; i < cn; i += 32) {
          if (LM && !((bits[i >> 5] >> (i & 31)) & 1u)) continue;
          const uint32_t sb = __ldg(a.Sb + c0 + i);
          if (__popc(sb & xb) != G.y) continue;
          const uint32_t s = sa | (sb << 16);
          double amp = 0.0;
          if (gz >> 63) {   // single-Z group (K1 pass 2, exact)
            const SzTerm* __restrict__ sz = reinterpret_cast<const SzTerm*>(a.szt);
            for (int t = G.z; t < G.w; ++t) {
              const uint4 qq = __ldg(reinterpret_cast<const uint4*>(sz + t));
              const uint32_t sb31 = (s << qq.z) & qq.w;
              amp += __hiloint2double((int)qq.y ^ (int)sb31, (int)qq.x);
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
          const double2 p = prow[__ldg(a.Rb + (sb ^ xb))];
          double2 yv = y[i];
          yv.x = fma(amp, p.x, yv.x);
          yv.y = fma(amp, p.y, yv.y);
          y[i] = yv;
        }
      }
    }
    __syncwarp();
    // output rows of the chunk (+ this unit's <psi|H psi> share)
    double er = 0.0, ei = 0.0;
    for (uint32_t i = lane; i < cn; i += 32) {
      if (LM && !((bits[i >> 5] >> (i & 31)) & 1u)) continue;   // zeroed by the combine pass
      const uint32_t row = rowbase + c0 + i;
      const double2 acc = y[i];
      if (a.out) {
        if (a.nsplit > 1) {
          a.ypart[(int64_t)sp * a.part_stride + (row - (uint32_t)a.a_lo * Nb)] = acc;
        } else {
          double2 yv = acc;
          if (a.prune > 0.0 && sqrt(yv.x * yv.x + yv.y * yv.y) < a.prune) yv = make_double2(0.0, 0.0);
          put_row(a.out, a.peer_rows, a.n_peer_rows, row, yv);
        }
      }
      if (a.upart) {
        const double2 pv = a.psi[row];
        er += pv.x * acc.x + pv.y * acc.y;
        ei += pv.x * acc.y - pv.y * acc.x;
      }
    }
    if (a.upart) {
      er = warp_sum(er);
      ei = warp_sum(ei);
      if (lane == 0) { a.upart[2 * uw] = er; a.upart[2 * uw + 1] = ei; }
    }
    __syncwarp();   // y is reused by the warp's next unit
  }
}

}  // namespace

int launch_apply_v(const hsv_op_s* op, const ApplyArgs& a0, int S, bool* done) {
  *done = false;
  if (!op->d_vl || op->sec->wide || tuning().apply_v != 1) return HSV_OK;
  if (a0.n_peer_rows > 0 && S == 1 && a0.smap) return HSV_OK;   // K1r + peers need the combine
  ApplyArgs a = a0;
  a.vl = op->d_vl;
  a.vloff = op->d_vloff;
  a.vgslot = op->d_vgslot;
  a.vl_chunk = op->vl_chunk;
  a.vl_nchunks = op->vl_nchunks;
  a.nsplit = S;
  use_split_table(op, S, a);
  if (S <= 1) { a.split_bk = nullptr; a.buckets = op->d_buckets; a.n_buckets = (int)op->n_buckets;
                a.n_buckets_h = (int)op->n_buckets_h; }
  const int64_t units1 = (a.a_hi - a.a_lo) * op->vl_nchunks;
  a.units = units1 * S;
  if (a.units == 0) { *done = true; return HSV_OK; }
  const size_t smem = (size_t)kVWarps * kVChunk * sizeof(double2) + kVWarps * (kVChunk / 32) * 4;
  const void* fn = a.smap ? (const void*)k_apply_v<1> : (const void*)k_apply_v<0>;
  static bool attr[2] = {false, false};
  if (!attr[a.smap ? 1 : 0]) {
    HSV_TRY_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr[a.smap ? 1 : 0] = true;
  }
  int occ = 0;
  HSV_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 32 * kVWarps, smem));
  occ = std::max(occ, 1);
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx().num_sms * occ,
                                                              (a.units + kVWarps - 1) / kVWarps));
  unsigned int* ucounter = nullptr;
  double* upart = nullptr;
  HSV_TRY(dalloc(&ucounter, 1));
  HSV_TRY_CUDA(cudaMemsetAsync(ucounter, 0, sizeof(unsigned), stream()));
  a.ucounter = ucounter;
  a.upart = nullptr;
  if (a.epart) {
    HSV_TRY(dalloc(&upart, 2 * a.units));
    HSV_TRY_CUDA(cudaMemsetAsync(upart, 0, 2 * a.units * sizeof(double), stream()));
    a.upart = upart;
  }
  const int64_t rows = (a.a_hi - a.a_lo) * a.Nb;
  double2* ypart = nullptr;
  if (S > 1 && a.out) {
    HSV_TRY(dalloc(&ypart, S * rows));
    a.ypart = ypart;
    a.part_stride = rows;
  }
  if (a.smap && a.out && !ypart)   // rows outside the support are exact zeros
    HSV_TRY_CUDA(cudaMemsetAsync(a.out + a.a_lo * a.Nb, 0, rows * sizeof(double2), stream()));
  {
    ProfScope prof(a.smap ? "apply_rows" : "apply");
    void* params[] = {&a};
    HSV_TRY_CUDA(cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(32 * kVWarps), params, smem,
                                  stream()));
    if (ypart) {
      if (a.smap)
        launch_combine_splits_map(ypart, S, rows, a.out, a.a_lo * a.Nb, a.smap, a.peer_rows,
                                  a.n_peer_rows);
      else
        launch_combine_splits(ypart, S, rows, a.out, a.a_lo * a.Nb, a.prune, a.peer_rows,
                              a.n_peer_rows);
    }
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
