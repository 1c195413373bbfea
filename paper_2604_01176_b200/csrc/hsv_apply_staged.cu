// K1s: the K1 pull kernel with each bucket's partner alpha row staged in
// shared memory by TMA bulk copies (double-buffered, mbarrier-signalled), for
// sectors whose beta rows and rank table fit on chip (Nb <= 1024 and
// 2^norb <= 8192: H12 and below).
//
// One CTA per (alpha row, bucket split); warp w owns the 64 rows
// [64w, 64w + 64) of the alpha row, two per lane.  The CTA first compacts the
// list of buckets that pass its (CTA-uniform) alpha test and whose partner row
// holds a nonzero, then walks it: while the warps gather psi[b ^ x] from the
// staged partner row (and Rb from a staged copy of the rank table) for bucket
// i, the copy engine is already bringing in the row of bucket i + 1.  The
// per-row arithmetic and the summation order are those of k_apply with the
// same split, so results are bitwise identical to it (tests/test_gpu_staged.py).
// In k_apply every (row, group) pays an L1/L2 Rb lookup and an L1/L2 psi
// gather with 64-bit address math; here both are shared-memory loads.
#include <algorithm>

#include "hsv_common.cuh"
#include "hsv_kernels.cuh"

namespace hsv {

namespace {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arm(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// 1-D TMA bulk copy global -> shared, completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace

struct StagedArgs {
  ApplyArgs a;
  int rb_size;        // 2^norb entries of the rank table
  int stage_rb;       // 1: Rb staged in shared memory
};

constexpr int kStagedMaxWarps = 16;

template <int SH>
__global__ void __launch_bounds__(kStagedMaxWarps * 32, 2) k_apply_staged(const StagedArgs sa_) {
  using W = uint32_t;
  constexpr int R = 2;
  const ApplyArgs& a = sa_.a;
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t Nb = (uint32_t)a.Nb;
  double2* rows = reinterpret_cast<double2*>(smem);                       // [2][Nb]
  uint32_t* rb_s = reinterpret_cast<uint32_t*>(rows + 2 * Nb);            // [rb_size]
  int2* blist = reinterpret_cast<int2*>(rb_s + (sa_.stage_rb ? sa_.rb_size : 0));  // {bk, ra2}
  __shared__ uint64_t bar[2];
  __shared__ int n_list;
  __shared__ double esh[kStagedMaxWarps][2];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int sp = (int)(blockIdx.x % (unsigned)a.nsplit);
  const uint32_t ra = (uint32_t)a.a_lo + blockIdx.x / (unsigned)a.nsplit;
  const int bk0 = a.nsplit > 1 ? __ldg(a.split_bk + sp) : 0;
  const int bk1 = a.nsplit > 1 ? __ldg(a.split_bk + sp + 1) : a.n_buckets;
  const uint32_t sa = __ldg(a.Sa + ra);
  const uint32_t rowbase = ra * Nb;

  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (sa_.stage_rb)
    for (int i = threadIdx.x; i < sa_.rb_size; i += blockDim.x) rb_s[i] = __ldg(a.Rb + i);
  // ordered compaction of this CTA's active buckets (warp 0, 32 at a time)
  if (warp == 0) {
    int cnt = 0;
    for (int b0 = bk0; b0 < bk1; b0 += 32) {
      const int bk = b0 + lane;
      bool ok = false;
      uint32_t ra2 = 0;
      if (bk < bk1) {
        const int4 B = __ldg(a.buckets + bk);
        if (__popc(sa & (uint32_t)B.x) == B.y) {
          ra2 = __ldg(a.Ra + (sa ^ (uint32_t)B.x));
          ok = !a.arow || __ldg(a.arow + ra2);
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      if (ok) blist[cnt + __popc(m & ((1u << lane) - 1u))] = make_int2(bk, (int)ra2);
      cnt += __popc(m);
    }
    if (lane == 0) n_list = cnt;
  }
  __syncthreads();
  const int nl = n_list;
  const unsigned row_bytes = Nb * (unsigned)sizeof(double2);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 && i < nl; ++i) {
      mbar_arm(&bar[i], row_bytes);
      bulk_g2s(rows + i * Nb, a.psi + (size_t)blist[i].y * Nb, row_bytes, &bar[i]);
    }
  }

  // this warp's rows
  W s[R];
  uint32_t sb[R];
  double2 acc[R];
  unsigned live = 0u;
  const uint32_t rb0 = (uint32_t)warp * (32 * R) + lane;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const uint32_t rb = rb0 + k * 32;
    const bool inr = rb < Nb;
    sb[k] = inr ? __ldg(a.Sb + rb) : 0u;
    s[k] = (W)sa | ((W)sb[k] << SH);
    const double2 pv = inr ? a.psi[rowbase + rb] : make_double2(0.0, 0.0);
    const bool lv = inr && (!a.energy_only || pv.x != 0.0 || pv.y != 0.0);
    const double d = (a.diag && lv && sp == 0) ? a.diag[rowbase + rb] : 0.0;
    acc[k] = make_double2(d * pv.x, d * pv.y);
    live |= lv ? (1u << k) : 0u;
  }
  const bool any_live = __any_sync(0xffffffffu, live != 0u);
  const uint32_t* __restrict__ rbt = sa_.stage_rb ? rb_s : a.Rb;

  for (int i = 0; i < nl; ++i) {
    const int buf = i & 1;
    const int2 E = blist[i];
    const int4 B = __ldg(a.buckets + E.x);
    mbar_wait(&bar[buf], (unsigned)(i >> 1) & 1u);
    const double2* __restrict__ prow = rows + buf * Nb;
    if (any_live) {
      if (E.x < a.n_buckets_h) {   // x-local groups: amp = sign * table[hash(pattern)]
        const Rec<W>* __restrict__ rp = reinterpret_cast<const Rec<W>*>(a.recs);
        for (int g = B.z; g < B.w; ++g) {
          const Rec<W> cur = ldrec(rp + g);
          const uint32_t xb = cur.xb;
          const int hb = (int)(cur.meta & 0xffu);
          unsigned v = 0u;
#pragma unroll
          for (int k = 0; k < R; ++k)
            v |= ((live >> k) & 1u) && __popc(sb[k] & xb) == hb ? (1u << k) : 0u;
          if (__any_sync(0xffffffffu, v != 0u)) {
#pragma unroll
            for (int k = 0; k < R; ++k) {
              const double amp = rec_amp<W>(cur, s[k], a.tabs);
              if ((v >> k) & 1u) {
                const double2 p = prow[rbt[sb[k] ^ xb]];
                acc[k].x = fma(amp, p.x, acc[k].x);
                acc[k].y = fma(amp, p.y, acc[k].y);
              }
            }
          }
        }
      } else {   // term-loop groups (single-Z or generic), reference term order
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
          if (gz >> 63) {
            const SzTerm* __restrict__ sz = reinterpret_cast<const SzTerm*>(a.szt);
            for (int t = G.z; t < G.w; ++t) {
              const uint4 q = __ldg(reinterpret_cast<const uint4*>(sz + t));
#pragma unroll
              for (int k = 0; k < R; ++k) {
                const uint32_t sb31 = ((uint32_t)s[k] << q.z) & q.w;
                amp[k] += __hiloint2double((int)q.y ^ (int)sb31, (int)q.x);
              }
            }
#pragma unroll
            for (int k = 0; k < R; ++k) {
              const int sgn = popc(s[k] & (W)gz) << 31;
              amp[k] = __hiloint2double(__double2hiint(amp[k]) ^ sgn, __double2loint(amp[k]));
            }
          } else {
            for (int t = G.z; t < G.w; ++t) {
              const double c = __ldg(&a.terms[t].c);
              const W z = (W)__ldg(&a.terms[t].z);
#pragma unroll
              for (int k = 0; k < R; ++k) {
                const int sgn = popc(s[k] & z) << 31;
                amp[k] += __hiloint2double(__double2hiint(c) ^ sgn, __double2loint(c));
              }
            }
          }
#pragma unroll
          for (int k = 0; k < R; ++k) {
            if ((v >> k) & 1u) {
              const double2 p = prow[rbt[sb[k] ^ xb]];
              acc[k].x = fma(amp[k], p.x, acc[k].x);
              acc[k].y = fma(amp[k], p.y, acc[k].y);
            }
          }
        }
      }
    }
    __syncthreads();   // every warp is done with buffer `buf`
    if (threadIdx.x == 0 && i + 2 < nl) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arm(&bar[buf], row_bytes);
      bulk_g2s(rows + buf * Nb, a.psi + (size_t)blist[i + 2].y * Nb, row_bytes, &bar[buf]);
    }
  }

  // outputs (as k_apply) and the CTA's energy partial (fixed order)
  double er = 0.0, ei = 0.0;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const uint32_t rb = rb0 + k * 32;
    if (rb >= Nb) continue;
    if (a.out) {
      if (a.nsplit > 1) {
        a.ypart[(int64_t)sp * a.part_stride + (rowbase + rb - (uint32_t)a.a_lo * Nb)] = acc[k];
      } else {
        double2 y = acc[k];
        if (a.prune > 0.0 && sqrt(y.x * y.x + y.y * y.y) < a.prune) y = make_double2(0.0, 0.0);
        put_row(a.out, a.peer_rows, a.n_peer_rows, rowbase + rb, y);
      }
    }
    if (a.epart && ((live >> k) & 1u)) {
      const double2 pv = a.psi[rowbase + rb];
      er += pv.x * acc[k].x + pv.y * acc[k].y;
      ei += pv.x * acc[k].y - pv.y * acc[k].x;
    }
  }
  if (a.epart) {
    er = warp_sum(er);
    ei = warp_sum(ei);
    if (lane == 0) { esh[warp][0] = er; esh[warp][1] = ei; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double r = 0.0, m = 0.0;
      for (int w2 = 0; w2 < nwarps; ++w2) { r += esh[w2][0]; m += esh[w2][1]; }
      a.epart[2 * blockIdx.x] = r;
      a.epart[2 * blockIdx.x + 1] = m;
    }
  }
}

// Launch K1s when the sector fits (see the file comment); *done = false: use k_apply.
int launch_apply_staged(const hsv_op_s* op, const ApplyArgs& a0, int64_t* n_warps, bool* done) {
  *done = false;
  const hsv_sector_s* s = op->sec;
  if (tuning().staged == 0 || s->wide) return HSV_OK;
  const int64_t Nb = s->Nb, arows = a0.a_hi - a0.a_lo;
  const int rb_size = 1 << s->norb;
  if (Nb < 1 || Nb > 32 * 2 * kStagedMaxWarps || arows <= 0) return HSV_OK;
  const int stage_rb = rb_size <= 8192 ? 1 : 0;
  const int warps = (int)((Nb + 63) / 64);
  const size_t smem = 2 * Nb * sizeof(double2) + (stage_rb ? rb_size * sizeof(uint32_t) : 0) +
                      (size_t)std::max<int64_t>(op->n_buckets, 1) * sizeof(int2);
  if (smem > 100 * 1024) return HSV_OK;
  StagedArgs sa{};
  sa.a = a0;
  sa.rb_size = rb_size;
  sa.stage_rb = stage_rb;
  // splits: enough CTAs for several waves (2 resident per SM)
  int S = tuning().apply_split;
  if (S <= 0) {
    S = 1;
    while (S < 4 && arows * S < 8 * 2 * (int64_t)ctx().num_sms) S *= 2;
  }
  if (!a0.split_bk) S = 1;
  sa.a.nsplit = S;
  use_split_table(op, S, sa.a);
  const int64_t grid = arows * S;
  if (n_warps) *n_warps = grid;   // one energy partial per CTA
  if (a0.epart) HSV_REQUIRE(grid <= (int64_t)ctx().num_sms * 64, HSV_ERR_UNSUPPORTED,
                            "staged apply: too many CTAs for the energy partial buffer");
  const int64_t rows = arows * Nb;
  double2* ypart = nullptr;
  if (S > 1 && a0.out) {
    HSV_TRY(dalloc(&ypart, S * rows));
    sa.a.ypart = ypart;
    sa.a.part_stride = rows;
  }
  static bool attr = false;
  if (!attr) {
    HSV_TRY_CUDA(cudaFuncSetAttribute(k_apply_staged<16>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
    attr = true;
  }
  {
    ProfScope prof("apply");
    k_apply_staged<16><<<(unsigned)grid, warps * 32, smem, stream()>>>(sa);
    if (ypart)
      launch_combine_splits(ypart, S, rows, a0.out, a0.a_lo * Nb, a0.prune, a0.peer_rows,
                            a0.n_peer_rows);
  }
  count_launch(ypart ? 2 : 1);
  HSV_CHECK_LAUNCH();
  dfree(ypart);
  *done = true;
  return HSV_OK;
}

}  // namespace hsv
