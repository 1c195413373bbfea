// Matrix-free Pauli operator: upload/validation (replaces the CSR assembly of
// svengine.py:115-171) and the K1 pull kernel computing H|psi> and
// <psi|H|psi> (replaces spmspv + dot, sparse.py:163-219).
//
// Row b of H|psi> is   y_b = D_b psi_b + sum_{groups g, b^x_g in sector} amp_g(b) psi_{b^x_g}
// with amp_g(b) = sum_{t in g, ascending z} c_t (-1)^{popcount(b & z_t)}, the
// same sequential sum the reference forms per x-group (svengine.py:137-146),
// so every matrix element is bit-identical to the reference CSR value.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

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
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= Na * Nb) return;
  const int64_t ra = idx / Nb, rb = idx - ra * Nb;
  const W s = (W)Sa[ra] | ((W)Sb[rb] << SH);
  double amp = 0.0;
  for (int t = t0; t < t1; ++t) {
    const Term T = terms[t];
    amp += (popc(s & (W)T.z) & 1) ? -T.c : T.c;
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
template <typename W, int SH, int R>
__global__ void __launch_bounds__(256) k_apply(const ApplyArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t tw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t u0 = gw * a.units / tw, u1 = (gw + 1) * a.units / tw;
  double er = 0.0, ei = 0.0;
  for (int64_t u = u0; u < u1; ++u) {
    const int64_t ra = a.a_lo + u / a.upr;
    const int64_t ch = u % a.upr;
    const uint32_t sa = __ldg(a.Sa + ra);
    const int64_t rowbase = ra * a.Nb;
    W s[R];
    uint32_t sb[R];
    int64_t idx[R];
    bool live[R], inr[R];
    double2 acc[R], pv[R];
    bool anyl = false;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int64_t rb = ch * (32 * R) + k * 32 + lane;
      inr[k] = rb < a.Nb;
      sb[k] = inr[k] ? __ldg(a.Sb + rb) : 0u;
      s[k] = (W)sa | ((W)sb[k] << SH);
      idx[k] = rowbase + rb;
      pv[k] = inr[k] ? a.psi[idx[k]] : make_double2(0.0, 0.0);
      live[k] = inr[k] && (!a.energy_only || pv[k].x != 0.0 || pv[k].y != 0.0);
      const double d = (a.diag && live[k]) ? a.diag[idx[k]] : 0.0;
      acc[k] = make_double2(d * pv[k].x, d * pv[k].y);
      anyl |= live[k];
    }
    if (__any_sync(0xffffffffu, anyl)) {
      for (int bk = 0; bk < a.n_buckets; ++bk) {
        const int4 B = __ldg(a.buckets + bk);
        if (__popc(sa & (uint32_t)B.x) != B.y) continue;
        const double2* __restrict__ prow =
            a.psi + (int64_t)__ldg(a.Ra + (sa ^ (uint32_t)B.x)) * a.Nb;
        for (int g = B.z; g < B.w; ++g) {
          const int4 G = __ldg(a.groups + g);
          const uint32_t xb = (uint32_t)G.x;
          bool v[R];
          bool anyv = false;
#pragma unroll
          for (int k = 0; k < R; ++k) {
            v[k] = live[k] && __popc(sb[k] & xb) == G.y;
            anyv |= v[k];
          }
          if (!__any_sync(0xffffffffu, anyv)) continue;
          double amp[R];
#pragma unroll
          for (int k = 0; k < R; ++k) amp[k] = 0.0;
          for (int t = G.z; t < G.w; ++t) {
            const double c = __ldg(&a.terms[t].c);
            const W z = (W)__ldg(&a.terms[t].z);
#pragma unroll
            for (int k = 0; k < R; ++k) amp[k] += (popc(s[k] & z) & 1) ? -c : c;
          }
#pragma unroll
          for (int k = 0; k < R; ++k) {
            if (v[k]) {
              const double2 p = prow[__ldg(a.Rb + (sb[k] ^ xb))];
              acc[k].x = fma(amp[k], p.x, acc[k].x);
              acc[k].y = fma(amp[k], p.y, acc[k].y);
            }
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (!inr[k]) continue;
      if (a.out) {
        double2 y = acc[k];
        if (a.prune > 0.0 && sqrt(y.x * y.x + y.y * y.y) < a.prune) y = make_double2(0.0, 0.0);
        a.out[idx[k]] = y;
      }
      er += pv[k].x * acc[k].x + pv[k].y * acc[k].y;
      ei += pv[k].x * acc[k].y - pv[k].y * acc[k].x;
    }
  }
  if (a.epart) {
    er = warp_sum(er);
    ei = warp_sum(ei);
    if (lane == 0) {
      a.epart[2 * gw] = er;
      a.epart[2 * gw + 1] = ei;
    }
  }
}

template <typename W, int SH, int R>
static int launch_apply_t(const ApplyArgs& a0, int64_t* n_warps_out) {
  ApplyArgs a = a0;
  a.upr = (int)((a.Nb + 32 * R - 1) / (32 * R));
  a.units = (a.a_hi - a.a_lo) * a.upr;
  int occ = 0;
  HSV_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_apply<W, SH, R>, 256, 0));
  occ = std::max(occ, 1);
  int64_t grid = (int64_t)ctx().num_sms * occ;
  const int64_t need = (a.units + 7) / 8;
  grid = std::max<int64_t>(1, std::min(grid, need));
  if (n_warps_out) *n_warps_out = grid * 8;
  if (a.units == 0) return HSV_OK;
  ProfScope prof("apply");
  k_apply<W, SH, R><<<(unsigned)grid, 256, 0, stream()>>>(a);
  count_launch();
  HSV_CHECK_LAUNCH();
  return HSV_OK;
}

int apply_warps(const hsv_op_s* op) {
  // number of warps the apply kernel will use (for energy-partial sizing)
  int occ = 0;
  if (op->sec->wide)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_apply<uint64_t, 32, kApplyR>, 256, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_apply<uint32_t, 16, kApplyR>, 256, 0);
  return ctx().num_sms * std::max(occ, 1) * 8;
}

int launch_apply(const hsv_op_s* op, const double2* psi, double2* out, double* epart,
                 int64_t a_lo, int64_t a_hi, double prune, int energy_only, int64_t* n_warps) {
  const hsv_sector_s* s = op->sec;
  ApplyArgs a{};
  a.Sa = s->d_Sa; a.Sb = s->d_Sb; a.Ra = s->d_Ra; a.Rb = s->d_Rb;
  a.buckets = op->d_buckets; a.n_buckets = (int)op->n_buckets;
  a.groups = op->d_groups; a.terms = op->d_terms; a.diag = op->d_diag;
  a.psi = psi; a.out = out; a.epart = epart;
  a.Nb = s->Nb; a.a_lo = a_lo; a.a_hi = a_hi; a.prune = prune; a.energy_only = energy_only;
  if (s->wide) return launch_apply_t<uint64_t, 32, kApplyR>(a, n_warps);
  return launch_apply_t<uint32_t, 16, kApplyR>(a, n_warps);
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

  // ---- device validation: sector leak per off-diagonal group ----
  Term* d_all = nullptr;
  if ((rc = dalloc(&d_all, all_terms.size()))) return fail(rc);
  if (!all_terms.empty())
    HSV_TRY_CUDA(cudaMemcpyAsync(d_all, all_terms.data(), all_terms.size() * sizeof(Term),
                                 cudaMemcpyHostToDevice, stream()));
  std::vector<int> offd;
  for (int g = 0; g < (int)hg.size(); ++g)
    if (hg[g].x != 0) offd.push_back(g);
  const int n_off = (int)offd.size();
  std::vector<unsigned long long> leak(n_off, 0ull);
  if (n_off > 0 && s->dim > 0) {
    std::vector<uint32_t> gxa(n_off), gxb(n_off);
    std::vector<int32_t> gha(n_off), ghb(n_off), gt0(n_off), gt1(n_off);
    for (int j = 0; j < n_off; ++j) {
      const HGroup& g = hg[offd[j]];
      gxa[j] = g.xa; gxb[j] = g.xb;
      // odd popcount can never match: use an impossible target count
      gha[j] = g.pa % 2 ? -1 : g.pa / 2;
      ghb[j] = g.pb % 2 ? -1 : g.pb / 2;
      gt0[j] = g.t0; gt1[j] = g.t1;
    }
    uint32_t *d_gxa, *d_gxb;
    int32_t *d_gha, *d_ghb, *d_gt0, *d_gt1;
    unsigned long long* d_leak;
    if ((rc = dalloc(&d_gxa, n_off)) || (rc = dalloc(&d_gxb, n_off)) ||
        (rc = dalloc(&d_gha, n_off)) || (rc = dalloc(&d_ghb, n_off)) ||
        (rc = dalloc(&d_gt0, n_off)) || (rc = dalloc(&d_gt1, n_off)) ||
        (rc = dalloc(&d_leak, n_off)))
      return fail(rc);
    cudaStream_t st = stream();
    HSV_TRY_CUDA(cudaMemcpyAsync(d_gxa, gxa.data(), n_off * 4, cudaMemcpyHostToDevice, st));
    HSV_TRY_CUDA(cudaMemcpyAsync(d_gxb, gxb.data(), n_off * 4, cudaMemcpyHostToDevice, st));
    HSV_TRY_CUDA(cudaMemcpyAsync(d_gha, gha.data(), n_off * 4, cudaMemcpyHostToDevice, st));
    HSV_TRY_CUDA(cudaMemcpyAsync(d_ghb, ghb.data(), n_off * 4, cudaMemcpyHostToDevice, st));
    HSV_TRY_CUDA(cudaMemcpyAsync(d_gt0, gt0.data(), n_off * 4, cudaMemcpyHostToDevice, st));
    HSV_TRY_CUDA(cudaMemcpyAsync(d_gt1, gt1.data(), n_off * 4, cudaMemcpyHostToDevice, st));
    HSV_TRY_CUDA(cudaMemsetAsync(d_leak, 0, n_off * 8, st));
    dim3 grid((unsigned)((s->Nb + 127) / 128), (unsigned)s->Na);
    if (s->wide)
      k_leak<uint64_t, 32><<<grid, 128, 0, st>>>(s->d_Sa, s->d_Sb, s->Na, s->Nb, d_gxa, d_gxb,
                                                 d_gha, d_ghb, d_gt0, d_gt1, n_off, d_all, d_leak);
    else
      k_leak<uint32_t, 16><<<grid, 128, 0, st>>>(s->d_Sa, s->d_Sb, s->Na, s->Nb, d_gxa, d_gxb,
                                                 d_gha, d_ghb, d_gt0, d_gt1, n_off, d_all, d_leak);
    count_launch();
    HSV_CHECK_LAUNCH();
    HSV_TRY_CUDA(cudaMemcpyAsync(leak.data(), d_leak, n_off * 8, cudaMemcpyDeviceToHost, st));
    if ((rc = stream_sync())) return fail(rc);
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
  // ---- diagonal table ----
  for (const HGroup& g : hg) {
    if (g.x != 0 || s->dim == 0) continue;
    if ((rc = dalloc(&op->d_diag, s->dim))) return fail(rc);
    const unsigned nb = (unsigned)((s->dim + 255) / 256);
    if (s->wide)
      k_diag<uint64_t, 32><<<nb, 256, 0, stream()>>>(s->d_Sa, s->d_Sb, s->Na, s->Nb, d_all,
                                                     g.t0, g.t1, op->d_diag);
    else
      k_diag<uint32_t, 16><<<nb, 256, 0, stream()>>>(s->d_Sa, s->d_Sb, s->Na, s->Nb, d_all,
                                                     g.t0, g.t1, op->d_diag);
    count_launch();
    HSV_CHECK_LAUNCH();
  }
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
  if ((rc = dalloc(&op->d_buckets, op->buckets.size())) ||
      (rc = dalloc(&op->d_groups, op->groups.size())) ||
      (rc = dalloc(&op->d_terms, op->terms.size())))
    return fail(rc);
  cudaStream_t st = stream();
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
  delete op;
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
  HSV_TRY(launch_apply(op, in->d_amp, out->d_amp, nullptr, 0, op->sec->Na, prune, 0, nullptr));
  out->norm2_valid = false;
  return stream_sync();
}

int hsv_apply_h_rows_async(hsv_op op, hsv_state in, hsv_state out, int64_t a_lo, int64_t a_hi,
                           double prune) {
  HSV_REQUIRE(op && in && out && in != out, HSV_ERR_INVALID, "bad argument");
  HSV_REQUIRE(in->sec == op->sec && out->sec == op->sec, HSV_ERR_INVALID, "dimension mismatch");
  HSV_REQUIRE(0 <= a_lo && a_lo <= a_hi && a_hi <= op->sec->Na, HSV_ERR_INVALID,
              "bad alpha-row range");
  HSV_TRY(launch_apply(op, in->d_amp, out->d_amp, nullptr, a_lo, a_hi, prune, 0, nullptr));
  out->norm2_valid = false;
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
  HSV_TRY(launch_apply(op, psi->d_amp, nullptr, part, 0, op->sec->Na, 0.0, 1, &used));
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
