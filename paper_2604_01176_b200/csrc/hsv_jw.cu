// Device-side Jordan-Wigner build of the qubit Hamiltonian (reference
// mapping.py:79-126 + pauli.py:165-198): the spin-orbital tables h[P,Q],
// g[P,Q,R,S] (chemists' order, mapping.py:48-76) -> the merged, pruned,
// (x, z)-sorted real Pauli sum that hsv_op_create consumes.
//
//  * every nonzero table entry is a product of ladder operators (a+_p a_q, or
//    0.5 g a+_p a+_r a_s a_q); each ladder operator is two words (X_p Z_<p with
//    0.5, Y_p Z_<p with -+0.5i), so a product expands to 4 or 16 words, generated
//    in the reference's nested order (mapping.py:86-99) with its phase rule
//    (pauli.py:37-50).  Every contribution is exactly (+-scale / 2^m) times a
//    power of i, so the values are exact;
//  * a stable radix sort by the packed word (x << 32 | z) keeps, inside each
//    word, the reference's generation order (np.nonzero row-major, then the
//    expansion order), and each word's contributions are summed sequentially
//    from 0 in that order -- the reference's dict accumulation
//    (mapping.py:96-99), so the merged coefficients are bit-identical;
//  * residual imaginary parts above 1e-12 raise (mapping.py:116-121), and
//    coefficients with |c| <= drop_tol are dropped (pauli.py:190-198).
// Up to 32 qubits (packed 64-bit keys).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "hsv_common.cuh"
#include "hsv_kernels.cuh"

namespace hsv {

namespace {

struct Prod {        // one nonzero table entry: up to 4 ladder operators
  int8_t op[4];      // qubit of each factor
  int8_t dag[4];     // 1: creation
  int n;             // 2 or 4 factors
  double scale;
};

__device__ __forceinline__ int pc(uint64_t v) { return __popcll(v); }

// term (x1, z1, c1) times ladder word w of factor (p, dag): the reference's
// mul_words phase and complex product c1 * c2 * i^k (exact values)
__device__ __forceinline__ void mul_ladder(uint64_t& x, uint64_t& z, double& cr, double& ci, int p,
                                           int dag, int w) {
  const uint64_t x2 = 1ull << p;
  const uint64_t z2 = w ? ((x2 - 1) | x2) : (x2 - 1);
  // ladder coefficient: w = 0 -> 0.5, w = 1 -> -0.5i (creation) / +0.5i (annihilation)
  const double c2r = w ? 0.0 : 0.5;
  const double c2i = w ? (dag ? -0.5 : 0.5) : 0.0;
  const uint64_t x3 = x ^ x2, z3 = z ^ z2;
  const int k = ((pc(x & z) + pc(x2 & z2) - pc(x3 & z3) + 2 * pc(z & x2)) % 4 + 4) % 4;
  // c1 * c2 (each operand purely real or purely imaginary: exact)
  double pr = __dadd_rn(__dmul_rn(cr, c2r), -__dmul_rn(ci, c2i));
  double pi = __dadd_rn(__dmul_rn(cr, c2i), __dmul_rn(ci, c2r));
  // times i^k
  for (int q = 0; q < k; ++q) {
    const double t = pr;
    pr = -pi;
    pi = t;
  }
  x = x3;
  z = z3;
  cr = pr;
  ci = pi;
}

// word j of product i (j in [0, 2^n)): the reference's nested expansion order
__global__ void k_jw_words(const Prod* __restrict__ prods, const int64_t* __restrict__ off,
                           int64_t n_prod, int64_t n_words, int n_qubits,
                           uint64_t* __restrict__ keys, uint32_t* __restrict__ idx,
                           double2* __restrict__ vals) {
  // slot 0 is the core (identity) word; product words fill slots 1..n_words-1
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + 1;
  if (t >= n_words) return;
  int64_t lo = 0, hi = n_prod;   // product of slot t (off[i] = first slot of product i)
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) / 2;
    if (off[mid] <= t) lo = mid; else hi = mid;
  }
  const Prod P = prods[lo];
  const int j = (int)(t - off[lo]);
  uint64_t x = 0, z = 0;
  double cr = P.scale, ci = 0.0;
  for (int f = 0; f < P.n; ++f) {
    const int w = (j >> (P.n - 1 - f)) & 1;   // first factor = most significant choice
    mul_ladder(x, z, cr, ci, P.op[f], P.dag[f], w);
  }
  (void)n_qubits;
  keys[t] = (x << 32) | z;
  idx[t] = (uint32_t)t;
  vals[t] = make_double2(cr, ci);
}

// one thread per word: segment heads (first key of a run)
__global__ void k_jw_heads(const uint64_t* __restrict__ keys, int64_t n, int* __restrict__ head) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) head[t] = (t == 0 || keys[t] != keys[t - 1]) ? 1 : 0;
}

// one thread per distinct word: its contributions summed in generation order
__global__ void k_jw_sum(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ gen,
                         const double2* __restrict__ vals, const int* __restrict__ start,
                         int64_t n_seg, int64_t n, double2* __restrict__ out_c,
                         uint64_t* __restrict__ out_k) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n_seg) return;
  const int64_t a = start[s];
  const int64_t b = s + 1 < n_seg ? start[s + 1] : n;
  double re = 0.0, im = 0.0;
  for (int64_t i = a; i < b; ++i) {
    const double2 v = vals[gen[i]];
    re = __dadd_rn(re, v.x);
    im = __dadd_rn(im, v.y);
  }
  out_c[s] = make_double2(re, im);
  out_k[s] = keys[a];
}

}  // namespace

}  // namespace hsv

using namespace hsv;

extern "C" {

int hsv_jordan_wigner(int n_qubits, const double* h, const double* g, double core_energy,
                      double drop_tol, int64_t* xs, int64_t* zs, double* coeffs, int64_t cap,
                      int64_t* n_out) {
  HSV_TRY(ensure_init());
  HSV_REQUIRE(n_qubits > 0 && n_qubits <= 32 && h && g && n_out, HSV_ERR_INVALID,
              "hsv_jordan_wigner: bad argument (1..32 qubits, tables required)");
  const int n = n_qubits;
  // products in the reference's order: core, one-body (np.nonzero row-major),
  // two-body (row-major over P, Q, R, S) -- mapping.py:105-114
  std::vector<Prod> prods;
  std::vector<int64_t> off(1, 0);
  for (int p = 0; p < n; ++p)
    for (int q = 0; q < n; ++q) {
      const double v = h[p * n + q];
      if (v == 0.0) continue;
      Prod P{};
      P.n = 2;
      P.op[0] = (int8_t)p; P.dag[0] = 1;
      P.op[1] = (int8_t)q; P.dag[1] = 0;
      P.scale = v;
      prods.push_back(P);
      off.push_back(off.back() + 4);
    }
  for (int p = 0; p < n; ++p)
    for (int q = 0; q < n; ++q)
      for (int r = 0; r < n; ++r)
        for (int s = 0; s < n; ++s) {
          const double v = g[(((int64_t)p * n + q) * n + r) * n + s];
          if (v == 0.0) continue;
          Prod P{};
          P.n = 4;
          P.op[0] = (int8_t)p; P.dag[0] = 1;
          P.op[1] = (int8_t)r; P.dag[1] = 1;
          P.op[2] = (int8_t)s; P.dag[2] = 0;
          P.op[3] = (int8_t)q; P.dag[3] = 0;
          P.scale = 0.5 * v;
          prods.push_back(P);
          off.push_back(off.back() + 16);
        }
  const int64_t n_prod = (int64_t)prods.size();
  const int64_t n_words = off.back() + 1;            // + the core word, generation index 0
  HSV_REQUIRE(n_words < (int64_t)UINT32_MAX, HSV_ERR_UNSUPPORTED, "too many Pauli words");
  Prod* d_prod = nullptr;
  int64_t* d_off = nullptr;
  uint64_t *keys = nullptr, *keys2 = nullptr, *ok = nullptr;
  uint32_t *gen = nullptr, *gen2 = nullptr;
  double2 *vals = nullptr, *sums = nullptr;
  int *head = nullptr, *start = nullptr, *n_seg_d = nullptr;
  HSV_TRY(dalloc(&d_prod, std::max<int64_t>(n_prod, 1)));
  HSV_TRY(dalloc(&d_off, n_prod + 1));
  HSV_TRY(dalloc(&keys, n_words));
  HSV_TRY(dalloc(&keys2, n_words));
  HSV_TRY(dalloc(&gen, n_words));
  HSV_TRY(dalloc(&gen2, n_words));
  HSV_TRY(dalloc(&vals, n_words));
  cudaStream_t st = stream();
  if (n_prod)
    HSV_TRY_CUDA(cudaMemcpyAsync(d_prod, prods.data(), n_prod * sizeof(Prod),
                                 cudaMemcpyHostToDevice, st));
  // word 0 = core (identity), then the products' words shifted by one
  std::vector<int64_t> off1(off);
  for (auto& o : off1) o += 1;
  HSV_TRY_CUDA(cudaMemcpyAsync(d_off, off1.data(), (n_prod + 1) * sizeof(int64_t),
                               cudaMemcpyHostToDevice, st));
  const uint64_t zero_key = 0;
  const uint32_t zero_gen = 0;
  const double2 core = make_double2(core_energy, 0.0);
  HSV_TRY_CUDA(cudaMemcpyAsync(keys, &zero_key, 8, cudaMemcpyHostToDevice, st));
  HSV_TRY_CUDA(cudaMemcpyAsync(gen, &zero_gen, 4, cudaMemcpyHostToDevice, st));
  HSV_TRY_CUDA(cudaMemcpyAsync(vals, &core, 16, cudaMemcpyHostToDevice, st));
  if (n_words > 1) {
    // generation index t + 1 for word t of the products
    k_jw_words<<<(unsigned)((n_words - 1 + 255) / 256), 256, 0, st>>>(
        d_prod, d_off, n_prod, n_words, n, keys, gen, vals);
    count_launch();
    HSV_CHECK_LAUNCH();
  }
  size_t tb = 0;
  cub::DoubleBuffer<uint64_t> dk(keys, keys2);
  cub::DoubleBuffer<uint32_t> dv(gen, gen2);
  // key = x << 32 | z: bits [0, n) and [32, 32 + n)
  HSV_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int)n_words, 0, 32 + n, st));
  char* tmp = nullptr;
  HSV_TRY(dalloc(&tmp, tb));
  HSV_TRY_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, (int)n_words, 0, 32 + n, st));
  count_launch();
  dfree(tmp);
  const uint64_t* sk = dk.Current();
  const uint32_t* sg = dv.Current();
  HSV_TRY(dalloc(&head, n_words));
  HSV_TRY(dalloc(&start, n_words));
  HSV_TRY(dalloc(&n_seg_d, 1));
  k_jw_heads<<<(unsigned)((n_words + 255) / 256), 256, 0, st>>>(sk, n_words, head);
  count_launch();
  tb = 0;
  cub::CountingInputIterator<int> ci(0);
  HSV_TRY_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, ci, head, start, n_seg_d, (int)n_words, st));
  HSV_TRY(dalloc(&tmp, tb));
  HSV_TRY_CUDA(cub::DeviceSelect::Flagged(tmp, tb, ci, head, start, n_seg_d, (int)n_words, st));
  count_launch();
  dfree(tmp);
  int n_seg = 0;
  HSV_TRY_CUDA(cudaMemcpyAsync(&n_seg, n_seg_d, sizeof(int), cudaMemcpyDeviceToHost, st));
  HSV_TRY(stream_sync());
  HSV_TRY(dalloc(&sums, std::max(n_seg, 1)));
  HSV_TRY(dalloc(&ok, std::max(n_seg, 1)));
  k_jw_sum<<<(unsigned)((n_seg + 255) / 256), 256, 0, st>>>(sk, sg, vals, start, n_seg, n_words,
                                                            sums, ok);
  count_launch();
  HSV_CHECK_LAUNCH();
  std::vector<double2> hc(n_seg);
  std::vector<uint64_t> hk(n_seg);
  HSV_TRY_CUDA(cudaMemcpyAsync(hc.data(), sums, n_seg * sizeof(double2), cudaMemcpyDeviceToHost, st));
  HSV_TRY_CUDA(cudaMemcpyAsync(hk.data(), ok, n_seg * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  HSV_TRY(stream_sync());
  dfree(d_prod); dfree(d_off); dfree(keys); dfree(keys2); dfree(gen); dfree(gen2); dfree(vals);
  dfree(head); dfree(start); dfree(n_seg_d); dfree(sums); dfree(ok);
  double worst = 0.0;
  for (const double2& c : hc) worst = std::max(worst, std::fabs(c.y));
  HSV_REQUIRE(worst <= 1e-12, HSV_ERR_NONREAL,
              "residual imaginary Pauli coefficient %.3e; input is not Hermitian", worst);
  int64_t m = 0;
  for (int i = 0; i < n_seg; ++i) {
    if (!(std::fabs(hc[i].x) > drop_tol)) continue;
    if (xs && m < cap) {
      xs[m] = (int64_t)(hk[i] >> 32);
      zs[m] = (int64_t)(hk[i] & 0xffffffffull);
      coeffs[m] = hc[i].x;
    }
    ++m;
  }
  *n_out = m;
  HSV_REQUIRE(!xs || m <= cap, HSV_ERR_INVALID, "output capacity %lld < %lld terms",
              (long long)cap, (long long)m);
  return HSV_OK;
}

}  // extern "C"
