// Shared internals of libhsv: context, error plumbing, object layouts and
// small device helpers.  See DESIGN.md for the data layout rationale.
#pragma once

#include <cuda_runtime.h>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/hsv.h"

namespace hsv {

constexpr int kMaxNorb = 20;          // dense alpha-major layout limit (C(20,10)^2 ~ 3.4e10 rows)
constexpr int kBinomN = 64;
constexpr double kSectorLeakTol = 1e-10;   // svengine.py:112
constexpr double kNormDriftTol = 1e-9;     // svengine.py:27

// ---------------------------------------------------------------- errors
void set_error(int code, const char* fmt, ...);
int last_code();

#define HSV_TRY_CUDA(call)                                                              \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      if (e_ == cudaErrorMemoryAllocation) {                                            \
        cudaGetLastError();                                                             \
        ::hsv::set_error(HSV_ERR_OOM, "device allocation failed (%s) at %s:%d",         \
                         cudaGetErrorString(e_), __FILE__, __LINE__);                   \
        return HSV_ERR_OOM;                                                             \
      }                                                                                 \
      ::hsv::set_error(HSV_ERR_CUDA, "CUDA error '%s' in %s at %s:%d",                  \
                       cudaGetErrorString(e_), #call, __FILE__, __LINE__);              \
      return HSV_ERR_CUDA;                                                              \
    }                                                                                   \
  } while (0)

#define HSV_CHECK_LAUNCH() HSV_TRY_CUDA(cudaGetLastError())

#define HSV_TRY(expr)             \
  do {                            \
    int rc_ = (expr);             \
    if (rc_ != HSV_OK) return rc_; \
  } while (0)

#define HSV_REQUIRE(cond, code, ...)              \
  do {                                            \
    if (!(cond)) {                                \
      ::hsv::set_error((code), __VA_ARGS__);      \
      return (code);                              \
    }                                             \
  } while (0)

// --------------------------------------------------------------- context
struct Context {
  int device = -1;
  cudaStream_t stream = nullptr;   // stream all work goes to
  cudaStream_t own = nullptr;      // library-owned stream
  int num_sms = 148;
  int64_t l2_bytes = 126ll << 20;
  int64_t launches = 0;
  // set by hsv_eg_forward_peer_async around its H application: K1 also stores
  // every output row into these peer buffers (NVLink), see ApplyArgs::peer_rows
  double2* const* peer_rows = nullptr;
  int n_peer_rows = 0;
  // device work counters (hsv_stats): exact units processed by the ADAPT
  // evaluation kernels, for the bench's algorithmic-byte accounting
  unsigned long long* d_stats = nullptr;
  // second stream (K4 phases overlapped with the K1a stream) and its events
  cudaStream_t aux = nullptr;
  std::vector<cudaEvent_t> aux_ev;
};
enum StatKey { kStatPairsFwd = 0, kStatPairsAdj = 1, kStatRowsK1r = 2, kStatCacheIdle = 4,
               kStatCacheMisses = 5, kStatPoolReserved = 6, kStatPoolUsed = 7, kStatCount = 8 };
Context& ctx();
int ensure_init();
inline cudaStream_t stream() { return ctx().stream; }
inline void count_launch(int n = 1) { ctx().launches += n; }

// Host-stall watch (diagnostics): with HSV_WATCH_MS=t in the environment, a
// watched host call that takes longer than t ms is reported on stderr with its
// label (allocations, synchronizations, copies and launches on the ADAPT path).
class HostWatch {
 public:
  explicit HostWatch(const char* what, int64_t bytes = -1);
  ~HostWatch();
 private:
  const char* what_;
  int64_t bytes_;
  int64_t t0_ = -1;
};

// Device scratch allocation, stream-ordered on the library stream, from the
// library's device arena (hsv_core.cu): large chunks taken from the driver once
// and sub-allocated, so the ADAPT loop does not go back to the driver once warm.
int cache_alloc(void** p, size_t bytes);
void cache_free(void* p);
template <typename T>
int dalloc(T** p, size_t n) {
  if (n == 0) n = 1;
  return cache_alloc(reinterpret_cast<void**>(p), n * sizeof(T));
}
template <typename T>
void dfree(T* p) {
  if (p) cache_free(const_cast<void*>(reinterpret_cast<const void*>(p)));
}
int stream_sync();   // stream sync + error mapping

// ------------------------------------------------------------- binomials
struct BinomTable {
  int64_t c[kBinomN][kBinomN];
};
const BinomTable& binom_host();
__device__ __forceinline__ int64_t dbinom(const int64_t* tab, int n, int k);

}  // namespace hsv

// ---------------------------------------------------------------- objects
// Sector: (n_alpha, n_beta) strings of norb spatial orbitals.  Compressed
// strings (bit p = spatial orbital p of that spin) are ranked in ascending
// order; the internal row index of (sa, sb) is Ra[sa] * Nb + Rb[sb].
struct hsv_sector_s {
  int n_qubits = 0, norb = 0, n_alpha = 0, n_beta = 0, ordering = 0;
  int64_t Na = 0, Nb = 0, dim = 0;
  int wide = 0;                     // 0: 32-bit packed words (norb<=16), 1: 64-bit
  int qa[32] = {0}, qb[32] = {0};   // qubit carrying alpha/beta orbital p
  std::vector<uint32_t> Sa, Sb;     // host: compressed string of each rank
  std::vector<uint32_t> Ra, Rb;     // host: rank of each compressed string (or ~0u)
  uint32_t *d_Sa = nullptr, *d_Sb = nullptr, *d_Ra = nullptr, *d_Rb = nullptr;
  uint32_t* d_Rb0 = nullptr;        // Rb with out-of-sector strings mapped to rank 0
  int64_t* d_perm = nullptr;        // internal row -> reference position
  int64_t* d_iperm = nullptr;       // reference position -> internal row
  int64_t* d_binom = nullptr;       // kBinomN x kBinomN
  int8_t* d_spin = nullptr;         // spin of each qubit (0 alpha, 1 beta)
  int32_t *d_aslot = nullptr, *d_bslot = nullptr;  // alpha/beta qubits below q
  uint32_t compress_a(uint64_t key) const {
    uint32_t s = 0;
    for (int p = 0; p < norb; ++p) s |= (uint32_t)((key >> qa[p]) & 1ull) << p;
    return s;
  }
  uint32_t compress_b(uint64_t key) const {
    uint32_t s = 0;
    for (int p = 0; p < norb; ++p) s |= (uint32_t)((key >> qb[p]) & 1ull) << p;
    return s;
  }
  uint64_t expand(uint32_t sa, uint32_t sb) const {
    uint64_t k = 0;
    for (int p = 0; p < norb; ++p) {
      k |= (uint64_t)((sa >> p) & 1u) << qa[p];
      k |= (uint64_t)((sb >> p) & 1u) << qb[p];
    }
    return k;
  }
};

// Matrix-free operator.  Off-diagonal x-groups that can map the sector into
// itself are bucketed by their alpha flip part; the diagonal group (x = 0) is
// pre-evaluated into a dense per-row table.
struct Term {          // 16 B: one pre-signed coefficient and its packed z mask
  double c;            // coeff * (-1)^(nY/2)   (svengine.py:140-144)
  uint64_t z;          // packed z: za | zb << SH
};
// Per active group: sign mask, pattern mask and perfect multiply-shift hash of
// an x-local group (tab >= 0), or tab = -1 for the sequential term loop.
struct GroupHash {
  uint64_t z0;
  uint64_t xm;
  uint64_t mul;
  int32_t shift;
  int32_t tab;
};

// Bucket split table for S = 2 << i parts (hsv_op_create): S runs of virtual
// buckets; split k is [cut[k], cut[k + 1]) of the table's virtual buckets.
constexpr int kSplitTables = 5;   // S = 2, 4, 8, 16, 32
struct SplitTable {
  int vb_off = 0, nb = 0, nbh = 0;   // in d_vbuckets; entries; of them hashed (first)
  int cut_off = 0;                   // S + 1 entries in d_splits
};

struct hsv_op_s {
  hsv_sector sec = nullptr;
  int64_t n_terms = 0, n_groups = 0, n_active = 0, n_buckets = 0;
  int4* d_buckets = nullptr;   // {xa, xa_pop/2, g0, g1}
  int4* d_groups = nullptr;    // {xb, xb_pop/2, t0, t1}
  Term* d_terms = nullptr;
  double* d_diag = nullptr;    // per internal row; nullptr if no diagonal terms
  GroupHash* d_ghash = nullptr;
  void* d_recs = nullptr;       // packed Rec<W> per group (kernel layout)
  uint16_t* d_bperm = nullptr;  // per-xb beta rank permutations (Rec.pad0 = slot), or nullptr
  uint32_t* d_vgslot = nullptr; // K1v: per group, its valid list's offset slot
  // K1v valid lists (hsv_apply_v.cu): for each distinct beta flip xb of a hashed
  // group, the beta strings whose partner sb ^ xb stays in the sector, in rank
  // order, as {rb | rank(sb ^ xb) << 16, sb}; d_vloff[Rec.pad1 + c] = first
  // entry with rb >= c * vl_chunk (vl_nchunks + 1 per list).  nullptr: not built.
  uint2* d_vl = nullptr;
  int* d_vloff = nullptr;
  int vl_chunk = 0, vl_nchunks = 0;
  int64_t n_buckets_h = 0;      // buckets [0, n_buckets_h) are x-local (hashed)
  int* d_splits = nullptr;      // split cuts (SplitTable::cut_off)
  int4* d_vbuckets = nullptr;   // virtual buckets of the split tables
  SplitTable split[kSplitTables];
  double* d_tabs = nullptr;
  int64_t n_hashed = 0;
  // term-loop groups whose terms differ from the first only by the flip
  // pattern and at most one extra Z ("single-Z" form, the singles):
  // d_gsz[g] = 1<<63 | z0 (0: generic loop), d_szt[t] per term
  uint64_t* d_gsz = nullptr;
  void* d_szt = nullptr;
  int64_t n_single_z = 0;
  uint32_t* d_gxa = nullptr;    // per group: alpha flip part (push path)
  int64_t g_hashed = 0;         // groups [0, g_hashed) are x-local
  // host copies of the active group table (for CSR materialization)
  std::vector<int4> buckets, groups;
  std::vector<Term> terms;
  // K1a: alpha-string rows [lo, hi) assembled once as a sliced ELL matrix
  // (chunks of 32 rows, entry j of a chunk's lane at off + 32 j), one segment
  // per bucket split in K1's accumulation order (hsv_apply.cu build_sell).
  // A few row ranges are kept (a rank's shard and the full range); declined
  // ranges (over the budget) are remembered so they are not counted again.
  struct Sell {
    int64_t lo = 0, hi = 0, chunks = 0, entries = 0;
    int S = 1;
    uint32_t* cols = nullptr;
    double* amps = nullptr;
    uint32_t* rcnt = nullptr;  // [row][split] stored elements (before padding; full ranges)
    uint64_t* off = nullptr;   // [chunk][split]
    uint32_t* len = nullptr;   // [chunk][split] entries per lane
  };
  std::vector<Sell> sells;
  std::vector<int4> sell_declined;   // {lo, hi, S, 0}
  // K1s: the support rows of one sweep plan's map, with only the elements whose
  // partner is in the map (psi is exactly zero elsewhere), compacted from the
  // range's K1a rows; rebuilt when the map changes (once per ADAPT iteration)
  Sell sup;
  uint32_t* sup_rows = nullptr;      // local rows of the support, ascending
  int64_t sup_n = 0;
  uint64_t sup_version = 0;
  uint64_t sup_seen = 0;             // the map version the last evaluation used, and
  int64_t sup_seen_evals = 0;        // how many evaluations in a row used it
};

struct hsv_pool_s {
  hsv_sector sec = nullptr;
  int64_t n = 0;
  int4* d = nullptr;          // {oa, va, ob, vb} compressed masks
  int* d_order = nullptr;     // operators in alpha-part order (screen kernel)
  int2* d_opl = nullptr;      // per operator: beta list {offset, length}, length -1: empty beta half
  int4* d_qa = nullptr;       // per screen slot q (alpha-part order): {oa, va, op, list offset}
  int* d_qn = nullptr;        // per slot: beta list length (-1: empty beta half)
  int2* d_blist = nullptr;    // beta source lists {rb_src, rb_tgt}
  std::vector<int4> h;
};

// NVLink peer exchange buffer (hsv_peer.cu): `bytes` of data then `world`
// arrival flags, one cudaMalloc allocation shared with the other ranks by IPC.
struct hsv_peer_s {
  int world = 1, rank = 0;
  int64_t bytes = 0, flags_off = 0;
  char* base = nullptr;                 // local allocation
  std::vector<char*> bases;             // every rank's mapping (bases[rank] == base)
  char** d_bases = nullptr;             // the same, in device memory
  unsigned int* d_counter = nullptr;    // last-CTA detection in the put kernel
  uint64_t epoch = 0;
  bool opened = false;
  int* d_err = nullptr;                 // 1: a wait timed out, 2: a peer aborted (hsv_peer_check)
};

struct hsv_state_s {
  hsv_sector sec = nullptr;
  double2* d_amp = nullptr;    // dim complex128, alpha-major internal order
  double* d_norm2 = nullptr;   // cached <psi|psi> (device scalar)
  bool norm2_valid = false;
  // Conservative alpha-row occupancy: d_arow[ra] != 0 if row ra may hold a
  // nonzero.  Kernels skip work whose inputs lie in empty alpha rows, which
  // changes no result (skipped terms are exact zeros).
  uint32_t* d_arow = nullptr;
  bool arow_valid = false;
  // Set when the K1 push path found psi too dense (skip its probe next time);
  // cleared by every write.  Only ever disables the push path.
  bool dense_hint = false;
  // Norm-drift flags of the forward sweep that built this state
  // (hsv_eg_forward_async), read by the hsv_eg_backward that consumes it: the
  // forward call does not wait for the device.
  int* d_pend_err = nullptr;
  double* d_pend_val = nullptr;
  // Structural support of an ansatz state (1 byte per row, allocated on first
  // use): the closure of the HF row under every rotation of the forward sweep
  // that built psi, theta = 0 included (hsv_eg_forward_async).  A superset of
  // the nonzeros, independent of exact cancellations, closed under each
  // rotation; the adjoint sweep reads w = H psi only there, so the
  // support-restricted K1 computes those rows only (hsv_apply.cu, K1r).
  uint8_t* d_smap = nullptr;
  bool smap_valid = false;
};

namespace hsv {
// Device helpers --------------------------------------------------------
__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int popc(uint32_t v) { return __popc(v); }
__device__ __forceinline__ int popc(uint64_t v) { return __popcll(v); }

__device__ __forceinline__ int64_t dbinom(const int64_t* tab, int n, int k) {
  return (k < 0 || n < 0 || k > n) ? 0 : tab[n * kBinomN + k];
}

// Deterministic block reductions (fixed shuffle tree + fixed smem order).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}

// Launch helpers
// RAII CUDA-event pair around a launch when profiling is enabled.
class ProfScope {
 public:
  explicit ProfScope(const char* name, cudaStream_t st = nullptr);   // nullptr: stream()
  ~ProfScope();
 private:
  const char* name_;
  cudaStream_t st_ = nullptr;
  cudaEvent_t a_ = nullptr;
  bool active_ = false;
};

// RAII host-time scope, accumulated under "h:<name>" next to the kernel
// scopes while profiling is enabled (hsv_prof_get("h:eg_fwd", ...)).
class HostProf {
 public:
  explicit HostProf(const char* name);
  ~HostProf();
 private:
  const char* name_;
  int64_t t0_ = -1;
};

int reduce_sum_f64(const double* d_in, int64_t n, int64_t stride, int64_t count,
                   double* d_out);   // d_out[j] = sum_i d_in[i*stride + j], j<count
int state_norm2_async(hsv_state st);
int state_fill_zero_async(hsv_state st);
// alpha-row occupancy flags of a raw amplitude array / of a state (lazy)
int arow_flags_async(const double2* amp, int64_t Na, int64_t Nb, uint32_t* flags);
int state_arow_async(hsv_state st);
}  // namespace hsv
