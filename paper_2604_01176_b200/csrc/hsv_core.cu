// libhsv core: context/errors, sectors (CiBasis replacement), states
// (SparseVector replacement) and deterministic reductions.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <unordered_map>

#include <chrono>
#include <cstdlib>

#include "hsv_common.cuh"
#include "hsv_kernels.cuh"

namespace hsv {

// ---------------------------------------------------------------- errors
static thread_local std::string g_err;
static thread_local int g_code = HSV_OK;

void set_error(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  g_code = code;
}
int last_code() { return g_code; }

// --------------------------------------------------------------- context
static Context g_ctx;
Context& ctx() { return g_ctx; }

int ensure_init() {
  if (g_ctx.device >= 0) return HSV_OK;
  int dev = 0;
  HSV_TRY_CUDA(cudaGetDevice(&dev));
  return hsv_init(dev);
}

static int64_t watch_ms() {
  static const int64_t v = [] {
    const char* e = getenv("HSV_WATCH_MS");
    return e ? (int64_t)atoll(e) : (int64_t)-1;
  }();
  return v;
}
static int64_t now_us() {
  return std::chrono::duration_cast<std::chrono::microseconds>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}
HostWatch::HostWatch(const char* what, int64_t bytes) : what_(what), bytes_(bytes) {
  if (watch_ms() >= 0) t0_ = now_us();
}
HostWatch::~HostWatch() {
  if (t0_ < 0) return;
  const int64_t dt = now_us() - t0_;
  if (dt < watch_ms() * 1000) return;
  if (bytes_ >= 0) {
    fprintf(stderr, "[hsv watch] %s %.3f ms (%lld bytes)\n", what_, dt * 1e-3, (long long)bytes_);
  } else {
    fprintf(stderr, "[hsv watch] %s %.3f ms\n", what_, dt * 1e-3);
  }
}

// ------------------------------------------------------ device arena
// Scratch and states are carved from large chunks the library owns (cudaMalloc
// once, kept): best-fit free ranges with splitting and coalescing inside a
// chunk, stream-ordered like cudaMallocAsync (one library stream; a block freed
// by earlier work is handed to later work on the same stream).  On the GPU
// boxes every trip to the driver -- cudaMallocAsync pool growth, and even pool
// remaps of an unchanged reservation -- cost 3-550 ms (profiles/r02/alloc_stalls.txt),
// so the ADAPT loop must not make any once warm.
namespace {
constexpr size_t kAlign = 512;
constexpr size_t kChunk = (size_t)512 << 20;   // new chunks: max(request, 512 MB)
struct Arena {
  std::mutex mu;
  struct Chunk { char* base; size_t size; };
  std::vector<Chunk> chunks;
  std::multimap<size_t, char*> free_by_size;        // size -> start
  std::map<char*, std::pair<size_t, int>> free_by_addr;   // start -> (size, chunk)
  std::unordered_map<char*, std::pair<size_t, int>> live;  // start -> (size, chunk)
  size_t reserved = 0, in_use = 0;
  int64_t driver_allocs = 0;
};
Arena& arena() {
  static Arena a;
  return a;
}
void erase_free(Arena& A, std::map<char*, std::pair<size_t, int>>::iterator it) {
  auto r = A.free_by_size.equal_range(it->second.first);
  for (auto q = r.first; q != r.second; ++q)
    if (q->second == it->first) { A.free_by_size.erase(q); break; }
  A.free_by_addr.erase(it);
}
void insert_free(Arena& A, char* p, size_t n, int chunk) {
  // coalesce with the free neighbours of the same chunk
  auto nx = A.free_by_addr.lower_bound(p);
  if (nx != A.free_by_addr.end() && nx->second.second == chunk && p + n == nx->first) {
    n += nx->second.first;
    erase_free(A, nx);
  }
  auto pv = A.free_by_addr.lower_bound(p);
  if (pv != A.free_by_addr.begin()) {
    --pv;
    if (pv->second.second == chunk && pv->first + pv->second.first == p) {
      p = pv->first;
      n += pv->second.first;
      erase_free(A, pv);
    }
  }
  A.free_by_addr[p] = {n, chunk};
  A.free_by_size.emplace(n, p);
}
// give wholly free chunks back to the driver (synchronizes)
int arena_trim_locked(Arena& A) {
  if (cudaStreamSynchronize(stream()) != cudaSuccess) cudaGetLastError();
  for (size_t c = 0; c < A.chunks.size(); ++c) {
    auto it = A.free_by_addr.find(A.chunks[c].base);
    if (A.chunks[c].base && it != A.free_by_addr.end() && it->second.first == A.chunks[c].size) {
      erase_free(A, it);
      cudaFree(A.chunks[c].base);
      A.reserved -= A.chunks[c].size;
      A.chunks[c] = {nullptr, 0};
    }
  }
  return HSV_OK;
}
}  // namespace

int cache_alloc(void** p, size_t bytes) {
  HostWatch hw("device allocation", (int64_t)bytes);
  bytes = (bytes + kAlign - 1) & ~(kAlign - 1);
  Arena& A = arena();
  std::lock_guard<std::mutex> lk(A.mu);
  auto it = A.free_by_size.lower_bound(bytes);
  if (it == A.free_by_size.end()) {   // new chunk
    // 25 % headroom: a buffer rebuilt a little larger each ADAPT iteration
    // (support-compacted rows) reuses its chunk after coalescing instead of
    // taking a new one from the driver every time
    size_t csz = std::max(((bytes + bytes / 4) + ((size_t)2 << 20) - 1) & ~(((size_t)2 << 20) - 1),
                          kChunk);
    char* base = nullptr;
    cudaError_t e = cudaMalloc(&base, csz);
    if (e != cudaSuccess && csz > bytes) {   // no room for a full chunk: exact size
      cudaGetLastError();
      csz = bytes;
      e = cudaMalloc(&base, csz);
    }
    if (e != cudaSuccess) {   // return wholly free chunks, retry once
      cudaGetLastError();
      arena_trim_locked(A);
      e = cudaMalloc(&base, csz);
    }
    if (e != cudaSuccess) {
      cudaGetLastError();
      set_error(HSV_ERR_OOM, "device allocation of %zu bytes failed: %s", bytes,
                cudaGetErrorString(e));
      return HSV_ERR_OOM;
    }
    A.chunks.push_back({base, csz});
    A.reserved += csz;
    ++A.driver_allocs;
    insert_free(A, base, csz, (int)A.chunks.size() - 1);
    it = A.free_by_size.lower_bound(bytes);
  }
  char* start = it->second;
  auto fa = A.free_by_addr.find(start);
  const size_t have = fa->second.first;
  const int chunk = fa->second.second;
  erase_free(A, fa);
  if (have > bytes) insert_free(A, start + bytes, have - bytes, chunk);   // split off the tail
  A.live[start] = {bytes, chunk};
  A.in_use += bytes;
  *p = start;
  return HSV_OK;
}

void cache_free(void* p) {
  Arena& A = arena();
  std::lock_guard<std::mutex> lk(A.mu);
  auto it = A.live.find(static_cast<char*>(p));
  if (it == A.live.end()) return;   // not an arena block (never happens: dalloc is the only source)
  A.in_use -= it->second.first;
  insert_free(A, it->first, it->second.first, it->second.second);
  A.live.erase(it);
}

int stream_sync() {
  HostWatch hw("cudaStreamSynchronize");
  cudaError_t e = cudaStreamSynchronize(stream());
  if (e != cudaSuccess) {
    set_error(HSV_ERR_CUDA, "CUDA error during stream synchronize: %s", cudaGetErrorString(e));
    return HSV_ERR_CUDA;
  }
  return HSV_OK;
}

const BinomTable& binom_host() {
  static BinomTable t;
  static std::once_flag once;
  std::call_once(once, [] {
    memset(&t, 0, sizeof(t));
    for (int n = 0; n < kBinomN; ++n) {
      t.c[n][0] = 1;
      for (int k = 1; k <= n; ++k) t.c[n][k] = t.c[n - 1][k - 1] + (k <= n - 1 ? t.c[n - 1][k] : 0);
    }
  });
  return t;
}

// ------------------------------------------------------------ reductions
// Column sums of a row-major [n x stride] array, fixed summation order.
// Coalesced variant: one thread per column, sequential over a chunk of rows.
__global__ void k_colsum_seq(const double* __restrict__ in, int64_t n, int64_t stride,
                             int64_t count, int64_t chunk, double* __restrict__ out) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t c = blockIdx.y;
  if (j >= count) return;
  int64_t i0 = c * chunk, i1 = min(n, i0 + chunk);
  double acc = 0.0;
  for (int64_t i = i0; i < i1; ++i) acc += in[i * stride + j];
  out[c * count + j] = acc;
}
// Tree variant for few columns: a block reduces `chunk` rows of one column.
__global__ void k_colsum_tree(const double* __restrict__ in, int64_t n, int64_t stride,
                              int64_t count, int64_t chunk, double* __restrict__ out) {
  __shared__ double sh[32];
  int64_t j = blockIdx.x;
  int64_t c = blockIdx.y;
  int64_t i0 = c * chunk, i1 = min(n, i0 + chunk);
  double acc = 0.0;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) acc += in[i * stride + j];
  acc = warp_sum(acc);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = acc;
  __syncthreads();
  if (w == 0) {
    double v = (l < (int)(blockDim.x >> 5)) ? sh[l] : 0.0;
    v = warp_sum(v);
    if (l == 0) out[c * count + j] = v;
  }
}

int reduce_sum_f64(const double* d_in, int64_t n, int64_t stride, int64_t count, double* d_out) {
  if (count <= 0) return HSV_OK;
  if (n <= 0) {
    HSV_TRY_CUDA(cudaMemsetAsync(d_out, 0, count * sizeof(double), stream()));
    return HSV_OK;
  }
  const bool seq = count >= 64;
  const double* src = d_in;
  int64_t src_n = n, src_stride = stride;
  double* tmp[2] = {nullptr, nullptr};
  int ping = 0;
  while (true) {
    // sequential column sums: enough (column block, row chunk) blocks for the
    // whole GPU (the screen's [rows x ops] partials: 38 -> ~8 us at H12), rows
    // per chunk fixed by (n, count) alone, so the sums stay deterministic
    int64_t chunk = 8192;
    if (seq) {
      const int64_t gx = (count + 127) / 128;
      const int64_t want = std::max<int64_t>(1, 2 * (int64_t)ctx().num_sms / gx);
      chunk = std::max<int64_t>(16, std::min<int64_t>(256, (src_n + want - 1) / want));
      if (src_n <= 256) chunk = src_n;   // short tail: finish in one launch
    } else if (src_n <= (1 << 20)) {
      chunk = src_n;   // few columns (energy partials of K1's units): one launch
    }
    int64_t nch = (src_n + chunk - 1) / chunk;
    double* dst;
    if (nch == 1) {
      dst = d_out;
    } else {
      if (!tmp[ping]) HSV_TRY(dalloc(&tmp[ping], (size_t)nch * count));
      dst = tmp[ping];
    }
    if (seq) {
      dim3 grid((unsigned)((count + 127) / 128), (unsigned)nch);
      k_colsum_seq<<<grid, 128, 0, stream()>>>(src, src_n, src_stride, count, chunk, dst);
    } else {
      dim3 grid((unsigned)count, (unsigned)nch);
      k_colsum_tree<<<grid, chunk >= 8192 ? 1024 : 256, 0, stream()>>>(src, src_n, src_stride,
                                                                        count, chunk, dst);
    }
    count_launch();
    HSV_CHECK_LAUNCH();
    if (nch == 1) break;
    src = dst;
    src_n = nch;
    src_stride = count;
    ping ^= 1;
  }
  dfree(tmp[0]);
  dfree(tmp[1]);
  return HSV_OK;
}

// ---------------------------------------------------------------- sector
// Reference position of every internal row: the closed-form rank of its key
// among the ascending sector keys (equals CiBasis position, cibasis.py:126-146).
__global__ void k_sector_perm(const uint32_t* __restrict__ Sa, const uint32_t* __restrict__ Sb,
                              int64_t Na, int64_t Nb, int n_qubits, int n_alpha, int n_beta,
                              const int32_t* __restrict__ qa, const int32_t* __restrict__ qb,
                              int norb, const int8_t* __restrict__ spin,
                              const int32_t* __restrict__ aslot, const int32_t* __restrict__ bslot,
                              const int64_t* __restrict__ binom, int64_t* __restrict__ perm,
                              int64_t* __restrict__ iperm) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= Na * Nb) return;
  int64_t ra = idx / Nb, rb = idx - ra * Nb;
  uint32_t sa = Sa[ra], sb = Sb[rb];
  uint64_t key = 0;
  for (int p = 0; p < norb; ++p) {
    key |= (uint64_t)((sa >> p) & 1u) << qa[p];
    key |= (uint64_t)((sb >> p) & 1u) << qb[p];
  }
  int al = n_alpha, bl = n_beta;
  int64_t pos = 0;
  for (int q = n_qubits - 1; q >= 0; --q) {
    if ((key >> q) & 1ull) {
      pos += dbinom(binom, aslot[q], al) * dbinom(binom, bslot[q], bl);
      if (spin[q] == 0) --al; else --bl;
    }
  }
  perm[idx] = pos;
  iperm[pos] = idx;
}

}  // namespace hsv

using namespace hsv;

extern "C" {

int hsv_abi_version(void) { return HSV_ABI_VERSION; }

int hsv_last_error(char* buf, size_t n) {
  if (buf && n) {
    size_t m = std::min(n - 1, g_err.size());
    memcpy(buf, g_err.data(), m);
    buf[m] = 0;
  }
  return g_code;
}

int hsv_init(int device) {
  if (g_ctx.device == device && g_ctx.stream) return HSV_OK;
  // one device per process: the device arena, the plans and every handle
  // belong to the first device
  HSV_REQUIRE(g_ctx.device < 0, HSV_ERR_INVALID,
              "libhsv is bound to CUDA device %d; one device per process (got %d)",
              g_ctx.device, device);
  HSV_TRY_CUDA(cudaSetDevice(device));
  HSV_TRY_CUDA(cudaFree(0));
  cudaDeviceProp prop;
  HSV_TRY_CUDA(cudaGetDeviceProperties(&prop, device));
  HSV_REQUIRE(prop.major >= 10, HSV_ERR_UNSUPPORTED,
              "libhsv is built for sm_100a (B200); device %d is sm_%d%d", device, prop.major,
              prop.minor);
  g_ctx.num_sms = prop.multiProcessorCount;
  g_ctx.l2_bytes = prop.l2CacheSize;
  if (!g_ctx.own) HSV_TRY_CUDA(cudaStreamCreateWithFlags(&g_ctx.own, cudaStreamNonBlocking));
  g_ctx.stream = g_ctx.own;
  g_ctx.device = device;
  cudaMemPool_t pool;
  HSV_TRY_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thr = UINT64_MAX;
  HSV_TRY_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  if (!g_ctx.d_stats) {
    HSV_TRY_CUDA(cudaMalloc(&g_ctx.d_stats, kStatCount * sizeof(unsigned long long)));
    HSV_TRY_CUDA(cudaMemset(g_ctx.d_stats, 0, kStatCount * sizeof(unsigned long long)));
  }
  return HSV_OK;
}

int hsv_stats(int64_t* out, int reset) {
  HSV_TRY(ensure_init());
  if (out) {
    HSV_TRY(stream_sync());
    HSV_TRY_CUDA(cudaMemcpy(out, g_ctx.d_stats, kStatCount * sizeof(int64_t),
                            cudaMemcpyDeviceToHost));
    // host-side slots: the stream-ordered pool's reserved / used bytes
    cudaMemPool_t pool;
    HSV_TRY_CUDA(cudaDeviceGetDefaultMemPool(&pool, g_ctx.device));
    uint64_t v = 0;
    HSV_TRY_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &v));
    out[kStatPoolReserved] = (int64_t)v;
    HSV_TRY_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &v));
    out[kStatPoolUsed] = (int64_t)v;
    Arena& A = arena();
    std::lock_guard<std::mutex> lk(A.mu);
    out[kStatCacheIdle] = (int64_t)(A.reserved - A.in_use);
    out[kStatCacheMisses] = A.driver_allocs;
  }
  if (reset)
    HSV_TRY_CUDA(cudaMemsetAsync(g_ctx.d_stats, 0, kStatCount * sizeof(unsigned long long),
                                 stream()));
  return HSV_OK;
}

int hsv_set_stream(void* s) {
  HSV_TRY(ensure_init());
  // blocks freed on the old stream may still be in use by its queued work:
  // drain it before they can be handed to work on the new one
  HSV_TRY(stream_sync());
  g_ctx.stream = s ? reinterpret_cast<cudaStream_t>(s) : g_ctx.own;
  return HSV_OK;
}
void* hsv_get_stream(void) {
  if (ensure_init() != HSV_OK) return nullptr;
  return reinterpret_cast<void*>(g_ctx.stream);
}
int64_t hsv_launch_count(int reset) {
  int64_t n = g_ctx.launches;
  if (reset) g_ctx.launches = 0;
  return n;
}
int hsv_mem_trim(void) {
  HSV_TRY(ensure_init());
  {
    Arena& A = arena();
    std::lock_guard<std::mutex> lk(A.mu);
    arena_trim_locked(A);
  }
  cudaMemPool_t pool;
  HSV_TRY_CUDA(cudaDeviceGetDefaultMemPool(&pool, g_ctx.device));
  HSV_TRY_CUDA(cudaMemPoolTrimTo(pool, 0));
  return HSV_OK;
}

int hsv_synchronize(void) {
  HSV_TRY(ensure_init());
  return stream_sync();
}

int hsv_sum_rows_async(const double* d_in, int64_t n_rows, int64_t n_cols, double* d_out) {
  HSV_TRY(ensure_init());
  HSV_REQUIRE(n_rows >= 0 && n_cols >= 0 && (n_cols == 0 || (d_in && d_out)), HSV_ERR_INVALID,
              "bad argument");
  if (n_cols == 0) return HSV_OK;
  if (n_rows == 0) {
    HSV_TRY_CUDA(cudaMemsetAsync(d_out, 0, n_cols * sizeof(double), stream()));
    return HSV_OK;
  }
  // one chunk: ((0 + row 0) + row 1) + ... per column, the rank-order sum
  dim3 grid((unsigned)((n_cols + 127) / 128), 1);
  k_colsum_seq<<<grid, 128, 0, stream()>>>(d_in, n_rows, n_cols, n_cols, n_rows, d_out);
  count_launch();
  HSV_CHECK_LAUNCH();
  return HSV_OK;
}

// ---------------------------------------------------------------- sector
int hsv_sector_create(int n_qubits, int n_alpha, int n_beta, int ordering, hsv_sector* out) {
  HSV_TRY(ensure_init());
  HSV_REQUIRE(out, HSV_ERR_INVALID, "null output handle");
  HSV_REQUIRE(ordering == HSV_INTERLEAVED || ordering == HSV_BLOCKED, HSV_ERR_INVALID,
              "unknown ordering %d; expected interleaved (0) or blocked (1)", ordering);
  HSV_REQUIRE(n_qubits > 0 && n_qubits % 2 == 0, HSV_ERR_INVALID,
              "n_qubits must be even (spin orbital pairs)");
  const int norb = n_qubits / 2;
  HSV_REQUIRE(0 <= n_alpha && n_alpha <= norb && 0 <= n_beta && n_beta <= norb, HSV_ERR_INVALID,
              "per-spin occupation exceeds the orbital count");
  HSV_REQUIRE(norb <= kMaxNorb, HSV_ERR_UNSUPPORTED,
              "n_qubits=%d exceeds the dense device layout limit (%d spatial orbitals)", n_qubits,
              kMaxNorb);
  auto* s = new hsv_sector_s();
  s->n_qubits = n_qubits;
  s->norb = norb;
  s->n_alpha = n_alpha;
  s->n_beta = n_beta;
  s->ordering = ordering;
  s->wide = norb > 16 ? 1 : 0;
  for (int p = 0; p < norb; ++p) {
    // cibasis.py:37-41 qubit_index
    s->qa[p] = ordering == HSV_INTERLEAVED ? 2 * p : p;
    s->qb[p] = ordering == HSV_INTERLEAVED ? 2 * p + 1 : p + norb;
  }
  const uint32_t nv = 1u << norb;
  s->Ra.assign(nv, ~0u);
  s->Rb.assign(nv, ~0u);
  for (uint32_t v = 0; v < nv; ++v) {
    int pc = __builtin_popcount(v);
    if (pc == n_alpha) { s->Ra[v] = (uint32_t)s->Sa.size(); s->Sa.push_back(v); }
    if (pc == n_beta) { s->Rb[v] = (uint32_t)s->Sb.size(); s->Sb.push_back(v); }
  }
  s->Na = (int64_t)s->Sa.size();
  s->Nb = (int64_t)s->Sb.size();
  s->dim = s->Na * s->Nb;

  int rc = HSV_OK;
  auto fail = [&](int code) { hsv_sector_destroy(s); return code; };
  if ((rc = dalloc(&s->d_Sa, s->Na)) || (rc = dalloc(&s->d_Sb, s->Nb)) ||
      (rc = dalloc(&s->d_Ra, nv)) || (rc = dalloc(&s->d_Rb, nv)) || (rc = dalloc(&s->d_Rb0, nv)) ||
      (rc = dalloc(&s->d_perm, s->dim)) || (rc = dalloc(&s->d_iperm, s->dim)) ||
      (rc = dalloc(&s->d_binom, kBinomN * kBinomN)) || (rc = dalloc(&s->d_spin, 64)) ||
      (rc = dalloc(&s->d_aslot, 64)) || (rc = dalloc(&s->d_bslot, 64)))
    return fail(rc);
  std::vector<int8_t> spin(64, 0);
  std::vector<int32_t> aslot(64, 0), bslot(64, 0), qa(32), qb(32);
  for (int q = 0; q < n_qubits; ++q)
    spin[q] = ordering == HSV_INTERLEAVED ? (q & 1) : (q < norb ? 0 : 1);
  int na = 0, nb = 0;
  for (int q = 0; q < n_qubits; ++q) {
    aslot[q] = na;
    bslot[q] = nb;
    if (spin[q] == 0) ++na; else ++nb;
  }
  for (int p = 0; p < 32; ++p) { qa[p] = s->qa[p]; qb[p] = s->qb[p]; }
  int32_t *d_qa = nullptr, *d_qb = nullptr;
  if ((rc = dalloc(&d_qa, 32)) || (rc = dalloc(&d_qb, 32))) return fail(rc);
  cudaStream_t st = stream();
  cudaError_t e = cudaSuccess;
  e = e ? e : cudaMemcpyAsync(s->d_Sa, s->Sa.data(), s->Na * 4, cudaMemcpyHostToDevice, st);
  e = e ? e : cudaMemcpyAsync(s->d_Sb, s->Sb.data(), s->Nb * 4, cudaMemcpyHostToDevice, st);
  e = e ? e : cudaMemcpyAsync(s->d_Ra, s->Ra.data(), nv * 4ull, cudaMemcpyHostToDevice, st);
  e = e ? e : cudaMemcpyAsync(s->d_Rb, s->Rb.data(), nv * 4ull, cudaMemcpyHostToDevice, st);
  std::vector<uint32_t> rb0(s->Rb);
  for (auto& r : rb0)
    if (r == ~0u) r = 0u;
  e = e ? e : cudaMemcpy(s->d_Rb0, rb0.data(), nv * 4ull, cudaMemcpyHostToDevice);
  e = e ? e : cudaMemcpyAsync(s->d_binom, binom_host().c, sizeof(BinomTable), cudaMemcpyHostToDevice, st);
  e = e ? e : cudaMemcpyAsync(s->d_spin, spin.data(), 64, cudaMemcpyHostToDevice, st);
  e = e ? e : cudaMemcpyAsync(s->d_aslot, aslot.data(), 64 * 4, cudaMemcpyHostToDevice, st);
  e = e ? e : cudaMemcpyAsync(s->d_bslot, bslot.data(), 64 * 4, cudaMemcpyHostToDevice, st);
  e = e ? e : cudaMemcpyAsync(d_qa, qa.data(), 32 * 4, cudaMemcpyHostToDevice, st);
  e = e ? e : cudaMemcpyAsync(d_qb, qb.data(), 32 * 4, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) {
    set_error(HSV_ERR_CUDA, "sector upload failed: %s", cudaGetErrorString(e));
    return fail(HSV_ERR_CUDA);
  }
  if (s->dim > 0) {
    int64_t nblk = (s->dim + 255) / 256;
    k_sector_perm<<<(unsigned)nblk, 256, 0, st>>>(s->d_Sa, s->d_Sb, s->Na, s->Nb, n_qubits,
                                                  n_alpha, n_beta, d_qa, d_qb, norb, s->d_spin,
                                                  s->d_aslot, s->d_bslot, s->d_binom,
                                                  s->d_perm, s->d_iperm);
    count_launch();
  }
  dfree(d_qa);
  dfree(d_qb);
  if ((rc = stream_sync())) return fail(rc);
  *out = s;
  return HSV_OK;
}

int hsv_sector_destroy(hsv_sector s) {
  if (!s) return HSV_OK;
  release_sweep_plans(s);   // cached sweep plans of this sector (hsv_sweep.cu)
  dfree(s->d_Sa); dfree(s->d_Sb); dfree(s->d_Ra); dfree(s->d_Rb); dfree(s->d_Rb0);
  dfree(s->d_perm); dfree(s->d_iperm); dfree(s->d_binom); dfree(s->d_spin);
  dfree(s->d_aslot); dfree(s->d_bslot);
  delete s;
  return HSV_OK;
}

int64_t hsv_sector_dim(hsv_sector s) { return s ? s->dim : -1; }

int hsv_sector_shape(hsv_sector s, int64_t* na, int64_t* nb) {
  HSV_REQUIRE(s, HSV_ERR_INVALID, "null sector");
  if (na) *na = s->Na;
  if (nb) *nb = s->Nb;
  return HSV_OK;
}

}  // extern "C"
