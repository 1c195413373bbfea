// NVLink peer exchange without NCCL: every rank maps the others' buffers by
// CUDA IPC, kernels store into peer memory directly, and arrival is published
// with system-scope release stores of an epoch counter into per-rank flags and
// observed with acquire loads on the device (stream-ordered, no host sync).
//
// Buffers are double-buffered by epoch parity: a rank can run ahead into the
// next exchange (writing the other half) while a slower peer still reads the
// current one; it cannot get two exchanges ahead, because every exchange ends
// with a wait for all ranks' arrival.
//
// Two users:
//  * hsv_peer_allgather_async: the per-rank (E, g) partials of the energy +
//    gradient step (replaces the NCCL all-gather in bench.py / distributed.py);
//  * hsv_eg_forward_peer_async: the rank's rows of w = H psi are stored into
//    every rank's buffer by the K1 epilogue itself (put_row), so the all-gather
//    of w rides on NVLink while K1 is still computing other rows -- the
//    compute + collective fusion of the multi-GPU adjoint sweep.
#include <cstdlib>
#include <cstring>
#include <string>

#include "hsv_common.cuh"
#include "hsv_kernels.cuh"

namespace hsv {

namespace {

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr uint64_t kAbortBit = 1ull << 63;   // flag value of a rank that gave up this exchange

// Publish `epoch` (or, abort != 0, epoch | kAbortBit) to every rank's flag slot
// of this rank, then wait -- bounded by timeout_ns -- until every rank has
// published this epoch.  A timeout or a peer's abort sets *err (1 timeout,
// 2 peer abort) and returns: the host reads it (hsv_peer_check) instead of the
// stream hanging forever on a dead or failed peer.
__device__ void publish_and_wait(char* const* bases, int world, int rank, int64_t flags_off,
                                 uint64_t epoch, int abort, uint64_t timeout_ns, int* err,
                                 unsigned sleep_ns) {
  __threadfence_system();
  const uint64_t mark = abort ? (epoch | kAbortBit) : epoch;
  for (int r = 0; r < world; ++r)
    st_release_sys(reinterpret_cast<uint64_t*>(bases[r] + flags_off) + rank, mark);
  const uint64_t* mine = reinterpret_cast<const uint64_t*>(bases[rank] + flags_off);
  const uint64_t t0 = globaltimer_ns();
  for (int r = 0; r < world; ++r) {
    while (true) {
      const uint64_t v = ld_acquire_sys(mine + r);
      if (v & kAbortBit) {
        if ((v & ~kAbortBit) >= epoch) { atomicMax(err, 2); break; }
      } else if (v >= epoch) {
        break;
      }
      if (globaltimer_ns() - t0 > timeout_ns) { atomicMax(err, 1); return; }
      __nanosleep(sleep_ns);
    }
  }
  __threadfence_system();
}

// copy n bytes (multiple of 16) from src to bases[r] + off for every rank r
__global__ void k_peer_put(const uint4* __restrict__ src, int64_t n16, char* const* bases,
                           int world, int64_t off) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
    const uint4 v = src[i];
    for (int r = 0; r < world; ++r) reinterpret_cast<uint4*>(bases[r] + off)[i] = v;
  }
}

// publish this rank's arrival for `epoch` to every rank, then wait for all
__global__ void k_peer_barrier(char* const* bases, int world, int rank, int64_t flags_off,
                               uint64_t epoch, int abort, uint64_t timeout_ns, int* err) {
  if (threadIdx.x != 0) return;
  publish_and_wait(bases, world, rank, flags_off, epoch, abort, timeout_ns, err, 64);
}

// all-gather + barrier + rank-order sum in one CTA: puts, then thread 0 publishes
// and waits (its system-scope fence is cumulative over the CTA's stores ordered
// before it by the barrier), then the sums read every rank's block
__global__ void __launch_bounds__(1024) k_peer_allreduce(const double* __restrict__ src,
                                                         int64_t n, char* const* bases,
                                                         int world, int rank, int64_t half,
                                                         int64_t flags_off, uint64_t epoch,
                                                         double* __restrict__ out,
                                                         uint64_t timeout_ns, int* err) {
  const int64_t n16 = n / 2;
  for (int64_t i = threadIdx.x; i < n16; i += blockDim.x) {
    const uint4 v = reinterpret_cast<const uint4*>(src)[i];
    for (int r = 0; r < world; ++r)
      reinterpret_cast<uint4*>(bases[r] + half + rank * n * (int64_t)sizeof(double))[i] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0)
    publish_and_wait(bases, world, rank, flags_off, epoch, 0, timeout_ns, err, 32);
  __syncthreads();
  const double* data = reinterpret_cast<const double*>(bases[rank] + half);
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    double acc = 0.0;
    for (int r = 0; r < world; ++r) acc += data[r * n + j];
    out[j] = acc;
  }
}

uint64_t peer_timeout_ns() {
  const char* e = getenv("HSV_PEER_TIMEOUT_S");
  const double s = e ? atof(e) : 60.0;
  return (uint64_t)((s > 0 ? s : 60.0) * 1e9);
}

int peer_barrier(hsv_peer_s* p, int abort = 0) {
  k_peer_barrier<<<1, 32, 0, stream()>>>(p->d_bases, p->world, p->rank, p->flags_off, p->epoch,
                                         abort, peer_timeout_ns(), p->d_err);
  count_launch();
  HSV_CHECK_LAUNCH();
  return HSV_OK;
}

}  // namespace

}  // namespace hsv

using namespace hsv;

extern "C" {

int hsv_peer_create(int world, int rank, int64_t bytes, hsv_peer* out, void* handle_out) {
  HSV_TRY(ensure_init());
  HSV_REQUIRE(out && handle_out && world >= 1 && rank >= 0 && rank < world && bytes > 0,
              HSV_ERR_INVALID, "bad argument");
  auto* p = new hsv_peer_s();
  p->world = world;
  p->rank = rank;
  p->bytes = (bytes + 255) / 256 * 256;
  p->flags_off = 2 * p->bytes;                          // two halves, then the flags
  const size_t total = (size_t)p->flags_off + (size_t)world * sizeof(uint64_t);
  cudaError_t e = cudaMalloc(&p->base, total);          // IPC needs a plain allocation
  if (e != cudaSuccess) {
    cudaGetLastError();
    delete p;
    set_error(HSV_ERR_OOM, "peer buffer of %zu bytes: %s", total, cudaGetErrorString(e));
    return HSV_ERR_OOM;
  }
  cudaMemset(p->base + p->flags_off, 0, (size_t)world * sizeof(uint64_t));
  if (cudaMalloc(&p->d_err, sizeof(int)) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(p->base);
    delete p;
    set_error(HSV_ERR_OOM, "peer error flag allocation failed");
    return HSV_ERR_OOM;
  }
  cudaMemset(p->d_err, 0, sizeof(int));
  cudaIpcMemHandle_t h;
  e = cudaIpcGetMemHandle(&h, p->base);
  if (e != cudaSuccess) {
    cudaGetLastError();
    cudaFree(p->base);
    delete p;
    set_error(HSV_ERR_CUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    return HSV_ERR_CUDA;
  }
  static_assert(sizeof(h) == 64, "IPC handle size");
  std::memcpy(handle_out, &h, sizeof(h));
  p->bases.assign(world, nullptr);
  p->bases[rank] = p->base;
  *out = p;
  return HSV_OK;
}

int hsv_peer_open(hsv_peer p, const void* handles) {
  HSV_REQUIRE(p && handles && !p->opened, HSV_ERR_INVALID, "bad argument");
  const char* hs = static_cast<const char*>(handles);
  for (int r = 0; r < p->world; ++r) {
    if (r == p->rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, hs + 64 * r, sizeof(h));
    void* ptr = nullptr;
    HSV_TRY_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    p->bases[r] = static_cast<char*>(ptr);
  }
  HSV_TRY_CUDA(cudaMalloc(&p->d_bases, p->world * sizeof(char*)));
  HSV_TRY_CUDA(cudaMemcpy(p->d_bases, p->bases.data(), p->world * sizeof(char*),
                          cudaMemcpyHostToDevice));
  HSV_TRY_CUDA(cudaDeviceSynchronize());   // flags zeroed everywhere before first use
  p->opened = true;
  return HSV_OK;
}

int hsv_peer_destroy(hsv_peer p) {
  if (!p) return HSV_OK;
  cudaDeviceSynchronize();
  for (int r = 0; r < p->world; ++r)
    if (r != p->rank && p->bases[r]) cudaIpcCloseMemHandle(p->bases[r]);
  if (p->d_bases) cudaFree(p->d_bases);
  if (p->base) cudaFree(p->base);
  if (p->d_err) cudaFree(p->d_err);
  delete p;
  return HSV_OK;
}

int hsv_peer_check(hsv_peer p) {
  HSV_REQUIRE(p, HSV_ERR_INVALID, "null peer");
  int h = 0;
  HSV_TRY(stream_sync());
  HSV_TRY_CUDA(cudaMemcpy(&h, p->d_err, sizeof(int), cudaMemcpyDeviceToHost));
  if (h) HSV_TRY_CUDA(cudaMemset(p->d_err, 0, sizeof(int)));
  HSV_REQUIRE(h != 1, HSV_ERR_CUDA,
              "NVLink peer exchange timed out (a peer did not arrive within "
              "HSV_PEER_TIMEOUT_S); its results are invalid");
  HSV_REQUIRE(h != 2, HSV_ERR_CUDA,
              "a peer rank aborted the NVLink exchange (its call failed); results are invalid");
  return HSV_OK;
}

int hsv_peer_data(hsv_peer p, void** d_data, int64_t* bytes) {
  HSV_REQUIRE(p, HSV_ERR_INVALID, "null peer");
  if (d_data) *d_data = p->base + (p->epoch & 1) * p->bytes;   // the latest exchange
  if (bytes) *bytes = p->bytes;
  return HSV_OK;
}

int hsv_peer_allgather_async(hsv_peer p, const void* d_src, int64_t n) {
  HSV_REQUIRE(p && p->opened && d_src, HSV_ERR_INVALID, "peer buffer not opened");
  HSV_REQUIRE(n > 0 && n % 16 == 0 && n * p->world <= p->bytes, HSV_ERR_INVALID,
              "allgather block of %lld bytes does not fit the peer buffer",
              (long long)n);
  ++p->epoch;
  const int64_t off = (p->epoch & 1) * p->bytes + p->rank * n;
  const int64_t n16 = n / 16;
  const int grid = (int)std::min<int64_t>((n16 + 255) / 256, (int64_t)ctx().num_sms * 4);
  {
    ProfScope prof("peer");
    k_peer_put<<<std::max(grid, 1), 256, 0, stream()>>>(static_cast<const uint4*>(d_src), n16,
                                                       p->d_bases, p->world, off);
    count_launch();
    HSV_CHECK_LAUNCH();
    HSV_TRY(peer_barrier(p));
  }
  return HSV_OK;
}

int hsv_peer_allreduce_async(hsv_peer p, const double* d_src, int64_t n, double* d_out) {
  HSV_REQUIRE(p && p->opened && d_src && d_out, HSV_ERR_INVALID, "peer buffer not opened");
  HSV_REQUIRE(n > 0 && n % 2 == 0 && n * 8 * p->world <= p->bytes, HSV_ERR_INVALID,
              "allreduce block of %lld doubles does not fit the peer buffer", (long long)n);
  ++p->epoch;
  {
    ProfScope prof("peer");
    k_peer_allreduce<<<1, 1024, 0, stream()>>>(d_src, n, p->d_bases, p->world, p->rank,
                                               (p->epoch & 1) * p->bytes, p->flags_off, p->epoch,
                                               d_out, peer_timeout_ns(), p->d_err);
    count_launch();
    HSV_CHECK_LAUNCH();
  }
  return HSV_OK;
}

int hsv_eg_forward_peer_async(hsv_op op, uint64_t hf_key, const uint64_t* occ,
                              const uint64_t* virt, const double* cs, const double* sn, int64_t k,
                              int64_t a_lo, int64_t a_hi, hsv_state psi, hsv_state w,
                              hsv_peer p) {
  HSV_REQUIRE(op && w && p && p->opened && w->sec == op->sec, HSV_ERR_INVALID, "bad argument");
  const int64_t wbytes = op->sec->dim * (int64_t)sizeof(double2);
  HSV_REQUIRE(wbytes <= p->bytes, HSV_ERR_INVALID, "peer buffer smaller than a state");
  ++p->epoch;
  const int64_t half = (p->epoch & 1) * p->bytes;
  // every rank's half for this epoch, as double2 row arrays
  std::vector<double2*> sinks(p->world);
  for (int r = 0; r < p->world; ++r) sinks[r] = reinterpret_cast<double2*>(p->bases[r] + half);
  double2** d_sinks = nullptr;
  HSV_TRY(dalloc(&d_sinks, p->world));
  HSV_TRY_CUDA(cudaMemcpyAsync(d_sinks, sinks.data(), p->world * sizeof(double2*),
                               cudaMemcpyHostToDevice, stream()));
  ctx().peer_rows = d_sinks;
  ctx().n_peer_rows = p->world;
  int rc = hsv_eg_forward_async(op, hf_key, occ, virt, cs, sn, k, a_lo, a_hi, psi, w);
  ctx().peer_rows = nullptr;
  ctx().n_peer_rows = 0;
  dfree(d_sinks);
  if (rc) {
    // still take part in this epoch's barrier, flagged as an abort, so the
    // other ranks stop waiting and report the failure (hsv_peer_check)
    const int saved = rc;
    std::string msg(256, '\0');
    hsv_last_error(&msg[0], msg.size());
    peer_barrier(p, 1);
    set_error(saved, "%s", msg.c_str());
    return saved;
  }
  {
    ProfScope prof("peer");
    HSV_TRY(peer_barrier(p));
  }
  // the local half now holds every rank's rows
  HSV_TRY_CUDA(cudaMemcpyAsync(w->d_amp, p->base + half, wbytes, cudaMemcpyDeviceToDevice,
                               stream()));
  w->norm2_valid = w->arow_valid = false;
  w->dense_hint = false;
  return HSV_OK;
}

}  // extern "C"
