// Live per-kernel timing (CUDA events on the launching stream) and the
// persistent device operator pool used by the screen kernel.
#include <chrono>
#include <map>
#include <string>
#include <vector>

#include "hsv_common.cuh"
#include "hsv_kernels.cuh"

namespace hsv {

struct ProfPair {
  const char* name;
  cudaEvent_t a, b;
};
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> free_ev;
  std::vector<ProfPair> pending;
  std::map<std::string, std::pair<double, int64_t>> acc;
};
static Prof g_prof;
static Tuning g_tuning;
Tuning& tuning() { return g_tuning; }

static cudaEvent_t take_event() {
  if (g_prof.free_ev.empty()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  cudaEvent_t e = g_prof.free_ev.back();
  g_prof.free_ev.pop_back();
  return e;
}

static int64_t host_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}
HostProf::HostProf(const char* name) : name_(name) {
  if (g_prof.on) t0_ = host_ns();
}
HostProf::~HostProf() {
  if (t0_ < 0) return;
  auto& slot = g_prof.acc[std::string("h:") + name_];
  slot.first += (host_ns() - t0_) * 1e-6;
  slot.second += 1;
}

ProfScope::ProfScope(const char* name, cudaStream_t st) : name_(name), st_(st) {
  if (!g_prof.on) return;
  if (!st_) st_ = stream();
  a_ = take_event();
  cudaEventRecord(a_, st_);
  active_ = true;
}
ProfScope::~ProfScope() {
  if (!active_) return;
  cudaEvent_t b = take_event();
  cudaEventRecord(b, st_);
  g_prof.pending.push_back(ProfPair{name_, a_, b});
}

}  // namespace hsv

using namespace hsv;

extern "C" {

int hsv_set_tuning(const char* key, int64_t value) {
  HSV_REQUIRE(key, HSV_ERR_INVALID, "null key");
  const std::string k(key);
  if (k == "apply_r") {
    HSV_REQUIRE(value == 0 || value == 1 || value == 2 || value == 4 || value == 8,
                HSV_ERR_INVALID, "apply_r must be 0 (auto), 1, 2, 4 or 8");
    g_tuning.apply_r = (int)value;
  } else if (k == "apply_minb") {
    HSV_REQUIRE(value >= 0 && value <= 6, HSV_ERR_INVALID, "apply_minb must be in [0, 6]");
    g_tuning.apply_minb = (int)value;
  } else if (k == "apply_interleave") {
    HSV_REQUIRE(value >= -1 && value <= 2, HSV_ERR_INVALID,
                "apply_interleave must be -1, 0, 1 or 2");
    g_tuning.apply_interleave = (int)value;
  } else if (k == "apply_split") {
    HSV_REQUIRE(value >= 0 && value <= 32 && (value & (value - 1)) == 0, HSV_ERR_INVALID,
                "apply_split must be 0 (auto), 1, 2, 4, 8, 16 or 32");
    g_tuning.apply_split = (int)value;
  } else if (k == "bperm") {
    HSV_REQUIRE(value >= -1 && value <= 1, HSV_ERR_INVALID, "bperm must be -1, 0 or 1");
    g_tuning.bperm = (int)value;
  } else if (k == "rb0_smem") {
    HSV_REQUIRE(value >= -1 && value <= 1, HSV_ERR_INVALID, "rb0_smem must be -1, 0 or 1");
    g_tuning.rb0_smem = (int)value;
  } else if (k == "apply_t") {
    HSV_REQUIRE(value >= -1 && value <= 1, HSV_ERR_INVALID, "apply_t must be -1, 0 or 1");
    g_tuning.apply_t = (int)value;
  } else if (k == "apply_v") {
    HSV_REQUIRE(value >= -1 && value <= 1, HSV_ERR_INVALID, "apply_v must be -1, 0 or 1");
    g_tuning.apply_v = (int)value;
  } else if (k == "sweep_incr") {
    HSV_REQUIRE(value == 0 || value == 1, HSV_ERR_INVALID, "sweep_incr must be 0 or 1");
    g_tuning.sweep_incr = (int)value;
  } else if (k == "sweep_p2p") {
    HSV_REQUIRE(value == 0 || value == 1, HSV_ERR_INVALID, "sweep_p2p must be 0 or 1");
    g_tuning.sweep_p2p = (int)value;
  } else if (k == "restrict_rows") {
    HSV_REQUIRE(value >= -1 && value <= 1, HSV_ERR_INVALID, "restrict_rows must be -1, 0 or 1");
    g_tuning.restrict_rows = (int)value;
  } else if (k == "push") {
    HSV_REQUIRE(value >= -1 && value <= 1, HSV_ERR_INVALID, "push must be -1, 0 or 1");
    g_tuning.push = (int)value;
  } else if (k == "sweep") {
    HSV_REQUIRE(value >= 0 && value <= 2, HSV_ERR_INVALID, "sweep must be 0, 1 or 2");
    g_tuning.sweep = (int)value;
  } else if (k == "staged") {
    HSV_REQUIRE(value == 0 || value == 1, HSV_ERR_INVALID, "staged must be 0 or 1");
    g_tuning.staged = (int)value;
  } else if (k == "sell") {
    HSV_REQUIRE(value >= -1 && value <= 1, HSV_ERR_INVALID, "sell must be -1, 0 or 1");
    g_tuning.sell = (int)value;
  } else if (k == "screen_overlap") {
    HSV_REQUIRE(value >= 0 && value <= 64, HSV_ERR_INVALID, "screen_overlap must be 0..64");
    g_tuning.screen_overlap = (int)value;
  } else if (k == "sup") {
    HSV_REQUIRE(value >= -1 && value <= 1, HSV_ERR_INVALID, "sup must be -1, 0 or 1");
    g_tuning.sup = (int)value;
  } else if (k == "sell_sp") {
    HSV_REQUIRE(value >= -1 && value <= 1, HSV_ERR_INVALID, "sell_sp must be -1, 0 or 1");
    g_tuning.sell_sp = (int)value;
  } else if (k == "sell_kernel") {
    HSV_REQUIRE(value >= 0 && value <= 4, HSV_ERR_INVALID, "sell_kernel must be 0..4");
    g_tuning.sell_kernel = (int)value;
  } else if (k == "sell_budget_mb") {
    HSV_REQUIRE(value >= 0, HSV_ERR_INVALID, "sell_budget_mb must be >= 0");
    g_tuning.sell_budget_mb = value;
  } else if (k == "sweep_bar") {
    HSV_REQUIRE(value == 0 || value == 1, HSV_ERR_INVALID, "sweep_bar must be 0 or 1");
    g_tuning.sweep_bar = (int)value;
  } else if (k == "sweep_threads") {
    HSV_REQUIRE(value == 128 || value == 256, HSV_ERR_INVALID, "sweep_threads must be 128 or 256");
    g_tuning.sweep_threads = (int)value;
  } else if (k == "sweep_grid") {
    HSV_REQUIRE(value >= 0 && value <= (1 << 20), HSV_ERR_INVALID, "sweep_grid out of range");
    g_tuning.sweep_grid = (int)value;
  } else if (k == "push_keys") {
    HSV_REQUIRE(value >= 0 && value <= 4096, HSV_ERR_INVALID, "push_keys out of range");
    g_tuning.push_keys = (int)value;
  } else if (k == "screen_pivot") {
    HSV_REQUIRE(value >= -1 && value <= 1, HSV_ERR_INVALID, "screen_pivot must be -1, 0 or 1");
    g_tuning.screen_pivot = (int)value;
  } else if (k == "screen_rows") {
    HSV_REQUIRE(value >= 64 && value <= 8192, HSV_ERR_INVALID, "screen_rows out of range");
    g_tuning.screen_rows = (int)value;
  } else {
    set_error(HSV_ERR_INVALID, "unknown tuning key '%s'", key);
    return HSV_ERR_INVALID;
  }
  return HSV_OK;
}

int hsv_prof_enable(int on) {
  g_prof.on = on != 0;
  return HSV_OK;
}

int hsv_prof_collect(void) {
  HSV_TRY(stream_sync());
  for (auto& p : g_prof.pending) {
    float ms = 0.f;
    HSV_TRY_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    auto& slot = g_prof.acc[p.name];
    slot.first += ms;
    slot.second += 1;
    g_prof.free_ev.push_back(p.a);
    g_prof.free_ev.push_back(p.b);
  }
  g_prof.pending.clear();
  return HSV_OK;
}

int hsv_prof_get(const char* name, double* total_ms, int64_t* count) {
  auto it = g_prof.acc.find(name);
  if (total_ms) *total_ms = it == g_prof.acc.end() ? 0.0 : it->second.first;
  if (count) *count = it == g_prof.acc.end() ? 0 : it->second.second;
  return HSV_OK;
}

int hsv_prof_reset(void) {
  g_prof.acc.clear();
  return HSV_OK;
}

// ---- operator pool (compressed QEB masks resident on the device) ----
int hsv_pool_create(hsv_sector s, const uint64_t* occ, const uint64_t* virt, int64_t n,
                    hsv_pool* out) {
  HSV_TRY(ensure_init());
  HSV_REQUIRE(s && out && (n == 0 || (occ && virt)), HSV_ERR_INVALID, "null argument");
  auto* p = new hsv_pool_s();
  p->sec = s;
  p->n = n;
  p->h.resize(n);
  for (int64_t i = 0; i < n; ++i) {
    if ((occ[i] & virt[i]) || !occ[i] || !virt[i]) {
      delete p;
      set_error(HSV_ERR_INVALID, "excitation indices must be distinct");
      return HSV_ERR_INVALID;
    }
    OpMasks m = compress_op(s, occ[i], virt[i]);
    p->h[i] = make_int4((int)m.oa, (int)m.va, (int)m.ob, (int)m.vb);
  }
  int rc = dalloc(&p->d, n);
  if (rc) { delete p; return rc; }
  if (n) HSV_TRY_CUDA(cudaMemcpyAsync(p->d, p->h.data(), n * sizeof(int4), cudaMemcpyHostToDevice, stream()));
  if ((rc = pool_prepare(p))) { hsv_pool_destroy(p); return rc; }
  *out = p;
  return HSV_OK;
}

int hsv_pool_destroy(hsv_pool p) {
  if (!p) return HSV_OK;
  dfree(p->d);
  dfree(p->d_order);
  dfree(p->d_opl);
  dfree(p->d_qa);
  dfree(p->d_qn);
  dfree(p->d_blist);
  delete p;
  return HSV_OK;
}

}  // extern "C"
