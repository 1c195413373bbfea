// Kernel argument blocks and cross-file launch helpers.
#pragma once
#include "hsv_common.cuh"

namespace hsv {

// Runtime tuning knobs (hsv_set_tuning); defaults are the measured best.
struct Tuning {
  int apply_r = 0;        // rows per lane in the K1 apply kernel (1, 2, 4, 8; 0 = auto)
  int apply_minb = 0;     // __launch_bounds__ min blocks/SM: 0 = default (R=2: 4, R=4: 3,
                          // R=8: 2); alternatives R=2: 3, 5 or 6, R=4: 2
  int screen_rows = 1024; // rows staged per chunk in the screen kernel
  int screen_pivot = -1;  // K4 rows: -1 auto (psi rows when psi is sparse), 0 w rows, 1 psi rows
  int apply_split = 0;    // bucket splits per row unit in K1 (0 = auto, else 1/2/4/8/16/32)
  int apply_interleave = -1;  // K1 unit schedule: -1 auto (= 2), 0 contiguous, 1 interleaved, 2 dynamic
  int push = -1;          // sparse-psi push path: -1 auto, 0 off, 1 whenever it fits in memory
  int push_keys = 32;     // auto: push while nnz(psi) * (1 + groups) <= push_keys * rows - 2^20
  int sweep = 2;          // adjoint/forward sweeps: 2 batched (orbits of kBatch rotations per
                          // grid barrier, hsv_sweep.cu), 1 one barrier per rotation, 0 launch per op
  int sell = -1;          // K1a (assembled sliced-ELL rows, built once per operator and
                          // row range when it fits sell_budget_mb): -1/1 on, 0 off
  int64_t sell_budget_mb = 32768;
  int screen_overlap = 2; // energy + screen with K1a: K4 on alpha-row phases, on a second
                          // stream, as the K1a stream finishes their rows (0/1: serial).
                          // H12 step 2.509 (serial) / 2.435 (2) / 2.494 (4) / 2.561 ms (8):
                          // K1a and K4 contend for L1 and issue, little overlaps
  int sup = -1;           // K1s (support-compacted assembled rows in the ADAPT evaluation):
                          // 1 always, 0 off, -1 auto: once a support map has served more than
                          // 10 evaluations (a plateau of the support, not a growing one).  A
                          // rebuild per iteration costs more than its evaluations save (H12
                          // depth 400: 26.3 vs 23.2 ms per iteration; depth 200 15.6 vs 15.8;
                          // tools/sup_probe.py); a map that outlives its iteration pays
  int sell_sp = -1;       // K1a work units: 1 (chunk, split) segments + in-order combine,
                          // 0 one chunk per warp (all splits in registers), -1 auto (split
                          // segments below ~2 chunks per resident warp)
  int sell_kernel = 3;    // K1a variant (elements per stage, blocks per SM): 0 (4,4) 1 (4,6)
                          // 2 (8,3) 3 (8,4) 4 (2,8); H12: 1.74 1.70 1.72 1.58 1.85 ms
  int sweep_bar = 0;      // batched sweep barrier: 0 grid.sync(), 1 counting (release/acquire;
                          // measured equal at H12 depth 100/400, profiles/r02/sweep_probe_bar.jsonl)
  int sweep_threads = 256;   // batched sweep block size (128 or 256)
  int sweep_grid = 0;     // sweep blocks: 0 = min(co-resident, work items)
  int sweep_incr = 1;     // sweep plans: 1 refilter only the batches an operator list change
                          // touched (ADAPT appends), 0 refilter every batch
  int sweep_p2p = 0;      // batched sweeps without grid barriers (per-row versions, k_psweep):
                          // 1 on, 0 off.  Exact, but measured 2.9x slower at H12 depth 400
                          // (2.60 vs 0.88 ms forward): consecutive batches share rows densely
                          // (a batch touches ~25% of the support), so the version waits
                          // chain batch after batch and the spinning adds latency
  int bperm = -1;         // K1 (R=8) pass-1 ranks from per-xb 16-bit permutation rows (built
                          // for 32-bit words, Nb <= 65536, <= 256 MB): -1/1 on, 0 off
  int rb0_smem = 0;       // K1 (R=8) pass-1 Rb0 table in shared memory: 1 on (norb <= 15),
                          // 0/-1 off (default: measured 1-3% slower at H12/H14)
  int restrict_rows = -1; // K1r in the adjoint evaluation (w = H psi on the structural
                          // support of psi only): -1/1 on, 0 off (full K1 / push)
  int apply_t = 0;        // K1t (alpha tiles: 8 alpha rows x 1 beta string per lane,
                          // hsv_apply_t.cu): 1 on, 0/-1 off.  Bitwise equal to K1 but
                          // measured 2.2x slower at H12 (5.21 vs 2.39 ms): 1.88e9 vs 1.25e9
                          // warp instructions (per-row predication of the alpha mask) and
                          // L1 hit 66 vs 78% (a lane gathers from 8 partner alpha rows)
  int apply_v = 0;        // K1v (per-group valid beta lists, shared-memory row accumulators):
                          // 1 on where built, 0/-1 off.  Bitwise equal to K1 but measured
                          // 2.4x slower at H12 (5.80 vs 2.40 ms): the per-group chain (record
                          // -> list offsets -> entries -> gathers -> shared-memory update,
                          // __syncwarp) serializes groups that K1 pipelines in registers
  int staged = 0;         // K1s (TMA-staged partner rows) where the sector fits: 1 on, 0 off.
                          // Off by default: it cuts K1's global load sectors 8.4x at H12
                          // but not its time (K1 is issue-bound; 3.04 vs 3.07 ms)
};
Tuning& tuning();

struct ApplyArgs {
  const uint32_t* Sa;
  const uint32_t* Sb;
  const uint32_t* Ra;
  const uint32_t* Rb;
  const uint32_t* Rb0;     // Rb with out-of-sector strings mapped to rank 0 (K1 pass 1)
  const int4* buckets;
  int n_buckets;
  int n_buckets_h;     // buckets [0, n_buckets_h) hold x-local (hashed) groups
  const void* recs;    // Rec<W> per hashed group (same index as groups)
  const int4* groups;
  const Term* terms;
  const double* diag;
  const GroupHash* ghash;
  const double* tabs;
  const uint64_t* gsz;     // per group: 1<<63 | z0 for single-Z groups, else 0
  const void* szt;         // SzTerm per term (single-Z groups)
  const uint32_t* gxa;     // per group: alpha flip part (its bucket's x)
  int g_hashed;            // groups [0, g_hashed) are x-local (hashed)
  const double2* psi;
  const uint32_t* arow;  // alpha-row occupancy of psi (skip empty partner rows) or nullptr
  double2* out;      // nullptr: energy only
  double* epart;     // [warps][2] energy partials or nullptr
  int64_t Nb;
  const uint16_t* bperm;   // per-xb beta rank permutations (Rec.pad0 = slot offset) or nullptr
  int rb0_n;               // Rb0 words staged in shared memory by K1 (0: read from global)
  int64_t a_lo, a_hi;
  int64_t units;
  int upr;
  int nsplit;              // bucket splits per row unit (1: none), 2..32 (use_split_table)
  int interleave;          // unit schedule: 0 contiguous, 1 interleaved, 2 dynamic (counter)
  int64_t dim_bytes;       // size of psi in bytes (schedule choice)
  const int* split_bk;     // nsplit + 1 bucket boundaries (in this launch's buckets)
  double2* ypart;          // [nsplit][rows of a_lo..a_hi] partial rows when nsplit > 1
  int64_t part_stride;
  double prune;
  int energy_only;
  unsigned int* ucounter;     // dynamic schedule: next work unit
  double* upart;              // dynamic schedule: [units][2] energy partials
  double2* const* peer_rows;  // device array: other ranks' w buffers (NVLink), or nullptr
  int n_peer_rows;
  // K1r (row-list mode): rows of alpha row ra are rlist[(ra - a_lo) * Nb + i],
  // i < rcnt[ra - a_lo]; work unit u covers list chunk utab[u].y of alpha row
  // a_lo + utab[u].x; *d_units list units (device count, no host sync)
  const uint32_t* rlist;
  const uint32_t* rcnt;
  const uint2* utab;
  const uint32_t* d_units;
  // K1v (valid lists, hsv_apply_v.cu)
  const uint2* vl;
  const int* vloff;
  int vl_chunk, vl_nchunks;
  const uint8_t* smap;     // K1v row-restricted mode: rows outside the map are skipped
  const uint32_t* vgslot;  // K1v: per group, its list's offset slot
  // K1 enumeration modes (SELL build, hsv_apply.cu): per (row, split) entry
  // counts, or the entries themselves at their sliced-ELL slots
  uint32_t* sell_cnt;        // [row - a_lo*Nb][split]
  const uint64_t* sell_off;  // [chunk][split] first slot (lane 0) of the segment
  uint32_t* sell_cols;
  double* sell_amps;
};

// K1r: row lists of the rows marked in smap (or, smap == nullptr, of the
// nonzero rows of amp) for alpha rows [a_lo, a_hi), and the unit table.
struct RowList {
  uint32_t* rlist = nullptr;
  uint32_t* rcnt = nullptr;
  uint2* utab = nullptr;
  uint32_t* d_units = nullptr;
  int64_t max_units = 0;
  int build(const hsv_sector_s* s, const uint8_t* smap, const double2* amp, int64_t a_lo,
            int64_t a_hi, int rows_per_unit);
  void release();
};

// Final value of output row `row`: local store plus the same store into every
// peer buffer (compute and all-gather fused: rows cross NVLink as they finish).
__device__ __forceinline__ void put_row(double2* out, double2* const* peers, int n_peers,
                                        int64_t row, double2 y) {
  out[row] = y;
  for (int p = 0; p < n_peers; ++p) peers[p][row] = y;
}

// Packed per-group record of an x-local group, loaded with one or two 16-byte
// uniform loads: meta = hb | shift << 8.
template <typename W> struct Rec;
template <> struct __align__(16) Rec<uint32_t> {
  uint32_t xb, meta, xm, z0, mul, tab, pad0, pad1;
};
template <> struct __align__(16) Rec<uint64_t> {
  uint32_t xb, meta, tab, pad0;
  uint64_t xm, z0, mul, pad1;
};
template <typename W>
__device__ __forceinline__ Rec<W> ldrec(const Rec<W>* p) {
  Rec<W> r;
  const uint4* q = reinterpret_cast<const uint4*>(p);
  uint4* d = reinterpret_cast<uint4*>(&r);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(Rec<W>) / 16); ++i) d[i] = __ldg(q + i);
  return r;
}

// Term of a single-Z group: z_t = z_0 ^ (0 or the whole flip mask) ^ (0 or one
// bit r).  For in-sector rows parity(s & flip) is fixed, so
//   (-1)^popc(s & z_t) c_t = (-1)^popc(s & z_0) * (-1)^{s_r} c'_t,
// c'_t = c_t with that fixed sign folded in; the sign bit of term t is
// (s << sh) & fm for 32-bit rows (sh = 31 - r), ((s >> sh) << 31) & fm for
// 64-bit rows (sh = r); fm = 0 when z_t has no extra Z.
struct __align__(16) SzTerm {
  double c;
  uint32_t sh, fm;
};

// Matrix element of an x-local group at row s: (-1)^popc(s & z0) * A[h(s & x)].
template <typename W>
__device__ __forceinline__ double rec_amp(const Rec<W>& r, W s, const double* __restrict__ tabs) {
  const int shift = (int)((r.meta >> 8) & 0xffu);
  const uint32_t h = r.tab + (uint32_t)((W)((s & r.xm) * r.mul) >> shift);
  const double A = __ldg(tabs + h);
  const int sgn = popc(s & r.z0) << 31;
  return __hiloint2double(__double2hiint(A) ^ sgn, __double2loint(A));
}

int grid_for(int64_t n, int block);
int state_dot_async(hsv_state a, hsv_state b, double* d_r);   // <a|b> -> d_r[0..1]
int state_dot_norm2_async(hsv_state a, hsv_state b, double* d_r);   // and <b|b> -> b's norm
void use_split_table(const hsv_op_s* op, int St, ApplyArgs& a);
int apply_warps(const hsv_op_s* op);
// Push (scatter + sort-reduce) K1 for sparse psi; *done = false: use the pull kernel.
// dense_hint (optional, per state): skip when set, set when psi is found dense.
int launch_push(const hsv_op_s* op, const ApplyArgs& a, bool* done, int64_t* n_warps,
                bool* dense_hint);
// K1t (hsv_apply_t.cu): *done = false when not selected (tuning apply_t) or wide words.
int launch_apply_t(const hsv_op_s* op, const ApplyArgs& a, int S, bool* done);
// K1v (hsv_apply_v.cu): *done = false when the operator has no valid lists.
// S = the bucket split count the register-row K1 would use (same row values).
int launch_apply_v(const hsv_op_s* op, const ApplyArgs& a, int S, bool* done);
// K1s (hsv_apply_staged.cu): *done = false when the sector does not fit on chip.
int launch_apply_staged(const hsv_op_s* op, const ApplyArgs& a, int64_t* n_warps, bool* done);
void launch_combine_splits(const double2* part, int S, int64_t rows, double2* out, int64_t off,
                           double prune, double2* const* peers, int n_peers);
void launch_combine_splits_map(const double2* part, int S, int64_t rows, double2* out,
                               int64_t off, const uint8_t* smap, double2* const* peers,
                               int n_peers);
int k1_default_split(const hsv_op_s* op, int64_t a_lo, int64_t a_hi, bool has_out);
int launch_apply(const hsv_op_s* op, const double2* psi, double2* out, double* epart,
                 int64_t a_lo, int64_t a_hi, double prune, int energy_only, int64_t* n_warps,
                 const uint32_t* arow = nullptr, bool* dense_hint = nullptr);
// K1r: out = H psi on the rows marked in smap (exactly the K1 values there),
// 0 on every other row of [a_lo, a_hi); no energy partials.
int launch_apply_rows(const hsv_op_s* op, const double2* psi, double2* out, int64_t a_lo,
                      int64_t a_hi, const uint32_t* arow, const uint8_t* smap,
                      int64_t support_rows = -1, uint64_t smap_version = 0);

// Compressed QEB masks of one excitation operator.
struct OpMasks {
  uint32_t oa, va, ob, vb;
};
OpMasks compress_op(const hsv_sector_s* s, uint64_t occ, uint64_t virt);
int64_t src_count(int norb, int n, uint32_t occ, uint32_t virt);

// Device scratch for pair lists (src rank, partner rank) of one operator.
struct PairLists {
  int2* la = nullptr;
  int2* lb = nullptr;
  int64_t ca = 0, cb = 0;
};
int build_pair_lists_async(const hsv_sector_s* s, const OpMasks& m, PairLists& pl);

// K3b/K5b batched sweeps (hsv_sweep.cu): mode 0 forward, 1 adjoint.
int launch_bsweep(const hsv_sector_s* sec, int mode, int64_t hf_row,
                  const std::vector<OpMasks>& ops, const double* cs, const double* sn,
                  double2* psi, double2* lam, uint8_t* smap_out, double* norm2, double* d_grads,
                  int* err, double* err_val, bool* used);
int smap_arow_async(const hsv_sector_s* sec, const uint8_t* smap, uint32_t* flags);
// rows of the cached plan's support map (-1: no plan for this sector)
int64_t sweep_plan_support(const hsv_sector_s* s);
// identity of the cached plan's support map contents (0: none)
uint64_t sweep_plan_version(const hsv_sector_s* s);
// drop the cached sweep plan (of sector s only, when s != nullptr)
void release_sweep_plans(const hsv_sector_s* s = nullptr);

// K1a by chunk ranges (the overlapped energy + screen, hsv_screen.cu): the
// range's assembled rows if built (*chunks = their 32-row chunk count, 0: not
// assembled -- the caller runs the serial path); rows of chunks [c0, c1) into
// out, their energy partials into cpart[2 c] (reduced by the caller in chunk order)
int sell_chunks(const hsv_op_s* op, int64_t a_lo, int64_t a_hi, int64_t* chunks);
int sell_apply_chunks(const hsv_op_s* op, const double2* psi, double2* out, int64_t a_lo,
                      int64_t a_hi, int64_t c0, int64_t c1, double* cpart);
int launch_screen(const hsv_op_s* op, const double2* psi, const double2* w,
                  const hsv_pool_s* pool, int64_t a_lo, int64_t a_hi, double* d_grads,
                  const uint32_t* psi_arow = nullptr, const uint32_t* w_arow = nullptr,
                  bool sparse_psi = false);
int pool_prepare(hsv_pool_s* p);

}  // namespace hsv
