/*
 * hsv.h -- C ABI of the B200-native exact sparse state-vector engine
 * (Hyperion-1 path of arxiv/paper_2604_01176, reference package `svmps`).
 *
 * Plain C types only (no torch, no C++ in signatures).  Every entry point
 * returns an int status (HSV_OK = 0); on failure hsv_last_error() holds a
 * message whose wording mirrors the reference exception it replaces, and the
 * Python host layer re-raises the same exception type (ValueError /
 * RuntimeError / MemoryError).
 *
 * Object model (all opaque, device resident, explicitly destroyed):
 *   hsv_sector  one (n_alpha, n_beta) particle-number sector of an n-qubit
 *               register: replaces svmps.cibasis.CiBasis / enumerate_basis
 *               (cibasis.py:98-181).  Reference positions (ascending key
 *               order) are exposed; internally amplitudes are stored
 *               alpha-string-major ("HBM layout").
 *   hsv_op      a real, number-conserving Pauli sum bound to a sector, stored
 *               matrix-free as x-grouped term tables: replaces the CSR built
 *               by svmps.svengine.assemble_subspace_hamiltonian
 *               (svengine.py:115-171) and its validation (odd-Y, sector leak).
 *   hsv_state   a complex128 amplitude vector over a sector; support is the
 *               set of exactly-nonzero amplitudes, which is how the reference
 *               SparseVector (sparse.py:20-70) drops exact zeros.
 *
 * Calls are synchronous on return unless named *_async; all device work is
 * enqueued on the library stream (hsv_set_stream).  Results are bitwise
 * deterministic run to run (no floating-point atomics).
 */
#ifndef HSV_H_
#define HSV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HSV_ABI_VERSION 1

#if defined(__GNUC__)
#define HSV_API __attribute__((visibility("default")))
#else
#define HSV_API
#endif

enum hsv_status {
  HSV_OK = 0,
  HSV_ERR_INVALID = 1,      /* bad argument / dimension mismatch  -> ValueError   */
  HSV_ERR_SECTOR = 2,       /* configuration outside the sector   -> ValueError   */
  HSV_ERR_NONREAL = 3,      /* odd-Y Pauli word                   -> ValueError   */
  HSV_ERR_LEAK = 4,         /* Hamiltonian not spin-conserving    -> ValueError   */
  HSV_ERR_NORM_DRIFT = 5,   /* QEB rotation norm drift            -> RuntimeError */
  HSV_ERR_CUDA = 6,         /* CUDA runtime failure               -> RuntimeError */
  HSV_ERR_OOM = 7,          /* device allocation failed           -> MemoryError  */
  HSV_ERR_UNSUPPORTED = 8   /* sector too large for dense layout  -> ValueError   */
};

enum hsv_ordering { HSV_INTERLEAVED = 0, HSV_BLOCKED = 1 };

typedef struct hsv_sector_s* hsv_sector;
typedef struct hsv_op_s* hsv_op;
typedef struct hsv_state_s* hsv_state;
typedef struct hsv_pool_s* hsv_pool;
typedef struct hsv_peer_s* hsv_peer;

/* ---- library / device ------------------------------------------------- */
HSV_API int hsv_abi_version(void);
/* Copies the last error message of the calling thread into buf. */
HSV_API int hsv_last_error(char* buf, size_t n);
/* Select the CUDA device for subsequent objects: one device per process; a
 * second call with another device fails (HSV_ERR_INVALID). */
HSV_API int hsv_init(int device);
/* Enqueue all work on this cudaStream_t (0 = library-owned stream). */
HSV_API int hsv_set_stream(void* cuda_stream);
HSV_API void* hsv_get_stream(void);
/* Number of CUDA kernels this library launched since the last reset. */
HSV_API int64_t hsv_launch_count(int reset);
/* Device work counters of the ADAPT evaluation kernels (8 slots): [0] rotation
 * pairs processed by forward sweeps, [1] by adjoint sweeps, [2] rows computed by
 * the support-restricted H application (K1r); host-read, not reset: [4] idle
 * bytes of the library's device arena, [5] arena chunks taken from the driver
 * so far, [6] / [7] the CUDA default pool's reserved / used bytes.
 * Synchronizes when out != NULL; reset != 0 zeroes the device counters. */
HSV_API int hsv_stats(int64_t* out, int reset);
HSV_API int hsv_synchronize(void);
/* Return the wholly idle chunks of the library's device arena (and the CUDA
 * default pool's idle memory) to the driver; synchronizes.  Freed scratch is
 * otherwise kept for reuse. */
HSV_API int hsv_mem_trim(void);

/* ---- sector: replaces CiBasis / enumerate_basis (cibasis.py:98-181) ---- */
HSV_API int hsv_sector_create(int n_qubits, int n_alpha, int n_beta, int ordering,
                      hsv_sector* out);
HSV_API int hsv_sector_destroy(hsv_sector s);
HSV_API int64_t hsv_sector_dim(hsv_sector s);
/* Alpha-string count and beta-string count (dim = n_alpha_strings * n_beta_strings). */
HSV_API int hsv_sector_shape(hsv_sector s, int64_t* n_alpha_strings, int64_t* n_beta_strings);
/* Reference positions of keys (CiBasis.try_positions, cibasis.py:133-138):
 * pos[i] = -1 when keys[i] is outside the sector. */
HSV_API int hsv_sector_positions(hsv_sector s, const uint64_t* keys, int64_t n, int64_t* pos);
/* Keys (occupation integers) of reference positions (CiBasis.states[pos]). */
HSV_API int hsv_sector_keys(hsv_sector s, const int64_t* pos, int64_t n, uint64_t* keys);

/* ---- operator: replaces assemble_subspace_hamiltonian (svengine.py:115-171) */
/* xs/zs: symplectic masks, coeffs: real weights (PauliSum arrays, pauli.py:87-107).
 * Raises NONREAL for an odd-Y word, LEAK for a group whose net amplitude
 * escapes the sector by more than 1e-10 (first offending x in ascending order). */
HSV_API int hsv_op_create(hsv_sector s, int n_qubits, const int64_t* xs, const int64_t* zs,
                  const double* coeffs, int64_t n_terms, hsv_op* out);
HSV_API int hsv_op_destroy(hsv_op op);
/* n_terms, n_groups (distinct x incl. diagonal), number of in-sector nonzero
 * matrix elements is not stored (matrix-free). */
/* Note on the *_async entry points: the first dense H application of an
 * alpha-row range assembles that range's rows (K1a, below), which synchronizes
 * once; every later call is asynchronous. */
/* K1a: stored slots (elements incl. sliced-ELL padding; 12 B each) and split
 * count of the assembled rows for alpha rows [a_lo, a_hi), 0 if not assembled
 * (K1a is built on the first H application of a range whose rows fit
 * sell_budget_mb; the matrix-free K1 runs otherwise). */
HSV_API int hsv_op_sell_info(hsv_op op, int64_t a_lo, int64_t a_hi, int64_t* slots,
                             int64_t* splits);
HSV_API int hsv_op_info(hsv_op op, int64_t* n_terms, int64_t* n_groups, int64_t* n_active_groups);
/* Number of structurally nonzero matrix elements (== reference CSR nnz). */
HSV_API int hsv_op_count_nnz(hsv_op op, int64_t* nnz);
/* Materialize the CSR (reference positions, ascending columns per row) for
 * small sectors: row_offsets[dim+1], cols[nnz], vals[nnz] (host buffers). */
HSV_API int hsv_op_to_csr(hsv_op op, int64_t* row_offsets, int64_t* cols, double* vals, int64_t nnz_cap);

/* ---- states (SparseVector / SvState, sparse.py:20-70, svengine.py:89-109) */
HSV_API int hsv_state_create(hsv_sector s, hsv_state* out);              /* all zero */
HSV_API int hsv_state_destroy(hsv_state st);
HSV_API int hsv_state_copy(hsv_state dst, hsv_state src);
HSV_API int hsv_state_zero(hsv_state st);
/* Basis state |key> (SvState.from_configuration, svengine.py:96-101). */
HSV_API int hsv_state_set_basis(hsv_state st, uint64_t key, double re, double im);
/* Replace contents from (ascending) reference positions; amps interleaved
 * (re, im) pairs, amps_im may be NULL for real input. */
HSV_API int hsv_state_set_sparse(hsv_state st, const int64_t* pos, const double* amps_re,
                         const double* amps_im, int64_t n);
/* Replace contents from all dim amplitudes in reference position order (a
 * SparseVector whose support is the whole sector: the binding sends the values
 * only, half the host-to-device bytes of hsv_state_set_sparse for real input). */
HSV_API int hsv_state_set_dense(hsv_state st, const double* amps_re, const double* amps_im);
HSV_API int hsv_state_set_keys(hsv_state st, const uint64_t* keys, const double* amps_re,
                       const double* amps_im, int64_t n);
HSV_API int hsv_state_nnz(hsv_state st, int64_t* nnz);
/* Support in ascending reference position order (drops exact zeros, or
 * |v| < prune when prune > 0). cap = capacity of the output buffers. */
HSV_API int hsv_state_get_sparse(hsv_state st, double prune, int64_t* pos, double* amps_re,
                         double* amps_im, int64_t cap, int64_t* n_out);
/* Amplitudes at given reference positions (zero where not in the support);
 * a cheap peek for sampled validation of very large states. */
HSV_API int hsv_state_get_positions(hsv_state st, const int64_t* pos, int64_t n, double* amps_re,
                                    double* amps_im);
/* <a|b> (dot, sparse.py:210-219). */
HSV_API int hsv_state_dot(hsv_state a, hsv_state b, double* re, double* im);
HSV_API int hsv_state_norm(hsv_state st, double* norm);
/* y <- a*x + y, then exact zeros drop (axpy, sparse.py:222-228). */
HSV_API int hsv_state_axpy(double a_re, double a_im, hsv_state x, hsv_state y);
HSV_API int hsv_state_scale(hsv_state st, double a_re, double a_im);

/* ---- hot path --------------------------------------------------------- */
/* out <- H|in> over all rows (spmspv, sparse.py:177-201); |y| < prune -> 0.
 * out must not alias in. */
HSV_API int hsv_apply_h(hsv_op op, hsv_state in, hsv_state out, double prune);
/* <psi|H|psi> (expectation, svengine.py:174-176). */
HSV_API int hsv_expect_h(hsv_op op, hsv_state psi, double* e_re, double* e_im);
/* exp(theta T)|in> for the QEB generator with occ/virt qubit masks, given
 * c = cos(theta), s = sin(theta) computed by the caller (svengine.py:209-237).
 * out may alias in. Raises NORM_DRIFT like svengine.py:234-236. */
HSV_API int hsv_apply_qeb(hsv_state in, hsv_state out, uint64_t occ_mask, uint64_t virt_mask,
                  double c, double s);
/* T|in> (apply_generator, svengine.py:187-206). out must not alias in. */
HSV_API int hsv_apply_generator(hsv_state in, hsv_state out, uint64_t occ_mask, uint64_t virt_mask);
/* Pool gradients g_k = 2 Re <H psi | T_k psi> for M operators plus the
 * energy <psi|H|psi> (SvAdaptEngine.energy + .screen, adapt.py:205-214). */
HSV_API int hsv_energy_screen(hsv_op op, hsv_state psi, const uint64_t* occ_masks,
                      const uint64_t* virt_masks, int64_t n_ops, double* energy,
                      double* grads);
/* psi <- exp(t_{k-1}T_{k-1})...exp(t_0 T_0)|hf> (apply_ansatz, svengine.py:240-244)
 * in one fused sweep; rotations with (c, s) == (1, 0) are skipped as theta == 0 is.
 * Synchronizes (norm-drift check, like hsv_apply_qeb). */
HSV_API int hsv_ansatz_state(hsv_sector sector, uint64_t hf_key, const uint64_t* occ_masks,
                             const uint64_t* virt_masks, const double* c, const double* s,
                             int64_t k, hsv_state psi_out);
/* Adjoint energy + analytic gradient of exp(t_{k-1}T_{k-1})...exp(t_0 T_0)|hf>
 * (ansatz_energy_gradient, svengine.py:260-281); cs[i], sn[i] = cos/sin(theta_i). */
HSV_API int hsv_energy_gradient(hsv_op op, uint64_t hf_key, const uint64_t* occ_masks,
                        const uint64_t* virt_masks, const double* cs, const double* sn,
                        int64_t k, double* energy, double* grads);
/* The same sweep in two phases for multi-GPU (owner computes H psi rows):
 * forward: psi <- exp(...)|hf> on all rows (replicated), w rows [a_lo, a_hi)
 * <- (H psi) rows (stream-ordered: a norm drift of the forward sweep is reported by
 * the hsv_eg_backward that consumes psi); the caller makes
 * w complete on every rank (all-gather of the row blocks);
 * backward: E = Re<psi|w> and the adjoint sweep; psi and w are consumed. */
HSV_API int hsv_eg_forward_async(hsv_op op, uint64_t hf_key, const uint64_t* occ_masks,
                                 const uint64_t* virt_masks, const double* cs, const double* sn,
                                 int64_t k, int64_t a_lo, int64_t a_hi, hsv_state psi_out,
                                 hsv_state w_out);
HSV_API int hsv_eg_backward(hsv_op op, hsv_state psi, hsv_state w, const uint64_t* occ_masks,
                            const uint64_t* virt_masks, const double* cs, const double* sn,
                            int64_t k, double* energy, double* grads);
/* Owner-computes shard variants for multi-GPU (rows = alpha-strings
 * [a_lo, a_hi)).  Write, without synchronizing, to DEVICE memory:
 *   d_out[0..1] = partial <psi|H|psi> (re, im), d_out[2..2+n_ops) = partial
 *   gradients (already multiplied by 2).  psi must be replicated. */
HSV_API int hsv_energy_screen_partial_async(hsv_op op, hsv_state psi, const uint64_t* occ_masks,
                                    const uint64_t* virt_masks, int64_t n_ops,
                                    int64_t a_lo, int64_t a_hi, double* d_out);
/* Device pointer to the amplitude array (alpha-major, complex128) and its
 * element count, for collectives issued by the host (e.g. NCCL all-gather). */
HSV_API int hsv_state_device_ptr(hsv_state st, void** ptr, int64_t* n);
/* out rows [a_lo, a_hi) <- (H in) rows; other rows untouched. */
HSV_API int hsv_apply_h_rows_async(hsv_op op, hsv_state in, hsv_state out, int64_t a_lo,
                           int64_t a_hi, double prune);

/* ---- operator pools (build_qeb_pool, adapt.py:78-108, resident on the device) ---- */
HSV_API int hsv_pool_create(hsv_sector s, const uint64_t* occ_masks, const uint64_t* virt_masks,
                            int64_t n_ops, hsv_pool* out);
HSV_API int hsv_pool_destroy(hsv_pool p);
/* energy + all pool gradients of rows [a_lo, a_hi) into DEVICE d_out
 * (layout as hsv_energy_screen_partial_async); no host synchronization. */
HSV_API int hsv_energy_screen_pool_async(hsv_op op, hsv_state psi, hsv_pool pool, int64_t a_lo,
                                         int64_t a_hi, double* d_out);
/* synchronous full-range variant with host outputs */
HSV_API int hsv_energy_screen_pool(hsv_op op, hsv_state psi, hsv_pool pool, double* energy,
                                   double* grads);
/* d_out[j] = sum over i in ascending order of d_in[i * n_cols + j] (DEVICE
 * pointers, one launch, no host synchronization): combines the per-rank
 * partials all-gathered by NCCL in rank order, as the reference concatenates
 * row blocks in worker order (sparse.py:199-201). */
HSV_API int hsv_sum_rows_async(const double* d_in, int64_t n_rows, int64_t n_cols, double* d_out);

/* ---- NVLink peer exchange (one process per GPU, replaces NCCL on the path) ----
 * A peer buffer is `bytes` of device memory that every rank maps (CUDA IPC),
 * plus per-rank arrival flags.  Collective use:
 *   hsv_peer_create   -> writes this rank's 64-byte IPC handle to handle_out;
 *   (host all-gathers the handles, e.g. torch.distributed.all_gather_object)
 *   hsv_peer_open     -> maps the other ranks' buffers (handles: world x 64 B);
 *   hsv_peer_allgather_async(p, d_src, n): copy n bytes from d_src to offset
 *     rank * n of every rank's buffer over NVLink, publish an arrival flag
 *     (system-scope release) and wait on the device until every rank's block
 *     has arrived; afterwards hsv_peer_data() holds all blocks in rank order.
 *     Stream-ordered, no host synchronization, no NCCL.
 * The same buffers carry whole H|psi> rows: hsv_eg_forward_peer_async writes
 * the rank's rows of w into every rank's buffer from the K1 epilogue
 * (compute + all-gather fused), then publishes/waits like the all-gather. */
HSV_API int hsv_peer_create(int world, int rank, int64_t bytes, hsv_peer* out, void* handle_out);
HSV_API int hsv_peer_open(hsv_peer p, const void* handles);
HSV_API int hsv_peer_destroy(hsv_peer p);
/* Synchronize and report the exchanges since the last check: HSV_ERR_CUDA if a
 * device-side wait timed out (HSV_PEER_TIMEOUT_S, default 60 s) or a peer rank
 * aborted its side of an exchange because its own call failed.  The waits are
 * bounded, so a dead or failed peer surfaces here instead of hanging the stream. */
HSV_API int hsv_peer_check(hsv_peer p);
HSV_API int hsv_peer_data(hsv_peer p, void** d_data, int64_t* bytes);
HSV_API int hsv_peer_allgather_async(hsv_peer p, const void* d_src, int64_t n);
/* All-gather + rank-order sum in ONE launch: the n float64 values at d_src go
 * to every rank's buffer, then (after the arrival barrier) d_out[j] =
 * ((0 + x_0[j]) + x_1[j]) + ... in rank order -- the same bits on every rank
 * and the same sum as hsv_sum_rows_async over hsv_peer_data().  n * 8 must be a
 * multiple of 16.  Replaces the NCCL all-reduce of the (E, gradients) partials
 * (bench.py; reference engine: the scalar combine of SURVEY.md 8(e)). */
HSV_API int hsv_peer_allreduce_async(hsv_peer p, const double* d_src, int64_t n, double* d_out);
/* Phase 1 of the adjoint sweep (as hsv_eg_forward_async) with the rows
 * [a_lo, a_hi) of w = H psi written by the K1 epilogue straight into every
 * rank's peer buffer (bytes >= dim * 16, rows at their natural offsets), then
 * the arrival barrier and a copy of the complete local buffer into `w`. */
HSV_API int hsv_eg_forward_peer_async(hsv_op op, uint64_t hf_key, const uint64_t* occ_masks,
                                      const uint64_t* virt_masks, const double* c,
                                      const double* s, int64_t k, int64_t a_lo, int64_t a_hi,
                                      hsv_state psi, hsv_state w, hsv_peer p);

/* ---- tuning knobs (defaults are the measured best): "apply_r" (rows per
 * lane 0 auto/1/2/4/8), "apply_minb", "apply_split" (0 auto/1/2/4/8/16/32),
 * "apply_interleave" (-1 auto = 2 dynamic, 0 contiguous, 1 interleaved),
 * "screen_rows", "push" (-1 auto, 0 pull only, 1 push whenever it fits),
 * "push_keys" (push budget factor), "sweep" (1 fused cooperative sweeps, 0 one
 * launch per rotation), "sweep_grid" (0 auto), "staged" (1: TMA-staged K1s),
 * "bperm" (K1 partner beta ranks from per-xb 16-bit rows: -1/1 on, 0 Rb0 gather),
 * "rb0_smem" (1: Rb0 staged in shared memory, opt-in) ---- */
HSV_API int hsv_set_tuning(const char* key, int64_t value);

/* ---- device Hamiltonian build (mapping.py:79-126, pauli.py:165-198) ---- */
/* Jordan-Wigner image of the spin-orbital tables h[n*n], g[n^4] (chemists'
 * order, mapping.py:48-76) plus core_energy: the merged real Pauli sum with
 * |c| > drop_tol, sorted by (x, z) -- the PauliSum hsv_op_create takes.  The
 * products are expanded and summed on the device in the reference's order, so
 * the coefficients are bit-identical to its dict accumulation.  n <= 32.
 * Call with xs == NULL to get *n_out, then with capacity cap >= *n_out.
 * HSV_ERR_NONREAL: residual imaginary coefficient > 1e-12 (not Hermitian). */
HSV_API int hsv_jordan_wigner(int n_qubits, const double* h, const double* g, double core_energy,
                              double drop_tol, int64_t* xs, int64_t* zs, double* coeffs,
                              int64_t cap, int64_t* n_out);

/* ---- Krylov basis blocks (FCI reference: thick-restart Lanczos, fci.py;
 * replaces scipy eigsh in oracle.py:99-142) ---- */
/* c_j = <q_j|w> (complex, c_out[2j], c_out[2j+1]; c_out may be NULL) for the m
 * basis states in one launch; subtract != 0: then w -= sum_j c_j q_j (one pass).
 * Fixed-order reductions (repeatable bit for bit).  Synchronizes. */
HSV_API int hsv_krylov_project(const hsv_state* q, int64_t m, hsv_state w, int subtract,
                               double* c_out);
/* out = sum_j coeff[j] q_j (real coefficients; a Ritz vector).  Synchronizes. */
HSV_API int hsv_krylov_combine(const hsv_state* q, int64_t m, const double* coeff,
                               hsv_state out);

/* ---- live kernel timing (CUDA events on the launch stream) ---- */
HSV_API int hsv_prof_enable(int on);
/* synchronize, then fold recorded event pairs into per-kernel totals */
HSV_API int hsv_prof_collect(void);
/* kernels: "apply", "screen", "qeb", "adjoint", "generator" */
HSV_API int hsv_prof_get(const char* kernel, double* total_ms, int64_t* count);
HSV_API int hsv_prof_reset(void);

/* ---- generic CSR x sparse vector (K1b; spmspv on arbitrary CsrMatrix) ---- */
/* y = M x with M in CSR (int64 offsets/cols, f64 values), x dense-scattered
 * from (x_idx, x_val, x_nnz); output is the compacted support (y != 0, or
 * |y| >= prune) in ascending row order.  Host buffers; y buffers sized n_rows. */
HSV_API int hsv_csr_spmspv(int64_t n_rows, int64_t n_cols, const int64_t* row_offsets,
                   const int64_t* cols, const double* vals, int64_t nnz,
                   const int64_t* x_idx, const double* x_val, int64_t x_nnz, double prune,
                   int64_t* y_idx, double* y_val, int64_t* y_nnz);

/* ---- generic sparse vectors (host arrays; SparseVector, sparse.py:20-245) ---- */
/* sum over shared indices of u_val*v_val; u_idx ascending (dot, sparse.py:210-219). */
HSV_API int hsv_vec_dot(const int64_t* u_idx, const double* u_val, int64_t nu, const int64_t* v_idx,
                const double* v_val, int64_t nv, double* out);
/* a*x + y merged in ascending index order, exact zeros (or |v| < prune) dropped
 * (axpy, sparse.py:222-228); out buffers sized nx + ny. */
HSV_API int hsv_vec_axpy(int64_t dim, double a, const int64_t* x_idx, const double* x_val, int64_t nx,
                 const int64_t* y_idx, const double* y_val, int64_t ny, double prune,
                 int64_t* out_idx, double* out_val, int64_t* n_out);
/* y = a*x (divide=0, scale sparse.py:231-234) or y = x/a (divide=1, normalize :242-245). */
HSV_API int hsv_vec_scale(const double* x, int64_t n, double a, int divide, double* y);

#ifdef __cplusplus
}
#endif
#endif /* HSV_H_ */
