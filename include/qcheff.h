/* qcheff.h — C-ABI of libqcheff, the B200 (sm_100a) implementation of the two
 * data-parallel hot paths of the effham reference (arXiv 2411.09982):
 * NPAD Givens-rotation block diagonalisation and Magnus time coarse-graining.
 *
 * Conventions (all entry points):
 *  - Pointers named d_* are DEVICE pointers (caller-owned; never freed here).
 *    Complex matrices are complex128, row-major, C-contiguous, interleaved
 *    (re, im) — exactly numpy's complex128 layout.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls that
 *    return host scalars synchronise that stream; the others are asynchronous.
 *  - Return value: QCH_OK or one of the QCH_ERR_* codes below, one per
 *    exception class of the reference (errors.py:4-64).  The message of the
 *    last failure on the calling thread is available from qch_last_error().
 *
 * The reference has no FFI: its boundary is the Python API in
 * /root/reference/pkg/src/effham.  Each function cites the reference function
 * it replaces.  INTEGRATION.md shows the ctypes binding.
 */
#ifndef QCHEFF_H_
#define QCHEFF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  QCH_OK = 0,
  QCH_ERR_VALUE = 1,            /* ValueError (argument validation)        */
  QCH_ERR_INDEX = 2,            /* errors.IndexOutOfRange                  */
  QCH_ERR_ZERO_COUPLING = 3,    /* errors.ZeroCoupling                     */
  QCH_ERR_OVERLAPPING = 4,      /* errors.OverlappingPairs                 */
  QCH_ERR_UNITARITY_DRIFT = 5,  /* errors.UnitarityDrift                   */
  QCH_ERR_NONFINITE = 6,        /* errors.NonFinite                        */
  QCH_ERR_GRID = 7,             /* errors.GridMismatch                     */
  QCH_ERR_DIMENSION = 8,        /* errors.DimensionMismatch                */
  QCH_ERR_NORM_DRIFT = 9,       /* errors.NormDrift                        */
  QCH_ERR_HERMITICITY = 10,     /* errors.HermiticityViolation             */
  QCH_ERR_UNSUPPORTED = 11,     /* size/shape this build does not handle   */
  QCH_ERR_CUDA = 12             /* CUDA runtime failure                    */
};

int qch_version(void);
/* Copies the last error message of this thread into buf (NUL-terminated);
 * returns the full message length. */
size_t qch_last_error(char* buf, size_t len);
/* Number of device kernels this library has launched in this process
 * (bench/evidence counter). */
int64_t qch_launch_count(void);

/* ---------------------------------------------------------------- NPAD --- */

/* HermitianOperator.max_abs (operators.py:92-99): max_ij |H_ij| with numpy's
 * |z| rounding, written to the device double *d_out. */
int qch_max_abs_c128(const void* d_h, int64_t n_elems, double* d_out, void* stream);
/* The same for a contiguous batch of items of n_elems each (one launch):
 * d_out[b] = max_abs of item b. */
int qch_max_abs_batch_c128(const void* d_h, int64_t batch, int64_t n_elems, double* d_out, void* stream);

/* *d_nonherm = 0 iff H[x,y] == conj(H[y,x]) for all x, y (exact compare), else 1.
 * Selects the mirrored-column fast path of the rotation kernels. */
int qch_hermitian_exact_c128(const void* d_h, int64_t n, int* d_nonherm, void* stream);
/* HermitianOperator validation (operators.py:104-116) on the device:
 * *d_defect = max |H - H^dag| with numpy's |z| (the caller compares it with
 * 1e-12 * max_abs, as the reference). */
int qch_hermitian_defect_c128(const void* d_h, int64_t n, double* d_defect, void* stream);

/* givens_rotation_matrix (npad.py:101-123) for n_pairs (i, j) index pairs of
 * one operator.  d_pairs: int64[2*n_pairs].  d_params: double[8*n_pairs] =
 * {cos_half, sin_half, phase, degenerate, s_re, s_im, 0, 0} where
 * s = -sin_half*exp(i*phase) (_block_params, npad.py:126-128).
 * d_status[k] = QCH_ERR_ZERO_COUPLING when H[j,i] == 0 (npad.py:112-113).
 * Index checks (npad.py:109-110) are the caller's (host) job. */
int qch_givens_params_c128(const void* d_h, int64_t n, const int64_t* d_pairs, int64_t n_pairs,
                           double* d_params, int* d_status, void* stream);

/* unitary_transformation / eliminate_couplings (npad.py:131-145, 235-241,
 * 274-297): conjugate H in place by n_pairs index-disjoint rotations, in the
 * reference's sequential order, in one launch.  d_params as produced by
 * qch_givens_params_c128.  herm_exact selects mirrored column writes (valid
 * when qch_hermitian_exact_c128 reported 0).  d_u (nullable): accumulated
 * unitary, rows i, j updated like _apply_left (npad.py:244-251).  d_h may be
 * NULL: only d_u is updated (sparse operators keep their CSR path). */
int qch_npad_apply_rotations_c128(void* d_h, int64_t n, const int64_t* d_pairs, const double* d_params,
                                  int64_t n_pairs, int herm_exact, void* d_u, void* stream);

/* npad_run (npad.py:320-354) on one device-resident dense operator, entire
 * greedy loop on the device.  threshold = tol * max_abs(input) (caller).
 * d_target (int32, nullable) / n_target: subspace mode (npad.py:300-317).
 * d_u (nullable): track the accumulated unitary; audited for drift every
 * 100 rotations (npad.py:254-259) -> QCH_ERR_UNITARITY_DRIFT.
 * d_pivots (nullable): int32[2*pivot_cap] log of the (i, j) picks.
 * Outputs: *applied, *converged (host). */
int qch_npad_run_dense_c128(void* d_h, int64_t n, const int32_t* d_target, int64_t n_target,
                            double threshold, int64_t max_iter, void* d_u, int32_t* d_pivots,
                            int64_t pivot_cap, int64_t* applied, int* converged, void* stream);

/* Batched npad_run (new API: a parameter sweep of independent operators).
 * d_h: (batch, n, n) contiguous.  d_thresholds: double[batch].
 * Outputs on device: d_applied int64[batch], d_converged int32[batch].
 * Asynchronous.  All operators must be exactly Hermitian (builders are). */
int qch_npad_run_batch_c128(void* d_h, int64_t batch, int64_t n, const int32_t* d_target,
                            int64_t n_target, const double* d_thresholds, int64_t max_iter,
                            int64_t* d_applied, int32_t* d_converged, void* stream);

/* _conjugate_sparse (npad.py:148-232) on a device CSR (indptr int64 (n+1),
 * sorted int32 column indices, complex128 values, no explicit zeros): the
 * NEW CSR of U H U^dag for the rotation (i < j; c = cos_half and
 * s = -sin_half e^{i phase} as _block_params, npad.py:126-128), fill-in
 * below 1e-15 * max_abs dropped.  Output capacity out_cap entries (the new
 * nnz is at most nnz + 4 (len(row i) + len(row j)) + 8); *nnz_out (host)
 * receives the new nnz.  Synchronous.  Bit-identical to the reference. */
int qch_npad_sparse_rotate_c128(const int64_t* d_indptr, const int32_t* d_indices, const void* d_data, int64_t n,
                                int64_t nnz, int64_t i, int64_t j, double cos_half, double s_re, double s_im,
                                double max_abs, int64_t* d_out_indptr, int32_t* d_out_indices, void* d_out_data,
                                int64_t out_cap, int64_t* nnz_out, void* stream);
/* _largest_relevant (npad.py:300-317) on a device CSR: host out[3] =
 * (i, j, numpy |H[j, i]|) of the largest strict-lower-triangle entry (subspace
 * mode: d_mask n bytes, exactly one endpoint in the target), ties to the
 * smallest (i, j); i = j = -1 when there is none.  n < 65536.  Synchronous. */
int qch_npad_sparse_select_c128(const int64_t* d_indptr, const int32_t* d_indices, const void* d_data, int64_t n,
                                const unsigned char* d_mask, int exact_keys, double* out, void* stream);
/* ladder_test_hamiltonian (models.py:194-209), the bench_givens operator
 * a^dag a + (a + a^dag) on n levels, built on the device as a CSR:
 * d_indptr (n+1) int64, d_indices / d_data (3n - 3; the zero diagonal entry (0,0) is
 * not stored, as HermitianOperator eliminates explicit zeros). */
int qch_build_ladder_csr_c128(int64_t n, int64_t* d_indptr, int32_t* d_indices, void* d_data, void* stream);
/* HermitianOperator.entry on a device CSR: d_out (3 complex, device) =
 * H[j,i], H[i,i], H[j,j] — the inputs of givens_rotation_matrix
 * (npad.py:111-117). */
int qch_npad_sparse_entries_c128(const int64_t* d_indptr, const int32_t* d_indices, const void* d_data, int64_t n,
                                 int64_t i, int64_t j, void* d_out, void* stream);

/* Device-side builder of the transmon (x) resonator Hamiltonians of the NPAD
 * configs: for each b, params[4b..4b+3] =
 * {omega_q, alpha, omega_r, g}; H = wq n + a/2 n(n-1) (x) I + I (x) wr a^dag a
 * + g (b + b^dag) (x) (a + a^dag), index q*n_r + k.  d_h: (batch, nq*nr)^2.
 * d_maxabs (nullable): double[batch] = max_abs of each operator
 * (operators.py:92-99), formed while the entries are written. */
int qch_build_transmon_resonator_c128(void* d_h, int64_t batch, int64_t n_q, int64_t n_r,
                                      const double* d_params, double* d_maxabs, void* stream);
/* spin_chain_hamiltonians (models.py:288-325), the drift built on the device
 * as a CSR: d_indptr (2^L + 1) int64, d_indices / d_data (capacity 2^L; the
 * diagonal's exact zeros are not stored, as scipy's diags -> csr drops them),
 * *nnz (host) = stored entries.  1 <= length <= 30 (one CTA compacts the
 * diagonal: sized for the dense-propagation chains, L <= 20).  Synchronous. */
int qch_build_spin_chain_drift_c128(int64_t length, double qubit_freq, double j_nn, double g_nnn,
                                    int64_t* d_indptr, int32_t* d_indices, void* d_data, int64_t* nnz,
                                    void* stream);
/* The chain's global controls sum_j sx_j and sum_j sy_j (models.py:311-320)
 * on the device: two CSRs of L 2^L entries each, sorted columns.
 * Asynchronous. */
int qch_build_global_xy_c128(int64_t length, int64_t* d_indptr_x, int32_t* d_indices_x, void* d_data_x,
                             int64_t* d_indptr_y, int32_t* d_indices_y, void* d_data_y, void* stream);

/* -------------------------------------------------------------- Magnus --- */

/* magnus_coefficients (magnus.py:151-169) and, for order 2, the second-order
 * coefficients alpha (M,K) and beta (M, K(K-1)/2) of SURVEY.md Appendix B.
 * d_sig: (K, S) float64.  d_c1: (M, K).  d_c2 (order 2, else nullable):
 * (M, K + K(K-1)/2) = [alpha_0..alpha_{K-1}, beta_01, beta_02, ..].
 * dt = grid spacing.  Returns QCH_ERR_GRID for M < 1 or M not dividing S-1. */
int qch_magnus_coefficients(const double* d_sig, int64_t K, int64_t S, int64_t M, double dt, int order,
                            double* d_c1, double* d_c2, void* stream);

/* Basis commutators [A,B] = AB - (AB)^dag of Hermitian operands: d_out gets
 * [H0,H_k] for k < K then [H_k,H_l] for k < l, each (N,N). */
int qch_magnus_commutators_c128(const void* d_h0, const void* d_hk, int64_t K, int64_t N, void* d_out,
                                void* stream);

/* assemble_effective_hams (magnus.py:172-190), intervals [m0, m0+mb):
 * Hbar_n = dt_int*H0 + sum_k c1[n,k] H_k  (+ (-i/2) X_n for order 2). */
int qch_magnus_assemble_c128(const void* d_h0, const void* d_hk, const void* d_comm, int64_t K, int64_t N,
                             const double* d_c1, const double* d_c2, int64_t m0, int64_t mb, double dt_int,
                             int order, void* d_hbar, void* stream);

/* _expm_minus_i (expm.py:56-71) for a batch: U_b = exp(-i H_b), scaling and
 * squaring Taylor (degree <= 18; Hermitian batches as cos - i sin by
 * Paterson-Stockmeyer on half (Hermitian) GEMMs).  d_work: scratch of 8*batch*n*n complex128.
 * Checks finiteness (expm.py:81-82, 97-99): QCH_ERR_NONFINITE, first bad
 * item index in *bad_index (host, nullable). */
int qch_expm_minus_i_batch_c128(const void* d_h, int64_t batch, int64_t n, void* d_u, void* d_work,
                                int64_t* bad_index, void* stream);

/* The scaling norm of _expm_minus_i (expm.py:59) for a batch: d_out[b] =
 * max_r sum_c |(-i H_b)_rc|, numpy's pairwise summation order bit for bit
 * (the value that picks the number of squarings).  Asynchronous. */
int qch_expm_norm_c128(const void* d_h, int64_t batch, int64_t n, double* d_out, void* stream);

/* UnitaryPropagator.validate (expm.py:40-47) for a batch: returns
 * QCH_ERR_NONFINITE (and *bad_index) for the first propagator with
 * ||UU^dag - I||_F > 1e-10*n or ||det U| - 1| > 1e-8. */
int qch_validate_unitary_batch_c128(const void* d_u, int64_t batch, int64_t n, int64_t* bad_index,
                                    void* stream);

/* evolve (magnus.py:214-267), whole pipeline on the device: coefficients,
 * assembly (order 1|2), propagators, ordered product and trajectory.
 * d_h0 (N,N), d_hk (K,N,N), d_sig (K,S), d_psi0 (N).  d_traj: (M+1, N).
 * d_comm (nullable): precomputed qch_magnus_commutators_c128 output for
 * order 2 (computed internally when NULL).
 * d_props (nullable): (M, N, N) propagators.  check: validate propagators.
 * NormDrift (magnus.py:270-273) -> QCH_ERR_NORM_DRIFT with the interval in
 * *bad_index. */
int qch_magnus_evolve_c128(const void* d_h0, const void* d_hk, const void* d_comm, int64_t K, int64_t N,
                           const double* d_sig, int64_t S, double t_start, double t_end, int64_t M, int order,
                           const void* d_psi0, void* d_traj, void* d_props, int check, int64_t* bad_index,
                           void* stream);

/* ||U_b U_b^dag - I||_F for a batch (DMMA GEMM with a fused reduction):
 * the unitarity audit of npad.py:257 and expm.py:35-38.  d_defect: (batch). */
int qch_unitarity_defect_c128(const void* d_u, int64_t batch, int64_t n, double* d_defect, void* stream);

/* Asynchronous evolve for N <= 4 (pipelined throughput): no host sync; the
 * two status words (first non-unitary interval, first norm-drift interval;
 * ~0 = none) are copied to d_flags (device, 2 x uint64) for a later check. */
int qch_magnus_evolve_async_c128(const void* d_h0, const void* d_hk, const void* d_comm, int64_t K, int64_t N,
                                 const double* d_sig, int64_t S, double t_start, double t_end, int64_t M, int order,
                                 const void* d_psi0, void* d_traj, void* d_props, int check, void* d_flags,
                                 void* stream);

/* Replayed evolve (new API, EvolvePlan): like qch_magnus_evolve_async_c128
 * but with a caller-owned self-cleaning workspace d_work of
 * qch_magnus_plan_workspace_bytes(N, M) bytes, prepared once by
 * qch_magnus_plan_workspace_init; the kernel's last block restores it after
 * every launch, so each launch is a single kernel (one CUDA-graph node).
 * One workspace per concurrently running evolve. */
int64_t qch_magnus_plan_workspace_bytes(int64_t N, int64_t M);
int qch_magnus_plan_workspace_init(void* d_work, int64_t N, int64_t M, void* stream);
int qch_magnus_evolve_plan_c128(const void* d_h0, const void* d_hk, const void* d_comm, int64_t K, int64_t N,
                                const double* d_sig, int64_t S, double t_start, double t_end, int64_t M, int order,
                                const void* d_psi0, void* d_traj, void* d_props, int check, void* d_work,
                                void* d_flags, void* stream);

/* evolve (magnus.py:214-267) with HOST buffers — the reference-facing call:
 * h_h0 (N,N), h_hk (K,N,N), h_sig (K,S) row-major, h_psi0 (N) are read from
 * host memory, the trajectory (M+1, N) is written to h_traj.  For N <= 4 ONE
 * single-pass fused kernel does everything: page-locked h_sig / h_traj are
 * read and written by the kernel itself over the host link (zero copy, the
 * transfers overlap the arithmetic); pageable buffers are staged by the
 * driver.  h_times (nullable, M+1 doubles) receives np.linspace(t_start,
 * t_end, M+1) bit for bit (magnus.py:263), filled on the host while the
 * kernel runs.  Synchronous.  Errors as qch_magnus_evolve_c128.  Not
 * re-entrant on one device (shares the device's workspace and side streams). */
int qch_magnus_evolve_host_c128(const void* h_h0, const void* h_hk, int64_t K, int64_t N, const double* h_sig,
                                int64_t S, double t_start, double t_end, int64_t M, int order, const void* h_psi0,
                                void* h_traj, int check, int64_t* bad_index, double* h_times, void* stream);

/* Fixed-step RK4 comparator (reference.py:11-65): psi' = -i H(t) psi with
 * H(t) = H0 + sum_k u_k(t) H_k read off grid samples (2*steps | S-1), all
 * steps in one call.  The operators come as ONE union-pattern CSR
 * (d_indptr int64 (n+1), d_indices int32 (nnz), d_vals complex128
 * (nnz, K+1): the H0 value then H_1..H_K at each stored position);
 * d_sig (K, S) f64; d_traj (steps+1, n) receives psi0 and every step.
 * Synchronous. */
int qch_rk4_evolve_c128(const int64_t* d_indptr, const int* d_indices, const void* d_vals, int64_t n, int64_t K,
                        const double* d_sig, int64_t S, double t_start, double t_end, int64_t steps,
                        const void* d_psi0, void* d_traj, void* stream);

/* ------------------------------------------------------------ GEMM ------- */

/* Batched complex128 GEMM on the FP64 tensor pipe (DMMA, mma.sync f64):
 * C_b = A_b @ B_b, (m,k) x (k,n), batch strides in elements; C must not
 * alias A or B. */
int qch_zgemm_batched(const void* d_a, const void* d_b, void* d_c, int64_t m, int64_t n, int64_t k,
                      int64_t batch, int64_t stride_a, int64_t stride_b, int64_t stride_c, void* stream);

/* C_b = A_b @ B_b for n x n factors whose product is Hermitian (commuting
 * Hermitian factors, e.g. two polynomials of one Hermitian matrix — every
 * product of the Hermitian exp(-iH) of expm.py:56-71): only the tiles meeting
 * the lower triangle are computed, the upper triangle is written as the
 * conjugate mirror (C is exactly Hermitian off the diagonal).  Contiguous
 * batch (stride n*n). */
int qch_zgemm_herm_batched(const void* d_a, const void* d_b, void* d_c, int64_t n, int64_t batch, void* stream);
/* Real DMMA products per complex product of the GEMMs above: 3 (Gauss / 3M,
 * the default: 6 N^3 tensor flops per complex GEMM) or 4 (QCH_ZGEMM_3M=0:
 * 8 N^3).  For roofline accounting. */
int qch_zgemm_real_products(void);
/* Executed DMMA flops of every TMA-kernel GEMM launched by this process
 * (computed tiles x 128 x 64 x K x 2 x real products; diagnostics: the
 * bench's tensor-pipe roofline divides its increase by the GEMM time). */
double qch_dmma_flops(void);

/* -------------------------------------- int8 tensor-core (tcgen05) ----- */

/* The Hermitian products of exp(-iH) (qch_zgemm_herm_batched and the
 * expm's Paterson-Stockmeyer / cos-sin steps) for any 512 <= n <= 16384 run
 * by default on the int8 tensor cores: each FP64 operand is cut into 8 exact
 * int8 slices (7 bits each, per-row power-of-two scale: the Ozaki scheme),
 * the 36 slice pairs with i + j <= 7 are multiplied with tcgen05.mma
 * kind::i8 (cta_group::2, 256 x 256 tiles, exact int32 in TMEM) and folded
 * into FP64 — FP64 level — in the Gauss / 3M complex form.  Inside the
 * expm, products that reach U only through small Taylor weights use fewer
 * leading slices (an error-bound plan, QCH_OZ_ADAPT=0 disables).  engine: 1 = int8 tensor
 * cores, 0 = DMMA, -1 = query; returns the previous setting. */
int qch_set_herm_gemm(int engine);
/* int8 tensor operations (2 per MAC) issued by the Ozaki GEMMs so far, and
 * the FP64 complex-product flops (8 M N K over the computed tiles) those
 * GEMMs stood in for (accounting). */
double qch_int8_ops(void);
double qch_int8_fp64_equiv_flops(void);
/* Diagnostics of the two building blocks: C_i32 (m x n) = A_i8 (m x k) .
 * B_i8 (n x k)^T on tcgen05 kind::i8 (k % 16 == 0), and P_f64 (m x n) =
 * X Y^T for one real component of complex matrices x (m x k), y (n x k)
 * (comp 0 Re, 1 Im, 2 Re+Im, 3 Re-Im, 4 -Im) through s slices (n even). */
int qch_i8gemm_test(const void* d_a, const void* d_b, void* d_c, int64_t m, int64_t n, int64_t k, void* stream);
int qch_oz_real_test(const void* d_x, int xcomp, const void* d_y, int ycomp, void* d_out, int64_t m, int64_t n,
                     int64_t k, int s, void* stream);

/* ------------------------------------------------ multi-GPU Magnus ------- */

/* The N > 4 pipeline in two halves (multi-GPU relay, sharding.RelayEvolvePlan):
 * qch_magnus_propagators_c128: U_m = exp(-i Hbar_m) (expm.py:56-71, the
 * batched propagators of evolve's dense path, magnus.py:247-248) for the M
 * intervals of a local signal window d_sig (K, S), S - 1 = M * sub; dt the
 * grid spacing, dt_int the interval length; d_comm: basis commutators (order
 * 2); d_u (M, N, N); check -> validate each (QCH_ERR_NONFINITE, local index).
 * qch_magnus_chain_c128: the sequential product psi <- U_m psi
 * (magnus.py:249-252) from d_psi_in, every state into d_rows (M, N), with the
 * NormDrift check (QCH_ERR_NORM_DRIFT, local index).  Both synchronous. */
int qch_magnus_propagators_c128(const void* d_h0, const void* d_hk, const void* d_comm, int64_t K, int64_t N,
                                const double* d_sig, int64_t S, double dt, double dt_int, int64_t M, int order,
                                int check, void* d_u, int64_t* bad_index, void* stream);
int qch_magnus_chain_c128(const void* d_u, int64_t N, int64_t M, const void* d_psi_in, void* d_rows,
                          int64_t* bad_index, void* stream);


/* Interval sharding, N <= 4.  Workspace bytes for M local
 * intervals. */
int64_t qch_magnus_shard_workspace_bytes(int64_t N, int64_t M);
/* Local intervals of one rank (pass 1, asynchronous): the fused single-pass
 * kernel in prefix mode — coefficients from the local signal slice (K, S)
 * with grid spacing dt and interval length dt_int, propagators, in-tile and
 * tile prefixes into d_work; writes the block product B = U_last...U_first
 * to d_block (N,N) — the tensor the ranks all-gather. */
int qch_magnus_shard_prepare_c128(const void* d_h0, const void* d_hk, const void* d_comm, int64_t K, int64_t N,
                                  const double* d_sig, int64_t S, double dt, double dt_int, int64_t M, int order,
                                  int check, void* d_work, void* d_block, void* stream);
/* psi_start = B_{rank-1} ... B_0 psi0 from the gathered blocks (world, N, N). */
int qch_magnus_apply_prefix_c128(const void* d_blocks, int64_t N, int64_t rank, const void* d_psi0,
                                 void* d_psi_start, void* stream);
/* Local trajectory (M+1, N) from psi_start; NormDrift / NonFinite checks. */
int qch_magnus_shard_finish_c128(int64_t N, int64_t M, void* d_work, const void* d_psi_start, void* d_traj,
                                 int check, int64_t* bad_index, void* stream);

/* qch_magnus_shard_finish_c128 without a host synchronisation: the two
 * status words (first non-unitary, first norm-drift local interval; ~0 =
 * none) are copied to d_flags (device, 2 x uint64). */
int qch_magnus_shard_finish_async_c128(int64_t N, int64_t M, void* d_work, const void* d_psi_start, void* d_traj,
                                       void* d_flags, void* stream);

/* ------------------------------------------------ measurement ------------ */

/* FP64 peak probes: kind 0 = DFMA pipe, kind 1 = DMMA (mma.sync f64).
 * *flops receives the launch's flop count (caller times it). */
int qch_peak_kernel(int kind, int blocks, int iters, double* d_sink, double* flops, void* stream);
/* CUDA-event timing of the hot kernels on their launching stream. */
void qch_profile_enable(int on);
int qch_profile_read(double* total_ms, int64_t* counts, char* names_buf, int64_t buf_len, int cap, int reset);

#ifdef __cplusplus
}
#endif
#endif /* QCHEFF_H_ */
