/*
 * iedd_b200.h -- C-ABI of the B200 (sm_100a) Schwarz-PCG hot path.
 *
 * This is the drop-in boundary for the reference package iedd 0.1.0
 * (/root/reference/pkg/src/iedd).  The reference is pure Python and binds no
 * FFI; its duck-typed protocol (pcg.py:26-33 "_as_callable", spectrum.py:147,
 * :161) is what these entry points replace.  The Python package
 * paper_2108_12574_b200 binds them with ctypes.
 *
 * Conventions
 *   - All double/int pointers named d_* are CUDA device pointers owned by the
 *     caller unless the function creates a handle.  h_* pointers are host.
 *   - All work is enqueued on the caller's stream (cudaStream_t passed as
 *     void*).  Functions never synchronise the host except where they return
 *     host scalars (ie_pcg_f64, ie_lanczos_f64, *_create with a bad_block out).
 *   - Return codes: 0 ok; <0 argument error (the Python layer raises
 *     ValueError with the reference's message); >0 numerical failure:
 *       IE_ERR_NOT_SPD        subdomain Cholesky hit a non-positive pivot
 *                             (NotPositiveDefinite, precond.py:197-200)
 *       IE_ERR_BREAKDOWN      PCG p^T A p <= 0 or non-finite (pcg.py:99-103)
 *       IE_ERR_NONFINITE      non-finite true residual (pcg.py:109-110)
 *       IE_ERR_NO_RITZ        Lanczos produced no Ritz value (spectrum.py:188-189)
 *       IE_ERR_CUDA           a CUDA runtime call failed (message via ie_last_error)
 *   - Vectors are length N = n^dim in the reference's C order (last axis
 *     fastest, geometry.py:42-44).
 */
#ifndef IEDD_B200_H
#define IEDD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IE_OK 0
#define IE_ERR_ARG (-1)
#define IE_ERR_NOT_SPD 1
#define IE_ERR_BREAKDOWN 2
#define IE_ERR_NONFINITE 3
#define IE_ERR_NO_RITZ 4
#define IE_ERR_CUDA 5

/* Operator metadata: replaces KernelOperator's scalar fields
 * (kernel.py:110-162: grid.dim, grid.n_per_dim, lattice_spacing, weight,
 * diag_value).  Entries are A_ij = weight * K(spacing * |a_i - a_j|) for
 * i != j with integer multi-indices a, K = -log(r)/(2 pi) for dim 1, 2 and
 * 1/(4 pi r) for dim 3 (kernel.py:146-149); A_ii = diag. */
typedef struct ie_geom {
    int32_t dim;
    int32_t n;
    double spacing;
    double weight;
    double diag;
} ie_geom;

/* ---------------------------------------------------------------- K1 ---- */
typedef struct ie_matvec ie_matvec;

#define IE_MATVEC_DIRECT 0 /* K1: O(N^2) direct sum, kernel evaluated per pair */
#define IE_MATVEC_FFT 1    /* K1b: O(N log N) circulant-embedding FFT (any n <= 4096) */

/* Replaces ToeplitzMatvec.__init__ (toeplitz.py:19-32).  ie_matvec_create
 * builds the direct-sum operator (device log table); ie_matvec_create_method
 * selects the method -- IE_MATVEC_FFT also computes the real, even symbol of
 * the M^dim circulant embedding on the device, M = the smallest power of two
 * >= 2n - 1 (= 2n, the reference's size, for power-of-two n; any M >= 2n - 1
 * gives the same Toeplitz product). */
int ie_matvec_create(const ie_geom* g, ie_matvec** out);
int ie_matvec_create_method(const ie_geom* g, int32_t method, ie_matvec** out);
void ie_matvec_destroy(ie_matvec* m);

/* Replaces ToeplitzMatvec.matvec (toeplitz.py:39-50), matrix-free:
 * Y[:, c] = A[row_begin:row_end, :] X[:, c] for c < nrhs (nrhs in {1, 2}).
 * X is N x nrhs column-major with leading dimension ldx (all N rows, full
 * vector); Y receives rows row_begin..row_end-1 at Y + (row - row_begin)
 * with leading dimension ldy.  Every row is summed in the same order for any
 * row range and any nrhs, so results are bitwise independent of sharding and
 * of RHS fusion. */
int ie_matvec_f64(const ie_matvec* m, const double* d_X, int64_t ldx, int32_t nrhs,
                  double* d_Y, int64_t ldy, int64_t row_begin, int64_t row_end,
                  void* stream);

/* Band (slab) passes of the FFT method for the sharded solver (2D, SURVEY.md
 * 8(e)); together they are ToeplitzMatvec.matvec (toeplitz.py:39-50) split
 * across ranks with two all-to-all transposes in between.  Rank g owns grid
 * rows [row_begin, row_end) (whole rows, point indices); the M spectrum
 * columns (M = the circulant size) are cut into `parts` slabs of
 * Mc = M / parts (a power of two).
 *   band_fwd: X (nrhs columns, ldx, band rows only) -> d_out, complex
 *             (nrows * M), destination-major: slab h at h * nrows * Mc;
 *   band_cols: d_buf = every grid row of columns [col_begin, col_end),
 *             row-major (n x ncols complex), in place: forward * symbol * inverse;
 *   band_inv: d_in (destination-major as band_fwd wrote it, after the reverse
 *             transpose) -> Y (band rows, ldy, nrhs columns).
 * With nrhs == 2 the exact power-of-two column scaling of the 2-RHS packing
 * uses d_scales = the two multipliers (device, 2 doubles: 2^-e0, 2^-e1) the
 * caller derived from GLOBAL quantities (pcg_scale_rule in distributed.py),
 * so every rank scales identically and the line arithmetic is bitwise that
 * of the single-GPU pass. */
int ie_matvec_band_fwd_f64(const ie_matvec* m, const double* d_X, int64_t ldx, int32_t nrhs,
                           int64_t row_begin, int64_t row_end, int32_t parts, void* d_out,
                           const double* d_scales, void* stream);
int ie_matvec_band_cols_f64(const ie_matvec* m, void* d_buf, int64_t col_begin, int64_t col_end,
                            void* stream);
int ie_matvec_band_inv_f64(const ie_matvec* m, const void* d_in, int64_t row_begin, int64_t row_end,
                           int32_t parts, double* d_Y, int64_t ldy, int32_t nrhs, const double* d_scales,
                           void* stream);
/* Per-2048-chunk partial maxima of |x0| and |x1| (x1 = x0 + ldx; ldx = 0:
 * x1 = x0) over n entries starting at a chunk boundary: d_out[2c], d_out[2c + 1]. */
int ie_absmax_partials_f64(const double* d_X, int64_t ldx, int64_t n, double* d_out, void* stream);

/* Replaces KernelOperator.assemble_block (kernel.py:170-184):
 * d_out (nr x nc row-major) = A[rows, cols]. */
int ie_assemble_block_f64(const ie_geom* g, const int64_t* d_rows, int64_t nr,
                          const int64_t* d_cols, int64_t nc, double* d_out, void* stream);

/* ----------------------------------------------------------- K2 / K3 ---- */
typedef struct ie_precond ie_precond;

#define IE_VARIANT_PACKED_INVERSE 0  /* apply = packed symmetric A_k^{-1} matvec */
#define IE_VARIANT_SUBST 1           /* apply = forward/back substitution with G_k */

/* Replaces precond.from_decomposition(op, dec, backend="exact")
 * (precond.py:157-215) + linalg.cholesky (linalg.py:36-45).
 * Subdomains are given as CSR on the HOST: h_offsets[D+1], h_indices[...],
 * each subdomain's index set sorted ascending (geometry.py:71-82).
 * share_translated bit 0 factorises one representative per translation class
 * (blocks whose points are translates of each other are bitwise identical
 * here, so this is exact); bit 1 (the reference's share_mirrored_subdomains,
 * precond.py:137-154, _MirroredSolver :43-62) also identifies blocks related
 * by grid reflections, each block's points taken in a canonical order.  On
 * IE_ERR_NOT_SPD, *bad_block = the first failing subdomain id. */
int ie_precond_create(const ie_geom* g, const int64_t* h_offsets, const int64_t* h_indices,
                      int64_t D, int32_t variant, int32_t share_translated,
                      ie_precond** out, int64_t* bad_block, void* stream);
void ie_precond_destroy(ie_precond* p);

/* Replaces Preconditioner.apply (precond.py:91-100): z = sum_k R_k^T A_k^{-1} R_k r,
 * summed per point in ascending subdomain id from exact zeros. */
int ie_precond_apply_f64(const ie_precond* p, const double* d_r, double* d_z, void* stream);

/* Replaces Preconditioner.stats (precond.py:122-130) plus device footprint:
 * out[0] = S (max block size), out[1] = reference memory_bytes (8*(s^2+s)
 * summed), out[2] = device factor bytes, out[3] = number of factorised blocks,
 * out[4] = D. */
int ie_precond_stats(const ie_precond* p, int64_t* out5);

/* Factor-level readback (test hook for linalg.cholesky, linalg.py:36-45):
 * subdomain k's stored block as an s x s row-major HOST matrix.  *kind = 1:
 * the Cholesky factor G, A_k = G^T G (variant SUBST, s <= 160); *kind = 0:
 * A_k^{-1}.  h_out = NULL returns *s_out only. */
int ie_precond_block_f64(const ie_precond* p, int64_t k, double* h_out, int64_t* s_out, int32_t* kind);

/* ---------------------------------------------------------- K4 / K5 ---- */
/* Replaces pcg.solve (pcg.py:54-136) for a native operator and
 * preconditioner (precond may be NULL = identity, pcg.py:68).  f, u are
 * device vectors of length N; u is overwritten with the iterate.
 * h_history must hold max_iters+1 doubles; *n_it = number of entries - 1.
 * h_flags[0] = converged, h_flags[1] = stagnated.  h_times[0] = t_pcg (s),
 * h_times[1] = mean preconditioner-apply time t_s (s, device events).
 * On IE_ERR_BREAKDOWN / IE_ERR_NONFINITE: *fail_iter, *fail_value hold the
 * iteration and p^T A p (resp. residual). */
int ie_pcg_f64(const ie_matvec* A, const ie_precond* T, const double* d_f, double* d_u,
               double tol, int64_t max_iters, double* h_history, int64_t* n_it,
               int32_t* h_flags, double* h_times, int64_t* fail_iter, double* fail_value,
               void* stream);

/* ie_pcg_f64 with the solution delivered to page-locked HOST memory h_u (the
 * reference's solve returns a host array, pcg.py:133-136): the device-to-host
 * copy starts when u is final -- after the last iteration's update, beside the
 * closing true-residual pass -- instead of after the solve.  Same solve
 * otherwise (bitwise). */
int ie_pcg_host_f64(const ie_matvec* A, const ie_precond* T, const double* d_f, double* h_u,
                    double tol, int64_t max_iters, double* h_history, int64_t* n_it,
                    int32_t* h_flags, double* h_times, int64_t* fail_iter, double* fail_value,
                    void* stream);
/* ie_pcg_f64 instrumented for the bench's per-kernel rooflines: iterations
 * launched one by one (no graph) with CUDA events between the kernel groups;
 * h_phase_ms[0..4] = mean device ms per steady-state (2-RHS) iteration of
 * the matvec, k_post_pass, k_iter_a, the preconditioner apply, k_iter_b. */
int ie_pcg_profile_f64(const ie_matvec* A, const ie_precond* T, const double* d_f, double* d_u,
                       double tol, int64_t max_iters, double* h_history, int64_t* n_it,
                       int32_t* h_flags, double* h_times, double* h_phase_ms, void* stream);

/* ------------------------------------------ sharded K4 (NVLink P2P) ---- */
/* Replaces pcg.solve (pcg.py:54-136) on G ranks, one per GPU (SURVEY.md
 * 8(e); the reference itself is single-process).  Rank g owns points
 * [h_bounds[g], h_bounds[g+1]) of every vector: equal, 2048-aligned bands of
 * whole grid rows; the 2D FFT operator with G | M (its circulant size) and
 * M/G a power of two.
 * T_local = the rank's preconditioner (subdomains intersecting its band,
 * ascending global ids; NULL = identity); h_need[2h], h_need[2h+1] bound the
 * points rank h's subdomains read (its r-halo; NULL without T).
 * Exchanges are direct stores into the peers' memory over NVLink plus a
 * mailbox counter per exchange (no collective library): four exchange points
 * per iteration (row->column transpose, column->need-rows transpose carrying
 * the r-halo, p.q/residual partials, the apply's r.z record).  n_it, history
 * and u are bitwise those of ie_pcg_f64 for every G.
 *   multi-process: ie_shard_create on every rank, ie_shard_export -> host
 *     all-gather of the ie_shard_handle_bytes() blobs (rank order) ->
 *     ie_shard_connect -> ie_pcg_sharded_f64 (collective: every rank calls it);
 *   one process, one device (tests): ie_shard_create for ranks 0..G-1,
 *     ie_shard_connect_local, ie_pcg_sharded_local_f64.
 * d_f_need = f on the rank's need rows [out2[0], out2[1]) of
 * ie_shard_need_rows; d_u_band = the band of u (out).  h_times[1] = mean
 * device time of rank 0's event-timed applies. */
typedef struct ie_shard ie_shard;
int ie_shard_create(const ie_matvec* A, const ie_precond* T_local, int32_t nranks, int32_t rank,
                    const int64_t* h_bounds, const int64_t* h_need, ie_shard** out);
void ie_shard_destroy(ie_shard* s);
int ie_shard_need_rows(const ie_shard* s, int64_t* out2);
int64_t ie_shard_handle_bytes(void);
int ie_shard_export(const ie_shard* s, void* h_out);
int ie_shard_connect(ie_shard* s, const void* h_handles);
int ie_shard_connect_local(ie_shard** shards, int32_t nranks);
int ie_pcg_sharded_f64(ie_shard* s, const double* d_f_need, double* d_u_band, double tol, int64_t max_iters,
                       double* h_history, int64_t* n_it, int32_t* h_flags, double* h_times, int64_t* fail_iter,
                       double* fail_value, void* stream);
int ie_pcg_sharded_local_f64(ie_shard** shards, int32_t nranks, const double* const* d_f_need,
                             double* const* d_u_band, double tol, int64_t max_iters, double* h_history,
                             int64_t* n_it, int32_t* h_flags, double* h_times, int64_t* fail_iter,
                             double* fail_value, void* stream);

/* Replaces spectrum.extremal_eigenvalue_lanczos (spectrum.py:133-190):
 * T = NULL is the identity preconditioner (precond.identity);
 * d_v0 = start vector (caller draws it from default_rng(seed), spectrum.py:148),
 * which = 0 (min) / 1 (max).  *steps = Lanczos steps taken. */
int ie_lanczos_f64(const ie_matvec* A, const ie_precond* T, const double* d_v0,
                   int32_t which, int64_t max_iters, double rtol, double* lambda,
                   int64_t* steps, void* stream);

/* Deterministic vector operations of the PCG iteration (for the sharded
 * driver; identical kernels and reduction order to ie_pcg_f64).
 * ie_dot_partials_f64: part[c] = fixed-tree sum over chunk c (ie_dot_chunk()
 *   elements) of x.y (mode 0) or |x-y|^2 (mode 1).
 * ie_sum_partials_f64: *out (device) = fixed-order sum of nch partials.
 * ie_update_f64: op 0 a += s*b, op 1 a -= s*b, op 2 a = b + s*a (products
 *   rounded first, as numpy does; pcg.py:105-106, :125). */
int64_t ie_dot_chunk(void);
int ie_dot_partials_f64(const double* d_x, const double* d_y, int64_t n, int32_t mode, double* d_part,
                        void* stream);
int ie_sum_partials_f64(const double* d_part, int64_t nch, double* d_out, void* stream);
int ie_update_f64(int32_t op, double* d_a, const double* d_b, double s, int64_t n, void* stream);
/* Per-line partials (nlines lines of n points; x.y for mode 0, |x-y|^2 for
 * mode 1) with the association ie_pcg_f64 uses when the post pass rides in
 * the FFT's last line transform of circulant size M (2D / 3D, M >= 64):
 * thread j < M/8 chains points j + (M/8) m by FMA, then a halving tree. */
int ie_line_partials_f64(const double* d_x, const double* d_y, int64_t nlines, int32_t n, int32_t M,
                         int32_t mode, double* d_part, void* stream);

/* FP64 issue-peak microbenchmark: DFMA instructions (lane ops) per second
 * over all SMs -- the roofline denominator for K1. */
int ie_fp64_peak(double* dfma_per_s, void* stream);
/* FP64 tensor-core (DMMA m8n8k4) throughput microbenchmark, flops/s over all
 * SMs -- the roofline denominator for the class-GEMM apply. */
int ie_dmma_peak(double* flops_per_s, void* stream);

/* Last error text for IE_ERR_CUDA / IE_ERR_ARG (thread-local). */
const char* ie_last_error(void);
/* Number of this library's kernels launched so far (process-wide counter). */
int64_t ie_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* IEDD_B200_H */
