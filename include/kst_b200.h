/*
 * kst_b200.h -- C ABI of libkst_b200.so, the B200 (sm_100a) Kron-STAP hot path.
 *
 * The reference (`kronstap`, pure Python, /root/reference/pkg/src/kronstap,
 * abbreviated src/) has no FFI: its boundary is the Python functions
 * re-exported by src/__init__.py:17-45. Each entry point below replaces one
 * of those functions; the citation on each names the reference interface.
 * INTEGRATION.md shows the ctypes binding a kronstap maintainer would add.
 *
 * Conventions
 *  - Complex data are interleaved (re, im) float64 pairs, i.e. numpy
 *    complex128 memory; row-major (C order) like numpy.
 *  - "dev" pointers are CUDA device pointers; "host" pointers are host
 *    memory. Every call is ordered on `stream` (a cudaStream_t passed as
 *    void*; NULL = legacy default stream). Calls that must report a
 *    data-dependent outcome (iteration counts, degenerate input, non-finite
 *    data) synchronise that stream before returning.
 *  - Return value: KST_OK or one of the KST_ERR_* codes, which the Python
 *    layer maps onto the reference's exception classes (src/errors.py:9-30).
 *    No C++ exception crosses this boundary. kst_last_error() gives text.
 *  - One kst_ctx per (device, host thread). The context owns a grow-only
 *    device workspace; callers own every input/output buffer. Contexts on
 *    different threads/streams may run concurrently; the small FFT / CRT
 *    plans live in device-global constant memory and are uploaded once per
 *    distinct plan, so concurrent callers should share shapes (the windowed
 *    estimator runs its first window alone, then fans out).
 *  - Results are deterministic: fixed-order reductions, no float atomics.
 */
#ifndef KST_B200_H
#define KST_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define KST_OK 0
#define KST_ERR_DIMENSION 1  /* -> DimensionError       */
#define KST_ERR_DATA 2       /* -> DataError            */
#define KST_ERR_DEGENERATE 3 /* -> DegenerateInputError */
#define KST_ERR_CUDA 100     /* CUDA runtime / launch failure */
#define KST_ERR_NOCONV 101   /* internal eigensolver failed to converge */

#define KST_KIND_KRON 0
#define KST_KIND_CLASSICAL 1

typedef struct kst_ctx kst_ctx;

/* Context lifetime. */
int kst_ctx_create(int device, kst_ctx** out);
int kst_ctx_destroy(kst_ctx* ctx);
const char* kst_last_error(const kst_ctx* ctx);
int kst_version(void);

/*
 * Pageable host <-> device copy (the boundary the reference's numpy inputs
 * cross; the reference itself never leaves the host): `bytes` from src to
 * dst through a ring of 4 MB pinned staging chunks filled / drained by
 * `threads` host threads while the copy engine moves the other chunks
 * (~33 GB/s from pageable numpy memory on the B200 box vs ~11 GB/s for a
 * plain pageable cudaMemcpy). dir 0: host src -> dev dst, enqueued on
 * `stream` (src may be reused on return); dir 1: dev src -> host dst,
 * complete on return.
 */
int kst_copy_staged(kst_ctx* ctx, void* dst, const void* src, size_t bytes, int dir, int threads,
                    void* stream);

/* Instrumentation (bench/profiling only; no effect on results):
 * kst_launch_count: kernels launched by this context so far.
 * kst_set_profiling(1): kst_pipeline records CUDA events at its stage
 *   boundaries; kst_stage_times then returns up to `max` stage durations in
 *   ms (scm, lrkron, bases, detect) of the last call, and the count. */
long long kst_launch_count(const kst_ctx* ctx);

/* Sample-covariance engine (K1). mode 0: FP64 tensor-core DMMA tiles (FP64
 * rounding only). mode 1: int8 tensor-core GEMMs on exact 7-bit slices
 * (`slices` per operand, 3..8; relative error ~(slices+1) 2^-7*slices of
 * max|x_a| max|x_b| n). mode 2: int8 residues modulo `slices` = 8..14
 * coprime moduli recombined by the Chinese remainder theorem, products on the
 * hand-written tcgen05 kernel (error: rounding x to beta bits, beta = 32 for
 * 10 moduli and n = 2001). mode 3: mode 2's numerics on cuBLAS int8 GEMMs.
 * Default: mode 2 with 10 moduli (else mode 1 with 6 slices, else mode 0);
 * env KST_GRAM=dmma|int8|crt|crt-cublas and KST_GRAM_SLICES override it at
 * context creation. */
int kst_set_gram(kst_ctx* ctx, int mode, int slices);
int kst_get_gram(const kst_ctx* ctx, int* mode, int* slices);
/* Detection (K5) precision. bits = 32 (default): FP64 load pass (spatial
 * reduction, temporal-projection coefficients) + FP32 prime-factor DFT and
 * pixel stage (detect_f32.cu) for single-map uniform-grid detection with
 * p <= 4, kb <= 3, q <= D and D a product of coprime factors <= 32 (or a*b,
 * a, b <= 32); every other case runs the FP64 kernels. bits = 64: the FP64
 * kernels everywhere. Env KST_DETECT=f32|f64 sets it at context creation. */
int kst_set_detect(kst_ctx* ctx, int bits);
int kst_get_detect(const kst_ctx* ctx, int* bits);
/* int8 tensor ops issued by the last int8 Gram (0 if none); with profiling on,
 * kst_stage_times entry 5 is that Gram's int8 GEMM span in ms. */
double kst_gram_int8_ops(const kst_ctx* ctx);
int kst_set_profiling(kst_ctx* ctx, int on);
int kst_stage_times(kst_ctx* ctx, double* ms, int max);

/*
 * Sample covariance -- replaces `sample_covariance(snapshots, p, q)`
 * (src/lrkron.py:53-78): S = (1/n) X^T conj(X), exactly Hermitian.
 *   X  dev, (n, d) complex, d = p*q snapshot rows (src/layout.py:35-41)
 *   S  dev, (d, d) complex, written in full (both triangles)
 */
int kst_scm(kst_ctx* ctx, const double* X, int64_t n, int64_t d, double* S,
            void* stream);

/*
 * LR-Kron estimate -- replaces `lr_kron_estimate(scm, rank_spatial,
 * rank_temporal, tol, max_iter, keep_iterates)` (src/lrkron.py:118-230).
 *   S            dev (pq, pq) complex
 *   validate     1: run the reference's input checks (src/lrkron.py:100-115)
 *   spatial      dev (p, p) complex   <- KronCovEstimate.spatial
 *   temporal     dev (q, q) complex   <- KronCovEstimate.temporal (may be NULL)
 *   tb_vectors   dev (q, rank_temporal) complex, tb_values host (rank_temporal):
 *                top eigenpairs of the final b with the reference's order and
 *                phase conventions (src/linalg.py:82-121); NULL to skip. Only
 *                filled when rank_temporal < q.
 *   residuals    host (max_iter) float64; *n_residuals entries written
 *   iter_spatial dev (max_iter, p, p), iter_b dev (max_iter, q, q): per-
 *                iteration (spatial, b) copies for keep_iterates; may be NULL
 */
int kst_lrkron(kst_ctx* ctx, const double* S, int p, int q, int rank_spatial,
               int rank_temporal, double tol, int max_iter, int validate,
               double* spatial, double* temporal, double* tb_vectors,
               double* tb_values, double* residuals, int* n_residuals,
               int* iterations, int* converged, double* iter_spatial,
               double* iter_b, void* stream);

/*
 * Hermitian eigen-helpers with the reference's conventions.
 * kst_heig_top: top `r` eigenpairs (descending; ties by dominant index;
 *   pivot entry real positive) of a dev (n, n) Hermitian matrix ->
 *   values host (r), vectors dev (n, r). Replaces hermitian_eig
 *   (src/linalg.py:82-121) restricted to the leading r pairs.
 * kst_eig_truncate: replaces eig_truncate (src/linalg.py:124-144).
 * kst_subspace_basis: replaces subspace_basis (src/filters.py:58-73);
 *   *keep = number of columns written (0 means the reference's None).
 */
int kst_heig_top(kst_ctx* ctx, const double* M, int n, int r, double* values,
                 double* vectors, void* stream);
int kst_eig_truncate(kst_ctx* ctx, const double* M, int n, int rank,
                     double* out, void* stream);
int kst_subspace_basis(kst_ctx* ctx, const double* M, int n, int rank,
                       double tol, double* basis, int* keep, void* stream);

/*
 * Detection image -- replaces `detection_image(filt, cube, dopplers,
 * spatial_grid)` (src/filters.py:243-275) for the projection filters
 * (`StapFilter.apply_matrix`, src/filters.py:88-116, kinds kron/classical),
 * and `pass_images` (src/multipass.py:83-102) when groups > 1.
 *   cube      dev (n, p, q) complex
 *   ua        dev (p, ka) complex or NULL (ka = 0)  -- spatial_basis
 *   ub        dev (q, kb) complex or NULL (kb = 0)  -- temporal_basis
 *   dopplers  host (D) float64 (any values; d/D grids take the folded-DFT path)
 *   grid      host (G, p) complex spatial candidates; rows split into
 *             `groups` equal consecutive blocks, one map per block
 *   values    dev (groups, n, D) float64
 */
int kst_detect(kst_ctx* ctx, const double* cube, int64_t n, int p, int q,
               const double* ua, int ka, const double* ub, int kb, int kind,
               int spatial_only, const double* dopplers, int D,
               const double* grid, int G, int groups, double* values,
               void* stream);

/*
 * Whole-cube clutter filter -- replaces StapFilter.apply_matrix
 * (src/filters.py:88-116) applied bin by bin, as `kronstap filter` does
 * (src/cli.py:177-206). cube/out dev (n, p, q) complex.
 */
int kst_filter(kst_ctx* ctx, const double* cube, int64_t n, int p, int q,
               const double* ua, int ka, const double* ub, int kb, int kind,
               int spatial_only, double* out, void* stream);

/*
 * "optimal" filter.
 * kst_chol replaces build_filter(kind="optimal") (src/filters.py:144-163:
 *   as_matrix finite check, then scipy cho_factor(sigma, lower=True)):
 *   sigma dev (d, d) complex row-major, only its lower triangle is read;
 *   L dev (d, d) complex (not aliasing sigma) receives the column-major
 *   lower Cholesky factor.
 *   KST_ERR_DATA if sigma has a non-finite entry or is not positive definite.
 * kst_chol_solve replaces StapFilter.apply_matrix for kind "optimal"
 *   (src/filters.py:98-100: cho_solve): X = sigma^-1 B for every column of the
 *   column-major (d, nrhs) matrix B, i.e. every bin of an (nrhs, p, q) cube
 *   with d = p q. X may equal B. KST_ERR_DATA if B has a non-finite entry.
 */
int kst_chol(kst_ctx* ctx, const double* sigma, int d, double* L, void* stream);
int kst_chol_solve(kst_ctx* ctx, const double* L, int d, const double* B,
                   int64_t nrhs, double* X, void* stream);

/* change_detect (src/multipass.py:105-123): out = |a - b| (or a - b). */
int kst_change(kst_ctx* ctx, const double* a, const double* b, int64_t count,
               int is_signed, double* out, void* stream);

/*
 * Fused frame pipeline -- the README library sequence (pkg/README.md:144-161):
 * sample_covariance -> lr_kron_estimate -> build_filter(kind) ->
 * detection_image, on one cube, without materialising host copies.
 *   cube dev (n, p, q); values dev (groups, n, D); summary host (8 doubles):
 *   [iterations, converged, ka, kb, last residual, 0, 0, 0]
 * Common case (p <= 4, q > 64, rank_temporal <= 24, rank_temporal < q): the
 * whole frame is enqueued without a host synchronisation (convergence, kept
 * ranks and validity decided on the device) and ONE synchronisation reads
 * the outcome; a frame whose device checks fail is recomputed on the
 * synchronous path (env KST_PIPE_ASYNC=0 forces it), so results and errors
 * are the same either way.
 */
int kst_pipeline(kst_ctx* ctx, const double* cube, int64_t n, int p, int q,
                 int rank_spatial, int rank_temporal, double tol, int max_iter,
                 int kind, const double* dopplers, int D, const double* grid,
                 int G, int groups, double* values, double* summary,
                 void* stream);

/*
 * Sync-free half of kst_pipeline, for CUDA-graph capture of a frame: enqueues
 * the common-case schedule (same arguments as kst_pipeline) with no host
 * synchronisation and writes the device outcome record rec (device, 8
 * doubles): [ok, iterations, converged, ka, kb, last residual, 0, 0]. When
 * rec[0] != 1 an assumption of the sync-free form failed and values are not
 * valid: recompute the frame with kst_pipeline. Returns KST_ERR_DIMENSION,
 * with nothing enqueued, outside the common case (p <= 4, q > 64,
 * 1 <= rank_temporal <= 24, rank_temporal < q). After one call with the same
 * arguments (workspaces allocated, resident tables staged) a further call
 * allocates nothing and can be captured with cudaStreamBeginCapture; the
 * capture stays valid while kst_state_epoch() is unchanged.
 */
int kst_pipeline_async(kst_ctx* ctx, const double* cube, int64_t n, int p,
                       int q, int rank_spatial, int rank_temporal, double tol,
                       int max_iter, int kind, const double* dopplers, int D,
                       const double* grid, int G, int groups, double* values,
                       double* rec, void* stream);

/* Resident-state epoch (process-wide): changes whenever device state a
 * captured frame depends on changes outside the capture -- a workspace or
 * pinned buffer reallocated, a constant bank uploaded, resident detection
 * tables restaged. */
long long kst_state_epoch(void);

/*
 * Windowed (L-mode) estimator, one call for a run of windows (SURVEY.md §8
 * "L-mode definition"; the reference has no windowed mode -- each window is
 * its README sequence, pkg/README.md:144-161: sample_covariance
 * (src/lrkron.py:53) -> lr_kron_estimate (src/lrkron.py:118) -> build_filter
 * (src/filters.py:137) -> detection_image (src/filters.py:243)).
 *   cube dev: frame bins [a, a + rows) (n_bins in the frame), (rows, p, q);
 *   windows s = s_begin, s_begin + s_step, ... < s_end train on bins
 *   [s, s + n_w) and detect the test bins whose window is s, clipped to the
 *   tile [lo, hi); values dev (hi - lo, D) float64 (row 0 = bin lo).
 */
int kst_windowed(kst_ctx* ctx, const double* cube, int64_t a, int64_t n_bins,
                 int p, int q, int n_w, int64_t lo, int64_t hi, int64_t s_begin,
                 int64_t s_end, int64_t s_step, int rank_spatial,
                 int rank_temporal, double tol, int max_iter, int kind,
                 int drop_temporal, const double* dopplers, int D,
                 const double* grid, int G, double* values, void* stream);

/*
 * Batched windowed (L-mode) estimator + detector for the test-bin tile
 * [lo, hi) (same semantics and arguments as kst_windowed over all the tile's
 * windows; the reference per-window sequence is pkg/README.md:144-161, i.e.
 * src/lrkron.py:53,118 and src/filters.py:137,243 per window). Every window
 * is estimated from the banded snapshot Gram (P x P blocks) in one CTA --
 * no (pq)^2 covariance or q^2 factor per window -- and each test bin is
 * detected from its window's bin spectra. Windows outside the batched
 * limits (p > 3, n_w > 128, rank_temporal > 6, G > 64, or a small
 * eigensolve that does not converge) run on the per-window step path.
 *   window_info host (optional): 8 ints per window s = window_start(lo) ..
 *   window_start(hi - 1): {status, iterations, converged, ka, kb,
 *   Rayleigh-Ritz rounds, r, n_w r}; status 64 = recomputed on the step
 *   path; all -1 when the whole call took the step path.
 */
int kst_lmode(kst_ctx* ctx, const double* cube, int64_t a, int64_t n_bins,
              int p, int q, int n_w, int64_t lo, int64_t hi, int rank_spatial,
              int rank_temporal, double tol, int max_iter, int kind,
              int drop_temporal, const double* dopplers, int D,
              const double* grid, int G, double* values, int* window_info,
              void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* KST_B200_H */
