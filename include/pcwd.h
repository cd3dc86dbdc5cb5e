/* pcwd.h — C ABI of the B200 product-convolution wavelet decomposition library (libpcwd.so).
 *
 * What it computes (PAPER.md arxiv 2005.09870):
 *   H f = Σ_{k=1..m} u_k ⋆ (v_k ⊙ f)                        Eq. (2)
 *   Θ = Ψ* H Ψ,  Θ[μ][λ] := θ[λ,μ] = <H ψ_λ, ψ_μ>             P:43, P:176 (R1)
 * in the periodic orthogonal wavelet basis of P:93-127 (depth J, filter h, g from P:100),
 * restricted to a retained index set (R14-R16).  This is the exact form of
 * Algorithm 1: A_k's circulant sub-band generators in spatial form
 * (Lemma 1) times B_k by the sparse cascade (Lemma 6), the
 * k-sum taken before the cascade; no truncation of A_k.
 *
 * Work unit: one test wavelet μ; the library produces row μ of Θ (all retained λ) as CSR.
 * Units are Λ indices (layout: coarse block, then levels J..1, orientations (0,1),(1,0),
 * (1,1), positions row-major — DESIGN.md R2/R3).  A handle owns the contiguous shard
 * [row0, row1) of units chosen by (rank, world) with a cost-balanced split.
 *
 * Conventions
 *   - All functions return a pcwd_status; pcwd_error_string() names it.  No global state:
 *     handles are independent; one handle must not be used from two threads at once.
 *   - "host or device" pointers are classified with cudaPointerGetAttributes.
 *   - Streams are passed as void* (a cudaStream_t; NULL = legacy default stream).
 *   - Nothing here blocks on the GPU unless stated ("synchronous").
 */
#ifndef PCWD_H
#define PCWD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PCWD_OK = 0,
  PCWD_E_SHAPE = 1,   /* d ∉ {1,2}, n not a power of two, n < 2  */
  PCWD_E_CONFIG = 2,  /* levels ∉ [1, log2 n], filter length odd / < 2 / > 20  */
  PCWD_E_PARAM = 3,   /* NULL pointer, m < 1, τ ≤ 0, L < 1 or L > N, rank ∉ [0, world) */
  PCWD_E_CUDA = 4,    /* a CUDA runtime call failed (message: pcwd_last_error)        */
  PCWD_E_OOM = 5,     /* device allocation failed                                     */
  PCWD_E_STATE = 6,   /* call order violated (e.g. CSR requested before decompose)    */
  PCWD_E_UNSUPPORTED = 7
} pcwd_status;

typedef enum { PCWD_F32 = 0, PCWD_F64 = 1 } pcwd_dtype;

typedef enum {
  PCWD_RETAIN_FULL = 0,       /* every (μ, λ): dense rows of length N, exact zeros kept (R14) */
  PCWD_RETAIN_THRESHOLD = 1,  /* |Θ[μ][λ]| ≥ tau_rel · max|Θ|, decided in fp64 (R15)           */
  PCWD_RETAIN_BAND = 2,       /* exactly band_L partners per unit, scale/position key (R16)    */
  PCWD_RETAIN_PATTERN = 3     /* the caller's retained set: pat_rowptr / pat_col, a CSR over units (the
                                 A_L pattern of Theorem 2's Remark, or any Θ_L of Eq. 7,
                                 P:858-863); exact zeros kept (R14)                                   */
} pcwd_retain;

typedef struct {
  int32_t d;            /* dimension, 1 or 2  */
  int32_t n;            /* side of the torus, power of two; N = n^d.  The paper's grid is
                           N_1 × … × N_d; the method is stated and analysed for
                           N_1 = … = N_d = 2^J ("to simplify the discussion"), which is
                           what this library implements: a single side n for every axis      */
  int32_t levels;       /* J = number of analysis steps, 1 ≤ J ≤ log2 n              (R3)    */
  int32_t filter_len;   /* 2δ, even, 2..20  */
  const double* h;      /* HOST, filter_len taps of the low-pass filter; g from P:100        */
  int32_t m;            /* number of product-convolution terms, ≥ 1  */
  const double* u;      /* host or device, m × N row-major fp64: u_k(z) at index z mod n     */
  const double* v;      /* host or device, m × N row-major fp64: v_k(y)                      */
  int32_t dtype;        /* pcwd_dtype: arithmetic and output precision (threshold rule always
                           decides and computes in fp64, values stored in dtype; R15)         */
  int32_t retain;       /* pcwd_retain                                                        */
  double tau_rel;       /* THRESHOLD: relative threshold τ_rel > 0                            */
  int32_t band_L;       /* BAND: partners per unit, 1 ≤ L ≤ N                                 */
  int32_t rank, world;  /* shard of units owned by this handle; world ≥ 1                    */
  int32_t device;       /* CUDA device ordinal used by create                                */
  const int64_t* pat_rowptr; /* PATTERN: host or device, N + 1 entries over ALL units (Λ order),
                           pat_rowptr[0] = 0, non-decreasing; a sharded handle reads its rows   */
  const int32_t* pat_col;    /* PATTERN: host or device, pat_rowptr[N] partner indices λ ∈ [0, N),
                           strictly increasing within each row (the CSR column order).  Checked
                           by pcwd_create (PCWD_E_PARAM); copied, the caller keeps ownership    */
} pcwd_desc;

typedef struct {
  int64_t n_rows;       /* units in this shard (= row1 - row0)                                */
  int64_t row0;         /* first global unit (Λ index) of the shard                           */
  int64_t nnz;          /* retained entries in this shard                                      */
  const int64_t* row_ptr;  /* DEVICE, n_rows + 1, row_ptr[0] = 0                              */
  const int32_t* col;      /* DEVICE, nnz global λ indices, strictly increasing within a row */
  const void* val;         /* DEVICE, nnz values of type dtype                                */
  int32_t dtype;
} pcwd_csr;

typedef struct {
  int64_t N, row0, row1, nnz;
  double global_max;        /* THRESHOLD: M = max|Θ| used for τ (fp64); else 0               */
  double fma_algorithmic;   /* algorithmic FMAs of one decompose over this shard */
  double bytes_algorithmic; /* algorithmic HBM bytes (inputs + templates + CSR output)       */
  int32_t kernel_launches;  /* kernels launched by the last pcwd_decompose                   */
  int32_t compute_dtype;    /* precision the path computed in                                */
} pcwd_info_t;

/* Validate desc and build the handle: plan (sub-band table, windows, band stencil, shard),
 * device buffers, copy of u and v cast to the compute precision.  Caller keeps ownership of
 * every pointer in desc and may free them when this returns.  Synchronous.
 * The low-pass filter h must be an orthogonal wavelet filter: ‖h‖₂ = 1, Σ h = √2 and
 * Σ_n h[n] h[n + 2k] = 0 for k ≠ 0, each to 1e-9; otherwise PCWD_E_CONFIG (Ψ would
 * not be orthogonal and Θ = Ψ*HΨ would not be the operator's representation).
 * PATTERN: pat_rowptr / pat_col are checked (monotone, in range, strictly increasing rows) and
 * copied; a violation is PCWD_E_PARAM. */
int pcwd_create(const pcwd_desc* desc, void** out_handle);

/* Compute the retained rows of this shard into handle-owned CSR (templates, k-sum, cascade,
 * retention, compaction — all on the GPU).  Enqueued on `stream`.  THRESHOLD with world > 1
 * needs the global max first: call pcwd_local_max, reduce over ranks, pcwd_set_global_max.
 * The CSR stays valid until the next decompose or destroy.  Returns when the work is
 * enqueued (THRESHOLD mode synchronises the stream once, to size the CSR). */
int pcwd_decompose(void* handle, void* stream);

/* THRESHOLD only: max|Θ[μ][·]| over this shard's units (fp64, synchronous). */
int pcwd_local_max(void* handle, void* stream, double* out_max);
/* THRESHOLD only: set M (e.g. the MAX all-reduce of pcwd_local_max over ranks). */
int pcwd_set_global_max(void* handle, double M);

/* Describe the CSR of the last decompose (device pointers owned by the handle). */
int pcwd_get_csr(void* handle, pcwd_csr* out);
/* Copy the CSR into caller buffers (host or device; sizes from pcwd_get_csr).  Any pointer
 * may be NULL to skip that array.  Enqueued on stream. */
int pcwd_copy_csr(void* handle, int64_t* row_ptr, int32_t* col, void* val, void* stream);

/* Replace the operator's kernels (u_k, v_k of H f = Σ_k u_k ⋆ (v_k ⊙ f)) on an existing
 * handle, keeping its plan (sub-band table, windows, stencil, shard, launch plan, buffers): the
 * "plan once, decompose many operators" use.  u, v: m·N fp64 each, layout as in pcwd_desc, host
 * (pinned for asynchronous copies) or device pointers; the caller keeps ownership.  The union of
 * supp u_k must lie inside the periodic bounding box of the u given to pcwd_create (the windows
 * of the plan are derived from it): checked on the GPU, PCWD_E_PARAM otherwise (the
 * handle then keeps its previous kernels).  Invalidates the last decompose.  Enqueued on stream,
 * then synchronises it once for the support check; BAND: v is then copied on an internal stream while
 * the templates of the new u are built on `stream` (the next decompose uses them instead of building
 * them), and both are synchronised before return, so u and v may be released on return. */
int pcwd_set_kernels(void* handle, const double* u, const double* v, void* stream);

/* The periodic bounding box of supp u_k the plan was built from (the windows of the plan follow
 * from it): per axis a start offset lo[a] (in [0, n)) and a width w[a] (1 ≤ w[a] ≤ n), axis 0 = rows
 * (d = 1: lo[0] = 0, w[0] = 1).  Host only; never fails on a valid handle. */
int pcwd_kernel_box(void* handle, int32_t lo[2], int32_t w[2]);

/* pcwd_set_kernels with u_k given on that box only (the compact impulse responses of P:234-246 are
 * naturally stored this way): u_box = m × w[0] × w[1] fp64, row-major, entry (k, i0, i1) = u_k at grid
 * point ((lo[0] + i0) mod n, (lo[1] + i1) mod n); u_k is zero elsewhere by construction, so there is no
 * support check and no synchronisation before the template build.  v, streams, synchronisation on
 * return and invalidation as pcwd_set_kernels; host (pinned) or device pointers, caller keeps ownership. */
int pcwd_set_kernels_box(void* handle, const double* u_box, const double* v, void* stream);

/* pcwd_decompose followed by the copy of the CSR into caller buffers (as pcwd_copy_csr; NULL
 * skips an array), with the copies overlapped with the computation: BAND and FULL rows have a
 * fixed width, so each launch's rows are copied (on a second stream, event-ordered) as soon as
 * that launch has finished, the largest level first.  THRESHOLD: decompose, then copy.  Enqueued
 * on `stream`: the host buffers are complete once `stream` has been synchronised.  Host buffers
 * should be pinned (pageable memory serialises the copies). */
int pcwd_decompose_to_host(void* handle, int64_t* row_ptr, int32_t* col, void* val, void* stream);

/* y = Θ_ret x (transpose = 0: x has N entries, y has n_rows) or y = Θ_retᵀ x (transpose = 1:
 * x has n_rows entries, y has N, overwritten).  x, y: DEVICE arrays of type dtype.
 * This is the Θ_L z product of Eq. (7).  Both are gathers (warp per row) in a fixed order:
 * the transposed product runs on a transposed copy of the CSR (columns' entries in increasing row
 * order; nnz·(4 + dtype size) bytes plus sort scratch), built by the first transposed call after each
 * decompose.  Enqueued on stream. */
int pcwd_apply(void* handle, const void* x, void* y, int transpose, void* stream);

/* ---- consumer of the decomposition ------------------------------------ */

/* Periodic orthogonal wavelet transform on the handle's grid, basis and depth:
 * inverse = 0: out = Ψ* in (coefficients in Λ order, the order of Θ's rows and columns);
 * inverse = 1: out = Ψ in.  in, out: DEVICE arrays of N values of the handle's dtype, not aliased.
 * Enqueued on stream (uses handle-owned scratch: one transform or FISTA per handle at a time). */
int pcwd_wavelet_transform(void* handle, const void* in, void* out, int inverse, void* stream);

/* FISTA in the wavelet domain on the decomposed Θ_L:
 *   z^(i) = Prox^Σ_{‖·‖_{1,w}}(y^(i) − τ Σ Θ_Lᵀ(Θ_L y^(i) − z0)),  y^(i+1) = z^(i) + (i−1)/(i+2)(z^(i) − z^(i−1)),
 * z^(0) = y^(1) = 0, for i = 1..iters.  precond = 0: Σ = I (FISTA-W); 1: Σ = diag(Θ_LᵀΘ_L)⁻¹ (FISTA-WP, Jacobi;
 * reading R-F1 of DESIGN.md).  Prox^Σ is the soft threshold at τ Σ_λλ w[λ].  *tau > 0 is used as the step;
 * *tau ≤ 0 computes τ = 0.99 / ‖Σ^½ Θ_LᵀΘ_L Σ^½‖₂ (power iteration until ‖M v‖ changes by < 1e-6 over 8
 * steps, at most 100) and returns it in *tau (this synchronises the stream every 8 power steps).  z0 (= Ψ* f0),
 * w (weights ≥ 0), z_out (= z^(iters)): DEVICE arrays of N values of the handle's dtype.  Needs a decompose first
 * and the whole Θ on this handle (a sharded Θ: pcwd_fista_sharded).  Θᵀ products are gathers over a transposed
 * copy of the CSR (built once per decompose, as for pcwd_apply with transpose = 1); the Jacobi diagonal and the
 * power-iteration norms accumulate in fp64 in a fixed order (the same bits on every run). */
int pcwd_fista(void* handle, const void* z0, const void* w, int iters, int precond, double* tau, void* z_out,
               void* stream);

/* FISTA over a row-sharded Θ_L (one handle per rank): the same iteration as pcwd_fista,
 * with Θ_L y computed on the handle's rows only and the gradient Θ_Lᵀ r = Σ_ranks Θ_rᵀ r_r summed by the caller:
 * after writing its partial into xg (DEVICE, N values of the handle's dtype) the library calls reduce(0, ctx),
 * which must replace xg by the sum over the ranks, ordered on `stream` (e.g. an NCCL all-reduce on that stream),
 * and return 0; with precond = 1 the Jacobi diagonal's partial column sums (DEVICE, N fp64 in xd) are summed the
 * same way once, by reduce(1, ctx).  z0 and w are the whole N-vectors (replicated); every rank computes the same
 * z_out and τ (the norms of the power iteration are summed in a fixed order, so all ranks stop it together).
 * A nonzero return of reduce stops the call with PCWD_E_PARAM.  The callback runs on the calling thread. */
typedef int (*pcwd_reduce_fn)(int which, void* ctx);
int pcwd_fista_sharded(void* handle, const void* z0, const void* w, int iters, int precond, double* tau, void* z_out,
                       pcwd_reduce_fn reduce, void* ctx, void* xg, double* xd, void* stream);

/* ---- Algorithm 1 proper: the η-approximation --------------------------------------- */

typedef enum {
  PCWD_TRUNC_INDEX = 0,     /* Theorem 2's Remark: drop |ℓ_λ − ℓ_μ| > S or ϑ(λ,μ) > 2^S (Definition 1)   */
  PCWD_TRUNC_MAGNITUDE = 1  /* "simply threshold A": keep |A_k[μ][ν]| ≥ 2^{−(S+1)} (power-of-two steps)  */
} pcwd_trunc_rule;

typedef struct {
  double eta;             /* the requested precision η                                                    */
  int32_t m;
  int32_t S[64];          /* per k: truncation index S_k of Ã_k (−1: Ã_k = 0); the rule's parameter        */
  double eps[64];         /* per k: ε_k = η / (m ‖v_k‖∞)    */
  double bound[64];       /* per k: Schur bound sqrt(‖E‖₁‖E‖_∞) ≥ ‖A_k − Ã_k‖₂ of the dropped part E       */
  int64_t nnz;            /* nonzeros of Θ̃                                                                 */
} pcwd_approx_info;

/* Algorithm 1: Θ̃ = Σ_k Ã_k B_k, an η-approximation of Θ (‖Θ − Θ̃‖₂ ≤ η), into the
 * handle's CSR (Θ̃ on its predicted support, columns increasing; replaces the last decompose — pcwd_get_csr,
 * pcwd_apply and pcwd_fista then work on Θ̃).  A_k = Ψ*U_kΨ, B_k = Ψ*V_kΨ; Ã_k is A_k truncated by `rule`
 * (pcwd_trunc_rule: the Remark's index rule, or power-of-two magnitude thresholds) with the smallest index S_k
 * whose dropped part has Schur bound sqrt(‖E‖₁‖E‖_∞) ≤ ε_k = η/(m‖v_k‖∞) (DESIGN.md R-A1..R-A4), so that
 * ‖A_k − Ã_k‖₂ ≤ ε_k.  η > 0 and rule ∈ {0, 1} (PCWD_E_PARAM).  Needs dtype F64 (the
 * paper's precision; PCWD_E_UNSUPPORTED otherwise), world = 1 and m ≤ 64 (PCWD_E_STATE /
 * PCWD_E_UNSUPPORTED); whole-torus transforms per class of units, so meant for N ≤ 512² (the paper's η sweep is
 * at 256²).  out (may be NULL) receives the per-k truncation.  Synchronous. */
int pcwd_approx(void* handle, double eta, int rule, void* stream, pcwd_approx_info* out);

/* y = H x (adjoint = 0) or y = H* x (adjoint = 1) on the handle's grid: H f = Σ_k u_k ⋆ (v_k ⊙ f) (Eq. 2,
 * P:29-32) by direct sums over the support box of the u_k.  x, y: DEVICE arrays of N values of the handle's dtype,
 * not aliased.  With pcwd_wavelet_transform this applies Θ = Ψ*HΨ to a vector (e.g. to measure ‖Θ − Θ̃‖₂).
 * Enqueued on stream. */
int pcwd_operator_apply(void* handle, const void* x, void* y, int adjoint, void* stream);

/* Algorithm 2's column orientation (ledger C1): for each λ of `lambdas` (host or
 * device, count Λ indices) the whole column Θ[·][λ] = Ψ*(H ψ_λ), w_λ = H ψ_λ = Σ_k u_k ⋆ (v_k ⊙ ψ_λ) by direct
 * sums over supp ψ_λ ⊕ supp u, then the whole-torus cascade.  out: DEVICE, count × N fp64 (row i = column λ_i).
 * About m·|supp u| / (window) times the row path's work per unit (SURVEY §0 finding 2); meant for columns on
 * demand and the C1 cross-check.  Synchronous. */
int pcwd_columns(void* handle, const int64_t* lambdas, int64_t count, double* out, void* stream);

/* The d = 3 variant (the grid is N_1 × … × N_d): rows of Θ = Ψ* H Ψ on the
 * periodic n × n × n grid, Θ[μ][·] = Ψ*(H* ψ_μ), H f = Σ_k u_k ⋆ (v_k ⊙ f) (R9), in the separable basis of
 * P:110-119 with axis 0 filtered first, then axis 1, then axis 2.  Λ layout: the (n >> levels)³ coarse block, then
 * levels J..1, orientations e = 4 e0 + 2 e1 + e2 = 1..7, positions row-major.  A handle-free call: n a power of two
 * ≤ 256; h: HOST, `taps` values of an orthogonal low-pass filter (else PCWD_E_CONFIG); u, v: DEVICE, m × n³ fp64,
 * u_k(z) at index z mod n, row-major (z0, z1, z2); units: HOST or DEVICE, `count` Λ indices in [0, n³) (else
 * PCWD_E_PARAM); out: DEVICE, count × n³ fp64 allocated by the caller (row i = row units[i] of Θ).  Computes in fp64,
 * each pass only on the product set of per-axis supports its result can be nonzero on (exact zeros elsewhere);
 * allocates and frees its scratch (≤ 4 GiB, else PCWD_E_OOM); synchronous. */
int pcwd_rows3d(int32_t n, int32_t levels, const double* h, int32_t taps, int32_t m, const double* u, const double* v,
                const int64_t* units, int64_t count, double* out, void* stream);

/* ---- constructing the product-convolution expansion (§3.3) ------------------
 * Both factor impulse responses given on the window [−R, R]^d around the origin (W = (2R+1)^d values per response,
 * row-major over the offsets (z0, z1) = (a − R, b − R); 2R + 1 ≤ n): u_k = the m leading left singular vectors of
 * the W × s matrix of responses (uncentred PCA, R10; sign: largest-|entry| positive), found on the GPU by
 * subspace iteration from a seeded Gaussian block with CholeskyQR2 re-orthonormalisation and a Rayleigh–Ritz step
 * (Jacobi).  Outputs: u (m × N, u_k(z) stored at index z mod n, taps that wrap accumulate) and v (m × N), both
 * DEVICE arrays allocated by the caller — they can be passed straight to pcwd_create / pcwd_set_kernels — and
 * sigma (HOST, m singular values).  Inputs host or device.  m + oversample ≤ 32.  Synchronous. */

/* §3.3.2: responses sampled at the g^d cell centres y_i = (n/g)(i + ½) (reading R11), irs = g^d × W
 * (sample-major, row-major grid); v_k = periodic bilinear interpolation of the projections <S(·, y_i), u_k>
 * between the cell centres (R12); g = n: one response per pixel, v_k(y) = the projection itself. */
int pcwd_pc_from_samples(int32_t d, int32_t n, int32_t R, int32_t g, int32_t m, const double* irs, double* u,
                         double* v, double* sigma, void* stream);
/* §3.3.3: randomized SVD of the space-varying impulse response S given at every pixel: svir = N × W
 * (row y = S(·, y) on the window), `oversample` extra columns, `power_iters` subspace iterations, `seed` of the
 * counter-based Gaussian start; v_k(y) = <S(·, y), u_k> (so Σ_k u_k v_kᵀ is the rank-m truncated SVD, the
 * Frobenius-optimal product-convolution expansion of P:241). */
int pcwd_pc_from_svir(int32_t d, int32_t n, int32_t R, int32_t m, const double* svir, int32_t oversample,
                      int32_t power_iters, uint64_t seed, double* u, double* v, double* sigma, void* stream);

int pcwd_info(void* handle, pcwd_info_t* out);

/* Phase timing with CUDA events recorded on the decompose stream around each phase
 * (enable = 1 before pcwd_decompose; read after the stream is synchronised).  enable = 2 also serialises the
 * unit-kernel launches (no concurrent coarse streams) so that pcwd_launch_profile reports each kernel's own
 * duration rather than overlapping stream spans.
 * Phases: 0 = templates (a1), 1 = unit kernels (a2+a3+a4), 2 = everything else (fills, scans,
 * threshold max/count passes).  out_ms[3] receives milliseconds of the last decompose;
 * out_fma[3] the algorithmic FMAs of phases 0 and 1 (phase 2: 0). */
int pcwd_profile(void* handle, int enable);
/* Per unit-kernel launch of the last decompose (profiling enabled): *count = launches; for the first
 * `max` of them, out_ms = duration (CUDA events on the decompose stream), out_fma = algorithmic FMAs of
 * the units it processed, out_kind = 0 generic / 1 tile / 2 fine / 3 batched (coarse),
 * out_level = wavelet level ℓ of its units.  Any output pointer may be NULL.  Synchronous. */
int pcwd_launch_profile(void* handle, int max, int* count, double* out_ms, double* out_fma, int* out_kind,
                        int* out_level);
int pcwd_phase_times(void* handle, double* out_ms, double* out_fma);
int pcwd_destroy(void* handle);

const char* pcwd_error_string(int code);
/* Last error message of this thread (CUDA detail, failing argument). */
const char* pcwd_last_error(void);

/* ---- host-only plan queries (no GPU needed; used by the CPU tests) ---------------------- */
int pcwd_validate(const pcwd_desc* desc);
/* Shard [row0, row1) that (desc->rank, desc->world) would own. */
int pcwd_plan_shard(const pcwd_desc* desc, int64_t* row0, int64_t* row1);
/* BAND: the stencil of unit sub-band `sb` (Λ order index): band_L entries of
 * (partner sub-band, offset o0, offset o1) in key order.  u and v may be NULL. */
int pcwd_plan_stencil(const pcwd_desc* desc, int32_t sb, int32_t* out_sb, int32_t* out_o0,
                      int32_t* out_o1);
/* Number of sub-bands of the Λ layout. */
int pcwd_plan_num_subbands(const pcwd_desc* desc, int32_t* out);
/* Host only.  The 1-D analysis atom of the separable fine path (reading R-S1; the analysis step of
 * P:96 iterated): W_{s,e}(y) for y = *out_start + i, i < *out_len, i.e. the level-s coefficient of
 * orientation e (0 = scaling, 1 = wavelet) at position 0 on the integer line is Σ_y x(y) W_{s,e}(y); the atom of
 * position l is W_{s,e}(y − 2^s l).  desc supplies the filter (validated like pcwd_create; u, v may be NULL).
 * out: caller-owned host array of cap doubles (may be NULL to query the length).  1 ≤ s ≤ 16, e ∈ {0, 1};
 * PCWD_E_PARAM on a bad argument or cap < length. */
int pcwd_plan_atom(const pcwd_desc* desc, int32_t s, int32_t e, double* out, int32_t cap, int32_t* out_len,
                   int32_t* out_start);

#ifdef __cplusplus
}
#endif
#endif /* PCWD_H */
