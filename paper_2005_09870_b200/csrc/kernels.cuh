// kernels.cuh — launch interface of the sm_100a kernels (implemented in kernels.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.h"
#include "geom.h"

namespace pcwd {

struct UnitArgs {
  const void* v;            // compute type, m × N
  const void* T;            // compute type, templates
  const int4* stencil;      // BAND: (sb, o0, o1, -)
  void* gscratch;           // compute type, per-CTA slices (global-scratch launches)
  int64_t gscratch_stride;  // elements per CTA slice
  int64_t u0, u1;           // global unit range of this launch
  int64_t row0;             // first unit of the shard (local row = unit - row0)
  const int64_t* row_ptr;   // TWRITE
  int32_t* col;
  void* val;                // output type
  double* unitmax;          // TMAX: per local row
  int32_t* cnt;             // TCOUNT / TWRITE: [row][sb]
  double tau;               // threshold (fp64)
  int use_smem;
  int hybrid;               // global-scratch launch with the step ≥ 2 buffers in shared memory (SubBand::hs_*)
  double* cand;             // TSTORE: every structural partner value of the unit, window by window in column order
  int dbg;                  // timing experiments only (PCWD_UNIT_DBG, results invalid): 1 = no k-sum, 2 = no candidate stores
};

struct TileArgs {
  const void* v;
  const void* T;
  const int4* stencil;
  const int4* box;          // nsb × nsb stencil offset boxes
  int64_t u0, u1;           // unit range (one level, whole rounds of G units)
  int64_t row0;
  int32_t* col;
  void* val;
  int G;                    // units per round
  int XS, YS;               // row strides of X and Yt (elements)
  int XR, YR;               // max rows of X and Yt
  int DMAX;                 // D buffer elements per unit
  int per_unit;             // (unused by the kernel)
  int Xsz, Ysz, Dsz;        // per-unit region sizes (elements)
  int64_t regY, regD, regEnd;  // region offsets of the CTA scratch layout (elements)
  int TS, VS, RC;           // k-sum staging: T / v tile row strides, rows per chunk
  unsigned long long* dbg;  // optional per-phase clock counters (PCWD_DEBUG_PHASES)
};

cudaError_t launch_band_tile(const Plan& P, const TileArgs& A, int real_bytes, int grid, size_t smem,
                             cudaStream_t st);

struct FGeom;
struct SepClass;
struct SepRun;
struct SepPart;

struct FineArgs {
  CUtensorMap tmV;          // TMA map of the periodically padded v (3-D: x, y, k), box VS × R0 × 1
  CUtensorMap tmT[3];       // TMA maps of the templates of the level's sub-bands (x, y, k), box TS × R0 × 1
  int vpad;                 // halo width P of the padded v (v_pad[y + P][x + P] = v[y mod n][x mod n])
  int sb_first;             // first sub-band of the launch (tmT index = sbi - sb_first)
  int TSZ, VSZ;             // staged T / v tile sizes (elements, multiples of 128 bytes)
  const void* v;
  const void* T;
  const int4* stencil;      // .w = level of the partner sub-band
  const FGeom* geom;        // class geometry records (plan), indexed by SubBand::fg_off
  int64_t u0, u1;           // unit range (one level, whole rounds of GU units)
  int64_t row0;
  int32_t* col;
  void* val;
  int64_t regS, regD;       // region offsets (elements): staging / Yt, D
  int RS, RSZ;              // R / approximation row stride, per-unit R region size
  int TS, VS;               // staged T row stride, staged v row stride
  int YS, YSZ;              // Yt row stride, per-slot Yt size (step 1, CG slots)
  int YS2, YSZ2;            // Yt row stride and per-unit size for steps ≥ 2 and the gather stage (GU units)
  int DS;                   // per-unit D size
  int nst;                  // staging buffers used (1 ≤ nst ≤ the kernel's NST)
  int direct;               // partner levels (0, 1 or 2, the coarsest ones) computed directly in the gather
  unsigned long long* dbg;  // optional phase clock counters (PCWD_DEBUG_PHASES): k-sum, cascade
  int dbg_flags;            // debug experiments (PCWD_FINE_DBG, results invalid): 2 = no cascade, 4 = step 1 only
  // separable direct a3 + a4 (geom.h "sep"; sep = 0: the cascade)
  int sep;
  int QS, QSZ;              // Q row stride, Q region size (elements); the gather stage follows Q in the slot
  const SepClass* sepc;     // indexed like geom
  const SepRun* seprun;
  const SepPart* seppart;
  const int* septask;
  const void* atoms;        // atom tap table (compute type, geom.h sep_toff layout), copied to shared memory
  int64_t regA;             // its shared-memory offset (elements; beyond everything the staging ring may use)
  int ntap;                 // its size (elements)
};

// Template configuration of the fine kernel for (real_bytes, level): units per round GU, template
// columns per thread GZ, tasks per thread NT, staging buffers NST, concurrent cascades CG (fine.cu).
struct FineCfg {
  int GU, GZ, NT, NST, CG;   // CG: units whose cascades run concurrently (256 / CG threads each)
};
bool fine_config(int real_bytes, int level, int L2, FineCfg* cfg);
cudaError_t launch_fine(const Plan& P, const FineArgs& A, int real_bytes, int level, int grid, size_t smem,
                        cudaStream_t st);

// Tiled k-sum (bk_ksum_tma): a tile row of Q0 column groups of width SH = 2^ℓ is staged as NB TMA boxes of
// SH·q columns (≤ 256 elements per box dimension); q is odd for SH ≤ 16 so that the rows a warp reads fall
// in distinct bank groups.
constexpr int kt_box_q(int SH, int Q0, int nb) {
  int q = (Q0 + nb - 1) / nb;
  if (SH <= 16 && q % 2 == 0) ++q;
  return q;
}
constexpr int kt_box_n(int SH, int Q0) {
  int nb = 1;
  while (SH * kt_box_q(SH, Q0, nb) > 256) ++nb;
  return nb;
}
constexpr int kt_units(int real_bytes) { return real_bytes == 4 ? 8 : 4; }   // G: units per tiled k-sum group
// A TMA box must start on a 16-byte boundary.  The periodic extension of v is built with a column offset
// (kt_offx) that puts every strip start of the levels ≥ 2 on one (their starts are ≡ −zhi mod 4), so a
// v box covers SH·q columns plus kt_vpadx columns of bank padding: SH for SH ≤ 16 with q even (fp32: a
// warp reads 32/SH rows, a row pitch ≡ SH mod 2SH keeps them in distinct banks), else none.
constexpr int kt_vpadx(int SH, int rb) { return rb == 8 ? 0 : (SH <= 16 ? SH : 0); }
constexpr int kt_vbox_q(int SH, int Q0, int nb, int rb) {
  int q = (Q0 + nb - 1) / nb;
  if (rb == 4 && SH <= 16 && q % 2 == 1) ++q;
  return q;
}
constexpr int kt_vbox_n(int SH, int Q0, int rb) {
  int nb = 1;
  while (SH * kt_vbox_q(SH, Q0, nb, rb) + kt_vpadx(SH, rb) > 256) ++nb;
  return nb;
}

struct BatchArgs {
  CUtensorMap tmV;          // tiled k-sum: TMA map of v (3-D: x, y, k), box (SH·qV + kt_vpadx) × TR × 1
  CUtensorMap tmT[4];       // tiled k-sum: TMA maps of the level's templates, box SH·qT × TR × 1 (whole-torus
                            // k-sum: box 256 × kf_rows × 1, one per sub-band of the level incl. the coarse block)
  int kf_rows;              // whole-torus k-sum with TMA (bk_ksum_full_tma): rows per thread; 0 = not planned
  int kt_gz;                // tiled k-sum: template column groups per thread (0 ⇒ not planned)
  int kt_sb_first;          // tiled k-sum: sub-band of tmT[0]
  int kt_flags;             // tiled k-sum debug: 1 = v strips by cp.async only
  int kt_vh, kt_vw;         // tiled k-sum: rows / columns of the periodically extended v that tmV maps
  int kt_offx;              // its column offset: v_wrap[y][x] = v[y mod n][(x − kt_offx) mod n]
  const CUtensorMap* amaps; // approximation steps: device array [step - 1][sub-band - kt_sb_first] of TMA maps
  unsigned am_steps;        // bit s: step s of every sub-band of the launch has a map (bk_approx_tma)
  int tail_s0;              // first step run by bk_tail (per-unit, shared memory); 0 = none
  const void* v;
  const void* T;
  const int4* stencil;      // .w = level of the partner sub-band
  void* scratch;            // batch × stride elements (generic per-unit layout of SubBand)
  int64_t stride;
  int64_t u0, u1;           // unit range of this launch (one level)
  int64_t batch;            // units per batch
  int64_t row0;
  int32_t* col;
  void* val;
};

// Template column groups per thread (GZ) of the tiled k-sum for the batched launch over [u0, u1), 0 when the
// tiled k-sum does not apply (host; api.cu encodes the TMA maps from it).
int ksum_tiled_gz(const Plan& P, int64_t u0, int64_t u1, int real_bytes);
// Tile side / input box of bk_approx_tma (TO outputs, TI × BW input box) for the compute type.
constexpr int ap_to(int rb) { return rb == 4 ? 32 : 16; }
constexpr int ap_ti(int rb, int L2) { return 2 * (ap_to(rb) - 1) + L2; }
constexpr int ap_bw(int rb, int L2) { return (ap_ti(rb, L2) + 16 / rb - 1 + 16 / rb - 1) / (16 / rb) * (16 / rb); }

// FISTA-W / FISTA-WP on a single-shard CSR Θ (fista.cu).  All arrays device, N entries of the compute type
// unless noted; dbuf: N + 1 doubles.
struct FistaArgs {
  int64_t N, nnz;
  const int64_t* row_ptr;
  const int32_t* col;
  const void* val;
  const int64_t* row_ptrT;   // Θᵀ as CSR over the columns (rows of Θ ascending in every column)
  const int32_t* rowT;
  const void* valT;
  const void* z0;     // Ψ* f0
  const void* w;      // ℓ1 weights w[λ]
  void *y, *zprev, *r, *g, *sigma, *sqrt_sigma, *z_out;
  double* D;          // Jacobi diagonal (N, fp64)
  double* dbuf;       // norm (1) + per-block partial sums (kFistaParts)
  int iters, precond, power_iters;
  int64_t rows, row0;                    // the handle's rows of Θ (rows = N, row0 = 0: the whole Θ)
  int (*reduce)(int which, void* ctx);   // sharded Θ: sum g (which = 0) / D (which = 1) over the ranks, in place,
  void* rctx;                            // ordered on the stream; null: the whole Θ is on this handle
};
constexpr int kFistaParts = 4096;        // ≥ the element-wise kernels' grid (grid_of in fista.cu)
// cb_failed: set when the reduce callback returned nonzero (the launch then stops and returns cudaErrorUnknown)
cudaError_t launch_fista(const Plan& P, const FistaArgs& F, int rb, cudaStream_t st, double* tau_io, int* cb_failed);
// Ψ* (inverse = 0) or Ψ (inverse = 1) of one length-N array on the plan's grid; work0/1: N elements each.
cudaError_t launch_wavelet_transform(const Plan& P, const void* in, void* out, void* work0, void* work1, int inverse,
                                     int rb, cudaStream_t st);

// Algorithm 1 (approx.cu): classes = (sub-band, position mod 2^{J−ℓ}), ordered by sub-band (clsbase[s] = first
// class of sub-band s).  Scratch per CTA: (5 + m) N doubles.
struct ApproxArgs {
  const double* T;          // templates (fp64)
  const double* v;          // m × N (fp64)
  double* scratch;
  int64_t cstride;          // doubles per CTA
  int64_t ncls;
  int64_t clsbase[kMaxSB + 1];
  int S[64];                // truncation index per k (−1: Ã_k = 0)
  int rule;                 // 0: Remark (i)/(ii) index rule; 1: magnitude, |a| ≥ 2^{-(S+1)}
  double* rowhist;          // stats: ncls × m × bins
  double* colhist;          // stats: ncls × m × bins (zeroed by the caller)
  int64_t* cnt;             // count pass: per unit
  const int64_t* row_ptr;   // write pass
  int32_t* col;
  void* val;
};
int approx_block();
int approx_bins();
cudaError_t launch_approx_stats(const Plan& P, const ApproxArgs& A, int grid, cudaStream_t st);
cudaError_t launch_approx_rows(const Plan& P, const ApproxArgs& A, int write, int out_bytes, int grid, cudaStream_t st);
// Algorithm 2's columns Θ[·][λ] = Ψ*(H ψ_λ) for count indices lam (device), out: count × N fp64; scratch per CTA
// cstride ≥ (3 + m) N doubles.
cudaError_t launch_columns(const Plan& P, const double* u, const void* v, const int64_t* lam, int64_t count,
                           double* scratch, int64_t cstride, int grid, double* out, int real_bytes, cudaStream_t st);
// y = H f or H* f on the plan's grid (direct sums over the planned box of supp u_k); f, out: N of the compute type.
cudaError_t launch_operator(const Plan& P, const double* u, const void* v, const void* f, void* out, int adjoint,
                            int real_bytes, cudaStream_t st);

cudaError_t launch_band_batched(const Plan& P, const BatchArgs& A, int real_bytes, int64_t maxX0, const int64_t* workA,
                                const int64_t* workB, const int64_t* appr0, const int64_t* appr1, int steps,
                                cudaStream_t st, int* launches);

struct TmplArgs {
  const double* phi_in;     // m × Win0 × Win1 (fp64)
  double* Y;                // m × 2 × Win0 × Wout1
  double* phi_out;          // m × Wout0 × Wout1
  void* T;                  // compute type templates
  int Sin[2], Win[2];       // input window per axis (W == n ⇒ whole line)
  int Sout[2][2], Wout[2];  // output window per axis and orientation
  int dil;                  // 2^{ℓ-1}
  int64_t toff[4];          // destination offset per orientation code (-1 = not stored)
  int64_t tstride;          // per-k stride of the destination sub-band templates
  int trs;                  // row stride of the destination templates
};

// dtype-dispatching launchers; return cudaError_t of the launch
cudaError_t launch_phi0(const Plan& P, const double* u, double* phi0, int S0, int W0, int S1, int W1,
                        cudaStream_t st);
cudaError_t launch_tmpl_level(const Plan& P, const TmplArgs& A, int real_bytes, int coarse_level,
                              cudaStream_t st);
cudaError_t launch_cast(const double* src, void* dst, int64_t count, int real_bytes, cudaStream_t st);
cudaError_t launch_box_scatter(const double* ub, int m, int n, int d, const int zlo[2], const int zhi[2], double* u,
                               cudaStream_t st);
cudaError_t launch_support_check(const double* u, int64_t total, int n, int d, const int zlo[2], const int zhi[2],
                                 int* flag, cudaStream_t st);
// K1: v_pad[k][y][x] = v[k][(y - P) mod n][(x - P) mod n], side n + 2P (compute type)
cudaError_t launch_pad_v(const void* v, void* vpad, int n, int P, int m, int real_bytes, cudaStream_t st);
// out[k][y][x] = v[k][(y - offy) mod n][(x - offx) mod n] for y < H, x < W (offsets ≤ 4n; n a power of two).
cudaError_t launch_wrap_v(const void* v, void* out, int n, int offy, int offx, int H, int W, int m, int real_bytes,
                          cudaStream_t st);
cudaError_t launch_units(const Plan& P, const UnitArgs& A, int mode, int real_bytes, int out_bytes,
                         int grid, size_t smem, cudaStream_t st);
size_t unit_smem_limit();
cudaError_t set_unit_smem_attr(size_t bytes);
cudaError_t launch_fill_band_rowptr(int64_t* row_ptr, int64_t rows, int64_t L, cudaStream_t st);
cudaError_t launch_fill_full(int64_t* row_ptr, int32_t* col, int64_t rows, int64_t N, cudaStream_t st);
// THRESHOLD store-then-filter: per unit of the shard, count / write the candidates ≥ tau stored by MODE_TSTORE.
// THRESHOLD, fp32 values: count + in-place compaction of the kept candidates (one read), then the copy into the CSR
cudaError_t launch_cand_compact(const Plan& P, double* cand, int64_t row0, int64_t rows, double tau, int32_t* cnt,
                                cudaStream_t st);
cudaError_t launch_cand_copy(const Plan& P, const double* cand, int64_t row0, int64_t rows, const int32_t* cnt,
                             const int64_t* row_ptr, int32_t* col, float* val, cudaStream_t st);
cudaError_t launch_cand_filter(const Plan& P, const double* cand, int64_t row0, int64_t rows, double tau, int write,
                               int32_t* cnt, const int64_t* row_ptr, int32_t* col, void* val, int out_bytes,
                               cudaStream_t st);
cudaError_t launch_row_counts(const int32_t* cnt, int64_t rows, int nsb, int64_t* rowcnt, cudaStream_t st);
cudaError_t launch_max_reduce(const double* x, int64_t n, double* out, cudaStream_t st);
cudaError_t launch_spmv(const int64_t* row_ptr, const int32_t* col, const void* val, const void* x,
                        void* y, int64_t rows, int64_t N, int transpose, int bytes, cudaStream_t st);
// Θᵀ of a CSR (rows × ncols) as CSR over the columns, entries of each column in increasing row order (deterministic).
size_t csr_transpose_bytes(int64_t nnz, int64_t ncols, int vbytes);
cudaError_t csr_transpose(const int64_t* rp, const int32_t* col, const void* val, int64_t rows, int64_t nnz,
                          int64_t ncols, int vbytes, int64_t* rpT, int32_t* rowT, void* valT, void* work,
                          size_t work_bytes, cudaStream_t st);
cudaError_t exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, void* tmp, size_t* tmp_bytes,
                               cudaStream_t st);

}  // namespace pcwd

// pca.cu: factorisation of impulse-response rows X (s × W, device) — see the file header.
namespace pcwd_pca {
int factor(const double* X, int64_t s, int W, int m, int oversample, int power_iters, uint64_t seed, double* U,
           double* c, double* sigma, cudaStream_t st);
int finish(const double* U, const double* c, int d, int n, int R, int g, int m, double* u, double* v, cudaStream_t st);
}  // namespace pcwd_pca

// volume.cu: the d = 3 variant — rows of Θ on the n³ torus (see the file header).  Returns a cudaError_t as int.
namespace pcwd_vol {
int rows3d(int n, int J, const double* h, int taps, int m, const double* u, const double* v, const int64_t* units,
           const int64_t* order, const int64_t* sorted_mu, int64_t count, double* out, cudaStream_t st);
}  // namespace pcwd_vol
