// kernels.cu — sm_100a kernels of the exact decomposition path.
//
//   a1  tmpl_*      T_{k,s} = ũ_k ⋆ ψ_{s,0} by the à-trous recursion (P:96 applied to ũ_k ⋆ φ):
//                   T_φ^{(ℓ)}(y) = Σ_j f_0[j] T_φ^{(ℓ-1)}(y - 2^{ℓ-1} j), detail templates with f_1;
//                   these are the spatial form of A_k's circulant sub-band generators (Lemma 1,
//                   P:1157-1159).  fp64.
//   a2  unit_kernel k-sum       R_μ(y) = Σ_k v_k(y) T_{k,s(μ)}(y - 2^ℓ p)   (B_k and A_kB_k of Alg. 1,
//                   P:186-190, fused with the accumulation: Row μ of Σ_k A_k B_k is Ψ*(Σ_k v_k ⊙ τT_k))
//   a3  unit_kernel cascade     c_μ = Ψ* R_μ on the windows R_μ can reach (sparse cascade,
//                   P:1266-1273, Lemma 6)
//   a4/a5 unit_kernel emit      retained gather: full rows / band stencil / threshold max-count-write
//
// One CTA processes one unit at a time (grid-stride over units in Λ order, coarse and costly
// first); its windows live in shared memory when they fit, else in a per-CTA global slice.
#include <mutex>
#include <cub/cub.cuh>

#include <algorithm>
#include <type_traits>
#include <climits>

#include "kernels.cuh"

namespace pcwd {

constexpr int kBlock = 256;
constexpr int kUB = 128;   // threads per CTA of the generic unit kernel (one unit per CTA; more CTAs per SM hide its barrier chain)

__device__ __forceinline__ float fmaT(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fmaT(double a, double b, double c) { return fma(a, b, c); }

// ============================================================================= templates (a1)

__global__ void phi0_kernel(const __grid_constant__ Plan P, const double* __restrict__ u,
                            double* __restrict__ phi0, int S0, int W0, int S1, int W1) {
  const int mask = P.n - 1;
  const int64_t total = int64_t(P.m) * W0 * W1;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    int64_t k = idx / (int64_t(W0) * W1);
    int64_t r = idx - k * W0 * W1;
    int i0 = int(r / W1), i1 = int(r - int64_t(i0) * W1);
    int z0 = P.d == 2 ? ((-(S0 + i0)) & mask) : 0;   // ũ(y) = u(-y)
    int z1 = (-(S1 + i1)) & mask;
    phi0[idx] = u[k * P.N + int64_t(z0) * P.n + z1];
  }
}

__device__ __forceinline__ double win_read(const double* buf, int y, int S, int W, int mask, int64_t stride) {
  int li = (y - S) & mask;
  return li < W ? buf[li * stride] : 0.0;
}

// One à-trous step of the template recursion along one axis, QT outputs per thread: the outputs at positions
// y, y + dil, …, y + (QT-1)·dil of one line share all but one input each (the filter is dilated by dil), so
// a thread reads QT + 2δ - 1 inputs for QT·2δ FMAs (fp64).
constexpr int QT = 8;

template <typename Real, int L2>
__global__ void tmpl_passA(const __grid_constant__ Plan P, const __grid_constant__ TmplArgs A, int coarse_level,
                           int level) {
  // along axis 1: Y[k][e1][i0][j1] = Σ_t f_{e1}[t] φ(i0, y1 - dil (o_{e1} + t)),  y1 = Sout[e1] + j1
  const int mask = P.n - 1, dil = A.dil;
  const int Win0 = A.Win[0], Win1 = A.Win[1], Wout1 = A.Wout[1];
  const int ngr = (Wout1 + dil * QT - 1) / (dil * QT);   // groups of QT outputs per residue
  const int64_t total = int64_t(P.m) * 2 * Win0 * dil * ngr;
  // index decomposition in 32 bits (the grids of every plan this library accepts stay below 2^31 threads)
  for (unsigned idx = blockIdx.x * blockDim.x + threadIdx.x; idx < unsigned(total); idx += gridDim.x * blockDim.x) {
    const int r = int(idx % unsigned(dil));
    unsigned t = idx / unsigned(dil);
    const int g = int(t % unsigned(ngr));
    t /= unsigned(ngr);
    const int i0 = int(t % unsigned(Win0));
    t /= unsigned(Win0);
    const int e1 = int(t & 1);
    const int64_t k = t >> 1;
    const int o = e1 ? 2 - L2 : 0;
    const double* line = A.phi_in + (k * Win0 + i0) * Win1;
    const int ybase = A.Sout[1][e1] + r + dil * (QT * g - o - (L2 - 1));
    double in[QT + L2 - 1];
#pragma unroll
    for (int i = 0; i < QT + L2 - 1; ++i) in[i] = win_read(line, (ybase + dil * i) & mask, A.Sin[1], Win1, mask, 1);
#pragma unroll
    for (int q = 0; q < QT; ++q) {
      const int j1 = r + dil * (QT * g + q);
      if (j1 >= Wout1) break;
      double acc = 0.0;
#pragma unroll
      for (int tt = 0; tt < L2; ++tt) acc = fma(P.td[e1][tt], in[q + (L2 - 1) - tt], acc);
      if (P.d == 2) {
        A.Y[((k * 2 + e1) * Win0 + i0) * Wout1 + j1] = acc;
      } else {  // d = 1: this is the output
        Real* T = reinterpret_cast<Real*>(A.T);
        if (e1 == 0) {
          A.phi_out[k * Wout1 + j1] = acc;
          if (level == coarse_level && A.toff[0] >= 0) T[A.toff[0] + k * A.tstride + j1] = Real(acc);
        } else if (A.toff[1] >= 0) {
          T[A.toff[1] + k * A.tstride + j1] = Real(acc);
        }
      }
    }
  }
}

template <typename Real, int L2>
__global__ void tmpl_passB(const __grid_constant__ Plan P, const __grid_constant__ TmplArgs A, int coarse_level,
                           int level) {
  // along axis 0, d = 2 only: out[k][e0 e1][j0][j1] = Σ_t f_{e0}[t] Y[k][e1](y0 - dil (o_{e0} + t), j1)
  const int mask = P.n - 1, dil = A.dil;
  const int Win0 = A.Win[0], Wout0 = A.Wout[0], Wout1 = A.Wout[1];
  const int ngr = (Wout0 + dil * QT - 1) / (dil * QT);
  const int64_t per = int64_t(Wout0) * Wout1;
  const int64_t total = int64_t(P.m) * 4 * dil * ngr * Wout1;
  Real* T = reinterpret_cast<Real*>(A.T);
  for (unsigned idx = blockIdx.x * blockDim.x + threadIdx.x; idx < unsigned(total); idx += gridDim.x * blockDim.x) {
    const int j1 = int(idx % unsigned(Wout1));
    unsigned t = idx / unsigned(Wout1);
    const int r = int(t % unsigned(dil));
    t /= unsigned(dil);
    const int g = int(t % unsigned(ngr));
    t /= unsigned(ngr);
    const int ec = int(t & 3);
    const int64_t k = t >> 2;
    const int e0 = ec >> 1, e1 = ec & 1;
    const int o = e0 ? 2 - L2 : 0;
    const double* col = A.Y + ((k * 2 + e1) * Win0) * Wout1 + j1;
    const int ybase = A.Sout[0][e0] + r + dil * (QT * g - o - (L2 - 1));
    double in[QT + L2 - 1];
#pragma unroll
    for (int i = 0; i < QT + L2 - 1; ++i) in[i] = win_read(col, (ybase + dil * i) & mask, A.Sin[0], Win0, mask, Wout1);
#pragma unroll
    for (int q = 0; q < QT; ++q) {
      const int j0 = r + dil * (QT * g + q);
      if (j0 >= Wout0) break;
      double acc = 0.0;
#pragma unroll
      for (int tt = 0; tt < L2; ++tt) acc = fma(P.td[e0][tt], in[q + (L2 - 1) - tt], acc);
      const int64_t rr = int64_t(j0) * Wout1 + j1;
      if (ec == 0) {
        A.phi_out[k * per + rr] = acc;
        if (level == coarse_level && A.toff[0] >= 0) T[A.toff[0] + k * A.tstride + int64_t(j0) * A.trs + j1] = Real(acc);
      } else if (A.toff[ec] >= 0) {
        T[A.toff[ec] + k * A.tstride + int64_t(j0) * A.trs + j1] = Real(acc);
      }
    }
  }
}

// Periodic extension of v: out[k][y][x] = v[k][(y - offy) mod n][(x - offx) mod n], y < H, x < W (row pitch W).
// Grid (ceil(W / 256), H, m): one thread per output element, coalesced along x.
template <typename Real>
__global__ void wrap_v_kernel(const Real* __restrict__ v, Real* __restrict__ out, int n, int offy, int offx, int H, int W) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y, k = blockIdx.z;
  if (x >= W) return;
  const int sy = (y - offy + n * 4) & (n - 1), sx = (x - offx + n * 4) & (n - 1);
  out[(int64_t(k) * H + y) * W + x] = v[(int64_t(k) * n + sy) * n + sx];
}

template <typename Real>
__global__ void cast_kernel(const double* __restrict__ src, Real* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = Real(src[i]);
}

// ============================================================================= per-unit kernel (a2-a5)

template <typename Real>
struct OutWin {
  const Real* buf;
  Range r0, r1;
  int sbi;
};

template <int NT = kUB>   // NT: threads of the calling CTA (the unit kernel's kUB, or kBlock)
__device__ __forceinline__ double block_reduce_max(double x, double* red) {
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    double y = threadIdx.x < NT / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) y = fmax(y, __shfl_xor_sync(0xffffffffu, y, o));
    if (threadIdx.x == 0) red[0] = y;
  }
  __syncthreads();
  return red[0];
}

template <int NT = kUB>
__device__ __forceinline__ int block_reduce_sum(int x, int* red) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    int y = threadIdx.x < NT / 32 ? red[threadIdx.x] : 0;
    for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
    if (threadIdx.x == 0) red[0] = y;
  }
  __syncthreads();
  return red[0];
}

template <int NT = kUB>
__device__ __forceinline__ int block_reduce_maxi(int x, int* red) {
  for (int o = 16; o > 0; o >>= 1) x = max(x, __shfl_xor_sync(0xffffffffu, x, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    int y = threadIdx.x < NT / 32 ? red[threadIdx.x] : 0;
    for (int o = 16; o > 0; o >>= 1) y = max(y, __shfl_xor_sync(0xffffffffu, y, o));
    if (threadIdx.x == 0) red[0] = y;
  }
  __syncthreads();
  return red[0];
}

// a / b for a ≥ 0, b ≥ 1: through a float reciprocal below 2^20 (the +0.5 keeps the truncation exact), else integer
__device__ __forceinline__ int qdiv(int a, int b, float inv_b) {
  return a < (1 << 20) ? __float2int_rz((float(a) + 0.5f) * inv_b) : a / b;
}

// ---- register-blocked cascade passes of the generic kernel (2-D, windows that do not wrap or cover the line) ----
// A task computes 8 consecutive outputs of one filter from one run of 14 + 2δ inputs held in registers (the
// outputs at 2j + t share all but two inputs): 14 + 2δ loads and one bounds test each for 8·2δ FMAs, instead of
// 2δ loads, tests and index computations per output.  TL2 = 2δ is a compile-time constant (taps from the
// kernel-parameter bank by compile-time index).  mode 0: window clear of wrapping (signed offset, zero outside);
// mode 1: whole periodic line (index mod the line); mode 2: a window whose taps can wrap onto it (local index
// mod the line, zero outside the window: local_index per input).
constexpr int kNQ = 4;   // outputs per task (4: the kernel keeps ≤ 80 registers, 3 CTAs per SM)

template <typename Real, int TL2>
__device__ __forceinline__ void run_load(const Real* __restrict__ base, int64_t stride, int q0, const Range& in, int mode,
                                         Real x[2 * kNQ - 2 + TL2]) {
  if (mode == 0) {
    int dq = (q0 - in.lo) & (in.nl - 1);
    if (dq >= in.nl - 2 * TL2) dq -= in.nl;
#pragma unroll
    for (int i = 0; i < 2 * kNQ - 2 + TL2; ++i)
      x[i] = unsigned(dq + i) < unsigned(in.len) ? base[int64_t(dq + i) * stride] : Real(0);
  } else if (mode == 1) {
#pragma unroll
    for (int i = 0; i < 2 * kNQ - 2 + TL2; ++i) x[i] = base[int64_t((q0 + i - in.lo) & (in.nl - 1)) * stride];
  } else {
#pragma unroll
    for (int i = 0; i < 2 * kNQ - 2 + TL2; ++i) {
      const int li = (q0 + i - in.lo) & (in.nl - 1);
      x[i] = li < in.len ? base[int64_t(li) * stride] : Real(0);
    }
  }
}

template <typename Real, int TL2>
__device__ void pass_a_blk(const Plan& P, const Real* __restrict__ cur, Real* __restrict__ Y, const Range& in0,
                           const Range& in1, const Range& a1, const Range& d1, int mode) {
  const int ycols = a1.len + d1.len;
  const int ga = (a1.len + kNQ - 1) / kNQ, gd = (d1.len + kNQ - 1) / kNQ;
  const int tot = in0.len * (ga + gd);
  const float inv = 1.0f / float(in0.len);
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    const int g = qdiv(idx, in0.len, inv), i0 = idx - g * in0.len;   // consecutive threads: consecutive rows
    const int e1 = g >= ga;
    const int j0 = kNQ * (e1 ? g - ga : g);
    const Range& R = e1 ? d1 : a1;
    Real x[2 * kNQ - 2 + TL2];
    run_load<Real, TL2>(cur + int64_t(i0) * in1.len, 1, 2 * (R.lo + j0) + P.to[e1], in1, mode, x);
    Real* out = Y + int64_t(i0) * ycols + (e1 ? a1.len : 0);
#pragma unroll
    for (int q = 0; q < kNQ; ++q) {
      Real acc = Real(0);
#pragma unroll
      for (int t = 0; t < TL2; ++t) acc = fmaT(TapsOf<Real>::get(P, e1, t), x[2 * q + t], acc);
      if (j0 + q < R.len) out[j0 + q] = acc;
    }
  }
}

template <typename Real, int TL2>
__device__ void pass_b_blk(const Plan& P, const Real* __restrict__ Y, Real* __restrict__ nxt, Real* __restrict__ Dd,
                           const Range& in0, const Range& a0, const Range& d0, const Range& a1, const Range& d1,
                           int mode) {
  const int ycols = a1.len + d1.len;
  const int s01 = a0.len * d1.len, s10 = d0.len * a1.len;
  const int ga = (a0.len + kNQ - 1) / kNQ, gd = (d0.len + kNQ - 1) / kNQ;
  const int tot = ycols * (ga + gd);
  const float inv = 1.0f / float(ycols);
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    const int g = qdiv(idx, ycols, inv), colY = idx - g * ycols;     // consecutive threads: consecutive columns
    const int e0 = g >= ga;
    const int j0 = kNQ * (e0 ? g - ga : g);
    const Range& R = e0 ? d0 : a0;
    Real x[2 * kNQ - 2 + TL2];
    run_load<Real, TL2>(Y + colY, ycols, 2 * (R.lo + j0) + P.to[e0], in0, mode, x);
    const int e1 = colY >= a1.len;
    const int j1 = e1 ? colY - a1.len : colY;
    const int w1 = e1 ? d1.len : a1.len;
    Real* out = e0 == 0 ? (e1 ? Dd : nxt) : (e1 ? Dd + s01 + s10 : Dd + s01);
#pragma unroll
    for (int q = 0; q < kNQ; ++q) {
      Real acc = Real(0);
#pragma unroll
      for (int t = 0; t < TL2; ++t) acc = fmaT(TapsOf<Real>::get(P, e0, t), x[2 * q + t], acc);
      if (j0 + q < R.len) out[(j0 + q) * w1 + j1] = acc;
    }
  }
}

// dispatch on 2δ (the Daubechies / Symmlet lengths of the configurations); false: use the per-output loops
template <typename Real>
__device__ __forceinline__ bool pass_a_dispatch(const Plan& P, const Real* cur, Real* Y, const Range& in0, const Range& in1,
                                                const Range& a1, const Range& d1, int mode) {
  switch (P.L2) {
    case 2: pass_a_blk<Real, 2>(P, cur, Y, in0, in1, a1, d1, mode); return true;
    case 4: pass_a_blk<Real, 4>(P, cur, Y, in0, in1, a1, d1, mode); return true;
    case 8: pass_a_blk<Real, 8>(P, cur, Y, in0, in1, a1, d1, mode); return true;
    case 12: pass_a_blk<Real, 12>(P, cur, Y, in0, in1, a1, d1, mode); return true;
  }
  return false;
}
template <typename Real>
__device__ __forceinline__ bool pass_b_dispatch(const Plan& P, const Real* Y, Real* nxt, Real* Dd, const Range& in0,
                                                const Range& a0, const Range& d0, const Range& a1, const Range& d1,
                                                int mode) {
  switch (P.L2) {
    case 2: pass_b_blk<Real, 2>(P, Y, nxt, Dd, in0, a0, d0, a1, d1, mode); return true;
    case 4: pass_b_blk<Real, 4>(P, Y, nxt, Dd, in0, a0, d0, a1, d1, mode); return true;
    case 8: pass_b_blk<Real, 8>(P, Y, nxt, Dd, in0, a0, d0, a1, d1, mode); return true;
    case 12: pass_b_blk<Real, 12>(P, Y, nxt, Dd, in0, a0, d0, a1, d1, mode); return true;
  }
  return false;
}

template <typename Real, typename OutT, int D, int MODE, int NT>
__global__ void __launch_bounds__(NT, NT == 128 ? 6 : 3) unit_kernel(const __grid_constant__ Plan P,
                                                      const __grid_constant__ UnitArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red_d[NT / 32];
  __shared__ int red_i[NT / 32];
  using BlockScan = cub::BlockScan<int, NT>;
  __shared__ typename BlockScan::TempStorage scan_tmp;

  Real* scratch = A.use_smem ? reinterpret_cast<Real*>(smem_raw)
                             : reinterpret_cast<Real*>(A.gscratch) + int64_t(blockIdx.x) * A.gscratch_stride;
  const int tid = threadIdx.x;
  const int n = P.n, mask = P.n - 1, L2 = P.L2;
  const Real* __restrict__ v = reinterpret_cast<const Real*>(A.v);

  for (int64_t unit = A.u0 + blockIdx.x; unit < A.u1; unit += gridDim.x) {
    const int sbi = find_subband(P, unit);
    const SubBand& S = P.sb[sbi];
    const int64_t row = unit - A.row0;
    const int64_t pos = unit - S.offset;
    const int p0 = D == 2 ? int(pos / S.nl) : 0;
    const int p1 = D == 2 ? int(pos - int64_t(p0) * S.nl) : int(pos);
    const Range r0 = D == 2 ? unit_window(P, S, 0, p0) : Range{0, 1, 1};
    const Range r1 = unit_window(P, S, 1, p1);
    Real* X0 = scratch + S.offX0;
    Real* hs = reinterpret_cast<Real*>(smem_raw);   // hybrid: shared-memory buffers of steps ≥ 2
    Real* X1 = A.hybrid ? hs + S.hs_X1 : scratch + S.offX1;
    Real* Y = scratch + S.offY;
    Real* Dd = scratch + S.offD;
    Real* stage_val = scratch + S.offStage;
    int* stage_col = reinterpret_cast<int*>(stage_val + P.band_Lpad);

    // ---- a2: R_μ(y) = Σ_k v_k(y) T_k(y - 2^ℓ p) on the unit window
    {
      const Real* __restrict__ T = reinterpret_cast<const Real*>(A.T) + S.toff;
      const bool f0 = D == 2 && S.tW[0] >= n;
      const bool f1 = S.tW[1] >= n;
      const int tw1 = S.tRS;
      const int total = r0.len * r1.len;
      const float inv_r1 = 1.0f / float(r1.len);
      for (int idx = tid; idx < total; idx += NT) {
        const int i0 = qdiv(idx, r1.len, inv_r1), i1 = idx - i0 * r1.len;
        const int y0 = D == 2 ? ((r0.lo + i0) & mask) : 0;
        const int y1 = (r1.lo + i1) & mask;
        const int t0 = f0 ? ((y0 - (p0 << S.level)) & mask) : i0;
        const int t1 = f1 ? ((y1 - (p1 << S.level)) & mask) : i1;
        const int64_t vy = int64_t(y0) * n + y1;
        const int64_t ti = int64_t(t0) * tw1 + t1;
        Real acc = Real(0);
        if (!(A.dbg & 1))
          for (int k = 0; k < P.m; ++k) acc = fmaT(v[k * P.N + vy], T[k * S.tstride + ti], acc);
        X0[idx] = acc;
      }
    }
    if (MODE == MODE_BAND) {
      for (int j = tid; j < P.band_Lpad; j += NT) { stage_col[j] = INT_MAX; stage_val[j] = Real(0); }
    }
    // PATTERN: the cascade runs up to the coarsest level among the unit's listed partners
    int nsteps = S.steps;
    if (A.dbg >> 4) nsteps = min(nsteps, A.dbg >> 4);   // timing experiment (PCWD_UNIT_DBG = 16·s): stop after step s
    if (MODE == MODE_PATTERN) {
      int mx = 0;
      for (int64_t j = A.row_ptr[row] + tid; j < A.row_ptr[row + 1]; j += NT) mx = max(mx, P.sb[find_subband(P, A.col[j])].level);
      nsteps = block_reduce_maxi<NT>(mx, red_i);
    }
    __syncthreads();

    // ---- a3: windowed periodic cascade, steps 1..S.steps, emitting after each step
    Real* cur = X0;
    Real* nxt = X1;
    Range in0 = r0, in1 = r1;
    double tmax = 0.0;
    int64_t crun = 0;   // TSTORE: candidates of this unit stored so far
    double* cbase = nullptr;
    if (MODE == MODE_TSTORE) cbase = A.cand + S.cand_off + (unit - (S.offset > A.row0 ? S.offset : A.row0)) * S.cand_slot;
    for (int s = 1; s <= nsteps; ++s) {
      const Range a0 = D == 2 ? step_out(in0, L2, 0) : Range{0, 1, 1};
      const Range d0 = D == 2 ? step_out(in0, L2, 1) : Range{0, 1, 1};
      const Range a1 = step_out(in1, L2, 0);
      const Range d1 = step_out(in1, L2, 1);
      int s01 = 0, s10 = 0;
      // window addressing: a window clear of wrapping (len + 2·2δ ≤ line) by a signed offset from its start, a
      // whole-line window modulo the line, otherwise local_index per tap
      auto kind = [&](const Range& r) { return r.len >= r.nl ? 1 : (r.len + 2 * L2 <= r.nl ? 0 : 2); };
      auto sdiff = [&](int g, const Range& r) {
        int dd = (g - r.lo) & (r.nl - 1);
        return dd >= r.nl - 2 * L2 ? dd - r.nl : dd;
      };
      if (D == 2) {
        const int ycols = a1.len + d1.len;
        const int totA = in0.len * ycols;
        const float inv_y = 1.0f / float(ycols), inv_a1 = 1.0f / float(a1.len), inv_d1 = 1.0f / float(d1.len);
        const int k1 = kind(in1);
        const bool blkA = pass_a_dispatch<Real>(P, cur, Y, in0, in1, a1, d1, k1);
        for (int idx = blkA ? totA : tid; idx < totA; idx += NT) {       // pass A: axis 1
          const int i0 = qdiv(idx, ycols, inv_y), j = idx - i0 * ycols;
          const int e1 = j >= a1.len;
          const int jj = e1 ? j - a1.len : j;
          const Range& R = e1 ? d1 : a1;
          const int q = 2 * (R.lo + jj) + P.to[e1];
          const Real* line = cur + i0 * in1.len;
          Real acc = Real(0);
          if (k1 == 0) {
            const int dq = sdiff(q, in1);
#pragma unroll 4
            for (int t = 0; t < L2; ++t)
              if (unsigned(dq + t) < unsigned(in1.len)) acc = fmaT(TapsOf<Real>::get(P, e1, t), line[dq + t], acc);
          } else if (k1 == 1) {
#pragma unroll 4
            for (int t = 0; t < L2; ++t)
              acc = fmaT(TapsOf<Real>::get(P, e1, t), line[(q + t - in1.lo) & (in1.nl - 1)], acc);
          } else {
#pragma unroll 4
            for (int t = 0; t < L2; ++t) {
              const int c = local_index(in1, q + t);
              if (c >= 0) acc = fmaT(TapsOf<Real>::get(P, e1, t), line[c], acc);
            }
          }
          Y[idx] = acc;
        }
        __syncthreads();
        const int k0 = kind(in0);
        const int s00 = a0.len * a1.len;
        s01 = a0.len * d1.len;
        s10 = d0.len * a1.len;
        const int s11 = d0.len * d1.len;
        const int totB = s00 + s01 + s10 + s11;
        const bool blkB = pass_b_dispatch<Real>(P, Y, nxt, Dd, in0, a0, d0, a1, d1, k0);
        for (int idx = blkB ? totB : tid; idx < totB; idx += NT) {       // pass B: axis 0
          int e0, e1, j0, j1, rem;
          Real* dst;
          if (idx < s00) { e0 = 0; e1 = 0; rem = idx; j0 = qdiv(rem, a1.len, inv_a1); j1 = rem - j0 * a1.len; dst = nxt + rem; }
          else if (idx < s00 + s01) { e0 = 0; e1 = 1; rem = idx - s00; j0 = qdiv(rem, d1.len, inv_d1); j1 = rem - j0 * d1.len; dst = Dd + rem; }
          else if (idx < s00 + s01 + s10) { e0 = 1; e1 = 0; rem = idx - s00 - s01; j0 = qdiv(rem, a1.len, inv_a1); j1 = rem - j0 * a1.len; dst = Dd + s01 + rem; }
          else { e0 = 1; e1 = 1; rem = idx - s00 - s01 - s10; j0 = qdiv(rem, d1.len, inv_d1); j1 = rem - j0 * d1.len; dst = Dd + s01 + s10 + rem; }
          const Range& R = e0 ? d0 : a0;
          const int q = 2 * (R.lo + j0) + P.to[e0];
          const int colY = (e1 ? a1.len : 0) + j1;
          Real acc = Real(0);
          if (k0 == 0) {
            const int dq = sdiff(q, in0);
#pragma unroll 4
            for (int t = 0; t < L2; ++t)
              if (unsigned(dq + t) < unsigned(in0.len)) acc = fmaT(TapsOf<Real>::get(P, e0, t), Y[(dq + t) * ycols + colY], acc);
          } else if (k0 == 1) {
#pragma unroll 4
            for (int t = 0; t < L2; ++t)
              acc = fmaT(TapsOf<Real>::get(P, e0, t), Y[((q + t - in0.lo) & (in0.nl - 1)) * ycols + colY], acc);
          } else {
#pragma unroll 4
            for (int t = 0; t < L2; ++t) {
              const int r = local_index(in0, q + t);
              if (r >= 0) acc = fmaT(TapsOf<Real>::get(P, e0, t), Y[r * ycols + colY], acc);
            }
          }
          *dst = acc;
        }
      } else {
        const int tot = a1.len + d1.len;
        for (int idx = tid; idx < tot; idx += NT) {
          const int e1 = idx >= a1.len;
          const int jj = e1 ? idx - a1.len : idx;
          const Range& R = e1 ? d1 : a1;
          const int q = 2 * (R.lo + jj) + P.to[e1];
          Real acc = Real(0);
          for (int t = 0; t < L2; ++t) {
            const int c = local_index(in1, q + t);
            if (c >= 0) acc = fmaT(TapsOf<Real>::get(P, e1, t), cur[c], acc);
          }
          if (e1) Dd[jj] = acc; else nxt[jj] = acc;
        }
      }
      __syncthreads();

      // ---- a4/a5: emit this step's sub-bands (and the coarse block at s == J)
      OutWin<Real> w[4];
      int nw = 0;
      const int base_sb = 1 + (P.J - s) * (D == 2 ? 3 : 1);
      if (D == 2) {
        w[nw++] = OutWin<Real>{Dd, a0, d1, base_sb + 0};
        w[nw++] = OutWin<Real>{Dd + s01, d0, a1, base_sb + 1};
        w[nw++] = OutWin<Real>{Dd + s01 + s10, d0, d1, base_sb + 2};
      } else {
        w[nw++] = OutWin<Real>{Dd, Range{0, 1, 1}, d1, base_sb};
      }
      if (s == P.J) w[nw++] = OutWin<Real>{nxt, a0, a1, 0};

      if (MODE == MODE_FULL) {
        OutT* out = reinterpret_cast<OutT*>(A.val) + row * P.N;
        for (int wi = 0; wi < nw; ++wi) {
          const OutWin<Real>& W = w[wi];
          const SubBand& L = P.sb[W.sbi];
          const int tot = W.r0.len * W.r1.len;
          for (int idx = tid; idx < tot; idx += NT) {
            const int i0 = idx / W.r1.len, i1 = idx - i0 * W.r1.len;
            const int g0 = (W.r0.lo + i0) & (W.r0.nl - 1);
            const int g1 = (W.r1.lo + i1) & (W.r1.nl - 1);
            out[L.offset + int64_t(g0) * L.nl + g1] = OutT(W.buf[idx]);
          }
        }
      } else if (MODE == MODE_BAND) {
        const int4* st = A.stencil + S.stencil_off;
        for (int j = tid; j < P.band_L; j += NT) {
          const int4 e = st[j];
          const SubBand& L = P.sb[e.x];
          if (L.level != s || (e.x == 0 && s != P.J)) continue;
          const OutWin<Real>* W = nullptr;
          for (int wi = 0; wi < nw; ++wi) if (w[wi].sbi == e.x) W = &w[wi];
          // partner position: base from μ's position on λ's grid, plus the stencil offset
          int b0, b1;
          if (L.level == S.level) { b0 = p0; b1 = p1; }
          else if (L.level < S.level) { b0 = p0 << (S.level - L.level); b1 = p1 << (S.level - L.level); }
          else { b0 = p0 >> (L.level - S.level); b1 = p1 >> (L.level - S.level); }
          const int l0 = D == 2 ? ((b0 + e.y) & (L.nl - 1)) : 0;
          const int l1 = (b1 + e.z) & (L.nl - 1);
          Real x = Real(0);
          if (W) {
            const int li0 = local_index(W->r0, l0), li1 = local_index(W->r1, l1);
            if (li0 >= 0 && li1 >= 0) x = W->buf[li0 * W->r1.len + li1];
          }
          stage_val[j] = x;
          stage_col[j] = int(L.offset + int64_t(l0) * L.nl + l1);
        }
      } else if (MODE == MODE_PATTERN) {   // the caller's partners of this step's sub-bands (columns given)
        OutT* outv = reinterpret_cast<OutT*>(A.val);
        for (int64_t j = A.row_ptr[row] + tid; j < A.row_ptr[row + 1]; j += NT) {
          const int c = A.col[j];
          const int sb = find_subband(P, c);
          const SubBand& L = P.sb[sb];
          if (L.level != s || (sb == 0 && s != P.J)) continue;
          const OutWin<Real>* W = nullptr;
          for (int wi = 0; wi < nw; ++wi) if (w[wi].sbi == sb) W = &w[wi];
          const int64_t lp = c - L.offset;
          const int l0 = D == 2 ? int(lp / L.nl) : 0;
          const int l1 = D == 2 ? int(lp - int64_t(l0) * L.nl) : int(lp);
          Real x = Real(0);
          if (W) {
            const int li0 = local_index(W->r0, l0), li1 = local_index(W->r1, l1);
            if (li0 >= 0 && li1 >= 0) x = W->buf[li0 * W->r1.len + li1];
          }
          outv[j] = OutT(x);
        }
      } else if (MODE == MODE_TMAX) {
        for (int wi = 0; wi < nw; ++wi) {
          const int tot = w[wi].r0.len * w[wi].r1.len;
          for (int idx = tid; idx < tot; idx += NT) tmax = fmax(tmax, fabs(double(w[wi].buf[idx])));
        }
      } else if (MODE == MODE_TSTORE) {   // TMAX + every value stored in column (sorted) order
        for (int wi = 0; wi < nw; ++wi) {
          const OutWin<Real>& W = w[wi];
          const int tot = W.r0.len * W.r1.len;
          auto ident = [](const Range& r) { return r.len >= r.nl || (r.lo & (r.nl - 1)) + r.len <= r.nl; };
          if (ident(W.r0) && ident(W.r1)) {   // no wrap: the window's row-major order is the column order
            for (int k = tid; k < tot; k += NT) {
              const double x = double(W.buf[k]);
              tmax = fmax(tmax, fabs(x));
              if (!(A.dbg & 2)) cbase[crun + k] = x;
            }
          } else {
            const float inv_w = 1.0f / float(W.r1.len);
            for (int k = tid; k < tot; k += NT) {
              const int ks0 = qdiv(k, W.r1.len, inv_w), ks1 = k - ks0 * W.r1.len;
              const double x = double(W.buf[sorted_to_local(W.r0, ks0) * W.r1.len + sorted_to_local(W.r1, ks1)]);
              tmax = fmax(tmax, fabs(x));
              if (!(A.dbg & 2)) cbase[crun + k] = x;
            }
          }
          crun += tot;
        }
      } else if (MODE == MODE_TCOUNT) {
        for (int wi = 0; wi < nw; ++wi) {
          int c = 0;
          const int tot = w[wi].r0.len * w[wi].r1.len;
          for (int idx = tid; idx < tot; idx += NT) c += fabs(double(w[wi].buf[idx])) >= A.tau;
          c = block_reduce_sum<NT>(c, red_i);
          if (tid == 0) A.cnt[row * P.nsb + w[wi].sbi] = c;
        }
      } else if (MODE == MODE_TWRITE) {
        OutT* outv = reinterpret_cast<OutT*>(A.val);
        for (int wi = 0; wi < nw; ++wi) {
          const OutWin<Real>& W = w[wi];
          const SubBand& L = P.sb[W.sbi];
          int64_t base = A.row_ptr[row];
          for (int q = 0; q < W.sbi; ++q) base += A.cnt[row * P.nsb + q];
          const int tot = W.r0.len * W.r1.len;
          int running = 0;
          for (int k0 = 0; k0 < tot; k0 += NT) {
            const int k = k0 + tid;
            int keep = 0, colv = 0;
            Real x = Real(0);
            if (k < tot) {
              const int ks0 = k / W.r1.len, ks1 = k - ks0 * W.r1.len;      // sorted (global) order
              const int i0 = sorted_to_local(W.r0, ks0), i1 = sorted_to_local(W.r1, ks1);
              x = W.buf[i0 * W.r1.len + i1];
              keep = fabs(double(x)) >= A.tau;
              const int g0 = (W.r0.lo + i0) & (W.r0.nl - 1);
              const int g1 = (W.r1.lo + i1) & (W.r1.nl - 1);
              colv = int(L.offset + int64_t(g0) * L.nl + g1);
            }
            int posn, agg;
            BlockScan(scan_tmp).ExclusiveSum(keep, posn, agg);
            if (keep) {
              A.col[base + running + posn] = colv;
              outv[base + running + posn] = OutT(x);
            }
            running += agg;
            __syncthreads();
          }
        }
      }
      __syncthreads();
      Real* tswap = cur; cur = nxt; nxt = tswap;
      if (A.hybrid && s == 1) {   // steps ≥ 2 work in shared memory: approximations X1 / X2, Y, D
        nxt = hs + S.hs_X2;
        Y = hs + S.hs_Y;
        Dd = hs + S.hs_D;
      }
      in0 = a0;
      in1 = a1;
    }

    // ---- finalize the unit
    if (MODE == MODE_BAND) {
      const int Lp = P.band_Lpad;
      for (int k = 2; k <= Lp; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
          for (int i = tid; i < Lp; i += NT) {
            const int ixj = i ^ j;
            if (ixj > i) {
              const bool up = (i & k) == 0;
              const int ci = stage_col[i], cj = stage_col[ixj];
              if ((ci > cj) == up) {
                stage_col[i] = cj; stage_col[ixj] = ci;
                const Real vi = stage_val[i]; stage_val[i] = stage_val[ixj]; stage_val[ixj] = vi;
              }
            }
          }
          __syncthreads();
        }
      }
      OutT* outv = reinterpret_cast<OutT*>(A.val);
      const int64_t base = row * P.band_L;
      for (int j = tid; j < P.band_L; j += NT) {
        A.col[base + j] = stage_col[j];
        outv[base + j] = OutT(stage_val[j]);
      }
    } else if (MODE == MODE_TMAX || MODE == MODE_TSTORE) {
      const double mx = block_reduce_max<NT>(tmax, red_d);
      if (tid == 0) A.unitmax[row] = mx;
    }
    __syncthreads();
  }
}

// THRESHOLD store-then-filter: one warp per unit walks the unit's window chain (the emission order of unit_kernel)
// over the candidates MODE_TSTORE stored in column order; WRITE = 0 counts per (unit, sub-band) the values with
// |x| ≥ tau (cnt), WRITE = 1 compacts them into the CSR (row_ptr from the counts) with ballot / popc.
template <typename OutT, int D, int WRITE>
__global__ void __launch_bounds__(kBlock) cand_filter_kernel(const __grid_constant__ Plan P, const double* __restrict__ cand,
                                                             int64_t row0, int64_t rows, double tau, int32_t* cnt,
                                                             const int64_t* __restrict__ row_ptr, int32_t* col, OutT* val) {
  const int lane = threadIdx.x & 31, L2 = P.L2;
  const int64_t warp0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t row = warp0; row < rows; row += nwarps) {
    const int64_t unit = row0 + row;
    const int sbi = find_subband(P, unit);
    const SubBand& S = P.sb[sbi];
    const int64_t pos = unit - S.offset;
    const int p0 = D == 2 ? int(pos / S.nl) : 0;
    const int p1 = D == 2 ? int(pos - int64_t(p0) * S.nl) : int(pos);
    Range in0 = D == 2 ? unit_window(P, S, 0, p0) : Range{0, 1, 1};
    Range in1 = unit_window(P, S, 1, p1);
    const double* cb = cand + S.cand_off + (unit - (S.offset > row0 ? S.offset : row0)) * S.cand_slot;
    int64_t crun = 0;
    int64_t base = 0;
    if (WRITE) base = row_ptr[row];
    for (int s = 1; s <= S.steps; ++s) {
      const Range a0 = D == 2 ? step_out(in0, L2, 0) : Range{0, 1, 1};
      const Range d0 = D == 2 ? step_out(in0, L2, 1) : Range{0, 1, 1};
      const Range a1 = step_out(in1, L2, 0);
      const Range d1 = step_out(in1, L2, 1);
      Range wr0[4], wr1[4];
      int wsb[4], nw = 0;
      const int base_sb = 1 + (P.J - s) * (D == 2 ? 3 : 1);
      if (D == 2) {
        wr0[nw] = a0; wr1[nw] = d1; wsb[nw++] = base_sb + 0;
        wr0[nw] = d0; wr1[nw] = a1; wsb[nw++] = base_sb + 1;
        wr0[nw] = d0; wr1[nw] = d1; wsb[nw++] = base_sb + 2;
      } else {
        wr0[nw] = Range{0, 1, 1}; wr1[nw] = d1; wsb[nw++] = base_sb;
      }
      if (s == P.J) { wr0[nw] = a0; wr1[nw] = a1; wsb[nw++] = 0; }
      for (int wi = 0; wi < nw; ++wi) {
        const int tot = wr0[wi].len * wr1[wi].len;
        const double* cw = cb + crun;
        if (!WRITE) {
          int c = 0;
          for (int k = lane; k < tot; k += 32) c += fabs(cw[k]) >= tau;
          c = __reduce_add_sync(0xffffffffu, c);
          if (lane == 0) cnt[row * P.nsb + wsb[wi]] = c;
        } else {
          // the count pass gave this window's kept entries: skip windows with none, stop once all are written,
          // and compute the column index only for the kept lanes
          const int want = cnt[row * P.nsb + wsb[wi]];
          const SubBand& L = P.sb[wsb[wi]];
          int64_t b = base;
          if (want > 0)
            for (int q = 0; q < wsb[wi]; ++q) b += cnt[row * P.nsb + q];
          int running = 0;
          for (int k0 = 0; k0 < tot && running < want; k0 += 32) {
            const int k = k0 + lane;
            const double x = k < tot ? cw[k] : 0.0;
            const int keep = k < tot && fabs(x) >= tau;
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep) {
              const int ks0 = k / wr1[wi].len, ks1 = k - ks0 * wr1[wi].len;
              const int i0 = sorted_to_local(wr0[wi], ks0), i1 = sorted_to_local(wr1[wi], ks1);
              const int g0 = (wr0[wi].lo + i0) & (wr0[wi].nl - 1);
              const int g1 = (wr1[wi].lo + i1) & (wr1[wi].nl - 1);
              const int posn = __popc(m & lt);
              col[b + running + posn] = int(L.offset + int64_t(g0) * L.nl + g1);
              val[b + running + posn] = OutT(x);
            }
            running += __popc(m);
          }
        }
        crun += tot;
      }
      in0 = a0;
      in1 = a1;
    }
  }
}

// THRESHOLD, fp32 values: one read of the candidates instead of two.  cand_compact_kernel walks a unit's windows in
// emission order (as cand_filter_kernel), counts the kept entries per (unit, sub-band) into cnt and compacts them IN
// PLACE at the front of the unit's own candidate slot as (fp32 value bits | column << 32) — the write position never
// passes the read position, and a chunk's loads complete before its ballot; cand_copy_kernel then moves each
// sub-band's compacted run to its CSR position (row_ptr from the counts; sub-bands in Λ order = column order).
constexpr int kCU = 4;   // candidate chunks of 32 loaded ahead per warp in the compaction

template <int D>
__global__ void __launch_bounds__(kBlock) cand_compact_kernel(const __grid_constant__ Plan P, double* cand, int64_t row0,
                                                              int64_t rows, double tau, int32_t* cnt) {
  const int lane = threadIdx.x & 31, L2 = P.L2;
  const int64_t warp0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t row = warp0; row < rows; row += nwarps) {
    const int64_t unit = row0 + row;
    const int sbi = find_subband(P, unit);
    const SubBand& S = P.sb[sbi];
    const int64_t pos = unit - S.offset;
    const int p0 = D == 2 ? int(pos / S.nl) : 0;
    const int p1 = D == 2 ? int(pos - int64_t(p0) * S.nl) : int(pos);
    Range in0 = D == 2 ? unit_window(P, S, 0, p0) : Range{0, 1, 1};
    Range in1 = unit_window(P, S, 1, p1);
    double* cb = cand + S.cand_off + (unit - (S.offset > row0 ? S.offset : row0)) * S.cand_slot;
    unsigned long long* out = reinterpret_cast<unsigned long long*>(cb);
    int64_t crun = 0, wpos = 0;
    for (int s = 1; s <= S.steps; ++s) {
      const Range a0 = D == 2 ? step_out(in0, L2, 0) : Range{0, 1, 1};
      const Range d0 = D == 2 ? step_out(in0, L2, 1) : Range{0, 1, 1};
      const Range a1 = step_out(in1, L2, 0);
      const Range d1 = step_out(in1, L2, 1);
      Range wr0[4], wr1[4];
      int wsb[4], nw = 0;
      const int base_sb = 1 + (P.J - s) * (D == 2 ? 3 : 1);
      if (D == 2) {
        wr0[nw] = a0; wr1[nw] = d1; wsb[nw++] = base_sb + 0;
        wr0[nw] = d0; wr1[nw] = a1; wsb[nw++] = base_sb + 1;
        wr0[nw] = d0; wr1[nw] = d1; wsb[nw++] = base_sb + 2;
      } else {
        wr0[nw] = Range{0, 1, 1}; wr1[nw] = d1; wsb[nw++] = base_sb;
      }
      if (s == P.J) { wr0[nw] = a0; wr1[nw] = a1; wsb[nw++] = 0; }
      for (int wi = 0; wi < nw; ++wi) {
        const int tot = wr0[wi].len * wr1[wi].len;
        const double* cw = cb + crun;
        const SubBand& L = P.sb[wsb[wi]];
        int running = 0;
        const float inv_w = 1.0f / float(wr1[wi].len);
        for (int k0 = 0; k0 < tot; k0 += kCU * 32) {   // kCU loads in flight per lane before the first ballot
          double xs[kCU];
#pragma unroll
          for (int u = 0; u < kCU; ++u) {
            const int k = k0 + 32 * u + lane;
            xs[u] = k < tot ? cw[k] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < kCU; ++u) {
            const int k = k0 + 32 * u + lane;
            const int keep = k < tot && fabs(xs[u]) >= tau;
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep) {
              const int ks0 = qdiv(k, wr1[wi].len, inv_w), ks1 = k - ks0 * wr1[wi].len;
              const int i0 = sorted_to_local(wr0[wi], ks0), i1 = sorted_to_local(wr1[wi], ks1);
              const int g0 = (wr0[wi].lo + i0) & (wr0[wi].nl - 1);
              const int g1 = (wr1[wi].lo + i1) & (wr1[wi].nl - 1);
              const unsigned c = unsigned(L.offset + int64_t(g0) * L.nl + g1);
              out[wpos + running + __popc(m & lt)] =
                  (static_cast<unsigned long long>(c) << 32) | __float_as_uint(float(xs[u]));
            }
            running += __popc(m);
          }
        }
        if (lane == 0) cnt[row * P.nsb + wsb[wi]] = running;
        wpos += running;
        crun += tot;
      }
      in0 = a0;
      in1 = a1;
    }
  }
}

template <int D>
__global__ void __launch_bounds__(kBlock) cand_copy_kernel(const __grid_constant__ Plan P, const double* __restrict__ cand,
                                                           int64_t row0, int64_t rows, const int32_t* __restrict__ cnt,
                                                           const int64_t* __restrict__ row_ptr, int32_t* col,
                                                           float* val) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t row = warp0; row < rows; row += nwarps) {
    const int64_t unit = row0 + row;
    const SubBand& S = P.sb[find_subband(P, unit)];
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(
        cand + S.cand_off + (unit - (S.offset > row0 ? S.offset : row0)) * S.cand_slot);
    const int32_t* c = cnt + row * P.nsb;
    const int64_t base = row_ptr[row];
    int64_t spos = 0;
    for (int s = 1; s <= S.steps; ++s) {   // emission order of the compaction
      const int base_sb = 1 + (P.J - s) * (D == 2 ? 3 : 1);
      const int nw = (D == 2 ? 3 : 1) + (s == P.J);
      for (int wi = 0; wi < nw; ++wi) {
        const int sb = wi < (D == 2 ? 3 : 1) ? base_sb + wi : 0;
        const int want = c[sb];
        if (want > 0) {
          int64_t dst = base;
          for (int q = 0; q < sb; ++q) dst += c[q];
          for (int k = lane; k < want; k += 32) {
            const unsigned long long e = src[spos + k];
            col[dst + k] = int32_t(e >> 32);
            val[dst + k] = __uint_as_float(unsigned(e & 0xffffffffull));
          }
        }
        spos += want;
      }
    }
  }
}

// ============================================================================= small kernels

__global__ void fill_band_rowptr(int64_t* row_ptr, int64_t rows, int64_t L) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i <= rows; i += int64_t(gridDim.x) * blockDim.x)
    row_ptr[i] = i * L;
}

__global__ void fill_full(int64_t* row_ptr, int32_t* col, int64_t rows, int64_t N) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i <= rows; i += int64_t(gridDim.x) * blockDim.x)
    row_ptr[i] = i * N;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < rows * N; i += int64_t(gridDim.x) * blockDim.x)
    col[i] = int32_t(i % N);
}

__global__ void row_counts_kernel(const int32_t* cnt, int64_t rows, int nsb, int64_t* rowcnt) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r <= rows; r += int64_t(gridDim.x) * blockDim.x) {
    int64_t c = 0;
    if (r < rows) for (int s = 0; s < nsb; ++s) c += cnt[r * nsb + s];
    rowcnt[r] = c;
  }
}

__global__ void max_reduce_kernel(const double* x, int64_t n, unsigned long long* out) {
  __shared__ double red[kBlock / 32];
  double m = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    m = fmax(m, x[i]);
  m = block_reduce_max<kBlock>(m, red);
  if (threadIdx.x == 0) atomicMax(out, __double_as_longlong(m));   // m ≥ 0: bit order = value order
}

template <typename T>
__global__ void spmv_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                            const T* __restrict__ val, const T* __restrict__ x, T* __restrict__ y, int64_t rows) {
  const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  double acc = 0.0;
  for (int64_t j = rp[warp] + lane; j < rp[warp + 1]; j += 32) acc += double(val[j]) * double(x[col[j]]);
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) y[warp] = T(acc);
}

template <typename T>
__global__ void spmv_t_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                              const T* __restrict__ val, const T* __restrict__ x, T* __restrict__ y, int64_t rows) {
  const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const T xr = x[warp];
  for (int64_t j = rp[warp] + lane; j < rp[warp + 1]; j += 32) atomicAdd(&y[col[j]], val[j] * xr);
}

// ============================================================================= launchers

static int grid_for(int64_t n, int per = kBlock) {
  int64_t g = (n + per - 1) / per;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return int(g);
}

cudaError_t launch_phi0(const Plan& P, const double* u, double* phi0, int S0, int W0, int S1, int W1,
                        cudaStream_t st) {
  phi0_kernel<<<grid_for(int64_t(P.m) * W0 * W1), kBlock, 0, st>>>(P, u, phi0, S0, W0, S1, W1);
  return cudaGetLastError();
}

template <typename Real, int L2>
static cudaError_t launch_tmpl_t(const Plan& P, const TmplArgs& A, int level, cudaStream_t st) {
  const int64_t ngA = (A.Wout[1] + int64_t(A.dil) * QT - 1) / (int64_t(A.dil) * QT);
  const int64_t ngB = (A.Wout[0] + int64_t(A.dil) * QT - 1) / (int64_t(A.dil) * QT);
  const int64_t totA = int64_t(P.m) * 2 * A.Win[0] * A.dil * ngA;
  const int64_t totB = int64_t(P.m) * 4 * A.dil * ngB * A.Wout[1];
  if (totA >= (int64_t(1) << 31) || totB >= (int64_t(1) << 31)) return cudaErrorInvalidValue;   // 32-bit indices
  tmpl_passA<Real, L2><<<grid_for(totA), kBlock, 0, st>>>(P, A, P.J, level);
  if (P.d == 2) tmpl_passB<Real, L2><<<grid_for(totB), kBlock, 0, st>>>(P, A, P.J, level);
  return cudaSuccess;
}

template <typename Real>
static cudaError_t launch_tmpl_r(const Plan& P, const TmplArgs& A, int level, cudaStream_t st) {
  switch (P.L2) {
    case 2: if (cudaError_t e = launch_tmpl_t<Real, 2>(P, A, level, st)) return e; break;
    case 4: if (cudaError_t e = launch_tmpl_t<Real, 4>(P, A, level, st)) return e; break;
    case 6: if (cudaError_t e = launch_tmpl_t<Real, 6>(P, A, level, st)) return e; break;
    case 8: if (cudaError_t e = launch_tmpl_t<Real, 8>(P, A, level, st)) return e; break;
    case 10: if (cudaError_t e = launch_tmpl_t<Real, 10>(P, A, level, st)) return e; break;
    case 12: if (cudaError_t e = launch_tmpl_t<Real, 12>(P, A, level, st)) return e; break;
    case 14: if (cudaError_t e = launch_tmpl_t<Real, 14>(P, A, level, st)) return e; break;
    case 16: if (cudaError_t e = launch_tmpl_t<Real, 16>(P, A, level, st)) return e; break;
    case 18: if (cudaError_t e = launch_tmpl_t<Real, 18>(P, A, level, st)) return e; break;
    case 20: if (cudaError_t e = launch_tmpl_t<Real, 20>(P, A, level, st)) return e; break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_tmpl_level(const Plan& P, const TmplArgs& A, int real_bytes, int level, cudaStream_t st) {
  return real_bytes == 4 ? launch_tmpl_r<float>(P, A, level, st) : launch_tmpl_r<double>(P, A, level, st);
}

cudaError_t launch_pad_v(const void* v, void* vpad, int n, int P, int m, int real_bytes, cudaStream_t st) {
  return launch_wrap_v(v, vpad, n, P, P, n + 2 * P, n + 2 * P, m, real_bytes, st);
}

cudaError_t launch_wrap_v(const void* v, void* out, int n, int offy, int offx, int H, int W, int m, int real_bytes,
                          cudaStream_t st) {
  const dim3 grid((W + 255) / 256, H, m);
  if (real_bytes == 4) wrap_v_kernel<float><<<grid, 256, 0, st>>>((const float*)v, (float*)out, n, offy, offx, H, W);
  else wrap_v_kernel<double><<<grid, 256, 0, st>>>((const double*)v, (double*)out, n, offy, offx, H, W);
  return cudaGetLastError();
}

// Support check of pcwd_set_kernels: flag = 1 if some u_k(z) != 0 lies outside the planned periodic
// box [zlo_a, zhi_a] of an axis (the plan's windows are derived from that box).
__global__ void support_check_kernel(const double* __restrict__ u, int64_t total, int n, int d, int zlo0, int w0,
                                     int zlo1, int w1, int* flag) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    if (u[i] == 0.0) continue;
    const int64_t z = d == 2 ? i % (int64_t(n) * n) : i % n;
    const int z1 = int(z % n), z0 = int(z / n);
    const bool in1 = ((z1 - zlo1) % n + n) % n < w1;
    const bool in0 = d == 1 || ((z0 - zlo0) % n + n) % n < w0;
    if (!(in0 && in1)) *flag = 1;
  }
}

cudaError_t launch_support_check(const double* u, int64_t total, int n, int d, const int zlo[2], const int zhi[2],
                                 int* flag, cudaStream_t st) {
  const int w0 = zhi[0] - zlo[0] + 1, w1 = zhi[1] - zlo[1] + 1;
  support_check_kernel<<<std::min(grid_for(total), 148 * 8), kBlock, 0, st>>>(u, total, n, d, zlo[0], w0, zlo[1], w1,
                                                                              flag);
  return cudaGetLastError();
}

// pcwd_set_kernels_box: u_k given on the plan's periodic bounding box only (m × w0 × w1, row-major);
// entry (k, i0, i1) goes to u_k at ((zlo0 + i0) mod n, (zlo1 + i1) mod n); the rest of u stays zero
__global__ void box_scatter_kernel(const double* __restrict__ ub, int64_t total, int n, int d, int zlo0, int w0,
                                   int zlo1, int w1, double* __restrict__ u) {
  const int mask = n - 1;
  const int64_t N = d == 2 ? int64_t(n) * n : n;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = i / (int64_t(w0) * w1);
    const int r = int(i - k * w0 * w1);
    const int i0 = r / w1, i1 = r - i0 * w1;
    const int z1 = (zlo1 + i1) & mask, z0 = d == 2 ? ((zlo0 + i0) & mask) : 0;
    u[k * N + int64_t(z0) * n + z1] = ub[i];
  }
}

cudaError_t launch_box_scatter(const double* ub, int m, int n, int d, const int zlo[2], const int zhi[2], double* u,
                               cudaStream_t st) {
  const int w0 = d == 2 ? zhi[0] - zlo[0] + 1 : 1, w1 = zhi[1] - zlo[1] + 1;
  const int64_t total = int64_t(m) * w0 * w1;
  box_scatter_kernel<<<std::max<int64_t>(1, std::min(grid_for(total), 148 * 8)), kBlock, 0, st>>>(
      ub, total, n, d, zlo[0], w0, zlo[1], w1, u);
  return cudaGetLastError();
}

cudaError_t launch_cast(const double* src, void* dst, int64_t count, int real_bytes, cudaStream_t st) {
  if (real_bytes == 4) cast_kernel<float><<<grid_for(count), kBlock, 0, st>>>(src, (float*)dst, count);
  else cast_kernel<double><<<grid_for(count), kBlock, 0, st>>>(src, (double*)dst, count);
  return cudaGetLastError();
}

template <typename Real, typename OutT, int D, int MODE, int NT>
static cudaError_t launch_one(const Plan& P, const UnitArgs& A, int grid, size_t smem, cudaStream_t st) {
  auto kern = unit_kernel<Real, OutT, D, MODE, NT>;
  // the kernel has static shared memory too (reductions, scan storage): opt in whenever static + dynamic
  // exceeds 48 KB; the attribute only ever grows (per instantiation, process-wide), under a lock so that
  // handles used from several threads never launch between another thread's check and its set
  static std::mutex mu;
  static int opted = -1, static_bytes = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (opted < 0) {
      cudaFuncAttributes fa;
      cudaError_t e = cudaFuncGetAttributes(&fa, kern);
      if (e != cudaSuccess) return e;
      static_bytes = int(fa.sharedSizeBytes);
      opted = 48 * 1024 - static_bytes;
    }
    if (int(smem) > opted) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e != cudaSuccess) return e;
      opted = int(smem);
    }
  }
  // the kernel strides over units: a grid larger than the CTAs that can be resident at once only adds a partial
  // second wave (each CTA has the same share of units), so clamp it to one full wave
  int per_sm = 0, dev = 0, nsm = 148;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem) == cudaSuccess && per_sm > 0 &&
      cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
    grid = std::min(grid, per_sm * nsm);
  kern<<<grid, NT, smem, st>>>(P, A);
  return cudaGetLastError();
}

// 128 threads per unit when the launch has many units (more units in flight per SM), 256 when it has few (the
// coarse levels: big windows, too few units to fill the GPU one per 128-thread CTA)
template <typename Real, typename OutT, int MODE>
static cudaError_t launch_d(const Plan& P, const UnitArgs& A, int grid, size_t smem, cudaStream_t st) {
  const bool few = A.u1 - A.u0 < 148 * 6;
  if (few)
    return P.d == 2 ? launch_one<Real, OutT, 2, MODE, 256>(P, A, grid, smem, st)
                    : launch_one<Real, OutT, 1, MODE, 256>(P, A, grid, smem, st);
  return P.d == 2 ? launch_one<Real, OutT, 2, MODE, 128>(P, A, grid, smem, st)
                  : launch_one<Real, OutT, 1, MODE, 128>(P, A, grid, smem, st);
}

cudaError_t launch_units(const Plan& P, const UnitArgs& A, int mode, int real_bytes, int out_bytes, int grid,
                         size_t smem, cudaStream_t st) {
  switch (mode) {
    case MODE_FULL:
      return real_bytes == 4 ? launch_d<float, float, MODE_FULL>(P, A, grid, smem, st)
                             : launch_d<double, double, MODE_FULL>(P, A, grid, smem, st);
    case MODE_BAND:
      return real_bytes == 4 ? launch_d<float, float, MODE_BAND>(P, A, grid, smem, st)
                             : launch_d<double, double, MODE_BAND>(P, A, grid, smem, st);
    case MODE_PATTERN:
      return real_bytes == 4 ? launch_d<float, float, MODE_PATTERN>(P, A, grid, smem, st)
                             : launch_d<double, double, MODE_PATTERN>(P, A, grid, smem, st);
    case MODE_TMAX:
      return launch_d<double, double, MODE_TMAX>(P, A, grid, smem, st);
    case MODE_TSTORE:
      return launch_d<double, double, MODE_TSTORE>(P, A, grid, smem, st);
    case MODE_TCOUNT:
      return launch_d<double, double, MODE_TCOUNT>(P, A, grid, smem, st);
    case MODE_TWRITE:
      return out_bytes == 4 ? launch_d<double, float, MODE_TWRITE>(P, A, grid, smem, st)
                            : launch_d<double, double, MODE_TWRITE>(P, A, grid, smem, st);
  }
  return cudaErrorInvalidValue;
}

size_t unit_smem_limit() { return 200 * 1024; }

cudaError_t launch_fill_band_rowptr(int64_t* row_ptr, int64_t rows, int64_t L, cudaStream_t st) {
  fill_band_rowptr<<<grid_for(rows + 1), kBlock, 0, st>>>(row_ptr, rows, L);
  return cudaGetLastError();
}

cudaError_t launch_fill_full(int64_t* row_ptr, int32_t* col, int64_t rows, int64_t N, cudaStream_t st) {
  fill_full<<<grid_for(rows * N), kBlock, 0, st>>>(row_ptr, col, rows, N);
  return cudaGetLastError();
}

cudaError_t launch_cand_filter(const Plan& P, const double* cand, int64_t row0, int64_t rows, double tau, int write,
                               int32_t* cnt, const int64_t* row_ptr, int32_t* col, void* val, int out_bytes,
                               cudaStream_t st) {
  const int grid = int(std::min<int64_t>((std::max<int64_t>(rows, 1) * 32 + kBlock - 1) / kBlock, 148 * 16));
  if (rows <= 0) return cudaSuccess;
#define PCWD_CF(OT, DD, W) cand_filter_kernel<OT, DD, W><<<grid, kBlock, 0, st>>>(P, cand, row0, rows, tau, cnt, row_ptr, col, static_cast<OT*>(val))
  if (!write) {
    if (P.d == 2) PCWD_CF(double, 2, 0); else PCWD_CF(double, 1, 0);
  } else if (out_bytes == 4) {
    if (P.d == 2) PCWD_CF(float, 2, 1); else PCWD_CF(float, 1, 1);
  } else {
    if (P.d == 2) PCWD_CF(double, 2, 1); else PCWD_CF(double, 1, 1);
  }
#undef PCWD_CF
  return cudaGetLastError();
}

cudaError_t launch_cand_compact(const Plan& P, double* cand, int64_t row0, int64_t rows, double tau, int32_t* cnt,
                                cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const int grid = int(std::min<int64_t>((rows * 32 + kBlock - 1) / kBlock, 148 * 16));
  if (P.d == 2) cand_compact_kernel<2><<<grid, kBlock, 0, st>>>(P, cand, row0, rows, tau, cnt);
  else cand_compact_kernel<1><<<grid, kBlock, 0, st>>>(P, cand, row0, rows, tau, cnt);
  return cudaGetLastError();
}

cudaError_t launch_cand_copy(const Plan& P, const double* cand, int64_t row0, int64_t rows, const int32_t* cnt,
                             const int64_t* row_ptr, int32_t* col, float* val, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const int grid = int(std::min<int64_t>((rows * 32 + kBlock - 1) / kBlock, 148 * 16));
  if (P.d == 2) cand_copy_kernel<2><<<grid, kBlock, 0, st>>>(P, cand, row0, rows, cnt, row_ptr, col, val);
  else cand_copy_kernel<1><<<grid, kBlock, 0, st>>>(P, cand, row0, rows, cnt, row_ptr, col, val);
  return cudaGetLastError();
}

cudaError_t launch_row_counts(const int32_t* cnt, int64_t rows, int nsb, int64_t* rowcnt, cudaStream_t st) {
  row_counts_kernel<<<grid_for(rows + 1), kBlock, 0, st>>>(cnt, rows, nsb, rowcnt);
  return cudaGetLastError();
}

cudaError_t launch_max_reduce(const double* x, int64_t n, double* out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), st);
  if (e != cudaSuccess) return e;
  max_reduce_kernel<<<grid_for(n), kBlock, 0, st>>>(x, n, reinterpret_cast<unsigned long long*>(out));
  return cudaGetLastError();
}

cudaError_t launch_spmv(const int64_t* row_ptr, const int32_t* col, const void* val, const void* x, void* y,
                        int64_t rows, int64_t N, int transpose, int bytes, cudaStream_t st) {
  const int grid = int((rows * 32 + kBlock - 1) / kBlock);
  if (grid == 0) return cudaSuccess;
  if (!transpose) {
    if (bytes == 4) spmv_kernel<float><<<grid, kBlock, 0, st>>>(row_ptr, col, (const float*)val, (const float*)x, (float*)y, rows);
    else spmv_kernel<double><<<grid, kBlock, 0, st>>>(row_ptr, col, (const double*)val, (const double*)x, (double*)y, rows);
  } else {
    cudaError_t e = cudaMemsetAsync(y, 0, size_t(N) * bytes, st);
    if (e != cudaSuccess) return e;
    if (bytes == 4) spmv_t_kernel<float><<<grid, kBlock, 0, st>>>(row_ptr, col, (const float*)val, (const float*)x, (float*)y, rows);
    else spmv_t_kernel<double><<<grid, kBlock, 0, st>>>(row_ptr, col, (const double*)val, (const double*)x, (double*)y, rows);
  }
  return cudaGetLastError();
}

}  // namespace pcwd
// exclusive_scan_i64 and csr_transpose (Θᵀ for apply ᵀ / FISTA) live in sort.cu (the library's own scan and stable
// radix sort).
