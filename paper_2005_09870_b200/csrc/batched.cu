// batched.cu — band rule for units with large windows (coarse levels), d = 2 (K3b).
//
// Units of one level are processed in batches; every phase is one grid-wide kernel over
// (unit, element) pairs with per-unit scratch slots in global memory (L2/HBM):
//   bk_ksum    R_μ(y) = Σ_k v_k(y) T_k(y - 2^ℓ p) on the unit window            (a2)
//   bk_passA   axis-1 analysis step of the current approximation window       (a3)
//   bk_passB   axis-0 step -> approximation (next input) and the 3 detail windows
//   bk_gather  the stencil entries of this level -> per-unit stage           (a4)
//   bk_write   sort the stage by column (CSR order), write the row
// Windows use the periodic Range arithmetic of common.h (a window may cover a whole line).
#include <climits>

#include "kernels.cuh"

namespace pcwd {

namespace {
constexpr int kB = 256;

__device__ __forceinline__ float fmaB(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fmaB(double a, double b, double c) { return fma(a, b, c); }

struct UnitPos {
  int sbi, p0, p1;
};

__device__ __forceinline__ UnitPos unit_pos(const Plan& P, int64_t unit) {
  UnitPos r;
  r.sbi = find_subband(P, unit);
  const SubBand& S = P.sb[r.sbi];
  const int64_t pos = unit - S.offset;
  r.p0 = int(pos / S.nl);
  r.p1 = int(pos - int64_t(r.p0) * S.nl);
  return r;
}

// input windows of step s (the level s-1 approximation) for a unit: iterate step_out
__device__ __forceinline__ void step_in(const Plan& P, const SubBand& S, const UnitPos& u, int s, Range& in0,
                                        Range& in1) {
  in0 = unit_window(P, S, 0, u.p0);
  in1 = unit_window(P, S, 1, u.p1);
  for (int q = 1; q < s; ++q) {
    in0 = step_out(in0, P.L2, 0);
    in1 = step_out(in1, P.L2, 0);
  }
}
}  // namespace

template <typename Real>
__global__ void __launch_bounds__(kB) bk_ksum(const __grid_constant__ Plan P, const __grid_constant__ BatchArgs A) {
  const int64_t unit = A.u0 + blockIdx.y;
  const UnitPos up = unit_pos(P, unit);
  const SubBand& S = P.sb[up.sbi];
  const Range r0 = unit_window(P, S, 0, up.p0), r1 = unit_window(P, S, 1, up.p1);
  const int total = r0.len * r1.len;
  Real* X0 = reinterpret_cast<Real*>(A.scratch) + int64_t(blockIdx.y) * A.stride + S.offX0;
  const Real* __restrict__ v = reinterpret_cast<const Real*>(A.v);
  const Real* __restrict__ T = reinterpret_cast<const Real*>(A.T) + S.toff;
  const int n = P.n, mask = n - 1;
  const bool f0 = S.tW[0] >= n, f1 = S.tW[1] >= n;
  const int tw1 = S.tRS;
  for (int idx = blockIdx.x * kB + threadIdx.x; idx < total; idx += gridDim.x * kB) {
    const int i0 = idx / r1.len, i1 = idx - i0 * r1.len;
    const int y0 = (r0.lo + i0) & mask, y1 = (r1.lo + i1) & mask;
    const int t0 = f0 ? ((y0 - (up.p0 << S.level)) & mask) : i0;
    const int t1 = f1 ? ((y1 - (up.p1 << S.level)) & mask) : i1;
    const int64_t vy = int64_t(y0) * n + y1;
    const int64_t ti = int64_t(t0) * tw1 + t1;
    Real acc = Real(0);
#pragma unroll 5
    for (int k = 0; k < P.m; ++k) acc = fmaB(__ldg(v + k * P.N + vy), __ldg(T + k * S.tstride + ti), acc);
    X0[idx] = acc;
  }
}

// Only the approximation chain is carried through the whole window (the stencil's coarse
// partners need all of it); the stencil's detail coefficients are computed directly in
// bk_gather from the step's input window (2δ × 2δ taps each).
//
// 4 consecutive outputs along a line from a window `in` stored contiguously (stride `st`
// between consecutive samples): out[q] = Σ_t f[t] x[2(lo+j0+q) + t]; contiguous fast path,
// periodic (full-line or wrapping) slow path.
template <typename Real>
__device__ __forceinline__ void line4(const Plan& P, const Real* __restrict__ x, int64_t st, const Range& in,
                                      int pos0, int nout, Real out[4]) {
  const int L2 = P.L2;
  int d = (2 * pos0 - in.lo) & (in.nl - 1);            // local index of the first tap, mod nl
  if (d > in.nl / 2) d -= in.nl;
  const bool fast = in.len < in.nl && d >= 0 && d + 2 * (nout - 1) + L2 <= in.len;
#pragma unroll
  for (int q = 0; q < 4; ++q) out[q] = Real(0);
  if (fast) {
    const Real* xp = x + int64_t(d) * st;
    for (int t = 0; t < L2; ++t) {
      const Real f = TapsOf<Real>::get(P, 0, t);
#pragma unroll
      for (int q = 0; q < 4; ++q) out[q] = fmaB(f, xp[int64_t(2 * q + t) * st], out[q]);
    }
  } else {
    for (int q = 0; q < nout; ++q)
      for (int t = 0; t < L2; ++t) {
        const int li = local_index(in, 2 * (pos0 + q) + t);
        if (li >= 0) out[q] = fmaB(TapsOf<Real>::get(P, 0, t), x[int64_t(li) * st], out[q]);
      }
  }
}

// pass A of step s (approximation along axis 1): Y[i0][jj], jj < a1.len
template <typename Real>
__global__ void __launch_bounds__(kB) bk_passA(const __grid_constant__ Plan P, const __grid_constant__ BatchArgs A,
                                               int s) {
  const int64_t unit = A.u0 + blockIdx.y;
  const UnitPos up = unit_pos(P, unit);
  const SubBand& S = P.sb[up.sbi];
  if (!(s < S.steps || s == P.J)) return;
  Range in0, in1;
  step_in(P, S, up, s, in0, in1);
  const Range a1 = step_out(in1, P.L2, 0);
  const int ng = (a1.len + 3) >> 2;
  const int total = in0.len * ng;
  Real* base = reinterpret_cast<Real*>(A.scratch) + int64_t(blockIdx.y) * A.stride;
  const Real* X = base + ((s & 1) ? S.offX0 : S.offX1);
  Real* Y = base + S.offY;
  for (int idx = blockIdx.x * kB + threadIdx.x; idx < total; idx += gridDim.x * kB) {
    const int i0 = idx / ng, g = idx - i0 * ng;
    const int jj = 4 * g, nout = min(4, a1.len - jj);
    Real out[4];
    line4<Real>(P, X + int64_t(i0) * in1.len, 1, in1, a1.lo + jj, nout, out);
    Real* yd = Y + int64_t(i0) * a1.len + jj;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q < nout) yd[q] = out[q];
  }
}

// pass B of step s (approximation along axis 0): next X = a0 × a1
template <typename Real>
__global__ void __launch_bounds__(kB) bk_passB(const __grid_constant__ Plan P, const __grid_constant__ BatchArgs A,
                                               int s) {
  const int64_t unit = A.u0 + blockIdx.y;
  const UnitPos up = unit_pos(P, unit);
  const SubBand& S = P.sb[up.sbi];
  if (!(s < S.steps || s == P.J)) return;
  Range in0, in1;
  step_in(P, S, up, s, in0, in1);
  const Range a0 = step_out(in0, P.L2, 0), a1 = step_out(in1, P.L2, 0);
  const int ng = (a0.len + 3) >> 2;
  const int total = ng * a1.len;
  Real* base = reinterpret_cast<Real*>(A.scratch) + int64_t(blockIdx.y) * A.stride;
  const Real* Y = base + S.offY;
  Real* Xn = base + ((s & 1) ? S.offX1 : S.offX0);
  for (int idx = blockIdx.x * kB + threadIdx.x; idx < total; idx += gridDim.x * kB) {
    const int g = idx / a1.len, j1 = idx - g * a1.len;
    const int j0 = 4 * g, nout = min(4, a0.len - j0);
    Real out[4];
    line4<Real>(P, Y + j1, a1.len, in0, a0.lo + j0, nout, out);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q < nout) Xn[int64_t(j0 + q) * a1.len + j1] = out[q];
  }
}

// gather the stencil entries of level s: details computed directly from the step's input
// window X (level s-1): d(l0,l1) = Σ_{t0,t1} f_{e0}[t0] f_{e1}[t1] X[2l0+o_{e0}+t0][2l1+o_{e1}+t1];
// the coarse block (e = 0, s = J) is read from the approximation output.
template <typename Real>
__global__ void __launch_bounds__(kB) bk_gather(const __grid_constant__ Plan P, const __grid_constant__ BatchArgs A,
                                                int s) {
  const int64_t unit = A.u0 + blockIdx.y;
  const UnitPos up = unit_pos(P, unit);
  const SubBand& S = P.sb[up.sbi];
  Range in0, in1;
  step_in(P, S, up, s, in0, in1);
  const Range a0 = step_out(in0, P.L2, 0), a1 = step_out(in1, P.L2, 0);
  Real* base = reinterpret_cast<Real*>(A.scratch) + int64_t(blockIdx.y) * A.stride;
  const Real* X = base + ((s & 1) ? S.offX0 : S.offX1);
  const Real* Xn = base + ((s & 1) ? S.offX1 : S.offX0);
  Real* sv = base + S.offStage;
  int* sc = reinterpret_cast<int*>(sv + P.band_Lpad);
  const int4* st = A.stencil + S.stencil_off;
  const int L2 = P.L2;
  for (int j = blockIdx.x * kB + threadIdx.x; j < P.band_Lpad; j += gridDim.x * kB) {
    if (j >= P.band_L) {
      if (s == 1) { sc[j] = INT_MAX; sv[j] = Real(0); }
      continue;
    }
    const int4 e = st[j];
    if (e.w != s) continue;
    const SubBand& L = P.sb[e.x];
    int b0, b1;
    if (L.level == S.level) { b0 = up.p0; b1 = up.p1; }
    else if (L.level < S.level) { b0 = up.p0 << (S.level - L.level); b1 = up.p1 << (S.level - L.level); }
    else { b0 = up.p0 >> (L.level - S.level); b1 = up.p1 >> (L.level - S.level); }
    const int l0 = (b0 + e.y) & (L.nl - 1), l1 = (b1 + e.z) & (L.nl - 1);
    Real val = Real(0);
    if (L.e == 0) {
      const int li0 = local_index(a0, l0), li1 = local_index(a1, l1);
      if (li0 >= 0 && li1 >= 0) val = Xn[int64_t(li0) * a1.len + li1];
    } else {
      const int e0 = L.e0, e1 = L.e1;
      for (int t0 = 0; t0 < L2; ++t0) {
        const int r = local_index(in0, 2 * l0 + P.to[e0] + t0);
        if (r < 0) continue;
        Real row = Real(0);
        for (int t1 = 0; t1 < L2; ++t1) {
          const int c = local_index(in1, 2 * l1 + P.to[e1] + t1);
          if (c >= 0) row = fmaB(TapsOf<Real>::get(P, e1, t1), X[int64_t(r) * in1.len + c], row);
        }
        val = fmaB(TapsOf<Real>::get(P, e0, t0), row, val);
      }
    }
    sv[j] = val;
    sc[j] = int(L.offset + int64_t(l0) * L.nl + l1);
  }
}

// one CTA per unit: bitonic sort of the stage by column, write the CSR row
template <typename Real>
__global__ void __launch_bounds__(kB) bk_write(const __grid_constant__ Plan P, const __grid_constant__ BatchArgs A) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int Lp = P.band_Lpad;
  int* kc = reinterpret_cast<int*>(sm);
  Real* kv = reinterpret_cast<Real*>(sm + ((Lp * 4 + 15) & ~15));
  const int64_t unit = A.u0 + blockIdx.x;
  const UnitPos up = unit_pos(P, unit);
  const SubBand& S = P.sb[up.sbi];
  const Real* sv = reinterpret_cast<const Real*>(A.scratch) + int64_t(blockIdx.x) * A.stride + S.offStage;
  const int* sc = reinterpret_cast<const int*>(sv + Lp);
  for (int i = threadIdx.x; i < Lp; i += kB) { kc[i] = sc[i]; kv[i] = sv[i]; }
  __syncthreads();
  for (int k = 2; k <= Lp; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < Lp; i += kB) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up2 = (i & k) == 0;
          const int ci = kc[i], cj = kc[ixj];
          if ((ci > cj) == up2) {
            kc[i] = cj; kc[ixj] = ci;
            const Real t = kv[i]; kv[i] = kv[ixj]; kv[ixj] = t;
          }
        }
      }
      __syncthreads();
    }
  }
  const int64_t base = (unit - A.row0) * P.band_L;
  Real* outv = reinterpret_cast<Real*>(A.val);
  for (int i = threadIdx.x; i < P.band_L; i += kB) {
    A.col[base + i] = kc[i];
    outv[base + i] = kv[i];
  }
}

// ----------------------------------------------------------------------------------- launcher

template <typename Real>
static cudaError_t run_batch_t(const Plan& P, const BatchArgs& A0, int64_t maxX0, const int64_t* workA,
                               const int64_t* workB, int steps, cudaStream_t st, int* launches) {
  const int64_t units = A0.u1 - A0.u0;
  for (int64_t b0 = 0; b0 < units; b0 += A0.batch) {
    BatchArgs A = A0;
    A.u0 = A0.u0 + b0;
    const int nb = int(std::min<int64_t>(A0.batch, units - b0));
    A.u1 = A.u0 + nb;
    auto gx = [](int64_t elems) { return int(std::max<int64_t>(1, std::min<int64_t>((elems + kB - 1) / kB, 64))); };
    bk_ksum<Real><<<dim3(gx(maxX0), nb), kB, 0, st>>>(P, A);
    ++*launches;
    for (int s = 1; s <= steps; ++s) {
      bk_passA<Real><<<dim3(gx(workA[s]), nb), kB, 0, st>>>(P, A, s);
      bk_passB<Real><<<dim3(gx(workB[s]), nb), kB, 0, st>>>(P, A, s);
      bk_gather<Real><<<dim3(1, nb), kB, 0, st>>>(P, A, s);
      *launches += 3;
    }
    const size_t sm = ((P.band_Lpad * 4 + 15) & ~15) + size_t(P.band_Lpad) * sizeof(Real);
    bk_write<Real><<<nb, kB, sm, st>>>(P, A);
    ++*launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_band_batched(const Plan& P, const BatchArgs& A, int real_bytes, int64_t maxX0, const int64_t* workA,
                                const int64_t* workB, int steps, cudaStream_t st, int* launches) {
  return real_bytes == 4 ? run_batch_t<float>(P, A, maxX0, workA, workB, steps, st, launches)
                         : run_batch_t<double>(P, A, maxX0, workA, workB, steps, st, launches);
}

}  // namespace pcwd
