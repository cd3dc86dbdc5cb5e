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
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"
#include "tma.h"

namespace pcwd {

namespace {
constexpr int kB = 256;

__device__ __forceinline__ float fmaB(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fmaB(double a, double b, double c) { return fma(a, b, c); }

// Row stride of the per-unit window buffers (R, approximations) in the batched scratch: 16-byte multiples so
// tile loads can use aligned vector copies.
__host__ __device__ __forceinline__ int rstride(int len) { return (len + 3) & ~3; }

inline int find_subband_host(const Plan& P, int64_t unit) {
  int s = P.nsb - 1;
  while (s > 0 && unit < P.sb[s].offset) --s;
  return s;
}

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

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
template <typename Real>
__device__ __forceinline__ void cp_async_el(Real* smem, const Real* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  if constexpr (sizeof(Real) == 4) asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}

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
  const int rs = rstride(r1.len);
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
    X0[int64_t(i0) * rs + i1] = acc;
  }
}

// Tiled k-sum for windows that do not cover a whole line (levels whose shift 2^ℓ ≥ 8): one CTA computes a
// (256/2^ℓ rows) × (2^ℓ·GZ columns) tile of template positions z for G units adjacent along axis 1.  Their
// windows are shifted by 2^ℓ columns, so unit u reads v at column z + 2^ℓ u: a thread owning template row r
// and columns res + 2^ℓ i (i < GZ) needs GZ template values and GZ+G-1 v values per k for G·GZ products.
// T_k and v_k tiles are staged in shared memory by cp.async, double-buffered over k; v columns wrap
// periodically (4-byte copies where the strip crosses the torus seam).
template <typename Real, int LEV, int G, int GZ>
__global__ void __launch_bounds__(kB) bk_ksum_tiled(const __grid_constant__ Plan P, const __grid_constant__ BatchArgs A,
                                                    int ntile1) {
  constexpr int SH = 1 << LEV;
  constexpr int TR = kB / SH;                 // template rows per tile
  constexpr int TW = SH * GZ;                 // template columns per tile
  constexpr int VW = 16 / int(sizeof(Real));  // elements per 16-byte vector
  constexpr int VWID = SH * (GZ + G - 1);     // v columns the G windows read
  constexpr int VS = VWID + VW;               // staged v row (aligned start + misalignment)
  extern __shared__ __align__(16) unsigned char ksm[];   // dynamic: Ts[2][TR][TW], Vs[2][TR][VS]
  auto Ts = reinterpret_cast<Real(*)[TR][TW]>(ksm);
  auto Vs = reinterpret_cast<Real(*)[TR][VS]>(ksm + sizeof(Real) * 2 * TR * TW);
  const int tid = threadIdx.x;
  const int n = P.n, mask = n - 1;
  const int64_t ug = A.u0 + int64_t(blockIdx.y) * G;            // first unit of the group
  const UnitPos up = unit_pos(P, ug);
  const SubBand& S = P.sb[up.sbi];
  const int R0 = S.tW[0], R1 = S.tW[1];
  const int t0 = blockIdx.x / ntile1, t1 = blockIdx.x - t0 * ntile1;
  const int z0 = t0 * TR, zc = t1 * TW;
  const int c0 = (up.p0 << LEV) + S.tSu[0];
  const int x0 = (up.p1 << LEV) + S.tSu[1] + zc;                // unwrapped first v column of the tile
  const int xa = x0 & ~(VW - 1), sh = x0 - xa;
  const bool nowrap = xa >= 0 && xa + VS <= n;
  const Real* __restrict__ v = reinterpret_cast<const Real*>(A.v);
  const Real* __restrict__ T = reinterpret_cast<const Real*>(A.T) + S.toff;
  auto stage = [&](int k, int b) {
    const Real* Tk = T + int64_t(k) * S.tstride;
    for (int i = tid; i < TR * (TW / VW); i += kB) {
      const int r = i / (TW / VW), c = (i - r * (TW / VW)) * VW;
      if (z0 + r < R0 && zc + c < S.tRS) cp_async16(&Ts[b][r][c], Tk + int64_t(z0 + r) * S.tRS + zc + c);
    }
    const Real* vk = v + int64_t(k) * P.N;
    if (nowrap) {
      for (int i = tid; i < TR * (VS / VW); i += kB) {
        const int r = i / (VS / VW), c = (i - r * (VS / VW)) * VW;
        cp_async16(&Vs[b][r][c], vk + int64_t((c0 + z0 + r) & mask) * n + xa + c);
      }
    } else {
      for (int i = tid; i < TR * VWID; i += kB) {
        const int r = i / VWID, c = i - r * VWID;
        cp_async_el(&Vs[b][r][sh + c], vk + int64_t((c0 + z0 + r) & mask) * n + ((x0 + c) & mask));
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int r = tid / SH, res = tid - r * SH;
  Real acc[G][GZ];
#pragma unroll
  for (int u = 0; u < G; ++u)
#pragma unroll
    for (int i = 0; i < GZ; ++i) acc[u][i] = Real(0);
  stage(0, 0);
  for (int k = 0; k < P.m; ++k) {
    if (k + 1 < P.m) {
      stage(k + 1, (k + 1) & 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const int b = k & 1;
    Real tv[GZ];
#pragma unroll
    for (int i = 0; i < GZ; ++i) tv[i] = Ts[b][r][res + SH * i];
#pragma unroll
    for (int mm = 0; mm < GZ + G - 1; ++mm) {
      const Real vm = Vs[b][r][sh + res + SH * mm];
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const int i = mm - u;
        if (i >= 0 && i < GZ) acc[u][i] = fmaB(vm, tv[i], acc[u][i]);
      }
    }
    __syncthreads();
  }
  if (z0 + r < R0) {
#pragma unroll
    for (int u = 0; u < G; ++u) {
      Real* X0 = reinterpret_cast<Real*>(A.scratch) + (ug + u - A.u0) * A.stride + S.offX0 + int64_t(z0 + r) * rstride(R1);
#pragma unroll
      for (int i = 0; i < GZ; ++i) {
        const int z = zc + res + SH * i;
        if (z < R1) X0[z] = acc[u][i];
      }
    }
  }
}

// Tiled k-sum with TMA staging (same tiling and register blocking as bk_ksum_tiled): per k, the T_k tile
// (TR rows × SH·GZ template columns) and the v_k strip of the G windows (TR rows × SH·(GZ+G-1) columns) are
// 3-D TMA boxes (kt_box_n / kt_box_q) issued by one thread into a ring of NST stage buffers, completion on
// an mbarrier per buffer — no per-thread copy or address arithmetic in the k loop.  v is read from its
// periodic extension (launch_wrap_v), so a strip that crosses the torus seam is still a run of TMA boxes.
template <typename Real, int LEV, int G, int GZ>
__global__ void __launch_bounds__(kB) bk_ksum_tma(const __grid_constant__ Plan P, const __grid_constant__ BatchArgs A,
                                                  int ntile1) {
  constexpr int SH = 1 << LEV;
  constexpr int TR = kB / SH;
  constexpr int RB = int(sizeof(Real)), VW = 16 / RB;
  constexpr int QT0 = GZ, QV0 = GZ + G - 1;
  constexpr int NTB = kt_box_n(SH, QT0), QT = kt_box_q(SH, QT0, NTB);
  constexpr int NVB = kt_vbox_n(SH, QV0, RB), QV = kt_vbox_q(SH, QV0, NVB, RB);
  constexpr int VBW = SH * QV + kt_vpadx(SH, RB);            // v box width (row pitch in shared memory)
  constexpr int TBOX = TR * SH * QT;                          // elements per box (TMA destinations: 128-byte aligned)
  constexpr int VBOX = (TR * VBW + 128 / RB - 1) / (128 / RB) * (128 / RB);
  constexpr int STAGE = NTB * TBOX + NVB * VBOX;
  constexpr int NST = 3;
  extern __shared__ __align__(16) unsigned char ktm[];
  __shared__ unsigned long long full[NST];
  Real* stg = reinterpret_cast<Real*>(ktm + ((128 - (smem_u32(ktm) & 127)) & 127));
  const int tid = threadIdx.x;
  const int n = P.n, mask = n - 1;
  const int64_t ug = A.u0 + int64_t(blockIdx.y) * G;
  const UnitPos up = unit_pos(P, ug);
  const SubBand& S = P.sb[up.sbi];
  const int R0 = S.tW[0], R1 = S.tW[1];
  const int t0 = blockIdx.x / ntile1, t1 = blockIdx.x - t0 * ntile1;
  const int z0 = t0 * TR, zc = t1 * SH * GZ;
  const int yr = ((up.p0 << LEV) + S.tSu[0] + z0) & mask;              // first v row of the tile
  const int xc = ((up.p1 << LEV) + S.tSu[1] + zc) & mask;              // first v column of the strip
  // v_wrap column of the strip start (kt_offx makes it 16-byte aligned: sh = 0 for every level ≥ 2)
  const int xw = xc + A.kt_offx, sh = xw & (VW - 1), xa = xw - sh;
  // each v box starts at its own wrapped column; the periodic extension (kt_vh × kt_vw ≥ (n + TR) × (n + VBW))
  // makes every box one TMA copy, wherever the strip crosses the torus seam
  const bool tma_v = yr + TR <= A.kt_vh && VBW + A.kt_offx <= A.kt_vw - n && sh + SH * QV <= VBW && !(A.kt_flags & 1);
  const CUtensorMap* tmT = &A.tmT[up.sbi - A.kt_sb_first];
  if (tid == 0) {
    for (int q = 0; q < NST; ++q) mbar_init(&full[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const Real* __restrict__ v = reinterpret_cast<const Real*>(A.v);
  auto issue = [&](int k) {
    if (k < P.m) {
      Real* b = stg + (k % NST) * STAGE;
      if (tid == 0) {
        mbar_expect_tx(&full[k % NST], unsigned(RB) * (NTB * TBOX + (tma_v ? NVB * TR * VBW : 0)));   // bytes of the boxes
#pragma unroll
        for (int j = 0; j < NTB; ++j) tma_load_3d(b + j * TBOX, tmT, zc + j * SH * QT, z0, k, &full[k % NST]);
        if (tma_v) {
#pragma unroll
          for (int j = 0; j < NVB; ++j)
            tma_load_3d(b + NTB * TBOX + j * VBOX, &A.tmV, ((xa + j * SH * QV - A.kt_offx) & mask) + A.kt_offx, yr, k,
                        &full[k % NST]);
        }
      }
      if (!tma_v) {   // strip across the torus seam: element copies into the same layout
        const Real* vk = v + int64_t(k) * P.N;
        Real* vb = b + NTB * TBOX;
        for (int i = tid; i < TR * SH * QV0; i += kB) {
          const int r = i / (SH * QV0), c = i - r * (SH * QV0);
          cp_async_el(vb + (c / (SH * QV)) * VBOX + r * VBW + sh + c % (SH * QV),
                      vk + int64_t((yr + r) & mask) * n + ((xc + c) & mask));
        }
      }
    }
    if (!tma_v) asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int q = 0; q < NST - 1; ++q) issue(q);
  const int r = tid / SH, res = tid - r * SH;
  const int offT = r * SH * QT + res, offV = r * VBW + sh + res;
  Real acc[G][GZ];
#pragma unroll
  for (int u = 0; u < G; ++u)
#pragma unroll
    for (int i = 0; i < GZ; ++i) acc[u][i] = Real(0);
  for (int k = 0; k < P.m; ++k) {
    issue(k + NST - 1);
    mbar_wait(&full[k % NST], unsigned(k / NST) & 1u);
    if (!tma_v) {
      asm volatile("cp.async.wait_group %0;" ::"n"(NST - 1) : "memory");
      __syncthreads();
    }
    const Real* Tb = stg + (k % NST) * STAGE;
    const Real* Vb = Tb + NTB * TBOX;
    Real tv[GZ];
#pragma unroll
    for (int i = 0; i < GZ; ++i) tv[i] = Tb[(i / QT) * TBOX + SH * (i % QT) + offT];
#pragma unroll
    for (int mm = 0; mm < QV0; ++mm) {
      const Real vm = Vb[(mm / QV) * VBOX + SH * (mm % QV) + offV];
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const int i = mm - u;
        if (i >= 0 && i < GZ) acc[u][i] = fmaB(vm, tv[i], acc[u][i]);
      }
    }
    __syncthreads();   // the buffer of k is refilled by issue(k + NST) at the next iteration
  }
  if (z0 + r < R0) {
#pragma unroll
    for (int u = 0; u < G; ++u) {
      Real* X0 = reinterpret_cast<Real*>(A.scratch) + (ug + u - A.u0) * A.stride + S.offX0 + int64_t(z0 + r) * rstride(R1);
#pragma unroll
      for (int i = 0; i < GZ; ++i) {
        const int z = zc + res + SH * i;
        if (z < R1) X0[z] = acc[u][i];
      }
    }
  }
}

template <typename Real, int LEV, int G, int GZ>
constexpr size_t ksum_tma_smem() {
  constexpr int SH = 1 << LEV, TR = kB / SH, RB = int(sizeof(Real));
  constexpr int NTB = kt_box_n(SH, GZ), QT = kt_box_q(SH, GZ, NTB);
  constexpr int NVB = kt_vbox_n(SH, GZ + G - 1, RB), QV = kt_vbox_q(SH, GZ + G - 1, NVB, RB);
  constexpr int VBOX = (TR * (SH * QV + kt_vpadx(SH, RB)) + 128 / RB - 1) / (128 / RB) * (128 / RB);
  return sizeof(Real) * 3 * size_t(NTB * TR * SH * QT + NVB * VBOX) + 128;
}

// Whole-torus k-sum with TMA staging, for 2^ℓ = 256·SHM (n = 2^ℓ·NL): as bk_ksum_full (units of a sub-band row
// share the v row; template columns shifted by 2^ℓ u), but a thread owns TRT rows and SHM residues (tid + 256 r),
// and the v rows (NL·SHM boxes of 256 columns) and the template strip ((2NL − 1)·SHM boxes of 256 columns, each
// starting on a multiple of 256 so none crosses the torus seam) are TMA boxes in a 3-stage mbarrier ring.
template <typename Real, int NL, int TRT, int SHM>
__global__ void __launch_bounds__(kB) bk_ksum_full_tma(const __grid_constant__ Plan P, const __grid_constant__ BatchArgs A) {
  constexpr int SH = 256 * SHM, G = NL, NTS = NL + G - 1;
  constexpr int BOX = TRT * 256;                    // elements per box (256 columns × TRT rows)
  constexpr int STAGE = (NL + NTS) * SHM * BOX;
  constexpr int NST = 3;
  extern __shared__ __align__(16) unsigned char kfm[];
  __shared__ unsigned long long full[NST];
  Real* stg = reinterpret_cast<Real*>(kfm + ((128 - (smem_u32(kfm) & 127)) & 127));
  const int tid = threadIdx.x;
  const int n = P.n, mask = n - 1;
  const int64_t ug = A.u0 + int64_t(blockIdx.y) * G;
  const UnitPos up = unit_pos(P, ug);
  const SubBand& S = P.sb[up.sbi];
  const int z0 = blockIdx.x * TRT;
  const int sy = up.p0 * SH;
  const int x0 = (-(up.p1 * SH + SH * (G - 1))) & mask;   // template column of strip column 0
  const int yt = (z0 - sy) & mask;                          // template row of tile row 0 (TRT | n: no wrap)
  const CUtensorMap* tmT = &A.tmT[up.sbi - A.kt_sb_first];
  if (tid == 0) {
    for (int q = 0; q < NST; ++q) mbar_init(&full[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int k) {
    if (tid == 0 && k < P.m) {
      Real* b = stg + (k % NST) * STAGE;
      mbar_expect_tx(&full[k % NST], unsigned(sizeof(Real) * STAGE));
#pragma unroll
      for (int i = 0; i < NL * SHM; ++i) tma_load_3d(b + i * BOX, &A.tmV, i * 256, z0, k, &full[k % NST]);
#pragma unroll
      for (int j = 0; j < NTS * SHM; ++j)
        tma_load_3d(b + (NL * SHM + j) * BOX, tmT, (x0 + j * 256) & mask, yt, k, &full[k % NST]);
    }
  };
  Real acc[TRT][SHM][G][NL];
#pragma unroll
  for (int t = 0; t < TRT; ++t)
#pragma unroll
    for (int r2 = 0; r2 < SHM; ++r2)
#pragma unroll
      for (int u = 0; u < G; ++u)
#pragma unroll
        for (int i = 0; i < NL; ++i) acc[t][r2][u][i] = Real(0);
#pragma unroll
  for (int q = 0; q < NST - 1; ++q) issue(q);
  for (int k = 0; k < P.m; ++k) {
    issue(k + NST - 1);
    mbar_wait(&full[k % NST], unsigned(k / NST) & 1u);
    const Real* Vb = stg + (k % NST) * STAGE;
    const Real* Tb = Vb + NL * SHM * BOX;
#pragma unroll
    for (int t = 0; t < TRT; ++t)
#pragma unroll
      for (int r2 = 0; r2 < SHM; ++r2) {
        Real vv[NL];
#pragma unroll
        for (int i = 0; i < NL; ++i) vv[i] = Vb[(i * SHM + r2) * BOX + t * 256 + tid];
        // unit u, column (tid + 256 r2) + SH i: strip chunk i − u + G − 1
#pragma unroll
        for (int mm = 0; mm < NTS; ++mm) {
          const Real tm = Tb[(mm * SHM + r2) * BOX + t * 256 + tid];
#pragma unroll
          for (int u = 0; u < G; ++u) {
            const int i = mm + u - (G - 1);
            if (i >= 0 && i < NL) acc[t][r2][u][i] = fmaB(vv[i], tm, acc[t][r2][u][i]);
          }
        }
      }
    __syncthreads();   // stage k % NST is refilled by issue(k + NST) next iteration
  }
  const int rs = rstride(n);
#pragma unroll
  for (int u = 0; u < G; ++u) {
    Real* X0 = reinterpret_cast<Real*>(A.scratch) + (ug + u - A.u0) * A.stride + S.offX0;
#pragma unroll
    for (int t = 0; t < TRT; ++t)
#pragma unroll
      for (int r2 = 0; r2 < SHM; ++r2)
#pragma unroll
        for (int i = 0; i < NL; ++i) X0[int64_t(z0 + t) * rs + tid + 256 * r2 + SH * i] = acc[t][r2][u][i];
  }
}

// Tiled k-sum for windows covering the whole torus on both axes (coarsest levels): the window is the torus,
// R(y) = Σ_k v_k(y) T_k((y - 2^ℓ p) mod n); G units adjacent along axis 1 read the same v tile and
// template columns shifted by 2^ℓ u.  A thread owns tile row r and the NL columns res + 2^ℓ i of one residue
// (a tile row spans the torus: 2^ℓ · NL = n); the template strip it reads is periodic.
template <typename Real, int LEV, int NL>
__global__ void __launch_bounds__(kB) bk_ksum_full(const __grid_constant__ Plan P, const __grid_constant__ BatchArgs A) {
  constexpr int SH = 1 << LEV;
  constexpr int TR = kB / SH > 0 ? kB / SH : 1;   // tile rows
  constexpr int G = NL;                            // units per group (a whole sub-band row)
  constexpr int TW = SH * NL;                      // = n
  constexpr int TSW = SH * (NL + G - 1);           // template strip width
  __shared__ Real Vt[2][TR][TW];
  __shared__ Real Tt[2][TR][TSW];
  const int tid = threadIdx.x;
  const int n = P.n, mask = n - 1;
  const int64_t ug = A.u0 + int64_t(blockIdx.y) * G;
  const UnitPos up = unit_pos(P, ug);
  const SubBand& S = P.sb[up.sbi];
  const int z0 = blockIdx.x * TR;                  // tile rows y0 = z0 .. z0 + TR - 1
  const int sy = up.p0 << LEV;                      // template row shift
  const int sx0 = (up.p1 << LEV) + SH * (G - 1);    // strip column 0 = template column (-sx0) mod n
  const Real* __restrict__ v = reinterpret_cast<const Real*>(A.v);
  const Real* __restrict__ T = reinterpret_cast<const Real*>(A.T) + S.toff;
  auto stage = [&](int k, int b) {
    const Real* vk = v + int64_t(k) * P.N;
    const Real* Tk = T + int64_t(k) * S.tstride;
    for (int i = tid; i < TR * TW; i += kB) {
      const int r = i / TW, c = i - r * TW;
      cp_async_el(&Vt[b][r][c], vk + int64_t(z0 + r) * n + c);
    }
    for (int i = tid; i < TR * TSW; i += kB) {
      const int r = i / TSW, c = i - r * TSW;
      cp_async_el(&Tt[b][r][c], Tk + int64_t((z0 + r - sy) & mask) * S.tRS + ((c - sx0) & mask));
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int r = tid / SH, res = tid - r * SH;
  const bool active = tid < TR * SH;
  Real acc[G][NL];
#pragma unroll
  for (int u = 0; u < G; ++u)
#pragma unroll
    for (int i = 0; i < NL; ++i) acc[u][i] = Real(0);
  stage(0, 0);
  for (int k = 0; k < P.m; ++k) {
    if (k + 1 < P.m) {
      stage(k + 1, (k + 1) & 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const int b = k & 1;
    if (active) {
      Real vv[NL];
#pragma unroll
      for (int i = 0; i < NL; ++i) vv[i] = Vt[b][r][res + SH * i];
      // unit u, column res + SH i: template column res + SH (i - u) - 2^ℓ p1  ->  strip index res + SH (i - u + G - 1)
#pragma unroll
      for (int mm = 0; mm < NL + G - 1; ++mm) {
        const Real tm = Tt[b][r][res + SH * mm];
#pragma unroll
        for (int u = 0; u < G; ++u) {
          const int i = mm + u - (G - 1);
          if (i >= 0 && i < NL) acc[u][i] = fmaB(vv[i], tm, acc[u][i]);
        }
      }
    }
    __syncthreads();
  }
  if (active) {
    const int rs = rstride(n);
#pragma unroll
    for (int u = 0; u < G; ++u) {
      Real* X0 = reinterpret_cast<Real*>(A.scratch) + (ug + u - A.u0) * A.stride + S.offX0 + int64_t(z0 + r) * rs;
#pragma unroll
      for (int i = 0; i < NL; ++i) X0[res + SH * i] = acc[u][i];
    }
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
    line4<Real>(P, X + int64_t(i0) * rstride(in1.len), 1, in1, a1.lo + jj, nout, out);
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
      if (q < nout) Xn[int64_t(j0 + q) * rstride(a1.len) + j1] = out[q];
  }
}

// Fused approximation step s (axis 1 then axis 0) for windows of any size: one CTA computes a 32 × 32 (fp64: 16 × 16) tile of
// the level-s approximation window of one unit.  The (62 + 2δ)² input tile is read from the unit's step
// input (zero outside its window, periodic where the window covers a line) into shared memory, filtered
// along axis 1 into a second tile, then along axis 0 into the next approximation (h taps only; the
// stencil's detail coefficients are computed directly by bk_gather).
template <typename Real, int L2, int TO>
__global__ void __launch_bounds__(kB) bk_approx(const __grid_constant__ Plan P, const __grid_constant__ BatchArgs A,
                                                int s, int ntx) {
  // TO: outputs per tile side (chosen per step by the launcher; static smem < 48 KB)
  constexpr int TI = 2 * (TO - 1) + L2;              // inputs per tile side
  constexpr int XS = ((TI + 1 + 1) / 2) * 2 % 4 == 2 ? ((TI + 1 + 1) / 2) * 2 : ((TI + 1 + 1) / 2) * 2 + 2;   // even, ≡ 2 mod 4
  constexpr int NI = 2 * 3 + L2;                     // inputs of 4 consecutive outputs
  __shared__ __align__(16) Real Xs[TI][XS];
  __shared__ Real Ys[TI][TO + 1];
  __shared__ int lr[TI], lc[TI];
  const int64_t unit = A.u0 + blockIdx.y;
  const UnitPos up = unit_pos(P, unit);
  const SubBand& S = P.sb[up.sbi];
  if (!(s < S.steps || s == P.J)) return;
  Range in0, in1;
  step_in(P, S, up, s, in0, in1);
  const Range a0 = step_out(in0, L2, 0), a1 = step_out(in1, L2, 0);
  const int ty = blockIdx.x / ntx, tx = blockIdx.x - ty * ntx;
  const int j0 = ty * TO, k0 = tx * TO;
  if (j0 >= a0.len || k0 >= a1.len) return;
  Real* base = reinterpret_cast<Real*>(A.scratch) + int64_t(blockIdx.y) * A.stride;
  const Real* X = base + ((s & 1) ? S.offX0 : S.offX1);
  Real* Xn = base + ((s & 1) ? S.offX1 : S.offX0);
  // input positions of the tile: 2·(a.lo + j0) + i on the input grid, i < TI; local indices are separable
  const int g0 = 2 * (a0.lo + j0), g1 = 2 * (a1.lo + k0);
  for (int i = threadIdx.x; i < TI; i += kB) {
    lr[i] = local_index(in0, g0 + i);
    lc[i] = local_index(in1, g1 + i);
  }
  __syncthreads();
  // tile rows/columns contiguous inside the window: 16-byte copies from the aligned-down column (the row
  // stride of the scratch is a 16-byte multiple), the misalignment `sh` is applied when reading Xs; otherwise
  // element copies with zero fill outside the window
  const bool fast = lr[0] >= 0 && lr[TI - 1] == lr[0] + TI - 1 && lc[0] >= 0 && lc[TI - 1] == lc[0] + TI - 1;
  const int rsx = rstride(in1.len);
  int sh = 0;
  if (fast) {
    constexpr int VWE = 8 / int(sizeof(Real));   // 8-byte copies: the even smem row stride stays bank-friendly
    const int ca = lc[0] & ~(VWE - 1);
    sh = lc[0] - ca;
    constexpr int NVEC = (TI + VWE - 1 + VWE - 1) / VWE;
    for (int idx = threadIdx.x; idx < TI * NVEC; idx += kB) {
      const int r = idx / NVEC, c = (idx - r * NVEC) * VWE;
      const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&Xs[r][c]));
      const Real* src = X + int64_t(lr[0] + r) * rsx + ca + c;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(src) : "memory");
    }
  } else {
    // edge tiles: the valid columns form one run [cf, cl] when the window does not wrap inside the tile (the
    // usual case); zero the tile, then copy each valid row's run with one warp (no per-element index math)
    __shared__ int crun[3];
    if (threadIdx.x < 32) {
      int first = TI, last = -1;
      for (int c = threadIdx.x; c < TI; c += 32)
        if (lc[c] >= 0) { first = min(first, c); last = max(last, c); }
      for (int o = 16; o > 0; o >>= 1) {
        first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
        last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
      }
      if (threadIdx.x == 0) {
        crun[0] = first;
        crun[1] = last;
        crun[2] = last >= first && lc[last] - lc[first] == last - first;
      }
    }
    for (int i = threadIdx.x; i < TI * XS; i += kB) (&Xs[0][0])[i] = Real(0);
    __syncthreads();
    const int cf = crun[0], cl = crun[1];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (crun[2]) {
      for (int r = w; r < TI; r += kB / 32) {
        const int li0 = lr[r];
        if (li0 < 0) continue;
        const Real* xrow = X + int64_t(li0) * rsx + lc[cf] - cf;
        for (int c = cf + lane; c <= cl; c += 32) {
          const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&Xs[r][c]));
          if constexpr (sizeof(Real) == 4)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(xrow + c) : "memory");
          else
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(xrow + c) : "memory");
        }
      }
    } else {
      for (int r = w; r < TI; r += kB / 32) {
        const int li0 = lr[r];
        if (li0 < 0) continue;
        const Real* xrow = X + int64_t(li0) * rsx;
        for (int c = lane; c < TI; c += 32) {
          const int li1 = lc[c];
          if (li1 < 0) continue;
          const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&Xs[r][c]));
          if constexpr (sizeof(Real) == 4)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(xrow + li1) : "memory");
          else
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(xrow + li1) : "memory");
        }
      }
    }
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  // axis 1: Ys[r][c] = Σ_t h[t] Xs[r][2c + t]; task = (row, 4 consecutive outputs), row fastest
  for (int idx = threadIdx.x; idx < TI * (TO / 4); idx += kB) {
    const int cq = idx / TI, r = idx - cq * TI;
    Real x[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) x[i] = Xs[r][sh + 8 * cq + i];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      Real acc = Real(0);
#pragma unroll
      for (int t = 0; t < L2; ++t) acc = fmaB(TapsOf<Real>::get(P, 0, t), x[2 * q + t], acc);
      Ys[r][4 * cq + q] = acc;
    }
  }
  __syncthreads();
  // axis 0: out[j][c] = Σ_t h[t] Ys[2j + t][c]; task = (4 consecutive output rows, column), column fastest
  for (int idx = threadIdx.x; idx < (TO / 4) * TO; idx += kB) {
    const int jq = idx / TO, c = idx - jq * TO;
    if (k0 + c >= a1.len) continue;
    Real y[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) y[i] = Ys[8 * jq + i][c];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = 4 * jq + q;
      if (j0 + j >= a0.len) break;
      Real acc = Real(0);
#pragma unroll
      for (int t = 0; t < L2; ++t) acc = fmaB(TapsOf<Real>::get(P, 0, t), y[2 * q + t], acc);
      Xn[int64_t(j0 + j) * rstride(a1.len) + k0 + c] = acc;
    }
  }
}

// Approximation step s with TMA tile loads, for steps whose input windows have one size across the launch's
// units and do not wrap (api.cu plans a 3-D tensor map per step and sub-band over the scratch buffer:
// columns × rows × unit slot).  A CTA computes `tpc` output tiles (TO × TO) of one unit; each input tile
// (TI rows × BW columns from a 16-byte aligned column, window outside read as zero by the TMA unit) lands in a
// double-buffered stage.  Axis 0 first (column-fastest tasks: conflict-free on the TMA row pitch), into Zs
// (odd pitch), then axis 1 (row-fastest tasks), 4 outputs per task, 16-byte stores (h taps only).
template <typename Real, int L2, int TO>
__global__ void __launch_bounds__(kB) bk_approx_tma(const __grid_constant__ Plan P, const __grid_constant__ BatchArgs A,
                                                    int s, int ntx, int ntiles, int tpc) {
  constexpr int RB = int(sizeof(Real)), VW = 16 / RB;
  constexpr int TI = 2 * (TO - 1) + L2;                     // input rows / columns per tile
  constexpr int BW = (TI + VW - 1 + VW - 1) / VW * VW;      // box width: aligned start + shift
  constexpr int XSZ = (TI * BW + 128 / RB - 1) / (128 / RB) * (128 / RB);
  constexpr int ZP = TI | 1;                                 // odd pitch of the axis-0 output
  constexpr int NI = 2 * 3 + L2;                             // inputs of 4 consecutive outputs
  extern __shared__ __align__(16) unsigned char atm[];
  __shared__ unsigned long long full[2];
  Real* Xs = reinterpret_cast<Real*>(atm + ((128 - (smem_u32(atm) & 127)) & 127));
  Real* Zs = Xs + 2 * XSZ;
  const int tid = threadIdx.x;
  const int64_t unit = A.u0 + blockIdx.y;
  const UnitPos up = unit_pos(P, unit);
  const SubBand& S = P.sb[up.sbi];
  if (!(s < S.steps || s == P.J)) return;
  Range in0, in1;
  step_in(P, S, up, s, in0, in1);
  const Range a0 = step_out(in0, L2, 0), a1 = step_out(in1, L2, 0);
  const int nty = (a0.len + TO - 1) / TO, ntxu = (a1.len + TO - 1) / TO;   // this unit's tiles
  const int t_first = blockIdx.x * tpc;
  const int t_last = min(t_first + tpc, nty * ntxu);
  if (t_first >= t_last) return;
  (void)ntx;
  (void)ntiles;
  const CUtensorMap* map = A.amaps + (s - 1) * 4 + (up.sbi - A.kt_sb_first);
  Real* Xn = reinterpret_cast<Real*>(A.scratch) + int64_t(blockIdx.y) * A.stride + ((s & 1) ? S.offX1 : S.offX0);
  const int rso = rstride(a1.len);
  // signed offset of input position g from the window start (g within L2 before the window .. its end)
  auto sdiff = [](int g, const Range& r) {
    int d = (g - r.lo) & (r.nl - 1);
    return d >= r.nl - 2 * L2 ? d - r.nl : d;
  };
  auto tile_org = [&](int t, int& d0, int& xs, int& sh, int& j0, int& k0) {
    const int ty = t / ntxu, tx = t - ty * ntxu;
    j0 = ty * TO;
    k0 = tx * TO;
    d0 = sdiff(2 * (a0.lo + j0), in0);
    const int d1 = sdiff(2 * (a1.lo + k0), in1);
    sh = d1 & (VW - 1);
    xs = d1 - sh;
  };
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int t, int b) {
    if (tid == 0 && t < t_last) {
      int d0, xs, sh, j0, k0;
      tile_org(t, d0, xs, sh, j0, k0);
      mbar_expect_tx(&full[b], unsigned(RB * TI * BW));
      tma_load_3d(Xs + b * XSZ, map, xs, d0, int(blockIdx.y), &full[b]);
    }
  };
  issue(t_first, 0);
  issue(t_first + 1, 1);
  for (int t = t_first, it = 0; t < t_last; ++t, ++it) {
    const int b = it & 1;
    int d0, xs, sh, j0, k0;
    tile_org(t, d0, xs, sh, j0, k0);
    mbar_wait(&full[b], unsigned(it >> 1) & 1u);
    const Real* X = Xs + b * XSZ;
    // axis 0: Zs[4jq + q][c] = Σ_t h[t] X[8jq + 2q + t][sh + c]
    for (int idx = tid; idx < TI * (TO / 4); idx += kB) {
      const int jq = idx / TI, c = idx - jq * TI;
      Real x[NI];
#pragma unroll
      for (int i = 0; i < NI; ++i) x[i] = X[(8 * jq + i) * BW + sh + c];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        Real acc = Real(0);
#pragma unroll
        for (int tt = 0; tt < L2; ++tt) acc = fmaB(TapsOf<Real>::get(P, 0, tt), x[2 * q + tt], acc);
        Zs[(4 * jq + q) * ZP + c] = acc;
      }
    }
    __syncthreads();   // Zs complete; stage b free
    issue(t + 2, b);
    // axis 1: out[j][4kq + q] = Σ_t h[t] Zs[j][8kq + 2q + t]
    for (int idx = tid; idx < TO * (TO / 4); idx += kB) {
      const int kq = idx / TO, j = idx - kq * TO;
      if (j0 + j >= a0.len || k0 + 4 * kq >= a1.len) continue;
      Real z[NI];
#pragma unroll
      for (int i = 0; i < NI; ++i) z[i] = Zs[j * ZP + 8 * kq + i];
      Real o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        Real acc = Real(0);
#pragma unroll
        for (int tt = 0; tt < L2; ++tt) acc = fmaB(TapsOf<Real>::get(P, 0, tt), z[2 * q + tt], acc);
        o[q] = acc;
      }
      Real* dst = Xn + int64_t(j0 + j) * rso + k0 + 4 * kq;   // rso is a multiple of 4: the row has room
      if constexpr (sizeof(Real) == 4) {
        *reinterpret_cast<float4*>(dst) = make_float4(o[0], o[1], o[2], o[3]);
      } else {
        reinterpret_cast<double2*>(dst)[0] = make_double2(o[0], o[1]);
        reinterpret_cast<double2*>(dst)[1] = make_double2(o[2], o[3]);
      }
    }
    __syncthreads();   // Zs reused by the next tile
  }
}

template <typename Real, int L2, int TO>
static void launch_approx_tma_t(const Plan& P, const BatchArgs& A, int s, int ntx, int nty, int nb, cudaStream_t st) {
  constexpr int RB = int(sizeof(Real)), VW = 16 / RB;
  constexpr int TI = 2 * (TO - 1) + L2;
  constexpr int BW = (TI + VW - 1 + VW - 1) / VW * VW;
  constexpr int XSZ = (TI * BW + 128 / RB - 1) / (128 / RB) * (128 / RB);
  constexpr size_t smem = size_t(RB) * (2 * XSZ + TO * (TI | 1)) + 128;
  auto k = bk_approx_tma<Real, L2, TO>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));   // per device, cheap
  const int ntiles = ntx * nty;
  const int tpc = ntiles <= 4 ? ntiles : (ntiles <= 16 ? 4 : 6);
  k<<<dim3((ntiles + tpc - 1) / tpc, nb), kB, smem, st>>>(P, A, s, ntx, ntiles, tpc);
}

template <typename Real, int TO>
static void launch_approx_to(const Plan& P, const BatchArgs& A, int s, dim3 grid, int ntx, cudaStream_t st) {
  switch (P.L2) {
    case 2: bk_approx<Real, 2, TO><<<grid, kB, 0, st>>>(P, A, s, ntx); break;
    case 4: bk_approx<Real, 4, TO><<<grid, kB, 0, st>>>(P, A, s, ntx); break;
    case 6: bk_approx<Real, 6, TO><<<grid, kB, 0, st>>>(P, A, s, ntx); break;
    case 8: bk_approx<Real, 8, TO><<<grid, kB, 0, st>>>(P, A, s, ntx); break;
    case 10: bk_approx<Real, 10, TO><<<grid, kB, 0, st>>>(P, A, s, ntx); break;
    case 12: bk_approx<Real, 12, TO><<<grid, kB, 0, st>>>(P, A, s, ntx); break;
  }
}

// Tile side per step: the TO ∈ {16, 24, 32} (fp64: {16}) with the least staged input Σ_tiles (2·TO + 2δ)²
// (edge tiles that run past the output window waste their share).
template <typename Real>
static void launch_approx(const Plan& P, const BatchArgs& A, int s, int64_t maxA0, int64_t maxA1, int nb,
                          cudaStream_t st) {
  static const bool no_tma = getenv("PCWD_NO_TMA_APPROX") != nullptr;
  if (A.amaps && ((A.am_steps >> s) & 1u) && !no_tma) {
    constexpr int TO = sizeof(Real) == 4 ? 32 : 16;
    const int ntx = int((maxA1 + TO - 1) / TO), nty = int((maxA0 + TO - 1) / TO);
    switch (P.L2) {
      case 2: launch_approx_tma_t<Real, 2, TO>(P, A, s, ntx, nty, nb, st); return;
      case 4: launch_approx_tma_t<Real, 4, TO>(P, A, s, ntx, nty, nb, st); return;
      case 6: launch_approx_tma_t<Real, 6, TO>(P, A, s, ntx, nty, nb, st); return;
      case 8: launch_approx_tma_t<Real, 8, TO>(P, A, s, ntx, nty, nb, st); return;
      case 10: launch_approx_tma_t<Real, 10, TO>(P, A, s, ntx, nty, nb, st); return;
      case 12: launch_approx_tma_t<Real, 12, TO>(P, A, s, ntx, nty, nb, st); return;
      default: break;
    }
  }
  if (P.L2 > 12 || (P.L2 & 1)) {
    auto gx = [](int64_t elems) { return int(std::max<int64_t>(1, std::min<int64_t>((elems + kB - 1) / kB, 64))); };
    bk_passA<Real><<<dim3(gx(maxA0 * 2 * maxA1 / 4 + 1), nb), kB, 0, st>>>(P, A, s);
    bk_passB<Real><<<dim3(gx(maxA0 * maxA1 / 4 + 1), nb), kB, 0, st>>>(P, A, s);
    return;
  }
  int best_to = 16;
  int64_t best = -1;
  const int cands[3] = {32, 24, 16};
  for (int c = 0; c < (sizeof(Real) == 4 ? 3 : 1); ++c) {
    const int to = sizeof(Real) == 4 ? cands[c] : 16;
    const int64_t ti = 2 * (to - 1) + P.L2;
    const int64_t cost = ((maxA0 + to - 1) / to) * ((maxA1 + to - 1) / to) * (ti * ti + 2048);   // + per-CTA overhead
    if (best < 0 || cost < best) { best = cost; best_to = to; }
  }
  const int ntx = int((maxA1 + best_to - 1) / best_to), nty = int((maxA0 + best_to - 1) / best_to);
  const dim3 grid(ntx * nty, nb);
  if constexpr (sizeof(Real) == 4) {
    if (best_to == 32) launch_approx_to<Real, 32>(P, A, s, grid, ntx, st);
    else if (best_to == 24) launch_approx_to<Real, 24>(P, A, s, grid, ntx, st);
    else launch_approx_to<Real, 16>(P, A, s, grid, ntx, st);
  } else {
    launch_approx_to<Real, 16>(P, A, s, grid, ntx, st);
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
      if (li0 >= 0 && li1 >= 0) val = Xn[int64_t(li0) * rstride(a1.len) + li1];
    } else {
      const int e0 = L.e0, e1 = L.e1;
      for (int t0 = 0; t0 < L2; ++t0) {
        const int r = local_index(in0, 2 * l0 + P.to[e0] + t0);
        if (r < 0) continue;
        Real row = Real(0);
        for (int t1 = 0; t1 < L2; ++t1) {
          const int c = local_index(in1, 2 * l1 + P.to[e1] + t1);
          if (c >= 0) row = fmaB(TapsOf<Real>::get(P, e1, t1), X[int64_t(r) * rstride(in1.len) + c], row);
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

// Tail of the cascade of one unit (one CTA per unit), steps s0 .. steps in shared memory: the step-s0 input
// window is read once from the scratch; each step computes its approximation (axis 1 then axis 0, periodic
// windows through local_index) and the stencil entries of its level — details directly from the step
// input (2δ × 2δ taps), the coarse block from the approximation (as bk_gather) — then the row (entries of the
// earlier steps from the stage in the scratch) is sorted by column and written (as bk_write).
template <typename Real, int L2, int NTT>
__global__ void __launch_bounds__(NTT) bk_tail(const __grid_constant__ Plan P, const __grid_constant__ BatchArgs A,
                                              int s0, int steps, int amax, int ymax) {
  extern __shared__ __align__(16) unsigned char tsm[];
  const int Lp = P.band_Lpad;
  int* kc = reinterpret_cast<int*>(tsm);
  Real* kv = reinterpret_cast<Real*>(tsm + ((Lp * 4 + 15) & ~15));
  Real* buf0 = kv + ((Lp + 3) & ~3);
  Real* buf1 = buf0 + amax;
  Real* Ys = buf1 + amax;
  const int tid = threadIdx.x;
  const int64_t unit = A.u0 + blockIdx.x;
  const UnitPos up = unit_pos(P, unit);
  const SubBand& S = P.sb[up.sbi];
  const Real* base = reinterpret_cast<const Real*>(A.scratch) + int64_t(blockIdx.x) * A.stride;
  Range in0, in1;
  step_in(P, S, up, s0, in0, in1);
  {  // step-s0 input window
    const Real* X = base + ((s0 & 1) ? S.offX0 : S.offX1);
    const int rs = rstride(in1.len);
    for (int i = tid; i < in0.len * in1.len; i += NTT) {
      const int r = i / in1.len, c = i - r * in1.len;
      buf0[i] = X[int64_t(r) * rs + c];
    }
  }
  // stage: entries of the steps before s0 come from bk_gather (scratch), the rest are computed below
  const Real* sv = base + S.offStage;
  const int* sc = reinterpret_cast<const int*>(sv + Lp);
  const int4* st = A.stencil + S.stencil_off;
  for (int j = tid; j < Lp; j += NTT) {
    if (j >= P.band_L) { kc[j] = INT_MAX; kv[j] = Real(0); }
    else if (st[j].w < s0) { kc[j] = sc[j]; kv[j] = sv[j]; }
  }
  __syncthreads();
  Real* X = buf0;
  Real* Xn = buf1;
  for (int s = s0; s <= steps; ++s) {
    const bool appr = s < S.steps || s == P.J;
    const Range a0 = step_out(in0, L2, 0), a1 = step_out(in1, L2, 0);
    if (appr) {
      // a window clear of wrapping (len + 2·2δ ≤ line) is addressed by a signed offset from its start; a
      // whole-line window wraps modulo the line; otherwise local_index per tap
      auto kind = [](const Range& r) { return r.len >= r.nl ? 1 : (r.len + 2 * L2 <= r.nl ? 0 : 2); };
      auto sdiff = [](int g, const Range& r) {
        int d = (g - r.lo) & (r.nl - 1);
        return d >= r.nl - 2 * L2 ? d - r.nl : d;
      };
      const int k1 = kind(in1), k0 = kind(in0);
      // axis 1: Ys[i0][l1] = Σ_t h[t] X[i0][2(a1.lo + l1) + t]
      for (int i = tid; i < in0.len * a1.len; i += NTT) {
        const int i0 = i / a1.len, l1 = i - i0 * a1.len;
        const int g = 2 * (a1.lo + l1);
        const Real* xr = X + i0 * in1.len;
        Real acc = Real(0);
        if (k1 == 0) {
          const int d = sdiff(g, in1);
#pragma unroll
          for (int t = 0; t < L2; ++t)
            if (unsigned(d + t) < unsigned(in1.len)) acc = fmaB(TapsOf<Real>::get(P, 0, t), xr[d + t], acc);
        } else if (k1 == 1) {
#pragma unroll
          for (int t = 0; t < L2; ++t) acc = fmaB(TapsOf<Real>::get(P, 0, t), xr[(g + t - in1.lo) & (in1.nl - 1)], acc);
        } else {
#pragma unroll
          for (int t = 0; t < L2; ++t) {
            const int c = local_index(in1, g + t);
            if (c >= 0) acc = fmaB(TapsOf<Real>::get(P, 0, t), xr[c], acc);
          }
        }
        Ys[i] = acc;
      }
      __syncthreads();
      // axis 0: Xn[l0][l1] = Σ_t h[t] Ys[2(a0.lo + l0) + t][l1]
      for (int i = tid; i < a0.len * a1.len; i += NTT) {
        const int l0 = i / a1.len, l1 = i - l0 * a1.len;
        const int g = 2 * (a0.lo + l0);
        const Real* yc = Ys + l1;
        Real acc = Real(0);
        if (k0 == 0) {
          const int d = sdiff(g, in0);
#pragma unroll
          for (int t = 0; t < L2; ++t)
            if (unsigned(d + t) < unsigned(in0.len)) acc = fmaB(TapsOf<Real>::get(P, 0, t), yc[(d + t) * a1.len], acc);
        } else if (k0 == 1) {
#pragma unroll
          for (int t = 0; t < L2; ++t)
            acc = fmaB(TapsOf<Real>::get(P, 0, t), yc[((g + t - in0.lo) & (in0.nl - 1)) * a1.len], acc);
        } else {
#pragma unroll
          for (int t = 0; t < L2; ++t) {
            const int r = local_index(in0, g + t);
            if (r >= 0) acc = fmaB(TapsOf<Real>::get(P, 0, t), yc[r * a1.len], acc);
          }
        }
        Xn[i] = acc;
      }
      __syncthreads();
    }
    // stencil entries of level s
    for (int j = tid; j < P.band_L; j += NTT) {
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
        if (appr && li0 >= 0 && li1 >= 0) val = Xn[li0 * a1.len + li1];
      } else {
        const int e0 = L.e0, e1 = L.e1;
        for (int t0 = 0; t0 < L2; ++t0) {
          const int r = local_index(in0, 2 * l0 + P.to[e0] + t0);
          if (r < 0) continue;
          Real row = Real(0);
#pragma unroll
          for (int t1 = 0; t1 < L2; ++t1) {
            const int c = local_index(in1, 2 * l1 + P.to[e1] + t1);
            if (c >= 0) row = fmaB(TapsOf<Real>::get(P, e1, t1), X[r * in1.len + c], row);
          }
          val = fmaB(TapsOf<Real>::get(P, e0, t0), row, val);
        }
      }
      kv[j] = val;
      kc[j] = int(L.offset + int64_t(l0) * L.nl + l1);
    }
    __syncthreads();
    if (appr) {
      Real* t = X;
      X = Xn;
      Xn = t;
      in0 = a0;
      in1 = a1;
    }
  }
  // CSR write in column order: the stencil order already is the column order unless a partner wraps around
  // the torus; then each entry goes to its rank (columns are distinct)
  const int L = P.band_L;
  int unsorted = 0;
  for (int i = tid; i + 1 < L; i += NTT) unsorted |= kc[i] > kc[i + 1];
  unsorted = __syncthreads_or(unsorted);
  const int64_t row = (unit - A.row0) * L;
  Real* outv = reinterpret_cast<Real*>(A.val);
  for (int i = tid; i < L; i += NTT) {
    const int c = kc[i];
    int rank = i;
    if (unsorted) {
      rank = 0;
      for (int j = 0; j < L; ++j) rank += kc[j] < c;
    }
    A.col[row + rank] = c;
    outv[row + rank] = kv[i];
  }
}

// ----------------------------------------------------------------------------------- launcher

// Tiled k-sum when every window of the launch's level stays inside one period per axis, the shift 2^ℓ is
// in [8, 128], and groups of G units stay in one sub-band row.  Returns false to use bk_ksum instead.
template <typename Real, int LEV, int G, int GZ>
static void launch_tiled_t(const Plan& P, const BatchArgs& A, dim3 grid, int ntile1, cudaStream_t st) {
  constexpr int SH = 1 << LEV, TR = kB / SH, TW = SH * GZ, VW = 16 / int(sizeof(Real));
  constexpr int VS = SH * (GZ + G - 1) + VW;
  constexpr size_t smem = sizeof(Real) * 2 * (size_t(TR) * TW + size_t(TR) * VS);
  auto k = bk_ksum_tiled<Real, LEV, G, GZ>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));   // per device, cheap
  k<<<grid, kB, smem, st>>>(P, A, ntile1);
}

template <typename Real, int LEV, int G, int GZ>
static void launch_tma_t(const Plan& P, const BatchArgs& A, dim3 grid, int ntile1, cudaStream_t st) {
  constexpr size_t smem = ksum_tma_smem<Real, LEV, G, GZ>();
  auto k = bk_ksum_tma<Real, LEV, G, GZ>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));   // per device, cheap
  BatchArgs B = A;
  B.kt_flags = getenv("PCWD_KT_FLAGS") ? atoi(getenv("PCWD_KT_FLAGS")) : 0;
  if (getenv("PCWD_KT_LEVMASK") && !((atoi(getenv("PCWD_KT_LEVMASK")) >> LEV) & 1)) B.kt_flags |= 1;
  k<<<grid, kB, smem, st>>>(P, B, ntile1);
}

int ksum_tiled_gz(const Plan& P, int64_t u0, int64_t u1, int real_bytes) {
  const int G = kt_units(real_bytes);
  if (getenv("PCWD_NO_TILED_KSUM") || u1 <= u0) return 0;
  const int s0 = find_subband_host(P, u0), s1 = find_subband_host(P, u1 - 1);
  const SubBand& S = P.sb[s0];
  const int lev = S.level;
  if (lev < 3 || lev > 8 || S.nl % G || (u0 - S.offset) % G || (u1 - u0) % G) return 0;
  for (int q = s0; q <= s1; ++q)
    if (P.sb[q].level != lev || P.sb[q].tW[0] >= P.n || P.sb[q].tW[1] >= P.n || P.sb[q].tW[0] != S.tW[0] ||
        P.sb[q].tW[1] != S.tW[1] || P.sb[q].e == 0)
      return 0;
  // template column groups per thread: the GZ ∈ {4, ..., 10} (fp64: {2, 4}) whose tiles waste the fewest columns
  const int SH = 1 << lev;
  const int cand_f[] = {8, 9, 10, 6, 5, 4}, cand_d[] = {4, 2};
  const int* cand = real_bytes == 4 ? cand_f : cand_d;
  const int ncand = real_bytes == 4 ? 6 : 2;
  int GZ = cand[0];
  int64_t best = -1;
  for (int c = 0; c < ncand; ++c) {
    const int tw = SH * cand[c], nt = (S.tW[1] + tw - 1) / tw;
    const int64_t cost = int64_t(nt) * (tw + SH * (G - 1));   // staged v columns per tile row ≈ traffic + work
    if (best < 0 || cost < best) { best = cost; GZ = cand[c]; }
  }
  return GZ;
}

template <typename Real>
static bool launch_ksum_tiled(const Plan& P, const BatchArgs& A, int nb, cudaStream_t st) {
  constexpr int G = sizeof(Real) == 4 ? 8 : 4;
  static_assert(G == kt_units(int(sizeof(Real))), "G");
  const int GZ = ksum_tiled_gz(P, A.u0, A.u1, int(sizeof(Real)));
  if (!GZ || nb % G) return false;
  const SubBand& S = P.sb[find_subband_host(P, A.u0)];
  const int lev = S.level, SH = 1 << lev, TR = kB / SH;
  const int ntile0 = (S.tW[0] + TR - 1) / TR, ntile1 = (S.tW[1] + SH * GZ - 1) / (SH * GZ);
  const dim3 grid(ntile0 * ntile1, nb / G);
  static const bool no_tma = getenv("PCWD_NO_TMA_KSUM") != nullptr;
  const bool tma = A.kt_gz == GZ && !no_tma;
#define PCWD_KT(L, Z)                                                                   \
  if (lev == L && GZ == Z) {                                                            \
    if (tma) launch_tma_t<Real, L, G, Z>(P, A, grid, ntile1, st);                       \
    else launch_tiled_t<Real, L, G, Z>(P, A, grid, ntile1, st);                         \
    return true;                                                                        \
  }
  if constexpr (sizeof(Real) == 4) {
    PCWD_KT(3, 8) PCWD_KT(3, 9) PCWD_KT(3, 10) PCWD_KT(3, 6) PCWD_KT(3, 5) PCWD_KT(3, 4)
    PCWD_KT(4, 8) PCWD_KT(4, 9) PCWD_KT(4, 10) PCWD_KT(4, 6) PCWD_KT(4, 5) PCWD_KT(4, 4)
    PCWD_KT(5, 8) PCWD_KT(5, 9) PCWD_KT(5, 10) PCWD_KT(5, 6) PCWD_KT(5, 5) PCWD_KT(5, 4)
    PCWD_KT(6, 8) PCWD_KT(6, 9) PCWD_KT(6, 10) PCWD_KT(6, 6) PCWD_KT(6, 5) PCWD_KT(6, 4)
    PCWD_KT(7, 8) PCWD_KT(7, 9) PCWD_KT(7, 10) PCWD_KT(7, 6) PCWD_KT(7, 5) PCWD_KT(7, 4)
    PCWD_KT(8, 8) PCWD_KT(8, 9) PCWD_KT(8, 10) PCWD_KT(8, 6) PCWD_KT(8, 5) PCWD_KT(8, 4)
  } else {
    PCWD_KT(3, 4) PCWD_KT(3, 2) PCWD_KT(4, 4) PCWD_KT(4, 2) PCWD_KT(5, 4) PCWD_KT(5, 2)
    PCWD_KT(6, 4) PCWD_KT(6, 2) PCWD_KT(7, 4) PCWD_KT(7, 2) PCWD_KT(8, 4) PCWD_KT(8, 2)
  }
#undef PCWD_KT
  return false;
}

// Full-torus windows: bk_ksum_full when 2^ℓ ≤ 256, a row of the sub-band is one group (nl ∈ {2, 4, 8}).
template <typename Real>
static bool launch_ksum_full(const Plan& P, const BatchArgs& A, int nb, cudaStream_t st) {
  if (getenv("PCWD_NO_TILED_KSUM")) return false;
  const int s0 = find_subband_host(P, A.u0), s1 = find_subband_host(P, A.u1 - 1);
  const SubBand& S = P.sb[s0];
  const int lev = S.level, nl = S.nl;
  if (P.d != 2 || (1 << lev) > 4 * kB || (nl != 2 && nl != 4 && nl != 8) || (nl << lev) != P.n) return false;
  for (int q = s0; q <= s1; ++q)
    if (P.sb[q].level != lev || P.sb[q].tW[0] < P.n || P.sb[q].tW[1] < P.n) return false;
  if (nb % nl || (A.u0 - S.offset) % nl) return false;
  if (A.kf_rows > 0 && lev >= 8 && lev <= 10 && (nl == 2 || nl == 4 || nl == 8) && !getenv("PCWD_NO_TMA_KSUM")) {
    const int shm = (1 << lev) / 256;
    auto launch = [&](auto kern, int NLV, int TRT, int SHMV) {
      const size_t smem = sizeof(Real) * 3 * size_t(2 * NLV - 1 + NLV) * SHMV * TRT * 256 + 128;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      kern<<<dim3(P.n / TRT, nb / NLV), kB, smem, st>>>(P, A);
    };
    if (shm == 1 && A.kf_rows == 2) {
      if (nl == 4) { launch(bk_ksum_full_tma<Real, 4, 2, 1>, 4, 2, 1); return true; }
      if (nl == 2) { launch(bk_ksum_full_tma<Real, 2, 2, 1>, 2, 2, 1); return true; }
    } else if (shm == 2 && A.kf_rows == 1) {
      if (nl == 4) { launch(bk_ksum_full_tma<Real, 4, 1, 2>, 4, 1, 2); return true; }
      if (nl == 2) { launch(bk_ksum_full_tma<Real, 2, 1, 2>, 2, 1, 2); return true; }
    } else if (shm == 4 && A.kf_rows == 1) {
      if (nl == 2) { launch(bk_ksum_full_tma<Real, 2, 1, 4>, 2, 1, 4); return true; }
    }
  }
  // cp.async kernel: 2^ℓ ≤ 256 (one residue per thread), static shared memory
  if ((1 << lev) > kB || (sizeof(Real) == 8 && nl == 8)) return false;
  const int TR = std::max(1, kB >> lev);
  const dim3 grid((P.n + TR - 1) / TR, nb / nl);
#define PCWD_KF(L, NLV)                                                                      \
  if constexpr (!(sizeof(Real) == 8 && NLV == 8)) {                                          \
    if (lev == L && nl == NLV) { bk_ksum_full<Real, L, NLV><<<grid, kB, 0, st>>>(P, A); return true; } \
  }
  PCWD_KF(8, 4) PCWD_KF(8, 2) PCWD_KF(7, 4) PCWD_KF(7, 2) PCWD_KF(6, 4) PCWD_KF(6, 2) PCWD_KF(5, 4) PCWD_KF(5, 2)
  PCWD_KF(7, 8) PCWD_KF(6, 8) PCWD_KF(5, 8) PCWD_KF(4, 8) PCWD_KF(4, 4) PCWD_KF(4, 2)
#undef PCWD_KF
  return false;
}

template <typename Real>
static cudaError_t run_batch_t(const Plan& P, const BatchArgs& A0, int64_t maxX0, const int64_t* workA,
                               const int64_t* workB, const int64_t* appr0, const int64_t* appr1, int steps,
                               cudaStream_t st, int* launches) {
  const int64_t units = A0.u1 - A0.u0;
  for (int64_t b0 = 0; b0 < units; b0 += A0.batch) {
    BatchArgs A = A0;
    A.u0 = A0.u0 + b0;
    const int nb = int(std::min<int64_t>(A0.batch, units - b0));
    A.u1 = A.u0 + nb;
    auto gx = [](int64_t elems) { return int(std::max<int64_t>(1, std::min<int64_t>((elems + kB - 1) / kB, 64))); };
    if (!launch_ksum_tiled<Real>(P, A, nb, st) && !launch_ksum_full<Real>(P, A, nb, st))
      bk_ksum<Real><<<dim3(gx(maxX0), nb), kB, 0, st>>>(P, A);
    ++*launches;
    static const bool old_passes = getenv("PCWD_OLD_PASSES") != nullptr;
    // steps ≥ tail_s0 (windows that fit in shared memory): one per-unit kernel with the gathers and the write
    const int s0 = A.tail_s0 > 0 && A.tail_s0 <= steps && !getenv("PCWD_NO_TAIL") ? A.tail_s0 : steps + 1;
    for (int s = 1; s < s0; ++s) {
      if (old_passes) {
        bk_passA<Real><<<dim3(gx(workA[s]), nb), kB, 0, st>>>(P, A, s);
        bk_passB<Real><<<dim3(gx(workB[s]), nb), kB, 0, st>>>(P, A, s);
        *launches += 2;
      } else {
        launch_approx<Real>(P, A, s, appr0[s], appr1[s], nb, st);
        *launches += 1;
      }
      bk_gather<Real><<<dim3(1, nb), kB, 0, st>>>(P, A, s);
      *launches += 1;
    }
    if (s0 <= steps) {
      const int64_t amax = (appr0[s0 - 1] * appr1[s0 - 1] + 3) & ~int64_t(3);
      const int64_t ymax = appr0[s0 - 1] * appr1[s0];
      const size_t sm = ((P.band_Lpad * 4 + 15) & ~15) + size_t((P.band_Lpad + 3) & ~3) * sizeof(Real) +
                        size_t(2 * amax + ymax) * sizeof(Real);
      // threads per unit: 128 for launches of many units (more resident CTAs; c5 level 4, 12,288 units: 297 ->
      // 210 us), 256 for fewer (c5 levels 5-8 are slower at 128); PCWD_TAIL_NT = 64 / 128 / 256 forces one
      static const int tnt_env = getenv("PCWD_TAIL_NT") ? atoi(getenv("PCWD_TAIL_NT")) : 0;
      const int tnt = tnt_env ? tnt_env : (nb >= 148 * 32 ? 128 : 256);
      auto launch_tail = [&](auto kern, int nt) {
        if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        kern<<<nb, nt, sm, st>>>(P, A, s0, steps, int(amax), int(ymax));
      };
#define PCWD_TAIL(L2V)                                                            \
  if (tnt == 64) launch_tail(bk_tail<Real, L2V, 64>, 64);                         \
  else if (tnt == 128) launch_tail(bk_tail<Real, L2V, 128>, 128);                 \
  else launch_tail(bk_tail<Real, L2V, 256>, 256);
      switch (P.L2) {
        case 2: PCWD_TAIL(2) break;
        case 4: PCWD_TAIL(4) break;
        case 6: PCWD_TAIL(6) break;
        case 8: PCWD_TAIL(8) break;
        case 10: PCWD_TAIL(10) break;
        case 12: PCWD_TAIL(12) break;
        default: return cudaErrorInvalidValue;
      }
#undef PCWD_TAIL
      ++*launches;
    } else {
      const size_t sm = ((P.band_Lpad * 4 + 15) & ~15) + size_t(P.band_Lpad) * sizeof(Real);
      bk_write<Real><<<nb, kB, sm, st>>>(P, A);
      ++*launches;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_band_batched(const Plan& P, const BatchArgs& A, int real_bytes, int64_t maxX0, const int64_t* workA,
                                const int64_t* workB, const int64_t* appr0, const int64_t* appr1, int steps,
                                cudaStream_t st, int* launches) {
  return real_bytes == 4 ? run_batch_t<float>(P, A, maxX0, workA, workB, appr0, appr1, steps, st, launches)
                         : run_batch_t<double>(P, A, maxX0, workA, workB, appr0, appr1, steps, st, launches);
}

}  // namespace pcwd
