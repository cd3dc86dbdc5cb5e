// fine.cu — band rule, fine levels (windows fit in shared memory): kernel K3f.
//
// One CTA (256 threads) processes rounds of GU units of one sub-band that are adjacent along axis 1
// (positions p1 .. p1+GU-1 of one row p0; their R windows are shifted by 2^ℓ columns).
//
//   a2 k-sum    R_j(y) = Σ_k v_k(c_j + y) T_k(y) for the GU windows at once (k-sum fused
//               before the cascade).  T_k and the v_k strip the GU windows read are staged in shared
//               memory by 3-D TMA boxes (one per k) in a ring of NST buffers (mbarrier completion).  A thread owns one template row r and GZ
//               template columns z_i = res + 2^ℓ(zb·GZ + i) of one residue class mod 2^ℓ; unit j reads
//               v at column z_i + 2^ℓ j = res + 2^ℓ(zb·GZ + i + j), so the GU·GZ products of one k need
//               only GZ template values and GU+GZ-1 v values (register blocking along the shift).
//   a3 cascade  one thread group per unit (warp at ℓ = 1), restricted to the stencil's needs (geom.h):
//               pass A filters input rows along axis 1 into a transposed buffer, pass B filters those
//               along axis 0; each task computes 8 consecutive outputs of one 2δ-tap filter from one run
//               of 16-byte loads (taps are compile-time indices into the kernel-parameter bank).
//   a4 gather   the stencil entries, written in CSR column order (rank sort when a partner wraps).
//
// Geometry comes from the host plan (one record per sub-band and class p mod 2^{steps-ℓ}, geom.h),
// translated to the unit's position.
#include <climits>
#include <cstdlib>
#include <type_traits>

#include "geom.h"
#include "kernels.cuh"
#include "tma.h"

// the SEP instances return from the round before the cascade loop (if constexpr + continue)
#pragma nv_diag_suppress 128

namespace pcwd {

namespace {

constexpr int kFT = 256;   // threads per CTA
constexpr int kSlack = 32; // elements of slack before / after each region (vector over-reads)

template <typename Real>
struct FVec;
template <>
struct FVec<float> {
  static constexpr int W = 4;
  using T = float4;
};
template <>
struct FVec<double> {
  static constexpr int W = 2;
  using T = double2;
};

__device__ __forceinline__ float ffma_(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double ffma_(double a, double b, double c) { return fma(a, b, c); }

__device__ __forceinline__ void bar_group(int id, int nthreads) {
  if (nthreads == 32) __syncwarp();
  else asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// 8 consecutive outputs out[q] = Σ_t f_TY[t] x[2(j0+q) + o_TY + t - base] of a row (taps are compile-time
// indices into the kernel-parameter bank).  `base` is even, so the 14 + 2δ inputs start at an even local
// index and are read as pairs (8-byte float2 / 16-byte double2 loads).  MASK: the row's valid entries are
// [vlo, vhi) and everything else must read as zero; without MASK the caller guarantees zeros around the
// valid entries (zero-padded rows), so no select is needed.
template <typename Real, int L2, int TY, bool MASK>
__device__ __forceinline__ void filt8(const Plan& P, const Real* __restrict__ row, int base, int j0, int nout,
                                      int vlo, int vhi, Real out[8]) {
  using V2 = typename std::conditional<sizeof(Real) == 4, float2, double2>::type;
  constexpr int o = TY ? 2 - L2 : 0;
  constexpr int SPAN = 14 + L2;                                 // inputs of 8 outputs (even)
  const int s0 = 2 * j0 + o - base;
  Real x[SPAN];
  const V2* p = reinterpret_cast<const V2*>(row + s0);
#pragma unroll
  for (int i = 0; i < SPAN / 2; ++i) {
    const V2 t = p[i];
    x[2 * i] = t.x;
    x[2 * i + 1] = t.y;
  }
  if constexpr (MASK) {
    const int lo = vlo - s0, hi = vhi - s0;
    if (lo > 0 || hi < 2 * (nout - 1) + L2) {
#pragma unroll
      for (int i = 0; i < SPAN; ++i) x[i] = (i >= lo && i < hi) ? x[i] : Real(0);
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    Real acc = Real(0);
#pragma unroll
    for (int t = 0; t < L2; ++t) acc = ffma_(TapsOf<Real>::get(P, TY, t), x[2 * q + t], acc);
    out[q] = acc;
  }
}

// Both filters of one analysis step on the same 8 output positions j0..j0+7 of a row (pass A, where the
// detail columns lie inside the approximation columns): one run of loads covers the union of the inputs,
// x[i] = row[2 j0 + (2 - L2) + i - base]; the g outputs read x[2q + t], the h outputs x[L2 - 2 + 2q + t].
template <typename Real, int L2, bool MASK>
__device__ __forceinline__ void filt8hg(const Plan& P, const Real* __restrict__ row, int base, int j0, bool doh,
                                        bool dog, int nh, int ng, int vlo, int vhi, Real oh[8], Real og[8]) {
  using V2 = typename std::conditional<sizeof(Real) == 4, float2, double2>::type;
  constexpr int SPAN = 12 + 2 * L2;
  const int s0 = 2 * j0 + 2 - L2 - base;
  Real x[SPAN];
  const V2* p = reinterpret_cast<const V2*>(row + s0);
#pragma unroll
  for (int i = 0; i < SPAN / 2; ++i) {
    const V2 t = p[i];
    x[2 * i] = t.x;
    x[2 * i + 1] = t.y;
  }
  if constexpr (MASK) {
    const int lo = vlo - s0, hi = vhi - s0;
    if (lo > 0 || hi < SPAN) {
#pragma unroll
      for (int i = 0; i < SPAN; ++i) x[i] = (i >= lo && i < hi) ? x[i] : Real(0);
    }
  }
  (void)nh;
  (void)ng;
  if (doh) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      Real acc = Real(0);
#pragma unroll
      for (int t = 0; t < L2; ++t) acc = ffma_(TapsOf<Real>::get(P, 0, t), x[L2 - 2 + 2 * q + t], acc);
      oh[q] = acc;
    }
  }
  if (dog) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      Real acc = Real(0);
#pragma unroll
      for (int t = 0; t < L2; ++t) acc = ffma_(TapsOf<Real>::get(P, 1, t), x[2 * q + t], acc);
      og[q] = acc;
    }
  }
}

// ---- separable direct a3 + a4 (geom.h "sep")
// BM atoms W (taps in shared memory, zero-padded to whole blocks of 2^S) at offsets c + 2^S b of a contiguous
// line x:  out[b·ostr] = Σ_i W[i] x[c + 2^S b + i]  for b < B ≤ BM.  MASK: entries outside [lo, hi) read 0
// (predicated loads); otherwise the caller guarantees zeros (or, beyond the B real atoms, finite values) there.
// Register window over the shift: for each residue r < 2^S the BM inputs x[c + 2^S j + r], j = k .. k + BM − 1,
// are held in registers (slot j mod BM); a block of 2^S taps costs 2^S tap loads (vectorised), 2^S new inputs
// and 2^S·BM FMAs.  Blocks are unrolled (compile-time count from 2δ), so the window rotates without moves.
template <typename Real, int L2, int S, int BM, bool MASK>
__device__ __noinline__ void sep_slide(const Real* __restrict__ x, int c, int lo, int hi, const Real* __restrict__ taps,
                                       int B, Real* __restrict__ out, int ostr) {
  constexpr int ST = 1 << S, NB = sep_atom_blk(S, L2);
  Real xr[ST][BM];
  Real acc[BM];
  const Real* xc = x + c;
  const unsigned span = unsigned(hi - lo);
  auto ld = [&](int j) -> Real {   // x[c + j]
    if constexpr (MASK) {
      Real v = Real(0);
      if (unsigned(c + j - lo) < span) v = xc[j];
      return v;
    } else {
      return xc[j];
    }
  };
#pragma unroll
  for (int b = 0; b < BM; ++b) acc[b] = Real(0);
#pragma unroll
  for (int r = 0; r < ST; ++r)
#pragma unroll
    for (int b = 0; b < BM; ++b) xr[r][b] = ld(r + ST * b);
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    Real w[ST];
    if constexpr (ST * sizeof(Real) >= 16) {
      using V = typename std::conditional<sizeof(Real) == 4, float4, double2>::type;
      constexpr int VW = 16 / sizeof(Real);
#pragma unroll
      for (int v = 0; v < ST / VW; ++v) {
        const V t = reinterpret_cast<const V*>(taps + k * ST)[v];
        const Real* tp = reinterpret_cast<const Real*>(&t);
#pragma unroll
        for (int q = 0; q < VW; ++q) w[VW * v + q] = tp[q];
      }
    } else {
#pragma unroll
      for (int r = 0; r < ST; ++r) w[r] = taps[k * ST + r];
    }
#pragma unroll
    for (int r = 0; r < ST; ++r)
#pragma unroll
      for (int b = 0; b < BM; ++b) acc[b] = ffma_(w[r], xr[r][(b + k) % BM], acc[b]);
    if (k + 1 < NB) {   // slot k mod BM (atom 0's entry of this block) takes the entry atom BM − 1 needs next
#pragma unroll
      for (int r = 0; r < ST; ++r) xr[r][k % BM] = ld((k + BM) * ST + r);
    }
  }
#pragma unroll
  for (int b = 0; b < BM; ++b)
    if (b < B) out[b * ostr] = acc[b];
}

template <typename Real, int L2, bool MASK>
__device__ __forceinline__ void sep_dispatch(int s, int B, const Real* x, int c, int lo, int hi, const Real* taps,
                                             Real* out, int ostr) {
#define SEP_CASE(SS, BB) \
  case SS * 16 + BB: sep_slide<Real, L2, SS, BB, MASK>(x, c, lo, hi, taps, B, out, ostr); break;
  switch (s * 16 + sep_bsel(s, B)) {
    SEP_CASE(1, 1) SEP_CASE(1, 2) SEP_CASE(1, 3) SEP_CASE(1, 4) SEP_CASE(1, 6) SEP_CASE(1, 8)
    SEP_CASE(2, 1) SEP_CASE(2, 2) SEP_CASE(2, 3) SEP_CASE(2, 4) SEP_CASE(2, 6) SEP_CASE(2, 8)
    SEP_CASE(3, 1) SEP_CASE(3, 2) SEP_CASE(3, 3) SEP_CASE(3, 4) SEP_CASE(3, 6)
    SEP_CASE(4, 1) SEP_CASE(4, 2)
    SEP_CASE(5, 1)
    default: break;
  }
#undef SEP_CASE
}

// a3 + a4 by the separable direct form: for each unit of the round (CG at a time, one thread group each),
// stage 1 filters the needed rows of R with the distinct column atoms of the stencil into Q, stage 2
// contracts the partners' row atoms with their Q columns, then the row is written in CSR column order.
// Rwin: window (0, 0) of unit 0 (rows of stride RS); taps: the shared-memory atom table (sep_toff).
template <typename Real, int L2, int GU, int CG>
__device__ __forceinline__ void sep_units(const Plan& P, const FineArgs& A, const SubBand& S, int p0, int p1f,
                                          int64_t ufirst, const Real* Rwin, Real* Ybase, const Real* taps, int slot,
                                          int gt, int* wflag) {
  constexpr int GT = kFT / CG;
  const int lev = S.level;
  const int4* st = A.stencil + S.stencil_off;
  const int L = P.band_L;
  const int R1 = S.tW[1];
  Real* outv = reinterpret_cast<Real*>(A.val);
  for (int w0 = 0; w0 < GU; w0 += CG) {
    const int u = w0 + slot;
    const int p1 = p1f + u;
    const int cls0 = p0 & (S.fg_m - 1), cls1 = p1 & (S.fg_m - 1);
    const SepClass C = A.sepc[S.fg_off + cls0 * S.fg_m + cls1];
    const Real* X = Rwin + u * A.RSZ;
    Real* Q = Ybase + slot * A.YSZ;
    Real* sv = Q + A.QSZ;
    int* sc = reinterpret_cast<int*>(sv + P.band_Lpad);
    SepRun* srun = reinterpret_cast<SepRun*>(sc + P.band_Lpad);
    if (gt == 0) wflag[slot] = 0;
    for (int jj = gt; jj < L; jj += GT) sv[jj] = Real(0);   // entries whose atoms miss the window stay 0
    for (int r = gt; r < C.nrun; r += GT) srun[r] = A.seprun[C.run_off + r];
    bar_group(1 + slot, GT);
    // stage 1: Q[q + b][row] = Σ_i W_{s,e}[i] · R[row][c + 2^s b + i]   (Q column-major, column stride QS)
    // tasks (run << 16 | row) grouped by code path in whole warps; -1 = padding.  The next task is fetched one
    // iteration ahead (run records in shared memory).
    int tk = gt < C.ntask ? __ldg(A.septask + C.task_off + gt) : -1;
    for (int t = gt; t < C.ntask; t += GT) {
      const int cur = tk;
      tk = t + GT < C.ntask ? __ldg(A.septask + C.task_off + t + GT) : -1;
      if (cur < 0) continue;
      const SepRun& R = srun[cur >> 16];
      const int row = cur & 0xffff;
      if constexpr (L2 >= 4) {
        if (R.mask)
          sep_dispatch<Real, L2, true>(R.s, R.B, X + row * A.RS, R.c, 0, R1, taps + R.toff, Q + R.q * A.QS + row,
                                       A.QS);
        else
          sep_dispatch<Real, L2, false>(R.s, R.B, X + row * A.RS, R.c, 0, R1, taps + R.toff, Q + R.q * A.QS + row,
                                        A.QS);
      }
    }
    bar_group(1 + slot, GT);
    // stage 2: Θ[μ][λ] = Σ_i W_{s,e}[i] · Q[g][fs + 2^s b + i]  (rows outside the computed [r0, r1) read 0)
    for (int t = gt; t < C.npart; t += GT) {
      const SepPart R = A.seppart[C.part_off + t];
      if (R.g < 0) continue;
      if constexpr (L2 >= 4)
        sep_dispatch<Real, L2, true>(R.s, R.B, Q + R.g * A.QS, R.fs, R.r0, R.r1, taps + R.toff,
                                     sv + R.jj, R.jstr);
    }
    // CSR columns in stencil order
    const int64_t base = (ufirst + u - A.row0) * L;
    int wrap = 0;
    for (int jj = gt; jj < L; jj += GT) {
      const int4 e = st[jj];
      const SubBand& Lb = P.sb[e.x];
      const int D = e.w - lev;
      const int b0 = D == 0 ? p0 : (D < 0 ? (p0 << -D) : (p0 >> D));
      const int b1 = D == 0 ? p1 : (D < 0 ? (p1 << -D) : (p1 >> D));
      const int l0 = b0 + e.y, l1 = b1 + e.z;
      wrap |= (l0 < 0) | (l0 >= Lb.nl) | (l1 < 0) | (l1 >= Lb.nl);
      sc[jj] = int(Lb.offset + int64_t(l0 & (Lb.nl - 1)) * Lb.nl + (l1 & (Lb.nl - 1)));
    }
    if (wrap) wflag[slot] = 1;
    bar_group(1 + slot, GT);
    wrap = wflag[slot];
    for (int jj = gt; jj < L; jj += GT) {
      const int c = sc[jj];
      int rank = jj;
      if (wrap) {
        rank = 0;
        for (int i = 0; i < L; ++i) rank += sc[i] < c;
      }
      A.col[base + rank] = c;
      outv[base + rank] = sv[jj];
    }
    __syncthreads();
  }
}

}  // namespace

// Shared-memory layout (elements of Real), all offsets from the dynamic smem base:
//   [slack] R_0 .. R_{GU-1} (RS × R0 each; later the approximation of each step, row stride RS) [slack]
//   [slack] staging: NST × (T_k tile R0 × TS, v_k strip R0 × VS)  ∪  Yt_0 .. Yt_{GU-1} (YC × YS)  [slack]
//   D_0 .. D_{GU-1} (DS each)
template <typename Real, int L2, int LEV, int GU, int GZ, int NT, int NST, int CG, int MINB, bool SEP>
__global__ void __launch_bounds__(kFT, MINB) fine_kernel(const __grid_constant__ Plan P, const __grid_constant__ FineArgs A) {
  extern __shared__ __align__(16) unsigned char fsm[];
  __shared__ int wflag[CG];
  __shared__ int nheavy[CG];
  __shared__ Real onef[2][kMaxTaps];              // f_0 = h, f_1 = g taps (gather's direct partners)
  __shared__ Real comp[2][3 * kMaxTaps - 2];      // two-step composites: c_e[x] = Σ_{2t+u=x} f_e[t] h[u]
  if (threadIdx.x < 2 * (3 * kMaxTaps - 2)) {
    const int e = threadIdx.x / (3 * kMaxTaps - 2), x = threadIdx.x % (3 * kMaxTaps - 2);
    double c = 0.0;
    for (int t = 0; t < L2; ++t) {
      const int uu = x - 2 * t;
      if (uu >= 0 && uu < L2) c += P.td[e][t] * P.td[0][uu];
    }
    comp[e][x] = Real(c);
    if (x < L2) onef[e][x] = Real(P.td[e][x]);
  }
  __shared__ int sdesc[CG][kFMS][32];   // per slot: translated step geometry (FStep fields)
  Real* sm = reinterpret_cast<Real*>(fsm);
  constexpr int SH = 1 << LEV;           // window shift between adjacent units (2^ℓ)
  constexpr int VW = FVec<Real>::W;
  const int tid = threadIdx.x;
  constexpr int GT = kFT / CG;           // threads per unit group in the cascade (CG units at a time)
  const int slot = tid / GT, gt = tid - slot * GT;
  Real* Rbase = sm + kSlack;
  // k-sum staging aliases the R region (R is written only after the last k); base aligned to 128 bytes for
  // the TMA boxes, derived from `sm` by an integer offset so the compiler keeps the shared address space
  const unsigned s_raw = smem_u32(sm + kSlack);
  Real* Sbase = sm + kSlack + (((s_raw + 127u) & ~127u) - s_raw) / sizeof(Real);
  Real* Ybase = sm + A.regS + kSlack;
  for (int i = tid; i < kSlack; i += kFT) sm[i] = Real(0);   // zero rows before R_0 row 0 (left pad)
  if constexpr (SEP) {   // the separable path's atom taps (geom.h sep_toff layout)
    const Real* at = reinterpret_cast<const Real*>(A.atoms);
    for (int i = tid; i < A.ntap; i += kFT) sm[A.regA + i] = at[i];
  }
  Real* Dbase = sm + A.regD;
  const int64_t rounds = (A.u1 - A.u0) / GU;
  __shared__ __align__(8) unsigned long long fullbar[NST];
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < NST; ++q) mbar_init(&fullbar[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned phase = 0u;   // bit b: parity of the next completion of fullbar[b]
  static_assert(NST >= 1 && NST <= 8, "staging depth");

  long long t_ksum = 0, t_casc = 0, t_last = 0;
  for (int64_t rd = blockIdx.x; rd < rounds; rd += gridDim.x) {
    if (A.dbg && tid == 0) t_last = clock64();
    const int64_t ufirst = A.u0 + rd * GU;
    const int sbi = find_subband(P, ufirst);
    const SubBand& S = P.sb[sbi];
    const int64_t pos = ufirst - S.offset;
    const int p0 = int(pos / S.nl), p1f = int(pos - int64_t(p0) * S.nl);
    const int R0 = S.tW[0], R1 = S.tW[1];
    const int c0 = (p0 << LEV) + S.tSu[0];
    const int c1f = (p1f << LEV) + S.tSu[1];
    const int roff = c1f & 1;                     // R row offset: makes every row base even (pair loads)
    const Real* __restrict__ T = reinterpret_cast<const Real*>(A.T) + S.toff;

    // ------------------------------------------------------------------ a2: k-sum
    {
      const int c1a = c1f & ~(VW - 1);                      // aligned strip start (may be < 0: padded v)
      const int sh = c1f - c1a;
      // stage T_k (template box) and the v_k strip (box of the periodically padded v) into buffer `buf`:
      // two TMA tile loads issued by one thread, completion counted in bytes on fullbar[buf].
      const unsigned stage_bytes = unsigned((R0 * A.TS + R0 * A.VS) * sizeof(Real));
      auto stage = [&](int k, int buf) {
        if (tid == kFT - 1) {
          Real* Ts = Sbase + buf * (A.TSZ + A.VSZ);
          Real* Vs = Ts + A.TSZ;
          fence_proxy_async();
          mbar_expect_tx(&fullbar[buf], stage_bytes);
          tma_load_3d(Ts, &A.tmT[sbi - A.sb_first], 0, 0, k, &fullbar[buf]);
          tma_load_3d(Vs, &A.tmV, c1a + A.vpad, c0 + A.vpad, k, &fullbar[buf]);
        }
      };
      // task t of this thread: q = t % Q (residue, z-block), r = t / Q
      const int NZB = ((R1 + SH - 1) / SH + GZ - 1) / GZ;
      const int Q = SH * NZB;
      Real acc[NT][GU][GZ];
#pragma unroll
      for (int a = 0; a < NT; ++a)
#pragma unroll
        for (int j = 0; j < GU; ++j)
#pragma unroll
          for (int i = 0; i < GZ; ++i) acc[a][j][i] = Real(0);
      stage(0, 0);
      const int nst = A.nst;           // staging buffers in use (≤ NST, as many as fit in the R region)
      for (int q = 1; q < nst; ++q)
        if (q < P.m) stage(q, q);
      // per-task offsets into the staged T / v tiles (loop-invariant over k)
      int tofs[NT], vofs[NT];
      bool tact[NT];
#pragma unroll
      for (int a = 0; a < NT; ++a) {
        const int t = tid + a * kFT;
        const int r = t / Q;
        const int q = t - r * Q;
        const int res = q % SH, zb = q / SH;
        const int z0 = res + SH * zb * GZ;
        tact[a] = r < R0;
        tofs[a] = r * A.TS + z0;
        vofs[a] = A.TSZ + r * A.VS + sh + z0;
      }
      int b = 0;
      for (int k = 0; k < P.m; ++k) {
        mbar_wait(&fullbar[b], (phase >> b) & 1u);
        phase ^= 1u << b;
        const Real* Ts = Sbase + b * (A.TSZ + A.VSZ);
#pragma unroll
        for (int a = 0; a < NT; ++a) {
          if (tact[a]) {
            const Real* tr = Ts + tofs[a];
            const Real* vr = Ts + vofs[a];
            Real tv[GZ];
#pragma unroll
            for (int i = 0; i < GZ; ++i) tv[i] = tr[SH * i];
#pragma unroll
            for (int mm = 0; mm < GU + GZ - 1; ++mm) {
              const Real vm = vr[SH * mm];
#pragma unroll
              for (int j = 0; j < GU; ++j) {
                const int i = mm - j;
                if (i >= 0 && i < GZ) acc[a][j][i] = ffma_(vm, tv[i], acc[a][j][i]);
              }
            }
          }
        }
        __syncthreads();
        if (k + nst < P.m) stage(k + nst, b);
        b = (b + 1 == nst) ? 0 : b + 1;
      }
      // R_j[r][z] (row stride RS), z < R1
#pragma unroll
      for (int a = 0; a < NT; ++a) {
        const int t = tid + a * kFT;
        const int r = t / Q;
        if (r < R0) {
          const int q = t - r * Q;
          const int res = q % SH, zb = q / SH;
          const int z0 = res + SH * zb * GZ;
          if (z0 + SH * (GZ - 1) < R1) {   // the whole block inside the window: plain stores
#pragma unroll
            for (int j = 0; j < GU; ++j) {
              Real* dst = Rbase + j * A.RSZ + r * A.RS + roff + z0;
#pragma unroll
              for (int i = 0; i < GZ; ++i) dst[SH * i] = acc[a][j][i];
            }
          } else {
#pragma unroll
            for (int j = 0; j < GU; ++j) {
              Real* dst = Rbase + j * A.RSZ + r * A.RS + roff;
#pragma unroll
              for (int i = 0; i < GZ; ++i)
                if (z0 + SH * i < R1) dst[z0 + SH * i] = acc[a][j][i];
            }
          }
        }
      }
      // zero the row pads (the staging boxes overwrote them): columns [0, roff) and [roff + R1, RS)
      for (int i = tid; i < GU * R0; i += kFT) {     // rows of all units are contiguous (RSZ = R0·RS)
        Real* row = Rbase + i * A.RS;
        if (roff) row[0] = Real(0);
        for (int c = roff + R1; c < A.RS; ++c) row[c] = Real(0);
      }
      __syncthreads();
    }

    if (A.dbg && tid == 0) { const long long t = clock64(); t_ksum += t - t_last; t_last = t; }
    // ------------------------------------------------------------------ a3: cascade of unit u
    // (CG units at a time, one thread group each; Yt, D and the step descriptors are per group slot)
    if constexpr (SEP) {
      sep_units<Real, L2, GU, CG>(P, A, S, p0, p1f, ufirst, Rbase + roff, Ybase, sm + A.regA, slot, gt, wflag);
      continue;
    }
    for (int w0 = 0; w0 < GU; w0 += CG) {
    const int u = w0 + slot;
    const int p1 = p1f + u;
    const int cls0 = p0 & (S.fg_m - 1), cls1 = p1 & (S.fg_m - 1);
    const FGeom& G = A.geom[S.fg_off + cls0 * S.fg_m + cls1];
    const int d0 = p0 - cls0, d1 = p1 - cls1;
    const int steps = S.steps;
    Real* X = Rbase + u * A.RSZ;                 // step input (R, then each step's approximation)
    Real* Yt = Ybase + slot * A.YSZ;
    Real* Dd = Dbase + slot * A.DS;
    int* sd = &sdesc[slot][0][0];
    // step descriptors: the class record's FStep fields translated to this unit (lane-parallel).
    // field layout (FStep): 0 xr 1 xrl 2 xc 3 xcl 4 ar 5 arl 6 hlo 7 hlen 8 glo 9 glen
    //                       10+ec blo0  14+ec blen0  18+ec blo1  22+ec blen1  26+ec doff
    // only what is read: every field of the cascade steps 1..S1, and the input box (fields 0-3) of step S1 + 1
    // (the X_{S1} box of the direct partners)
    const int S1 = steps <= A.direct ? 1 : steps - A.direct;   // A.direct levels (≤ 2) computed directly in the gather
    const int nfield = S1 * 32 + (S1 < steps ? 4 : 0);
    for (int i = gt; i < nfield; i += GT) {
      const int si = i >> 5, fi = i & 31;
      int val = 0;
      if (fi < 30) {
        // which shift a field takes: xr, ar (axis 0, level s-1); xc (axis 1, level s-1); hlo, glo, blo1 (axis 1,
        // level s); blo0 (axis 0, level s)
        const bool a0p = fi == 0 || fi == 4, a1p = fi == 2;
        const bool a1s = fi == 6 || fi == 8 || (fi >= 18 && fi < 22), a0s = fi >= 10 && fi < 14;
        const int dd = (a0p || a0s) ? d0 : d1;
        const int lv = (a0p || a1p) ? si : si + 1;
        const int sh = lv <= LEV ? dd * (1 << (LEV - lv)) : (dd >> (lv - LEV));
        val = reinterpret_cast<const int*>(&G.st[si])[fi] + ((a0p || a1p || a0s || a1s) ? sh : 0);
      }
      sd[i] = val;
    }
    if (gt == 0) { wflag[slot] = 0; nheavy[slot] = 0; }
    bar_group(1 + slot, GT);
    int xb = (p1 << LEV) + S.tSu[1] - roff;      // column of X's local index 0 (even)
    int xr0 = c0;                                // row of X's local index 0
    // cascade steps 1..S1; the partners of the last two levels are computed in the gather directly from the
    // step-S1 approximation (2δ × 2δ taps for level S1 + 1, composite (3·2δ − 2)² taps for S1 + 2), which
    // replaces the two smallest, latency-bound cascade steps
    int steps_run = (A.dbg_flags & 2) ? 0 : (A.dbg_flags & 4) ? 1 : steps;   // debug: skip cascade steps
    steps_run = min(steps_run, S1);
    for (int s = 1; s <= steps_run; ++s) {
      const int* d = sd + (s - 1) * 32;
      const int ar = d[4], arl = d[5];
      const int hlo = d[6], hlen = d[7], glo = d[8], glen = d[9];
      // pass A: rows of X (axis 1) -> Yt[col][row - yb]; task = (8-column block of the union of the h and
      // g output ranges, row), row fastest; a block inside both ranges computes both filters from one load
      const int yb = ar & ~(VW - 1);
      {
        const int gend = glo + glen, hend = hlo + hlen;
        const int ulo = glen ? (hlen ? min(hlo, glo) : glo) : hlo;
        const int uhi = glen ? (hlen ? max(hend, gend) : gend) : hend;
        const int nb = (uhi - ulo + 7) >> 3;
        const int rows = arl;
        const int ntask = (hlen + glen) ? nb * rows : 0;
        const int vlo = d[2] - xb, vhi = vlo + d[3];
        const float inv = 1.0f / float(max(rows, 1));
        for (int t = gt; t < ntask; t += GT) {
          const int q = __float2int_rz((float(t) + 0.5f) * inv);   // t / rows (exact for t < 2^20)
          const int rr = t - q * rows;
          const int j0 = ulo + 8 * q;
          const bool doh = j0 < hend && j0 + 8 > hlo, dog = j0 < gend && j0 + 8 > glo;
          const int r = ar + rr;
          const Real* xrow = X + (r - xr0) * A.RS;
          Real oh[8], og[8];
          if (s == 1) filt8hg<Real, L2, false>(P, xrow, xb, j0, doh, dog, 8, 8, vlo, vhi, oh, og);
          else filt8hg<Real, L2, true>(P, xrow, xb, j0, doh, dog, 8, 8, vlo, vhi, oh, og);
          Real* yh = Yt + (j0 - hlo) * A.YS + (r - yb);
          Real* yg = Yt + (hlen + j0 - glo) * A.YS + (r - yb);
          if (doh) {
            if (j0 >= hlo && j0 + 8 <= hend) {   // whole block inside the h range: plain stores
#pragma unroll
              for (int i = 0; i < 8; ++i) yh[i * A.YS] = oh[i];
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i)
                if (j0 + i >= hlo && j0 + i < hend) yh[i * A.YS] = oh[i];
            }
          }
          if (dog) {
            if (j0 >= glo && j0 + 8 <= gend) {
#pragma unroll
              for (int i = 0; i < 8; ++i) yg[i * A.YS] = og[i];
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i)
                if (j0 + i >= glo && j0 + i < gend) yg[i * A.YS] = og[i];
            }
          }
        }
      }
      bar_group(1 + slot, GT);
      // pass B: Yt rows (axis 0) -> approximation box (next X) and detail boxes (D); one flat task index
      // over the four boxes (box, row block, column), column fastest
      int nxb = 0, nxr = 0;
      if (s < steps) {
        nxb = d[32 + 2] & ~(VW - 1);
        nxr = d[32 + 0];
      }
      {
        const bool want0 = s < steps || s == P.J;
        const int vlo = ar - yb, vhi = vlo + arl;
        const int n0 = want0 ? ((d[14] + 7) >> 3) * d[22] : 0;
        const int n1 = n0 + ((d[15] + 7) >> 3) * d[23];
        const int n2 = n1 + ((d[16] + 7) >> 3) * d[24];
        const int n3 = n2 + ((d[17] + 7) >> 3) * d[25];
        for (int t = gt; t < n3; t += GT) {
          const int ec = (t >= n0) + (t >= n1) + (t >= n2);
          const int idx = t - (ec == 0 ? 0 : ec == 1 ? n0 : ec == 2 ? n1 : n2);
          const int bl0 = d[14 + ec], bl1 = d[22 + ec];
          const int q = __float2int_rz((float(idx) + 0.5f) * __frcp_rn(float(bl1)));   // idx / bl1
          const int cc = idx - q * bl1;
          const int l0 = d[10 + ec] + 8 * q;
          const int nrow = min(8, bl0 - 8 * q);
          const int j = d[18 + ec] + cc;
          const int e0 = ec >> 1, e1 = ec & 1;
          const int ycol = e1 ? hlen + (j - glo) : (j - hlo);
          Real out[8];
          if (e0) filt8<Real, L2, 1, true>(P, Yt + ycol * A.YS, yb, l0, nrow, vlo, vhi, out);
          else filt8<Real, L2, 0, true>(P, Yt + ycol * A.YS, yb, l0, nrow, vlo, vhi, out);
          Real* dst;
          int dstr;
          if (ec == 0 && s < steps) {
            dst = X + (l0 - nxr) * A.RS + (j - nxb);
            dstr = A.RS;
          } else {
            dst = Dd + d[26 + ec] + (8 * q) * bl1 + cc;
            dstr = bl1;
          }
          if (nrow == 8) {
#pragma unroll
            for (int i = 0; i < 8; ++i) dst[i * dstr] = out[i];
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (i < nrow) dst[i * dstr] = out[i];
          }
        }
      }
      bar_group(1 + slot, GT);
      xb = nxb;
      xr0 = nxr;
    }

    // ------------------------------------------------------------------ a4: gather + write row
    {
      const int lev = LEV;
      const int4* st = A.stencil + S.stencil_off;
      const int L = P.band_L;
      const int64_t base = (ufirst + u - A.row0) * L;
      Real* outv = reinterpret_cast<Real*>(A.val);
      Real* sv = Yt;                              // wrap-case stage (Yt is dead now)
      int* sc = reinterpret_cast<int*>(sv + P.band_Lpad);
      int wrap = 0;
      int* hl = sc + P.band_Lpad;                  // heavy (two-step) partners of this unit
      // X_{S1} (the step-S1 approximation) in the R region: box rows [bxr, bxr + bxrl), columns [bxc, bxc + bxcl),
      // local origin (xr0, xb)
      const int* dn = sd + min(S1, steps - 1) * 32;
      const int bxr = dn[0], bxrl = dn[1], bxc = dn[2], bxcl = dn[3];
      for (int jj = gt; jj < L; jj += GT) {
        const int4 e = st[jj];
        const int s = e.w;                        // level of the partner sub-band
        const SubBand& Lb = P.sb[e.x];
        const int D = s - lev;
        const int b0 = D == 0 ? p0 : (D < 0 ? (p0 << -D) : (p0 >> D));
        const int b1 = D == 0 ? p1 : (D < 0 ? (p1 << -D) : (p1 >> D));
        const int l0 = b0 + e.y, l1 = b1 + e.z;
        const int ec = Lb.e;
        const int e0 = ec >> 1, e1 = ec & 1;
        Real x = Real(0);
        if (s <= S1) {
          const int* dl = sd + (s - 1) * 32;
          const int i0 = l0 - dl[10 + ec], i1 = l1 - dl[18 + ec];
          const int bl1 = dl[22 + ec];
          if (i0 >= 0 && i0 < dl[14 + ec] && i1 >= 0 && i1 < bl1) x = Dd[dl[26 + ec] + i0 * bl1 + i1];
        } else if (s == S1 + 1) {
          // one analysis step applied to X_{S1} at this coefficient only (2δ × 2δ taps)
          const int r0 = 2 * l0 + (e0 ? 2 - L2 : 0), q0 = 2 * l1 + (e1 ? 2 - L2 : 0);
          const int ta = max(0, bxr - r0), tb = min(L2, bxr + bxrl - r0);
          const int ua = max(0, bxc - q0), ub = min(L2, bxc + bxcl - q0);
          const Real* row0 = X + (r0 - xr0) * A.RS + (q0 - xb);
          if (ta == 0 && tb == L2 && ua == 0 && ub == L2) {
            // rows of 2δ taps start at an even column (q0 - xb even, even row stride): pair loads
            using V2 = typename std::conditional<sizeof(Real) == 4, float2, double2>::type;
#pragma unroll
            for (int t = 0; t < L2; ++t) {
              const V2* rp = reinterpret_cast<const V2*>(row0 + t * A.RS);
              Real acc = Real(0);
#pragma unroll
              for (int u2 = 0; u2 < L2 / 2; ++u2) {
                const V2 pr = rp[u2];
                acc = ffma_(onef[e1][2 * u2], pr.x, acc);
                acc = ffma_(onef[e1][2 * u2 + 1], pr.y, acc);
              }
              x = ffma_(onef[e0][t], acc, x);
            }
          } else {
            for (int t = ta; t < tb; ++t) {
              Real acc = Real(0);
              for (int u2 = ua; u2 < ub; ++u2) acc = ffma_(onef[e1][u2], row0[t * A.RS + u2], acc);
              x = ffma_(onef[e0][t], acc, x);
            }
          }
        } else {
          // two steps (composite taps): deferred to the warp-cooperative pass below
          hl[atomicAdd(&nheavy[slot], 1)] = jj;
        }
        wrap |= (l0 < 0) | (l0 >= Lb.nl) | (l1 < 0) | (l1 >= Lb.nl);
        const int c = int(Lb.offset + int64_t(l0 & (Lb.nl - 1)) * Lb.nl + (l1 & (Lb.nl - 1)));
        sv[jj] = x;
        sc[jj] = c;
      }
      // any partner wraps around the torus -> place by rank of the column
      if (wrap) wflag[slot] = 1;
      bar_group(1 + slot, GT);
      // partners two levels past S1: one warp per coefficient, lanes over the (3·2δ − 2) rows of its
      // composite footprint, warp reduction
      {
        const int nh = nheavy[slot];
        const int wg = gt >> 5, lane = gt & 31, nw = GT >> 5;
        constexpr int NT2 = 3 * L2 - 2;
        for (int h = wg; h < nh; h += nw) {
          const int jj = hl[h];
          const int4 e = st[jj];
          const SubBand& Lb = P.sb[e.x];
          const int D = e.w - lev;
          const int b0 = D == 0 ? p0 : (D < 0 ? (p0 << -D) : (p0 >> D));
          const int b1 = D == 0 ? p1 : (D < 0 ? (p1 << -D) : (p1 >> D));
          const int l0 = b0 + e.y, l1 = b1 + e.z;
          const int e0 = Lb.e >> 1, e1 = Lb.e & 1;
          const int r0 = 4 * l0 + 2 * (e0 ? 2 - L2 : 0), q0 = 4 * l1 + 2 * (e1 ? 2 - L2 : 0);
          const int ua = max(0, bxc - q0), ub = min(NT2, bxc + bxcl - q0);
          Real part = Real(0);
          if (ua == 0 && ub == NT2) {
            using V2 = typename std::conditional<sizeof(Real) == 4, float2, double2>::type;
            for (int t = lane; t < NT2; t += 32) {
              if (r0 + t < bxr || r0 + t >= bxr + bxrl) continue;
              const V2* rp = reinterpret_cast<const V2*>(X + (r0 + t - xr0) * A.RS + (q0 - xb));
              Real acc = Real(0);
#pragma unroll
              for (int u2 = 0; u2 < NT2 / 2; ++u2) {   // q0 - xb even: pair loads
                const V2 pr = rp[u2];
                acc = ffma_(comp[e1][2 * u2], pr.x, acc);
                acc = ffma_(comp[e1][2 * u2 + 1], pr.y, acc);
              }
              part = ffma_(comp[e0][t], acc, part);
            }
          } else {
            for (int t = lane; t < NT2; t += 32) {
              if (r0 + t < bxr || r0 + t >= bxr + bxrl) continue;
              const Real* row = X + (r0 + t - xr0) * A.RS + (q0 - xb);
              Real acc = Real(0);
              for (int u2 = ua; u2 < ub; ++u2) acc = ffma_(comp[e1][u2], row[u2], acc);
              part = ffma_(comp[e0][t], acc, part);
            }
          }
          for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
          if (lane == 0) sv[jj] = part;
        }
      }
      bar_group(1 + slot, GT);
      wrap = wflag[slot];
      for (int jj = gt; jj < L; jj += GT) {
        const int c = sc[jj];
        int rank = jj;
        if (wrap) {
          rank = 0;
          for (int i = 0; i < L; ++i) rank += sc[i] < c;
        }
        A.col[base + rank] = c;
        outv[base + rank] = sv[jj];
      }
    }
    __syncthreads();
    }
    if (A.dbg && tid == 0) { const long long t = clock64(); t_casc += t - t_last; t_last = t; }
  }
  if (A.dbg && tid == 0) {
    atomicAdd(A.dbg, (unsigned long long)t_ksum);
    atomicAdd(A.dbg + 1, (unsigned long long)t_casc);
  }
}

// ---------------------------------------------------------------------------------- launcher

// "wide" fp32 variants: twice the units per round at one CTA per SM (up to 255 registers, ~200 KB smem):
// more template reuse per staged tile.  PCWD_FINE_WIDE = bit mask over levels 1..3 (default: level 3).
static int fine_wide(int level) {
  static const int mask = getenv("PCWD_FINE_WIDE") ? atoi(getenv("PCWD_FINE_WIDE")) : 4;
  return (mask >> (level - 1)) & 1;
}

bool fine_config(int real_bytes, int level, int L2, FineCfg* c) {
  if (L2 != 2 && L2 != 4 && L2 != 8 && L2 != 12) return false;
  if (real_bytes == 4) {
    const int wide = fine_wide(level);
    if (level == 1) { *c = wide ? FineCfg{16, 11, 1, 4, 8} : FineCfg{8, 11, 1, 4, 4}; return true; }
    if (level == 2) { *c = wide ? FineCfg{8, 15, 1, 2, 4} : FineCfg{4, 15, 1, 2, 4}; return true; }
    if (level == 3) { *c = wide ? FineCfg{4, 11, 3, 2, 4} : FineCfg{2, 11, 3, 1, 2}; return true; }
  } else {
    if (level == 1) { *c = FineCfg{4, 11, 1, 4, 4}; return true; }
    if (level == 2) { *c = FineCfg{2, 15, 1, 4, 2}; return true; }
    if (level == 3) { *c = FineCfg{2, 11, 3, 4, 2}; return true; }
  }
  return false;
}

// The separable variant is a separate instance (SEP = true) so the cascade instances carry none of its code; it is
// built only where build_sep can plan it (2δ ∈ {4, 8, 12}).
template <typename Real, int L2, int LEV, int GU, int GZ, int NT, int NST, int CG, int MINB>
static cudaError_t launch_fine_t(const Plan& P, const FineArgs& A, int grid, size_t smem, cudaStream_t st) {
  auto k = fine_kernel<Real, L2, LEV, GU, GZ, NT, NST, CG, MINB, false>;
  if constexpr (L2 >= 4) {
    if (A.sep) k = fine_kernel<Real, L2, LEV, GU, GZ, NT, NST, CG, MINB, true>;
  }
  if (A.sep && L2 < 4) return cudaErrorInvalidValue;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
  }
  k<<<grid, kFT, smem, st>>>(P, A);
  return cudaGetLastError();
}

template <int L2>
static cudaError_t launch_fine_l2(const Plan& P, const FineArgs& A, int real_bytes, int level, int grid, size_t smem,
                                  cudaStream_t st) {
  if (real_bytes == 4) {
    const int wide = fine_wide(level);
    if (level == 1) {
      if (wide) return launch_fine_t<float, L2, 1, 16, 11, 1, 4, 8, 1>(P, A, grid, smem, st);
      return launch_fine_t<float, L2, 1, 8, 11, 1, 4, 4, 2>(P, A, grid, smem, st);
    }
    if (level == 2) {
      if (wide) return launch_fine_t<float, L2, 2, 8, 15, 1, 2, 4, 1>(P, A, grid, smem, st);
      return launch_fine_t<float, L2, 2, 4, 15, 1, 2, 4, 2>(P, A, grid, smem, st);
    }
    if (level == 3) {
      if (wide) return launch_fine_t<float, L2, 3, 4, 11, 3, 2, 4, 1>(P, A, grid, smem, st);
      return launch_fine_t<float, L2, 3, 2, 11, 3, 1, 2, 2>(P, A, grid, smem, st);
    }
  } else {
    if (level == 1) return launch_fine_t<double, L2, 1, 4, 11, 1, 4, 4, 1>(P, A, grid, smem, st);
    if (level == 2) return launch_fine_t<double, L2, 2, 2, 15, 1, 4, 2, 2>(P, A, grid, smem, st);
    if (level == 3) return launch_fine_t<double, L2, 3, 2, 11, 3, 4, 2, 1>(P, A, grid, smem, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_fine(const Plan& P, const FineArgs& A, int real_bytes, int level, int grid, size_t smem,
                        cudaStream_t st) {
  switch (P.L2) {
    case 2: return launch_fine_l2<2>(P, A, real_bytes, level, grid, smem, st);
    case 4: return launch_fine_l2<4>(P, A, real_bytes, level, grid, smem, st);
    case 8: return launch_fine_l2<8>(P, A, real_bytes, level, grid, smem, st);
    case 12: return launch_fine_l2<12>(P, A, real_bytes, level, grid, smem, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace pcwd
