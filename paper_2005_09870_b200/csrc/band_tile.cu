// band_tile.cu — the fast path of the band rule (kernel K3t).
//
// One CTA processes rounds of G units of one sub-band that are adjacent along axis 1
// (positions p1 .. p1+G-1 of row p0).  Per round:
//   a2  k-sum    R_u(y) = Σ_k v_k(y) T_k(y - c_u) for the G windows at once; each thread
//                holds a 4-wide strip of T_k and the (4 + (G-1)·2^ℓ)-wide strip of v_k that
//                the G shifted windows read, so one v load feeds up to G FMAs.
//   a3  cascade  restricted to what the unit's stencil needs (Lemma 6, made
//                exact): step s computes the approximation only where steps s+1.. read it, and
//                the detail coefficients only inside the stencil's boxes at level s.
//                Separable: pass A filters rows (axis 1) into a transposed buffer, pass B
//                filters those rows (axis 0); both compute 4 outputs per thread from
//                vector loads of a zero-padded, 16-byte-aligned row (the filter taps are
//                uniform and come from the constant bank).
//   a4  gather   stencil entries are read from the detail boxes, written in (sb, o0, o1)
//                order (= CSR column order unless a partner wraps around the torus; then
//                the entry's rank among the unit's columns is used).
// All windows are in unwrapped coordinates; a plan flag guarantees no window covers a
// whole periodic line for the sub-bands routed here (wk_ok).
#include <climits>

#include "kernels.cuh"

namespace pcwd {

namespace {

constexpr int kTB = 256;          // threads per CTA (G units × WPU warps)
constexpr int kMS = 6;            // max cascade steps on this path
constexpr int kG = 4;             // max units per round
constexpr int kSL = 32;           // slack elements before / after each row buffer (vector over-reads)

struct Box {
  int lo0, len0, lo1, len1;
};

struct UGeom {
  int p0, p1, wrap, c0, c1;              // position, wrap flag, R window start (unwrapped)
  int R0, R1;                            // R window lengths
  // step s (index s-1): input region X (rows [xr, xr+xrl), cols [xc, xc+xcl), stored from column xb)
  int xr[kMS], xrl[kMS], xc[kMS], xcl[kMS], xb[kMS];
  // pass A: rows [ar, ar+arl) of X, stored in Yt from row-coordinate yb; h cols, g cols
  int ar[kMS], arl[kMS], yb[kMS], hlo[kMS], hlen[kMS], glo[kMS], glen[kMS];
  Box box[kMS][4];                       // outputs per orientation code 0..3 at level s
  int doff[kMS][4];                      // box offsets in the D buffer (all steps kept)
};

__device__ __forceinline__ float fmaT(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fmaT(double a, double b, double c) { return fma(a, b, c); }

template <typename Real>
struct Vec;
template <>
struct Vec<float> {
  static constexpr int W = 4;
  using T = float4;
};
template <>
struct Vec<double> {
  static constexpr int W = 2;
  using T = double2;
};

__device__ __forceinline__ int imin(int a, int b) { return a < b ? a : b; }
__device__ __forceinline__ int imax(int a, int b) { return a > b ? a : b; }
__device__ __forceinline__ int align_down(int a, int w) { return a & ~(w - 1); }

// intersect [lo, lo+len) with [alo, alo+alen)
__device__ __forceinline__ void clip(int& lo, int& len, int alo, int alen) {
  int a = imax(lo, alo), b = imin(lo + len, alo + alen);
  lo = a;
  len = imax(0, b - a);
}
// union bounding interval of [lo, lo+len) and [lo2, lo2+len2) (empty intervals ignored)
__device__ __forceinline__ void hull(int& lo, int& len, int lo2, int len2) {
  if (len2 <= 0) return;
  if (len <= 0) { lo = lo2; len = len2; return; }
  int a = imin(lo, lo2), b = imax(lo + len, lo2 + len2);
  lo = a;
  len = b - a;
}

__device__ __forceinline__ void group_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// 4 consecutive outputs out[q] = Σ_t f_TY[t] · x[2(j0+q) + o_TY + t - base] of a row whose valid
// (computed) entries are the local indices [vlo, vhi); everything else is zero (outside the exact
// support window).  Always 16-byte vector loads (the buffers carry kSL slack on both sides); the
// few edge groups mask the loaded values.  Taps come from the kernel-parameter (constant) bank.
template <typename Real, int L2, int TY>
__device__ __forceinline__ void filt4(const Plan& P, const Real* __restrict__ row, int base, int j0, int nout,
                                      int vlo, int vhi, Real out[4]) {
  constexpr int VW = Vec<Real>::W;
  constexpr int o = TY ? 2 - L2 : 0;
  constexpr int NV = ((2 + 6 + L2) + VW - 1) / VW * VW;     // loads incl. alignment slack
  const int s0 = 2 * j0 + o - base;
  const int a = s0 & ~(VW - 1);
  const int off = s0 - a;                                    // 0 or 2 (float), 0 (double)
  Real x[NV];
  const typename Vec<Real>::T* p = reinterpret_cast<const typename Vec<Real>::T*>(row + a);
#pragma unroll
  for (int i = 0; i < NV / VW; ++i) {
    typename Vec<Real>::T t = p[i];
    if constexpr (VW == 4) {
      x[4 * i] = t.x; x[4 * i + 1] = t.y; x[4 * i + 2] = t.z; x[4 * i + 3] = t.w;
    } else {
      x[2 * i] = t.x; x[2 * i + 1] = t.y;
    }
  }
  if (s0 < vlo || s0 + 2 * (nout - 1) + L2 > vhi) {
#pragma unroll
    for (int i = 0; i < NV; ++i)
      if (a + i < vlo || a + i >= vhi) x[i] = Real(0);
  }
  if (off == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      Real acc = Real(0);
#pragma unroll
      for (int t = 0; t < L2; ++t) acc = fmaT(TapsOf<Real>::get(P, TY, t), x[2 * q + t], acc);
      out[q] = acc;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      Real acc = Real(0);
#pragma unroll
      for (int t = 0; t < L2; ++t) acc = fmaT(TapsOf<Real>::get(P, TY, t), x[2 + 2 * q + t], acc);
      out[q] = acc;
    }
  }
}

}  // namespace

// CTA scratch layout (elements):  [X_0 .. X_{G-1}] [Yt_0 .. Yt_{G-1} ∪ k-sum staging] [D_0 .. D_{G-1}]
// X_u / Yt_u carry kSL slack elements before and after (vector over-reads); D_u is followed by
// the unit's wrap-case stage.  The k-sum staging (two T_k/v_k tile buffers) aliases the Yt
// region, which is idle during the k-sum.
template <typename Real>
__device__ __forceinline__ Real* unit_X(Real* scr, const TileArgs& A, int u) { return scr + u * A.Xsz + kSL; }
template <typename Real>
__device__ __forceinline__ Real* unit_Y(Real* scr, const TileArgs& A, int u) {
  return scr + A.regY + u * A.Ysz + kSL;
}
template <typename Real>
__device__ __forceinline__ Real* unit_D(Real* scr, const TileArgs& A, int u) { return scr + A.regD + u * A.Dsz; }

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// k-sum for G units adjacent along axis 1 (window shift STEP = 2^ℓ per unit): each task holds a
// 4-wide strip of T_k and the (4 + (G-1)·STEP)-wide strip of v_k the G windows read, so one v
// value feeds up to G FMAs.  Both strips are read with 16-byte loads (T rows are aligned; the v
// strip starts at a uniform misalignment c1 mod VW, fixed by a register shift).
template <typename Real, int G, int STEP, int SHIFT>
__device__ __forceinline__ void ksum_task(const Plan& P, const SubBand& S, const Real* __restrict__ vrow,
                                          const Real* __restrict__ trow, Real acc[G][4]) {
  constexpr int VW = Vec<Real>::W;
  constexpr int SPAN = 4 + (G - 1) * STEP;
  constexpr int NV = (SPAN + SHIFT + VW - 1) / VW;
  using V = typename Vec<Real>::T;
#pragma unroll 2
  for (int k = 0; k < P.m; ++k) {
    Real tv[4], vb[NV * VW];
    if constexpr (VW == 4) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(trow));
      tv[0] = q.x; tv[1] = q.y; tv[2] = q.z; tv[3] = q.w;
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const float4 w = __ldg(reinterpret_cast<const float4*>(vrow) + i);
        vb[4 * i] = w.x; vb[4 * i + 1] = w.y; vb[4 * i + 2] = w.z; vb[4 * i + 3] = w.w;
      }
    } else {
      const double2 q0 = __ldg(reinterpret_cast<const double2*>(trow));
      const double2 q1 = __ldg(reinterpret_cast<const double2*>(trow) + 1);
      tv[0] = q0.x; tv[1] = q0.y; tv[2] = q1.x; tv[3] = q1.y;
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const double2 w = __ldg(reinterpret_cast<const double2*>(vrow) + i);
        vb[2 * i] = w.x; vb[2 * i + 1] = w.y;
      }
    }
#pragma unroll
    for (int u = 0; u < G; ++u)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[u][i] = fmaT(vb[SHIFT + u * STEP + i], tv[i], acc[u][i]);
    vrow += P.N;
    trow += S.tstride;
  }
}

template <typename Real, int G, int STEP>
__device__ void ksum_tile(const Plan& P, const TileArgs& A, const SubBand& S, const UGeom* geo, Real* scr) {
  constexpr int VW = Vec<Real>::W;
  constexpr int SPAN = 4 + (G - 1) * STEP;
  const Real* __restrict__ v = reinterpret_cast<const Real*>(A.v);
  const Real* __restrict__ T = reinterpret_cast<const Real*>(A.T) + S.toff;
  const int n = P.n, mask = n - 1;
  const int W0 = geo[0].R0, W1 = geo[0].R1;
  const int groups = (W1 + 3) >> 2;
  const int tasks = W0 * groups;
  const int c0 = geo[0].c0, c1 = geo[0].c1;
  const int sh = c1 & (VW - 1);
  const int c1a = c1 - sh;
  // fast path: every strip inside the row without wrapping, T rows 16-byte aligned
  const bool fast = c1a >= 0 && c1a + ((W1 + 3) & ~3) + SPAN + VW <= n && (S.tRS & 3) == 0 && (S.toff & 3) == 0;
  for (int task = threadIdx.x; task < tasks; task += blockDim.x) {
    const int r = task / groups;
    const int z = (task - r * groups) << 2;
    Real acc[G][4];
#pragma unroll
    for (int u = 0; u < G; ++u)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[u][i] = Real(0);
    const int y0 = (c0 + r) & mask;
    if (fast) {
      const Real* vrow = v + int64_t(y0) * n + c1a + z;
      const Real* trow = T + int64_t(r) * S.tRS + z;
      if constexpr (VW == 4) {
        if (sh == 0) ksum_task<Real, G, STEP, 0>(P, S, vrow, trow, acc);
        else if (sh == 1) ksum_task<Real, G, STEP, 1>(P, S, vrow, trow, acc);
        else if (sh == 2) ksum_task<Real, G, STEP, 2>(P, S, vrow, trow, acc);
        else ksum_task<Real, G, STEP, 3>(P, S, vrow, trow, acc);
      } else {
        if (sh == 0) ksum_task<Real, G, STEP, 0>(P, S, vrow, trow, acc);
        else ksum_task<Real, G, STEP, 1>(P, S, vrow, trow, acc);
      }
    } else {
      const Real* vrow = v + int64_t(y0) * n;
      const Real* trow = T + int64_t(r) * S.tRS + z;
      for (int k = 0; k < P.m; ++k) {
        Real tv[4], vr[SPAN];
#pragma unroll
        for (int i = 0; i < 4; ++i) tv[i] = (z + i < W1) ? __ldg(trow + i) : Real(0);
#pragma unroll
        for (int i = 0; i < SPAN; ++i) vr[i] = __ldg(vrow + ((c1 + z + i) & mask));
#pragma unroll
        for (int u = 0; u < G; ++u)
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[u][i] = fmaT(vr[u * STEP + i], tv[i], acc[u][i]);
        vrow += P.N;
        trow += S.tstride;
      }
    }
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const UGeom& g = geo[u];
      Real* dst = unit_X(scr, A, u) + r * A.XS + (g.c1 + z - g.xb[0]);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (z + i < W1) dst[i] = acc[u][i];
    }
  }
}

template <typename Real, int L2>
__device__ void unit_geometry(const Plan& P, const SubBand& S, int sbi, int sb_first, const int4* sbox,
                              int64_t pos, UGeom& g) {
  constexpr int VW = Vec<Real>::W;
  const int lev = S.level, nl = S.nl, steps = S.steps;
  g.p0 = int(pos / nl);
  g.p1 = int(pos - int64_t(g.p0) * nl);
  g.c0 = (g.p0 << lev) + S.tSu[0];
  g.c1 = (g.p1 << lev) + S.tSu[1];
  g.R0 = S.tW[0];
  g.R1 = S.tW[1];
  // forward: actual windows per step (approx aw, detail dw) per axis
  int aw0[kMS + 1], awl0[kMS + 1], aw1[kMS + 1], awl1[kMS + 1];
  int dw0[kMS + 1], dwl0[kMS + 1], dw1[kMS + 1], dwl1[kMS + 1];
  aw0[0] = g.c0; awl0[0] = g.R0; aw1[0] = g.c1; awl1[0] = g.R1;
#pragma unroll
  for (int s = 1; s <= kMS; ++s) {
    if (s > steps) break;
    int a = aw0[s - 1], b = aw0[s - 1] + awl0[s - 1] - 1;
    aw0[s] = -((-(a - L2 + 1)) >> 1); awl0[s] = (b >> 1) - aw0[s] + 1;
    dw0[s] = -((-(a - 1)) >> 1); dwl0[s] = ((b + L2 - 2) >> 1) - dw0[s] + 1;
    a = aw1[s - 1]; b = aw1[s - 1] + awl1[s - 1] - 1;
    aw1[s] = -((-(a - L2 + 1)) >> 1); awl1[s] = (b >> 1) - aw1[s] + 1;
    dw1[s] = -((-(a - 1)) >> 1); dwl1[s] = ((b + L2 - 2) >> 1) - dw1[s] + 1;
  }
  // backward: needed boxes, clipped to the actual windows
  int wrap = 0;
  int nA0 = 0, nAl0 = 0, nA1 = 0, nAl1 = 0;
  int doff = 0;
#pragma unroll
  for (int s = kMS; s >= 1; --s) {
    if (s > steps) continue;
    const int nls = P.n >> s;
    const int D = s - lev;
    const int b0 = D == 0 ? g.p0 : (D < 0 ? (g.p0 << -D) : (g.p0 >> D));
    const int b1 = D == 0 ? g.p1 : (D < 0 ? (g.p1 << -D) : (g.p1 >> D));
    Box bx[4];
    if (s == steps) {
      nAl0 = nAl1 = 0;
      if (s == P.J) {
        const int4 cb = sbox[(sbi - sb_first) * P.nsb + 0];
        if (cb.x <= cb.y) {
          nA0 = b0 + cb.x; nAl0 = cb.y - cb.x + 1; nA1 = b1 + cb.z; nAl1 = cb.w - cb.z + 1;
          if (nA0 < 0 || nA0 + nAl0 > nls || nA1 < 0 || nA1 + nAl1 > nls) wrap = 1;
        }
      }
    }
    bx[0] = Box{nA0, nAl0, nA1, nAl1};
    clip(bx[0].lo0, bx[0].len0, aw0[s], awl0[s]);
    clip(bx[0].lo1, bx[0].len1, aw1[s], awl1[s]);
    if (bx[0].len0 == 0 || bx[0].len1 == 0) bx[0].len0 = bx[0].len1 = 0;
    for (int ec = 1; ec < 4; ++ec) {
      const int sl = 1 + (P.J - s) * 3 + (ec - 1);
      const int4 b = sbox[(sbi - sb_first) * P.nsb + sl];
      Box o{0, 0, 0, 0};
      if (b.x <= b.y) {
        o = Box{b0 + b.x, b.y - b.x + 1, b1 + b.z, b.w - b.z + 1};
        if (o.lo0 < 0 || o.lo0 + o.len0 > nls || o.lo1 < 0 || o.lo1 + o.len1 > nls) wrap = 1;
        const int e0 = ec >> 1, e1 = ec & 1;
        clip(o.lo0, o.len0, e0 ? dw0[s] : aw0[s], e0 ? dwl0[s] : awl0[s]);
        clip(o.lo1, o.len1, e1 ? dw1[s] : aw1[s], e1 ? dwl1[s] : awl1[s]);
        if (o.len0 == 0 || o.len1 == 0) o.len0 = o.len1 = 0;
      }
      bx[ec] = o;
    }
    const int si = s - 1;
#pragma unroll
    for (int ec = 0; ec < 4; ++ec) g.box[si][ec] = bx[ec];
    int hlo = 0, hlen = 0, glo = 0, glen = 0;
    hull(hlo, hlen, bx[0].lo1, bx[0].len0 ? bx[0].len1 : 0);
    hull(hlo, hlen, bx[2].lo1, bx[2].len0 ? bx[2].len1 : 0);
    hull(glo, glen, bx[1].lo1, bx[1].len0 ? bx[1].len1 : 0);
    hull(glo, glen, bx[3].lo1, bx[3].len0 ? bx[3].len1 : 0);
    g.hlo[si] = hlo; g.hlen[si] = hlen; g.glo[si] = glo; g.glen[si] = glen;
    int rlo = 0, rlen = 0;
    for (int ec = 0; ec < 4; ++ec) {
      if (!bx[ec].len0) continue;
      const int e0 = ec >> 1;
      const int lo = 2 * bx[ec].lo0 + (e0 ? 2 - L2 : 0);
      hull(rlo, rlen, lo, 2 * (bx[ec].len0 - 1) + L2);
    }
    int clo = 0, clen = 0;
    if (hlen) hull(clo, clen, 2 * hlo, 2 * (hlen - 1) + L2);
    if (glen) hull(clo, clen, 2 * glo + 2 - L2, 2 * (glen - 1) + L2);
    clip(rlo, rlen, aw0[s - 1], awl0[s - 1]);
    clip(clo, clen, aw1[s - 1], awl1[s - 1]);
    g.ar[si] = rlo; g.arl[si] = rlen;
    g.yb[si] = align_down(rlo, VW);
    g.xr[si] = rlo; g.xrl[si] = rlen; g.xc[si] = clo; g.xcl[si] = clen;
    g.xb[si] = align_down(clo, VW);
    nA0 = rlo; nAl0 = rlen; nA1 = clo; nAl1 = clen;
    for (int ec = 0; ec < 4; ++ec) {
      g.doff[si][ec] = doff;
      if (ec || s == P.J) doff += bx[ec].len0 * bx[ec].len1;
    }
  }
  g.xr[0] = g.c0; g.xrl[0] = g.R0; g.xc[0] = g.c1; g.xcl[0] = g.R1;
  g.xb[0] = align_down(g.c1, VW);
  g.wrap = wrap;
}

template <typename Real, int L2>
__global__ void __launch_bounds__(kTB) band_tile_kernel(const __grid_constant__ Plan P,
                                                        const __grid_constant__ TileArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ UGeom geo[kG];
  __shared__ int4 sbox[3 * kMaxSB];
  Real* scr = reinterpret_cast<Real*>(smem_raw);
  const int tid = threadIdx.x;
  const int G = A.G;
  const int GT = blockDim.x / G;              // threads per unit group (whole warps)
  const int u = tid / GT, gt = tid - u * GT;  // this thread's unit and rank inside its group
  // stage this launch's stencil rows and offset boxes (≤ 3 sub-bands of one level) in smem
  const int sb_first = find_subband(P, A.u0);
  const int nsbl = find_subband(P, A.u1 - 1) - sb_first + 1;
  int4* sst = reinterpret_cast<int4*>(scr + A.regEnd);
  for (int i = tid; i < nsbl * P.nsb; i += blockDim.x) sbox[i] = A.box[sb_first * P.nsb + i];
  for (int i = tid; i < nsbl * P.band_L; i += blockDim.x) {
    const int q = i / P.band_L, j = i - q * P.band_L;
    sst[i] = A.stencil[P.sb[sb_first + q].stencil_off + j];
  }
  __syncthreads();
  const int64_t rounds = (A.u1 - A.u0) / G;
  unsigned long long* dbg = A.dbg;
  long long acc_[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tlast_ = 0;

  for (int64_t rd = blockIdx.x; rd < rounds; rd += gridDim.x) {
    const int64_t ufirst = A.u0 + rd * G;
    const int sbi = find_subband(P, ufirst);
    const SubBand& S = P.sb[sbi];
    const int lev = S.level, steps = S.steps;
    if (dbg && tid == 0) tlast_ = clock64();
    if (tid < G) unit_geometry<Real, L2>(P, S, sbi, sb_first, sbox, ufirst + tid - S.offset, geo[tid]);
    __syncthreads();
    if (dbg && tid == 0) { long long t_ = clock64(); acc_[2] += t_ - tlast_; tlast_ = t_; }
    // ---------------------------------------------------------------- a2: k-sum (whole CTA)
    if (G == 4 && lev == 1) ksum_tile<Real, 4, 2>(P, A, S, geo, scr);
    else if (G == 2 && lev == 1) ksum_tile<Real, 2, 2>(P, A, S, geo, scr);
    else if (G == 2 && lev == 2) ksum_tile<Real, 2, 4>(P, A, S, geo, scr);
    else if (G == 2 && lev == 3) ksum_tile<Real, 2, 8>(P, A, S, geo, scr);
    else ksum_tile<Real, 1, 1>(P, A, S, geo, scr);
    __syncthreads();
    if (dbg && tid == 0) { long long t_ = clock64(); acc_[3] += t_ - tlast_; tlast_ = t_; }

    // ---------------------------------------------------------------- a3: cascade of unit u
    const UGeom& g = geo[u];
    Real* X = unit_X(scr, A, u);
    Real* Yt = unit_Y(scr, A, u);
    Real* Dd = unit_D(scr, A, u);
    for (int s = 1; s <= steps; ++s) {
      const int si = s - 1;
      // pass A: rows of X (axis-1 filter) -> Yt[col][row]; task = (column group, row), row fastest
      {
        const int hg = (g.hlen[si] + 3) >> 2, gg = (g.glen[si] + 3) >> 2;
        const int rows = g.arl[si];
        const int ntask = (hg + gg) * rows;
        const int xb = g.xb[si], vlo = g.xc[si] - xb, vhi = vlo + g.xcl[si];
        for (int t = gt; t < ntask; t += GT) {
          const int q = t / rows;
          const int rr = t - q * rows;
          const int ty = q >= hg;
          const int j0 = ty ? g.glo[si] + 4 * (q - hg) : g.hlo[si] + 4 * q;
          const int jend = ty ? g.glo[si] + g.glen[si] : g.hlo[si] + g.hlen[si];
          const int nout = imin(4, jend - j0);
          const int r = g.ar[si] + rr;
          const Real* xrow = X + (r - g.xr[si]) * A.XS;
          Real out[4];
          if (ty) filt4<Real, L2, 1>(P, xrow, xb, j0, nout, vlo, vhi, out);
          else filt4<Real, L2, 0>(P, xrow, xb, j0, nout, vlo, vhi, out);
          const int ycol0 = ty ? g.hlen[si] + (j0 - g.glo[si]) : (j0 - g.hlo[si]);
          Real* yd = Yt + ycol0 * A.YS + (r - g.yb[si]);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (i < nout) yd[i * A.YS] = out[i];
        }
      }
      group_sync(1 + u, GT);
      // pass B: Yt rows (axis-0 filter) -> approx box (next X) and detail boxes (D);
      // task = (box, row group, column), column fastest
      {
        const bool want0 = s < steps || s == P.J;
        int cnt[4];
#pragma unroll
        for (int ec = 0; ec < 4; ++ec) {
          const Box& b = g.box[si][ec];
          cnt[ec] = (ec == 0 && !want0) ? 0 : ((b.len0 + 3) >> 2) * b.len1;
        }
        const int ntask = cnt[0] + cnt[1] + cnt[2] + cnt[3];
        const int yb = g.yb[si], vlo = g.ar[si] - yb, vhi = vlo + g.arl[si];
        for (int t = gt; t < ntask; t += GT) {
          int ec = 0, idx = t;
          while (idx >= cnt[ec]) { idx -= cnt[ec]; ++ec; }
          const Box& b = g.box[si][ec];
          const int q = idx / b.len1;
          const int cc = idx - q * b.len1;
          const int e0 = ec >> 1, e1 = ec & 1;
          const int l0 = b.lo0 + 4 * q;
          const int nrow = imin(4, b.len0 - 4 * q);
          const int j = b.lo1 + cc;
          const int ycol = e1 ? g.hlen[si] + (j - g.glo[si]) : (j - g.hlo[si]);
          Real out[4];
          if (e0) filt4<Real, L2, 1>(P, Yt + ycol * A.YS, yb, l0, nrow, vlo, vhi, out);
          else filt4<Real, L2, 0>(P, Yt + ycol * A.YS, yb, l0, nrow, vlo, vhi, out);
          if (ec == 0 && s < steps) {
            Real* xd = X + (l0 - g.xr[si + 1]) * A.XS + (j - g.xb[si + 1]);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (i < nrow) xd[i * A.XS] = out[i];
          } else {
            Real* dd = Dd + g.doff[si][ec] + (4 * q) * b.len1 + cc;
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (i < nrow) dd[i * b.len1] = out[i];
          }
        }
      }
      group_sync(1 + u, GT);
    }
    if (dbg && tid == 0) { long long t_ = clock64(); acc_[4] += t_ - tlast_; tlast_ = t_; }
    // ---------------------------------------------------------------- a4: gather + write row
    {
      const int4* st = sst + (sbi - sb_first) * P.band_L;
      const int L = P.band_L;
      const int64_t base = (ufirst + u - A.row0) * L;
      Real* outv = reinterpret_cast<Real*>(A.val);
      Real* sv = Dd + A.DMAX;   // wrap-case stage follows D
      int* sc = reinterpret_cast<int*>(sv + P.band_Lpad);
      for (int jj = gt; jj < L; jj += GT) {
        const int4 e = st[jj];
        const int s = e.w, si = s - 1;              // .w = level of the partner sub-band
        const SubBand& Lb = P.sb[e.x];
        const int D = s - lev;
        const int b0 = D == 0 ? g.p0 : (D < 0 ? (g.p0 << -D) : (g.p0 >> D));
        const int b1 = D == 0 ? g.p1 : (D < 0 ? (g.p1 << -D) : (g.p1 >> D));
        const int l0 = b0 + e.y, l1 = b1 + e.z;
        const Box& b = g.box[si][Lb.e];
        Real x = Real(0);
        const int i0 = l0 - b.lo0, i1 = l1 - b.lo1;
        if (i0 >= 0 && i0 < b.len0 && i1 >= 0 && i1 < b.len1) x = Dd[g.doff[si][Lb.e] + i0 * b.len1 + i1];
        const int c = int(Lb.offset + int64_t(l0 & (Lb.nl - 1)) * Lb.nl + (l1 & (Lb.nl - 1)));
        if (!g.wrap) {
          A.col[base + jj] = c;
          outv[base + jj] = x;
        } else {
          sv[jj] = x;
          sc[jj] = c;
        }
      }
      if (g.wrap) {          // a partner wraps around the torus: place by rank of the column
        group_sync(1 + u, GT);
        for (int jj = gt; jj < L; jj += GT) {
          const int c = sc[jj];
          int rank = 0;
          for (int i = 0; i < L; ++i) rank += sc[i] < c;
          A.col[base + rank] = c;
          outv[base + rank] = sv[jj];
        }
      }
    }
    __syncthreads();
    if (dbg && tid == 0) { long long t_ = clock64(); acc_[5] += t_ - tlast_; tlast_ = t_; }
  }
  if (dbg && tid == 0)
    for (int i = 0; i < 8; ++i) atomicAdd(dbg + i, (unsigned long long)acc_[i]);
}

// ---------------------------------------------------------------------------------- launcher

template <typename Real, int L2>
static cudaError_t launch_tile_t(const Plan& P, const TileArgs& A, int grid, size_t smem, cudaStream_t st) {
  auto k = band_tile_kernel<Real, L2>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
  }
  k<<<grid, kTB, smem, st>>>(P, A);
  return cudaGetLastError();
}

cudaError_t launch_band_tile(const Plan& P, const TileArgs& A, int real_bytes, int grid, size_t smem,
                             cudaStream_t st) {
#define PCWD_TILE_CASE(LL)                                                                   \
  case LL:                                                                                   \
    return real_bytes == 4 ? launch_tile_t<float, LL>(P, A, grid, smem, st)                  \
                           : launch_tile_t<double, LL>(P, A, grid, smem, st);
  switch (P.L2) {
    PCWD_TILE_CASE(2)
    PCWD_TILE_CASE(4)
    PCWD_TILE_CASE(6)
    PCWD_TILE_CASE(8)
    PCWD_TILE_CASE(12)
  }
#undef PCWD_TILE_CASE
  return cudaErrorInvalidValue;
}

}  // namespace pcwd
