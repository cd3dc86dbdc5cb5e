// common.h — plan structures and window arithmetic shared by the host planner and the kernels.
//
// Index conventions:
//   * grid row-major, axis 0 = rows, axis 1 = columns; d = 1 is stored as axis 1 only
//     (axis 0 has one position and is never filtered)
//   * one analysis step on a periodic line of length n':
//         out_e[l] = Σ_j f_e[j] · x[(2l + o_e + j) mod n'],  j ∈ [0, 2δ)
//     with f_0 = h, o_0 = 0 (approximation) and f_1[j] = g[2-2δ+j] = (-1)^{1-i} h[1-i]
//     (i = 2-2δ+j), o_1 = 2-2δ (detail)
//   * a window is a Range: positions (lo + i) mod nl for i < len, the signal being exactly
//     zero elsewhere on the line (Lemma 6, made exact by index arithmetic).
//     len == nl means the whole periodic line (lo = 0).
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define PCWD_HD __host__ __device__ __forceinline__
#else
#define PCWD_HD inline
#endif

namespace pcwd {

constexpr int kMaxJ = 16;
constexpr int kMaxSB = 1 + 3 * kMaxJ;
constexpr int kMaxTaps = 20;

enum Mode : int { MODE_FULL = 0, MODE_BAND = 1, MODE_TMAX = 2, MODE_TCOUNT = 3, MODE_TWRITE = 4, MODE_TSTORE = 5,
                  MODE_PATTERN = 6 };

struct Range {
  int lo, len, nl;
};

PCWD_HD int floordiv2(int a) { return a >> 1; }          // arithmetic shift: floor(a/2)
PCWD_HD int ceildiv2(int a) { return -((-a) >> 1); }

PCWD_HD Range full_range(int nl) { return Range{0, nl, nl}; }

// Output window of one analysis step (approximation: detail = 0; detail: detail = 1).
// a[l] touches x[2l .. 2l+L2-1]; d[l] touches x[2l+2-L2 .. 2l+1].
PCWD_HD Range step_out(Range in, int L2, int detail) {
  int half = in.nl >> 1;
  if (in.len >= in.nl) return full_range(half);
  int a = in.lo, b = in.lo + in.len - 1;
  int lo = detail ? ceildiv2(a - 1) : ceildiv2(a - L2 + 1);
  int hi = detail ? floordiv2(b + L2 - 2) : floordiv2(b);
  int len = hi - lo + 1;
  if (len >= half) return full_range(half);
  return Range{lo & (half - 1), len, half};
}

// Upper bound of step_out(...).len over the parity of in.lo.
PCWD_HD int step_out_maxlen(int len_in, int nl_in, int L2) {
  int half = nl_in >> 1;
  if (len_in >= nl_in) return half;
  int l = (len_in >> 1) + (L2 >> 1);
  return l < half ? l : half;
}

// Local index of global position g in r, or -1 when g is outside the window.
PCWD_HD int local_index(const Range& r, int g) {
  int li = (g - r.lo) & (r.nl - 1);
  return li < r.len ? li : -1;
}

// k-th smallest global position of a window -> its local index (CSR column order).
PCWD_HD int sorted_to_local(const Range& r, int k) {
  if (r.len >= r.nl) return k;
  int start = r.lo & (r.nl - 1);
  if (start + r.len <= r.nl) return k;
  int i = k + (r.nl - start);
  return i >= r.len ? i - r.len : i;
}

struct SubBand {
  int level;        // ℓ: number of analysis steps (1 = finest)
  int e;            // 0 = coarse scaling block (ℓ = J); d=2: 1=(0,1) 2=(1,0) 3=(1,1); d=1: 1
  int e0, e1;       // orientation bit per axis
  int nl;           // positions per axis (n >> ℓ)
  int steps;        // cascade steps a unit of this sub-band needs
  int64_t offset;   // first Λ index
  int64_t count;    // nl^d
  // convolved template T_{k,s} = ũ_k ⋆ ψ_{s,0}: window per axis (tW == n ⇒ whole line, tS = 0)
  int tS[2], tW[2];
  int64_t toff;     // template buffer offset of k = 0 (elements); k-th at toff + k * tstride
  int64_t tstride;  // = tW[0] * tRS
  int tRS;          // template row stride (tW[1] rounded up to 4 unless the row is a whole line)
  // per-unit scratch layout (elements of the compute type)
  int64_t offX0, offX1, offY, offD, offStage, scratch;
  // hybrid layout (global-scratch launches): the buffers of steps ≥ 2 and the step-1 approximation in shared
  // memory (elements): approximations X1 (steps 1, 3, …) and X2 (steps 2, 4, …), pass-A output Y and detail
  // boxes D of steps ≥ 2; hs_size = their total
  int64_t hs_X1, hs_X2, hs_Y, hs_D, hs_size;
  int stencil_off;  // BAND: first entry of this sub-band's stencil
  int any_full;     // some window of this sub-band covers a whole line (general path only)
  int tSu[2];       // template window start, unwrapped: -zhi + (e_a ? 2^{ℓ-1}(2-2δ) : 0)
  // warp-per-unit band kernel (band_warp.cu): eligibility and per-warp scratch layout
  int wk_ok;
  int64_t wk_offY, wk_offD, wk_offStage, wk_scratch;
  double fma;       // algorithmic FMA per unit (k-sum + cascade, max windows)
  int fg_off, fg_m; // fine path: first geometry record of this sub-band, class modulus per axis (geom.h)
  // THRESHOLD store-then-filter: candidate slot of this sub-band's first shard unit, and per-unit slot size
  int64_t cand_off, cand_slot;
};

struct Plan {
  int d, n, J, L2, m, nsb;
  int64_t N;
  int retain;       // pcwd_retain
  int band_L, band_Lpad;
  int zlo[2], zhi[2];   // periodic bounding box of the nonzeros of all u_k (offsets)
  float tf[2][kMaxTaps];
  double td[2][kMaxTaps];
  int to[2];            // tap offsets o_0 = 0, o_1 = 2 - L2
  SubBand sb[kMaxSB];
};

template <typename Real>
struct TapsOf;
template <>
struct TapsOf<float> {
  PCWD_HD static float get(const Plan& P, int e, int j) { return P.tf[e][j]; }
};
template <>
struct TapsOf<double> {
  PCWD_HD static double get(const Plan& P, int e, int j) { return P.td[e][j]; }
};

// Window of unit μ = (sub-band s, position p) on axis a: the template window shifted by 2^ℓ p.
PCWD_HD Range unit_window(const Plan& P, const SubBand& s, int a, int p) {
  if (s.tW[a] >= P.n) return full_range(P.n);
  return Range{((p << s.level) + s.tS[a]) & (P.n - 1), s.tW[a], P.n};
}

PCWD_HD int find_subband(const Plan& P, int64_t unit) {   // largest s with sb[s].offset <= unit
  int lo = 0, hi = P.nsb - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (P.sb[mid].offset <= unit) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

}  // namespace pcwd
