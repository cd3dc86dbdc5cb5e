// approx.cu — Algorithm 1 of the paper, the η-approximation Θ̃ = Σ_k Ã_k B_k,
// and the operator application H f = Σ_k u_k ⋆ (v_k ⊙ f) / H* g (Eq. 2) used to check ‖Θ − Θ̃‖₂ ≤ η.
//
// Algorithm 1 on the GPU (fp64, as the paper ran it):
//   * A_k = Ψ* U_k Ψ has circulant sub-bands (Lemma 1): row μ is Ψ*(ũ_k ⋆ ψ_μ) = Ψ*(τ_{2^ℓ p} T_{k,s}), the
//     cascade of the shifted convolved template (a1), and every row of a (sub-band s, class q = p mod 2^{J−ℓ}) is a
//     translate of the class representative's row by a multiple of 2^J pixels — a whole number of positions at
//     every level.  One CTA per class computes the representative row of every A_k once.
//   * Ã_k: A_k truncated by Theorem 2's Remark: entries with (i) |ℓ_λ − ℓ_μ| > S_k or (ii)
//     ϑ(λ,μ) > 2^{S_k} (Definition 1) are zeroed; S_k is the smallest S whose dropped part has Schur bound
//     sqrt(‖E‖₁‖E‖_∞) ≤ ε_k = η/(m‖v_k‖∞), so ‖A_k − Ã_k‖₂ ≤ ε_k (DESIGN.md R-A1..R-A3).  The row sums of
//     E come from the class representatives' rows, the column sums from the same rows folded by the translation
//     group (column ν of E sums the representatives' entries over ν's class) — approx_stats_kernel.
//   * C_k = Ã_k B_k, B_k = Ψ*V_kΨ: row μ of Ã_kB_k = (B_k ã_μ)ᵀ = (Ψ*(v_k ⊙ Ψ ã_μ))ᵀ — the product
//     over the predicted locations taken in the spatial domain.  Per class: G_k = Ψ ã_{k,q} (inverse
//     cascade of the truncated representative row); per unit of the class: R = Σ_k v_k ⊙ τ_{2^J t} G_k, then
//     Θ̃[μ][·] = Ψ* R (accumulation over k before the cascade, by linearity).
//   * The output is Θ̃ on its predicted support (𝒮 of Lemma 9): the λ whose ψ_λ meets some
//     ψ_ν with Ã_k[μ][ν] ≠ 0, found by |tap| cascades (no cancellation) — CSR with increasing columns, by a count
//     pass and a write pass (the per-unit work is recomputed).
// Every transform is a whole-torus periodic cascade of one CTA in global (L2) scratch: this path is meant for the
// paper's η sweeps (Fig. 3, N = 256²), not for the 1024² exact-path sizes.
#include <algorithm>
#include <cstdint>

#include "kernels.cuh"

namespace pcwd {

namespace {
constexpr int kAB = 512;   // threads per CTA
constexpr int kSB = 64;    // histogram bins of the truncation index S (S ≥ 63 clamps)

__device__ __forceinline__ int wrap(int a, int n) { return a & (n - 1); }

// One periodic analysis step of a line family.  In: x[r][i] rows of length ns (stride ns), `lines` lines.
// Out: approximation a[r][l], detail d[r][l] (stride half) — P:96, P:100:
//   a[l] = Σ_t h[t] x[(2l + t) mod ns],  d[l] = Σ_j g_j x[(2l + o1 + j) mod ns]  (taps fold when 2δ > ns)
// `col` = true filters along the slow axis (x[i][c], lines = columns), else along rows.
template <bool ABS>
__device__ __forceinline__ double tap(const Plan& P, int e, int t) { return ABS ? fabs(P.td[e][t]) : P.td[e][t]; }

template <bool ABS = false>
__device__ void analysis_pass(const Plan& P, const double* __restrict__ x, double* __restrict__ a, double* __restrict__ d,
                              int ns, int lines, bool col, int64_t a_ld, int64_t d_ld) {
  const int half = ns >> 1, L2 = P.L2, o1 = P.to[1];
  const int total = half * lines;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int l = col ? idx / lines : idx % half;
    const int r = col ? idx % lines : idx / half;
    double sa = 0.0, sd = 0.0;
    for (int t = 0; t < L2; ++t) {
      const int ia = wrap(2 * l + t, ns), id = wrap(2 * l + o1 + t, ns);
      const double xa = col ? x[int64_t(ia) * ns + r] : x[int64_t(r) * ns + ia];
      const double xd = col ? x[int64_t(id) * ns + r] : x[int64_t(r) * ns + id];
      sa = fma(tap<ABS>(P, 0, t), xa, sa);
      sd = fma(tap<ABS>(P, 1, t), xd, sd);
    }
    if (col) { a[int64_t(l) * a_ld + r] = sa; d[int64_t(l) * d_ld + r] = sd; }
    else { a[int64_t(r) * a_ld + l] = sa; d[int64_t(r) * d_ld + l] = sd; }
  }
}

// Its adjoint (= inverse, the step is orthogonal) as a gather: x[i] = Σ_t h[t] a[(i − t)/2] over the t with
// i − t even, plus Σ_j g_j d[(i − o1 − j)/2] over the j with i − o1 − j even (indices mod ns).
template <bool ABS = false>
__device__ void synthesis_pass(const Plan& P, const double* __restrict__ a, const double* __restrict__ d,
                               double* __restrict__ x, int ns, int lines, bool col, int64_t a_ld, int64_t d_ld) {
  const int L2 = P.L2, o1 = P.to[1];
  const int total = ns * lines;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int i = col ? idx / lines : idx % ns;
    const int r = col ? idx % lines : idx / ns;
    double s = 0.0;
    for (int t = (i & 1); t < L2; t += 2) {
      const int l = wrap(i - t, ns) >> 1;
      s = fma(tap<ABS>(P, 0, t), col ? a[int64_t(l) * a_ld + r] : a[int64_t(r) * a_ld + l], s);
    }
    for (int j = ((i - o1) & 1); j < L2; j += 2) {
      const int l = wrap(i - o1 - j, ns) >> 1;
      s = fma(tap<ABS>(P, 1, j), col ? d[int64_t(l) * d_ld + r] : d[int64_t(r) * d_ld + l], s);
    }
    if (col) x[int64_t(i) * lines + r] = s;
    else x[int64_t(r) * ns + i] = s;
  }
}

// Ψ*: x (N, destroyed) → c (N, Λ layout).  y: N scratch.  ABS: the same cascade with |h|, |g| — on a nonnegative
// input, coefficient λ is > 0 exactly when supp ψ_λ meets the input's support (no cancellation).
template <bool ABS = false>
__device__ void forward_full(const Plan& P, double* x, double* c, double* y) {
  const int n = P.n, J = P.J;
  for (int s = 1; s <= J; ++s) {
    const int ns = n >> (s - 1), half = ns >> 1;
    const int base = 1 + (J - s) * (P.d == 2 ? 3 : 1);
    if (P.d == 1) {
      analysis_pass<ABS>(P, x, y, c + P.sb[base].offset, ns, 1, false, half, half);
      __syncthreads();
      for (int i = threadIdx.x; i < half; i += blockDim.x) x[i] = y[i];
      __syncthreads();
      continue;
    }
    // axis 0 (columns): y[0 .. half) = approximation rows, y[half .. ns) = detail rows
    analysis_pass<ABS>(P, x, y, y + int64_t(half) * ns, ns, ns, true, ns, ns);
    __syncthreads();
    // axis 1 (rows): approximation rows → (0,0) into x, (0,1); detail rows → (1,0), (1,1)
    analysis_pass<ABS>(P, y, x, c + P.sb[base].offset, ns, half, false, half, half);
    analysis_pass<ABS>(P, y + int64_t(half) * ns, c + P.sb[base + 1].offset, c + P.sb[base + 2].offset, ns, half, false,
                  half, half);
    __syncthreads();
  }
  const int nJ = n >> J;
  const int cnt = P.d == 2 ? nJ * nJ : nJ;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) c[i] = x[i];
  __syncthreads();
}

// Ψ: c (N, Λ layout) → x (N).  y: N scratch.  ABS: |taps| (a nonnegative c gives x > 0 exactly on the union of
// the supports of the ψ_ν with c_ν > 0).
template <bool ABS = false>
__device__ void inverse_full(const Plan& P, const double* c, double* x, double* y) {
  const int n = P.n, J = P.J;
  const int nJ = n >> J;
  const int cnt = P.d == 2 ? nJ * nJ : nJ;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) x[i] = c[i];
  __syncthreads();
  for (int s = J; s >= 1; --s) {
    const int ns = n >> (s - 1), half = ns >> 1;
    const int base = 1 + (J - s) * (P.d == 2 ? 3 : 1);
    if (P.d == 1) {
      for (int i = threadIdx.x; i < half; i += blockDim.x) y[i] = x[i];
      __syncthreads();
      synthesis_pass<ABS>(P, y, c + P.sb[base].offset, x, ns, 1, false, half, half);
      __syncthreads();
      continue;
    }
    // rows: (x, (0,1)) → y[0 .. half) rows of length ns; ((1,0), (1,1)) → y[half .. ns)
    synthesis_pass<ABS>(P, x, c + P.sb[base].offset, y, ns, half, false, half, half);
    synthesis_pass<ABS>(P, c + P.sb[base + 1].offset, c + P.sb[base + 2].offset, y + int64_t(half) * ns, ns, half, false,
                   half, half);
    __syncthreads();
    // columns: (y rows 0..half, y rows half..ns) → x (ns × ns)
    synthesis_pass<ABS>(P, y, y + int64_t(half) * ns, x, ns, ns, true, ns, ns);
    __syncthreads();
  }
}

// Periodic support box of ψ_(s, p) on axis a (P:103-104 with reading R7): start (mod n) and length.
__device__ __forceinline__ void supp_box(const Plan& P, const SubBand& S, int a, int p, int* st, int* len) {
  const int delta = P.L2 >> 1;
  const int64_t L = (int64_t(1) << S.level) - 1;
  const int64_t Ll = L * (2 * delta - 1) + 1;
  const int bit = a == 0 ? S.e0 : S.e1;
  if (Ll >= P.n) { *st = 0; *len = P.n; return; }
  const int64_t s0 = (int64_t(p) << S.level) + (bit ? (int64_t(1) << (S.level - 1)) * (2 - 2 * delta) : 0);
  *st = int(((s0 % P.n) + P.n) % P.n);
  *len = int(Ll);
}

__device__ __forceinline__ int64_t axis_gap(int s1, int L1, int s2, int L2, int n) {
  if (L1 >= n || L2 >= n) return 0;
  const int d = wrap(s2 - s1, n);
  if (d <= L1 - 1 || n - d <= L2 - 1) return 0;
  return min(d - (L1 - 1), (n - d) - (L2 - 1));
}

// Truncation index of Theorem 2's Remark: the smallest S with |ℓ_μ − ℓ_ν| ≤ S and
// dist(supp ψ_μ, supp ψ_ν) ≤ (2^S − 1)·2^{ℓ_c} (ϑ ≤ 2^S, Definition 1; ℓ_c the coarser level).
__device__ int s_keep(const Plan& P, int sm, int pm0, int pm1, int sn, int pn0, int pn1) {
  const SubBand& A = P.sb[sm];
  const SubBand& B = P.sb[sn];
  int64_t dist2 = 0;
  for (int a = (P.d == 2 ? 0 : 1); a < 2; ++a) {
    int s1, l1, s2, l2;
    supp_box(P, A, a, a == 0 ? pm0 : pm1, &s1, &l1);
    supp_box(P, B, a, a == 0 ? pn0 : pn1, &s2, &l2);
    const int64_t g = axis_gap(s1, l1, s2, l2, P.n);
    dist2 += g * g;
  }
  int S = abs(A.level - B.level);
  const int lc = max(A.level, B.level);
  while (S < kSB - 1) {
    const int64_t reach = ((int64_t(1) << S) - 1) << lc;
    if (reach * reach >= dist2) break;
    ++S;
  }
  return S;
}

// Magnitude rule ("simply threshold A", the Remark's alternative): bin b of |a| ∈ [2^{-b-1}, 2^{-b}) (exact,
// from the binary exponent), clamped to [0, 62]; index S keeps the bins b ≤ S, i.e. |a| ≥ 2^{-(S+1)} (S = −1: none).
// Power-of-two thresholds keep the decision away from rounding (a GPU/oracle flip needs |a| within an ulp of 2^-e).
__device__ __forceinline__ int mag_bin(double a) {
  int x;
  frexp(fabs(a), &x);   // |a| = f·2^x, f ∈ [½, 1)
  return min(max(-x, 0), 62);
}

// Λ index → (sub-band, p0, p1)
__device__ __forceinline__ void locate(const Plan& P, int64_t idx, int* s, int* p0, int* p1) {
  *s = find_subband(P, idx);
  const SubBand& S = P.sb[*s];
  const int64_t pos = idx - S.offset;
  *p0 = P.d == 2 ? int(pos / S.nl) : 0;
  *p1 = P.d == 2 ? int(pos - int64_t(*p0) * S.nl) : int(pos);
}

// x = τ_{2^ℓ p} T_{k,s} on the torus (zero elsewhere): the template window placed as in unit_kernel's k-sum.
__device__ void place_template(const Plan& P, const SubBand& S, const double* __restrict__ T, int k, int p0, int p1,
                               double* x) {
  const int n = P.n;
  const int64_t N = P.N;
  for (int64_t i = threadIdx.x; i < N; i += blockDim.x) x[i] = 0.0;
  __syncthreads();
  const int w0 = P.d == 2 ? min(S.tW[0], n) : 1, w1 = min(S.tW[1], n);
  const int b0 = P.d == 2 ? (S.tW[0] >= n ? (p0 << S.level) : S.tS[0] + (p0 << S.level)) : 0;
  const int b1 = S.tW[1] >= n ? (p1 << S.level) : S.tS[1] + (p1 << S.level);
  const double* Tk = T + S.toff + int64_t(k) * S.tstride;
  for (int idx = threadIdx.x; idx < w0 * w1; idx += blockDim.x) {
    const int i0 = idx / w1, i1 = idx - i0 * w1;
    const int y0 = P.d == 2 ? wrap(b0 + i0, n) : 0, y1 = wrap(b1 + i1, n);
    x[int64_t(y0) * n + y1] = Tk[int64_t(i0) * S.tRS + i1];
  }
  __syncthreads();
}

__device__ __forceinline__ int class_mod(const Plan& P, const SubBand& S) { return 1 << (P.J - S.level); }

__device__ __forceinline__ int64_t class_of(const Plan& P, const ApproxArgs& A, int s, int p0, int p1) {
  const int M = class_mod(P, P.sb[s]);
  return A.clsbase[s] + (P.d == 2 ? int64_t(p0 & (M - 1)) * M + (p1 & (M - 1)) : (p1 & (M - 1)));
}

// class c → (sub-band, representative position q)
__device__ __forceinline__ void class_rep(const Plan& P, const ApproxArgs& A, int64_t c, int* s, int* q0, int* q1) {
  int sb = 0;
  while (sb + 1 < P.nsb && A.clsbase[sb + 1] <= c) ++sb;
  const int M = class_mod(P, P.sb[sb]);
  const int64_t r = c - A.clsbase[sb];
  *s = sb;
  *q0 = P.d == 2 ? int(r / M) : 0;
  *q1 = P.d == 2 ? int(r % M) : int(r);
}

// Pass 0: for every class and k, |A_k[μ_c][ν]| summed by truncation index S (row sums) and into ν's class
// (column sums, global fp64 atomics).
__global__ void __launch_bounds__(kAB) approx_stats_kernel(const __grid_constant__ Plan P,
                                                           const __grid_constant__ ApproxArgs A) {
  __shared__ double hist[kSB];
  double* x = A.scratch + int64_t(blockIdx.x) * A.cstride;
  double* y = x + P.N;
  double* c = y + P.N;
  for (int64_t cl = blockIdx.x; cl < A.ncls; cl += gridDim.x) {
    int s, q0, q1;
    class_rep(P, A, cl, &s, &q0, &q1);
    for (int k = 0; k < P.m; ++k) {
      for (int i = threadIdx.x; i < kSB; i += blockDim.x) hist[i] = 0.0;
      place_template(P, P.sb[s], A.T, k, q0, q1, x);
      forward_full(P, x, c, y);
      for (int64_t i = threadIdx.x; i < P.N; i += blockDim.x) {
        const double a = fabs(c[i]);
        if (a == 0.0) continue;
        int sn, p0, p1;
        locate(P, i, &sn, &p0, &p1);
        const int S = A.rule == 0 ? s_keep(P, s, q0, q1, sn, p0, p1) : mag_bin(c[i]);
        atomicAdd(&hist[S], a);
        atomicAdd(&A.colhist[(class_of(P, A, sn, p0, p1) * P.m + k) * kSB + S], a);
      }
      __syncthreads();
      for (int i = threadIdx.x; i < kSB; i += blockDim.x) A.rowhist[(cl * P.m + k) * kSB + i] = hist[i];
      __syncthreads();
    }
  }
}

// Passes 1 (count) and 2 (write): per class, G_k = Ψ ã_{k,q}; per unit of the class, Θ̃[μ][·] = Ψ*(Σ_k v_k ⊙ τ G_k),
// output on the predicted support (Lemma 9's 𝒮 = supp F·I): the λ whose support meets the
// support of some ψ_ν with Ã_k[μ][ν] ≠ 0 — index arithmetic done by the |tap| cascades (the spatial round trip
// leaves rounding noise outside it, which is not part of Θ̃).
template <bool WRITE, typename OutT>
__global__ void __launch_bounds__(kAB) approx_rows_kernel(const __grid_constant__ Plan P,
                                                          const __grid_constant__ ApproxArgs A) {
  __shared__ int wsum[kAB / 32];
  const int64_t N = P.N;
  double* x = A.scratch + int64_t(blockIdx.x) * A.cstride;
  double* y = x + N;
  double* c = y + N;
  double* kap = c + N;                     // kept-ν indicator of the class row, then each unit's support
  double* mk = kap + N;                    // ∪ supp ψ_ν over the kept ν (> 0 there)
  double* G = mk + N;                      // m × N
  const int n = P.n, nJ = n >> P.J;
  const int tcount = P.d == 2 ? nJ * nJ : nJ;
  OutT* val = reinterpret_cast<OutT*>(A.val);
  for (int64_t cl = blockIdx.x; cl < A.ncls; cl += gridDim.x) {
    int s, q0, q1;
    class_rep(P, A, cl, &s, &q0, &q1);
    const SubBand& S = P.sb[s];
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) kap[i] = 0.0;
    __syncthreads();
    for (int k = 0; k < P.m; ++k) {
      double* Gk = G + int64_t(k) * N;
      if (A.S[k] < 0) {   // Ã_k = 0
        for (int64_t i = threadIdx.x; i < N; i += blockDim.x) Gk[i] = 0.0;
        __syncthreads();
        continue;
      }
      place_template(P, S, A.T, k, q0, q1, x);
      forward_full(P, x, c, y);
      for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {   // Ã_k row: rule (i)/(ii) with S_k
        if (c[i] == 0.0) continue;
        int sn, p0, p1;
        locate(P, i, &sn, &p0, &p1);
        if ((A.rule == 0 ? s_keep(P, s, q0, q1, sn, p0, p1) : mag_bin(c[i])) > A.S[k]) c[i] = 0.0;
        else kap[i] = 1.0;
      }
      __syncthreads();
      inverse_full(P, c, Gk, y);
    }
    inverse_full<true>(P, kap, mk, y);
    const int M = class_mod(P, S);
    for (int t = 0; t < tcount; ++t) {
      const int t0 = P.d == 2 ? t / nJ : 0, t1 = P.d == 2 ? t % nJ : t;
      const int p0 = q0 + M * t0, p1 = q1 + M * t1;
      const int64_t unit = S.offset + (P.d == 2 ? int64_t(p0) * S.nl + p1 : p1);
      const int sh0 = P.d == 2 ? (t0 << P.J) : 0, sh1 = t1 << P.J;   // τ_{2^J t}: 2^ℓ (p − q) pixels
      for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
        const int y0 = P.d == 2 ? int(i / n) : 0, y1 = int(i - int64_t(y0) * n);
        const int64_t src = P.d == 2 ? int64_t(wrap(y0 - sh0, n)) * n + wrap(y1 - sh1, n) : wrap(y1 - sh1, n);
        x[i] = mk[src];
      }
      __syncthreads();
      forward_full<true>(P, x, kap, y);   // kap[λ] > 0: λ in the predicted support of this row
      for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
        const int y0 = P.d == 2 ? int(i / n) : 0, y1 = int(i - int64_t(y0) * n);
        const int64_t src = P.d == 2 ? int64_t(wrap(y0 - sh0, n)) * n + wrap(y1 - sh1, n) : wrap(y1 - sh1, n);
        double r = 0.0;
        for (int k = 0; k < P.m; ++k) r = fma(A.v[int64_t(k) * N + i], G[int64_t(k) * N + src], r);
        x[i] = r;
      }
      __syncthreads();
      forward_full(P, x, c, y);
      if (!WRITE) {
        int64_t cnt = 0;
        for (int64_t i0 = 0; i0 < N; i0 += blockDim.x) {
          const int64_t i = i0 + threadIdx.x;
          cnt += __syncthreads_count(i < N && kap[i] > 0.0);
        }
        if (threadIdx.x == 0) A.cnt[unit] = cnt;
      } else {
        int64_t base = A.row_ptr[unit];
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        for (int64_t i0 = 0; i0 < N; i0 += blockDim.x) {   // compaction in column (Λ) order
          const int64_t i = i0 + threadIdx.x;
          const bool keep = i < N && kap[i] > 0.0;
          const unsigned b = __ballot_sync(0xffffffffu, keep);
          if (lane == 0) wsum[w] = __popc(b);
          __syncthreads();
          int before = 0, total = 0;
          for (int q = 0; q < int(blockDim.x >> 5); ++q) {
            if (q < w) before += wsum[q];
            total += wsum[q];
          }
          if (keep) {
            const int64_t pos = base + before + __popc(b & ((1u << lane) - 1u));
            A.col[pos] = int32_t(i);
            val[pos] = OutT(c[i]);
          }
          base += total;
          __syncthreads();
        }
      }
      __syncthreads();
    }
  }
}

// Algorithm 2's column orientation, fixed λ: w_λ = H ψ_λ = Σ_k u_k ⋆ (v_k ⊙ ψ_λ), then Θ[·][λ] = Ψ* w_λ.
// One CTA per requested λ: ψ_λ = Ψ e_λ (whole-torus inverse cascade); q_k = v_k ⊙ ψ_λ on supp ψ_λ; w_λ(x) =
// Σ_{y ∈ supp ψ_λ} Σ_k q_k(y) u_k(x − y) over the box supp ψ_λ ⊕ box(u) (zero elsewhere); Ψ* w_λ by the whole-torus
// forward cascade.  Scratch per CTA: (3 + m) N doubles.
template <typename Real>
__global__ void __launch_bounds__(kAB) column_kernel(const __grid_constant__ Plan P, const double* __restrict__ u,
                                                     const Real* __restrict__ v, const int64_t* __restrict__ lam,
                                                     int64_t count, double* __restrict__ scratch, int64_t cstride,
                                                     double* __restrict__ out) {
  const int64_t N = P.N;
  const int n = P.n;
  double* psi = scratch + int64_t(blockIdx.x) * cstride;
  double* w = psi + N;
  double* y = w + N;
  double* q = y + N;   // m × (box of supp ψ_λ)
  for (int64_t it = blockIdx.x; it < count; it += gridDim.x) {
    const int64_t l = lam[it];
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) w[i] = i == l ? 1.0 : 0.0;
    __syncthreads();
    inverse_full(P, w, psi, y);
    int s, p0, p1;
    locate(P, l, &s, &p0, &p1);
    int st[2] = {0, 0}, ln[2] = {1, 1};
    for (int a = (P.d == 2 ? 0 : 1); a < 2; ++a) supp_box(P, P.sb[s], a, a == 0 ? p0 : p1, &st[a], &ln[a]);
    const int B = ln[0] * ln[1];
    for (int t = threadIdx.x; t < B * P.m; t += blockDim.x) {
      const int k = t / B, b = t - k * B;
      const int b0 = b / ln[1], b1 = b - b0 * ln[1];
      const int64_t yi = P.d == 2 ? int64_t(wrap(st[0] + b0, n)) * n + wrap(st[1] + b1, n) : wrap(st[1] + b1, n);
      q[t] = double(v[int64_t(k) * N + yi]) * psi[yi];
    }
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) w[i] = 0.0;
    __syncthreads();
    // output box: supp ψ_λ ⊕ [zlo, zhi] per axis (the whole line when it covers it)
    int xs[2], xl[2];
    for (int a = 0; a < 2; ++a) {
      if (a == 0 && P.d == 1) { xs[0] = 0; xl[0] = 1; continue; }
      const int wz = P.zhi[a] - P.zlo[a] + 1;
      xl[a] = min(n, ln[a] + wz - 1);
      xs[a] = xl[a] >= n ? 0 : wrap(st[a] + P.zlo[a], n);
    }
    for (int t = threadIdx.x; t < xl[0] * xl[1]; t += blockDim.x) {
      const int i0 = t / xl[1], i1 = t - i0 * xl[1];
      const int x0 = P.d == 2 ? wrap(xs[0] + i0, n) : 0, x1 = wrap(xs[1] + i1, n);
      double acc = 0.0;
      const int wu0 = P.d == 2 ? P.zhi[0] - P.zlo[0] + 1 : 1, wu1 = P.zhi[1] - P.zlo[1] + 1;
      if (B <= wu0 * wu1) {   // gather over y ∈ supp ψ_λ
        for (int b0 = 0; b0 < ln[0]; ++b0) {
          const int y0 = P.d == 2 ? wrap(st[0] + b0, n) : 0;
          const int z0 = P.d == 2 ? wrap(x0 - y0, n) : 0;
          for (int b1 = 0; b1 < ln[1]; ++b1) {
            const int y1 = wrap(st[1] + b1, n);
            const int64_t zi = int64_t(z0) * n + wrap(x1 - y1, n);
            const int b = b0 * ln[1] + b1;
            for (int k = 0; k < P.m; ++k) {
              const double uz = u[int64_t(k) * N + zi];
              if (uz != 0.0) acc = fma(q[int64_t(k) * B + b], uz, acc);
            }
          }
        }
      } else {                // gather over z ∈ box(u): y = x − z must fall in supp ψ_λ
        for (int a0 = 0; a0 < wu0; ++a0) {
          const int z0 = P.d == 2 ? wrap(P.zlo[0] + a0, n) : 0;
          const int b0 = P.d == 2 ? wrap(x0 - z0 - st[0], n) : 0;
          if (b0 >= ln[0]) continue;
          for (int a1 = 0; a1 < wu1; ++a1) {
            const int z1 = wrap(P.zlo[1] + a1, n);
            const int b1 = wrap(x1 - z1 - st[1], n);
            if (b1 >= ln[1]) continue;
            const int64_t zi = int64_t(z0) * n + z1;
            const int b = b0 * ln[1] + b1;
            for (int k = 0; k < P.m; ++k) {
              const double uz = u[int64_t(k) * N + zi];
              if (uz != 0.0) acc = fma(q[int64_t(k) * B + b], uz, acc);
            }
          }
        }
      }
      w[P.d == 2 ? int64_t(x0) * n + x1 : x1] = acc;
    }
    __syncthreads();
    forward_full(P, w, out + it * N, y);
  }
}

// y = H f (adjoint = 0) or H* f (adjoint = 1), direct sums over the planned box of supp u_k:
//   H f (x) = Σ_k Σ_z u_k(z) v_k(x − z) f(x − z),   H* g (y) = Σ_k v_k(y) Σ_z u_k(z) g(y + z).
template <typename Real>
__global__ void operator_kernel(const __grid_constant__ Plan P, const double* __restrict__ u, const Real* __restrict__ v,
                                const Real* __restrict__ f, Real* __restrict__ out, int adjoint) {
  const int n = P.n;
  const int64_t N = P.N;
  const int w0 = P.d == 2 ? P.zhi[0] - P.zlo[0] + 1 : 1, w1 = P.zhi[1] - P.zlo[1] + 1;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < N; i += int64_t(gridDim.x) * blockDim.x) {
    const int x0 = P.d == 2 ? int(i / n) : 0, x1 = int(i - int64_t(x0) * n);
    double acc = 0.0;
    for (int k = 0; k < P.m; ++k) {
      const double* uk = u + int64_t(k) * N;
      const Real* vk = v + int64_t(k) * N;
      double ak = 0.0;
      for (int a = 0; a < w0; ++a) {
        const int z0 = P.d == 2 ? wrap(P.zlo[0] + a, n) : 0;
        for (int b = 0; b < w1; ++b) {
          const int z1 = wrap(P.zlo[1] + b, n);
          const double uz = uk[int64_t(z0) * n + z1];
          if (uz == 0.0) continue;
          if (!adjoint) {
            const int64_t j = P.d == 2 ? int64_t(wrap(x0 - z0, n)) * n + wrap(x1 - z1, n) : wrap(x1 - z1, n);
            ak = fma(uz, double(vk[j]) * double(f[j]), ak);
          } else {
            const int64_t j = P.d == 2 ? int64_t(wrap(x0 + z0, n)) * n + wrap(x1 + z1, n) : wrap(x1 + z1, n);
            ak = fma(uz, double(f[j]), ak);
          }
        }
      }
      acc = adjoint ? fma(double(vk[i]), ak, acc) : acc + ak;
    }
    out[i] = Real(acc);
  }
}

}  // namespace

int approx_block() { return kAB; }
int approx_bins() { return kSB; }

cudaError_t launch_approx_stats(const Plan& P, const ApproxArgs& A, int grid, cudaStream_t st) {
  approx_stats_kernel<<<grid, kAB, 0, st>>>(P, A);
  return cudaGetLastError();
}

cudaError_t launch_approx_rows(const Plan& P, const ApproxArgs& A, int write, int out_bytes, int grid,
                               cudaStream_t st) {
  if (!write) approx_rows_kernel<false, double><<<grid, kAB, 0, st>>>(P, A);
  else if (out_bytes == 8) approx_rows_kernel<true, double><<<grid, kAB, 0, st>>>(P, A);
  else approx_rows_kernel<true, float><<<grid, kAB, 0, st>>>(P, A);
  return cudaGetLastError();
}

cudaError_t launch_columns(const Plan& P, const double* u, const void* v, const int64_t* lam, int64_t count,
                           double* scratch, int64_t cstride, int grid, double* out, int real_bytes, cudaStream_t st) {
  if (real_bytes == 8)
    column_kernel<double><<<grid, kAB, 0, st>>>(P, u, static_cast<const double*>(v), lam, count, scratch, cstride, out);
  else
    column_kernel<float><<<grid, kAB, 0, st>>>(P, u, static_cast<const float*>(v), lam, count, scratch, cstride, out);
  return cudaGetLastError();
}

cudaError_t launch_operator(const Plan& P, const double* u, const void* v, const void* f, void* out, int adjoint,
                            int real_bytes, cudaStream_t st) {
  const int grid = int(std::min<int64_t>((P.N + 255) / 256, 148 * 16));
  if (real_bytes == 8)
    operator_kernel<double><<<grid, 256, 0, st>>>(P, u, static_cast<const double*>(v), static_cast<const double*>(f),
                                                  static_cast<double*>(out), adjoint);
  else
    operator_kernel<float><<<grid, 256, 0, st>>>(P, u, static_cast<const float*>(v), static_cast<const float*>(f),
                                                 static_cast<float*>(out), adjoint);
  return cudaGetLastError();
}

}  // namespace pcwd
