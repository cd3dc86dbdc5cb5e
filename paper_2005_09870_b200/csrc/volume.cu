// d = 3 variant: rows of Θ = Ψ* H Ψ on the periodic n × n × n grid.
//
// Row μ is Ψ*(H* ψ_μ) (R1; H* g = Σ_k v_k ⊙ (ũ_k ⋆ g), R9).  One CTA per unit, taken from a launch-wide counter, coarse
// units first; the unit's two n³ work arrays (the analysis cascade's ping-pong) in a global scratch slice:
//   1. ψ_μ = Ψ e_μ = f_0 ⊗ f_1 ⊗ f_2 (tensor-product basis): three 1-D synthesis cascades (P:94-96
//      transposed) in shared memory;
//   2. w(y) = Σ_k v_k(y) Σ_c u_k(c) ψ_μ((y + c) mod n) over the cyclic support box of the u_k, on O_0 × O_1 × O_2 only
//      (O_a = supp f_a dilated by the box: supp w is inside this product set);
//   3. c = Ψ* w by the analysis cascade, axis 0 first (R6 carried to three axes), every pass on the product set its
//      outputs can be nonzero on (1-D masks pushed through the steps), written in the Λ layout (coarse block, levels
//      J..1, orientations 4 e0 + 2 e1 + e2 = 1..7, positions row-major).
// fp64.  Supports are tracked as data (no class geometry, templates, TMA staging or retention rule as in the d ≤ 2
// pipeline): a variant path, see DESIGN.md §6b for what bounds it.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "common.h"
#include "kernels.cuh"

namespace pcwd_vol {

struct Args {
  int n, J, taps, m;
  int lo[3], cnt[3];            // cyclic support box of the u_k: offsets lo[a] .. lo[a] + cnt[a] − 1 per axis
  double h[pcwd::kMaxTaps];     // h[t], t = 0..taps−1
  double g[pcwd::kMaxTaps];     // g at offset 2 − taps + j: (−1)^{1−i} h[1−i]
  const double* u;
  const double* v;
  const int64_t* units;
  const int64_t* order;         // positions into units, most expensive (coarsest, lowest Λ index) first
  unsigned long long* next;     // launch-wide counter: CTAs take the next position as they finish
  int64_t count;
  double* out;
  double* scratch;              // 2 n³ doubles per CTA
};

// Largest cyclic offset per axis over the nonzeros of every u_k.
__global__ void support_kernel(const double* u, int64_t total, int n, int* rad) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    if (u[i] == 0.0) continue;
    const int64_t z = i % (int64_t(n) * n * n);
    const int z0 = int(z / (int64_t(n) * n)), z1 = int(z / n) % n, z2 = int(z % n);
    atomicMax(&rad[0], min(z0, n - z0));
    atomicMax(&rad[1], min(z1, n - z1));
    atomicMax(&rad[2], min(z2, n - z2));
  }
}

// q / d for q < 2^24, 1 ≤ d ≤ 256 by one multiply: M = ⌈2^32 / d⌉ overshoots q/d by < q / 2^32 < 1/256 ≤ 1/d, so the
// floor is exact; d = 1 (M would be 2^32) is passed through.
struct FastDiv {
  unsigned M, d;
  __device__ explicit FastDiv(int dd) : M(dd > 1 ? 0xFFFFFFFFu / unsigned(dd) + 1u : 0u), d(unsigned(dd)) {}
  __device__ __forceinline__ unsigned div(unsigned q) const { return d > 1 ? __umulhi(q, M) : q; }
};

// Index lists of three 1-D masks (one warp per axis, ballot compaction); all threads of the CTA call it.
__device__ void build_lists(const unsigned char (*mask)[256], int len, short (*list)[256], int* cnt) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w < 3) {
    int base = 0;
    for (int c = 0; c < len; c += 32) {
      const int i = c + lane;
      const bool on = i < len && mask[w][i];
      const unsigned b = __ballot_sync(0xffffffffu, on);
      if (on) list[w][base + __popc(b & ((1u << lane) - 1u))] = short(i);
      base += __popc(b);
    }
    if (lane == 0) cnt[w] = base;
  }
  __syncthreads();
}

// One analysis step along axis `ax` of a cube of side s (power of two), out = a | d concatenated on that axis,
// restricted to a product set: outputs (i0, i1, i2) ∈ L0 × L1 × L2 only, inputs read where `min` (the input's mask
// along `ax`) is set — everything off the product set is an exact zero that is neither stored nor loaded.
__device__ void analysis_pass(const Args& A, const double* x, double* y, int s, int ax,
                              const short* L0, int c0, const short* L1, int c1, const short* L2, int c2,
                              const unsigned char* min) {
  const int half = s >> 1, mask = s - 1;
  const int stride = ax == 0 ? s * s : (ax == 1 ? s : 1);
  const int total = c0 * c1 * c2;
  const FastDiv d2(c2), d1(c1);
  for (int q = threadIdx.x; q < total; q += blockDim.x) {
    const unsigned t = d2.div(q), j0 = d1.div(t);
    const int i2 = L2[q - t * c2], i1 = L1[t - j0 * c1], i0 = L0[j0];
    const int idx = (i0 * s + i1) * s + i2;
    const int i = ax == 0 ? i0 : (ax == 1 ? i1 : i2);
    const double* line = x + (idx - i * stride);
    double acc = 0.0;
    if (i < half) {
      for (int t = 0; t < A.taps; ++t) {
        const int xi = (2 * i + t) & mask;
        if (min[xi]) acc += A.h[t] * line[xi * stride];
      }
    } else {
      const int l = i - half;
      for (int j = 0; j < A.taps; ++j) {
        const int xi = (2 * l + 2 - A.taps + j) & mask;
        if (min[xi]) acc += A.g[j] * line[xi * stride];
      }
    }
    y[idx] = acc;
  }
}

__device__ __forceinline__ int64_t subband_offset(int n, int J, int lev, int e) {
  const int64_t nJ = n >> J;
  int64_t off = nJ * nJ * nJ;
  for (int l = J; l > lev; --l) {
    const int64_t nl = n >> l;
    off += 7 * nl * nl * nl;
  }
  const int64_t nl = n >> lev;
  return off + (e - 1) * nl * nl * nl;
}

template <int NT>
__global__ void __launch_bounds__(NT) rows3d_kernel(const Args A) {
  const int n = A.n, J = A.J;
  const int64_t N = int64_t(n) * n * n;
  __shared__ unsigned char S[3][256];    // supp f_a
  __shared__ unsigned char M[3][256];    // per-axis support of the cascade's current input (a product set)
  __shared__ unsigned char P[3][256];    // … of the current level's output (a | d coordinates)
  __shared__ short LM[3][256], LP[3][256];
  __shared__ int cM[3], cP[3];
  __shared__ double fa[3][256], fb[3][256];   // the 1-D factors of ψ_μ (ping-pong)
  double (*f)[256] = fa;
  double* X = A.scratch + 2 * N * blockIdx.x;
  double* Y = X + N;
  __shared__ unsigned long long taken;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) taken = atomicAdd(A.next, 1ull);
    __syncthreads();
    if (taken >= (unsigned long long)A.count) break;
    const int64_t ui = A.order[taken];
    const int64_t mu = A.units[ui];
    // 1. ψ_μ = Ψ e_μ is a tensor product: ψ_μ(x) = f_0(x0) f_1(x1) f_2(x2), f_a = the 1-D scaling
    //    function (e_a = 0) or wavelet (e_a = 1) of level ℓ at position l_a — three 1-D synthesis cascades in shared
    //    memory instead of the 3-D one; ψ_μ is never written out.
    int lev = J, e = 0;
    int64_t pos = mu;
    {
      const int64_t nJ = n >> J;
      if (mu >= nJ * nJ * nJ) {
        for (lev = J; lev >= 1; --lev) {
          const int64_t nl = n >> lev, cube = nl * nl * nl, base = subband_offset(n, J, lev, 1);
          if (mu < base + 7 * cube) {
            e = 1 + int((mu - base) / cube);
            pos = (mu - base) % cube;
            break;
          }
        }
      }
    }
    {
      const int nl = n >> lev;
      const int l3[3] = {int(pos / (int64_t(nl) * nl)), int(pos / nl) % nl, int(pos % nl)};
      double (*src)[256] = fa, (*dst)[256] = fb;
      for (int idx = threadIdx.x; idx < 3 * nl; idx += blockDim.x) {
        const int a = idx / nl, i = idx % nl;
        src[a][i] = (i == (a == 0 ? l3[0] : (a == 1 ? l3[1] : l3[2]))) ? 1.0 : 0.0;
      }
      __syncthreads();
      for (int lv = lev; lv >= 1; --lv) {
        const int s = 2 * (n >> lv), smask = s - 1;
        for (int idx = threadIdx.x; idx < 3 * s; idx += blockDim.x) {
          const int a = idx / s, i = idx % s;
          const bool detail = lv == lev && ((e >> (2 - a)) & 1);
          double acc = 0.0;
          if (detail) {
            for (int j = 0; j < A.taps; ++j) {
              const int r = i - (2 - A.taps + j);
              if ((r & 1) == 0) acc += A.g[j] * src[a][(r & smask) >> 1];
            }
          } else {
            for (int t = 0; t < A.taps; ++t) {
              const int r = i - t;
              if ((r & 1) == 0) acc += A.h[t] * src[a][(r & smask) >> 1];
            }
          }
          dst[a][i] = acc;
        }
        __syncthreads();
        double (*tmp)[256] = src; src = dst; dst = tmp;
      }
      f = src;
    }
    // 2. w = H* ψ_μ on its support only.  supp ψ_μ = S_0 × S_1 × S_2 (S_a = supp f_a) is a product set, so supp w ⊂
    //    O_0 × O_1 × O_2 with O_a = S_a dilated by the box; everything else is an exact zero and is never touched.
    double* row = A.out + ui * N;
    {
      const int mask = n - 1;
      for (int idx = threadIdx.x; idx < 3 * n; idx += blockDim.x) S[idx / n][idx % n] = f[idx / n][idx % n] != 0.0;
      __syncthreads();
      for (int idx = threadIdx.x; idx < 3 * n; idx += blockDim.x) {
        const int a = idx / n, y = idx % n;
        bool any = false;
        for (int c = 0; c < A.cnt[a]; ++c) any |= S[a][(y + A.lo[a] + c) & mask] != 0;
        M[a][y] = any;
      }
      __syncthreads();
      build_lists(M, n, LM, cM);
      const int c0 = cM[0], c1 = cM[1], c2 = cM[2];
      const FastDiv d2(c2), d1(c1);
      for (int q = threadIdx.x; q < c0 * c1 * c2; q += blockDim.x) {
        const unsigned t = d2.div(q), j0 = d1.div(t);
        const int y2 = LM[2][q - t * c2], y1 = LM[1][t - j0 * c1], y0 = LM[0][j0];
        const int y = (y0 * n + y1) * n + y2;
        double acc = 0.0;
        for (int k = 0; k < A.m; ++k) {
          const double* uk = A.u + k * N;
          double s = 0.0;
          for (int a = 0; a < A.cnt[0]; ++a) {
            const int c0i = (A.lo[0] + a) & mask, x0 = (y0 + c0i) & mask;
            if (!S[0][x0]) continue;
            for (int b = 0; b < A.cnt[1]; ++b) {
              const int c1i = (A.lo[1] + b) & mask, x1 = (y1 + c1i) & mask;
              if (!S[1][x1]) continue;
              const double* ur = uk + (c0i * n + c1i) * n;
              double t = 0.0;
              for (int c = 0; c < A.cnt[2]; ++c) {
                const int c2i = (A.lo[2] + c) & mask;
                t += ur[c2i] * f[2][(y2 + c2i) & mask];
              }
              s += (f[0][x0] * f[1][x1]) * t;
            }
          }
          acc += A.v[k * N + y] * s;
        }
        Y[y] = acc;
      }
      __syncthreads();
    }
    // 3. c = Ψ* w, each pass on the product set its outputs can be nonzero on
    {
      for (int lv = 1; lv <= J; ++lv) {
        const int s = n >> (lv - 1), nl = s >> 1, smask = s - 1;
        for (int idx = threadIdx.x; idx < 3 * s; idx += blockDim.x) {
          const int a = idx / s, i = idx % s;
          bool any = false;
          if (i < nl) {
            for (int t = 0; t < A.taps; ++t) any |= M[a][(2 * i + t) & smask] != 0;
          } else {
            for (int j = 0; j < A.taps; ++j) any |= M[a][(2 * (i - nl) + 2 - A.taps + j) & smask] != 0;
          }
          P[a][i] = any;
        }
        __syncthreads();
        build_lists(P, s, LP, cP);
        analysis_pass(A, Y, X, s, 0, LP[0], cP[0], LM[1], cM[1], LM[2], cM[2], M[0]);
        __syncthreads();
        analysis_pass(A, X, Y, s, 1, LP[0], cP[0], LP[1], cP[1], LM[2], cM[2], M[1]);
        __syncthreads();
        analysis_pass(A, Y, X, s, 2, LP[0], cP[0], LP[1], cP[1], LP[2], cP[2], M[2]);
        __syncthreads();
        const int64_t base = subband_offset(n, J, lv, 1);
        const int64_t cube = int64_t(nl) * nl * nl;
        const int c0 = cP[0], c1 = cP[1], c2 = cP[2];
        const FastDiv d2(c2), d1(c1);
        for (int q = threadIdx.x; q < c0 * c1 * c2; q += blockDim.x) {
          const unsigned t = d2.div(q), j0 = d1.div(t);
          const int i2 = LP[2][q - t * c2], i1 = LP[1][t - j0 * c1], i0 = LP[0][j0];
          const int e = (i0 >= nl ? 4 : 0) | (i1 >= nl ? 2 : 0) | (i2 >= nl ? 1 : 0);
          const int pos = ((i0 % nl) * nl + (i1 % nl)) * nl + (i2 % nl);
          const double val = X[(i0 * s + i1) * s + i2];
          if (e == 0) Y[pos] = val;
          else row[base + (e - 1) * cube + pos] = val;
        }
        for (int idx = threadIdx.x; idx < 3 * nl; idx += blockDim.x) M[idx / nl][idx % nl] = P[idx / nl][idx % nl];
        __syncthreads();
        build_lists(M, nl, LM, cM);
      }
      const int nJ = n >> J;
      const int c0 = cM[0], c1 = cM[1], c2 = cM[2];
      for (int q = threadIdx.x; q < c0 * c1 * c2; q += blockDim.x) {
        const int i = (LM[0][q / (c2 * c1)] * nJ + LM[1][(q / c2) % c1]) * nJ + LM[2][q % c2];
        row[i] = Y[i];
      }
      __syncthreads();
    }
  }
}

// units, order, u, v, out: DEVICE.  h, sorted_mu (the Λ indices in `order`'s order, ascending): HOST.  Returns a
// cudaError_t as int (0 = success); synchronises `st` (the support box comes back to the host before the launches).
// Two launches side by side: the units whose 1-D supports cover at least half an axis (levels ≥ ℓ_c, the leading
// entries of `order`) on 1024-thread CTAs, the fine ones — a few thousand outputs each, latency-bound — on many
// 128-thread CTAs.
int rows3d(int n, int J, const double* h, int taps, int m, const double* u, const double* v, const int64_t* units,
           const int64_t* order, const int64_t* sorted_mu, int64_t count, double* out, cudaStream_t st) {
  if (count == 0) return 0;
  Args A{};
  A.n = n; A.J = J; A.taps = taps; A.m = m;
  for (int t = 0; t < taps; ++t) A.h[t] = h[t];
  for (int j = 0; j < taps; ++j) {
    const int i = 2 - taps + j;                       // g[i] = (−1)^{1−i} h[1−i]
    A.g[j] = (((1 - i) & 1) ? -1.0 : 1.0) * h[1 - i];
  }
  A.u = u; A.v = v; A.units = units; A.out = out;
  const int64_t N = int64_t(n) * n * n;
  int* rad = nullptr;
  cudaError_t e = cudaMalloc(&rad, 8 * sizeof(int));   // [0..2] support radii, [4..5], [6..7] the two unit counters
  if (e != cudaSuccess) return int(e);
  int rh[3] = {0, 0, 0};
  e = cudaMemsetAsync(rad, 0, 8 * sizeof(int), st);
  if (e == cudaSuccess) {
    support_kernel<<<296, 256, 0, st>>>(u, m * N, n, rad);
    e = cudaMemcpyAsync(rh, rad, 3 * sizeof(int), cudaMemcpyDeviceToHost, st);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) { cudaFree(rad); return int(e); }
  for (int a = 0; a < 3; ++a) {
    const bool whole = 2 * rh[a] + 1 >= n;
    A.lo[a] = whole ? 0 : -rh[a];
    A.cnt[a] = whole ? n : 2 * rh[a] + 1;
  }
  // ℓ_c: the first level whose dilated 1-D support (2^ℓ − 1)(taps − 1) + 1 + 2R reaches n/2; units of levels ≥ ℓ_c
  // are exactly those with Λ index < (n >> (ℓ_c − 1))³ (the layout is coarse first).
  const int R = std::max(rh[0], std::max(rh[1], rh[2]));
  int lc = 1;
  while (lc <= J && ((int64_t(1) << lc) - 1) * (taps - 1) + 1 + 2 * R < n / 2) ++lc;
  const int64_t side = n >> (lc - 1), bound = lc > J ? 0 : side * side * side;
  int64_t n_coarse = 0;
  while (n_coarse < count && sorted_mu[n_coarse] < bound) ++n_coarse;
  const int64_t n_fine = count - n_coarse;
  const int64_t per_cta = 2 * N * int64_t(sizeof(double));
  const int64_t cap = std::max<int64_t>(1, (int64_t(4) << 30) / per_cta);
  const int64_t ctas_c = std::min<int64_t>(std::min<int64_t>(n_coarse, 148 * 2), cap);
  const int64_t ctas_f = std::min<int64_t>(std::min<int64_t>(n_fine, 148 * 8), cap);
  double* scratch = nullptr;
  e = cudaMalloc(&scratch, size_t((ctas_c + ctas_f) * per_cta));
  if (e != cudaSuccess) { cudaFree(rad); return int(e); }
  cudaStream_t s2 = nullptr;
  cudaEvent_t ev = nullptr;
  e = cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaMemsetAsync(out, 0, size_t(count) * N * sizeof(double), st);   // the rows' exact zeros
  if (e == cudaSuccess) e = cudaEventRecord(ev, st);
  if (e == cudaSuccess && n_coarse > 0) {
    e = cudaStreamWaitEvent(s2, ev, 0);
    Args C = A;
    C.order = order; C.count = n_coarse; C.scratch = scratch;
    C.next = reinterpret_cast<unsigned long long*>(rad + 4);
    // few coarse units: ask for more than half an SM's shared memory so that every CTA gets an SM of its own
    const size_t pad = n_coarse <= 148 ? size_t(120) << 10 : 0;
    if (e == cudaSuccess && pad)
      e = cudaFuncSetAttribute(rows3d_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pad));
    if (e == cudaSuccess) rows3d_kernel<1024><<<unsigned(ctas_c), 1024, pad, s2>>>(C);
    if (e == cudaSuccess) e = cudaGetLastError();
  }
  if (e == cudaSuccess && n_fine > 0) {
    Args F = A;
    F.order = order + n_coarse; F.count = n_fine; F.scratch = scratch + ctas_c * 2 * N;
    F.next = reinterpret_cast<unsigned long long*>(rad + 6);
    rows3d_kernel<128><<<unsigned(ctas_f), 128, 0, st>>>(F);
    e = cudaGetLastError();
  }
  cudaError_t e2 = s2 ? cudaStreamSynchronize(s2) : cudaSuccess;
  cudaError_t e1 = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = e1 != cudaSuccess ? e1 : e2;
  if (ev) cudaEventDestroy(ev);
  if (s2) cudaStreamDestroy(s2);
  cudaFree(scratch);
  cudaFree(rad);
  return int(e);
}

}  // namespace pcwd_vol
