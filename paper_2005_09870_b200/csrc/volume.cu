// d = 3 variant: rows of Θ = Ψ* H Ψ on the periodic n × n × n grid.
//
// Row μ is Ψ*(H* ψ_μ) (R1; H* g = Σ_k v_k ⊙ (ũ_k ⋆ g), R9).  One CTA per unit, the unit's two n³ work arrays in a
// global scratch slice (they stay in L2 for the sizes this path is meant for):
//   1. ψ_μ = Ψ e_μ by the synthesis cascade (P:94-96 transposed), axes undone in the order 2, 1, 0 per level;
//   2. w(y) = Σ_k v_k(y) Σ_c u_k(c) ψ_μ((y + c) mod n) over the cyclic support box of the u_k, skipping the
//      (x0, x1) lines on which ψ_μ is identically zero;
//   3. c = Ψ* w by the analysis cascade, axis 0 first (R6 carried to three axes), written in the Λ layout
//      (coarse block, levels J..1, orientations 4 e0 + 2 e1 + e2 = 1..7, positions row-major).
// Whole-torus passes in fp64, no windowing: a plain variant path for small volumes, not the tuned d ≤ 2 pipeline.
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

// One analysis step along axis `ax` of a cube of side s (power of two): out holds a | d concatenated on that axis.
__device__ void analysis_pass(const Args& A, const double* __restrict__ x, double* __restrict__ y, int s, int ax) {
  const int half = s >> 1, mask = s - 1;
  const int stride = ax == 0 ? s * s : (ax == 1 ? s : 1);
  const int total = s * s * s;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int i = (idx / stride) & mask;
    const double* line = x + (idx - i * stride);
    double acc = 0.0;
    if (i < half) {
      for (int t = 0; t < A.taps; ++t) acc += A.h[t] * line[((2 * i + t) & mask) * stride];
    } else {
      const int l = i - half;
      for (int j = 0; j < A.taps; ++j) acc += A.g[j] * line[((2 * l + 2 - A.taps + j) & mask) * stride];
    }
    y[idx] = acc;
  }
}

// The adjoint step: x holds a | d on axis `ax`; y[i] = Σ_{(2l+t) ≡ i} h[t] a[l] + Σ_{(2l+o) ≡ i} g[o] d[l].
__device__ void synthesis_pass(const Args& A, const double* __restrict__ x, double* __restrict__ y, int s, int ax) {
  const int half = s >> 1, mask = s - 1;
  const int stride = ax == 0 ? s * s : (ax == 1 ? s : 1);
  const int total = s * s * s;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int i = (idx / stride) & mask;
    const double* line = x + (idx - i * stride);
    double acc = 0.0;
    for (int t = 0; t < A.taps; ++t) {
      const int r = i - t;
      if ((r & 1) == 0) acc += A.h[t] * line[((r & mask) >> 1) * stride];
    }
    for (int j = 0; j < A.taps; ++j) {
      const int r = i - (2 - A.taps + j);
      if ((r & 1) == 0) acc += A.g[j] * line[(half + ((r & mask) >> 1)) * stride];
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

__global__ void __launch_bounds__(512) rows3d_kernel(const Args A) {
  const int n = A.n, J = A.J;
  const int64_t N = int64_t(n) * n * n;
  __shared__ unsigned linemask[2048];   // one bit per (x0, x1) line of the torus, n ≤ 256
  __shared__ unsigned outmask[2048];
  double* X = A.scratch + 2 * N * blockIdx.x;
  double* Y = X + N;
  for (int64_t ui = blockIdx.x; ui < A.count; ui += gridDim.x) {
    const int64_t mu = A.units[ui];
    // 1. ψ_μ = Ψ e_μ
    {
      const int nJ = n >> J;
      for (int i = threadIdx.x; i < nJ * nJ * nJ; i += blockDim.x) X[i] = (i == mu) ? 1.0 : 0.0;
      __syncthreads();
      for (int lev = J; lev >= 1; --lev) {
        const int nl = n >> lev, s = 2 * nl;
        const int64_t base = subband_offset(n, J, lev, 1);
        const int64_t cube = int64_t(nl) * nl * nl;
        for (int idx = threadIdx.x; idx < s * s * s; idx += blockDim.x) {
          const int i0 = idx / (s * s), i1 = (idx / s) % s, i2 = idx % s;
          const int e = (i0 >= nl ? 4 : 0) | (i1 >= nl ? 2 : 0) | (i2 >= nl ? 1 : 0);
          const int pos = ((i0 % nl) * nl + (i1 % nl)) * nl + (i2 % nl);
          Y[idx] = e == 0 ? X[pos] : ((base + (e - 1) * cube + pos == mu) ? 1.0 : 0.0);
        }
        __syncthreads();
        synthesis_pass(A, Y, X, s, 2);
        __syncthreads();
        synthesis_pass(A, X, Y, s, 1);
        __syncthreads();
        synthesis_pass(A, Y, X, s, 0);
        __syncthreads();
      }
    }
    // 2. w = H* ψ_μ.  ψ_μ is exactly zero off its support (a fine-level wavelet fills a few (x0, x1) lines of the
    //    torus): lines without a nonzero are skipped — they would add exact zeros.
    {
      const int mask = n - 1;
      for (int i = threadIdx.x; i < (n * n + 31) / 32; i += blockDim.x) linemask[i] = 0u;
      __syncthreads();
      for (int idx = threadIdx.x; idx < N; idx += blockDim.x)
        if (X[idx] != 0.0) atomicOr(&linemask[(idx / n) >> 5], 1u << ((idx / n) & 31));
      __syncthreads();
      // output lines (y0, y1) that see a nonzero line through the box; the others are exact zeros
      for (int i = threadIdx.x; i < (n * n + 31) / 32; i += blockDim.x) outmask[i] = 0u;
      __syncthreads();
      for (int l = threadIdx.x; l < n * n; l += blockDim.x) {
        const int y0 = l / n, y1 = l & mask;
        bool any = false;
        for (int a = 0; a < A.cnt[0] && !any; ++a) {
          const int x0 = (y0 + A.lo[0] + a) & mask;
          for (int b = 0; b < A.cnt[1]; ++b) {
            const int line = x0 * n + ((y1 + A.lo[1] + b) & mask);
            if ((linemask[line >> 5] >> (line & 31)) & 1u) { any = true; break; }
          }
        }
        if (any) atomicOr(&outmask[l >> 5], 1u << (l & 31));
      }
      __syncthreads();
      for (int y = threadIdx.x; y < N; y += blockDim.x) {
        const int y0 = y / (n * n), y1 = (y / n) & mask, y2 = y & mask;
        if (!((outmask[(y / n) >> 5] >> ((y / n) & 31)) & 1u)) { Y[y] = 0.0; continue; }
        double acc = 0.0;
        for (int k = 0; k < A.m; ++k) {
          const double* uk = A.u + k * N;
          double s = 0.0;
          for (int a = 0; a < A.cnt[0]; ++a) {
            const int c0 = (A.lo[0] + a) & mask, x0 = (y0 + c0) & mask;
            for (int b = 0; b < A.cnt[1]; ++b) {
              const int c1 = (A.lo[1] + b) & mask, x1 = (y1 + c1) & mask;
              const int line = x0 * n + x1;
              if (!((linemask[line >> 5] >> (line & 31)) & 1u)) continue;
              const double* ur = uk + (c0 * n + c1) * n;
              const double* xr = X + (x0 * n + x1) * n;
              for (int c = 0; c < A.cnt[2]; ++c) {
                const int c2 = (A.lo[2] + c) & mask;
                s += ur[c2] * xr[(y2 + c2) & mask];
              }
            }
          }
          acc += A.v[k * N + y] * s;
        }
        Y[y] = acc;
      }
      __syncthreads();
    }
    // 3. c = Ψ* w
    {
      double* row = A.out + ui * N;
      for (int lev = 1; lev <= J; ++lev) {
        const int s = n >> (lev - 1), nl = s >> 1;
        analysis_pass(A, Y, X, s, 0);
        __syncthreads();
        analysis_pass(A, X, Y, s, 1);
        __syncthreads();
        analysis_pass(A, Y, X, s, 2);
        __syncthreads();
        const int64_t base = subband_offset(n, J, lev, 1);
        const int64_t cube = int64_t(nl) * nl * nl;
        for (int idx = threadIdx.x; idx < s * s * s; idx += blockDim.x) {
          const int i0 = idx / (s * s), i1 = (idx / s) % s, i2 = idx % s;
          const int e = (i0 >= nl ? 4 : 0) | (i1 >= nl ? 2 : 0) | (i2 >= nl ? 1 : 0);
          const int pos = ((i0 % nl) * nl + (i1 % nl)) * nl + (i2 % nl);
          if (e == 0) Y[pos] = X[idx];
          else row[base + (e - 1) * cube + pos] = X[idx];
        }
        __syncthreads();
      }
      const int nJ = n >> J;
      for (int i = threadIdx.x; i < nJ * nJ * nJ; i += blockDim.x) row[i] = Y[i];
      __syncthreads();
    }
  }
}

// units, u, v, out: DEVICE.  h: HOST.  Returns a cudaError_t as int (0 = success); synchronises `st` once (the
// support box comes back to the host before the launch).
int rows3d(int n, int J, const double* h, int taps, int m, const double* u, const double* v, const int64_t* units,
           int64_t count, double* out, cudaStream_t st) {
  if (count == 0) return 0;
  Args A{};
  A.n = n; A.J = J; A.taps = taps; A.m = m;
  for (int t = 0; t < taps; ++t) A.h[t] = h[t];
  for (int j = 0; j < taps; ++j) {
    const int i = 2 - taps + j;                       // g[i] = (−1)^{1−i} h[1−i]
    A.g[j] = (((1 - i) & 1) ? -1.0 : 1.0) * h[1 - i];
  }
  A.u = u; A.v = v; A.units = units; A.count = count; A.out = out;
  const int64_t N = int64_t(n) * n * n;
  int* rad = nullptr;
  cudaError_t e = cudaMalloc(&rad, 3 * sizeof(int));
  if (e != cudaSuccess) return int(e);
  int rh[3] = {0, 0, 0};
  e = cudaMemsetAsync(rad, 0, 3 * sizeof(int), st);
  if (e == cudaSuccess) {
    support_kernel<<<296, 256, 0, st>>>(u, m * N, n, rad);
    e = cudaMemcpyAsync(rh, rad, 3 * sizeof(int), cudaMemcpyDeviceToHost, st);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(rad);
  if (e != cudaSuccess) return int(e);
  for (int a = 0; a < 3; ++a) {
    const bool whole = 2 * rh[a] + 1 >= n;
    A.lo[a] = whole ? 0 : -rh[a];
    A.cnt[a] = whole ? n : 2 * rh[a] + 1;
  }
  const int64_t per_cta = 2 * N * int64_t(sizeof(double));
  int64_t ctas = std::min<int64_t>(count, 148 * 4);
  ctas = std::max<int64_t>(1, std::min<int64_t>(ctas, (int64_t(2) << 30) / per_cta));
  double* scratch = nullptr;
  e = cudaMalloc(&scratch, size_t(ctas * per_cta));
  if (e != cudaSuccess) return int(e);
  A.scratch = scratch;
  rows3d_kernel<<<unsigned(ctas), 512, 0, st>>>(A);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(scratch);
  return int(e);
}

}  // namespace pcwd_vol
