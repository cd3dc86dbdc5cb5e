// pca.cu — constructing the product-convolution expansion on the GPU (§3.3):
//
//   * §3.3.2: principal components of impulse responses sampled on a grid, the coefficient maps v_k
//     interpolated from the samples' projection coefficients (periodic bilinear between cell centres, reading R12).
//   * §3.3.3: a randomized SVD ("the couples (u_k, v_k) can be obtained using a randomized SVD of
//     the matrix S") of the space-varying impulse response S given at every pixel; v_k(y) = <S(·, y), u_k>.
//
// Both factor a matrix X (s × W): row i is one impulse response on the window [−R, R]^d (W = (2R+1)^d values).
// u_k = the m leading right singular vectors of X (uncentred PCA, reading R10), found by subspace iteration on XᵀX
// started from a seeded Gaussian block (counter-based generator), re-orthonormalised (modified Gram–Schmidt, twice)
// after every product, then a Rayleigh–Ritz step (cyclic Jacobi on the r × r projected matrix).  Sign: the largest-|entry| of
// each u_k is positive.  c = X u (the projections).  All of it runs in these kernels; the host only sequences them.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/pcwd.h"
#include "kernels.cuh"

namespace pcwd_pca {

namespace {

constexpr int kT = 256;
constexpr int kMaxR = 32;

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

// Y[w][j] ~ N(0, 1) from (seed, w, j) (Box–Muller on two counter-based uniforms)
__global__ void gauss_kernel(double* Y, int W, int r, uint64_t seed) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < W * r; i += gridDim.x * blockDim.x) {
    const uint64_t a = splitmix64(seed ^ (uint64_t(i) * 2 + 1)), b = splitmix64(seed + 0x632BE59BD9B4E019ULL * (uint64_t(i) + 7));
    const double u1 = (double(a >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    const double u2 = double(b >> 11) * (1.0 / 9007199254740992.0);
    Y[i] = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
  }
}

// Z (s × r) = X (s × W) · Y (W × r): a warp per row of X, lanes over W, shuffle reduction per column of Y.
__global__ void xy_kernel(const double* __restrict__ X, const double* __restrict__ Y, double* __restrict__ Z, int64_t s,
                          int W, int r) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = warp; i < s; i += nw) {
    double acc[kMaxR];
#pragma unroll
    for (int j = 0; j < kMaxR; ++j) acc[j] = 0.0;
    for (int w = lane; w < W; w += 32) {
      const double x = X[i * W + w];
#pragma unroll
      for (int j = 0; j < kMaxR; ++j)
        if (j < r) acc[j] = fma(x, Y[int64_t(w) * r + j], acc[j]);
    }
#pragma unroll
    for (int j = 0; j < kMaxR; ++j) {
      if (j >= r) break;
      double v = acc[j];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) Z[i * r + j] = v;
    }
  }
}

// Y (W × r) = Xᵀ (W × s) · Z (s × r): a thread per (w, j), summing over all rows in order (deterministic).
__global__ void xtz_kernel(const double* __restrict__ X, const double* __restrict__ Z, double* __restrict__ Y, int64_t s,
                           int W, int r) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < W * r; t += gridDim.x * blockDim.x) {
    const int w = t % W, j = t / W;
    double acc = 0.0;
    for (int64_t i = 0; i < s; ++i) acc = fma(X[i * W + w], Z[i * r + j], acc);
    Y[int64_t(w) * r + j] = acc;
  }
}

// Partial Gram sums of the columns of Z (rows [b·chunk, (b+1)·chunk)): part[b][a][c] = Σ_i Z[i][a] Z[i][c].
__global__ void gram_part_kernel(const double* __restrict__ Z, int64_t s, int r, int64_t chunk, double* __restrict__ part) {
  const int64_t i0 = blockIdx.x * chunk, i1 = min(s, i0 + chunk);
  for (int t = threadIdx.x; t < r * r; t += blockDim.x) {
    const int a = t / r, c = t % r;
    double acc = 0.0;
    for (int64_t i = i0; i < i1; ++i) acc = fma(Z[i * r + a], Z[i * r + c], acc);
    part[int64_t(blockIdx.x) * r * r + t] = acc;
  }
}

// One CTA: G = Σ_b part[b] (in block order); then either
//   mode 0 (CholeskyQR of Y, L × r): G = LLᵀ (Cholesky, one thread), Y ← Y L⁻ᵀ;
//   mode 1 (Rayleigh–Ritz): G = V Λ Vᵀ by cyclic Jacobi (one thread: r ≤ 32), eigenpairs sorted by decreasing λ
//          into lam[r] and V (r × r, column j = eigenvector j).
__global__ void small_kernel(const double* __restrict__ part, int nb, int r, int mode, double* Y, int L, double* lam,
                             double* V) {
  __shared__ double G[kMaxR * kMaxR];
  __shared__ double Vs[kMaxR * kMaxR];
  for (int t = threadIdx.x; t < r * r; t += blockDim.x) {
    double acc = 0.0;
    for (int b = 0; b < nb; ++b) acc += part[int64_t(b) * r * r + t];
    G[t] = acc;
  }
  __syncthreads();
  if (mode == 0) {
    if (threadIdx.x == 0) {   // in place: lower triangle of G becomes L
      for (int j = 0; j < r; ++j) {
        double d = G[j * r + j];
        for (int k = 0; k < j; ++k) d -= G[j * r + k] * G[j * r + k];
        d = d > 0.0 ? sqrt(d) : 1e-300;
        G[j * r + j] = d;
        for (int i = j + 1; i < r; ++i) {
          double x = G[i * r + j];
          for (int k = 0; k < j; ++k) x -= G[i * r + k] * G[j * r + k];
          G[i * r + j] = x / d;
        }
      }
    }
    __syncthreads();
    for (int w = threadIdx.x; w < L; w += blockDim.x) {   // row y ← y L⁻ᵀ: forward substitution per row
      double y[kMaxR];
      for (int j = 0; j < r; ++j) y[j] = Y[int64_t(w) * r + j];
      for (int j = 0; j < r; ++j) {
        double x = y[j];
        for (int k = 0; k < j; ++k) x -= G[j * r + k] * y[k];
        y[j] = x / G[j * r + j];
      }
      for (int j = 0; j < r; ++j) Y[int64_t(w) * r + j] = y[j];
    }
    return;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < r * r; ++i) Vs[i] = (i / r == i % r) ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 60; ++sweep) {
      double off = 0.0, tot = 0.0;
      for (int i = 0; i < r; ++i)
        for (int j = 0; j < r; ++j) {
          tot += G[i * r + j] * G[i * r + j];
          if (i != j) off += G[i * r + j] * G[i * r + j];
        }
      if (off <= 1e-34 * tot) break;
      for (int p = 0; p < r - 1; ++p)
        for (int q = p + 1; q < r; ++q) {
          const double apq = G[p * r + q];
          if (apq == 0.0) continue;
          const double theta = (G[q * r + q] - G[p * r + p]) / (2.0 * apq);
          const double tt = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
          const double c = 1.0 / sqrt(tt * tt + 1.0), sn = tt * c;
          for (int k = 0; k < r; ++k) {   // G ← Jᵀ G J
            const double gkp = G[k * r + p], gkq = G[k * r + q];
            G[k * r + p] = c * gkp - sn * gkq;
            G[k * r + q] = sn * gkp + c * gkq;
          }
          for (int k = 0; k < r; ++k) {
            const double gpk = G[p * r + k], gqk = G[q * r + k];
            G[p * r + k] = c * gpk - sn * gqk;
            G[q * r + k] = sn * gpk + c * gqk;
          }
          for (int k = 0; k < r; ++k) {
            const double vkp = Vs[k * r + p], vkq = Vs[k * r + q];
            Vs[k * r + p] = c * vkp - sn * vkq;
            Vs[k * r + q] = sn * vkp + c * vkq;
          }
        }
    }
    int ord[kMaxR];
    for (int i = 0; i < r; ++i) ord[i] = i;
    for (int i = 0; i < r; ++i)   // selection sort by decreasing eigenvalue (stable on ties)
      for (int j = i + 1; j < r; ++j)
        if (G[ord[j] * r + ord[j]] > G[ord[i] * r + ord[i]]) { const int t = ord[i]; ord[i] = ord[j]; ord[j] = t; }
    for (int j = 0; j < r; ++j) {
      lam[j] = G[ord[j] * r + ord[j]];
      for (int k = 0; k < r; ++k) V[k * r + j] = Vs[k * r + ord[j]];
    }
  }
}

__device__ double block_sum(double x, double* red) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = x;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < int(blockDim.x >> 5); ++i) s += red[i];
  return s;
}

// One CTA: Y (W × r) ← an orthonormal basis of its column span by modified Gram–Schmidt, each column orthogonalised
// twice; a column that (numerically) lies in the span of the previous ones — the null space of a rank-deficient X —
// is replaced by a fresh seeded Gaussian column and orthogonalised again.
__global__ void mgs_kernel(double* Y, int W, int r, uint64_t seed) {
  __shared__ double red[32];
  for (int j = 0; j < r; ++j) {
    for (int attempt = 0; attempt < 8; ++attempt) {
      double n0 = 0.0;
      for (int w = threadIdx.x; w < W; w += blockDim.x) n0 += Y[int64_t(w) * r + j] * Y[int64_t(w) * r + j];
      n0 = sqrt(block_sum(n0, red));
      for (int pass = 0; pass < 2; ++pass)
        for (int i = 0; i < j; ++i) {
          double dp = 0.0;
          for (int w = threadIdx.x; w < W; w += blockDim.x) dp += Y[int64_t(w) * r + i] * Y[int64_t(w) * r + j];
          dp = block_sum(dp, red);
          for (int w = threadIdx.x; w < W; w += blockDim.x) Y[int64_t(w) * r + j] -= dp * Y[int64_t(w) * r + i];
          __syncthreads();
        }
      double nj = 0.0;
      for (int w = threadIdx.x; w < W; w += blockDim.x) nj += Y[int64_t(w) * r + j] * Y[int64_t(w) * r + j];
      nj = sqrt(block_sum(nj, red));
      if (nj > 1e-12 * n0 && nj > 1e-300) {
        for (int w = threadIdx.x; w < W; w += blockDim.x) Y[int64_t(w) * r + j] /= nj;
        __syncthreads();
        break;
      }
      for (int w = threadIdx.x; w < W; w += blockDim.x) {   // dependent column: restart it from noise
        const uint64_t a = splitmix64(seed ^ (0xABCDULL + uint64_t(attempt) * 1000003ULL + uint64_t(j) * 7919ULL +
                                              uint64_t(w) * 104729ULL));
        const uint64_t b = splitmix64(a + 0x9E3779B97F4A7C15ULL);
        const double u1 = (double(a >> 11) + 0.5) * (1.0 / 9007199254740992.0);
        const double u2 = double(b >> 11) * (1.0 / 9007199254740992.0);
        Y[int64_t(w) * r + j] = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
      }
      __syncthreads();
    }
  }
}

// U (W × m) = Y (W × r) · V[:, :m], then the sign rule: the largest-|entry| of each column positive (first on ties).
__global__ void ritz_kernel(const double* __restrict__ Y, const double* __restrict__ V, int W, int r, int m,
                            double* __restrict__ U) {
  __shared__ double sv[kT];
  __shared__ int si[kT];
  for (int k = 0; k < m; ++k) {
    for (int w = threadIdx.x; w < W; w += blockDim.x) {
      double acc = 0.0;
      for (int j = 0; j < r; ++j) acc = fma(Y[int64_t(w) * r + j], V[j * r + k], acc);
      U[int64_t(w) * m + k] = acc;
    }
    __syncthreads();
    double best = -1.0;
    int bi = 0;
    for (int w = threadIdx.x; w < W; w += blockDim.x) {
      const double a = fabs(U[int64_t(w) * m + k]);
      if (a > best) { best = a; bi = w; }
    }
    sv[threadIdx.x] = best;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) {
        const double b2 = sv[threadIdx.x + o];
        const int i2 = si[threadIdx.x + o];
        if (b2 > sv[threadIdx.x] || (b2 == sv[threadIdx.x] && i2 < si[threadIdx.x])) { sv[threadIdx.x] = b2; si[threadIdx.x] = i2; }
      }
      __syncthreads();
    }
    const bool flip = U[int64_t(si[0]) * m + k] < 0.0;
    __syncthreads();
    if (flip)
      for (int w = threadIdx.x; w < W; w += blockDim.x) U[int64_t(w) * m + k] = -U[int64_t(w) * m + k];
    __syncthreads();
  }
}

// u_k on the torus: u_k(z mod n) += U[w][k], z = window offset of w (taps that wrap accumulate, as synth embeds them)
__global__ void embed_kernel(const double* __restrict__ U, int d, int n, int R, int m, double* __restrict__ u) {
  const int side = 2 * R + 1;
  const int W = d == 2 ? side * side : side;
  const int64_t N = d == 2 ? int64_t(n) * n : n;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int k = 0; k < m; ++k)
      for (int w = 0; w < W; ++w) {
        const int a = d == 2 ? w / side : 0, b = d == 2 ? w % side : w;
        const int z0 = d == 2 ? (((a - R) % n) + n) % n : 0, z1 = (((b - R) % n) + n) % n;
        u[int64_t(k) * N + (d == 2 ? int64_t(z0) * n + z1 : z1)] += U[int64_t(w) * m + k];
      }
  }
}

// v_k(y) from the projections c (s × m) at the cell centres (n/g)(i + ½): periodic bilinear interpolation (R12);
// g = n means one sample per pixel (v_k(y) = c_k(y)).
__global__ void interp_kernel(const double* __restrict__ c, int d, int n, int g, int m, double* __restrict__ v) {
  const int64_t N = d == 2 ? int64_t(n) * n : n;
  const double sp = double(n) / g;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < N * m; t += int64_t(gridDim.x) * blockDim.x) {
    const int k = int(t / N);
    const int64_t y = t - int64_t(k) * N;
    if (g == n) {   // one impulse response per pixel: v_k(y) = <S(·, y), u_k> itself
      v[t] = c[y * m + k];
      continue;
    }
    const int y0 = d == 2 ? int(y / n) : 0, y1 = int(y - int64_t(y0) * n);
    auto axis = [&](int yy, int* i0, int* i1, double* f) {
      const double tt = yy / sp - 0.5;
      const double fl = floor(tt);
      *f = tt - fl;
      const int ii = int(fl);
      *i0 = ((ii % g) + g) % g;
      *i1 = (((ii + 1) % g) + g) % g;
    };
    int a0, a1, b0, b1;
    double fa, fb;
    axis(y1, &b0, &b1, &fb);
    double val;
    if (d == 2) {
      axis(y0, &a0, &a1, &fa);
      const double c00 = c[(int64_t(a0) * g + b0) * m + k], c01 = c[(int64_t(a0) * g + b1) * m + k];
      const double c10 = c[(int64_t(a1) * g + b0) * m + k], c11 = c[(int64_t(a1) * g + b1) * m + k];
      const double r0 = c00 * (1.0 - fa) + c10 * fa, r1 = c01 * (1.0 - fa) + c11 * fa;
      val = r0 * (1.0 - fb) + r1 * fb;
    } else {
      val = c[int64_t(b0) * m + k] * (1.0 - fb) + c[int64_t(b1) * m + k] * fb;
    }
    v[t] = val;
  }
}

}  // namespace

// X (s × W) device; outputs U (W × m), c (s × m) device and sigma (host, m).
int factor(const double* X, int64_t s, int W, int m, int oversample, int power_iters, uint64_t seed, double* U,
           double* c, double* sigma, cudaStream_t st) {
  const int r = std::min(std::min<int64_t>(m + oversample, kMaxR), std::min<int64_t>(W, s));
  if (m > r) return PCWD_E_PARAM;
  double *Y = nullptr, *Z = nullptr, *part = nullptr, *lam = nullptr, *V = nullptr;
  const int64_t chunk = 4096;
  const int nb = int((s + chunk - 1) / chunk);
  const int nbW = int((W + chunk - 1) / chunk);
  struct Free { double** p[5]; ~Free() { for (auto q : p) if (*q) cudaFree(*q); } } fr{{&Y, &Z, &part, &lam, &V}};
  if (cudaMalloc(&Y, sizeof(double) * W * r) || cudaMalloc(&Z, sizeof(double) * s * r) ||
      cudaMalloc(&part, sizeof(double) * std::max(nb, nbW) * r * r) || cudaMalloc(&lam, sizeof(double) * r) ||
      cudaMalloc(&V, sizeof(double) * r * r))
    return PCWD_E_OOM;
  const int gw = int(std::min<int64_t>((s * 32 + kT - 1) / kT, 148 * 16));
  const int gt = int(std::min<int64_t>((int64_t(W) * r + kT - 1) / kT, 148 * 16));
  // (CholeskyQR squares the condition number of Y, which the power iterations drive to ~(σ_1/σ_r)^2: modified
  // Gram–Schmidt with re-orthogonalisation instead)
  auto orth = [&]() { mgs_kernel<<<1, kT, 0, st>>>(Y, W, r, seed); };
  (void)nbW;
  gauss_kernel<<<gt, kT, 0, st>>>(Y, W, r, seed);
  orth();
  for (int it = 0; it < power_iters; ++it) {   // Y ← orth(Xᵀ X Y)
    xy_kernel<<<gw, kT, 0, st>>>(X, Y, Z, s, W, r);
    xtz_kernel<<<gt, kT, 0, st>>>(X, Z, Y, s, W, r);
    orth();
  }
  // Rayleigh–Ritz on span(Y): (XY)ᵀ(XY) = V Λ Vᵀ, u = Y V, σ = sqrt(λ)
  xy_kernel<<<gw, kT, 0, st>>>(X, Y, Z, s, W, r);
  gram_part_kernel<<<nb, kT, 0, st>>>(Z, s, r, chunk, part);
  small_kernel<<<1, kT, 0, st>>>(part, nb, r, 1, nullptr, 0, lam, V);
  ritz_kernel<<<1, kT, 0, st>>>(Y, V, W, r, m, U);
  xy_kernel<<<gw, kT, 0, st>>>(X, U, c, s, W, m);   // projections c = X u
  std::vector<double> lh(r);
  if (cudaMemcpyAsync(lh.data(), lam, sizeof(double) * r, cudaMemcpyDeviceToHost, st) != cudaSuccess) return PCWD_E_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return PCWD_E_CUDA;
  for (int k = 0; k < m; ++k) sigma[k] = std::sqrt(std::max(lh[k], 0.0));
  return cudaGetLastError() == cudaSuccess ? PCWD_OK : PCWD_E_CUDA;
}

int finish(const double* U, const double* c, int d, int n, int R, int g, int m, double* u, double* v, cudaStream_t st) {
  const int64_t N = d == 2 ? int64_t(n) * n : n;
  if (cudaMemsetAsync(u, 0, sizeof(double) * m * N, st) != cudaSuccess) return PCWD_E_CUDA;
  embed_kernel<<<1, 1, 0, st>>>(U, d, n, R, m, u);
  interp_kernel<<<int(std::min<int64_t>((N * m + kT - 1) / kT, 148 * 16)), kT, 0, st>>>(c, d, n, g, m, v);
  return cudaGetLastError() == cudaSuccess ? PCWD_OK : PCWD_E_CUDA;
}

}  // namespace pcwd_pca
