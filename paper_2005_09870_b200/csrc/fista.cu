// fista.cu — consumer of the decomposition: the periodic orthogonal wavelet transform
// Ψ* / Ψ on the plan's grid and FISTA-W / FISTA-WP in the wavelet domain.
//
//   dwt_step    one analysis step of Ψ* (P:94-100): every output of the four (d = 2) or two (d = 1) sub-bands
//               as the direct separable 2δ × 2δ (2δ) tap sum over the periodic input — a[l] = Σ_t h[t] x[2l+t],
//               d[l] = Σ_i g[i] x[2l+i], i ∈ [2−2δ, 1], axis 0 then axis 1; taps fold when the
//               filter is longer than the line
//   idwt_step   its adjoint (the step is orthogonal), as a gather over the taps that reach each output
//   fista_*     the iteration of P:1537-1546: z = Prox^Σ(y − τ Σ Θᵀ(Θ y − z0)), y ← z + (i−1)/(i+2)(z − z_prev),
//               with Σ = I (FISTA-W) or the Jacobi preconditioner diag(ΘᵀΘ)⁻¹ (FISTA-WP, reading R-F1), the
//               Θᵀ products as gathers over the transposed CSR (deterministic), the
//               weighted soft threshold as the Σ-metric prox, τ = 0.99 / ‖Σ^½ ΘᵀΘ Σ^½‖₂ by power iteration.
#include <cstdint>

#include "kernels.cuh"

namespace pcwd {

namespace {
constexpr int kFB = 256;

__device__ __forceinline__ int fold_mod(int a, int n) {   // a mod n for any int a (n a power of two)
  return a & (n - 1);
}

// One analysis step on a (ns × ns) (d = 2) or ns (d = 1) approximation `x`; the approximation goes to `a_out`
// (row-major (ns/2)²), the details straight into their Λ sub-band slots of `c` (offsets off[e − 1]).
template <typename Real>
__global__ void dwt_step(const Plan P, const Real* __restrict__ x, Real* __restrict__ a_out, Real* __restrict__ c,
                         int ns, int64_t off1, int64_t off2, int64_t off3) {
  const int half = ns >> 1, L2 = P.L2;
  const int64_t total = P.d == 2 ? int64_t(half) * half : half;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    if (P.d == 1) {
      const int l = int(i);
      Real a = Real(0), dd = Real(0);
      for (int t = 0; t < L2; ++t) {
        const Real xv = x[fold_mod(2 * l + t, ns)];
        a += Real(P.td[0][t]) * xv;
      }
      for (int t = 0; t < L2; ++t) dd += Real(P.td[1][t]) * x[fold_mod(2 * l + P.to[1] + t, ns)];
      a_out[l] = a;
      c[off1 + l] = dd;
      continue;
    }
    const int l0 = int(i / half), l1 = int(i - int64_t(l0) * half);
    Real o[4] = {Real(0), Real(0), Real(0), Real(0)};   // e = (e0, e1): 0 = (0,0), 1 = (0,1), 2 = (1,0), 3 = (1,1)
    for (int e0 = 0; e0 < 2; ++e0) {
      for (int t0 = 0; t0 < L2; ++t0) {
        const Real* row = x + int64_t(fold_mod(2 * l0 + P.to[e0] + t0, ns)) * ns;
        Real rh = Real(0), rg = Real(0);   // the row filtered along axis 1 by h and by g
        for (int t1 = 0; t1 < L2; ++t1) {
          rh += Real(P.td[0][t1]) * row[fold_mod(2 * l1 + t1, ns)];
          rg += Real(P.td[1][t1]) * row[fold_mod(2 * l1 + P.to[1] + t1, ns)];
        }
        const Real f0 = Real(P.td[e0][t0]);
        o[2 * e0] += f0 * rh;
        o[2 * e0 + 1] += f0 * rg;
      }
    }
    const int64_t p = int64_t(l0) * half + l1;
    a_out[p] = o[0];
    c[off1 + p] = o[1];
    c[off2 + p] = o[2];
    c[off3 + p] = o[3];
  }
}

// Adjoint of dwt_step: x[i] = Σ_e Σ_{t: (i − o_e − t) even} f_e[t] s_e[(i − o_e − t)/2 mod half] per axis.
template <typename Real>
__global__ void idwt_step(const Plan P, const Real* __restrict__ a_in, const Real* __restrict__ c, Real* __restrict__ x,
                          int ns, int64_t off1, int64_t off2, int64_t off3) {
  const int half = ns >> 1, L2 = P.L2;
  const int64_t total = P.d == 2 ? int64_t(ns) * ns : ns;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    if (P.d == 1) {
      const int y = int(i);
      Real acc = Real(0);
      for (int e = 0; e < 2; ++e)
        for (int t = 0; t < L2; ++t) {
          const int q = fold_mod(y - P.to[e] - t, ns);
          if (q & 1) continue;
          acc += Real(P.td[e][t]) * (e ? c[off1 + (q >> 1)] : a_in[q >> 1]);
        }
      x[y] = acc;
      continue;
    }
    const int y0 = int(i / ns), y1 = int(i - int64_t(y0) * ns);
    const Real* src[4] = {a_in, c + off1, c + off2, c + off3};
    Real acc = Real(0);
    for (int e0 = 0; e0 < 2; ++e0)
      for (int t0 = 0; t0 < L2; ++t0) {
        const int q0 = fold_mod(y0 - P.to[e0] - t0, ns);
        if (q0 & 1) continue;
        const int l0 = q0 >> 1;
        Real part = Real(0);
        for (int e1 = 0; e1 < 2; ++e1) {
          const Real* s = src[2 * e0 + e1] + int64_t(l0) * half;
          for (int t1 = 0; t1 < L2; ++t1) {
            const int q1 = fold_mod(y1 - P.to[e1] - t1, ns);
            if (q1 & 1) continue;
            part += Real(P.td[e1][t1]) * s[q1 >> 1];
          }
        }
        acc += Real(P.td[e0][t0]) * part;
      }
    x[i] = acc;
  }
}

template <typename Real>
__global__ void copy_kernel(const Real* __restrict__ s, Real* __restrict__ d, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) d[i] = s[i];
}

// r = Θy − z0 (r holds Θy on entry)
template <typename Real>
__global__ void sub_kernel(Real* __restrict__ r, const Real* __restrict__ z0, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) r[i] -= z0[i];
}

// z = soft(y − τ Σ g, τ Σ w) ;  y ← z + β (z − z_prev) ;  z_prev ← z
template <typename Real>
__global__ void fista_update(Real* __restrict__ y, Real* __restrict__ zprev, Real* __restrict__ zout,
                             const Real* __restrict__ g, const Real* __restrict__ w, const Real* __restrict__ sigma,
                             Real tau, Real beta, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const Real s = sigma ? sigma[i] : Real(1);
    const Real u = y[i] - tau * s * g[i];
    const Real th = tau * s * w[i];
    const Real z = u > th ? u - th : (u < -th ? u + th : Real(0));
    const Real zp = zprev[i];
    zprev[i] = z;
    zout[i] = z;
    y[i] = z + beta * (z - zp);
  }
}

// Jacobi diagonal: D[λ] = Σ_μ Θ[μ][λ]² (fp64), over column λ of the transposed CSR in its fixed (row) order —
// the same bits on every run; then σ = 1 / D (0 where D = 0)
template <typename Real>
__global__ void colsq_kernel(const int64_t* __restrict__ row_ptrT, const Real* __restrict__ valT,
                             double* __restrict__ D, int64_t n) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < n; c += int64_t(gridDim.x) * blockDim.x) {
    double acc = 0.0;
    for (int64_t j = row_ptrT[c]; j < row_ptrT[c + 1]; ++j) acc += double(valT[j]) * double(valT[j]);
    D[c] = acc;
  }
}
template <typename Real>
__global__ void inv_kernel(const double* __restrict__ D, Real* __restrict__ sigma, int64_t n, Real* __restrict__ ssig) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double s = D[i] > 0.0 ? 1.0 / D[i] : 0.0;
    sigma[i] = Real(s);
    ssig[i] = Real(sqrt(s));
  }
}

// out = s ⊙ in (s may be null: copy); the block's sum of squares of out (fp64) into parts[blockIdx.x]
template <typename Real>
__global__ void scale_norm(const Real* __restrict__ in, const Real* __restrict__ s, Real* __restrict__ out, int64_t n,
                           double* __restrict__ parts) {
  __shared__ double red[kFB / 32];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const Real v = s ? in[i] * s[i] : in[i];
    out[i] = v;
    acc += double(v) * double(v);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < kFB / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) parts[blockIdx.x] = acc;
  }
}
// *nrm = Σ parts in a fixed order (one warp): the norm is the same bits on every run and on every rank
__global__ void sum_parts(const double* __restrict__ parts, int np, double* __restrict__ nrm) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += 32) acc += parts[i];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (threadIdx.x == 0) *nrm = acc;
}
// v = in / sqrt(*nrm)
template <typename Real>
__global__ void normalize(const Real* __restrict__ in, Real* __restrict__ v, int64_t n, const double* __restrict__ nrm) {
  const double inv = *nrm > 0.0 ? 1.0 / sqrt(*nrm) : 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    v[i] = Real(double(in[i]) * inv);
}
__global__ void init_vec(float* f, double* dd, int64_t n, unsigned seed) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    unsigned x = unsigned(i) * 2654435761u ^ seed;   // fixed pseudo-random start vector (deterministic)
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    const double v = 0.5 + double(x & 0xffffu) / 65536.0;
    if (f) f[i] = float(v);
    if (dd) dd[i] = v;
  }
}

int grid_of(int64_t n) {
  int64_t g = (n + kFB - 1) / kFB;
  return int(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}
}  // namespace

cudaError_t launch_wavelet_transform(const Plan& P, const void* in, void* out, void* work0, void* work1, int inverse,
                                     int rb, cudaStream_t st) {
  const int n = P.n, J = P.J;
  auto run = [&](auto tag) -> cudaError_t {
    using Real = decltype(tag);
    const Real* src = static_cast<const Real*>(in);
    Real* c = static_cast<Real*>(out);
    Real* w0 = static_cast<Real*>(work0);
    Real* w1 = static_cast<Real*>(work1);
    // sub-band offsets of level ℓ (Λ order): coarse block, then levels J..1 × orientations
    auto off = [&](int lev, int e) -> int64_t {
      const int nJ = n >> J;
      int64_t o = P.d == 2 ? int64_t(nJ) * nJ : nJ;
      for (int l = J; l > lev; --l) {
        const int nl = n >> l;
        o += (P.d == 2 ? 3 : 1) * (P.d == 2 ? int64_t(nl) * nl : nl);
      }
      const int nl = n >> lev;
      return o + int64_t(e - 1) * (P.d == 2 ? int64_t(nl) * nl : nl);
    };
    const int64_t N = P.d == 2 ? int64_t(n) * n : n;
    if (!inverse) {
      const Real* cur = src;
      Real* bufs[2] = {w0, w1};
      for (int lev = 1; lev <= J; ++lev) {
        const int ns = n >> (lev - 1);
        Real* a = lev == J ? c : bufs[lev & 1];   // the last approximation is the coarse block (offset 0)
        const int64_t o1 = off(lev, 1), o2 = P.d == 2 ? off(lev, 2) : 0, o3 = P.d == 2 ? off(lev, 3) : 0;
        dwt_step<Real><<<grid_of(P.d == 2 ? int64_t(ns / 2) * (ns / 2) : ns / 2), kFB, 0, st>>>(P, cur, a, c, ns, o1, o2, o3);
        cur = a;
      }
      (void)N;
    } else {
      const Real* a = src;   // coarse block at offset 0
      Real* bufs[2] = {w0, w1};
      for (int lev = J; lev >= 1; --lev) {
        const int ns = n >> (lev - 1);
        Real* xo = lev == 1 ? c : bufs[lev & 1];
        const int64_t o1 = off(lev, 1), o2 = P.d == 2 ? off(lev, 2) : 0, o3 = P.d == 2 ? off(lev, 3) : 0;
        idwt_step<Real><<<grid_of(P.d == 2 ? int64_t(ns) * ns : ns), kFB, 0, st>>>(P, a, src, xo, ns, o1, o2, o3);
        a = xo;
      }
    }
    return cudaGetLastError();
  };
  return rb == 4 ? run(float()) : run(double());
}

cudaError_t launch_fista(const Plan& P, const FistaArgs& F, int rb, cudaStream_t st, double* tau_io, int* cb_failed) {
  const int64_t N = F.N, rows = F.rows;
  *cb_failed = 0;
  // sharded Θ (rows [row0, row0 + rows)): Θ y is local to the rows, Θᵀ r = Σ_ranks Θ_rᵀ r_r is summed by the
  // caller's reduce; every other vector is replicated and updated identically on every rank
  auto reduce = [&](int which) -> cudaError_t {
    if (!F.reduce) return cudaSuccess;
    if (F.reduce(which, F.rctx) != 0) { *cb_failed = 1; return cudaErrorUnknown; }
    return cudaSuccess;
  };
  auto run = [&](auto tag) -> cudaError_t {
    using Real = decltype(tag);
    Real* y = static_cast<Real*>(F.y);
    Real* zp = static_cast<Real*>(F.zprev);
    Real* r = static_cast<Real*>(F.r);
    Real* g = static_cast<Real*>(F.g);
    Real* sig = F.precond ? static_cast<Real*>(F.sigma) : nullptr;
    const Real* z0 = static_cast<const Real*>(F.z0) + F.row0;
    const Real* w = static_cast<const Real*>(F.w);
    Real* zo = static_cast<Real*>(F.z_out);
    cudaError_t e;
    Real* ssig = sig ? static_cast<Real*>(F.sqrt_sigma) : nullptr;
    if (F.precond) {   // Jacobi diagonal of ΘᵀΘ (column sums of squares over all rows), σ = D⁻¹, and σ^½
      colsq_kernel<Real><<<grid_of(N), kFB, 0, st>>>(F.row_ptrT, static_cast<const Real*>(F.valT), F.D, N);
      if ((e = reduce(1))) return e;
      inv_kernel<Real><<<grid_of(N), kFB, 0, st>>>(F.D, sig, N, ssig);
    }
    double tau = *tau_io;
    if (tau <= 0.0) {   // power iteration on M = Σ^½ ΘᵀΘ Σ^½ (Σ = I for FISTA-W): v ← M v / ‖M v‖
      Real* v = y;
      double* nrm = F.dbuf;
      double* parts = F.dbuf + 1;
      const int gN = grid_of(N);
      init_vec<<<gN, kFB, 0, st>>>(rb == 4 ? reinterpret_cast<float*>(v) : nullptr,
                                   rb == 8 ? reinterpret_cast<double*>(v) : nullptr, N, 12345u);
      double lam = 0.0;
      for (int it = 0; it < F.power_iters; ++it) {
        // u = Σ^½ v (into g), r = Θ u, g = Θᵀ r, u = Σ^½ g (into r), ‖u‖
        if (ssig) scale_norm<Real><<<gN, kFB, 0, st>>>(v, ssig, g, N, parts);
        else copy_kernel<Real><<<gN, kFB, 0, st>>>(v, g, N);
        if ((e = launch_spmv(F.row_ptr, F.col, F.val, g, r, rows, N, 0, rb, st))) return e;
        if ((e = launch_spmv(F.row_ptrT, F.rowT, F.valT, r, g, N, rows, 0, rb, st))) return e;
        if ((e = reduce(0))) return e;
        scale_norm<Real><<<gN, kFB, 0, st>>>(g, ssig, r, N, parts);
        sum_parts<<<1, 32, 0, st>>>(parts, gN, nrm);
        normalize<Real><<<gN, kFB, 0, st>>>(r, v, N, nrm);
        // every 8 iterations: stop once ‖M v‖ changes by less than 1e-6 (relative); the norm is deterministic and
        // g is the same on every rank after the reduce, so every rank takes the same decision
        if ((it + 1) % 8 == 0 && it + 1 < F.power_iters) {
          double cur = 0.0;
          if ((e = cudaMemcpyAsync(&cur, nrm, sizeof(double), cudaMemcpyDeviceToHost, st))) return e;
          if ((e = cudaStreamSynchronize(st))) return e;
          if (lam > 0.0 && fabs(cur - lam) <= 1e-6 * cur) break;
          lam = cur;
        }
      }
      if ((e = cudaMemcpyAsync(&lam, nrm, sizeof(double), cudaMemcpyDeviceToHost, st))) return e;
      if ((e = cudaStreamSynchronize(st))) return e;
      lam = sqrt(lam);   // ‖M v‖ with ‖v‖ = 1 → the top eigenvalue of M at convergence
      tau = lam > 0.0 ? 0.99 / lam : 1.0;
      *tau_io = tau;
    }
    // iterations: z^(0) = y^(1) = 0
    if ((e = cudaMemsetAsync(y, 0, N * rb, st))) return e;
    if ((e = cudaMemsetAsync(zp, 0, N * rb, st))) return e;
    for (int i = 1; i <= F.iters; ++i) {
      if ((e = launch_spmv(F.row_ptr, F.col, F.val, y, r, rows, N, 0, rb, st))) return e;    // r = Θ y (rows)
      sub_kernel<Real><<<grid_of(rows), kFB, 0, st>>>(r, z0, rows);                          // r −= z0 (rows)
      if ((e = launch_spmv(F.row_ptrT, F.rowT, F.valT, r, g, N, rows, 0, rb, st))) return e;  // g = Θᵀ r (gather)
      if ((e = reduce(0))) return e;                                                         // Σ over the shards
      const Real beta = Real(double(i - 1) / double(i + 2));
      fista_update<Real><<<grid_of(N), kFB, 0, st>>>(y, zp, zo, g, w, sig, Real(tau), beta, N);
    }
    return cudaGetLastError();
  };
  return rb == 4 ? run(float()) : run(double());
}

}  // namespace pcwd
