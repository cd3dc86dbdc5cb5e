/* ORACLE (test infrastructure only) — plain fp64 rows of Θ = Ψ* H Ψ, one unit at a time.
 *
 * Θ[μ][λ] = <H ψ_λ, ψ_μ> = <ψ_λ, H* ψ_μ>  (reading R1), so the
 * row of unit μ is Ψ*(H* ψ_μ):
 *   1. ψ_μ = Ψ e_μ by the plain inverse cascade over the whole torus
 *   2. H* ψ_μ (y) = Σ_k v_k(y) Σ_x u_k(x - y) ψ_μ(x)  — the definition of Eq. (2)'s
 *      adjoint, summed over the nonzeros of ψ_μ and of u_k
 *   3. Ψ* of that by the plain forward cascade over the whole torus
 * Filter step on a periodic line of length n' (reading R5):
 *   a[l] = Σ_t h[t] x[(2l+t) mod n'],  d[l] = Σ_i g[i] x[(2l+i) mod n'],
 *   g[i] = (-1)^{1-i} h[1-i], i ∈ [2-2δ, 1].
 * 2-D: axis 0 then axis 1 (reading R6); Λ layout of oracle/basis.py (reading R2/R3).
 *
 * This file shares nothing with the CUDA library; it is called from oracle/rows.py.
 * No windowing, no blocking: every step runs over the full periodic array.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int d, n, J, L;          /* dimension, side, depth, filter length 2δ */
  const double* h;         /* L taps */
  int m;
  const double* u;         /* m × N */
  const double* v;         /* m × N */
} oracle_problem;

static double g_tap(const double* h, int L, int i) { /* g[i], i in [2-L, 1] */
  double s = ((1 - i) % 2 == 0) ? 1.0 : -1.0;
  (void)L;
  return s * h[1 - i];
}

static int md(long a, int n) { /* a mod n in [0, n) */
  while (a >= n) a -= n;
  while (a < 0) a += n;
  return (int)a;
}

/* analysis along a strided line: in[0..n2-1] (stride is), out a/d (stride os).
 * The line is first copied into its periodic extension ext[j] = in[(j - L) mod n2],
 * j < n2 + 2L, so that every tap index 2l+t (t ∈ [0,L)) and 2l+i (i ∈ [2-L,1]) is a
 * plain array index (L > n2, i.e. a folding filter, is covered by the mod). */
static void step_line(const double* in, int n2, long is, double* a, double* dd, long os,
                      const double* h, int L, double* ext) {
  int half = n2 / 2;
  for (int j = 0; j < n2 + 2 * L; ++j) ext[j] = in[(long)md((long)j - L, n2) * is];
  const double* x = ext + L;     /* x[q] = in[q mod n2] for q in [-L, n2+L) */
  for (int l = 0; l < half; ++l) {
    double sa = 0.0, sd = 0.0;
    for (int t = 0; t < L; ++t) sa += h[t] * x[2 * l + t];
    for (int i = 2 - L; i <= 1; ++i) sd += g_tap(h, L, i) * x[2 * l + i];
    a[(long)l * os] = sa;
    dd[(long)l * os] = sd;
  }
}

/* adjoint of step_line: out[...] += ; lines whose a and d are both zero add nothing */
static void unstep_line(const double* a, const double* dd, long os, int n2, double* out, long is,
                        const double* h, int L) {
  int half = n2 / 2;
  for (int l = 0; l < half; ++l) {
    double al = a[(long)l * os], dl = dd[(long)l * os];
    if (al == 0.0 && dl == 0.0) continue;
    for (int t = 0; t < L; ++t) out[(long)md(2L * l + t, n2) * is] += h[t] * al;
    for (int i = 2 - L; i <= 1; ++i) out[(long)md(2L * l + i, n2) * is] += g_tap(h, L, i) * dl;
  }
}

static long sb_offset(int d, int n, int J, int lev, int e) {
  /* Λ layout: coarse (level J) first, then levels J..1 with e = 1,2,3 (d=2) or 1 (d=1) */
  long nJ = n >> J;
  long off = (d == 2) ? nJ * nJ : nJ;
  int ne = (d == 2) ? 3 : 1;
  if (e == 0) return 0;
  for (int l = J; l > lev; --l) {
    long nl = n >> l;
    off += ne * ((d == 2) ? nl * nl : nl);
  }
  long nl = n >> lev;
  return off + (long)(e - 1) * ((d == 2) ? nl * nl : nl);
}

/* forward cascade: x (N, destroyed) -> c (N, Λ layout). work: 2N */
static void forward(const oracle_problem* p, double* x, double* c, double* work, double* ext) {
  int n = p->n, d = p->d, J = p->J, L = p->L;
  double* cur = x;
  for (int lev = 1; lev <= J; ++lev) {
    int n2 = n >> (lev - 1), half = n2 / 2;
    if (d == 1) {
      double* a = work;
      double* dd = c + sb_offset(d, n, J, lev, 1);
      step_line(cur, n2, 1, a, dd, 1, p->h, L, ext);
      memcpy(cur, a, sizeof(double) * half);
    } else {
      /* axis 0: columns of the n2×n2 block (row stride n2) -> t0 (half × n2), t1 */
      double* t0 = work;
      double* t1 = work + (long)half * n2;
      for (int col = 0; col < n2; ++col)
        step_line(cur + col, n2, n2, t0 + col, t1 + col, n2, p->h, L, ext);
      /* axis 1: rows of t0 -> (0,0) and (0,1); rows of t1 -> (1,0), (1,1) */
      double* e01 = c + sb_offset(d, n, J, lev, 1);
      double* e10 = c + sb_offset(d, n, J, lev, 2);
      double* e11 = c + sb_offset(d, n, J, lev, 3);
      double* a00 = cur; /* overwrite in place: cur no longer needed */
      for (int r = 0; r < half; ++r) {
        step_line(t0 + (long)r * n2, n2, 1, a00 + (long)r * half, e01 + (long)r * half, 1, p->h, L, ext);
        step_line(t1 + (long)r * n2, n2, 1, e10 + (long)r * half, e11 + (long)r * half, 1, p->h, L, ext);
      }
    }
  }
  long nJ = n >> J;
  memcpy(c, cur, sizeof(double) * (d == 2 ? nJ * nJ : nJ));
}

/* inverse cascade: c (N, Λ layout) -> x (N). work: 3N */
static void inverse(const oracle_problem* p, const double* c, double* x, double* work) {
  int n = p->n, d = p->d, J = p->J, L = p->L;
  long nJ = n >> J;
  double* cur = work;              /* current approximation, up to N */
  double* nxt = work + (long)n * (d == 2 ? n : 1);
  memcpy(cur, c, sizeof(double) * (d == 2 ? nJ * nJ : nJ));
  for (int lev = J; lev >= 1; --lev) {
    int half = n >> lev, n2 = 2 * half;
    if (d == 1) {
      memset(nxt, 0, sizeof(double) * n2);
      unstep_line(cur, c + sb_offset(d, n, J, lev, 1), 1, n2, nxt, 1, p->h, L);
    } else {
      const double* e01 = c + sb_offset(d, n, J, lev, 1);
      const double* e10 = c + sb_offset(d, n, J, lev, 2);
      const double* e11 = c + sb_offset(d, n, J, lev, 3);
      double* t0 = x;                          /* half × n2 */
      double* t1 = x + (long)half * n2;        /* half × n2 */
      memset(t0, 0, sizeof(double) * (long)half * n2 * 2);
      for (int r = 0; r < half; ++r) {
        unstep_line(cur + (long)r * half, e01 + (long)r * half, 1, n2, t0 + (long)r * n2, 1, p->h, L);
        unstep_line(e10 + (long)r * half, e11 + (long)r * half, 1, n2, t1 + (long)r * n2, 1, p->h, L);
      }
      memset(nxt, 0, sizeof(double) * (long)n2 * n2);
      for (int col = 0; col < n2; ++col)
        unstep_line(t0 + col, t1 + col, n2, n2, nxt + col, n2, p->h, L);
    }
    double* s = cur; cur = nxt; nxt = s;
  }
  memcpy(x, cur, sizeof(double) * (long)n * (d == 2 ? n : 1));
}

/* nonzeros of u_k, listed once (plain bookkeeping, no arithmetic): position (zr, zc), value */
typedef struct { int* zr; int* zc; double* val; long cnt; } nzlist;

/* g = H* psi:  g(y) = Σ_k Σ_x v_k(y) u_k(x - y) psi(x)   (adjoint of Eq. 2):
 * for every nonzero psi(x) and every nonzero u_k(z), y = x - z (mod n per axis). */
static void adjoint_apply(const oracle_problem* p, const nzlist* unz, const double* psi, double* g) {
  int n = p->n, d = p->d;
  long N = (d == 2) ? (long)n * n : n;
  memset(g, 0, sizeof(double) * N);
  for (long x = 0; x < N; ++x) {
    double px = psi[x];
    if (px == 0.0) continue;
    int xr = (d == 2) ? (int)(x / n) : 0;
    int xc = (d == 2) ? (int)(x % n) : (int)x;
    for (int k = 0; k < p->m; ++k) {
      const int* zr = unz[k].zr;
      const int* zc = unz[k].zc;
      const double* uv = unz[k].val;
      const double* vk = p->v + (long)k * N;
      for (long j = 0; j < unz[k].cnt; ++j) {
        int yr = xr - zr[j]; if (yr < 0) yr += n;
        int yc = xc - zc[j]; if (yc < 0) yc += n;
        long y = (long)yr * n + yc;
        g[y] += vk[y] * uv[j] * px;
      }
    }
  }
}

/* Rows of Θ for the given units.  rows: count × N (or NULL); rowmax: count (or NULL) = max|Θ[μ][·]|.
 * bound > 0 (rows == NULL only): a unit whose ‖H*ψ_μ‖₂ is below bound·(1 - 1e-9) cannot hold an
 * entry ≥ bound (Parseval: max_λ |Θ[μ][λ]| ≤ ‖Θ[μ][·]‖₂ = ‖H*ψ_μ‖₂, Ψ orthogonal, P:127,
 * P:1483), so its forward cascade is skipped and rowmax = -‖H*ψ_μ‖₂ is returned instead.
 * Returns 0 on success. */
int oracle_rows(const oracle_problem* p, const int64_t* units, int64_t count, double* rows,
                double* rowmax, int nthreads, double bound) {
  long N = (p->d == 2) ? (long)p->n * p->n : p->n;
  int err = 0;
  nzlist* unz = (nzlist*)calloc(p->m, sizeof(nzlist));
  if (!unz) return 1;
  for (int k = 0; k < p->m; ++k) {
    const double* uk = p->u + (long)k * N;
    unz[k].zr = (int*)malloc(sizeof(int) * N);
    unz[k].zc = (int*)malloc(sizeof(int) * N);
    unz[k].val = (double*)malloc(sizeof(double) * N);
    if (!unz[k].zr || !unz[k].zc || !unz[k].val) return 1;
    for (long z = 0; z < N; ++z)
      if (uk[z] != 0.0) {
        long c = unz[k].cnt++;
        unz[k].zr[c] = (p->d == 2) ? (int)(z / p->n) : 0;
        unz[k].zc[c] = (p->d == 2) ? (int)(z % p->n) : (int)z;
        unz[k].val[c] = uk[z];
      }
  }
#pragma omp parallel num_threads(nthreads > 0 ? nthreads : 1)
  {
    double* buf = (double*)malloc(sizeof(double) * (N * 8 + 2 * (long)p->n + 4 * (long)p->L));
    if (!buf) {
#pragma omp atomic write
      err = 1;
    } else {
      double* e = buf;
      double* psi = buf + N;
      double* g = buf + 2 * N;
      double* c = buf + 3 * N;
      double* work = buf + 4 * N;   /* 3N */
      double* acc = buf + 7 * N;
      double* ext = buf + 8 * N;
#pragma omp for schedule(dynamic, 1)
      for (int64_t i = 0; i < count; ++i) {
        memset(e, 0, sizeof(double) * N);
        e[units[i]] = 1.0;
        inverse(p, e, psi, work);
        adjoint_apply(p, unz, psi, g);
        if (bound > 0.0 && rows == NULL) {
          double s2 = 0.0;
          for (long j = 0; j < N; ++j) s2 += g[j] * g[j];
          double nrm = sqrt(s2);
          if (nrm < bound * (1.0 - 1e-9)) { if (rowmax) rowmax[i] = -nrm; continue; }
        }
        forward(p, g, c, work, ext);
        if (rows) memcpy(rows + i * N, c, sizeof(double) * N);
        if (rowmax) {
          double mx = 0.0;
          for (long j = 0; j < N; ++j) { double a = fabs(c[j]); if (a > mx) mx = a; }
          rowmax[i] = mx;
        }
      }
      free(buf);
    }
  }
  for (int k = 0; k < p->m; ++k) { free(unz[k].zr); free(unz[k].zc); free(unz[k].val); }
  free(unz);
  return err;
}

/* ---- per-unit statistics of the threshold-retained row (all-unit pattern sweeps) ----------------
 * For each unit: cnt = #{λ : |Θ[μ][λ]| ≥ tau} (the closed inequality of reading R15), hash = FNV-1a
 * (32 bit) over the little-endian bytes of the retained λ (int32, increasing), ssq = Σ retained θ²,
 * sketch = Σ retained θ·s(λ) with s(λ) = ±1 from the top bit of splitmix64(λ), rmax = max|Θ[μ][·]|,
 * near = #{λ : ||θ| − tau| ≤ 1e-12·tau} (decisions an fp64 rounding difference could flip).
 * These are bookkeeping over the oracle's own fp64 row; nothing here is the method's arithmetic.
 * A unit whose ‖H*ψ_μ‖₂ < tau retains nothing (Parseval, as in oracle_rows) and skips the cascade. */
static uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

int oracle_row_stats(const oracle_problem* p, const int64_t* units, int64_t count, double tau,
                     int64_t* cnt, uint32_t* hash, double* ssq, double* sketch, double* rmax,
                     int64_t* near, int nthreads) {
  long N = (p->d == 2) ? (long)p->n * p->n : p->n;
  int err = 0;
  nzlist* unz = (nzlist*)calloc(p->m, sizeof(nzlist));
  if (!unz) return 1;
  for (int k = 0; k < p->m; ++k) {
    const double* uk = p->u + (long)k * N;
    unz[k].zr = (int*)malloc(sizeof(int) * N);
    unz[k].zc = (int*)malloc(sizeof(int) * N);
    unz[k].val = (double*)malloc(sizeof(double) * N);
    if (!unz[k].zr || !unz[k].zc || !unz[k].val) return 1;
    for (long z = 0; z < N; ++z)
      if (uk[z] != 0.0) {
        long c = unz[k].cnt++;
        unz[k].zr[c] = (p->d == 2) ? (int)(z / p->n) : 0;
        unz[k].zc[c] = (p->d == 2) ? (int)(z % p->n) : (int)z;
        unz[k].val[c] = uk[z];
      }
  }
#pragma omp parallel num_threads(nthreads > 0 ? nthreads : 1)
  {
    double* buf = (double*)malloc(sizeof(double) * (N * 8 + 2 * (long)p->n + 4 * (long)p->L));
    if (!buf) {
#pragma omp atomic write
      err = 1;
    } else {
      double* e = buf;
      double* psi = buf + N;
      double* g = buf + 2 * N;
      double* c = buf + 3 * N;
      double* work = buf + 4 * N;
      double* ext = buf + 8 * N;
#pragma omp for schedule(dynamic, 1)
      for (int64_t i = 0; i < count; ++i) {
        memset(e, 0, sizeof(double) * N);
        e[units[i]] = 1.0;
        inverse(p, e, psi, work);
        adjoint_apply(p, unz, psi, g);
        double s2 = 0.0;
        for (long j = 0; j < N; ++j) s2 += g[j] * g[j];
        int64_t nc = 0, nn = 0;
        uint32_t hh = 2166136261u;
        double sq = 0.0, sk = 0.0, mx = 0.0;
        if (sqrt(s2) >= tau * (1.0 - 1e-9)) {
          forward(p, g, c, work, ext);
          for (long j = 0; j < N; ++j) {
            double a = fabs(c[j]);
            if (a > mx) mx = a;
            if (fabs(a - tau) <= 1e-12 * tau) ++nn;
            if (a >= tau) {
              ++nc;
              uint32_t col = (uint32_t)j;
              for (int b = 0; b < 4; ++b) { hh ^= (col >> (8 * b)) & 0xffu; hh *= 16777619u; }
              sq += c[j] * c[j];
              sk += (splitmix64((uint64_t)j) >> 63) ? -c[j] : c[j];
            }
          }
        } else {
          mx = -sqrt(s2);
        }
        cnt[i] = nc; hash[i] = hh; ssq[i] = sq; sketch[i] = sk; rmax[i] = mx; near[i] = nn;
      }
      free(buf);
    }
  }
  for (int k = 0; k < p->m; ++k) { free(unz[k].zr); free(unz[k].zc); free(unz[k].val); }
  free(unz);
  return err;
}
