// plan.cpp — validation, sub-band table, template / unit windows, band stencil, shard split.
//
// Passages: Λ and its layout P:113-125 (R2/R3); supports P:99-104 and the
// recursion P:96 (R7); Lemma 6 P:1294-1301 for the cascade windows; Theorem 2 / Remark
// P:1163-1180 for the band rule (R16); cost-balanced unit sharding.
#include "plan.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <set>
#include <tuple>

namespace pcwd {

static bool is_pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }
static int ilog2(int64_t x) {
  int l = 0;
  while ((int64_t(1) << l) < x) ++l;
  return l;
}

int validate_desc(const pcwd_desc* d, std::string* msg) {
  if (!d) { *msg = "desc is NULL"; return PCWD_E_PARAM; }
  if (d->d != 1 && d->d != 2) { *msg = "d must be 1 or 2"; return PCWD_E_SHAPE; }
  if (!is_pow2(d->n) || d->n < 2) { *msg = "n must be a power of two >= 2"; return PCWD_E_SHAPE; }
  if (d->d == 2 && d->n > (1 << 14)) { *msg = "n too large for d = 2 (max 16384)"; return PCWD_E_SHAPE; }
  if (d->d == 1 && d->n > (1 << 24)) { *msg = "n too large for d = 1"; return PCWD_E_SHAPE; }
  int lg = ilog2(d->n);
  if (d->levels < 1 || d->levels > lg || d->levels > kMaxJ) { *msg = "levels must be in [1, log2 n]"; return PCWD_E_CONFIG; }
  if (d->filter_len < 2 || d->filter_len > kMaxTaps || (d->filter_len & 1)) {
    *msg = "filter_len must be even, 2..20"; return PCWD_E_CONFIG;
  }
  if (!d->h) { *msg = "h is NULL"; return PCWD_E_PARAM; }
  {  // an orthogonal wavelet filter: ‖h‖₂ = 1, Σ h = √2, Σ_n h[n] h[n+2k] = 0 (k ≠ 0)
    const int L = d->filter_len;
    double s1 = 0.0;
    for (int i = 0; i < L; ++i) s1 += d->h[i];
    if (std::fabs(s1 - std::sqrt(2.0)) > 1e-9) { *msg = "h: sum must be sqrt(2) (low-pass filter of an orthogonal wavelet)"; return PCWD_E_CONFIG; }
    for (int k = 0; 2 * k < L; ++k) {
      double a = 0.0;
      for (int i = 0; i + 2 * k < L; ++i) a += d->h[i] * d->h[i + 2 * k];
      if (std::fabs(a - (k == 0 ? 1.0 : 0.0)) > 1e-9) {
        *msg = k == 0 ? "h: norm must be 1" : "h: not orthogonal to its even shifts (sum h[n]h[n+2k] != 0)";
        return PCWD_E_CONFIG;
      }
    }
  }
  if (d->m < 1) { *msg = "m must be >= 1"; return PCWD_E_PARAM; }
  if (d->dtype != PCWD_F32 && d->dtype != PCWD_F64) { *msg = "dtype"; return PCWD_E_PARAM; }
  int64_t N = d->d == 2 ? int64_t(d->n) * d->n : d->n;
  if (d->retain == PCWD_RETAIN_THRESHOLD) {
    if (!(d->tau_rel > 0.0)) { *msg = "tau_rel must be > 0"; return PCWD_E_PARAM; }
  } else if (d->retain == PCWD_RETAIN_BAND) {
    if (d->band_L < 1 || d->band_L > N) { *msg = "band_L must be in [1, N]"; return PCWD_E_PARAM; }
    if (d->band_L > 4096) { *msg = "band_L > 4096 not supported"; return PCWD_E_UNSUPPORTED; }
  } else if (d->retain == PCWD_RETAIN_PATTERN) {
    if (!d->pat_rowptr || !d->pat_col) { *msg = "PATTERN needs pat_rowptr and pat_col"; return PCWD_E_PARAM; }
  } else if (d->retain != PCWD_RETAIN_FULL) {
    *msg = "retain"; return PCWD_E_PARAM;
  }
  if (d->retain == PCWD_RETAIN_FULL && N > (1 << 16)) { *msg = "full retention limited to N <= 65536"; return PCWD_E_UNSUPPORTED; }
  if (d->world < 1 || d->rank < 0 || d->rank >= d->world) { *msg = "rank must be in [0, world)"; return PCWD_E_PARAM; }
  return PCWD_OK;
}

int sb_index(int d, int J, int level, int e) {
  if (e == 0) return 0;
  int ne = d == 2 ? 3 : 1;
  return 1 + (J - level) * ne + (e - 1);
}

// Periodic bounding box [zlo, zhi] (zlo may be negative) of the nonzeros along one axis.
static void axis_bbox(const std::vector<char>& occ, int n, int* zlo, int* zhi) {
  int cnt = 0;
  for (char c : occ) cnt += c != 0;
  if (cnt == 0) { *zlo = 0; *zhi = 0; return; }
  if (cnt == n) { *zlo = 0; *zhi = n - 1; return; }
  // largest circular run of zeros
  int best_len = 0, best_end = -1;  // run ends at best_end (inclusive)
  for (int start = 0; start < n; ++start) {
    if (occ[start] || !occ[(start - 1 + n) % n]) continue;  // run must start after a nonzero
    int len = 0;
    while (len < n && !occ[(start + len) % n]) ++len;
    if (len > best_len) { best_len = len; best_end = (start + len - 1) % n; }
  }
  int first = (best_end + 1) % n;            // first occupied position of the arc
  int arc = n - best_len;
  int lo = first > n / 2 ? first - n : first;
  *zlo = lo;
  *zhi = lo + arc - 1;
}

// Window of one template axis after the à-trous step (dilation dil, orientation e).
struct Win1 {
  int S, W;  // W == n ⇒ whole line, S = 0
};

static Win1 win_next(Win1 in, int n, int dil, int L2, int e) {
  int64_t W = int64_t(in.W) + int64_t(dil) * (L2 - 1);
  if (in.W >= n || W >= n) return Win1{0, n};
  int o = e ? 2 - L2 : 0;
  int S = int(((int64_t(in.S) + int64_t(dil) * o) % n + n) % n);
  return Win1{S, int(W)};
}

// ---------------------------------------------------------------- band rule (R16)
namespace {
struct Cand {
  int key0, delta, rho, level, e, o2, o0, o1, sb;
  bool operator<(const Cand& b) const {
    return std::tie(key0, delta, rho, level, e, o2, o0, o1) <
           std::tie(b.key0, b.delta, b.rho, b.level, b.e, b.o2, b.o0, b.o1);
  }
};
inline int canon(int64_t raw, int nl) {   // [-nl/2, nl/2)
  int64_t half = nl / 2;
  int64_t r = ((raw + half) % nl + nl) % nl;
  return int(r - half);
}
inline int pdist(int64_t q, int nc) {
  int64_t r = ((q % nc) + nc) % nc;
  return int(std::min<int64_t>(r, nc - r));
}
inline int64_t floordiv(int64_t a, int64_t b) {  // b > 0
  return a >= 0 ? a / b : -((-a + b - 1) / b);
}
}  // namespace

static void build_stencil(const Plan& P, int s_mu, int L, std::vector<Stencil>* out) {
  const SubBand& mu = P.sb[s_mu];
  int d = P.d;
  for (int S = 0;; ++S) {
    std::vector<Cand> cands;
    for (int s = 0; s < P.nsb; ++s) {
      const SubBand& lam = P.sb[s];
      int delta = std::abs(lam.level - mu.level);
      if (delta > S) continue;
      int rmax = S - delta;
      int nl = lam.nl;
      int lc = std::max(lam.level, mu.level);
      int nc = P.n >> lc;
      bool finer = lam.level < mu.level;
      // candidate offsets per axis
      std::vector<int> offs;
      {
        std::set<int> seen;
        int64_t lo, hi;
        if (finer) { lo = -int64_t(rmax) << delta; hi = ((int64_t(rmax) + 1) << delta) - 1; }
        else { lo = -rmax; hi = rmax; }
        for (int64_t o = lo; o <= hi; ++o) {
          int c = canon(o, nl);
          if (seen.insert(c).second) offs.push_back(c);
          if ((int64_t)seen.size() >= nl) break;
        }
      }
      auto rho_of = [&](int o) {
        int64_t q = finer ? floordiv(o, int64_t(1) << delta) : o;
        return pdist(q, nc);
      };
      if (d == 1) {
        for (int o1 : offs) {
          int rho = rho_of(o1);
          if (delta + rho > S) continue;
          cands.push_back(Cand{delta + rho, delta, rho, lam.level, lam.e, o1 * o1, 0, o1, s});
        }
      } else {
        for (int o0 : offs)
          for (int o1 : offs) {
            int rho = std::max(rho_of(o0), rho_of(o1));
            if (delta + rho > S) continue;
            cands.push_back(Cand{delta + rho, delta, rho, lam.level, lam.e, o0 * o0 + o1 * o1, o0, o1, s});
          }
      }
    }
    bool exhausted = S > P.J + P.n;
    if ((int)cands.size() >= L || exhausted) {
      std::sort(cands.begin(), cands.end());
      std::vector<Stencil> pick;
      for (int i = 0; i < L && i < (int)cands.size(); ++i)
        pick.push_back(Stencil{cands[i].sb, cands[i].o0, cands[i].o1, 0});
      // storage order (sb, o0, o1): the CSR column order of every unit whose partners do not wrap
      std::sort(pick.begin(), pick.end(), [](const Stencil& a, const Stencil& b) {
        return std::tie(a.sb, a.o0, a.o1) < std::tie(b.sb, b.o0, b.o1);
      });
      out->insert(out->end(), pick.begin(), pick.end());
      return;
    }
  }
}

// Base atom W_{s,e} of the separable path (geom.h): the level-s analysis functional of orientation e at position
// 0 on the integer line, W_{1,e}(y) = f_e[y − o_e], W_{s,e}(y) = Σ_j f_e[j] · W_{s−1,0}(y − 2^{s−1}(o_e + j)) (P:96,
// R5); w[i] = W_{s,e}(sep_atom_start(s, e) + i), i < sep_atom_len(s).  fp64.
void sep_base_atom(const Plan& P, int s, int e, std::vector<double>* out) {
  const int L2 = P.L2;
  std::vector<double> prev;   // W_{s'-1,0}
  for (int s2 = 1; s2 <= s; ++s2) {
    const int len = sep_atom_len(s2, L2);
    const int ee = s2 == s ? e : 0;
    std::vector<double> w(len, 0.0);
    if (s2 == 1) {
      for (int j = 0; j < L2; ++j) w[j] = P.td[ee][j];
    } else {
      const int dil = 1 << (s2 - 1);
      for (int j = 0; j < L2; ++j)
        for (size_t i = 0; i < prev.size(); ++i) w[dil * j + i] += P.td[ee][j] * prev[i];
    }
    if (s2 == s) *out = w;
    else prev = w;
  }
}

// Separable direct path of the fine kernel (geom.h): base atoms W_{s,e} and, per fine sub-band and class,
// the stage-1 runs over the distinct column atoms and the stage-2 partner records.  A level is marked usable
// only if every one of its class records could be built (no atom wraps onto the window, partner levels
// ≤ sep_smax).
static void build_sep(HostPlan* hp) {
  Plan& P = hp->P;
  const int L2 = P.L2, n = P.n, J = P.J, ns = P.nsb;
  hp->atoms.clear();
  hp->sepcls.assign(hp->fgeom.size(), SepClass{});
  hp->seprun.clear();
  hp->seppart.clear();
  hp->septask.clear();
  for (int l = 0; l <= kMaxJ; ++l) hp->sep_ok[l] = hp->sep_nq[l] = hp->sep_nrun[l] = 0;
  if (P.retain != PCWD_RETAIN_BAND || P.d != 2 || hp->fgeom.empty() || (L2 != 4 && L2 != 8 && L2 != 12)) return;
  const int smax = std::min(J, kSepSmax);
  hp->sep_smax = smax;
  for (int s = 1; s <= smax; ++s) {
    hp->atom_len[s] = sep_atom_len(s, L2);
    for (int e = 0; e < 2; ++e) {
      std::vector<double> w;
      sep_base_atom(P, s, e, &w);
      hp->atom_off[s][e] = int(hp->atoms.size());
      hp->atoms.insert(hp->atoms.end(), w.begin(), w.end());
    }
  }
  auto sstart = [&](int s, int e) { return sep_atom_start(s, e, L2); };   // support start of W_{s,e}
  const int PADC = L2;    // zero columns guaranteed on both sides of every R row (fine kernel layout)
  int ok_lev[kMaxJ + 1], seen[kMaxJ + 1];
  for (int l = 0; l <= kMaxJ; ++l) ok_lev[l] = 1, seen[l] = 0;
  for (int sbi = 0; sbi < ns; ++sbi) {
    const SubBand& S = P.sb[sbi];
    if (S.fg_m <= 0) continue;
    const int lev = S.level, M = S.fg_m;
    seen[lev] = 1;
    const int R0 = S.tW[0], R1 = S.tW[1];
    for (int q0 = 0; q0 < M && ok_lev[lev]; ++q0)
      for (int q1 = 0; q1 < M && ok_lev[lev]; ++q1) {
        SepClass& C = hp->sepcls[S.fg_off + q0 * M + q1];
        const int w0 = (q0 << lev) + S.tSu[0], w1 = (q1 << lev) + S.tSu[1];
        struct Ent { int sp, e0, e1, l0, l1; };
        std::vector<Ent> ents(P.band_L);
        std::vector<std::tuple<int, int, int>> keys;   // distinct column atoms (s, e1, l1)
        for (int jj = 0; jj < P.band_L; ++jj) {
          const Stencil& st = hp->stencil[S.stencil_off + jj];
          const SubBand& T = P.sb[st.sb];
          const int sp = T.level, D = sp - lev;
          if (sp > smax || hp->atom_len[sp] + std::max(R0, R1) > n) { ok_lev[lev] = 0; break; }
          const int b0 = D == 0 ? q0 : (D < 0 ? (q0 << -D) : (q0 >> D));
          const int b1 = D == 0 ? q1 : (D < 0 ? (q1 << -D) : (q1 >> D));
          ents[jj] = Ent{sp, T.e0, T.e1, b0 + st.o0, b1 + st.o1};
          keys.emplace_back(sp, T.e1, b1 + st.o1);
        }
        if (!ok_lev[lev]) break;
        std::sort(keys.begin(), keys.end());
        keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
        // stage-1 runs: consecutive positions of one (s, e1), at most sep_bmax(s) atoms; Q columns in run order
        std::vector<int> qcol(keys.size(), -1), qrun(keys.size(), -1);
        std::vector<SepRun> runs;
        int nq = 0;
        bool open = false;
        int last_sp = -1, last_e = -1, last_l = 0;
        for (size_t k = 0; k < keys.size(); ++k) {
          const int sp = std::get<0>(keys[k]), e1 = std::get<1>(keys[k]), l1 = std::get<2>(keys[k]);
          const int len = hp->atom_len[sp];
          const int st1 = l1 * (1 << sp) + sstart(sp, e1) - w1;
          if (st1 >= R1 || st1 + len <= 0) { open = false; continue; }   // misses the window: its partners are 0
          if (open && sp == last_sp && e1 == last_e && l1 == last_l + 1 && runs.back().B < sep_bmax(sp)) {
            runs.back().B++;
          } else {
            runs.push_back(SepRun{sp, e1, st1, 1, nq, 1 << 30, -(1 << 30), 0, sep_toff(sp, e1, L2), 0});
            open = true;
          }
          last_sp = sp; last_e = e1; last_l = l1;
          qcol[k] = nq++;
          qrun[k] = int(runs.size()) - 1;
        }
        // partners: Q column, row atom (clipped range → rows stage 1 must provide)
        struct PR { int g, sp, e0, l0, jj, st0; };
        std::vector<PR> prs;
        for (int jj = 0; jj < P.band_L; ++jj) {
          const Ent& E = ents[jj];
          const size_t k = std::lower_bound(keys.begin(), keys.end(), std::make_tuple(E.sp, E.e1, E.l1)) - keys.begin();
          const int len = hp->atom_len[E.sp];
          const int st0 = E.l0 * (1 << E.sp) + sstart(E.sp, E.e0) - w0;
          const int ta = std::max(0, -st0), tb = std::min(len, R0 - st0);
          if (qcol[k] < 0 || tb <= ta) continue;   // Θ entry 0 (the kernel zeroes every slot first)
          SepRun& r = runs[qrun[k]];
          r.r0 = std::min(r.r0, st0 + ta);
          r.r1 = std::max(r.r1, st0 + tb);
          prs.push_back(PR{qcol[k], E.sp, E.e0, E.l0, jj, st0});
        }
        // stage-2 runs: partners of one (g, s, e0) at consecutive l0 with a constant slot stride
        std::sort(prs.begin(), prs.end(), [](const PR& x, const PR& y) {
          return std::tie(x.g, x.sp, x.e0, x.l0) < std::tie(y.g, y.sp, y.e0, y.l0);
        });
        std::vector<SepPart> parts;
        for (size_t i = 0; i < prs.size(); ++i) {
          const PR& x = prs[i];
          if (!parts.empty() && i > 0) {
            SepPart& pp = parts.back();
            const PR& y = prs[i - 1];
            const bool same = x.g == y.g && x.sp == y.sp && x.e0 == y.e0 && x.l0 == y.l0 + 1;
            const int js = x.jj - y.jj;
            if (same && pp.B < kSepPartB && (pp.B == 1 || js == pp.jstr)) {
              pp.jstr = js;
              pp.B++;
              continue;
            }
          }
          parts.push_back(SepPart{x.g, x.sp, x.e0, x.st0, 1, x.jj, 0, 0, 0, sep_toff(x.sp, x.e0, L2), {0, 0}});
        }
        for (auto& r : runs) {
          if (r.r1 <= r.r0) r.r0 = r.r1 = 0;
          // columns read by the register window (incl. the rounded-up atoms) vs the zero pads around the row
          const int end = r.c + (sep_atom_blk(r.s, L2) << r.s) + (sep_bsel(r.s, r.B) - 1) * (1 << r.s);
          r.mask = (r.c < -kSepPad || end > R1 + kSepPad) ? 1 : 0;
        }
        std::vector<int> colrun(nq, 0);
        for (size_t r = 0; r < runs.size(); ++r)
          for (int b = 0; b < runs[r].B; ++b) colrun[runs[r].q + b] = int(r);
        for (auto& pp : parts) { pp.r0 = runs[colrun[pp.g]].r0; pp.r1 = runs[colrun[pp.g]].r1; }
        // stage-2 tasks grouped by kernel variant (atom level), each group padded to whole warps (g = -1: no-op)
        std::stable_sort(parts.begin(), parts.end(), [](const SepPart& x, const SepPart& y) { return x.s < y.s; });
        C.part_off = int(hp->seppart.size());
        for (size_t i = 0; i < parts.size(); ++i) {
          hp->seppart.push_back(parts[i]);
          if (i + 1 == parts.size() || parts[i + 1].s != parts[i].s)
            while ((hp->seppart.size() - C.part_off) % 32) hp->seppart.push_back(SepPart{-1, parts[i].s, 0, 0, 0, 0, 0, 0, 0, 0, {0, 0}});
        }
        C.npart = int(hp->seppart.size()) - C.part_off;
        C.run_off = int(hp->seprun.size());
        C.nrun = int(runs.size());
        C.task_off = int(hp->septask.size());
        if (runs.size() > size_t(kSepMaxRuns)) { ok_lev[lev] = 0; break; }
        // stage-1 tasks (run << 16 | row) grouped by kernel variant (atom level, register-window width, mask) so
        // that a warp's 32 consecutive tasks take one code path; each group padded to whole warps (-1: no-op)
        std::vector<int> ord(runs.size());
        for (size_t r = 0; r < runs.size(); ++r) ord[r] = int(r);
        auto vkey = [&](int r) { return std::make_tuple(runs[r].s, sep_bsel(runs[r].s, runs[r].B), runs[r].mask); };
        std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return vkey(x) < vkey(y); });
        for (size_t i = 0; i < ord.size(); ++i) {
          const int r = ord[i];
          runs[r].tbeg = int(hp->septask.size()) - C.task_off;
          for (int row = runs[r].r0; row < runs[r].r1; ++row) hp->septask.push_back(r << 16 | row);
          if (i + 1 == ord.size() || vkey(ord[i + 1]) != vkey(r))
            while ((hp->septask.size() - C.task_off) % 32) hp->septask.push_back(-1);
        }
        hp->seprun.insert(hp->seprun.end(), runs.begin(), runs.end());
        C.ntask = int(hp->septask.size()) - C.task_off;
        C.nq = nq;
        hp->sep_nq[lev] = std::max(hp->sep_nq[lev], nq);
        hp->sep_nrun[lev] = std::max(hp->sep_nrun[lev], C.nrun);
      }
  }
  for (int l = 1; l <= kMaxJ; ++l) hp->sep_ok[l] = seen[l] && ok_lev[l];
  if (getenv("PCWD_DEBUG_SEP")) {   // per level: executed FMAs per unit (padded runs) by atom level, both stages
    for (int lev = 1; lev <= J; ++lev) {
      if (!hp->sep_ok[lev]) continue;
      double f1[kSepSmax + 1] = {}, f2[kSepSmax + 1] = {}, ncls = 0, ntask = 0, npart = 0, nmask = 0;
      for (int sbi = 0; sbi < ns; ++sbi) {
        const SubBand& S = P.sb[sbi];
        if (S.fg_m <= 0 || S.level != lev) continue;
        for (int c = 0; c < S.fg_m * S.fg_m; ++c) {
          const SepClass& C = hp->sepcls[S.fg_off + c];
          ncls += 1; ntask += C.ntask; npart += C.npart;
          for (int r = 0; r < C.nrun; ++r) {
            const SepRun& R = hp->seprun[C.run_off + r];
            f1[R.s] += double(sep_bsel(R.s, R.B)) * (sep_atom_blk(R.s, L2) << R.s) * (R.r1 - R.r0);
            nmask += R.mask * (R.r1 - R.r0);
          }
          for (int r = 0; r < C.npart; ++r) {
            const SepPart& R = hp->seppart[C.part_off + r];
            f2[R.s] += double(sep_bsel(R.s, R.B)) * (sep_atom_blk(R.s, L2) << R.s);
          }
        }
      }
      fprintf(stderr, "[pcwd sep] level %d classes %.0f stage-1 tasks/unit %.1f (masked %.1f) stage-2 runs/unit %.1f nq %d | executed FMA/unit"
              " by s=1..5: stage 1 %.0f %.0f %.0f %.0f %.0f, stage 2 %.0f %.0f %.0f %.0f %.0f\n", lev, ncls, ntask / ncls, nmask / ncls,
              npart / ncls, hp->sep_nq[lev], f1[1] / ncls, f1[2] / ncls, f1[3] / ncls, f1[4] / ncls, f1[5] / ncls,
              f2[1] / ncls, f2[2] / ncls, f2[3] / ncls, f2[4] / ncls, f2[5] / ncls);
    }
  }
}

int build_plan(const pcwd_desc* d, const double* u_host, HostPlan* hp, std::string* msg) {
  int rc = validate_desc(d, msg);
  if (rc) return rc;
  Plan& P = hp->P;
  std::memset(&P, 0, sizeof(Plan));
  P.d = d->d;
  P.n = d->n;
  P.J = d->levels;
  P.L2 = d->filter_len;
  P.m = d->m;
  P.N = d->d == 2 ? int64_t(d->n) * d->n : d->n;
  P.retain = d->retain;
  P.band_L = d->retain == PCWD_RETAIN_BAND ? d->band_L : 0;
  P.band_Lpad = 1;
  while (P.band_Lpad < P.band_L) P.band_Lpad <<= 1;
  const int n = P.n, J = P.J, L2 = P.L2;
  // taps: f_0 = h (o_0 = 0); f_1[j] = g[i], i = 2 - L2 + j, g[i] = (-1)^{1-i} h[1-i]
  P.to[0] = 0;
  P.to[1] = 2 - L2;
  for (int j = 0; j < L2; ++j) {
    int i = 2 - L2 + j;
    double g = (((1 - i) % 2) == 0 ? 1.0 : -1.0) * d->h[1 - i];
    P.td[0][j] = d->h[j];
    P.td[1][j] = g;
    P.tf[0][j] = float(d->h[j]);
    P.tf[1][j] = float(g);
  }
  hp->real_bytes = (d->dtype == PCWD_F64 || d->retain == PCWD_RETAIN_THRESHOLD) ? 8 : 4;
  hp->out_bytes = d->dtype == PCWD_F64 ? 8 : 4;

  // periodic bounding box of supp u_k (union over k), per axis
  if (u_host) {
    std::vector<char> occ0(n, 0), occ1(n, 0);
    for (int k = 0; k < P.m; ++k)
      for (int64_t z = 0; z < P.N; ++z)
        if (u_host[k * P.N + z] != 0.0) {
          if (P.d == 2) { occ0[z / n] = 1; occ1[z % n] = 1; }
          else occ1[z] = 1;
        }
    axis_bbox(occ1, n, &P.zlo[1], &P.zhi[1]);
    if (P.d == 2) axis_bbox(occ0, n, &P.zlo[0], &P.zhi[0]);
  } else {
    P.zlo[1] = 0; P.zhi[1] = n - 1;
    if (P.d == 2) { P.zlo[0] = 0; P.zhi[0] = n - 1; }
  }

  // sub-band table in Λ order
  int ns = 0;
  auto add = [&](int level, int e, int e0, int e1) {
    SubBand& s = P.sb[ns++];
    s.level = level; s.e = e; s.e0 = e0; s.e1 = e1;
    s.nl = n >> level;
    s.count = P.d == 2 ? int64_t(s.nl) * s.nl : s.nl;
  };
  add(J, 0, 0, 0);
  for (int lev = J; lev >= 1; --lev) {
    if (P.d == 2) { add(lev, 1, 0, 1); add(lev, 2, 1, 0); add(lev, 3, 1, 1); }
    else add(lev, 1, 0, 1);
  }
  P.nsb = ns;
  int64_t off = 0;
  for (int s = 0; s < ns; ++s) { P.sb[s].offset = off; off += P.sb[s].count; }

  // template windows: φ chain from ũ (window [-zhi, -zlo]) by the à-trous recursion
  std::array<std::vector<Win1>, 2> phi;  // phi[a][ℓ] = window of ũ ⋆ φ_{ℓ,0} on axis a
  for (int a = 0; a < 2; ++a) {
    phi[a].resize(J + 1);
    if (a == 0 && P.d == 1) { for (auto& w : phi[a]) w = Win1{0, 1}; continue; }
    int W0 = P.zhi[a] - P.zlo[a] + 1;
    phi[a][0] = W0 >= n ? Win1{0, n} : Win1{((-P.zhi[a]) % n + n) % n, W0};
    for (int lev = 1; lev <= J; ++lev) phi[a][lev] = win_next(phi[a][lev - 1], n, 1 << (lev - 1), L2, 0);
  }
  for (int a = 0; a < 2; ++a)
    for (int lev = 0; lev <= J; ++lev) {
      hp->phiS[a][lev] = phi[a][lev].S;
      hp->phiW[a][lev] = phi[a][lev].W;
      hp->psiS[a][lev] = lev == 0 ? 0
          : (a == 0 && P.d == 1 ? 0 : win_next(phi[a][lev - 1], n, 1 << (lev - 1), L2, 1).S);
    }
  int64_t toff = 0;
  hp->phi_elems = 0;
  hp->y_elems = 0;
  hp->fma_templates = 0.0;
  for (int lev = 1; lev <= J; ++lev) {
    Win1 in0 = phi[0][lev - 1], in1 = phi[1][lev - 1];
    Win1 o1 = win_next(in1, n, 1 << (lev - 1), L2, 0);
    Win1 o0 = P.d == 2 ? win_next(in0, n, 1 << (lev - 1), L2, 0) : Win1{0, 1};
    hp->phi_elems = std::max<int64_t>(hp->phi_elems, int64_t(in0.W) * in1.W);
    hp->phi_elems = std::max<int64_t>(hp->phi_elems, int64_t(o0.W) * o1.W);
    hp->y_elems = std::max<int64_t>(hp->y_elems, 2 * int64_t(in0.W) * o1.W);
    const double tf = double(P.m) * L2 * (2.0 * in0.W * o1.W + (P.d == 2 ? 4.0 * o0.W * o1.W : 0.0));
    hp->fma_templates += tf;
    hp->tmpl_fma_level[lev] = tf;
  }
  for (int s = 0; s < ns; ++s) {
    SubBand& S = P.sb[s];
    int lev = S.level;
    for (int a = 0; a < 2; ++a) {
      if (a == 0 && P.d == 1) { S.tS[0] = 0; S.tW[0] = 1; continue; }
      int e_a = a == 0 ? S.e0 : S.e1;
      Win1 w = win_next(phi[a][lev - 1], n, 1 << (lev - 1), L2, e_a);
      S.tS[a] = w.S;
      S.tW[a] = w.W;
      S.tSu[a] = -P.zhi[a] + (e_a ? (1 << (lev - 1)) * (2 - L2) : 0);
    }
    S.tRS = S.tW[1] >= n ? S.tW[1] : (S.tW[1] + 3) / 4 * 4;
    S.tstride = int64_t(S.tW[0]) * S.tRS;
    S.toff = toff;
    toff += S.tstride * P.m;
    toff = (toff + 3) & ~int64_t(3);
  }
  hp->tmpl_elems = toff;

  // band stencils (per unit sub-band), then the steps each sub-band needs
  hp->stencil.clear();
  for (int s = 0; s < ns; ++s) {
    P.sb[s].stencil_off = int(hp->stencil.size());
    if (P.retain == PCWD_RETAIN_BAND) build_stencil(P, s, P.band_L, &hp->stencil);
    int steps = J;
    if (P.retain == PCWD_RETAIN_BAND) {
      steps = 1;
      for (int j = 0; j < P.band_L; ++j) {
        const Stencil& st = hp->stencil[P.sb[s].stencil_off + j];
        steps = std::max(steps, P.sb[st.sb].level);
      }
    }
    P.sb[s].steps = steps;
  }
  if (P.retain == PCWD_RETAIN_BAND) {
    hp->stencil_box.assign(size_t(ns) * ns * 4, 0);
    for (int s = 0; s < ns; ++s) {
      for (int t = 0; t < ns; ++t) {
        int* b = &hp->stencil_box[(size_t(s) * ns + t) * 4];
        b[0] = b[2] = 1 << 30;
        b[1] = b[3] = -(1 << 30);
      }
      for (int j = 0; j < P.band_L; ++j) {
        const Stencil& st = hp->stencil[P.sb[s].stencil_off + j];
        int* b = &hp->stencil_box[(size_t(s) * ns + st.sb) * 4];
        b[0] = std::min(b[0], st.o0); b[1] = std::max(b[1], st.o0);
        b[2] = std::min(b[2], st.o1); b[3] = std::max(b[3], st.o1);
      }
    }
  }

  // per-unit scratch layout and algorithmic FMA (max windows over the unit's parity)
  const int rb = hp->real_bytes;
  for (int s = 0; s < ns; ++s) {
    SubBand& S = P.sb[s];
    int64_t w0 = P.d == 2 ? std::min(S.tW[0], n) : 1;
    int64_t w1 = std::min(S.tW[1], n);
    int64_t nl0 = P.d == 2 ? n : 1, nl1 = n;
    auto rs4 = [](int64_t x) { return (x + 3) & ~int64_t(3); };   // batched path: 16-byte row strides
    int64_t X0 = w0 * rs4(w1);
    int64_t maxA = 0, maxY = 0, maxD = 0;
    int64_t hA1 = 0, hA2 = 0, hY = 0, hD = 0;   // hybrid layout: step-1 / step-2 approximations, steps ≥ 2
    double fma = double(P.m) * X0;
    S.any_full = (S.tW[1] >= n) || (P.d == 2 && S.tW[0] >= n);
    for (int st = 1; st <= S.steps; ++st) {
      int64_t o0 = P.d == 2 ? step_out_maxlen(int(w0), int(nl0), L2) : 1;
      int64_t o1 = step_out_maxlen(int(w1), int(nl1), L2);
      if (P.d == 2) {
        maxY = std::max(maxY, w0 * 2 * o1);
        maxA = std::max(maxA, o0 * rs4(o1));
        maxD = std::max(maxD, 3 * o0 * o1);
        if (st % 2) hA1 = std::max(hA1, o0 * o1); else hA2 = std::max(hA2, o0 * o1);
        if (st >= 2) { hY = std::max(hY, w0 * 2 * o1); hD = std::max(hD, 3 * o0 * o1); }
        fma += double(L2) * (w0 * 2.0 * o1 + 4.0 * o0 * o1);
      } else {
        maxA = std::max(maxA, o1);
        maxD = std::max(maxD, o1);
        if (st % 2) hA1 = std::max(hA1, o1); else hA2 = std::max(hA2, o1);
        if (st >= 2) { hY = std::max(hY, 2 * o1); hD = std::max(hD, o1); }
        fma += double(L2) * 2.0 * o1;
      }
      w0 = o0; w1 = o1;
      nl0 = P.d == 2 ? nl0 / 2 : 1;
      nl1 /= 2;
    }
    auto al = [](int64_t x) { return (x + 3) & ~int64_t(3); };
    S.offX0 = 0;
    S.offX1 = al(std::max(X0, maxA));
    S.offY = S.offX1 + al(maxA);
    S.offD = S.offY + al(maxY);
    S.offStage = S.offD + al(maxD);
    int64_t stage = 0;
    if (P.retain == PCWD_RETAIN_BAND) stage = P.band_Lpad + (int64_t(P.band_Lpad) * 4 + rb - 1) / rb;
    S.scratch = S.offStage + al(stage);
    S.hs_X1 = 0;
    S.hs_X2 = al(hA1);
    S.hs_Y = S.hs_X2 + al(hA2);
    S.hs_D = S.hs_Y + al(hY);
    S.hs_size = S.hs_D + al(hD);
    S.fma = fma;

    // warp kernel: band rule, d = 2, windows never cover a whole line, per-warp scratch small
    S.wk_ok = 0;
    if (P.retain == PCWD_RETAIN_BAND && P.d == 2 && (L2 == 2 || L2 == 4 || L2 == 6 || L2 == 8 || L2 == 12)) {
      bool ok = S.tW[0] < n && S.tW[1] < n;
      int64_t a0 = S.tW[0], a1 = S.tW[1];
      int64_t nl = n;
      int64_t maxY2 = 0, maxX = a0 * a1, maxD2 = 0;
      for (int st = 1; st <= S.steps && ok; ++st) {
        int64_t o0 = (a0 >> 1) + (L2 >> 1), o1 = (a1 >> 1) + (L2 >> 1);   // unclipped max lengths
        nl >>= 1;
        if (o0 >= nl || o1 >= nl) ok = false;
        maxY2 = std::max(maxY2, a0 * 2 * o1);
        maxX = std::max(maxX, o0 * o1);
        maxD2 = std::max(maxD2, 3 * o0 * o1);
        a0 = o0; a1 = o1;
      }
      // detail boxes are bounded by the stencil boxes
      int64_t boxmax = 0;
      for (int t = 0; t < ns; ++t) {
        const int* b = &hp->stencil_box[(size_t(s) * ns + t) * 4];
        if (b[0] <= b[1]) boxmax += int64_t(b[1] - b[0] + 1) * (b[3] - b[2] + 1);
      }
      int64_t dmax = std::min(maxD2, boxmax);
      S.wk_offY = al(maxX);
      S.wk_offD = S.wk_offY + al(maxY2);
      S.wk_offStage = S.wk_offD + al(dmax);
      S.wk_scratch = S.wk_offStage + al(P.band_Lpad + (int64_t(P.band_Lpad) * 4 + rb - 1) / rb);
      if (ok && S.wk_scratch * rb <= 200 * 1024) S.wk_ok = 1;
    }
  }

  // fine-path geometry: one record per sub-band and class q = p mod 2^{steps-ℓ} (geom.h)
  hp->fgeom.clear();
  for (int s = 0; s < ns; ++s) {
    SubBand& S = P.sb[s];
    S.fg_off = 0;
    S.fg_m = 0;
    if (!(P.retain == PCWD_RETAIN_BAND && P.d == 2 && S.e != 0 && S.level <= 3 && S.steps <= kFMS && S.wk_ok)) continue;
    const int M = 1 << std::max(0, S.steps - S.level);
    S.fg_off = int(hp->fgeom.size());
    S.fg_m = M;
    auto boxfn = [&](int t, int* b) {
      const int* q = &hp->stencil_box[(size_t(s) * ns + t) * 4];
      b[0] = q[0]; b[1] = q[1]; b[2] = q[2]; b[3] = q[3];
    };
    for (int q0 = 0; q0 < M; ++q0)
      for (int q1 = 0; q1 < M; ++q1) {
        FGeom g;
        std::memset(&g, 0, sizeof(g));
        compute_fgeom(P, S, q0, q1, boxfn, g);
        hp->fgeom.push_back(g);
      }
  }
  build_sep(hp);

  // shard: contiguous unit ranges (Λ order) with equal estimated time.  A unit's time is its algorithmic
  // FMA count times a per-path weight: time per algorithmic FMA of each level's kernel path relative to
  // the fine level-1 kernel, measured on B200 at c5 (profiles/r01: fine ℓ = 1, 2, 3 at 1.0, 0.9, 1.5;
  // batched ℓ = 4..7 at 1.36, 1.06, 0.95, 1.13, whole-torus windows 2.4 — ℓ ≥ 5 at the r1d figures × 0.9, the coarse
  // levels of a shard running on concurrent streams since r1f).  The template chain up
  // to level ℓ is charged to the first unit of level ℓ (its owner builds it).  Boundaries are rounded to
  // 16 units so every shard keeps whole rounds of the fine and tiled kernels.
  std::vector<double> ucost(ns, 0.0), lump(ns, 0.0);
  for (int s = 0; s < ns; ++s) {
    const SubBand& S = P.sb[s];
    double w = 1.0;
    if (P.retain == PCWD_RETAIN_BAND) {
      static const double wl[8] = {1.0, 1.0, 0.9, 1.5, 1.36, 1.06, 0.95, 1.13};
      w = S.any_full ? 2.4 : wl[std::min(S.level, 7)];
    }
    ucost[s] = S.fma * w;
  }
  for (int lev = 1; lev <= J; ++lev) {
    const int s = sb_index(P.d, J, lev, 1);   // first detail sub-band of the level in Λ order
    lump[lev == J ? 0 : s] += hp->tmpl_fma_level[lev] * 4.0;   // fp64 template passes (DFMA half rate, L2-bound): ≈4× per FMA
  }
  double total = 0.0;
  for (int s = 0; s < ns; ++s) total += ucost[s] * double(P.sb[s].count) + lump[s];
  auto unit_at_cost = [&](double c) -> int64_t {   // first unit whose prefix cost ≥ c
    double acc = 0.0;
    for (int s = 0; s < ns; ++s) {
      double sc = ucost[s] * double(P.sb[s].count) + lump[s];
      if (acc + sc >= c) {
        int64_t k = ucost[s] > 0 ? int64_t(std::ceil((c - acc - lump[s]) / ucost[s] - 1e-9)) : 0;
        k = std::max<int64_t>(0, std::min<int64_t>(k, P.sb[s].count));
        return P.sb[s].offset + k;
      }
      acc += sc;
    }
    return P.N;
  };
  auto align16 = [&](int64_t u) { return P.N >= 256 ? std::min<int64_t>(P.N, (u + 8) / 16 * 16) : u; };
  hp->row0 = d->rank == 0 ? 0 : align16(unit_at_cost(total * d->rank / d->world));
  hp->row1 = d->rank == d->world - 1 ? P.N : align16(unit_at_cost(total * (d->rank + 1) / d->world));
  if (hp->row1 < hp->row0) hp->row1 = hp->row0;
  // THRESHOLD store-then-filter: every structural partner value of a unit (the windows the cascade emits, in
  // emission order) gets a slot; per sub-band, the slot is the per-axis worst case over positions
  hp->cand_total = 0;
  if (d->retain == PCWD_RETAIN_THRESHOLD) {
    for (int s = 0; s < ns; ++s) {
      SubBand& S = P.sb[s];
      int mA[2][kMaxJ + 1] = {}, mD[2][kMaxJ + 1] = {};
      for (int a = (P.d == 2 ? 0 : 1); a < 2; ++a)
        for (int p = 0; p < S.nl; ++p) {
          Range in = unit_window(P, S, a, p);
          for (int st = 1; st <= S.steps; ++st) {
            const Range ra = step_out(in, L2, 0), rd = step_out(in, L2, 1);
            mA[a][st] = std::max(mA[a][st], ra.len);
            mD[a][st] = std::max(mD[a][st], rd.len);
            in = ra;
          }
        }
      int64_t slot = 0;
      for (int st = 1; st <= S.steps; ++st) {
        if (P.d == 2) {
          slot += int64_t(mA[0][st]) * mD[1][st] + int64_t(mD[0][st]) * mA[1][st] + int64_t(mD[0][st]) * mD[1][st];
          if (st == J) slot += int64_t(mA[0][st]) * mA[1][st];
        } else {
          slot += mD[1][st] + (st == J ? mA[1][st] : 0);
        }
      }
      const int64_t a0 = std::max(hp->row0, S.offset), a1 = std::min(hp->row1, S.offset + S.count);
      S.cand_slot = slot;
      S.cand_off = hp->cand_total;
      if (a1 > a0) hp->cand_total += (a1 - a0) * slot;
    }
  }
  double f = 0.0;
  for (int s = 0; s < ns; ++s) {
    int64_t a = std::max(hp->row0, P.sb[s].offset);
    int64_t b = std::min(hp->row1, P.sb[s].offset + P.sb[s].count);
    if (b > a) f += P.sb[s].fma * double(b - a);
  }
  hp->fma_shard = f + hp->fma_templates;
  return PCWD_OK;
}

}  // namespace pcwd
