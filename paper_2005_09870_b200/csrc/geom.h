// geom.h — per-unit cascade geometry of the band rule, restricted to what the unit's stencil needs.
//
// For a unit μ at level ℓ, position p, the a3 cascade only has to produce the detail
// coefficients inside the stencil's boxes (reading R16) and the approximation coefficients that later
// steps read.  Working backwards from the coarsest needed step, each step s needs
//   * pass B (axis 0) outputs: the detail boxes of level s and the approximation box the next step reads;
//   * pass A (axis 1) outputs: the columns those boxes read (h- and g-filtered separately);
//   * input rows / columns: the taps those outputs touch (Lemma 6, made exact),
// all clipped to the unit's actual support windows (step_out of common.h).
// Coordinates are UNWRAPPED (no reduction mod n) so that a unit's geometry is a translate of its
// class representative: every start on the level-s grid moves by (p - q)·2^{ℓ-s} (s ≤ ℓ) or by
// (p - q) >> (s - ℓ) (s > ℓ, exact since p ≡ q mod 2^{steps-ℓ}).  The host plan tabulates one record
// per sub-band and class q = p mod 2^{steps-ℓ}; kernels translate it.
#pragma once
#include "common.h"

namespace pcwd {

constexpr int kFMS = 6;   // max cascade steps on the fine path

struct FStep {
  int xr, xrl, xc, xcl;   // input region of the step (level s-1): rows, columns
  int ar, arl;            // rows of the input filtered by pass A (⊆ input rows)
  int hlo, hlen, glo, glen;   // pass-A output columns (level s): h-filtered (e1 = 0), g-filtered (e1 = 1)
  int blo0[4], blen0[4], blo1[4], blen1[4];   // pass-B output boxes per orientation code ec = 2 e0 + e1
  int doff[4];            // offset of each detail box (and the coarse block at s = J) in the D buffer
};

struct FGeom {
  int c0, c1;             // R window start (level 0), unwrapped
  int R0, R1;             // R window size
  int steps;
  int dsize;              // D buffer elements used
  FStep st[kFMS];
};

PCWD_HD int g_imin(int a, int b) { return a < b ? a : b; }
PCWD_HD int g_imax(int a, int b) { return a > b ? a : b; }
PCWD_HD void g_clip(int& lo, int& len, int alo, int alen) {
  int a = g_imax(lo, alo), b = g_imin(lo + len, alo + alen);
  lo = a;
  len = g_imax(0, b - a);
}
PCWD_HD void g_hull(int& lo, int& len, int lo2, int len2) {
  if (len2 <= 0) return;
  if (len <= 0) { lo = lo2; len = len2; return; }
  int a = g_imin(lo, lo2), b = g_imax(lo + len, lo2 + len2);
  lo = a;
  len = b - a;
}

// Geometry of unit (p0, p1) of sub-band S (index sbi).  box(t) returns the stencil offset box
// {omin0, omax0, omin1, omax1} of partner sub-band t for this unit sub-band (omin > omax: none).
template <typename BoxFn>
PCWD_HD void compute_fgeom(const Plan& P, const SubBand& S, int p0, int p1, BoxFn box, FGeom& g) {
  const int lev = S.level, steps = S.steps, L2 = P.L2;
  g.c0 = (p0 << lev) + S.tSu[0];
  g.c1 = (p1 << lev) + S.tSu[1];
  g.R0 = S.tW[0];
  g.R1 = S.tW[1];
  g.steps = steps;
  // forward: actual windows per step (approximation aw, detail dw) per axis
  int aw0[kFMS + 1], awl0[kFMS + 1], aw1[kFMS + 1], awl1[kFMS + 1];
  int dw0[kFMS + 1], dwl0[kFMS + 1], dw1[kFMS + 1], dwl1[kFMS + 1];
  aw0[0] = g.c0; awl0[0] = g.R0; aw1[0] = g.c1; awl1[0] = g.R1;
  dw0[0] = dwl0[0] = dw1[0] = dwl1[0] = 0;
  for (int s = 1; s <= steps; ++s) {
    int a = aw0[s - 1], b = aw0[s - 1] + awl0[s - 1] - 1;
    aw0[s] = -((-(a - L2 + 1)) >> 1); awl0[s] = (b >> 1) - aw0[s] + 1;
    dw0[s] = -((-(a - 1)) >> 1); dwl0[s] = ((b + L2 - 2) >> 1) - dw0[s] + 1;
    a = aw1[s - 1]; b = aw1[s - 1] + awl1[s - 1] - 1;
    aw1[s] = -((-(a - L2 + 1)) >> 1); awl1[s] = (b >> 1) - aw1[s] + 1;
    dw1[s] = -((-(a - 1)) >> 1); dwl1[s] = ((b + L2 - 2) >> 1) - dw1[s] + 1;
  }
  // backward: needed boxes, clipped to the actual windows
  int nA0 = 0, nAl0 = 0, nA1 = 0, nAl1 = 0;
  for (int s = steps; s >= 1; --s) {
    const int D = s - lev;
    const int b0 = D == 0 ? p0 : (D < 0 ? (p0 << -D) : (p0 >> D));
    const int b1 = D == 0 ? p1 : (D < 0 ? (p1 << -D) : (p1 >> D));
    FStep& f = g.st[s - 1];
    int lo0[4], len0[4], lo1[4], len1[4];
    if (s == steps) {
      nAl0 = nAl1 = 0;
      if (s == P.J) {   // coarse block partners come from the last approximation
        int cb[4];
        box(0, cb);
        if (cb[0] <= cb[1]) { nA0 = b0 + cb[0]; nAl0 = cb[1] - cb[0] + 1; nA1 = b1 + cb[2]; nAl1 = cb[3] - cb[2] + 1; }
      }
    }
    lo0[0] = nA0; len0[0] = nAl0; lo1[0] = nA1; len1[0] = nAl1;
    g_clip(lo0[0], len0[0], aw0[s], awl0[s]);
    g_clip(lo1[0], len1[0], aw1[s], awl1[s]);
    if (len0[0] == 0 || len1[0] == 0) len0[0] = len1[0] = 0;
    for (int ec = 1; ec < 4; ++ec) {
      const int sl = 1 + (P.J - s) * 3 + (ec - 1);
      int b[4];
      box(sl, b);
      lo0[ec] = lo1[ec] = len0[ec] = len1[ec] = 0;
      if (b[0] <= b[1]) {
        lo0[ec] = b0 + b[0]; len0[ec] = b[1] - b[0] + 1; lo1[ec] = b1 + b[2]; len1[ec] = b[3] - b[2] + 1;
        const int e0 = ec >> 1, e1 = ec & 1;
        g_clip(lo0[ec], len0[ec], e0 ? dw0[s] : aw0[s], e0 ? dwl0[s] : awl0[s]);
        g_clip(lo1[ec], len1[ec], e1 ? dw1[s] : aw1[s], e1 ? dwl1[s] : awl1[s]);
        if (len0[ec] == 0 || len1[ec] == 0) len0[ec] = len1[ec] = 0;
      }
    }
    for (int ec = 0; ec < 4; ++ec) { f.blo0[ec] = lo0[ec]; f.blen0[ec] = len0[ec]; f.blo1[ec] = lo1[ec]; f.blen1[ec] = len1[ec]; }
    int hlo = 0, hlen = 0, glo = 0, glen = 0;
    g_hull(hlo, hlen, lo1[0], len0[0] ? len1[0] : 0);
    g_hull(hlo, hlen, lo1[2], len0[2] ? len1[2] : 0);
    g_hull(glo, glen, lo1[1], len0[1] ? len1[1] : 0);
    g_hull(glo, glen, lo1[3], len0[3] ? len1[3] : 0);
    f.hlo = hlo; f.hlen = hlen; f.glo = glo; f.glen = glen;
    int rlo = 0, rlen = 0;
    for (int ec = 0; ec < 4; ++ec) {
      if (!len0[ec]) continue;
      const int e0 = ec >> 1;
      g_hull(rlo, rlen, 2 * lo0[ec] + (e0 ? 2 - L2 : 0), 2 * (len0[ec] - 1) + L2);
    }
    int clo = 0, clen = 0;
    if (hlen) g_hull(clo, clen, 2 * hlo, 2 * (hlen - 1) + L2);
    if (glen) g_hull(clo, clen, 2 * glo + 2 - L2, 2 * (glen - 1) + L2);
    g_clip(rlo, rlen, aw0[s - 1], awl0[s - 1]);
    g_clip(clo, clen, aw1[s - 1], awl1[s - 1]);
    f.ar = rlo; f.arl = rlen;
    f.xr = rlo; f.xrl = rlen; f.xc = clo; f.xcl = clen;
    nA0 = rlo; nAl0 = rlen; nA1 = clo; nAl1 = clen;
  }
  // the R window is the step-1 input as computed by the k-sum (whole window)
  g.st[0].xr = g.c0; g.st[0].xrl = g.R0; g.st[0].xc = g.c1; g.st[0].xcl = g.R1;
  int doff = 0;
  for (int s = 1; s <= steps; ++s)
    for (int ec = 0; ec < 4; ++ec) {
      g.st[s - 1].doff[ec] = doff;
      if (ec || s == P.J) doff += g.st[s - 1].blen0[ec] * g.st[s - 1].blen1[ec];
    }
  g.dsize = doff;
}

// Translate a class record computed at position q to position p (p ≡ q mod 2^{steps-ℓ} per axis).
PCWD_HD int g_shift(int dp, int lev, int s) { return s <= lev ? dp * (1 << (lev - s)) : (dp >> (s - lev)); }

// ---------------------------------------------------------------------------------------------------
// Separable direct path of the fine kernel ("sep").  The 2-D basis is a tensor product
// (P:93-127): the analysis atom of coefficient λ = (s, e0, e1, l0, l1) is
//     ψ_λ(y0, y1) = w_{s,e0,l0}(y0) · w_{s,e1,l1}(y1),   w_{s,e,l}(y) = W_{s,e}(y − 2^s l),
// with the 1-D base atoms of the analysis step of common.h:
//     W_{1,e}(y) = f_e[y − o_e],   W_{s,e}(y) = Σ_j f_e[j] · W_{s−1,0}(y − 2^{s−1}(o_e + j)),
// supported on [2^{s−1} o_e, 2^{s−1} o_e + (2^s − 1)(2δ − 1) + 1).  Entry Θ[μ][λ] = ⟨R_μ, ψ_λ⟩ over μ's
// window therefore factorises:  Q[y0][g] = Σ_{y1} R_μ(y0, y1) w_g(y1)  (stage 1, one column per distinct
// column atom g of the stencil), then  Θ[μ][λ] = Σ_{y0} w_{s,e0,l0}(y0) Q[y0][g(λ)]  (stage 2).
// Every position is relative to the unit's window; for a unit of class q = p mod 2^{steps−ℓ} the whole
// record is a translate of its class representative's (see g_shift), so one record per class suffices.
struct SepRun {            // stage 1: B column atoms of one (s, e1) at consecutive positions, one row per task
  int s, e;                // atom level and orientation bit
  int c;                   // window column of the first atom's tap 0 (unclipped; columns outside [0, R1) read 0)
  int B;                   // atoms in the run (≤ sep_bmax(s))
  int q;                   // Q column of the first atom
  int r0, r1;              // Q rows the stage-2 partners read: [r0, r1)
  int mask;                // 1: some tap read lies beyond the kSepPad zero columns around the row (masked loads)
  int toff;                // sep_toff(s, e): the atom's taps in the shared-memory table
  int tbeg;                // first stage-1 task of the run (tasks of a class are its runs' rows, in run order)
};
struct SepPart {           // stage 2: B partners of one Q column g, row atoms W_{s,e} at consecutive positions
  int g;                   // Q column
  int s, e;
  int fs;                  // window row of the first atom's tap 0 (unclipped)
  int B;
  int jj, jstr;            // stencil slots jj + b·jstr
  int r0, r1;              // rows of column g computed by stage 1 (everything else reads 0)
  int toff;                // sep_toff(s, e)
  int pad[2];
};
constexpr int kSepSmax = 5;
constexpr int kSepMaxRuns = 64;
constexpr int kSepPartB = 1;      // partners per stage-2 task (1: balanced over the unit's threads)   // stage-1 runs per class (staged in shared memory per unit)
constexpr int kSepPad = 12;   // zero columns the fine kernel keeps on both sides of every R row in sep mode
// register-window widths instantiated per atom level (the run's B is rounded up to the next one)
PCWD_HD constexpr int sep_bsel(int s, int B) {
  return B <= 1 ? 1 : B <= 2 ? 2 : (s >= 4 ? 2 : B <= 3 ? 3 : B <= 4 ? 4 : B <= 6 ? 6 : 8);
}   // atom levels of the separable path (plan.cpp keeps the cascade beyond)
PCWD_HD constexpr int sep_atom_len(int s, int L2) { return ((1 << s) - 1) * (L2 - 1) + 1; }
PCWD_HD constexpr int sep_atom_start(int s, int e, int L2) { return e ? (1 << (s - 1)) * (2 - L2) : 0; }
PCWD_HD constexpr int sep_bmax(int s) { return s <= 2 ? 8 : (s == 3 ? 6 : (s == 4 ? 2 : 1)); }   // atoms per run (max)
// shared-memory tap table: W_{s,e} (s ≤ kSepSmax) at 16-byte aligned offsets, each followed by zeros up to a
// whole number of 2^s-tap blocks
PCWD_HD constexpr int sep_atom_blk(int s, int L2) { return (sep_atom_len(s, L2) + (1 << s) - 1) >> s; }
PCWD_HD constexpr int sep_atom_slot(int s, int L2) { return ((sep_atom_blk(s, L2) << s) + 3) & ~3; }
PCWD_HD constexpr int sep_toff(int s, int e, int L2) {
  return s <= 1 ? e * sep_atom_slot(1, L2) : sep_toff(s - 1, 1, L2) + sep_atom_slot(s - 1, L2) + e * sep_atom_slot(s, L2);
}
PCWD_HD constexpr int sep_ttot(int L2) { return sep_toff(kSepSmax, 1, L2) + sep_atom_slot(kSepSmax, L2); }
struct SepClass {
  int run_off, nrun;       // stage-1 runs of this class
  int task_off, ntask;     // stage-1 tasks (run << 16 | row), grouped by run
  int part_off, npart;     // stage-2 runs
  int nq;                  // Q columns
  int pad;
};

}  // namespace pcwd
