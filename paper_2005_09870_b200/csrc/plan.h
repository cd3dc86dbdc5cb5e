// plan.h — host-side planning for one handle (no CUDA calls).
#pragma once
#include <string>
#include <vector>

#include "../../include/pcwd.h"
#include "common.h"
#include "geom.h"

namespace pcwd {

struct Stencil {
  int sb, o0, o1, pad;
};

struct HostPlan {
  Plan P;
  std::vector<Stencil> stencil;   // nsb × band_L (BAND only), each sub-band's entries sorted by (sb, o0, o1)
  std::vector<int> stencil_box;   // BAND: nsb × nsb × 4 (omin0, omax0, omin1, omax1) of μ-sub-band × λ-sub-band
                                  //       (omin > omax: no entry)
  int real_bytes = 4;             // compute precision
  int out_bytes = 4;              // stored value precision
  int64_t row0 = 0, row1 = 0;     // shard
  int64_t tmpl_elems = 0;         // template buffer size (elements of the compute type)
  int64_t phi_elems = 0;          // per-k φ-chain window max (fp64 elements)
  int64_t y_elems = 0;            // per-k template pass-A buffer max (fp64 elements)
  double fma_shard = 0.0;         // algorithmic FMA of the shard (k-sum + cascade + templates)
  // template φ-chain windows per axis and level (ℓ = 0..J), and the ψ-window start per level
  int phiS[2][kMaxJ + 1] = {}, phiW[2][kMaxJ + 1] = {}, psiS[2][kMaxJ + 1] = {};
  double fma_templates = 0.0;
  double tmpl_fma_level[kMaxJ + 1] = {};   // template FMAs of each level's à-trous step
  std::vector<FGeom> fgeom;       // BAND, fine levels: class geometry records (SubBand::fg_off / fg_m)
  int64_t cand_total = 0;         // THRESHOLD: candidate slots of the shard (store-then-filter), fp64 values
  // separable direct path of the fine kernel (geom.h SepRun / SepPart / SepClass), records indexed like fgeom
  std::vector<double> atoms;      // base atoms W_{s,e}, s = 1..sep_smax, e = 0, 1 (fp64; cast on upload)
  int atom_off[kMaxJ + 1][2] = {};
  int atom_len[kMaxJ + 1] = {};
  int sep_smax = 0;
  std::vector<SepClass> sepcls;   // one per fgeom record (valid where SubBand::fg_m > 0 and sep_ok[level])
  std::vector<SepRun> seprun;
  std::vector<SepPart> seppart;
  std::vector<int> septask;
  int sep_ok[kMaxJ + 1] = {};     // level ℓ: every class record of every sub-band built
  int sep_nq[kMaxJ + 1] = {};     // max Q columns over the level's classes
  int sep_nrun[kMaxJ + 1] = {};   // max stage-1 runs over the level's classes
};

// Returns a pcwd_status; msg receives the reason on error.
int validate_desc(const pcwd_desc* d, std::string* msg);

// u_host: m × N fp64 on the host (may be NULL: then the bounding box is the whole torus).
int build_plan(const pcwd_desc* d, const double* u_host, HostPlan* hp, std::string* msg);

// Base atom W_{s,e} of the separable fine path (fp64, sep_atom_len(s) taps from sep_atom_start(s, e)).
void sep_base_atom(const Plan& P, int s, int e, std::vector<double>* out);

// Λ order index of sub-band (level, e).
int sb_index(int d, int J, int level, int e);

}  // namespace pcwd
