// api.cu — the C ABI of include/pcwd.h: handle lifetime, device buffers, launch sequencing.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pcwd.h"
#include "kernels.cuh"
#include "plan.h"

using namespace pcwd;

static thread_local std::string g_err;

namespace {

constexpr size_t kSmemBudget = 200 * 1024;  // dynamic smem per CTA for in-smem units

struct Launch {
  int64_t u0, u1;
  int grid;
  size_t smem;      // 0 ⇒ global scratch (generic kernel)
  int tile = 0;     // 1 ⇒ band_tile_kernel with the parameters below
  TileArgs ta{};
  int fine = 0;     // 1 ⇒ fine_kernel (fine.cu) for level `level`
  int level = 0;
  int box[3] = {0, 0, 0};   // fine: TMA box rows R0, T box width TS, v box width VS
  FineArgs fa{};
  int batched = 0;  // 1 ⇒ batched grid kernels (batched.cu)
  BatchArgs ba{};
  int64_t maxX0 = 0, maxY = 0, maxB = 0;
  int64_t workA[kMaxJ + 1] = {}, workB[kMaxJ + 1] = {};   // batched: per-step work items of pass A / B
  int64_t appr0[kMaxJ + 1] = {}, appr1[kMaxJ + 1] = {};   // batched: per-step max approximation window
  int steps = 0;
  int gu = 1;       // fine: units per round (chunks of a launch are multiples of it)
  int hybrid = 0;   // generic kernel, global scratch: smem (bytes) holds the buffers of steps ≥ 2
  size_t bs_off = 0;  // batched: byte offset of this launch's slice of the batched scratch
  int64_t gs_off = -1, gs_stride = 0;   // generic, global scratch: element offset of this launch's slice, per-CTA stride
};

struct Handle {
  pcwd_desc desc{};
  HostPlan hp;
  double* u_d = nullptr;
  void* v_d = nullptr;
  void* T_d = nullptr;
  double* phi[2] = {nullptr, nullptr};
  double* Ytmp = nullptr;
  int4* stencil_d = nullptr;
  int4* box_d = nullptr;
  FGeom* fgeom_d = nullptr;
  SepClass* sepc_d = nullptr;   // separable direct path tables (plan.cpp build_sep)
  SepRun* seprun_d = nullptr;
  SepPart* seppart_d = nullptr;
  int* septask_d = nullptr;
  void* atoms_d = nullptr;
  void* vpad_d = nullptr;   // periodically padded v (fine path TMA source)
  void* vwrap_d = nullptr;  // v extended periodically by kt_pr rows / kt_pc columns (tiled k-sum TMA source)
  CUtensorMap* amaps_d = nullptr;   // TMA maps of the batched approximation steps
  int kt_pr = 0, kt_pc = 0, kt_offx = 0;
  int vpad = 0;
  void* gscratch = nullptr;
  void* bscratch = nullptr;
  size_t bscratch_bytes = 0;
  bool conc = false;                // coarse levels on concurrent streams (each with its own scratch slice)
  bool conc_t = false;              // threshold rule: the generic launches of the one cascade pass on concurrent streams
  static constexpr int kNCS = 5;
  cudaStream_t cstream[kNCS] = {};
  cudaEvent_t efork = nullptr, ejoin[kNCS] = {};
  std::vector<Launch> launches;
  int64_t* row_ptr = nullptr;
  int32_t* col = nullptr;
  void* val = nullptr;
  int64_t nnz = 0, cap = 0;
  double* unitmax = nullptr;
  int32_t* cnt = nullptr;
  int64_t* rowcnt = nullptr;
  void* cubtmp = nullptr;
  size_t cubbytes = 0;
  double* dmax = nullptr;
  double* cand = nullptr;           // THRESHOLD store-then-filter: candidate values (hp.cand_total fp64)
  bool cand_valid = false;
  double M = 0.0;
  bool M_set = false, tmpl_fresh = false, decomposed = false;
  bool tmpl_ready = false;   // BAND: templates of the current u built by pcwd_set_kernels, consumed by the next decompose
  cudaStream_t cv = nullptr; // pcwd_set_kernels: v's host-to-device copy beside the template build
  int nlaunch = 0;
  bool profile = false;
  bool profile_serial = false;      // pcwd_profile(h, 2): launches serialised (per-kernel times, no overlap)
  cudaEvent_t ev[8] = {};
  std::vector<cudaEvent_t> lev;     // profile: one event pair per unit launch (run_units)
  cudaStream_t cs = nullptr;        // decompose_to_host: copy stream
  std::vector<cudaEvent_t> cev;     // decompose_to_host: chunk-done events
  cudaEvent_t cjoin = nullptr;      // decompose_to_host: copies done
  double* ustage = nullptr;         // set_kernels: staging of u (swapped with u_d once checked)
  void* vstage = nullptr;           // set_kernels: staging of v (fp64; swapped with v_d in fp64 compute)
  double* ubox = nullptr;           // set_kernels_box: u_k on the plan's bounding box (m × w0 × w1)
  int64_t ubox_cap = 0;
  struct Sink { int64_t width; int32_t* col; char* val; int ob; };
  const Sink* sink = nullptr;       // decompose_to_host: caller buffers the finished rows go to
  int* flag_d = nullptr;            // set_kernels: support check flag
  void* fbuf = nullptr;             // FISTA / wavelet transform scratch (allocated on first use)
  size_t fbuf_bytes = 0;
  int64_t* rpT = nullptr;           // Θᵀ as CSR over the columns (apply ᵀ, FISTA), built on first use per decompose
  int32_t* rowT = nullptr;
  void* valT = nullptr;
  void* twork = nullptr;
  size_t twork_bytes = 0;
  int64_t tcap = -1;
  bool tvalid = false;
  int64_t rows() const { return hp.row1 - hp.row0; }
};

inline bool L2OK(int L2) { return L2 >= 2 && L2 <= 12 && L2 % 2 == 0; }

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess) {                                                                      \
      return fail(e_ == cudaErrorMemoryAllocation ? PCWD_E_OOM : PCWD_E_CUDA,                     \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                            \
    }                                                                                             \
  } while (0)

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

void free_all(Handle* h) {
  void* ptrs[] = {h->u_d, h->v_d, h->T_d, h->phi[0], h->phi[1], h->Ytmp, h->stencil_d, h->box_d, h->fgeom_d, h->sepc_d, h->seprun_d, h->seppart_d, h->septask_d, h->atoms_d, h->vpad_d, h->vwrap_d, h->amaps_d, h->gscratch, h->bscratch,
                  h->row_ptr, h->col, h->val, h->unitmax, h->cnt, h->rowcnt, h->cubtmp, h->dmax, h->cand, h->ustage, h->vstage, h->ubox, h->flag_d, h->fbuf, h->rpT, h->rowT, h->valT, h->twork};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto& e : h->cev) cudaEventDestroy(e);
  h->cev.clear();
  if (h->cjoin) cudaEventDestroy(h->cjoin);
  h->cjoin = nullptr;
  if (h->cs) cudaStreamDestroy(h->cs);
  if (h->cv) cudaStreamDestroy(h->cv);
  h->cs = nullptr;
  for (int i = 0; i < Handle::kNCS; ++i) {
    if (h->cstream[i]) cudaStreamDestroy(h->cstream[i]);
    if (h->ejoin[i]) cudaEventDestroy(h->ejoin[i]);
    h->cstream[i] = nullptr;
    h->ejoin[i] = nullptr;
  }
  if (h->efork) cudaEventDestroy(h->efork);
  h->efork = nullptr;
}

template <typename T>
cudaError_t dalloc(T** p, size_t bytes) {
  return cudaMalloc(reinterpret_cast<void**>(p), bytes < 16 ? 16 : bytes);
}

// 3-D tiled TMA descriptor over a row-major (z, y, x) array of rb-byte reals: extents (dx, dy, dz), strides in
// elements (sy, sz), box (bx, by, 1), out-of-range elements read as zero.  Returns 0 or the CUresult.
int encode_map3(CUtensorMap* map, void* base, int rb, int64_t dx, int64_t dy, int64_t dz, int64_t sy, int64_t sz, int bx,
                int by) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p) return -1;
    fn = reinterpret_cast<EncodeFn>(p);
  }
  const cuuint64_t dims[3] = {cuuint64_t(dx), cuuint64_t(dy), cuuint64_t(dz)};
  const cuuint64_t strides[2] = {cuuint64_t(sy * rb), cuuint64_t(sz * rb)};
  const cuuint32_t box[3] = {cuuint32_t(bx), cuuint32_t(by), 1u};
  const cuuint32_t es[3] = {1u, 1u, 1u};
  CUresult r = fn(map, rb == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return int(r);
}

// Templates T_{k,s} for every sub-band (a1).
int build_templates(Handle* h, cudaStream_t st) {
  const Plan& P = h->hp.P;
  const HostPlan& hp = h->hp;
  CK(launch_phi0(P, h->u_d, h->phi[0], hp.phiS[0][0], hp.phiW[0][0], hp.phiS[1][0], hp.phiW[1][0], st));
  h->nlaunch++;
  // only the levels of the sub-bands this shard owns (the à-trous chain runs up to the coarsest of them)
  int maxlev = 1;
  for (int s = 0; s < P.nsb; ++s)
    if (P.sb[s].offset < hp.row1 && P.sb[s].offset + P.sb[s].count > hp.row0) maxlev = std::max(maxlev, P.sb[s].level);
  int cur = 0;
  for (int lev = 1; lev <= maxlev; ++lev) {
    TmplArgs A{};
    A.phi_in = h->phi[cur];
    A.phi_out = h->phi[cur ^ 1];
    A.Y = h->Ytmp;
    A.T = h->T_d;
    A.dil = 1 << (lev - 1);
    for (int a = 0; a < 2; ++a) {
      A.Sin[a] = hp.phiS[a][lev - 1];
      A.Win[a] = hp.phiW[a][lev - 1];
      A.Wout[a] = hp.phiW[a][lev];
      A.Sout[a][0] = hp.phiS[a][lev];
      A.Sout[a][1] = hp.psiS[a][lev];
    }
    for (int ec = 0; ec < 4; ++ec) A.toff[ec] = -1;
    if (lev == P.J) A.toff[0] = P.sb[0].toff;
    if (P.d == 2) {
      for (int ec = 1; ec < 4; ++ec) A.toff[ec] = P.sb[sb_index(2, P.J, lev, ec)].toff;
    } else {
      A.toff[1] = P.sb[sb_index(1, P.J, lev, 1)].toff;
    }
    A.trs = A.Wout[1] >= P.n ? A.Wout[1] : (A.Wout[1] + 3) / 4 * 4;
    A.tstride = int64_t(A.Wout[0]) * A.trs;
    CK(launch_tmpl_level(P, A, hp.real_bytes, lev, st));
    h->nlaunch += P.d == 2 ? 2 : 1;
    cur ^= 1;
  }
  return PCWD_OK;
}

// Algorithmic FMA (SURVEY §8(d) per-unit figure, SubBand::fma) of the units [u0, u1).
double units_fma(const Plan& P, int64_t u0, int64_t u1) {
  double f = 0.0;
  for (int s = 0; s < P.nsb; ++s) {
    const int64_t a = std::max(u0, P.sb[s].offset), b = std::min(u1, P.sb[s].offset + P.sb[s].count);
    if (b > a) f += P.sb[s].fma * double(b - a);
  }
  return f;
}

int run_units(Handle* h, int mode, cudaStream_t st, double tau) {
  const Plan& P = h->hp.P;
  if (h->profile && h->lev.size() < 2 * h->launches.size()) {
    for (auto& e : h->lev) cudaEventDestroy(e);
    h->lev.assign(2 * h->launches.size(), nullptr);
    for (auto& e : h->lev) CK(cudaEventCreate(&e));
  }
  // decompose_to_host: after each launch, its rows (fixed width in BAND / FULL) are copied on the
  // copy stream, ordered by an event; the largest level runs first so that the copies start early
  const Handle::Sink* sk = h->sink;
  int ci = 0;
  cudaStream_t ls = st;   // stream of the current launch
  auto emit = [&](int64_t a, int64_t b) -> int {
    if (!sk || b <= a) return PCWD_OK;
    if (ci >= int(h->cev.size())) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      h->cev.push_back(e);
    }
    cudaEvent_t e = h->cev[ci++];
    CK(cudaEventRecord(e, ls));
    CK(cudaStreamWaitEvent(h->cs, e, 0));
    const int64_t off = (a - h->hp.row0) * sk->width, cnt = (b - a) * sk->width;
    if (sk->col) CK(cudaMemcpyAsync(sk->col + off, h->col + off, cnt * sizeof(int32_t), cudaMemcpyDefault, h->cs));
    if (sk->val)
      CK(cudaMemcpyAsync(sk->val + off * sk->ob, static_cast<char*>(h->val) + off * sk->ob, cnt * sk->ob,
                         cudaMemcpyDefault, h->cs));
    return PCWD_OK;
  };
  // coarse (batched) levels are independent: each runs on its own stream with its own scratch slice,
  // forked from `st` after the templates and joined back before the next non-batched launch
  const bool conc = h->conc && mode == MODE_BAND && !h->profile_serial;
  const bool conc_t = h->conc_t && (mode == MODE_TSTORE || mode == MODE_TMAX) && !h->profile_serial;
  // the fine kernels (on `st`) may also run beside the coarse streams: they share no data (all but the first,
  // largest one, which runs alone)
  static const bool overlap = getenv("PCWD_COARSE_OVERLAP") ? atoi(getenv("PCWD_COARSE_OVERLAP")) != 0 : true;
  bool forked = false;
  int bi = 0, used = 0;
  auto fork = [&]() -> int {
    if (forked) return PCWD_OK;
    CK(cudaEventRecord(h->efork, st));
    for (int i = 0; i < Handle::kNCS; ++i) CK(cudaStreamWaitEvent(h->cstream[i], h->efork, 0));
    forked = true;
    used = 0;
    return PCWD_OK;
  };
  auto join = [&]() -> int {
    if (!forked) return PCWD_OK;
    for (int i = 0; i < used; ++i) {
      CK(cudaEventRecord(h->ejoin[i], h->cstream[i]));
      CK(cudaStreamWaitEvent(st, h->ejoin[i], 0));
    }
    forked = false;
    return PCWD_OK;
  };
  struct JoinGuard {   // on an error return the coarse streams are still joined back into `st`
    Handle* h; cudaStream_t st; bool* forked; int* used;
    ~JoinGuard() {
      if (!*forked) return;
      for (int i = 0; i < *used; ++i) {
        cudaEventRecord(h->ejoin[i], h->cstream[i]);
        cudaStreamWaitEvent(st, h->ejoin[i], 0);
      }
    }
  } join_guard{h, st, &forked, &used};
  const int nL = int(h->launches.size());
  for (int it = 0; it < nL; ++it) {
    // order: the largest level (the finest) first when the output streams to the host or the coarse
    // levels overlap the other fine levels; it runs alone, then the coarse streams fork beside the rest
    const int li = (sk || (conc && overlap)) ? nL - 1 - it : it;
    const Launch& L = h->launches[li];
    {   // timing experiment only (results invalid): PCWD_SKIP_LEVELS = bit mask of levels whose launches are skipped
      static const int skip = getenv("PCWD_SKIP_LEVELS") ? atoi(getenv("PCWD_SKIP_LEVELS")) : 0;
      if (skip && ((skip >> P.sb[find_subband(P, L.u0)].level) & 1)) continue;
    }
    ls = st;
    // level 1 beside the coarse streams too (default: the shorter step, c5 r01 15.36 vs 15.74 ms); PCWD_OVERLAP_ALL=0
    // runs the first (largest) level alone
    static const bool overlap_all = !(getenv("PCWD_OVERLAP_ALL") && atoi(getenv("PCWD_OVERLAP_ALL")) == 0);
    if (conc && overlap && it == (overlap_all ? 0 : 1))
      if (int rc = fork()) return rc;   // after the first launch: coarse streams wait for it only
    if (conc_t) {   // threshold rule's cascade pass: every level on its own stream (own scratch slices)
      if (int rc = fork()) return rc;
      const int k = bi++ % Handle::kNCS;
      ls = h->cstream[k];
      used = std::max(used, k + 1);
    } else if (L.batched && conc) {
      if (int rc = fork()) return rc;
      const int k = bi++ % Handle::kNCS;
      ls = h->cstream[k];
      used = std::max(used, k + 1);
    } else if (forked && !overlap) {
      if (int rc = join()) return rc;
    }
    if (h->profile) cudaEventRecord(h->lev[2 * li], ls);
    struct Rec {   // record the launch's end event on every path out of this iteration
      Handle* h; int i; cudaStream_t st;
      ~Rec() { if (h->profile) cudaEventRecord(h->lev[2 * i + 1], st); }
    } rec_end{h, li, ls};
    if (L.batched) {
      if (mode != MODE_BAND) return fail(PCWD_E_STATE, "batched launch outside BAND mode");
      BatchArgs B = L.ba;
      B.v = h->v_d;
      B.T = h->T_d;
      B.stencil = h->stencil_d;
      B.scratch = static_cast<char*>(h->bscratch) + L.bs_off;
      B.row0 = h->hp.row0;
      B.col = h->col;
      B.val = h->val;
      int nl = 0;
      CK(launch_band_batched(P, B, h->hp.real_bytes, L.maxX0, L.workA, L.workB, L.appr0, L.appr1, L.steps, ls, &nl));
      h->nlaunch += nl;
      if (int rc = emit(L.u0, L.u1)) return rc;
      continue;
    }
    if (L.fine) {
      if (mode != MODE_BAND) return fail(PCWD_E_STATE, "fine launch outside BAND mode");
      FineArgs F = L.fa;
      F.v = h->v_d;
      F.T = h->T_d;
      F.stencil = h->stencil_d;
      F.geom = h->fgeom_d;
      F.sepc = h->sepc_d;
      F.seprun = h->seprun_d;
      F.seppart = h->seppart_d;
      F.septask = h->septask_d;
      F.atoms = h->atoms_d;
      F.row0 = h->hp.row0;
      F.col = h->col;
      F.val = h->val;
      static const bool dbg_on = getenv("PCWD_DEBUG_PHASES") != nullptr;
      unsigned long long* dbg = nullptr;
      if (dbg_on) {
        CK(cudaMalloc(&dbg, 8 * sizeof(unsigned long long)));
        CK(cudaMemset(dbg, 0, 8 * sizeof(unsigned long long)));
      }
      F.dbg = dbg;
      F.dbg_flags = getenv("PCWD_FINE_DBG") ? atoi(getenv("PCWD_FINE_DBG")) : 0;
      {
        // chunks of about 64K units when the rows stream to the host (each chunk's copy overlaps the next)
        const int64_t GU = L.gu, units = L.u1 - L.u0;
        int64_t chunk = units;
        if (sk) {
          const int64_t nch = std::max<int64_t>(1, (units + 65535) / 65536);
          chunk = ((units + nch - 1) / nch + GU - 1) / GU * GU;
        }
        for (int64_t a = L.u0; a < L.u1; a += chunk) {
          const int64_t b = std::min(L.u1, a + chunk);
          F.u0 = a;
          F.u1 = b;
          CK(launch_fine(P, F, h->hp.real_bytes, L.level, int(std::min<int64_t>(L.grid, (b - a) / GU)), L.smem, st));
          h->nlaunch++;
          if (int rc = emit(a, b)) return rc;
        }
      }
      if (dbg_on) {
        unsigned long long c[8];
        CK(cudaMemcpy(c, dbg, sizeof(c), cudaMemcpyDeviceToHost));
        const double tot = double(c[0] + c[1]);
        fprintf(stderr, "[pcwd fine] level %d grid %d: ksum %.1f%% cascade+gather %.1f%%\n", L.level, L.grid,
                100.0 * c[0] / tot, 100.0 * c[1] / tot);
        cudaFree(dbg);
      }
      continue;
    }
    if (L.tile) {
      if (mode != MODE_BAND) return fail(PCWD_E_STATE, "tile launch outside BAND mode");
      TileArgs T = L.ta;
      T.v = h->v_d;
      T.T = h->T_d;
      T.stencil = h->stencil_d;
      T.box = h->box_d;
      T.row0 = h->hp.row0;
      T.col = h->col;
      T.val = h->val;
      T.dbg = nullptr;
      static const bool dbg_on = getenv("PCWD_DEBUG_PHASES") != nullptr;
      unsigned long long* dbg = nullptr;
      if (dbg_on) {
        CK(cudaMalloc(&dbg, 8 * sizeof(unsigned long long)));
        CK(cudaMemset(dbg, 0, 8 * sizeof(unsigned long long)));
        T.dbg = dbg;
      }
      CK(launch_band_tile(P, T, h->hp.real_bytes, L.grid, L.smem, st));
      h->nlaunch++;
      if (int rc = emit(L.u0, L.u1)) return rc;
      if (dbg_on) {
        unsigned long long c[8];
        CK(cudaMemcpy(c, dbg, sizeof(c), cudaMemcpyDeviceToHost));
        double tot = 0;
        for (int i = 2; i < 8; ++i) tot += double(c[i]);
        fprintf(stderr, "[pcwd tile] level %d G %d grid %d smem %zu: geom %.1f%% ksum %.1f%% cascade %.1f%% gather+write %.1f%%\n",
                P.sb[find_subband(P, L.u0)].level, L.ta.G, L.grid, L.smem, 100 * c[2] / tot, 100 * c[3] / tot,
                100 * c[4] / tot, 100 * c[5] / tot);
        cudaFree(dbg);
      }
      continue;
    }
    UnitArgs A{};
    A.v = h->v_d;
    A.T = h->T_d;
    A.stencil = h->stencil_d;
    A.gscratch = L.gs_off >= 0 ? static_cast<char*>(h->gscratch) + size_t(L.gs_off) * h->hp.real_bytes : nullptr;
    A.gscratch_stride = L.gs_stride;
    A.u0 = L.u0;
    A.u1 = L.u1;
    A.row0 = h->hp.row0;
    A.row_ptr = h->row_ptr;
    A.col = h->col;
    A.val = h->val;
    A.unitmax = h->unitmax;
    A.cnt = h->cnt;
    A.tau = tau;
    A.use_smem = L.smem > 0 && !L.hybrid;
    A.hybrid = L.hybrid;
    A.cand = h->cand;
    static const int unit_dbg = getenv("PCWD_UNIT_DBG") ? atoi(getenv("PCWD_UNIT_DBG")) : 0;
    A.dbg = unit_dbg;
    CK(launch_units(P, A, mode, h->hp.real_bytes, h->hp.out_bytes, L.grid, L.smem, ls));
    h->nlaunch++;
    if (mode == MODE_BAND || mode == MODE_FULL)
      if (int rc = emit(L.u0, L.u1)) return rc;
  }
  return join();
}

int local_max_impl(Handle* h, cudaStream_t st, double* out) {
  int rc = build_templates(h, st);
  if (rc) return rc;
  // with a candidate buffer the one cascade pass also stores every structural partner (store-then-filter:
  // the count and write passes then only read it); without one, they recompute the cascade
  rc = run_units(h, h->cand ? MODE_TSTORE : MODE_TMAX, st, 0.0);
  if (rc) return rc;
  h->cand_valid = h->cand != nullptr;
  CK(launch_max_reduce(h->unitmax, h->rows(), h->dmax, st));
  h->nlaunch++;
  CK(cudaMemcpyAsync(out, h->dmax, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  h->tmpl_fresh = true;
  return PCWD_OK;
}

}  // namespace

extern "C" {

const char* pcwd_error_string(int code) {
  switch (code) {
    case PCWD_OK: return "ok";
    case PCWD_E_SHAPE: return "shape error (d, n)";
    case PCWD_E_CONFIG: return "configuration error (levels, filter length)";
    case PCWD_E_PARAM: return "parameter error";
    case PCWD_E_CUDA: return "CUDA error";
    case PCWD_E_OOM: return "out of device memory";
    case PCWD_E_STATE: return "invalid call order";
    case PCWD_E_UNSUPPORTED: return "unsupported configuration";
  }
  return "unknown status";
}

const char* pcwd_last_error(void) { return g_err.c_str(); }

int pcwd_validate(const pcwd_desc* desc) {
  std::string msg;
  int rc = validate_desc(desc, &msg);
  if (rc) g_err = msg;
  return rc;
}

int pcwd_plan_shard(const pcwd_desc* desc, int64_t* row0, int64_t* row1) {
  HostPlan hp;
  std::string msg;
  int rc = build_plan(desc, desc ? desc->u : nullptr, &hp, &msg);
  if (rc) return fail(rc, msg);
  *row0 = hp.row0;
  *row1 = hp.row1;
  return PCWD_OK;
}

int pcwd_plan_num_subbands(const pcwd_desc* desc, int32_t* out) {
  std::string msg;
  int rc = validate_desc(desc, &msg);
  if (rc) return fail(rc, msg);
  *out = 1 + desc->levels * (desc->d == 2 ? 3 : 1);
  return PCWD_OK;
}

int pcwd_plan_stencil(const pcwd_desc* desc, int32_t sb, int32_t* out_sb, int32_t* out_o0, int32_t* out_o1) {
  if (!desc || desc->retain != PCWD_RETAIN_BAND) return fail(PCWD_E_PARAM, "stencil needs BAND retention");
  HostPlan hp;
  std::string msg;
  int rc = build_plan(desc, nullptr, &hp, &msg);
  if (rc) return fail(rc, msg);
  if (sb < 0 || sb >= hp.P.nsb) return fail(PCWD_E_PARAM, "sub-band index out of range");
  const int L = hp.P.band_L;
  for (int j = 0; j < L; ++j) {
    const Stencil& s = hp.stencil[hp.P.sb[sb].stencil_off + j];
    out_sb[j] = s.sb;
    out_o0[j] = s.o0;
    out_o1[j] = s.o1;
  }
  return PCWD_OK;
}

int pcwd_plan_atom(const pcwd_desc* desc, int32_t s, int32_t e, double* out, int32_t cap, int32_t* out_len,
                   int32_t* out_start) {
  std::string msg;
  int rc = validate_desc(desc, &msg);
  if (rc) return fail(rc, msg);
  if (s < 1 || s > kMaxJ || (e != 0 && e != 1) || !out_len || !out_start) return fail(PCWD_E_PARAM, "pcwd_plan_atom arguments");
  Plan P{};
  P.L2 = desc->filter_len;
  for (int j = 0; j < P.L2; ++j) {   // f_0 = h, f_1[j] = g[2 − 2δ + j] = (−1)^{1−i} h[1−i], i = 2 − 2δ + j (common.h)
    const int i = 2 - P.L2 + j;
    P.td[0][j] = desc->h[j];
    P.td[1][j] = ((1 - i) % 2 == 0 ? 1.0 : -1.0) * desc->h[1 - i];
  }
  std::vector<double> w;
  sep_base_atom(P, s, e, &w);
  *out_len = int32_t(w.size());
  *out_start = sep_atom_start(s, e, P.L2);
  if (out) {
    if (cap < int32_t(w.size())) return fail(PCWD_E_PARAM, "pcwd_plan_atom: cap smaller than the atom");
    std::copy(w.begin(), w.end(), out);
  }
  return PCWD_OK;
}

int pcwd_create(const pcwd_desc* desc, void** out_handle) {
  if (!out_handle) return fail(PCWD_E_PARAM, "out_handle is NULL");
  *out_handle = nullptr;
  std::string msg;
  int rc = validate_desc(desc, &msg);
  if (rc) return fail(rc, msg);
  if (!desc->u || !desc->v) return fail(PCWD_E_PARAM, "u or v is NULL");
  CK(cudaSetDevice(desc->device));
  const int64_t N = desc->d == 2 ? int64_t(desc->n) * desc->n : desc->n;
  const int64_t mN = int64_t(desc->m) * N;
  const bool u_dev = is_device_ptr(desc->u), v_dev = is_device_ptr(desc->v);
  std::vector<double> u_host;
  const double* uh = desc->u;
  if (u_dev) {
    u_host.resize(mN);
    CK(cudaMemcpy(u_host.data(), desc->u, mN * sizeof(double), cudaMemcpyDeviceToHost));
    uh = u_host.data();
  }
  // PATTERN: the caller's CSR over all units, checked on the host (monotone row pointers, columns in range and
  // strictly increasing within each row); the handle keeps its shard's rows
  std::vector<int64_t> pat_rp;
  std::vector<int32_t> pat_col;
  if (desc->retain == PCWD_RETAIN_PATTERN) {
    pat_rp.resize(N + 1);
    CK(cudaMemcpy(pat_rp.data(), desc->pat_rowptr, (N + 1) * sizeof(int64_t), cudaMemcpyDefault));
    if (pat_rp[0] != 0) return fail(PCWD_E_PARAM, "pat_rowptr[0] must be 0");
    for (int64_t i = 0; i < N; ++i)
      if (pat_rp[i + 1] < pat_rp[i]) return fail(PCWD_E_PARAM, "pat_rowptr must be non-decreasing");
    if (pat_rp[N] > (int64_t(1) << 40)) return fail(PCWD_E_PARAM, "pattern too large");
    pat_col.resize(std::max<int64_t>(pat_rp[N], 1));
    if (pat_rp[N] > 0) CK(cudaMemcpy(pat_col.data(), desc->pat_col, pat_rp[N] * sizeof(int32_t), cudaMemcpyDefault));
    for (int64_t i = 0; i < N; ++i)
      for (int64_t j = pat_rp[i]; j < pat_rp[i + 1]; ++j) {
        if (pat_col[j] < 0 || pat_col[j] >= N) return fail(PCWD_E_PARAM, "pat_col out of range at row " + std::to_string(i));
        if (j > pat_rp[i] && pat_col[j] <= pat_col[j - 1])
          return fail(PCWD_E_PARAM, "pat_col not strictly increasing in row " + std::to_string(i));
      }
  }
  Handle* h = new Handle();
  h->desc = *desc;
  rc = build_plan(desc, uh, &h->hp, &msg);
  if (rc) { delete h; return fail(rc, msg); }
  const Plan& P = h->hp.P;
  const int rb = h->hp.real_bytes, ob = h->hp.out_bytes;
  auto bail = [&](int code, const std::string& m) { free_all(h); delete h; return fail(code, m); };
#define CKB(call)                                                                                  \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess)                                                                         \
      return bail(e_ == cudaErrorMemoryAllocation ? PCWD_E_OOM : PCWD_E_CUDA,                      \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                             \
  } while (0)

  // inputs: u in fp64 (template build), v in the compute type (host → device boundary)
  CKB(dalloc(&h->u_d, mN * sizeof(double)));
  CKB(cudaMemcpy(h->u_d, desc->u, mN * sizeof(double), u_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
  CKB(dalloc(&h->v_d, mN * rb));
  if (rb == 8) {
    CKB(cudaMemcpy(h->v_d, desc->v, mN * sizeof(double), v_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
  } else {
    double* tmp = nullptr;
    CKB(dalloc(&tmp, mN * sizeof(double)));
    CKB(cudaMemcpy(tmp, desc->v, mN * sizeof(double), v_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
    CKB(launch_cast(tmp, h->v_d, mN, 4, 0));
    CKB(cudaDeviceSynchronize());
    cudaFree(tmp);
  }
  CKB(dalloc(&h->T_d, std::max<int64_t>(h->hp.tmpl_elems, 1) * rb));
  CKB(dalloc(&h->phi[0], int64_t(P.m) * h->hp.phi_elems * sizeof(double)));
  CKB(dalloc(&h->phi[1], int64_t(P.m) * h->hp.phi_elems * sizeof(double)));
  CKB(dalloc(&h->Ytmp, int64_t(P.m) * std::max<int64_t>(h->hp.y_elems, 1) * sizeof(double)));
  if (!h->hp.stencil.empty()) {
    std::vector<int4> st(h->hp.stencil.size());
    for (size_t i = 0; i < st.size(); ++i)
      st[i] = make_int4(h->hp.stencil[i].sb, h->hp.stencil[i].o0, h->hp.stencil[i].o1,
                        P.sb[h->hp.stencil[i].sb].level);
    CKB(dalloc(&h->stencil_d, st.size() * sizeof(int4)));
    CKB(cudaMemcpy(h->stencil_d, st.data(), st.size() * sizeof(int4), cudaMemcpyHostToDevice));
  }

  // launch plan: one launch per level inside the shard; in-smem when the unit scratch fits
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, desc->device);
  int smem_optin = 0;
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, desc->device);
  const size_t budget = std::min<size_t>(kSmemBudget, size_t(smem_optin > 0 ? smem_optin : 48 * 1024) - 8 * 1024);
  if (!h->hp.stencil_box.empty()) {
    std::vector<int4> bx(h->hp.stencil_box.size() / 4);
    for (size_t i = 0; i < bx.size(); ++i)
      bx[i] = make_int4(h->hp.stencil_box[4 * i], h->hp.stencil_box[4 * i + 1], h->hp.stencil_box[4 * i + 2],
                        h->hp.stencil_box[4 * i + 3]);
    CKB(dalloc(&h->box_d, bx.size() * sizeof(int4)));
    CKB(cudaMemcpy(h->box_d, bx.data(), bx.size() * sizeof(int4), cudaMemcpyHostToDevice));
  }
  if (!h->hp.fgeom.empty()) {
    CKB(dalloc(&h->fgeom_d, h->hp.fgeom.size() * sizeof(FGeom)));
    CKB(cudaMemcpy(h->fgeom_d, h->hp.fgeom.data(), h->hp.fgeom.size() * sizeof(FGeom), cudaMemcpyHostToDevice));
  }
  if (!h->hp.sepcls.empty() && !h->hp.seprun.empty()) {
    const HostPlan& hp = h->hp;
    auto up = [&](auto** dst, const auto& vec) -> cudaError_t {
      cudaError_t e = dalloc(dst, vec.size() * sizeof(vec[0]));
      if (e != cudaSuccess) return e;
      return cudaMemcpy(*dst, vec.data(), vec.size() * sizeof(vec[0]), cudaMemcpyHostToDevice);
    };
    CKB(up(&h->sepc_d, hp.sepcls));
    CKB(up(&h->seprun_d, hp.seprun));
    CKB(up(&h->seppart_d, hp.seppart));
    CKB(up(&h->septask_d, hp.septask));
    {   // tap table in the kernel's shared-memory layout (geom.h sep_toff), compute type
      std::vector<double> tab(sep_ttot(P.L2), 0.0);
      for (int s2 = 1; s2 <= hp.sep_smax; ++s2)
        for (int e2 = 0; e2 < 2; ++e2)
          for (int i = 0; i < hp.atom_len[s2]; ++i) tab[sep_toff(s2, e2, P.L2) + i] = hp.atoms[hp.atom_off[s2][e2] + i];
      if (rb == 8) {
        CKB(up(reinterpret_cast<double**>(&h->atoms_d), tab));
      } else {
        std::vector<float> tf(tab.begin(), tab.end());
        CKB(up(reinterpret_cast<float**>(&h->atoms_d), tf));
      }
    }
  }
  int64_t gmax = 0;
  h->conc = P.retain == PCWD_RETAIN_BAND && !getenv("PCWD_COARSE_SERIAL");
  auto add_generic = [&](int64_t u0, int64_t u1, int64_t scr) {
    if (u1 <= u0) return;
    size_t bytes = size_t(scr) * rb;
    Launch L{u0, u1, 0, 0};
    // shared-memory scratch only up to 48 KB per unit (c4 sweep 32-100 KB: 74 ms at 32-56, 78 at 72-100); larger
    // windows work in global (L2) scratch with 4 units per SM in flight
    static const size_t smem_cap = size_t(getenv("PCWD_GENERIC_SMEM_KB") ? atoi(getenv("PCWD_GENERIC_SMEM_KB")) : 48) << 10;
    if (bytes <= std::min<size_t>(budget, smem_cap)) {
      L.smem = std::max<size_t>(bytes, 16);
      int per_sm = int(std::min<size_t>(8, (228 * 1024) / (L.smem + 2048)));
      per_sm = std::max(per_sm, 1);
      L.grid = int(std::min<int64_t>(u1 - u0, int64_t(nsm) * per_sm));
    } else {   // its own slice of the global scratch (launches may run concurrently)
      L.grid = int(std::min<int64_t>(u1 - u0, int64_t(nsm) * 8));   // 128-thread CTAs, up to 6-8 per SM
      L.gs_stride = (scr + 31) & ~int64_t(31);
      L.gs_off = gmax;
      gmax += L.gs_stride * L.grid;
      // hybrid: the step-1 approximation and every buffer of steps ≥ 2 (small windows, latency-bound chains of
      // barriers) in shared memory; the k-sum window and the step-1 pass-A / detail buffers stay in global
      int64_t hs = 0;
      for (int q = 0; q < P.nsb; ++q)
        if (P.sb[q].offset < u1 && P.sb[q].offset + P.sb[q].count > u0) hs = std::max(hs, P.sb[q].hs_size);
      static const size_t hcap = size_t(getenv("PCWD_HYBRID_KB") ? atoi(getenv("PCWD_HYBRID_KB")) : 40) << 10;
      if (hs > 0 && size_t(hs) * rb <= std::min<size_t>(budget, hcap)) {
        L.smem = size_t(hs) * rb;
        L.hybrid = 1;
      }
    }
    h->launches.push_back(L);
  };
  for (int s = 0; s < P.nsb;) {
    int lev = P.sb[s].level;
    int e = s;
    int64_t scr = 0;
    bool tile_ok = P.retain == PCWD_RETAIN_BAND && P.d == 2 && lev <= P.J;
    while (e < P.nsb && P.sb[e].level == lev) {
      scr = std::max(scr, P.sb[e].scratch);
      tile_ok = tile_ok && P.sb[e].wk_ok && P.sb[e].steps <= 6 && P.sb[e].e != 0;
      ++e;
    }
    int64_t u0 = std::max(h->hp.row0, P.sb[s].offset);
    int64_t u1 = std::min(h->hp.row1, P.sb[e - 1].offset + P.sb[e - 1].count);
    if (u1 <= u0) { s = e; continue; }
    // fine kernel (fine.cu): levels 1..3 whose every sub-band has a class geometry table
    {
      FineCfg fc{};
      bool ok = P.retain == PCWD_RETAIN_BAND && P.d == 2 && fine_config(rb, lev, P.L2, &fc) && !getenv("PCWD_NO_FINE") &&
                lev <= (getenv("PCWD_FINE_MAXLEV") ? atoi(getenv("PCWD_FINE_MAXLEV")) : 3);
      for (int q = s; q < e && ok; ++q) ok = P.sb[q].fg_m > 0 && P.sb[q].e != 0 && P.sb[q].nl % fc.GU == 0;
      if (ok) {
        const int VW = 16 / rb, SH = 1 << lev;
        const SubBand& S0 = P.sb[s];
        const int R0 = S0.tW[0], R1 = S0.tW[1];
        for (int q = s; q < e; ++q) ok = ok && P.sb[q].tW[0] == R0 && P.sb[q].tW[1] == R1;
        const int NZB = ((R1 + SH - 1) / SH + fc.GZ - 1) / fc.GZ;
        ok = ok && int64_t(R0) * SH * NZB <= int64_t(fc.NT) * 256;
        // strides: multiples of VW with an odd vector count (8 consecutive rows -> distinct bank groups)
        auto odd_stride = [&](int w) { int x = (w + VW - 1) / VW * VW; if ((x / VW) % 2 == 0) x += VW; return x; };
        int arl = 0, ycols = 0, dsz = 0, arl2 = 0, ycols2 = 0;
        for (int q = s; q < e && ok; ++q) {
          const SubBand& Sq = P.sb[q];
          ok = ok && Sq.steps <= lev + 2;     // sdesc capacity of the kernel
          for (int c = 0; c < Sq.fg_m * Sq.fg_m; ++c) {
            const FGeom& g = h->hp.fgeom[Sq.fg_off + c];
            dsz = std::max(dsz, g.dsize);
            for (int st = 0; st < g.steps; ++st) {
              if (st == 0) {
                arl = std::max(arl, g.st[st].arl);
                ycols = std::max(ycols, g.st[st].hlen + g.st[st].glen);
              } else {
                arl2 = std::max(arl2, g.st[st].arl);
                ycols2 = std::max(ycols2, g.st[st].hlen + g.st[st].glen);
              }
              // the approximations of steps ≥ 1 are stored in the unit's R region (row stride RS)
              if (st > 0) ok = ok && g.st[st].xcl + VW - 1 <= ((R1 + VW - 1) / VW * VW) && g.st[st].xrl <= R0;
            }
          }
        }
        // R rows: [roff, roff + R1) valid, zero pad of ≥ 2δ + 2 after (serves as the next row's left pad);
        // even stride with an odd number of pairs (16 lanes of 8-byte loads hit distinct banks)
        auto pair_stride = [&](int w) { int x = (w + 1) / 2 * 2; if ((x / 2) % 2 == 0) x += 2; return x; };
        int roffmax = 0;   // R rows are shifted by one column when a window starts at an odd column
        for (int q = s; q < e; ++q) roffmax |= P.sb[q].tSu[1] & 1;
        // separable direct a3 + a4 (plan.cpp build_sep): odd R row stride (a warp's lanes read 32 rows of one column)
        // PCWD_SEP: bit mask over fine levels 1..3; default fp32 4 = level 3 only (c5, B200: level 3 1.95 ms separable
        // vs 2.11 ms cascade; levels 1 / 2 8.1 / 2.66 ms vs 7.3 / 2.54 ms), fp64 6 = levels 2-3 (7.91 / 5.68 ms vs
        // 8.35 / 6.15; level 1 17.1 vs 16.3 ms) — DESIGN.md §6
        static const int sep_env = getenv("PCWD_SEP") ? atoi(getenv("PCWD_SEP")) : -1;
        const int sep_mask = sep_env >= 0 ? sep_env : (rb == 8 ? 6 : 4);
        const bool sep = h->hp.sep_ok[lev] && ((sep_mask >> (lev - 1)) & 1);
        const int RS = sep ? ((R1 + std::max(kSepPad, roffmax + P.L2 + 2)) | 1) : pair_stride(R1 + roffmax + P.L2 + 2);
        const int zmaxT = (SH - 1) + SH * fc.GZ * (NZB - 1) + SH * (fc.GZ - 1);
        const int zmaxV = zmaxT + SH * (fc.GU - 1);
        const int TS = odd_stride(std::max(S0.tRS, zmaxT + 1));
        const int VS = odd_stride(VW - 1 + std::max(R1 + SH * (fc.GU - 1), zmaxV + 1));
        const int YS = pair_stride(arl + VW - 1);
        const int64_t lpad = P.band_Lpad + (int64_t(P.band_Lpad) * 8 + rb - 1) / rb;   // gather: values, columns, heavy list
        const int64_t YSZ = (int64_t(ycols) * YS + VW - 1) / VW * VW;
        const int YS2 = pair_stride(arl2 + VW - 1);
        const int64_t YSZ2 = (std::max<int64_t>(int64_t(ycols2) * YS2, lpad) + VW - 1) / VW * VW;
        const int64_t RSZ = int64_t(R0) * RS;
        const int64_t DS = (dsz + VW - 1) / VW * VW;
        const int SLK = 32;
        const int64_t regR = SLK + fc.GU * RSZ + SLK;
        const int al = 128 / rb;   // TMA destinations: 128-byte aligned boxes
        const int TSZ = (R0 * TS + al - 1) / al * al, VSZ = (R0 * VS + al - 1) / al * al;
        // staging ring depth: the ring may use the whole dynamic smem (R, Yt and D regions are all idle
        // during the k-sum); as many buffers as fit, up to the kernel's NST
        // Yt slots (pass-A output of any step, then the gather stage) are max(YSZ, YSZ2) apart
        int64_t YSL = std::max<int64_t>(YSZ, YSZ2);
        // separable path: Q (R0 rows × QS) then the gather stage in each slot
        int QS = 0;
        int64_t QSZ = 0;
        if (sep) {
          QS = R0 | 1;   // Q is column-major: column stride (rows)
          QSZ = (int64_t(h->hp.sep_nq[lev]) * QS + VW - 1) / VW * VW;
          // Q, the gather stage (values, columns) and the class's stage-1 runs; no Yt / D buffers (cascade only)
          YSL = QSZ + (2 * int64_t(P.band_Lpad) + int64_t(h->hp.sep_nrun[lev]) * int64_t(sizeof(SepRun)) / rb + VW - 1) / VW * VW;
        }
        const int64_t regS = SLK + (sep ? fc.CG * YSL : std::max<int64_t>(fc.CG * YSL, fc.GU * YSZ2)) + SLK;
        const int64_t regD = regR + regS;
        int64_t total_el = regD + (sep ? 0 : fc.GU * DS);
        int nst = int(std::min<int64_t>(fc.NST, (total_el - SLK - al) / (TSZ + VSZ)));
        if (nst < 1) {   // enlarge the allocation to hold one staging buffer
          total_el = SLK + al + (TSZ + VSZ);
          nst = 1;
        }
        const int64_t stg = int64_t(nst) * (TSZ + VSZ) + al;
        const int64_t elA = (std::max<int64_t>(total_el, regD + (sep ? 0 : fc.GU * DS)) + 3) & ~int64_t(3);   // atom taps (sep)
        const int ntap = sep ? sep_ttot(P.L2) : 0;
        const size_t smem = size_t(elA + ntap) * rb;
        ok = ok && smem + 4096 <= size_t(smem_optin > 0 ? smem_optin : 48 * 1024);
        int64_t a0 = (u0 + fc.GU - 1) / fc.GU * fc.GU, a1 = u1 / fc.GU * fc.GU;
        if (getenv("PCWD_DEBUG_PLAN"))
          fprintf(stderr, "[pcwd fine] level %d ok %d GU %d R %dx%d RS %d TS %d VS %d YS %d ycols %d arl %d dsz %d "
                  "regR %lld stg %lld yt %lld smem %zu\n", lev, int(ok), fc.GU, R0, R1, RS, TS, VS, YS, ycols, arl, dsz,
                  (long long)regR, (long long)stg, (long long)std::max<int64_t>(fc.CG * YSZ, fc.GU * YSZ2), smem);
        if (ok && a1 > a0) {
          Launch F{a0, a1, 0, 0};
          F.fine = 1;
          F.gu = fc.GU;
          F.level = lev;
          F.smem = smem;
          const int per_sm = int(std::max<size_t>(1, std::min<size_t>(2, (228 * 1024) / (smem + 4096))));
          // (MINB = 1 instances use up to 255 registers: one CTA per SM regardless of smem)
          F.grid = int(std::min<int64_t>((a1 - a0) / fc.GU, int64_t(nsm) * per_sm));
          FineArgs& A = F.fa;
          A.u0 = a0; A.u1 = a1;
          A.regS = regR; A.regD = regD;
          A.TSZ = TSZ; A.VSZ = VSZ;
          A.nst = nst;
          A.sep = sep ? 1 : 0;
          A.regA = elA;
          A.ntap = ntap;
          A.QS = QS;
          A.QSZ = int(QSZ);
          // partner levels computed directly from the last cascade approximation: PCWD_FINE_DIRECT = "d1,d2,d3"
          // per fine level (2 = one step of 2δ × 2δ taps plus one composite step, 1 = the 2δ × 2δ step only)
          {
            int dl[3] = {2, 2, 1};   // measured on c5: level 3 faster with one more cascade step
            if (const char* e = getenv("PCWD_FINE_DIRECT")) sscanf(e, "%d,%d,%d", &dl[0], &dl[1], &dl[2]);
            A.direct = getenv("PCWD_NO_DIRECT") ? 0 : std::max(0, std::min(2, dl[lev - 1]));
          }
          (void)stg;
          A.sb_first = s;
          // halo of the padded v that every round's boxes stay inside
          int tmin0 = 1 << 30, tmax0 = -(1 << 30), tmin1 = 1 << 30, tmax1 = -(1 << 30);
          for (int q = s; q < e; ++q) {
            tmin0 = std::min(tmin0, P.sb[q].tSu[0]); tmax0 = std::max(tmax0, P.sb[q].tSu[0]);
            tmin1 = std::min(tmin1, P.sb[q].tSu[1]); tmax1 = std::max(tmax1, P.sb[q].tSu[1]);
          }
          const int nl = S0.nl;
          auto fl = [&](int x) { return x >= 0 ? x / VW * VW : -((-x + VW - 1) / VW) * VW; };
          const int need = std::max({-tmin0, -fl(tmin1), ((nl - 1) << lev) + tmax0 + R0 - P.n,
                                     fl(((nl - fc.GU) << lev) + tmax1) + VS - P.n, 0});
          h->vpad = std::max(h->vpad, (need + 3) / 4 * 4);
          F.box[0] = R0; F.box[1] = TS; F.box[2] = VS;
          A.RS = RS; A.RSZ = int(RSZ); A.TS = TS; A.VS = VS; A.YS = YS; A.YSZ = int(YSL); A.DS = int(DS);
          A.YS2 = YS2; A.YSZ2 = int(YSZ2);
          add_generic(u0, a0, scr);
          h->launches.push_back(F);
          add_generic(a1, u1, scr);
          s = e;
          continue;
        }
      }
    }
    Launch T{0, 0, 0, 0};
    // the tile kernel only where the fine kernel does not apply and windows are small (levels ≤ 3); coarser
    // levels run faster on the batched path (tiled k-sum + fused approximation steps)
    if (tile_ok && lev <= 3 && !getenv("PCWD_NO_TILE")) {
      // per-unit scratch of the tile kernel: X (R window and approximations), Yt, D boxes, stage
      const SubBand& S0 = P.sb[s];
      const int VW = 16 / rb;
      // row stride: window + alignment and vector-read slack, ≡ VW (mod 2·VW) so that 8
      // consecutive rows hit distinct 16-byte bank groups
      auto stride = [&](int w) {
        int x = (w + P.L2 + 16 + VW - 1) / VW * VW;
        while (x % (2 * VW) != VW) x += VW;
        return x;
      };
      int W0 = S0.tW[0], W1 = S0.tW[1];
      int XR = W0, XS = stride(W1), YS = stride(W0);
      // Yt rows (pass-A outputs) and D boxes, per step: approximation width + stencil boxes
      int YR = 0;
      int64_t dmax = 0;
      for (int q = s; q < e; ++q) {
        int a1 = W1;
        for (int st = 1; st <= P.sb[q].steps; ++st) {
          a1 = (a1 >> 1) + (P.L2 >> 1);
          int64_t area = 0;
          int gw = 0, hw = 0;
          for (int t = 0; t < P.nsb; ++t) {
            if (P.sb[t].level != st) continue;
            const int* b = &h->hp.stencil_box[(size_t(q) * P.nsb + t) * 4];
            if (b[0] > b[1]) continue;
            area += int64_t(b[1] - b[0] + 1) * (b[3] - b[2] + 1);
            if (P.sb[t].e1) gw = std::max(gw, b[3] - b[2] + 1);
            else hw = std::max(hw, b[3] - b[2] + 1);
          }
          const int hcols = (st < P.sb[q].steps || st == P.J) ? a1 : std::min(a1, hw);
          YR = std::max(YR, hcols + std::min(a1, gw) + 1);
          dmax = std::max(dmax, area);
        }
      }
      // D keeps every step's boxes (gather at the end): total stencil box area of the sub-band
      dmax = 0;
      for (int q = s; q < e; ++q) {
        int64_t area = 0;
        for (int t = 0; t < P.nsb; ++t) {
          const int* b = &h->hp.stencil_box[(size_t(q) * P.nsb + t) * 4];
          if (b[0] <= b[1]) area += int64_t(b[1] - b[0] + 1) * (b[3] - b[2] + 1);
        }
        dmax = std::max(dmax, area);
      }
      dmax = (dmax + VW - 1) / VW * VW;
      int64_t stage = P.band_Lpad + (int64_t(P.band_Lpad) * 4 + rb - 1) / rb;
      const int SL = 32;   // kSL of band_tile.cu
      const int64_t Xsz = int64_t(XR) * XS + 2 * SL, Ysz = int64_t(YR) * YS + 2 * SL;
      const int64_t Dsz = (dmax + stage + VW - 1) / VW * VW;
      int G = lev == 1 ? 4 : lev <= 3 ? 2 : 1;
      const int nl = P.sb[s].nl;
      const size_t st_bytes = size_t(e - s) * P.band_L * sizeof(int4);
      auto layout = [&](int g, int64_t* regY, int64_t* regD, int64_t* regEnd, int* TS, int* VS, int* RC) {
        const int step = 1 << lev;
        const int groups = (W1 + 3) / 4;
        *RC = std::max(1, std::min(W0, (2 * 256) / groups));
        *TS = (W1 + 3) / 4 * 4;
        *VS = (W1 + (g - 1) * step + 3 + 4) / 4 * 4;
        const int64_t stg = 2 * int64_t(*RC) * (*TS + *VS);
        *regY = g * Xsz;
        *regD = *regY + std::max<int64_t>(g * Ysz, stg);
        *regD = (*regD + VW - 1) / VW * VW;
        *regEnd = *regD + g * Dsz;
        *regEnd = (*regEnd + 3) / 4 * 4;
        return size_t(*regEnd) * rb + st_bytes;
      };
      int64_t regY = 0, regD = 0, regEnd = 0;
      int TS = 0, VS = 0, RC = 0;
      const size_t two_per_sm = 110 * 1024;
      while (G > 1 && (layout(G, &regY, &regD, &regEnd, &TS, &VS, &RC) > two_per_sm || nl % G)) G >>= 1;
      size_t smem = layout(G, &regY, &regD, &regEnd, &TS, &VS, &RC);
      int64_t per_unit = Xsz + Ysz + Dsz;
      if (smem <= budget && nl % G == 0) {
        // whole rounds of G units inside [u0, u1); the ragged ends go to the generic kernel
        int64_t a0 = (u0 + G - 1) / G * G, a1 = u1 / G * G;
        if (a1 > a0) {
          T.u0 = a0;
          T.u1 = a1;
          T.tile = 1;
          T.smem = smem;
          int per_sm = int(std::max<size_t>(1, std::min<size_t>(8, (228 * 1024) / (smem + 4096))));
          T.grid = int(std::min<int64_t>((a1 - a0) / G, int64_t(nsm) * per_sm));
          T.ta.u0 = a0;
          T.ta.u1 = a1;
          T.ta.G = G;
          T.ta.XS = XS;
          T.ta.YS = YS;
          T.ta.XR = XR;
          T.ta.YR = YR;
          T.ta.DMAX = int(dmax);
          T.ta.per_unit = int(per_unit);
          T.ta.Xsz = int(Xsz);
          T.ta.Ysz = int(Ysz);
          T.ta.Dsz = int(Dsz);
          T.ta.regY = regY;
          T.ta.regD = regD;
          T.ta.regEnd = regEnd;
          T.ta.TS = TS;
          T.ta.VS = VS;
          T.ta.RC = RC;
          add_generic(u0, a0, scr);
          h->launches.push_back(T);
          add_generic(a1, u1, scr);
          s = e;
          continue;
        }
      }
    }
    if (P.retain == PCWD_RETAIN_BAND && P.d == 2 && !getenv("PCWD_NO_BATCHED")) {
      // batched grid kernels: per-unit slots of the generic layout in one global buffer
      Launch B{u0, u1, 0, 0};
      B.batched = 1;
      int64_t stride = (scr + 31) & ~int64_t(31);
      // units per batch: up to 32 GiB of slots per level (one batch per level at c5 and 2048²); the sum over
      // the levels is fitted to the free device memory after the plan (below)
      static const size_t cap = size_t(getenv("PCWD_BATCH_MB") ? atol(getenv("PCWD_BATCH_MB")) : 32768) << 20;
      int64_t batch = std::max<int64_t>(1, std::min<int64_t>(u1 - u0, int64_t(cap / (size_t(stride) * rb))));
      batch = std::min<int64_t>(batch, 65535);
      B.ba.stride = stride;
      B.ba.u0 = u0;
      B.ba.u1 = u1;
      B.ba.batch = batch;
      int steps = 0;
      int64_t mx0 = 0, my = 0, mb = 0;
      for (int q = s; q < e; ++q) {
        const SubBand& S = P.sb[q];
        steps = std::max(steps, S.steps);
        int64_t w0 = std::min(S.tW[0], P.n), w1 = std::min(S.tW[1], P.n);
        mx0 = std::max(mx0, w0 * w1);
        int64_t nl0 = P.n, nl1 = P.n;
        for (int st = 1; st <= S.steps; ++st) {
          int64_t o0 = step_out_maxlen(int(w0), int(nl0), P.L2), o1 = step_out_maxlen(int(w1), int(nl1), P.L2);
          my = std::max(my, w0 * 2 * o1);
          mb = std::max(mb, 4 * o0 * o1);
          B.workA[st] = std::max(B.workA[st], w0 * ((o1 + 3) / 4));
          B.workB[st] = std::max(B.workB[st], ((o0 + 3) / 4) * o1);
          B.appr0[st] = std::max(B.appr0[st], o0);
          B.appr1[st] = std::max(B.appr1[st], o1);
          w0 = o0; w1 = o1; nl0 >>= 1; nl1 >>= 1;
        }
      }
      B.maxX0 = mx0;
      B.maxY = my;
      B.maxB = mb;
      B.steps = steps;
      // tiled k-sum with TMA staging (levels ≤ 5): maps of the level's templates here, of the periodically
      // extended v once its extent (max strip over the levels) is known
      B.level = lev;
      static const int tma_maxlev = getenv("PCWD_TMA_KSUM_MAXLEV") ? atoi(getenv("PCWD_TMA_KSUM_MAXLEV")) : 8;
      const int gz = lev <= tma_maxlev && !getenv("PCWD_NO_TMA_KSUM") ? ksum_tiled_gz(P, u0, u1, rb) : 0;
      if (gz) {
        const int SH = 1 << lev, TR = 256 / SH, G = kt_units(rb);
        const int qT = kt_box_q(SH, gz, kt_box_n(SH, gz));
        const int qV = kt_vbox_q(SH, gz + G - 1, kt_vbox_n(SH, gz + G - 1, rb), rb);
        h->kt_pr = std::max(h->kt_pr, TR);
        h->kt_pc = std::max(h->kt_pc, SH * qV + kt_vpadx(SH, rb));   // one v box past the seam
        int rc2 = 0;
        for (int q = s, i = 0; q < e && i < 3 && !rc2; ++q, ++i)
          rc2 = encode_map3(&B.ba.tmT[i], static_cast<char*>(h->T_d) + P.sb[q].toff * rb, rb, P.sb[q].tRS, P.sb[q].tW[0],
                            P.m, P.sb[q].tRS, P.sb[q].tstride, SH * qT, TR);
        if (rc2) return bail(PCWD_E_CUDA, "cuTensorMapEncodeTiled (k-sum) failed: " + std::to_string(rc2));
        B.ba.kt_gz = gz;
        B.ba.kt_sb_first = s;
      }
      B.ba.kt_sb_first = s;
      // whole-torus k-sum with TMA (2^ℓ = 256, a sub-band row of 2 or 4 units): v and template maps, 256 × 2 boxes
      // (2^ℓ = 256·SHM with SHM ∈ {1, 2, 4}: rows per thread 2 at SHM = 1, else 1)
      const int kshm = lev >= 8 && lev <= 10 ? (1 << lev) / 256 : 0;
      const int knl = P.sb[s].nl;
      const bool kf_ok = (kshm == 1 && (knl == 2 || knl == 4)) || (kshm == 2 && (knl == 2 || knl == 4)) ||
                         (kshm == 4 && knl == 2);
      if (!gz && P.d == 2 && kf_ok && (1 << lev) * knl == P.n && e - s <= 4 && !getenv("PCWD_NO_TMA_KSUM")) {
        const int trt = kshm == 1 ? 2 : 1;
        bool full = true;
        for (int q = s; q < e; ++q) full = full && P.sb[q].tW[0] >= P.n && P.sb[q].tW[1] >= P.n;
        int rc2 = full ? encode_map3(&B.ba.tmV, h->v_d, rb, P.n, P.n, P.m, P.n, int64_t(P.n) * P.n, 256, trt) : 1;
        for (int q = s, i = 0; full && q < e && !rc2; ++q, ++i)
          rc2 = encode_map3(&B.ba.tmT[i], static_cast<char*>(h->T_d) + P.sb[q].toff * rb, rb, P.sb[q].tRS, P.n, P.m,
                            P.sb[q].tRS, P.sb[q].tstride, 256, trt);
        if (full && rc2) return bail(PCWD_E_CUDA, "cuTensorMapEncodeTiled (whole-torus k-sum) failed: " + std::to_string(rc2));
        if (full) B.ba.kf_rows = trt;
      }
      // approximation steps on the TMA path: every participating sub-band's step-s input window has one size
      // over its units and stays clear of wrapping (maps encoded once the scratch exists)
      for (int st = 1; st <= steps && st < 32; ++st) {
        bool ok = e - s <= 4 && !getenv("PCWD_NO_TMA_APPROX");
        for (int q = s; q < e && ok; ++q) {
          const SubBand& Sq = P.sb[q];
          if (!(st < Sq.steps || st == P.J)) continue;
          for (int a = 0; a < 2 && ok; ++a) {
            int len = -1;
            for (int p = 0; p < Sq.nl && ok; ++p) {
              Range w = unit_window(P, Sq, a, p);
              for (int t = 1; t < st; ++t) w = step_out(w, P.L2, 0);
              ok = (len < 0 || w.len == len) && w.len + 2 * P.L2 <= w.nl;
              len = w.len;
            }
          }
        }
        if (ok) B.ba.am_steps |= 1u << st;
      }
      // per-unit tail: from the first step ≥ 3 (measured best on c5) whose input window, pass-A output and
      // approximation fit in 64 KB
      if (L2OK(P.L2)) {
        static const int smin = getenv("PCWD_TAIL_S0_MIN") ? atoi(getenv("PCWD_TAIL_S0_MIN")) : 3;
        for (int st = std::max(2, smin); st <= steps; ++st) {
          const int64_t am = (B.appr0[st - 1] * B.appr1[st - 1] + 3) & ~int64_t(3);
          if ((2 * am + B.appr0[st - 1] * B.appr1[st]) * rb <= 64 * 1024) { B.ba.tail_s0 = st; break; }
        }
      }
      if (h->conc) {   // concurrent coarse levels: one scratch slice each
        B.bs_off = h->bscratch_bytes;
        h->bscratch_bytes += (size_t(batch) * stride * rb + 1023) & ~size_t(1023);
      } else {
        h->bscratch_bytes = std::max(h->bscratch_bytes, size_t(batch) * stride * rb);
      }
      h->launches.push_back(B);
      s = e;
      continue;
    }
    add_generic(u0, u1, scr);
    s = e;
  }
  if (h->bscratch_bytes) {
    // fit the coarse scratch into half of the free device memory (the CSR, candidates and templates need the
    // rest): concurrent levels share the budget equally, serial levels share one slice; batches shrink to fit
    size_t freeb = 0, totb = 0;
    CKB(cudaMemGetInfo(&freeb, &totb));
    const size_t budget = freeb / 2;
    if (h->bscratch_bytes > budget) {
      int nb = 0;
      for (const Launch& L : h->launches) nb += L.batched;
      const size_t per = h->conc ? budget / size_t(std::max(nb, 1)) : budget;
      size_t off = 0, mx = 0;
      for (Launch& L : h->launches) {
        if (!L.batched) continue;
        const size_t ub = size_t(L.ba.stride) * rb;
        L.ba.batch = std::max<int64_t>(1, std::min<int64_t>(L.ba.batch, int64_t(per / ub)));
        const size_t bytes = size_t(L.ba.batch) * ub;
        if (h->conc) { L.bs_off = off; off += (bytes + 1023) & ~size_t(1023); }
        mx = std::max(mx, bytes);
      }
      h->bscratch_bytes = h->conc ? off : mx;
    }
    CKB(dalloc(&h->bscratch, h->bscratch_bytes + 1024));   // + vector over-read slack
  }
  {
    int nb = 0;
    for (const Launch& L : h->launches) nb += L.batched;
    h->conc = h->conc && nb > 1;
    int ng = 0;
    for (const Launch& L : h->launches) ng += !L.batched && !L.fine && !L.tile;
    h->conc_t = P.retain == PCWD_RETAIN_THRESHOLD && ng > 1 && !getenv("PCWD_COARSE_SERIAL");
    if (h->conc || h->conc_t) {
      CKB(cudaEventCreateWithFlags(&h->efork, cudaEventDisableTiming));
      for (int i = 0; i < Handle::kNCS; ++i) {
        CKB(cudaStreamCreateWithFlags(&h->cstream[i], cudaStreamNonBlocking));
        CKB(cudaEventCreateWithFlags(&h->ejoin[i], cudaEventDisableTiming));
      }
    }
  }
  {  // TMA maps of the approximation steps: [launch][step - 1][sub-band - first] over the scratch input buffer
    std::vector<CUtensorMap> maps;
    std::vector<size_t> first;
    for (Launch& L : h->launches) {
      first.push_back(maps.size());
      if (!L.batched || !L.ba.am_steps) continue;
      maps.resize(maps.size() + 32 * 4);
      CUtensorMap* M = maps.data() + first.back();
      const int TI = ap_ti(rb, P.L2), BW = ap_bw(rb, P.L2);
      for (int st = 1; st < 32; ++st) {
        if (!((L.ba.am_steps >> st) & 1u)) continue;
        for (int q = L.ba.kt_sb_first, i = 0; q < P.nsb && i < 4 && P.sb[q].offset < L.u1; ++q, ++i) {
          const SubBand& Sq = P.sb[q];
          if (!(st < Sq.steps || st == P.J)) continue;
          Range w0 = unit_window(P, Sq, 0, 0), w1 = unit_window(P, Sq, 1, 0);
          for (int t = 1; t < st; ++t) { w0 = step_out(w0, P.L2, 0); w1 = step_out(w1, P.L2, 0); }
          char* base = static_cast<char*>(h->bscratch) + L.bs_off + ((st & 1) ? Sq.offX0 : Sq.offX1) * rb;
          const int rc2 = encode_map3(&M[(st - 1) * 4 + i], base, rb, w1.len, w0.len, L.ba.batch, (w1.len + 3) & ~3,
                                      L.ba.stride, BW, TI);
          if (rc2) return bail(PCWD_E_CUDA, "cuTensorMapEncodeTiled (approximation) failed: " + std::to_string(rc2));
        }
      }
    }
    if (!maps.empty()) {
      CKB(dalloc(&h->amaps_d, maps.size() * sizeof(CUtensorMap)));
      CKB(cudaMemcpy(h->amaps_d, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
      for (size_t i = 0; i < h->launches.size(); ++i)
        if (h->launches[i].batched && h->launches[i].ba.am_steps) h->launches[i].ba.amaps = h->amaps_d + first[i];
    }
  }
  if (h->kt_pc > 0) {   // v extended periodically by kt_pr rows and kt_pc columns: every k-sum v box is one TMA copy
    h->kt_offx = ((P.zhi[1] % 4) + 4) % 4;   // strip starts ≡ −zhi (mod 4) at levels ≥ 2: shift them onto 16 bytes
    h->kt_pc = (h->kt_pc + h->kt_offx + 31) / 32 * 32;
    const int H = P.n + h->kt_pr, W = P.n + h->kt_pc;
    CKB(dalloc(&h->vwrap_d, size_t(P.m) * H * W * rb));
    for (Launch& L : h->launches) {
      if (!L.batched || !L.ba.kt_gz) continue;
      const int SH = 1 << L.level, TR = 256 / SH, G = kt_units(rb), q0 = L.ba.kt_gz + G - 1;
      const int qV = kt_vbox_q(SH, q0, kt_vbox_n(SH, q0, rb), rb);
      const int rc2 = encode_map3(&L.ba.tmV, h->vwrap_d, rb, W, H, P.m, W, int64_t(W) * H, SH * qV + kt_vpadx(SH, rb), TR);
      if (rc2) return bail(PCWD_E_CUDA, "cuTensorMapEncodeTiled (k-sum v) failed: " + std::to_string(rc2));
      L.ba.kt_vh = H;
      L.ba.kt_vw = W;
      L.ba.kt_offx = h->kt_offx;
    }
  }
  // fine path: periodically padded v (K1) and the TMA descriptors of every fine launch
  bool any_fine = false;
  for (const Launch& L : h->launches) any_fine = any_fine || L.fine;
  if (any_fine) {
    const int W = P.n + 2 * h->vpad;
    CKB(dalloc(&h->vpad_d, size_t(P.m) * W * W * rb));   // filled by every decompose (pad_v_kernel)
    for (Launch& L : h->launches) {
      if (!L.fine) continue;
      int rc2 = encode_map3(&L.fa.tmV, h->vpad_d, rb, W, W, P.m, int64_t(W), int64_t(W) * W, L.box[2], L.box[0]);
      if (rc2) return bail(PCWD_E_CUDA, "cuTensorMapEncodeTiled (v) failed: " + std::to_string(rc2));
      L.fa.vpad = h->vpad;
      for (int q = L.fa.sb_first, i = 0; q < P.nsb && i < 3 && P.sb[q].level == L.level; ++q, ++i) {
        const SubBand& Sq = P.sb[q];
        rc2 = encode_map3(&L.fa.tmT[i], static_cast<char*>(h->T_d) + Sq.toff * rb, rb, Sq.tRS, Sq.tW[0], P.m, Sq.tRS,
                          Sq.tstride, L.box[1], L.box[0]);
        if (rc2) return bail(PCWD_E_CUDA, "cuTensorMapEncodeTiled (T) failed: " + std::to_string(rc2));
      }
    }
  }
  if (gmax > 0) CKB(dalloc(&h->gscratch, size_t(gmax) * rb));

  // output CSR
  const int64_t rows = h->rows();
  CKB(dalloc(&h->row_ptr, (rows + 1) * sizeof(int64_t)));
  if (P.retain == PCWD_RETAIN_BAND) {
    h->cap = h->nnz = rows * P.band_L;
  } else if (P.retain == PCWD_RETAIN_FULL) {
    h->cap = h->nnz = rows * P.N;
  } else if (P.retain == PCWD_RETAIN_PATTERN) {
    // the shard's rows of the caller's pattern: row pointers rebased to the shard, columns copied once
    const int64_t base = pat_rp[h->hp.row0];
    h->cap = h->nnz = pat_rp[h->hp.row1] - base;
    std::vector<int64_t> rp(rows + 1);
    for (int64_t i = 0; i <= rows; ++i) rp[i] = pat_rp[h->hp.row0 + i] - base;
    CKB(cudaMemcpy(h->row_ptr, rp.data(), (rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
  } else {
    CKB(dalloc(&h->unitmax, std::max<int64_t>(rows, 1) * sizeof(double)));
    CKB(dalloc(&h->cnt, std::max<int64_t>(rows * P.nsb, 1) * sizeof(int32_t)));
    CKB(dalloc(&h->rowcnt, (rows + 1) * sizeof(int64_t)));
    CKB(dalloc(&h->dmax, sizeof(double)));
    size_t tb = 0;
    CKB(exclusive_scan_i64(nullptr, nullptr, rows + 1, nullptr, &tb, 0));
    h->cubbytes = tb;
    CKB(dalloc(&h->cubtmp, tb));
    h->cap = 0;
    // store-then-filter buffer: if it does not fit, the count / write passes recompute
    if (h->hp.cand_total > 0 && !getenv("PCWD_NO_CAND")) {
      if (dalloc(&h->cand, size_t(h->hp.cand_total) * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        h->cand = nullptr;
      }
    }
  }
  if (h->cap > 0) {
    CKB(dalloc(&h->col, h->cap * sizeof(int32_t)));
    CKB(dalloc(&h->val, h->cap * ob));
  }
  if (P.retain == PCWD_RETAIN_PATTERN && h->nnz > 0)
    CKB(cudaMemcpy(h->col, pat_col.data() + pat_rp[h->hp.row0], h->nnz * sizeof(int32_t), cudaMemcpyHostToDevice));
  CKB(cudaDeviceSynchronize());
#undef CKB
  *out_handle = h;
  return PCWD_OK;
}

int pcwd_local_max(void* handle, void* stream, double* out_max) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h || !out_max) return fail(PCWD_E_PARAM, "NULL argument");
  if (h->hp.P.retain != PCWD_RETAIN_THRESHOLD) return fail(PCWD_E_STATE, "local_max needs THRESHOLD");
  CK(cudaSetDevice(h->desc.device));
  h->nlaunch = 0;
  return local_max_impl(h, static_cast<cudaStream_t>(stream), out_max);
}

int pcwd_set_global_max(void* handle, double M) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h) return fail(PCWD_E_PARAM, "NULL handle");
  if (!(M >= 0.0)) return fail(PCWD_E_PARAM, "M must be >= 0");
  h->M = M;
  h->M_set = true;
  return PCWD_OK;
}

int pcwd_decompose(void* handle, void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h) return fail(PCWD_E_PARAM, "NULL handle");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(h->desc.device));
  const Plan& P = h->hp.P;
  const int64_t rows = h->rows();
  int rc;
  if (P.retain != PCWD_RETAIN_THRESHOLD || !h->M_set) h->nlaunch = 0;
  h->tvalid = false;
  auto rec = [&](int i) { if (h->profile) cudaEventRecord(h->ev[i], st); };
  if (P.retain == PCWD_RETAIN_BAND) {
    rec(0);
    if (h->vpad_d) {   // periodically padded copy of v, the TMA source of the fine kernels
      CK(launch_pad_v(h->v_d, h->vpad_d, P.n, h->vpad, P.m, h->hp.real_bytes, st));
      h->nlaunch++;
    }
    if (h->vwrap_d) {  // periodic extension of v, the TMA source of the tiled coarse k-sums
      CK(launch_wrap_v(h->v_d, h->vwrap_d, P.n, 0, h->kt_offx, P.n + h->kt_pr, P.n + h->kt_pc, P.m, h->hp.real_bytes, st));
      h->nlaunch++;
    }
    if (h->tmpl_ready) h->tmpl_ready = false;   // built by pcwd_set_kernels beside v's copy (same u)
    else if ((rc = build_templates(h, st))) return rc;
    rec(1);
    if ((rc = run_units(h, MODE_BAND, st, 0.0))) return rc;
    rec(2);
    CK(launch_fill_band_rowptr(h->row_ptr, rows, P.band_L, st));
    h->nlaunch++;
    rec(3);
  } else if (P.retain == PCWD_RETAIN_PATTERN) {
    rec(0);
    if ((rc = build_templates(h, st))) return rc;
    rec(1);
    rec(2);
    if ((rc = run_units(h, MODE_PATTERN, st, 0.0))) return rc;
    rec(3);
  } else if (P.retain == PCWD_RETAIN_FULL) {
    rec(0);
    if ((rc = build_templates(h, st))) return rc;
    rec(1);
    CK(cudaMemsetAsync(h->val, 0, size_t(h->cap) * h->hp.out_bytes, st));
    CK(launch_fill_full(h->row_ptr, h->col, rows, P.N, st));
    h->nlaunch++;
    rec(2);
    if ((rc = run_units(h, MODE_FULL, st, 0.0))) return rc;
    rec(3);
  } else {
    if (!h->M_set) {
      if (h->desc.world > 1) return fail(PCWD_E_STATE, "THRESHOLD with world > 1 needs pcwd_set_global_max");
      double M = 0.0;
      if ((rc = local_max_impl(h, st, &M))) return rc;
      h->M = M;
    } else if (!h->tmpl_fresh) {
      if ((rc = build_templates(h, st))) return rc;
    }
    const double tau = h->desc.tau_rel * h->M;
    CK(cudaMemsetAsync(h->cnt, 0, size_t(std::max<int64_t>(rows * P.nsb, 1)) * sizeof(int32_t), st));
    // fp32 values: count and compact in one read of the candidates (the CSR copy follows the scan)
    static const bool no_compact = getenv("PCWD_NO_COMPACT") != nullptr;
    const bool compact = h->cand_valid && h->hp.out_bytes == 4 && !no_compact;
    if (compact) {
      CK(launch_cand_compact(P, static_cast<double*>(h->cand), h->hp.row0, rows, tau, h->cnt, st));
      h->nlaunch++;
      h->cand_valid = false;   // the buffer now holds the compacted rows (a failed decompose must recompute)
    } else if (h->cand_valid) {
      CK(launch_cand_filter(P, h->cand, h->hp.row0, rows, tau, 0, h->cnt, nullptr, nullptr, nullptr, h->hp.out_bytes, st));
      h->nlaunch++;
    } else if ((rc = run_units(h, MODE_TCOUNT, st, tau))) {
      return rc;
    }
    CK(launch_row_counts(h->cnt, rows, P.nsb, h->rowcnt, st));
    size_t tb = h->cubbytes;
    CK(exclusive_scan_i64(h->rowcnt, h->row_ptr, rows + 1, h->cubtmp, &tb, st));
    h->nlaunch += 2;
    int64_t nnz = 0;
    CK(cudaMemcpyAsync(&nnz, h->row_ptr + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (nnz > h->cap) {
      // free first (room for the larger CSR), with the handle left consistent (no CSR) if the allocation fails
      if (h->col) { cudaFree(h->col); h->col = nullptr; }
      if (h->val) { cudaFree(h->val); h->val = nullptr; }
      h->cap = 0;
      h->nnz = 0;
      h->decomposed = false;
      int32_t* ncol = nullptr;
      void* nval = nullptr;
      int64_t got = 0;
      auto grow = [&](int64_t c) {
        if (dalloc(&ncol, c * sizeof(int32_t)) != cudaSuccess) { cudaGetLastError(); ncol = nullptr; return false; }
        if (dalloc(&nval, c * h->hp.out_bytes) != cudaSuccess) {
          cudaGetLastError(); cudaFree(ncol); ncol = nullptr; nval = nullptr; return false;
        }
        got = c;
        return true;
      };
      bool ok = grow(nnz + nnz / 8 + 1024) || grow(nnz);
      if (!ok && h->cand && !compact) {
        // the store-then-filter buffer starves the CSR: drop it and write the rows by the recompute pass (not after
        // a compaction: the compacted rows live in that buffer)
        cudaFree(h->cand);
        h->cand = nullptr;
        h->cand_valid = false;
        ok = grow(nnz + nnz / 8 + 1024) || grow(nnz);
      }
      if (!ok) return fail(PCWD_E_OOM, "CSR of " + std::to_string(nnz) + " entries does not fit in device memory");
      h->col = ncol;
      h->val = nval;
      h->cap = got;
    }
    h->nnz = nnz;
    if (compact) {
      CK(launch_cand_copy(P, static_cast<const double*>(h->cand), h->hp.row0, rows, h->cnt, h->row_ptr, h->col,
                          static_cast<float*>(h->val), st));
      h->nlaunch++;
    } else if (h->cand_valid) {
      CK(launch_cand_filter(P, h->cand, h->hp.row0, rows, tau, 1, h->cnt, h->row_ptr, h->col, h->val,
                            h->hp.out_bytes, st));
      h->nlaunch++;
    } else if ((rc = run_units(h, MODE_TWRITE, st, tau))) {
      return rc;
    }
    h->M_set = false;
    h->tmpl_fresh = false;
    h->cand_valid = false;
  }
  h->decomposed = true;
  return PCWD_OK;
}

int pcwd_get_csr(void* handle, pcwd_csr* out) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h || !out) return fail(PCWD_E_PARAM, "NULL argument");
  if (!h->decomposed) return fail(PCWD_E_STATE, "decompose first");
  out->n_rows = h->rows();
  out->row0 = h->hp.row0;
  out->nnz = h->nnz;
  out->row_ptr = h->row_ptr;
  out->col = h->col;
  out->val = h->val;
  out->dtype = h->desc.dtype;
  return PCWD_OK;
}

int pcwd_copy_csr(void* handle, int64_t* row_ptr, int32_t* col, void* val, void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h) return fail(PCWD_E_PARAM, "NULL handle");
  if (!h->decomposed) return fail(PCWD_E_STATE, "decompose first");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(h->desc.device));
  if (row_ptr) CK(cudaMemcpyAsync(row_ptr, h->row_ptr, (h->rows() + 1) * sizeof(int64_t), cudaMemcpyDefault, st));
  if (col && h->nnz) CK(cudaMemcpyAsync(col, h->col, h->nnz * sizeof(int32_t), cudaMemcpyDefault, st));
  if (val && h->nnz) CK(cudaMemcpyAsync(val, h->val, h->nnz * h->hp.out_bytes, cudaMemcpyDefault, st));
  return PCWD_OK;
}

// pcwd_set_kernels / pcwd_set_kernels_box after the new u is staged (and checked) in h->ustage: swap it in, copy v
// (BAND: on a second stream beside the template build), invalidate the last decompose
static int set_kernels_finish(Handle* h, const double* v, cudaStream_t st, bool overlap) {
  const Plan& P = h->hp.P;
  const int64_t mN = int64_t(P.m) * P.N;
  const int rb = h->hp.real_bytes;
  std::swap(h->u_d, h->ustage);
  h->tmpl_ready = false;
  // v_d stays in place: the k-sum TMA maps hold its address
  cudaStream_t vs = st;
  if (overlap) {
    if (!h->cv) CK(cudaStreamCreateWithFlags(&h->cv, cudaStreamNonBlocking));
    vs = h->cv;
    CK(cudaMemcpyAsync(h->vstage, v, mN * sizeof(double), cudaMemcpyDefault, vs));
  }
  if (rb == 8) CK(cudaMemcpyAsync(h->v_d, h->vstage, mN * sizeof(double), cudaMemcpyDeviceToDevice, vs));
  else CK(launch_cast(static_cast<const double*>(h->vstage), h->v_d, mN, 4, vs));
  if (overlap) {
    if (int rc = build_templates(h, st)) return rc;
    CK(cudaStreamSynchronize(vs));   // the caller may release v on return
    CK(cudaStreamSynchronize(st));   // the templates are complete whatever stream the next decompose uses
    h->tmpl_ready = true;
  }
  h->M_set = false;
  h->tmpl_fresh = false;
  h->cand_valid = false;
  h->decomposed = false;
  return PCWD_OK;
}

int pcwd_set_kernels(void* handle, const double* u, const double* v, void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h || !u || !v) return fail(PCWD_E_PARAM, "NULL argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(h->desc.device));
  const Plan& P = h->hp.P;
  const int64_t mN = int64_t(P.m) * P.N;
  if (!h->ustage) CK(dalloc(&h->ustage, mN * sizeof(double)));
  if (!h->vstage) CK(dalloc(&h->vstage, mN * sizeof(double)));
  if (!h->flag_d) CK(dalloc(&h->flag_d, sizeof(int)));
  CK(cudaMemsetAsync(h->flag_d, 0, sizeof(int), st));
  CK(cudaMemcpyAsync(h->ustage, u, mN * sizeof(double), cudaMemcpyDefault, st));
  CK(launch_support_check(h->ustage, mN, P.n, P.d, P.zlo, P.zhi, h->flag_d, st));
  // BAND: v is copied on a second stream while the templates (which read only u) are built, so the next decompose
  // need not build them; other rules copy v behind u as before
  const bool overlap = P.retain == PCWD_RETAIN_BAND && !getenv("PCWD_NO_SETK_OVERLAP");
  if (!overlap) CK(cudaMemcpyAsync(h->vstage, v, mN * sizeof(double), cudaMemcpyDefault, st));
  int flag = 0;
  CK(cudaMemcpyAsync(&flag, h->flag_d, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (flag)
    return fail(PCWD_E_PARAM, "supp u_k leaves the periodic bounding box the plan was built for (create a new handle)");
  return set_kernels_finish(h, v, st, overlap);
}

int pcwd_kernel_box(void* handle, int32_t lo[2], int32_t w[2]) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h || !lo || !w) return fail(PCWD_E_PARAM, "NULL argument");
  const Plan& P = h->hp.P;
  lo[0] = P.d == 2 ? P.zlo[0] : 0;
  w[0] = P.d == 2 ? P.zhi[0] - P.zlo[0] + 1 : 1;
  lo[1] = P.zlo[1];
  w[1] = P.zhi[1] - P.zlo[1] + 1;
  return PCWD_OK;
}

int pcwd_set_kernels_box(void* handle, const double* u_box, const double* v, void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h || !u_box || !v) return fail(PCWD_E_PARAM, "NULL argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(h->desc.device));
  const Plan& P = h->hp.P;
  const int64_t mN = int64_t(P.m) * P.N;
  int32_t lo[2], w[2];
  pcwd_kernel_box(handle, lo, w);
  const int64_t nb = int64_t(P.m) * w[0] * w[1];
  if (!h->ustage) CK(dalloc(&h->ustage, mN * sizeof(double)));
  if (!h->vstage) CK(dalloc(&h->vstage, mN * sizeof(double)));
  if (h->ubox_cap < nb) {
    if (h->ubox) cudaFree(h->ubox);
    h->ubox = nullptr;
    h->ubox_cap = 0;
    CK(dalloc(&h->ubox, nb * sizeof(double)));
    h->ubox_cap = nb;
  }
  // the support is inside the box by construction: no check, no synchronisation before the template build
  const bool overlap = P.retain == PCWD_RETAIN_BAND && !getenv("PCWD_NO_SETK_OVERLAP");
  CK(cudaMemcpyAsync(h->ubox, u_box, nb * sizeof(double), cudaMemcpyDefault, st));
  CK(cudaMemsetAsync(h->ustage, 0, mN * sizeof(double), st));
  CK(launch_box_scatter(h->ubox, P.m, P.n, P.d, P.zlo, P.zhi, h->ustage, st));
  if (!overlap) CK(cudaMemcpyAsync(h->vstage, v, mN * sizeof(double), cudaMemcpyDefault, st));
  return set_kernels_finish(h, v, st, overlap);
}

int pcwd_decompose_to_host(void* handle, int64_t* row_ptr, int32_t* col, void* val, void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h) return fail(PCWD_E_PARAM, "NULL handle");
  CK(cudaSetDevice(h->desc.device));
  const Plan& P = h->hp.P;
  if (P.retain == PCWD_RETAIN_THRESHOLD || P.retain == PCWD_RETAIN_PATTERN) {   // rows of varying width
    int rc = pcwd_decompose(handle, stream);
    return rc ? rc : pcwd_copy_csr(handle, row_ptr, col, val, stream);
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!h->cs) CK(cudaStreamCreateWithFlags(&h->cs, cudaStreamNonBlocking));
  const Handle::Sink sk{P.retain == PCWD_RETAIN_BAND ? int64_t(P.band_L) : P.N, col, static_cast<char*>(val),
                        h->hp.out_bytes};
  h->sink = &sk;
  int rc = pcwd_decompose(handle, stream);
  h->sink = nullptr;
  if (rc) return rc;
  if (row_ptr) CK(cudaMemcpyAsync(row_ptr, h->row_ptr, (h->rows() + 1) * sizeof(int64_t), cudaMemcpyDefault, st));
  // join: `stream` waits for the last copy
  if (!h->cjoin) CK(cudaEventCreateWithFlags(&h->cjoin, cudaEventDisableTiming));
  CK(cudaEventRecord(h->cjoin, h->cs));
  CK(cudaStreamWaitEvent(st, h->cjoin, 0));
  return PCWD_OK;
}

// FISTA / transform scratch: 8 vectors of N compute-type elements + N + 1 doubles, 256-byte aligned slices
int fista_scratch(Handle* h, char** base, size_t* slice) {
  const int64_t N = h->hp.P.N;
  const size_t sl = (size_t(N) * h->hp.out_bytes + 255) & ~size_t(255);
  const size_t need = 8 * sl + ((size_t(N + 1 + kFistaParts) * 8 + 255) & ~size_t(255));
  if (h->fbuf_bytes < need) {
    if (h->fbuf) cudaFree(h->fbuf);
    h->fbuf = nullptr;
    h->fbuf_bytes = 0;
    CK(dalloc(&h->fbuf, need));
    h->fbuf_bytes = need;
  }
  *base = static_cast<char*>(h->fbuf);
  *slice = sl;
  return PCWD_OK;
}

// Θᵀ of the shard's CSR (deterministic order), built once per decompose
int ensure_transpose(Handle* h, cudaStream_t st) {
  if (h->tvalid) return PCWD_OK;
  const int64_t N = h->hp.P.N, nnz = h->nnz;
  const int vb = h->hp.out_bytes;
  if (nnz > h->tcap) {
    void* ptrs[] = {h->rpT, h->rowT, h->valT};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    h->rpT = nullptr; h->rowT = nullptr; h->valT = nullptr;
    h->tcap = -1;   // consistent if an allocation below fails
    const int64_t cap = std::max<int64_t>(nnz, 1);
    CK(dalloc(&h->rpT, (N + 1) * sizeof(int64_t)));
    CK(dalloc(&h->rowT, cap * sizeof(int32_t)));
    CK(dalloc(&h->valT, cap * vb));
    h->tcap = cap;
  }
  // the sort's work space only lives while the transpose is built (Θ̃ of pcwd_approx can have billions of entries)
  h->twork_bytes = csr_transpose_bytes(std::max<int64_t>(nnz, 1), N, vb) + ((N + 1) * 8 + 255);
  CK(dalloc(&h->twork, h->twork_bytes));
  const cudaError_t e = csr_transpose(h->row_ptr, h->col, h->val, h->rows(), nnz, N, vb, h->rpT, h->rowT, h->valT,
                                      h->twork, h->twork_bytes, st);
  const cudaError_t e2 = cudaStreamSynchronize(st);
  cudaFree(h->twork);
  h->twork = nullptr;
  h->twork_bytes = 0;
  CK(e);
  CK(e2);
  h->tvalid = true;
  return PCWD_OK;
}

int pcwd_wavelet_transform(void* handle, const void* in, void* out, int inverse, void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h || !in || !out) return fail(PCWD_E_PARAM, "NULL argument");
  if (in == out) return fail(PCWD_E_PARAM, "in and out must not alias");
  CK(cudaSetDevice(h->desc.device));
  char* base;
  size_t sl;
  if (int rc = fista_scratch(h, &base, &sl)) return rc;
  CK(launch_wavelet_transform(h->hp.P, in, out, base + 6 * sl, base + 7 * sl, inverse, h->hp.out_bytes,
                              static_cast<cudaStream_t>(stream)));
  return PCWD_OK;
}

static int fista_common(Handle* h, const void* z0, const void* w, int iters, int precond, double* tau, void* z_out,
                        int (*reduce)(int, void*), void* ctx, void* xg, double* xd, void* stream) {
  if (!h->decomposed) return fail(PCWD_E_STATE, "decompose first");
  if (iters < 0) return fail(PCWD_E_PARAM, "iters < 0");
  CK(cudaSetDevice(h->desc.device));
  char* base;
  size_t sl;
  if (int rc = fista_scratch(h, &base, &sl)) return rc;
  FistaArgs F{};
  F.N = h->hp.P.N;
  F.nnz = h->nnz;
  F.row_ptr = h->row_ptr;
  F.col = h->col;
  F.val = h->val;
  F.z0 = z0;
  F.w = w;
  F.y = base;
  F.zprev = base + sl;
  F.r = base + 2 * sl;
  F.g = xg ? xg : base + 3 * sl;
  F.sigma = base + 4 * sl;
  F.sqrt_sigma = base + 5 * sl;
  F.D = xd ? xd : reinterpret_cast<double*>(base + 8 * sl);
  F.dbuf = reinterpret_cast<double*>(base + 8 * sl) + F.N;
  F.z_out = z_out;
  if (int rc = ensure_transpose(h, static_cast<cudaStream_t>(stream))) return rc;
  F.row_ptrT = h->rpT;
  F.rowT = h->rowT;
  F.valT = h->valT;
  F.iters = iters;
  F.precond = precond ? 1 : 0;
  F.power_iters = 100;   // at most; stops earlier when ‖M v‖ settles (relative change < 1e-6 over 8 iterations)
  F.rows = h->rows();
  F.row0 = h->hp.row0;
  F.reduce = reduce;
  F.rctx = ctx;
  int cb_failed = 0;
  const cudaError_t e = launch_fista(h->hp.P, F, h->hp.out_bytes, static_cast<cudaStream_t>(stream), tau, &cb_failed);
  if (cb_failed) return fail(PCWD_E_PARAM, "the reduce callback failed");
  CK(e);
  return PCWD_OK;
}

int pcwd_fista(void* handle, const void* z0, const void* w, int iters, int precond, double* tau, void* z_out,
               void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h || !z0 || !w || !z_out || !tau) return fail(PCWD_E_PARAM, "NULL argument");
  if (h->decomposed && h->rows() != h->hp.P.N)
    return fail(PCWD_E_STATE, "FISTA needs the whole Θ on one handle (world = 1); use pcwd_fista_sharded");
  return fista_common(h, z0, w, iters, precond, tau, z_out, nullptr, nullptr, nullptr, nullptr, stream);
}

int pcwd_fista_sharded(void* handle, const void* z0, const void* w, int iters, int precond, double* tau, void* z_out,
                       pcwd_reduce_fn reduce, void* ctx, void* xg, double* xd, void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h || !z0 || !w || !z_out || !tau || !reduce || !xg || (precond && !xd)) return fail(PCWD_E_PARAM, "NULL argument");
  return fista_common(h, z0, w, iters, precond, tau, z_out, reduce, ctx, xg, xd, stream);
}

int pcwd_apply(void* handle, const void* x, void* y, int transpose, void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h || !x || !y) return fail(PCWD_E_PARAM, "NULL argument");
  if (!h->decomposed) return fail(PCWD_E_STATE, "decompose first");
  CK(cudaSetDevice(h->desc.device));
  if (transpose) {   // Θᵀ x as a gather over the transposed CSR (deterministic)
    if (int rc = ensure_transpose(h, static_cast<cudaStream_t>(stream))) return rc;
    CK(launch_spmv(h->rpT, h->rowT, h->valT, x, y, h->hp.P.N, h->rows(), 0, h->hp.out_bytes,
                   static_cast<cudaStream_t>(stream)));
  } else {
    CK(launch_spmv(h->row_ptr, h->col, h->val, x, y, h->rows(), h->hp.P.N, 0, h->hp.out_bytes,
                   static_cast<cudaStream_t>(stream)));
  }
  return PCWD_OK;
}

int pcwd_operator_apply(void* handle, const void* x, void* y, int adjoint, void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h || !x || !y) return fail(PCWD_E_PARAM, "NULL argument");
  if (x == y) return fail(PCWD_E_PARAM, "x and y must not alias");
  CK(cudaSetDevice(h->desc.device));
  CK(launch_operator(h->hp.P, h->u_d, h->v_d, x, y, adjoint, h->hp.real_bytes, static_cast<cudaStream_t>(stream)));
  return PCWD_OK;
}

int pcwd_columns(void* handle, const int64_t* lambdas, int64_t count, double* out, void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h || (count > 0 && (!lambdas || !out))) return fail(PCWD_E_PARAM, "NULL argument");
  if (count < 0) return fail(PCWD_E_PARAM, "count < 0");
  if (count == 0) return PCWD_OK;
  CK(cudaSetDevice(h->desc.device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Plan& P = h->hp.P;
  std::vector<int64_t> lh(count);
  CK(cudaMemcpy(lh.data(), lambdas, count * sizeof(int64_t), cudaMemcpyDefault));
  for (int64_t i = 0; i < count; ++i)
    if (lh[i] < 0 || lh[i] >= P.N) return fail(PCWD_E_PARAM, "lambda index out of range");
  const int64_t cstride = (3 + int64_t(P.m)) * P.N;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->desc.device);
  const int64_t budget = int64_t(4) << 30;   // scratch: at most 4 GiB of CTA slices
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>({count, int64_t(nsm) * 2, budget / (cstride * 8)})));
  struct B { double* s = nullptr; int64_t* l = nullptr; ~B() { cudaFree(s); cudaFree(l); } } b;
  CK(dalloc(&b.s, size_t(grid) * cstride * sizeof(double)));
  CK(dalloc(&b.l, count * sizeof(int64_t)));
  CK(cudaMemcpyAsync(b.l, lh.data(), count * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  CK(launch_columns(P, h->u_d, h->v_d, b.l, count, b.s, cstride, grid, out, h->hp.real_bytes, st));
  CK(cudaStreamSynchronize(st));
  return PCWD_OK;
}

// ---- constructing the product-convolution expansion (pca.cu) ---------------------------------------------------
static int pc_common(int d, int n, int R, int m, int64_t s, const double* X, int g, int oversample, int power_iters,
                     uint64_t seed, double* u, double* v, double* sigma, cudaStream_t st) {
  if (!X || !u || !v || !sigma) return fail(PCWD_E_PARAM, "NULL argument");
  if (d != 1 && d != 2) return fail(PCWD_E_SHAPE, "d must be 1 or 2");
  if (n < 2 || (n & (n - 1))) return fail(PCWD_E_SHAPE, "n must be a power of two >= 2");
  if (R < 0 || 2 * R + 1 > n) return fail(PCWD_E_PARAM, "window 2R+1 must fit the torus");
  const int W = d == 2 ? (2 * R + 1) * (2 * R + 1) : 2 * R + 1;
  if (m < 1 || m > W || m > s || m + std::max(oversample, 0) > 32)
    return fail(PCWD_E_PARAM, "need 1 <= m <= min(W, samples) and m + oversample <= 32");
  if (power_iters < 1) return fail(PCWD_E_PARAM, "power_iters must be >= 1");
  const bool dev = is_device_ptr(X);
  double *Xd = nullptr, *U = nullptr, *c = nullptr;
  struct F { double** p[3]; bool own; ~F() { if (own && *p[0]) cudaFree(*p[0]); cudaFree(*p[1]); cudaFree(*p[2]); } } fr{{&Xd, &U, &c}, !dev};
  if (dev) Xd = const_cast<double*>(X);
  else {
    CK(dalloc(&Xd, sizeof(double) * s * W));
    CK(cudaMemcpyAsync(Xd, X, sizeof(double) * s * W, cudaMemcpyHostToDevice, st));
  }
  CK(dalloc(&U, sizeof(double) * W * m));
  CK(dalloc(&c, sizeof(double) * s * m));
  int rc = pcwd_pca::factor(Xd, s, W, m, oversample, power_iters, seed, U, c, sigma, st);
  if (rc) return fail(rc, "factorisation failed");
  rc = pcwd_pca::finish(U, c, d, n, R, g, m, u, v, st);
  if (rc) return fail(rc, "embedding / interpolation failed");
  CK(cudaStreamSynchronize(st));
  return PCWD_OK;
}

int pcwd_pc_from_samples(int32_t d, int32_t n, int32_t R, int32_t g, int32_t m, const double* irs, double* u,
                         double* v, double* sigma, void* stream) {
  if (g < 1 || g > n) return fail(PCWD_E_PARAM, "g must be in [1, n]");
  const int64_t s = d == 2 ? int64_t(g) * g : g;
  return pc_common(d, n, R, m, s, irs, g, 8, 24, 0x5eed5eedULL, u, v, sigma, static_cast<cudaStream_t>(stream));
}

int pcwd_pc_from_svir(int32_t d, int32_t n, int32_t R, int32_t m, const double* svir, int32_t oversample,
                      int32_t power_iters, uint64_t seed, double* u, double* v, double* sigma, void* stream) {
  const int64_t s = d == 2 ? int64_t(n) * n : n;
  return pc_common(d, n, R, m, s, svir, n, oversample, power_iters, seed, u, v, sigma,
                   static_cast<cudaStream_t>(stream));
}

int pcwd_rows3d(int32_t n, int32_t levels, const double* h, int32_t taps, int32_t m, const double* u, const double* v,
                const int64_t* units, int64_t count, double* out, void* stream) {
  if (n < 2 || n > 256 || (n & (n - 1))) return fail(PCWD_E_SHAPE, "pcwd_rows3d: n must be a power of two in [2, 256]");
  int lg = 0;
  while ((1 << lg) < n) ++lg;
  if (levels < 1 || levels > lg) return fail(PCWD_E_CONFIG, "pcwd_rows3d: levels must be in [1, log2 n]");
  if (taps < 2 || taps > kMaxTaps || (taps & 1)) return fail(PCWD_E_CONFIG, "pcwd_rows3d: taps must be even, 2..20");
  if (!h || !u || !v || m < 1 || count < 0 || (count > 0 && (!units || !out))) return fail(PCWD_E_PARAM, "pcwd_rows3d: NULL argument or m < 1");
  double s1 = 0.0;   // an orthogonal wavelet filter, as pcwd_validate checks it
  for (int i = 0; i < taps; ++i) s1 += h[i];
  if (std::fabs(s1 - std::sqrt(2.0)) > 1e-9) return fail(PCWD_E_CONFIG, "pcwd_rows3d: h must sum to sqrt(2)");
  for (int k = 0; 2 * k < taps; ++k) {
    double a = 0.0;
    for (int i = 0; i + 2 * k < taps; ++i) a += h[i] * h[i + 2 * k];
    if (std::fabs(a - (k == 0 ? 1.0 : 0.0)) > 1e-9) return fail(PCWD_E_CONFIG, "pcwd_rows3d: h is not an orthogonal wavelet filter");
  }
  if (!is_device_ptr(u) || !is_device_ptr(v) || (count > 0 && !is_device_ptr(out)))
    return fail(PCWD_E_PARAM, "pcwd_rows3d: u, v and out must be device pointers");
  const int64_t N = int64_t(n) * n * n;
  std::vector<int64_t> uh(count);
  if (count > 0) CK(cudaMemcpy(uh.data(), units, count * sizeof(int64_t), cudaMemcpyDefault));
  for (int64_t i = 0; i < count; ++i)
    if (uh[i] < 0 || uh[i] >= N) return fail(PCWD_E_PARAM, "pcwd_rows3d: unit index out of range");
  if (count == 0) return PCWD_OK;
  // coarse units (low Λ indices: the widest supports) first, the CTAs take units from a counter as they finish
  std::vector<int64_t> order(count);
  for (int64_t i = 0; i < count; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return uh[a] < uh[b]; });
  std::vector<int64_t> sorted_mu(count);
  for (int64_t i = 0; i < count; ++i) sorted_mu[i] = uh[order[i]];
  uh.insert(uh.end(), order.begin(), order.end());
  int64_t* ud = nullptr;
  CK(cudaMalloc(&ud, 2 * count * sizeof(int64_t)));
  cudaError_t e = cudaMemcpy(ud, uh.data(), 2 * count * sizeof(int64_t), cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaError_t(pcwd_vol::rows3d(n, levels, h, taps, m, u, v, ud, ud + count, sorted_mu.data(), count, out,
                                     static_cast<cudaStream_t>(stream)));
  cudaFree(ud);
  if (e != cudaSuccess)
    return fail(e == cudaErrorMemoryAllocation ? PCWD_E_OOM : PCWD_E_CUDA, std::string("pcwd_rows3d: ") + cudaGetErrorString(e));
  return PCWD_OK;
}

int pcwd_approx(void* handle, double eta, int rule, void* stream, pcwd_approx_info* out) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h) return fail(PCWD_E_PARAM, "NULL handle");
  if (!(eta > 0.0)) return fail(PCWD_E_PARAM, "eta must be > 0");
  if (rule != PCWD_TRUNC_INDEX && rule != PCWD_TRUNC_MAGNITUDE) return fail(PCWD_E_PARAM, "rule");
  const Plan& P = h->hp.P;
  if (h->hp.real_bytes != 8) return fail(PCWD_E_UNSUPPORTED, "pcwd_approx computes in fp64: create the handle with dtype F64");
  if (h->desc.world != 1) return fail(PCWD_E_STATE, "pcwd_approx needs world = 1");
  if (P.m > 64) return fail(PCWD_E_UNSUPPORTED, "pcwd_approx supports m <= 64");
  CK(cudaSetDevice(h->desc.device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t N = P.N;
  const int bins = approx_bins();
  // classes: (sub-band, position mod 2^{J-ℓ}) in sub-band order
  ApproxArgs A{};
  int64_t nc = 0;
  for (int s = 0; s < P.nsb; ++s) {
    A.clsbase[s] = nc;
    const int64_t M = int64_t(1) << (P.J - P.sb[s].level);
    nc += P.d == 2 ? M * M : M;
  }
  A.clsbase[P.nsb] = nc;
  A.ncls = nc;
  A.rule = rule;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->desc.device);
  const int grid = int(std::min<int64_t>(nc, int64_t(nsm) * 2));
  A.cstride = (5 + int64_t(P.m)) * N;
  struct Bufs {
    double *scratch = nullptr, *rowh = nullptr, *colh = nullptr;
    int64_t* cnt = nullptr;
    ~Bufs() { cudaFree(scratch); cudaFree(rowh); cudaFree(colh); cudaFree(cnt); }
  } B;
  CK(dalloc(&B.scratch, size_t(grid) * A.cstride * sizeof(double)));
  CK(dalloc(&B.rowh, size_t(nc) * P.m * bins * sizeof(double)));
  CK(dalloc(&B.colh, size_t(nc) * P.m * bins * sizeof(double)));
  CK(dalloc(&B.cnt, size_t(N) * sizeof(int64_t)));
  CK(cudaMemsetAsync(B.colh, 0, size_t(nc) * P.m * bins * sizeof(double), st));
  if (int rc = build_templates(h, st)) return rc;
  A.T = static_cast<const double*>(h->T_d);
  A.v = static_cast<const double*>(h->v_d);
  A.scratch = B.scratch;
  A.rowhist = B.rowh;
  A.colhist = B.colh;
  A.cnt = B.cnt;
  // pass 0: |A_k| by truncation index (row and column sums of every class)
  CK(launch_approx_stats(P, A, grid, st));
  std::vector<double> rowh(size_t(nc) * P.m * bins), colh(size_t(nc) * P.m * bins), vh(size_t(P.m) * N);
  CK(cudaMemcpyAsync(rowh.data(), B.rowh, rowh.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(colh.data(), B.colh, colh.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(vh.data(), h->v_d, vh.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  pcwd_approx_info info{};
  info.eta = eta;
  info.m = P.m;
  for (int k = 0; k < P.m; ++k) {
    double vinf = 0.0;
    for (int64_t i = 0; i < N; ++i) vinf = std::max(vinf, std::fabs(vh[size_t(k) * N + i]));
    const double eps = vinf > 0.0 ? eta / (P.m * vinf) : HUGE_VAL;
    // dropped part at index S: entries with S_keep > S; its max row / column abs sums over the classes
    int smax = -1;
    for (int64_t c = 0; c < nc; ++c)
      for (int b = 0; b < bins; ++b)
        if (rowh[(size_t(c) * P.m + k) * bins + b] > 0.0) smax = std::max(smax, b);
    int Sk = smax;
    double bk = 0.0;
    for (int S = -1; S <= smax; ++S) {
      double mr = 0.0, mc = 0.0;
      for (int64_t c = 0; c < nc; ++c) {
        double r = 0.0, q = 0.0;
        for (int b = S + 1; b < bins; ++b) {
          r += rowh[(size_t(c) * P.m + k) * bins + b];
          q += colh[(size_t(c) * P.m + k) * bins + b];
        }
        mr = std::max(mr, r);
        mc = std::max(mc, q);
      }
      const double bound = std::sqrt(mr * mc);
      if (bound <= eps) { Sk = S; bk = bound; break; }
    }
    A.S[k] = Sk;
    info.S[k] = Sk;
    info.eps[k] = eps;
    info.bound[k] = bk;
  }
  // pass 1: nonzeros per row of Θ̃; host scan; pass 2: write
  CK(launch_approx_rows(P, A, 0, 8, grid, st));
  std::vector<int64_t> cnt(N), rp(N + 1, 0);
  CK(cudaMemcpyAsync(cnt.data(), B.cnt, N * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < N; ++i) rp[i + 1] = rp[i] + cnt[i];
  const int64_t nnz = rp[N];
  if (nnz > h->cap) {
    if (h->col) { cudaFree(h->col); h->col = nullptr; }
    if (h->val) { cudaFree(h->val); h->val = nullptr; }
    h->cap = 0;
    h->nnz = 0;
    h->decomposed = false;
    CK(dalloc(&h->col, std::max<int64_t>(nnz, 1) * sizeof(int32_t)));
    if (dalloc(&h->val, std::max<int64_t>(nnz, 1) * h->hp.out_bytes) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(h->col);
      h->col = nullptr;
      return fail(PCWD_E_OOM, "CSR of Θ̃ does not fit in device memory");
    }
    h->cap = nnz;
  }
  CK(cudaMemcpyAsync(h->row_ptr, rp.data(), (N + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  A.row_ptr = h->row_ptr;
  A.col = h->col;
  A.val = h->val;
  CK(launch_approx_rows(P, A, 1, h->hp.out_bytes, grid, st));
  CK(cudaStreamSynchronize(st));
  h->nnz = nnz;
  h->decomposed = true;
  h->tvalid = false;
  h->M_set = false;
  h->cand_valid = false;
  info.nnz = nnz;
  if (out) *out = info;
  return PCWD_OK;
}

int pcwd_info(void* handle, pcwd_info_t* out) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h || !out) return fail(PCWD_E_PARAM, "NULL argument");
  const Plan& P = h->hp.P;
  out->N = P.N;
  out->row0 = h->hp.row0;
  out->row1 = h->hp.row1;
  out->nnz = h->nnz;
  out->global_max = h->M;
  out->fma_algorithmic = h->hp.fma_shard;
  const int rb = h->hp.real_bytes;
  out->bytes_algorithmic = double(P.m) * P.N * rb + double(h->hp.tmpl_elems) * rb +
                           double(h->nnz) * (4 + h->hp.out_bytes) + double(h->rows() + 1) * 8;
  out->kernel_launches = h->nlaunch;
  out->compute_dtype = rb == 8 ? PCWD_F64 : PCWD_F32;
  return PCWD_OK;
}

int pcwd_profile(void* handle, int enable) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h) return fail(PCWD_E_PARAM, "NULL handle");
  CK(cudaSetDevice(h->desc.device));
  if (enable && !h->ev[0])
    for (auto& e : h->ev) CK(cudaEventCreate(&e));
  h->profile = enable != 0;
  h->profile_serial = enable == 2;
  return PCWD_OK;
}

int pcwd_phase_times(void* handle, double* out_ms, double* out_fma) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h || !out_ms || !out_fma) return fail(PCWD_E_PARAM, "NULL argument");
  if (!h->profile || h->hp.P.retain == PCWD_RETAIN_THRESHOLD)
    return fail(PCWD_E_STATE, "profiling not enabled (or THRESHOLD: not instrumented)");
  float t[3] = {0, 0, 0};
  CK(cudaEventElapsedTime(&t[0], h->ev[0], h->ev[1]));
  if (h->hp.P.retain == PCWD_RETAIN_BAND || h->hp.P.retain == PCWD_RETAIN_PATTERN) {
    CK(cudaEventElapsedTime(&t[1], h->ev[1], h->ev[2]));
    CK(cudaEventElapsedTime(&t[2], h->ev[2], h->ev[3]));
  } else {
    CK(cudaEventElapsedTime(&t[2], h->ev[1], h->ev[2]));
    CK(cudaEventElapsedTime(&t[1], h->ev[2], h->ev[3]));
  }
  for (int i = 0; i < 3; ++i) out_ms[i] = t[i];
  out_fma[0] = h->hp.fma_templates;
  out_fma[1] = h->hp.fma_shard - h->hp.fma_templates;
  out_fma[2] = 0.0;
  return PCWD_OK;
}

int pcwd_launch_profile(void* handle, int max, int* count, double* out_ms, double* out_fma, int* out_kind,
                        int* out_level) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h || !count) return fail(PCWD_E_PARAM, "NULL argument");
  if (!h->profile || h->lev.size() < 2 * h->launches.size())
    return fail(PCWD_E_STATE, "profiling not enabled before the last decompose");
  CK(cudaSetDevice(h->desc.device));
  const int n = int(h->launches.size());
  *count = n;
  for (int i = 0; i < n && i < max; ++i) {
    const Launch& L = h->launches[i];
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->lev[2 * i], h->lev[2 * i + 1]));
    if (out_ms) out_ms[i] = ms;
    if (out_fma) out_fma[i] = units_fma(h->hp.P, L.u0, L.u1);
    if (out_kind) out_kind[i] = L.fine ? 2 : L.tile ? 1 : L.batched ? 3 : 0;
    if (out_level) out_level[i] = h->hp.P.sb[find_subband(h->hp.P, L.u0)].level;
  }
  return PCWD_OK;
}

int pcwd_destroy(void* handle) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h) return PCWD_OK;
  cudaSetDevice(h->desc.device);
  for (auto& e : h->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : h->lev)
    if (e) cudaEventDestroy(e);
  free_all(h);
  delete h;
  return PCWD_OK;
}

}  // extern "C"
