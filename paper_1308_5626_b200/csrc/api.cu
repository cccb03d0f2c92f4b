// api.cu -- the C ABI of libpspgmres (include/pspgmres.h): context, workspace plan, and the
// host control flow of Algorithm 1, Algorithm 2 and the time-step
// driver (Eq.3-4).  Every numeric step runs in the kernels of stencil.cu,
// krylov.cu, mrep.cu and banded.cu; the host only sequences launches and reads the O(1)
// scalars the control flow branches on (beta, R(k), flags, gate decision).
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "internal.h"

using namespace psp;

namespace {
// NVTX ranges around the host API (header-only NVTX3: free unless a profiler is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

struct psp_ctx {
  // configuration
  psp_grid grid{};
  int d = 1, nA = 30;
  double tol = 1e-8, dt = 0.0;
  psp_opts opts{};
  cudaStream_t stream = nullptr;
  psp_comm* comm = nullptr;
  int64_t n = 0, row0 = 0;
  int64_t n_global = 0;
  Stencil st{};
  // multi-rank (slab decomposition along the slowest axis)
  bool multi = false;
  int nranks = 1, rank = 0;
  int64_t plane = 1;             // rows per slab unit (halo size of the stencil)
  double* hx_lo = nullptr;       // halo planes of the matvec input (received per matvec)
  double* hx_hi = nullptr;
  double* hf_lo = nullptr;       // halo planes of the coefficient field (received at create)
  double* hf_hi = nullptr;
  double* mh_send = nullptr;     // MREP halo rows: [lo|hi] x m_max x d, packed for the send
  double* mh_recv = nullptr;     //   and received ([lo|hi] x m_max x d)
  double* bmisc = nullptr;       // banded multi-rank scratch (maps, states)
  // f2: the device-resident solve's scratch (resident.cu)
  double* res_out = nullptr;     // 16-double summary
  unsigned long long* res_bar = nullptr;
  double* res_part = nullptr;
  double* res_hist = nullptr;
  double* res_beta = nullptr;
  int res_hist_cap = 0, res_beta_cap = 0;
  // f3: streaming MREP -- the lagged sums of every probe recorded since the last fit (mrep.cu)
  double* ssums = nullptr;       // (4d+4) x n
  int scount = 0;
  // workspace carve
  double* ring_px = nullptr;      // column starts, ldr apart
  double* ring_py = nullptr;
  int64_t ldr = 0;               // ring column stride: n, or n + 2 planes (multi-rank ghost planes)
  int64_t goff = 0;              // the owned rows start goff into a column (a ghost plane when multi)
  double* Wbase = nullptr;       // W's column start (W = Wbase + goff)
  double* kpad = nullptr;        // multi-rank: the coefficient field with its ghost planes
  double* slot_scale = nullptr;  // per physical slot: the recorded probe is scale * column
  int ring_cap = 0, ring_count = 0, ring_head = 0;
  int ring_phys = 0;             // ring_cap + 1: the slot after the newest is always free
  // fused Arnoldi cycle (N = I): V(:,j) lives in ring slot vslot[j] (unnormalised)
  bool cycle_fused = false;
  int vslot[kMaxRestart + 2] = {};
  double* V = nullptr;
  int64_t ldv = 0;
  double* X0 = nullptr;
  double* B = nullptr;
  double* W = nullptr;
  double* bands = nullptr;
  double* lu = nullptr;
  double* intercept = nullptr;
  uint8_t* rowkind = nullptr;
  double* kappa = nullptr;
  bool n_identity = true;
  DevState ds{};
  RedCfg rc{};
  MrepScratch ms{};
  BandedScratch bs{};
  // host
  double* hp = nullptr;  // pinned scalars
  std::string err;
  psp_status sticky = PSP_OK;
  int64_t launches = 0;
  int last_k = 0;
  int combined_k = 0;      // the last step of this ring cycle already formed X0 + Z0, Z1 (krylov.cu)
  int combined_slot = -1;  // ring slot whose P_x / P_y columns hold them
  cudaEvent_t ev[6] = {};
  // multi-rank matvec: the halo exchange runs on a side stream beside the slab's interior planes
  cudaStream_t hstream = nullptr;
  cudaEvent_t hev[2] = {};
  // per-kernel-class event timing (opts.timing >= 2)
  struct KRec {
    int klass;
    double bytes;
    int ev;
  };
  std::vector<cudaEvent_t> kev;
  std::vector<KRec> krec;
  int kev_used = 0;
  double kms[PSP_KC_COUNT] = {};
  double kbytes[PSP_KC_COUNT] = {};
  int64_t kcount[PSP_KC_COUNT] = {};
};

namespace {
void kt_flush(psp_ctx* c) {
  if (c->krec.empty()) return;
  cudaStreamSynchronize(c->stream);
  for (const auto& r : c->krec) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->kev[r.ev], c->kev[r.ev + 1]);
    c->kms[r.klass] += ms;
    c->kbytes[r.klass] += r.bytes;
    c->kcount[r.klass] += 1;
  }
  c->krec.clear();
  c->kev_used = 0;
}
// returns a handle (or -1 when timing is off); pair with kt_end after the launch(es)
int kt_begin(psp_ctx* c) {
  if (c->opts.timing < 2) return -1;
  // the event pool grows (it is reused after every flush): no synchronisation in the middle of
  // a timed region; psp_kernel_stats flushes
  while ((int)c->kev.size() < c->kev_used + 2) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->kev.push_back(e);
  }
  const int h = c->kev_used;
  c->kev_used += 2;
  cudaEventRecord(c->kev[h], c->stream);
  return h;
}
void kt_end(psp_ctx* c, int h, int klass, double bytes) {
  if (h < 0) return;
  cudaEventRecord(c->kev[h + 1], c->stream);
  c->krec.push_back({klass, bytes, h});
}
// algorithmic bytes of one matvec: x (+ field or DIA bands) read, y written (+ probe copy)
double matvec_bytes(const psp_ctx* c, bool copy) {
  double per = 16.0;
  if (c->st.kind == PSP_OP_CELL_DIFF || c->st.kind == PSP_OP_CELL_ADVDIFF) per += 8.0;
  if (c->st.kind == PSP_OP_DIA) per += 8.0 * (2 * c->st.dA + 1);
  if (copy) per += 8.0;
  return per * (double)c->n;
}
}  // namespace

static std::string g_err;

namespace psp {
std::string cuda_err_str(cudaError_t e) { return std::string(cudaGetErrorName(e)) + ": " + cudaGetErrorString(e); }
int device_ordinal() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) dev = 0;
  return dev < kMaxDev ? dev : kMaxDev - 1;
}
int device_sms() {
  static std::atomic<int> sms[kMaxDev];
  const int dev = device_ordinal();
  int v = sms[dev].load(std::memory_order_relaxed);
  if (v <= 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    sms[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}
}  // namespace psp

static psp_status fail(psp_ctx* c, psp_status s, const std::string& msg) {
  if (c) c->err = msg;
  g_err = msg;
  return s;
}

static psp_status check_cuda(psp_ctx* c, const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    if (c) c->sticky = PSP_E_CUDA;
    return fail(c, PSP_E_CUDA, std::string(where) + ": " + cuda_err_str(e));
  }
  return PSP_OK;
}

#define PSP_TRY(expr)                 \
  do {                                \
    psp_status _s = (expr);           \
    if (_s != PSP_OK) return _s;      \
  } while (0)

// ------------------------------------------------------------------------------------------
// Workspace plan
// ------------------------------------------------------------------------------------------
namespace {

struct Plan {
  size_t off_px, off_py, off_V, off_X0, off_B, off_W, off_bands, off_lu, off_icpt, off_kind,
      off_kappa, off_H, off_Hraw, off_G, off_C, off_S, off_Q, off_Lm, off_alpha, off_scal, off_resid,
      off_sscale, off_halo, off_rpart, off_mhalo, off_bmisc,
      off_partials, off_tickets, off_mpart, off_mtick, off_mres, off_banded, off_res, off_rhist, off_rbeta,
      off_ssums, off_kpad, total;
  int hist_cap, beta_cap;
  int nblocks;
};

int sm_count() { return device_sms(); }

Plan make_plan(int64_t n, int d, int nA, int m_max, int max_cycles, int64_t plane = 1, int nranks = 1,
               int mrep_stream = 0) {
  Plan p{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o += (bytes + 255) & ~(size_t)255;
    return at;
  };
  const size_t vec = (size_t)n * 8;
  p.nblocks = 8 * sm_count();
  // multi-rank: every ring column (and W) carries a ghost plane below / above the slab (the
  // neighbours' boundary planes), so the fused passes run on slabs (fused.cu, FusedLayout)
  const size_t gvec = (size_t)(n + (nranks > 1 ? 2 * plane : 0)) * 8;
  p.off_px = take(gvec * (m_max + 1));  // m_max probes + the free slot (fused path)
  p.off_py = take(gvec * (m_max + 1));
  p.off_sscale = take((size_t)(m_max + 1) * 8);
  p.off_V = take(vec * (nA + 1));
  p.off_X0 = take(vec);
  p.off_B = take(vec);
  p.off_W = take(gvec);
  p.off_kpad = nranks > 1 ? take(gvec) : 0;
  p.off_bands = take(vec * (2 * d + 1));
  p.off_lu = take(vec * (2 * d + 1));
  p.off_icpt = p.off_kind = p.off_kappa = 0;   // (diagnostics: psp_mrep_fit_raw only)
  const size_t hs = (size_t)(nA + 1) * nA * 8;
  p.off_H = take(hs);
  p.off_Hraw = take(hs);
  p.off_G = take((size_t)(nA + 1) * 8);
  p.off_C = take((size_t)nA * 8);
  p.off_S = take((size_t)nA * 8);
  p.off_Q = take((size_t)nA * 8);
  p.off_Lm = take((size_t)(nA + 1) * (nA + 1) * 8);
  p.off_alpha = take((size_t)(nA + 1) * 8);
  p.off_scal = take(SC_NSCAL * 8);
  p.off_resid = take((size_t)nA * 8);
  p.off_partials = take((size_t)2 * kMaxRestart * p.nblocks * 8);
  p.off_tickets = take(TK_N * 4);
  p.off_mpart = take((size_t)6 * kMrepMaxBlocks * 8);
  p.off_mtick = take(64);
  p.off_mres = take(16 * 8);
  p.off_banded = take(banded_scratch_bytes(n, d));
  p.off_halo = take((size_t)4 * plane * 8);
  p.off_rpart = take((size_t)(2 * kMaxRestart + 16) * 8);
  p.off_mhalo = take((size_t)4 * (m_max + 1) * d * 8);
  p.off_bmisc = take(banded_misc_doubles(d, nranks) * 8);
  // f2 (resident.cu): barrier word + summary, double-buffered grid partials, R(k) / beta history
  p.off_res = take(256 + resident_scratch_doubles(nA, sm_count()) * 8);
  const int64_t hc = (int64_t)nA * max_cycles;
  p.hist_cap = (int)(hc < ((int64_t)1 << 22) ? hc : ((int64_t)1 << 22));
  p.beta_cap = max_cycles;
  p.off_rhist = take((size_t)p.hist_cap * 8);
  p.off_rbeta = take((size_t)p.beta_cap * 8);
  p.off_ssums = mrep_stream ? take((size_t)(4 * d + 4) * (size_t)n * 8) : o;   // f3
  p.total = o + 256;  // alignment slack for the base pointer
  return p;
}

int64_t grid_rows(const psp_grid* g) {
  int64_t r = 1;
  for (int a = 0; a < g->ndim; ++a) r *= g->n[a];
  return r;
}

psp_status validate(const psp_grid* grid, const psp_stencil* st, int d, int restart, const psp_opts* o) {
  if (!grid || !st) return fail(nullptr, PSP_E_ARG, "grid/stencil is NULL");
  if (grid->ndim < 1 || grid->ndim > 3) return fail(nullptr, PSP_E_DIM, "ndim must be 1..3");
  for (int a = 0; a < grid->ndim; ++a)
    if (grid->n[a] < 1) return fail(nullptr, PSP_E_DIM, "grid extent < 1");
  if (st->kind < PSP_OP_CONST_DIFF || st->kind > PSP_OP_DIA) return fail(nullptr, PSP_E_ARG, "bad stencil kind");
  if ((st->kind == PSP_OP_CELL_DIFF || st->kind == PSP_OP_CELL_ADVDIFF) && !st->d_field)
    return fail(nullptr, PSP_E_ARG, "cell operator needs d_field");
  if (st->kind == PSP_OP_DIA && (!st->d_bands || st->dA < 0)) return fail(nullptr, PSP_E_ARG, "DIA operator needs d_bands");
  if (st->kind == PSP_OP_CELL_ADVDIFF)
    for (int a = 0; a < 3; ++a)
      if (st->c[a] < 0) return fail(nullptr, PSP_E_ARG, "upwind velocity must be >= 0 (v1)");
  if (d < 1 || d > kMaxD) return fail(nullptr, PSP_E_ARG, "d must be 1..4");
  if (restart < 1 || restart > kMaxRestart) return fail(nullptr, PSP_E_ARG, "restart must be 1..128");
  if (o) {
    if (o->m_max < 1 || o->m_max > 256) return fail(nullptr, PSP_E_ARG, "m_max must be 1..256");
    if (o->max_cycles < 1) return fail(nullptr, PSP_E_ARG, "max_cycles must be >= 1");
  }
  if (grid_rows(grid) < 2 * d + 1) return fail(nullptr, PSP_E_DIM, "n < 2d+1 (S:207)");
  return PSP_OK;
}

}  // namespace

// ------------------------------------------------------------------------------------------
extern "C" {

void psp_default_opts(psp_opts* o) {
  memset(o, 0, sizeof(*o));
  o->max_cycles = 1000;
  o->tol_mode = PSP_TOL_REL_B;
  o->m_max = 64;
  o->reset_history_per_step = 0;
  o->ortho = PSP_MGS_1REDUCE;
  o->gate = 1;
  o->timing = 0;
  o->fused = 1;
  o->fused_kmin = 2;
  o->fused_kmax = 16;
  o->fused_split_cols = 16;
  o->resident = 1;
}

const char* psp_version(void) { return "libpspgmres 0.1 (sm_100a, FP64)"; }

const char* psp_status_str(psp_status s) {
  switch (s) {
    case PSP_OK: return "ok";
    case PSP_E_ARG: return "bad argument";
    case PSP_E_DIM: return "dimension mismatch";
    case PSP_E_SAMPLES: return "insufficient samples (m < 2d+2)";
    case PSP_E_RANK: return "rank deficient";
    case PSP_E_SINGULAR: return "singular";
    case PSP_E_NONFINITE: return "non-finite value";
    case PSP_E_NOCONV: return "not converged";
    case PSP_E_CUDA: return "CUDA error";
    case PSP_E_NCCL: return "NCCL error";
    case PSP_E_NOMEM: return "workspace too small";
  }
  return "unknown";
}

const char* psp_last_error(const psp_ctx* c) { return c ? c->err.c_str() : g_err.c_str(); }

// Slab decomposition: contiguous blocks of the slowest axis (z for 3-D, y for
// 2-D, the index for 1-D), balanced to within one plane; the global lexicographic row order is
// kept, so rank r owns rows [row0, row0 + nrows).
psp_status psp_partition(const psp_grid* grid, int nranks, int rank, int64_t* row0, int64_t* nrows,
                         int64_t* slab0, int64_t* slab_len) {
  if (!grid || grid->ndim < 1 || grid->ndim > 3 || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(nullptr, PSP_E_ARG, "psp_partition: bad argument");
  const int ax = grid->ndim - 1;
  const int64_t N = grid->n[ax];
  if (N < nranks) return fail(nullptr, PSP_E_DIM, "psp_partition: fewer planes than ranks");
  int64_t plane = 1;
  for (int a = 0; a < ax; ++a) plane *= grid->n[a];
  const int64_t base = N / nranks, rem = N % nranks;
  const int64_t s0 = rank * base + (rank < rem ? rank : rem);
  const int64_t len = base + (rank < rem ? 1 : 0);
  if (row0) *row0 = s0 * plane;
  if (nrows) *nrows = len * plane;
  if (slab0) *slab0 = s0;
  if (slab_len) *slab_len = len;
  return PSP_OK;
}

static psp_status local_layout(const psp_grid* grid, const psp_stencil* st, int d, const psp_comm* comm,
                               int64_t* n_loc, int64_t* row0, int64_t* slab0, int64_t* slab_len,
                               int64_t* plane) {
  const int nr = comm ? comm->nranks : 1, rk = comm ? comm->rank : 0;
  PSP_TRY(psp_partition(grid, nr, rk, row0, n_loc, slab0, slab_len));
  *plane = *n_loc / *slab_len;
  if (nr > 1) {
    if (st->kind == PSP_OP_DIA) return fail(nullptr, PSP_E_ARG, "multi-rank: DIA operators are single-rank only");
    if (*n_loc < 2 * d + 1) return fail(nullptr, PSP_E_DIM, "multi-rank: each rank needs >= 2d+1 rows");
  }
  return PSP_OK;
}

psp_status psp_workspace_bytes(const psp_grid* grid, const psp_stencil* st, int d, int restart,
                               const psp_opts* opts, const psp_comm* comm, size_t* bytes) {
  psp_opts o;
  if (opts) o = *opts; else psp_default_opts(&o);
  PSP_TRY(validate(grid, st, d, restart, &o));
  int64_t n_loc, row0, s0, sl, plane;
  PSP_TRY(local_layout(grid, st, d, comm, &n_loc, &row0, &s0, &sl, &plane));
  Plan p = make_plan(n_loc, d, restart, o.m_max, o.max_cycles, plane, comm ? comm->nranks : 1, o.mrep_stream);
  *bytes = p.total;
  return PSP_OK;
}

psp_status psp_create(const psp_grid* grid, const psp_stencil* st, double dt, int d, int restart,
                      double tol, const psp_opts* opts, void* d_ws, size_t ws_bytes, void* stream,
                      psp_comm* comm, psp_ctx** out) {
  if (!out) return fail(nullptr, PSP_E_ARG, "out is NULL");
  *out = nullptr;
  psp_opts o;
  if (opts) o = *opts; else psp_default_opts(&o);
  PSP_TRY(validate(grid, st, d, restart, &o));
  if (!(tol > 0.0) || !(dt >= 0.0)) return fail(nullptr, PSP_E_ARG, "tol must be > 0 and dt >= 0");
  if (o.method != PSP_METHOD_GMRES && o.method != PSP_METHOD_CG) return fail(nullptr, PSP_E_ARG, "bad method");
  if (o.mrep_stream && comm && comm->nranks > 1)
    return fail(nullptr, PSP_E_ARG, "streaming MREP is single-rank");
  if (o.method == PSP_METHOD_CG && comm && comm->nranks > 1)
    return fail(nullptr, PSP_E_ARG, "PSP-CG is single-rank (the symmetric part of N needs the neighbours' rows)");
  int64_t n, row0, slab0, slab_len, plane;
  PSP_TRY(local_layout(grid, st, d, comm, &n, &row0, &slab0, &slab_len, &plane));
  const int nranks = comm ? comm->nranks : 1;
  Plan p = make_plan(n, d, restart, o.m_max, o.max_cycles, plane, nranks, o.mrep_stream);
  if (!d_ws || ws_bytes < p.total) return fail(nullptr, PSP_E_NOMEM, "workspace smaller than psp_workspace_bytes");

  psp_ctx* c = new psp_ctx();
  c->grid = *grid;
  c->d = d;
  c->nA = restart;
  c->tol = tol;
  c->dt = dt;
  c->opts = o;
  c->stream = (cudaStream_t)stream;
  c->comm = comm;
  c->n = n;
  c->row0 = row0;
  c->n_global = grid_rows(grid);
  c->nranks = nranks;
  c->rank = comm ? comm->rank : 0;
  c->multi = nranks > 1;
  c->plane = plane;
  // operator coefficients (R24): h_a = 1/(n_a+1) of the GLOBAL grid; local extents per slab
  Stencil& S = c->st;
  S.kind = st->kind;
  S.ndim = grid->ndim;
  S.nx = grid->n[0];
  S.ny = grid->ndim >= 2 ? grid->n[1] : 1;
  S.nz = grid->ndim >= 3 ? grid->n[2] : 1;
  if (grid->ndim == 3) S.nz = slab_len;
  else if (grid->ndim == 2) S.ny = slab_len;
  else S.nx = slab_len;
  S.n = n;
  for (int a = 0; a < 3; ++a) {
    const double na = a < grid->ndim ? (double)grid->n[a] : 1.0;
    const double h = 1.0 / (na + 1.0);
    const double coef = (st->kind == PSP_OP_CONST_DIFF) ? st->nu : 1.0;
    S.s[a] = a < grid->ndim ? dt * coef / (h * h) : 0.0;
    S.a[a] = (a < grid->ndim && st->kind == PSP_OP_CELL_ADVDIFF) ? dt * st->c[a] / h : 0.0;
  }
  S.field = st->d_field;
  S.dA = st->dA;
  S.bands = st->d_bands;
  S.x_lo = S.x_hi = S.f_lo = S.f_hi = nullptr;

  char* base = (char*)(((uintptr_t)d_ws + 255) & ~(uintptr_t)255);
  auto at = [&](size_t off) { return base + off; };
  c->ring_px = (double*)at(p.off_px);
  c->ring_py = (double*)at(p.off_py);
  c->goff = c->multi ? plane : 0;
  c->ldr = n + 2 * c->goff;
  c->ring_cap = o.m_max;
  c->ring_phys = o.m_max + 1;
  c->slot_scale = (double*)at(p.off_sscale);
  c->V = (double*)at(p.off_V);
  c->ldv = n;
  c->X0 = (double*)at(p.off_X0);
  c->B = (double*)at(p.off_B);
  c->Wbase = (double*)at(p.off_W);
  c->W = c->Wbase + c->goff;
  c->kpad = c->multi ? (double*)at(p.off_kpad) : nullptr;
  c->bands = (double*)at(p.off_bands);
  c->lu = (double*)at(p.off_lu);
  c->intercept = nullptr;
  c->rowkind = nullptr;
  c->kappa = nullptr;
  c->ds.H = (double*)at(p.off_H);
  c->ds.Hraw = (double*)at(p.off_Hraw);
  c->ds.G = (double*)at(p.off_G);
  c->ds.C = (double*)at(p.off_C);
  c->ds.S = (double*)at(p.off_S);
  c->ds.Q = (double*)at(p.off_Q);
  c->ds.Lm = (double*)at(p.off_Lm);
  c->ds.alpha = (double*)at(p.off_alpha);
  c->ds.scal = (double*)at(p.off_scal);
  c->ds.resid = (double*)at(p.off_resid);
  c->ds.partials = (double*)at(p.off_partials);
  c->ds.tickets = (unsigned*)at(p.off_tickets);
  c->ds.rpart = (double*)at(p.off_rpart);
  c->ds.slot_scale = c->slot_scale;
  c->ds.multi = c->multi ? 1 : 0;
  c->rc.nblocks = p.nblocks;
  c->rc.max_vals = 2 * kMaxRestart;
  c->ms.partials = (double*)at(p.off_mpart);
  c->ms.ticket = (unsigned*)at(p.off_mtick);
  c->ms.result = (double*)at(p.off_mres);
  // the split MREP's lagged-sum rows live in the Krylov basis storage (unused in ring mode, and
  // free between solves in split mode: psp_mrep_fit runs after the solve, Alg.2 / P:30)
  if (4 * c->d + 4 <= c->nA + 1) {
    c->ms.sums = c->V;
    c->ms.sums_n = c->ldv;
  }
  c->bs = banded_scratch(at(p.off_banded), n, d);
  c->hx_lo = (double*)at(p.off_halo);
  c->hx_hi = c->hx_lo + plane;
  c->hf_lo = c->hx_hi + plane;
  c->hf_hi = c->hf_lo + plane;
  c->mh_send = (double*)at(p.off_mhalo);
  c->mh_recv = c->mh_send + 2 * (size_t)(o.m_max + 1) * d;
  c->bmisc = (double*)at(p.off_bmisc);
  c->res_bar = (unsigned long long*)at(p.off_res);
  c->res_out = (double*)at(p.off_res + 64);
  c->res_part = (double*)at(p.off_res + 256);
  c->res_hist = (double*)at(p.off_rhist);
  c->res_beta = (double*)at(p.off_rbeta);
  c->res_hist_cap = p.hist_cap;
  c->res_beta_cap = p.beta_cap;
  c->ssums = o.mrep_stream ? (double*)at(p.off_ssums) : nullptr;
  // zero the small control state (tickets, epochs, Hessenberg)
  cudaMemsetAsync(at(p.off_H), 0, p.off_partials - p.off_H, c->stream);
  cudaMemsetAsync(at(p.off_tickets), 0, TK_N * 4, c->stream);
  cudaMemsetAsync(at(p.off_mtick), 0, 64, c->stream);
  cudaMemsetAsync(at(p.off_banded), 0, banded_scratch_bytes(n, d), c->stream);
  cudaMemsetAsync(at(p.off_halo), 0, (size_t)4 * plane * 8, c->stream);
  if (cudaMallocHost((void**)&c->hp, 64 * sizeof(double)) != cudaSuccess) {
    delete c;
    return fail(nullptr, PSP_E_CUDA, "cudaMallocHost failed");
  }
  memset(c->hp, 0, 64 * sizeof(double));
  c->hp[32] = 1.0;  // the pinned constant 1.0 (scale of probes recorded normalised)
  for (int i = 0; i < 6; ++i) cudaEventCreate(&c->ev[i]);
  if (c->multi) {
    cudaStreamCreateWithFlags(&c->hstream, cudaStreamNonBlocking);
    for (int i = 0; i < 2; ++i) cudaEventCreateWithFlags(&c->hev[i], cudaEventDisableTiming);
  }
  // multi-rank: the coefficient field's halo planes, once (the field is fixed per context)
  if (c->multi && S.field) {
    if (comm->sendrecv(S.field, c->hf_lo, plane, S.field + (n - plane), c->hf_hi, plane, c->stream)) {
      cudaFreeHost(c->hp);
      delete c;
      return fail(nullptr, PSP_E_NCCL, "psp_create: field halo exchange failed");
    }
    S.f_lo = c->rank > 0 ? c->hf_lo : nullptr;
    S.f_hi = c->rank < nranks - 1 ? c->hf_hi : nullptr;
  }
  if (c->multi) {
    // ghost planes: zero (the Dirichlet value at the global boundary) until a neighbour fills them
    for (int q = 0; q <= o.m_max; ++q) {
      for (double* base : {c->ring_px, c->ring_py}) {
        double* col = base + (int64_t)q * c->ldr;
        cudaMemsetAsync(col, 0, (size_t)plane * 8, c->stream);
        cudaMemsetAsync(col + plane + n, 0, (size_t)plane * 8, c->stream);
      }
    }
    cudaMemsetAsync(c->Wbase, 0, (size_t)c->ldr * 8, c->stream);
    cudaMemsetAsync(c->kpad, 0, (size_t)c->ldr * 8, c->stream);
    if (S.field) {                                 // [kappa ghost below | kappa | kappa ghost above]
      cudaMemcpyAsync(c->kpad + plane, S.field, (size_t)n * 8, cudaMemcpyDeviceToDevice, c->stream);
      if (S.f_lo) cudaMemcpyAsync(c->kpad, S.f_lo, (size_t)plane * 8, cudaMemcpyDeviceToDevice, c->stream);
      if (S.f_hi) cudaMemcpyAsync(c->kpad + plane + n, S.f_hi, (size_t)plane * 8, cudaMemcpyDeviceToDevice, c->stream);
    }
  }
  psp_status s = check_cuda(c, "psp_create");
  if (s != PSP_OK) {
    cudaFreeHost(c->hp);
    delete c;
    return s;
  }
  *out = c;
  return PSP_OK;
}

psp_status psp_destroy(psp_ctx* c) {
  if (!c) return PSP_OK;
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (int i = 0; i < 6; ++i)
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  for (int i = 0; i < 2; ++i)
    if (c->hev[i]) cudaEventDestroy(c->hev[i]);
  if (c->hstream) cudaStreamDestroy(c->hstream);
  for (auto e : c->kev) cudaEventDestroy(e);
  if (c->hp) cudaFreeHost(c->hp);
  delete c;
  return PSP_OK;
}

psp_status psp_local_rows(const psp_ctx* c, int64_t* row0, int64_t* nrows) {
  if (!c) return PSP_E_ARG;
  if (row0) *row0 = c->row0;
  if (nrows) *nrows = c->n;
  return PSP_OK;
}

psp_status psp_launch_count(const psp_ctx* c, int64_t* l) {
  if (!c || !l) return PSP_E_ARG;
  *l = c->launches;
  return PSP_OK;
}

psp_status psp_set_timing(psp_ctx* c, int level) {
  if (!c) return PSP_E_ARG;
  if (level < 0 || level > 2) return fail(c, PSP_E_ARG, "psp_set_timing: level must be 0, 1 or 2");
  c->opts.timing = level;
  return PSP_OK;
}

psp_status psp_kernel_stats(psp_ctx* c, double* ms, double* bytes, int64_t* launches, int reset) {
  if (!c) return PSP_E_ARG;
  kt_flush(c);
  for (int k = 0; k < PSP_KC_COUNT; ++k) {
    if (ms) ms[k] = c->kms[k];
    if (bytes) bytes[k] = c->kbytes[k];
    if (launches) launches[k] = c->kcount[k];
    if (reset) {
      c->kms[k] = 0.0;
      c->kbytes[k] = 0.0;
      c->kcount[k] = 0;
    }
  }
  return PSP_OK;
}

const char* psp_kernel_class_name(int k) {
  static const char* names[PSP_KC_COUNT] = {"matvec", "precond_solve", "ortho_dots", "ortho_update",
                                            "mgs_literal", "normalize", "combine", "residual",
                                            "mrep_fit", "banded_factor", "other", "arnoldi_fused",
                                            "resident_solve", "cg"};
  return (k >= 0 && k < PSP_KC_COUNT) ? names[k] : "?";
}

}  // extern "C"

// ------------------------------------------------------------------------------------------
// internal steps
// ------------------------------------------------------------------------------------------
namespace {

// The probe ring (FIFO of capacity m_max, R20) over m_max+1 physical slots: the slot after the
// newest probe is always free, so a fused pass can write the next probe before it is known
// whether it will be recorded (a cycle may converge first).
int ring_peek(const psp_ctx* c) { return (c->ring_head + c->ring_count) % c->ring_phys; }
// record a probe column: returns its slot (the free slot), evicting the oldest when full
int ring_next(psp_ctx* c) {
  const int slot = ring_peek(c);
  if (c->ring_count < c->ring_cap) c->ring_count += 1;
  else c->ring_head = (c->ring_head + 1) % c->ring_phys;
  return slot;
}
int ring_slot(const psp_ctx* c, int q) { return (c->ring_head + q) % c->ring_phys; }  // q-th oldest
double* px_col(psp_ctx* c, int slot) { return c->ring_px + (int64_t)slot * c->ldr + c->goff; }
double* py_col(psp_ctx* c, int slot) { return c->ring_py + (int64_t)slot * c->ldr + c->goff; }
// f3: the probe just recorded in `slot` (its data and scale final in stream order) joins the
// streaming MREP's lagged sums
void stream_add(psp_ctx* c, int slot) {
  if (!c->ssums) return;
  launch_mrep_accumulate(px_col(c, slot), py_col(c, slot), c->slot_scale, slot,
                         c->n, c->d, c->ssums, c->n, c->scount == 0 ? 1 : 0, c->stream);
  c->scount += 1;
  c->launches += 1;
}
double* Vcol(psp_ctx* c, int j /*1-based*/) { return c->V + (int64_t)(j - 1) * c->ldv; }
// a probe recorded normalised (scale 1)
void set_unit_scale(psp_ctx* c, int slot) {
  cudaMemcpyAsync(c->slot_scale + slot, c->hp + 32, sizeof(double), cudaMemcpyHostToDevice, c->stream);
}
// the Krylov basis of the current cycle
Basis basis(const psp_ctx* c) {
  if (c->cycle_fused) return Basis{c->ring_px + c->goff, c->ldr, c->vslot[1], c->ring_phys};
  return Basis{c->V, c->ldv, 0, c->nA + 1};
}
// a ring-resident cycle: the Krylov basis lives in the probe ring (single rank: the fused pass
// would need the halo planes of u in the middle of the pass)
bool fused_eligible(const psp_ctx* c) {
  // multi-rank: the ring columns carry ghost planes (exchanged after every pass), so the fused
  // passes run on slabs; 1-D grids shard along x, which the fused pass does not march
  return c->opts.fused && c->n_identity && c->opts.ortho == PSP_MGS_1REDUCE && c->ring_cap >= c->nA + 1 &&
         (!c->multi || c->grid.ndim >= 2);
}

// multi-rank ring steps: the boundary planes of a freshly written column go to the neighbours'
// ghost planes (one plane each way); no-op on one rank
psp_status ghost_exchange(psp_ctx* c, double* col /* owned start */) {
  if (!c->multi) return PSP_OK;
  const int64_t pl = c->plane;
  if (c->comm->sendrecv(col, col - pl, (size_t)pl, col + c->n - pl, col + c->n, (size_t)pl, c->stream))
    return fail(c, PSP_E_NCCL, "ghost plane exchange failed");
  return PSP_OK;
}
FusedLayout flayout(const psp_ctx* c) {
  FusedLayout l;
  l.ld = c->ldr;
  l.zoff = c->multi ? 1 : 0;
  l.lo_in = c->multi && c->rank > 0;
  l.hi_in = c->multi && c->rank < c->nranks - 1;
  l.field = c->multi ? c->kpad : c->st.field;
  return l;
}

// y = A (xs x) [+ probe copy]; multi-rank: first the slab halo planes of x from rank-1 / rank+1
// planes [p0, p0 + cnt) of this rank's slab as a stencil of their own: the planes just outside
// are local data or the received halo (lo / hi), so the march kernels treat them as halo planes
static Stencil slab_part(const psp_ctx* c, int64_t p0, int64_t cnt, const double* x, const double* lo,
                         const double* hi) {
  Stencil v = c->st;
  const int64_t pl = c->plane, nzl = c->n / pl;
  if (v.ndim == 3) v.nz = cnt;
  else v.ny = cnt;
  v.n = cnt * pl;
  v.field = c->st.field ? c->st.field + p0 * pl : nullptr;
  v.x_lo = p0 > 0 ? x + (p0 - 1) * pl : lo;
  v.x_hi = p0 + cnt < nzl ? x + (p0 + cnt) * pl : hi;
  v.f_lo = c->st.field ? (p0 > 0 ? c->st.field + (p0 - 1) * pl : c->st.f_lo) : nullptr;
  v.f_hi = c->st.field ? (p0 + cnt < nzl ? c->st.field + (p0 + cnt) * pl : c->st.f_hi) : nullptr;
  return v;
}

// y = A (xs x) [+ probe copy].  Multi-rank: the halo planes of x from rank-1 / rank+1 (NCCL
// send/recv) travel on a side stream while the slab's interior planes [1, nz-1) -- whose
// neighbour planes are all local -- are computed; the two boundary planes follow the exchange.
psp_status matvec(psp_ctx* c, const double* x, const double* xs, double* y, double* xcopy) {
  Stencil st = c->st;
  if (c->multi) {
    const int64_t pl = c->plane, nzl = c->n / pl;
    const double* lo = c->rank > 0 ? c->hx_lo : nullptr;
    const double* hi = c->rank < c->nranks - 1 ? c->hx_hi : nullptr;
    if (nzl >= 3 && st.ndim >= 2 && st.kind != PSP_OP_DIA) {
      cudaEventRecord(c->hev[0], c->stream);               // x is ready
      const int64_t off = pl;                              // the interior planes (enqueued first: a
      launch_matvec(slab_part(c, 1, nzl - 2, x, lo, hi), x + off, xs, y + off,   // host-mediated exchange
                    xcopy ? xcopy + off : nullptr, c->stream);                   // blocks the host thread)
      cudaStreamWaitEvent(c->hstream, c->hev[0], 0);
      if (c->comm->sendrecv(x, c->hx_lo, (size_t)pl, x + (c->n - pl), c->hx_hi, (size_t)pl, c->hstream))
        return fail(c, PSP_E_NCCL, "matvec halo exchange failed");
      cudaEventRecord(c->hev[1], c->hstream);
      cudaStreamWaitEvent(c->stream, c->hev[1], 0);       // then the two boundary planes
      launch_matvec(slab_part(c, 0, 1, x, lo, hi), x, xs, y, xcopy, c->stream);
      const int64_t last = (nzl - 1) * pl;
      launch_matvec(slab_part(c, nzl - 1, 1, x, lo, hi), x + last, xs, y + last, xcopy ? xcopy + last : nullptr,
                    c->stream);
      c->launches += 3;
      return PSP_OK;
    }
    if (c->comm->sendrecv(x, c->hx_lo, (size_t)pl, x + (c->n - pl), c->hx_hi, (size_t)pl, c->stream))
      return fail(c, PSP_E_NCCL, "matvec halo exchange failed");
    st.x_lo = lo;
    st.x_hi = hi;
  }
  launch_matvec(st, x, xs, y, xcopy, c->stream);
  c->launches += 1;
  return PSP_OK;
}

// multi-rank: all-reduce this rank's reduction totals, then run the scalar epilogue on every
// rank (identical inputs -> identical decisions on every rank)
psp_status finish_reduce(psp_ctx* c, int kind, int nv, int k, int j, int slot) {
  if (!c->multi) return PSP_OK;
  if (c->comm->allreduce(c->ds.rpart, (size_t)nv, 0, c->stream))
    return fail(c, PSP_E_NCCL, "all-reduce failed");
  launch_epilogue(kind, c->ds, k, c->nA, j, slot, c->stream);
  c->launches += 1;
  return PSP_OK;
}

psp_status sync_read(psp_ctx* c, const double* dsrc, int count, double* hdst) {
  cudaMemcpyAsync(c->hp, dsrc, count * sizeof(double), cudaMemcpyDeviceToHost, c->stream);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    c->sticky = PSP_E_CUDA;
    return fail(c, PSP_E_CUDA, "stream sync: " + cuda_err_str(e));
  }
  PSP_TRY(check_cuda(c, "sync_read"));
  memcpy(hdst, c->hp, count * sizeof(double));
  return PSP_OK;
}

psp_status set_eps(psp_ctx* c, const double* d_b, double* eps_out) {
  double eps;
  if (c->opts.tol_mode == PSP_TOL_ABS) {
    eps = c->tol;
  } else {
    launch_norm(d_b, c->n, c->ds, SC_NORM, c->rc, c->stream);
    c->launches += 1;
    PSP_TRY(finish_reduce(c, EPI_NORM, 1, 0, 0, SC_NORM));
    double nb;
    PSP_TRY(sync_read(c, c->ds.scal + SC_NORM, 1, &nb));
    eps = c->tol * nb;  // R1
  }
  c->hp[8] = eps;
  cudaMemcpyAsync(c->ds.scal + SC_EPS, c->hp + 8, sizeof(double), cudaMemcpyHostToDevice, c->stream);
  cudaStreamSynchronize(c->stream);
  *eps_out = eps;
  return check_cuda(c, "set_eps");
}

// z = x0 + N^{-1} (vs v) with the accepted N (banded LU of K4), multi-rank aware
psp_status precond_scaled(psp_ctx* c, const double* v, const double* vs, double* z, const double* x0 = nullptr) {
  if (banded_solve(c->lu, c->n, c->d, v, vs, x0, z, c->bs, c->stream, &c->launches, c->multi ? c->comm : nullptr,
                   c->bmisc))
    return fail(c, PSP_E_NCCL, "banded solve: collective failed");
  return PSP_OK;
}

psp_status precond(psp_ctx* c, const double* v, const double* x0, double* z) {
  if (c->n_identity) {
    if (x0) return fail(c, PSP_E_ARG, "internal: identity precond with addend");
    launch_copy(v, z, c->n, c->stream);
    c->launches += 1;
    return PSP_OK;
  }
  return precond_scaled(c, v, nullptr, z, x0);
}

}  // namespace

extern "C" {

psp_status psp_matvec(psp_ctx* c, const double* x, double* y, int record) {
  if (!c || !x || !y) return fail(c, PSP_E_ARG, "psp_matvec: NULL argument");
  if (c->sticky != PSP_OK) return c->sticky;
  if (record) {
    const int slot = ring_next(c);
    set_unit_scale(c, slot);
    PSP_TRY(matvec(c, x, nullptr, py_col(c, slot), px_col(c, slot)));
    stream_add(c, slot);
    launch_copy(py_col(c, slot), y, c->n, c->stream);
    c->launches += 1;
  } else {
    PSP_TRY(matvec(c, x, nullptr, y, nullptr));
  }
  return check_cuda(c, "psp_matvec");
}

psp_status psp_precond_apply(psp_ctx* c, const double* v, double* z) {
  if (!c || !v || !z) return fail(c, PSP_E_ARG, "psp_precond_apply: NULL argument");
  if (c->sticky != PSP_OK) return c->sticky;
  PSP_TRY(precond(c, v, nullptr, z));
  return check_cuda(c, "psp_precond_apply");
}

// step k of a ring-resident cycle as one fused pass (update + matvec + dots) or as separate
// passes: the policy of opts.fused_kmin / fused_kmax
// the fused kernels pay per tile plane, not per byte, below a few million rows (C2, 512^2: a
// step 9.9 ms with split passes, 45 ms fused; C3, 2048^2: 336 -> 292 ms fused): opts.fused = 1
// uses them from kFusedMinRows rows on, opts.fused = 2 always (the parity tests' small cases)
constexpr int64_t kFusedMinRows = (int64_t)1 << 21;
static bool fused_big(const psp_ctx* c) { return c->opts.fused >= 2 || c->n >= kFusedMinRows; }

static bool fused_pass(const psp_ctx* c, int k) {
  // (the pass streams k basis columns: the restart length itself may exceed the fused kernel's 32)
  return fused_big(c) && k >= c->opts.fused_kmin && k <= c->opts.fused_kmax && fused_supported(c->st, k);
}

static double fused_bytes(const psp_ctx* c, int k);

// split-column step: a step wider than the fused band whose newest fused_split_cols basis columns
// go through the fused pass and the older J = k - fused_split_cols through an update and a dots
// pass (both stream those columns once each, with no stencil halo)
static bool hyb_pass(const psp_ctx* c, int k) {
  const int kb = c->opts.fused_split_cols;
  return fused_big(c) && kb > 0 && kb <= 16 && k > c->opts.fused_kmax && k - kb >= 1 && fused_supported(c->st, kb);
}

// Step k as three passes over the ring: [A] u' = alpha_k w~_k - sum_{j<J} h_j alpha_j V(:,j) into
// the scratch vector W (l.13-16, the first J MGS terms); [B] the fused pass over the columns
// [J, k): u = u' - sum_{J<=j<k} h_j alpha_j V(:,j) -> V(:,k+1) (the next slot), w~_{k+1} = A u
// (l.11-12) and their inner products with those columns, u and w~; [C] the inner products of
// V(:,0..J-1) with w~_{k+1} and u, then H(k+1,k), Givens, alpha_{k+1} (l.17-32) and step k+1's
// MGS coefficients (R11) in its last block.
static psp_status ring_hyb_step(psp_ctx* c, int k, int src_slot, int dst) {
  const int64_t n = c->n;
  const double dn = (double)n;
  const int kb = c->opts.fused_split_cols, J = k - kb;
  int h = kt_begin(c);
  launch_icwy_update(basis(c), py_col(c, src_slot), c->ds.alpha + (k - 1), c->W, k, c->nA, n, c->ds, c->rc,
                     c->stream, J);
  kt_end(c, h, PSP_KC_ORTHO_UPDATE, 8.0 * (J + 2) * dn);
  PSP_TRY(ghost_exchange(c, c->W));                 // multi-rank: u' on the ghost planes
  h = kt_begin(c);
  const int fe = launch_fused(c->st, c->ring_px, c->ring_py, c->vslot[1], c->ring_phys, k, c->nA, src_slot, 0,
                              px_col(c, dst), py_col(c, dst), c->slot_scale, dst, c->ds, c->stream, flayout(c), J,
                              c->Wbase);
  if (fe) return fail(c, PSP_E_CUDA, "fused pass: " + fused_error(fe));
  kt_end(c, h, PSP_KC_FUSED, fused_bytes(c, kb));
  if (c->multi) {
    if (c->comm->allreduce(c->ds.rpart + kHybOff, (size_t)(2 * kb + 2), 0, c->stream))
      return fail(c, PSP_E_NCCL, "all-reduce failed");
    PSP_TRY(ghost_exchange(c, px_col(c, dst)));
    PSP_TRY(ghost_exchange(c, py_col(c, dst)));
  }
  h = kt_begin(c);
  launch_icwy_dots_hyb(basis(c), py_col(c, dst), px_col(c, dst), J, k, c->nA, n, c->ds, c->rc, c->stream);
  PSP_TRY(finish_reduce(c, EPI_HYB, 2 * J + 1, k, J, 0));
  kt_end(c, h, PSP_KC_ORTHO_DOTS, 8.0 * (J + 2) * dn);
  cudaMemcpyAsync(c->slot_scale + dst, c->ds.alpha + k, sizeof(double), cudaMemcpyDeviceToDevice, c->stream);
  c->launches += 3;
  return PSP_OK;
}

// The ring-resident step without the fused pass (k = 0: the cycle start, V(:,1) already in its
// slot): [k >= 1: V(:,k+1) = alpha_k w~_k - sum_j h_j alpha_j V(:,j) into the next slot, H(k+1,k),
// Givens, alpha_{k+1} (l.13-32)]; w~_{k+1} = A V(:,k+1) unnormalised into the slot's P_y
// (l.11-12, no probe copy); the MGS coefficients of step k+1 (l.13-16 / R11).
static psp_status ring_split_step(psp_ctx* c, int k, int src_slot, int dst) {
  const int64_t n = c->n;
  const double dn = (double)n;
  int h;
  if (k >= 1) {
    h = kt_begin(c);
    launch_icwy_update(basis(c), py_col(c, src_slot), c->ds.alpha + (k - 1), px_col(c, dst), k, c->nA, n, c->ds,
                       c->rc, c->stream);
    PSP_TRY(finish_reduce(c, EPI_UPDATE, 1, k, 0, 0));
    kt_end(c, h, PSP_KC_ORTHO_UPDATE, 8.0 * (k + 2) * dn);
    c->launches += 1;
  }
  cudaMemcpyAsync(c->slot_scale + dst, c->ds.alpha + k, sizeof(double), cudaMemcpyDeviceToDevice, c->stream);
  h = kt_begin(c);
  PSP_TRY(matvec(c, px_col(c, dst), nullptr, py_col(c, dst), nullptr));
  kt_end(c, h, PSP_KC_MATVEC, matvec_bytes(c, false));
  h = kt_begin(c);
  launch_icwy_dots(basis(c), py_col(c, dst), k + 1, c->nA, n, 1, c->ds, c->rc, c->stream);
  PSP_TRY(finish_reduce(c, EPI_DOTS_RAW, 2 * k + 1, k + 1, 0, 0));
  kt_end(c, h, PSP_KC_ORTHO_DOTS, 8.0 * (k + 2) * dn);
  c->launches += 1;
  if (c->multi) {                                   // ghost planes for the fused passes that follow
    PSP_TRY(ghost_exchange(c, px_col(c, dst)));
    PSP_TRY(ghost_exchange(c, py_col(c, dst)));
  }
  return PSP_OK;
}

// algorithmic bytes of the fused pass of step k (k = 0: the cycle-start pass)
static double fused_bytes(const psp_ctx* c, int k) {
  const bool cell = c->st.kind == PSP_OP_CELL_DIFF || c->st.kind == PSP_OP_CELL_ADVDIFF;
  const double per = 8.0 * (k + 1 + (cell ? 1 : 0) + (k > 0 ? 1 : 0) + 1);
  return per * (double)c->n;
}

psp_status psp_cycle_begin(psp_ctx* c, const double* b, const double* x0, double* h_beta) {
  NvtxRange nv("psp_cycle_begin");
  if (!c || !b || !x0) return fail(c, PSP_E_ARG, "psp_cycle_begin: NULL argument");
  if (c->sticky != PSP_OK) return c->sticky;
  if (x0 != c->X0) {
    launch_copy(x0, c->X0, c->n, c->stream);
    c->launches += 1;
  }
  c->cycle_fused = fused_eligible(c);
  // l.4: P_x(:,i) <- X0, P_y(:,i) <- A X0
  const int slot = ring_next(c);
  set_unit_scale(c, slot);
  int h = kt_begin(c);
  PSP_TRY(matvec(c, c->X0, nullptr, py_col(c, slot), px_col(c, slot)));
  kt_end(c, h, PSP_KC_MATVEC, matvec_bytes(c, true));
  stream_add(c, slot);
  // l.5-7: R_bar = B - P_y(:,i); beta = ||R_bar||; G(1) = beta.  V(:,1) <- R_bar/beta
  // (l.6) is stored unnormalised with alpha_1 = 1/beta.  On the fused path V(:,1) goes straight
  // into the ring slot where it will be recorded as the probe Y_1 (N = I, l.11).
  double* v1 = Vcol(c, 1);
  if (c->cycle_fused) {
    c->vslot[1] = ring_peek(c);
    v1 = px_col(c, c->vslot[1]);
  }
  h = kt_begin(c);
  launch_residual(b, py_col(c, slot), v1, c->n, c->nA, c->ds, c->rc, c->stream);
  kt_end(c, h, PSP_KC_RESIDUAL, 24.0 * c->n);
  c->launches += 1;
  PSP_TRY(finish_reduce(c, EPI_RESIDUAL, 1, 0, 0, 0));
  double beta;
  PSP_TRY(sync_read(c, c->ds.scal + SC_BETA, 1, &beta));
  if (h_beta) *h_beta = beta;
  if (c->cycle_fused && beta > 0.0 && isfinite(beta)) {
    // cycle-start pass: A V(:,1) -> P_y of the next slot and step 1's MGS coefficient
    if (fused_pass(c, 0)) {
      PSP_TRY(ghost_exchange(c, px_col(c, c->vslot[1])));   // multi-rank: V(:,1) on the ghost planes
      h = kt_begin(c);
      const int fe = launch_fused(c->st, c->ring_px, c->ring_py, c->vslot[1], c->ring_phys, 0, c->nA, c->vslot[1],
                                  1, nullptr, py_col(c, c->vslot[1]), c->slot_scale, c->vslot[1], c->ds, c->stream,
                                  flayout(c));
      if (fe) return fail(c, PSP_E_CUDA, "fused pass: " + fused_error(fe));
      kt_end(c, h, PSP_KC_FUSED, fused_bytes(c, 0));
      c->launches += 1;
      if (c->multi) {
        PSP_TRY(ghost_exchange(c, py_col(c, c->vslot[1])));
        PSP_TRY(finish_reduce(c, EPI_FUSED, 2, 0, 0, c->vslot[1]));
      }
    } else {
      PSP_TRY(ring_split_step(c, 0, c->vslot[1], c->vslot[1]));
    }
  }
  c->last_k = 0;
  c->combined_k = 0;
  return check_cuda(c, "psp_cycle_begin");
}

psp_status psp_arnoldi_step(psp_ctx* c, int k, double* h_resid, int* h_flags) {
  if (!c) return fail(c, PSP_E_ARG, "psp_arnoldi_step: NULL ctx");
  if (k < 1 || k > c->nA) return fail(c, PSP_E_ARG, "psp_arnoldi_step: k out of 1..restart");
  if (c->sticky != PSP_OK) return c->sticky;
  const int64_t n = c->n;
  const double dn = (double)n;
  int h;
  if (c->cycle_fused) {
    // l.10-12: the probe (Y_k, A Y_k) = (V_k, A V_k) was written by the previous pass into the
    // free slot; recording it makes it the newest probe.
    const int slot = ring_next(c);
    if (slot != c->vslot[k]) return fail(c, PSP_E_ARG, "psp_arnoldi_step: steps out of order (fused cycle)");
    stream_add(c, slot);
    if (k < c->nA) {
      // l.13-18 of step k, then l.10-16 of step k+1: one fused pass or three ring passes
      const int dst = ring_peek(c);
      c->vslot[k + 1] = dst;
      if (fused_pass(c, k)) {
        h = kt_begin(c);
        const int fe = launch_fused(c->st, c->ring_px, c->ring_py, c->vslot[1], c->ring_phys, k, c->nA, slot, 0,
                                    px_col(c, dst), py_col(c, dst), c->slot_scale, dst, c->ds, c->stream, flayout(c));
        if (fe) return fail(c, PSP_E_CUDA, "fused pass: " + fused_error(fe));
        kt_end(c, h, PSP_KC_FUSED, fused_bytes(c, k));
        c->launches += 1;
        if (c->multi) {                               // ghost planes of V(:,k+1), w~_{k+1}; the sums
          PSP_TRY(ghost_exchange(c, px_col(c, dst)));
          PSP_TRY(ghost_exchange(c, py_col(c, dst)));
          PSP_TRY(finish_reduce(c, EPI_FUSED, 2 * k + 2, k, 0, dst));
        }
      } else if (hyb_pass(c, k)) {
        PSP_TRY(ring_hyb_step(c, k, slot, dst));
      } else {
        PSP_TRY(ring_split_step(c, k, slot, dst));
      }
    } else {
      // the last step of the cycle: only H(k+1,k) = ||U|| is needed (V(:,k+1) is never used).
      // With N = I it is fused with the cycle's combine (Z = Z0 + y_k Z1, krylov.cu): one pass
      // over the basis forms ||U||, X0 + Z0 and Z1 into the free ring slot's columns
      h = kt_begin(c);
      if (c->n_identity && c->opts.fused) {
        const int spare = ring_peek(c);
        launch_update_combine(basis(c), py_col(c, slot), c->ds.alpha + (k - 1), c->X0, px_col(c, spare),
                              py_col(c, spare), k, c->nA, n, c->ds, c->rc, c->stream);
        PSP_TRY(finish_reduce(c, EPI_UPDCOMB, 1, k, 0, 0));
        c->combined_k = k;
        c->combined_slot = spare;
        kt_end(c, h, PSP_KC_ORTHO_UPDATE, 8.0 * (k + 4) * dn);
        c->launches += 2;
      } else {
        launch_icwy_update(basis(c), py_col(c, slot), c->ds.alpha + (k - 1), c->W, k, c->nA, n, c->ds,
                           c->rc, c->stream);
        PSP_TRY(finish_reduce(c, EPI_UPDATE, 1, k, 0, 0));
        kt_end(c, h, PSP_KC_ORTHO_UPDATE, 8.0 * (k + 2) * dn);
        c->launches += 1;
      }
    }
    c->launches += 1;
  } else {
    const int slot = ring_next(c);
    set_unit_scale(c, slot);
    double* px = px_col(c, slot);
    double* py = py_col(c, slot);
    const double* Vk = Vcol(c, k);
    // l.10-12: Y_k = N^{-1} V(:,k) -> P_x(:,i); P_y(:,i) = A Y_k
    if (c->n_identity) {
      h = kt_begin(c);
      PSP_TRY(matvec(c, Vk, c->ds.alpha + (k - 1), py, px));  // N = I: probe copy fused
      kt_end(c, h, PSP_KC_MATVEC, matvec_bytes(c, true));
    } else {
      h = kt_begin(c);
      PSP_TRY(precond_scaled(c, Vk, c->ds.alpha + (k - 1), px));
      kt_end(c, h, PSP_KC_PRECOND, 8.0 * (2 * c->d + 5) * dn);
      h = kt_begin(c);
      PSP_TRY(matvec(c, px, nullptr, py, nullptr));
      kt_end(c, h, PSP_KC_MATVEC, matvec_bytes(c, false));
    }
    stream_add(c, slot);
    double* U = Vcol(c, k + 1);
    // l.13-17: MGS (R11) + H(k+1,k) + Givens (l.19-32) in the last block
    if (c->opts.ortho == PSP_MGS_LITERAL) {
      h = kt_begin(c);
      launch_mgs_literal(py, U, nullptr, Vcol(c, 1), 1, k, c->nA, n, c->ds, c->rc, c->stream);
      PSP_TRY(finish_reduce(c, EPI_MGS, 1, k, 1, 0));
      for (int j = 2; j <= k; ++j) {
        launch_mgs_literal(U, U, Vcol(c, j - 1), Vcol(c, j), j, k, c->nA, n, c->ds, c->rc, c->stream);
        PSP_TRY(finish_reduce(c, EPI_MGS, 1, k, j, 0));
      }
      launch_mgs_literal_final(U, Vcol(c, k), k, c->nA, n, c->ds, c->rc, c->stream);
      PSP_TRY(finish_reduce(c, EPI_MGS_FINAL, 1, k, 0, 0));
      kt_end(c, h, PSP_KC_MGS_LITERAL, (24.0 + 32.0 * (k - 1) + 24.0) * dn);
      c->launches += k + 1;
    } else {
      h = kt_begin(c);
      launch_icwy_dots(basis(c), py, k, c->nA, n, 0, c->ds, c->rc, c->stream);
      PSP_TRY(finish_reduce(c, EPI_DOTS, 2 * k - 1, k, 0, 0));
      kt_end(c, h, PSP_KC_ORTHO_DOTS, 8.0 * (k + 1) * dn);
      h = kt_begin(c);
      launch_icwy_update(basis(c), py, nullptr, U, k, c->nA, n, c->ds, c->rc, c->stream);
      PSP_TRY(finish_reduce(c, EPI_UPDATE, 1, k, 0, 0));
      kt_end(c, h, PSP_KC_ORTHO_UPDATE, 8.0 * (k + 2) * dn);
      c->launches += 2;
    }
  }
  // l.18: V(:,k+1) = U / H(k+1,k) (R4: 0 on breakdown) -- lagged: alpha_{k+1} is set
  // by the Givens epilogue and folded into every reader of V(:,k+1)
  double sc[2];
  PSP_TRY(sync_read(c, c->ds.scal + SC_RK, 2, sc));
  if (h_resid) *h_resid = sc[0];
  if (h_flags) *h_flags = (int)sc[1];
  c->last_k = k;
  return PSP_OK;
}

psp_status psp_cycle_end(psp_ctx* c, int k, double* x) {
  if (!c || !x) return fail(c, PSP_E_ARG, "psp_cycle_end: NULL argument");
  if (k < 0 || k > c->nA) return fail(c, PSP_E_ARG, "psp_cycle_end: bad k");
  if (c->sticky != PSP_OK) return c->sticky;
  if (k == 0) {
    if (x != c->X0) launch_copy(c->X0, x, c->n, c->stream);
    return check_cuda(c, "psp_cycle_end");
  }
  // l.38-42: Q = H^{-1}G; Z = sum Q_j V_j; X = X0 + N^{-1} Z
  if (c->cycle_fused && c->combined_k == k && k == c->nA) {
    // the last step already formed X0 + Z0 and Z1: X = (X0 + Z0) + y_k Z1
    int h = kt_begin(c);
    launch_combine_finish(px_col(c, c->combined_slot), py_col(c, c->combined_slot), c->X0, c->n, c->ds,
                          c->stream);
    kt_end(c, h, PSP_KC_COMBINE, 24.0 * (double)c->n);
    c->launches += 1;
  } else if (c->n_identity) {
    int h = kt_begin(c);
    launch_combine(basis(c), k, c->nA, c->X0, c->X0, c->n, c->ds, c->stream);
    kt_end(c, h, PSP_KC_COMBINE, 8.0 * (k + 2) * (double)c->n);
    c->launches += 1;
  } else {
    int h = kt_begin(c);
    launch_combine(basis(c), k, c->nA, nullptr, c->W, c->n, c->ds, c->stream);
    kt_end(c, h, PSP_KC_COMBINE, 8.0 * (k + 1) * (double)c->n);
    c->launches += 1;
    h = kt_begin(c);
    PSP_TRY(precond(c, c->W, c->X0, c->X0));
    kt_end(c, h, PSP_KC_PRECOND, 8.0 * (2 * c->d + 6) * (double)c->n);
  }
  // l.43: X0 <- X
  if (x != c->X0) {
    launch_copy(c->X0, x, c->n, c->stream);
    c->launches += 1;
  }
  double st;
  PSP_TRY(sync_read(c, c->ds.scal + SC_STATUS, 1, &st));
  if (st != 0.0) return fail(c, PSP_E_SINGULAR, "back-substitution: zero pivot (R6)");
  return check_cuda(c, "psp_cycle_end");
}

// f4: PSP with preconditioned conjugate gradients (readings R27-R31; oracle/oracle.c orc_pcg).
// Vectors: x in X0, r = V(:,1), z = V(:,2) (z aliases r when N = I); the direction p_k and A p_k
// live in the probe ring slot of step k (the probe (p_k, A p_k) / ||p_k|| is recorded with
// slot_scale = 1/||p_k||, so recording costs no copy), p_{k-1} in the previous slot.
static psp_status cg_solve(psp_ctx* c, const double* b, const double* x0, psp_report* R, double eps) {
  const int64_t n = c->n;
  const double dn = (double)n;
  const bool ident = c->n_identity;
  if (x0 != c->X0) {
    launch_copy(x0, c->X0, n, c->stream);
    c->launches += 1;
  }
  c->cycle_fused = false;
  double* r = Vcol(c, 1);
  double* z = ident ? r : Vcol(c, 2);
  // the probe (x0, A x0) (as Alg.1 l.4), r0 = b - A x0
  const int s0 = ring_next(c);
  set_unit_scale(c, s0);
  int h = kt_begin(c);
  PSP_TRY(matvec(c, c->X0, nullptr, py_col(c, s0), px_col(c, s0)));
  kt_end(c, h, PSP_KC_MATVEC, matvec_bytes(c, true));
  stream_add(c, s0);
  h = kt_begin(c);
  launch_cg_start(b, py_col(c, s0), r, n, c->ds, c->rc, c->stream);
  c->launches += 1;
  PSP_TRY(finish_reduce(c, EPI_CG_START, 1, 0, 1, 0));
  kt_end(c, h, PSP_KC_CG, 24.0 * dn);
  R->matvecs = 1;
  R->cycles = 1;
  if (!ident) {                                       // z0 = M^-1 r0, rho = r0'z0
    h = kt_begin(c);
    PSP_TRY(precond_scaled(c, r, nullptr, z));
    kt_end(c, h, PSP_KC_PRECOND, 8.0 * (2 * c->d + 5) * dn);
    launch_cg_rz(r, z, n, c->ds, c->rc, c->stream);
    c->launches += 1;
    PSP_TRY(finish_reduce(c, EPI_CG_RHO, 1, 0, 0, 0));
    R->precond_applies += 1;
  }
  double beta;
  PSP_TRY(sync_read(c, c->ds.scal + SC_BETA, 1, &beta));
  R->r0 = beta;
  R->final_resid_est = beta;
  if (R->h_beta_history && R->beta_cap > 0) R->h_beta_history[0] = beta;
  R->beta_len = 1;
  if (!isfinite(beta)) return PSP_E_NONFINITE;
  if (beta <= eps) return PSP_OK;                      // R3
  const int64_t max_iters = (int64_t)c->nA * c->opts.max_cycles;   // R31
  int prev = -1;
  for (int64_t k = 1; k <= max_iters; ++k) {
    const int s = ring_next(c);
    const double* pold = prev >= 0 ? px_col(c, prev) : nullptr;
    // p = z + beta p_old -> P_x slot, q = A p -> P_y slot, p'q, p'p (alpha, the probe scale)
    h = kt_begin(c);
    if (!c->multi && launch_cg_dir_fused(c->st, z, pold, px_col(c, s), py_col(c, s), s, c->ds, c->stream)) {
      c->launches += 1;
      kt_end(c, h, PSP_KC_CG, (pold ? 40.0 : 32.0) * dn);
    } else {
      launch_cg_pupdate(z, pold, px_col(c, s), n, c->ds, c->stream);
      PSP_TRY(matvec(c, px_col(c, s), nullptr, py_col(c, s), nullptr));
      launch_cg_dirdots(px_col(c, s), py_col(c, s), n, s, c->ds, c->rc, c->stream);
      c->launches += 2;
      PSP_TRY(finish_reduce(c, EPI_CG_DIR, 2, 0, 1, s));
      kt_end(c, h, PSP_KC_CG, (pold ? 24.0 : 16.0) * dn + matvec_bytes(c, false) + 16.0 * dn);
    }
    R->matvecs += 1;
    stream_add(c, s);                                 // (after the pass that set its scale)
    // x += alpha p, r -= alpha q, R(k) = ||r||
    h = kt_begin(c);
    launch_cg_update(c->X0, px_col(c, s), py_col(c, s), r, n, ident ? 1 : 0, c->ds, c->rc, c->stream);
    c->launches += 1;
    PSP_TRY(finish_reduce(c, EPI_CG_UPD, 1, 0, ident ? 1 : 0, 0));
    kt_end(c, h, PSP_KC_CG, 48.0 * dn);
    if (!ident) {                                     // z = M^-1 r, rho' = r'z, beta
      h = kt_begin(c);
      PSP_TRY(precond_scaled(c, r, nullptr, z));
      kt_end(c, h, PSP_KC_PRECOND, 8.0 * (2 * c->d + 5) * dn);
      launch_cg_rz(r, z, n, c->ds, c->rc, c->stream);
      c->launches += 1;
      PSP_TRY(finish_reduce(c, EPI_CG_RHO, 1, 0, 0, 0));
      R->precond_applies += 1;
    }
    double sc[2];
    PSP_TRY(sync_read(c, c->ds.scal + SC_RK, 2, sc));
    const int flags = (int)sc[1];
    if (flags & PSP_FLAG_NONFINITE) return PSP_E_NONFINITE;
    if (flags & PSP_FLAG_BREAKDOWN) return fail(c, PSP_E_SINGULAR, "CG: p'Ap <= 0 (A or N_s not SPD, R30)");
    if (R->h_resid_history && R->resid_len < R->resid_cap) R->h_resid_history[R->resid_len] = sc[0];
    R->resid_len += 1;
    R->iterations += 1;
    R->final_resid_est = sc[0];
    if (flags & PSP_FLAG_CONVERGED) return PSP_OK;
    prev = s;
  }
  return PSP_E_NOCONV;
}

// f2: the device-resident solve (resident.cu) -- single rank, one-reduction MGS, n_A <= 64, up to
// 2^20 rows by default (a banded N: one CTA's sequential sweeps, n <= 16384)
static bool resident_eligible(const psp_ctx* c) {
  if (c->opts.resident <= 0 || c->multi || c->opts.ortho != PSP_MGS_1REDUCE) return false;
  if (c->opts.method != PSP_METHOD_GMRES || c->ssums) return false;
  if (!resident_supported(c->n, c->nA, !c->n_identity)) return false;
  return c->opts.resident >= 2 || c->n <= kResidentAutoRows;
}

static psp_status resident_solve(psp_ctx* c, const double* b, const double* x0, double* x, psp_report* R) {
  if (x0 != c->X0) {
    launch_copy(x0, c->X0, c->n, c->stream);
    c->launches += 1;
  }
  ResidentCall rc{};
  rc.st = c->st;
  rc.b = b;
  rc.X0 = c->X0;
  rc.V = c->V;
  rc.ldv = c->ldv;
  rc.ring_px = c->ring_px;
  rc.ring_py = c->ring_py;
  rc.slot_scale = c->slot_scale;
  rc.ring_cap = c->ring_cap;
  rc.ring_phys = c->ring_phys;
  rc.ring_head = c->ring_head;
  rc.ring_count = c->ring_count;
  rc.lu = c->n_identity ? nullptr : c->lu;
  rc.d = c->d;
  rc.y = c->W;
  rc.z = c->bs.y;
  rc.nA = c->nA;
  rc.max_cycles = c->opts.max_cycles;
  rc.tol_abs = c->opts.tol_mode == PSP_TOL_ABS;
  rc.tol = c->tol;
  rc.grid = resident_grid(c->n, !c->n_identity);
  rc.partials = c->res_part;
  rc.bar = c->res_bar;
  rc.hist = c->res_hist;
  rc.hist_cap = c->res_hist_cap;
  rc.betas = c->res_beta;
  rc.beta_cap = c->res_beta_cap;
  rc.out = c->res_out;
  rc.ds = c->ds;
  const int h = kt_begin(c);
  if (launch_resident(rc, c->stream)) {
    c->sticky = PSP_E_CUDA;
    return fail(c, PSP_E_CUDA, "resident solve: launch failed: " + cuda_err_str(cudaGetLastError()));
  }
  c->launches += 1;
  double o[24];
  PSP_TRY(sync_read(c, c->res_out, 24, o));
  if (getenv("PSP_RES_PROFILE"))   // instrumented builds: per-phase cycles of CTA 0 (resident.cu)
    fprintf(stderr, "resident phases (cycles): probe+matvec %.3g dots %.3g solve %.3g update+norm %.3g givens %.3g"
            " | grid reductions: local work %.3g, CTA totals + barrier %.3g\n",
            o[17], o[18], o[19], o[20], o[21], o[22], o[23]);
  const int iters = (int)o[0];
  // algorithmic bytes: step k reads V_k, k columns twice, writes P_x, P_y,
  // V_{k+1}: 8(2k+4) per row; a cycle start 40, a cycle end 8(k+2)
  {
    double per = 0.0;
    int left = iters;
    for (int cy = 0; cy < (int)o[1]; ++cy) {
      const int kk = left < c->nA ? left : c->nA;
      per += 40.0 + 8.0 * (kk + 2);
      for (int k = 1; k <= kk; ++k) per += 8.0 * (2 * k + 4);
      left -= kk;
    }
    kt_end(c, h, PSP_KC_RESIDENT, per * (double)c->n);
  }
  R->iterations = iters;
  R->cycles = (int)o[1];
  R->matvecs = (int)o[2];
  R->precond_applies = (int)o[3];
  const bool finish = o[4] != 0.0;
  const int status = (int)o[5];
  R->r0 = o[6];
  R->eps = o[7];
  R->final_resid_est = o[8];
  R->resid_len = (int)o[10];
  R->beta_len = (int)o[11];
  c->ring_head = (int)o[12];
  c->ring_count = (int)o[13];
  c->cycle_fused = false;
  c->last_k = 0;
  c->combined_k = 0;
  if (R->h_resid_history && R->resid_cap > 0) {
    int cnt = R->resid_len < R->resid_cap ? R->resid_len : R->resid_cap;
    if (cnt > c->res_hist_cap) cnt = c->res_hist_cap;
    if (cnt > 0) cudaMemcpyAsync(R->h_resid_history, c->res_hist, (size_t)cnt * 8, cudaMemcpyDeviceToHost, c->stream);
  }
  if (R->h_beta_history && R->beta_cap > 0) {
    int cnt = R->beta_len < R->beta_cap ? R->beta_len : R->beta_cap;
    if (cnt > c->res_beta_cap) cnt = c->res_beta_cap;
    if (cnt > 0) cudaMemcpyAsync(R->h_beta_history, c->res_beta, (size_t)cnt * 8, cudaMemcpyDeviceToHost, c->stream);
  }
  if (x != c->X0) {
    launch_copy(c->X0, x, c->n, c->stream);
    c->launches += 1;
  }
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) {
    c->sticky = PSP_E_CUDA;
    return fail(c, PSP_E_CUDA, "resident solve: " + cuda_err_str(cudaGetLastError()));
  }
  psp_status st = PSP_OK;
  if (status == PSP_E_NONFINITE) st = PSP_E_NONFINITE;
  else if (status == PSP_E_SINGULAR) st = PSP_E_SINGULAR;
  if (st == PSP_OK) {
    R->final_resid_true = o[9];
    R->converged = finish ? 1 : 0;
    R->resid_verified = (finish && o[9] <= R->eps) ? 1 : 0;
    if (!finish) st = PSP_E_NOCONV;
  }
  return st;
}

psp_status psp_solve(psp_ctx* c, const double* b, const double* x0, double* x, psp_report* rep) {
  NvtxRange nv("psp_solve");
  if (!c || !b || !x0 || !x) return fail(c, PSP_E_ARG, "psp_solve: NULL argument");
  if (c->sticky != PSP_OK) return c->sticky;
  psp_report dummy;
  memset(&dummy, 0, sizeof(dummy));
  psp_report* R = rep ? rep : &dummy;
  R->status = PSP_OK;
  R->converged = R->iterations = R->cycles = R->matvecs = R->precond_applies = 0;
  R->resid_len = R->beta_len = 0;
  R->resid_verified = 0;
  R->precond_identity = c->n_identity ? 1 : 0;
  if (c->opts.timing) cudaEventRecord(c->ev[0], c->stream);
  if (c->opts.method == PSP_METHOD_CG) {
    double eps;
    PSP_TRY(set_eps(c, b, &eps));
    R->eps = eps;
    psp_status status = cg_solve(c, b, x0, R, eps);
    const bool finish = status == PSP_OK;
    if (finish || status == PSP_E_NOCONV) {
      if (x != c->X0) {
        launch_copy(c->X0, x, c->n, c->stream);
        c->launches += 1;
      }
      PSP_TRY(matvec(c, x, nullptr, c->W, nullptr));  // R13: true residual, not recorded
      launch_diff_norm(b, c->W, c->n, c->ds, SC_TMP, c->rc, c->stream);
      c->launches += 1;
      PSP_TRY(finish_reduce(c, EPI_NORM, 1, 0, 0, SC_TMP));
      double tr;
      PSP_TRY(sync_read(c, c->ds.scal + SC_TMP, 1, &tr));
      R->final_resid_true = tr;
      R->converged = finish ? 1 : 0;
      R->resid_verified = (finish && tr <= eps) ? 1 : 0;
    }
    if (c->opts.timing) {
      cudaEventRecord(c->ev[1], c->stream);
      cudaEventSynchronize(c->ev[1]);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
      R->t_solve_ms = ms;
    }
    R->status = status;
    if (status != PSP_OK && status != PSP_E_NOCONV)
      return fail(c, status, std::string("psp_solve (CG): ") + psp_status_str(status));
    if (status == PSP_E_NOCONV) fail(c, status, "psp_solve (CG): iteration limit reached");
    return status;
  }
  if (resident_eligible(c)) {
    psp_status status = resident_solve(c, b, x0, x, R);
    if (c->opts.timing) {
      cudaEventRecord(c->ev[1], c->stream);
      cudaEventSynchronize(c->ev[1]);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
      R->t_solve_ms = ms;
    }
    R->status = status;
    if (status != PSP_OK && status != PSP_E_NOCONV)
      return fail(c, status, std::string("psp_solve (resident): ") + psp_status_str(status));
    if (status == PSP_E_NOCONV) fail(c, status, "psp_solve: n_r restart cycles exhausted");
    return status;
  }
  double eps;
  PSP_TRY(set_eps(c, b, &eps));
  R->eps = eps;
  psp_status status = PSP_OK;
  bool finish = false;
  if (x0 != c->X0) {
    launch_copy(x0, c->X0, c->n, c->stream);
    c->launches += 1;
  }
  for (int l = 1; l <= c->opts.max_cycles; ++l) {  // l.3
    double beta;
    PSP_TRY(psp_cycle_begin(c, b, c->X0, &beta));
    R->matvecs += 1;
    R->cycles += 1;
    if (R->h_beta_history && R->beta_len < R->beta_cap) R->h_beta_history[R->beta_len] = beta;
    R->beta_len += 1;
    if (l == 1) R->r0 = beta;
    if (!isfinite(beta)) { status = PSP_E_NONFINITE; break; }
    if (beta <= eps) {  // R3
      finish = true;
      R->final_resid_est = beta;
      break;
    }
    int kdone = 0;
    for (int k = 1; k <= c->nA; ++k) {  // l.8
      double Rk;
      int flags;
      PSP_TRY(psp_arnoldi_step(c, k, &Rk, &flags));
      R->matvecs += 1;
      if (!c->n_identity) R->precond_applies += 1;
      if (R->h_resid_history && R->resid_len < R->resid_cap) R->h_resid_history[R->resid_len] = Rk;
      R->resid_len += 1;
      R->iterations += 1;
      R->final_resid_est = Rk;
      kdone = k;
      if (flags & PSP_FLAG_NONFINITE) { status = PSP_E_NONFINITE; break; }
      if (flags & (PSP_FLAG_CONVERGED | PSP_FLAG_BREAKDOWN)) { finish = true; break; }  // l.33-36
    }
    if (status != PSP_OK) break;
    psp_status s = psp_cycle_end(c, kdone, c->X0);  // l.38-44
    if (!c->n_identity) R->precond_applies += 1;
    if (s != PSP_OK) { status = s; break; }
    if (finish) break;  // l.45-48
  }
  if (status == PSP_OK) {
    if (x != c->X0) {
      launch_copy(c->X0, x, c->n, c->stream);
      c->launches += 1;
    }
    // R13: true residual with one unrecorded matvec
    PSP_TRY(matvec(c, x, nullptr, c->W, nullptr));
    launch_diff_norm(b, c->W, c->n, c->ds, SC_TMP, c->rc, c->stream);
    c->launches += 1;
    PSP_TRY(finish_reduce(c, EPI_NORM, 1, 0, 0, SC_TMP));
    double tr;
    PSP_TRY(sync_read(c, c->ds.scal + SC_TMP, 1, &tr));
    R->final_resid_true = tr;
    R->converged = finish ? 1 : 0;
    R->resid_verified = (finish && tr <= eps) ? 1 : 0;
    if (!finish) status = PSP_E_NOCONV;
  }
  if (c->opts.timing) {
    cudaEventRecord(c->ev[1], c->stream);
    cudaEventSynchronize(c->ev[1]);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
    R->t_solve_ms = ms;
  }
  R->status = status;
  if (status != PSP_OK && status != PSP_E_NOCONV)
    return fail(c, status, std::string("psp_solve: ") + psp_status_str(status));
  if (status == PSP_E_NOCONV) fail(c, status, "psp_solve: n_r restart cycles exhausted");
  return status;
}

psp_status psp_raw_scratch_bytes(int64_t n, int d, size_t* bytes) {
  if (!bytes || n < 1 || d < 1 || d > kMaxD) return fail(nullptr, PSP_E_ARG, "psp_raw_scratch_bytes: bad argument");
  // + the split MREP's lagged-sum rows ((4d+4) x n doubles)
  *bytes = banded_scratch_bytes(n, d) + 6 * kMrepMaxBlocks * 8 + 64 + 16 * 8 + 1024 +
           (size_t)(4 * d + 4) * (size_t)n * 8 + 256;
  return PSP_OK;
}

static void raw_carve(void* scratch, int64_t n, int d, MrepScratch* ms, BandedScratch* bs) {
  char* p = (char*)(((uintptr_t)scratch + 255) & ~(uintptr_t)255);
  ms->partials = (double*)p;
  p += 6 * kMrepMaxBlocks * 8;
  ms->ticket = (unsigned*)p;
  p += 64;
  ms->result = (double*)p;
  p += 16 * 8;
  p = (char*)(((uintptr_t)p + 255) & ~(uintptr_t)255);
  ms->sums = (double*)p;
  ms->sums_n = n;
  p += (size_t)(4 * d + 4) * (size_t)n * 8;
  p = (char*)(((uintptr_t)p + 255) & ~(uintptr_t)255);
  *bs = banded_scratch(p, n, d);
}

psp_status psp_mrep_fit_raw(const double* px, const double* py, int64_t n, int m, int64_t ld,
                            const int32_t* h_order, int d, double* bands, double* icpt,
                            uint8_t* kind, double* kappa, void* scratch, size_t sbytes,
                            void* stream, psp_mrep_info* info) {
  size_t need;
  PSP_TRY(psp_raw_scratch_bytes(n, d, &need));
  if (!px || !py || !bands || !scratch) return fail(nullptr, PSP_E_ARG, "psp_mrep_fit_raw: NULL argument");
  if (sbytes < need) return fail(nullptr, PSP_E_NOMEM, "psp_mrep_fit_raw: scratch too small");
  if (n < 2 * d + 1) return fail(nullptr, PSP_E_DIM, "n < 2d+1");
  if (m > 256) return fail(nullptr, PSP_E_ARG, "m > 256");
  if (m < 2 * d + 2) {
    if (info) { memset(info, 0, sizeof(*info)); info->status = PSP_E_SAMPLES; }
    return PSP_E_SAMPLES;
  }
  cudaStream_t s = (cudaStream_t)stream;
  MrepScratch ms;
  BandedScratch bs;
  raw_carve(scratch, n, d, &ms, &bs);
  cudaMemsetAsync(ms.ticket, 0, 64, s);
  std::vector<int32_t> slots(m);
  for (int c2 = 0; c2 < m; ++c2) slots[c2] = h_order ? h_order[c2] : c2;
  MrepOut out{bands, icpt, kind, kappa};
  mrep_launch(px, py, nullptr, ld, slots.data(), m, n, d, out, ms, s, MrepMulti{nullptr, nullptr, nullptr, 0, n});
  double r[16];
  if (cudaMemcpyAsync(r, ms.result, sizeof(r), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return fail(nullptr, PSP_E_CUDA, "psp_mrep_fit_raw: " + cuda_err_str(cudaGetLastError()));
  PSP_TRY(check_cuda(nullptr, "psp_mrep_fit_raw"));
  if (info) {
    info->max_abs_diag = r[0];
    info->rows_ridge = (int64_t)r[3];
    info->rows_fallback = (int64_t)(r[4] + r[8]);
    info->rows_nondominant = (int64_t)r[5];
    info->gate_accepted = r[7] != 0.0;
    info->status = PSP_OK;
  }
  return PSP_OK;
}

psp_status psp_banded_factor_raw(const double* bands, int64_t n, int d, double* lu, void* scratch,
                                 size_t sbytes, void* stream) {
  size_t need;
  PSP_TRY(psp_raw_scratch_bytes(n, d, &need));
  if (!bands || !lu || !scratch) return fail(nullptr, PSP_E_ARG, "psp_banded_factor_raw: NULL argument");
  if (sbytes < need) return fail(nullptr, PSP_E_NOMEM, "scratch too small");
  MrepScratch ms;
  BandedScratch bs;
  raw_carve(scratch, n, d, &ms, &bs);
  cudaStream_t s = (cudaStream_t)stream;
  int passes = 0;
  int st = banded_factor(bands, n, d, lu, bs, s, &passes, nullptr, nullptr, nullptr);
  PSP_TRY(check_cuda(nullptr, "psp_banded_factor_raw"));
  if (st != PSP_OK) return fail(nullptr, PSP_E_SINGULAR, "banded LU: zero pivot or growth (S:272, S:293)");
  return PSP_OK;
}

psp_status psp_banded_solve_raw(const double* lu, int64_t n, int d, const double* v, const double* x0,
                                double* z, void* scratch, size_t sbytes, void* stream) {
  size_t need;
  PSP_TRY(psp_raw_scratch_bytes(n, d, &need));
  if (!lu || !v || !z || !scratch) return fail(nullptr, PSP_E_ARG, "psp_banded_solve_raw: NULL argument");
  if (sbytes < need) return fail(nullptr, PSP_E_NOMEM, "scratch too small");
  if (z == v) return fail(nullptr, PSP_E_ARG, "z and v may not alias");
  MrepScratch ms;
  BandedScratch bs;
  raw_carve(scratch, n, d, &ms, &bs);
  banded_solve(lu, n, d, v, nullptr, x0, z, bs, (cudaStream_t)stream, nullptr, nullptr, nullptr);
  return check_cuda(nullptr, "psp_banded_solve_raw");
}

static psp_status install_bands(psp_ctx* c, bool gate_ok, psp_report* R) {
  NvtxRange nv("banded_factor");
  bool accept = gate_ok;
  if (accept) {
    if (c->opts.timing) cudaEventRecord(c->ev[4], c->stream);
    int passes = 0;
    int h = kt_begin(c);
    int st = banded_factor(c->bands, c->n, c->d, c->lu, c->bs, c->stream, &passes, &c->launches,
                           c->multi ? c->comm : nullptr, c->bmisc);
    if (st == PSP_E_NCCL) return fail(c, PSP_E_NCCL, "banded factor: collective failed");
    kt_end(c, h, PSP_KC_FACTOR, 16.0 * (2 * c->d + 1) * (double)c->n);
    PSP_TRY(check_cuda(c, "banded_factor"));
    if (st != PSP_OK) accept = false;  // fall back to identity
    if (c->opts.timing && R) {
      cudaEventRecord(c->ev[5], c->stream);
      cudaEventSynchronize(c->ev[5]);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, c->ev[4], c->ev[5]);
      R->t_factor_ms = ms;
    }
  }
  c->n_identity = !accept;
  if (R) R->mrep_gate_accepted = accept ? 1 : 0;
  return PSP_OK;
}

psp_status psp_mrep_fit(psp_ctx* c, psp_report* rep) {
  NvtxRange nv("psp_mrep_fit");
  if (!c) return fail(c, PSP_E_ARG, "psp_mrep_fit: NULL ctx");
  if (c->sticky != PSP_OK) return c->sticky;
  psp_report dummy;
  memset(&dummy, 0, sizeof(dummy));
  psp_report* R = rep ? rep : &dummy;
  // f3 (opts.mrep_stream): the window is every probe since the last fit, already summed
  const int m = c->ssums ? c->scount : c->ring_count;
  R->mrep_ran = 0;
  if (m < 2 * c->d + 2) {  // R19
    c->scount = 0;
    R->mrep_status = PSP_E_SAMPLES;
    return PSP_E_SAMPLES;
  }
  if (c->opts.timing) cudaEventRecord(c->ev[2], c->stream);
  // the per-row diagnostics (intercept R15, row kind, condition estimate R17) are not written on
  // the hot path: psp_mrep_fit_raw returns them (17 bytes a row less traffic)
  MrepOut out{c->bands, nullptr, nullptr, nullptr};
  cudaMemsetAsync(c->ms.ticket, 0, 64, c->stream);
  int h = kt_begin(c);
  if (c->ssums) {
    MrepScratch sc = c->ms;
    sc.sums = c->ssums;
    sc.sums_n = c->n;
    mrep_fit_sums(m, c->n, c->d, out, sc, c->stream);
    c->scount = 0;
    kt_end(c, h, PSP_KC_MREP, (8.0 * (4 * c->d + 4) + 8.0 * (2 * c->d + 1)) * (double)c->n);
  } else {
    std::vector<int32_t> slots(m);
    for (int q = 0; q < m; ++q) slots[q] = ring_slot(c, q);
    MrepMulti mm{c->multi ? c->comm : nullptr, c->mh_send, c->mh_recv, c->row0, c->n_global};
    if (mrep_launch(c->ring_px + c->goff, c->ring_py + c->goff, c->slot_scale, c->ldr, slots.data(), m, c->n, c->d,
                    out, c->ms, c->stream, mm))
      return fail(c, PSP_E_NCCL, "MREP: collective failed");
    kt_end(c, h, PSP_KC_MREP, (16.0 * m + 8.0 * (2 * c->d + 1)) * (double)c->n);
  }
  c->launches += 3;
  double r[16];
  PSP_TRY(sync_read(c, c->ms.result, 16, r));
  if (c->opts.timing) {
    cudaEventRecord(c->ev[3], c->stream);
    cudaEventSynchronize(c->ev[3]);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]);
    R->t_mrep_ms = ms;
  }
  R->mrep_ran = 1;
  R->mrep_status = PSP_OK;
  R->mrep_max_abs_diag = r[0];
  R->mrep_rows_ridge = (int64_t)r[3];
  R->mrep_rows_fallback = (int64_t)(r[4] + r[8]);
  R->mrep_rows_nondominant = (int64_t)r[5];
  bool gate_ok = c->opts.gate ? (r[7] != 0.0) : true;
  if (c->opts.method == PSP_METHOD_CG) {
    // R29: CG takes the symmetric part N_s = (N + N^T) / 2, accepted when it is SPD by positive-
    // diagonal strict dominance (the factors' buffer is the scratch: it is refactored below)
    launch_sym_bands(c->bands, c->lu, c->n, c->d, c->stream);
    cudaMemcpyAsync(c->bands, c->lu, (size_t)c->n * (2 * c->d + 1) * 8, cudaMemcpyDeviceToDevice, c->stream);
    launch_gate_count(c->bands, c->n, c->d, c->row0, c->n_global, c->ds.scal + SC_TMP, c->stream, 1);
    c->launches += 2;
    double nondom;
    PSP_TRY(sync_read(c, c->ds.scal + SC_TMP, 1, &nondom));
    R->mrep_rows_nondominant = (int64_t)nondom;
    gate_ok = c->opts.gate ? (nondom == 0.0) : true;
  }
  return install_bands(c, gate_ok, R);
}

psp_status psp_step(psp_ctx* c, const double* u_n, double* u_np1, psp_report* rep) {
  NvtxRange nv("psp_step");
  if (!c || !u_n || !u_np1) return fail(c, PSP_E_ARG, "psp_step: NULL argument");
  if (c->sticky != PSP_OK) return c->sticky;
  if (c->opts.reset_history_per_step) { c->ring_count = 0; c->ring_head = 0; c->scount = 0; }
  // b := u^n (kept in B: u_np1 may alias u_n); X0 := u^n (R2)
  launch_copy(u_n, c->B, c->n, c->stream);
  c->launches += 1;
  psp_status s = psp_solve(c, c->B, c->B, u_np1, rep);
  if (s != PSP_OK && s != PSP_E_NOCONV) return s;
  psp_report dummy;
  memset(&dummy, 0, sizeof(dummy));
  psp_status m = psp_mrep_fit(c, rep ? rep : &dummy);
  if (m != PSP_OK && m != PSP_E_SAMPLES) return m;
  return s;
}

psp_status psp_set_bands(psp_ctx* c, const double* d_bands, int* h_accepted) {
  if (!c) return fail(c, PSP_E_ARG, "psp_set_bands: NULL ctx");
  if (c->sticky != PSP_OK) return c->sticky;
  if (!d_bands) {  // N = I
    c->n_identity = true;
    if (h_accepted) *h_accepted = 0;
    return PSP_OK;
  }
  if (d_bands != c->bands)
    cudaMemcpyAsync(c->bands, d_bands, (size_t)c->n * (2 * c->d + 1) * 8, cudaMemcpyDeviceToDevice, c->stream);
  bool ok = true;
  if (c->opts.gate) {
    // R21 on the given bands: a device count of the non-dominant rows (one scalar read back),
    // summed over the ranks for one decision for the whole matrix
    launch_gate_count(c->bands, c->n, c->d, c->row0, c->n_global, c->ds.scal + SC_TMP, c->stream,
                      c->opts.method == PSP_METHOD_CG ? 1 : 0);
    c->launches += 1;
    if (c->multi && c->comm->allreduce(c->ds.scal + SC_TMP, 1, 0, c->stream))
      return fail(c, PSP_E_NCCL, "psp_set_bands: gate all-reduce failed");
    double nondom;
    PSP_TRY(sync_read(c, c->ds.scal + SC_TMP, 1, &nondom));
    ok = nondom == 0.0;
  }
  PSP_TRY(install_bands(c, ok, nullptr));
  if (h_accepted) *h_accepted = c->n_identity ? 0 : 1;
  return check_cuda(c, "psp_set_bands");
}

// AC10: zero the given local rows of the current N (all 2d+1 bands), then re-install it
// through the gate and the factorisation, exactly as psp_set_bands: a gated N with a zero row is
// rejected (R21), an ungated one fails the factorisation (zero pivot) -- either way the
// identity fallback takes over and the next solve runs with N = I.
psp_status psp_inject_fault_rows(psp_ctx* c, const int64_t* h_rows, int count, int* h_accepted) {
  if (!c || (count > 0 && !h_rows)) return fail(c, PSP_E_ARG, "psp_inject_fault_rows: bad argument");
  if (c->sticky != PSP_OK) return c->sticky;
  for (int q = 0; q < count; ++q) {
    if (h_rows[q] < 0 || h_rows[q] >= c->n) return fail(c, PSP_E_DIM, "psp_inject_fault_rows: row out of range");
    for (int o = 0; o <= 2 * c->d; ++o)
      cudaMemsetAsync(c->bands + (int64_t)o * c->n + h_rows[q], 0, sizeof(double), c->stream);
  }
  return psp_set_bands(c, c->bands, h_accepted);
}

psp_status psp_get_bands(const psp_ctx* c, double* d_out, int* h_ident) {
  if (!c) return PSP_E_ARG;
  if (d_out)
    cudaMemcpyAsync(d_out, c->bands, (size_t)c->n * (2 * c->d + 1) * 8, cudaMemcpyDeviceToDevice, c->stream);
  if (h_ident) *h_ident = c->n_identity ? 1 : 0;
  cudaStreamSynchronize(c->stream);
  return PSP_OK;
}

psp_status psp_ring_view(const psp_ctx* c, int* count, int32_t* slots, double* scale,
                         const double** px, const double** py, int64_t* ld) {
  if (!c) return PSP_E_ARG;
  if (count) *count = c->ring_count;
  if (slots)
    for (int q = 0; q < c->ring_count; ++q) slots[q] = ring_slot(c, q);
  if (scale && c->ring_count > 0) {
    std::vector<double> all(c->ring_phys);
    cudaMemcpyAsync(all.data(), c->slot_scale, all.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream);
    if (cudaStreamSynchronize(c->stream) != cudaSuccess) return PSP_E_CUDA;
    for (int q = 0; q < c->ring_count; ++q) scale[q] = all[ring_slot(c, q)];
  }
  if (px) *px = c->ring_px + c->goff;
  if (py) *py = c->ring_py + c->goff;
  if (ld) *ld = c->ldr;
  return PSP_OK;
}

psp_status psp_ring_reset(psp_ctx* c) {
  if (!c) return PSP_E_ARG;
  c->ring_count = 0;
  c->ring_head = 0;
  c->scount = 0;
  return PSP_OK;
}

psp_status psp_get_hessenberg(const psp_ctx* c, double* H, double* Hraw, double* G, double* C, double* S) {
  if (!c) return PSP_E_ARG;
  const size_t hs = (size_t)(c->nA + 1) * c->nA * 8;
  if (H) cudaMemcpyAsync(H, c->ds.H, hs, cudaMemcpyDeviceToHost, c->stream);
  if (Hraw) cudaMemcpyAsync(Hraw, c->ds.Hraw, hs, cudaMemcpyDeviceToHost, c->stream);
  if (G) cudaMemcpyAsync(G, c->ds.G, (c->nA + 1) * 8, cudaMemcpyDeviceToHost, c->stream);
  if (C) cudaMemcpyAsync(C, c->ds.C, c->nA * 8, cudaMemcpyDeviceToHost, c->stream);
  if (S) cudaMemcpyAsync(S, c->ds.S, c->nA * 8, cudaMemcpyDeviceToHost, c->stream);
  return cudaStreamSynchronize(c->stream) == cudaSuccess ? PSP_OK : PSP_E_CUDA;
}

psp_status psp_get_basis(const psp_ctx* c, int j, const double** d_vj, double* h_scale) {
  if (!c || !d_vj || j < 1 || j > c->nA + 1) return PSP_E_ARG;
  *d_vj = c->cycle_fused ? c->ring_px + (int64_t)c->vslot[j] * c->ldr + c->goff : c->V + (int64_t)(j - 1) * c->ldv;
  if (h_scale) {
    cudaMemcpyAsync(c->hp + 16, c->ds.alpha + (j - 1), sizeof(double), cudaMemcpyDeviceToHost, c->stream);
    if (cudaStreamSynchronize(c->stream) != cudaSuccess) return PSP_E_CUDA;
    *h_scale = c->hp[16];
  }
  return PSP_OK;
}

}  // extern "C"
