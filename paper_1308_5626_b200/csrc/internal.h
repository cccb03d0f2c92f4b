// internal.h -- shared declarations of libpspgmres's translation units (not part of the ABI).
//
// The public boundary is include/pspgmres.h.  Everything here is sm_100a CUDA + host C++
// of the product; nothing is shared with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/pspgmres.h"

// The communicator (comm.cu): NCCL for real ranks, a host-mediated loopback group for testing.
// op: 0 sum, 1 max, 2 min.  sendrecv exchanges with rank-1 (lo) and rank+1 (hi): send_lo goes
// to rank-1 and recv_lo receives rank-1's send_hi, and symmetrically.  Return 0 on success.
struct psp_comm {
  int nranks = 1, rank = 0;
  virtual ~psp_comm() {}
  virtual int allreduce(double* d, size_t count, int op, cudaStream_t s) = 0;
  virtual int sendrecv(const double* send_lo, double* recv_lo, size_t n_lo, const double* send_hi,
                       double* recv_hi, size_t n_hi, cudaStream_t s) = 0;
  virtual int allgather(const double* send, double* recv, size_t count, cudaStream_t s) = 0;
};

namespace psp {

constexpr int kMaxD = 4;         // MREP / banded half-bandwidth supported by the kernels
constexpr int kMaxRestart = 128; // n_A limit (device Hessenberg state is O(n_A^2))
constexpr int kRedThreads = 256; // block size of the grid-reduction kernels
constexpr int kHybOff = 2 * kMaxRestart + 16;   // ds.rpart offset of a split-column fused pass's sums

// ------------------------------------------------------------------------------------------
// Operator data (A = I - dt L, Eq.4).  Coefficients are precomputed on the host.
// ------------------------------------------------------------------------------------------
struct Stencil {
  int kind;            // PSP_OP_*
  int ndim;
  int64_t nx, ny, nz;  // LOCAL extents (nz = this rank's planes for 3-D; ny lines for 2-D)
  int64_t n;           // local rows
  double s[3];         // dt * nu / h_a^2 (CONST_DIFF) or dt / h_a^2 (CELL_*)
  double a[3];         // dt * c_a / h_a (CELL_ADVDIFF)
  const double* field; // kappa / nu of the local rows (CELL_*)
  int dA;              // DIA half-bandwidth
  const double* bands; // DIA bands (2dA+1) x n
  // slab halo (multi-rank): the plane / line of x and field just below / above the local
  // block, NULL on the global boundary.
  const double* x_lo;
  const double* x_hi;
  const double* f_lo;
  const double* f_hi;
};

// y = A (xs * x); optionally xcopy = xs * x (the probe column P_x).
// xs: device scalar (the lagged normalisation of a Krylov column) or NULL for 1.
void launch_matvec(const Stencil& st, const double* x, const double* xs, double* y, double* xcopy,
                   cudaStream_t s);

// ------------------------------------------------------------------------------------------
// Device state of one GMRES cycle (Hessenberg, Givens, scalars) -- lives in the workspace.
// ------------------------------------------------------------------------------------------
struct DevState {
  double* H;         // (nA+1) x nA column-major, rotated in place
  double* Hraw;      // pre-rotation copy (test hook, R4 breakdown test)
  double* G;         // nA+1
  double* C;         // nA
  double* S;         // nA
  double* Q;         // nA (back-substitution, R6)
  double* Lm;        // (nA+1) x (nA+1): strictly-lower part of V'V (ICWY MGS, R11)
  double* alpha;     // nA+1: V(:,j) = alpha[j-1] * stored column (lagged normalisation)
  double* scal;      // scalars, see enum below
  double* resid;     // R(k) of the current cycle, nA
  double* partials;  // grid-reduction partials: kMaxPartialVals x nblocks
  unsigned* tickets; // last-block counters (one per reduction slot)
  double* rpart;     // multi-rank: this rank's totals, all-reduced before the epilogue
  double* slot_scale;  // per probe-ring slot: the recorded probe is slot_scale[slot] * column
  int multi;         // 1: reductions stop at rpart (the host all-reduces, then epilogue_kernel)
};
// scalar epilogues of the grid reductions (krylov.cu); multi-rank runs them as a 1-thread
// kernel on the all-reduced ds.rpart
// EPI_DOTS_RAW: the ring-resident step, w = A V_k unnormalised (scale alpha_k), so h_j carries alpha_k too
// EPI_HYB: the split-column ring step (fused pass over the last columns + dots over the rest)
enum { EPI_NORM = 0, EPI_RESIDUAL = 1, EPI_MGS = 2, EPI_MGS_FINAL = 3, EPI_DOTS = 4, EPI_UPDATE = 5, EPI_DOTS_RAW = 6,
       EPI_HYB = 7,
       // f4, PSP-CG (cg.cuh): r0 = b - A x0; p'q and p'p of a direction; the x / r update; r'z
       EPI_CG_START = 8, EPI_CG_DIR = 9, EPI_CG_UPD = 10, EPI_CG_RHO = 11,
       // multi-rank ring steps: the fused pass's tail (givens.cuh fused_tail; slot = dst slot) and
       // the last step's update + combine coefficients (krylov.cu)
       EPI_FUSED = 12, EPI_UPDCOMB = 13 };
void launch_epilogue(int kind, DevState ds, int k, int nA, int j, int slot, cudaStream_t s);
enum { SC_BETA = 0, SC_EPS = 1, SC_RK = 2, SC_FLAGS = 3, SC_STATUS = 4, SC_NORM = 5,
       SC_MAXDIAG = 6, SC_GATE = 7, SC_TMP = 8, SC_RHO = 9, SC_ALPHA = 10, SC_BETACG = 11, SC_NSCAL = 16 };
enum { TK_MAIN = 0, TK_AUX = 1, TK_MREP = 2, TK_N = 8 };

struct RedCfg {
  int nblocks;       // grid of every reduction kernel (multiple of the SM count)
  int max_vals;      // partials per block the partials buffer holds
};

// Krylov basis columns V(:,j), j = 0..: either a plain column-major array (s1 = 0, cap large)
// or consecutive slots of the probe ring (the fused path stores V(:,j) in P_x slots).
struct Basis {
  const double* base;
  int64_t ld;
  int s1;
  int cap;
  __host__ __device__ const double* col(int j) const { return base + (int64_t)((s1 + j) % cap) * ld; }
};

// ---- Krylov kernels (krylov.cu) ----
// ||x||_2 -> scal[slot] (deterministic tree order; sqrt applied)
void launch_norm(const double* x, int64_t n, DevState ds, int slot, const RedCfg& rc, cudaStream_t s);
// r = b - y into v (unnormalised), beta = ||r|| -> scal[SC_BETA], G(1) = beta
void launch_residual(const double* b, const double* y, double* v, int64_t n, int nA, DevState ds,
                     const RedCfg& rc, cudaStream_t s);
// literal MGS: one launch per j; src -> dst (U) with the lagged axpy of j-1
void launch_mgs_literal(const double* src, double* U, const double* Vprev, const double* Vj,
                        int j, int k, int nA, int64_t n, DevState ds, const RedCfg& rc,
                        cudaStream_t s);
// literal MGS tail: U -= H(k,k) V_k; H(k+1,k) = ||U||; then the Givens update
void launch_mgs_literal_final(double* U, const double* Vk, int k, int nA, int64_t n,
                              DevState ds, const RedCfg& rc, cudaStream_t s);
// ICWY one-reduction MGS (R11): pass A = dots V_j'w (j<=k), V_j'V_k (j<k); solve (I+L)h = s
// w_raw: w = A V(:,k) unnormalised (ring-resident basis), h_j = alpha_j alpha_k V_j'w
void launch_icwy_dots(Basis V, const double* w, int k, int nA, int64_t n, int w_raw,
                      DevState ds, const RedCfg& rc, cudaStream_t s);
// pass B = U = w - sum_j h_j V_j ; H(k+1,k) = ||U|| ; Givens update
// ncols >= 0 and < k: only columns [0, ncols), no norm / epilogue (split-column step, pass A)
void launch_icwy_update(Basis V, const double* w, const double* ws, double* U, int k,
                        int nA, int64_t n, DevState ds, const RedCfg& rc, cudaStream_t s, int ncols = -1);
// split-column step k, pass C: dots of V_0..V_{J-1} and u with w, then the step's epilogue
// (EPI_HYB, with the fused pass's sums in ds.rpart)
void launch_icwy_dots_hyb(Basis V, const double* w, const double* u, int J, int k, int nA, int64_t n,
                          DevState ds, const RedCfg& rc, cudaStream_t s);
// the last step of a full ring cycle fused with the combine (krylov.cu): ||U_k|| + Givens,
// z0 = x0 + Z0, z1 = Z1 (Z = Z0 + y_k Z1), then x = z0 + y_k z1 at the cycle end
void launch_update_combine(Basis V, const double* w, const double* ws, const double* x0, double* z0, double* z1,
                           int k, int nA, int64_t n, DevState ds, const RedCfg& rc, cudaStream_t s);
void launch_combine_finish(const double* z0, const double* z1, double* x, int64_t n, DevState ds, cudaStream_t s);
// Q = H^{-1} G (R6) and out = base + sum_j Q_j V_j; base may be NULL (Z only)
void launch_combine(Basis V, int k, int nA, const double* base, double* out,
                    int64_t n, DevState ds, cudaStream_t s);
// y = x (plain copy on the stream)
void launch_copy(const double* x, double* y, int64_t n, cudaStream_t s);
// ||b - y|| -> scal[slot]
void launch_diff_norm(const double* b, const double* y, int64_t n, DevState ds, int slot,
                      const RedCfg& rc, cudaStream_t s);

// ---- f4: PSP-CG passes (krylov.cu; the fused direction pass in stencil.cu) ----
// r = b - y (y = A x0, the recorded x0 probe), r'r -> EPI_CG_START (beta, rho for N = I)
void launch_cg_start(const double* b, const double* y, double* r, int64_t n, DevState ds, const RedCfg& rc,
                     cudaStream_t s);
// p = z + beta p_old (p_old NULL: p = z), into the ring slot (no reduction)
void launch_cg_pupdate(const double* z, const double* pold, double* p, int64_t n, DevState ds, cudaStream_t s);
// p'q, p'p -> EPI_CG_DIR (alpha, the slot's probe scale 1/||p||)
void launch_cg_dirdots(const double* p, const double* q, int64_t n, int slot, DevState ds, const RedCfg& rc,
                       cudaStream_t s);
// x += alpha p, r -= alpha q, r'r -> EPI_CG_UPD (R(k), flags; N = I: beta, rho)
void launch_cg_update(double* x, const double* p, const double* q, double* r, int64_t n, int identity,
                      DevState ds, const RedCfg& rc, cudaStream_t s);
// r'z -> EPI_CG_RHO (beta, rho)
void launch_cg_rz(const double* r, const double* z, int64_t n, DevState ds, const RedCfg& rc, cudaStream_t s);
// the fused direction pass (stencil.cu): p = z + beta p_old -> px, q = A p -> py, p'q and p'p ->
// EPI_CG_DIR, one pass over HBM (3-D grids with nx % 4 == 0 and 16-byte aligned vectors, one
// rank); returns false when the shape is not supported (the caller runs the three passes)
bool launch_cg_dir_fused(const Stencil& st, const double* z, const double* pold, double* px, double* py, int slot,
                         DevState ds, cudaStream_t s);

// ---- fused single-pass Arnoldi step for N = I (fused.cu) ----
bool fused_supported(const Stencil& st, int k);
// finish step k (u = V_{k+1} -> dstx, A u -> dsty, H(k+1,k), Givens, alpha_{k+1} ->
// slot_scale[dst_slot]) and compute step k+1's MGS coefficients; k = 0 is the cycle-start pass
// returns 0, or the cuTensorMapEncodeTiled error of the operand maps.
// Layout of the ring columns: ring_px / ring_py / lay.field / src_vec are column STARTS, columns
// lay.ld apart; with lay.zoff = 1 (multi-rank slabs) every column carries a ghost plane below and
// above the nz owned planes (the neighbour ranks' boundary planes, zero at the global boundary),
// and lo_in / hi_in say whether the neighbour exists (its ghost plane is interior, not Dirichlet).
struct FusedLayout {
  int64_t ld;
  int zoff, lo_in, hi_in;
  const double* field;   // the coefficient field's column start (NULL: constant coefficients)
};
int launch_fused(const Stencil& st, const double* ring_px, const double* ring_py, int vs1, int cap, int k, int nA,
                  int src_slot, int src_px, double* dstx, double* dsty, double* slot_scale, int dst_slot,
                  DevState ds, cudaStream_t s, const FusedLayout& lay, int jb = 0, const double* src_vec = nullptr);

// ---- f2: the device-resident solve (resident.cu) ----
constexpr int kResidentMaxRestart = 64;       // replicated per-CTA scalar state in shared memory
constexpr int64_t kResidentSeqRows = 16384;   // a banded N: one thread's sequential sweeps
constexpr int64_t kResidentOneCtaRows = 4096; // one CTA (no grid barrier)
constexpr int64_t kResidentAutoRows = (int64_t)1 << 20;   // opts.resident = 1: up to here
struct ResidentCall {
  Stencil st;
  const double* b;
  double* X0;
  double* V;
  int64_t ldv;
  double* ring_px;
  double* ring_py;
  double* slot_scale;
  int ring_cap, ring_phys, ring_head, ring_count;
  const double* lu;     // NULL: N = I
  int d;
  double* y;            // n (N != I)
  double* z;            // n (N != I)
  int nA, max_cycles, tol_abs;
  double tol;
  int grid;
  double* partials;     // resident_scratch_doubles
  unsigned long long* bar;
  double* hist;
  int hist_cap;
  double* betas;
  int beta_cap;
  double* out;          // 16 doubles: iterations, cycles, matvecs, precond applies, finish, status,
                        // r0, eps, est, true resid, hist len, beta len, ring head, ring count
  DevState ds;
};
bool resident_supported(int64_t n, int nA, bool banded_n);
int resident_grid(int64_t n, bool banded_n);
size_t resident_scratch_doubles(int nA, int grid);
int launch_resident(const ResidentCall& c, cudaStream_t s);   // 0 ok, 1 launch failure

// ---- MREP (mrep.cu) ----
struct MrepOut {
  double* bands;      // (2d+1) x n
  double* intercept;  // n or NULL
  uint8_t* kind;      // n or NULL
  double* kappa;      // n or NULL
};
struct MrepScratch {
  double* partials;   // 6 x kMrepMaxBlocks
  unsigned* ticket;
  double* result;     // 16: [0] max|diag| [1] max|diag| over non-dominant rows [2] min|diag|
                      // [3] rows_ridge [4] rows_fallback [5] rows_nondominant (pre-R18)
                      // [6] R18 patch needed [7] gate accepted (R21) [8] rows patched by R18
  double* sums = nullptr;   // optional (4d+4) x sums_n lagged-sum rows: the split MREP (mrep.cu)
  int64_t sums_n = 0;
};
constexpr int kMrepMaxBlocks = 148 * 8;
// Alg.2 on probe columns px + slots[c]*ld (c = 0..m-1 oldest -> newest), then R18 + gate stats.
// Multi-rank MREP: the d P_x rows on each side of this rank's block come from the neighbours
// (send/recv: [lo|hi] x m x d doubles each), rows are global row0 + local, of gN in total;
// the gate statistics are all-reduced.  comm NULL: one rank (row0 = 0, gN = n).
struct MrepMulti {
  psp_comm* comm;
  double* send;
  double* recv;
  int64_t row0;
  int64_t gN;
};
// slot_scale (device, per slot, may be NULL): the recorded probe is slot_scale[slot] * column.
// Returns 0, or 1 when a collective failed.
int mrep_launch(const double* px, const double* py, const double* slot_scale, int64_t ld,
                const int32_t* slots, int m, int64_t n, int d, MrepOut out, MrepScratch sc,
                cudaStream_t s, MrepMulti mm);

// f3: streaming MREP.  Add the probe (scale[slot] * x, scale[slot] * y) to the (4d+4) x ns lagged
// sums (first != 0: overwrite, the first probe of a window); then fit every row from the sums
// (m probes), R18 and the gate statistics into sc.result as mrep_launch.  One rank.
void launch_mrep_accumulate(const double* x, const double* y, const double* scale, int slot, int64_t n, int d,
                            double* sums, int64_t ns, int first, cudaStream_t s);
void mrep_fit_sums(int m, int64_t n, int d, MrepOut out, MrepScratch sc, cudaStream_t s);
// R21 gate of a given N: the number of rows that are not strictly diagonally dominant -> *count
// (device scalar; zeroed first).  grow0 / gN: global index of local row 0 and the global rows.
// spd != 0 (PSP-CG, R29): a non-positive diagonal also counts
void launch_gate_count(const double* bands, int64_t n, int d, int64_t grow0, int64_t gN, double* count,
                       cudaStream_t s, int spd = 0);
// R29: sym = (N + N^T) / 2 in DIA storage (one rank); sym must not alias bands
void launch_sym_bands(const double* bands, double* sym, int64_t n, int d, cudaStream_t s);

// ---- banded LU (banded.cu) ----
struct BandedScratch {
  double* states;     // fixed-point states (factor) / look-back descriptors (solve)
  unsigned long long* tickets;
  int* changed;
  double* y;          // n: intermediate of the two sweeps
  int64_t desc_count;
};
size_t banded_scratch_bytes(int64_t n, int d);
BandedScratch banded_scratch(void* base, int64_t n, int d);
// multi-rank scratch of the banded solver (doubles): chunk states, rank maps, gathered states
size_t banded_misc_doubles(int d, int nranks);
// factor; returns PSP_OK / PSP_E_SINGULAR / PSP_E_NCCL (synchronises); *passes = fixed-point
// passes.  comm (may be NULL) + misc: the rows are this rank's block of a global banded matrix.
int banded_factor(const double* bands, int64_t n, int d, double* lu, BandedScratch sc,
                  cudaStream_t s, int* passes, int64_t* launches, psp_comm* comm, double* misc);
// z = x0 + N^{-1} (vs * v) (x0 may be NULL; vs: device scalar or NULL for 1)
int banded_solve(const double* lu, int64_t n, int d, const double* v, const double* vs,
                 const double* x0, double* z, BandedScratch sc, cudaStream_t s, int64_t* launches,
                 psp_comm* comm, double* misc);

// ---- misc ----
std::string cuda_err_str(cudaError_t e);
// Per-device launch state (function attributes, tensor maps, occupancy, side streams) is keyed by
// the CURRENT device, so contexts on several GPUs of one process each get their own.
constexpr int kMaxDev = 64;
int device_ordinal();   // cudaGetDevice, clamped to [0, kMaxDev)
int device_sms();       // multiprocessor count of the current device (cached per device)
// fused.cu: text of a launch_fused error code
std::string fused_error(int code);

}  // namespace psp
