// Device-resident problem + state of one DLRA solve (behind pnd_handle).
#pragma once

#include "pnd.h"

namespace pnd {

// phase timer: CUDA events on the handle's stream around each phase of the
// step (pnd_timing / pnd_timing_get), used by bench.py for per-kernel
// durations and roofline fractions
enum Phase {
  PH_KSTAGE, PH_LGRAM, PH_LSIDE, PH_ORTH, PH_TSQR_M, PH_SGRAM, PH_SRK4, PH_SVD, PH_ROTATE,
  PH_SCATK1, PH_SCATGRAM, PH_SCATSMALL, PH_DOSE, PH_DEFECT, PH_COUNT
};

struct TimerState {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<int> ids;  // mark i uses pool[i]
  cudaEvent_t ev[8] = {};
};

struct Handle {
  int device = 0;
  cudaStream_t st = nullptr;
  cudaStream_t st2 = nullptr;       // side stream: independent passes overlapped with st
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  Geom g{};
  int m = 0;
  std::string err;
  std::string stencil_error;  // non-empty for a 2-cell axis

  // operators and coefficients
  DBuf amat;        // ns x m x m, A_s in stencil order
  DBuf inv_s;       // ld (1/S per cell)
  DBuf isp;         // (n + 2 halo) x 2: rows [1/S, 0] with zero halo rows (TMA segments)
  DBuf s_field;     // ld (S at E_mid, for the "steps" tally)
  IBuf cls;         // n
  DBuf cls_atomic;  // n_cls x 12
  DBuf cls_val;     // n_cls (staging)
  int n_cls = 0;
  DBuf gdiag;       // 12 x m
  DBuf sigt;        // 12
  int n_beams = 0;
  DBuf psi;         // n_beams x ld (source slice, E_mid)
  DBuf psi_lo;      // n_beams x ld (tally slice, E_lo)
  DBuf tm;          // n_beams x m
  DBuf flux;        // n_beams x G x ld (group tables, column-major)
  int n_groups = 0;
  // separable group tables (pnd_set_flux_separable): psi(c, g) = lat(x, y) depth(z, g),
  // kept as the factors (n_beams x nx ny, n_beams x nz x G) -- a 512^3 x 128-group
  // dense table is 137 GB per beam; the per-step slices are formed from the factors
  DBuf sep_lat, sep_depth;
  bool flux_sep = false;
  // ray-footprint (sparse) group tables (pnd_set_flux_table_sparse): per beam
  // the cells its rays touched and their nnz x G values -- a traced 121-ray
  // pencil at 256^3 touches ~0.2 % of the cells; the dense table would be
  // 17 GB per beam at 128 groups
  std::vector<IBuf> sp_cells;
  std::vector<DBuf> sp_vals;
  std::vector<int> sp_nnz;
  bool flux_sparse = false;
  bool have_flux() const { return flux.p != nullptr || flux_sep || flux_sparse; }
  bool have_angular = false, have_inv_s = false, have_mat = false, have_scat = false;
  // per-step coefficient tables (coeff.cu, pnd_set_coefficient_tables):
  // [log E | log S (12 x K each) | rho (n_cls) | w (n_cls x 12) | E_mom (P) |
  //  g (12 x P x nd) | xi1 (12 x P) | flux (e_min, e_max) per beam]
  DBuf ctab;
  DBuf csel;        // device-side flux selections (j0, j1; w0, w1)
  int ct_K = 0, ct_P = 0, ct_nd = 0, ct_model = 0, ct_pn = 0, ct_bcorr = 0;
  double ct_fpscale = 0.0;
  bool have_ctab = false;
  // ranks above 32 (wide.cu): 32-column block copies and chain workspaces
  std::vector<NBuf> wide_u0b, wide_qb, wide_w1b, wide_w2b, wide_gb;
  NBuf wide_base, wide_tmp[2];
  DBuf wide_m, wide_t, wide_i, wide_g;
  // ranks above 64 (xwide.cu): the n-side matrices as 32-column cell-major
  // blocks; `blocked` = the state's U / Q live in xU / xQ
  std::vector<NBuf> xU, xQ, xUn, xW1, xW2;  // the CGS scratch Y shares xW1
  std::vector<DBuf> xsm;
  bool blocked = false;
  DBuf cq_work;  // pivoted-Cholesky work matrices that do not fit in shared memory
  // full-rank state (fullrank.cu): ceil(m / 32) cell-major column blocks
  std::vector<NBuf> fr_u, fr_w1, fr_w2;
  NBuf fr_t[2];
  DBuf fr_scr, fr_scr2, fr_scr3, fr_eye;
  bool have_fr = false;

  // state: U^ = [U (ua cols) | Q (uq cols)] cell-major, S (ru x rv row-major),
  // V (m x rv row-major); ru = ua + uq
  NBuf U, Q, Un, Qa, W1, W2, Xs;
  DBuf S, V;
  int ua = 0, uq = 0;
  int ru = 0, rv = 0;

  // workspaces
  DBuf part;                  // gram partials
  DBuf bcat;                  // K-stage [M; S0] (stream-ordered reuse within this handle)
  TsqrWork tq_m;
  DBuf sm[48];                // small / m-side scratch (see step.cu Slot)
  IBuf iflag;
  DBuf dep, prev;             // dose tally
  double* pinned = nullptr;   // small pinned readback buffer
  Comm* comm = nullptr;       // z-slab communicator (multi-GPU), null on one device
  TimerState timer;
  bool nvtx_open = false;  // an NVTX phase range is open
  bool singular_pending = false;  // scattering solve flag awaiting the next sync

  // speculative steps (step.cu spec_*): the host predicts every shape the
  // step's device-side decisions produce (the augmentation ranks, the
  // truncation ranks), launches the whole step without a host round trip and
  // the device flags any disagreement; one synchronisation at the end reads
  // the flag, and a mismatch restores the snapshot taken at the step's start
  // and recomputes the step on the synchronous path. Small grids only (the
  // snapshot is a copy of the state), one device.
  bool spec = false;              // inside a speculative step
  int spec_pause = 0;             // steps to run synchronously after a mismatch
  int spec_r1[2] = {-1, -1};      // truncation ranks of the last step (the predictions)
  int spec_tr = 0;                // which substep of the step is running (0, 1)
  bool spec_kfull[2] = {false, false};  // its last augmentation was full
  IBuf spec_flag;                 // [mismatch, singular]
  NBuf snap_u;
  DBuf snap_s, snap_v, snap_dep, snap_prev;
  int snap_ua = 0, snap_ru = 0, snap_rv = 0;
  long long spec_hits = 0, spec_misses = 0;
};

// phase mark: when timing is on, records an event on the handle's stream;
// the time until the next mark is attributed to `id` (id < 0 closes)
void phase(Handle& h, int id);

// views of the current state
NMat state_u(Handle& h);
NMat state_q(Handle& h);
void consolidate(Handle& h);   // fold Q into U (uq -> 0)
void set_isp(Handle& h);       // refresh the [1/S, 0] halo rows from inv_s
// step coefficients at e_mid (and the uncollided tally slice at e_lo) from the
// device-resident tables: no host->device copy per step (coeff.cu)
void coefficients_at(Handle& h, double e_mid, double e_lo, bool want_lo);

// ranks above 32 (wide.cu): 32-column blocks of an n-side matrix, the
// K-stage chained over blocks, the S-Grams over block pairs
std::vector<NMat> block_views(Handle& h, std::vector<NBuf>& bufs, int cols);
std::vector<NMat> split_blocks(Handle& h, NMat src, std::vector<NBuf>& bufs);
// balanced blocks of <= maxw columns of [X1 | X2] (the S-Gram pairs)
std::vector<NMat> split_joint(Handle& h, NMat X1, NMat X2, int maxw, std::vector<NBuf>& bufs);
void kstage_blocks(Handle& h, const std::vector<NMat>& X, NMat U0, const double* S0,
                   const double* M, const std::vector<NMat>& out, bool in_scaled,
                   bool out_scaled);
void stencil_grams_blocks(Handle& h, const std::vector<NMat>& B, const double* isp, double* G);

// rank-revealing pivoted Cholesky of the augmentation's small Gram (step.cu);
// mode 0 deflate, 1 re-orthogonalise, 2 deflated residuals, 3 level-2 scaled
void cholqr_build(const double* G, const double* C, int a, int b, int mode, double tol2,
                  const double* dinv, double* TA, double* TB, int* info, double* d0out,
                  DBuf& work, cudaStream_t st, const double* gate = nullptr);

// ranks above 64 (xwide.cu): column-blocked storage, every product a chain
// over 32-column blocks
using BMat = std::vector<NMat>;
struct XTerm {
  const BMat* in;
  const double* T;  // in.cols x out.cols row-major (ld: 0 = out.cols); null = identity
  double scale;
  int ld = 0;
};
BMat bview(Handle& h, std::vector<NBuf>& bufs, int cols);
int bcols(const BMat& m);
void bm_gram(Handle& h, const BMat& X, const BMat& Y, double* out, const double* w, bool sym);
void bm_lincomb(Handle& h, const std::vector<XTerm>& terms, const BMat& out);
void to_blocked(Handle& h);
void from_blocked(Handle& h);
void release_narrow(Handle& h);
void release_blocked(Handle& h);
BMat xstate_u(Handle& h);
BMat xstate_q(Handle& h);
void consolidate_x(Handle& h);
int orth_complement_x(Handle& h, const BMat& X, const double* C1, int rank_bound);
void streaming_step_x(Handle& h, double dt);
void scattering_step_x(Handle& h, double dt);
void rotate_x(Handle& h, const double* P, int p, int kcols, int r1, bool all_zero,
              double* ugram);
void dose_accumulate_x(Handle& h, const double* coef, double half_dt, const double* psi,
                       double* dep, double* prev);
double orth_defect_x(Handle& h, double* G, bool have_ugram);
void upload_blocked(Handle& h, const double* u, int ru);
void download_blocked(Handle& h, double* u, int ld);
int random_state_x(Handle& h, int r, unsigned long long seed);

// full-rank oracle on the device (fullrank.cu, fullrank.py:16-45)
void fullrank_reset(Handle& h);                    // u = 0
NMat fullrank_block(Handle& h, int b);             // columns [32 b, 32 b + 32)
int fullrank_blocks(const Handle& h);
void fullrank_streaming_step(Handle& h, double dt);
void fullrank_scattering_step(Handle& h, double dt);
void fullrank_dose_step(Handle& h, double dt, bool tally_steps);

void streaming_step(Handle& h, double dt);
void scattering_step(Handle& h, double dt);
// ugram (optional, r1 x r1): also form U1^T U1 in the rotation pass
void truncate(Handle& h, double theta, int rmin, int rmax, double* tail, int* rank,
              double* ugram = nullptr);
void dose_accumulate_step(Handle& h, double dt, bool tally_steps);
// have_ugram: U^T U is already in defect_gram_slot (from the last truncation)
double orth_defect(Handle& h, bool have_ugram = false);
double* defect_gram_slot(Handle& h, int ru, int rv);
// speculative steps: eligibility, snapshot + flag reset, and the one
// synchronisation (false: the prediction failed and the state is restored)
bool spec_eligible(Handle& h, int truncate_after);
void spec_begin(Handle& h);
bool spec_end(Handle& h, bool abort);
// Q (k columns) = orthonormal basis of (I - U U^T) X; C1 = U^T X (device, ua x b; null
// when U is empty). Returns k; the result is installed as the state's Q.
// rank_bound: an upper bound on rank(X) known from its construction (the
// scattering source rows); directions beyond it are rounding noise, so the
// graded-increment second level is skipped once k reaches it.
int orth_complement(Handle& h, NMat X, const double* C1, NMat X2 = NMat{},
                    int rank_bound = 1 << 30);

}  // namespace pnd
