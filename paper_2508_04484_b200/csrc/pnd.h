// Internal header of libpndose_b200: errors, geometry, device buffers, kernel
// entry points. The public C-ABI is include/pndose_b200.h.
//
// Device layout:
//   * n-side matrices (U0, the augmentation Q, the K-stage iterates, dK) are
//     CELL-MAJOR: row c holds the r coefficients of cell c contiguously, with
//     an even row stride rs (16-byte aligned rows). H zero rows precede row 0
//     and follow row n-1, so every stencil halo segment [c0 + off, c0 + off + CH)
//     is one contiguous, in-bounds block that a single cp.async.bulk copies;
//   * small and m-side matrices (S, Grams, V, A_d^+-) are dense row-major,
//     exactly the numpy C-order the Python boundary passes in.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#define PND_OK 0
#define PND_ECONFIG 2
#define PND_EPHYSICS 3
#define PND_ENUMERICAL 4
#define PND_EIO 5
#define PND_EDEVICE 6

namespace pnd {

struct Error {
  int code;
  std::string msg;
};

// thrown inside the library, caught at the C-ABI boundary
[[noreturn]] void fail(int code, const std::string& msg);
void check_cuda(cudaError_t e, const char* what);
#define CK(x) ::pnd::check_cuda((x), #x)

// Allow a kernel the device's whole opt-in shared memory (227 KB). The
// attribute is a per-function cap shared by every host thread, so it is set
// to the maximum once instead of to each launch's size (a per-launch value
// would let a concurrent smaller launch on another handle shrink the cap
// under a larger one).
constexpr int kMaxDynSmem = 227 * 1024;
int max_smem_optin();  // cudaDevAttrMaxSharedMemoryPerBlockOptin of the current device
// Both queries below are cached per kernel (and launch shape): the driver
// calls cost microseconds each, paid on every launch of the launch-bound small
// problems otherwise.
bool smem_set_once(const void* fn);   // true the first time fn is seen
template <class F>
inline void allow_max_smem(F* fn) {
  if (!smem_set_once((const void*)fn)) return;
  cudaFuncAttributes fa{};
  check_cuda(cudaFuncGetAttributes(&fa, (const void*)fn), "cudaFuncGetAttributes");
  check_cuda(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  max_smem_optin() - (int)fa.sharedSizeBytes),
             "cudaFuncSetAttribute");
}
// cudaOccupancyMaxActiveBlocksPerMultiprocessor, cached per (kernel, threads, smem); >= 1
int occupancy_cached(const void* fn, int threads, size_t smem);
// after every kernel launch: surface launch errors, count the launch
void launched();
long long launch_count();
int sm_count();

// ------------------------------------------------------------ geometry
struct Geom {
  int nx, ny, nz;
  int n;          // cells
  int ld;         // padded length of per-cell vectors (inv_s, psi, dose)
  int halo;       // zero rows before/after every n-side matrix
  double h[3];
  double ih[3];   // 1/h   (the stencil coefficients, no FP64 division in kernels)
  double i2h[3];  // 1/(2h)
  int na;         // number of active axes
  int axis[3];    // active axis ids in x, y, z order (the first has stride 1)
  int ns;         // number of stencils = 2 * na (order: axis-major, + then -)
  // z-slab of a multi-GPU grid (comm.cu): this device holds global planes
  // [z0, z0 + nz) of nzg; comm != null -> halo planes and Gram sums go over NCCL
  int z0 = 0;
  int nzg = 0;    // 0: single device (nzg = nz)
  double inv_nx = 0.0, inv_nxy = 0.0;  // 1/nx, 1/(nx ny): cell -> (i, j, k) without division
  // the same by integer reciprocals: q = umulhi64(c, m) for c < 2^32 with
  // m = floor((2^64 - 1) / d) + 1 (d >= 2; m = 0 marks d = 1)
  unsigned long long mnx = 0, mnxy = 0;
  void* comm = nullptr;
  // 1/S is the same in every cell (one material class): the stencil Grams then
  // form only the D+ stencils and take D- = -(D+)^T + boundary rows (stencil.cu)
  int uniform_s = 0;
};

// ------------------------------------------------------------ slab communication (comm.cu)
struct Comm;
void comm_unique_id(char* out128);
Comm* comm_create(const char* id128, int rank, int world);
void comm_destroy(Comm* c);
// ranks of the slab communicator (1 without one)
int comm_world(const Geom& g);
// sum a small device block over the slabs (no-op on one device)
void comm_allreduce(const Geom& g, double* p, size_t count, cudaStream_t st);
// fill the 2-plane halo rows of an n-side matrix from the neighbouring slabs
void comm_halo_rows(const Geom& g, double* rows, int rs, cudaStream_t st);

// ------------------------------------------------------------ device buffers
struct DBuf {
  double* p = nullptr;
  size_t cap = 0;  // doubles
  double* get(size_t count);  // grow-only allocation (contents not preserved)
  void free_();
};

struct IBuf {
  int* p = nullptr;
  size_t cap = 0;
  int* get(size_t count);
  void free_();
};

// cell-major n-side matrix view: element (cell c, column j) at p[c * rs + j]
struct NMat {
  double* p = nullptr;
  int rs = 0;
  int cols = 0;
};

// owner of one n-side matrix buffer (halo rows kept zero for the current rs)
struct NBuf {
  DBuf d;
  int rs = -1;
  // a view with `cols` columns (rs = cols rounded up to even); the contents
  // survive when the stride does not change
  NMat view(const Geom& g, int cols, cudaStream_t st);
};

inline int even(int c) { return (c + 1) & ~1; }

// ------------------------------------------------------------ n-side kernels (stencil.cu, nside.cu)
// K-phase Horner stage / full-rank streaming operator:
//   out = [D_0 S^-1 X, ..., D_ns-1 S^-1 X | U0] . [M_0; ...; M_ns-1; S0]
struct KStageArgs {
  Geom geo;
  NMat X;             // stencil input (xc = X.cols)
  NMat U0;            // base rows (ra = U0.cols), p == nullptr -> no base
  const double* S0;   // ra x r row-major
  const double* M;    // ns x xc x r row-major contraction matrices
  const double* inv_s;
  NMat out;           // r = out.cols
  DBuf* bcat = nullptr;     // per-handle scratch for the fragment-ordered [M; S0]
  bool in_scaled = false;   // X holds S^-1 x (the Horner intermediates)
  bool out_scaled = false;  // store S^-1 out instead of out
  int zpart = 0;            // 0: all cells; 1: planes 2 .. nz-3; 2: planes 0, 1, nz-2, nz-1
};
void kstage(const KStageArgs& a, cudaStream_t st);
// the plane split of kstage applies (whole chunks per plane, nz >= 5)
bool kstage_can_split(const Geom& g);

// stencil Grams: out[s] = [X1 | X2]^T D_s S^-1 [X1 | X2]  (ns x w x w, w = X1.cols + X2.cols)
void stencil_grams(const Geom& g, NMat X1, NMat X2, const double* inv_s, double* out,
                   DBuf& partial, cudaStream_t st);
// one material class: the D- stencil Grams from the D+ ones (out holds the D+
// Grams in its even slots): D- = -(D+)^T + boundary rows, per axis
void minus_from_plus(const Geom& g, NMat X1, NMat X2, const double* isp, double* out,
                     DBuf& partial, cudaStream_t st);
// rectangular stencil Grams of two <= 32-column blocks, placed into an
// ns x w x w Gram at rows r0.., columns c0..: G_s[r0 + i][c0 + j] = (XA^T D_s S^-1 XB)_ij
// (not summed over slabs: the caller allreduces the assembled Gram)
void stencil_grams_rect(const Geom& g, NMat XA, NMat XB, const double* isp, double* G, int w,
                        int r0, int c0, DBuf& partial, cudaStream_t st);
// general stencil Grams for the unit API: out[s] = X^T D_s S^-1 Y
void stencil_grams_xy(const Geom& g, NMat X, NMat Y, const double* inv_s, double* out,
                      DBuf& partial, cudaStream_t st);

// out = [Y1 | Y2] TA - X TB (rows written when out.p != null) and, when grams != null,
// grams = [X^T out (X.cols x nb) ; out^T out (nb x nb)]. TA == nullptr means
// TA = I (out = [Y1 | Y2] - X TB: the Y rows are added, not multiplied).
void lincomb(const Geom& g, NMat Y1, NMat Y2, NMat X, const double* TA, const double* TB,
             NMat out, double* grams, DBuf& partial, cudaStream_t st);
// Gram out = X^T diag(w) Y (X.cols x Y.cols, row-major; w = null: plain) in one
// streaming pass (lincomb.cu)
void gram_xy(const Geom& g, NMat X, NMat Y, double* out, DBuf& partial, cudaStream_t st,
             const double* w = nullptr);
// out = X^T diag(w) [Y1 | Y2] (X.cols x (Y1.cols + Y2.cols)) in one pass
void gram_xy2(const Geom& g, NMat X, NMat Y1, NMat Y2, double* out, DBuf& partial,
              cudaStream_t st, const double* w = nullptr);
// Z[c][b*12 + i] = N_{cls(c),i} psi_b(c) / S(c): the scattering source rows (dlra.py:244-251)
void source_rows(const Geom& g, const double* inv_s, const int* cls, const double* cls_atomic,
                 const double* psi, int n_beams, NMat Z, cudaStream_t st);

// pointwise Grams
enum PGen { PG_PLAIN = 0, PG_WEIGHT = 1, PG_SOURCE = 2 };
struct PGramArgs {
  Geom geo;
  NMat X;                 // A operand (na = X.cols)
  NMat Y;                 // plain / weight input
  int nb;                 // T columns
  int nphase;
  int gen;
  const double* inv_s;
  const int* cls;
  const double* wtab;     // class x 12 atomic densities
  int wmode;              // weight: 0 class indicator, 1 wtab[cls][phase]
  const double* psi;      // source: n_beams x ld
  int ld;
  double* out;            // nphase x na x nb
};
void pgram(const PGramArgs& a, DBuf& partial, cudaStream_t st);

// dK = dt * inv_s * sum_b psi_b * (N_cls . rows_b)  (scattering source rows, dlra.py:244-251)
void scat_dk(const Geom& g, double dt, const double* inv_s, const int* cls,
             const double* cls_atomic, int n_cls, const double* psi, int n_beams,
             const double* rows /* B x 12 x r */, NMat out, cudaStream_t st);

void dose_accumulate(const Geom& g, NMat U, const double* coef /* U.cols */, double half_dt,
                     const double* s_field, const double* psi, int n_beams, double* deposited,
                     double* prev, cudaStream_t st);

void unit_rows(const Geom& g, NMat U, cudaStream_t st);        // U[:, j] = e_j
void random_rows(const Geom& g, NMat U, unsigned long long seed, cudaStream_t st);
void class_gather_inv(const int* cls, const double* class_val, int n, double* out_inv,
                      double* out_val, cudaStream_t st);
// psi = w0 lat depth[:, j0] + w1 lat depth[:, j1] of a separable table (the same
// arithmetic as psi_lerp on the expanded table); sel_j/sel_w: device selections
// (nullptr: the host scalars)
void psi_lerp_separable(const double* lat, const double* depth, int nxy, int G, int n,
                        const int* sel_j, const double* sel_w, int j0, double w0, int j1,
                        double w1, double* out, cudaStream_t st);
void psi_lerp(const double* values, int ldv, int n, int j0, double w0, int j1, double w1,
              double* out, cudaStream_t st);
// sparse (ray-footprint) table: out = 0, then out[cells[i]] = w0 v[i][j0] + w1 v[i][j1]
// (v: nnz x G row-major; sel_j / sel_w on the device, or the host scalars)
void psi_lerp_sparse(const int* cells, const double* values, int nnz, int G, int n,
                     const int* sel_j, const double* sel_w, int j0, double w0, int j1, double w1,
                     double* out, cudaStream_t st);
// row-major host-layout (n x c) <-> column-major (ld) device layout (flux tables, TSQR)
void transpose_in(const double* src_rowmajor, int n, int c, double* dst, int ldd, cudaStream_t st);
void transpose_out(const double* src, int lds, int n, int c, double* dst_rowmajor,
                   cudaStream_t st);
void fill_zero(double* p, size_t count, cudaStream_t st);

// ------------------------------------------------------------ dense small / m-side (dense.cu)
struct Mat {  // strided matrix view: element (i, j) at p[i * rs + j * cs]
  double* p;
  long rs, cs;
};
inline Mat rowm(double* p, int ncols) { return Mat{p, ncols, 1}; }
inline Mat colm(double* p, int ld) { return Mat{p, 1, ld}; }
inline Mat tr(Mat a) { return Mat{a.p, a.cs, a.rs}; }

// C[b] = alpha * A[b] B[b] + beta * C[b], b < batch (batch strides in doubles)
void gemm(int M, int N, int K, double alpha, Mat A, long sA, Mat B, long sB, double beta, Mat C,
          long sC, int batch, cudaStream_t st);
void axpby(int count, double a, const double* x, double b, double* y, cudaStream_t st);

// TSQR of an (rows x cols) column-major matrix, rows >= 1. On return `q`
// (rows x min(rows, cols), ld = ldq) holds the explicit orthonormal factor and
// `rfac` (min(rows,cols) x cols row-major) the triangular factor.
struct TsqrWork {
  DBuf tau, tree, rbuf, cbuf;
  std::vector<int> level_nodes;
};
int tsqr(double* a, int rows, int cols, int lda, double* q, int ldq, double* rfac, TsqrWork& w,
         cudaStream_t st);

// one-CTA Jacobi SVD of (p x q row-major) s: s = P diag(sig) Qt, k = min(p, q)
void svd_small(const double* s, int p, int q, double* P /* p x k */, double* sig /* k */,
               double* Qt /* k x q */, double* work, cudaStream_t st);

// truncation rule on sigma (device) -> info[0] = r1 (or -r1raw-1 on rank_max), tail
void tail_rule(const double* sig, int k, double theta, int rmin, int rmax, int* info,
               double* tail, cudaStream_t st);

// batched implicit solves of scattering substep 1 (dlra.py:286-298)
void scat_solves(const double* B /* 12 x r x r */, const double* coeffs /* 12 x m */,
                 const double* lcols /* r x m */, int r, int m, double dt, double* lnew /* r x m */,
                 int* singular_col, cudaStream_t st);

// L-phase RK4 of the streaming substep, fused (one cluster launch) when the
// moment count is small: L1 (m x a row-major) and BV = [L1 | V] column-major;
// false = not applicable (the GEMM path is used)
bool l_rk4(const double* V, const double* S, const double* G, int ru, const double* amat, int m,
           int a, int b, int ns, double dt, double* L1, double* BV, cudaStream_t st);
// S-phase RK4 on an (p x q) matrix: S' = -sum_s G_s S F_s (G: p x p, F: q x q)
void s_rk4(double* S, int p, int q, const double* G, const double* F, int ns, double dt,
           double* work, cudaStream_t st);

// uncollided energy march + deposit (march.cu)
void march_steppers(int nl, const double* D, const double* L, const double* U, const double* mass,
                    int ng, int n_steppers, const int* key, const double* dz, double* Dinv,
                    double* E, int* bad, cudaStream_t st);
void march_rays(int nl, const double* D, const double* L, const double* U, const double* mass,
                int ng, const double* Dinv, const double* E, const double* st_dz, int n_marches,
                const int* seg_off, const int* seg_key, const double* half_dz, const int* half_n,
                const int* half_st, const double* s_min, double e_min, const double* psi0,
                const double* p_lo, double* psi, double* tmp, double* averages,
                double* residual, int* bad, cudaStream_t st);
void deposit_rays(int n_rays, const int* ray_seg_off, const long long* cells,
                  const double* lengths, const int* ray_march, const int* march_seg_off,
                  const double* weight, double volume, const double* averages,
                  const double* mres, double* values, int ld, double* residual, int ng,
                  cudaStream_t st);

// per-element Legendre moments of the screened kernel on an energy grid
// (moments.cu, moliere.py:111-147): g (n_el x n_e x (L+1)), xi1 (n_el x n_e);
// returns -1, or the first element * n_e + energy whose quadrature failed rtol
int moment_tables(const double* energies, int n_e, const int* z, const int* a, int n_el,
                  const double* x1, const double* w1, const double* x2, const double* w2, int nn,
                  int max_degree, double exponent, double rtol, double* g, double* xi1,
                  cudaStream_t st);

// ray traversal (trace.cu)
void traverse(const Geom& g, const double* origin, int n_rays, const double* starts,
              const double* dirs, int* counts, const long long* offsets, long long* cells,
              double* t0, double* t1, cudaStream_t st);

}  // namespace pnd
