// Internal header of libpndose_b200: handle, error plumbing, kernel entry
// points. The public C-ABI is include/pndose_b200.h.
//
// Device layout:
//   * n-side matrices (U, K, W, U^, TSQR workspace) are column-major with a
//     padded leading dimension `ld` (multiple of 32 doubles = 256 B), so a
//     warp's 32 consecutive cells of one column are one 256-byte segment;
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
// after every kernel launch: surface launch errors, count the launch
void launched();
long long launch_count();

// ------------------------------------------------------------ geometry
struct Geom {
  int nx, ny, nz;
  int n;          // cells
  int ld;         // padded leading dimension of n-side matrices
  double h[3];
  double ih[3];   // 1/h   (the stencil coefficients, no FP64 division in kernels)
  double i2h[3];  // 1/(2h)
  int na;         // number of active axes
  int axis[3];    // active axis ids in x, y, z order
  int ns;         // number of stencils = 2 * na (order: axis-major, + then -)
};

// stencil s -> (axis, plus)
__host__ __device__ inline int stencil_axis(const Geom& g, int s) { return g.axis[s >> 1]; }
__host__ __device__ inline bool stencil_plus(int s) { return (s & 1) == 0; }

// ------------------------------------------------------------ device buffers
struct DBuf {
  double* p = nullptr;
  size_t cap = 0;  // doubles
  double* get(size_t count);  // grow-only allocation
  void free_();
};

struct IBuf {
  int* p = nullptr;
  size_t cap = 0;
  int* get(size_t count);
  void free_();
};

// ------------------------------------------------------------ kernels API
// Gram engine (gram.cu): out[g][a][b] = sum_c X[c][a] * T_g[c][b]
enum GramGen { GEN_STENCIL = 0, GEN_WEIGHT = 1, GEN_SOURCE = 2, GEN_PLAIN = 3, GEN_LINCOMB = 4 };

struct GramArgs {
  Geom geo;
  const double* X; int ldx; int na;          // n x na col-major
  const double* Y; int ldy; int nb;          // n x nb col-major (stencil/weight/plain)
  int nphase;                                // number of Grams produced
  int gen;
  const double* inv_s;                       // (n)
  // weight generator: phase k uses w_k(c)
  const int* cls; const double* wtab; int n_cls; int wmode;  // see gram.cu
  // source generator: T[c][b] = N[cls][b%12] * inv_s[c] * psi[b/12][c]
  const double* psi; int ldpsi; int n_beams;
  // lincomb generator: T = Y TA - X TB (TA: ny x nb, TB: na x nb, row-major),
  // written to Yout (ld = ldo) when non-null; Y has ny columns
  int ny; const double* TA; const double* TB; double* Yout; int ldo;
  int self_phase;                            // phase whose A operand is T (-1: none)
  double* out;                               // per phase rows x nb (row-major), phases
                                             // concatenated; rows = nb for self_phase
};
void gram(GramArgs a, DBuf& partial, cudaStream_t st);
// engine.cu: DMMA chunk kernels behind gram() for GEN_STENCIL and GEN_LINCOMB
void stencil_grams(const GramArgs& a, DBuf& partial, cudaStream_t st);
void lincomb(const GramArgs& a, DBuf& partial, bool grams, cudaStream_t st);

// n-side streaming kernels (nside.cu)
struct KStageArgs {
  Geom geo;
  const double* X; int ldx; int xc;  // stencil input (xc cols)
  const double* U0; int ldu; int ra; // base U0 (ra cols), null -> no base
  const double* S0;                  // ra x r row-major (base = U0 S0)
  const double* M;                   // ns x xc x r row-major contraction matrices
  const double* inv_s;
  int r;                             // output columns
  double* out; int ldo;
  double* copy_u; int ldc;           // optional: copy of U0 (ra cols)
};
void kstage(const KStageArgs& a, cudaStream_t st);

// out (n x b) = X (n x a) * P (a x b row-major)  [+ options]
void rotate(const Geom& g, const double* X, int ldx, int a, const double* P, int b, double* out,
            int ldo, cudaStream_t st);
void rotate_ld(const Geom& g, const double* X, int ldx, int a, const double* P, int ldp, int b,
               double* out, int ldo, cudaStream_t st);

// scattering K1 = U0 S0 + dt * inv_s * sum_b psi_b * (N_cls . rows_b) into A[:, :r],
// U0 (ra cols) copied into A[:, r:r+ra]
void scat_k1(const Geom& g, const double* U0, int ldu, int ra, const double* S0, int r, double dt,
             const double* inv_s, const int* cls, const double* cls_atomic, const double* psi,
             int ldpsi, int n_beams, const double* rows /* B x 12 x r */, double* A, int lda,
             cudaStream_t st);

void apply_streaming_full(const Geom& g, const double* U, int ldu, int m, const double* inv_s,
                          const double* Acat /* ns x m x m */, double* W /* n x ns*m scratch */,
                          double* out, int ldo, cudaStream_t st);

void dose_accumulate(const Geom& g, const double* U, int ldu, const double* coef /* r */, int r,
                     double half_dt, const double* s_field, const double* psi, int ldpsi,
                     int n_beams, double* deposited, double* prev, cudaStream_t st);

void class_gather_inv(const int* cls, const double* class_val, int n, double* out_inv,
                      double* out_val, cudaStream_t st);
void psi_lerp(const double* values, int ldv, int n, int j0, double w0, int j1, double w1,
              double* out, cudaStream_t st);
void transpose_in(const double* src_rowmajor, int n, int c, double* dst, int ldd, cudaStream_t st);
void transpose_out(const double* src, int lds, int n, int c, double* dst_rowmajor,
                   cudaStream_t st);
void fill_zero(double* p, size_t count, cudaStream_t st);

// dense small / m-side kernels (dense.cu)
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

// S-phase RK4 on an (p x q) matrix: S' = -sum_s G_s S F_s (G: p x p, F: q x q)
void s_rk4(double* S, int p, int q, const double* G, const double* F, int ns, double dt,
           double* work, cudaStream_t st);

}  // namespace pnd
