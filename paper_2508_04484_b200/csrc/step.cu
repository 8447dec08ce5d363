// Orchestration of one pseudo-time (energy) step on the device.
//
// Shapes follow the reference: U0 (n x a), S0 (a x b), V0 (m x b).
//
// Horner RK4. Every RK4 here integrates a linear autonomous right-hand side
// (K, L and S phases, dlra.py:118-123), for which classic RK4 equals
//   y1 = y0 + h L (y0 + h/2 L (y0 + h/3 L (y0 + h/4 L y0)))
// exactly in exact arithmetic: 4 passes over n-side data instead of the
// classic scheme's 4 evaluations plus 3 combinations.
//
// Augmentation. The reference orthonormalises [K1, U0] with Householder QR
// (dlra.py:26-43, 220, 304). Since U0 is already orthonormal and
// K1 = U0 S0 + dK, span[K1, U0] = span[U0, dK]; the device builds
// U^ = [U0 | Q] with Q an orthonormal basis of (I - U0 U0^T) dK, where dK is
// the increment itself (the last Horner stage without its base, or the
// scattering source term), so no cancellation against U0 S0 occurs. Q comes
// from Gram passes only (block classical Gram-Schmidt with reorthogonalisation
// + SVQB, Stathopoulos & Wu 2002): directions of the projected increment below
// 1e-7 of its largest singular value (numerical noise for a one-pass Gram
// method) are deflated rather than normalised into noise directions. Then
// U^T U0 = [I; 0] exactly, and the truncation handles the exact-zero case
// (S^ == 0) with the reference's canonical basis.
// The moment side (m x 2r, small) keeps Householder TSQR.
#include <cmath>
#include <cstring>

#include "handle.h"

namespace pnd {

namespace {

enum Slot {
  S_FV, S_MST, S_YST, S_HU, S_QV, S_L0, S_LW, S_ZST, S_BV, S_VHC, S_RV, S_SHAT, S_G,
  S_FH, S_VHR, S_GT, S_ROWS, S_H, S_BI, S_COEF, S_LCOL, S_LNEW, S_RT, S_VTC, S_LEFT, S_PROJ,
  S_PROJ2, S_GTV, S_P, S_SIG, S_QTM, S_TAIL, S_DEF, S_COEFD, S_VNEW, S_M2,
  S_C1, S_OG, S_OTA, S_OTB, S_EYE, S_PC, S_TAZ, S_COUNT
};
static_assert(S_COUNT <= 43, "slots 43..47 are reserved by abi.cu");

double* slot(Handle& h, int s, size_t count) { return h.sm[s].get(count > 0 ? count : 1); }

void need(bool ok, const char* what) {
  if (!ok) fail(PND_ECONFIG, std::string("handle is missing ") + what);
}

// F_s(W) = W^T A_s W for every stencil s; W row-major (m x c) -> out ns x c x c
void moment_factors(Handle& h, double* W, int c, double* out) {
  const int m = h.m, ns = h.g.ns;
  double* Y = slot(h, S_YST, (size_t)ns * m * c);
  gemm(ns * m, c, m, 1.0, rowm(h.amat.p, m), 0, rowm(W, c), 0, 0.0, rowm(Y, c), 0, 1, h.st);
  gemm(c, c, m, 1.0, tr(rowm(W, c)), 0, rowm(Y, c), (long)m * c, 0.0, rowm(out, c), (long)c * c,
       ns, h.st);
}

__global__ void eye_kernel(double* I, int b) {
  for (int i = threadIdx.x; i < b * b; i += blockDim.x) I[i] = (i / b == i % b) ? 1.0 : 0.0;
}

__global__ void zero_rows_kernel(double* S, int row0, int rows, int cols) {
  for (int i = threadIdx.x; i < rows * cols; i += blockDim.x) S[(size_t)row0 * cols + i] = 0.0;
}

__global__ void isp_kernel(const double* inv_s, int n, double* isp) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    isp[2 * c] = inv_s[c];
    isp[2 * c + 1] = 0.0;
  }
}

double* eye(Handle& h, int b) {
  double* I = slot(h, S_EYE, (size_t)b * b);
  eye_kernel<<<1, 256, 0, h.st>>>(I, b);
  launched();
  return I;
}

// max(|G - I|, |C|) (the block's orthonormality defect) into out[0]
__global__ void defect_gc_kernel(const double* G, const double* C, int a, int b, double* out) {
  __shared__ double red[256];
  double d = 0.0;
  for (int i = threadIdx.x; i < b * b + a * b; i += blockDim.x) {
    const double v = i < b * b ? fabs(G[i] - ((i / b == i % b) ? 1.0 : 0.0)) : fabs(C[i - b * b]);
    d = v > d ? v : d;
  }
  red[threadIdx.x] = d;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

// Level 2 of the augmentation (graded increments). W = [Q | Z] from
// cholqr mode 2, G3 = W^T W, C3 = U0^T W formed from the explicit vectors, so
// every entry is accurate to eps |w_i| |w_j| -- unlike the level-1 Gram, whose
// small directions are lost below eps |Y|^2. M = G3 - C3^T C3 (W projected out
// of U0); the columns kept are Q's and every Z column with norm above
// *floor_p (1e-13 |X|_F: the rounding noise of forming and projecting the
// increment X = U0 C1 + Y is ~eps |X|, so only real content passes);
// Ms = D^-1 M_JJ D^-1 (unit diagonal, zero rows and columns outside J) is
// the well-conditioned Gram of the scaled columns.
__global__ void level2_gram(const double* G3, const double* C3, int a, int b, int k1, int kb,
                            const double* floor_p, double* Ms, double* dinv) {
  const int tid = threadIdx.x;
  __shared__ double d[512];
  const double floor_abs = *floor_p;
  for (int j = tid; j < b; j += blockDim.x) {
    double mjj = G3[j * b + j];
    for (int t = 0; t < a; ++t) mjj -= C3[t * b + j] * C3[t * b + j];
    const double nj = mjj > 0.0 ? sqrt(mjj) : 0.0;
    d[j] = nj;
  }
  __syncthreads();
  // at most kb - k1 of the deflated columns can be real when the increment's
  // rank is known to be <= kb: the largest residuals above the floor
  for (int j = tid; j < b; j += blockDim.x) {
    const double nj = d[j];
    int above = 0;
    for (int i = k1; i < b; ++i) above += d[i] > nj || (d[i] == nj && i < j);
    const bool keep = j < k1 || (above < kb - k1 && nj > floor_abs);
    dinv[j] = keep ? 1.0 / nj : 0.0;
  }
  __syncthreads();
  for (int j = tid; j < b; j += blockDim.x) d[j] = dinv[j];
  __syncthreads();
  for (int i = tid; i < b * b; i += blockDim.x) {
    const int r = i / b, c = i % b;
    double v = G3[i];
    for (int t = 0; t < a; ++t) v -= C3[t * b + r] * C3[t * b + c];
    Ms[i] = v * d[r] * d[c];
  }
}

// out[0] = rel * |X|_F, |X|_F^2 = trace(Y^T Y) + |U0^T X|_F^2 (the level-2 floor)
__global__ void xnorm_kernel(const double* G2, const double* C1, int a, int b, double rel,
                             double* out) {
  __shared__ double red[256];
  const int tid = threadIdx.x;
  double x2 = 0.0;
  for (int j = tid; j < b; j += blockDim.x) x2 += G2[j * b + j];
  if (C1)
    for (int i = tid; i < a * b; i += blockDim.x) x2 += C1[i] * C1[i];
  red[tid] = x2;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (tid < w) red[tid] += red[tid + w];
    __syncthreads();
  }
  if (tid == 0) out[0] = rel * sqrt(red[0] > 0.0 ? red[0] : 0.0);
}

}  // namespace

// Rank-revealing pivoted Cholesky of the small Gram of the augmentation
// (CholeskyQR with diagonal pivoting): G = P R^T R P^T,
// pivots taken while the largest remaining diagonal -- the squared residual
// norm of that column after projecting out the columns already taken --
// exceeds tol2 x the first pivot. Every column left out therefore has a
// residual below sqrt(tol2) of the largest column (the deflation guarantee the
// second level builds on). Replaces an eigen-decomposition (SVQB) of the same
// Gram: one pass over b^2 entries instead of Jacobi sweeps.
//   mode 0: TA (b x k) = P_J R^-1, so Q = (Y - U0 C) TA has orthonormal columns
//   mode 1: the same without the deflation threshold (re-orthogonalisation)
//   mode 2: TA (b x b) = [P_J R^-1 | e_rest - P_J G_JJ^-1 G_J,rest]: the
//           deflated columns' residuals after Q, unnormalised (level 2 input)
//   mode 3: G is the unit-scaled level-2 Gram (dinv: the column scales):
//           TA (b x k) = D^-1 P_J R^-1
// TB = C TA (a x ncol); info[0] = k. work: 2 b^2 doubles (global) when the
// matrices do not fit in shared memory.
__global__ void __launch_bounds__(256)
    cholqr_kernel(const double* __restrict__ G, const double* __restrict__ C, int a, int b,
                  int mode, double tol2, const double* __restrict__ dinv, double* TA,
                  double* TB, int* info, double* d0out, double* work, int in_smem,
                  const double* __restrict__ gate) {
  // gate (speculative steps): the re-orthogonalisation is not needed when the
  // block's defect is within the 1e-12 trigger -- spec_select_kernel then
  // supplies TA = I, TB = 0
  if (gate && gate[0] <= 1e-12) return;
  extern __shared__ double sm[];
  double* A = in_smem ? sm : work;               // b x b working copy (R in its upper part)
  double* Ri = A + (size_t)b * b;                // k x k inverse of R
  __shared__ int perm[512];
  __shared__ int k_s, piv_s;
  __shared__ double d0_s;
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < b * b; i += nthr) A[i] = G[i];
  for (int i = tid; i < b; i += nthr) perm[i] = i;
  if (tid == 0) {
    k_s = b;
    d0_s = 0.0;
  }
  __syncthreads();
  for (int j = 0; j < b; ++j) {
    if (warp == 0) {
      double best = -1.0;
      int bi = j;
      for (int i = j + lane; i < b; i += 32) {
        const double v = A[(size_t)i * b + i];
        if (v > best) { best = v; bi = i; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (lane == 0) {
        if (j == 0) d0_s = best;
        const double d0 = j == 0 ? best : d0_s;
        if (!(best > 0.0) || best <= tol2 * d0) k_s = j;
        piv_s = bi;
      }
    }
    __syncthreads();
    if (k_s == j) break;
    const int p = piv_s;
    if (p != j) {  // symmetric swap of rows / columns j and p
      for (int i = tid; i < b; i += nthr) {
        const double t = A[(size_t)j * b + i];
        A[(size_t)j * b + i] = A[(size_t)p * b + i];
        A[(size_t)p * b + i] = t;
      }
      __syncthreads();
      for (int i = tid; i < b; i += nthr) {
        const double t = A[(size_t)i * b + j];
        A[(size_t)i * b + j] = A[(size_t)i * b + p];
        A[(size_t)i * b + p] = t;
      }
      if (tid == 0) {
        const int t = perm[j];
        perm[j] = perm[p];
        perm[p] = t;
      }
      __syncthreads();
    }
    const double rjj = sqrt(A[(size_t)j * b + j]);
    __syncthreads();
    if (tid == 0) A[(size_t)j * b + j] = rjj;
    for (int i = j + 1 + tid; i < b; i += nthr) A[(size_t)j * b + i] /= rjj;
    __syncthreads();
    const int w = b - j - 1;
    for (int e = tid; e < w * w; e += nthr) {
      const int r = j + 1 + e / w, c = j + 1 + e % w;
      A[(size_t)r * b + c] -= A[(size_t)j * b + r] * A[(size_t)j * b + c];
    }
    __syncthreads();
  }
  const int k = k_s;
  if (tid == 0) {
    info[0] = k;
    if (d0out) d0out[0] = d0_s;
  }
  // R^-1 (k x k upper), one column per thread: R x = e_c by back substitution
  for (int c = tid; c < k; c += nthr) {
    for (int r = k - 1; r >= 0; --r) {
      double v = r == c ? 1.0 : 0.0;
      for (int t = r + 1; t <= c; ++t) v -= A[(size_t)r * b + t] * Ri[(size_t)t * k + c];
      Ri[(size_t)r * k + c] = r > c ? 0.0 : v / A[(size_t)r * b + r];
    }
  }
  __syncthreads();
  const int ncol = mode == 2 ? b : k;
  for (int e = tid; e < b * ncol; e += nthr) TA[e] = 0.0;
  __syncthreads();
  for (int e = tid; e < k * k; e += nthr) {
    const int i = e / k, c = e % k;
    const double sc = mode == 3 ? dinv[perm[i]] : 1.0;
    TA[(size_t)perm[i] * ncol + c] = sc * Ri[e];
  }
  if (mode == 2) {
    // rest column t (original index q = perm[k + t]): e_q - P_J c, c = R^-1 R^-T G[J, q]
    for (int t = tid; t < b - k; t += nthr) {
      const int q = perm[k + t];
      double y[512 / 8];  // R^-T g, chunked: k <= 64 in registers, else recomputed
      if (k <= 64) {
        for (int i = 0; i < k; ++i) {
          double v = 0.0;
          for (int l = 0; l <= i; ++l) v += Ri[(size_t)l * k + i] * G[(size_t)perm[l] * b + q];
          y[i] = v;
        }
        for (int i = 0; i < k; ++i) {
          double v = 0.0;
          for (int l = i; l < k; ++l) v += Ri[(size_t)i * k + l] * y[l];
          TA[(size_t)perm[i] * ncol + k + t] = -v;
        }
      } else {
        for (int i = 0; i < k; ++i) {
          double v = 0.0;
          for (int l = i; l < k; ++l) {
            double yl = 0.0;
            for (int m = 0; m <= l; ++m) yl += Ri[(size_t)m * k + l] * G[(size_t)perm[m] * b + q];
            v += Ri[(size_t)i * k + l] * yl;
          }
          TA[(size_t)perm[i] * ncol + k + t] = -v;
        }
      }
      TA[(size_t)q * ncol + k + t] = 1.0;
    }
  }
  __syncthreads();
  for (int e = tid; e < a * ncol; e += nthr) {
    const int r = e / ncol, c = e % ncol;
    double v = 0.0;
    for (int j = 0; j < b; ++j) v += C[(size_t)r * b + j] * TA[(size_t)j * ncol + c];
    TB[e] = v;
  }
}

void cholqr_build(const double* G, const double* C, int a, int b, int mode, double tol2,
                  const double* dinv, double* TA, double* TB, int* info, double* d0out,
                  DBuf& work, cudaStream_t st, const double* gate) {
  if (b > 512) fail(PND_ECONFIG, "augmentation block wider than 512 columns");
  const size_t need = 2 * (size_t)b * b * sizeof(double);
  const bool in_smem = need + 8192 <= (size_t)kMaxDynSmem;
  double* w = nullptr;
  if (in_smem) {
    static bool init = false;
    if (!init) {
      allow_max_smem(cholqr_kernel);
      init = true;
    }
  } else {
    w = work.get(2 * (size_t)b * b);
  }
  cholqr_kernel<<<1, 256, in_smem ? need : 0, st>>>(G, C, a, b, mode, tol2, dinv, TA, TB, info,
                                                   d0out, w, in_smem ? 1 : 0, gate);
  launched();
}

NMat state_u(Handle& h) { return h.U.view(h.g, h.ua, h.st); }
NMat state_q(Handle& h) {
  if (h.uq <= 0) return NMat{};
  return h.Q.view(h.g, h.uq, h.st);
}

void set_isp(Handle& h) {
  const size_t rows = (size_t)h.g.n + 2 * (size_t)h.g.halo;
  if (h.isp.cap < 2 * rows) {
    h.isp.get(2 * rows);
    fill_zero(h.isp.p, 2 * rows, h.st);
  }
  isp_kernel<<<148 * 8, 256, 0, h.st>>>(h.inv_s.p, h.g.n, h.isp.p + 2 * (size_t)h.g.halo);
  launched();
  comm_halo_rows(h.g, h.isp.p + 2 * (size_t)h.g.halo, 2, h.st);  // slab faces
}

static const double* isp_rows(Handle& h) { return h.isp.p + 2 * (size_t)h.g.halo; }

void consolidate(Handle& h) {
  if (h.uq <= 0) return;
  if (h.blocked || h.ua + h.uq > 64) {  // ranks above 64: the blocked layout (xwide.cu)
    to_blocked(h);
    consolidate_x(h);
    return;
  }
  const int ru = h.ua + h.uq;
  NMat u = state_u(h), q = state_q(h);
  NMat out = h.Un.view(h.g, ru, h.st);
  lincomb(h.g, u, q, NMat{}, eye(h, ru), nullptr, out, nullptr, h.part, h.st);
  std::swap(h.U, h.Un);
  h.ua = ru;
  h.uq = 0;
}

// the scattering step's implicit solves report a singular column through a
// flag read back with the next synchronisation (the augmentation's)
void check_singular(Handle& h) {
  if (!h.singular_pending) return;
  h.singular_pending = false;
  const int singular = *(int*)(h.pinned + 10);
  if (singular != (1 << 30)) {
    fail(PND_ENUMERICAL, "implicit scattering solve singular at moment column " +
                             std::to_string(singular) +
                             "; the step size is too large for the scattering stiffness");
  }
}

// ------------------------------------------------------------ speculative steps
namespace {
// flag[0] |= the device-side decision differs from the host's prediction
__global__ void spec_check_kernel(const int* got, int want, int* flag) {
  if (threadIdx.x == 0 && got[0] != want) atomicOr(flag, 1);
}
__global__ void spec_check_trunc_kernel(const int* r1, const double* sig, int want, int* flag) {
  if (threadIdx.x == 0 && (r1[0] != want || sig[0] == 0.0)) atomicOr(flag, 2);
}
// the re-orthogonalisation pass of orth_complement, predicated on the device:
// when the block's defect is within the trigger the pass applies TA = I,
// TB = 0 (Q TA - U0 TB = Q exactly)
__global__ void spec_select_kernel(const double* defect, double trigger, int a, int k, double* TA,
                                   double* TB) {
  if (defect[0] > trigger) return;
  for (int i = threadIdx.x; i < k * k; i += blockDim.x) TA[i] = (i / k == i % k) ? 1.0 : 0.0;
  for (int i = threadIdx.x; i < a * k; i += blockDim.x) TB[i] = 0.0;
}
}  // namespace

// orth_complement after its pass-2 pivoted Cholesky, without a host round
// trip: the increment is predicted to be full (k = min(b, rank_bound): no
// deflated column, so no second level), the device checks the prediction,
// and the re-orthogonalisation pass always runs, predicated by its defect.
static int orth_complement_spec(Handle& h, NMat Y, NMat U0, int a, int b, int rank_bound,
                                double* grams, double* TA, double* TB, int* info,
                                double* dinfo) {
  const Geom& g = h.g;
  cudaStream_t st = h.st;
  const int k = b < rank_bound ? b : rank_bound;
  spec_check_kernel<<<1, 32, 0, st>>>(info, k, h.spec_flag.p);
  launched();
  NMat Qv = h.Q.view(g, k, st);
  lincomb(g, Y, NMat{}, U0, TA, TB, Qv, grams, h.part, st);
  double* C3 = grams;
  double* G3 = grams + (size_t)a * k;
  defect_gc_kernel<<<1, 256, 0, st>>>(G3, C3, a, k, dinfo);
  launched();
  double* G3c = slot(h, S_M2, (size_t)k * k);
  CK(cudaMemcpyAsync(G3c, G3, sizeof(double) * k * k, cudaMemcpyDeviceToDevice, st));
  if (a > 0) gemm(k, k, a, -1.0, tr(rowm(C3, k)), 0, rowm(C3, k), 0, 1.0, rowm(G3c, k), 0, 1, st);
  cholqr_build(G3c, C3, a, k, 1, 0.0, nullptr, TA, TB, info + 1, nullptr, h.cq_work, st, dinfo);
  spec_select_kernel<<<1, 256, 0, st>>>(dinfo, 1e-12, a, k, TA, TB);
  launched();
  NMat Q2 = h.Qa.view(g, k, st);
  lincomb(g, Qv, NMat{}, U0, TA, TB, Q2, nullptr, h.part, st);
  std::swap(h.Q, h.Qa);
  h.uq = k;
  return k;
}

int orth_complement(Handle& h, NMat X, const double* C1, NMat X2, int rank_bound) {
  const int a = h.ua, b = X.cols + (X2.p ? X2.cols : 0);
  cudaStream_t st = h.st;
  const Geom& g = h.g;
  NMat U0 = a > 0 ? state_u(h) : NMat{};
  double* grams = slot(h, S_OG, (size_t)b * (a + b));
  double* TA = slot(h, S_OTA, (size_t)b * b);
  double* TB = slot(h, S_OTB, (size_t)(a > 0 ? a : 1) * b);
  double* sig = slot(h, S_SIG, (size_t)b + 2);
  int* info = h.iflag.get(8);
  double* dinfo = slot(h, S_TAIL, 4);
  // pass 2: Y = X - U0 C1 -> Qa, C2 = U0^T Y, G2 = Y^T Y
  NMat Y = h.Qa.view(g, b, st);
  lincomb(g, X, X2, U0, nullptr, C1, Y, grams, h.part, st);
  double* C2 = grams;                  // a x b
  double* G2 = grams + (size_t)a * b;  // b x b
  if (a > 0) gemm(b, b, a, -1.0, tr(rowm(C2, b)), 0, rowm(C2, b), 0, 1.0, rowm(G2, b), 0, 1, st);
  // rank-revealing pivoted Cholesky of the projected Gram: columns whose
  // residual falls below 1e-7 of the largest are deflated (to level 2)
  cholqr_build(G2, C2, a, b, 0, 1e-14, nullptr, TA, TB, info, sig, h.cq_work, st);
  if (h.spec) return orth_complement_spec(h, Y, U0, a, b, rank_bound, grams, TA, TB, info, dinfo);
  CK(cudaMemcpyAsync(h.pinned + 8, info, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h.pinned + 11, sig, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  check_singular(h);
  int k = *(int*)(h.pinned + 8);
  const double lam0 = h.pinned[11];
  h.uq = 0;
  h.spec_kfull[h.spec_tr] = k == (b < rank_bound ? b : rank_bound);
  // Level 2 (graded increments): the one-pass Gram resolves directions only
  // down to ~1e-7 of the largest column (its entries carry eps |Y|^2 absolute
  // error), where the reference's Householder QR keeps every direction. When
  // columns were deflated and the increment's rank bound allows more, their
  // residuals after Q are formed explicitly (W = Y' [P_J R^-1 | rest residual
  // columns], cholqr mode 2), their Gram recomputed from the vectors
  // themselves and re-orthonormalised after column scaling: directions down to
  // 1e-13 of |X| are kept (the content below that is under T2's 1e-11
  // bound), rounding noise is not.
  const bool level2 = k < b && k < rank_bound && lam0 > 0.0;
  if (k == 0 && !level2) return 0;
  NMat Qv;
  double* C3 = grams;
  double* G3 = nullptr;
  if (level2) {
    cholqr_build(G2, C2, a, b, 2, 1e-14, nullptr, TA, TB, info, nullptr, h.cq_work, st);
    xnorm_kernel<<<1, 256, 0, st>>>(G2, a > 0 ? C1 : nullptr, a, b, 1e-13, dinfo + 1);
    launched();
    // pass 3': W = Y TA - U0 TB (b cols) -> Q, C3 = U0^T W, G3 = W^T W
    NMat W = h.Q.view(g, b, st);
    lincomb(g, Y, NMat{}, U0, TA, TB, W, grams, h.part, st);
    double* Ms = slot(h, S_M2, (size_t)b * b);
    double* dinv = slot(h, S_PC, (size_t)b);
    level2_gram<<<1, 256, 0, st>>>(grams + (size_t)a * b, grams, a, b, k,
                                   rank_bound < b ? rank_bound : b, dinfo + 1, Ms, dinv);
    launched();
    cholqr_build(Ms, grams, a, b, 3, 1e-14, dinv, TA, TB, info + 2, nullptr, h.cq_work, st);
    CK(cudaMemcpyAsync(h.pinned + 8, info + 2, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    k = *(int*)(h.pinned + 8);
    if (k == 0) return 0;
    // pass 4': Q = W T - U0 TB (k cols) -> Qa, then swapped into Q
    Qv = h.Qa.view(g, k, st);
    lincomb(g, W, NMat{}, U0, TA, TB, Qv, grams, h.part, st);
    std::swap(h.Q, h.Qa);
    Qv = h.Q.view(g, k, st);
  } else {
    // pass 3: Q = Y TA - U0 TB (k cols) -> Q, C3 = U0^T Q, G3 = Q^T Q
    Qv = h.Q.view(g, k, st);
    lincomb(g, Y, NMat{}, U0, TA, TB, Qv, grams, h.part, st);
  }
  G3 = grams + (size_t)a * k;
  // the block's defect max(|Q^T Q - I|, |U0^T Q|) decides on a further pass;
  // its SVQB coefficients are only formed when it is needed
  defect_gc_kernel<<<1, 256, 0, st>>>(G3, C3, a, k, dinfo);
  launched();
  CK(cudaMemcpyAsync(h.pinned + 9, dinfo, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  // re-orthogonalise when the block's defect exceeds the reference's own
  // re-orthonormalisation trigger (orthonormal_columns, dlra.py:36-41: 1e-12)
  if (h.pinned[9] > 1e-12) {
    double* G3c = slot(h, S_M2, (size_t)k * k);
    CK(cudaMemcpyAsync(G3c, G3, sizeof(double) * k * k, cudaMemcpyDeviceToDevice, st));
    if (a > 0)
      gemm(k, k, a, -1.0, tr(rowm(C3, k)), 0, rowm(C3, k), 0, 1.0, rowm(G3c, k), 0, 1, st);
    cholqr_build(G3c, C3, a, k, 1, 0.0, nullptr, TA, TB, info + 1, nullptr, h.cq_work, st);
    // pass 4: Q <- Q TA - U0 TB (into Qa, then swap)
    NMat Q2 = h.Qa.view(g, k, st);
    lincomb(g, Qv, NMat{}, U0, TA, TB, Q2, nullptr, h.part, st);
    std::swap(h.Q, h.Qa);
  }
  h.uq = k;
  return k;
}

// One K stage with the halo exchange of its input overlapped: the exchange
// (NCCL send/recv of the two boundary planes each way) runs on the side
// stream while the planes 2 .. nz-3 are computed; the four boundary planes
// follow once it has landed. The split is over whole chunks, so the result is
// the unsplit launch's, bit for bit.
static void kstage_overlapped(Handle& h, KStageArgs ka, cudaStream_t st) {
  CK(cudaEventRecord(h.ev_fork, st));
  CK(cudaStreamWaitEvent(h.st2, h.ev_fork, 0));
  comm_halo_rows(h.g, ka.X.p, ka.X.rs, h.st2);
  CK(cudaEventRecord(h.ev_join, h.st2));
  ka.zpart = 1;
  kstage(ka, st);
  CK(cudaStreamWaitEvent(st, h.ev_join, 0));
  ka.zpart = 2;
  kstage(ka, st);
}

void streaming_step(Handle& h, double dt) {
  h.singular_pending = false;
  if (!h.stencil_error.empty()) fail(PND_ECONFIG, h.stencil_error);
  need(h.have_angular, "angular operators (pnd_set_angular)");
  need(h.have_inv_s, "stopping power (pnd_set_inv_s)");
  consolidate(h);
  const Geom& g = h.g;
  const int m = h.m, ns = g.ns;
  const int a = h.ua, b = h.rv;
  if (a <= 0 || b <= 0) fail(PND_ECONFIG, "empty low-rank state");
  if (h.blocked || a > 64 || b > 64) return streaming_step_x(h, dt);  // xwide.cu
  cudaStream_t st = h.st;
  const NMat U0 = state_u(h);
  const double* isp = isp_rows(h);
  // ranks above 32: the stencil kernels run on 32-column blocks (wide.cu)
  const bool wide = a > 32 || b > 32;
  // z-slabs: overlap each K stage's halo exchange with its interior planes
  const bool split =
      !wide && kstage_can_split(g) && (comm_world(g) > 1 || getenv("PND_KSTAGE_SPLIT"));
  // U0's neighbour planes (K stage 0, L- and S-Grams): with the split, inside K stage 0
  if (!split) comm_halo_rows(g, U0.p, U0.rs, st);
  std::vector<NMat> u0b, w1b, w2b;
  if (wide) {
    u0b = split_blocks(h, U0, h.wide_u0b);
    w1b = block_views(h, h.wide_w1b, b);
    w2b = block_views(h, h.wide_w2b, b);
  }

  // --- K phase: K1 = K0 + dK, K' = -sum_s (D_s S^-1 K) F_s(V0), K0 = U0 S0
  phase(h, PH_LSIDE);
  double* F = slot(h, S_FV, (size_t)ns * b * b);
  moment_factors(h, h.V.p, b, F);
  const int xmax = a > b ? a : b;
  double* M = slot(h, S_MST, (size_t)ns * xmax * b);
  const NMat W1 = h.W1.view(g, b, st);
  const NMat W2 = h.W2.view(g, b, st);
  const double coef[4] = {0.25, 1.0 / 3.0, 0.5, 1.0};
  for (int stage = 0; stage < 4; ++stage) {
    KStageArgs ka{};
    ka.bcat = &h.bcat;
    ka.geo = g;
    ka.inv_s = isp;
    ka.U0 = stage == 3 ? NMat{} : U0;  // the last stage returns dK = h L(W2) only
    ka.S0 = h.S.p;
    ka.M = M;
    const double c = -coef[stage] * dt;
    if (stage == 0) {
      // L(U0 S0) = -sum_s (D_s U0)(S0 F_s): X = U0, M_s = -(h/4) S0 F_s
      gemm(a, b, b, c, rowm(h.S.p, b), 0, rowm(F, b), (long)b * b, 0.0, rowm(M, b),
           (long)a * b, ns, st);
      ka.X = U0;
      ka.out = W1;
    } else {
      axpby(ns * b * b, c, F, 0.0, M, st);
      ka.X = stage == 2 ? W2 : W1;
      ka.out = stage == 2 ? W1 : W2;
    }
    // the Horner intermediates W1/W2 are stored pre-scaled by 1/S; dK is not
    ka.in_scaled = stage > 0;
    ka.out_scaled = stage < 3;
    phase(h, PH_KSTAGE);
    if (wide) {
      const std::vector<NMat>& xin = stage == 0 ? u0b : stage == 2 ? w2b : w1b;
      if (stage > 0)
        for (const NMat& x : xin) comm_halo_rows(g, x.p, x.rs, st);
      // the same buffer rotation as below: U0 -> W1 -> W2 -> W1 -> W2
      kstage_blocks(h, xin, ka.U0, h.S.p, M, stage == 0 || stage == 2 ? w1b : w2b,
                    ka.in_scaled, ka.out_scaled);
    } else if (split) {
      // the input's boundary planes go to the neighbours (side stream) while
      // the interior planes -- which read no halo row -- run
      kstage_overlapped(h, ka, st);
    } else {
      if (stage > 0) comm_halo_rows(g, ka.X.p, ka.X.rs, st);  // the previous stage's output
      kstage(ka, st);
    }
    phase(h, PH_LSIDE);
  }
  // dK = W2 (one matrix, or its <= 2 column blocks at ranks above 32)
  const NMat dK = wide ? w2b[0] : W2;
  const NMat dK2 = wide && w2b.size() > 1 ? w2b[1] : NMat{};

  double* C1 = slot(h, S_C1, (size_t)a * b);
  phase(h, PH_LGRAM);
  if (dK2.p) gram_xy2(g, U0, dK, dK2, C1, h.part, st);  // C1 = U0^T dK
  else gram_xy(g, U0, dK, C1, h.part, st);

  // --- U augmentation: U^ = [U0 | orth((I - U0 U0^T) dK)]
  phase(h, PH_ORTH);
  const int k = orth_complement(h, dK, C1, dK2);
  const int ru = a + k;

  // --- S-phase Grams G_s = U^T D_s S^-1 U^ (dlra.py:199-209). Their leading
  // a x a block is the L phase's U0^T D_s S^-1 U0 = Q_s^T (dlra.py:183-184):
  // same factor, same 1/S, so the L phase reads it there instead of a
  // separate pass over n (the L phase does not depend on the augmentation).
  double* G = slot(h, S_G, (size_t)ns * ru * ru);
  phase(h, PH_SGRAM);
  if (k > 0) comm_halo_rows(g, state_q(h).p, state_q(h).rs, st);
  if (ru > 64 || wide) {
    // [U0 | Q] in balanced blocks of <= 32 columns, one rectangular S-Gram
    // launch per block pair (stencil_grams_blocks)
    const std::vector<NMat> blocks =
        split_joint(h, U0, k > 0 ? state_q(h) : NMat{}, 32, h.wide_gb);
    stencil_grams_blocks(h, blocks, isp, G);
  } else {
    stencil_grams(g, U0, k > 0 ? state_q(h) : NMat{}, isp, G, h.part, st);
  }

  // --- L phase: L' = -sum_s A_s L Q_s, Q_s^T = G_s[:a, :a], L0 = V0 S0^T
  phase(h, PH_LSIDE);
  const int cols = a + b;
  double* BV = slot(h, S_BV, (size_t)m * cols);
  if (!l_rk4(h.V.p, h.S.p, G, ru, h.amat.p, m, a, b, ns, dt, slot(h, S_M2, (size_t)m * a), BV,
             st)) {
  double* L0 = slot(h, S_L0, (size_t)m * a);
  double* LW = slot(h, S_LW, (size_t)m * a);
  double* Z = slot(h, S_ZST, (size_t)ns * m * a);
  gemm(m, a, b, 1.0, rowm(h.V.p, b), 0, tr(rowm(h.S.p, b)), 0, 0.0, rowm(L0, a), 0, 1, st);
  CK(cudaMemcpyAsync(LW, L0, sizeof(double) * m * a, cudaMemcpyDeviceToDevice, st));
  for (int stage = 0; stage < 4; ++stage) {
    gemm(m, a, a, 1.0, rowm(LW, a), 0, tr(rowm(G, ru)), (long)ru * ru, 0.0, rowm(Z, a),
         (long)m * a, ns, st);
    double* dst = stage == 3 ? slot(h, S_M2, (size_t)m * a) : LW;
    CK(cudaMemcpyAsync(dst, L0, sizeof(double) * m * a, cudaMemcpyDeviceToDevice, st));
    // dst = L0 - c h sum_s A_s Z_s  (A_s symmetric: [A_0..A_ns-1] = (stacked A)^T)
    gemm(m, a, ns * m, -coef[stage] * dt, tr(rowm(h.amat.p, m)), 0, rowm(Z, a), 0, 1.0,
         rowm(dst, a), 0, 1, st);
    if (stage == 3) transpose_in(dst, m, a, BV, m, st);
  }
  transpose_in(h.V.p, m, b, BV + (size_t)a * m, m, st);
  }

  // --- V augmentation: V^ = orth([L1, V0])
  double* Vhc = slot(h, S_VHC, (size_t)m * cols);
  double* Rv = slot(h, S_RV, (size_t)cols * cols);
  phase(h, PH_TSQR_M);
  const int rv = tsqr(BV, m, cols, m, Vhc, m, Rv, h.tq_m, st);
  phase(h, PH_SRK4);

  // --- S^0 = (U^T U0) S0 (V0^T V^) = [S0 Rv[:, a:]^T ; 0]
  double* Sh = slot(h, S_SHAT, (size_t)ru * rv);
  gemm(a, rv, b, 1.0, rowm(h.S.p, b), 0, Mat{Rv + a, 1, cols}, 0, 0.0, rowm(Sh, rv), 0, 1, st);
  if (k > 0) {
    zero_rows_kernel<<<1, 256, 0, st>>>(Sh, a, k, rv);
    launched();
  }

  // --- S phase: S' = -sum_s (U^T D_s S^-1 U^) S F_s(V^), precontracted Grams G
  double* Vhr = slot(h, S_VHR, (size_t)m * rv);
  transpose_out(Vhc, m, m, rv, Vhr, st);
  double* Fh = slot(h, S_FH, (size_t)ns * rv * rv);
  moment_factors(h, Vhr, rv, Fh);
  s_rk4(Sh, ru, rv, G, Fh, ns, dt, nullptr, st);

  // --- new (augmented) state: [U0 | Q]
  double* Snew = h.S.get((size_t)ru * rv);
  CK(cudaMemcpyAsync(Snew, Sh, sizeof(double) * ru * rv, cudaMemcpyDeviceToDevice, st));
  double* Vnew = h.V.get((size_t)m * rv);
  CK(cudaMemcpyAsync(Vnew, Vhr, sizeof(double) * m * rv, cudaMemcpyDeviceToDevice, st));
  h.ru = ru;
  h.rv = rv;
  phase(h, -1);
}

namespace {

__global__ void gt_kernel(const double* g, const double* tm, int m, int nb, double* gt) {
  const int total = nb * 12 * m;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int b = i / (12 * m), rem = i - b * 12 * m, q = rem % m;
    gt[i] = g[rem] * tm[b * m + q];
  }
}

__global__ void coeff_kernel(const double* g, const double* sig, int m, double* c) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 12 * m; i += gridDim.x * blockDim.x)
    c[i] = sig[i / m] - g[i];
}

__global__ void init_int(int* p, int v) { *p = v; }

// One material class and one beam: dK = dt (psi/S) w^T with w = N^T rows (a
// b-vector), so span((I - U0 U0^T) dK) = span((I - U0 U0^T) z) for the single
// column z = dt |w| psi/S -- zero exactly when dK is. zscale: s = dt |w|_2.
__global__ void zscale_kernel(const double* __restrict__ atomic, const double* __restrict__ rows,
                              int b, double dt, double* s) {
  double v = 0.0;
  for (int j = threadIdx.x; j < b; j += 32) {
    double w = 0.0;
    for (int i = 0; i < 12; ++i) w = fma(atomic[i], rows[i * b + j], w);
    v = fma(w, w, v);
  }
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (threadIdx.x == 0) s[0] = dt * sqrt(v);
}

// z = s psi / S (column 0; the padding column of the even stride is zero)
__global__ void zcol_kernel(int n, const double* __restrict__ s, const double* __restrict__ inv_s,
                            const double* __restrict__ psi, NMat z) {
  const double sc = s[0];
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const double2 v{sc * inv_s[c] * psi[c], 0.0};
    *reinterpret_cast<double2*>(z.p + (size_t)c * 2) = v;
  }
}

// U0^T z = s U0^T diag(1/S) psi (u: stride us)
__global__ void zcoef_kernel(const double* __restrict__ s, const double* __restrict__ u, int us,
                             int a, double* out) {
  for (int i = threadIdx.x; i < a; i += blockDim.x) out[i] = s[0] * u[(size_t)i * us];
}

// per-cell weight of Gram i: [cls == i] / S (phase < 0) or wtab[cls][phase] / S;
// zero past n (the chunked staging reads up to 64 rows beyond)
__global__ void class_weight_kernel(const int* cls, const double* wtab, const double* inv_s, int n,
                                    int phase, int cl, double* w) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n + 64; c += gridDim.x * blockDim.x) {
    double v = 0.0;
    if (c < n) v = inv_s[c] * (phase < 0 ? (cls[c] == cl ? 1.0 : 0.0) : wtab[cls[c] * 12 + phase]);
    w[c] = v;
  }
}

}  // namespace

void scattering_step(Handle& h, double dt) {
  h.singular_pending = false;
  need(h.have_inv_s, "stopping power (pnd_set_inv_s)");
  need(h.have_mat, "materials (pnd_set_materials)");
  need(h.have_scat, "scattering tables (pnd_set_scattering)");
  consolidate(h);
  const Geom& g = h.g;
  const int m = h.m;
  const int a = h.ua, b = h.rv;
  const int B = h.n_beams;
  cudaStream_t st = h.st;
  if (a <= 0 || b <= 0) fail(PND_ECONFIG, "empty low-rank state");
  if (h.blocked || a > 64 || b > 64) return scattering_step_x(h, dt);  // xwide.cu
  const NMat U0 = state_u(h);

  // gt_b = g o T_M^b (12 x m), rows_b = gt_b V0 (12 x b)
  phase(h, PH_SCATSMALL);
  double* gt = slot(h, S_GT, (size_t)(B > 0 ? B : 1) * 12 * m);
  double* rows = slot(h, S_ROWS, (size_t)(B > 0 ? B : 1) * 12 * b);
  if (B > 0) {
    gt_kernel<<<64, 256, 0, st>>>(h.gdiag.p, h.tm.p, m, B, gt);
    launched();
    gemm(12 * B, b, m, 1.0, rowm(gt, m), 0, rowm(h.V.p, b), 0, 0.0, rowm(rows, b), 0, 1, st);
  }

  // One material class and one beam: the source rows are rank one,
  // Z[c][i] = N_i psi(c) / S(c), so Z is never formed -- dK = dt (psi/S) (N^T rows)
  // row by row, and every projection X^T Z = (X^T diag(1/S) psi) N^T comes
  // out of a Gram-only pass against the psi column (the one with B_0 for U0).
  const bool rank1 = h.n_cls == 1 && B == 1;
  const NMat psi_col{h.psi.p, 1, 1};

  // substep 2 increment: dK = dt src_rows(V0) = dt Z rows  (dlra.py:303; K1 = U0 S0 + dK)
  // with the source rows Z[c][b*12 + i] = N_{cls,i} psi_b / S materialised once
  phase(h, PH_SCATK1);
  NMat Z{}, dK{};
  bool forked = false;
  double* C1 = slot(h, S_C1, (size_t)a * b + 72);
  double* zs = C1 + 64;  // rank one: the scale s of z (C1 holds U0^T z, a <= 64)
  if (rank1) {
    // the increment's one direction z (memory-bound, on the side stream)
    // overlaps the B_0 / projection Gram pass below (reads only U0 and psi);
    // joined before z is used
    zscale_kernel<<<1, 32, 0, st>>>(h.cls_atomic.p, rows, b, dt, zs);
    launched();
    CK(cudaEventRecord(h.ev_fork, st));
    CK(cudaStreamWaitEvent(h.st2, h.ev_fork, 0));
    dK = h.Xs.view(g, 1, h.st2);
    zcol_kernel<<<sm_count() * 8, 256, 0, h.st2>>>(g.n, zs, h.inv_s.p, h.psi.p, dK);
    launched();
    CK(cudaEventRecord(h.ev_join, h.st2));
    forked = true;
  } else if (B > 0) {
    dK = h.W2.view(g, b, st);
    Z = h.Xs.view(g, 12 * B, st);
    source_rows(g, h.inv_s.p, h.cls.p, h.cls_atomic.p, h.psi.p, B, Z, st);
    double* TAz = slot(h, S_TAZ, (size_t)12 * B * b);
    axpby(12 * B * b, dt, rows, 0.0, TAz, st);
    lincomb(g, Z, NMat{}, NMat{}, TAz, nullptr, dK, nullptr, h.part, st);
  } else {
    dK = h.W2.view(g, b, st);
    scat_dk(g, dt, h.inv_s.p, h.cls.p, h.cls_atomic.p, h.n_cls, nullptr, 0, rows, dK, st);
  }

  // substep 1: B_i = U0^T diag(N_i / S) U0 (dlra.py:284-285)
  const int nw = h.n_cls <= 12 ? h.n_cls : 12;
  double* H = slot(h, S_H, (size_t)nw * a * a);
  phase(h, PH_SCATGRAM);
  double* left = slot(h, S_LEFT, (size_t)a * 12 * (B > 0 ? B : 1));
  if (rank1) {
    // [H | u] = U0^T diag(1/S) [U0 | psi]; left = U0^T Z = u N^T
    double* Hu = slot(h, S_HU, (size_t)a * (a + 1));
    if (a + 1 <= 64) {
      gram_xy2(g, U0, U0, psi_col, Hu, h.part, st, h.inv_s.p);
      CK(cudaMemcpy2DAsync(H, a * sizeof(double), Hu, (a + 1) * sizeof(double),
                           a * sizeof(double), a, cudaMemcpyDeviceToDevice, st));
      gemm(a, 12, 1, 1.0, Mat{Hu + a, a + 1, 1}, 0, rowm(h.cls_atomic.p, 12), 0, 0.0,
           rowm(left, 12), 0, 1, st);
      zcoef_kernel<<<1, 64, 0, st>>>(zs, Hu + a, a + 1, a, C1);
    } else {  // 64 columns: the Gram-only pass takes at most 64
      gram_xy(g, U0, U0, H, h.part, st, h.inv_s.p);
      gram_xy(g, U0, psi_col, Hu, h.part, st, h.inv_s.p);
      gemm(a, 12, 1, 1.0, Mat{Hu, 1, 1}, 0, rowm(h.cls_atomic.p, 12), 0, 0.0, rowm(left, 12), 0,
           1, st);
      zcoef_kernel<<<1, 64, 0, st>>>(zs, Hu, 1, a, C1);
    }
    launched();
  } else if (h.n_cls == 1) {
    gram_xy(g, U0, U0, H, h.part, st, h.inv_s.p);  // one class: U0^T diag(1/S) U0
  } else if (a > 32) {
    // ranks above 32: one weighted Gram-only pass per class / phase
    double* wv = h.wide_t.get((size_t)g.ld + 64);
    for (int i = 0; i < nw; ++i) {
      class_weight_kernel<<<148 * 8, 256, 0, st>>>(h.cls.p, h.cls_atomic.p, h.inv_s.p, g.n,
                                                   h.n_cls <= 12 ? -1 : i, i, wv);
      launched();
      gram_xy(g, U0, U0, H + (size_t)i * a * a, h.part, st, wv);
    }
  } else {
    PGramArgs pa{};
    pa.geo = g;
    pa.X = U0;
    pa.Y = U0;
    pa.nb = a;
    pa.nphase = nw;
    pa.gen = PG_WEIGHT;
    pa.inv_s = h.inv_s.p;
    pa.cls = h.cls.p;
    pa.wtab = h.cls_atomic.p;
    pa.wmode = h.n_cls <= 12 ? 0 : 1;
    pa.out = H;
    pgram(pa, h.part, st);
  }
  phase(h, PH_SCATSMALL);
  double* Bi = slot(h, S_BI, (size_t)12 * a * a);
  if (h.n_cls <= 12) {
    // B_i = sum_k N_{k,i} H_k
    gemm(12, a * a, h.n_cls, 1.0, tr(rowm(h.cls_atomic.p, 12)), 0, rowm(H, a * a), 0, 0.0,
         rowm(Bi, a * a), 0, 1, st);
  } else {
    CK(cudaMemcpyAsync(Bi, H, sizeof(double) * 12 * a * a, cudaMemcpyDeviceToDevice, st));
  }
  // source projections U0^T (N psi_b / S)  (a x 12B)
  phase(h, PH_SCATGRAM);
  if (B > 0 && !rank1) gram_xy(g, U0, Z, left, h.part, st);
  phase(h, PH_SCATSMALL);
  // C1 = U0^T dK = dt sum_b left_b rows_b  (no n-side pass; rank one: U0^T z above)
  if (B > 0 && !rank1) {
    for (int beam = 0; beam < B; ++beam)
      gemm(a, b, 12, dt, Mat{left + beam * 12, 12 * B, 1}, 0, rowm(rows + (size_t)beam * 12 * b, b),
           0, beam == 0 ? 0.0 : 1.0, rowm(C1, b), 0, 1, st);
  } else if (B == 0) {
    fill_zero(C1, (size_t)a * b, st);
  }
  double* coeffs = slot(h, S_COEF, (size_t)12 * m);
  coeff_kernel<<<16, 256, 0, st>>>(h.gdiag.p, h.sigt.p, m, coeffs);
  launched();
  double* lcols = slot(h, S_LCOL, (size_t)a * m);
  gemm(a, m, b, 1.0, rowm(h.S.p, b), 0, tr(rowm(h.V.p, b)), 0, 0.0, rowm(lcols, m), 0, 1, st);
  double* lnew = slot(h, S_LNEW, (size_t)a * m);
  int* flag = h.iflag.get(8);
  init_int<<<1, 1, 0, st>>>(flag + 4, 1 << 30);
  launched();
  scat_solves(Bi, coeffs, lcols, a, m, dt, lnew, flag + 4, st);
  // the singular-column flag is read back with the augmentation's first
  // synchronisation below (no extra host round trip)
  CK(cudaMemcpyAsync(h.pinned + 10, flag + 4, sizeof(int), cudaMemcpyDeviceToHost, st));
  h.singular_pending = true;
  // V~, R~ = qr(L1^T): lnew row-major (a x m) is L1^T column-major (m x a)
  phase(h, PH_TSQR_M);
  const int kt = m < a ? m : a;
  double* Vtc = slot(h, S_VTC, (size_t)m * kt);
  double* Rt = slot(h, S_RT, (size_t)kt * a);
  tsqr(lnew, m, a, m, Vtc, m, Rt, h.tq_m, st);  // S~ = R~^T  (a x kt)

  // substep 2: U^ = [U0 | orth((I - U0 U0^T) dK)]
  phase(h, PH_ORTH);
  if (forked) CK(cudaStreamWaitEvent(st, h.ev_join, 0));  // dK from the side stream
  // rank(dK) <= rank of the source rows: one per (material class, beam);
  // rank one: the column z spans it
  const int bound = rank1 ? 1 : (long)h.n_cls * B < b ? h.n_cls * B : b;
  const int k = orth_complement(h, dK, C1, NMat{}, bound);
  const int ru = a + k;
  phase(h, PH_SCATSMALL);

  // substep 3: l3 = V~ S~^T + dt proj^T, V^ = orth([l3, V~])  (dlra.py:306-312)
  const int vcols = a + kt;
  double* BV = slot(h, S_BV, (size_t)m * vcols);
  double* proj = slot(h, S_PROJ, (size_t)a * m);
  gemm(m, a, kt, 1.0, colm(Vtc, m), 0, rowm(Rt, a), 0, 0.0, colm(BV, m), 0, 1, st);
  if (B > 0) {
    for (int beam = 0; beam < B; ++beam) {
      gemm(a, m, 12, 1.0, Mat{left + beam * 12, 12 * B, 1}, 0, rowm(gt + (size_t)beam * 12 * m, m),
           0, beam == 0 ? 0.0 : 1.0, rowm(proj, m), 0, 1, st);
    }
    axpby(a * m, dt, proj, 1.0, BV, st);  // col-major (m x a) == row-major (a x m) layout
  }
  CK(cudaMemcpyAsync(BV + (size_t)a * m, Vtc, sizeof(double) * m * kt, cudaMemcpyDeviceToDevice,
                     st));
  double* Vhc = slot(h, S_VHC, (size_t)m * vcols);
  double* Rv = slot(h, S_RV, (size_t)vcols * vcols);
  phase(h, PH_TSQR_M);
  const int rv = tsqr(BV, m, vcols, m, Vhc, m, Rv, h.tq_m, st);
  phase(h, PH_SCATSMALL);

  // substep 4: S1 = (U^T U0) S~ (V~^T V^) + dt U^T (N psi / S)(g o T_M) V^, U^T U0 = [I; 0]
  double* Sh = slot(h, S_SHAT, (size_t)ru * rv);
  gemm(a, rv, kt, 1.0, tr(rowm(Rt, a)), 0, Mat{Rv + a, 1, vcols}, 0, 0.0, rowm(Sh, rv), 0, 1,
       st);
  if (k > 0) {
    zero_rows_kernel<<<1, 256, 0, st>>>(Sh, a, k, rv);
    launched();
  }
  if (B > 0) {
    // U^T X_b = [left_b ; Q^T X_b]
    double* proj2 = slot(h, S_PROJ2, (size_t)ru * 12 * B);
    CK(cudaMemcpyAsync(proj2, left, sizeof(double) * a * 12 * B, cudaMemcpyDeviceToDevice, st));
    if (k > 0) {
      phase(h, PH_SCATGRAM);
      if (rank1) {
        // Q^T Z = (Q^T diag(1/S) psi) N^T
        double* qv = slot(h, S_QV, (size_t)k);
        gram_xy(g, state_q(h), psi_col, qv, h.part, st, h.inv_s.p);
        gemm(k, 12, 1, 1.0, Mat{qv, 1, 1}, 0, rowm(h.cls_atomic.p, 12), 0, 0.0,
             rowm(proj2 + (size_t)a * 12, 12), 0, 1, st);
      } else {
        gram_xy(g, state_q(h), Z, proj2 + (size_t)a * 12 * B, h.part, st);
      }
      phase(h, PH_SCATSMALL);
    }
    double* gtv = slot(h, S_GTV, (size_t)B * 12 * rv);
    gemm(12 * B, rv, m, 1.0, rowm(gt, m), 0, colm(Vhc, m), 0, 0.0, rowm(gtv, rv), 0, 1, st);
    for (int beam = 0; beam < B; ++beam) {
      gemm(ru, rv, 12, dt, Mat{proj2 + beam * 12, 12 * B, 1}, 0,
           rowm(gtv + (size_t)beam * 12 * rv, rv), 0, 1.0, rowm(Sh, rv), 0, 1, st);
    }
  }

  double* Snew = h.S.get((size_t)ru * rv);
  CK(cudaMemcpyAsync(Snew, Sh, sizeof(double) * ru * rv, cudaMemcpyDeviceToDevice, st));
  double* Vnew = h.V.get((size_t)m * rv);
  transpose_out(Vhc, m, m, rv, Vnew, st);
  h.ru = ru;
  h.rv = rv;
  phase(h, -1);
}

namespace {
__global__ void diag_kernel(const double* sig, int r, double* S) {
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) S[i] = (i / r == i % r) ? sig[i / r] : 0.0;
}

__global__ void defect_kernel(const double* G, int r, double* out) {
  __shared__ double red[256];
  double mx = 0.0;
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) {
    const double v = fabs(G[i] - ((i / r == i % r) ? 1.0 : 0.0));
    mx = v > mx ? v : mx;
  }
  red[threadIdx.x] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int i = 0; i < blockDim.x; ++i) m = red[i] > m ? red[i] : m;
    out[0] = out[0] > m ? out[0] : m;
  }
}
}  // namespace

void truncate(Handle& h, double theta, int rmin, int rmax, double* tail_out, int* rank_out,
              double* ugram) {
  const int p = h.ru, q = h.rv, k = p < q ? p : q;
  cudaStream_t st = h.st;
  phase(h, PH_SVD);
  double* P = slot(h, S_P, (size_t)p * k);
  double* sig = slot(h, S_SIG, (size_t)k);
  double* Qt = slot(h, S_QTM, (size_t)k * q);
  svd_small(h.S.p, p, q, P, sig, Qt, nullptr, st);
  double* dtail = slot(h, S_TAIL, 2);
  int* info = h.iflag.get(8);
  tail_rule(sig, k, theta, rmin, rmax, info + 1, dtail, st);
  int r1;
  double tail;
  bool all_zero;
  if (h.spec) {
    // predicted: the rank this truncation kept last step (the fixed rank in
    // fixed-rank runs), a nonzero S^; the tail is read after the step
    const int which = h.spec_tr;
    r1 = h.spec_r1[which] < k ? h.spec_r1[which] : k;
    spec_check_trunc_kernel<<<1, 32, 0, st>>>(info + 1, sig, r1, h.spec_flag.p);
    launched();
    CK(cudaMemcpyAsync(h.pinned + 20 + which, dtail, sizeof(double), cudaMemcpyDeviceToHost, st));
    tail = 0.0;
    all_zero = false;
  } else {
    CK(cudaMemcpyAsync(h.pinned, dtail, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync((int*)(h.pinned + 1), info + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h.pinned + 2, sig, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    check_singular(h);
    r1 = *(int*)(h.pinned + 1);
    tail = h.pinned[0];
    all_zero = h.pinned[2] == 0.0;
    if (r1 >= 0) h.spec_r1[h.spec_tr] = r1;
  }
  if (r1 < 0) {
    fail(PND_ENUMERICAL, "adaptive rank " + std::to_string(-r1 - 1) + " exceeds rank_max=" +
                             std::to_string(rmax) + "; increase the truncation threshold");
  }
  const Geom& g = h.g;
  const int m = h.m;
  phase(h, PH_ROTATE);
  if (h.blocked || r1 > 64) {
    // ranks above 64: the rotation into 32-column blocks (xwide.cu); back to
    // the row-major layout when the rank has come down to 64 or less
    rotate_x(h, P, p, k, r1, all_zero, ugram);
    phase(h, PH_SVD);
    double* Vn = slot(h, S_VNEW, (size_t)m * r1);
    gemm(m, r1, q, 1.0, rowm(h.V.p, q), 0, Mat{Qt, 1, q}, 0, 0.0, rowm(Vn, r1), 0, 1, st);
    double* V = h.V.get((size_t)m * r1);
    CK(cudaMemcpyAsync(V, Vn, sizeof(double) * m * r1, cudaMemcpyDeviceToDevice, st));
    double* S = h.S.get((size_t)r1 * r1);
    diag_kernel<<<1, 256, 0, st>>>(sig, r1, S);
    launched();
    h.ru = h.rv = r1;
    if (r1 <= 64) from_blocked(h);
    phase(h, -1);
    if (tail_out) *tail_out = tail;
    if (rank_out) *rank_out = r1;
    return;
  }
  const NMat Un = h.Un.view(g, r1, st);
  if (all_zero) {
    // S^ == 0: the reference's Householder basis of [0 | U0] starts with e_0..e_{r-1}
    // and svd(0) = (I, 0, I), so U1 is the canonical cell basis (Appendix C.4)
    unit_rows(g, Un, st);
  } else {
    // U1 = [U | Q] P[:, :r1]
    double* Pc = slot(h, S_PC, (size_t)p * r1);
    CK(cudaMemcpy2DAsync(Pc, r1 * sizeof(double), P, k * sizeof(double), r1 * sizeof(double), p,
                         cudaMemcpyDeviceToDevice, st));
    // ugram: the rotated basis' Gram U1^T U1 (the orthonormality diagnostic)
    // comes out of the same pass
    lincomb(g, state_u(h), state_q(h), NMat{}, Pc, nullptr, Un, ugram, h.part, st);
  }
  if (ugram && all_zero) gram_xy(g, Un, Un, ugram, h.part, st);
  phase(h, PH_SVD);
  double* Vn = slot(h, S_VNEW, (size_t)m * r1);
  gemm(m, r1, q, 1.0, rowm(h.V.p, q), 0, Mat{Qt, 1, q}, 0, 0.0, rowm(Vn, r1), 0, 1, st);
  std::swap(h.U, h.Un);
  h.ua = r1;
  h.uq = 0;
  double* V = h.V.get((size_t)m * r1);
  CK(cudaMemcpyAsync(V, Vn, sizeof(double) * m * r1, cudaMemcpyDeviceToDevice, st));
  double* S = h.S.get((size_t)r1 * r1);
  diag_kernel<<<1, 256, 0, st>>>(sig, r1, S);
  launched();
  h.ru = h.rv = r1;
  phase(h, -1);
  if (tail_out) *tail_out = tail;
  if (rank_out) *rank_out = r1;
}

void dose_accumulate_step(Handle& h, double dt, bool tally_steps) {
  consolidate(h);
  const Geom& g = h.g;
  cudaStream_t st = h.st;
  phase(h, PH_DOSE);
  double* coef = slot(h, S_COEFD, (size_t)h.ru);
  // integrand = sqrt(4 pi) U (S V[0, :]) (+ S psi_u(E_lo))  (driver.py:606, 613-621)
  gemm(h.ru, 1, h.rv, 1.0, rowm(h.S.p, h.rv), 0, Mat{h.V.p, 1, 0}, 0, 0.0, Mat{coef, 1, 0}, 0, 1,
       st);
  double* dep = h.dep.get((size_t)g.ld);
  double* prev = h.prev.get((size_t)g.ld);
  if (h.blocked) {
    dose_accumulate_x(h, coef, 0.5 * dt, tally_steps && h.n_beams > 0 ? h.psi_lo.p : nullptr,
                      dep, prev);
    phase(h, -1);
    return;
  }
  pnd::dose_accumulate(g, state_u(h), coef, 0.5 * dt, h.s_field.p,
                       tally_steps && h.n_beams > 0 ? h.psi_lo.p : nullptr, h.n_beams, dep, prev,
                       st);
  phase(h, -1);
}

double* defect_gram_slot(Handle& h, int ru, int rv) {
  return slot(h, S_DEF, (size_t)ru * ru + (size_t)rv * rv + 2);
}

double orth_defect(Handle& h, bool have_ugram) {
  consolidate(h);
  const Geom& g = h.g;
  cudaStream_t st = h.st;
  phase(h, PH_DEFECT);
  double* G = defect_gram_slot(h, h.ru, h.rv);
  double* out = G + (size_t)h.ru * h.ru + (size_t)h.rv * h.rv;
  if (h.blocked) {
    const double d = orth_defect_x(h, G, have_ugram);
    phase(h, -1);
    return d;
  }
  if (!have_ugram) gram_xy(g, state_u(h), state_u(h), G, h.part, st);  // U^T U
  double* GV = G + (size_t)h.ru * h.ru;
  gemm(h.rv, h.rv, h.m, 1.0, tr(rowm(h.V.p, h.rv)), 0, rowm(h.V.p, h.rv), 0, 0.0,
       rowm(GV, h.rv), 0, 1, st);
  fill_zero(out, 1, st);
  defect_kernel<<<1, 256, 0, st>>>(G, h.ru, out);
  launched();
  defect_kernel<<<1, 256, 0, st>>>(GV, h.rv, out);
  launched();
  phase(h, -1);
  if (h.spec) {  // read with the speculative step's one synchronisation
    CK(cudaMemcpyAsync(h.pinned + 22, out, sizeof(double), cudaMemcpyDeviceToHost, st));
    return 0.0;
  }
  CK(cudaMemcpyAsync(h.pinned + 2, out, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return h.pinned[2];
}

// ------------------------------------------------------------ speculative step driver
bool spec_eligible(Handle& h, int truncate_after) {
  if (getenv("PND_NO_SPEC") || h.spec_pause > 0 || truncate_after != 3) return false;
  // the last synchronous step's augmentations were full (the prediction)
  if (!h.spec_kfull[0] || !h.spec_kfull[1]) return false;
  if (h.blocked || h.ua > 64 || h.rv > 64 || h.ua <= 0 || h.rv <= 0) return false;
  if (h.spec_r1[0] < 1 || h.spec_r1[1] < 1) return false;  // no prediction yet
  if (comm_world(h.g) != 1) return false;
  // the snapshot is a copy of the state: small grids only (the launch-bound regime)
  return (size_t)h.g.n * (size_t)(h.ua + h.uq) <= ((size_t)1 << 22);
}

void spec_begin(Handle& h) {
  consolidate(h);
  cudaStream_t st = h.st;
  const Geom& g = h.g;
  const NMat u = state_u(h);
  const size_t rows = (size_t)g.n + 2 * (size_t)g.halo;
  double* su = h.snap_u.d.get(rows * u.rs);
  CK(cudaMemcpyAsync(su, u.p - (size_t)g.halo * u.rs, rows * u.rs * sizeof(double),
                     cudaMemcpyDeviceToDevice, st));
  h.snap_u.rs = u.rs;
  CK(cudaMemcpyAsync(h.snap_s.get((size_t)h.ru * h.rv), h.S.p, sizeof(double) * h.ru * h.rv,
                     cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(h.snap_v.get((size_t)h.m * h.rv), h.V.p, sizeof(double) * h.m * h.rv,
                     cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(h.snap_dep.get(g.ld), h.dep.get(g.ld), sizeof(double) * g.ld,
                     cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(h.snap_prev.get(g.ld), h.prev.get(g.ld), sizeof(double) * g.ld,
                     cudaMemcpyDeviceToDevice, st));
  h.snap_ua = h.ua;
  h.snap_ru = h.ru;
  h.snap_rv = h.rv;
  int* f = h.spec_flag.get(2);
  CK(cudaMemsetAsync(f, 0, 2 * sizeof(int), st));
  h.spec = true;
}

bool spec_end(Handle& h, bool abort) {
  cudaStream_t st = h.st;
  h.spec = false;
  CK(cudaMemcpyAsync((int*)(h.pinned + 24), h.spec_flag.p, sizeof(int), cudaMemcpyDeviceToHost,
                     st));
  CK(cudaStreamSynchronize(st));
  const int flag = *(int*)(h.pinned + 24);
  // the scattering solves' singular-column flag (the synchronous path raises)
  const bool singular = h.singular_pending && *(int*)(h.pinned + 10) != (1 << 30);
  h.singular_pending = false;
  // test hook: PND_SPEC_TEST_MISS=k rejects every k-th speculative step (the
  // restore-and-recompute path, which must reproduce the accepted result)
  bool forced = false;
  if (const char* e = getenv("PND_SPEC_TEST_MISS")) {
    const long long k = atoll(e);
    forced = k > 0 && (h.spec_hits + h.spec_misses) % k == 0;
  }
  if (flag == 0 && !singular && !abort && !forced) {
    ++h.spec_hits;
    return true;
  }
  ++h.spec_misses;
  h.spec_pause = 2;
  // restore the step's input state
  const Geom& g = h.g;
  h.ua = h.snap_ua;
  h.uq = 0;
  h.ru = h.snap_ru;
  h.rv = h.snap_rv;
  const NMat u = h.U.view(g, h.ua, st);
  if (u.rs != h.snap_u.rs) fail(PND_ECONFIG, "speculative step: snapshot stride mismatch");
  const size_t rows = (size_t)g.n + 2 * (size_t)g.halo;
  CK(cudaMemcpyAsync(u.p - (size_t)g.halo * u.rs, h.snap_u.d.p, rows * u.rs * sizeof(double),
                     cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(h.S.get((size_t)h.ru * h.rv), h.snap_s.p, sizeof(double) * h.ru * h.rv,
                     cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(h.V.get((size_t)h.m * h.rv), h.snap_v.p, sizeof(double) * h.m * h.rv,
                     cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(h.dep.p, h.snap_dep.p, sizeof(double) * g.ld, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(h.prev.p, h.snap_prev.p, sizeof(double) * g.ld, cudaMemcpyDeviceToDevice,
                     st));
  return false;
}

}  // namespace pnd
