#include <cstdlib>
// Dense small / m-side linear algebra on the device, so no step leaves the GPU.
//
//   gemm        strided batched FP64 GEMM for the m-side factors
//               (dlra.py:155-166, 176-194) and all R x R products;
//   tsqr        communication-avoiding Householder QR (TSQR) used for every
//               orthonormal_columns call (dlra.py:26-43) and the moment-side
//               qr(L1^T) (dlra.py:299): Householder leaves of 128 rows in
//               shared memory (LAPACK dlarfg conventions, so an exactly zero
//               column yields tau = 0 and the unit vector, reproducing the
//               reference's canonical step-0 basis),
//               a tree of stacked R factors, then top-down formation of the
//               explicit Q;
//   svd_small   one-CTA one-sided (Hestenes) Jacobi SVD of the augmented
//               coefficient matrix (dlra.py:99), with exact zero singular
//               values completed by canonical unit vectors (svd(0) = I, I);
//   tail_rule   the truncation rank rule (dlra.py:100-109), same summation
//               order as numpy's reversed cumsum;
//   scat_solves the m independent r x r implicit solves of scattering
//               substep 1 (dlra.py:286-298), partial-pivoting LU per column;
//   s_rk4       Horner-form RK4 of the precontracted Galerkin S-phase.
#include <float.h>

#include <cooperative_groups.h>

#include "pnd.h"

namespace pnd {

namespace cg = cooperative_groups;

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// all threads of the block get the sum; red must hold >= 32 doubles
__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < nw; ++w) s += red[w];
  __syncthreads();
  return s;
}

// ----------------------------------------------------------------- gemm
// Ktot > 0: split-K -- batch b covers k in [b K, b K + K) of Ktot (the last clipped)
__global__ void gemm_kernel(int M, int N, int K, double alpha, Mat A, long sA, Mat B, long sB,
                            double beta, Mat C, long sC, int Ktot) {
  __shared__ double As[16][17];
  __shared__ double Bs[16][17];
  const int b = blockIdx.z;
  const double* a = A.p + (size_t)b * sA;
  const double* bb = B.p + (size_t)b * sB;
  double* c = C.p + (size_t)b * sC;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int row = blockIdx.y * 16 + ty, col = blockIdx.x * 16 + tx;
  if (Ktot > 0 && K > Ktot - b * K) K = Ktot - b * K;  // the last slice
  double acc = 0.0;
  for (int k0 = 0; k0 < K; k0 += 16) {
    // A tile: (row block, k0..k0+15); load with tx running along k
    const int ar = blockIdx.y * 16 + ty, ak = k0 + tx;
    As[ty][tx] = (ar < M && ak < K) ? a[ar * A.rs + ak * A.cs] : 0.0;
    const int bk = k0 + ty, bc = blockIdx.x * 16 + tx;
    Bs[ty][tx] = (bk < K && bc < N) ? bb[bk * B.rs + bc * B.cs] : 0.0;
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) acc = fma(As[ty][kk], Bs[kk][tx], acc);
    __syncthreads();
  }
  if (row < M && col < N) {
    double* dst = c + row * C.rs + col * C.cs;
    *dst = beta == 0.0 ? alpha * acc : alpha * acc + beta * (*dst);
  }
}

__global__ void axpby_kernel(int n, double a, const double* x, double b, double* y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    y[i] = b == 0.0 ? a * x[i] : a * x[i] + b * y[i];
}

// ----------------------------------------------------------------- TSQR
struct Part {
  int rows, cols, br, nblk;
  __host__ __device__ int start(int b) const { return b * br; }
  __host__ __device__ int count(int b) const { return b == nblk - 1 ? rows - b * br : br; }
};

__global__ void hh_qr_kernel(double* A, int lda, Part pt, int first, double* tau, double* Rn,
                             int ldn) {
  extern __shared__ double sm[];
  const int b = first + blockIdx.x;
  const int r0 = pt.start(b), rb = pt.count(b), cols = pt.cols;
  const int LDS = cols + 1;
  double* S = sm;                      // rb x LDS
  double* red = sm + rb * LDS;         // 32
  double* wk = red + 32;               // cols
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nw = nthr >> 5;
  for (int idx = tid; idx < rb * cols; idx += nthr) {
    const int i = idx % rb, j = idx / rb;
    S[i * LDS + j] = A[(size_t)(r0 + i) + (size_t)j * lda];
  }
  __syncthreads();
  const int kk = rb < cols ? rb : cols;
  for (int j = 0; j < kk; ++j) {
    double part = 0.0;
    for (int i = j + 1 + tid; i < rb; i += nthr) part += S[i * LDS + j] * S[i * LDS + j];
    const double xnorm2 = block_sum(part, red);
    double tj = 0.0;
    if (xnorm2 > 0.0) {
      const double alpha = S[j * LDS + j];
      const double beta = -copysign(sqrt(alpha * alpha + xnorm2), alpha);
      tj = (beta - alpha) / beta;
      const double scl = 1.0 / (alpha - beta);
      for (int i = j + 1 + tid; i < rb; i += nthr) S[i * LDS + j] *= scl;
      __syncthreads();
      for (int k = j + 1 + warp; k < cols; k += nw) {
        double s = 0.0;
        for (int i = j + 1 + lane; i < rb; i += 32) s += S[i * LDS + j] * S[i * LDS + k];
        s = warp_sum(s);
        if (lane == 0) wk[k] = S[j * LDS + k] + s;
      }
      __syncthreads();
      const int w = cols - j - 1;
      if (w > 0) {
        for (int idx = tid; idx < (rb - j) * w; idx += nthr) {
          const int i = j + idx / w, k = j + 1 + idx % w;
          const double v = (i == j) ? 1.0 : S[i * LDS + j];
          S[i * LDS + k] -= tj * v * wk[k];
        }
      }
      __syncthreads();
      if (tid == 0) S[j * LDS + j] = beta;
      __syncthreads();
    }
    if (tid == 0) tau[(size_t)b * cols + j] = tj;
  }
  for (int j = kk + tid; j < cols; j += nthr) tau[(size_t)b * cols + j] = 0.0;
  for (int idx = tid; idx < rb * cols; idx += nthr) {
    const int i = idx % rb, j = idx / rb;
    A[(size_t)(r0 + i) + (size_t)j * lda] = S[i * LDS + j];
  }
  if (Rn) {
    for (int idx = tid; idx < cols * cols; idx += nthr) {
      const int i = idx % cols, j = idx / cols;
      const double v = (i < kk && i <= j) ? S[i * LDS + j] : 0.0;
      Rn[(size_t)(b * cols + i) + (size_t)j * ldn] = v;
    }
  }
}

// X = H_0 ... H_{kk-1} [C_b; 0] for every block b of the partition
__global__ void hh_applyq_kernel(const double* V, int ldv, Part pt, int first, const double* tau,
                                 const double* C, int ldc, int kc, double* Q, int ldq) {
  extern __shared__ double sm[];
  const int b = first + blockIdx.x;
  const int r0 = pt.start(b), rb = pt.count(b), cols = pt.cols;
  const int LDV = cols + 1, LDX = kc + 1;
  double* Vs = sm;                // rb x LDV
  double* X = Vs + rb * LDV;      // rb x LDX
  double* wk = X + rb * LDX;      // kc
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nw = nthr >> 5;
  const int kk = rb < cols ? rb : cols;
  for (int idx = tid; idx < rb * cols; idx += nthr) {
    const int i = idx % rb, j = idx / rb;
    Vs[i * LDV + j] = V[(size_t)(r0 + i) + (size_t)j * ldv];
  }
  for (int idx = tid; idx < rb * kc; idx += nthr) {
    const int i = idx % rb, c = idx / rb;
    double v = 0.0;
    if (i < cols) {
      if (C) v = C[(size_t)(b * cols + i) + (size_t)c * ldc];
      else v = (i == c) ? 1.0 : 0.0;
    }
    X[i * LDX + c] = v;
  }
  __syncthreads();
  for (int j = kk - 1; j >= 0; --j) {
    const double tj = tau[(size_t)b * cols + j];
    if (tj == 0.0) continue;
    for (int c = warp; c < kc; c += nw) {
      double s = 0.0;
      for (int i = j + 1 + lane; i < rb; i += 32) s += Vs[i * LDV + j] * X[i * LDX + c];
      s = warp_sum(s);
      if (lane == 0) wk[c] = X[j * LDX + c] + s;
    }
    __syncthreads();
    for (int idx = tid; idx < (rb - j) * kc; idx += nthr) {
      const int i = j + idx / kc, c = idx % kc;
      const double v = (i == j) ? 1.0 : Vs[i * LDV + j];
      X[i * LDX + c] -= tj * v * wk[c];
    }
    __syncthreads();
  }
  for (int idx = tid; idx < rb * kc; idx += nthr) {
    const int i = idx % rb, c = idx / rb;
    Q[(size_t)(r0 + i) + (size_t)c * ldq] = X[i * LDX + c];
  }
}

__global__ void copy_rfac_kernel(const double* Rn, int ldn, int kc, int cols, double* rfac) {
  for (int idx = threadIdx.x + blockIdx.x * blockDim.x; idx < kc * cols;
       idx += blockDim.x * gridDim.x) {
    const int i = idx / cols, j = idx % cols;
    rfac[idx] = Rn[(size_t)i + (size_t)j * ldn];
  }
}

// ----------------------------------------------------------------- SVD
template <int MT>  // column elements per lane: M <= 32 MT
__global__ void __launch_bounds__(1024, 1)
    svd_kernel(const double* s, int p, int q, double* P, double* sig, double* Qt, double* gw) {
  extern __shared__ double sm[];
  const bool tall = p >= q;
  const int M = tall ? p : q, N = tall ? q : p;
  const int N2 = N + (N & 1);
  // gw: V and U in a global (L2-resident) work buffer when they do not fit in
  // shared memory (the wide R x R case); A (the dot products of every round),
  // sg and perm stay in shared memory
  // a_in_gw (the widest, R > ~160): A lives in the global work buffer as well
  const bool a_in_gw = gw && ((size_t)M * N2 + N2) * sizeof(double) + N * sizeof(int) + 1024 >
                                 (size_t)kMaxDynSmem;
  double* A = a_in_gw ? gw + (size_t)N2 * N2 + (size_t)M * N : sm;  // column-major M x N2
  double* Vm = gw ? gw : A + M * N2;       // column-major N2 x N2
  double* U = Vm + N2 * N2;        // column-major M x N (sorted, completed)
  double* sg = a_in_gw ? sm : gw ? A + M * N2 : U + M * N;  // N2
  int* perm = (int*)(sg + N2);     // N
  __shared__ int rotated;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nw = nthr >> 5;
  for (int idx = tid; idx < M * N2; idx += nthr) {
    const int i = idx % M, j = idx / M;
    double v = 0.0;
    if (j < N) v = tall ? s[i * q + j] : s[j * q + i];
    A[idx] = v;
  }
  for (int idx = tid; idx < N2 * N2; idx += nthr) Vm[idx] = (idx % N2 == idx / N2) ? 1.0 : 0.0;
  __syncthreads();
  const int npair = N2 / 2;
  // Hestenes one-sided Jacobi, round-robin pairs; per pair one warp holds the
  // two columns in registers (MT per lane), so a rotation costs one
  // dot product (the column norms are carried: a' = a - t g, b' = b + t g,
  // recomputed exactly at the start of every sweep)
  double* nrm = sg;  // column norms^2 during the sweeps (sg is rewritten below)
  for (int sweep = 0; sweep < 60 && N2 > 1; ++sweep) {
    for (int j = warp; j < N2; j += nw) {
      double x = 0.0;
      for (int i = lane; i < M; i += 32) x += A[j * M + i] * A[j * M + i];
      x = warp_sum(x);
      if (lane == 0) nrm[j] = x;
    }
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int round = 0; round < N2 - 1; ++round) {
      for (int k = warp; k < npair; k += nw) {
        int a, b;
        if (k == 0) {
          a = round;
          b = N2 - 1;
        } else {
          a = (round + k) % (N2 - 1);
          b = (round + N2 - 1 - k) % (N2 - 1);
        }
        if (a > b) { const int t = a; a = b; b = t; }
        double xa[MT], yb[MT];
        double ga = 0.0;
#pragma unroll
        for (int t = 0; t < MT; ++t) {
          const int i = lane + 32 * t;
          xa[t] = i < M ? A[a * M + i] : 0.0;
          yb[t] = i < M ? A[b * M + i] : 0.0;
          ga = fma(xa[t], yb[t], ga);
        }
        ga = warp_sum(ga);
        const double al = nrm[a], be = nrm[b];
        if (ga != 0.0 && fabs(ga) > 1e-15 * sqrt(al * be)) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = rsqrt(1.0 + t * t), sn = c * t;
#pragma unroll
          for (int u = 0; u < MT; ++u) {
            const int i = lane + 32 * u;
            if (i < M) {
              A[a * M + i] = c * xa[u] - sn * yb[u];
              A[b * M + i] = sn * xa[u] + c * yb[u];
            }
          }
          for (int i = lane; i < N2; i += 32) {
            const double x = Vm[a * N2 + i], y = Vm[b * N2 + i];
            Vm[a * N2 + i] = c * x - sn * y;
            Vm[b * N2 + i] = sn * x + c * y;
          }
          if (lane == 0) {
            nrm[a] = al - t * ga;
            nrm[b] = be + t * ga;
            rotated = 1;
          }
        }
      }
      __syncthreads();
    }
    const int any = rotated;
    __syncthreads();
    if (!any) break;
  }
  // singular values
  for (int j = warp; j < N; j += nw) {
    double x = 0.0;
    for (int i = lane; i < M; i += 32) x += A[j * M + i] * A[j * M + i];
    x = warp_sum(x);
    if (lane == 0) sg[j] = sqrt(x);
  }
  __syncthreads();
  if (tid == 0) {  // stable selection sort, descending
    for (int j = 0; j < N; ++j) perm[j] = j;
    for (int j = 0; j < N; ++j) {
      int best = j;
      for (int k = j + 1; k < N; ++k)
        if (sg[perm[k]] > sg[perm[best]]) best = k;
      const int t = perm[j];
      perm[j] = perm[best];
      perm[best] = t;
    }
  }
  __syncthreads();
  // left vectors for nonzero singular values
  for (int idx = tid; idx < M * N; idx += nthr) {
    const int i = idx % M, j = idx / M;
    const double sv = sg[perm[j]];
    U[idx] = sv > 0.0 ? A[perm[j] * M + i] / sv : 0.0;
  }
  __syncthreads();
  // complete the zero ones with canonical unit vectors (Gram-Schmidt x2)
  if (warp == 0) {
    int cand = 0;
    for (int j = 0; j < N; ++j) {
      if (sg[perm[j]] > 0.0) continue;
      for (; cand < M; ++cand) {
        double vloc[16];
        // v = e_cand - sum_k U_k U_k[cand] over filled columns, twice
        for (int t = 0; t < 16; ++t) vloc[t] = 0.0;
        for (int i = lane, t = 0; i < M; i += 32, ++t) vloc[t] = (i == cand) ? 1.0 : 0.0;
        for (int pass = 0; pass < 2; ++pass) {
          for (int k = 0; k < N; ++k) {
            if (k == j || (sg[perm[k]] == 0.0 && k > j)) continue;
            double d = 0.0;
            for (int i = lane, t = 0; i < M; i += 32, ++t) d += U[k * M + i] * vloc[t];
            d = warp_sum(d);
            for (int i = lane, t = 0; i < M; i += 32, ++t) vloc[t] -= d * U[k * M + i];
          }
        }
        double nn = 0.0;
        for (int i = lane, t = 0; i < M; i += 32, ++t) nn += vloc[t] * vloc[t];
        nn = warp_sum(nn);
        if (nn > 0.25) {
          const double inv = 1.0 / sqrt(nn);
          for (int i = lane, t = 0; i < M; i += 32, ++t) U[j * M + i] = vloc[t] * inv;
          __syncwarp();
          ++cand;
          break;
        }
      }
    }
  }
  __syncthreads();
  // outputs: s = P diag(sig) Qt
  for (int j = tid; j < N; j += nthr) sig[j] = sg[perm[j]];
  if (tall) {
    for (int idx = tid; idx < p * N; idx += nthr) {
      const int i = idx / N, j = idx % N;
      P[idx] = U[j * M + i];
    }
    for (int idx = tid; idx < N * q; idx += nthr) {
      const int j = idx / q, c = idx % q;
      Qt[idx] = Vm[perm[j] * N2 + c];
    }
  } else {
    for (int idx = tid; idx < p * N; idx += nthr) {
      const int i = idx / N, j = idx % N;
      P[idx] = Vm[perm[j] * N2 + i];
    }
    for (int idx = tid; idx < N * q; idx += nthr) {
      const int j = idx / q, c = idx % q;
      Qt[idx] = U[j * M + c];
    }
  }
}

// QR-preconditioned one-sided Jacobi for the small truncation SVDs (M <= 64),
// everything in shared memory. A Pi = Q R by Householder with column pivoting
// (the hh_qr conventions: beta = -sign(alpha) |x|, tau = 0 for a zero
// sub-column), then Hestenes Jacobi on X = R^T, whose columns are the rows of
// R: X Vx = Ux Sigma, so R = Vx Sigma Ux^T and A = (Q Vx) Sigma (Pi Ux)^T.
// On the graded augmented S^ of the DLRA steps the pivoted triangular factor
// needs ~5 sweeps where the plain matrix needs 9-16 (its rounding-noise
// columns converge slowly). Q Vx is formed by applying the reflectors to
// [Vx; 0] backwards. Exact zero singular values are completed with canonical
// unit vectors as in svd_kernel (svd(0) = I, I: no pivoting, tau = 0).
//
// These matrices are tiny, so the kernel is instruction-bound, not
// latency-bound (ncu: IPC 2 on the one SM with 20 warps doing redundant
// scalar work): every Jacobi pair and every column update is handled by a
// group of 8 lanes (RPL rows per lane), so a round costs 5 warps, not 20.
constexpr int QJ_G = 8;

// T[:, k0:k1] <- H_j T[:, k0:k1] (column-major, leading dimension M) for the
// reflector in column j of V (v_j = 1, v_i = V[j M + i] below), one 8-lane
// group per column
template <int RPL>
__device__ __forceinline__ void qj_apply(const double* V, double* T, int M, int j, int k0, int k1,
                                         double tj) {
  const int nc = k1 - k0;
  const int tid = threadIdx.x, grp = tid / QJ_G, l = tid % QJ_G, ngrp = blockDim.x / QJ_G;
  const int trips = (nc + ngrp - 1) / ngrp;
  for (int t = 0; t < trips; ++t) {
    const int c = grp + t * ngrp;
    const bool act = c < nc;
    const int k = k0 + (act ? c : 0);
    double v[RPL], x[RPL];
    double w = 0.0;
#pragma unroll
    for (int u = 0; u < RPL; ++u) {
      const int i = j + 1 + l + QJ_G * u;
      const bool in = act && i < M;
      v[u] = in ? V[j * M + i] : 0.0;
      x[u] = in ? T[k * M + i] : 0.0;
      w = fma(v[u], x[u], w);
    }
    const double tjk = act ? T[k * M + j] : 0.0;
    w += __shfl_xor_sync(0xffffffffu, w, 4);
    w += __shfl_xor_sync(0xffffffffu, w, 2);
    w += __shfl_xor_sync(0xffffffffu, w, 1);
    if (act) {
      w = tj * (w + tjk);
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        const int i = j + 1 + l + QJ_G * u;
        if (i < M) T[k * M + i] = x[u] - w * v[u];
      }
      if (l == 0) T[k * M + j] = tjk - w;
    }
  }
}

template <int RPL>
__global__ void __launch_bounds__(512, 1)
    svd_qrj_kernel(const double* s, int p, int q, double* P, double* sig, double* Qt,
                   int stop) {
  extern __shared__ double sm[];
  const bool tall = p >= q;
  const int M = tall ? p : q, N = tall ? q : p;
  const int N2 = N + (N & 1);
  double* V = sm;                // N x M: reflector j below row j (V[j M + i], i > j)
  double* X = V + N * M;         // N x N2 column-major, X = R^T
  double* Vm = X + N * N2;       // N2 x N2 column-major
  double* U = Vm + N2 * N2;      // N x N: normalised X columns in singular value order
  double* tau = U + N * N;       // N
  double* nrm = tau + N;         // N2 (QR: trailing norms by position; Jacobi: column norms)
  double* sg = nrm + N2;         // N2
  int* perm = (int*)(sg + N2);   // N: column pivots (A Pi)[:, j] = A[:, perm[j]]
  int* order = perm + N;         // N: singular values, descending
  __shared__ int rotated, large;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nw = nthr >> 5;
  const int grp = tid / QJ_G, l = tid % QJ_G, ngrp = nthr / QJ_G;
  const unsigned gm = 0xffu << (lane & ~7);
  // ---- Householder QR with column pivoting, column c of A in the registers
  // of 8-lane group c (rows l + 8u); pivoting renames positions (no data
  // moves): group c sits at position `at` (initially c)
  const bool own = grp < N;
  double xa[RPL];
  double nn = 0.0;
#pragma unroll
  for (int u = 0; u < RPL; ++u) {
    const int i = l + QJ_G * u;
    xa[u] = (own && i < M) ? (tall ? s[i * q + grp] : s[grp * q + i]) : 0.0;
    nn = fma(xa[u], xa[u], nn);
  }
  nn += __shfl_xor_sync(0xffffffffu, nn, 4);
  nn += __shfl_xor_sync(0xffffffffu, nn, 2);
  nn += __shfl_xor_sync(0xffffffffu, nn, 1);
  int at = grp;
  bool done = !own;
  if (own && l == 0) nrm[grp] = nn;
  __syncthreads();
  for (int j = 0; j < N; ++j) {
    // pivot (every group redundantly): the first position p >= j with the
    // largest trailing norm
    double best = -1.0;
    int bp = j;
    for (int pp = j + l; pp < N; pp += QJ_G)
      if (nrm[pp] > best) { best = nrm[pp]; bp = pp; }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      if (ob > best || (ob == best && op < bp)) { best = ob; bp = op; }
    }
    // the group at position bp moves to position j, the one at j to bp
    if (!done) {
      if (at == bp) at = j;
      else if (at == j) at = bp;
    }
    if (!done && at == j) {
      // owner: reflector of row j from its registers
      double sq = 0.0, al = 0.0;
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        const int i = l + QJ_G * u;
        if (i > j) sq = fma(xa[u], xa[u], sq);
        if (i == j) al = xa[u];
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        sq += __shfl_xor_sync(gm, sq, o);
        al += __shfl_xor_sync(gm, al, o);
      }
      double tj = 0.0;
      if (sq > 0.0) {
        const double beta = -copysign(sqrt(al * al + sq), al);
        tj = (beta - al) / beta;
        const double scl = 1.0 / (al - beta);
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
          const int i = l + QJ_G * u;
          if (i > j && i < M) V[j * M + i] = xa[u] * scl;
          if (i == j) xa[u] = beta;
        }
      } else {
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
          const int i = l + QJ_G * u;
          if (i > j && i < M) V[j * M + i] = 0.0;
        }
      }
      // R column j -> row j of X = R^T (X[j + i N] = R[i][j], zero below the diagonal)
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        const int i = l + QJ_G * u;
        if (i < N) X[j + i * N] = i <= j ? xa[u] : 0.0;
      }
      if (l == 0) {
        tau[j] = tj;
        perm[j] = grp;
      }
      done = true;
    }
    __syncthreads();
    if (!done) {
      // H_j on this column, then its trailing norm (rows > j) at its position
      const double tj = tau[j];
      double v[RPL];
      double w = 0.0;
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        const int i = l + QJ_G * u;
        v[u] = i == j ? 1.0 : (i > j && i < M) ? V[j * M + i] : 0.0;
        w = fma(v[u], xa[u], w);
      }
      w += __shfl_xor_sync(gm, w, 4);
      w += __shfl_xor_sync(gm, w, 2);
      w += __shfl_xor_sync(gm, w, 1);
      w *= tj;
      double t2 = 0.0;
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        xa[u] -= w * v[u];
        const int i = l + QJ_G * u;
        if (i > j) t2 = fma(xa[u], xa[u], t2);
      }
      t2 += __shfl_xor_sync(gm, t2, 4);
      t2 += __shfl_xor_sync(gm, t2, 2);
      t2 += __shfl_xor_sync(gm, t2, 1);
      if (l == 0) nrm[at] = t2;
    }
    __syncthreads();
  }
  if (stop == 1) return;  // profiling: the QR phase alone
  // X's pad column and Vx = I
  for (int idx = tid; idx < N * (N2 - N); idx += nthr) X[N * N + idx] = 0.0;
  for (int idx = tid; idx < N2 * N2; idx += nthr) Vm[idx] = (idx % N2 == idx / N2) ? 1.0 : 0.0;
  __syncthreads();
  // ---- Hestenes sweeps on the columns of X (svd_kernel's rotation and stopping
  // rule), round-robin pairs, one 8-lane group per pair
  const int npair = N2 / 2;
  for (int sweep = 0; sweep < 60 && N2 > 1; ++sweep) {
    for (int t = 0; t < (N2 + ngrp - 1) / ngrp; ++t) {
      const int j = grp + t * ngrp;
      double x = 0.0;
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        const int i = l + QJ_G * u;
        const double v = (j < N2 && i < N) ? X[j * N + i] : 0.0;
        x = fma(v, v, x);
      }
      x += __shfl_xor_sync(0xffffffffu, x, 4);
      x += __shfl_xor_sync(0xffffffffu, x, 2);
      x += __shfl_xor_sync(0xffffffffu, x, 1);
      if (l == 0 && j < N2) nrm[j] = x;
    }
    if (tid == 0) rotated = large = 0;
    __syncthreads();
    for (int round = 0; round < N2 - 1; ++round) {
      const int k = grp;
      if (k < npair || (grp * QJ_G < ((npair * QJ_G + 31) & ~31))) {
        const bool act = k < npair;
        int a = 0, b = 1;
        if (act) {
          if (k == 0) {
            a = round;
            b = N2 - 1;
          } else {
            a = round + k;
            if (a >= N2 - 1) a -= N2 - 1;
            b = round + N2 - 1 - k;
            if (b >= N2 - 1) b -= N2 - 1;
          }
          if (a > b) { const int t = a; a = b; b = t; }
        }
        // every load of the round first (the rotation's operands do not depend
        // on it): the measured round was a chain of load, shuffle, rotation
        // parameters and a load-after-store of V
        double x[RPL], y[RPL], vx[RPL], vy[RPL];
        double ga = 0.0;
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
          const int i = l + QJ_G * u;
          const bool in = act && i < N;
          const bool inv = act && i < N2;
          x[u] = in ? X[a * N + i] : 0.0;
          y[u] = in ? X[b * N + i] : 0.0;
          vx[u] = inv ? Vm[a * N2 + i] : 0.0;
          vy[u] = inv ? Vm[b * N2 + i] : 0.0;
          ga = fma(x[u], y[u], ga);
        }
        const double al = act ? nrm[a] : 0.0, be = act ? nrm[b] : 0.0;
        const double thr = 1e-15 * sqrt(al * be);  // off the shuffle chain (dsqrt: ~100 cycles)
        ga += __shfl_xor_sync(0xffffffffu, ga, 4);
        ga += __shfl_xor_sync(0xffffffffu, ga, 2);
        ga += __shfl_xor_sync(0xffffffffu, ga, 1);
        if (act && ga != 0.0 && fabs(ga) > thr) {
          // tan(2 theta) = 2 ga / (al - be), the smaller rotation (|theta| <= pi/4):
          // cos 2theta = |d| / h, sin 2theta = sgn(d) g / h (d = be - al, g = 2 ga,
          // h = |(d, g)|), c = sqrt(q), s = sin 2theta / (2 c), t = s / c with
          // q = (1 + cos 2theta) / 2 in [1/2, 1]: two reciprocal square roots
          // instead of two divisions, a square root and a reciprocal square root
          // (the same rotation as zeta = d / g, t = sgn(zeta) / (|zeta| + sqrt(1 + zeta^2)))
          const double d = be - al, gg = 2.0 * ga;
          const double h2 = fma(d, d, gg * gg);
          double c, sn, t;
          if (h2 > 1e-290 && h2 < 1e290) {
            const double r = rsqrt(h2);
            const double c2 = fabs(d) * r, s2 = (d >= 0.0 ? gg : -gg) * r;
            const double q = fma(0.5, c2, 0.5);
            const double rq = rsqrt(q);
            c = q * rq;
            sn = 0.5 * s2 * rq;
            t = sn * rq;
          } else {  // extreme magnitudes: the scale-free formula
            const double zeta = d / gg;
            t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            c = rsqrt(1.0 + t * t);
            sn = c * t;
          }
#pragma unroll
          for (int u = 0; u < RPL; ++u) {
            const int i = l + QJ_G * u;
            if (i < N) {
              X[a * N + i] = c * x[u] - sn * y[u];
              X[b * N + i] = sn * x[u] + c * y[u];
            }
            if (i < N2) {
              Vm[a * N2 + i] = c * vx[u] - sn * vy[u];
              Vm[b * N2 + i] = sn * vx[u] + c * vy[u];
            }
          }
          if (l == 0) {
            nrm[a] = al - t * ga;
            nrm[b] = be + t * ga;
            rotated = 1;
            if (fabs(ga) > 1e7 * thr) large = 1;  // |cos angle| above 1e-8
          }
        }
      }
      __syncthreads();
    }
    // converged: no rotation, or every rotation of this sweep was below 1e-8
    // relative -- the next sweep's (quadratically smaller, below 1e-15) would
    // all be skipped, so it is not run
    const int any = rotated && large;
    __syncthreads();
    if (!any) break;
  }
  if (stop == 2) return;  // profiling: QR + Jacobi
  // singular values and their order (rank by counting: descending, stable)
  for (int j = warp; j < N; j += nw) {
    double x = 0.0;
    for (int i = lane; i < N; i += 32) x += X[j * N + i] * X[j * N + i];
    x = warp_sum(x);
    if (lane == 0) sg[j] = sqrt(x);
  }
  __syncthreads();
  for (int j = tid; j < N; j += nthr) {
    int rk = 0;
    const double v = sg[j];
    for (int k = 0; k < N; ++k) rk += (sg[k] > v) || (sg[k] == v && k < j);
    order[rk] = j;
  }
  __syncthreads();
  for (int idx = tid; idx < N * N; idx += nthr) {
    const int i = idx % N, j = idx / N;
    const double sv = sg[order[j]];
    U[idx] = sv > 0.0 ? X[order[j] * N + i] / sv : 0.0;
  }
  __syncthreads();
  // complete the zero ones with canonical unit vectors (Gram-Schmidt x2)
  if (warp == 0 && sg[order[N - 1]] == 0.0) {
    int cand = 0;
    for (int j = 0; j < N; ++j) {
      if (sg[order[j]] > 0.0) continue;
      for (; cand < N; ++cand) {
        double v0 = lane == cand ? 1.0 : 0.0, v1 = lane + 32 == cand ? 1.0 : 0.0;
        for (int pass = 0; pass < 2; ++pass) {
          for (int k = 0; k < N; ++k) {
            if (k == j || (sg[order[k]] == 0.0 && k > j)) continue;
            const double u0 = lane < N ? U[k * N + lane] : 0.0;
            const double u1 = lane + 32 < N ? U[k * N + lane + 32] : 0.0;
            const double d = warp_sum(fma(u0, v0, u1 * v1));
            v0 -= d * u0;
            v1 -= d * u1;
          }
        }
        const double nn = warp_sum(fma(v0, v0, v1 * v1));
        if (nn > 0.25) {
          const double inv = 1.0 / sqrt(nn);
          if (lane < N) U[j * N + lane] = v0 * inv;
          if (lane + 32 < N) U[j * N + lane + 32] = v1 * inv;
          __syncwarp();
          ++cand;
          break;
        }
      }
    }
  }
  __syncthreads();
  // left vectors of A: B = Q [Vx(:, order); 0], column k in the registers of
  // group k, the reflectors applied backwards from shared memory (no barrier)
  if (grp < N) {
    const int k = grp;
#pragma unroll
    for (int u = 0; u < RPL; ++u) {
      const int i = l + QJ_G * u;
      xa[u] = i < N ? Vm[order[k] * N2 + i] : 0.0;
    }
    for (int j = N - 1; j >= 0; --j) {
      const double tj = tau[j];
      if (tj == 0.0) continue;
      double v[RPL];
      double w = 0.0;
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        const int i = l + QJ_G * u;
        v[u] = i == j ? 1.0 : (i > j && i < M) ? V[j * M + i] : 0.0;
        w = fma(v[u], xa[u], w);
      }
      w += __shfl_xor_sync(gm, w, 4);
      w += __shfl_xor_sync(gm, w, 2);
      w += __shfl_xor_sync(gm, w, 1);
      w *= tj;
#pragma unroll
      for (int u = 0; u < RPL; ++u) xa[u] -= w * v[u];
    }
#pragma unroll
    for (int u = 0; u < RPL; ++u) {
      const int i = l + QJ_G * u;
      if (i < M) {
        if (tall) P[i * N + k] = xa[u];
        else Qt[k * q + i] = xa[u];
      }
    }
  }
  for (int j = tid; j < N; j += nthr) sig[j] = sg[order[j]];
  // right vectors of A: Pi U
  if (tall) {
    for (int idx = tid; idx < N * N; idx += nthr) {
      const int i = idx % N, k = idx / N;
      Qt[k * q + perm[i]] = U[k * N + i];
    }
  } else {
    for (int idx = tid; idx < N * N; idx += nthr) {
      const int i = idx % N, k = idx / N;
      P[perm[i] * N + k] = U[k * N + i];
    }
  }
}

__global__ void tail_kernel(const double* sig, int k, double theta, int rmin, int rmax, int* info,
                            double* tail) {
  __shared__ double tails[513];
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  // tails[j] = sum_{i >= j} sigma_i accumulated from the smallest (np.cumsum of sigma[::-1])
  tails[k] = 0.0;
  double acc = 0.0;
  for (int j = k - 1; j >= 0; --j) {
    acc = (j == k - 1) ? sig[j] : acc + sig[j];
    tails[j] = acc;
  }
  int r1 = k;
  for (int j = 0; j <= k; ++j)
    if (tails[j] <= theta) { r1 = j; break; }
  if (r1 > rmax) {
    info[0] = -r1 - 1;
    tail[0] = 0.0;
    return;
  }
  int r = r1 < rmin ? rmin : r1;
  if (r > rmax) r = rmax;
  if (r > k) r = k;
  info[0] = r;
  tail[0] = tails[r];
}

__global__ void scat_solve_kernel(const double* B, const double* coeffs, const double* lcols,
                                  int r, int m, double dt, double* lnew, int* singular,
                                  double* gw) {
  extern __shared__ double sm[];
  const int q = blockIdx.x;
  const int LD = r + 1;
  // gw: ranks whose r x r system does not fit in shared memory (r > ~160)
  double* const base = gw ? gw + (size_t)q * ((size_t)r * LD + r) : sm;
  double* Mx = base;           // r x LD
  double* x = base + r * LD;   // r
  __shared__ int piv;
  __shared__ int bad;
  const int tid = threadIdx.x, nthr = blockDim.x;
  for (int idx = tid; idx < r * r; idx += nthr) {
    const int a = idx / r, b = idx % r;
    double s = 0.0;
    for (int i = 0; i < 12; ++i) s += coeffs[i * m + q] * B[(size_t)i * r * r + idx];
    Mx[a * LD + b] = (a == b ? 1.0 : 0.0) + dt * s;
  }
  for (int a = tid; a < r; a += nthr) x[a] = lcols[a * m + q];
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < r; ++j) {
    if (tid == 0) {
      int p = j;
      double best = fabs(Mx[j * LD + j]);
      for (int i = j + 1; i < r; ++i) {
        const double v = fabs(Mx[i * LD + j]);
        if (v > best) { best = v; p = i; }
      }
      piv = p;
      if (best == 0.0) bad = 1;
    }
    __syncthreads();
    if (bad) break;
    const int p = piv;
    if (p != j) {
      for (int k = tid; k < r; k += nthr) {
        const double t = Mx[j * LD + k];
        Mx[j * LD + k] = Mx[p * LD + k];
        Mx[p * LD + k] = t;
      }
      if (tid == 0) { const double t = x[j]; x[j] = x[p]; x[p] = t; }
    }
    __syncthreads();
    const double inv = 1.0 / Mx[j * LD + j];
    for (int i = j + 1 + tid; i < r; i += nthr) {
      const double l = Mx[i * LD + j] * inv;
      Mx[i * LD + j] = l;
      for (int k = j + 1; k < r; ++k) Mx[i * LD + k] -= l * Mx[j * LD + k];
      x[i] -= l * x[j];
    }
    __syncthreads();
  }
  if (bad) {
    if (tid == 0) atomicMin(singular, q);
    return;
  }
  if (tid == 0) {
    for (int i = r - 1; i >= 0; --i) {
      double s = x[i];
      for (int k = i + 1; k < r; ++k) s -= Mx[i * LD + k] * x[k];
      x[i] = s / Mx[i * LD + i];
    }
  }
  __syncthreads();
  for (int a = tid; a < r; a += nthr) lnew[a * m + q] = x[a];
}

// RK4 (Horner form) of S' = -sum_s G_s S F_s on the R x R coefficient matrix in
// one CTA; with `staged` the Grams and moment factors are copied to shared
// memory first (the products then read only shared memory), and every
// product element is formed from two interleaved partial sums.
__global__ void s_rk4_kernel(double* S, int p, int q, const double* G, const double* F, int ns,
                             double dt, int staged, double* __restrict__ gw) {
  extern __shared__ double sm[];
  const int pq = p * q;
  double* S0 = gw ? gw : sm;  // gw: global work for the wide (R > ~90) case
  double* W = S0 + pq;
  double* T = W + pq;
  double* Acc = T + pq;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const double* Gb = G;
  const double* Fb = F;
  if (staged) {
    double* sg = Acc + pq;
    double* sf = sg + (size_t)ns * p * p;
    for (int i = tid; i < ns * p * p; i += nthr) sg[i] = G[i];
    for (int i = tid; i < ns * q * q; i += nthr) sf[i] = F[i];
    Gb = sg;
    Fb = sf;
  }
  for (int i = tid; i < pq; i += nthr) S0[i] = W[i] = S[i];
  __syncthreads();
  const double coef[4] = {0.25, 1.0 / 3.0, 0.5, 1.0};
  for (int st = 0; st < 4; ++st) {
    for (int i = tid; i < pq; i += nthr) Acc[i] = 0.0;
    for (int s = 0; s < ns; ++s) {
      const double* Gs = Gb + (size_t)s * p * p;
      const double* Fs = Fb + (size_t)s * q * q;
      __syncthreads();
      for (int i = tid; i < pq; i += nthr) {
        const int a = i / q, b = i % q;
        double t0 = 0.0, t1 = 0.0;
        int k = 0;
        for (; k + 1 < p; k += 2) {
          t0 = fma(Gs[a * p + k], W[k * q + b], t0);
          t1 = fma(Gs[a * p + k + 1], W[(k + 1) * q + b], t1);
        }
        if (k < p) t0 = fma(Gs[a * p + k], W[k * q + b], t0);
        T[i] = t0 + t1;
      }
      __syncthreads();
      for (int i = tid; i < pq; i += nthr) {
        const int a = i / q, b = i % q;
        double t0 = 0.0, t1 = 0.0;
        int k = 0;
        for (; k + 1 < q; k += 2) {
          t0 = fma(T[a * q + k], Fs[k * q + b], t0);
          t1 = fma(T[a * q + k + 1], Fs[(k + 1) * q + b], t1);
        }
        if (k < q) t0 = fma(T[a * q + k], Fs[k * q + b], t0);
        Acc[i] -= t0 + t1;
      }
    }
    __syncthreads();
    const double c = coef[st] * dt;
    for (int i = tid; i < pq; i += nthr) W[i] = S0[i] + c * Acc[i];
    __syncthreads();
  }
  for (int i = tid; i < pq; i += nthr) S[i] = W[i];
}

// S[:, k0:k1] <- H_j S[:, k0:k1] for the reflector stored in column j of the
// row-major S (v_j = 1, v_i = S[i][j] below): each column is one group of G
// threads (8 up to 128 rows, else 32) that forms w = tau (S[j][k] + v^T
// S[j+1:, k]) by a partial sum per thread and a G-lane xor reduction, then
// updates its own column -- no block barrier between the dot product and the
// update, and no redundant per-column scalar work across whole warps.
// tau_la: look-ahead -- the group of column k0 (= j + 1) then forms that
// column's reflector (the same dlarfg conventions) and stores it with its tau
// in tau_la[k0], so the next column step needs no serial reflector phase
__device__ void hh_apply_groups(double* S, int LDS, int rows, int j, int k0, int k1, double tj,
                                double* tau_la = nullptr) {
  const int nc = k1 - k0;
  if (nc <= 0) return;
  const int G = rows <= 128 ? 8 : 32;
  const int tid = threadIdx.x, ngrp = blockDim.x / G, grp = tid / G, g = tid - grp * G;
  const int trips = (nc + ngrp - 1) / ngrp;
  if (((tid >> 5) << 5) / G >= nc) return;  // whole warp past the last column
  for (int t = 0; t < trips; ++t) {
    const int c = grp + t * ngrp;
    const bool act = c < nc;
    const int k = k0 + (act ? c : 0);
    double w = 0.0;
    const double sjk = act ? S[j * LDS + k] : 0.0;
    if (act)
      for (int i = j + 1 + g; i < rows; i += G) w = fma(S[i * LDS + j], S[i * LDS + k], w);
    for (int o = G >> 1; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    if (act) {
      w = tj * (w + sjk);
      for (int i = j + 1 + g; i < rows; i += G) S[i * LDS + k] -= w * S[i * LDS + j];
      if (g == 0) S[j * LDS + k] = sjk - w;
      if (tau_la && c == 0) {
        const int lane = tid & 31;
        const unsigned gm = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
        __syncwarp(gm);
        double x = 0.0;
        for (int i = k + 1 + g; i < rows; i += G) x = fma(S[i * LDS + k], S[i * LDS + k], x);
        for (int o = G >> 1; o > 0; o >>= 1) x += __shfl_xor_sync(gm, x, o);
        const double alpha = S[k * LDS + k];
        double tk = 0.0;
        if (x > 0.0) {
          const double beta = -copysign(sqrt(alpha * alpha + x), alpha);
          tk = (beta - alpha) / beta;
          const double scl = 1.0 / (alpha - beta);
          for (int i = k + 1 + g; i < rows; i += G) S[i * LDS + k] *= scl;
          __syncwarp(gm);
          if (g == 0) S[k * LDS + k] = beta;
        }
        if (g == 0) tau_la[k] = tk;
      }
    }
  }
}

// The same RK4 over a cluster of SRK_CL CTAs: CTA c owns a block of rows of
// the R x R iterate, forms its rows of G_s W (all of W needed) and of
// (G_s W) F_s (its rows only), and broadcasts its rows of the next stage's W
// into every CTA's shared memory (DSMEM stores; W double-buffered, so one
// cluster barrier per stage). Same products, same summation order as
// s_rk4_kernel, so the result is bit-identical; the work is spread over 8 SMs.
constexpr int SRK_CL = 8;
__global__ void __cluster_dims__(SRK_CL, 1, 1) __launch_bounds__(256)
    s_rk4_cluster_kernel(double* S, int p, int q, const double* G, const double* F, int ns,
                         double dt) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int cr = (int)cl.block_rank();
  const int per = (p + SRK_CL - 1) / SRK_CL;
  const int r0 = cr * per;
  const int nr = r0 < p ? (p - r0 < per ? p - r0 : per) : 0;
  const int pq = p * q;
  double* W0 = sm;                 // p x q, double-buffered across stages
  double* W1 = W0 + pq;
  double* S0 = W1 + pq;            // own rows (per x q)
  double* T = S0 + per * q;        // per x q
  double* Acc = T + per * q;       // per x q
  double* sg = Acc + per * q;      // ns x per x p: own rows of every G_s
  double* sf = sg + (size_t)ns * per * p;  // ns x q x q
  const int tid = threadIdx.x, nthr = blockDim.x;
  for (int i = tid; i < ns * nr * p; i += nthr) {
    const int s = i / (nr * p), rem = i - s * nr * p, a = rem / p, k = rem - a * p;
    sg[(s * per + a) * p + k] = G[(size_t)s * p * p + (size_t)(r0 + a) * p + k];
  }
  for (int i = tid; i < ns * q * q; i += nthr) sf[i] = F[i];
  for (int i = tid; i < pq; i += nthr) W0[i] = S[i];
  for (int i = tid; i < nr * q; i += nthr) S0[i] = S[(size_t)r0 * q + i];
  __syncthreads();
  const double coef[4] = {0.25, 1.0 / 3.0, 0.5, 1.0};
  for (int st = 0; st < 4; ++st) {
    const double* W = (st & 1) ? W1 : W0;
    double* Wn = (st & 1) ? W0 : W1;
    for (int i = tid; i < nr * q; i += nthr) Acc[i] = 0.0;
    for (int s = 0; s < ns; ++s) {
      const double* Gs = sg + (size_t)s * per * p;
      const double* Fs = sf + (size_t)s * q * q;
      __syncthreads();
      for (int i = tid; i < nr * q; i += nthr) {
        const int a = i / q, b = i % q;
        double t0 = 0.0, t1 = 0.0;
        int k = 0;
        for (; k + 1 < p; k += 2) {
          t0 = fma(Gs[a * p + k], W[k * q + b], t0);
          t1 = fma(Gs[a * p + k + 1], W[(k + 1) * q + b], t1);
        }
        if (k < p) t0 = fma(Gs[a * p + k], W[k * q + b], t0);
        T[i] = t0 + t1;
      }
      __syncthreads();
      for (int i = tid; i < nr * q; i += nthr) {
        const int a = i / q, b = i % q;
        double t0 = 0.0, t1 = 0.0;
        int k = 0;
        for (; k + 1 < q; k += 2) {
          t0 = fma(T[a * q + k], Fs[k * q + b], t0);
          t1 = fma(T[a * q + k + 1], Fs[(k + 1) * q + b], t1);
        }
        if (k < q) t0 = fma(T[a * q + k], Fs[k * q + b], t0);
        Acc[i] -= t0 + t1;
      }
    }
    const double c = coef[st] * dt;
    if (st < 3) {
      for (int i = tid; i < nr * q; i += nthr) {
        const double v = S0[i] + c * Acc[i];
        for (int rr = 0; rr < SRK_CL; ++rr) cl.map_shared_rank(Wn, rr)[(size_t)r0 * q + i] = v;
      }
      cl.sync();  // the next stage's W complete in every CTA
    } else {
      for (int i = tid; i < nr * q; i += nthr) S[(size_t)r0 * q + i] = S0[i] + c * Acc[i];
    }
  }
}

// Householder QR with the columns held in registers (rows <= 8 MAXR, cols <= 64):
// one 8-lane group per column for the whole factorisation. Step j: the owner
// of column j forms its reflector from its registers (dlarfg conventions:
// beta = -sign(alpha) |x|, tau = 0 for a zero sub-column) and publishes v_j
// and tau_j in shared memory; after one barrier every later column applies
// H_j from its registers (one group reduction). The explicit Q needs no
// barrier at all: group c applies H_c ... H_0 to e_c from the stored
// reflectors. One barrier per column instead of the shared-matrix kernel's
// serial reflector phase and two barriers (the m-side QRs are latency-bound).
template <int G, int MAXR>
__global__ void __launch_bounds__(G == 8 ? 512 : 640)
    qr_reg_kernel(const double* __restrict__ A, int rows, int cols, int lda,
                  double* __restrict__ Q, int ldq, double* __restrict__ rfac) {
  // G lanes per column (8 up to 128 rows, 16 for the P19 moment count, 400
  // rows); with G = 16 the reflector is re-read from shared memory instead of
  // being held twice in registers
  constexpr bool VREG = MAXR <= 16;
  extern __shared__ double sm[];
  const int kk = rows < cols ? rows : cols;
  double* V = sm;                       // kk x rows: v_j below row j
  double* tau = V + (size_t)kk * rows;  // kk
  const int tid = threadIdx.x, lane = tid & 31, c = tid / G, l = tid % G;
  const unsigned gm = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << (lane & ~(G - 1));
  const bool act = c < cols;
  double x[MAXR];
#pragma unroll
  for (int u = 0; u < MAXR; ++u) {
    const int i = l + G * u;
    x[u] = (act && i < rows) ? A[(size_t)i + (size_t)c * lda] : 0.0;
  }
  for (int j = 0; j < kk; ++j) {
    if (c == j) {
      double s = 0.0, al = 0.0;
#pragma unroll
      for (int u = 0; u < MAXR; ++u) {
        const int i = l + G * u;
        if (i > j) s = fma(x[u], x[u], s);
        if (i == j) al = x[u];
      }
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) {
        s += __shfl_xor_sync(gm, s, o);
        al += __shfl_xor_sync(gm, al, o);
      }
      double tj = 0.0;
      if (s > 0.0) {
        const double beta = -copysign(sqrt(al * al + s), al);
        tj = (beta - al) / beta;
        const double scl = 1.0 / (al - beta);
#pragma unroll
        for (int u = 0; u < MAXR; ++u) {
          const int i = l + G * u;
          if (i > j && i < rows) {
            V[(size_t)j * rows + i] = x[u] * scl;
            x[u] = 0.0;
          }
          if (i == j) x[u] = beta;
        }
      } else {
#pragma unroll
        for (int u = 0; u < MAXR; ++u) {
          const int i = l + G * u;
          if (i > j && i < rows) V[(size_t)j * rows + i] = 0.0;
        }
      }
      if (l == 0) tau[j] = tj;
    }
    __syncthreads();
    if (act && c > j) {
      const double tj = tau[j];
      if (tj != 0.0) {
        double v[VREG ? MAXR : 1];
        double w = 0.0;
#pragma unroll
        for (int u = 0; u < MAXR; ++u) {
          const int i = l + G * u;
          const double vi = i == j ? 1.0 : (i > j && i < rows) ? V[(size_t)j * rows + i] : 0.0;
          if constexpr (VREG) v[u] = vi;
          w = fma(vi, x[u], w);
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) w += __shfl_xor_sync(gm, w, o);
        w *= tj;
#pragma unroll
        for (int u = 0; u < MAXR; ++u) {
          double vi;
          if constexpr (VREG) {
            vi = v[u];
          } else {
            const int i = l + G * u;
            vi = i == j ? 1.0 : (i > j && i < rows) ? V[(size_t)j * rows + i] : 0.0;
          }
          x[u] -= w * vi;
        }
      }
    }
  }
  // triangular factor (kk x cols, row-major): column c is final after step c
  if (act) {
#pragma unroll
    for (int u = 0; u < MAXR; ++u) {
      const int i = l + G * u;
      if (i < kk) rfac[(size_t)i * cols + c] = i <= c ? x[u] : 0.0;
    }
  }
  __syncthreads();
  // explicit Q (rows x kk): column c = H_0 ... H_c e_c (H_j e_c = e_c for j > c)
  if (c < kk) {
#pragma unroll
    for (int u = 0; u < MAXR; ++u) x[u] = (l + G * u == c) ? 1.0 : 0.0;
    for (int j = c; j >= 0; --j) {
      const double tj = tau[j];
      if (tj == 0.0) continue;
      double v[VREG ? MAXR : 1];
      double w = 0.0;
#pragma unroll
      for (int u = 0; u < MAXR; ++u) {
        const int i = l + G * u;
        const double vi = i == j ? 1.0 : (i > j && i < rows) ? V[(size_t)j * rows + i] : 0.0;
        if constexpr (VREG) v[u] = vi;
        w = fma(vi, x[u], w);
      }
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) w += __shfl_xor_sync(gm, w, o);
      w *= tj;
#pragma unroll
      for (int u = 0; u < MAXR; ++u) {
        double vi;
        if constexpr (VREG) {
          vi = v[u];
        } else {
          const int i = l + G * u;
          vi = i == j ? 1.0 : (i > j && i < rows) ? V[(size_t)j * rows + i] : 0.0;
        }
        x[u] -= w * vi;
      }
    }
#pragma unroll
    for (int u = 0; u < MAXR; ++u) {
      const int i = l + G * u;
      if (i < rows) Q[(size_t)i + (size_t)c * ldq] = x[u];
    }
  }
}

// The streaming substep's L phase on the moment side (dlra.py:176-194) for
// small moment counts, fused over a cluster of LRK_CL CTAs: L0 = V0 S0^T, then
// the Horner RK4 of L' = -sum_s A_s L Q_s (Q_s^T = the leading a x a block of
// the S-phase Gram G_s): CTA c owns a block of rows, forms its rows of
// Z_s = L Q_s^T (broadcast into every CTA's shared memory: A_s L needs all of
// Z) and its rows of the next iterate (broadcast as well). Writes L1 (m x a
// row-major) and BV = [L1 | V0] column-major, the next orthonormalisation's
// input. Replaces ~20 small launches per step (GEMMs, split-K reductions,
// copies, transposes) by one.
constexpr int LRK_CL = 8;
__global__ void __cluster_dims__(LRK_CL, 1, 1) __launch_bounds__(256)
    l_rk4_cluster_kernel(const double* __restrict__ V, const double* __restrict__ S,
                         const double* __restrict__ G, int ru, const double* __restrict__ amat,
                         int m, int a, int b, int ns, double dt, double* __restrict__ L1,
                         double* __restrict__ BV) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int cr = (int)cl.block_rank();
  const int per = (m + LRK_CL - 1) / LRK_CL;
  const int r0 = cr * per;
  const int nr = r0 < m ? (m - r0 < per ? m - r0 : per) : 0;
  const int ma = m * a;
  double* LW0 = sm;                          // m x a (all rows), double-buffered
  double* LW1 = LW0 + ma;
  double* Z = LW1 + ma;                      // ns x m x a
  double* Ar = Z + (size_t)ns * ma;          // ns x per x m: own rows of every A_s
  double* Gs = Ar + (size_t)ns * per * m;    // ns x a x a: Q_s^T blocks
  double* L0r = Gs + (size_t)ns * a * a;     // per x a
  const int tid = threadIdx.x, nthr = blockDim.x;
  for (int i = tid; i < ns * nr * m; i += nthr) {
    const int s = i / (nr * m), rem = i - s * nr * m, r = rem / m, p = rem - r * m;
    Ar[(s * per + r) * m + p] = amat[((size_t)s * m + r0 + r) * m + p];
  }
  for (int i = tid; i < ns * a * a; i += nthr) {
    const int s = i / (a * a), rem = i - s * a * a, j = rem / a, k = rem - j * a;
    Gs[i] = G[(size_t)s * ru * ru + (size_t)j * ru + k];
  }
  // L0 = V S^T, own rows; broadcast as the first iterate
  for (int i = tid; i < nr * a; i += nthr) {
    const int r = i / a, j = i - r * a;
    double acc = 0.0;
    for (int k = 0; k < b; ++k) acc = fma(V[(size_t)(r0 + r) * b + k], S[(size_t)j * b + k], acc);
    L0r[i] = acc;
    for (int rr = 0; rr < LRK_CL; ++rr) cl.map_shared_rank(LW0, rr)[(r0 + r) * a + j] = acc;
  }
  // V0 into BV's last b columns (column-major)
  for (int i = tid; i < nr * b; i += nthr) {
    const int r = i / b, k = i - r * b;
    BV[(size_t)a * m + (size_t)k * m + r0 + r] = V[(size_t)(r0 + r) * b + k];
  }
  cl.sync();
  const double coef[4] = {0.25, 1.0 / 3.0, 0.5, 1.0};
  for (int st = 0; st < 4; ++st) {
    const double* W = (st & 1) ? LW1 : LW0;
    double* Wn = (st & 1) ? LW0 : LW1;
    // Z_s rows: Z_s[r][j] = sum_i W[r][i] Q_s^T[j][i]
    for (int i = tid; i < ns * nr * a; i += nthr) {
      const int s = i / (nr * a), rem = i - s * nr * a, r = rem / a, j = rem - r * a;
      const double* w = W + (r0 + r) * a;
      const double* g = Gs + (s * a + j) * a;
      double acc = 0.0;
      for (int k = 0; k < a; ++k) acc = fma(w[k], g[k], acc);
      for (int rr = 0; rr < LRK_CL; ++rr)
        cl.map_shared_rank(Z, rr)[(size_t)s * ma + (r0 + r) * a + j] = acc;
    }
    cl.sync();  // every row of every Z_s in every CTA
    const double c = -coef[st] * dt;
    for (int i = tid; i < nr * a; i += nthr) {
      const int r = i / a, j = i - r * a;
      double t0 = 0.0, t1 = 0.0;
      for (int s = 0; s < ns; ++s) {
        const double* ar = Ar + (s * per + r) * m;
        const double* z = Z + (size_t)s * ma + j;
        int p = 0;
        for (; p + 1 < m; p += 2) {
          t0 = fma(ar[p], z[p * a], t0);
          t1 = fma(ar[p + 1], z[(p + 1) * a], t1);
        }
        if (p < m) t0 = fma(ar[p], z[p * a], t0);
      }
      const double v = fma(c, t0 + t1, L0r[i]);
      if (st < 3) {
        for (int rr = 0; rr < LRK_CL; ++rr) cl.map_shared_rank(Wn, rr)[(r0 + r) * a + j] = v;
      } else {
        L1[(size_t)(r0 + r) * a + j] = v;
        BV[(size_t)j * m + r0 + r] = v;
      }
    }
    if (st < 3) cl.sync();  // the next iterate complete (and Z free) in every CTA
  }
}

// Householder QR of a whole (rows x cols) column-major matrix in one CTA
// (the m-side factors: rows = m moments <= ~600): the matrix lives in shared
// memory, the reflectors are those of hh_qr_kernel (beta = -sign(alpha) ||x||,
// tau = 0 for a zero sub-column), and the explicit Q is then formed in place by
// applying the reflectors backwards (LAPACK dorg2r order). Replaces a TSQR
// tree of several launches by one launch for the small m-side QRs.
// gw: when the matrix does not fit in shared memory (wide factors: cols > 64)
// it lives in this global (L2-resident) work buffer instead -- same algorithm
__global__ void __launch_bounds__(512)
    qr_small_kernel(const double* __restrict__ A, int rows, int cols, int lda,
                    double* __restrict__ Q, int ldq, double* __restrict__ rfac,
                    double* __restrict__ gw) {
  extern __shared__ double sm[];
  const int LDS = cols | 1;  // odd row length: conflict-free column walks
  double* S = gw ? gw : sm;            // rows x LDS
  double* tau = (gw ? sm : S + (size_t)rows * LDS) + 32 + cols;  // cols
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  for (int idx = tid; idx < rows * cols; idx += nthr) {
    const int i = idx % rows, j = idx / rows;
    S[i * LDS + j] = A[(size_t)i + (size_t)j * lda];
  }
  __syncthreads();
  const int kk = rows < cols ? rows : cols;
  for (int j = 0; j < kk && j < 1; ++j) {
    // the reflector of column 0 in one warp; the later ones are formed by the
    // column groups one step ahead (hh_apply_groups look-ahead)
    if (warp == 0) {
      double part = 0.0;
      for (int i = j + 1 + lane; i < rows; i += 32) part += S[i * LDS + j] * S[i * LDS + j];
      const double xnorm2 = warp_sum(part);
      double tj = 0.0;
      if (xnorm2 > 0.0) {
        const double alpha = S[j * LDS + j];
        const double beta = -copysign(sqrt(alpha * alpha + xnorm2), alpha);
        tj = (beta - alpha) / beta;
        const double scl = 1.0 / (alpha - beta);
        for (int i = j + 1 + lane; i < rows; i += 32) S[i * LDS + j] *= scl;
        __syncwarp();
        if (lane == 0) S[j * LDS + j] = beta;
      }
      if (lane == 0) tau[j] = tj;
    }
    __syncthreads();
  }
  for (int j = 0; j < kk; ++j) {
    // H_j on the trailing columns; with a next reflector to form, the apply
    // runs even for tau_j = 0 (w = 0) so the look-ahead group forms it
    if (tau[j] != 0.0 || j + 1 < kk)
      hh_apply_groups(S, LDS, rows, j, j + 1, cols, tau[j], j + 1 < kk ? tau : nullptr);
    __syncthreads();
  }
  // triangular factor (kk x cols, row-major)
  for (int idx = tid; idx < kk * cols; idx += nthr) {
    const int i = idx / cols, j = idx - i * cols;
    rfac[idx] = i <= j ? S[i * LDS + j] : 0.0;
  }
  __syncthreads();
  // explicit Q (rows x kk) in place, reflectors applied backwards
  for (int j = kk - 1; j >= 0; --j) {
    const double tj = tau[j];
    if (j < kk - 1 && tj != 0.0) {
      hh_apply_groups(S, LDS, rows, j, j + 1, kk, tj);
      __syncthreads();
    }
    for (int i = tid; i < rows; i += nthr) {
      double v;
      if (i < j) v = 0.0;
      else if (i == j) v = 1.0 - tj;
      else v = -tj * S[i * LDS + j];
      S[i * LDS + j] = v;
    }
    __syncthreads();
  }
  for (int idx = tid; idx < rows * kk; idx += nthr) {
    const int i = idx % rows, j = idx / rows;
    Q[(size_t)i + (size_t)j * ldq] = S[i * LDS + j];
  }
}

void set_smem(const void* fn, size_t bytes) {
  if (bytes > (size_t)kMaxDynSmem) fail(PND_ECONFIG, "kernel tile exceeds shared memory");
  allow_max_smem(fn);
}

// partition of a level: leaves of `br` rows, a short tail merged into the
// previous block so every block but a lone one has >= cols rows
Part make_part(int rows, int cols, int br) {
  Part p{rows, cols, br, 0};
  if (rows <= br) {
    p.nblk = 1;
    p.br = rows;
    return p;
  }
  int nb = rows / br;
  const int tail = rows - nb * br;
  if (tail >= cols) nb += 1;  // tail is its own block (count = tail)
  p.nblk = nb;                // else the tail is merged into the last block
  return p;
}

}  // namespace

namespace {
// C = beta C + alpha sum_s P_s over the split-K partials (fixed order)
__global__ void splitk_reduce(const double* __restrict__ P, int splits, int M, int N, double alpha,
                              double beta, Mat C) {
  const int total = M * N;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < splits; ++b) s += P[(size_t)b * total + e];
    const int i = e / N, j = e - i * N;
    double* c = C.p + (long)i * C.rs + (long)j * C.cs;
    *c = beta == 0.0 ? alpha * s : alpha * s + beta * (*c);
  }
}
}  // namespace

void gemm(int M, int N, int K, double alpha, Mat A, long sA, Mat B, long sB, double beta, Mat C,
          long sC, int batch, cudaStream_t st) {
  if (M <= 0 || N <= 0 || batch <= 0) return;
  const int tiles = ((N + 15) / 16) * ((M + 15) / 16);
  if (batch == 1 && K >= 256 && tiles < 148) {
    // long-K, few tiles (the L phase's A^T Z, K = ns m): split K over CTAs,
    // partials reduced in a fixed order
    int splits = K / 128;
    if (splits > 16) splits = 16;
    const int kb = (K + splits - 1) / splits;
    splits = (K + kb - 1) / kb;
    double* P = nullptr;
    CK(cudaMallocAsync((void**)&P, (size_t)splits * M * N * sizeof(double), st));
    dim3 grid((N + 15) / 16, (M + 15) / 16, splits), block(16, 16);
    const Mat Pm{P, N, 1};
    // batch b multiplies K-slice [b kb, b kb + kb): A advanced along k (cs), B along k (rs)
    gemm_kernel<<<grid, block, 0, st>>>(M, N, kb, 1.0, A, (long)kb * A.cs, B, (long)kb * B.rs, 0.0,
                                         Pm, (long)M * N, K);
    launched();
    splitk_reduce<<<(M * N + 255) / 256, 256, 0, st>>>(P, splits, M, N, alpha, beta, C);
    launched();
    CK(cudaFreeAsync(P, st));
    return;
  }
  dim3 grid((N + 15) / 16, (M + 15) / 16, batch), block(16, 16);
  gemm_kernel<<<grid, block, 0, st>>>(M, N, K, alpha, A, sA, B, sB, beta, C, sC, 0);
  launched();
}

void axpby(int count, double a, const double* x, double b, double* y, cudaStream_t st) {
  if (count <= 0) return;
  int blocks = (count + 255) / 256;
  if (blocks > 1024) blocks = 1024;
  axpby_kernel<<<blocks, 256, 0, st>>>(count, a, x, b, y);
  launched();
}

int tsqr(double* a, int rows, int cols, int lda, double* q, int ldq, double* rfac, TsqrWork& w,
         cudaStream_t st) {
  if (cols > 512) fail(PND_ECONFIG, "orthonormalisation supports at most 512 columns");
  const int kc = rows < cols ? rows : cols;
  {
    // whole matrix in one CTA when it fits (the m-side QRs)
    const size_t sm = ((size_t)rows * (cols | 1) + 32 + 2 * (size_t)cols) * sizeof(double);
    const size_t smr = ((size_t)kc * rows + kc) * sizeof(double);
    if (!getenv("PND_QR_SHARED") && smr + 1024 <= (size_t)kMaxDynSmem &&
        ((rows <= 128 && cols <= 64) || (rows <= 416 && cols <= 40))) {
      // columns in registers: one 8-lane group per column up to 128 rows, 16 lanes
      // up to 416 (the P19 moment count)
      if (rows <= 128) {
        const int thr = ((8 * cols + 31) / 32) * 32;
        if (rows <= 64) {
          set_smem((const void*)qr_reg_kernel<8, 8>, smr);
          qr_reg_kernel<8, 8><<<1, thr, smr, st>>>(a, rows, cols, lda, q, ldq, rfac);
        } else {
          set_smem((const void*)qr_reg_kernel<8, 16>, smr);
          qr_reg_kernel<8, 16><<<1, thr, smr, st>>>(a, rows, cols, lda, q, ldq, rfac);
        }
      } else {
        const int thr = ((16 * cols + 31) / 32) * 32;
        set_smem((const void*)qr_reg_kernel<16, 26>, smr);
        qr_reg_kernel<16, 26><<<1, thr, smr, st>>>(a, rows, cols, lda, q, ldq, rfac);
      }
      launched();
      return kc;
    }
    if (sm + 1024 <= (size_t)kMaxDynSmem) {
      // one 8-lane group per column up to 128 rows, 16 warps from a few hundred rows
      int thr = rows <= 128 ? 8 * cols : 512;  // one 8-lane group per column
      thr = thr > 512 ? 512 : ((thr + 31) / 32) * 32;
      set_smem((const void*)qr_small_kernel, sm);
      qr_small_kernel<<<1, thr, sm, st>>>(a, rows, cols, lda, q, ldq, rfac, nullptr);
      launched();
      return kc;
    }
    if (cols > 64) {
      // wide factors (more than 64 columns): the same one-CTA Householder QR
      // with the matrix in a global, L2-resident work buffer
      if ((size_t)rows * cols > ((size_t)1 << 24))
        fail(PND_ECONFIG, "orthonormalisation of more than 64 columns supports <= 2^24 entries");
      double* gw = w.rbuf.get((size_t)rows * (cols | 1));
      const size_t sms = (32 + 2 * (size_t)cols) * sizeof(double);
      qr_small_kernel<<<1, 512, sms, st>>>(a, rows, cols, lda, q, ldq, rfac, gw);
      launched();
      return kc;
    }
  }
  // level matrices: level 0 is `a`; level l+1 holds the stacked R's of level l
  struct Level {
    double* mat;
    int ld;
    Part part;
    double* tau;
    double* qexp;  // explicit Q of this level (non-leaf levels)
  };
  std::vector<Level> lv;
  const int br0 = 128;
  const int grp = cols > 32 ? 2 : (cols > 16 ? 4 : 8);
  // sizes
  size_t tree_need = 0, tau_need = 0, q_need = 0;
  {
    int r = rows;
    Part p = make_part(r, cols, br0);
    for (;;) {
      tau_need += (size_t)p.nblk * cols;
      const int next_rows = p.nblk * cols;
      tree_need += (size_t)next_rows * cols;
      if (p.nblk == 1) break;
      q_need += (size_t)next_rows * cols;
      p = make_part(next_rows, cols, grp * cols);
    }
  }
  double* tree = w.tree.get(tree_need);
  double* taus = w.tau.get(tau_need);
  double* qbuf = w.cbuf.get(q_need > 0 ? q_need : 1);
  {
    double* mat = a;
    int ld = lda;
    Part p = make_part(rows, cols, br0);
    size_t toff = 0, taoff = 0, qoff = 0;
    for (;;) {
      Level L{mat, ld, p, taus + taoff, nullptr};
      taoff += (size_t)p.nblk * cols;
      double* Rn = tree + toff;
      const int ldn = p.nblk * cols;
      toff += (size_t)ldn * cols;
      // QR of every block of this level
      const int tail_b = p.nblk - 1;
      const int nreg = p.nblk - 1;
      if (nreg > 0) {
        const size_t sm = ((size_t)p.br * (cols + 1) + 32 + cols) * sizeof(double);
        set_smem((const void*)hh_qr_kernel, sm);
        hh_qr_kernel<<<nreg, 128, sm, st>>>(mat, ld, p, 0, L.tau, Rn, ldn);
        launched();
      }
      {
        const size_t sm = ((size_t)p.count(tail_b) * (cols + 1) + 32 + cols) * sizeof(double);
        set_smem((const void*)hh_qr_kernel, sm);
        hh_qr_kernel<<<1, 128, sm, st>>>(mat, ld, p, tail_b, L.tau, Rn, ldn);
        launched();
      }
      lv.push_back(L);
      if (p.nblk == 1) {
        // root: its R block (kc x cols) is the triangular factor
        copy_rfac_kernel<<<1, 256, 0, st>>>(Rn, ldn, p.rows < cols ? p.rows : cols, cols, rfac);
        launched();
        break;
      }
      lv.back().qexp = qbuf + qoff;  // explicit Q of the NEXT level is stored per level below
      qoff += (size_t)ldn * cols;
      mat = Rn;
      ld = ldn;
      p = make_part(ldn, cols, grp * cols);
    }
  }
  // top-down explicit Q: level L-1 (root) down to 0
  const double* C = nullptr;
  int ldc = 0;
  for (int l = (int)lv.size() - 1; l >= 0; --l) {
    Level& L = lv[l];
    const Part& p = L.part;
    const int kcl = (l == (int)lv.size() - 1) ? (p.rows < cols ? p.rows : cols) : cols;
    double* out;
    int ldo;
    if (l == 0) {
      out = q;
      ldo = ldq;
    } else {
      out = lv[l - 1].qexp;
      ldo = p.rows;
    }
    const int nreg = p.nblk - 1;
    if (nreg > 0) {
      const size_t sm = ((size_t)p.br * (cols + 1 + kcl + 1) + kcl) * sizeof(double);
      set_smem((const void*)hh_applyq_kernel, sm);
      hh_applyq_kernel<<<nreg, 128, sm, st>>>(L.mat, L.ld, p, 0, L.tau, C, ldc, kcl, out, ldo);
      launched();
    }
    {
      const size_t sm =
          ((size_t)p.count(p.nblk - 1) * (cols + 1 + kcl + 1) + kcl) * sizeof(double);
      set_smem((const void*)hh_applyq_kernel, sm);
      hh_applyq_kernel<<<1, 128, sm, st>>>(L.mat, L.ld, p, p.nblk - 1, L.tau, C, ldc, kcl, out,
                                           ldo);
      launched();
    }
    C = out;
    ldc = ldo;
  }
  return kc;
}

void svd_small(const double* s, int p, int q, double* P, double* sig, double* Qt, double*,
               cudaStream_t st) {
  const int M = p >= q ? p : q, N = p >= q ? q : p;
  if (M > 512 || N > 512) fail(PND_ECONFIG, "truncation SVD supports at most 512 x 512");
  const int N2 = N + (N & 1);
  const size_t mats = (size_t)M * N2 + (size_t)N2 * N2 + (size_t)M * N;
  size_t sm = (mats + N2) * sizeof(double) + N * sizeof(int);
  double* gw = nullptr;
  if (sm + 1024 > (size_t)kMaxDynSmem) {
    // wide R x R: V and U in a global (L2-resident) work buffer, stream-ordered;
    // above ~160 columns A as well (svd_kernel a_in_gw)
    const size_t vu = (size_t)N2 * N2 + (size_t)M * N + (size_t)M * N2;
    CK(cudaMallocAsync((void**)&gw, vu * sizeof(double), st));
    sm = ((size_t)M * N2 + N2) * sizeof(double) + N * sizeof(int);
    if (sm + 1024 > (size_t)kMaxDynSmem) sm = (size_t)N2 * sizeof(double) + N * sizeof(int);
  }
  // one warp per Jacobi pair of a round (two per warp above 64 columns)
  int threads = 32 * (N2 / 2);
  if (threads < 64) threads = 64;
  if (threads > 1024) threads = 1024;
  if (M <= 64 && !getenv("PND_SVD_PLAIN")) {
    const size_t smq = ((size_t)M * N + (size_t)N * N2 + (size_t)N2 * N2 + (size_t)N * N +
                        N + 2 * N2) * sizeof(double) + 2 * N * sizeof(int);
    // one 8-lane group per Jacobi pair; rows per lane = ceil(M / 8)
    // one 8-lane group per column in the QR, per Jacobi pair in the sweeps
    int thq = ((QJ_G * (N > N2 / 2 ? N : N2 / 2) + 31) / 32) * 32;
    if (thq < 64) thq = 64;
    const int rpl = (M + QJ_G - 1) / QJ_G;
    auto kq = svd_qrj_kernel<8>;
    switch (rpl) {
      case 1: kq = svd_qrj_kernel<1>; break;
      case 2: kq = svd_qrj_kernel<2>; break;
      case 3: kq = svd_qrj_kernel<3>; break;
      case 4: kq = svd_qrj_kernel<4>; break;
      case 5: kq = svd_qrj_kernel<5>; break;
      case 6: kq = svd_qrj_kernel<6>; break;
      case 7: kq = svd_qrj_kernel<7>; break;
      default: break;
    }
    set_smem((const void*)kq, smq);
    // PND_SVD_STOP=1/2: stop after the QR / the Jacobi sweeps (phase timing only)
    const char* stop = getenv("PND_SVD_STOP");
    kq<<<1, thq, smq, st>>>(s, p, q, P, sig, Qt, stop ? atoi(stop) : 0);
  } else if (M <= 64) {
    set_smem((const void*)svd_kernel<2>, sm);
    svd_kernel<2><<<1, threads, sm, st>>>(s, p, q, P, sig, Qt, gw);
  } else if (M <= 128) {
    set_smem((const void*)svd_kernel<4>, sm);
    svd_kernel<4><<<1, threads, sm, st>>>(s, p, q, P, sig, Qt, gw);
  } else if (M <= 256) {
    set_smem((const void*)svd_kernel<8>, sm);
    svd_kernel<8><<<1, threads, sm, st>>>(s, p, q, P, sig, Qt, gw);
  } else {
    set_smem((const void*)svd_kernel<16>, sm);
    svd_kernel<16><<<1, threads, sm, st>>>(s, p, q, P, sig, Qt, gw);
  }
  launched();
  if (gw) CK(cudaFreeAsync(gw, st));
}

void tail_rule(const double* sig, int k, double theta, int rmin, int rmax, int* info,
               double* tail, cudaStream_t st) {
  if (k > 512) fail(PND_ECONFIG, "tail rule supports at most 512 singular values");
  tail_kernel<<<1, 32, 0, st>>>(sig, k, theta, rmin, rmax, info, tail);
  launched();
}

void scat_solves(const double* B, const double* coeffs, const double* lcols, int r, int m,
                 double dt, double* lnew, int* singular, cudaStream_t st) {
  const size_t sm = ((size_t)r * (r + 1) + r) * sizeof(double);
  if (sm + 1024 > (size_t)kMaxDynSmem) {
    double* gw = nullptr;
    CK(cudaMallocAsync((void**)&gw, sm * m, st));
    scat_solve_kernel<<<m, 128, 0, st>>>(B, coeffs, lcols, r, m, dt, lnew, singular, gw);
    launched();
    CK(cudaFreeAsync(gw, st));
    return;
  }
  set_smem((const void*)scat_solve_kernel, sm);
  scat_solve_kernel<<<m, 64, sm, st>>>(B, coeffs, lcols, r, m, dt, lnew, singular, nullptr);
  launched();
}

bool l_rk4(const double* V, const double* S, const double* G, int ru, const double* amat, int m,
           int a, int b, int ns, double dt, double* L1, double* BV, cudaStream_t st) {
  if (getenv("PND_LRK4_GEMM")) return false;
  const int per = (m + LRK_CL - 1) / LRK_CL;
  const size_t smem = (2 * (size_t)m * a + (size_t)ns * m * a + (size_t)ns * per * m +
                       (size_t)ns * a * a + (size_t)per * a) * sizeof(double);
  if (smem + 1024 > (size_t)kMaxDynSmem) return false;
  set_smem((const void*)l_rk4_cluster_kernel, smem);
  l_rk4_cluster_kernel<<<LRK_CL, 256, smem, st>>>(V, S, G, ru, amat, m, a, b, ns, dt, L1, BV);
  launched();
  return true;
}

void s_rk4(double* S, int p, int q, const double* G, const double* F, int ns, double dt, double*,
           cudaStream_t st) {
  const size_t sm = 4 * (size_t)p * q * sizeof(double);
  const size_t sm_staged = sm + ((size_t)ns * ((size_t)p * p + (size_t)q * q)) * sizeof(double);
  const bool staged = sm_staged + 1024 <= (size_t)kMaxDynSmem;
  if (!staged && sm + 1024 > (size_t)kMaxDynSmem) {
    // wide: the four R x R work matrices in global memory (stream-ordered)
    double* gw = nullptr;
    CK(cudaMallocAsync((void**)&gw, 4 * (size_t)p * q * sizeof(double), st));
    s_rk4_kernel<<<1, 1024, 0, st>>>(S, p, q, G, F, ns, dt, 0, gw);
    launched();
    CK(cudaFreeAsync(gw, st));
    return;
  }
  const int per = (p + SRK_CL - 1) / SRK_CL;
  const size_t sm_cl = (2 * (size_t)p * q + 3 * (size_t)per * q + (size_t)ns * per * p +
                        (size_t)ns * q * q) * sizeof(double);
  if (sm_cl + 1024 <= (size_t)kMaxDynSmem && !getenv("PND_SRK4_ONE")) {
    set_smem((const void*)s_rk4_cluster_kernel, sm_cl);
    s_rk4_cluster_kernel<<<SRK_CL, 256, sm_cl, st>>>(S, p, q, G, F, ns, dt);
    launched();
    return;
  }
  set_smem((const void*)s_rk4_kernel, staged ? sm_staged : sm);
  s_rk4_kernel<<<1, 1024, staged ? sm_staged : sm, st>>>(S, p, q, G, F, ns, dt, staged ? 1 : 0,
                                                           nullptr);
  launched();
}

}  // namespace pnd
