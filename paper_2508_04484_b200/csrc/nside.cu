// Cell-parallel (n-side) kernels of the energy step.
//
// kstage: one Horner stage of the K-phase RK4 (dlra.py:168-174, 118-123),
//   out = U0 S0 + sum_s (D_s S^-1 X) M_s, thread per cell. The 13-point
//   neighbourhood of the cell (+-1, +-2 along each active axis) is read per
//   column through L1/L2 (column-major layout: x neighbours are in the same
//   256-byte segment, y/z neighbours are re-reads the L2 holds), the ns
//   r x r contraction matrices sit in shared memory and are read as warp
//   broadcasts. With U0 = null and M_s = -A_s it is the full-rank streaming
//   operator F_S (spatial.py:148-167).
// rotate / scat_k1 / dose: row-local contractions of the truncation
//   (dlra.py:111-113), the scattering K-step (dlra.py:303, 244-251) and the
//   dose trapezoid (driver.py:606, 613-622).
#include "pnd.h"

namespace pnd {

namespace {

struct Nbr {
  // per active axis: f at offsets -2..+2 (index 2 = centre), valid flags by position
  int idx[3], len[3], st[3];
};

template <int NB>
__global__ void __launch_bounds__(128) kstage_kernel(KStageArgs a) {
  extern __shared__ double sm[];
  const Geom& g = a.geo;
  const int ns = g.ns;
  const int r = a.r, xc = a.xc, ra = a.ra;
  double* sM = sm;                   // ns * xc * NB
  double* sS = sm + ns * xc * NB;    // ra * NB
  for (int i = threadIdx.x; i < ns * xc * NB; i += blockDim.x) {
    const int s = i / (xc * NB), rem = i - s * xc * NB, j = rem / NB, k = rem - j * NB;
    sM[i] = k < r ? a.M[(s * xc + j) * r + k] : 0.0;
  }
  if (a.U0) {
    for (int i = threadIdx.x; i < ra * NB; i += blockDim.x) {
      const int j = i / NB, k = i - j * NB;
      sS[i] = k < r ? a.S0[j * r + k] : 0.0;
    }
  }
  __syncthreads();
  const int nxy = g.nx * g.ny;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < g.n; c += gridDim.x * blockDim.x) {
    const int ck = c / nxy, rem = c - ck * nxy;
    const int cj = rem / g.nx, ci = rem - cj * g.nx;
    // per active axis: neighbour offsets and inv_s at -2..+2
    double is[3][5];
    int off[3][5];
    bool ok[3][5];
#pragma unroll
    for (int ai = 0; ai < 3; ++ai) {
      if (ai < g.na) {
        const int axis = g.axis[ai];
        const int len = axis == 0 ? g.nx : (axis == 1 ? g.ny : g.nz);
        const int idx = axis == 0 ? ci : (axis == 1 ? cj : ck);
        const int st = axis == 0 ? 1 : (axis == 1 ? g.nx : nxy);
#pragma unroll
        for (int d = 0; d < 5; ++d) {
          const int q = idx + d - 2;
          ok[ai][d] = q >= 0 && q < len;
          off[ai][d] = c + (d - 2) * st;
          is[ai][d] = ok[ai][d] ? a.inv_s[off[ai][d]] : 0.0;
        }
      }
    }
    double acc[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) acc[k] = 0.0;
    if (a.U0) {
      for (int j = 0; j < ra; ++j) {
        const double u = a.U0[(size_t)j * a.ldu + c];
        if (a.copy_u) a.copy_u[(size_t)j * a.ldc + c] = u;
        const double* srow = sS + j * NB;
#pragma unroll
        for (int k = 0; k < NB; ++k) acc[k] = fma(u, srow[k], acc[k]);
      }
    }
    for (int j = 0; j < xc; ++j) {
      const double* col = a.X + (size_t)j * a.ldx;
#pragma unroll
      for (int ai = 0; ai < 3; ++ai) {
        if (ai < g.na) {
          const int axis = g.axis[ai];
          const double ih = g.ih[axis], i2h = g.i2h[axis];
          double f[5];
#pragma unroll
          for (int d = 0; d < 5; ++d) f[d] = ok[ai][d] ? col[off[ai][d]] * is[ai][d] : 0.0;
          // D^+ (minus-biased) and D^- (plus-biased), spatial.py:81-118
          double tp, tm;
          if (ok[ai][0]) tp = (3.0 * f[2] - 4.0 * f[1] + f[0]) * i2h;
          else if (ok[ai][1]) tp = (f[2] - f[1]) * ih;
          else tp = f[2] * ih;
          if (ok[ai][4]) tm = (-3.0 * f[2] + 4.0 * f[3] - f[4]) * i2h;
          else if (ok[ai][3]) tm = (f[3] - f[2]) * ih;
          else tm = -f[2] * ih;
          const double* mp = sM + ((2 * ai) * xc + j) * NB;
          const double* mm = sM + ((2 * ai + 1) * xc + j) * NB;
#pragma unroll
          for (int k = 0; k < NB; ++k) acc[k] = fma(tp, mp[k], fma(tm, mm[k], acc[k]));
        }
      }
    }
#pragma unroll
    for (int k = 0; k < NB; ++k)
      if (k < r) a.out[(size_t)k * a.ldo + c] = acc[k];
  }
}

template <int NB>
void kstage_launch(const KStageArgs& a, cudaStream_t st) {
  const size_t smem = ((size_t)a.geo.ns * a.xc * NB + (size_t)a.ra * NB) * sizeof(double);
  CK(cudaFuncSetAttribute(kstage_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)smem));
  int dev = 0, sms = 148;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int blocks = (a.geo.n + 127) / 128;
  const int cap = sms * 8;
  if (blocks > cap) blocks = cap;
  kstage_kernel<NB><<<blocks, 128, smem, st>>>(a);
  launched();
}

template <int NB>
__global__ void __launch_bounds__(128) rotate_kernel(Geom g, const double* __restrict__ X, int ldx,
                                                     int na, const double* __restrict__ P, int ldp,
                                                     int nb, double* __restrict__ out, int ldo) {
  extern __shared__ double sP[];  // na x NB
  for (int i = threadIdx.x; i < na * NB; i += blockDim.x) {
    const int j = i / NB, k = i - j * NB;
    sP[i] = k < nb ? P[j * ldp + k] : 0.0;
  }
  __syncthreads();
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < g.n; c += gridDim.x * blockDim.x) {
    double acc[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) acc[k] = 0.0;
    for (int j = 0; j < na; ++j) {
      const double x = X[(size_t)j * ldx + c];
      const double* pr = sP + j * NB;
#pragma unroll
      for (int k = 0; k < NB; ++k) acc[k] = fma(x, pr[k], acc[k]);
    }
#pragma unroll
    for (int k = 0; k < NB; ++k)
      if (k < nb) out[(size_t)k * ldo + c] = acc[k];
  }
}

template <int NB>
__global__ void __launch_bounds__(128) scat_k1_kernel(
    Geom g, const double* __restrict__ U0, int ldu, int ra, const double* __restrict__ S0, int r,
    double dt, const double* __restrict__ inv_s, const int* __restrict__ cls,
    const double* __restrict__ atomic, const double* __restrict__ psi, int ldpsi, int n_beams,
    const double* __restrict__ rows, double* __restrict__ A, int lda) {
  extern __shared__ double sm[];
  double* sS = sm;                    // ra x NB
  double* sR = sm + ra * NB;          // n_beams x 12 x NB
  for (int i = threadIdx.x; i < ra * NB; i += blockDim.x) {
    const int j = i / NB, k = i - j * NB;
    sS[i] = k < r ? S0[j * r + k] : 0.0;
  }
  for (int i = threadIdx.x; i < n_beams * 12 * NB; i += blockDim.x) {
    const int bi = i / NB, k = i - bi * NB;
    sR[i] = k < r ? rows[bi * r + k] : 0.0;
  }
  __syncthreads();
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < g.n; c += gridDim.x * blockDim.x) {
    double acc[NB], src[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) acc[k] = src[k] = 0.0;
    for (int j = 0; j < ra; ++j) {
      const double u = U0[(size_t)j * ldu + c];
      A[(size_t)(r + j) * lda + c] = u;
      const double* srow = sS + j * NB;
#pragma unroll
      for (int k = 0; k < NB; ++k) acc[k] = fma(u, srow[k], acc[k]);
    }
    // source rows: sum_b sum_i (N_i S^-1 psi_b)(c) * rows_b[i]  (dlra.py:244-251)
    const double is = inv_s[c];
    const int kc = cls[c];
    for (int b = 0; b < n_beams; ++b) {
      const double sp = is * psi[(size_t)b * ldpsi + c];
      for (int i = 0; i < 12; ++i) {
        const double x = atomic[kc * 12 + i] * sp;
        const double* rr = sR + (b * 12 + i) * NB;
#pragma unroll
        for (int k = 0; k < NB; ++k) src[k] = fma(x, rr[k], src[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < NB; ++k)
      if (k < r) A[(size_t)k * lda + c] = acc[k] + dt * src[k];
  }
}

__global__ void dose_kernel(Geom g, const double* __restrict__ U, int ldu,
                            const double* __restrict__ coef, int r, double half_dt,
                            const double* __restrict__ s_field, const double* __restrict__ psi,
                            int ldpsi, int n_beams, double* __restrict__ dep,
                            double* __restrict__ prev) {
  const double sqrt4pi = 3.5449077018110318;  // sqrt(4 pi), driver.py:59
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < g.n; c += gridDim.x * blockDim.x) {
    double u0 = 0.0;
    for (int j = 0; j < r; ++j) u0 = fma(U[(size_t)j * ldu + c], coef[j], u0);
    double integrand = sqrt4pi * u0;
    if (psi) {
      double ps = 0.0;
      for (int b = 0; b < n_beams; ++b) ps += psi[(size_t)b * ldpsi + c];
      integrand = integrand + s_field[c] * ps;
    }
    dep[c] += half_dt * (prev[c] + integrand);
    prev[c] = integrand;
  }
}

__global__ void class_gather_kernel(const int* __restrict__ cls, const double* __restrict__ val,
                                    int n, double* __restrict__ inv, double* __restrict__ out) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const double s = val[cls[c]];
    if (inv) inv[c] = 1.0 / s;
    if (out) out[c] = s;
  }
}

__global__ void lerp_kernel(const double* __restrict__ v, int ldv, int n, int j0, double w0,
                            int j1, double w1, double* __restrict__ out) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    double x;
    if (w1 == 0.0) {
      x = w0 == 1.0 ? v[(size_t)j0 * ldv + c] : w0 * v[(size_t)j0 * ldv + c];
    } else {
      x = w0 * v[(size_t)j0 * ldv + c] + w1 * v[(size_t)j1 * ldv + c];
    }
    out[c] = x;
  }
}

// row-major (n x c) host layout <-> column-major (ld) device layout
__global__ void tin_kernel(const double* __restrict__ src, int n, int cdim, double* __restrict__ dst,
                           int ldd) {
  __shared__ double tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int row = r0 + i, col = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (row < n && col < cdim) ? src[(size_t)row * cdim + col] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int col = c0 + i, row = r0 + threadIdx.x;
    if (row < n && col < cdim) dst[(size_t)col * ldd + row] = tile[threadIdx.x][i];
  }
}

__global__ void tout_kernel(const double* __restrict__ src, int lds, int n, int cdim,
                            double* __restrict__ dst) {
  __shared__ double tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int col = c0 + i, row = r0 + threadIdx.x;
    tile[threadIdx.x][i] = (row < n && col < cdim) ? src[(size_t)col * lds + row] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int row = r0 + i, col = c0 + threadIdx.x;
    if (row < n && col < cdim) dst[(size_t)row * cdim + col] = tile[i][threadIdx.x];
  }
}

__global__ void zero_kernel(double* p, size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x)
    p[i] = 0.0;
}

int grid_for(int n, int block) {
  int b = (n + block - 1) / block;
  if (b > 148 * 16) b = 148 * 16;
  return b < 1 ? 1 : b;
}

}  // namespace


template <int NB>
static void rotate_launch(const Geom& g, const double* X, int ldx, int a, const double* P,
                          int ldp, int b, double* out, int ldo, cudaStream_t st) {
  const size_t smem = (size_t)a * NB * sizeof(double);
  CK(cudaFuncSetAttribute(rotate_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)smem));
  rotate_kernel<NB><<<grid_for(g.n, 128), 128, smem, st>>>(g, X, ldx, a, P, ldp, b, out, ldo);
  launched();
}

void rotate_ld(const Geom& g, const double* X, int ldx, int a, const double* P, int ldp, int b,
               double* out, int ldo, cudaStream_t st) {
  if (b <= 0) return;
  if (b <= 8) rotate_launch<8>(g, X, ldx, a, P, ldp, b, out, ldo, st);
  else if (b <= 16) rotate_launch<16>(g, X, ldx, a, P, ldp, b, out, ldo, st);
  else if (b <= 24) rotate_launch<24>(g, X, ldx, a, P, ldp, b, out, ldo, st);
  else if (b <= 32) rotate_launch<32>(g, X, ldx, a, P, ldp, b, out, ldo, st);
  else if (b <= 48) rotate_launch<48>(g, X, ldx, a, P, ldp, b, out, ldo, st);
  else if (b <= 64) rotate_launch<64>(g, X, ldx, a, P, ldp, b, out, ldo, st);
  else fail(PND_ECONFIG, "rotate supports at most 64 output columns");
}

void rotate(const Geom& g, const double* X, int ldx, int a, const double* P, int b, double* out,
            int ldo, cudaStream_t st) {
  rotate_ld(g, X, ldx, a, P, b, b, out, ldo, st);
}

template <int NB>
static void scat_k1_launch(const Geom& g, const double* U0, int ldu, int ra, const double* S0,
                           int r, double dt, const double* inv_s, const int* cls,
                           const double* atomic, const double* psi, int ldpsi, int n_beams,
                           const double* rows, double* A, int lda, cudaStream_t st) {
  const size_t smem = ((size_t)ra * NB + (size_t)n_beams * 12 * NB) * sizeof(double);
  CK(cudaFuncSetAttribute(scat_k1_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)smem));
  scat_k1_kernel<NB><<<grid_for(g.n, 128), 128, smem, st>>>(g, U0, ldu, ra, S0, r, dt, inv_s,
                                                            cls, atomic, psi, ldpsi, n_beams,
                                                            rows, A, lda);
  launched();
}

void scat_k1(const Geom& g, const double* U0, int ldu, int ra, const double* S0, int r, double dt,
             const double* inv_s, const int* cls, const double* cls_atomic, const double* psi,
             int ldpsi, int n_beams, const double* rows, double* A, int lda, cudaStream_t st) {
#define PND_K1(NBV) scat_k1_launch<NBV>(g, U0, ldu, ra, S0, r, dt, inv_s, cls, cls_atomic, psi, \
                                        ldpsi, n_beams, rows, A, lda, st)
  if (r <= 8) PND_K1(8);
  else if (r <= 16) PND_K1(16);
  else if (r <= 24) PND_K1(24);
  else if (r <= 32) PND_K1(32);
  else if (r <= 48) PND_K1(48);
  else if (r <= 64) PND_K1(64);
  else fail(PND_ECONFIG, "scattering K-step supports rank <= 64");
#undef PND_K1
}

void apply_streaming_full(const Geom& g, const double* U, int ldu, int m, const double* inv_s,
                          const double* Mneg, double*, double* out, int ldo, cudaStream_t st) {
  KStageArgs a{};
  a.geo = g;
  a.X = U;
  a.ldx = ldu;
  a.xc = m;
  a.ra = 0;
  a.U0 = nullptr;
  a.S0 = nullptr;
  a.M = Mneg;
  a.inv_s = inv_s;
  a.r = m;
  a.out = out;
  a.ldo = ldo;
  a.copy_u = nullptr;
  kstage(a, st);
}

void dose_accumulate(const Geom& g, const double* U, int ldu, const double* coef, int r,
                     double half_dt, const double* s_field, const double* psi, int ldpsi,
                     int n_beams, double* deposited, double* prev, cudaStream_t st) {
  dose_kernel<<<grid_for(g.n, 256), 256, 0, st>>>(g, U, ldu, coef, r, half_dt, s_field, psi,
                                                   ldpsi, n_beams, deposited, prev);
  launched();
}

void class_gather_inv(const int* cls, const double* class_val, int n, double* out_inv,
                      double* out_val, cudaStream_t st) {
  class_gather_kernel<<<grid_for(n, 256), 256, 0, st>>>(cls, class_val, n, out_inv, out_val);
  launched();
}

void psi_lerp(const double* values, int ldv, int n, int j0, double w0, int j1, double w1,
              double* out, cudaStream_t st) {
  lerp_kernel<<<grid_for(n, 256), 256, 0, st>>>(values, ldv, n, j0, w0, j1, w1, out);
  launched();
}

void transpose_in(const double* src, int n, int c, double* dst, int ldd, cudaStream_t st) {
  if (n <= 0 || c <= 0) return;
  dim3 grid((c + 31) / 32, (n + 31) / 32), block(32, 8);
  tin_kernel<<<grid, block, 0, st>>>(src, n, c, dst, ldd);
  launched();
}

void transpose_out(const double* src, int lds, int n, int c, double* dst, cudaStream_t st) {
  if (n <= 0 || c <= 0) return;
  dim3 grid((c + 31) / 32, (n + 31) / 32), block(32, 8);
  tout_kernel<<<grid, block, 0, st>>>(src, lds, n, c, dst);
  launched();
}

void fill_zero(double* p, size_t count, cudaStream_t st) {
  if (!count) return;
  size_t blocks = (count + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  zero_kernel<<<(int)blocks, 256, 0, st>>>(p, count);
  launched();
}

}  // namespace pnd
