// Per-element angular moments of the screened elastic-scattering kernel on
// the device (the MomentTables of driver.py:269-307,
// physics/moliere.py:38-147).
//
// One CTA per (element, energy): the screening offset chi and the amplitude
// C from the proton kinematics (kinematics.py:8-32), the de-peaked
// Gauss-Legendre quadrature of moliere.py:81-108 -- mu0 in [0, 1] under
// s = ln(1 - mu0 + chi) (1 - mu0 as chi expm1(s - ln chi)), mu0 in [-1, 0]
// under t = sqrt(1 + mu0) -- the lab-frame factor tau_lab, and the Legendre
// moments g_0..g_L plus xi1 = 2 pi Int sigma (1 - mu0), each node's P_l by the
// three-term recurrence; evaluated with n and 2n nodes and the doubled-node
// convergence test of legendre_moments (rtol, moliere.py:111-147). The
// Gauss-Legendre nodes are the host's (numpy leggauss, as the reference).
#include <cmath>

#include "pnd.h"

namespace pnd {

namespace {

constexpr double PROTON_REST_MEV = 938.272;
constexpr double ELECTRON_REST_MEV = 0.51099895;
constexpr double FINE_STRUCTURE = 7.2973525693e-3;
constexpr double HBARC_MEV_CM = 1.9732698045930252e-11;
constexpr double TWO_PI = 6.283185307179586;
constexpr int MAXDEG = 96;

__device__ double tau_lab(double mu0, double r) {
  const double num = pow(1.0 + 2.0 * mu0 * r + r * r, 1.5);
  const double den = 1.0 + mu0 * r;
  return den > 0.0 ? num / den : 0.0;
}

// block-wide sum of v (all threads get it); red: >= 32 doubles
__device__ double bsum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s += red[i];
  return s;
}

// moments of one (element, energy) with nn Gauss-Legendre nodes per piece;
// out[0..L] = g, out[L+1] = xi1 (thread 0 holds the sums)
__device__ void moments_nn(double chi, double c, double r, double q, const double* x,
                           const double* w, int nn, int L, double* acc, double* red,
                           double* out) {
  for (int l = 0; l <= L + 1; ++l) acc[l] = 0.0;
  const double s_lo = log(chi), s_hi = log(1.0 + chi);
  for (int i = threadIdx.x; i < 2 * nn; i += blockDim.x) {
    double mu0, omm, jac;
    if (i < nn) {
      const double s = 0.5 * (s_hi - s_lo) * x[i] + 0.5 * (s_hi + s_lo);
      jac = 0.5 * (s_hi - s_lo) * exp(s) * w[i];
      omm = chi * expm1(s - s_lo);
      mu0 = 1.0 - omm;
    } else {
      const double t = 0.5 * (x[i - nn] + 1.0);
      jac = 0.5 * 2.0 * t * w[i - nn];
      mu0 = -1.0 + t * t;
      omm = 2.0 - t * t;
    }
    const double val = tau_lab(mu0, r) * c / pow(omm + chi, q) * jac;
    double p0 = 1.0, p1 = mu0;
    acc[0] += val;
    if (L >= 1) acc[1] += val * mu0;
    for (int l = 2; l <= L; ++l) {
      // numpy legvander's order: (v[l-1] x (2l - 1) - v[l-2] (l - 1)) / l
      const double p2 = (p1 * mu0 * (2.0 * l - 1.0) - p0 * (l - 1.0)) / l;
      acc[l] += val * p2;
      p0 = p1;
      p1 = p2;
    }
    acc[L + 1] += val * omm;
  }
  for (int l = 0; l <= L + 1; ++l) {
    const double s = bsum(acc[l], red);
    if (threadIdx.x == 0) out[l] = TWO_PI * s;
  }
}

__global__ void __launch_bounds__(128)
    moment_table_kernel(const double* __restrict__ energies, int n_e, const int* __restrict__ z,
                        const int* __restrict__ a, const double* x1, const double* w1,
                        const double* x2, const double* w2, int nn, int L, double q, double rtol,
                        double* __restrict__ g, double* __restrict__ xi1, int* bad) {
  __shared__ double red[32];
  __shared__ double o1[MAXDEG + 2], o2[MAXDEG + 2];
  double acc[MAXDEG + 2];
  const int j = blockIdx.x, el = blockIdx.y;
  const double e = energies[j];
  // kinematics.py:8-32 and moliere.py:38-54
  const double p = sqrt(e * (e + 2.0 * PROTON_REST_MEV));
  const double beta = p / (e + PROTON_REST_MEV);
  const double chi0 = 1.13 * FINE_STRUCTURE * pow((double)z[el], 1.0 / 3.0) * ELECTRON_REST_MEV / p;
  const double aa = z[el] * FINE_STRUCTURE / beta;
  const double chi = chi0 * chi0 * (1.13 + 3.76 * aa * aa);
  const double k = p / HBARC_MEV_CM;
  const double c = 4.0 * FINE_STRUCTURE * FINE_STRUCTURE / (k * k);
  const double r = 1.0 / a[el];
  moments_nn(chi, c, r, q, x1, w1, nn, L, acc, red, o1);
  moments_nn(chi, c, r, q, x2, w2, 2 * nn, L, acc, red, o2);
  if (threadIdx.x == 0) {
    const double scale = fmax(fabs(o2[0]), fabs(o2[L + 1]));
    double err = fabs(o1[L + 1] - o2[L + 1]);
    for (int l = 0; l <= L; ++l) err = fmax(err, fabs(o1[l] - o2[l]));
    if (err / scale > rtol) atomicMin(bad, el * n_e + j);
    for (int l = 0; l <= L; ++l) g[((size_t)el * n_e + j) * (L + 1) + l] = o2[l];
    xi1[(size_t)el * n_e + j] = o2[L + 1];
  }
}

}  // namespace

int moment_tables(const double* energies, int n_e, const int* z, const int* a, int n_el,
                  const double* x1, const double* w1, const double* x2, const double* w2, int nn,
                  int max_degree, double exponent, double rtol, double* g, double* xi1,
                  cudaStream_t st) {
  if (max_degree < 0 || max_degree > MAXDEG) fail(PND_ECONFIG, "moment tables: degree 0..96");
  DBuf de, dx1, dw1, dx2, dw2, dg, dxi;
  IBuf dz, da, db;
  auto up = [&](DBuf& b, const double* src, size_t cnt) {
    double* p = b.get(cnt);
    CK(cudaMemcpyAsync(p, src, cnt * sizeof(double), cudaMemcpyHostToDevice, st));
    return p;
  };
  auto upi = [&](IBuf& b, const int* src, size_t cnt) {
    int* p = b.get(cnt);
    CK(cudaMemcpyAsync(p, src, cnt * sizeof(int), cudaMemcpyHostToDevice, st));
    return p;
  };
  const double* pe = up(de, energies, n_e);
  const double* px1 = up(dx1, x1, nn);
  const double* pw1 = up(dw1, w1, nn);
  const double* px2 = up(dx2, x2, 2 * nn);
  const double* pw2 = up(dw2, w2, 2 * nn);
  const int* pz = upi(dz, z, n_el);
  const int* pa = upi(da, a, n_el);
  int* bad = db.get(1);
  const int init = 1 << 30;
  CK(cudaMemcpyAsync(bad, &init, sizeof(int), cudaMemcpyHostToDevice, st));
  const size_t ng = (size_t)n_el * n_e * (max_degree + 1);
  double* pg = dg.get(ng);
  double* pxi = dxi.get((size_t)n_el * n_e);
  moment_table_kernel<<<dim3(n_e, n_el), 128, 0, st>>>(pe, n_e, pz, pa, px1, pw1, px2, pw2, nn,
                                                       max_degree, exponent, rtol, pg, pxi, bad);
  launched();
  int hb = 0;
  CK(cudaMemcpyAsync(g, pg, ng * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(xi1, pxi, (size_t)n_el * n_e * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (DBuf* b : {&de, &dx1, &dw1, &dx2, &dw2, &dg, &dxi}) b->free_();
  for (IBuf* b : {&dz, &da, &db}) b->free_();
  return hb == init ? -1 : hb;  // -1: converged; else the first (element * n_e + energy)
}

}  // namespace pnd
