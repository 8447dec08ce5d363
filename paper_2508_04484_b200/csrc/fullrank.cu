// Full-rank solver on the device (fullrank.py:16-40).
//
// The oracle of the low-rank path evolves the dense n x m moment matrix with
// the same Lie splitting: RK4 on u' = F_S(u) (apply_streaming,
// spatial.py:148-167) and implicit Euler on the per-(cell, moment)
// self-scattering with an explicit Euler source (fullrank.py:30-45). On the
// device the dense matrix is kept as ceil(m / 32) column blocks, each a
// cell-major n x 32 matrix with the zero halo rows of every n-side factor,
// so the streaming operator is the K-stage kernel applied block by block:
//   one Horner stage  out[:, ob] = u[:, ob] + c F_S(W)[:, ob]
//                  = u[:, ob] - c sum_xb sum_s (D_s S^-1 W[:, xb]) A_s[xb, ob],
// a chain over the input blocks xb in which each K-stage takes the previous
// partial sum as its base rows (S0 = I). The Horner form of RK4 equals the
// classical one for this linear autonomous right-hand side (to rounding).
// The scattering update is one elementwise kernel; the dose tally reuses
// the low-rank path's trapezoid with U = block 0 and coefficient e_0.
// Memory: four n x m matrices (u, two Horner buffers, the partial-sum pair
// is two blocks), e.g. 64^3 x 400 = 0.84 GB each.
#include <cmath>
#include <cstdio>

#include "handle.h"

namespace pnd {

namespace {

constexpr int FB = 32;  // column block

int nblk(const Handle& h) { return (h.m + FB - 1) / FB; }
int bw(const Handle& h, int b) { return b + 1 < nblk(h) ? FB : h.m - FB * (nblk(h) - 1); }

// M[s][p][q] = c A_s[x0 + p][o0 + q] (ns x bx x bo), A_s in stencil order (m x m)
__global__ void mblock_kernel(const double* __restrict__ amat, int m, int ns, int x0, int bx,
                              int o0, int bo, double c, double* __restrict__ M) {
  const int total = ns * bx * bo;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int s = i / (bx * bo), rem = i - s * bx * bo, p = rem / bo, q = rem - p * bo;
    M[i] = c * amat[((size_t)s * m + x0 + p) * m + o0 + q];
  }
}

__global__ void unit_kernel(double* e, int b) {
  for (int i = threadIdx.x; i < b; i += blockDim.x) e[i] = i == 0 ? 1.0 : 0.0;
}

__global__ void eye_rows_kernel(double* I, int b) {
  for (int i = threadIdx.x; i < b * b; i += blockDim.x) I[i] = (i / b == i % b) ? 1.0 : 0.0;
}

// per-block max |u| (the amplification check of fullrank_streaming_step)
__global__ void absmax_kernel(NMat u, int n, double* __restrict__ out) {
  __shared__ double red[256];
  double mx = 0.0;
  const long total = (long)n * u.rs;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const double v = fabs(u.p[i]);
    mx = v > mx ? v : mx;
  }
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = red[0];
}

// u <- u / (1 + dt rates) + dt source  (fullrank_scattering_step)
//   rates[c][q]  = sum_i N_{cls(c),i} / S(c) (sigma_t,i - g_{i,q})
//   source[c][q] = sum_b sum_i N_{cls(c),i} psi_b(c) / S(c) g_{i,q} T_M^b[q]
__global__ void fr_scatter_kernel(NMat u, int n, int q0, double dt, const double* __restrict__ inv_s,
                                  const int* __restrict__ cls, const double* __restrict__ atomic,
                                  const double* __restrict__ gdiag, const double* __restrict__ sigt,
                                  int m, const double* __restrict__ psi, int ld, int n_beams,
                                  const double* __restrict__ tm) {
  const long total = (long)n * u.cols;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
       e += (long)gridDim.x * blockDim.x) {
    const int c = (int)(e / u.cols), j = (int)(e - (long)c * u.cols), q = q0 + j;
    const double* N = atomic + (size_t)cls[c] * 12;
    const double is = inv_s[c];
    double rate = 0.0, gsum = 0.0;
    for (int i = 0; i < 12; ++i) {
      const double w = N[i] * is;
      rate = fma(w, sigt[i] - gdiag[(size_t)i * m + q], rate);
      gsum = fma(w, gdiag[(size_t)i * m + q], gsum);
    }
    double src = 0.0;
    for (int b = 0; b < n_beams; ++b) src = fma(psi[(size_t)b * ld + c] * gsum, tm[(size_t)b * m + q], src);
    double* x = u.p + (size_t)c * u.rs + j;
    *x = *x / (1.0 + dt * rate) + dt * src;
  }
}

NMat blk(Handle& h, std::vector<NBuf>& v, int b) {
  if ((int)v.size() < nblk(h)) v.resize(nblk(h));
  return v[b].view(h.g, bw(h, b), h.st);
}

double absmax_all(Handle& h, std::vector<NBuf>& v) {
  double* part = h.fr_scr.get(148 * 4 * (size_t)nblk(h) + 8);
  for (int b = 0; b < nblk(h); ++b) {
    absmax_kernel<<<148 * 4, 256, 0, h.st>>>(blk(h, v, b), h.g.n, part + (size_t)b * 148 * 4);
    launched();
  }
  std::vector<double> hp((size_t)148 * 4 * nblk(h));
  CK(cudaMemcpyAsync(hp.data(), part, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, h.st));
  CK(cudaStreamSynchronize(h.st));
  double mx = 0.0;
  for (double x : hp) mx = x > mx ? x : mx;
  return mx;
}

}  // namespace

void fullrank_reset(Handle& h) {
  for (int b = 0; b < nblk(h); ++b) {
    const NMat u = blk(h, h.fr_u, b);
    fill_zero(u.p, (size_t)h.g.n * u.rs, h.st);
  }
  h.have_fr = true;
}

NMat fullrank_block(Handle& h, int b) { return blk(h, h.fr_u, b); }
int fullrank_blocks(const Handle& h) { return nblk(h); }

void fullrank_streaming_step(Handle& h, double dt) {
  if (!h.stencil_error.empty()) fail(PND_ECONFIG, h.stencil_error);
  if (!h.have_angular || !h.have_inv_s) fail(PND_ECONFIG, "set angular and inv_s first");
  if (!h.have_fr) fail(PND_ECONFIG, "no full-rank state (pnd_fullrank_set / reset)");
  const Geom& g = h.g;
  const int nb = nblk(h), ns = g.ns, m = h.m;
  const double scale0 = absmax_all(h, h.fr_u);
  const double coef[4] = {0.25, 1.0 / 3.0, 0.5, 1.0};
  double* M = h.fr_scr2.get((size_t)ns * FB * FB + 1);
  double* I = h.fr_eye.get((size_t)FB * FB);
  // Horner buffers: u -> A -> B -> A -> B (the base is u in every stage)
  std::vector<NBuf>* const src[4] = {&h.fr_u, &h.fr_w1, &h.fr_w2, &h.fr_w1};
  std::vector<NBuf>* const dst[4] = {&h.fr_w1, &h.fr_w2, &h.fr_w1, &h.fr_w2};
  for (int stage = 0; stage < 4; ++stage) {
    std::vector<NBuf>* const W = src[stage];
    std::vector<NBuf>* const Wn = dst[stage];
    for (int b = 0; b < nb; ++b) comm_halo_rows(g, blk(h, *W, b).p, blk(h, *W, b).rs, h.st);
    for (int ob = 0; ob < nb; ++ob) {
      const int bo = bw(h, ob);
      eye_rows_kernel<<<1, 256, 0, h.st>>>(I, bo);
      launched();
      NMat base = blk(h, h.fr_u, ob);
      for (int xb = 0; xb < nb; ++xb) {
        const int bx = bw(h, xb);
        mblock_kernel<<<64, 256, 0, h.st>>>(h.amat.p, m, ns, FB * xb, bx, FB * ob, bo,
                                            -coef[stage] * dt, M);
        launched();
        NMat out = xb + 1 < nb ? h.fr_t[xb & 1].view(g, bo, h.st) : blk(h, *Wn, ob);
        KStageArgs a{};
        a.bcat = &h.bcat;
        a.geo = g;
        a.X = blk(h, *W, xb);
        a.U0 = base;
        a.S0 = I;
        a.M = M;
        a.inv_s = h.isp.p + 2 * (size_t)g.halo;
        a.out = out;
        kstage(a, h.st);
        base = out;
      }
    }
  }
  // u1 = the last stage's output
  std::swap(h.fr_u, h.fr_w2);
  const double scale1 = absmax_all(h, h.fr_u);
  if (scale0 > 0.0 && scale1 > 1e6 * scale0) {
    char buf[160];
    snprintf(buf, sizeof buf,
             "streaming step amplified the solution by %.2e; reduce the step size",
             scale1 / scale0);
    fail(PND_ENUMERICAL, buf);
  }
}

void fullrank_scattering_step(Handle& h, double dt) {
  if (!h.have_inv_s || !h.have_mat || !h.have_scat)
    fail(PND_ECONFIG, "full-rank scattering needs inv_s, materials and scattering tables");
  if (!h.have_fr) fail(PND_ECONFIG, "no full-rank state (pnd_fullrank_set / reset)");
  for (int b = 0; b < nblk(h); ++b) {
    fr_scatter_kernel<<<148 * 8, 256, 0, h.st>>>(
        blk(h, h.fr_u, b), h.g.n, FB * b, dt, h.inv_s.p, h.cls.p, h.cls_atomic.p, h.gdiag.p,
        h.sigt.p, h.m, h.psi.p, h.g.ld, h.n_beams, h.tm.p);
    launched();
  }
}

void fullrank_dose_step(Handle& h, double dt, bool tally_steps) {
  // integrand = sqrt(4 pi) u[:, 0] (+ S psi_u(E_lo)) (driver.py:610-621)
  double* e0 = h.fr_scr3.get(FB);
  unit_kernel<<<1, 32, 0, h.st>>>(e0, FB);
  launched();
  double* dep = h.dep.get((size_t)h.g.ld);
  double* prev = h.prev.get((size_t)h.g.ld);
  dose_accumulate(h.g, blk(h, h.fr_u, 0), e0, 0.5 * dt, h.s_field.p,
                  tally_steps && h.n_beams > 0 ? h.psi_lo.p : nullptr, h.n_beams, dep, prev,
                  h.st);
}

}  // namespace pnd
