// Per-step coefficient assembly on the device.
//
// The step contexts (driver.py:523-538) need, at every energy step, the
// stopping power of every material class, the 12 per-element scattering
// diagonals and total cross sections, and the uncollided-flux slice. The
// tables they come from are uploaded once (pnd_set_coefficient_tables); one
// single-CTA kernel then evaluates them at e_mid (and e_lo for the
// per-step uncollided tally) straight into the device buffers the step
// reads, so a step needs no host->device copy:
//   - class S(E): log-log linear interpolation of each element's mass
//     stopping-power table (stopping.py:48-56, np.interp semantics: clamped
//     at the table ends) and Bragg additivity rho_k sum_i w_ki s_i
//     (stopping.py:107-120; host restatement problem.class_stopping);
//   - scattering tables (driver.py:337-362, angular.py:217-248): moment
//     tables linearly interpolated in energy (MomentTables._interp,
//     driver.py:290-296); Boltzmann: g_l per degree minus g_{N+1} (transport
//     correction), sigma_t = g_0 - g_{N+1}; Fokker-Planck: -xi1/2 l(l+1) minus
//     scale * lambda_{N+1}, sigma_t = -scale * lambda_{N+1};
//   - uncollided-flux lerp weights between group centres
//     (raytracer.py:440-449; host restatement UncollidedSlices.lerp_weights),
//     then the same lerp kernel as the host-driven path, reading its
//     (j0, w0, j1, w1) from device memory.
#include "handle.h"

namespace pnd {

namespace {

constexpr int NEL = 12;

struct CoeffArgs {
  const double* log_e;   // 12 x K
  const double* log_s;   // 12 x K
  int K;
  const double* dens;    // n_cls
  const double* wts;     // n_cls x 12 mass fractions
  int n_cls;
  const double* mom_e;   // P
  int P;
  const double* mom_g;   // 12 x P x nd (Boltzmann)
  int nd;
  const double* xi1;     // 12 x P (Fokker-Planck)
  int model;             // 0 Boltzmann, 1 Fokker-Planck
  int pn_order;
  int boltz_corr;
  double fp_scale;
  int m;
  const double* flux_range;  // n_beams x 2 (e_min, e_max)
  int n_groups, n_beams;
};

// np.interp(x, xp, fp) for increasing xp: clamped ends, else the segment
// [xp[j], xp[j+1]) that holds x, slope * (x - xp[j]) + fp[j]
__device__ double interp(double x, const double* xp, const double* fp, int K) {
  if (!(x > xp[0])) return fp[0];
  if (!(x < xp[K - 1])) return fp[K - 1];
  int lo = 0, hi = K - 1;  // xp[lo] <= x < xp[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (xp[mid] <= x) lo = mid;
    else hi = mid;
  }
  const double slope = (fp[lo + 1] - fp[lo]) / (xp[lo + 1] - xp[lo]);
  return slope * (x - xp[lo]) + fp[lo];
}

// MomentTables._interp: idx = clip(searchsorted(en, e) - 1, 0, P - 2)
__device__ void moment_index(const double* en, int P, double e, int& idx, double& w) {
  int s = 0;  // searchsorted (left): first index with en[s] >= e
  while (s < P && en[s] < e) ++s;
  idx = s - 1;
  if (idx < 0) idx = 0;
  if (idx > P - 2) idx = P - 2;
  w = (e - en[idx]) / (en[idx + 1] - en[idx]);
}

// UncollidedSlices.lerp_weights on the group centres of [e_min, e_max]
__device__ void lerp_weights(double e, double e_min, double e_max, int G, int& j0, double& w0,
                             int& j1, double& w1) {
  const double step = (e_max - e_min) / G;  // np.linspace(e_min, e_max, G + 1)
  auto edge = [&](int i) { return i == G ? e_max : e_min + i * step; };
  auto centre = [&](int j) { return 0.5 * (edge(j) + edge(j + 1)); };
  const double c0 = centre(0), cl = centre(G - 1);
  if (e <= c0 || e >= cl) {
    const int j = e <= c0 ? 0 : G - 1;
    const bool inside = e_min <= e && e <= e_max;
    j0 = j1 = j;
    w0 = inside ? 1.0 : 0.0;
    w1 = 0.0;
    return;
  }
  int s = 0;  // searchsorted(c, e) (left)
  while (s < G && centre(s) < e) ++s;
  const int j = s - 1;
  const double w = (e - centre(j)) / (centre(j + 1) - centre(j));
  j0 = j;
  w0 = 1.0 - w;
  j1 = j + 1;
  w1 = w;
}

__global__ void coeff_kernel(CoeffArgs a, double e_mid, double e_lo, int want_lo,
                             double* __restrict__ class_s, double* __restrict__ gdiag,
                             double* __restrict__ sigt, int* __restrict__ sel_j,
                             double* __restrict__ sel_w) {
  __shared__ double s_el[NEL];
  __shared__ double mom[NEL][2];  // Boltzmann: g_{N+1} per element; FP: xi1
  const int tid = threadIdx.x;
  // element stopping powers at e_mid
  if (tid < NEL) {
    const double x = log(e_mid);
    s_el[tid] = exp(interp(x, a.log_e + (size_t)tid * a.K, a.log_s + (size_t)tid * a.K, a.K));
  }
  int idx;
  double w;
  moment_index(a.mom_e, a.P, e_mid, idx, w);
  if (tid < NEL) {
    if (a.model == 0) {
      const double* t = a.mom_g + (size_t)tid * a.P * a.nd;
      const int d = a.pn_order + 1;
      mom[tid][0] = (1.0 - w) * t[(size_t)idx * a.nd + d] + w * t[(size_t)(idx + 1) * a.nd + d];
      mom[tid][1] = (1.0 - w) * t[(size_t)idx * a.nd] + w * t[(size_t)(idx + 1) * a.nd];
    } else {
      const double* t = a.xi1 + (size_t)tid * a.P;
      mom[tid][0] = (1.0 - w) * t[idx] + w * t[idx + 1];
      mom[tid][1] = 0.0;
    }
  }
  __syncthreads();
  // class S(E) = rho_k * (w_k . s)
  for (int k = tid; k < a.n_cls; k += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < NEL; ++i) s += a.wts[(size_t)k * NEL + i] * s_el[i];
    class_s[k] = a.dens[k] * s;
  }
  // scattering diagonals (12 x m) and sigma_t (12)
  const int N = a.pn_order;
  for (int e = tid; e < NEL * a.m; e += blockDim.x) {
    const int i = e / a.m, p = e - i * a.m;
    int l = (int)sqrt((double)p);
    while (l * l > p) --l;
    while ((l + 1) * (l + 1) <= p) ++l;
    double g;
    if (a.model == 0) {
      const double* t = a.mom_g + (size_t)i * a.P * a.nd;
      g = (1.0 - w) * t[(size_t)idx * a.nd + l] + w * t[(size_t)(idx + 1) * a.nd + l];
      if (a.boltz_corr) g = g - mom[i][0];
    } else {
      const double x = mom[i][0];
      g = -(x / 2.0) * (l * (l + 1.0));
      if (a.fp_scale > 0.0) g = g - a.fp_scale * (-(x / 2.0) * (N + 1.0) * (N + 2.0));
    }
    gdiag[e] = g;
  }
  if (tid < NEL) {
    double s;
    if (a.model == 0) {
      s = mom[tid][1];
      if (a.boltz_corr) s = s - mom[tid][0];
    } else {
      s = 0.0;
      if (a.fp_scale > 0.0) s = s - a.fp_scale * (-(mom[tid][0] / 2.0) * (N + 1.0) * (N + 2.0));
    }
    sigt[tid] = s;
  }
  // uncollided-flux selections: [which][beam] -> (j0, j1), (w0, w1)
  if (tid < a.n_beams * 2) {
    const int which = tid / a.n_beams, b = tid - which * a.n_beams;
    if (which == 0 || want_lo) {
      int j0, j1;
      double w0, w1;
      lerp_weights(which == 0 ? e_mid : e_lo, a.flux_range[2 * b], a.flux_range[2 * b + 1],
                   a.n_groups, j0, w0, j1, w1);
      sel_j[2 * tid] = j0;
      sel_j[2 * tid + 1] = j1;
      sel_w[2 * tid] = w0;
      sel_w[2 * tid + 1] = w1;
    }
  }
}

// psi = w0 v[:, j0] + w1 v[:, j1] with the selection read on the device (the
// same arithmetic as lerp_kernel in nside.cu)
__global__ void lerp_dev_kernel(const double* __restrict__ v, int ldv, int n,
                                const int* __restrict__ sel_j, const double* __restrict__ sel_w,
                                double* __restrict__ out) {
  const int j0 = sel_j[0], j1 = sel_j[1];
  const double w0 = sel_w[0], w1 = sel_w[1];
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

}  // namespace

void coefficients_at(Handle& h, double e_mid, double e_lo, bool want_lo) {
  if (!h.have_ctab) fail(PND_ECONFIG, "coefficient tables not set (pnd_set_coefficient_tables)");
  CoeffArgs a{};
  a.log_e = h.ctab.p;
  a.log_s = h.ctab.p + (size_t)NEL * h.ct_K;
  a.K = h.ct_K;
  a.dens = a.log_s + (size_t)NEL * h.ct_K;
  a.wts = a.dens + h.n_cls;
  a.n_cls = h.n_cls;
  a.mom_e = a.wts + (size_t)h.n_cls * NEL;
  a.P = h.ct_P;
  a.mom_g = a.mom_e + h.ct_P;
  a.nd = h.ct_nd;
  a.xi1 = a.mom_g + (size_t)NEL * h.ct_P * h.ct_nd;
  a.flux_range = a.xi1 + (size_t)NEL * h.ct_P;
  a.model = h.ct_model;
  a.pn_order = h.ct_pn;
  a.boltz_corr = h.ct_bcorr;
  a.fp_scale = h.ct_fpscale;
  a.m = h.m;
  a.n_groups = h.n_groups;
  a.n_beams = h.have_flux() ? h.n_beams : 0;
  double* cs = h.cls_val.get(h.n_cls);
  double* gd = h.gdiag.get((size_t)NEL * h.m);
  double* sg = h.sigt.get(NEL);
  int* sj = reinterpret_cast<int*>(h.csel.get(32));
  double* sw = h.csel.p + 16;
  coeff_kernel<<<1, 256, 0, h.st>>>(a, e_mid, e_lo, want_lo ? 1 : 0, cs, gd, sg, sj, sw);
  launched();
  // stopping-power fields (S, 1/S per cell, the staged [1/S, 0] rows)
  double* d = h.inv_s.get(h.g.ld + 64);
  double* sf = h.s_field.get(h.g.ld);
  fill_zero(d + h.g.n, h.g.ld + 64 - h.g.n, h.st);
  class_gather_inv(h.cls.p, cs, h.g.n, d, sf, h.st);
  set_isp(h);
  h.have_inv_s = true;
  h.g.uniform_s = h.n_cls == 1;
  h.have_scat = true;
  // uncollided slices
  for (int which = 0; which < (want_lo ? 2 : 1); ++which) {
    double* dst = which == 0 ? h.psi.p : h.psi_lo.p;
    if (!dst) continue;
    for (int b = 0; b < a.n_beams; ++b) {
      const int s = which * a.n_beams + b;
      if (h.flux_sep) {
        const int nxy = h.g.nx * h.g.ny;
        psi_lerp_separable(h.sep_lat.p + (size_t)b * nxy,
                           h.sep_depth.p + (size_t)b * h.g.nz * h.n_groups, nxy, h.n_groups,
                           h.g.n, sj + 2 * s, sw + 2 * s, 0, 0.0, 0, 0.0,
                           dst + (size_t)b * h.g.ld, h.st);
        continue;
      }
      if (h.flux_sparse) {
        psi_lerp_sparse(h.sp_cells[b].p, h.sp_vals[b].p, h.sp_nnz[b], h.n_groups, h.g.n,
                        sj + 2 * s, sw + 2 * s, 0, 0.0, 0, 0.0, dst + (size_t)b * h.g.ld, h.st);
        continue;
      }
      lerp_dev_kernel<<<sm_count() * 8, 256, 0, h.st>>>(
          h.flux.p + (size_t)b * h.n_groups * h.g.ld, h.g.ld, h.g.n, sj + 2 * s, sw + 2 * s,
          dst + (size_t)b * h.g.ld);
      launched();
    }
  }
}

}  // namespace pnd
