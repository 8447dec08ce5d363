// Uncollided flux: Crank-Nicolson energy march along ray paths and the
// track-length deposit (raytracer.py:285-350 march_ray, 486-519 trace_beam).
//
// The energy operator G of one material (assemble_energy_operators,
// raytracer.py:169-274: DG with nl = degree+1 Legendre modes per group,
// Lax-Friedrichs slowing-down faces, SIPG straggling, absorption) couples a
// group only to its neighbours, so A = M + dz/2 G and B = M - dz/2 G are
// block tridiagonal with nl x nl blocks. The reference factors A densely
// (scipy lu_factor); here each (material, dz) "stepper" is factored once by
// block elimination (one thread per stepper) and every CN substep
//   psi <- A^-1 (B psi)
// is a block-tridiagonal multiply, a forward sweep and a back sweep.
//
// march_kernel: one thread per distinct ray signature (rays whose
// (material, length) sequence coincides share one march, as in the reference),
// serial over its segments and substeps; it records the group averages (the
// P0 coefficients) after the first half of every segment and the energy
// carried below e_min (trapezoidal trace rule), exactly the reference's
// bookkeeping.
// deposit_kernel: one CTA walks the rays in enumeration order and adds
// weight * length / V * averages into the (group x cell) flux table and the
// residual energy per cell; a ray visits each cell at most once, so the
// per-ray adds are conflict-free and the summation order is the reference's.
#include "pnd.h"

namespace pnd {

namespace {

template <int NL>
__device__ __forceinline__ void inv_small(const double* a, double* inv) {
  // Gauss-Jordan with partial pivoting on an NL x NL block (row-major)
  double m[NL][2 * NL];
#pragma unroll
  for (int i = 0; i < NL; ++i)
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      m[i][j] = a[i * NL + j];
      m[i][NL + j] = i == j ? 1.0 : 0.0;
    }
#pragma unroll
  for (int c = 0; c < NL; ++c) {
    int p = c;
#pragma unroll
    for (int r = c + 1; r < NL; ++r)
      if (fabs(m[r][c]) > fabs(m[p][c])) p = r;
    if (p != c) {
#pragma unroll
      for (int j = 0; j < 2 * NL; ++j) {
        const double t = m[c][j];
        m[c][j] = m[p][j];
        m[p][j] = t;
      }
    }
    const double d = 1.0 / m[c][c];
#pragma unroll
    for (int j = 0; j < 2 * NL; ++j) m[c][j] *= d;
#pragma unroll
    for (int r = 0; r < NL; ++r) {
      if (r == c) continue;
      const double f = m[r][c];
#pragma unroll
      for (int j = 0; j < 2 * NL; ++j) m[r][j] -= f * m[c][j];
    }
  }
#pragma unroll
  for (int i = 0; i < NL; ++i)
#pragma unroll
    for (int j = 0; j < NL; ++j) inv[i * NL + j] = m[i][NL + j];
}

// blocks of G per key: D[k][g], L[k][g] (row block g, column block g-1),
// U[k][g] (row block g, column block g+1), each NL x NL row-major
struct MarchOps {
  const double* D;
  const double* L;
  const double* U;
  const double* mass;  // NG * NL
  int ng;
};

// stepper s: key[s], dz[s] -> Dinv[s][g] (factored diagonal blocks of A) and
// E[s][g] = A_L[g] Dinv[g-1] (forward-elimination multipliers)
template <int NL>
__global__ void stepper_kernel(MarchOps op, int n_steppers, const int* __restrict__ key,
                               const double* __restrict__ dz, double* __restrict__ Dinv,
                               double* __restrict__ E, int* __restrict__ bad) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_steppers) return;
  constexpr int B2 = NL * NL;
  const int k = key[s], G = op.ng;
  const double h = 0.5 * dz[s];
  const double* Dk = op.D + (size_t)k * G * B2;
  const double* Lk = op.L + (size_t)k * G * B2;
  const double* Uk = op.U + (size_t)k * G * B2;
  double* di = Dinv + (size_t)s * G * B2;
  double* e = E + (size_t)s * G * B2;
  double prev[B2];  // Dinv[g-1]
  for (int g = 0; g < G; ++g) {
    double a[B2];
#pragma unroll
    for (int i = 0; i < NL; ++i)
#pragma unroll
      for (int j = 0; j < NL; ++j)
        a[i * NL + j] = (i == j ? op.mass[g * NL + i] : 0.0) + h * Dk[g * B2 + i * NL + j];
    if (g > 0) {
      // E_g = (h L_g) Dinv_{g-1};  a -= E_g (h U_{g-1})
      double eg[B2];
#pragma unroll
      for (int i = 0; i < NL; ++i)
#pragma unroll
        for (int j = 0; j < NL; ++j) {
          double v = 0.0;
#pragma unroll
          for (int t = 0; t < NL; ++t) v += h * Lk[g * B2 + i * NL + t] * prev[t * NL + j];
          eg[i * NL + j] = v;
        }
#pragma unroll
      for (int i = 0; i < NL; ++i)
#pragma unroll
        for (int j = 0; j < NL; ++j) {
          double v = 0.0;
#pragma unroll
          for (int t = 0; t < NL; ++t) v += eg[i * NL + t] * h * Uk[(g - 1) * B2 + t * NL + j];
          a[i * NL + j] -= v;
        }
#pragma unroll
      for (int i = 0; i < B2; ++i) e[g * B2 + i] = eg[i];
    } else {
#pragma unroll
      for (int i = 0; i < B2; ++i) e[i] = 0.0;
    }
    inv_small<NL>(a, prev);
#pragma unroll
    for (int i = 0; i < B2; ++i) {
      if (!isfinite(prev[i])) atomicExch(bad, 1);
      di[g * B2 + i] = prev[i];
    }
  }
}

struct MarchJob {
  int n_marches;
  const int* seg_off;     // n_marches + 1
  const int* seg_key;     // per segment
  const double* half_dz;  // 2 per segment: dz of each half
  const int* half_n;      // 2 per segment: substeps of each half
  const int* half_st;     // 2 per segment: stepper index
  const double* st_dz;    // per stepper: the dz its factors were built with
  const double* s_min;    // per key: s*(e_min)
  double e_min;
  const double* psi0;
  const double* p_lo;     // NL: Legendre values at xi = -1
  double* psi;            // n_marches x ndof (work / exit spectra)
  double* tmp;            // n_marches x ndof
  double* averages;       // n_segments x ng
  double* residual;       // n_segments
  int* bad;
};

template <int NL>
__global__ void march_kernel(MarchOps op, MarchJob j, const double* __restrict__ Dinv,
                             const double* __restrict__ E) {
  const int mi = blockIdx.x * blockDim.x + threadIdx.x;
  if (mi >= j.n_marches) return;
  constexpr int B2 = NL * NL;
  const int G = op.ng, ndof = G * NL;
  double* psi = j.psi + (size_t)mi * ndof;
  double* y = j.tmp + (size_t)mi * ndof;
  for (int i = 0; i < ndof; ++i) psi[i] = j.psi0[i];
  double plo[NL];
#pragma unroll
  for (int t = 0; t < NL; ++t) plo[t] = j.p_lo[t];
  for (int sg = j.seg_off[mi]; sg < j.seg_off[mi + 1]; ++sg) {
    const int k = j.seg_key[sg];
    const double* Dk = op.D + (size_t)k * G * B2;
    const double* Lk = op.L + (size_t)k * G * B2;
    const double* Uk = op.U + (size_t)k * G * B2;
    const double smin = j.s_min[k];
    double res = 0.0;
    for (int half = 0; half < 2; ++half) {
      const int ns = j.half_n[2 * sg + half];
      if (ns <= 0) continue;
      // the operators are the stepper's (built at the first dz that rounds
      // to this one, as the reference's LU cache), the residual uses this dz
      const double dz = j.half_dz[2 * sg + half];
      const double h = 0.5 * j.st_dz[j.half_st[2 * sg + half]];
      const double* di = Dinv + (size_t)j.half_st[2 * sg + half] * G * B2;
      const double* e = E + (size_t)j.half_st[2 * sg + half] * G * B2;
      for (int it = 0; it < ns; ++it) {
        double tb = 0.0;
#pragma unroll
        for (int t = 0; t < NL; ++t) tb += psi[t] * plo[t];
        // y = B psi = M psi - h G psi, then forward sweep y_g -= E_g y_{g-1}
        for (int g = 0; g < G; ++g) {
          double v[NL];
#pragma unroll
          for (int i = 0; i < NL; ++i) {
            double gpsi = 0.0;
#pragma unroll
            for (int t = 0; t < NL; ++t) {
              gpsi += Dk[g * B2 + i * NL + t] * psi[g * NL + t];
              if (g > 0) gpsi += Lk[g * B2 + i * NL + t] * psi[(g - 1) * NL + t];
              if (g + 1 < G) gpsi += Uk[g * B2 + i * NL + t] * psi[(g + 1) * NL + t];
            }
            v[i] = op.mass[g * NL + i] * psi[g * NL + i] - h * gpsi;
          }
          if (g > 0) {
#pragma unroll
            for (int i = 0; i < NL; ++i) {
              double c = 0.0;
#pragma unroll
              for (int t = 0; t < NL; ++t) c += e[g * B2 + i * NL + t] * y[(g - 1) * NL + t];
              v[i] -= c;
            }
          }
#pragma unroll
          for (int i = 0; i < NL; ++i) y[g * NL + i] = v[i];
        }
        // back sweep: x_g = Dinv_g (y_g - h U_g x_{g+1})
        for (int g = G - 1; g >= 0; --g) {
          double r[NL];
#pragma unroll
          for (int i = 0; i < NL; ++i) {
            double c = y[g * NL + i];
            if (g + 1 < G) {
#pragma unroll
              for (int t = 0; t < NL; ++t) c -= h * Uk[g * B2 + i * NL + t] * psi[(g + 1) * NL + t];
            }
            r[i] = c;
          }
#pragma unroll
          for (int i = 0; i < NL; ++i) {
            double x = 0.0;
#pragma unroll
            for (int t = 0; t < NL; ++t) x += di[g * B2 + i * NL + t] * r[t];
            psi[g * NL + i] = x;
          }
        }
        double ta = 0.0;
#pragma unroll
        for (int t = 0; t < NL; ++t) ta += psi[t] * plo[t];
        res += j.e_min * smin * 0.5 * (tb + ta) * dz;
      }
      if (half == 0) {
        for (int g = 0; g < G; ++g) j.averages[(size_t)sg * G + g] = psi[g * NL];
      }
    }
    j.residual[sg] = res;
    for (int i = 0; i < ndof; ++i)
      if (!isfinite(psi[i])) {
        atomicExch(j.bad, 2);
        break;
      }
  }
}

struct DepositJob {
  int n_rays;
  const int* ray_seg_off;   // n_rays + 1: this ray's segments in the flat list
  const long long* cells;   // per ray segment
  const double* lengths;    // per ray segment
  const int* ray_march;     // march index per ray
  const int* march_seg_off; // first march segment per march
  const double* weight;     // per ray: beam weight * ray weight
  double volume;
  const double* averages;   // march segments x ng
  const double* mres;       // march segments
  double* values;           // ng x ld (device flux table layout)
  int ld;
  double* residual;         // n
  int ng;
};

__global__ void deposit_kernel(DepositJob d) {
  for (int r = 0; r < d.n_rays; ++r) {
    const int s0 = d.ray_seg_off[r], s1 = d.ray_seg_off[r + 1];
    const int ms0 = d.march_seg_off[d.ray_march[r]];
    const double w = d.weight[r];
    const int nseg = s1 - s0;
    for (int e = threadIdx.x; e < nseg * d.ng; e += blockDim.x) {
      const int q = e / d.ng, g = e - q * d.ng;
      const long long cell = d.cells[s0 + q];
      const double track = d.lengths[s0 + q] / d.volume;
      d.values[(size_t)g * d.ld + cell] += w * track * d.averages[(size_t)(ms0 + q) * d.ng + g];
    }
    for (int q = threadIdx.x; q < nseg; q += blockDim.x)
      d.residual[d.cells[s0 + q]] += w * d.mres[ms0 + q] / d.volume;
    __syncthreads();
  }
}

}  // namespace

void march_steppers(int nl, const double* D, const double* L, const double* U, const double* mass,
                    int ng, int n_steppers, const int* key, const double* dz, double* Dinv,
                    double* E, int* bad, cudaStream_t st) {
  MarchOps op{D, L, U, mass, ng};
  const int blocks = (n_steppers + 63) / 64;
  switch (nl) {
    case 1: stepper_kernel<1><<<blocks, 64, 0, st>>>(op, n_steppers, key, dz, Dinv, E, bad); break;
    case 2: stepper_kernel<2><<<blocks, 64, 0, st>>>(op, n_steppers, key, dz, Dinv, E, bad); break;
    case 3: stepper_kernel<3><<<blocks, 64, 0, st>>>(op, n_steppers, key, dz, Dinv, E, bad); break;
    case 4: stepper_kernel<4><<<blocks, 64, 0, st>>>(op, n_steppers, key, dz, Dinv, E, bad); break;
    default: fail(PND_ECONFIG, "energy DG degree above 3 is not supported");
  }
  launched();
}

void march_rays(int nl, const double* D, const double* L, const double* U, const double* mass,
                int ng, const double* Dinv, const double* E, const double* st_dz, int n_marches,
                const int* seg_off, const int* seg_key, const double* half_dz, const int* half_n,
                const int* half_st, const double* s_min, double e_min, const double* psi0,
                const double* p_lo, double* psi, double* tmp, double* averages,
                double* residual, int* bad, cudaStream_t st) {
  MarchOps op{D, L, U, mass, ng};
  MarchJob j{n_marches, seg_off, seg_key, half_dz, half_n, half_st, st_dz, s_min, e_min,
             psi0, p_lo, psi, tmp, averages, residual, bad};
  const int blocks = (n_marches + 31) / 32;
  switch (nl) {
    case 1: march_kernel<1><<<blocks, 32, 0, st>>>(op, j, Dinv, E); break;
    case 2: march_kernel<2><<<blocks, 32, 0, st>>>(op, j, Dinv, E); break;
    case 3: march_kernel<3><<<blocks, 32, 0, st>>>(op, j, Dinv, E); break;
    case 4: march_kernel<4><<<blocks, 32, 0, st>>>(op, j, Dinv, E); break;
    default: fail(PND_ECONFIG, "energy DG degree above 3 is not supported");
  }
  launched();
}

void deposit_rays(int n_rays, const int* ray_seg_off, const long long* cells,
                  const double* lengths, const int* ray_march, const int* march_seg_off,
                  const double* weight, double volume, const double* averages,
                  const double* mres, double* values, int ld, double* residual, int ng,
                  cudaStream_t st) {
  DepositJob d{n_rays, ray_seg_off, cells, lengths, ray_march, march_seg_off, weight,
               volume, averages, mres, values, ld, residual, ng};
  deposit_kernel<<<1, 1024, 0, st>>>(d);
  launched();
}

}  // namespace pnd
