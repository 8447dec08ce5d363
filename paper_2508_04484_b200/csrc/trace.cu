// Uncollided ray traversal: thread per ray, bit-exact Amanatides-Woo walk.
//
// Restates raytracer.traverse_grid (/root/reference/pkg/src/pndose/raytracer.py:353-403)
// with every float64 operation written as an explicit round-to-nearest
// intrinsic (__dadd_rn, __dmul_rn, ...), so no multiply-add is ever fused and
// each operation happens in the reference's order. Ties in the axis choice go
// to the first axis (np.argmin); Python's max/min keep their first argument on
// ties, which the explicit comparisons below reproduce, signed zeros included.
// Two launches: the first counts segments per ray, the caller scans the
// counts, the second writes (cell, t_enter, t_exit) at the ray's offset.
#include "pnd.h"

namespace pnd {

namespace {

struct TraceGrid {
  int n[3];
  double h[3];
  double lo[3], hi[3];
  double eps;
};

__device__ __forceinline__ double pmax(double a, double b) { return b > a ? b : a; }
__device__ __forceinline__ double pmin(double a, double b) { return b < a ? b : a; }

template <bool WRITE>
__global__ void traverse_kernel(TraceGrid tg, int n_rays, const double* __restrict__ starts,
                                const double* __restrict__ dirs, int* __restrict__ counts,
                                const long long* __restrict__ offsets, long long* __restrict__ cells,
                                double* __restrict__ t0, double* __restrict__ t1) {
  const int ray = blockIdx.x * blockDim.x + threadIdx.x;
  if (ray >= n_rays) return;
  double p0[3], d[3];
  for (int a = 0; a < 3; ++a) {
    p0[a] = starts[ray * 3 + a];
    d[a] = dirs[ray * 3 + a];
  }
  int emitted = 0;
  long long base = WRITE ? offsets[ray] : 0;
  double t_lo = 0.0, t_hi = __longlong_as_double(0x7ff0000000000000ULL);  // +inf
  bool miss = false;
  for (int a = 0; a < 3; ++a) {
    if (fabs(d[a]) < 1e-14) {
      if (!(tg.lo[a] <= p0[a] && p0[a] <= tg.hi[a])) miss = true;
      continue;
    }
    const double ta = __ddiv_rn(__dsub_rn(tg.lo[a], p0[a]), d[a]);
    const double tb = __ddiv_rn(__dsub_rn(tg.hi[a], p0[a]), d[a]);
    t_lo = pmax(t_lo, pmin(ta, tb));
    t_hi = pmin(t_hi, pmax(ta, tb));
  }
  if (!miss && t_hi > t_lo) {
    const double te = __dadd_rn(t_lo, tg.eps);
    int idx[3], step[3];
    double tmax[3], tdel[3];
    for (int a = 0; a < 3; ++a) {
      const double p = __dadd_rn(p0[a], __dmul_rn(te, d[a]));
      int i = (int)__ddiv_rn(__dsub_rn(p, tg.lo[a]), tg.h[a]);
      i = i < 0 ? 0 : i;
      i = i > tg.n[a] - 1 ? tg.n[a] - 1 : i;
      idx[a] = i;
      step[a] = 0;
      tmax[a] = __longlong_as_double(0x7ff0000000000000ULL);
      tdel[a] = tmax[a];
      if (d[a] > 1e-14) {
        step[a] = 1;
        const double nxt = __dadd_rn(tg.lo[a], __dmul_rn((double)(i + 1), tg.h[a]));
        tmax[a] = __ddiv_rn(__dsub_rn(nxt, p0[a]), d[a]);
        tdel[a] = __ddiv_rn(tg.h[a], d[a]);
      } else if (d[a] < -1e-14) {
        step[a] = -1;
        const double nxt = __dadd_rn(tg.lo[a], __dmul_rn((double)i, tg.h[a]));
        tmax[a] = __ddiv_rn(__dsub_rn(nxt, p0[a]), d[a]);
        tdel[a] = __ddiv_rn(-tg.h[a], d[a]);
      }
    }
    double t = t_lo;
    const double t_end = __dsub_rn(t_hi, 1e-14);
    const long long nxy = (long long)tg.n[0] * tg.n[1];
    while (t < t_end) {
      int axis = 0;
      if (tmax[1] < tmax[axis]) axis = 1;
      if (tmax[2] < tmax[axis]) axis = 2;
      const double tn = pmin(tmax[axis], t_hi);
      if (tn > t) {
        if (WRITE) {
          const long long o = base + emitted;
          cells[o] = (long long)idx[2] * nxy + (long long)idx[1] * tg.n[0] + idx[0];
          t0[o] = t;
          t1[o] = tn;
        }
        ++emitted;
      }
      t = tn;
      idx[axis] += step[axis];
      if (!(0 <= idx[axis] && idx[axis] < tg.n[axis])) break;
      tmax[axis] = __dadd_rn(tmax[axis], tdel[axis]);
    }
  }
  if (!WRITE) counts[ray] = emitted;
}

}  // namespace

void traverse(const Geom& g, const double* origin, int n_rays, const double* starts,
              const double* dirs, int* counts, const long long* offsets, long long* cells,
              double* t0, double* t1, cudaStream_t st) {
  TraceGrid tg;
  tg.n[0] = g.nx;
  tg.n[1] = g.ny;
  tg.n[2] = g.nz;
  double hmax = g.h[0];
  for (int a = 0; a < 3; ++a) {
    tg.h[a] = g.h[a];
    tg.lo[a] = origin[a];
    // bounds: origin + n * h, evaluated in double like Grid3D.extent (spatial.py:73-78)
    tg.hi[a] = origin[a] + (double)tg.n[a] * g.h[a];
    if (a > 0 && g.h[a] > hmax) hmax = g.h[a];
  }
  tg.eps = 1e-10 * hmax;
  const int threads = 128, blocks = (n_rays + threads - 1) / threads;
  if (n_rays <= 0) return;
  if (cells) {
    traverse_kernel<true><<<blocks, threads, 0, st>>>(tg, n_rays, starts, dirs, counts, offsets,
                                                      cells, t0, t1);
  } else {
    traverse_kernel<false><<<blocks, threads, 0, st>>>(tg, n_rays, starts, dirs, counts, offsets,
                                                       cells, t0, t1);
  }
  launched();
}

}  // namespace pnd
