// Tall-skinny Gram engine: out[g][a][b] = sum_c X[c][a] * T_g[c][b].
//
// Every n-side reduction of the step is one of these:
//   * GEN_STENCIL  T_g = D_g (S^-1 Y): L-phase factors (D U0)^T U0
//                  (dlra.py:183-184) and S-phase Grams U^T D U^
//                  (dlra.py:199-209, precontracted);
//   * GEN_WEIGHT   T_g = w_g(c) Y: the 12 weighted Grams B_i of the implicit
//                  scattering substep (dlra.py:285), by material class;
//   * GEN_SOURCE   T[c][b] = N_i(c) S^-1(c) psi_beam(c): source projections
//                  U^T (N psi / S) (dlra.py:307-319);
//   * GEN_PLAIN    T = Y.
// A persistent grid (fixed size, so the reduction order is fixed and reruns
// are bit-identical) walks 64-cell chunks. The chunk's X rows are staged in
// shared memory once, each phase's T rows are generated into shared memory,
// and the 8x8 output tiles are accumulated with FP64 tensor-core
// mma.sync.m8n8k4 (DMMA) in registers across all chunks. Per-block partials
// go to a workspace and a second kernel sums them in block order.
#include "pnd.h"

namespace pnd {

namespace {

constexpr int CH = 64;  // cells per chunk (16 k-steps of the m8n8k4 MMA)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ double fval(const double* __restrict__ col,
                                       const double* __restrict__ inv_s, int c) {
  return col[c] * inv_s[c];
}

// D_s (S^-1 y) at cell c for one column (spatial.py:81-118 row formulas)
__device__ __forceinline__ double stencil_one(const Geom& g, int s, const double* __restrict__ col,
                                              const double* __restrict__ inv_s, int c, int ci,
                                              int cj, int ck) {
  const int axis = g.axis[s >> 1];
  const bool plus = (s & 1) == 0;
  const int len = axis == 0 ? g.nx : (axis == 1 ? g.ny : g.nz);
  const int idx = axis == 0 ? ci : (axis == 1 ? cj : ck);
  const int st = axis == 0 ? 1 : (axis == 1 ? g.nx : g.nx * g.ny);
  const double h = g.h[axis];
  const double f0 = fval(col, inv_s, c);
  if (plus) {
    if (idx >= 2) {
      return (3.0 * f0 - 4.0 * fval(col, inv_s, c - st) + fval(col, inv_s, c - 2 * st)) /
             (2.0 * h);
    }
    if (idx == 1) return (f0 - fval(col, inv_s, c - st)) / h;
    return f0 / h;
  }
  if (idx <= len - 3) {
    return (-3.0 * f0 + 4.0 * fval(col, inv_s, c + st) - fval(col, inv_s, c + 2 * st)) /
           (2.0 * h);
  }
  if (idx == len - 2) return (fval(col, inv_s, c + st) - f0) / h;
  return -f0 / h;
}

template <int T, int NPH, int NW>
__global__ void __launch_bounds__(NW * 32) gram_kernel(GramArgs a, double* __restrict__ partial) {
  constexpr int W = T * 8;       // padded width
  constexpr int LDS = W + 1;     // smem row stride (doubles)
  constexpr int NT = T * T;      // tiles per phase
  constexpr int TPW = (NT + NW - 1) / NW;
  extern __shared__ double smem[];
  double* sX = smem;             // [CH][LDS]
  double* sT = smem + CH * LDS;  // [CH][LDS]

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int nthr = NW * 32;
  const Geom& g = a.geo;
  const int nchunks = (g.n + CH - 1) / CH;

  double acc[NPH][TPW][2];
#pragma unroll
  for (int p = 0; p < NPH; ++p)
#pragma unroll
    for (int t = 0; t < TPW; ++t) acc[p][t][0] = acc[p][t][1] = 0.0;

  const int nxy = g.nx * g.ny;
  for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
    const int c0 = chunk * CH;
    // stage X rows (coalesced along cells)
    for (int idx = tid; idx < CH * W; idx += nthr) {
      const int cell = idx % CH, col = idx / CH;
      const int c = c0 + cell;
      sX[cell * LDS + col] = (c < g.n && col < a.na) ? a.X[(size_t)col * a.ldx + c] : 0.0;
    }
#pragma unroll
    for (int p = 0; p < NPH; ++p) {
      if (p < a.nphase) {
        __syncthreads();  // previous phase's MMAs are done with sT
        for (int idx = tid; idx < CH * W; idx += nthr) {
          const int cell = idx % CH, col = idx / CH;
          const int c = c0 + cell;
          double v = 0.0;
          if (c < g.n && col < a.nb) {
            if (a.gen == GEN_STENCIL) {
              const int ck = c / nxy, rem = c - ck * nxy;
              const int cj = rem / g.nx, ci = rem - cj * g.nx;
              v = stencil_one(g, p, a.Y + (size_t)col * a.ldy, a.inv_s, c, ci, cj, ck);
            } else if (a.gen == GEN_WEIGHT) {
              const int k = a.cls[c];
              const double w = a.wmode == 0 ? (k == p ? a.inv_s[c] : 0.0)
                                            : a.wtab[k * 12 + p] * a.inv_s[c];
              v = w * a.Y[(size_t)col * a.ldy + c];
            } else if (a.gen == GEN_SOURCE) {
              const int beam = col / 12, el = col - beam * 12;
              v = a.wtab[a.cls[c] * 12 + el] * (a.inv_s[c] * a.psi[(size_t)beam * a.ldpsi + c]);
            } else {
              v = a.Y[(size_t)col * a.ldy + c];
            }
          }
          sT[cell * LDS + col] = v;
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < TPW; ++t) {
          const int tile = warp + t * NW;
          if (tile < NT) {
            const int ti = tile / T, tj = tile - (tile / T) * T;
            const double* xa = sX + (lane & 3) * LDS + ti * 8 + (lane >> 2);
            const double* tb = sT + (lane & 3) * LDS + tj * 8 + (lane >> 2);
#pragma unroll 4
            for (int k0 = 0; k0 < CH; k0 += 4) {
              dmma(acc[p][t][0], acc[p][t][1], xa[k0 * LDS], tb[k0 * LDS]);
            }
          }
        }
      }
    }
    __syncthreads();
  }
  // write this block's partial (row-major na x nb per phase)
  double* out = partial + (size_t)blockIdx.x * a.nphase * a.na * a.nb;
#pragma unroll
  for (int p = 0; p < NPH; ++p) {
    if (p < a.nphase) {
#pragma unroll
      for (int t = 0; t < TPW; ++t) {
        const int tile = warp + t * NW;
        if (tile < NT) {
          const int ti = tile / T, tj = tile - (tile / T) * T;
          const int row = ti * 8 + (lane >> 2);
          const int col = tj * 8 + 2 * (lane & 3);
          if (row < a.na) {
            if (col < a.nb) out[((size_t)p * a.na + row) * a.nb + col] = acc[p][t][0];
            if (col + 1 < a.nb) out[((size_t)p * a.na + row) * a.nb + col + 1] = acc[p][t][1];
          }
        }
      }
    }
  }
}

__global__ void reduce_partials(const double* __restrict__ partial, int nblk, int count,
                                double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int b = 0; b < nblk; ++b) s += partial[(size_t)b * count + i];
  out[i] = s;
}

template <int T, int NPH, int NW>
void launch(const GramArgs& a, DBuf& partial, cudaStream_t st) {
  const int W = T * 8;
  const size_t smem = 2 * (size_t)CH * (W + 1) * sizeof(double);
  static bool configured = false;
  if (!configured) {
    CK(cudaFuncSetAttribute(gram_kernel<T, NPH, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem));
    configured = true;
  }
  int dev = 0, sms = 148;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int nchunks = (a.geo.n + CH - 1) / CH;
  int grid = sms * 2;
  if (grid > nchunks) grid = nchunks;
  if (grid < 1) grid = 1;
  const size_t count = (size_t)a.nphase * a.na * a.nb;
  double* part = partial.get(count * grid);
  gram_kernel<T, NPH, NW><<<grid, NW * 32, smem, st>>>(a, part);
  launched();
  reduce_partials<<<(int)((count + 255) / 256), 256, 0, st>>>(part, grid, (int)count, a.out);
  launched();
}

template <int NPH>
void dispatch_t(int t, const GramArgs& a, DBuf& partial, cudaStream_t st) {
  switch (t) {
    case 1: launch<1, NPH, 8>(a, partial, st); break;
    case 2: launch<2, NPH, 8>(a, partial, st); break;
    case 3: launch<3, NPH, 8>(a, partial, st); break;
    case 4: launch<4, NPH, 8>(a, partial, st); break;
    case 5: launch<5, NPH, 8>(a, partial, st); break;
    case 6: launch<6, NPH, 16>(a, partial, st); break;
    case 7: launch<7, NPH, 16>(a, partial, st); break;
    case 8: launch<8, NPH, 16>(a, partial, st); break;
    default: fail(PND_ECONFIG, "gram width above 64 columns is not supported");
  }
}

}  // namespace

void gram(GramArgs a, DBuf& partial, cudaStream_t st) {
  const int w = a.na > a.nb ? a.na : a.nb;
  const int t = (w + 7) / 8;
  if (a.na <= 0 || a.nb <= 0 || a.nphase <= 0) return;
  if (a.gen == GEN_STENCIL) {
    if (a.nphase > 6) fail(PND_ECONFIG, "at most 6 stencils");
    dispatch_t<6>(t, a, partial, st);
  } else if (a.gen == GEN_WEIGHT) {
    if (a.nphase > 12) fail(PND_ECONFIG, "at most 12 weighted Grams");
    if (t > 4) fail(PND_ECONFIG, "weighted Grams support rank <= 32");
    switch (t) {
      case 1: launch<1, 12, 8>(a, partial, st); break;
      case 2: launch<2, 12, 8>(a, partial, st); break;
      case 3: launch<3, 12, 8>(a, partial, st); break;
      default: launch<4, 12, 8>(a, partial, st); break;
    }
  } else {
    if (a.nphase != 1) fail(PND_ECONFIG, "plain/source Grams have one phase");
    dispatch_t<1>(t, a, partial, st);
  }
}

}  // namespace pnd
