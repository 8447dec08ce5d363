// Tall-skinny Gram engine: out[g] = A_g^T T_g summed over all cells.
//
// Every n-side reduction of the step is one of these:
//   * GEN_STENCIL  T_g = D_g (S^-1 Y): L-phase factors (D U0)^T U0
//                  (dlra.py:183-184) and S-phase Grams U^T D U^
//                  (dlra.py:199-209, precontracted);
//   * GEN_WEIGHT   T_g = w_g(c) Y: the weighted Grams B_i of the implicit
//                  scattering substep (dlra.py:285), by material class;
//   * GEN_SOURCE   T[c][b] = N_i(c) S^-1(c) psi_beam(c): source projections
//                  U^T (N psi / S) (dlra.py:307-319);
//   * GEN_PLAIN    T = Y;
//   * GEN_LINCOMB  T = Y TA - X TB, also written back to memory: one pass of
//                  the block Gram-Schmidt / SVQB orthonormalisation of the
//                  augmentation (phase 0: X^T T, phase 1: T^T T).
// The A operand of phase g is the staged X tile, or T itself for the
// `self_phase`. A persistent grid (fixed size, so the summation order is
// fixed and reruns are bit-identical) walks 64-cell chunks; the 8x8 output
// tiles are accumulated across all chunks with FP64 tensor-core
// mma.sync.m8n8k4 (DMMA) in registers; per-block partials are summed in block
// order by a second kernel.
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

struct CellPos {
  int c;         // flat index (valid if c < n)
  int idx[3];    // axis coordinates
};

// D_s (S^-1 y) at one cell for one column (spatial.py:81-118 row formulas)
__device__ __forceinline__ double stencil_one(const Geom& g, int s, const double* __restrict__ col,
                                              const double* __restrict__ inv_s,
                                              const CellPos& p) {
  const int axis = g.axis[s >> 1];
  const bool plus = (s & 1) == 0;
  const int len = axis == 0 ? g.nx : (axis == 1 ? g.ny : g.nz);
  const int idx = p.idx[axis];
  const int st = axis == 0 ? 1 : (axis == 1 ? g.nx : g.nx * g.ny);
  const int c = p.c;
  const double f0 = col[c] * inv_s[c];
  if (plus) {
    if (idx >= 2) {
      const double f1 = col[c - st] * inv_s[c - st], f2 = col[c - 2 * st] * inv_s[c - 2 * st];
      return (3.0 * f0 - 4.0 * f1 + f2) * g.i2h[axis];
    }
    if (idx == 1) return (f0 - col[c - st] * inv_s[c - st]) * g.ih[axis];
    return f0 * g.ih[axis];
  }
  if (idx <= len - 3) {
    const double f1 = col[c + st] * inv_s[c + st], f2 = col[c + 2 * st] * inv_s[c + 2 * st];
    return (-3.0 * f0 + 4.0 * f1 - f2) * g.i2h[axis];
  }
  if (idx == len - 2) return (col[c + st] * inv_s[c + st] - f0) * g.ih[axis];
  return -f0 * g.ih[axis];
}

template <int T, int NPH, int NW>
__global__ void __launch_bounds__(NW * 32) gram_kernel(GramArgs a, double* __restrict__ partial) {
  constexpr int W = T * 8;       // padded width
  constexpr int LDS = W + 1;     // smem row stride (doubles)
  constexpr int NT = T * T;      // tiles per phase
  constexpr int TPW = (NT + NW - 1) / NW;
  constexpr int NTHR = NW * 32;
  static_assert(NTHR % CH == 0, "thread count must be a multiple of the chunk");
  extern __shared__ double smem[];
  double* sX = smem;             // [CH][LDS] A operand rows (X)
  double* sT = sX + CH * LDS;    // [CH][LDS] generated rows (T)
  double* sY = sT + CH * LDS;    // [CH][LDS] second input rows (LINCOMB)
  double* sTA = sY + CH * LDS;   // [W][W]   LINCOMB coefficients on Y
  double* sTB = sTA + W * W;     // [W][W]   LINCOMB coefficients on X

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const Geom& g = a.geo;
  const int nchunks = (g.n + CH - 1) / CH;
  const bool lincomb = a.gen == GEN_LINCOMB;

  if (lincomb) {
    for (int i = tid; i < W * W; i += NTHR) {
      const int r = i / W, c = i - r * W;
      sTA[i] = (r < a.ny && c < a.nb) ? a.TA[r * a.nb + c] : 0.0;
      sTB[i] = (r < a.na && c < a.nb) ? a.TB[r * a.nb + c] : 0.0;
    }
  }

  double acc[NPH][TPW][2];
#pragma unroll
  for (int p = 0; p < NPH; ++p)
#pragma unroll
    for (int t = 0; t < TPW; ++t) acc[p][t][0] = acc[p][t][1] = 0.0;

  const int my_cell = tid & (CH - 1);  // fixed: NTHR is a multiple of CH
  const int col0 = tid / CH;
  constexpr int CSTEP = NTHR / CH;
  const int nxy = g.nx * g.ny;
  for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
    const int c0 = chunk * CH;
    CellPos pos;
    pos.c = c0 + my_cell;
    const bool valid = pos.c < g.n;
    {
      const int k = pos.c / nxy, rem = pos.c - k * nxy;
      pos.idx[2] = k;
      pos.idx[1] = rem / g.nx;
      pos.idx[0] = rem - pos.idx[1] * g.nx;
    }
    __syncthreads();  // previous chunk is done with every tile
    for (int col = col0; col < W; col += CSTEP) {
      sX[my_cell * LDS + col] = (valid && col < a.na) ? a.X[(size_t)col * a.ldx + pos.c] : 0.0;
      if (lincomb)
        sY[my_cell * LDS + col] = (valid && col < a.ny) ? a.Y[(size_t)col * a.ldy + pos.c] : 0.0;
    }
    if (lincomb) __syncthreads();
#pragma unroll
    for (int p = 0; p < NPH; ++p) {
      if (p < a.nphase) {
        // phase 0 generates T; later phases regenerate it unless it is reused
        const bool gen = (p == 0) || a.gen == GEN_STENCIL || a.gen == GEN_WEIGHT;
        if (gen) {
          if (p > 0) __syncthreads();  // previous phase's MMAs are done with sT
          for (int col = col0; col < W; col += CSTEP) {
            double v = 0.0;
            if (valid && col < a.nb) {
              if (a.gen == GEN_STENCIL) {
                v = stencil_one(g, p, a.Y + (size_t)col * a.ldy, a.inv_s, pos);
              } else if (a.gen == GEN_WEIGHT) {
                const int k = a.cls[pos.c];
                const double w = a.wmode == 0 ? (k == p ? a.inv_s[pos.c] : 0.0)
                                              : a.wtab[k * 12 + p] * a.inv_s[pos.c];
                v = w * a.Y[(size_t)col * a.ldy + pos.c];
              } else if (a.gen == GEN_SOURCE) {
                const int beam = col / 12, el = col - beam * 12;
                v = a.wtab[a.cls[pos.c] * 12 + el] *
                    (a.inv_s[pos.c] * a.psi[(size_t)beam * a.ldpsi + pos.c]);
              } else if (a.gen == GEN_LINCOMB) {
                double s = 0.0;
                const double* yr = sY + my_cell * LDS;
                const double* xr = sX + my_cell * LDS;
                for (int k = 0; k < a.ny; ++k) s = fma(yr[k], sTA[k * W + col], s);
                for (int k = 0; k < a.na; ++k) s = fma(-xr[k], sTB[k * W + col], s);
                v = s;
                if (a.Yout) a.Yout[(size_t)col * a.ldo + pos.c] = v;
              } else {
                v = a.Y[(size_t)col * a.ldy + pos.c];
              }
            }
            sT[my_cell * LDS + col] = v;
          }
          __syncthreads();
        }
        const double* sA = (p == a.self_phase) ? sT : sX;
#pragma unroll
        for (int t = 0; t < TPW; ++t) {
          const int tile = warp + t * NW;
          if (tile < NT) {
            const int ti = tile / T, tj = tile - (tile / T) * T;
            const double* xa = sA + (lane & 3) * LDS + ti * 8 + (lane >> 2);
            const double* tb = sT + (lane & 3) * LDS + tj * 8 + (lane >> 2);
#pragma unroll 4
            for (int k0 = 0; k0 < CH; k0 += 4) {
              dmma(acc[p][t][0], acc[p][t][1], xa[k0 * LDS], tb[k0 * LDS]);
            }
          }
        }
      }
    }
  }
  // write this block's partial: phase p is rows_p x nb (rows = na, or nb for the self phase)
  const size_t total = (size_t)a.nb * (a.nphase * a.na + (a.self_phase >= 0 ? a.nb - a.na : 0));
  double* out = partial + (size_t)blockIdx.x * total;
#pragma unroll
  for (int p = 0; p < NPH; ++p) {
    if (p < a.nphase) {
      const int rows = (p == a.self_phase) ? a.nb : a.na;
      size_t off = 0;
      for (int q = 0; q < p; ++q) off += (size_t)((q == a.self_phase) ? a.nb : a.na) * a.nb;
#pragma unroll
      for (int t = 0; t < TPW; ++t) {
        const int tile = warp + t * NW;
        if (tile < NT) {
          const int ti = tile / T, tj = tile - (tile / T) * T;
          const int row = ti * 8 + (lane >> 2);
          const int col = tj * 8 + 2 * (lane & 3);
          if (row < rows) {
            if (col < a.nb) out[off + (size_t)row * a.nb + col] = acc[p][t][0];
            if (col + 1 < a.nb) out[off + (size_t)row * a.nb + col + 1] = acc[p][t][1];
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

int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  return sms;
}

template <int T, int NPH, int NW>
void launch(const GramArgs& a, DBuf& partial, cudaStream_t st) {
  const int W = T * 8;
  const bool lc = a.gen == GEN_LINCOMB;
  const size_t smem = ((lc ? 3 : 2) * (size_t)CH * (W + 1) + (lc ? 2 * (size_t)W * W : 0)) *
                      sizeof(double);
  static size_t configured = 0;
  if (smem > configured) {
    CK(cudaFuncSetAttribute(gram_kernel<T, NPH, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem));
    configured = smem;
  }
  const int nchunks = (a.geo.n + CH - 1) / CH;
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gram_kernel<T, NPH, NW>, NW * 32,
                                                   smem));
  int grid = sm_count() * (per_sm > 0 ? per_sm : 1);
  if (grid > nchunks) grid = nchunks;
  if (grid < 1) grid = 1;
  const size_t count =
      (size_t)a.nb * (a.nphase * a.na + (a.self_phase >= 0 ? a.nb - a.na : 0));
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
  if (a.gen == GEN_STENCIL) {
    if (a.nphase != a.geo.ns) fail(PND_ECONFIG, "stencil Grams cover every stencil");
    stencil_grams(a, partial, st);
    return;
  }
  if (a.gen == GEN_LINCOMB) {
    lincomb(a, partial, a.nphase >= 2, st);
    return;
  }
  int w = a.na > a.nb ? a.na : a.nb;
  if (a.gen == GEN_LINCOMB && a.ny > w) w = a.ny;
  const int t = (w + 7) / 8;
  if (a.na <= 0 || a.nb <= 0 || a.nphase <= 0) return;
  if (a.self_phase >= a.nphase) a.self_phase = -1;
  if (a.gen == GEN_STENCIL) {
    if (a.nphase > 6) fail(PND_ECONFIG, "at most 6 stencils");
    a.self_phase = -1;
    dispatch_t<6>(t, a, partial, st);
  } else if (a.gen == GEN_WEIGHT) {
    if (a.nphase > 12) fail(PND_ECONFIG, "at most 12 weighted Grams");
    if (t > 4) fail(PND_ECONFIG, "weighted Grams support rank <= 32");
    a.self_phase = -1;
    switch (t) {
      case 1: launch<1, 12, 8>(a, partial, st); break;
      case 2: launch<2, 12, 8>(a, partial, st); break;
      case 3: launch<3, 12, 8>(a, partial, st); break;
      default: launch<4, 12, 8>(a, partial, st); break;
    }
  } else if (a.gen == GEN_LINCOMB) {
    if (a.nphase > 2) fail(PND_ECONFIG, "lincomb Grams have at most two phases");
    if (t > 4) fail(PND_ECONFIG, "orthonormalisation supports at most 32 columns per block");
    switch (t) {
      case 1: launch<1, 2, 8>(a, partial, st); break;
      case 2: launch<2, 2, 8>(a, partial, st); break;
      case 3: launch<3, 2, 8>(a, partial, st); break;
      default: launch<4, 2, 8>(a, partial, st); break;
    }
  } else {
    if (a.nphase != 1) fail(PND_ECONFIG, "plain/source Grams have one phase");
    a.self_phase = -1;
    dispatch_t<1>(t, a, partial, st);
  }
}

}  // namespace pnd
