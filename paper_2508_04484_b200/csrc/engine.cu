// Chunked FP64 tensor-core engine for the n-side hot kernels.
//
// Every n-side operation of the step is "generate per-cell feature rows, then
// contract them": the K-phase Horner stage (stencil values of 6 stencils x r
// columns plus the U0 row, contracted with [M_s ; S0]), the orthonormalisation
// passes and the truncation rotation (rows of [Y | X] contracted with
// [TA ; -TB]), and the stencil Grams (U^T D_s U^). A persistent grid walks
// chunks of consecutive cells; each chunk's feature rows are generated into a
// shared-memory tile (global loads coalesced along cells; stencil
// neighbours read through L1/L2), then contracted with FP64 mma.sync.m8n8k4
// (DMMA): row GEMMs (cells x K) . (K x r) for the per-cell outputs, and
// transposed tile products accumulated in registers across chunks for the
// Grams. Shared-memory tiles use row strides = 4 (mod 16) doubles, which
// makes the DMMA fragment loads of a half-warp hit 16 distinct 8-byte banks.
#include "pnd.h"

namespace pnd {

namespace {

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// smallest stride >= w with stride % 16 == 4 (conflict-free DMMA fragment loads)
__host__ __device__ constexpr int padded(int w) {
  return ((w + 11) / 16) * 16 + 4 >= w ? ((w + 11) / 16) * 16 + 4 : ((w + 11) / 16) * 16 + 20;
}

int sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

template <class K>
int resident_blocks(K kernel, int threads, size_t smem) {
  int nb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, smem));
  return nb < 1 ? 1 : nb;
}

// 13-point neighbourhood of one cell: offsets and 1/S at -2..+2 per active axis
struct Hood {
  int off[3][5];
  double is[3][5];
  bool ok[3][5];
};

__device__ __forceinline__ void make_hood(const Geom& g, const double* __restrict__ inv_s, int c,
                                          bool valid, Hood& hd) {
  const int nxy = g.nx * g.ny;
  const int ck = c / nxy, rem = c - ck * nxy;
  const int cj = rem / g.nx, ci = rem - cj * g.nx;
#pragma unroll
  for (int ai = 0; ai < 3; ++ai) {
    const int axis = ai < g.na ? g.axis[ai] : 0;
    const int len = axis == 0 ? g.nx : (axis == 1 ? g.ny : g.nz);
    const int idx = axis == 0 ? ci : (axis == 1 ? cj : ck);
    const int st = axis == 0 ? 1 : (axis == 1 ? g.nx : nxy);
#pragma unroll
    for (int d = 0; d < 5; ++d) {
      const int q = idx + d - 2;
      const bool ok = valid && ai < g.na && q >= 0 && q < len;
      hd.ok[ai][d] = ok;
      hd.off[ai][d] = ok ? c + (d - 2) * st : 0;
      hd.is[ai][d] = ok ? inv_s[c + (d - 2) * st] : 0.0;
    }
  }
}

// the 2*na stencil values D_s (S^-1 y) of one column at the hood's cell
// (spatial.py:81-118: (3,-4,1)/2h interior, first order next to the inflow
// boundary, zero-inflow ghost on the boundary cell)
__device__ __forceinline__ void stencils_of(const Geom& g, const Hood& hd,
                                            const double* __restrict__ col, double* t) {
#pragma unroll
  for (int ai = 0; ai < 3; ++ai) {
    if (ai < g.na) {
      const int axis = g.axis[ai];
      const double ih = g.ih[axis], i2h = g.i2h[axis];
      double f[5];
#pragma unroll
      for (int d = 0; d < 5; ++d) f[d] = hd.ok[ai][d] ? col[hd.off[ai][d]] * hd.is[ai][d] : 0.0;
      double tp, tm;
      if (hd.ok[ai][0]) tp = (3.0 * f[2] - 4.0 * f[1] + f[0]) * i2h;
      else if (hd.ok[ai][1]) tp = (f[2] - f[1]) * ih;
      else tp = f[2] * ih;
      if (hd.ok[ai][4]) tm = (-3.0 * f[2] + 4.0 * f[3] - f[4]) * i2h;
      else if (hd.ok[ai][3]) tm = (f[3] - f[2]) * ih;
      else tm = -f[2] * ih;
      t[2 * ai] = tp;
      t[2 * ai + 1] = tm;
    }
  }
}

// --------------------------------------------------------------------------
// K-phase Horner stage: out = [D_0 S^-1 X, ..., D_ns-1 S^-1 X, U0] . [M_0; ...; M_ns-1; S0]
constexpr int KCH = 64;

template <int RB>
__global__ void __launch_bounds__(256, 2) kstage2_kernel(KStageArgs a, int K, int K4, int KS,
                                                         int BS) {
  constexpr int NT = RB / 8;          // n-tiles
  constexpr int TILES = (KCH / 8) * NT;
  constexpr int TPW = (TILES + 7) / 8;
  extern __shared__ double sm[];
  double* sA = sm;                    // [KCH][KS]
  double* sB = sA + KCH * KS;         // [K4][BS]
  const Geom& g = a.geo;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ns = g.ns, xc = a.xc, ra = a.U0 ? a.ra : 0, r = a.r;
  for (int i = tid; i < K4 * BS; i += 256) {
    const int k = i / BS, n = i - k * BS;
    double v = 0.0;
    if (n < r && k < K) v = k < ns * xc ? a.M[(size_t)k * r + n] : a.S0[(size_t)(k - ns * xc) * r + n];
    sB[i] = v;
  }
  for (int i = tid; i < KCH * (K4 - K); i += 256) {
    const int cell = i / (K4 - K), k = K + i % (K4 - K);
    sA[cell * KS + k] = 0.0;
  }
  const int cell = tid & (KCH - 1), cgrp = tid >> 6;
  const int nchunks = (g.n + KCH - 1) / KCH;
  for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
    const int c0 = chunk * KCH, c = c0 + cell;
    const bool valid = c < g.n;
    Hood hd;
    make_hood(g, a.inv_s, valid ? c : 0, valid, hd);
    double* arow = sA + cell * KS;
    for (int j = cgrp; j < xc; j += 4) {
      double t[6];
      stencils_of(g, hd, a.X + (size_t)j * a.ldx, t);
#pragma unroll
      for (int s = 0; s < 6; ++s)
        if (s < ns) arow[s * xc + j] = valid ? t[s] : 0.0;
    }
    for (int j = cgrp; j < ra; j += 4) arow[ns * xc + j] = valid ? a.U0[(size_t)j * a.ldu + c] : 0.0;
    __syncthreads();
    double acc[TPW][2];
#pragma unroll
    for (int t = 0; t < TPW; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll
    for (int t = 0; t < TPW; ++t) {
      const int tile = warp + 8 * t;
      if (tile < TILES) {
        const int mt = tile / NT, nt = tile - mt * NT;
        const double* pa = sA + (mt * 8 + (lane >> 2)) * KS + (lane & 3);
        const double* pb = sB + (lane & 3) * BS + nt * 8 + (lane >> 2);
        for (int k0 = 0; k0 < K4; k0 += 4) dmma(acc[t][0], acc[t][1], pa[k0], pb[k0 * BS]);
      }
    }
#pragma unroll
    for (int t = 0; t < TPW; ++t) {
      const int tile = warp + 8 * t;
      if (tile < TILES) {
        const int mt = tile / NT, nt = tile - mt * NT;
        const int cc = c0 + mt * 8 + (lane >> 2);
        const int n = nt * 8 + 2 * (lane & 3);
        if (cc < g.n) {
          if (n < r) a.out[(size_t)n * a.ldo + cc] = acc[t][0];
          if (n + 1 < r) a.out[(size_t)(n + 1) * a.ldo + cc] = acc[t][1];
        }
      }
    }
    __syncthreads();
  }
}

template <int RB>
void kstage2_launch(const KStageArgs& a, cudaStream_t st) {
  const int ns = a.geo.ns;
  const int ra = a.U0 ? a.ra : 0;
  const int K = ns * a.xc + ra;
  const int K4 = (K + 3) / 4 * 4;
  const int KS = padded(K4);
  const int BS = padded(RB);
  const size_t smem = ((size_t)KCH * KS + (size_t)K4 * BS) * sizeof(double);
  CK(cudaFuncSetAttribute(kstage2_kernel<RB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)smem));
  const int nchunks = (a.geo.n + KCH - 1) / KCH;
  int grid = sms() * resident_blocks(kstage2_kernel<RB>, 256, smem);
  if (grid > nchunks) grid = nchunks;
  kstage2_kernel<RB><<<grid, 256, smem, st>>>(a, K, K4, KS, BS);
  launched();
}

// --------------------------------------------------------------------------
// Linear combination (+ Grams): T = [Y | X] . [TA ; -TB]  (cells x nb), written to
// out; phase 0 accumulates X^T T, phase 1 T^T T.
constexpr int LCH = 64;

template <int NB8, bool GRAMS>
__global__ void __launch_bounds__(256) lincomb2_kernel(GramArgs a, int K4, int KS, int BS, int TS,
                                                       double* __restrict__ partial) {
  constexpr int OT = (LCH / 8) * NB8;          // output tiles
  constexpr int OPW = (OT + 7) / 8;
  constexpr int XT = NB8;                      // max x-gram row tiles (na <= NBP assumed)
  constexpr int GTILES = GRAMS ? (XT * NB8 + NB8 * NB8) : 0;
  constexpr int GPW = GRAMS ? (GTILES + 7) / 8 : 1;
  extern __shared__ double sm[];
  double* sA = sm;                             // [LCH][KS]  rows [Y | X]
  double* sB = sA + LCH * KS;                  // [K4][BS]   [TA ; -TB]
  double* sT = sB + K4 * BS;                   // [LCH][TS]  output rows
  const Geom& g = a.geo;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ny = a.ny, na = a.na, nb = a.nb, K = ny + na;
  for (int i = tid; i < K4 * BS; i += 256) {
    const int k = i / BS, n = i - k * BS;
    double v = 0.0;
    if (n < nb && k < K) v = k < ny ? a.TA[k * nb + n] : -a.TB[(k - ny) * nb + n];
    sB[i] = v;
  }
  for (int i = tid; i < LCH * (K4 - K); i += 256) {
    const int cell = i / (K4 - K), k = K + i % (K4 - K);
    sA[cell * KS + k] = 0.0;
  }
  double gacc[GPW][2];
#pragma unroll
  for (int t = 0; t < GPW; ++t) gacc[t][0] = gacc[t][1] = 0.0;
  const int cell = tid & (LCH - 1), cgrp = tid >> 6;
  const int nchunks = (g.n + LCH - 1) / LCH;
  for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
    const int c0 = chunk * LCH, c = c0 + cell;
    const bool valid = c < g.n;
    double* arow = sA + cell * KS;
    for (int j = cgrp; j < K; j += 4) {
      double v = 0.0;
      if (valid) v = j < ny ? a.Y[(size_t)j * a.ldy + c] : a.X[(size_t)(j - ny) * a.ldx + c];
      arow[j] = v;
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < OPW; ++t) {
      const int tile = warp + 8 * t;
      if (tile < OT) {
        const int mt = tile / NB8, nt = tile - mt * NB8;
        double d0 = 0.0, d1 = 0.0;
        const double* pa = sA + (mt * 8 + (lane >> 2)) * KS + (lane & 3);
        const double* pb = sB + (lane & 3) * BS + nt * 8 + (lane >> 2);
        for (int k0 = 0; k0 < K4; k0 += 4) dmma(d0, d1, pa[k0], pb[k0 * BS]);
        const int row = mt * 8 + (lane >> 2), n = nt * 8 + 2 * (lane & 3);
        const bool rv = c0 + row < g.n;
        sT[row * TS + n] = rv ? d0 : 0.0;
        sT[row * TS + n + 1] = rv ? d1 : 0.0;
      }
    }
    __syncthreads();
    if (a.Yout) {
      for (int j = cgrp; j < nb; j += 4)
        if (valid) a.Yout[(size_t)j * a.ldo + c] = sT[cell * TS + j];
    }
    if (GRAMS) {
#pragma unroll
      for (int t = 0; t < GPW; ++t) {
        const int tile = warp + 8 * t;
        if (tile < GTILES) {
          const bool xg = tile < XT * NB8;
          const int tt = xg ? tile : tile - XT * NB8;
          const int ti = tt / NB8, tj = tt - ti * NB8;
          // A = (X or T)^T : A[m = col][k = cell]; B = T[cell][col]
          const double* pa = xg ? sA + (lane & 3) * KS + ny + ti * 8 + (lane >> 2)
                                : sT + (lane & 3) * TS + ti * 8 + (lane >> 2);
          const int sa = xg ? KS : TS;
          const double* pb = sT + (lane & 3) * TS + tj * 8 + (lane >> 2);
          if (!xg || ti * 8 < na) {
#pragma unroll 4
            for (int k0 = 0; k0 < LCH; k0 += 4)
              dmma(gacc[t][0], gacc[t][1], xg && ti * 8 + (lane >> 2) >= na ? 0.0 : pa[k0 * sa],
                   pb[k0 * TS]);
          }
        }
      }
    }
    __syncthreads();
  }
  if (GRAMS) {
    // partial layout: [X^T T (na x nb)] [T^T T (nb x nb)]
    double* out = partial + (size_t)blockIdx.x * (na + nb) * nb;
#pragma unroll
    for (int t = 0; t < GPW; ++t) {
      const int tile = warp + 8 * t;
      if (tile < GTILES) {
        const bool xg = tile < XT * NB8;
        const int tt = xg ? tile : tile - XT * NB8;
        const int ti = tt / NB8, tj = tt - ti * NB8;
        const int row = ti * 8 + (lane >> 2), col = tj * 8 + 2 * (lane & 3);
        const int rows = xg ? na : nb;
        const size_t off = xg ? 0 : (size_t)na * nb;
        if (row < rows) {
          if (col < nb) out[off + (size_t)row * nb + col] = gacc[t][0];
          if (col + 1 < nb) out[off + (size_t)row * nb + col + 1] = gacc[t][1];
        }
      }
    }
  }
}

__global__ void reduce_blocks(const double* __restrict__ partial, int nblk, int count,
                              double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int b = 0; b < nblk; ++b) s += partial[(size_t)b * count + i];
  out[i] = s;
}

template <int NB8, bool GRAMS>
void lincomb2_launch(const GramArgs& a, DBuf& partial, cudaStream_t st) {
  const int K = a.ny + a.na;
  const int K4 = (K + 3) / 4 * 4;
  const int KS = padded(K4), BS = padded(NB8 * 8), TS = padded(NB8 * 8);
  const size_t smem =
      ((size_t)LCH * KS + (size_t)K4 * BS + (size_t)LCH * TS) * sizeof(double);
  CK(cudaFuncSetAttribute(lincomb2_kernel<NB8, GRAMS>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int nchunks = (a.geo.n + LCH - 1) / LCH;
  int grid = sms() * resident_blocks(lincomb2_kernel<NB8, GRAMS>, 256, smem);
  if (grid > nchunks) grid = nchunks;
  const size_t count = (size_t)(a.na + a.nb) * a.nb;
  double* part = GRAMS ? partial.get(count * grid) : nullptr;
  lincomb2_kernel<NB8, GRAMS><<<grid, 256, smem, st>>>(a, K4, KS, BS, TS, part);
  launched();
  if (GRAMS) {
    reduce_blocks<<<(int)((count + 255) / 256), 256, 0, st>>>(part, grid, (int)count, a.out);
    launched();
  }
}

// --------------------------------------------------------------------------
// Stencil Grams: out_s = X^T D_s (S^-1 Y) for every stencil s, all stencils of a
// (cell, column) generated at once from its 13-point neighbourhood.
constexpr int SCH = 32;

template <int T8>
__global__ void __launch_bounds__(256) sgram_kernel(GramArgs a, int LS,
                                                    double* __restrict__ partial) {
  constexpr int W = T8 * 8;
  constexpr int NT = T8 * T8;
  constexpr int TPW = (NT + 7) / 8;
  extern __shared__ double sm[];
  double* sX = sm;              // [SCH][LS]
  double* sT = sX + SCH * LS;   // [6][SCH][LS]
  const Geom& g = a.geo;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ns = g.ns;
  double acc[6][TPW][2];
#pragma unroll
  for (int s = 0; s < 6; ++s)
#pragma unroll
    for (int t = 0; t < TPW; ++t) acc[s][t][0] = acc[s][t][1] = 0.0;
  const int cell = tid & (SCH - 1), cgrp = tid >> 5;
  const int nchunks = (g.n + SCH - 1) / SCH;
  for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
    const int c = chunk * SCH + cell;
    const bool valid = c < g.n;
    Hood hd;
    make_hood(g, a.inv_s, valid ? c : 0, valid, hd);
    for (int j = cgrp; j < W; j += 8) {
      double t[6] = {0, 0, 0, 0, 0, 0};
      double x = 0.0;
      if (valid && j < a.nb) stencils_of(g, hd, a.Y + (size_t)j * a.ldy, t);
      if (valid && j < a.na) x = a.X[(size_t)j * a.ldx + c];
      sX[cell * LS + j] = x;
#pragma unroll
      for (int s = 0; s < 6; ++s)
        if (s < ns) sT[(s * SCH + cell) * LS + j] = valid && j < a.nb ? t[s] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      if (s < ns) {
        const double* tb0 = sT + s * SCH * LS;
#pragma unroll
        for (int t = 0; t < TPW; ++t) {
          const int tile = warp + 8 * t;
          if (tile < NT) {
            const int ti = tile / T8, tj = tile - ti * T8;
            const double* xa = sX + (lane & 3) * LS + ti * 8 + (lane >> 2);
            const double* tb = tb0 + (lane & 3) * LS + tj * 8 + (lane >> 2);
#pragma unroll
            for (int k0 = 0; k0 < SCH; k0 += 4)
              dmma(acc[s][t][0], acc[s][t][1], xa[k0 * LS], tb[k0 * LS]);
          }
        }
      }
    }
    __syncthreads();
  }
  double* out = partial + (size_t)blockIdx.x * ns * a.na * a.nb;
#pragma unroll
  for (int s = 0; s < 6; ++s) {
    if (s < ns) {
#pragma unroll
      for (int t = 0; t < TPW; ++t) {
        const int tile = warp + 8 * t;
        if (tile < NT) {
          const int ti = tile / T8, tj = tile - ti * T8;
          const int row = ti * 8 + (lane >> 2), col = tj * 8 + 2 * (lane & 3);
          if (row < a.na) {
            double* o = out + ((size_t)s * a.na + row) * a.nb;
            if (col < a.nb) o[col] = acc[s][t][0];
            if (col + 1 < a.nb) o[col + 1] = acc[s][t][1];
          }
        }
      }
    }
  }
}

template <int T8>
void sgram_launch(const GramArgs& a, DBuf& partial, cudaStream_t st) {
  const int LS = padded(T8 * 8);
  const size_t smem = (size_t)7 * SCH * LS * sizeof(double);
  CK(cudaFuncSetAttribute(sgram_kernel<T8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)smem));
  const int nchunks = (a.geo.n + SCH - 1) / SCH;
  int grid = sms() * resident_blocks(sgram_kernel<T8>, 256, smem);
  if (grid > nchunks) grid = nchunks;
  const size_t count = (size_t)a.geo.ns * a.na * a.nb;
  double* part = partial.get(count * grid);
  sgram_kernel<T8><<<grid, 256, smem, st>>>(a, LS, part);
  launched();
  reduce_blocks<<<(int)((count + 255) / 256), 256, 0, st>>>(part, grid, (int)count, a.out);
  launched();
}

}  // namespace

void lincomb(const GramArgs& a, DBuf& partial, bool grams, cudaStream_t st) {
  const int w = a.nb > a.na ? a.nb : a.na;
  if (a.ny + a.na > 128) fail(PND_ECONFIG, "lincomb supports at most 128 input columns");
#define PND_LC(N8)                                                         \
  do {                                                                     \
    if (grams) lincomb2_launch<N8, true>(a, partial, st);                  \
    else lincomb2_launch<N8, false>(a, partial, st);                       \
  } while (0)
  if (w <= 8) PND_LC(1);
  else if (w <= 16) PND_LC(2);
  else if (w <= 24) PND_LC(3);
  else if (w <= 32) PND_LC(4);
  else if (w <= 40) PND_LC(5);
  else if (w <= 48) PND_LC(6);
  else if (w <= 64) PND_LC(8);
  else fail(PND_ECONFIG, "lincomb supports at most 64 output columns");
#undef PND_LC
}


}  // namespace pnd
