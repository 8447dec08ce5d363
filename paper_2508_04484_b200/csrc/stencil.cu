// Stencil kernels: K-phase Horner stage and stencil Grams (cell-major layout).
//
// The upwind stencils (spatial.py:81-118) reach +-2 cells along every active
// axis. For a chunk of CH consecutive cells the kernel stages, per input
// matrix, box 0 = rows [c0-2, c0+CH+2) (the first active axis has stride 1)
// and rows [c0 + d*st, c0 + d*st + CH), d = -2,-1,+1,+2, for every further
// axis: 1 + 4 (na - 1) contiguous segments, each one cp.async.bulk copy (TMA)
// onto an mbarrier; the zero halo rows around every matrix keep all segments
// in bounds. Lanes run along cells: each thread computes its cell's axis
// indices and the 13 values of 1/S once per chunk, then the 2*na stencil
// values of its columns, written k-major into the DMMA operand tile
// (row length = 4 mod 16 doubles, conflict-free fragment loads). The kernels
// are templated on the number of active axes so all segment indexing is
// static. Two CTAs per SM overlap one CTA's segment copies and stencil
// formation with the other's tensor-core work.
//
//   kstage: out = [D_0 S^-1 X, ..., D_ns-1 S^-1 X | U0] . [M_0; ...; M_ns-1; S0]
//           one Horner stage of the K-phase RK4 (dlra.py:168-174), FP64 DMMA
//           m8n8k4, B fragments from the L1-resident concatenated [M; S0];
//   sgram:  G_s += X^T D_s S^-1 X over all chunks for X = [X1 | X2] (the L- and
//           S-phase factors, dlra.py:183-184, 199-209), accumulated in registers,
//           per-CTA partials summed in fixed order (bit-reproducible).
#include "tma.cuh"

namespace pnd {

namespace {

__host__ __device__ constexpr int pad4(int w) { return ((w + 11) / 16) * 16 + 4; }
__host__ __device__ constexpr int up16(int w) { return (w + 15) / 16 * 16; }

struct Seg {
  int nbox;
  int off[9];      // first row of box b relative to c0
  int nrows;       // staged rows per input (CH + 4 + (nbox - 1) CH)
  int xoff[2];     // smem offset of input 0 / 1 rows
  int ioff;        // smem offset of the [1/S, 0] rows
  int coff;        // smem offset of separate centre rows (-1: none)
  int total;       // doubles staged
  unsigned bytes;  // bytes per chunk
};

template <int CH>
Seg make_seg(const Geom& g, const NMat* in, int nin, const NMat* centre) {
  Seg s{};
  s.nbox = 1;
  s.off[0] = -2;
  const int nxy = g.nx * g.ny;
  for (int ai = 1; ai < g.na; ++ai) {
    const int st = g.axis[ai] == 1 ? g.nx : nxy;
    const int ds[4] = {-2, -1, 1, 2};
    for (int q = 0; q < 4; ++q) s.off[s.nbox++] = ds[q] * st;
  }
  s.nrows = CH + 4 + (s.nbox - 1) * CH;
  int o = 0;
  unsigned bytes = 0;
  for (int k = 0; k < 2; ++k) {
    s.xoff[k] = o;
    if (k < nin) {
      o += up16(s.nrows * in[k].rs);
      bytes += s.nrows * in[k].rs * 8;
    }
  }
  s.ioff = o;
  o += up16(2 * s.nrows);
  bytes += 2 * s.nrows * 8;
  s.coff = -1;
  if (centre) {
    s.coff = o;
    o += up16(CH * centre->rs);
    bytes += CH * centre->rs * 8;
  }
  s.total = up16(o);
  s.bytes = bytes;
  return s;
}

template <int CH>
__device__ __forceinline__ int box_row(int b) {
  return b == 0 ? 0 : CH + 4 + (b - 1) * CH;
}

template <int CH, int NA>
__device__ __forceinline__ void issue_seg(const Seg& S, double* dst, uint64_t* bar, int c0,
                                          const NMat& a, const NMat& b, int nin,
                                          const double* isp, const NMat& c) {
  mbar_expect_tx(bar, S.bytes);
#pragma unroll
  for (int q = 0; q < 1 + 4 * (NA - 1); ++q) {
    const int rows = q == 0 ? CH + 4 : CH;
    const long row = (long)c0 + S.off[q];
    const int drow = box_row<CH>(q);
    bulk_load(dst + S.xoff[0] + drow * a.rs, a.p + row * a.rs, rows * a.rs * 8, bar);
    if (nin > 1) bulk_load(dst + S.xoff[1] + drow * b.rs, b.p + row * b.rs, rows * b.rs * 8, bar);
    bulk_load(dst + S.ioff + 2 * drow, isp + 2 * row, rows * 16, bar);
  }
  if (S.coff >= 0) bulk_load(dst + S.coff, c.p + (long)c0 * c.rs, CH * c.rs * 8, bar);
}

// per-thread stencil context of one cell (its axis indices); the staged rows
// are pre-scaled by 1/S (scale_rows), so f = S^-1 x is read directly
template <int CH, int NA>
struct Ctx {
  int idx[NA], len[NA];

  __device__ __forceinline__ void init(const Geom& g, int c) {
    const int nxy = g.nx * g.ny;
    const int ck = c / nxy, rem = c - ck * nxy;
    const int cj = rem / g.nx, ci = rem - cj * g.nx;
#pragma unroll
    for (int ai = 0; ai < NA; ++ai) {
      const int axis = g.axis[ai];
      idx[ai] = axis == 0 ? ci : axis == 1 ? cj : ck;
      len[ai] = axis == 0 ? g.nx : axis == 1 ? g.ny : g.nz;
    }
  }

  // the 2 NA stencil values of column j (staged rows X with row length rs)
  __device__ __forceinline__ void apply(const Geom& g, const double* X, int rs, int i, int j,
                                        double* t) const {
#pragma unroll
    for (int ai = 0; ai < NA; ++ai) {
      double f[5];
      if (ai == 0) {
#pragma unroll
        for (int d = 0; d < 5; ++d) f[d] = X[(i + d) * rs + j];
      } else {
        const int b = 1 + 4 * (ai - 1);
        f[0] = X[(box_row<CH>(b) + i) * rs + j];
        f[1] = X[(box_row<CH>(b + 1) + i) * rs + j];
        f[2] = X[(i + 2) * rs + j];
        f[3] = X[(box_row<CH>(b + 2) + i) * rs + j];
        f[4] = X[(box_row<CH>(b + 3) + i) * rs + j];
      }
      const int id = idx[ai], ln = len[ai];
      const int axis = g.axis[ai];
      const double ih = axis == 0 ? g.ih[0] : axis == 1 ? g.ih[1] : g.ih[2];
      const double i2h = axis == 0 ? g.i2h[0] : axis == 1 ? g.i2h[1] : g.i2h[2];
      double tp, tm;
      if (id >= 2) tp = (3.0 * f[2] - 4.0 * f[1] + f[0]) * i2h;
      else if (id == 1) tp = (f[2] - f[1]) * ih;
      else tp = f[2] * ih;
      if (id <= ln - 3) tm = (-3.0 * f[2] + 4.0 * f[3] - f[4]) * i2h;
      else if (id == ln - 2) tm = (f[3] - f[2]) * ih;
      else tm = -f[2] * ih;
      t[2 * ai] = tp;
      t[2 * ai + 1] = tm;
    }
  }
};

// in-place X[row][:] *= 1/S[row] over the staged rows of one input; calls
// keep(row, col, unscaled value) first (the kstage base rows)
template <class Keep>
__device__ __forceinline__ void scale_rows(double* X, int rs, int nrows, const double* I,
                                           Keep keep) {
  const int total = nrows * rs;
  const int drow = blockDim.x / rs, dcol = blockDim.x - drow * rs;
  int row = threadIdx.x / rs, col = threadIdx.x - row * rs;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const double v = X[e];
    keep(row, col, v);
    X[e] = v * I[2 * row];
    row += drow;
    col += dcol;
    if (col >= rs) {
      col -= rs;
      ++row;
    }
  }
}

template <class Kern>
int resident(Kern k, int threads, size_t smem) {
  int nb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, threads, smem));
  return nb < 1 ? 1 : nb;
}

// ===================================================================== kstage
constexpr int KC = 32;
constexpr int KCS = pad4(KC);  // 36: k-major A tile row length

template <int NA, int RB>
__global__ void __launch_bounds__(256, 2)
    kstage_kernel(Geom g, NMat X, NMat U0, NMat out, const double* __restrict__ Bcat, int K,
                  int K4, Seg S, const double* __restrict__ isp) {
  constexpr int NS = 2 * NA;
  constexpr int NT = RB / 8;
  constexpr int TILES = (KC / 8) * NT;
  extern __shared__ __align__(128) double sm[];
  double* buf = sm;
  double* sA = sm + S.total;                 // [K4][KCS] k-major
  uint64_t* bar = (uint64_t*)(sA + K4 * KCS);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int xc = X.cols, ra = U0.p ? U0.cols : 0, rso = out.rs;
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  for (int i = tid; i < (K4 - K) * KCS; i += 256) sA[K * KCS + i] = 0.0;
  __syncthreads();
  const bool sepc = S.coff >= 0;
  const int nchunks = (g.n + KC - 1) / KC;
  int it = 0;
  for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, ++it) {
    const int c0 = chunk * KC;
    if (tid == 0) {
      fence_proxy_async();
      issue_seg<KC, NA>(S, buf, bar, c0, X, X, 1, isp, U0);
    }
    mbar_wait(bar, it & 1);
    // rows past n (chunk tail) read zero halo rows; their results are not stored
    double* Xs = buf + S.xoff[0];
    double* base = sA + NS * xc * KCS;
    if (sepc) {
      for (int e = tid; e < ra * KC; e += 256) {
        const int j = e / KC, i = e - j * KC;
        base[j * KCS + i] = buf[S.coff + i * U0.rs + j];
      }
      scale_rows(Xs, X.rs, S.nrows, buf + S.ioff, [](int, int, double) {});
    } else {
      scale_rows(Xs, X.rs, S.nrows, buf + S.ioff, [&](int row, int col, double v) {
        if (row >= 2 && row < KC + 2 && col < ra) base[col * KCS + row - 2] = v;
      });
    }
    __syncthreads();
    const int i = lane;
    Ctx<KC, NA> cx;
    cx.init(g, c0 + i);
    for (int j = warp; j < xc; j += 8) {
      double t[NS];
      cx.apply(g, Xs, X.rs, i, j, t);
#pragma unroll
      for (int s = 0; s < NS; ++s) sA[(s * xc + j) * KCS + i] = t[s];
    }
    __syncthreads();
    for (int tile = warp; tile < TILES; tile += 8) {
      const int mt = tile / NT, nt = tile - mt * NT;
      double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
      const double* pa = sA + (lane & 3) * KCS + mt * 8 + (lane >> 2);
      const double* pb = Bcat + (lane & 3) * RB + nt * 8 + (lane >> 2);
      int k0 = 0;
      for (; k0 + 8 <= K4; k0 += 8) {
        dmma884(d0, d1, pa[k0 * KCS], __ldg(pb + k0 * RB));
        dmma884(e0, e1, pa[(k0 + 4) * KCS], __ldg(pb + (k0 + 4) * RB));
      }
      if (k0 < K4) dmma884(d0, d1, pa[k0 * KCS], __ldg(pb + k0 * RB));
      const int row = c0 + mt * 8 + (lane >> 2);
      const int n = nt * 8 + 2 * (lane & 3);
      if (row < g.n) {
        double* o = out.p + (long)row * rso + n;
        if (n + 1 < rso) {
          *reinterpret_cast<double2*>(o) = make_double2(d0 + e0, d1 + e1);
        } else if (n < rso) {
          o[0] = d0 + e0;
        }
      }
    }
    __syncthreads();
  }
}

__global__ void bcat_kernel(const double* M, int kM, const double* S0, int kS, int r, int K4,
                            int RB, double* B) {
  for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < K4 * RB; i += blockDim.x * gridDim.x) {
    const int k = i / RB, n = i % RB;
    double v = 0.0;
    if (n < r) {
      if (k < kM) v = M[(size_t)k * r + n];
      else if (k < kM + kS) v = S0[(size_t)(k - kM) * r + n];
    }
    B[i] = v;
  }
}

template <int NA, int RB>
void kstage_launch(const KStageArgs& a, DBuf& bcat, cudaStream_t st) {
  const Geom& g = a.geo;
  const int ra = a.U0.p ? a.U0.cols : 0;
  const bool sepc = ra > 0 && !(a.U0.p == a.X.p && a.U0.rs == a.X.rs);
  const int K = 2 * NA * a.X.cols + ra;
  const int K4 = (K + 7) / 8 * 8;
  double* B = bcat.get((size_t)K4 * RB);
  bcat_kernel<<<16, 256, 0, st>>>(a.M, 2 * NA * a.X.cols, a.S0, ra, a.out.cols, K4, RB, B);
  launched();
  const Seg S = make_seg<KC>(g, &a.X, 1, sepc ? &a.U0 : nullptr);
  const size_t smem = ((size_t)S.total + (size_t)K4 * KCS) * sizeof(double) + 16;
  if (smem > 227 * 1024) fail(PND_ECONFIG, "kstage tile exceeds shared memory");
  CK(cudaFuncSetAttribute(kstage_kernel<NA, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)smem));
  const int nchunks = (g.n + KC - 1) / KC;
  int grid = sm_count() * resident(kstage_kernel<NA, RB>, 256, smem);
  if (grid > nchunks) grid = nchunks;
  kstage_kernel<NA, RB><<<grid, 256, smem, st>>>(g, a.X, a.U0, a.out, B, K, K4, S, a.inv_s);
  launched();
}

template <int NA>
void kstage_na(const KStageArgs& a, DBuf& bcat, cudaStream_t st) {
  const int r = a.out.cols;
  if (r <= 8) kstage_launch<NA, 8>(a, bcat, st);
  else if (r <= 16) kstage_launch<NA, 16>(a, bcat, st);
  else if (r <= 24) kstage_launch<NA, 24>(a, bcat, st);
  else if (r <= 32) kstage_launch<NA, 32>(a, bcat, st);
  else fail(PND_ECONFIG, "kstage supports at most 32 output columns");
}

// ===================================================================== sgram
constexpr int GC = 16;
constexpr int GTL = pad4(GC);  // 20

template <int NA, int T8>
__global__ void __launch_bounds__(256, T8 <= 5 ? 2 : 1)
    sgram_kernel(Geom g, NMat X1, NMat X2, Seg S, const double* __restrict__ isp,
                 double* __restrict__ partial) {
  constexpr int NS = 2 * NA;
  constexpr int W = T8 * 8;
  constexpr int TILES = NS * T8 * T8;
  constexpr int TPW = (TILES + 7) / 8;
  extern __shared__ __align__(128) double sm[];
  double* buf = sm;
  constexpr int XS = pad4(W);
  double* sT = sm + S.total;                   // [NS][W][GTL] stencils, k = cell
  double* sX = sT + NS * W * GTL;              // [GC][XS] unscaled centre rows
  uint64_t* bar = (uint64_t*)(sX + GC * XS);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int a1 = X1.cols, a2 = X2.p ? X2.cols : 0, w = a1 + a2;
  const int nin = X2.p ? 2 : 1;
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  for (int i = tid; i < NS * W * GTL + GC * XS; i += 256) sT[i] = 0.0;
  __syncthreads();
  double acc[TPW][2];
#pragma unroll
  for (int t = 0; t < TPW; ++t) acc[t][0] = acc[t][1] = 0.0;
  const int nchunks = (g.n + GC - 1) / GC;
  const int i = lane & (GC - 1), jh = lane >> 4;
  int it = 0;
  for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, ++it) {
    const int c0 = chunk * GC;
    if (tid == 0) {
      fence_proxy_async();
      issue_seg<GC, NA>(S, buf, bar, c0, X1, X2, nin, isp, X1);
    }
    mbar_wait(bar, it & 1);
    // keep the unscaled centre rows (the A = X^T operand), then scale by 1/S;
    // rows past n are zero halo rows and contribute nothing
    {
      double* X1s = buf + S.xoff[0];
      scale_rows(X1s, X1.rs, S.nrows, buf + S.ioff, [&](int row, int col, double v) {
        if (row >= 2 && row < GC + 2 && col < a1) sX[(row - 2) * XS + col] = v;
      });
      if (a2)
        scale_rows(buf + S.xoff[1], X2.rs, S.nrows, buf + S.ioff,
                   [&](int row, int col, double v) {
                     if (row >= 2 && row < GC + 2 && col < a2) sX[(row - 2) * XS + a1 + col] = v;
                   });
    }
    __syncthreads();
    Ctx<GC, NA> cx;
    cx.init(g, c0 + i);
    for (int j = 2 * warp + jh; j < w; j += 16) {
      double t[NS];
      if (j < a1) cx.apply(g, buf + S.xoff[0], X1.rs, i, j, t);
      else cx.apply(g, buf + S.xoff[1], X2.rs, i, j - a1, t);
#pragma unroll
      for (int s = 0; s < NS; ++s) sT[(s * W + j) * GTL + i] = t[s];
    }
    __syncthreads();
    // A = X^T: fragment (m = column, k = cell) from the unscaled centre rows
    const int m0 = lane >> 2, kq = lane & 3;
#pragma unroll
    for (int t = 0; t < TPW; ++t) {
      const int tile = warp + 8 * t;
      if (tile < TILES) {
        const int s = tile / (T8 * T8), rem = tile - s * T8 * T8;
        const int ti = rem / T8, tj = rem - ti * T8;
        const double* pa = sX + kq * XS + ti * 8 + m0;
        const double* pb = sT + (s * W + tj * 8 + m0) * GTL + kq;
#pragma unroll
        for (int k0 = 0; k0 < GC; k0 += 4) dmma884(acc[t][0], acc[t][1], pa[k0 * XS], pb[k0]);
      }
    }
    __syncthreads();
  }
  double* out = partial + (size_t)blockIdx.x * NS * w * w;
#pragma unroll
  for (int t = 0; t < TPW; ++t) {
    const int tile = warp + 8 * t;
    if (tile < TILES) {
      const int s = tile / (T8 * T8), rem = tile - s * T8 * T8;
      const int ti = rem / T8, tj = rem - ti * T8;
      const int row = ti * 8 + (lane >> 2), col = tj * 8 + 2 * (lane & 3);
      if (row < w) {
        double* o = out + ((size_t)s * w + row) * w;
        if (col < w) o[col] = acc[t][0];
        if (col + 1 < w) o[col + 1] = acc[t][1];
      }
    }
  }
}

__global__ void reduce_parts(const double* __restrict__ partial, int nblk, int count,
                             double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int b = 0; b < nblk; ++b) s += partial[(size_t)b * count + i];
  out[i] = s;
}

template <int NA, int T8>
void sgram_launch(const Geom& g, NMat X1, NMat X2, const double* isp, double* out, DBuf& partial,
                  cudaStream_t st) {
  const NMat ins[2] = {X1, X2};
  const Seg S = make_seg<GC>(g, ins, X2.p ? 2 : 1, nullptr);
  const int W = T8 * 8;
  const size_t smem =
      ((size_t)S.total + (size_t)2 * NA * W * GTL + (size_t)GC * pad4(W)) * sizeof(double) + 16;
  if (smem > 227 * 1024) fail(PND_ECONFIG, "stencil Gram tile exceeds shared memory");
  CK(cudaFuncSetAttribute(sgram_kernel<NA, T8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)smem));
  const int nchunks = (g.n + GC - 1) / GC;
  int grid = sm_count() * resident(sgram_kernel<NA, T8>, 256, smem);
  if (grid > nchunks) grid = nchunks;
  const int w = X1.cols + (X2.p ? X2.cols : 0);
  const size_t count = (size_t)2 * NA * w * w;
  double* part = partial.get(count * grid);
  sgram_kernel<NA, T8><<<grid, 256, smem, st>>>(g, X1, X2, S, isp, part);
  launched();
  reduce_parts<<<(int)((count + 255) / 256), 256, 0, st>>>(part, grid, (int)count, out);
  launched();
}

template <int NA>
void sgram_na(const Geom& g, NMat X1, NMat X2, const double* isp, double* out, DBuf& partial,
              cudaStream_t st) {
  const int w = X1.cols + (X2.p ? X2.cols : 0);
  switch ((w + 7) / 8) {
    case 1: sgram_launch<NA, 1>(g, X1, X2, isp, out, partial, st); break;
    case 2: sgram_launch<NA, 2>(g, X1, X2, isp, out, partial, st); break;
    case 3: sgram_launch<NA, 3>(g, X1, X2, isp, out, partial, st); break;
    case 4: sgram_launch<NA, 4>(g, X1, X2, isp, out, partial, st); break;
    case 5: sgram_launch<NA, 5>(g, X1, X2, isp, out, partial, st); break;
    case 6: sgram_launch<NA, 6>(g, X1, X2, isp, out, partial, st); break;
    case 7:
    case 8: sgram_launch<NA, 8>(g, X1, X2, isp, out, partial, st); break;
    default: fail(PND_ECONFIG, "stencil Grams support at most 64 columns");
  }
}

DBuf g_bcat;  // concatenated [M; S0] of the current kstage launch (stream-ordered reuse)

}  // namespace

void kstage(const KStageArgs& a, cudaStream_t st) {
  if (a.X.cols > 32 || (a.U0.p && a.U0.cols > 32))
    fail(PND_ECONFIG, "kstage supports <= 32 input columns");
  switch (a.geo.na) {
    case 1: kstage_na<1>(a, g_bcat, st); break;
    case 2: kstage_na<2>(a, g_bcat, st); break;
    case 3: kstage_na<3>(a, g_bcat, st); break;
    default: fail(PND_ECONFIG, "grid has no active axis");
  }
}

void stencil_grams(const Geom& g, NMat X1, NMat X2, const double* isp, double* out,
                   DBuf& partial, cudaStream_t st) {
  switch (g.na) {
    case 1: sgram_na<1>(g, X1, X2, isp, out, partial, st); break;
    case 2: sgram_na<2>(g, X1, X2, isp, out, partial, st); break;
    case 3: sgram_na<3>(g, X1, X2, isp, out, partial, st); break;
    default: return;
  }
}

void stencil_grams_xy(const Geom& g, NMat X, NMat Y, const double* isp, double* out,
                      DBuf& partial, cudaStream_t st) {
  // Grams of [Y | X] against its stencils, then the (X, D Y) block
  const int a = X.cols, b = Y.cols, w = a + b;
  DBuf full;
  double* f = full.get((size_t)g.ns * w * w);
  stencil_grams(g, Y, X, isp, f, partial, st);
  for (int s = 0; s < g.ns; ++s) {
    CK(cudaMemcpy2DAsync(out + (size_t)s * a * b, b * sizeof(double),
                         f + (size_t)s * w * w + (size_t)b * w, w * sizeof(double),
                         b * sizeof(double), a, cudaMemcpyDeviceToDevice, st));
  }
  CK(cudaStreamSynchronize(st));
  full.free_();
}

}  // namespace pnd
