// Stencil kernels with TMA-staged halos and FP64 tensor-core (DMMA) contractions.
//
// The upwind stencils (spatial.py:81-118) reach +-2 cells along every active
// axis. A chunk of consecutive cells [c0, c0 + CH) needs, per input column,
//   box 0: cells [c0 - 2, c0 + CH + 2)   (the first active axis has stride 1,
//          since every inactive axis has one cell)
//   boxes 1..: [c0 + d*st, c0 + d*st + CH) for d = -2, -1, +1, +2 along each
//          further active axis (stride nx or nx*ny)
// Each box is one cp.async.bulk.tensor.2d of {cells, columns} from the
// column-major matrix into shared memory; cells outside the grid arrive as
// zeros. One thread issues the boxes of chunk i+1 while all warps compute chunk
// i (double buffer, one mbarrier per buffer). The stencil values are then
// formed from shared memory (the boundary closures need the cell's axis index)
// and contracted with DMMA:
//   kstage3: out = [D_0 S^-1 X ... D_ns-1 S^-1 X | U0] . [M_0; ...; M_ns-1; S0]
//            (one Horner stage of the K-phase RK4, dlra.py:168-174);
//   sgram3:  G_s += X^T D_s S^-1 Y over all chunks (the L- and S-phase
//            factors, dlra.py:183-184, 199-209), accumulated in registers.
// Shared-memory tiles are laid out [column][cell] with row lengths = 4
// (mod 16) doubles, so DMMA fragment loads and the warp-per-column stencil
// reads are bank-conflict free.
#include "tma.cuh"

namespace pnd {

namespace {

__host__ __device__ constexpr int pad4(int w) { return ((w + 11) / 16) * 16 + 4; }
__host__ __device__ constexpr int up16(int w) { return (w + 15) / 16 * 16; }

int sm_count2() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

struct BoxPlan {
  int nbox;     // 1 + 4 (na - 1)
  int off[9];   // first cell of box b relative to c0 (box 0 starts at -2)
};

BoxPlan make_plan(const Geom& g) {
  BoxPlan p{};
  p.nbox = 1;
  p.off[0] = -2;
  const int nxy = g.nx * g.ny;
  for (int ai = 1; ai < g.na; ++ai) {
    const int axis = g.axis[ai];
    const int st = axis == 1 ? g.nx : nxy;
    const int ds[4] = {-2, -1, 1, 2};
    for (int q = 0; q < 4; ++q) p.off[p.nbox++] = ds[q] * st;
  }
  return p;
}

struct CellCoord {
  int idx[3];
  int len[3];
};

__device__ __forceinline__ CellCoord coord_of(const Geom& g, int c) {
  const int nxy = g.nx * g.ny;
  const int ck = c / nxy, rem = c - ck * nxy;
  const int cj = rem / g.nx, ci = rem - cj * g.nx;
  const int all[3] = {ci, cj, ck};
  const int lens[3] = {g.nx, g.ny, g.nz};
  CellCoord cc;
#pragma unroll
  for (int ai = 0; ai < 3; ++ai) {
    const int axis = ai < g.na ? g.axis[ai] : 0;
    cc.idx[ai] = all[axis];
    cc.len[ai] = lens[axis];
  }
  return cc;
}

// A TMA box of FP64 must start on a 16-byte boundary in its innermost
// dimension: with an odd row stride (odd nx) the +-nx boxes would start on odd
// cells, so then every box b >= 1 is fetched one cell early with the long
// (CH + 4) box and read with shift[b] = 1.
struct KLayout {
  int nbox;
  int off[9];      // first cell of box b relative to c0 (the TMA start is off - shift)
  int shift[9];    // 0 or 1
  int blen;        // cells per box for b >= 1 (CH, or CH + 4 with odd offsets)
  int xbox[9];     // offset (doubles) of X box b inside a buffer
  int ibox[9];     // offset of inv_s box b
  int ubox;        // offset of the separate centre box (-1: none)
  int buf;         // doubles per buffer (multiple of 16)
  unsigned bytes;  // TMA bytes per chunk
};

// the 2*na stencil values of column j at chunk cell i from the staged boxes
// (box 0: length CH + 4 starting at cell -2; boxes b >= 1: length CH)
template <int CH>
__device__ __forceinline__ void stencils_smem(const Geom& g, const CellCoord& cc, int i,
                                              const double* B, const KLayout& L, int j,
                                              double* t) {
  const double* xb0 = B + L.xbox[0] + j * (CH + 4);
  const double* ib0 = B + L.ibox[0];
#pragma unroll
  for (int ai = 0; ai < 3; ++ai) {
    if (ai < g.na) {
      const int axis = g.axis[ai];
      const double ih = g.ih[axis], i2h = g.i2h[axis];
      double f[5];
      if (ai == 0) {
#pragma unroll
        for (int d = 0; d < 5; ++d) f[d] = xb0[i + d] * ib0[i + d];
      } else {
        const int b = 1 + 4 * (ai - 1);
        const int bl = L.blen;
        f[0] = B[L.xbox[b] + j * bl + i + L.shift[b]] * B[L.ibox[b] + i + L.shift[b]];
        f[1] = B[L.xbox[b + 1] + j * bl + i + L.shift[b + 1]] * B[L.ibox[b + 1] + i + L.shift[b + 1]];
        f[2] = xb0[i + 2] * ib0[i + 2];
        f[3] = B[L.xbox[b + 2] + j * bl + i + L.shift[b + 2]] * B[L.ibox[b + 2] + i + L.shift[b + 2]];
        f[4] = B[L.xbox[b + 3] + j * bl + i + L.shift[b + 3]] * B[L.ibox[b + 3] + i + L.shift[b + 3]];
      }
      const int idx = cc.idx[ai], len = cc.len[ai];
      double tp, tm;
      if (idx >= 2) tp = (3.0 * f[2] - 4.0 * f[1] + f[0]) * i2h;
      else if (idx == 1) tp = (f[2] - f[1]) * ih;
      else tp = f[2] * ih;
      if (idx <= len - 3) tm = (-3.0 * f[2] + 4.0 * f[3] - f[4]) * i2h;
      else if (idx == len - 2) tm = (f[3] - f[2]) * ih;
      else tm = -f[2] * ih;
      t[2 * ai] = tp;
      t[2 * ai + 1] = tm;
    }
  }
}

// -------------------------------------------------------------------- kstage3
constexpr int KC = 32;          // cells per chunk
constexpr int KL0 = KC + 4;     // box 0 length
constexpr int KCS = pad4(KC);   // k-major A tile stride (36)

struct KMaps {
  CUtensorMap xr, xs, ir, is, uc;
};

template <int RB>
__global__ void __launch_bounds__(256, 1)
    kstage3_kernel(const __grid_constant__ KMaps maps, KStageArgs a, KLayout L, int K, int K4,
                   int BS) {
  constexpr int NT = RB / 8;
  constexpr int TILES = (KC / 8) * NT;
  constexpr int TPW = (TILES + 7) / 8;
  extern __shared__ __align__(128) double sm[];
  double* buf0 = sm;
  double* sA = sm + 2 * L.buf;        // [K4][KCS]
  double* sB = sA + K4 * KCS;         // [K4][BS]
  double* sO = sB + K4 * BS;          // [RB][KCS]
  uint64_t* bar = (uint64_t*)(sO + RB * KCS);
  const Geom& g = a.geo;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ns = g.ns, xc = a.xc, ra = a.U0 ? a.ra : 0, r = a.r;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  for (int i = tid; i < K4 * BS; i += 256) {
    const int k = i / BS, n = i - k * BS;
    double v = 0.0;
    if (n < r && k < K) v = k < ns * xc ? a.M[(size_t)k * r + n] : a.S0[(size_t)(k - ns * xc) * r + n];
    sB[i] = v;
  }
  for (int i = tid; i < (K4 - K) * KCS; i += 256) sA[K * KCS + i] = 0.0;
  __syncthreads();

  const int nchunks = (g.n + KC - 1) / KC;
  auto issue = [&](int chunk, int b) {
    double* dst = buf0 + b * L.buf;
    const int c0 = chunk * KC;
    mbar_expect_tx(&bar[b], L.bytes);
    tma_load_2d(dst + L.xbox[0], &maps.xr, &bar[b], c0 + L.off[0], 0);
    tma_load_2d(dst + L.ibox[0], &maps.ir, &bar[b], c0 + L.off[0], 0);
    const bool lng = L.blen != KC;
    for (int q = 1; q < L.nbox; ++q) {
      const int s0 = c0 + L.off[q] - L.shift[q];
      tma_load_2d(dst + L.xbox[q], lng ? &maps.xr : &maps.xs, &bar[b], s0, 0);
      tma_load_2d(dst + L.ibox[q], lng ? &maps.ir : &maps.is, &bar[b], s0, 0);
    }
    if (L.ubox >= 0) tma_load_2d(dst + L.ubox, &maps.uc, &bar[b], c0, 0);
  };
  if (tid == 0 && blockIdx.x < nchunks) issue(blockIdx.x, 0);

  const int cell = tid & (KC - 1), cgrp = warp;
  int it = 0;
  for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, ++it) {
    const int b = it & 1;
    const int next = chunk + gridDim.x;
    if (tid == 0 && next < nchunks) {
      fence_proxy_async();
      issue(next, b ^ 1);
    }
    mbar_wait(&bar[b], (it >> 1) & 1);
    const double* B = buf0 + b * L.buf;
    const int c0 = chunk * KC, c = c0 + cell;
    const bool valid = c < g.n;
    const CellCoord cc = coord_of(g, valid ? c : 0);
    for (int j = cgrp; j < xc; j += 8) {
      double t[6];
      stencils_smem<KC>(g, cc, cell, B, L, j, t);
#pragma unroll
      for (int s = 0; s < 6; ++s)
        if (s < ns) sA[(s * xc + j) * KCS + cell] = valid ? t[s] : 0.0;
    }
    for (int j = cgrp; j < ra; j += 8) {
      const double u = L.ubox >= 0 ? B[L.ubox + j * KC + cell] : B[L.xbox[0] + j * KL0 + cell + 2];
      sA[(ns * xc + j) * KCS + cell] = valid ? u : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < TPW; ++t) {
      const int tile = warp + 8 * t;
      if (tile < TILES) {
        const int mt = tile / NT, nt = tile - mt * NT;
        double d0 = 0.0, d1 = 0.0;
        const double* pa = sA + (lane & 3) * KCS + mt * 8 + (lane >> 2);
        const double* pb = sB + (lane & 3) * BS + nt * 8 + (lane >> 2);
        for (int k0 = 0; k0 < K4; k0 += 4) dmma884(d0, d1, pa[k0 * KCS], pb[k0 * BS]);
        const int m = mt * 8 + (lane >> 2), n = nt * 8 + 2 * (lane & 3);
        sO[n * KCS + m] = d0;
        sO[(n + 1) * KCS + m] = d1;
      }
    }
    __syncthreads();
    if (valid)
      for (int j = cgrp; j < r; j += 8) a.out[(size_t)j * a.ldo + c] = sO[j * KCS + cell];
    // the next iteration's writes into sA / sO and its TMA into this buffer
    // happen after every thread passed this barrier
    __syncthreads();
  }
}

// box layout of one buffer: X boxes, 1/S boxes, optional centre box
KLayout box_layout(const Geom& g, int ch, int cols, int sep_cols) {
  const BoxPlan p = make_plan(g);
  KLayout L{};
  L.nbox = p.nbox;
  bool odd = false;
  for (int q = 0; q < p.nbox; ++q) {
    L.off[q] = p.off[q];
    odd = odd || (q > 0 && (p.off[q] & 1));
  }
  L.blen = odd ? ch + 4 : ch;
  for (int q = 0; q < p.nbox; ++q) L.shift[q] = (q > 0 && odd) ? (p.off[q] & 1) : 0;
  int o = 0;
  unsigned bytes = 0;
  for (int q = 0; q < p.nbox; ++q) {
    const int len = q == 0 ? ch + 4 : L.blen;
    L.xbox[q] = o;
    o += up16(len * cols);
    bytes += len * cols * 8;
  }
  for (int q = 0; q < p.nbox; ++q) {
    const int len = q == 0 ? ch + 4 : L.blen;
    L.ibox[q] = o;
    o += up16(len);
    bytes += len * 8;
  }
  L.ubox = -1;
  if (sep_cols > 0) {
    L.ubox = o;
    o += up16(ch * sep_cols);
    bytes += ch * sep_cols * 8;
  }
  L.buf = up16(o);
  L.bytes = bytes;
  return L;
}

KLayout klayout(const Geom& g, int xc, int ra_sep) { return box_layout(g, KC, xc, ra_sep); }

template <int RB>
void kstage3_launch(const KStageArgs& a, cudaStream_t st) {
  const Geom& g = a.geo;
  const int ns = g.ns;
  const int ra = a.U0 ? a.ra : 0;
  const bool x_is_u = a.U0 && a.X == a.U0 && a.ldx == a.ldu && a.xc >= ra;
  const int K = ns * a.xc + ra;
  const int K4 = (K + 3) / 4 * 4;
  const int BS = pad4(RB);
  const KLayout L = klayout(g, a.xc, (ra > 0 && !x_is_u) ? ra : 0);
  KMaps maps;
  make_tmap(&maps.xr, a.X, g.n, a.ldx, a.xc, KL0, a.xc);
  make_tmap(&maps.xs, a.X, g.n, a.ldx, a.xc, KC, a.xc);
  make_tmap(&maps.ir, a.inv_s, g.n, g.ld, 1, KL0, 1);
  make_tmap(&maps.is, a.inv_s, g.n, g.ld, 1, KC, 1);
  if (ra > 0 && !x_is_u) make_tmap(&maps.uc, a.U0, g.n, a.ldu, ra, KC, ra);
  else maps.uc = maps.xs;
  const size_t smem = (2 * (size_t)L.buf + (size_t)K4 * KCS + (size_t)K4 * BS +
                       (size_t)RB * KCS) * sizeof(double) + 64;
  if (smem > 227 * 1024) fail(PND_ECONFIG, "kstage tile exceeds shared memory");
  CK(cudaFuncSetAttribute(kstage3_kernel<RB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)smem));
  const int nchunks = (g.n + KC - 1) / KC;
  int grid = sm_count2();
  if (grid > nchunks) grid = nchunks;
  kstage3_kernel<RB><<<grid, 256, smem, st>>>(maps, a, L, K, K4, BS);
  launched();
}

// -------------------------------------------------------------------- sgram3
constexpr int GC = 16;          // cells per chunk
constexpr int GL0 = GC + 4;     // box 0 length (= 20, = 4 mod 16: conflict-free A reads)
constexpr int GTL = GC + 4;     // T tile row length

struct GMaps {
  CUtensorMap yr, ys, ir, is, xc;
};

template <int T8>
__global__ void __launch_bounds__(256, 1)
    sgram3_kernel(const __grid_constant__ GMaps maps, GramArgs a, KLayout L, int xsep,
                  double* __restrict__ partial) {
  constexpr int W = T8 * 8;
  constexpr int TILES = 6 * T8 * T8;
  constexpr int TPW = (TILES + 7) / 8;
  extern __shared__ __align__(128) double sm[];
  double* buf0 = sm;
  double* sT = sm + 2 * L.buf;        // [6][W][GTL]
  uint64_t* bar = (uint64_t*)(sT + 6 * W * GTL);
  const Geom& g = a.geo;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ns = g.ns, na = a.na, nb = a.nb;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  double acc[TPW][2];
#pragma unroll
  for (int t = 0; t < TPW; ++t) acc[t][0] = acc[t][1] = 0.0;
  const int nchunks = (g.n + GC - 1) / GC;
  auto issue = [&](int chunk, int b) {
    double* dst = buf0 + b * L.buf;
    const int c0 = chunk * GC;
    mbar_expect_tx(&bar[b], L.bytes);
    tma_load_2d(dst + L.xbox[0], &maps.yr, &bar[b], c0 + L.off[0], 0);
    tma_load_2d(dst + L.ibox[0], &maps.ir, &bar[b], c0 + L.off[0], 0);
    const bool lng = L.blen != GC;
    for (int q = 1; q < L.nbox; ++q) {
      const int s0 = c0 + L.off[q] - L.shift[q];
      tma_load_2d(dst + L.xbox[q], lng ? &maps.yr : &maps.ys, &bar[b], s0, 0);
      tma_load_2d(dst + L.ibox[q], lng ? &maps.ir : &maps.is, &bar[b], s0, 0);
    }
    if (L.ubox >= 0) tma_load_2d(dst + L.ubox, &maps.xc, &bar[b], c0, 0);
  };
  if (tid == 0 && blockIdx.x < nchunks) issue(blockIdx.x, 0);
  const int cell = tid & (GC - 1), cgrp = tid >> 4;
  int it = 0;
  for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, ++it) {
    const int b = it & 1;
    const int next = chunk + gridDim.x;
    if (tid == 0 && next < nchunks) {
      fence_proxy_async();
      issue(next, b ^ 1);
    }
    mbar_wait(&bar[b], (it >> 1) & 1);
    const double* B = buf0 + b * L.buf;
    const int c = chunk * GC + cell;
    const bool valid = c < g.n;
    const CellCoord cc = coord_of(g, valid ? c : 0);
    for (int j = cgrp; j < W; j += 16) {
      double t[6] = {0, 0, 0, 0, 0, 0};
      if (j < nb) stencils_smem<GC>(g, cc, cell, B, L, j, t);
#pragma unroll
      for (int s = 0; s < 6; ++s)
        if (s < ns) sT[(s * W + j) * GTL + cell] = (valid && j < nb) ? t[s] : 0.0;
    }
    __syncthreads();
    // A = X^T: A[m = column][k = cell] from the centre of Y's box 0 (X == Y) or X's box
    const double* xa = xsep ? B + L.ubox : B + L.xbox[0] + 2;
    const int xl = xsep ? GC : GL0;
#pragma unroll
    for (int t = 0; t < TPW; ++t) {
      const int tile = warp + 8 * t;
      if (tile < TILES) {
        const int s = tile / (T8 * T8), rem = tile - s * T8 * T8;
        const int ti = rem / T8, tj = rem - ti * T8;
        if (s < ns) {
          const int m = ti * 8 + (lane >> 2);
          const bool mv = m < na;
          const double* pa = xa + (mv ? m : 0) * xl + (lane & 3);
          const double* pb = sT + (s * W + tj * 8 + (lane >> 2)) * GTL + (lane & 3);
#pragma unroll
          for (int k0 = 0; k0 < GC; k0 += 4)
            dmma884(acc[t][0], acc[t][1], mv ? pa[k0] : 0.0, pb[k0]);
        }
      }
    }
    __syncthreads();
  }
  double* out = partial + (size_t)blockIdx.x * ns * na * nb;
#pragma unroll
  for (int t = 0; t < TPW; ++t) {
    const int tile = warp + 8 * t;
    if (tile < TILES) {
      const int s = tile / (T8 * T8), rem = tile - s * T8 * T8;
      const int ti = rem / T8, tj = rem - ti * T8;
      const int row = ti * 8 + (lane >> 2), col = tj * 8 + 2 * (lane & 3);
      if (s < ns && row < na) {
        double* o = out + ((size_t)s * na + row) * nb;
        if (col < nb) o[col] = acc[t][0];
        if (col + 1 < nb) o[col + 1] = acc[t][1];
      }
    }
  }
}

__global__ void reduce_blocks2(const double* __restrict__ partial, int nblk, int count,
                               double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int b = 0; b < nblk; ++b) s += partial[(size_t)b * count + i];
  out[i] = s;
}

KLayout glayout(const Geom& g, int ny, int xsep_cols) { return box_layout(g, GC, ny, xsep_cols); }

template <int T8>
void sgram3_launch(const GramArgs& a, DBuf& partial, cudaStream_t st) {
  const Geom& g = a.geo;
  const bool x_is_y = a.X == a.Y && a.ldx == a.ldy && a.na <= a.nb;
  const int xsep = x_is_y ? 0 : a.na;
  const KLayout L = glayout(g, a.nb, xsep);
  GMaps maps;
  make_tmap(&maps.yr, a.Y, g.n, a.ldy, a.nb, GL0, a.nb);
  make_tmap(&maps.ys, a.Y, g.n, a.ldy, a.nb, GC, a.nb);
  make_tmap(&maps.ir, a.inv_s, g.n, g.ld, 1, GL0, 1);
  make_tmap(&maps.is, a.inv_s, g.n, g.ld, 1, GC, 1);
  if (xsep) make_tmap(&maps.xc, a.X, g.n, a.ldx, a.na, GC, a.na);
  else maps.xc = maps.ys;
  const int W = T8 * 8;
  const size_t smem = (2 * (size_t)L.buf + (size_t)6 * W * GTL) * sizeof(double) + 64;
  if (smem > 227 * 1024) fail(PND_ECONFIG, "stencil Gram tile exceeds shared memory");
  CK(cudaFuncSetAttribute(sgram3_kernel<T8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)smem));
  const int nchunks = (g.n + GC - 1) / GC;
  int grid = sm_count2();
  if (grid > nchunks) grid = nchunks;
  const size_t count = (size_t)g.ns * a.na * a.nb;
  double* part = partial.get(count * grid);
  sgram3_kernel<T8><<<grid, 256, smem, st>>>(maps, a, L, xsep ? 1 : 0, part);
  launched();
  reduce_blocks2<<<(int)((count + 255) / 256), 256, 0, st>>>(part, grid, (int)count, a.out);
  launched();
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess)
      fail(PND_EDEVICE, "cuTensorMapEncodeTiled is unavailable in this driver");
    fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

}  // namespace

void make_tmap(CUtensorMap* map, const double* base, int n, int ld, int cols, int box_cells,
               int box_cols) {
  cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  cuuint32_t box[2] = {(cuuint32_t)box_cells, (cuuint32_t)box_cols};
  cuuint32_t es[2] = {1, 1};
  const CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims,
                                 strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(PND_EDEVICE, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
}

void kstage(const KStageArgs& a, cudaStream_t st) {
  if (a.copy_u) fail(PND_ECONFIG, "kstage copy_u is not supported");
  if (a.r <= 8) kstage3_launch<8>(a, st);
  else if (a.r <= 16) kstage3_launch<16>(a, st);
  else if (a.r <= 24) kstage3_launch<24>(a, st);
  else if (a.r <= 32) kstage3_launch<32>(a, st);
  else if (a.r <= 48) kstage3_launch<48>(a, st);
  else if (a.r <= 64) kstage3_launch<64>(a, st);
  else fail(PND_ECONFIG, "kstage supports at most 64 output columns");
}

void stencil_grams(const GramArgs& a, DBuf& partial, cudaStream_t st) {
  const int w = a.na > a.nb ? a.na : a.nb;
  if (a.geo.ns == 0) return;
  switch ((w + 7) / 8) {
    case 1: sgram3_launch<1>(a, partial, st); break;
    case 2: sgram3_launch<2>(a, partial, st); break;
    case 3: sgram3_launch<3>(a, partial, st); break;
    case 4: sgram3_launch<4>(a, partial, st); break;
    case 5: sgram3_launch<5>(a, partial, st); break;
    case 6: sgram3_launch<6>(a, partial, st); break;
    default: fail(PND_ECONFIG, "stencil Grams support at most 48 columns");
  }
}

}  // namespace pnd
