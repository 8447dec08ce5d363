// LINCOMB: out = [Y1 | Y2] TA - X TB over all cells, with the Grams
//   grams = [X^T out (X.cols x nb) ; out^T out (nb x nb)]
// -- the streaming passes of the block CGS2/SVQB augmentation and the
// truncation rotation U1 = U^ P (dlra.py:26-43, 111-113).
//
// HBM-streaming kernel, warp-specialised like the stencil kernels:
//   producer warp: one cp.async.bulk per input per 64-cell chunk into a ring
//     of staging buffers (the rows of a chunk are contiguous in the
//     cell-major layout; chunks past n read the zero halo rows);
//   8 compute warps: warp w owns m-tile w (8 cells) of the chunk and all
//     NB8 n-tiles of out: FP64 DMMA with A fragments straight from the staged
//     rows (row length = 4 mod 16 doubles: conflict-free) and B fragments
//     from a shared copy of [TA; -TB] in fragment order; out is stored from
//     the accumulators and parked in a double-buffered shared tile, from which
//     the Grams (k = cell) accumulate in registers across all chunks.
// Per-CTA Gram partials are summed in a fixed order (deterministic).
#include "tma.cuh"

namespace pnd {

namespace {

__host__ __device__ constexpr int lpad4(int w) { return ((w + 11) / 16) * 16 + 4; }

constexpr int LCH = 64;                 // cells per chunk
constexpr int LCW = 8;                  // compute warps
constexpr int LTH = 32 * (LCW + 1);     // + producer warp
constexpr int LNSTG_MAX = 4;
constexpr int LZPAD = 16;               // zero doubles after each staged input block

struct LBars {
  uint64_t sfull[LNSTG_MAX], sempty[LNSTG_MAX];
};

// Gram tile index -> (row tile, column tile): X^T out tiles (row tiles < XT)
// first, then the upper triangle (column tile >= row tile - XT) of out^T out
__device__ __forceinline__ void gram_tile(int tile, int XT, int NB8, int& ti, int& tj) {
  if (tile < XT * NB8) {
    ti = tile / NB8;
    tj = tile - ti * NB8;
    return;
  }
  int u = tile - XT * NB8, r = 0;
  while (u >= NB8 - r) {
    u -= NB8 - r;
    ++r;
  }
  ti = XT + r;
  tj = r + u;
}

struct LIn {
  const double* p[3];
  int cols[3], rs[3];
  int off[3];   // smem offset of the staged rows of input q (doubles)
  int ks0[3];   // first k-step of input q
  int nin;      // inputs in use (Y1, then Y2 and/or X)
  int xq;       // index of the X input (-1: none)
  int stage;    // doubles per staging slot
  unsigned bytes;
  int ks;       // total k-steps
  int ident;        // TA = I: out = [Y1 | Y2] - X TB; the number of Y inputs added
  const double* w;  // optional per-cell weight (Gram-only mode: T = diag(w) Y1)
  int woff;         // smem offset of the staged weights
};

// element q of a per-input array of LIn. A runtime index into the kernel's
// by-value parameter struct makes the compiler copy it to local memory
// (LDL in the chunk loops -- 11 % of the stall samples of the CGS passes);
// selects over constant indices keep every field in registers / the
// constant bank
template <class T>
__device__ __forceinline__ T sel3(const T (&a)[3], int q) {
  return q == 0 ? a[0] : q == 1 ? a[1] : a[2];
}

template <int NB8, int TBUF = 2>
__global__ void __launch_bounds__(LTH, NB8 >= 7 ? 1 : 2)
    lincomb_kernel(int n, LIn in, const double* __restrict__ TA, const double* __restrict__ TB,
                   int ny, int nb, NMat out, int nstg, int grams, int copy_y, int skip_tt,
                   double* __restrict__ partial, int) {
  constexpr int tb = TBUF;
  constexpr int TS = lpad4(NB8 * 8);            // out tile row length
  extern __shared__ __align__(128) double sm[];
  double* const sB = sm + nstg * in.stage;      // [ks][NB8][32] fragment order
  double* const sT = sB + in.ks * NB8 * 32;     // tb x [LCH][TS] (tb = 1: 128 wide inputs)
  LBars* bars = reinterpret_cast<LBars*>(sT + tb * LCH * TS);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int xcn = in.xq >= 0 ? sel3(in.cols, in.xq) : 0;
  const int XT = (xcn + 7) / 8;                  // X^T out row tiles
  // Gram tiles: X^T out (XT x NB8), then the upper triangle of the symmetric
  // out^T out (mirrored when stored)
  const int GT = grams ? XT * NB8 + (skip_tt ? 0 : NB8 * (NB8 + 1) / 2) : 0;
  if (tid == 0) {
    for (int b = 0; b < nstg; ++b) {
      mbar_init(&bars->sfull[b], 1);
      mbar_init(&bars->sempty[b], LCW);
    }
    mbar_fence_init();
  }
  // zero pads after each staged block (k-steps past a block's columns read them)
  for (int s = 0; s < nstg; ++s)
    for (int q = 0; q < in.nin; ++q)
      for (int i = tid; i < LZPAD; i += LTH)
        sm[s * in.stage + sel3(in.off, q) + LCH * sel3(in.rs, q) + i] = 0.0;
  // B = [TA; -TB] in fragment order (zero rows past each input's columns)
  for (int i = tid; i < in.ks * NB8 * 32; i += LTH) {
    const int l = i & 31, f = i >> 5, ks = f / NB8, nt = f - ks * NB8;
    int q = 0;
    while (q + 1 < in.nin && ks >= sel3(in.ks0, q + 1)) ++q;
    const int j = 4 * (ks - sel3(in.ks0, q)) + (l & 3), col = nt * 8 + (l >> 2);
    double v = 0.0;
    if (j < sel3(in.cols, q) && col < nb && !copy_y) {
      if (q == in.xq) v = -TB[(size_t)j * nb + col];
      else if (!in.ident) v = TA[(size_t)((q == 0 ? 0 : in.cols[0]) + j) * nb + col];
    }
    sB[i] = v;
  }
  for (int i = tid; i < tb * LCH * TS; i += LTH) sT[i] = 0.0;
  __syncthreads();
  const int nchunks = (n + LCH - 1) / LCH;

  if (warp == LCW) {  // producer
    if (lane == 0) {
      Ring r(nstg);
      for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, r.next()) {
        if (r.k) mbar_wait_sleep(&bars->sempty[r.s], (r.k - 1) & 1);
        mbar_expect_tx(&bars->sfull[r.s], in.bytes);
        const long c0 = (long)chunk * LCH;
        for (int q = 0; q < in.nin; ++q)
          bulk_load(sm + r.s * in.stage + sel3(in.off, q), sel3(in.p, q) + c0 * sel3(in.rs, q),
                    LCH * sel3(in.rs, q) * 8, &bars->sfull[r.s]);
        if (in.w) bulk_load(sm + r.s * in.stage + in.woff, in.w + c0, LCH * 8, &bars->sfull[r.s]);
      }
    }
    return;
  }

  const int m = lane >> 2, kq = lane & 3;
  constexpr int GPW_MAX = (NB8 * NB8 + NB8 * (NB8 + 1) / 2 + LCW - 1) / LCW;
  double gacc[GPW_MAX][2], gacc2[GPW_MAX][2];  // even / odd k-steps: two chains per tile
#pragma unroll
  for (int t = 0; t < GPW_MAX; ++t) gacc[t][0] = gacc[t][1] = gacc2[t][0] = gacc2[t][1] = 0.0;
  // this warp's Gram tiles, resolved once (the triangular index walk was a
  // per-chunk loop of branches)
  int g_ti[GPW_MAX], g_tj[GPW_MAX];
#pragma unroll
  for (int t = 0; t < GPW_MAX; ++t) {
    g_ti[t] = g_tj[t] = -1;
    if (warp + LCW * t < GT) gram_tile(warp + LCW * t, XT, NB8, g_ti[t], g_tj[t]);
  }
  Ring r(nstg);
  int it = 0;
  for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, r.next(), ++it) {
    const long c0 = (long)chunk * LCH;
    mbar_wait(&bars->sfull[r.s], r.k & 1);
    const double* sb = sm + r.s * in.stage;
    double* T = sT + (tb == 2 ? (it & 1) : 0) * LCH * TS;
    if (copy_y) {
      // Gram-only mode: out = Y1 (no contraction), parked for X^T Y1
      const double* y = sb + in.off[0];
      const double* wv = in.w ? sb + in.woff : nullptr;
      const int y2 = in.nin > 1 && in.xq != 1 ? 1 : -1;  // second Y input, if any
      const int c1 = in.cols[0], c2 = y2 >= 0 ? sel3(in.cols, y2) : 0;
      for (int e = lane; e < 8 * NB8 * 8; e += 32) {
        const int i = warp * 8 + e / (NB8 * 8), c = e % (NB8 * 8);
        // rows past n are halo rows (possibly a neighbour slab's): no Gram input
        double v = 0.0;
        if (c0 + i < n) {
          if (c < c1) v = y[i * in.rs[0] + c];
          else if (c - c1 < c2) v = sb[sel3(in.off, y2) + i * sel3(in.rs, y2) + c - c1];
        }
        T[i * TS + c] = wv ? wv[i] * v : v;
      }
      __syncwarp();
    } else {
    // ---- out tile: m-tile `warp`, all n-tiles; two accumulator sets
    double acc[2][NB8][2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int nt = 0; nt < NB8; ++nt) acc[h][nt][0] = acc[h][nt][1] = 0.0;
    if (in.ident) {
      // TA = I: start from the Y1 rows (accumulator layout: row m, columns
      // 2 kq, 2 kq + 1), then Y2's after Y1's columns (two Y blocks)
      const double* y = sb + in.off[0] + (warp * 8 + m) * in.rs[0];
#pragma unroll
      for (int nt = 0; nt < NB8; ++nt) {
        const int col = nt * 8 + 2 * kq;
        if (col < in.cols[0]) acc[0][nt][0] = y[col];
        if (col + 1 < in.cols[0]) acc[0][nt][1] = y[col + 1];
      }
      if (in.ident == 2) {
        const int c1 = in.cols[0], c2 = in.cols[1];
        const double* y2 = sb + in.off[1] + (warp * 8 + m) * in.rs[1];
#pragma unroll
        for (int nt = 0; nt < NB8; ++nt) {
          const int col = nt * 8 + 2 * kq;
          if (col >= c1 && col < c1 + c2) acc[0][nt][0] = y2[col - c1];
          if (col + 1 >= c1 && col + 1 < c1 + c2) acc[0][nt][1] = y2[col + 1 - c1];
        }
      }
    }
    for (int q = in.ident; q < in.nin; ++q) {
      const double* pa = sb + sel3(in.off, q) + (warp * 8 + m) * sel3(in.rs, q) + kq;
      const int k0 = sel3(in.ks0, q), k1 = q + 1 < in.nin ? sel3(in.ks0, q + 1) : in.ks;
      int ks = k0;
      for (; ks + 1 < k1; ks += 2) {
        const double a0 = pa[4 * (ks - k0)], a1 = pa[4 * (ks + 1 - k0)];
#pragma unroll
        for (int nt = 0; nt < NB8; ++nt) {
          dmma884(acc[0][nt][0], acc[0][nt][1], a0, sB[(ks * NB8 + nt) * 32 + lane]);
          dmma884(acc[1][nt][0], acc[1][nt][1], a1, sB[((ks + 1) * NB8 + nt) * 32 + lane]);
        }
      }
      if (ks < k1) {
        const double a0 = pa[4 * (ks - k0)];
#pragma unroll
        for (int nt = 0; nt < NB8; ++nt)
          dmma884(acc[0][nt][0], acc[0][nt][1], a0, sB[(ks * NB8 + nt) * 32 + lane]);
      }
    }
    const int il = warp * 8 + m;
    const long row = c0 + il;
#pragma unroll
    for (int nt = 0; nt < NB8; ++nt) {
      const double v0 = acc[0][nt][0] + acc[1][nt][0], v1 = acc[0][nt][1] + acc[1][nt][1];
      const int col = nt * 8 + 2 * kq;
      // rows past n (halo rows, possibly a neighbour slab's) stay out of the Grams
      *reinterpret_cast<double2*>(T + il * TS + col) =
          row < n ? make_double2(v0, v1) : make_double2(0.0, 0.0);
      if (out.p && row < n) {
        double* o = out.p + row * out.rs + col;
        if (col + 1 < out.rs) *reinterpret_cast<double2*>(o) = make_double2(v0, v1);
        else if (col < out.rs) o[0] = v0;
      }
    }
    }
    if (grams) {
      named_sync(1, 32 * LCW);  // out tile of this chunk complete
      const double* sx = in.xq >= 0 ? sb + sel3(in.off, in.xq) : nullptr;
      const int rsx = in.xq >= 0 ? sel3(in.rs, in.xq) : 0;
#pragma unroll
      for (int t = 0; t < GPW_MAX; ++t) {
        if (g_ti[t] >= 0) {
          const int ti = g_ti[t], tj = g_tj[t];
          const bool xg = ti < XT;
          const double* pa = xg ? sx + (ti * 8 + m) : T + ((ti - XT) * 8 + m);
          const int sa = xg ? rsx : TS;
          const double* pb = T + tj * 8 + m;
          // rows past n: zero staged rows and zero out rows -> no contribution
#pragma unroll
          for (int k0 = 0; k0 < LCH; k0 += 8) {
            dmma884(gacc[t][0], gacc[t][1], pa[(k0 + kq) * sa], pb[(k0 + kq) * TS]);
            dmma884(gacc2[t][0], gacc2[t][1], pa[(k0 + 4 + kq) * sa], pb[(k0 + 4 + kq) * TS]);
          }
        }
      }
      // one out tile: every warp is done reading it before the next chunk's writes
      if constexpr (TBUF == 1) named_sync(1, 32 * LCW);
    }
    warp_arrive(&bars->sempty[r.s]);
  }
  if (grams) {
    double* o = partial + (size_t)blockIdx.x * (xcn + (skip_tt ? 0 : nb)) * nb;
#pragma unroll
    for (int t = 0; t < GPW_MAX; ++t) {
      gacc[t][0] += gacc2[t][0];
      gacc[t][1] += gacc2[t][1];
    }
#pragma unroll
    for (int t = 0; t < GPW_MAX; ++t) {
      const int tile = warp + LCW * t;
      if (tile < GT) {
        int ti, tj;
        gram_tile(tile, XT, NB8, ti, tj);
        const bool xg = ti < XT;
        const int rrow = (xg ? ti : ti - XT) * 8 + m, col = tj * 8 + 2 * kq;
        const int nrow = xg ? xcn : nb;
        const size_t base = xg ? 0 : (size_t)xcn * nb;  // (skip_tt: only X^T out tiles)
        if (rrow < nrow) {
          if (col < nb) o[base + (size_t)rrow * nb + col] = gacc[t][0];
          if (col + 1 < nb) o[base + (size_t)rrow * nb + col + 1] = gacc[t][1];
        }
        if (!xg && ti - XT != tj) {  // mirror the off-diagonal out^T out tile
          if (rrow < nb) {
            if (col < nb) o[base + (size_t)col * nb + rrow] = gacc[t][0];
            if (col + 1 < nb) o[base + (size_t)(col + 1) * nb + rrow] = gacc[t][1];
          }
        }
      }
    }
  }
}

// Per-warp Gram variant (out tiles up to 32 columns): warp w's Gram work is
// its own 8 cells of the chunk -- X^T out and out^T out over those cells, all
// tiles, 2 k-steps each (every tile an independent DMMA chain) -- so no
// CTA-wide barrier per chunk: the out tile goes through a private shared
// tile (only __syncwarp), and in Gram-only mode the staged Y rows are the B
// operand directly. The out^T out A and B fragments are the same loads. Each
// warp writes its own partial; lreduce sums grid x 8 partials in fixed order.
// SYM (Gram-only, X = Y1, Y1 covering every out tile but the last): the
// tiles below the diagonal are mirrors -- not formed (left zero), copied
// after the reduction (mirror_tiles_kernel).
template <int NB8, int NO8 = NB8, bool SYM = false>
__global__ void __launch_bounds__(LTH, 2)
    lincomb_pw_kernel(int n, LIn in, const double* __restrict__ TA, const double* __restrict__ TB,
                      int ny, int nb, NMat out, int nstg, int grams, int copy_y, int skip_tt,
                      double* __restrict__ partial, int) {
  constexpr int TS = lpad4(NO8 * 8);            // out tile row length
  constexpr int NTT = NO8 * (NO8 + 1) / 2;      // upper-triangle out^T out tiles
  extern __shared__ __align__(128) double sm[];
  double* const sB = sm + nstg * in.stage;      // [ks][NO8][32] fragment order
  double* const sT = sB + in.ks * NO8 * 32;     // per warp [8][TS]
  LBars* bars = reinterpret_cast<LBars*>(sT + LCW * 8 * TS);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int xcn = in.xq >= 0 ? sel3(in.cols, in.xq) : 0;
  const int XT = (xcn + 7) / 8;
  if (tid == 0) {
    for (int b = 0; b < nstg; ++b) {
      mbar_init(&bars->sfull[b], 1);
      mbar_init(&bars->sempty[b], LCW);
    }
    mbar_fence_init();
  }
  for (int s = 0; s < nstg; ++s)
    for (int q = 0; q < in.nin; ++q)
      for (int i = tid; i < LZPAD; i += LTH)
        sm[s * in.stage + sel3(in.off, q) + LCH * sel3(in.rs, q) + i] = 0.0;
  for (int i = tid; i < in.ks * NO8 * 32; i += LTH) {
    const int l = i & 31, f = i >> 5, ks = f / NO8, nt = f - ks * NO8;
    int q = 0;
    while (q + 1 < in.nin && ks >= sel3(in.ks0, q + 1)) ++q;
    const int j = 4 * (ks - sel3(in.ks0, q)) + (l & 3), col = nt * 8 + (l >> 2);
    double v = 0.0;
    if (j < sel3(in.cols, q) && col < nb && !copy_y) {
      if (q == in.xq) v = -TB[(size_t)j * nb + col];
      else if (!in.ident) v = TA[(size_t)((q == 0 ? 0 : in.cols[0]) + j) * nb + col];
    }
    sB[i] = v;
  }
  for (int i = tid; i < LCW * 8 * TS; i += LTH) sT[i] = 0.0;
  __syncthreads();
  const int nchunks = (n + LCH - 1) / LCH;

  if (warp == LCW) {  // producer
    if (lane == 0) {
      Ring r(nstg);
      for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, r.next()) {
        if (r.k) mbar_wait_sleep(&bars->sempty[r.s], (r.k - 1) & 1);
        mbar_expect_tx(&bars->sfull[r.s], in.bytes);
        const long c0 = (long)chunk * LCH;
        for (int q = 0; q < in.nin; ++q)
          bulk_load(sm + r.s * in.stage + sel3(in.off, q), sel3(in.p, q) + c0 * sel3(in.rs, q),
                    LCH * sel3(in.rs, q) * 8, &bars->sfull[r.s]);
        if (in.w) bulk_load(sm + r.s * in.stage + in.woff, in.w + c0, LCH * 8, &bars->sfull[r.s]);
      }
    }
    return;
  }

  const int m = lane >> 2, kq = lane & 3;
  double gx[NB8][NO8][2], gt[NTT][2];
#pragma unroll
  for (int ti = 0; ti < NB8; ++ti)
#pragma unroll
    for (int tj = 0; tj < NO8; ++tj) gx[ti][tj][0] = gx[ti][tj][1] = 0.0;
#pragma unroll
  for (int t = 0; t < NTT; ++t) gt[t][0] = gt[t][1] = 0.0;
  double* const T = sT + warp * 8 * TS;
  const int rsx = in.xq >= 0 ? sel3(in.rs, in.xq) : 0;
  // Gram-only second Y input: staged at index 1 unless that is X
  const int y2 = copy_y && in.nin > 1 && in.xq != 1 ? 1 : -1;
  Ring r(nstg);
  for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, r.next()) {
    const long c0 = (long)chunk * LCH;
    const long w0 = c0 + warp * 8;  // this warp's first cell
    mbar_wait(&bars->sfull[r.s], r.k & 1);
    const double* sb = sm + r.s * in.stage;
    const double* sy;
    int rsy;
    if (copy_y) {
      sy = sb + in.off[0] + warp * 8 * in.rs[0];
      rsy = in.rs[0];
    } else {
      // ---- out tile: m-tile `warp`, all n-tiles (NB8 independent chains)
      double acc[NO8][2];
#pragma unroll
      for (int nt = 0; nt < NO8; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
      if (in.ident) {
        // TA = I: start from the Y rows (accumulator layout: row m, columns
        // 2 kq, 2 kq + 1), Y2's after Y1's columns
        const double* y = sb + in.off[0] + (warp * 8 + m) * in.rs[0];
        const int c1 = in.cols[0];
#pragma unroll
        for (int nt = 0; nt < NO8; ++nt) {
          const int col = nt * 8 + 2 * kq;
          if (col < c1) acc[nt][0] = y[col];
          if (col + 1 < c1) acc[nt][1] = y[col + 1];
        }
        if (in.ident == 2) {
          const int c2 = in.cols[1];
          const double* y2 = sb + in.off[1] + (warp * 8 + m) * in.rs[1];
#pragma unroll
          for (int nt = 0; nt < NO8; ++nt) {
            const int col = nt * 8 + 2 * kq;
            if (col >= c1 && col < c1 + c2) acc[nt][0] = y2[col - c1];
            if (col + 1 >= c1 && col + 1 < c1 + c2) acc[nt][1] = y2[col + 1 - c1];
          }
        }
      }
      for (int q = in.ident; q < in.nin; ++q) {
        const double* pa = sb + sel3(in.off, q) + (warp * 8 + m) * sel3(in.rs, q) + kq;
        const int k0 = sel3(in.ks0, q), k1 = q + 1 < in.nin ? sel3(in.ks0, q + 1) : in.ks;
#pragma unroll 2
        for (int ks = k0; ks < k1; ++ks) {
          const double a0 = pa[4 * (ks - k0)];
#pragma unroll
          for (int nt = 0; nt < NO8; ++nt)
            dmma884(acc[nt][0], acc[nt][1], a0, sB[(ks * NO8 + nt) * 32 + lane]);
        }
      }
      const long row = w0 + m;
#pragma unroll
      for (int nt = 0; nt < NO8; ++nt) {
        const double v0 = acc[nt][0], v1 = acc[nt][1];
        const int col = nt * 8 + 2 * kq;
        // rows past n (halo rows, possibly a neighbour slab's) stay out of the Grams
        *reinterpret_cast<double2*>(T + m * TS + col) =
            row < n ? make_double2(v0, v1) : make_double2(0.0, 0.0);
        if (out.p && row < n) {
          double* o = out.p + row * out.rs + col;
          if (col + 1 < out.rs) *reinterpret_cast<double2*>(o) = make_double2(v0, v1);
          else if (col < out.rs) o[0] = v0;
        }
      }
      __syncwarp();
      sy = T;
      rsy = TS;
    }
    if (grams) {
      const double* sx = in.xq >= 0 ? sb + sel3(in.off, in.xq) + warp * 8 * rsx : nullptr;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int cl = 4 * s + kq;  // k index = this lane's cell
        double bf[NO8];
        if (copy_y) {
          // Gram-only: B = diag(w) [Y1 | Y2]; rows past n contribute nothing
          const bool live = w0 + cl < n;
          const double wv = in.w ? sb[in.woff + warp * 8 + cl] : 1.0;
          if (y2 < 0) {
#pragma unroll
            for (int tj = 0; tj < NO8; ++tj)
              bf[tj] = live ? wv * sy[cl * rsy + tj * 8 + m] : 0.0;
          } else {
            const int c1 = in.cols[0];
            const double* s2 = sb + sel3(in.off, y2) + (warp * 8 + cl) * sel3(in.rs, y2);
#pragma unroll
            for (int tj = 0; tj < NO8; ++tj) {
              const int col = tj * 8 + m;
              const double v = col < c1 ? sy[cl * rsy + col]
                               : col - c1 < sel3(in.cols, y2) ? s2[col - c1] : 0.0;
              bf[tj] = live ? wv * v : 0.0;
            }
          }
        } else {
#pragma unroll
          for (int tj = 0; tj < NO8; ++tj) bf[tj] = sy[cl * rsy + tj * 8 + m];
        }
#pragma unroll
        for (int ti = 0; ti < NB8; ++ti) {
          if (ti < XT) {
            const double a = sx[cl * rsx + ti * 8 + m];
#pragma unroll
            for (int tj = 0; tj < NO8; ++tj)
              if (!(SYM && tj < ti)) dmma884(gx[ti][tj][0], gx[ti][tj][1], a, bf[tj]);
          }
        }
        if (!skip_tt) {
          // out^T out: the A fragment of row tile ti is the B fragment of tile ti
#pragma unroll
          for (int ti = 0, t = 0; ti < NO8; ++ti)
#pragma unroll
            for (int tj = ti; tj < NO8; ++tj, ++t) dmma884(gt[t][0], gt[t][1], bf[ti], bf[tj]);
        }
      }
    }
    warp_arrive(&bars->sempty[r.s]);
  }
  if (grams) {
    const size_t count = (size_t)(xcn + (skip_tt ? 0 : nb)) * nb;
    double* o = partial + ((size_t)blockIdx.x * LCW + warp) * count;
    const int col = 2 * kq;
#pragma unroll
    for (int ti = 0; ti < NB8; ++ti) {
      const int rrow = ti * 8 + m;
#pragma unroll
      for (int tj = 0; tj < NO8; ++tj) {
        const int c = tj * 8 + col;
        if (ti < XT && rrow < xcn) {
          if (c < nb) o[(size_t)rrow * nb + c] = gx[ti][tj][0];
          if (c + 1 < nb) o[(size_t)rrow * nb + c + 1] = gx[ti][tj][1];
        }
      }
    }
    if (!skip_tt) {
      double* ot = o + (size_t)xcn * nb;
#pragma unroll
      for (int ti = 0, t = 0; ti < NO8; ++ti)
#pragma unroll
        for (int tj = ti; tj < NO8; ++tj, ++t) {
          const int rrow = ti * 8 + m, c = tj * 8 + col;
          if (rrow < nb) {
            if (c < nb) ot[(size_t)rrow * nb + c] = gt[t][0];
            if (c + 1 < nb) ot[(size_t)rrow * nb + c + 1] = gt[t][1];
          }
          if (ti != tj && rrow < nb) {  // mirror the off-diagonal tile
            if (c < nb) ot[(size_t)c * nb + rrow] = gt[t][0];
            if (c + 1 < nb) ot[(size_t)(c + 1) * nb + rrow] = gt[t][1];
          }
        }
    }
  }
}

// the mirrored tiles of a symmetric Gram-only pass: rows r of X against
// out columns c < r in an earlier tile
__global__ void mirror_tiles_kernel(double* g, int xc, int nb) {
  for (int e = threadIdx.x; e < xc * nb; e += blockDim.x) {
    const int r = e / nb, c = e - r * nb;
    if (c / 8 < r / 8) g[e] = g[(size_t)c * nb + r];
  }
}

// sums nblk partials of `count` entries: 32 consecutive entries per block
// (coalesced), 8 fixed strided subsets of the partials per entry, combined in
// a fixed order (bit-reproducible)
__global__ void __launch_bounds__(256) lreduce(const double* __restrict__ partial, int nblk,
                                               int count, double* __restrict__ out) {
  __shared__ double red[8][33];
  const int i = blockIdx.x * 32 + threadIdx.x;
  double s = 0.0;
  if (i < count)
    for (int b = threadIdx.y; b < nblk; b += 8) s += partial[(size_t)b * count + i];
  red[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && i < count) {
    double t = red[0][threadIdx.x];
#pragma unroll
    for (int y = 1; y < 8; ++y) t += red[y][threadIdx.x];
    out[i] = t;
  }
}

// One output column (the CGS passes of a one-column increment):
//   out = y ta - X tb  (ident: ta = 1), Grams [X^T out ; out^T out]
// The contraction is a 1 x XC dot product per cell -- FP64 FMAs on the CUDA
// cores, not tensor-core tiles padded to 8 output columns. One thread per
// cell, its X row read straight from global memory (the warp's 32 rows are
// one contiguous span, every sector used across the row's loads), two cells
// per thread in flight; Gram partials reduced per warp, summed by lreduce.
// Gram-only (out.p null, TB null): X^T diag(w) y.
constexpr int L1TH = 256;
template <int XCM>
__global__ void __launch_bounds__(L1TH, 2)
    lincomb1_kernel(int n, const double* __restrict__ y, int rsy, const double* __restrict__ X,
                    int rsx, int xc, const double* __restrict__ TA, const double* __restrict__ TB,
                    NMat out, double* __restrict__ partial, const double* __restrict__ w,
                    int gram_only) {
  __shared__ double sc[XCM];
  for (int j = threadIdx.x; j < XCM; j += blockDim.x) sc[j] = TB && j < xc ? TB[j] : 0.0;
  const double ta = TA ? TA[0] : 1.0;
  __syncthreads();
  double gx[XCM], gt = 0.0;
#pragma unroll
  for (int j = 0; j < XCM; ++j) gx[j] = 0.0;
  const long stride = (long)gridDim.x * blockDim.x;
  for (long c = (long)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += stride) {
    const double* xr = X + c * rsx;
    double x[XCM];
#pragma unroll
    for (int j = 0; j < XCM; j += 2) {
      if (j < xc) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(xr + j));
        x[j] = v.x;
        x[j + 1] = v.y;
      } else {
        x[j] = x[j + 1] = 0.0;
      }
    }
    double v = ta * __ldg(y + c * rsy);
#pragma unroll
    for (int j = 0; j < XCM; ++j) v = fma(-sc[j], x[j], v);
    if (out.p) *reinterpret_cast<double2*>(out.p + c * out.rs) = make_double2(v, 0.0);
    if (partial) {
      const double vg = w ? v * __ldg(w + c) : v;
#pragma unroll
      for (int j = 0; j < XCM; ++j) gx[j] = fma(x[j], vg, gx[j]);
      gt = fma(v, v, gt);
    }
  }
  if (!partial) return;
  const int lane = threadIdx.x & 31;
  double* o = partial + ((size_t)blockIdx.x * (L1TH / 32) + (threadIdx.x >> 5)) *
                             (xc + (gram_only ? 0 : 1));
#pragma unroll
  for (int j = 0; j < XCM; ++j) {
    double t = gx[j];
    for (int s = 16; s > 0; s >>= 1) t += __shfl_xor_sync(0xffffffffu, t, s);
    if (lane == 0 && j < xc) o[j] = t;
  }
  if (gram_only) return;
  for (int s = 16; s > 0; s >>= 1) gt += __shfl_xor_sync(0xffffffffu, gt, s);
  if (lane == 0) o[xc] = gt;
}

template <int XCM>
void lincomb1_launch(const Geom& g, NMat Y1, NMat X, const double* TA, const double* TB, NMat out,
                     double* grams, DBuf& partial, cudaStream_t st, const double* w = nullptr) {
  const bool gram_only = out.p == nullptr;
  auto kern = lincomb1_kernel<XCM>;
  const int nblk = occupancy_cached((const void*)kern, L1TH, 0);
  int grid = sm_count() * nblk;
  const int need = (g.n + L1TH - 1) / L1TH;
  if (grid > need) grid = need;
  const size_t count = (size_t)X.cols + (gram_only ? 0 : 1);
  const int nparts = grid * (L1TH / 32);
  double* part = grams ? partial.get(count * nparts) : nullptr;
  kern<<<grid, L1TH, 0, st>>>(g.n, Y1.p, Y1.rs, X.p, X.rs, X.cols, TA, TB, out, part, w,
                              gram_only ? 1 : 0);
  launched();
  if (grams) {
    lreduce<<<(int)((count + 31) / 32), dim3(32, 8), 0, st>>>(part, nparts, (int)count, grams);
    launched();
    comm_allreduce(g, grams, count, st);
  }
}

template <int NB8>
void lincomb_launch(const Geom& g, NMat Y1, NMat Y2, NMat X, const double* TA, const double* TB,
                    NMat out, double* grams, DBuf& partial, cudaStream_t st, bool gram_only,
                    const double* weight = nullptr) {
  LIn in{};
  const NMat ms[3] = {Y1, Y2, X};
  int o = 0, ks = 0;
  // Gram-only X^T diag(w) X: the one matrix is staged once and read as both operands
  const bool same = gram_only && X.p == Y1.p && X.rs == Y1.rs && X.cols == Y1.cols;
  for (int q = 0; q < 3; ++q) {
    if (!ms[q].p || ms[q].cols <= 0) continue;
    if (q == 2 && same) continue;
    const int i = in.nin++;
    in.p[i] = ms[q].p;
    in.cols[i] = ms[q].cols;
    in.rs[i] = ms[q].rs;
    in.off[i] = o;
    in.ks0[i] = ks;
    if (q == 2) in.xq = i;
    o += ((LCH * ms[q].rs + LZPAD) + 15) / 16 * 16;
    ks += (ms[q].cols + 3) / 4;
    in.bytes += LCH * ms[q].rs * 8;
  }
  if (!X.p || X.cols <= 0) in.xq = -1;
  if (same) in.xq = 0;
  in.ident = (!gram_only && TA == nullptr) ? (Y2.p && Y2.cols > 0 ? 2 : 1) : 0;
  if (in.ident && Y1.cols + (Y2.p ? Y2.cols : 0) != out.cols)
    fail(PND_ECONFIG, "lincomb: TA = I needs out = [Y1 | Y2] - X TB with matching columns");
  if (weight) {
    in.w = weight;
    in.woff = o;
    o += LCH;
    in.bytes += LCH * 8;
  }
  in.stage = o;
  in.ks = ks;
  const int ny = Y1.cols + (Y2.p ? Y2.cols : 0);
  const int nb = out.cols;
  constexpr int TS = lpad4(NB8 * 8);
  // per-warp Grams (lincomb_pw_kernel) while the registers allow
  constexpr bool PWOK = NB8 <= 3;
  // (Gram-only passes and the CGS passes' contraction + Grams: 0.4 operand
  // loads per Gram DMMA instead of 2 and no CTA barrier per chunk -- the
  // barrier was 7.7 % of the CTA variant's stall samples; at 256^3 r = 20 the
  // two augmentations take 9.05 instead of 9.88 ms. The rotation's U^T U
  // alone (no X) stays on the CTA variant, which is faster there.)
  // one output tile against a wider X (the CGS passes of a one-column
  // increment): the per-warp kernel with its out tile, B fragments and Grams
  // sized for 8 columns, with or without Grams
  const bool narrow = !gram_only && NB8 > 1 && nb <= 8 && X.p != nullptr;
  const bool PW = narrow || (PWOK && (gram_only || (grams != nullptr && X.p != nullptr &&
                                                   !getenv("PND_LINCOMB_CTA_GRAMS"))));
  const int no8 = narrow ? 1 : NB8;
  int tb = 2;  // out-tile buffers
  size_t tile = PW ? (size_t)LCW * 8 * (narrow ? lpad4(8) : TS) : 2 * (size_t)LCH * TS;
  size_t fixed = ((size_t)ks * no8 * 32 + tile) * sizeof(double) + sizeof(LBars);
  // two CTAs per SM: keep the whole CTA under ~113 KB
  const size_t cap = 113 * 1024;
  int nstg = 0;
  while (nstg < LNSTG_MAX && fixed + (size_t)(nstg + 1) * in.stage * sizeof(double) <= cap)
    ++nstg;
  if (nstg < 2) {
    nstg = 2;
    if (!PW && fixed + 2 * (size_t)in.stage * sizeof(double) > (size_t)kMaxDynSmem) {
      // 128 input columns x 64 outputs: one out tile (a barrier per chunk)
      tb = 1;
      tile = (size_t)LCH * TS;
      fixed = ((size_t)ks * NB8 * 32 + tile) * sizeof(double) + sizeof(LBars);
    }
    if (fixed + 2 * (size_t)in.stage * sizeof(double) > (size_t)kMaxDynSmem)
      fail(PND_ECONFIG, "lincomb tile exceeds shared memory");
  }
  const size_t smem = fixed + (size_t)nstg * in.stage * sizeof(double);
  auto kern = lincomb_kernel<NB8>;
  if (tb == 1) kern = lincomb_kernel<NB8, 1>;
  // symmetric Gram-only pass: every out tile below the diagonal lies in Y1
  // (large grids: on small ones the mirror launch costs more than it saves)
  const bool sym = PWOK && gram_only && same && NB8 > 1 && Y1.cols >= 8 * (NB8 - 1) &&
                   (g.n >= (1 << 18) || getenv("PND_LINCOMB_SYM")) &&
                   !getenv("PND_LINCOMB_NOSYM");
  if (narrow) kern = lincomb_pw_kernel<NB8, 1>;
  if constexpr (PWOK) {
    if (PW && !narrow) kern = sym ? lincomb_pw_kernel<NB8, NB8, true> : lincomb_pw_kernel<NB8>;
  }
  allow_max_smem(kern);
  const int nblk = occupancy_cached((const void*)kern, LTH, smem);
  const int nchunks = (g.n + LCH - 1) / LCH;
  int grid = sm_count() * nblk;
  if (grid > nchunks) grid = nchunks;
  const int xcn = X.p ? X.cols : 0;
  const size_t count = (size_t)(xcn + (gram_only ? 0 : nb)) * nb;
  const int nparts = PW ? grid * LCW : grid;  // per-warp or per-CTA partials
  double* part = grams ? partial.get(count * nparts) : nullptr;
  kern<<<grid, LTH, smem, st>>>(g.n, in, TA, TB, ny, nb, out, nstg, grams ? 1 : 0,
                                gram_only ? 1 : 0, gram_only ? 1 : 0, part, tb);
  launched();
  if (grams) {
    lreduce<<<(int)((count + 31) / 32), dim3(32, 8), 0, st>>>(part, nparts, (int)count, grams);
    launched();
    if (sym) {
      mirror_tiles_kernel<<<1, 256, 0, st>>>(grams, xcn, nb);
      launched();
    }
    comm_allreduce(g, grams, count, st);
  }
}

}  // namespace

void lincomb(const Geom& g, NMat Y1, NMat Y2, NMat X, const double* TA, const double* TB,
             NMat out, double* grams, DBuf& partial, cudaStream_t st) {
  const int w = out.cols > (X.p ? X.cols : 0) ? out.cols : X.cols;
  const int K = Y1.cols + (Y2.p ? Y2.cols : 0) + (X.p ? X.cols : 0);
  if (K > 128) fail(PND_ECONFIG, "lincomb supports at most 128 input columns");
  if (grams && X.p && X.cols > 64) fail(PND_ECONFIG, "lincomb Grams support at most 64 X columns");
  if (out.cols == 1 && out.p && Y1.cols == 1 && !(Y2.p && Y2.cols > 0) && X.p && X.cols > 0 &&
      X.cols <= 32 && X.rs % 2 == 0 && out.rs == 2 && !getenv("PND_LINCOMB1_OFF")) {
    if (X.cols <= 8) return lincomb1_launch<8>(g, Y1, X, TA, TB, out, grams, partial, st);
    if (X.cols <= 16) return lincomb1_launch<16>(g, Y1, X, TA, TB, out, grams, partial, st);
    if (X.cols <= 24) return lincomb1_launch<24>(g, Y1, X, TA, TB, out, grams, partial, st);
    return lincomb1_launch<32>(g, Y1, X, TA, TB, out, grams, partial, st);
  }
  switch ((w + 7) / 8) {
    case 1: lincomb_launch<1>(g, Y1, Y2, X, TA, TB, out, grams, partial, st, false); break;
    case 2: lincomb_launch<2>(g, Y1, Y2, X, TA, TB, out, grams, partial, st, false); break;
    case 3: lincomb_launch<3>(g, Y1, Y2, X, TA, TB, out, grams, partial, st, false); break;
    case 4: lincomb_launch<4>(g, Y1, Y2, X, TA, TB, out, grams, partial, st, false); break;
    case 5: lincomb_launch<5>(g, Y1, Y2, X, TA, TB, out, grams, partial, st, false); break;
    case 6: lincomb_launch<6>(g, Y1, Y2, X, TA, TB, out, grams, partial, st, false); break;
    case 7:
    case 8: lincomb_launch<8>(g, Y1, Y2, X, TA, TB, out, grams, partial, st, false); break;
    default: fail(PND_ECONFIG, "lincomb supports at most 64 output columns");
  }
}

void gram_xy2(const Geom& g, NMat X, NMat Y1, NMat Y2, double* out, DBuf& partial,
              cudaStream_t st, const double* weight) {
  // out = X^T diag(weight) [Y1 | Y2]: the Gram-only pass with two staged Y inputs
  const int ny = Y1.cols + Y2.cols;
  const int w = ny > X.cols ? ny : X.cols;
  if (w > 64) fail(PND_ECONFIG, "Grams support at most 64 columns");
  const NMat o{nullptr, 0, ny};
  switch ((w + 7) / 8) {
    case 1: lincomb_launch<1>(g, Y1, Y2, X, nullptr, nullptr, o, out, partial, st, true, weight); break;
    case 2: lincomb_launch<2>(g, Y1, Y2, X, nullptr, nullptr, o, out, partial, st, true, weight); break;
    case 3: lincomb_launch<3>(g, Y1, Y2, X, nullptr, nullptr, o, out, partial, st, true, weight); break;
    case 4: lincomb_launch<4>(g, Y1, Y2, X, nullptr, nullptr, o, out, partial, st, true, weight); break;
    case 5: lincomb_launch<5>(g, Y1, Y2, X, nullptr, nullptr, o, out, partial, st, true, weight); break;
    case 6: lincomb_launch<6>(g, Y1, Y2, X, nullptr, nullptr, o, out, partial, st, true, weight); break;
    default: lincomb_launch<8>(g, Y1, Y2, X, nullptr, nullptr, o, out, partial, st, true, weight); break;
  }
}

void gram_xy(const Geom& g, NMat X, NMat Y, double* out, DBuf& partial, cudaStream_t st,
             const double* weight) {
  // out = X^T diag(weight) Y (X.cols x Y.cols) in one streaming pass: the
  // LINCOMB kernel with out = diag(weight) Y parked in shared memory and only
  // the X^T out Grams formed
  const int w = Y.cols > X.cols ? Y.cols : X.cols;
  if (w > 64) fail(PND_ECONFIG, "Grams support at most 64 columns");
  const NMat none{}, o{nullptr, 0, Y.cols};
  if (Y.cols == 1 && X.cols <= 8 && X.rs % 2 == 0 && !getenv("PND_LINCOMB1_OFF"))
    return lincomb1_launch<8>(g, Y, X, nullptr, nullptr, o, out, partial, st, weight);
  switch ((w + 7) / 8) {
    case 1: lincomb_launch<1>(g, Y, none, X, nullptr, nullptr, o, out, partial, st, true, weight); break;
    case 2: lincomb_launch<2>(g, Y, none, X, nullptr, nullptr, o, out, partial, st, true, weight); break;
    case 3: lincomb_launch<3>(g, Y, none, X, nullptr, nullptr, o, out, partial, st, true, weight); break;
    case 4: lincomb_launch<4>(g, Y, none, X, nullptr, nullptr, o, out, partial, st, true, weight); break;
    case 5: lincomb_launch<5>(g, Y, none, X, nullptr, nullptr, o, out, partial, st, true, weight); break;
    case 6: lincomb_launch<6>(g, Y, none, X, nullptr, nullptr, o, out, partial, st, true, weight); break;
    default: lincomb_launch<8>(g, Y, none, X, nullptr, nullptr, o, out, partial, st, true, weight); break;
  }
}

}  // namespace pnd
