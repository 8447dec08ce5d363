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
#include <cstdlib>

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
  int cpp, nz;     // chunk order: cpp > 0 -> z-fastest (cpp chunks per z-plane)
  int plus_only;   // D+ stencils only: the +1 / +2 segments of the y and z axes are not staged
  int no_isp;      // the [1/S, 0] rows are not staged (inputs already scaled by 1/S)
  // the planes a launch covers (cpp > 0): zlo .. zlo + nzr - 1, or with zb the
  // four boundary planes 0, 1, nz - 2, nz - 1; nchunks = nzr * cpp (all: nz planes)
  int zlo, nzr, zb, nchunks;
};

// first cell of the p-th processed chunk. With whole chunks per z-plane the
// chunks are visited z-fastest: the CTAs of one grid-stride step then cover
// consecutive planes of the same (x, y) run, so the +-1/+-2 plane halo rows are
// read by neighbouring CTAs at the same time (L2 hits) instead of
// 2 planes apart in time (which falls out of L2 at 256^3).
__device__ __forceinline__ int chunk_cell(const Seg& S, int p, int ch) {
  if (S.cpp == 0) return p * ch;
  const int zi = p % S.nzr, r = p / S.nzr;
  const int zq = S.zb ? (zi < 2 ? zi : S.nz - 4 + zi) : S.zlo + zi;
  return (zq * S.cpp + r) * ch;
}

template <int CH>
Seg make_seg(const Geom& g, const NMat* in, int nin, const NMat* centre, bool plus_only = false,
             bool no_isp = false) {
  Seg s{};
  s.plus_only = plus_only ? 1 : 0;
  s.no_isp = no_isp ? 1 : 0;
  s.nbox = 1;
  s.off[0] = -2;
  const int nxy = g.nx * g.ny;
  for (int ai = 1; ai < g.na; ++ai) {
    const int st = g.axis[ai] == 1 ? g.nx : nxy;
    const int ds[4] = {-2, -1, 1, 2};
    for (int q = 0; q < 4; ++q) s.off[s.nbox++] = ds[q] * st;
  }
  s.nrows = CH + 4 + (plus_only ? (s.nbox - 1) / 2 : s.nbox - 1) * CH;
  int o = 0;
  unsigned bytes = 0;
  // staged rows per input: all segments, or without the +1 / +2 ones (plus_only)
  const int srows = s.nrows;
  for (int k = 0; k < 2; ++k) {
    s.xoff[k] = o;
    if (k < nin) {
      o += up16(s.nrows * in[k].rs);
      bytes += srows * in[k].rs * 8;
    }
  }
  s.ioff = o;
  if (!no_isp) {
    o += up16(2 * s.nrows);
    bytes += 2 * srows * 8;
  }
  s.coff = -1;
  if (centre) {
    s.coff = o;
    o += up16(CH * centre->rs);
    bytes += CH * centre->rs * 8;
  }
  s.total = up16(o);
  s.bytes = bytes;
  s.cpp = (nxy % CH == 0 && g.nz > 1) ? nxy / CH : 0;
  s.nz = g.nz;
  s.zlo = 0;
  s.nzr = g.nz;
  s.zb = 0;
  s.nchunks = (g.n + CH - 1) / CH;
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
    // D+ only (the one-material S-Grams): the +1 / +2 neighbours are never
    // read, and the staged segments are packed back to back
    if (S.plus_only && q > 0 && ((q - 1) & 3) >= 2) continue;
    const int rows = q == 0 ? CH + 4 : CH;
    const long row = (long)c0 + S.off[q];
    const int drow = box_row<CH>(S.plus_only && q > 0 ? 1 + 2 * ((q - 1) >> 2) + ((q - 1) & 3) : q);
    bulk_load(dst + S.xoff[0] + drow * a.rs, a.p + row * a.rs, rows * a.rs * 8, bar);
    if (nin > 1) bulk_load(dst + S.xoff[1] + drow * b.rs, b.p + row * b.rs, rows * b.rs * 8, bar);
    if (!S.no_isp) bulk_load(dst + S.ioff + 2 * drow, isp + 2 * row, rows * 16, bar);
  }
  if (S.coff >= 0) bulk_load(dst + S.coff, c.p + (long)c0 * c.rs, CH * c.rs * 8, bar);
}

// Per-thread stencil context of one cell for one chunk: the staged-row
// pointers of its 1 + 4 NA stencil points (centre, then d = -2,-1,+1,+2 per
// axis; column offset folded in), 1/S at those points, and the boundary class.
// apply<FAST>() forms the 2 NA values D_s S^-1 x of column (col0 + off):
// FAST = every cell of the warp is >= 2 cells from every face (branch-free
// interior formula); otherwise the boundary closures of spatial.py:81-118.
// CMP: the compact plus-only staging (only the -2 / -1 segments of the y and
// z axes are staged, back to back); the +1 / +2 points then alias the -2 row
// and are never read (D+ only)
template <int CH, int NA, bool PRE = false, bool CMP = false>
struct Ctx {
  static constexpr int NP = 1 + 4 * NA;
  const double* xr[NP];
  double is[NP];
  int idx[NA], len[NA];
  bool inner;

  __device__ __forceinline__ static int row_of(int p, int i) {
    if (p == 0) return i + 2;
    const int ai = (p - 1) >> 2, q = (p - 1) & 3;
    if (ai == 0) return i + (q < 2 ? q : q + 1);
    if (CMP) return box_row<CH>(1 + 2 * (ai - 1) + (q < 2 ? q : 0)) + i;
    return box_row<CH>(1 + 4 * (ai - 1) + q) + i;
  }

  __device__ __forceinline__ void init(const Geom& g, int c, int i, const double* I) {
    // cell -> (i, j, k) by exact integer reciprocals (the double-product
    // version's int->double conversions were the formers' top stall)
    const int nxy = g.nx * g.ny;
    const int ck = g.mnxy ? (int)__umul64hi((unsigned long long)c, g.mnxy) : c;
    const int rem = c - ck * nxy;
    const int cj = g.mnx ? (int)__umul64hi((unsigned long long)rem, g.mnx) : rem;
    const int ci = rem - cj * g.nx;
    inner = true;
    // z in global planes (a slab's faces are interior unless they are the grid's)
    const int gk = ck + g.z0, gnz = g.nzg > 0 ? g.nzg : g.nz;
#pragma unroll
    for (int ai = 0; ai < NA; ++ai) {
      const int axis = g.axis[ai];
      idx[ai] = axis == 0 ? ci : axis == 1 ? cj : gk;
      len[ai] = axis == 0 ? g.nx : axis == 1 ? g.ny : gnz;
      inner = inner && idx[ai] >= 2 && idx[ai] <= len[ai] - 3;
    }
    if (!PRE) {
#pragma unroll
      for (int p = 0; p < NP; ++p) is[p] = I[2 * row_of(p, i)];
    }
  }

  // rows of input X (row length rs), column offset col0 folded in
  __device__ __forceinline__ void rows(const double* X, int rs, int i, int col0) {
#pragma unroll
    for (int p = 0; p < NP; ++p) xr[p] = X + row_of(p, i) * rs + col0;
  }

  // The 1/(2h) of the second-order upwind differences is folded into the
  // operand each stencil is contracted with (bcat_kernel: M_s; reduce_parts:
  // G_s), so a feature costs 2 FP64 ops (+ one shared 3 x centre): the
  // formers share the FP64 pipe with the contraction warps' DMMAs. The
  // first-order boundary closures (1/h = 2 x 1/(2h)) carry the exact factor 2.
  template <bool FAST>
  __device__ __forceinline__ void apply(const Geom& g, int off, double* t) const {
    // PRE: the staged rows already hold S^-1 x
    const double fc = PRE ? xr[0][off] : xr[0][off] * is[0];
    const double c3 = 3.0 * fc;
#pragma unroll
    for (int ai = 0; ai < NA; ++ai) {
      const double f0 = PRE ? xr[1 + 4 * ai][off] : xr[1 + 4 * ai][off] * is[1 + 4 * ai];
      const double f1 = PRE ? xr[2 + 4 * ai][off] : xr[2 + 4 * ai][off] * is[2 + 4 * ai];
      const double f3 = PRE ? xr[3 + 4 * ai][off] : xr[3 + 4 * ai][off] * is[3 + 4 * ai];
      const double f4 = PRE ? xr[4 + 4 * ai][off] : xr[4 + 4 * ai][off] * is[4 + 4 * ai];
      double tp, tm;
      if (FAST) {
        tp = fma(-4.0, f1, c3) + f0;
        tm = fma(4.0, f3, -c3) - f4;
      } else {
        const int id = idx[ai], ln = len[ai];
        if (id >= 2) tp = fma(-4.0, f1, c3) + f0;
        else if (id == 1) tp = 2.0 * (fc - f1);
        else tp = 2.0 * fc;
        if (id <= ln - 3) tm = fma(4.0, f3, -c3) - f4;
        else if (id == ln - 2) tm = 2.0 * (f3 - fc);
        else tm = -2.0 * fc;
      }
      t[2 * ai] = tp;
      t[2 * ai + 1] = tm;
    }
  }
};

// 1/(2h) of the axis of each stencil s (= 2 ai + {0: D+, 1: D-})
struct StScale {
  double v[6];
};

StScale stencil_scale(const Geom& g) {
  StScale sc{};
  for (int s = 0; s < 2 * g.na && s < 6; ++s) sc.v[s] = g.i2h[g.axis[s / 2]];
  return sc;
}

template <class Kern>
int resident(Kern k, int threads, size_t smem) {
  return occupancy_cached((const void*)k, threads, smem);
}

// ============================================================ pipeline roles
// Both stencil kernels are warp-specialized, one persistent CTA per SM:
//   1 producer warp: lane 0 issues the bulk copies of each chunk into a ring
//     of NSTG staging buffers (sfull[s] completes on the bytes, sempty[s] on
//     the 8 former-warp releases);
//   8 "former" warps: wait for chunk k's staging, write its stencil features
//     F[f] (f = k & 1, double-buffered), release the staging buffer;
//   contraction warps: DMMA over F[f] while the formers work on k+1.
// Warps signal with one elected lane after __syncwarp; there is no CTA-wide
// barrier after the prologue.
constexpr int FORMW = 8;             // former warps
constexpr int CONW = 8;              // kstage contraction warps (m-tile x k-half)
constexpr int PTH = 32 * (FORMW + CONW + 1);
// sgram contraction warps: 8 (two per SM sub-partition, so the DMMA work is
// even across the four) while the accumulators fit the 120-register cap of
// 17 warps; 7 for the widest tiles
__host__ __device__ constexpr int gconw(int t8) { return t8 <= 5 ? 8 : 7; }
__host__ __device__ constexpr int gpth(int t8) { return 32 * (FORMW + gconw(t8) + 1); }
constexpr int NSTG_MAX = 4;

struct PipeBars {
  uint64_t sfull[NSTG_MAX], sempty[NSTG_MAX], ffull[2], fempty[2];
};

// staging ring depth that fits next to `fixed` bytes of shared memory
int stages_for(size_t fixed, int stage_doubles) {
  const size_t cap = 227 * 1024;
  int n = 0;
  while (n < NSTG_MAX && fixed + (size_t)(n + 1) * stage_doubles * sizeof(double) <= cap) ++n;
  return n;
}

__device__ __forceinline__ void pipe_init(PipeBars* pb, int nstg, int conw) {
  if (threadIdx.x == 0) {
    for (int b = 0; b < nstg; ++b) {
      mbar_init(&pb->sfull[b], 1);
      mbar_init(&pb->sempty[b], FORMW);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&pb->ffull[b], FORMW);
      mbar_init(&pb->fempty[b], conw);
    }
    mbar_fence_init();
  }
}


// ===================================================================== kstage
// out = [D_0 S^-1 X, ..., D_ns-1 S^-1 X | U0] . Bcat, Bcat = [M_0; ...; M_ns-1; S0]
// (zero-padded to K4 x RB). Chunk = 32 cells; F[b] = [K4][36] k-major.
// Former lane = (cell 4w + (lane & 3), column (lane >> 2) + 8t): conflict-free
// reads of the staged rows and writes of F. Contraction warp m owns m-tile m,
// all NT n-tiles, k-steps dealt round-robin to four accumulator sets (4 NT
// independent DMMA chains); B fragments come from a shared-memory copy of
// Bcat in fragment order.
// KHR > 0: the register-rebalanced variant. The CTA has 20 warps = 5
// warpgroups (formers, formers, contraction, contraction, producer + 3 idle
// warps); `setmaxnreg` moves registers from the producer and former
// warpgroups to the contraction ones, which then hold their k-half of the B
// fragments ([M; S0] is the same for every chunk) in registers for the whole
// kernel: per chunk a contraction warp loads only its KHR A fragments instead
// of KHR (1 + NT) fragments -- the B stream was the largest shared-memory
// stream of the kernel.
// setmaxnreg moves registers within the CTA's launch allocation (96 per
// thread x 640 = 61,440): 2 x 128 x 80 + 2 x 128 x 144 + 128 x 24 = 60,416
constexpr int RPTH = 32 * 20;
constexpr int REG_FORM = 80, REG_CON = 144, REG_PROD = 24;
static_assert(2 * 128 * REG_FORM + 2 * 128 * REG_CON + 128 * REG_PROD <= RPTH * 96,
              "register budget exceeds the CTA's launch allocation");
template <int N>
__device__ __forceinline__ void reg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void reg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(N));
}

template <int NA, int RB, bool PRE, int KC, int KHR = 0>
__global__ void __launch_bounds__(KHR > 0 ? RPTH : PTH, 1)
    kstage_kernel(Geom g, NMat X, NMat U0, NMat out, const double* __restrict__ Bcat, int K,
                  int K4, Seg S, int nstg, const double* __restrict__ isp, int oscale, int dbg) {
  constexpr int NTH = KHR > 0 ? RPTH : PTH;
  constexpr int NS = 2 * NA;
  constexpr int NT = RB / 8;
  constexpr int KCS = pad4(KC);       // feature tile row length (k-major: k = feature)
  constexpr int MT = KC / 8;          // m-tiles per chunk
  constexpr int CG = KC / 4;          // former cell groups (4 cells each)
  constexpr int JS = 8 * (FORMW / CG);  // former column stride
  constexpr int KSPLIT = CONW / MT;   // contraction k-parts
  extern __shared__ __align__(128) double sm[];
  // staging slot s: sm + s S.total; feature buffer f: F0 + f K4 KCS
  double* const F0 = sm + nstg * S.total;
  // Bcat in DMMA B-fragment order: sB[(ks NT + nt) 32 + lane] =
  // Bcat[4 ks + (lane & 3)][8 nt + (lane >> 2)] (one contiguous 256-byte load each)
  // (KHR: the B fragments live in the contraction warps' registers, loaded
  // from global memory once; no shared copy -- the room goes to a deeper ring)
  double* const sB = F0 + 2 * K4 * KCS;
  double* const red = sB + (KHR > 0 ? 0 : K4 * RB);  // [k-part - 1][MT][NT][64] partials
  PipeBars* pb = reinterpret_cast<PipeBars*>(red + (KSPLIT - 1) * MT * NT * 64);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int xc = X.cols, ra = U0.p ? U0.cols : 0;
  pipe_init(pb, nstg, CONW);
  for (int i = tid; i < (K4 - K) * KCS; i += NTH) {
    F0[K * KCS + i] = 0.0;
    F0[K4 * KCS + K * KCS + i] = 0.0;
  }
  if constexpr (KHR == 0) {
    for (int i = tid; i < K4 * RB; i += NTH) {
      const int l = i & 31, f = i >> 5, ks = f / NT, nt = f - ks * NT;
      sB[i] = Bcat[(4 * ks + (l & 3)) * RB + 8 * nt + (l >> 2)];
    }
  }
  __syncthreads();
  const bool sepc = S.coff >= 0;
  const int nchunks = S.nchunks;

  if (warp >= FORMW + CONW) {
    if constexpr (KHR > 0) reg_dec<REG_PROD>();
    if (warp == FORMW + CONW && lane == 0) {
      Ring r(nstg);
      for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, r.next()) {
        if (r.k) mbar_wait(&pb->sempty[r.s], (r.k - 1) & 1);
        issue_seg<KC, NA>(S, sm + r.s * S.total, &pb->sfull[r.s], chunk_cell(S, chunk, KC), X, X,
                          1, isp, U0);
      }
    }
  } else if (warp < FORMW) {
    if constexpr (KHR > 0) reg_dec<REG_FORM>();
    // lane = (cell 4 (w % CG) + (lane & 3), column (lane >> 2) + 8 (w / CG) + JS t)
    const int ci = 4 * (warp % CG) + (lane & 3), cj = (lane >> 2) + 8 * (warp / CG);
    Ring r(nstg);
    int it = 0;
    for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, ++it, r.next()) {
      const int f = it & 1, u = it >> 1;
      const int c0 = chunk_cell(S, chunk, KC);
      mbar_wait(&pb->sfull[r.s], r.k & 1);
      if (u >= 1) mbar_wait(&pb->fempty[f], (u - 1) & 1);
      const double* sb = sm + r.s * S.total;
      const double* Xs = sb + S.xoff[0];
      double* Fb = F0 + f * K4 * KCS;
      double* base = Fb + NS * xc * KCS;
      if (dbg & 1) {  // profiling (PND_KSTAGE_DBG): formers skip the features
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&pb->ffull[f]);
          mbar_arrive(&pb->sempty[r.s]);
        }
        continue;
      }
      // base rows = unscaled centre rows (rows past n are zero halo rows; their
      // results are not stored)
      if (sepc) {
        for (int j = cj; j < ra; j += JS) base[j * KCS + ci] = sb[S.coff + ci * U0.rs + j];
      } else if (ra > 0 && U0.p != X.p) {
        // KHR: U0's centre rows are not staged (the ring is deeper instead)
        const double* u0r = U0.p + (long)(c0 + ci) * U0.rs;
        for (int j = cj; j < ra; j += JS) base[j * KCS + ci] = __ldg(u0r + j);
      } else {
        for (int j = cj; j < ra; j += JS) base[j * KCS + ci] = Xs[(ci + 2) * X.rs + j];
      }
      Ctx<KC, NA, PRE> cx;
      cx.init(g, c0 + ci, ci, sb + S.ioff);
      cx.rows(Xs, X.rs, ci, cj);
      const bool fast = __all_sync(0xffffffffu, cx.inner);
#pragma unroll
      for (int t = 0; t < (RB + JS - 1) / JS; ++t) {
        const int j = cj + JS * t;
        if (j < xc) {
          double v[NS];
          if (fast) cx.template apply<true>(g, JS * t, v);
          else cx.template apply<false>(g, JS * t, v);
#pragma unroll
          for (int s = 0; s < NS; ++s) Fb[(s * xc + j) * KCS + ci] = v[s];
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&pb->ffull[f]);
        mbar_arrive(&pb->sempty[r.s]);
      }
    }
  } else {
    // contraction warp q: m-tile q % MT, k-part q / MT (two warps per SM
    // sub-partition, so one issues DMMAs while the other waits on its loads);
    // the k-parts' partials go through the consumed feature buffer
    if constexpr (KHR > 0) reg_inc<REG_CON>();
    const int q = warp - FORMW, mt = q % MT, kh = q / MT;
    const int nks = K4 / 4;
    const int ks0 = (nks * kh) / KSPLIT, ks1 = (nks * (kh + 1)) / KSPLIT;
    const double* pb0 = sB + lane;
    constexpr int KHA = KHR > 0 ? KHR : 1;
    double breg[KHA][NT];
    if constexpr (KHR > 0) {
#pragma unroll
      for (int i = 0; i < KHR; ++i)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          breg[i][nt] = __ldg(Bcat + (4 * (ks0 + i) + (lane & 3)) * RB + 8 * nt + (lane >> 2));
    }
    int it = 0;
    for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, ++it) {
      const int b = it & 1, u = it >> 1;
      const int c0 = chunk_cell(S, chunk, KC);
      // the output row's 1/S, fetched before the wait (its latency was an
      // epilogue stall)
      const int prow = c0 + mt * 8 + (lane >> 2);
      const double is_pre = (!kh && oscale && prow < g.n) ? __ldg(isp + 2 * (long)prow) : 1.0;
      mbar_wait(&pb->ffull[b], u & 1);
      double acc[2][NT][2];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[h][nt][0] = acc[h][nt][1] = 0.0;
      double* Fb = F0 + b * K4 * KCS;
      const double* pa = Fb + (lane & 3) * KCS + mt * 8 + (lane >> 2);
      int ks = (dbg & 2) ? ks1 : ks0;  // profiling: no DMMA (PND_KSTAGE_DBG & 2)
      if constexpr (KHR > 0) {
        const double* pak = pa + ks0 * 4 * KCS;
#pragma unroll
        for (int i = 0; i < KHR; ++i) {
          const double a0 = pak[i * 4 * KCS];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
            dmma884(acc[i & 1][nt][0], acc[i & 1][nt][1], a0, breg[i][nt]);
        }
        ks = ks1;
      }
      if (ks + 1 < ks1) {
        // software-pipelined: the next k-step pair's fragments are loaded
        // before this pair's DMMAs issue (the loads were the DMMAs' wait)
        double av[2], bv[2][NT];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          av[h] = pa[(ks + h) * 4 * KCS];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) bv[h][nt] = pb0[((ks + h) * NT + nt) * 32];
        }
        for (; ks + 1 < ks1; ks += 2) {
          double an[2], bn[2][NT];
          const bool more = ks + 3 < ks1;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            an[h] = more ? pa[(ks + 2 + h) * 4 * KCS] : 0.0;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
              bn[h][nt] = more ? pb0[((ks + 2 + h) * NT + nt) * 32] : 0.0;
          }
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              dmma884(acc[h][nt][0], acc[h][nt][1], av[h], bv[h][nt]);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            av[h] = an[h];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) bv[h][nt] = bn[h][nt];
          }
        }
      }
      if (ks < ks1) {
        const double a0 = pa[ks * 4 * KCS];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          dmma884(acc[0][nt][0], acc[0][nt][1], a0, pb0[(ks * NT + nt) * 32]);
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        acc[0][nt][0] += acc[1][nt][0];
        acc[0][nt][1] += acc[1][nt][1];
      }
      // F[b] is free as soon as this warp's DMMAs have read it; the k-parts
      // of an m-tile meet in their own partial buffer, synchronised pairwise
      // (named barrier 3 + m-tile, KSPLIT warps) instead of across all
      // contraction warps
      __syncwarp();
      warp_arrive(&pb->fempty[b]);
      if (kh) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          *reinterpret_cast<double2*>(red + (((kh - 1) * MT + mt) * NT + nt) * 64 + 2 * lane) =
              make_double2(acc[0][nt][0], acc[0][nt][1]);
      }
      named_sync(3 + mt, 32 * KSPLIT);  // the m-tile's partials written
      if (!kh) {
        const int row = c0 + mt * 8 + (lane >> 2);
        double v[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          v[nt][0] = acc[0][nt][0];
          v[nt][1] = acc[0][nt][1];
#pragma unroll
          for (int p = 1; p < KSPLIT; ++p) {
            const double2 pv = *reinterpret_cast<const double2*>(
                red + (((p - 1) * MT + mt) * NT + nt) * 64 + 2 * lane);
            v[nt][0] += pv.x;
            v[nt][1] += pv.y;
          }
        }
        named_sync(3 + mt, 32 * KSPLIT);  // read before the next chunk's partials
        if (row < g.n) {
          double* o = out.p + (long)row * out.rs;
          const double is = is_pre;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const int n = nt * 8 + 2 * (lane & 3);
            double v0 = v[nt][0], v1 = v[nt][1];
            if (oscale) {
              v0 *= is;
              v1 *= is;
            }
            if (n + 1 < out.rs) *reinterpret_cast<double2*>(o + n) = make_double2(v0, v1);
            else if (n < out.rs) o[n] = v0;
          }
        }
      } else {
        named_sync(3 + mt, 32 * KSPLIT);
      }
    }
  }
}

__global__ void bcat_kernel(const double* M, int kM, int xc, StScale sc, const double* S0, int kS,
                            int r, int K4, int RB, double* B) {
  for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < K4 * RB; i += blockDim.x * gridDim.x) {
    const int k = i / RB, n = i % RB;
    double v = 0.0;
    if (n < r) {
      if (k < kM) v = M[(size_t)k * r + n] * sc.v[k / xc];  // 1/(2h) of stencil k / xc
      else if (k < kM + kS) v = S0[(size_t)(k - kM) * r + n];
    }
    B[i] = v;
  }
}

template <int NA, int RB, bool PRE, int KC, int KHR = 0>
bool kstage_try(const KStageArgs& a, const double* B, int K, int K4, cudaStream_t st) {
  const Geom& g = a.geo;
  const int ra = a.U0.p ? a.U0.cols : 0;
  const bool sepc = ra > 0 && !(a.U0.p == a.X.p && a.U0.rs == a.X.rs);
  // PRE: the staged rows already hold S^-1 x, the formers read no 1/S row;
  // KHR: U0's centre rows are read from global memory instead of staged
  Seg S = make_seg<KC>(g, &a.X, 1, (sepc && KHR == 0) ? &a.U0 : nullptr, false, PRE);
  if (a.zpart) {
    // interior planes (no halo row read) / the four boundary planes: the
    // halo exchange of X overlaps the interior launch (streaming_step)
    if (S.cpp == 0 || g.nz < 5) fail(PND_ECONFIG, "kstage: plane split needs whole chunks per plane");
    S.zlo = a.zpart == 1 ? 2 : 0;
    S.nzr = a.zpart == 1 ? g.nz - 4 : 4;
    S.zb = a.zpart == 2 ? 1 : 0;
    S.nchunks = S.nzr * S.cpp;
  }
  constexpr int KSP = CONW / (KC / 8);
  const size_t fixed = (2 * (size_t)K4 * pad4(KC) + (KHR > 0 ? 0 : (size_t)K4 * RB) +
                        (size_t)(KSP - 1) * (KC / 8) * (RB / 8) * 64) * sizeof(double) +
                       sizeof(PipeBars);
  const int nstg = stages_for(fixed, S.total);
  if (nstg < (KHR > 0 ? 3 : 2)) return false;  // KHR only pays with a deeper ring
  const size_t smem = fixed + (size_t)nstg * S.total * sizeof(double);
  constexpr int nth = KHR > 0 ? RPTH : PTH;
  allow_max_smem(kstage_kernel<NA, RB, PRE, KC, KHR>);
  const int nchunks = S.nchunks;
  int grid = sm_count() * resident(kstage_kernel<NA, RB, PRE, KC, KHR>, nth, smem);
  // the interior launch of an overlapped halo exchange leaves two SMs to the
  // exchange's NCCL kernels (the persistent CTAs would otherwise hold every
  // SM and serialise the exchange behind them)
  if (a.zpart == 1 && grid > 2 * resident(kstage_kernel<NA, RB, PRE, KC, KHR>, nth, smem))
    grid -= 2 * resident(kstage_kernel<NA, RB, PRE, KC, KHR>, nth, smem);
  if (grid > nchunks) grid = nchunks;
  const char* dbg = getenv("PND_KSTAGE_DBG");
  kstage_kernel<NA, RB, PRE, KC, KHR><<<grid, nth, smem, st>>>(
      g, a.X, a.U0, a.out, B, K, K4, S, nstg, a.inv_s, a.out_scaled ? 1 : 0, dbg ? atoi(dbg) : 0);
  launched();
  return true;
}

template <int NA, int RB, bool PRE>
void kstage_launch(const KStageArgs& a, DBuf& bcat, cudaStream_t st) {
  const int ra = a.U0.p ? a.U0.cols : 0;
  const bool sepc = ra > 0 && !(a.U0.p == a.X.p && a.U0.rs == a.X.rs);
  if (PRE && ra > 0 && !sepc) fail(PND_ECONFIG, "kstage: scaled input needs separate base rows");
  const int K = 2 * NA * a.X.cols + ra;
  const int K4 = (K + 15) / 16 * 16;  // whole groups of four k-steps
  double* B = bcat.get((size_t)K4 * RB);
  bcat_kernel<<<16, 256, 0, st>>>(a.M, 2 * NA * a.X.cols, a.X.cols, stencil_scale(a.geo), a.S0,
                                  ra, a.out.cols, K4, RB, B);
  launched();
  // 32-cell chunks when the tiles fit, else 16-cell chunks (larger ranks);
  // the register-rebalanced variant for the bench's 3-D r = 20 tiles
  // The B fragments in registers (setmaxnreg-rebalanced warpgroups) free the
  // shared copy of [M; S0] for a third staging slot; measured a gain only for
  // the last Horner stage (no U0 base rows: 5.74 -> 5.30 ms at 256^3) and a
  // loss with them (the base rows then come from global memory: 6.21 -> 6.79)
  if (NA == 3 && RB == 24 && ra == 0 && !getenv("PND_KSTAGE_SMEM_B")) {
    const int khr = K4 / 8;  // k-steps per contraction k-half (KC = 32: 4 m-tiles x 2)
    if (khr == 18 && kstage_try<NA, RB, PRE, 32, 18>(a, B, K, K4, st)) return;
    if (khr == 16 && kstage_try<NA, RB, PRE, 32, 16>(a, B, K, K4, st)) return;
  }
  if (kstage_try<NA, RB, PRE, 32>(a, B, K, K4, st)) return;
  if (kstage_try<NA, RB, PRE, 16>(a, B, K, K4, st)) return;
  fail(PND_ECONFIG, "kstage tile exceeds shared memory");
}

template <int NA, int RB>
void kstage_rb(const KStageArgs& a, DBuf& bcat, cudaStream_t st) {
  if (a.in_scaled) kstage_launch<NA, RB, true>(a, bcat, st);
  else kstage_launch<NA, RB, false>(a, bcat, st);
}

template <int NA>
void kstage_na(const KStageArgs& a, DBuf& bcat, cudaStream_t st) {
  const int r = a.out.cols > a.X.cols ? a.out.cols : a.X.cols;
  if (r <= 8) kstage_rb<NA, 8>(a, bcat, st);
  else if (r <= 16) kstage_rb<NA, 16>(a, bcat, st);
  else if (r <= 24) kstage_rb<NA, 24>(a, bcat, st);
  else if (r <= 32) kstage_rb<NA, 32>(a, bcat, st);
  else fail(PND_ECONFIG, "kstage supports at most 32 output columns");
}

// ===================================================================== sgram
// G_s = [X1 | X2]^T D_s S^-1 [X1 | X2]. Chunk = GC cells (32 for w <= 24,
// else 16, so a chunk carries enough work per pipeline handoff); per buffer b:
// F[b] = [NS W][pad4(GC)] stencil features (k = cell), C[b] = [GC][pad4(W)] unscaled
// centre rows (the A = X^T operand). Contraction warp m (of 7) owns the
// stencil-column tiles bt = bt0 + m + 7u (bt = s T8 + tj) against all T8 row tiles, one
// accumulator per tile (T8 UPW independent chains); launches cover column-tile
// ranges of at most 32 tiles.
// PO (plus only): only the D+ stencil of every axis is formed and contracted
// (NA Grams); the D- Grams follow from them (reduce_minus: one material
// class, single device)
template <int NA, int T8, int GC, bool PO = false>
__global__ void __launch_bounds__(gpth(T8), 1)
    sgram_kernel(Geom g, NMat X1, NMat X2, Seg S, int nstg, const double* __restrict__ isp,
                 int bt0, int nbt, double* __restrict__ partial) {
  constexpr int NS = PO ? NA : 2 * NA;  // stencils formed
  constexpr int W = T8 * 8;
  constexpr int XS = pad4(W);
  constexpr int GCONW = gconw(T8), GPTH = gpth(T8);
  constexpr int GTL = pad4(GC);       // feature tile row length (k = cell)
  constexpr int CG = GC / 4;          // groups of 4 cells: 4 or 8
  constexpr int JS = 8 * (8 / CG);    // column stride of one former lane
  constexpr int NBMAX = 32;
  constexpr int UPW = ((NS * T8 < NBMAX ? NS * T8 : NBMAX) + GCONW - 1) / GCONW;
  constexpr int FT = NS * W * GTL + GC * XS;  // doubles per feature buffer
  extern __shared__ __align__(128) double sm[];
  // staging slot s: sm + s S.total; feature buffer f: F0 + f FT
  double* const F0 = sm + nstg * S.total;
  PipeBars* pb = reinterpret_cast<PipeBars*>(F0 + 2 * FT);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int a1 = X1.cols, a2 = X2.p ? X2.cols : 0, w = a1 + a2;
  const int nin = X2.p ? 2 : 1;
  pipe_init(pb, nstg, GCONW);
  for (int i = tid; i < 2 * FT; i += GPTH) F0[i] = 0.0;
  __syncthreads();
  const int nchunks = S.nchunks;

  if (warp == FORMW + GCONW) {
    if (lane == 0) {
      Ring r(nstg);
      for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, r.next()) {
        if (r.k) mbar_wait(&pb->sempty[r.s], (r.k - 1) & 1);
        issue_seg<GC, NA>(S, sm + r.s * S.total, &pb->sfull[r.s], chunk_cell(S, chunk, GC), X1,
                          X2, nin, isp, X1);
      }
    }
  } else if (warp < FORMW) {
    // lane = (cell 4 (w % CG) + (lane & 3), column (lane >> 2) + 8 (w / CG) + JS t)
    const int ci = 4 * (warp % CG) + (lane & 3), cj = (lane >> 2) + 8 * (warp / CG);
    Ring r(nstg);
    int it = 0;
    for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, ++it, r.next()) {
      const int f = it & 1, u = it >> 1;
      const int c0 = chunk_cell(S, chunk, GC);
      mbar_wait(&pb->sfull[r.s], r.k & 1);
      if (u >= 1) mbar_wait(&pb->fempty[f], (u - 1) & 1);
      const double* sb = sm + r.s * S.total;
      const double* X1s = sb + S.xoff[0];
      const double* X2s = sb + S.xoff[1];
      double* Fb = F0 + f * FT;
      double* Cb = Fb + NS * W * GTL;
      // unscaled centre rows (A operand); rows past n are zero halo rows
      for (int j = cj; j < w; j += JS)
        Cb[ci * XS + j] = c0 + ci >= g.n ? 0.0  // past n: halo rows (maybe a neighbour's)
                          : j < a1 ? X1s[(ci + 2) * X1.rs + j]
                                   : X2s[(ci + 2) * X2.rs + j - a1];
      // PO (one material class): 1/S is one number, so the formers difference
      // the raw rows and reduce_parts_po applies 1/S with 1/(2h)
      Ctx<GC, NA, PO, PO> cx;
      cx.init(g, c0 + ci, ci, sb + S.ioff);
      const bool fast = __all_sync(0xffffffffu, cx.inner);
      constexpr int TT = (W + JS - 1) / JS;
      cx.rows(X1s, X1.rs, ci, cj);
#pragma unroll
      for (int t = 0; t < TT; ++t) {
        const int j = cj + JS * t;
        if (j < a1) {
          double v[2 * NA];
          if (fast) cx.template apply<true>(g, JS * t, v);
          else cx.template apply<false>(g, JS * t, v);
#pragma unroll
          for (int s = 0; s < NS; ++s) Fb[(s * W + j) * GTL + ci] = v[PO ? 2 * s : s];
        }
      }
      if (a2) {
        const int j0 = cj >= a1 ? cj : cj + JS * ((a1 - cj + JS - 1) / JS);
        cx.rows(X2s, X2.rs, ci, j0 - a1);
#pragma unroll
        for (int t = 0; t < TT; ++t) {
          const int j = j0 + JS * t;
          if (j < w) {
            double v[2 * NA];
            if (fast) cx.template apply<true>(g, JS * t, v);
            else cx.template apply<false>(g, JS * t, v);
#pragma unroll
            for (int s = 0; s < NS; ++s) Fb[(s * W + j) * GTL + ci] = v[PO ? 2 * s : s];
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&pb->ffull[f]);
        mbar_arrive(&pb->sempty[r.s]);
      }
    }
  } else {
    const int m = warp - FORMW;
    double acc[UPW][T8][2];
#pragma unroll
    for (int q = 0; q < UPW; ++q)
#pragma unroll
      for (int ti = 0; ti < T8; ++ti) acc[q][ti][0] = acc[q][ti][1] = 0.0;
    const int m0 = lane >> 2, kq = lane & 3;
    int it = 0;
    for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, ++it) {
      const int b = it & 1, u = it >> 1;
      mbar_wait(&pb->ffull[b], u & 1);
      const double* pa = F0 + b * FT + NS * W * GTL + kq * XS + m0;
      const double* pbt = F0 + b * FT + ((bt0 + m) * 8 + m0) * GTL + kq;
      // software-pipelined over the chunk's GC / 4 k-steps (while the
      // registers allow: UPW T8 <= 10 accumulator tiles): the next k-step's
      // fragments are loaded before this one's DMMAs issue
      if constexpr (UPW * T8 > 10) {
#pragma unroll 1
        for (int k0 = 0; k0 < GC; k0 += 4) {
          double af[T8];
#pragma unroll
          for (int ti = 0; ti < T8; ++ti) af[ti] = pa[k0 * XS + ti * 8];
#pragma unroll
          for (int q = 0; q < UPW; ++q) {
            if (m + GCONW * q < nbt) {
              const double bf = pbt[q * GCONW * 8 * GTL + k0];
#pragma unroll
              for (int ti = 0; ti < T8; ++ti) dmma884(acc[q][ti][0], acc[q][ti][1], af[ti], bf);
            }
          }
        }
      } else {
      double af[T8], bf[UPW];
#pragma unroll
      for (int ti = 0; ti < T8; ++ti) af[ti] = pa[ti * 8];
#pragma unroll
      for (int q = 0; q < UPW; ++q)
        bf[q] = m + GCONW * q < nbt ? pbt[q * GCONW * 8 * GTL] : 0.0;
#pragma unroll
      for (int k0 = 0; k0 < GC; k0 += 4) {
        double an[T8], bn[UPW];
        if (k0 + 4 < GC) {
#pragma unroll
          for (int ti = 0; ti < T8; ++ti) an[ti] = pa[(k0 + 4) * XS + ti * 8];
#pragma unroll
          for (int q = 0; q < UPW; ++q)
            bn[q] = m + GCONW * q < nbt ? pbt[q * GCONW * 8 * GTL + k0 + 4] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < UPW; ++q) {
          if (m + GCONW * q < nbt) {
#pragma unroll
            for (int ti = 0; ti < T8; ++ti) dmma884(acc[q][ti][0], acc[q][ti][1], af[ti], bf[q]);
          }
        }
        if (k0 + 4 < GC) {
#pragma unroll
          for (int ti = 0; ti < T8; ++ti) af[ti] = an[ti];
#pragma unroll
          for (int q = 0; q < UPW; ++q) bf[q] = bn[q];
        }
      }
      }
      warp_arrive(&pb->fempty[b]);
    }
    double* out = partial + (size_t)blockIdx.x * NS * w * w;
#pragma unroll
    for (int q = 0; q < UPW; ++q) {
      if (m + GCONW * q < nbt) {
        const int bt = bt0 + m + GCONW * q;
        const int s = bt / T8, tj = bt - s * T8;
        const int col = tj * 8 + 2 * (lane & 3);
#pragma unroll
        for (int ti = 0; ti < T8; ++ti) {
          const int row = ti * 8 + (lane >> 2);
          if (row < w) {
            double* o = out + ((size_t)s * w + row) * w;
            if (col < w) o[col] = acc[q][ti][0];
            if (col + 1 < w) o[col + 1] = acc[q][ti][1];
          }
        }
      }
    }
  }
}

// Rectangular stencil Grams G_s = XA^T D_s S^-1 XB for the column-blocked
// layout of ranks above 64 (xwide.cu): the features are formed from ONE
// block XB (<= 32 columns, halo segments staged) and contracted against the
// centre rows of another block XA (<= 32 columns, staged without halo), so
// every (A, B) block pair is one launch of exactly its own work -- the
// square kernel above, run on [XA | XB], would also recompute both diagonal
// blocks and form XA's features. Same roles and pipeline as sgram_kernel.
template <int NA, int T8A, int T8B, int GC>
__global__ void __launch_bounds__(gpth(T8B), 1)
    sgram_rect_kernel(Geom g, NMat XA, NMat XB, Seg S, int nstg, const double* __restrict__ isp,
                      double* __restrict__ partial) {
  constexpr int NS = 2 * NA;
  constexpr int WA = T8A * 8, WB = T8B * 8;
  constexpr int XS = pad4(WA);
  constexpr int GCONW = gconw(T8B), GPTH = gpth(T8B);
  constexpr int GTL = pad4(GC);
  constexpr int CG = GC / 4;
  constexpr int JS = 8 * (8 / CG);
  constexpr int NBT = NS * T8B;                       // feature column tiles
  constexpr int UPW = (NBT + GCONW - 1) / GCONW;
  constexpr int FT = NS * WB * GTL + GC * XS;
  extern __shared__ __align__(128) double sm[];
  double* const F0 = sm + nstg * S.total;
  PipeBars* pb = reinterpret_cast<PipeBars*>(F0 + 2 * FT);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wa = XA.cols, wb = XB.cols;
  pipe_init(pb, nstg, GCONW);
  for (int i = tid; i < 2 * FT; i += GPTH) F0[i] = 0.0;
  __syncthreads();
  const int nchunks = S.nchunks;

  if (warp == FORMW + GCONW) {
    if (lane == 0) {
      Ring r(nstg);
      for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, r.next()) {
        if (r.k) mbar_wait(&pb->sempty[r.s], (r.k - 1) & 1);
        issue_seg<GC, NA>(S, sm + r.s * S.total, &pb->sfull[r.s], chunk_cell(S, chunk, GC), XB,
                          XB, 1, isp, XA);
      }
    }
  } else if (warp < FORMW) {
    const int ci = 4 * (warp % CG) + (lane & 3), cj = (lane >> 2) + 8 * (warp / CG);
    Ring r(nstg);
    int it = 0;
    for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, ++it, r.next()) {
      const int f = it & 1, u = it >> 1;
      const int c0 = chunk_cell(S, chunk, GC);
      mbar_wait(&pb->sfull[r.s], r.k & 1);
      if (u >= 1) mbar_wait(&pb->fempty[f], (u - 1) & 1);
      const double* sb = sm + r.s * S.total;
      const double* XBs = sb + S.xoff[0];
      double* Fb = F0 + f * FT;
      double* Cb = Fb + NS * WB * GTL;
      // XA centre rows (the A operand); rows past n stay out of the Grams
      for (int j = cj; j < wa; j += JS)
        Cb[ci * XS + j] = c0 + ci >= g.n ? 0.0 : sb[S.coff + ci * XA.rs + j];
      Ctx<GC, NA> cx;
      cx.init(g, c0 + ci, ci, sb + S.ioff);
      const bool fast = __all_sync(0xffffffffu, cx.inner);
      constexpr int TT = (WB + JS - 1) / JS;
      cx.rows(XBs, XB.rs, ci, cj);
#pragma unroll
      for (int t = 0; t < TT; ++t) {
        const int j = cj + JS * t;
        if (j < wb) {
          double v[NS];
          if (fast) cx.template apply<true>(g, JS * t, v);
          else cx.template apply<false>(g, JS * t, v);
#pragma unroll
          for (int s2 = 0; s2 < NS; ++s2) Fb[(s2 * WB + j) * GTL + ci] = v[s2];
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&pb->ffull[f]);
        mbar_arrive(&pb->sempty[r.s]);
      }
    }
  } else {
    const int m = warp - FORMW;
    double acc[UPW][T8A][2];
#pragma unroll
    for (int q = 0; q < UPW; ++q)
#pragma unroll
      for (int ti = 0; ti < T8A; ++ti) acc[q][ti][0] = acc[q][ti][1] = 0.0;
    const int m0 = lane >> 2, kq = lane & 3;
    int it = 0;
    for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, ++it) {
      const int b = it & 1, u = it >> 1;
      mbar_wait(&pb->ffull[b], u & 1);
      const double* pa = F0 + b * FT + NS * WB * GTL + kq * XS + m0;
      const double* pbt = F0 + b * FT + (m * 8 + m0) * GTL + kq;
#pragma unroll 1
      for (int k0 = 0; k0 < GC; k0 += 4) {
        double af[T8A];
#pragma unroll
        for (int ti = 0; ti < T8A; ++ti) af[ti] = pa[k0 * XS + ti * 8];
#pragma unroll
        for (int q = 0; q < UPW; ++q) {
          if (m + GCONW * q < NBT) {
            const double bf = pbt[q * GCONW * 8 * GTL + k0];
#pragma unroll
            for (int ti = 0; ti < T8A; ++ti) dmma884(acc[q][ti][0], acc[q][ti][1], af[ti], bf);
          }
        }
      }
      warp_arrive(&pb->fempty[b]);
    }
    double* out = partial + (size_t)blockIdx.x * NS * wa * wb;
#pragma unroll
    for (int q = 0; q < UPW; ++q) {
      if (m + GCONW * q < NBT) {
        const int bt = m + GCONW * q;
        const int s2 = bt / T8B, tj = bt - s2 * T8B;
        const int col = tj * 8 + 2 * (lane & 3);
#pragma unroll
        for (int ti = 0; ti < T8A; ++ti) {
          const int row = ti * 8 + (lane >> 2);
          if (row < wa) {
            double* o = out + ((size_t)s2 * wa + row) * wb;
            if (col < wb) o[col] = acc[q][ti][0];
            if (col + 1 < wb) o[col + 1] = acc[q][ti][1];
          }
        }
      }
    }
  }
}

// the D+ partials (NA x per) summed in fixed order into the even stencil slots
__global__ void reduce_parts_po(const double* __restrict__ partial, int nblk, int count, int per,
                                StScale sc, const double* __restrict__ isp,
                                double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int b = 0; b < nblk; ++b) s += partial[(size_t)b * count + i];
  const int a = i / per;
  // isp[0]: the one material's 1/S (the formers differenced the raw rows)
  out[(size_t)(2 * a) * per + (i - a * per)] = s * sc.v[a] * isp[0];
}

// sums the per-CTA Gram partials in a fixed order and applies the stencil's
// 1/(2h) (count = ns * per)
__global__ void reduce_parts(const double* __restrict__ partial, int nblk, int count, int per,
                             StScale sc, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int b = 0; b < nblk; ++b) s += partial[(size_t)b * count + i];
  out[i] = s * sc.v[i / per];
}

template <int NA, int T8, int GC, bool PO = false>
void sgram_launch(const Geom& g, NMat X1, NMat X2, const double* isp, double* out, DBuf& partial,
                  cudaStream_t st) {
  constexpr int GTL = pad4(GC);
  constexpr int NSF = PO ? NA : 2 * NA;
  const NMat ins[2] = {X1, X2};
  // PO: raw rows are differenced (1/S applied in the reduction): no 1/S rows staged
  const Seg S = make_seg<GC>(g, ins, X2.p ? 2 : 1, nullptr, PO && !getenv("PND_SGRAM_ALLSEG"), PO);
  const int W = T8 * 8;
  const size_t ft = (size_t)NSF * W * GTL + (size_t)GC * pad4(W);
  const size_t fixed = 2 * ft * sizeof(double) + sizeof(PipeBars);
  const int nstg = stages_for(fixed, S.total);
  if (nstg < 2) fail(PND_ECONFIG, "stencil Gram tile exceeds shared memory");
  const size_t smem = fixed + (size_t)nstg * S.total * sizeof(double);
  allow_max_smem(sgram_kernel<NA, T8, GC, PO>);
  const int nchunks = (g.n + GC - 1) / GC;
  int grid = sm_count() * resident(sgram_kernel<NA, T8, GC, PO>, gpth(T8), smem);
  if (grid > nchunks) grid = nchunks;
  const int w = X1.cols + (X2.p ? X2.cols : 0);
  const size_t count = (size_t)NSF * w * w;
  double* part = partial.get(count * grid);
  const int nb = NSF * T8;
  for (int bt0 = 0; bt0 < nb; bt0 += 32) {
    const int nbt = nb - bt0 < 32 ? nb - bt0 : 32;
    sgram_kernel<NA, T8, GC, PO><<<grid, gpth(T8), smem, st>>>(g, X1, X2, S, nstg, isp, bt0, nbt,
                                                            part);
    launched();
  }
  if (PO) {
    // the D+ Grams into the even stencil slots, then D- = -(D+)^T + boundary rows
    StScale sc = stencil_scale(g), sp{};
    for (int a = 0; a < NA; ++a) sp.v[a] = sc.v[2 * a];
    reduce_parts_po<<<(int)((count + 255) / 256), 256, 0, st>>>(part, grid, (int)count, w * w,
                                                                sp, isp, out);
    launched();
    minus_from_plus(g, X1, X2, isp, out, partial, st);
    comm_allreduce(g, out, (size_t)2 * NA * w * w, st);
    return;
  }
  reduce_parts<<<(int)((count + 255) / 256), 256, 0, st>>>(part, grid, (int)count, w * w,
                                                           stencil_scale(g), out);
  launched();
  comm_allreduce(g, out, count, st);
}

// the rectangular per-CTA partials (ns x wa x wb) summed in fixed order, scaled
// by 1/(2h), placed at rows r0.., columns c0.. of each ns x w x w Gram
__global__ void reduce_place(const double* __restrict__ partial, int nblk, int ns, int wa, int wb,
                             StScale sc, double* __restrict__ G, int w, int r0, int c0) {
  const int count = ns * wa * wb;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double v = 0.0;
  for (int b = 0; b < nblk; ++b) v += partial[(size_t)b * count + i];
  const int s2 = i / (wa * wb), rem = i - s2 * wa * wb, r = rem / wb, c = rem - r * wb;
  G[((size_t)s2 * w + r0 + r) * w + c0 + c] = v * sc.v[s2];
}

template <int NA, int GC>
void sgram_rect_launch(const Geom& g, NMat XA, NMat XB, const double* isp, double* G, int w,
                       int r0, int c0, DBuf& partial, cudaStream_t st) {
  constexpr int T8 = 4;  // 32-column blocks
  const Seg S = make_seg<GC>(g, &XB, 1, &XA);
  const size_t ft = (size_t)2 * NA * (T8 * 8) * pad4(GC) + (size_t)GC * pad4(T8 * 8);
  const size_t fixed = 2 * ft * sizeof(double) + sizeof(PipeBars);
  const int nstg = stages_for(fixed, S.total);
  if (nstg < 2) fail(PND_ECONFIG, "stencil Gram tile exceeds shared memory");
  const size_t smem = fixed + (size_t)nstg * S.total * sizeof(double);
  allow_max_smem(sgram_rect_kernel<NA, T8, T8, GC>);
  const int nchunks = (g.n + GC - 1) / GC;
  int grid = sm_count() * resident(sgram_rect_kernel<NA, T8, T8, GC>, gpth(T8), smem);
  if (grid > nchunks) grid = nchunks;
  const int ns = 2 * NA;
  const size_t count = (size_t)ns * XA.cols * XB.cols;
  double* part = partial.get(count * grid);
  sgram_rect_kernel<NA, T8, T8, GC><<<grid, gpth(T8), smem, st>>>(g, XA, XB, S, nstg, isp, part);
  launched();
  reduce_place<<<(int)((count + 255) / 256), 256, 0, st>>>(part, grid, ns, XA.cols, XB.cols,
                                                           stencil_scale(g), G, w, r0, c0);
  launched();
}

template <int NA>
void sgram_na(const Geom& g, NMat X1, NMat X2, const double* isp, double* out, DBuf& partial,
              cudaStream_t st) {
  const int w = X1.cols + (X2.p ? X2.cols : 0);
  // one material class on one device: half the stencil Grams (the D+ ones)
  if (g.uniform_s && comm_world(g) == 1 && !getenv("PND_SGRAM_FULL")) {
    switch ((w + 7) / 8) {
      case 1: sgram_launch<NA, 1, 32, true>(g, X1, X2, isp, out, partial, st); return;
      case 2: sgram_launch<NA, 2, 32, true>(g, X1, X2, isp, out, partial, st); return;
      case 3: sgram_launch<NA, 3, 32, true>(g, X1, X2, isp, out, partial, st); return;
      case 4: sgram_launch<NA, 4, 16, true>(g, X1, X2, isp, out, partial, st); return;
      case 5: sgram_launch<NA, 5, 16, true>(g, X1, X2, isp, out, partial, st); return;
      case 6: sgram_launch<NA, 6, 16, true>(g, X1, X2, isp, out, partial, st); return;
      case 7: sgram_launch<NA, 7, 8, true>(g, X1, X2, isp, out, partial, st); return;
      case 8: sgram_launch<NA, 8, 8, true>(g, X1, X2, isp, out, partial, st); return;
      default: break;
    }
  }
  switch ((w + 7) / 8) {
    case 1: sgram_launch<NA, 1, 32>(g, X1, X2, isp, out, partial, st); break;
    case 2: sgram_launch<NA, 2, 32>(g, X1, X2, isp, out, partial, st); break;
    case 3: sgram_launch<NA, 3, 32>(g, X1, X2, isp, out, partial, st); break;
    case 4: sgram_launch<NA, 4, 16>(g, X1, X2, isp, out, partial, st); break;
    case 5: sgram_launch<NA, 5, 16>(g, X1, X2, isp, out, partial, st); break;
    case 6: sgram_launch<NA, 6, 16>(g, X1, X2, isp, out, partial, st); break;
    case 7: sgram_launch<NA, 7, 8>(g, X1, X2, isp, out, partial, st); break;
    case 8: sgram_launch<NA, 8, 8>(g, X1, X2, isp, out, partial, st); break;
    default: fail(PND_ECONFIG, "stencil Grams support at most 64 columns");
  }
}


}  // namespace

bool kstage_can_split(const Geom& g) {
  // whole 32- and 16-cell chunks per plane, an interior to overlap
  return g.nz >= 5 && ((size_t)g.nx * g.ny) % 32 == 0 && g.axis[g.na - 1] == 2;
}

void kstage(const KStageArgs& a, cudaStream_t st) {
  if (!a.bcat) fail(PND_ECONFIG, "kstage: no [M; S0] scratch buffer");
  if (a.X.cols > 32 || (a.U0.p && a.U0.cols > 32))
    fail(PND_ECONFIG, "kstage supports <= 32 input columns");
  switch (a.geo.na) {
    case 1: kstage_na<1>(a, *a.bcat, st); break;
    case 2: kstage_na<2>(a, *a.bcat, st); break;
    case 3: kstage_na<3>(a, *a.bcat, st); break;
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

// ---------------------------------------------------------------- D- from D+
// One material class (1/S = sigma in every cell), one device: along an axis
// the reference's stencils (spatial.py:81-118) satisfy D- = -(D+)^T + E with
// E nonzero only in the rows of the first two and last two cells of each
// line, so X^T D- S^-1 X = -(X^T D+ S^-1 X)^T + sigma X^T E X: the D- Grams
// cost a pass over the boundary cells (2 x 2 planes per axis) instead of a
// stencil contraction over the whole grid.
namespace {

// coefficients x 2h of the reference's D+ (minus-biased) and D- rows
double dplus_c(int r, int c) {
  if (r >= 2) return c == r ? 3.0 : c == r - 1 ? -4.0 : c == r - 2 ? 1.0 : 0.0;
  if (r == 1) return c == 1 ? 2.0 : c == 0 ? -2.0 : 0.0;
  return c == 0 ? 2.0 : 0.0;
}
double dminus_c(int L, int r, int c) {
  if (r <= L - 3) return c == r ? -3.0 : c == r + 1 ? 4.0 : c == r + 2 ? -1.0 : 0.0;
  if (r == L - 2) return c == r ? -2.0 : c == r + 1 ? 2.0 : 0.0;
  return c == r ? -2.0 : 0.0;
}

struct ERows {
  int nb;          // boundary rows (<= 4)
  int row[4];
  double e[4][5];  // E[row][row + d], d = -2..2 (x 2h)
};

ERows e_rows(int L) {
  ERows er{};
  for (int i = 0; i < L; ++i) {
    double e[5];
    bool any = false;
    for (int d = -2; d <= 2; ++d) {
      const int j = i + d;
      e[d + 2] = (j >= 0 && j < L) ? dminus_c(L, i, j) + dplus_c(j, i) : 0.0;
      any = any || e[d + 2] != 0.0;
    }
    if (!any) continue;
    if (er.nb >= 4) fail(PND_ECONFIG, "stencil transpose: unexpected interior rows");
    er.row[er.nb] = i;
    for (int d = 0; d < 5; ++d) er.e[er.nb][d] = e[d];
    ++er.nb;
  }
  return er;
}

// boundary cells b of one axis -> Xb[b] = X[c], Zb[b] = sigma_c sum_d E[i][i+d] X[c + d s]
// (one warp row per boundary cell, lanes over the columns; 32-bit cell
// arithmetic: the 64-bit divisions of a flat element index dominated)
__global__ void e_gather_kernel(int n, int L, int s, ERows er, NMat X1, NMat X2,
                                const double* __restrict__ isp, NMat Xb, NMat Zb) {
  const int M = n / L;
  const int nb = er.nb * M;
  const int a1 = X1.cols, w = a1 + (X2.p ? X2.cols : 0);
  for (int b = blockIdx.x * blockDim.y + threadIdx.y; b < nb; b += gridDim.x * blockDim.y) {
    const int p = b / M;
    const int q = b - p * M;
    const long c = (long)(q / s) * ((long)s * L) + (long)er.row[p] * s + (q % s);
    double e[5];
#pragma unroll
    for (int d = 0; d < 5; ++d) e[d] = er.e[p][d];
    const double sc = isp[2 * c];
    for (int col = threadIdx.x; col < w; col += 32) {
      const double* base = col < a1 ? X1.p + col : X2.p + (col - a1);
      const long rs = col < a1 ? X1.rs : X2.rs;
      double z = 0.0;
#pragma unroll
      for (int d = 0; d < 5; ++d)
        if (e[d] != 0.0) z += e[d] * base[(c + (d - 2) * (long)s) * rs];
      Xb.p[(long)b * Xb.rs + col] = base[c * rs];
      Zb.p[(long)b * Zb.rs + col] = sc * z;
    }
  }
}

// out[2a + 1] = -out[2a]^T + corr * i2h
__global__ void minus_assemble_kernel(double* out, int w, int a, const double* corr, double i2h) {
  const int ww = w * w;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ww; e += gridDim.x * blockDim.x) {
    const int r = e / w, c = e - r * w;
    out[(size_t)(2 * a + 1) * ww + e] = -out[(size_t)(2 * a) * ww + (size_t)c * w + r] +
                                        corr[e] * i2h;
  }
}

}  // namespace

void minus_from_plus(const Geom& g, NMat X1, NMat X2, const double* isp, double* out,
                     DBuf& partial, cudaStream_t st) {
  const int w = X1.cols + (X2.p ? X2.cols : 0);
  const int rs = even(w);
  double* corr = nullptr;
  CK(cudaMallocAsync((void**)&corr, (size_t)w * w * sizeof(double), st));
  for (int ai = 0; ai < g.na; ++ai) {
    const int axis = g.axis[ai];
    const int L = axis == 0 ? g.nx : axis == 1 ? g.ny : g.nz;
    const long s = axis == 0 ? 1 : axis == 1 ? g.nx : (long)g.nx * g.ny;
    const ERows er = e_rows(L);
    const long nb = (long)er.nb * (g.n / L);
    // compact boundary-cell matrices with 64 zero rows after them (chunked Gram)
    Geom gb = g;
    gb.n = (int)nb;
    gb.halo = 64;
    gb.comm = nullptr;
    const size_t rows = (size_t)nb + 2 * 64;
    double* buf = nullptr;
    CK(cudaMallocAsync((void**)&buf, 2 * rows * rs * sizeof(double), st));
    if (rs > w || rows < (1 << 16)) {
      fill_zero(buf, 2 * rows * rs, st);  // the padding column too / one launch on small grids
    } else {  // the gather writes every row: zero only the 64-row margins
      for (size_t m0 : {(size_t)0, (size_t)nb + 64, rows, rows + (size_t)nb + 64})
        fill_zero(buf + m0 * rs, 64 * (size_t)rs, st);
    }
    NMat Xb{buf + 64 * (size_t)rs, rs, w}, Zb{buf + (rows + 64) * (size_t)rs, rs, w};
    int grid = (int)((nb + 7) / 8);
    if (grid > 148 * 16) grid = 148 * 16;
    e_gather_kernel<<<grid > 0 ? grid : 1, dim3(32, 8), 0, st>>>(g.n, L, (int)s, er, X1, X2, isp,
                                                                 Xb, Zb);
    launched();
    gram_xy(gb, Xb, Zb, corr, partial, st);
    minus_assemble_kernel<<<(w * w + 255) / 256, 256, 0, st>>>(out, w, ai, corr, g.i2h[axis]);
    launched();
    CK(cudaFreeAsync(buf, st));
  }
  CK(cudaFreeAsync(corr, st));
}

void stencil_grams_rect(const Geom& g, NMat XA, NMat XB, const double* isp, double* G, int w,
                        int r0, int c0, DBuf& partial, cudaStream_t st) {
  if (XA.cols > 32 || XB.cols > 32) fail(PND_ECONFIG, "rectangular stencil Grams take 32 columns");
  switch (g.na) {
    case 1: sgram_rect_launch<1, 32>(g, XA, XB, isp, G, w, r0, c0, partial, st); break;
    case 2: sgram_rect_launch<2, 16>(g, XA, XB, isp, G, w, r0, c0, partial, st); break;
    case 3: sgram_rect_launch<3, 16>(g, XA, XB, isp, G, w, r0, c0, partial, st); break;
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
