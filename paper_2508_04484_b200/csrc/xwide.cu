// Ranks above 64: the energy step on column-blocked n-side storage.
//
// Up to rank 64 the state U (and the augmentation Q) are cell-major matrices
// with one row per cell (step.cu, wide.cu). Above 64 every n-side matrix of
// the step is stored as a list of cell-major 32-column blocks, each its own
// buffer with its own zero halo rows -- the layout every n-side kernel
// already reads (one block = one <= 32-column matrix), so no kernel changes
// and no split copies: the state costs n x r doubles per factor whatever r
// is (256^3 at r = 200: U, Q, the two Horner iterates, the rotation output
// and the CGS scratch are 6 x 26.8 GB).
//
// Every product over columns becomes a chain over blocks:
//   bm_lincomb  out_j = sum_t s_t In_t T_t[:, j-block], the LINCOMB kernel
//               taking up to three 32-column input blocks per pass (the
//               running partial sum rides in a pass as [partial | In] [I; T]);
//   bm_gram     X^T diag(w) Y block pair by block pair (Gram-only LINCOMB,
//               two Y blocks per pass; symmetric Grams only j >= i);
//   K-stage     one chain per output block (wide.cu: base rows U0 S0 by
//               bm_lincomb, then one K-stage per input block);
//   S-Grams     one rectangular launch per (A, B) block pair of [U0 | Q]
//               (stencil_grams_rect: B's features contracted with A's rows);
// and the small side (R x R SVD / QR / RK4, m-side QR, the r x r implicit
// solves) runs on the same kernels with their work matrices in global
// (L2-resident) memory above the shared-memory sizes (dense.cu).
// The algorithm is step.cu's, line for line (dlra.py:213-322, 90-115).
#include <cmath>
#include <cstring>

#include "handle.h"

namespace pnd {

namespace {

constexpr int XB = 32;  // block width

int nblk(int cols) { return (cols + XB - 1) / XB; }

int gsz(long n) {
  long b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return b < 1 ? 1 : (int)b;
}

// dst (ld columns, row-major) [r0 + i][c0 + j] = src[i][j] (rows x cols contiguous)
__global__ void place_kernel(const double* __restrict__ src, int rows, int cols, double* dst,
                             int ld, int r0, int c0) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols;
       e += gridDim.x * blockDim.x) {
    const int i = e / cols, j = e - i * cols;
    dst[(size_t)(r0 + i) * ld + c0 + j] = src[e];
  }
}

// lower triangle of a symmetric Gram from its upper blocks: out[r][c] =
// out[c][r] where block(r) > block(c)
__global__ void mirror_kernel(double* out, int w) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < w * w; e += gridDim.x * blockDim.x) {
    const int r = e / w, c = e - r * w;
    if (r / XB > c / XB) out[e] = out[(size_t)c * w + r];
  }
}

// TA / TB of one LINCOMB pass: up to 4 row segments stacked, columns
// [c0, c0 + nb) of each source, scaled; ident segments are I (nb x nb)
struct TSeg {
  const double* src;
  int ld, r0, rows, ident;
  double scale;
};
struct TCat {
  TSeg s[4];
  int nseg, c0, nb;
};

__global__ void tcat_kernel(TCat tc, double* dst) {
  int total = 0;
  for (int q = 0; q < tc.nseg; ++q) total += tc.s[q].rows;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total * tc.nb;
       e += gridDim.x * blockDim.x) {
    int row = e / tc.nb;
    const int col = e - row * tc.nb;
    int q = 0;
    while (row >= tc.s[q].rows) row -= tc.s[q++].rows;
    const TSeg& sg = tc.s[q];
    dst[e] = sg.ident ? (row == col ? sg.scale : 0.0)
                      : sg.scale * sg.src[(size_t)(sg.r0 + row) * sg.ld + tc.c0 + col];
  }
}

// U[c][j] = (global cell == j0 + j): the canonical basis, block by block
__global__ void unit_block_kernel(Geom g, NMat U, int j0) {
  const long total = (long)g.n * U.rs;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
       e += (long)gridDim.x * blockDim.x) {
    const int c = (int)(e / U.rs), j = (int)(e - (long)c * U.rs);
    const long cg = c + (long)g.z0 * g.nx * g.ny;
    U.p[e] = (j < U.cols && cg == j0 + j) ? 1.0 : 0.0;
  }
}

// columns [c0, c0 + dst.cols) of a row-major matrix -> one block (and back)
__global__ void cut_kernel(NMat src, int c0, NMat dst, int n) {
  const long total = (long)n * dst.rs;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
       e += (long)gridDim.x * blockDim.x) {
    const long c = e / dst.rs;
    const int j = (int)(e - c * dst.rs);
    dst.p[e] = j < dst.cols ? src.p[c * src.rs + c0 + j] : 0.0;
  }
}
__global__ void paste_kernel(NMat src, int c0, NMat dst, int n) {
  const long total = (long)n * src.cols;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
       e += (long)gridDim.x * blockDim.x) {
    const long c = e / src.cols;
    const int j = (int)(e - c * src.cols);
    dst.p[c * dst.rs + c0 + j] = src.p[c * src.rs + j];
  }
}

// the dose trapezoid (driver.py:606, 613-621) over a blocked U
constexpr int DMAXB = 24;
struct BList {
  NMat b[DMAXB];
  int nb;
};
__global__ void dose_blocks_kernel(Geom g, BList U, const double* __restrict__ coef,
                                   double half_dt, const double* __restrict__ s_field,
                                   const double* __restrict__ psi, int n_beams,
                                   double* __restrict__ dep, double* __restrict__ prev) {
  const double sqrt4pi = 3.5449077018110318;
  __shared__ double sc[DMAXB * XB];
  int tot = 0;
  for (int q = 0; q < U.nb; ++q) tot += U.b[q].cols;
  for (int i = threadIdx.x; i < tot; i += blockDim.x) sc[i] = coef[i];
  __syncthreads();
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < g.n; c += gridDim.x * blockDim.x) {
    double u0 = 0.0;
    int j0 = 0;
    for (int q = 0; q < U.nb; ++q) {
      const double* row = U.b[q].p + (long)c * U.b[q].rs;
      for (int j = 0; j < U.b[q].cols; ++j) u0 = fma(row[j], sc[j0 + j], u0);
      j0 += U.b[q].cols;
    }
    double integrand = sqrt4pi * u0;
    if (psi) {
      double ps = 0.0;
      for (int b = 0; b < n_beams; ++b) ps += psi[(size_t)b * g.ld + c];
      integrand = integrand + s_field[c] * ps;
    }
    dep[c] += half_dt * (prev[c] + integrand);
    prev[c] = integrand;
  }
}

__global__ void eye_x_kernel(double* I, int b) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < b * b; i += gridDim.x * blockDim.x)
    I[i] = (i / b == i % b) ? 1.0 : 0.0;
}

__global__ void zero_rows_x_kernel(double* S, int row0, int rows, int cols) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows * cols;
       i += gridDim.x * blockDim.x)
    S[(size_t)row0 * cols + i] = 0.0;
}

__global__ void defect_x_kernel(const double* G, int r, double* out) {
  __shared__ double red[256];
  double mx = 0.0;
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) {
    const double v = fabs(G[i] - ((i / r == i % r) ? 1.0 : 0.0));
    mx = v > mx ? v : mx;
  }
  red[threadIdx.x] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int i = 0; i < (int)blockDim.x; ++i) m = red[i] > m ? red[i] : m;
    out[0] = out[0] > m ? out[0] : m;
  }
}

__global__ void class_weight_x_kernel(const int* cls, const double* wtab, const double* inv_s,
                                      int n, int phase, int cl, double* w) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n + 64; c += gridDim.x * blockDim.x) {
    double v = 0.0;
    if (c < n) v = inv_s[c] * (phase < 0 ? (cls[c] == cl ? 1.0 : 0.0) : wtab[cls[c] * 12 + phase]);
    w[c] = v;
  }
}

__global__ void gt_x_kernel(const double* g, const double* tm, int m, int nb, double* gt) {
  const int total = nb * 12 * m;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int b = i / (12 * m), rem = i - b * 12 * m, q = rem % m;
    gt[i] = g[rem] * tm[b * m + q];
  }
}

__global__ void coeff_x_kernel(const double* g, const double* sig, int m, double* c) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 12 * m; i += gridDim.x * blockDim.x)
    c[i] = sig[i / m] - g[i];
}

__global__ void init_int_x(int* p, int v) { *p = v; }

// the augmentation helpers of step.cu, for any b (<= 512)
__global__ void defect_gc_x(const double* G, const double* C, int a, int b, double* out) {
  __shared__ double red[256];
  double d = 0.0;
  for (int i = threadIdx.x; i < b * b + a * b; i += blockDim.x) {
    const double v = i < b * b ? fabs(G[i] - ((i / b == i % b) ? 1.0 : 0.0)) : fabs(C[i - b * b]);
    d = v > d ? v : d;
  }
  red[threadIdx.x] = d;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

__global__ void xnorm_x(const double* G2, const double* C1, int a, int b, double rel,
                        double* out) {
  __shared__ double red[256];
  const int tid = threadIdx.x;
  double x2 = 0.0;
  for (int j = tid; j < b; j += blockDim.x) x2 += G2[j * b + j];
  if (C1)
    for (int i = tid; i < a * b; i += blockDim.x) x2 += C1[i] * C1[i];
  red[tid] = x2;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (tid < w) red[tid] += red[tid + w];
    __syncthreads();
  }
  if (tid == 0) out[0] = rel * sqrt(red[0] > 0.0 ? red[0] : 0.0);
}

__global__ void level2_gram_x(const double* G3, const double* C3, int a, int b, int k1, int kb,
                              const double* floor_p, double* Ms, double* dinv) {
  const int tid = threadIdx.x;
  __shared__ double d[512];
  const double floor_abs = *floor_p;
  for (int j = tid; j < b; j += blockDim.x) {
    double mjj = G3[j * b + j];
    for (int t = 0; t < a; ++t) mjj -= C3[t * b + j] * C3[t * b + j];
    const double nj = mjj > 0.0 ? sqrt(mjj) : 0.0;
    d[j] = nj;
  }
  __syncthreads();
  for (int j = tid; j < b; j += blockDim.x) {
    const double nj = d[j];
    int above = 0;
    for (int i = k1; i < b; ++i) above += d[i] > nj || (d[i] == nj && i < j);
    const bool keep = j < k1 || (above < kb - k1 && nj > floor_abs);
    dinv[j] = keep ? 1.0 / nj : 0.0;
  }
  __syncthreads();
  for (int j = tid; j < b; j += blockDim.x) d[j] = dinv[j];
  __syncthreads();
  for (int i = tid; i < b * b; i += blockDim.x) {
    const int r = i / b, c = i % b;
    double v = G3[i];
    for (int t = 0; t < a; ++t) v -= C3[t * b + r] * C3[t * b + c];
    Ms[i] = v * d[r] * d[c];
  }
}

// small scratch of the x path (its own slots: step.cu's are file-local)
enum XSlot {
  X_C1, X_OG, X_TA, X_TB, X_SIG, X_M2, X_PC, X_INFO, X_EYE, X_TCA, X_TCB, X_GT,
  X_FV, X_MST, X_G, X_L0, X_LW, X_Z, X_BV, X_VHC, X_RV, X_SH, X_VHR, X_FH, X_ROWS, X_H, X_BI,
  X_LEFT, X_HU, X_COEF, X_LCOL, X_LNEW, X_VTC, X_RT, X_PROJ, X_PROJ2, X_GTV, X_TAZ, X_QV,
  X_VN, X_DEF, X_COEFD, X_ROWSJ, X_TMP, X_COUNT
};

}  // namespace

// ------------------------------------------------------------ blocked views
static double* xs(Handle& h, int s, size_t count) {
  if ((int)h.xsm.size() < X_COUNT) h.xsm.resize(X_COUNT);
  return h.xsm[s].get(count > 0 ? count : 1);
}

BMat bview(Handle& h, std::vector<NBuf>& bufs, int cols) {
  const int nb = nblk(cols);
  if ((int)bufs.size() < nb) bufs.resize(nb);
  BMat v;
  for (int b = 0; b < nb; ++b) v.push_back(bufs[b].view(h.g, b + 1 < nb ? XB : cols - XB * b, h.st));
  return v;
}

int bcols(const BMat& m) {
  int c = 0;
  for (const NMat& x : m) c += x.cols;
  return c;
}

// X^T diag(w) Y -> out (X.cols x Y.cols, row-major, ld = Y.cols); sym: X == Y
void bm_gram(Handle& h, const BMat& X, const BMat& Y, double* out, const double* w, bool sym) {
  const Geom& g = h.g;
  cudaStream_t st = h.st;
  const int ld = bcols(Y);
  double* tmp = xs(h, X_TMP, (size_t)XB * 2 * XB);
  for (size_t i = 0, r0 = 0; i < X.size(); r0 += X[i].cols, ++i) {
    size_t j = sym ? i : 0;
    int c0 = 0;
    for (size_t q = 0; q < j; ++q) c0 += Y[q].cols;
    for (; j < Y.size(); j += 2) {
      const bool two = j + 1 < Y.size();
      const int wc = Y[j].cols + (two ? Y[j + 1].cols : 0);
      if (two) gram_xy2(g, X[i], Y[j], Y[j + 1], tmp, h.part, st, w);
      else gram_xy(g, X[i], Y[j], tmp, h.part, st, w);
      place_kernel<<<gsz((long)X[i].cols * wc), 256, 0, st>>>(tmp, X[i].cols, wc, out, ld,
                                                               (int)r0, c0);
      launched();
      c0 += wc;
    }
  }
  if (sym) {
    mirror_kernel<<<gsz((long)ld * ld), 256, 0, st>>>(out, ld);
    launched();
  }
}

// out = sum_t scale_t In_t T_t (T_t: In_t.cols x out.cols row-major; T_t == nullptr:
// In_t has out's column blocks and is added as is)
void bm_lincomb(Handle& h, const std::vector<XTerm>& terms, const BMat& out) {
  const Geom& g = h.g;
  cudaStream_t st = h.st;
  const int nbo = bcols(out);
  double* TA = xs(h, X_TCA, (size_t)4 * XB * XB);
  double* TB = xs(h, X_TCB, (size_t)2 * XB * XB);
  struct Item {
    NMat m;
    TSeg seg;
  };
  for (size_t jb = 0, c0 = 0; jb < out.size(); c0 += out[jb].cols, ++jb) {
    const int bj = out[jb].cols;
    std::vector<Item> items;
    for (const XTerm& t : terms) {
      if (!t.T) {
        items.push_back({(*t.in)[jb], TSeg{nullptr, 0, 0, bj, 1, t.scale}});
        continue;
      }
      int r0 = 0;
      for (const NMat& blk : *t.in) {
        items.push_back({blk, TSeg{t.T, t.ld ? t.ld : nbo, r0, blk.cols, 0, t.scale}});
        r0 += blk.cols;
      }
    }
    if (items.empty()) fail(PND_ECONFIG, "bm_lincomb: no terms");
    size_t pos = 0;
    NMat partial{};
    int pingpong = 0;
    while (pos < items.size()) {
      // [Y1 | Y2] TA - X TB: first pass Y1, Y2 = items, later Y1 = the partial sum
      std::vector<const Item*> ys;
      TCat ta{};
      ta.c0 = (int)c0;
      ta.nb = bj;
      NMat Y1{}, Y2{}, Xm{};
      if (partial.p) {
        Y1 = partial;
        ta.s[ta.nseg++] = TSeg{nullptr, 0, 0, bj, 1, 1.0};
      } else {
        Y1 = items[pos].m;
        ta.s[ta.nseg++] = items[pos].seg;
        ++pos;
      }
      if (pos < items.size()) {
        Y2 = items[pos].m;
        ta.s[ta.nseg++] = items[pos].seg;
        ++pos;
      }
      TCat tb{};
      tb.c0 = (int)c0;
      tb.nb = bj;
      if (pos < items.size()) {
        Xm = items[pos].m;
        tb.s[tb.nseg] = items[pos].seg;
        tb.s[tb.nseg].scale = -tb.s[tb.nseg].scale;
        ++tb.nseg;
        ++pos;
      }
      // the ident segment of a TSeg is I_bj (the partial or an identity term)
      int rows = 0;
      for (int q = 0; q < ta.nseg; ++q) rows += ta.s[q].rows;
      tcat_kernel<<<gsz((long)rows * bj), 256, 0, st>>>(ta, TA);
      launched();
      if (tb.nseg) {
        tcat_kernel<<<gsz((long)Xm.cols * bj), 256, 0, st>>>(tb, TB);
        launched();
      }
      const bool last = pos >= items.size();
      // the partial sums share the K-stage chain temporaries (not live here)
      NMat dst = last ? out[jb] : h.wide_tmp[pingpong].view(g, bj, st);
      lincomb(g, Y1, Y2, Xm, TA, tb.nseg ? TB : nullptr, dst, nullptr, h.part, st);
      partial = dst;
      pingpong ^= 1;
    }
  }
}

// ------------------------------------------------------------ layout changes
// The two layouts never need their buffers at the same time: a layout change
// frees the other one's n-side buffers (at 256^3 a rank-64 row-major set and
// a rank-110 blocked set together exceed the 180 GB).
static void release(NBuf& b) {
  b.d.free_();
  b.rs = -1;
}

void release_narrow(Handle& h) {
  CK(cudaStreamSynchronize(h.st));
  for (NBuf* b : {&h.U, &h.Q, &h.Un, &h.Qa, &h.W1, &h.W2}) release(*b);
  for (std::vector<NBuf>* v : {&h.wide_u0b, &h.wide_qb, &h.wide_w1b, &h.wide_w2b, &h.wide_gb})
    for (NBuf& b : *v) release(b);
}

void release_blocked(Handle& h) {
  CK(cudaStreamSynchronize(h.st));
  for (std::vector<NBuf>* v : {&h.xU, &h.xQ, &h.xUn, &h.xW1, &h.xW2})
    for (NBuf& b : *v) release(b);
}

// the state's U (ua columns) in row-major form -> blocks (and Q likewise)
void to_blocked(Handle& h) {
  if (h.blocked) return;
  const Geom& g = h.g;
  auto cut = [&](NMat src, std::vector<NBuf>& dst) {
    BMat b = bview(h, dst, src.cols);
    for (size_t i = 0, c0 = 0; i < b.size(); c0 += b[i].cols, ++i) {
      cut_kernel<<<gsz((long)g.n * b[i].rs), 256, 0, h.st>>>(src, (int)c0, b[i], g.n);
      launched();
    }
  };
  if (h.ua > 0) cut(h.U.view(g, h.ua, h.st), h.xU);
  if (h.uq > 0) cut(h.Q.view(g, h.uq, h.st), h.xQ);
  h.blocked = true;
  release_narrow(h);
}

// blocks -> row-major U (ua <= 64) when the rank has come down again
void from_blocked(Handle& h) {
  if (!h.blocked) return;
  if (h.uq > 0 || h.ua > 64) return;
  const Geom& g = h.g;
  const BMat b = bview(h, h.xU, h.ua);
  const NMat U = h.U.view(g, h.ua, h.st);
  for (size_t i = 0, c0 = 0; i < b.size(); c0 += b[i].cols, ++i) {
    paste_kernel<<<gsz((long)g.n * b[i].cols), 256, 0, h.st>>>(b[i], (int)c0, U, g.n);
    launched();
  }
  h.blocked = false;
  release_blocked(h);
}

BMat xstate_u(Handle& h) { return bview(h, h.xU, h.ua); }
BMat xstate_q(Handle& h) { return h.uq > 0 ? bview(h, h.xQ, h.uq) : BMat{}; }

static double* eye_x(Handle& h, int b) {
  double* I = xs(h, X_EYE, (size_t)b * b);
  eye_x_kernel<<<gsz((long)b * b), 256, 0, h.st>>>(I, b);
  launched();
  return I;
}

void consolidate_x(Handle& h) {
  if (h.uq <= 0) return;
  const int a = h.ua, k = h.uq, ru = a + k;
  double* I = eye_x(h, ru);  // [I_a 0; 0 I_k] rows: U -> rows 0..a, Q -> rows a..
  BMat u = xstate_u(h), q = xstate_q(h);
  BMat out = bview(h, h.xUn, ru);
  bm_lincomb(h, {XTerm{&u, I, 1.0}, XTerm{&q, I + (size_t)a * ru, 1.0}}, out);
  std::swap(h.xU, h.xUn);
  h.ua = ru;
  h.uq = 0;
}

// ------------------------------------------------------------ augmentation
// orth_complement (step.cu) on blocks: Q = orthonormal basis of (I - U0 U0^T) X
int orth_complement_x(Handle& h, const BMat& X, const double* C1, int rank_bound) {
  const int a = h.ua, b = bcols(X);
  cudaStream_t st = h.st;
  const BMat U0 = a > 0 ? xstate_u(h) : BMat{};
  double* C2 = xs(h, X_OG, (size_t)b * (a + b) + 1);
  double* G2 = C2 + (size_t)a * b;
  double* TA = xs(h, X_TA, (size_t)b * b);
  double* TB = xs(h, X_TB, (size_t)(a > 0 ? a : 1) * b);
  double* sig = xs(h, X_SIG, (size_t)b + 2);
  double* dinfo = xs(h, X_DEF, 4);
  int* info = h.iflag.get(8);
  double* I = eye_x(h, b);
  // pass 2: Y = X - U0 C1 -> xW1 (free once the K stages are done; X is in
  // xW2), C2 = U0^T Y, G2 = Y^T Y
  const BMat Y = bview(h, h.xW1, b);
  if (a > 0) bm_lincomb(h, {XTerm{&X, nullptr, 1.0}, XTerm{&U0, C1, -1.0}}, Y);
  else bm_lincomb(h, {XTerm{&X, I, 1.0}}, Y);
  if (a > 0) bm_gram(h, U0, Y, C2, nullptr, false);
  bm_gram(h, Y, Y, G2, nullptr, true);
  if (a > 0) gemm(b, b, a, -1.0, tr(rowm(C2, b)), 0, rowm(C2, b), 0, 1.0, rowm(G2, b), 0, 1, st);
  cholqr_build(G2, C2, a, b, 0, 1e-14, nullptr, TA, TB, info, sig, h.cq_work, st);
  CK(cudaMemcpyAsync(h.pinned + 8, info, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h.pinned + 11, sig, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  int k = *(int*)(h.pinned + 8);
  const double lam0 = h.pinned[11];
  h.uq = 0;
  const bool level2 = k < b && k < rank_bound && lam0 > 0.0;
  if (k == 0 && !level2) return 0;
  double* C3 = C2;
  BMat Qv;
  if (level2) {
    cholqr_build(G2, C2, a, b, 2, 1e-14, nullptr, TA, TB, info, nullptr, h.cq_work, st);
    xnorm_x<<<1, 256, 0, st>>>(G2, a > 0 ? C1 : nullptr, a, b, 1e-13, dinfo + 1);
    launched();
    // pass 3': W = Y TA - U0 TB (b cols) -> xQ, C3 = U0^T W, G3 = W^T W
    const BMat W = bview(h, h.xQ, b);
    if (a > 0) bm_lincomb(h, {XTerm{&Y, TA, 1.0}, XTerm{&U0, TB, -1.0}}, W);
    else bm_lincomb(h, {XTerm{&Y, TA, 1.0}}, W);
    double* G3 = C3 + (size_t)a * b;
    if (a > 0) bm_gram(h, U0, W, C3, nullptr, false);
    bm_gram(h, W, W, G3, nullptr, true);
    double* Ms = xs(h, X_M2, (size_t)b * b);
    double* dinv = xs(h, X_PC, (size_t)b);
    level2_gram_x<<<1, 256, 0, st>>>(G3, C3, a, b, k, rank_bound < b ? rank_bound : b, dinfo + 1,
                                     Ms, dinv);
    launched();
    cholqr_build(Ms, C3, a, b, 3, 1e-14, dinv, TA, TB, info + 2, nullptr, h.cq_work, st);
    CK(cudaMemcpyAsync(h.pinned + 8, info + 2, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    k = *(int*)(h.pinned + 8);
    if (k == 0) return 0;
    // pass 4': Q = W T - U0 TB -> xUn blocks, swapped into xQ
    Qv = bview(h, h.xUn, k);
    if (a > 0) bm_lincomb(h, {XTerm{&W, TA, 1.0}, XTerm{&U0, TB, -1.0}}, Qv);
    else bm_lincomb(h, {XTerm{&W, TA, 1.0}}, Qv);
    std::swap(h.xQ, h.xUn);
    Qv = bview(h, h.xQ, k);
  } else {
    Qv = bview(h, h.xQ, k);
    if (a > 0) bm_lincomb(h, {XTerm{&Y, TA, 1.0}, XTerm{&U0, TB, -1.0}}, Qv);
    else bm_lincomb(h, {XTerm{&Y, TA, 1.0}}, Qv);
  }
  double* G3 = C3 + (size_t)a * k;
  if (a > 0) bm_gram(h, U0, Qv, C3, nullptr, false);
  bm_gram(h, Qv, Qv, G3, nullptr, true);
  defect_gc_x<<<1, 256, 0, st>>>(G3, C3, a, k, dinfo);
  launched();
  CK(cudaMemcpyAsync(h.pinned + 9, dinfo, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h.pinned[9] > 1e-12) {
    double* G3c = xs(h, X_M2, (size_t)k * k);
    CK(cudaMemcpyAsync(G3c, G3, sizeof(double) * k * k, cudaMemcpyDeviceToDevice, st));
    if (a > 0)
      gemm(k, k, a, -1.0, tr(rowm(C3, k)), 0, rowm(C3, k), 0, 1.0, rowm(G3c, k), 0, 1, st);
    cholqr_build(G3c, C3, a, k, 1, 0.0, nullptr, TA, TB, info + 1, nullptr, h.cq_work, st);
    const BMat Q2 = bview(h, h.xUn, k);
    if (a > 0) bm_lincomb(h, {XTerm{&Qv, TA, 1.0}, XTerm{&U0, TB, -1.0}}, Q2);
    else bm_lincomb(h, {XTerm{&Qv, TA, 1.0}}, Q2);
    std::swap(h.xQ, h.xUn);
  }
  h.uq = k;
  return k;
}

// ------------------------------------------------------------ streaming step
// K stage chained over blocks: out_j = S^-1? (U0 S0[:, j] + sum_x sum_s (D_s S^-1 X_x) M_s[x, j])
// (the base rows' bm_lincomb uses wide_tmp for its partial sums before the
// chain below takes them over)
static void kstage_x(Handle& h, const BMat& X, const BMat& U0, const double* S0, const double* M,
                     const BMat& out, bool in_scaled, bool out_scaled) {
  const Geom& g = h.g;
  cudaStream_t st = h.st;
  const int ns = g.ns, xc = bcols(X), b = bcols(out);
  double* I = h.wide_i.get((size_t)XB * XB);
  double* Ms = h.wide_m.get((size_t)ns * XB * XB + 1);
  for (size_t ob = 0, o0 = 0; ob < out.size(); o0 += out[ob].cols, ++ob) {
    const int bo = out[ob].cols;
    eye_x_kernel<<<1, 256, 0, st>>>(I, bo);
    launched();
    NMat base{};
    if (!U0.empty()) {
      // U0 S0[:, ob]: S0 is (a x b); the term's T restricted to block ob's columns
      BMat bb{h.wide_base.view(g, bo, st)};
      // bm_lincomb writes out-block 0 from columns [0, bo) of T: pass S0 shifted by o0
      // through a one-block output whose column offset is o0 (T = S0 + o0, ld b)
      std::vector<XTerm> t{XTerm{&U0, S0 + o0, 1.0, (int)b}};
      bm_lincomb(h, t, bb);
      base = bb[0];
    }
    for (size_t xb = 0, x0 = 0; xb < X.size(); x0 += X[xb].cols, ++xb) {
      const bool last = xb + 1 == X.size();
      // M (ns x xc x b) -> Ms (ns x bx x bo)
      const int bx = X[xb].cols;
      for (int s = 0; s < ns; ++s)
        CK(cudaMemcpy2DAsync(Ms + (size_t)s * bx * bo, bo * sizeof(double),
                             M + ((size_t)s * xc + x0) * b + o0, b * sizeof(double),
                             bo * sizeof(double), bx, cudaMemcpyDeviceToDevice, st));
      KStageArgs ka{};
      ka.bcat = &h.bcat;
      ka.geo = g;
      ka.inv_s = h.isp.p + 2 * (size_t)g.halo;
      ka.X = X[xb];
      ka.U0 = base;
      ka.S0 = I;
      ka.M = Ms;
      ka.out = last ? out[ob] : h.wide_tmp[xb & 1].view(g, bo, st);
      ka.in_scaled = in_scaled;
      ka.out_scaled = last && out_scaled;
      kstage(ka, st);
      base = ka.out;
    }
  }
}

void moment_factors_x(Handle& h, double* W, int c, double* out) {
  const int m = h.m, ns = h.g.ns;
  double* Y = xs(h, X_MST, (size_t)ns * m * c);
  gemm(ns * m, c, m, 1.0, rowm(h.amat.p, m), 0, rowm(W, c), 0, 0.0, rowm(Y, c), 0, 1, h.st);
  gemm(c, c, m, 1.0, tr(rowm(W, c)), 0, rowm(Y, c), (long)m * c, 0.0, rowm(out, c), (long)c * c,
       ns, h.st);
}

void streaming_step_x(Handle& h, double dt) {
  to_blocked(h);
  consolidate_x(h);
  const Geom& g = h.g;
  const int m = h.m, ns = g.ns;
  const int a = h.ua, b = h.rv;
  cudaStream_t st = h.st;
  const BMat U0 = xstate_u(h);
  const double* isp = h.isp.p + 2 * (size_t)g.halo;
  for (const NMat& x : U0) comm_halo_rows(g, x.p, x.rs, st);
  const BMat W1 = bview(h, h.xW1, b), W2 = bview(h, h.xW2, b);

  phase(h, PH_LSIDE);
  double* F = xs(h, X_FV, (size_t)ns * b * b);
  moment_factors_x(h, h.V.p, b, F);
  const int xmax = a > b ? a : b;
  double* M = xs(h, X_G, (size_t)ns * xmax * b);
  const double coef[4] = {0.25, 1.0 / 3.0, 0.5, 1.0};
  for (int stage = 0; stage < 4; ++stage) {
    const double c = -coef[stage] * dt;
    if (stage == 0)
      gemm(a, b, b, c, rowm(h.S.p, b), 0, rowm(F, b), (long)b * b, 0.0, rowm(M, b), (long)a * b,
           ns, st);
    else
      axpby(ns * b * b, c, F, 0.0, M, st);
    phase(h, PH_KSTAGE);
    const BMat& xin = stage == 0 ? U0 : stage == 2 ? W2 : W1;
    if (stage > 0)
      for (const NMat& x : xin) comm_halo_rows(g, x.p, x.rs, st);
    kstage_x(h, xin, stage == 3 ? BMat{} : U0, h.S.p, M, stage == 0 || stage == 2 ? W1 : W2,
             stage > 0, stage < 3);
    phase(h, PH_LSIDE);
  }
  const BMat& dK = W2;
  double* C1 = xs(h, X_C1, (size_t)a * b);
  phase(h, PH_LGRAM);
  bm_gram(h, U0, dK, C1, nullptr, false);
  phase(h, PH_ORTH);
  const int k = orth_complement_x(h, dK, C1, 1 << 30);
  const int ru = a + k;

  double* G = xs(h, X_Z, (size_t)ns * ru * ru);
  phase(h, PH_SGRAM);
  BMat blocks = U0;
  if (k > 0) {
    const BMat Q = xstate_q(h);
    for (const NMat& q : Q) {
      comm_halo_rows(g, q.p, q.rs, st);
      blocks.push_back(q);
    }
  }
  // every (A, B) block pair: one rectangular launch (features of B formed
  // once per pair, no diagonal-block recomputation), one allreduce at the end
  stencil_grams_blocks(h, blocks, isp, G);

  phase(h, PH_LSIDE);
  const int cols = a + b;
  double* L0 = xs(h, X_L0, (size_t)m * a);
  double* LW = xs(h, X_LW, (size_t)m * a);
  double* Z = xs(h, X_H, (size_t)ns * m * a);
  gemm(m, a, b, 1.0, rowm(h.V.p, b), 0, tr(rowm(h.S.p, b)), 0, 0.0, rowm(L0, a), 0, 1, st);
  CK(cudaMemcpyAsync(LW, L0, sizeof(double) * m * a, cudaMemcpyDeviceToDevice, st));
  double* BV = xs(h, X_BV, (size_t)m * cols);
  double* M2 = xs(h, X_M2, (size_t)m * a);
  for (int stage = 0; stage < 4; ++stage) {
    gemm(m, a, a, 1.0, rowm(LW, a), 0, tr(rowm(G, ru)), (long)ru * ru, 0.0, rowm(Z, a),
         (long)m * a, ns, st);
    double* dst = stage == 3 ? M2 : LW;
    CK(cudaMemcpyAsync(dst, L0, sizeof(double) * m * a, cudaMemcpyDeviceToDevice, st));
    gemm(m, a, ns * m, -coef[stage] * dt, tr(rowm(h.amat.p, m)), 0, rowm(Z, a), 0, 1.0,
         rowm(dst, a), 0, 1, st);
    if (stage == 3) transpose_in(dst, m, a, BV, m, st);
  }
  transpose_in(h.V.p, m, b, BV + (size_t)a * m, m, st);
  double* Vhc = xs(h, X_VHC, (size_t)m * cols);
  double* Rv = xs(h, X_RV, (size_t)cols * cols);
  phase(h, PH_TSQR_M);
  const int rv = tsqr(BV, m, cols, m, Vhc, m, Rv, h.tq_m, st);
  phase(h, PH_SRK4);
  double* Sh = xs(h, X_SH, (size_t)ru * rv);
  gemm(a, rv, b, 1.0, rowm(h.S.p, b), 0, Mat{Rv + a, 1, cols}, 0, 0.0, rowm(Sh, rv), 0, 1, st);
  if (k > 0) {
    zero_rows_x_kernel<<<gsz((long)k * rv), 256, 0, st>>>(Sh, a, k, rv);
    launched();
  }
  double* Vhr = xs(h, X_VHR, (size_t)m * rv);
  transpose_out(Vhc, m, m, rv, Vhr, st);
  double* Fh = xs(h, X_FH, (size_t)ns * rv * rv);
  moment_factors_x(h, Vhr, rv, Fh);
  s_rk4(Sh, ru, rv, G, Fh, ns, dt, nullptr, st);
  double* Snew = h.S.get((size_t)ru * rv);
  CK(cudaMemcpyAsync(Snew, Sh, sizeof(double) * ru * rv, cudaMemcpyDeviceToDevice, st));
  double* Vnew = h.V.get((size_t)m * rv);
  CK(cudaMemcpyAsync(Vnew, Vhr, sizeof(double) * m * rv, cudaMemcpyDeviceToDevice, st));
  h.ru = ru;
  h.rv = rv;
  phase(h, -1);
}

// ------------------------------------------------------------ scattering step
void scattering_step_x(Handle& h, double dt) {
  to_blocked(h);
  consolidate_x(h);
  const Geom& g = h.g;
  const int m = h.m;
  const int a = h.ua, b = h.rv;
  const int B = h.n_beams;
  cudaStream_t st = h.st;
  const BMat U0 = xstate_u(h);

  phase(h, PH_SCATSMALL);
  double* gt = xs(h, X_GT, (size_t)(B > 0 ? B : 1) * 12 * m);
  double* rows = xs(h, X_ROWS, (size_t)(B > 0 ? B : 1) * 12 * b);
  if (B > 0) {
    gt_x_kernel<<<64, 256, 0, st>>>(h.gdiag.p, h.tm.p, m, B, gt);
    launched();
    gemm(12 * B, b, m, 1.0, rowm(gt, m), 0, rowm(h.V.p, b), 0, 0.0, rowm(rows, b), 0, 1, st);
  }
  const bool rank1 = h.n_cls == 1 && B == 1;
  const BMat psi_col{NMat{h.psi.p, 1, 1}};

  // substep 2 increment dK = dt src_rows(V0) (dlra.py:303), block by block
  const BMat dK = bview(h, h.xW2, b);
  phase(h, PH_SCATK1);
  NMat Z{};
  double* rj = xs(h, X_ROWSJ, (size_t)(B > 0 ? B : 1) * 12 * XB);
  if (B > 0 && !rank1) {
    Z = h.Xs.view(g, 12 * B, st);
    source_rows(g, h.inv_s.p, h.cls.p, h.cls_atomic.p, h.psi.p, B, Z, st);
  }
  for (size_t j = 0, c0 = 0; j < dK.size(); c0 += dK[j].cols, ++j) {
    const int bj = dK[j].cols;
    if (B == 0) {
      fill_zero(dK[j].p, (size_t)g.n * dK[j].rs, st);
      continue;
    }
    CK(cudaMemcpy2DAsync(rj, bj * sizeof(double), rows + c0, b * sizeof(double),
                         bj * sizeof(double), 12 * B, cudaMemcpyDeviceToDevice, st));
    if (rank1) {
      scat_dk(g, dt, h.inv_s.p, h.cls.p, h.cls_atomic.p, 1, h.psi.p, 1, rj, dK[j], st);
    } else {
      axpby(12 * B * bj, dt, rj, 0.0, rj, st);
      lincomb(g, Z, NMat{}, NMat{}, rj, nullptr, dK[j], nullptr, h.part, st);
    }
  }

  // substep 1: B_i = U0^T diag(N_i / S) U0 (dlra.py:284-285)
  const int nw = h.n_cls <= 12 ? h.n_cls : 12;
  double* H = xs(h, X_H, (size_t)nw * a * a);
  phase(h, PH_SCATGRAM);
  double* left = xs(h, X_LEFT, (size_t)a * 12 * (B > 0 ? B : 1));
  if (rank1) {
    bm_gram(h, U0, U0, H, h.inv_s.p, true);
    double* u = xs(h, X_HU, (size_t)a);
    bm_gram(h, U0, psi_col, u, h.inv_s.p, false);
    gemm(a, 12, 1, 1.0, Mat{u, 1, 1}, 0, rowm(h.cls_atomic.p, 12), 0, 0.0, rowm(left, 12), 0, 1,
         st);
  } else if (h.n_cls == 1) {
    bm_gram(h, U0, U0, H, h.inv_s.p, true);
  } else {
    double* wv = h.wide_t.get((size_t)g.ld + 64);
    for (int i = 0; i < nw; ++i) {
      class_weight_x_kernel<<<148 * 8, 256, 0, st>>>(h.cls.p, h.cls_atomic.p, h.inv_s.p, g.n,
                                                      h.n_cls <= 12 ? -1 : i, i, wv);
      launched();
      bm_gram(h, U0, U0, H + (size_t)i * a * a, wv, true);
    }
  }
  phase(h, PH_SCATSMALL);
  double* Bi = xs(h, X_BI, (size_t)12 * a * a);
  if (h.n_cls <= 12)
    gemm(12, a * a, h.n_cls, 1.0, tr(rowm(h.cls_atomic.p, 12)), 0, rowm(H, a * a), 0, 0.0,
         rowm(Bi, a * a), 0, 1, st);
  else
    CK(cudaMemcpyAsync(Bi, H, sizeof(double) * 12 * a * a, cudaMemcpyDeviceToDevice, st));
  phase(h, PH_SCATGRAM);
  if (B > 0 && !rank1) bm_gram(h, U0, BMat{Z}, left, nullptr, false);
  phase(h, PH_SCATSMALL);
  double* C1 = xs(h, X_C1, (size_t)a * b);
  if (B > 0) {
    for (int beam = 0; beam < B; ++beam)
      gemm(a, b, 12, dt, Mat{left + beam * 12, 12 * B, 1}, 0,
           rowm(rows + (size_t)beam * 12 * b, b), 0, beam == 0 ? 0.0 : 1.0, rowm(C1, b), 0, 1,
           st);
  } else {
    fill_zero(C1, (size_t)a * b, st);
  }
  double* coeffs = xs(h, X_COEF, (size_t)12 * m);
  coeff_x_kernel<<<16, 256, 0, st>>>(h.gdiag.p, h.sigt.p, m, coeffs);
  launched();
  double* lcols = xs(h, X_LCOL, (size_t)a * m);
  gemm(a, m, b, 1.0, rowm(h.S.p, b), 0, tr(rowm(h.V.p, b)), 0, 0.0, rowm(lcols, m), 0, 1, st);
  double* lnew = xs(h, X_LNEW, (size_t)a * m);
  int* flag = h.iflag.get(8);
  init_int_x<<<1, 1, 0, st>>>(flag + 4, 1 << 30);
  launched();
  scat_solves(Bi, coeffs, lcols, a, m, dt, lnew, flag + 4, st);
  CK(cudaMemcpyAsync(h.pinned + 10, flag + 4, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (*(int*)(h.pinned + 10) != (1 << 30))
    fail(PND_ENUMERICAL, "implicit scattering solve singular at moment column " +
                             std::to_string(*(int*)(h.pinned + 10)) +
                             "; the step size is too large for the scattering stiffness");
  phase(h, PH_TSQR_M);
  const int kt = m < a ? m : a;
  double* Vtc = xs(h, X_VTC, (size_t)m * kt);
  double* Rt = xs(h, X_RT, (size_t)kt * a);
  tsqr(lnew, m, a, m, Vtc, m, Rt, h.tq_m, st);

  phase(h, PH_ORTH);
  const int bound = rank1 ? 1 : (long)h.n_cls * B < b ? h.n_cls * B : b;
  const int k = orth_complement_x(h, dK, C1, bound);
  const int ru = a + k;
  phase(h, PH_SCATSMALL);

  const int vcols = a + kt;
  double* BV = xs(h, X_BV, (size_t)m * vcols);
  double* proj = xs(h, X_PROJ, (size_t)a * m);
  gemm(m, a, kt, 1.0, colm(Vtc, m), 0, rowm(Rt, a), 0, 0.0, colm(BV, m), 0, 1, st);
  if (B > 0) {
    for (int beam = 0; beam < B; ++beam)
      gemm(a, m, 12, 1.0, Mat{left + beam * 12, 12 * B, 1}, 0,
           rowm(gt + (size_t)beam * 12 * m, m), 0, beam == 0 ? 0.0 : 1.0, rowm(proj, m), 0, 1,
           st);
    axpby(a * m, dt, proj, 1.0, BV, st);
  }
  CK(cudaMemcpyAsync(BV + (size_t)a * m, Vtc, sizeof(double) * m * kt, cudaMemcpyDeviceToDevice,
                     st));
  double* Vhc = xs(h, X_VHC, (size_t)m * vcols);
  double* Rv = xs(h, X_RV, (size_t)vcols * vcols);
  phase(h, PH_TSQR_M);
  const int rv = tsqr(BV, m, vcols, m, Vhc, m, Rv, h.tq_m, st);
  phase(h, PH_SCATSMALL);
  double* Sh = xs(h, X_SH, (size_t)ru * rv);
  gemm(a, rv, kt, 1.0, tr(rowm(Rt, a)), 0, Mat{Rv + a, 1, vcols}, 0, 0.0, rowm(Sh, rv), 0, 1,
       st);
  if (k > 0) {
    zero_rows_x_kernel<<<gsz((long)k * rv), 256, 0, st>>>(Sh, a, k, rv);
    launched();
  }
  if (B > 0) {
    double* proj2 = xs(h, X_PROJ2, (size_t)ru * 12 * B);
    CK(cudaMemcpyAsync(proj2, left, sizeof(double) * a * 12 * B, cudaMemcpyDeviceToDevice, st));
    if (k > 0) {
      phase(h, PH_SCATGRAM);
      const BMat Q = xstate_q(h);
      if (rank1) {
        double* qv = xs(h, X_QV, (size_t)k);
        bm_gram(h, Q, psi_col, qv, h.inv_s.p, false);
        gemm(k, 12, 1, 1.0, Mat{qv, 1, 1}, 0, rowm(h.cls_atomic.p, 12), 0, 0.0,
             rowm(proj2 + (size_t)a * 12, 12), 0, 1, st);
      } else {
        bm_gram(h, Q, BMat{Z}, proj2 + (size_t)a * 12 * B, nullptr, false);
      }
      phase(h, PH_SCATSMALL);
    }
    double* gtv = xs(h, X_GTV, (size_t)B * 12 * rv);
    gemm(12 * B, rv, m, 1.0, rowm(gt, m), 0, colm(Vhc, m), 0, 0.0, rowm(gtv, rv), 0, 1, st);
    for (int beam = 0; beam < B; ++beam)
      gemm(ru, rv, 12, dt, Mat{proj2 + beam * 12, 12 * B, 1}, 0,
           rowm(gtv + (size_t)beam * 12 * rv, rv), 0, 1.0, rowm(Sh, rv), 0, 1, st);
  }
  double* Snew = h.S.get((size_t)ru * rv);
  CK(cudaMemcpyAsync(Snew, Sh, sizeof(double) * ru * rv, cudaMemcpyDeviceToDevice, st));
  double* Vnew = h.V.get((size_t)m * rv);
  transpose_out(Vhc, m, m, rv, Vnew, st);
  h.ru = ru;
  h.rv = rv;
  phase(h, -1);
}

// ------------------------------------------------------------ truncation
// the rotation U1 = [U | Q] P[:, :r1] into blocks (from a blocked or a
// row-major augmented state); ugram (r1 x r1): U1^T U1 for the defect
void rotate_x(Handle& h, const double* P, int p, int kcols, int r1, bool all_zero,
              double* ugram) {
  const Geom& g = h.g;
  cudaStream_t st = h.st;
  const BMat Un = bview(h, h.xUn, r1);
  if (all_zero) {
    for (size_t j = 0, c0 = 0; j < Un.size(); c0 += Un[j].cols, ++j) {
      unit_block_kernel<<<gsz((long)g.n * Un[j].rs), 256, 0, st>>>(g, Un[j], (int)c0);
      launched();
    }
  } else {
    double* Pc = xs(h, X_PC, (size_t)p * r1);
    CK(cudaMemcpy2DAsync(Pc, r1 * sizeof(double), P, kcols * sizeof(double), r1 * sizeof(double),
                         p, cudaMemcpyDeviceToDevice, st));
    if (h.blocked) {
      const BMat u = xstate_u(h), q = xstate_q(h);
      std::vector<XTerm> t{XTerm{&u, Pc, 1.0}};
      if (!q.empty()) t.push_back(XTerm{&q, Pc + (size_t)h.ua * r1, 1.0});
      bm_lincomb(h, t, Un);
    } else {
      // row-major [U | Q] (<= 64 + 64 columns): one LINCOMB per output block
      const NMat u = state_u(h), q = state_q(h);
      double* Tj = xs(h, X_TCA, (size_t)p * XB);
      for (size_t j = 0, c0 = 0; j < Un.size(); c0 += Un[j].cols, ++j) {
        CK(cudaMemcpy2DAsync(Tj, Un[j].cols * sizeof(double), Pc + c0, r1 * sizeof(double),
                             Un[j].cols * sizeof(double), p, cudaMemcpyDeviceToDevice, st));
        lincomb(g, u, q, NMat{}, Tj, nullptr, Un[j], nullptr, h.part, st);
      }
    }
  }
  if (ugram) bm_gram(h, Un, Un, ugram, nullptr, true);
  std::swap(h.xU, h.xUn);
  if (!h.blocked) release_narrow(h);
  h.blocked = true;
  h.ua = r1;
  h.uq = 0;
}

void dose_accumulate_x(Handle& h, const double* coef, double half_dt, const double* psi,
                       double* dep, double* prev) {
  const BMat U = xstate_u(h);
  if ((int)U.size() > DMAXB) fail(PND_ECONFIG, "dose supports rank <= 768");
  BList bl{};
  bl.nb = (int)U.size();
  for (int i = 0; i < bl.nb; ++i) bl.b[i] = U[i];
  dose_blocks_kernel<<<gsz(h.g.n), 256, 0, h.st>>>(h.g, bl, coef, half_dt, h.s_field.p, psi,
                                                   h.n_beams, dep, prev);
  launched();
}

double orth_defect_x(Handle& h, double* G, bool have_ugram) {
  cudaStream_t st = h.st;
  double* out = G + (size_t)h.ru * h.ru + (size_t)h.rv * h.rv;
  if (!have_ugram) {
    const BMat U = xstate_u(h);
    bm_gram(h, U, U, G, nullptr, true);
  }
  double* GV = G + (size_t)h.ru * h.ru;
  gemm(h.rv, h.rv, h.m, 1.0, tr(rowm(h.V.p, h.rv)), 0, rowm(h.V.p, h.rv), 0, 0.0,
       rowm(GV, h.rv), 0, 1, st);
  fill_zero(out, 1, st);
  defect_x_kernel<<<1, 256, 0, st>>>(G, h.ru, out);
  launched();
  defect_x_kernel<<<1, 256, 0, st>>>(GV, h.rv, out);
  launched();
  CK(cudaMemcpyAsync(h.pinned + 2, out, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return h.pinned[2];
}

namespace {
__device__ __forceinline__ double hash_normal_x(unsigned long long x) {
  double s = 0.0;
  for (int i = 0; i < 4; ++i) {
    x += 0x9E3779B97F4A7C15ULL;
    unsigned long long z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    s += (double)(z >> 11) * (1.0 / 9007199254740992.0);
  }
  return (s - 2.0) * 1.7320508075688772;
}

// block of a pseudo-random n x cols matrix keyed by (global cell, global column)
__global__ void random_block_kernel(Geom g, NMat U, int c0, int cols, unsigned long long seed) {
  const long total = (long)g.n * U.rs;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
       e += (long)gridDim.x * blockDim.x) {
    const int c = (int)(e / U.rs), j = (int)(e - (long)c * U.rs);
    const unsigned long long key =
        (unsigned long long)(c + (long)g.z0 * g.nx * g.ny) * cols + c0 + j;
    U.p[e] = j < U.cols ? hash_normal_x(seed * 0x100000001B3ULL + key) : 0.0;
  }
}
}  // namespace

// U = orth(pseudo-random n x r) on blocks (pnd_state_random above rank 64)
int random_state_x(Handle& h, int r, unsigned long long seed) {
  if (!h.blocked) release_narrow(h);
  const BMat X = bview(h, h.xW2, r);
  for (size_t i = 0, c0 = 0; i < X.size(); c0 += X[i].cols, ++i) {
    random_block_kernel<<<gsz((long)h.g.n * X[i].rs), 256, 0, h.st>>>(h.g, X[i], (int)c0, r,
                                                                      seed);
    launched();
  }
  h.ua = 0;
  h.uq = 0;
  h.blocked = true;
  const int k = orth_complement_x(h, X, nullptr, 1 << 30);
  std::swap(h.xU, h.xQ);
  h.ua = k;
  h.uq = 0;
  return k;
}

// host <-> blocked state (pnd_state_set / pnd_state_get above rank 64)
void upload_blocked(Handle& h, const double* u, int ru) {
  if (!h.blocked) release_narrow(h);
  const BMat b = bview(h, h.xU, ru);
  for (size_t i = 0, c0 = 0; i < b.size(); c0 += b[i].cols, ++i) {
    if (b[i].rs != b[i].cols) fill_zero(b[i].p, (size_t)h.g.n * b[i].rs, h.st);
    CK(cudaMemcpy2DAsync(b[i].p, b[i].rs * sizeof(double), u + c0, ru * sizeof(double),
                         b[i].cols * sizeof(double), h.g.n, cudaMemcpyHostToDevice, h.st));
  }
  h.blocked = true;
}

void download_blocked(Handle& h, double* u, int ld) {
  const BMat b = xstate_u(h);
  int c0 = 0;
  for (const NMat& x : b) {
    CK(cudaMemcpy2DAsync(u + c0, ld * sizeof(double), x.p, x.rs * sizeof(double),
                         x.cols * sizeof(double), h.g.n, cudaMemcpyDeviceToHost, h.st));
    c0 += x.cols;
  }
  for (const NMat& x : xstate_q(h)) {
    CK(cudaMemcpy2DAsync(u + c0, ld * sizeof(double), x.p, x.rs * sizeof(double),
                         x.cols * sizeof(double), h.g.n, cudaMemcpyDeviceToHost, h.st));
    c0 += x.cols;
  }
}

}  // namespace pnd
