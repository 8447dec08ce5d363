// Ranks above 32: the stencil kernels on 32-column blocks.
//
// The K-stage and S-Gram kernels tile at most 32 input columns (the K-stage
// stages whole rows of its input, the S-Gram accumulators cover at most 64
// columns). For wider factors the n-side matrices they read are split into
// cell-major column blocks of <= 32 (the layout of the device full-rank
// solver, fullrank.cu) and the kernels are chained over the blocks:
//   K-stage:  out[:, ob] = S^-1? (U0 S0[:, ob] + sum_xb sum_s (D_s S^-1 X_xb) M_s[xb, ob])
//             -- the U0 S0 term as one LINCOMB pass, then one K-stage per input
//             block, each taking the previous partial sum as its base rows
//             (S0 = I); only the last one applies the output's 1/S;
//   S-Grams:  G_s block by block: one rectangular launch per (i, j) pair
//             (stencil_grams_rect), placed into the w x w Grams.
#include "handle.h"

namespace pnd {

namespace {

constexpr int WB = 32;

__global__ void split_kernel(NMat src, int c0, NMat dst, int n) {
  const long total = (long)n * dst.rs;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
       e += (long)gridDim.x * blockDim.x) {
    const long c = e / dst.rs;
    const int j = (int)(e - c * dst.rs);
    dst.p[e] = j < dst.cols ? src.p[c * src.rs + c0 + j] : 0.0;
  }
}

// dst = columns [c0, c0 + dst.cols) of [X1 | X2]
__global__ void split2_kernel(NMat x1, NMat x2, int c0, NMat dst, int n) {
  const long total = (long)n * dst.rs;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
       e += (long)gridDim.x * blockDim.x) {
    const long c = e / dst.rs;
    const int j = (int)(e - c * dst.rs), gc = c0 + j;
    double v = 0.0;
    if (j < dst.cols) v = gc < x1.cols ? x1.p[c * x1.rs + gc] : x2.p[c * x2.rs + gc - x1.cols];
    dst.p[e] = v;
  }
}

// M (ns x rows x ld, row-major) -> sub (ns x bx x bo): rows x0.., columns o0..
__global__ void msub_kernel(const double* __restrict__ M, int ns, int rows, int ld, int x0, int bx,
                            int o0, int bo, double* __restrict__ out) {
  const int total = ns * bx * bo;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int s = i / (bx * bo), rem = i - s * bx * bo, p = rem / bo, q = rem - p * bo;
    out[i] = M[((size_t)s * rows + x0 + p) * ld + o0 + q];
  }
}

__global__ void eye_b_kernel(double* I, int b) {
  for (int i = threadIdx.x; i < b * b; i += blockDim.x) I[i] = (i / b == i % b) ? 1.0 : 0.0;
}

int grid_n(long n) {
  long b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return b < 1 ? 1 : (int)b;
}

}  // namespace

// ceil(cols / 32) blocks of balanced width (40 -> 20 + 20: the kernels' tiles
// are fuller than with 32 + 8)
int block_width(int cols) {
  const int nb = (cols + WB - 1) / WB;
  return (cols + nb - 1) / nb;
}

std::vector<NMat> block_views(Handle& h, std::vector<NBuf>& bufs, int cols) {
  const int bw = block_width(cols), nb = (cols + bw - 1) / bw;
  if ((int)bufs.size() < nb) bufs.resize(nb);
  std::vector<NMat> v;
  for (int b = 0; b < nb; ++b) v.push_back(bufs[b].view(h.g, b + 1 < nb ? bw : cols - bw * b, h.st));
  return v;
}

std::vector<NMat> split_blocks(Handle& h, NMat src, std::vector<NBuf>& bufs) {
  std::vector<NMat> v = block_views(h, bufs, src.cols);
  int c0 = 0;
  for (size_t b = 0; b < v.size(); ++b) {
    split_kernel<<<grid_n((long)h.g.n * v[b].rs), 256, 0, h.st>>>(src, c0, v[b], h.g.n);
    launched();
    comm_halo_rows(h.g, v[b].p, v[b].rs, h.st);  // slab faces of the copy
    c0 += v[b].cols;
  }
  return v;
}

std::vector<NMat> split_joint(Handle& h, NMat X1, NMat X2, int maxw, std::vector<NBuf>& bufs) {
  const int cols = X1.cols + (X2.p ? X2.cols : 0);
  const int nb = (cols + maxw - 1) / maxw, bw = (cols + nb - 1) / nb;
  if ((int)bufs.size() < nb) bufs.resize(nb);
  std::vector<NMat> v;
  for (int b = 0, c0 = 0; b < nb; ++b, c0 += bw) {
    const NMat d = bufs[b].view(h.g, b + 1 < nb ? bw : cols - bw * b, h.st);
    split2_kernel<<<grid_n((long)h.g.n * d.rs), 256, 0, h.st>>>(X1, X2.p ? X2 : X1, c0, d, h.g.n);
    launched();
    comm_halo_rows(h.g, d.p, d.rs, h.st);
    v.push_back(d);
  }
  return v;
}

void kstage_blocks(Handle& h, const std::vector<NMat>& X, NMat U0, const double* S0,
                   const double* M, const std::vector<NMat>& out, bool in_scaled,
                   bool out_scaled) {
  const Geom& g = h.g;
  cudaStream_t st = h.st;
  const int ns = g.ns, a = U0.p ? U0.cols : 0;
  int xc = 0;
  for (const NMat& x : X) xc += x.cols;
  int b = 0;
  for (const NMat& o : out) b += o.cols;
  double* Ms = h.wide_m.get((size_t)ns * WB * WB + 1);
  double* Ts = h.wide_t.get((size_t)(a > 0 ? a : 1) * WB + 1);
  double* I = h.wide_i.get((size_t)WB * WB);
  int o0 = 0;
  for (size_t ob = 0; ob < out.size(); o0 += out[ob].cols, ++ob) {
    const int bo = out[ob].cols;
    eye_b_kernel<<<1, 256, 0, st>>>(I, bo);  // S0 of the chained partial sums
    launched();
    NMat base{};
    if (a > 0) {
      // U0 S0[:, ob] in one streaming pass
      msub_kernel<<<16, 256, 0, st>>>(S0, 1, a, b, 0, a, o0, bo, Ts);
      launched();
      base = h.wide_base.view(g, bo, st);
      lincomb(g, U0, NMat{}, NMat{}, Ts, nullptr, base, nullptr, h.part, st);
    }
    int x0 = 0;
    for (size_t xb = 0; xb < X.size(); x0 += X[xb].cols, ++xb) {
      const bool last = xb + 1 == X.size();
      msub_kernel<<<64, 256, 0, st>>>(M, ns, xc, b, x0, X[xb].cols, o0, bo, Ms);
      launched();
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

void stencil_grams_blocks(Handle& h, const std::vector<NMat>& B, const double* isp, double* G) {
  const Geom& g = h.g;
  const int ns = g.ns, nb = (int)B.size();
  int w = 0;
  std::vector<int> off;
  for (const NMat& x : B) {
    off.push_back(w);
    w += x.cols;
  }
  if (nb == 1) {
    stencil_grams(g, B[0], NMat{}, isp, G, h.part, h.st);
    return;
  }
  // every (A, B) block pair: one rectangular launch (B's features contracted
  // with A's rows), placed into the w x w Grams; one allreduce at the end
  (void)ns;
  for (int i = 0; i < nb; ++i)
    for (int j = 0; j < nb; ++j)
      stencil_grams_rect(g, B[i], B[j], isp, G, w, off[i], off[j], h.part, h.st);
  comm_allreduce(g, G, (size_t)g.ns * w * w, h.st);
}

}  // namespace pnd
