// Cell-parallel (n-side) kernels of the energy step, cell-major layout.
//
// Every n-side operation is "form per-cell feature rows, then contract them"
// and runs as FP64 tensor-core mma.sync.m8n8k4 (DMMA) on shared-memory tiles.
// The stencil kernels (kstage, stencil Grams) live in stencil.cu and the
// LINCOMB passes in lincomb.cu; this file holds the other pointwise /
// contraction kernels:
//   pgram    plain / weighted / source Grams (dlra.py:285, 307-319);
//   scat_dk, dose, transposes, unit/random rows, class gathers.
// Shared-memory tiles use row lengths = 4 (mod 16) doubles where DMMA
// fragments are read, which spreads a half-warp over 16 distinct banks.
#include "tma.cuh"

namespace pnd {

namespace {

__host__ __device__ constexpr int pad4(int w) { return ((w + 11) / 16) * 16 + 4; }
__host__ __device__ constexpr int up16(int w) { return (w + 15) / 16 * 16; }


__global__ void reduce_blocks(const double* __restrict__ partial, int nblk, int count,
                              double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int b = 0; b < nblk; ++b) s += partial[(size_t)b * count + i];
  out[i] = s;
}

template <class Kern>
int resident(Kern k, int threads, size_t smem) {
  return occupancy_cached((const void*)k, threads, smem);
}

// ===================================================================== pgram
constexpr int PC = 64;

template <int T8, int NPH>
__global__ void __launch_bounds__(256) pgram_kernel(PGramArgs a, int LS,
                                                    double* __restrict__ partial) {
  constexpr int W = T8 * 8;
  constexpr int NT = T8 * T8;
  constexpr int TPW = (NT + 7) / 8;
  extern __shared__ __align__(128) double sm[];
  double* sX = sm;             // [PC][LS]
  double* sT = sX + PC * LS;   // [PC][LS]
  const Geom& g = a.geo;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int na = a.X.cols, nb = a.nb;
  for (int i = tid; i < 2 * PC * LS; i += 256) sm[i] = 0.0;
  double acc[NPH][TPW][2];
#pragma unroll
  for (int p = 0; p < NPH; ++p)
#pragma unroll
    for (int t = 0; t < TPW; ++t) acc[p][t][0] = acc[p][t][1] = 0.0;
  const int nchunks = (g.n + PC - 1) / PC;
  for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
    const int c0 = chunk * PC;
    const int rows = g.n - c0 < PC ? g.n - c0 : PC;
    __syncthreads();
    for (int e = tid; e < PC * na; e += 256) {
      const int i = e / na, j = e - i * na;
      sX[i * LS + j] = i < rows ? a.X.p[(long)(c0 + i) * a.X.rs + j] : 0.0;
    }
#pragma unroll
    for (int p = 0; p < NPH; ++p) {
      if (p < a.nphase) {
        if (p > 0) __syncthreads();
        for (int e = tid; e < PC * nb; e += 256) {
          const int i = e / nb, j = e - i * nb;
          double v = 0.0;
          if (i < rows) {
            const int c = c0 + i;
            if (a.gen == PG_PLAIN) {
              v = a.Y.p[(long)c * a.Y.rs + j];
            } else if (a.gen == PG_WEIGHT) {
              const int k = a.cls[c];
              const double w = a.wmode == 0 ? (k == p ? a.inv_s[c] : 0.0)
                                            : a.wtab[k * 12 + p] * a.inv_s[c];
              v = w * a.Y.p[(long)c * a.Y.rs + j];
            } else {
              const int beam = j / 12, el = j - beam * 12;
              v = a.wtab[a.cls[c] * 12 + el] * (a.inv_s[c] * a.psi[(size_t)beam * a.ld + c]);
            }
          }
          sT[i * LS + j] = v;
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < TPW; ++t) {
          const int tile = warp + 8 * t;
          if (tile < NT) {
            const int ti = tile / T8, tj = tile - ti * T8;
            const double* xa = sX + (lane & 3) * LS + ti * 8 + (lane >> 2);
            const double* tb = sT + (lane & 3) * LS + tj * 8 + (lane >> 2);
#pragma unroll 4
            for (int k0 = 0; k0 < PC; k0 += 4)
              dmma884(acc[p][t][0], acc[p][t][1], xa[k0 * LS], tb[k0 * LS]);
          }
        }
      }
    }
  }
  double* out = partial + (size_t)blockIdx.x * a.nphase * na * nb;
#pragma unroll
  for (int p = 0; p < NPH; ++p) {
    if (p < a.nphase) {
#pragma unroll
      for (int t = 0; t < TPW; ++t) {
        const int tile = warp + 8 * t;
        if (tile < NT) {
          const int ti = tile / T8, tj = tile - ti * T8;
          const int row = ti * 8 + (lane >> 2), col = tj * 8 + 2 * (lane & 3);
          if (row < na) {
            double* o = out + ((size_t)p * na + row) * nb;
            if (col < nb) o[col] = acc[p][t][0];
            if (col + 1 < nb) o[col + 1] = acc[p][t][1];
          }
        }
      }
    }
  }
}

template <int T8, int NPH>
void pgram_launch(const PGramArgs& a, DBuf& partial, cudaStream_t st) {
  const int LS = pad4(T8 * 8);
  const size_t smem = 2 * (size_t)PC * LS * sizeof(double);
  allow_max_smem(pgram_kernel<T8, NPH>);
  const int nchunks = (a.geo.n + PC - 1) / PC;
  int grid = sm_count() * resident(pgram_kernel<T8, NPH>, 256, smem);
  if (grid > nchunks) grid = nchunks;
  const size_t count = (size_t)a.nphase * a.X.cols * a.nb;
  double* part = partial.get(count * grid);
  pgram_kernel<T8, NPH><<<grid, 256, smem, st>>>(a, LS, part);
  launched();
  reduce_blocks<<<(int)((count + 255) / 256), 256, 0, st>>>(part, grid, (int)count, a.out);
  launched();
  comm_allreduce(a.geo, a.out, count, st);
}

// ===================================================================== small kernels
// dK[c] = dt sum_b (psi_b(c) / S(c)) T[cls(c)][b], T[k][b] = N_k^T rows_b (r-vector
// per class and beam, in shared memory). One warp per 32 cells: the lanes
// load the cells' class and 1/S once, then write one row (rs <= 32 doubles)
// per store instruction.
template <bool WIDE>  // WIDE: rows of up to 64 doubles (ranks above 32)
__global__ void scat_dk_kernel(Geom g, double dt, const double* __restrict__ inv_s,
                               const int* __restrict__ cls, const double* __restrict__ atomic,
                               int n_cls, const double* __restrict__ psi, int n_beams,
                               const double* __restrict__ rows, NMat out) {
  extern __shared__ double sT[];  // n_cls x n_beams x r
  const int r = out.cols, rs = out.rs, nb = n_beams > 0 ? n_beams : 1;
  for (int idx = threadIdx.x; idx < n_cls * nb * r; idx += blockDim.x) {
    const int k = idx / (nb * r), rem = idx - k * nb * r, b = rem / r, j = rem - b * r;
    double t = 0.0;
    for (int i = 0; i < 12; ++i) t = fma(atomic[k * 12 + i], rows[(b * 12 + i) * r + j], t);
    sT[idx] = t;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5, nwarps = gridDim.x * wpb;
  for (int c0 = (blockIdx.x * wpb + (threadIdx.x >> 5)) * 32; c0 < g.n; c0 += nwarps * 32) {
    const int c = c0 + lane;
    const int kc = c < g.n ? cls[c] : 0;
    const double is = c < g.n ? inv_s[c] : 0.0;
    double sp[4];  // psi_b / S of this lane's cell (n_beams <= 4)
#pragma unroll
    for (int b = 0; b < 4; ++b)
      sp[b] = (psi && b < n_beams && c < g.n) ? dt * is * psi[(size_t)b * g.ld + c] : 0.0;
    const int nrow = g.n - c0 < 32 ? g.n - c0 : 32;
#pragma unroll 4
    for (int q = 0; q < nrow; ++q) {
      const int kr = __shfl_sync(0xffffffffu, kc, q);
      double v = 0.0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if (b < n_beams) {  // warp-uniform
          const double s = __shfl_sync(0xffffffffu, sp[b], q);
          if (lane < r) v = fma(s, sT[(kr * nb + b) * r + lane], v);
        }
      }
      if (lane < rs) out.p[(size_t)(c0 + q) * rs + lane] = v;
      // columns 32..63 (ranks above 32)
      if (WIDE) {
        double v2 = 0.0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          if (b < n_beams) {
            const double s = __shfl_sync(0xffffffffu, sp[b], q);
            if (lane + 32 < r) v2 = fma(s, sT[(kr * nb + b) * r + lane + 32], v2);
          }
        }
        if (lane + 32 < rs) out.p[(size_t)(c0 + q) * rs + lane + 32] = v2;
      }
    }
  }
}

__global__ void source_rows_kernel(int n, int ld, const double* __restrict__ inv_s,
                                   const int* __restrict__ cls, const double* __restrict__ atomic,
                                   const double* __restrict__ psi, int n_beams, NMat Z) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const double* at = atomic + cls[c] * 12;
    const double is = inv_s[c];
    double* z = Z.p + (long)c * Z.rs;
    for (int b = 0; b < n_beams; ++b) {
      const double sp = is * psi[(size_t)b * ld + c];
#pragma unroll
      for (int i = 0; i < 12; i += 2)
        *reinterpret_cast<double2*>(z + b * 12 + i) = make_double2(at[i] * sp, at[i + 1] * sp);
    }
  }
}

__global__ void dose_kernel(Geom g, NMat U, const double* __restrict__ coef, double half_dt,
                            const double* __restrict__ s_field, const double* __restrict__ psi,
                            int n_beams, double* __restrict__ dep, double* __restrict__ prev) {
  const double sqrt4pi = 3.5449077018110318;  // sqrt(4 pi), driver.py:59
  __shared__ double sc[64];
  for (int i = threadIdx.x; i < U.cols; i += blockDim.x) sc[i] = coef[i];
  __syncthreads();
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < g.n; c += gridDim.x * blockDim.x) {
    double u0 = 0.0;
    const double* row = U.p + (long)c * U.rs;
    for (int j = 0; j < U.cols; ++j) u0 = fma(row[j], sc[j], u0);
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

__global__ void unit_rows_kernel(Geom g, NMat U) {
  const long total = (long)g.n * U.rs;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
       e += (long)gridDim.x * blockDim.x) {
    const int c = (int)(e / U.rs), j = (int)(e - (long)c * U.rs);
    const long cg = c + (long)g.z0 * g.nx * g.ny;  // global cell index (slabs)
    U.p[e] = (j < U.cols && cg == j) ? 1.0 : 0.0;
  }
}

__device__ __forceinline__ double hash_normal(unsigned long long x) {
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

__global__ void random_rows_kernel(Geom g, NMat U, unsigned long long seed) {
  const long total = (long)g.n * U.rs;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
       e += (long)gridDim.x * blockDim.x) {
    const int c = (int)(e / U.rs), j = (int)(e - (long)c * U.rs);
    // keyed by the global cell, so a slab decomposition draws the same matrix
    const unsigned long long key = (unsigned long long)(c + (long)g.z0 * g.nx * g.ny) * U.rs + j;
    U.p[e] = j < U.cols ? hash_normal(seed * 0x100000001B3ULL + key) : 0.0;
  }
}

__global__ void class_gather_kernel(const int* __restrict__ cls, const double* __restrict__ val,
                                    int n, double* __restrict__ inv, double* __restrict__ out) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const double s = val[cls[c]];
    if (inv) inv[c] = 1.0 / s;
    if (out) out[c] = s;
  }
}

__global__ void lerp_kernel(const double* __restrict__ v, int ldv, int n, int j0, double w0,
                            int j1, double w1, double* __restrict__ out) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    double x;
    if (w1 == 0.0) {
      x = w0 == 1.0 ? v[(size_t)j0 * ldv + c] : w0 * v[(size_t)j0 * ldv + c];
    } else {
      x = w0 * v[(size_t)j0 * ldv + c] + w1 * v[(size_t)j1 * ldv + c];
    }
    out[c] = x;
  }
}

// lerp_kernel on the separable table: v[g][c] = lat[c % nxy] * depth[c / nxy][g],
// the product rounded as the expanded table stores it
__global__ void lerp_sep_kernel(const double* __restrict__ lat, const double* __restrict__ depth,
                                int nxy, int G, int n, const int* __restrict__ sel_j,
                                const double* __restrict__ sel_w, int j0, double w0, int j1,
                                double w1, double* __restrict__ out) {
  if (sel_j) {
    j0 = sel_j[0];
    j1 = sel_j[1];
    w0 = sel_w[0];
    w1 = sel_w[1];
  }
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const int k = c / nxy;
    const double l = lat[c - k * nxy];
    const double v0 = __dmul_rn(l, depth[(size_t)k * G + j0]);
    double x;
    if (w1 == 0.0) {
      x = w0 == 1.0 ? v0 : w0 * v0;
    } else {
      const double v1 = __dmul_rn(l, depth[(size_t)k * G + j1]);
      x = w0 * v0 + w1 * v1;
    }
    out[c] = x;
  }
}

__global__ void tin_kernel(const double* __restrict__ src, int n, int cdim, double* __restrict__ dst,
                           int ldd) {
  __shared__ double tile[32][33];
  // rows on grid x (up to 2^31 - 1 blocks), columns on grid y
  const int c0 = blockIdx.y * 32, r0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int row = r0 + i, col = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (row < n && col < cdim) ? src[(size_t)row * cdim + col] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int col = c0 + i, row = r0 + threadIdx.x;
    if (row < n && col < cdim) dst[(size_t)col * ldd + row] = tile[threadIdx.x][i];
  }
}

__global__ void tout_kernel(const double* __restrict__ src, int lds, int n, int cdim,
                            double* __restrict__ dst) {
  __shared__ double tile[32][33];
  const int c0 = blockIdx.y * 32, r0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int col = c0 + i, row = r0 + threadIdx.x;
    tile[threadIdx.x][i] = (row < n && col < cdim) ? src[(size_t)col * lds + row] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int row = r0 + i, col = c0 + threadIdx.x;
    if (row < n && col < cdim) dst[(size_t)row * cdim + col] = tile[i][threadIdx.x];
  }
}

__global__ void zero_kernel(double* p, size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x)
    p[i] = 0.0;
}

int grid_for(long n, int block) {
  long b = (n + block - 1) / block;
  if (b > 148 * 16) b = 148 * 16;
  return b < 1 ? 1 : (int)b;
}

}  // namespace

void pgram(const PGramArgs& a, DBuf& partial, cudaStream_t st) {
  const int w = a.X.cols > a.nb ? a.X.cols : a.nb;
  const int t = (w + 7) / 8;
  if (a.X.cols <= 0 || a.nb <= 0 || a.nphase <= 0) return;
  if (a.nphase > 1) {
    if (a.nphase > 12 || t > 4) fail(PND_ECONFIG, "weighted Grams support 12 phases, rank <= 32");
    switch (t) {
      case 1: pgram_launch<1, 12>(a, partial, st); break;
      case 2: pgram_launch<2, 12>(a, partial, st); break;
      case 3: pgram_launch<3, 12>(a, partial, st); break;
      default: pgram_launch<4, 12>(a, partial, st); break;
    }
    return;
  }
  switch (t) {
    case 1: pgram_launch<1, 1>(a, partial, st); break;
    case 2: pgram_launch<2, 1>(a, partial, st); break;
    case 3: pgram_launch<3, 1>(a, partial, st); break;
    case 4: pgram_launch<4, 1>(a, partial, st); break;
    case 5: pgram_launch<5, 1>(a, partial, st); break;
    case 6: pgram_launch<6, 1>(a, partial, st); break;
    case 7:
    case 8: pgram_launch<8, 1>(a, partial, st); break;
    default: fail(PND_ECONFIG, "Grams support at most 64 columns");
  }
}

void scat_dk(const Geom& g, double dt, const double* inv_s, const int* cls,
             const double* cls_atomic, int n_cls, const double* psi, int n_beams,
             const double* rows, NMat out, cudaStream_t st) {
  if (out.rs > 64) fail(PND_ECONFIG, "scattering increment supports rank <= 64");
  const size_t smem = (size_t)n_cls * (n_beams > 0 ? n_beams : 1) * out.cols * sizeof(double);
  if (smem > 48 * 1024) fail(PND_ECONFIG, "scattering increment: too many material classes");
  if (out.rs > 32)
    scat_dk_kernel<true><<<sm_count() * 8, 256, smem, st>>>(g, dt, inv_s, cls, cls_atomic, n_cls,
                                                            psi, n_beams, rows, out);
  else
    scat_dk_kernel<false><<<sm_count() * 8, 256, smem, st>>>(g, dt, inv_s, cls, cls_atomic, n_cls,
                                                             psi, n_beams, rows, out);
  launched();
}

void dose_accumulate(const Geom& g, NMat U, const double* coef, double half_dt,
                     const double* s_field, const double* psi, int n_beams, double* deposited,
                     double* prev, cudaStream_t st) {
  if (U.cols > 64) fail(PND_ECONFIG, "dose supports rank <= 64");
  dose_kernel<<<grid_for(g.n, 256), 256, 0, st>>>(g, U, coef, half_dt, s_field, psi, n_beams,
                                                   deposited, prev);
  launched();
}

void unit_rows(const Geom& g, NMat U, cudaStream_t st) {
  unit_rows_kernel<<<grid_for((long)g.n * U.rs, 256), 256, 0, st>>>(g, U);
  launched();
}

void random_rows(const Geom& g, NMat U, unsigned long long seed, cudaStream_t st) {
  random_rows_kernel<<<grid_for((long)g.n * U.rs, 256), 256, 0, st>>>(g, U, seed);
  launched();
}

void class_gather_inv(const int* cls, const double* class_val, int n, double* out_inv,
                      double* out_val, cudaStream_t st) {
  class_gather_kernel<<<grid_for(n, 256), 256, 0, st>>>(cls, class_val, n, out_inv, out_val);
  launched();
}

void psi_lerp_separable(const double* lat, const double* depth, int nxy, int G, int n,
                        const int* sel_j, const double* sel_w, int j0, double w0, int j1,
                        double w1, double* out, cudaStream_t st) {
  lerp_sep_kernel<<<grid_for(n, 256), 256, 0, st>>>(lat, depth, nxy, G, n, sel_j, sel_w, j0, w0,
                                                    j1, w1, out);
  launched();
}

namespace {
__global__ void lerp_sparse_kernel(const int* __restrict__ cells, const double* __restrict__ v,
                                   int nnz, int G, const int* __restrict__ sel_j,
                                   const double* __restrict__ sel_w, int j0h, double w0h, int j1h,
                                   double w1h, double* __restrict__ out) {
  const int j0 = sel_j ? sel_j[0] : j0h, j1 = sel_j ? sel_j[1] : j1h;
  const double w0 = sel_w ? sel_w[0] : w0h, w1 = sel_w ? sel_w[1] : w1h;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += gridDim.x * blockDim.x) {
    const double* row = v + (size_t)i * G;
    double x;
    if (w1 == 0.0) x = w0 == 1.0 ? row[j0] : w0 * row[j0];
    else x = w0 * row[j0] + w1 * row[j1];
    out[cells[i]] = x;
  }
}
}  // namespace

void psi_lerp_sparse(const int* cells, const double* values, int nnz, int G, int n,
                     const int* sel_j, const double* sel_w, int j0, double w0, int j1, double w1,
                     double* out, cudaStream_t st) {
  fill_zero(out, (size_t)n, st);
  if (nnz <= 0) return;
  lerp_sparse_kernel<<<grid_for(nnz, 256), 256, 0, st>>>(cells, values, nnz, G, sel_j, sel_w, j0,
                                                         w0, j1, w1, out);
  launched();
}

void psi_lerp(const double* values, int ldv, int n, int j0, double w0, int j1, double w1,
              double* out, cudaStream_t st) {
  lerp_kernel<<<grid_for(n, 256), 256, 0, st>>>(values, ldv, n, j0, w0, j1, w1, out);
  launched();
}

void transpose_in(const double* src, int n, int c, double* dst, int ldd, cudaStream_t st) {
  if (n <= 0 || c <= 0) return;
  dim3 grid((n + 31) / 32, (c + 31) / 32), block(32, 8);
  tin_kernel<<<grid, block, 0, st>>>(src, n, c, dst, ldd);
  launched();
}

void transpose_out(const double* src, int lds, int n, int c, double* dst, cudaStream_t st) {
  if (n <= 0 || c <= 0) return;
  dim3 grid((n + 31) / 32, (c + 31) / 32), block(32, 8);
  tout_kernel<<<grid, block, 0, st>>>(src, lds, n, c, dst);
  launched();
}

void fill_zero(double* p, size_t count, cudaStream_t st) {
  if (!count) return;
  size_t blocks = (count + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  zero_kernel<<<(int)blocks, 256, 0, st>>>(p, count);
  launched();
}

NMat NBuf::view(const Geom& g, int cols, cudaStream_t st) {
  const int nrs = even(cols > 0 ? cols : 1);
  const size_t total = (size_t)(g.n + 2 * g.halo) * nrs;
  if (d.cap < total || nrs != rs) {
    d.get(total > d.cap ? total : d.cap);
    // halo rows (and the whole buffer, once) are zero for the new stride
    fill_zero(d.p, (size_t)g.halo * nrs, st);
    fill_zero(d.p + (size_t)(g.halo + g.n) * nrs, (size_t)g.halo * nrs, st);
    rs = nrs;
  }
  NMat m;
  m.p = d.p + (size_t)g.halo * rs;
  m.rs = rs;
  m.cols = cols;
  return m;
}

void source_rows(const Geom& g, const double* inv_s, const int* cls, const double* cls_atomic,
                 const double* psi, int n_beams, NMat Z, cudaStream_t st) {
  source_rows_kernel<<<grid_for(g.n, 256), 256, 0, st>>>(g.n, g.ld, inv_s, cls, cls_atomic, psi,
                                                    n_beams, Z);
  launched();
}

}  // namespace pnd
