#include <atomic>
#include <vector>
// extern "C" boundary (include/pndose_b200.h): argument checks, host<->device
// staging, error mapping. Every exception raised inside the library becomes
// a status code plus a message stored in the handle.
#include <cmath>
#include <map>
#include <mutex>
#include <tuple>
#include <unordered_set>
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "../../include/pndose_b200.h"
#include <nvtx3/nvToolsExt.h>

#include "handle.h"

namespace pnd {

void fail(int code, const std::string& msg) { throw Error{code, msg}; }

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    fail(PND_EDEVICE, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
  }
}

double* DBuf::get(size_t count) {
  if (count > cap) {
    if (p) CK(cudaFree(p));
    p = nullptr;
    cap = 0;
    CK(cudaMalloc(&p, count * sizeof(double)));
    cap = count;
  }
  return p;
}
void DBuf::free_() {
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
}
int* IBuf::get(size_t count) {
  if (count > cap) {
    if (p) CK(cudaFree(p));
    p = nullptr;
    cap = 0;
    CK(cudaMalloc(&p, count * sizeof(int)));
    cap = count;
  }
  return p;
}
void IBuf::free_() {
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
}

static std::atomic<long long> g_launches{0};  // kernel launches (bench gpu_launches)

bool smem_set_once(const void* fn) {
  static std::mutex mu;
  static std::unordered_set<const void*> seen;
  std::lock_guard<std::mutex> lk(mu);
  return seen.insert(fn).second;
}

int occupancy_cached(const void* fn, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t>, int> cache;
  const auto key = std::make_tuple(fn, threads, smem);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  int nb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, threads, smem));
  if (nb < 1) nb = 1;
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = nb;
  return nb;
}

void launched() {
  CK(cudaGetLastError());
  ++g_launches;
}

long long launch_count() { return g_launches; }

int max_smem_optin() {
  static int v = 0;
  if (!v) {
    int dev = 0, x = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&x, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    v = x;
  }
  return v;
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

void phase(Handle& h, int id) {
  // NVTX ranges per phase (no-ops unless a profiler is attached)
  static const char* const names[PH_COUNT] = {
      "kstage", "l_gram", "l_side", "tsqr_n", "tsqr_m", "s_gram", "s_rk4",
      "svd", "rotate", "scat_k1", "scat_gram", "scat_small", "dose", "defect"};
  if (h.nvtx_open) nvtxRangePop();
  h.nvtx_open = id >= 0 && id < PH_COUNT;
  if (h.nvtx_open) nvtxRangePushA(names[id]);
  TimerState& t = h.timer;
  if (!t.on) return;
  if (t.used == t.pool.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    t.pool.push_back(e);
  }
  CK(cudaEventRecord(t.pool[t.used], h.st));
  t.ids.push_back(id);
  ++t.used;
}

namespace {

__global__ void logdiag_kernel(double* S, int r) {
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) {
    const int a = i / r, b = i % r;
    S[i] = a == b ? pow(10.0, r > 1 ? -3.0 * a / (r - 1) : 0.0) : 0.0;
  }
}

}  // namespace

}  // namespace pnd

struct pnd_handle {
  pnd::Handle h;
};

using pnd::Handle;
using pnd::NMat;

namespace {

template <class F>
int guard(pnd_handle* hh, F&& f) {
  if (!hh) return PND_ECONFIG;
  try {
    CK(cudaSetDevice(hh->h.device));
    f(hh->h);
    return PND_OK;
  } catch (const pnd::Error& e) {
    hh->h.err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    hh->h.err = e.what();
    return PND_EDEVICE;
  }
}

void up(double* dst, const double* src, size_t count, cudaStream_t st) {
  if (!count) return;
  CK(cudaMemcpyAsync(dst, src, count * sizeof(double), cudaMemcpyHostToDevice, st));
}
void down(double* dst, const double* src, size_t count, cudaStream_t st) {
  if (!count) return;
  CK(cudaMemcpyAsync(dst, src, count * sizeof(double), cudaMemcpyDeviceToHost, st));
}

// host (n x cols row-major) -> cell-major device view (rs >= cols, pad column zero)
void upload_rows(Handle& h, NMat m, const double* src) {
  if (m.rs != m.cols) pnd::fill_zero(m.p, (size_t)h.g.n * m.rs, h.st);
  CK(cudaMemcpy2DAsync(m.p, m.rs * sizeof(double), src, m.cols * sizeof(double),
                       m.cols * sizeof(double), h.g.n, cudaMemcpyHostToDevice, h.st));
}

// device view -> host rows [:, col0 : col0 + m.cols] of an (n x ldh) row-major array
void download_rows(Handle& h, NMat m, double* dst, int ldh, int col0) {
  CK(cudaMemcpy2DAsync(dst + col0, ldh * sizeof(double), m.p, m.rs * sizeof(double),
                       m.cols * sizeof(double), h.g.n, cudaMemcpyDeviceToHost, h.st));
}

}  // namespace

extern "C" {

int pnd_create(pnd_handle** out, int nx, int ny, int nz, double dx, double dy, double dz, int m,
               int device) {
  if (!out) return PND_ECONFIG;
  *out = nullptr;
  auto* hh = new pnd_handle();
  Handle& h = hh->h;
  h.device = device;
  try {
    const int dims[3] = {nx, ny, nz};
    const char* names[3] = {"nx", "ny", "nz"};
    for (int a = 0; a < 3; ++a) {
      if (dims[a] < 1) pnd::fail(PND_ECONFIG, "grid needs at least one cell per dimension");
      if (dims[a] == 2 && h.stencil_error.empty()) {
        // Grid3D allows it; only the stencil cannot be built (spatial.py:84-88)
        h.stencil_error = std::string("grid.") + names[a] +
                          "=2: grids with 2 cells along a used axis cannot host the 3-point "
                          "one-sided stencil; use 1 (inactive) or >= 3";
      }
    }
    if (!(dx > 0 && dy > 0 && dz > 0)) pnd::fail(PND_ECONFIG, "grid spacings must be positive");
    if (m < 1) pnd::fail(PND_ECONFIG, "need at least one moment");
    const long long n = (long long)nx * ny * nz;
    const long long halo = 2LL * nx * ny + 72;
    if (n + 2 * halo >= (1LL << 31) - 1024) pnd::fail(PND_ECONFIG, "grid exceeds 2^31 cells per device");
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&h.st, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&h.st2, cudaStreamNonBlocking));
    {
      // stream-ordered scratch (split-K partials, wide R x R work) stays in the
      // device pool instead of going back to the driver at every synchronisation
      cudaMemPool_t pool;
      CK(cudaDeviceGetDefaultMemPool(&pool, device));
      uint64_t keep = UINT64_MAX;
      CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    CK(cudaEventCreateWithFlags(&h.ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h.ev_join, cudaEventDisableTiming));
    CK(cudaMallocHost(&h.pinned, 64 * sizeof(double)));
    pnd::Geom& g = h.g;
    g.nx = nx;
    g.ny = ny;
    g.nz = nz;
    g.n = (int)n;
    g.ld = (int)((n + 31) / 32 * 32);
    g.inv_nx = 1.0 / nx;
    g.inv_nxy = 1.0 / ((double)nx * ny);
    auto magic = [](unsigned long long d) { return d < 2 ? 0ULL : ~0ULL / d + 1; };
    g.mnx = magic((unsigned long long)nx);
    g.mnxy = magic((unsigned long long)nx * ny);
    g.halo = (int)halo;
    g.h[0] = dx;
    g.h[1] = dy;
    g.h[2] = dz;
    for (int a = 0; a < 3; ++a) {
      g.ih[a] = 1.0 / g.h[a];
      g.i2h[a] = 1.0 / (2.0 * g.h[a]);
    }
    g.na = 0;
    for (int a = 0; a < 3; ++a)
      if (dims[a] > 1) g.axis[g.na++] = a;
    for (int a = g.na; a < 3; ++a) g.axis[a] = 0;
    g.ns = 2 * g.na;
    h.m = m;
    *out = hh;
    return PND_OK;
  } catch (const pnd::Error& e) {
    h.err = e.msg;
    *out = hh;  // caller reads the message, then destroys
    return e.code;
  }
}

int pnd_destroy(pnd_handle* hh) {
  if (!hh) return PND_OK;
  Handle& h = hh->h;
  cudaSetDevice(h.device);
  if (h.st) cudaStreamSynchronize(h.st);
  if (h.st2) cudaStreamSynchronize(h.st2);
  pnd::DBuf* bufs[] = {&h.amat, &h.inv_s, &h.isp, &h.s_field, &h.cls_atomic, &h.cls_val, &h.bcat,
                       &h.gdiag, &h.sigt, &h.psi, &h.psi_lo, &h.tm, &h.flux, &h.S, &h.V,
                       &h.part, &h.dep, &h.prev, &h.tq_m.tau, &h.tq_m.tree, &h.tq_m.rbuf,
                       &h.tq_m.cbuf, &h.ctab, &h.csel, &h.wide_m, &h.wide_t, &h.wide_i,
                       &h.wide_g, &h.fr_scr, &h.fr_scr2, &h.fr_scr3, &h.fr_eye,
                       &h.sep_lat, &h.sep_depth, &h.cq_work};
  for (auto* b : bufs) b->free_();
  // ranks above 64 (xwide.cu) and the sparse flux tables
  for (auto* v : {&h.xU, &h.xQ, &h.xUn, &h.xW1, &h.xW2})
    for (auto& b : *v) b.d.free_();
  for (auto& b : h.xsm) b.free_();
  for (auto& b : h.sp_vals) b.free_();
  for (auto& b : h.sp_cells) b.free_();
  pnd::NBuf* nb[] = {&h.U, &h.Q, &h.Un, &h.Qa, &h.W1, &h.W2, &h.Xs, &h.wide_base,
                     &h.wide_tmp[0], &h.wide_tmp[1], &h.fr_t[0], &h.fr_t[1]};
  for (auto* b : nb) b->d.free_();
  for (auto* v : {&h.wide_u0b, &h.wide_qb, &h.wide_w1b, &h.wide_w2b, &h.wide_gb, &h.fr_u,
                  &h.fr_w1, &h.fr_w2})
    for (auto& b : *v) b.d.free_();
  pnd::comm_destroy(h.comm);
  h.comm = nullptr;
  for (auto& b : h.sm) b.free_();
  h.cls.free_();
  h.iflag.free_();
  for (auto e : h.timer.pool) cudaEventDestroy(e);
  for (auto e : h.timer.ev)
    if (e) cudaEventDestroy(e);
  if (h.pinned) cudaFreeHost(h.pinned);
  if (h.st) cudaStreamDestroy(h.st);
  if (h.st2) cudaStreamDestroy(h.st2);
  if (h.ev_fork) cudaEventDestroy(h.ev_fork);
  if (h.ev_join) cudaEventDestroy(h.ev_join);
  delete hh;
  return PND_OK;
}

int pnd_last_error(pnd_handle* hh, char* buf, size_t len) {
  if (!hh || !buf || !len) return PND_ECONFIG;
  std::snprintf(buf, len, "%s", hh->h.err.c_str());
  return PND_OK;
}

int pnd_synchronize(pnd_handle* hh) {
  return guard(hh, [&](Handle& h) { CK(cudaStreamSynchronize(h.st)); });
}

int pnd_device_bytes(pnd_handle* hh, double* bytes) {
  return guard(hh, [&](Handle& h) {
    double total = 0;
    const pnd::DBuf* bufs[] = {&h.amat, &h.inv_s, &h.isp, &h.s_field, &h.cls_atomic, &h.gdiag,
                               &h.psi, &h.psi_lo, &h.tm, &h.flux, &h.S, &h.V, &h.part, &h.dep,
                               &h.prev, &h.sep_lat, &h.sep_depth, &h.tq_m.tau, &h.tq_m.tree, &h.tq_m.cbuf};
    for (auto* b : bufs) total += 8.0 * b->cap;
    const pnd::NBuf* nb[] = {&h.U, &h.Q, &h.Un, &h.Qa, &h.W1, &h.W2, &h.Xs};
    for (auto* b : nb) total += 8.0 * b->d.cap;
    for (auto& b : h.sm) total += 8.0 * b.cap;
    *bytes = total;
  });
}

int pnd_set_angular(pnd_handle* hh, const double* a_plus, const double* a_minus) {
  return guard(hh, [&](Handle& h) {
    const size_t mm = (size_t)h.m * h.m;
    double* d = h.amat.get(h.g.ns * mm + 1);
    for (int ai = 0; ai < h.g.na; ++ai) {
      const int axis = h.g.axis[ai];
      up(d + (2 * ai) * mm, a_plus + axis * mm, mm, h.st);
      up(d + (2 * ai + 1) * mm, a_minus + axis * mm, mm, h.st);
    }
    CK(cudaStreamSynchronize(h.st));
    h.have_angular = true;
  });
}

int pnd_set_materials(pnd_handle* hh, const int32_t* cell_class, int n_class,
                      const double* class_atomic) {
  return guard(hh, [&](Handle& h) {
    if (n_class < 1) pnd::fail(PND_ECONFIG, "need at least one material class");
    int* c = h.cls.get(h.g.n);
    CK(cudaMemcpyAsync(c, cell_class, sizeof(int) * h.g.n, cudaMemcpyHostToDevice, h.st));
    up(h.cls_atomic.get((size_t)n_class * 12), class_atomic, (size_t)n_class * 12, h.st);
    CK(cudaStreamSynchronize(h.st));
    h.n_cls = n_class;
    h.have_mat = true;
  });
}

int pnd_set_inv_s(pnd_handle* hh, const double* inv_s) {
  return guard(hh, [&](Handle& h) {
    // 64 doubles of zero slack: streaming kernels stage whole 64-cell chunks
    double* d = h.inv_s.get(h.g.ld + 64);
    pnd::fill_zero(d, h.g.ld + 64, h.st);
    up(d, inv_s, h.g.n, h.st);
    double* sf = h.s_field.get(h.g.ld);
    pnd::fill_zero(sf, h.g.ld, h.st);
    pnd::set_isp(h);
    CK(cudaStreamSynchronize(h.st));
    h.have_inv_s = true;
    int uni = 1;
    for (int i = 1; i < h.g.n && uni; ++i) uni = inv_s[i] == inv_s[0];
    h.g.uniform_s = uni;
  });
}

int pnd_set_class_stopping(pnd_handle* hh, const double* class_s) {
  return guard(hh, [&](Handle& h) {
    if (!h.have_mat) pnd::fail(PND_ECONFIG, "set materials before class stopping powers");
    double* v = h.cls_val.get(h.n_cls);
    up(v, class_s, h.n_cls, h.st);
    double* d = h.inv_s.get(h.g.ld + 64);
    double* sf = h.s_field.get(h.g.ld);
    pnd::fill_zero(d + h.g.n, h.g.ld + 64 - h.g.n, h.st);  // zero tail (chunked staging)
    pnd::class_gather_inv(h.cls.p, v, h.g.n, d, sf, h.st);
    pnd::set_isp(h);
    h.have_inv_s = true;
    h.g.uniform_s = h.n_cls == 1;
  });
}

int pnd_set_scattering(pnd_handle* hh, const double* g_diags, const double* sigma_t) {
  return guard(hh, [&](Handle& h) {
    // small pageable copies: staged by the driver at the call, no stream sync needed
    up(h.gdiag.get((size_t)12 * h.m), g_diags, (size_t)12 * h.m, h.st);
    up(h.sigt.get(12), sigma_t, 12, h.st);
    h.have_scat = true;
  });
}

int pnd_set_sources(pnd_handle* hh, int n_beams, const double* psi, const double* t_m) {
  return guard(hh, [&](Handle& h) {
    if (n_beams < 0 || n_beams > 4) pnd::fail(PND_ECONFIG, "0..4 uncollided sources supported");
    h.n_beams = n_beams;
    if (!n_beams) return;
    double* d = h.psi.get((size_t)n_beams * h.g.ld + 64);
    for (int b = 0; b < n_beams; ++b) up(d + (size_t)b * h.g.ld, psi + (size_t)b * h.g.n, h.g.n, h.st);
    up(h.tm.get((size_t)n_beams * h.m), t_m, (size_t)n_beams * h.m, h.st);
    CK(cudaStreamSynchronize(h.st));
  });
}

int pnd_set_flux_table(pnd_handle* hh, int beam, int n_beams, int n_groups, const double* values,
                       const double* t_m) {
  return guard(hh, [&](Handle& h) {
    if (n_beams < 1 || n_beams > 4) pnd::fail(PND_ECONFIG, "1..4 beams supported");
    if (beam < 0 || beam >= n_beams) pnd::fail(PND_ECONFIG, "beam index out of range");
    if (beam == 0) {
      h.n_groups = n_groups;
      h.n_beams = n_beams;
      h.flux_sep = false;
      h.flux_sparse = false;
      h.sep_lat.free_();
      h.sep_depth.free_();
      h.flux.get((size_t)n_beams * n_groups * h.g.ld);
      h.psi.get((size_t)n_beams * h.g.ld + 64);
      h.psi_lo.get((size_t)n_beams * h.g.ld);
      h.tm.get((size_t)n_beams * h.m);
    } else if (n_groups != h.n_groups || n_beams != h.n_beams || !h.flux.p) {
      pnd::fail(PND_ECONFIG, "all beams must share the group grid (set beam 0 first)");
    }
    // values (n x G row-major) -> G columns of length ld
    pnd::DBuf stage;
    double* s = stage.get((size_t)h.g.n * n_groups);
    up(s, values, (size_t)h.g.n * n_groups, h.st);
    pnd::transpose_in(s, h.g.n, n_groups, h.flux.p + (size_t)beam * n_groups * h.g.ld, h.g.ld,
                      h.st);
    up(h.tm.p + (size_t)beam * h.m, t_m, h.m, h.st);
    CK(cudaStreamSynchronize(h.st));
    stage.free_();
  });
}

int pnd_set_flux_table_sparse(pnd_handle* hh, int beam, int n_beams, int n_groups, int nnz,
                              const int32_t* cells, const double* values, const double* t_m) {
  return guard(hh, [&](Handle& h) {
    if (n_beams < 1 || n_beams > 4) pnd::fail(PND_ECONFIG, "1..4 beams supported");
    if (beam < 0 || beam >= n_beams) pnd::fail(PND_ECONFIG, "beam index out of range");
    if (nnz < 0 || nnz > h.g.n) pnd::fail(PND_ECONFIG, "sparse flux: bad cell count");
    for (int i = 0; i < nnz; ++i)
      if (cells[i] < 0 || cells[i] >= h.g.n || (i && cells[i] <= cells[i - 1]))
        pnd::fail(PND_ECONFIG, "sparse flux: cells must be increasing and inside the grid");
    if (beam == 0) {
      h.n_groups = n_groups;
      h.n_beams = n_beams;
      h.flux_sep = false;
      h.flux_sparse = true;
      h.flux.free_();
      h.sep_lat.free_();
      h.sep_depth.free_();
      h.sp_cells.resize(n_beams);
      h.sp_vals.resize(n_beams);
      h.sp_nnz.assign(n_beams, 0);
      h.psi.get((size_t)n_beams * h.g.ld + 64);
      h.psi_lo.get((size_t)n_beams * h.g.ld);
      h.tm.get((size_t)n_beams * h.m);
    } else if (n_groups != h.n_groups || n_beams != h.n_beams || !h.flux_sparse) {
      pnd::fail(PND_ECONFIG, "all beams must share the group grid (set beam 0 first)");
    }
    h.sp_nnz[beam] = nnz;
    int* dc = h.sp_cells[beam].get((size_t)(nnz > 0 ? nnz : 1));
    double* dv = h.sp_vals[beam].get((size_t)(nnz > 0 ? nnz : 1) * n_groups);
    if (nnz > 0) {
      CK(cudaMemcpyAsync(dc, cells, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, h.st));
      up(dv, values, (size_t)nnz * n_groups, h.st);
    }
    up(h.tm.p + (size_t)beam * h.m, t_m, h.m, h.st);
    CK(cudaStreamSynchronize(h.st));
  });
}

int pnd_moment_tables(pnd_handle* hh, int n_e, const double* energies, int n_el,
                      const int32_t* z, const int32_t* a, int nn, const double* x1,
                      const double* w1, const double* x2, const double* w2, int max_degree,
                      double exponent, double rtol, double* g, double* xi1) {
  return guard(hh, [&](Handle& h) {
    if (n_e < 1 || n_el < 1 || nn < 1) pnd::fail(PND_ECONFIG, "moment tables: empty grid");
    const int bad = pnd::moment_tables(energies, n_e, z, a, n_el, x1, w1, x2, w2, nn, max_degree,
                                       exponent, rtol, g, xi1, h.st);
    if (bad >= 0) {
      char msg[160];
      snprintf(msg, sizeof msg,
               "moment quadrature for element %d at %g MeV did not converge, tolerance %.3e",
               bad / n_e, energies[bad % n_e], rtol);
      pnd::fail(PND_ENUMERICAL, msg);
    }
  });
}

int pnd_set_coefficient_tables(pnd_handle* hh, int k, const double* log_e, const double* log_s,
                               const double* class_density, const double* class_weights, int p,
                               const double* mom_e, int nd, const double* mom_g,
                               const double* mom_xi1, int model, int pn_order,
                               int boltzmann_correction, double fp_correction_scale,
                               int n_beams, const double* flux_range) {
  return guard(hh, [&](Handle& h) {
    if (!h.have_mat) pnd::fail(PND_ECONFIG, "set materials before the coefficient tables");
    if (k < 2 || p < 2 || nd < pn_order + 2 || (model != 0 && model != 1))
      pnd::fail(PND_ECONFIG, "coefficient tables: bad sizes or model");
    if (n_beams < 0 || n_beams > 4) pnd::fail(PND_ECONFIG, "0..4 beams supported");
    const size_t nel = 12, nc = h.n_cls;
    const size_t total = 2 * nel * k + nc + nc * nel + p + nel * p * nd + nel * p + 2 * n_beams;
    double* d = h.ctab.get(total);
    size_t o = 0;
    auto put = [&](const double* src, size_t cnt) {
      if (cnt) up(d + o, src, cnt, h.st);
      o += cnt;
    };
    put(log_e, nel * k);
    put(log_s, nel * k);
    put(class_density, nc);
    put(class_weights, nc * nel);
    put(mom_e, p);
    put(mom_g, nel * p * nd);
    put(mom_xi1, nel * p);
    put(flux_range, 2 * (size_t)n_beams);
    h.ct_K = k;
    h.ct_P = p;
    h.ct_nd = nd;
    h.ct_model = model;
    h.ct_pn = pn_order;
    h.ct_bcorr = boltzmann_correction;
    h.ct_fpscale = fp_correction_scale;
    if (n_beams && (!h.have_flux() || n_beams != h.n_beams))
      pnd::fail(PND_ECONFIG, "coefficient tables: set the flux tables of every beam first");
    h.csel.get(32);
    CK(cudaStreamSynchronize(h.st));
    h.have_ctab = true;
  });
}

int pnd_coefficients_at(pnd_handle* hh, double e_mid, double e_lo, int want_lo) {
  return guard(hh, [&](Handle& h) { pnd::coefficients_at(h, e_mid, e_lo, want_lo != 0); });
}

int pnd_get_coefficients(pnd_handle* hh, double* class_s, double* g_diags, double* sigma_t,
                         double* psi, double* psi_lo) {
  return guard(hh, [&](Handle& h) {
    if (class_s) down(class_s, h.cls_val.p, h.n_cls, h.st);
    if (g_diags) down(g_diags, h.gdiag.p, (size_t)12 * h.m, h.st);
    if (sigma_t) down(sigma_t, h.sigt.p, 12, h.st);
    for (int b = 0; b < h.n_beams; ++b) {
      if (psi) down(psi + (size_t)b * h.g.n, h.psi.p + (size_t)b * h.g.ld, h.g.n, h.st);
      if (psi_lo) down(psi_lo + (size_t)b * h.g.n, h.psi_lo.p + (size_t)b * h.g.ld, h.g.n, h.st);
    }
    CK(cudaStreamSynchronize(h.st));
  });
}

int pnd_select_flux(pnd_handle* hh, int which, const int32_t* j0, const double* w0,
                    const int32_t* j1, const double* w1) {
  return guard(hh, [&](Handle& h) {
    double* dst = which == 0 ? h.psi.p : h.psi_lo.p;
    for (int b = 0; b < h.n_beams; ++b) {
      if (h.flux_sep) {
        const int nxy = h.g.nx * h.g.ny;
        pnd::psi_lerp_separable(h.sep_lat.p + (size_t)b * nxy,
                                h.sep_depth.p + (size_t)b * h.g.nz * h.n_groups, nxy, h.n_groups,
                                h.g.n, nullptr, nullptr, j0[b], w0[b], j1[b], w1[b],
                                dst + (size_t)b * h.g.ld, h.st);
        continue;
      }
      if (h.flux_sparse) {
        pnd::psi_lerp_sparse(h.sp_cells[b].p, h.sp_vals[b].p, h.sp_nnz[b], h.n_groups, h.g.n,
                             nullptr, nullptr, j0[b], w0[b], j1[b], w1[b],
                             dst + (size_t)b * h.g.ld, h.st);
        continue;
      }
      const double* tab = h.flux.p + (size_t)b * h.n_groups * h.g.ld;
      pnd::psi_lerp(tab, h.g.ld, h.g.n, j0[b], w0[b], j1[b], w1[b], dst + (size_t)b * h.g.ld,
                    h.st);
    }
  });
}

int pnd_state_set(pnd_handle* hh, int ru, int rv, const double* u, const double* s,
                  const double* v) {
  return guard(hh, [&](Handle& h) {
    if (ru < 1 || rv < 1) pnd::fail(PND_ECONFIG, "rank must be positive");
    // ranks up to 256 per factor, 512 for an augmented state (truncate input)
    if (ru > 512 || rv > 512) pnd::fail(PND_ECONFIG, "rank above 256 is not supported");
    if (ru > 64) {
      pnd::upload_blocked(h, u, ru);  // 32-column blocks (xwide.cu)
    } else {
      if (h.blocked) pnd::release_blocked(h);
      NMat U = h.U.view(h.g, ru, h.st);
      upload_rows(h, U, u);
      h.blocked = false;
    }
    up(h.S.get((size_t)ru * rv), s, (size_t)ru * rv, h.st);
    up(h.V.get((size_t)h.m * rv), v, (size_t)h.m * rv, h.st);
    CK(cudaStreamSynchronize(h.st));
    h.ua = ru;
    h.uq = 0;
    h.ru = ru;
    h.rv = rv;
  });
}

int pnd_state_shape(pnd_handle* hh, int* ru, int* rv) {
  return guard(hh, [&](Handle& h) {
    *ru = h.ru;
    *rv = h.rv;
  });
}

int pnd_state_get(pnd_handle* hh, double* u, double* s, double* v) {
  return guard(hh, [&](Handle& h) {
    if (u && h.blocked) {
      pnd::download_blocked(h, u, h.ru);
    } else if (u) {
      download_rows(h, pnd::state_u(h), u, h.ru, 0);
      if (h.uq > 0) download_rows(h, pnd::state_q(h), u, h.ru, h.ua);
    }
    if (s) down(s, h.S.p, (size_t)h.ru * h.rv, h.st);
    if (v) down(v, h.V.p, (size_t)h.m * h.rv, h.st);
    CK(cudaStreamSynchronize(h.st));
  });
}

int pnd_streaming_step(pnd_handle* hh, double dt) {
  return guard(hh, [&](Handle& h) { pnd::streaming_step(h, dt); });
}

int pnd_scattering_step(pnd_handle* hh, double dt) {
  return guard(hh, [&](Handle& h) { pnd::scattering_step(h, dt); });
}

int pnd_truncate(pnd_handle* hh, double theta, int rank_min, int rank_max, double* tail,
                 int* rank) {
  return guard(hh, [&](Handle& h) {
    if (theta < 0) pnd::fail(PND_ECONFIG, "truncation threshold must be nonnegative");
    if (!(1 <= rank_min && rank_min <= rank_max))
      pnd::fail(PND_ECONFIG, "need 1 <= rank_min <= rank_max");
    pnd::truncate(h, theta, rank_min, rank_max, tail, rank);
  });
}

int pnd_step(pnd_handle* hh, double dt, double theta, int rank_min, int rank_max,
             int truncate_after, int tally_steps, int want_defect, double* out) {
  return guard(hh, [&](Handle& h) {
    double t1 = 0.0, t2 = 0.0, defect = 0.0;
    int rank = 0;
    const int ru0 = h.ru, rv0 = h.rv;
    int ru1 = 0, rv1 = 0;
    auto body = [&]() {
      h.spec_tr = 0;
      pnd::streaming_step(h, dt);
      if (truncate_after & 1) pnd::truncate(h, theta, rank_min, rank_max, &t1, &rank);
      ru1 = h.ru;
      rv1 = h.rv;
      h.spec_tr = 1;
      pnd::scattering_step(h, dt);
      bool ugram = false;
      if (truncate_after & 2) {
        // the last rotation of the step also forms U^T U for the defect diagnostic
        const int kmax = h.ru < h.rv ? h.ru : h.rv;  // the truncated rank is at most this
        double* G = want_defect ? pnd::defect_gram_slot(h, kmax, kmax) : nullptr;
        pnd::truncate(h, theta, rank_min, rank_max, &t2, &rank, G);
        ugram = want_defect;
      }
      pnd::dose_accumulate_step(h, dt, tally_steps != 0);
      if (want_defect) defect = pnd::orth_defect(h, ugram);
    };
    if (h.spec_pause > 0) --h.spec_pause;
    bool done = false;
    if (pnd::spec_eligible(h, truncate_after)) {
      // no host round trip inside the step: one synchronisation at its end
      pnd::spec_begin(h);
      try {
        body();
      } catch (...) {
        pnd::spec_end(h, true);
        throw;
      }
      done = pnd::spec_end(h, false);
      if (done) {
        t1 = h.pinned[20];
        t2 = h.pinned[21];
        if (want_defect) defect = h.pinned[22];
      }
    }
    if (!done) body();
    if (out) {
      out[0] = t1;
      out[1] = t2;
      out[2] = (double)(h.ru < h.rv ? h.ru : h.rv);
      out[3] = defect;
      out[4] = ru0;  // factor ranks entering the streaming substep
      out[5] = rv0;
      out[6] = ru1;  // ... and entering the scattering substep
      out[7] = rv1;
    }
  });
}

int pnd_spec_stats(pnd_handle* hh, long long* hits_misses) {
  return guard(hh, [&](Handle& h) {
    hits_misses[0] = h.spec_hits;
    hits_misses[1] = h.spec_misses;
  });
}

int pnd_dose_reset(pnd_handle* hh) {
  return guard(hh, [&](Handle& h) {
    pnd::fill_zero(h.dep.get(h.g.ld), h.g.ld, h.st);
    pnd::fill_zero(h.prev.get(h.g.ld), h.g.ld, h.st);
    if (!h.s_field.p) pnd::fill_zero(h.s_field.get(h.g.ld), h.g.ld, h.st);
  });
}

int pnd_dose_accumulate(pnd_handle* hh, double dt, int tally_steps) {
  return guard(hh, [&](Handle& h) { pnd::dose_accumulate_step(h, dt, tally_steps != 0); });
}

int pnd_dose_state(pnd_handle* hh, double* deposited, double* prev) {
  return guard(hh, [&](Handle& h) {
    if (deposited) down(deposited, h.dep.get(h.g.ld), h.g.n, h.st);
    if (prev) down(prev, h.prev.get(h.g.ld), h.g.n, h.st);
    CK(cudaStreamSynchronize(h.st));
  });
}

int pnd_dose_restore(pnd_handle* hh, const double* deposited, const double* prev) {
  return guard(hh, [&](Handle& h) {
    pnd::fill_zero(h.dep.get(h.g.ld), h.g.ld, h.st);
    pnd::fill_zero(h.prev.get(h.g.ld), h.g.ld, h.st);
    up(h.dep.p, deposited, h.g.n, h.st);
    up(h.prev.p, prev, h.g.n, h.st);
    CK(cudaStreamSynchronize(h.st));
  });
}

int pnd_get_dose(pnd_handle* hh, double* deposited) {
  return guard(hh, [&](Handle& h) {
    down(deposited, h.dep.get(h.g.ld), h.g.n, h.st);
    CK(cudaStreamSynchronize(h.st));
  });
}

int pnd_orth_defect(pnd_handle* hh, double* defect) {
  return guard(hh, [&](Handle& h) { *defect = pnd::orth_defect(h); });
}

// ------------------------------------------------------------ unit parity
int pnd_apply_streaming(pnd_handle* hh, const double* u, double* out) {
  return guard(hh, [&](Handle& h) {
    if (!h.stencil_error.empty()) pnd::fail(PND_ECONFIG, h.stencil_error);
    if (!h.have_angular || !h.have_inv_s) pnd::fail(PND_ECONFIG, "set angular and inv_s first");
    if (h.m > 32) pnd::fail(PND_ECONFIG, "apply_streaming supports m <= 32");
    const int n = h.g.n, m = h.m, ns = h.g.ns;
    for (size_t i = 0; i < (size_t)n * m; ++i)
      if (!std::isfinite(u[i])) pnd::fail(PND_ENUMERICAL, "non-finite streaming input");
    NMat X = h.W1.view(h.g, m, h.st);
    upload_rows(h, X, u);
    pnd::DBuf mneg;
    double* M = mneg.get((size_t)ns * m * m + 1);
    pnd::axpby(ns * m * m, -1.0, h.amat.p, 0.0, M, h.st);
    NMat O = h.W2.view(h.g, m, h.st);
    pnd::KStageArgs a{};
    a.bcat = &h.bcat;
    a.geo = h.g;
    a.X = X;
    a.M = M;
    a.inv_s = h.isp.p + 2 * (size_t)h.g.halo;
    a.out = O;
    pnd::kstage(a, h.st);
    download_rows(h, O, out, m, 0);
    CK(cudaStreamSynchronize(h.st));
    mneg.free_();
  });
}

int pnd_fullrank_reset(pnd_handle* hh) {
  return guard(hh, [&](Handle& h) { pnd::fullrank_reset(h); });
}

int pnd_fullrank_set(pnd_handle* hh, const double* u) {
  return guard(hh, [&](Handle& h) {
    const int n = h.g.n, m = h.m;
    for (size_t i = 0; i < (size_t)n * m; ++i)
      if (!std::isfinite(u[i])) pnd::fail(PND_ENUMERICAL, "non-finite full-rank state");
    pnd::fullrank_reset(h);
    for (int b = 0; b < pnd::fullrank_blocks(h); ++b) {
      const NMat blk = pnd::fullrank_block(h, b);
      CK(cudaMemcpy2DAsync(blk.p, blk.rs * sizeof(double), u + 32 * b, m * sizeof(double),
                           blk.cols * sizeof(double), n, cudaMemcpyHostToDevice, h.st));
    }
    CK(cudaStreamSynchronize(h.st));
  });
}

int pnd_fullrank_get(pnd_handle* hh, double* u) {
  return guard(hh, [&](Handle& h) {
    if (!h.have_fr) pnd::fail(PND_ECONFIG, "no full-rank state");
    for (int b = 0; b < pnd::fullrank_blocks(h); ++b)
      download_rows(h, pnd::fullrank_block(h, b), u, h.m, 32 * b);
    CK(cudaStreamSynchronize(h.st));
  });
}

int pnd_fullrank_streaming_step(pnd_handle* hh, double dt) {
  return guard(hh, [&](Handle& h) { pnd::fullrank_streaming_step(h, dt); });
}

int pnd_fullrank_scattering_step(pnd_handle* hh, double dt) {
  return guard(hh, [&](Handle& h) { pnd::fullrank_scattering_step(h, dt); });
}

int pnd_fullrank_step(pnd_handle* hh, double dt, int tally_steps) {
  return guard(hh, [&](Handle& h) {
    pnd::fullrank_streaming_step(h, dt);
    pnd::fullrank_scattering_step(h, dt);
    pnd::fullrank_dose_step(h, dt, tally_steps != 0);
  });
}

int pnd_stencil_grams(pnd_handle* hh, const double* x, int a, const double* y, int b,
                      double* out) {
  return guard(hh, [&](Handle& h) {
    if (!h.stencil_error.empty()) pnd::fail(PND_ECONFIG, h.stencil_error);
    if (!h.have_inv_s) pnd::fail(PND_ECONFIG, "set inv_s first");
    NMat X = h.W1.view(h.g, a, h.st);
    NMat Y = h.W2.view(h.g, b, h.st);
    upload_rows(h, X, x);
    upload_rows(h, Y, y);
    pnd::DBuf o;
    double* O = o.get((size_t)h.g.ns * a * b + 1);
    if (a + b > 64) {
      // wider than one S-Gram launch: the block pairs of the streaming step
      std::vector<NMat> bl = pnd::split_blocks(h, Y, h.wide_u0b);
      const int nby = (int)bl.size();
      for (const NMat& q : pnd::split_blocks(h, X, h.wide_qb)) bl.push_back(q);
      const int w = a + b;
      pnd::DBuf full;
      double* F = full.get((size_t)h.g.ns * w * w);
      pnd::stencil_grams_blocks(h, bl, h.isp.p + 2 * (size_t)h.g.halo, F);
      (void)nby;
      // the (X, D Y) block: rows b.., columns 0..b (G = [Y | X]^T D [Y | X])
      for (int s2 = 0; s2 < h.g.ns; ++s2)
        CK(cudaMemcpy2DAsync(O + (size_t)s2 * a * b, b * sizeof(double),
                             F + ((size_t)s2 * w + b) * w, w * sizeof(double), b * sizeof(double),
                             a, cudaMemcpyDeviceToDevice, h.st));
      CK(cudaStreamSynchronize(h.st));
      full.free_();
    } else {
      pnd::stencil_grams_xy(h.g, X, Y, h.isp.p + 2 * (size_t)h.g.halo, O, h.part, h.st);
    }
    down(out, O, (size_t)h.g.ns * a * b, h.st);
    CK(cudaStreamSynchronize(h.st));
    o.free_();
  });
}

int pnd_augment_basis(pnd_handle* hh, const double* u, int a, const double* x, int b,
                      int rank_bound, double* q, int* k_out) {
  return guard(hh, [&](Handle& h) {
    if (a < 0 || b < 1 || a > 64 || b > 64) pnd::fail(PND_ECONFIG, "augment_basis: 0 <= a, 1 <= b <= 64");
    h.ua = a;
    h.uq = 0;
    if (a > 0) upload_rows(h, h.U.view(h.g, a, h.st), u);
    NMat X = h.W2.view(h.g, b, h.st);
    upload_rows(h, X, x);
    pnd::DBuf c1;
    double* C1 = c1.get((size_t)(a > 0 ? a : 1) * b);
    if (a > 0) pnd::gram_xy(h.g, pnd::state_u(h), X, C1, h.part, h.st);
    const int k = pnd::orth_complement(h, X, a > 0 ? C1 : nullptr, NMat{},
                                       rank_bound > 0 ? rank_bound : (1 << 30));
    if (k > 0) download_rows(h, pnd::state_q(h), q, b, 0);
    CK(cudaStreamSynchronize(h.st));
    *k_out = k;
    h.uq = 0;
    c1.free_();
  });
}

int pnd_k_rhs(pnd_handle* hh, const double* k, int r, const double* f, double* out) {
  return guard(hh, [&](Handle& h) {
    if (!h.stencil_error.empty()) pnd::fail(PND_ECONFIG, h.stencil_error);
    if (!h.have_inv_s) pnd::fail(PND_ECONFIG, "set inv_s first");
    const int ns = h.g.ns;
    NMat K = h.W1.view(h.g, r, h.st);
    upload_rows(h, K, k);
    pnd::DBuf dm;
    double* M = dm.get((size_t)ns * r * r + 1);
    up(M, f, (size_t)ns * r * r, h.st);
    pnd::axpby(ns * r * r, -1.0, M, 0.0, M, h.st);
    NMat O = h.W2.view(h.g, r, h.st);
    if (r > 32) {
      // ranks above 32: the block chain of the streaming step (wide.cu)
      const auto xb = pnd::split_blocks(h, K, h.wide_w1b);
      const auto ob = pnd::block_views(h, h.wide_w2b, r);
      pnd::kstage_blocks(h, xb, NMat{}, nullptr, M, ob, false, false);
      int c0 = 0;
      for (size_t b = 0; b < ob.size(); ++b) {
        download_rows(h, ob[b], out, r, c0);
        c0 += ob[b].cols;
      }
    } else {
      pnd::KStageArgs a{};
      a.bcat = &h.bcat;
      a.geo = h.g;
      a.X = K;
      a.M = M;
      a.inv_s = h.isp.p + 2 * (size_t)h.g.halo;
      a.out = O;
      pnd::kstage(a, h.st);
      download_rows(h, O, out, r, 0);
    }
    CK(cudaStreamSynchronize(h.st));
    dm.free_();
  });
}

int pnd_orthonormalize(pnd_handle* hh, const double* a, int rows, int cols, double* q,
                       double* r) {
  return guard(hh, [&](Handle& h) {
    if (rows < 1 || cols < 1) pnd::fail(PND_ECONFIG, "empty matrix");
    const int kc = rows < cols ? rows : cols;
    pnd::DBuf st, da, dq, dr;
    double* s = st.get((size_t)rows * cols);
    up(s, a, (size_t)rows * cols, h.st);
    double* A = da.get((size_t)rows * cols);
    pnd::transpose_in(s, rows, cols, A, rows, h.st);
    double* Q = dq.get((size_t)rows * kc);
    double* R = dr.get((size_t)kc * cols);
    pnd::TsqrWork w;
    pnd::tsqr(A, rows, cols, rows, Q, rows, R, w, h.st);
    pnd::transpose_out(Q, rows, rows, kc, s, h.st);
    down(q, s, (size_t)rows * kc, h.st);
    if (r) down(r, R, (size_t)kc * cols, h.st);
    CK(cudaStreamSynchronize(h.st));
    w.tau.free_(); w.tree.free_(); w.rbuf.free_(); w.cbuf.free_();
    st.free_(); da.free_(); dq.free_(); dr.free_();
  });
}

int pnd_svd_small(pnd_handle* hh, const double* s, int p, int q, double* pm, double* sig,
                  double* qt) {
  return guard(hh, [&](Handle& h) {
    const int k = p < q ? p : q;
    pnd::DBuf ds, dp, dsig, dq;
    double* S = ds.get((size_t)p * q);
    up(S, s, (size_t)p * q, h.st);
    double* P = dp.get((size_t)p * k);
    double* G = dsig.get(k);
    double* Q = dq.get((size_t)k * q);
    pnd::svd_small(S, p, q, P, G, Q, nullptr, h.st);
    down(pm, P, (size_t)p * k, h.st);
    down(sig, G, k, h.st);
    down(qt, Q, (size_t)k * q, h.st);
    CK(cudaStreamSynchronize(h.st));
    ds.free_(); dp.free_(); dsig.free_(); dq.free_();
  });
}

int pnd_traverse(pnd_handle* hh, const double* origin3, int n_rays, const double* starts,
                 const double* dirs, int32_t* counts, const int64_t* offsets, int64_t* cells,
                 double* t0, double* t1) {
  return guard(hh, [&](Handle& h) {
    if (n_rays <= 0) return;
    pnd::DBuf ds, dd, dt0, dt1;
    pnd::IBuf dc;
    double* S = ds.get((size_t)n_rays * 3);
    double* D = dd.get((size_t)n_rays * 3);
    up(S, starts, (size_t)n_rays * 3, h.st);
    up(D, dirs, (size_t)n_rays * 3, h.st);
    if (!cells) {
      int* C = dc.get(n_rays);
      pnd::traverse(h.g, origin3, n_rays, S, D, C, nullptr, nullptr, nullptr, nullptr, h.st);
      CK(cudaMemcpyAsync(counts, C, sizeof(int) * n_rays, cudaMemcpyDeviceToHost, h.st));
      CK(cudaStreamSynchronize(h.st));
    } else {
      const long long total = offsets[n_rays];
      long long* O = nullptr;
      long long* CE = nullptr;
      CK(cudaMalloc(&O, sizeof(long long) * (n_rays + 1)));
      CK(cudaMalloc(&CE, sizeof(long long) * (total > 0 ? total : 1)));
      double* T0 = dt0.get(total > 0 ? total : 1);
      double* T1 = dt1.get(total > 0 ? total : 1);
      CK(cudaMemcpyAsync(O, offsets, sizeof(long long) * (n_rays + 1), cudaMemcpyHostToDevice,
                         h.st));
      pnd::traverse(h.g, origin3, n_rays, S, D, nullptr, O, CE, T0, T1, h.st);
      CK(cudaMemcpyAsync(cells, CE, sizeof(long long) * total, cudaMemcpyDeviceToHost, h.st));
      down(t0, T0, total, h.st);
      down(t1, T1, total, h.st);
      CK(cudaStreamSynchronize(h.st));
      cudaFree(O);
      cudaFree(CE);
    }
    ds.free_(); dd.free_(); dt0.free_(); dt1.free_(); dc.free_();
  });
}

namespace {
// split dense block-tridiagonal G (ndof x ndof row-major, nl x nl blocks) into
// D / L / U block arrays [g][nl][nl]
void split_blocks(const double* G, int ng, int nl, double* D, double* L, double* U) {
  const int ndof = ng * nl, b2 = nl * nl;
  for (int g = 0; g < ng; ++g)
    for (int i = 0; i < nl; ++i)
      for (int j = 0; j < nl; ++j) {
        const size_t row = (size_t)(g * nl + i) * ndof;
        D[g * b2 + i * nl + j] = G[row + g * nl + j];
        L[g * b2 + i * nl + j] = g > 0 ? G[row + (g - 1) * nl + j] : 0.0;
        U[g * b2 + i * nl + j] = g + 1 < ng ? G[row + (g + 1) * nl + j] : 0.0;
      }
}
}  // namespace

int pnd_march(pnd_handle* hh, int nl, int ng, int n_keys, const double* gmats,
              const double* mass, const double* p_lo, double e_min, const double* s_min,
              const double* psi0, int n_steppers, const int32_t* st_key, const double* st_dz,
              int n_marches, const int32_t* seg_off, const int32_t* seg_key,
              const double* half_dz, const int32_t* half_n, const int32_t* half_st,
              double* averages, double* residual, double* psi_exit) {
  return guard(hh, [&](Handle& h) {
    if (nl < 1 || nl > 4 || ng < 1) pnd::fail(PND_ECONFIG, "bad energy DG space");
    if (n_marches <= 0) return;
    const int ndof = ng * nl, b2 = nl * nl;
    const int nseg = seg_off[n_marches];
    // operator blocks: reject couplings beyond the neighbour groups
    std::vector<double> D((size_t)n_keys * ng * b2), L(D.size()), U(D.size());
    for (int k = 0; k < n_keys; ++k) {
      const double* G = gmats + (size_t)k * ndof * ndof;
      for (int r = 0; r < ndof; ++r)
        for (int c = 0; c < ndof; ++c) {
          const int gr = r / nl, gc = c / nl;
          if ((gr - gc > 1 || gc - gr > 1) && G[(size_t)r * ndof + c] != 0.0)
            pnd::fail(PND_ECONFIG, "energy operator is not block tridiagonal");
        }
      split_blocks(G, ng, nl, D.data() + (size_t)k * ng * b2, L.data() + (size_t)k * ng * b2,
                   U.data() + (size_t)k * ng * b2);
    }
    pnd::DBuf dD, dL, dU, dm, dpl, dsm, dps, dsz, dhz, dinv, dE, dpsi, dtmp, dav, dres;
    pnd::IBuf ik, iso, isk, ihn, ihs, ibad;
    double* Dd = dD.get(D.size());
    double* Ld = dL.get(L.size());
    double* Ud = dU.get(U.size());
    up(Dd, D.data(), D.size(), h.st);
    up(Ld, L.data(), L.size(), h.st);
    up(Ud, U.data(), U.size(), h.st);
    double* md = dm.get(ndof);
    up(md, mass, ndof, h.st);
    double* pld = dpl.get(nl);
    up(pld, p_lo, nl, h.st);
    double* smd = dsm.get(n_keys);
    up(smd, s_min, n_keys, h.st);
    double* psd = dps.get(ndof);
    up(psd, psi0, ndof, h.st);
    int* kd = ik.get(n_steppers);
    CK(cudaMemcpyAsync(kd, st_key, sizeof(int) * n_steppers, cudaMemcpyHostToDevice, h.st));
    double* szd = dsz.get(n_steppers);
    up(szd, st_dz, n_steppers, h.st);
    int* sod = iso.get(n_marches + 1);
    CK(cudaMemcpyAsync(sod, seg_off, sizeof(int) * (n_marches + 1), cudaMemcpyHostToDevice,
                       h.st));
    int* skd = isk.get(nseg > 0 ? nseg : 1);
    CK(cudaMemcpyAsync(skd, seg_key, sizeof(int) * nseg, cudaMemcpyHostToDevice, h.st));
    double* hzd = dhz.get(2 * (size_t)(nseg > 0 ? nseg : 1));
    up(hzd, half_dz, 2 * (size_t)nseg, h.st);
    int* hnd = ihn.get(2 * (size_t)(nseg > 0 ? nseg : 1));
    CK(cudaMemcpyAsync(hnd, half_n, sizeof(int) * 2 * nseg, cudaMemcpyHostToDevice, h.st));
    int* hsd = ihs.get(2 * (size_t)(nseg > 0 ? nseg : 1));
    CK(cudaMemcpyAsync(hsd, half_st, sizeof(int) * 2 * nseg, cudaMemcpyHostToDevice, h.st));
    int* bad = ibad.get(1);
    CK(cudaMemsetAsync(bad, 0, sizeof(int), h.st));
    double* Dinv = dinv.get((size_t)n_steppers * ng * b2);
    double* E = dE.get((size_t)n_steppers * ng * b2);
    pnd::march_steppers(nl, Dd, Ld, Ud, md, ng, n_steppers, kd, szd, Dinv, E, bad, h.st);
    double* psi = dpsi.get((size_t)n_marches * ndof);
    double* tmp = dtmp.get((size_t)n_marches * ndof);
    double* av = dav.get((size_t)(nseg > 0 ? nseg : 1) * ng);
    double* rs = dres.get(nseg > 0 ? nseg : 1);
    pnd::march_rays(nl, Dd, Ld, Ud, md, ng, Dinv, E, szd, n_marches, sod, skd, hzd, hnd, hsd,
                    smd, e_min, psd, pld, psi, tmp, av, rs, bad, h.st);
    int hbad = 0;
    CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, h.st));
    if (averages) down(averages, av, (size_t)nseg * ng, h.st);
    if (residual) down(residual, rs, nseg, h.st);
    if (psi_exit) down(psi_exit, psi, (size_t)n_marches * ndof, h.st);
    CK(cudaStreamSynchronize(h.st));
    if (hbad == 1) pnd::fail(PND_ENUMERICAL, "Crank-Nicolson solve failed: singular block");
    if (hbad == 2) pnd::fail(PND_ENUMERICAL, "ray march produced non-finite flux");
  });
}

int pnd_deposit(pnd_handle* hh, int ng, int n_rays, const int32_t* ray_seg_off,
                const int64_t* cells, const double* lengths, const int32_t* ray_march,
                const int32_t* march_seg_off, const double* weight, double volume,
                int n_march_segs, const double* averages, const double* mres, double* values,
                double* residual) {
  return guard(hh, [&](Handle& h) {
    const int n = h.g.n, ld = h.g.ld;
    pnd::DBuf dv, dr, dl, dw, da, dm;
    pnd::IBuf io, im, ims;
    double* V = dv.get((size_t)ng * ld);
    double* R = dr.get(ld);
    pnd::fill_zero(V, (size_t)ng * ld, h.st);
    pnd::fill_zero(R, ld, h.st);
    if (n_rays > 0) {
      const int nseg = ray_seg_off[n_rays];
      int* od = io.get(n_rays + 1);
      CK(cudaMemcpyAsync(od, ray_seg_off, sizeof(int) * (n_rays + 1), cudaMemcpyHostToDevice,
                         h.st));
      long long* cd = nullptr;
      CK(cudaMalloc(&cd, sizeof(long long) * (nseg > 0 ? nseg : 1)));
      CK(cudaMemcpyAsync(cd, cells, sizeof(long long) * nseg, cudaMemcpyHostToDevice, h.st));
      double* ldv = dl.get(nseg > 0 ? nseg : 1);
      up(ldv, lengths, nseg, h.st);
      int* rmd = im.get(n_rays);
      CK(cudaMemcpyAsync(rmd, ray_march, sizeof(int) * n_rays, cudaMemcpyHostToDevice, h.st));
      int n_m = 0;
      for (int r = 0; r < n_rays; ++r) n_m = ray_march[r] + 1 > n_m ? ray_march[r] + 1 : n_m;
      int* msd = ims.get(n_m + 1);
      CK(cudaMemcpyAsync(msd, march_seg_off, sizeof(int) * (n_m + 1), cudaMemcpyHostToDevice,
                         h.st));
      double* wd = dw.get(n_rays);
      up(wd, weight, n_rays, h.st);
      double* ad = da.get((size_t)(n_march_segs > 0 ? n_march_segs : 1) * ng);
      up(ad, averages, (size_t)n_march_segs * ng, h.st);
      double* mrd = dm.get(n_march_segs > 0 ? n_march_segs : 1);
      up(mrd, mres, n_march_segs, h.st);
      pnd::deposit_rays(n_rays, od, cd, ldv, rmd, msd, wd, volume, ad, mrd, V, ld, R, ng, h.st);
      CK(cudaStreamSynchronize(h.st));
      cudaFree(cd);
    }
    pnd::DBuf dt;
    if (values) {
      double* T = dt.get((size_t)n * ng);
      pnd::transpose_out(V, ld, n, ng, T, h.st);  // (n x ng) row-major, the reference layout
      down(values, T, (size_t)n * ng, h.st);
    }
    if (residual) down(residual, R, n, h.st);
    CK(cudaStreamSynchronize(h.st));
  });
}

int pnd_comm_unique_id(char* out128) {
  try {
    pnd::comm_unique_id(out128);
    return PND_OK;
  } catch (const pnd::Error& e) {
    return e.code;
  } catch (...) {
    return PND_EDEVICE;
  }
}

int pnd_set_slab(pnd_handle* hh, int z0, int nz_global, const char* id128, int rank, int world) {
  return guard(hh, [&](Handle& h) {
    pnd::Geom& g = h.g;
    if (z0 < 0 || nz_global < g.nz || z0 + g.nz > nz_global)
      pnd::fail(PND_ECONFIG, "slab planes outside the global grid");
    if (world > 1 && g.nz < 2) pnd::fail(PND_ECONFIG, "a slab needs at least 2 planes");
    if (world < 1 || rank < 0 || rank >= world) pnd::fail(PND_ECONFIG, "bad rank / world");
    g.z0 = z0;
    g.nzg = nz_global;
    // active axes and the 2-cell rule follow the global grid (spatial.py:84-88)
    const int dims[3] = {g.nx, g.ny, nz_global};
    h.stencil_error.clear();
    const char* names[3] = {"nx", "ny", "nz"};
    for (int a = 0; a < 3; ++a)
      if (dims[a] == 2 && h.stencil_error.empty())
        h.stencil_error = std::string("grid.") + names[a] +
                          "=2: grids with 2 cells along a used axis cannot host the 3-point "
                          "one-sided stencil; use 1 (inactive) or >= 3";
    g.na = 0;
    for (int a = 0; a < 3; ++a)
      if (dims[a] > 1) g.axis[g.na++] = a;
    for (int a = g.na; a < 3; ++a) g.axis[a] = 0;
    g.ns = 2 * g.na;
    pnd::comm_destroy(h.comm);
    h.comm = nullptr;
    bool have_id = false;
    for (int i = 0; id128 && i < 128 && !have_id; ++i) have_id = id128[i] != 0;
    // a communicator whenever an id is given (world 1 included: exercises the
    // transport's setup on a single GPU; its exchanges are no-ops there)
    if (have_id) h.comm = pnd::comm_create(id128, rank, world);
    g.comm = h.comm;
  });
}

int pnd_timing(pnd_handle* hh, int enable) {
  return guard(hh, [&](Handle& h) {
    CK(cudaStreamSynchronize(h.st));
    h.timer.on = enable != 0;
    h.timer.used = 0;
    h.timer.ids.clear();
  });
}

int pnd_timing_get(pnd_handle* hh, int nphase, double* ms, int* count) {
  return guard(hh, [&](Handle& h) {
    CK(cudaStreamSynchronize(h.st));
    for (int i = 0; i < nphase; ++i) {
      ms[i] = 0.0;
      count[i] = 0;
    }
    pnd::TimerState& t = h.timer;
    for (size_t i = 0; i + 1 < t.used; ++i) {
      const int id = t.ids[i];
      if (id < 0 || id >= nphase) continue;
      float e = 0.f;
      CK(cudaEventElapsedTime(&e, t.pool[i], t.pool[i + 1]));
      ms[id] += e;
      count[id] += 1;
    }
    t.used = 0;
    t.ids.clear();
  });
}

int pnd_event_record(pnd_handle* hh, int slot) {
  return guard(hh, [&](Handle& h) {
    if (slot < 0 || slot >= 8) pnd::fail(PND_ECONFIG, "event slot out of range");
    if (!h.timer.ev[slot]) CK(cudaEventCreate(&h.timer.ev[slot]));
    CK(cudaEventRecord(h.timer.ev[slot], h.st));
  });
}

int pnd_event_elapsed(pnd_handle* hh, int a, int b, double* ms) {
  return guard(hh, [&](Handle& h) {
    CK(cudaEventSynchronize(h.timer.ev[b]));
    float e = 0.f;
    CK(cudaEventElapsedTime(&e, h.timer.ev[a], h.timer.ev[b]));
    *ms = e;
  });
}

int pnd_launch_count(pnd_handle* hh, long long* count) {
  return guard(hh, [&](Handle&) { *count = pnd::launch_count(); });
}

int pnd_set_flux_separable(pnd_handle* hh, int beam, int n_beams, int n_groups,
                           const double* lateral, const double* depth, const double* t_m) {
  return guard(hh, [&](Handle& h) {
    if (n_beams < 1 || n_beams > 4) pnd::fail(PND_ECONFIG, "1..4 beams supported");
    if (beam < 0 || beam >= n_beams) pnd::fail(PND_ECONFIG, "beam index out of range");
    const int nxy = h.g.nx * h.g.ny;
    if (beam == 0) {
      h.n_groups = n_groups;
      h.n_beams = n_beams;
      h.flux.free_();  // the factors replace any dense tables
      h.flux_sep = true;
      h.flux_sparse = false;
      h.sep_lat.get((size_t)n_beams * nxy);
      h.sep_depth.get((size_t)n_beams * h.g.nz * n_groups);
      h.psi.get((size_t)n_beams * h.g.ld + 64);
      h.psi_lo.get((size_t)n_beams * h.g.ld);
      h.tm.get((size_t)n_beams * h.m);
    } else if (!h.flux_sep || n_beams != h.n_beams || n_groups != h.n_groups) {
      pnd::fail(PND_ECONFIG, "separable flux: set beam 0 first with the same beam/group counts");
    }
    up(h.sep_lat.p + (size_t)beam * nxy, lateral, nxy, h.st);
    up(h.sep_depth.p + (size_t)beam * h.g.nz * n_groups, depth, (size_t)h.g.nz * n_groups, h.st);
    up(h.tm.p + (size_t)beam * h.m, t_m, h.m, h.st);
    CK(cudaStreamSynchronize(h.st));
  });
}

int pnd_state_random(pnd_handle* hh, int r, unsigned long long seed) {
  return guard(hh, [&](Handle& h) {
    if (r < 1 || r > 256) pnd::fail(PND_ECONFIG, "random state rank must be 1..256");
    const int m = h.m;
    // U = orth(random n x r) through the device Gram-Schmidt/SVQB passes
    int k;
    if (r > 64) {
      k = pnd::random_state_x(h, r, seed);
    } else {
      NMat X = h.Xs.view(h.g, r, h.st);
      pnd::random_rows(h.g, X, seed, h.st);
      h.ua = 0;
      h.uq = 0;
      h.blocked = false;
      k = pnd::orth_complement(h, X, nullptr);
      std::swap(h.U, h.Q);
      h.ua = k;
      h.uq = 0;
    }
    double* B = h.sm[44].get((size_t)m * r);
    double* Vc = h.sm[43].get((size_t)m * r);
    double* R = h.sm[45].get((size_t)r * r);
    // V = orth(random m x r) on the moment side (TSQR)
    {
      pnd::DBuf tmp;
      double* t = tmp.get((size_t)m * r);
      std::vector<double> host((size_t)m * r);
      unsigned long long x = seed * 7919ULL + 1;
      for (auto& v : host) {
        x = x * 6364136223846793005ULL + 1442695040888963407ULL;
        v = (double)(x >> 11) * (1.0 / 9007199254740992.0) - 0.5;
      }
      up(B, host.data(), host.size(), h.st);
      pnd::tsqr(B, m, r, m, Vc, m, R, h.tq_m, h.st);
      pnd::transpose_out(Vc, m, m, r, h.V.get((size_t)m * r), h.st);
      CK(cudaStreamSynchronize(h.st));
      tmp.free_();
    }
    double* S = h.S.get((size_t)k * r);
    pnd::logdiag_kernel<<<1, 256, 0, h.st>>>(S, k);
    pnd::launched();
    CK(cudaStreamSynchronize(h.st));
    h.ru = h.rv = k;
  });
}

}  // extern "C"
