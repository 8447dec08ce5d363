// Z-slab decomposition over NVLink: halo planes and Gram allreduces (NCCL).
//
// One process per GPU owns planes [z0, z0 + nz) of the global grid (SURVEY.md
// §8(e), paper_2508_04484_b200/slabs.py). The energy step needs only two kinds
// of communication:
//   - the upwind stencils reach 2 planes along z: before a stencil kernel reads
//     a matrix, its 2 boundary planes go to each neighbour, straight into the
//     neighbour's halo rows (the cell-major layout keeps 2 nx*ny zero rows
//     before and after every matrix, so a received plane lands where a local
//     one would be; at the global faces the halo stays zero, which is the
//     reference's zero-inflow closure);
//   - every reduction over cells (stencil Grams, augmentation Grams, B_i,
//     source projections, the defect Gram) is an FP64 sum of a small block:
//     one allreduce after the per-device reduction. All m-side and R x R work
//     then runs replicated on bit-identical inputs.
// NCCL is loaded with dlopen on first use (the library itself has no link-time
// NCCL dependency; single-GPU handles never touch it).
//
// A second transport, "local", serves the tests: several handles of one
// process (one host thread each) on one GPU exchange their halo planes with
// device-to-device copies and sum their Gram blocks on the host, meeting at a
// host barrier. No kernel ever waits on another rank, so this is safe on a
// single GPU (unlike NCCL ranks sharing one device) and checks the whole slab
// logic -- global boundary classes, halo placement, masked chunk tails, every
// allreduce site -- against the undecomposed solve.
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "pnd.h"

namespace pnd {

namespace {

struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  if (!a.lib) {
    a.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.lib) fail(PND_EDEVICE, std::string("cannot load libnccl.so.2: ") + dlerror());
    auto sym = [&](const char* name) {
      void* p = dlsym(a.lib, name);
      if (!p) fail(PND_EDEVICE, std::string("libnccl.so.2 lacks ") + name);
      return p;
    };
    a.getUniqueId = (decltype(a.getUniqueId))sym("ncclGetUniqueId");
    a.commInitRank = (decltype(a.commInitRank))sym("ncclCommInitRank");
    a.commDestroy = (decltype(a.commDestroy))sym("ncclCommDestroy");
    a.allReduce = (decltype(a.allReduce))sym("ncclAllReduce");
    a.send = (decltype(a.send))sym("ncclSend");
    a.recv = (decltype(a.recv))sym("ncclRecv");
    a.groupStart = (decltype(a.groupStart))sym("ncclGroupStart");
    a.groupEnd = (decltype(a.groupEnd))sym("ncclGroupEnd");
    a.errorString = (decltype(a.errorString))sym("ncclGetErrorString");
  }
  return a;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(PND_EDEVICE, std::string(what) + ": " + api().errorString(r));
}

}  // namespace

namespace {

struct LocalWorld {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  std::vector<double*> rows;            // published halo bases (row 0 of each rank)
  std::vector<int> n, rs;
  std::vector<std::vector<double>> red;  // published Gram blocks

  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else if (!cv.wait_for(lk, std::chrono::seconds(120),
                            [&] { return generation != gen; })) {
      // a rank that failed never arrives: report instead of hanging the caller
      --arrived;
      lk.unlock();
      fail(PND_EDEVICE, "local slab transport: a peer rank did not reach the barrier");
    }
  }
};

std::mutex g_worlds_mu;
std::map<std::string, std::shared_ptr<LocalWorld>> g_worlds;

}  // namespace

struct Comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  std::shared_ptr<LocalWorld> local;  // "local:" transport (tests on one GPU)
};

void comm_unique_id(char* out) {
  ncclUniqueId id;
  nck(api().getUniqueId(&id), "ncclGetUniqueId");
  for (int i = 0; i < NCCL_UNIQUE_ID_BYTES; ++i) out[i] = id.internal[i];
}

Comm* comm_create(const char* id_bytes, int rank, int world) {
  auto* c = new Comm();
  c->rank = rank;
  c->world = world;
  if (std::strncmp(id_bytes, "local:", 6) == 0) {
    const std::string key(id_bytes, strnlen(id_bytes, NCCL_UNIQUE_ID_BYTES));
    std::lock_guard<std::mutex> lk(g_worlds_mu);
    auto& w = g_worlds[key];
    if (!w) {
      w = std::make_shared<LocalWorld>();
      w->world = world;
      w->rows.assign(world, nullptr);
      w->n.assign(world, 0);
      w->rs.assign(world, 0);
      w->red.assign(world, {});
    }
    c->local = w;
    return c;
  }
  ncclUniqueId id;
  for (int i = 0; i < NCCL_UNIQUE_ID_BYTES; ++i) id.internal[i] = id_bytes[i];
  nck(api().commInitRank(&c->comm, world, id, rank), "ncclCommInitRank");
  return c;
}

void comm_destroy(Comm* c) {
  if (!c) return;
  if (c->comm) api().commDestroy(c->comm);
  delete c;
}

int comm_world(const Geom& g) {
  auto* c = static_cast<Comm*>(g.comm);
  return c ? c->world : 1;
}

void comm_allreduce(const Geom& g, double* p, size_t count, cudaStream_t st) {
  auto* c = static_cast<Comm*>(g.comm);
  if (!c || c->world <= 1 || count == 0) return;
  if (c->local) {
    LocalWorld& w = *c->local;
    std::vector<double>& mine = w.red[c->rank];
    mine.resize(count);
    CK(cudaMemcpyAsync(mine.data(), p, count * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    w.barrier();
    std::vector<double> sum(count, 0.0);
    for (int r = 0; r < w.world; ++r)  // rank order: every rank gets the same bits
      for (size_t i = 0; i < count; ++i) sum[i] += w.red[r][i];
    w.barrier();
    CK(cudaMemcpyAsync(p, sum.data(), count * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    return;
  }
  nck(api().allReduce(p, p, count, ncclFloat64, ncclSum, c->comm, st), "ncclAllReduce");
}

void comm_halo_rows(const Geom& g, double* rows, int rs, cudaStream_t st) {
  auto* c = static_cast<Comm*>(g.comm);
  if (!c || c->world <= 1) return;
  const size_t nxy = (size_t)g.nx * g.ny, cnt = 2 * nxy * rs;
  const size_t n = (size_t)g.n;
  if (c->local) {
    LocalWorld& w = *c->local;
    CK(cudaStreamSynchronize(st));
    w.rows[c->rank] = rows;
    w.n[c->rank] = g.n;
    w.rs[c->rank] = rs;
    w.barrier();
    // write my boundary planes into the neighbours' halo rows
    if (c->rank > 0) {
      if (w.rs[c->rank - 1] != rs) fail(PND_ECONFIG, "slab halo exchange: row length mismatch");
      double* dst = w.rows[c->rank - 1] + (size_t)w.n[c->rank - 1] * rs;
      CK(cudaMemcpyAsync(dst, rows, cnt * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    if (c->rank + 1 < c->world) {
      double* dst = w.rows[c->rank + 1] - 2 * nxy * rs;
      CK(cudaMemcpyAsync(dst, rows + (n - 2 * nxy) * rs, cnt * sizeof(double),
                         cudaMemcpyDeviceToDevice, st));
    }
    CK(cudaStreamSynchronize(st));
    w.barrier();
    return;
  }
  NcclApi& a = api();
  nck(a.groupStart(), "ncclGroupStart");
  if (c->rank > 0) {
    // my first 2 planes -> the lower neighbour's upper halo; its last 2 -> mine
    nck(a.send(rows, cnt, ncclFloat64, c->rank - 1, c->comm, st), "ncclSend");
    nck(a.recv(rows - 2 * nxy * rs, cnt, ncclFloat64, c->rank - 1, c->comm, st), "ncclRecv");
  }
  if (c->rank + 1 < c->world) {
    nck(a.send(rows + (n - 2 * nxy) * rs, cnt, ncclFloat64, c->rank + 1, c->comm, st),
        "ncclSend");
    nck(a.recv(rows + n * rs, cnt, ncclFloat64, c->rank + 1, c->comm, st), "ncclRecv");
  }
  nck(a.groupEnd(), "ncclGroupEnd");
}

void comm_halo(const Geom& g, NMat X, cudaStream_t st) { comm_halo_rows(g, X.p, X.rs, st); }

}  // namespace pnd
