// Rank-to-rank transports of the z-slab decomposition:
//   - NcclTransport: one process per GPU; halo planes by ncclSend / ncclRecv inside one group,
//     dot products by ncclAllReduce, the coarse right-hand side by ncclAllGather.  Everything is
//     enqueued on the caller's stream (capturable into the solve's CUDA graph).
//   - LoopTransport: several contexts of ONE process (one host thread each) for correctness tests
//     on a single GPU.  Every exchange first synchronises the caller's stream, meets the other
//     ranks at a host barrier and then copies device to device; no kernel ever waits for another
//     rank (B200_PROFILING.md: kernels that wait on one another must not share a GPU).
#include "comm.h"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>   // types only: the library is resolved at run time (below)

#include <condition_variable>
#include <mutex>
#include <type_traits>
#include <vector>

namespace pmg {

// NCCL is opened on first use with dlopen instead of being a link-time dependency: a process that
// already holds a libnccl.so.2 (torch ships its own) keeps using that one (RTLD_NOLOAD finds it),
// and a one-GPU process never loads NCCL at all -- two different libnccl.so.2 in one process
// break whichever of the two was resolved second.
namespace {
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string err;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW);
    if (!h) { api.err = std::string("cannot load libnccl.so.2: ") + dlerror(); return; }
    bool ok = true;
    auto get = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) ok = false;
    };
    get(api.GetUniqueId, "ncclGetUniqueId");
    get(api.CommInitRank, "ncclCommInitRank");
    get(api.CommDestroy, "ncclCommDestroy");
    get(api.GroupStart, "ncclGroupStart");
    get(api.GroupEnd, "ncclGroupEnd");
    get(api.Send, "ncclSend");
    get(api.Recv, "ncclRecv");
    get(api.AllReduce, "ncclAllReduce");
    get(api.AllGather, "ncclAllGather");
    get(api.GetErrorString, "ncclGetErrorString");
    if (!ok) api.err = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}
}  // namespace

// ------------------------------------------------------------------------------------ plan
int slab_plan(int k3, int nranks, int rank, SlabPlan* out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks || k3 < nranks) return -1;
  SlabPlan s;
  s.z0 = (int)((long long)rank * k3 / nranks);
  s.z1 = (int)((long long)(rank + 1) * k3 / nranks);
  s.zb = s.z0 > 0 ? s.z0 - 1 : 0;
  s.nplanes = s.z1 - s.zb + 1;
  s.own_lo = s.z0 - s.zb;
  s.own_hi = (rank == nranks - 1) ? s.nplanes : s.nplanes - 1;
  s.lower = rank > 0 ? rank - 1 : -1;
  s.upper = rank < nranks - 1 ? rank + 1 : -1;
  *out = s;
  return 0;
}

// ------------------------------------------------------------------------------------ NCCL
namespace {
std::string nccl_err(const char* what, ncclResult_t r) { return std::string(what) + ": " + nccl().GetErrorString(r); }

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  ~NcclTransport() override {
    if (comm) nccl().CommDestroy(comm);
  }
  bool graph_safe() const override { return true; }
  std::string halo(const double* send_lo, double* recv_lo, const double* send_hi, double* recv_hi, size_t n,
                   cudaStream_t st) override {
    ncclResult_t r = nccl().GroupStart();
    if (r != ncclSuccess) return nccl_err("ncclGroupStart", r);
    if (send_lo && rank > 0) {
      if ((r = nccl().Send(send_lo, n, ncclDouble, rank - 1, comm, st)) != ncclSuccess) { nccl().GroupEnd(); return nccl_err("ncclSend", r); }
      if ((r = nccl().Recv(recv_lo, n, ncclDouble, rank - 1, comm, st)) != ncclSuccess) { nccl().GroupEnd(); return nccl_err("ncclRecv", r); }
    }
    if (send_hi && rank < nranks - 1) {
      if ((r = nccl().Send(send_hi, n, ncclDouble, rank + 1, comm, st)) != ncclSuccess) { nccl().GroupEnd(); return nccl_err("ncclSend", r); }
      if ((r = nccl().Recv(recv_hi, n, ncclDouble, rank + 1, comm, st)) != ncclSuccess) { nccl().GroupEnd(); return nccl_err("ncclRecv", r); }
    }
    if ((r = nccl().GroupEnd()) != ncclSuccess) return nccl_err("ncclGroupEnd", r);
    return "";
  }
  std::string shift_up(const double* send, double* recv, size_t n, cudaStream_t st) override {
    ncclResult_t r = nccl().GroupStart();
    if (r != ncclSuccess) return nccl_err("ncclGroupStart", r);
    if (rank < nranks - 1 && (r = nccl().Send(send, n, ncclDouble, rank + 1, comm, st)) != ncclSuccess) { nccl().GroupEnd(); return nccl_err("ncclSend", r); }
    if (rank > 0 && (r = nccl().Recv(recv, n, ncclDouble, rank - 1, comm, st)) != ncclSuccess) { nccl().GroupEnd(); return nccl_err("ncclRecv", r); }
    if ((r = nccl().GroupEnd()) != ncclSuccess) return nccl_err("ncclGroupEnd", r);
    return "";
  }
  std::string allreduce_sum(double* dev, int n, cudaStream_t st) override {
    ncclResult_t r = nccl().AllReduce(dev, dev, (size_t)n, ncclDouble, ncclSum, comm, st);
    return r == ncclSuccess ? "" : nccl_err("ncclAllReduce", r);
  }
  std::string allgather(const double* send, double* recv, size_t n, cudaStream_t st) override {
    ncclResult_t r = nccl().AllGather(send, recv, n, ncclDouble, comm, st);
    return r == ncclSuccess ? "" : nccl_err("ncclAllGather", r);
  }
};

// ------------------------------------------------------------------------------------ loopback
struct LoopHub {
  int n;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<const void*> ptr;   // per rank: 4 published pointers
  std::vector<double> val;        // per rank: reduction inputs
  std::mutex excl;                // one cooperative kernel at a time on the shared GPU
  explicit LoopHub(int n_) : n(n_), ptr(4 * n_, nullptr), val(64 * n_, 0.0) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

std::string cuda_err(const char* what, cudaError_t e) { return std::string(what) + ": " + cudaGetErrorString(e); }

struct LoopTransport : Transport {
  LoopHub* hub = nullptr;
  int rank = 0;
  bool graph_safe() const override { return false; }
  std::string sync(cudaStream_t st) {
    cudaError_t e = cudaStreamSynchronize(st);
    return e == cudaSuccess ? "" : cuda_err("cudaStreamSynchronize", e);
  }
  std::string halo(const double* send_lo, double* recv_lo, const double* send_hi, double* recv_hi, size_t n,
                   cudaStream_t st) override {
    std::string err = sync(st);
    hub->ptr[4 * rank + 0] = send_lo;
    hub->ptr[4 * rank + 1] = send_hi;
    hub->barrier();
    cudaError_t e = cudaSuccess;
    if (err.empty() && recv_lo && rank > 0 && hub->ptr[4 * (rank - 1) + 1])
      e = cudaMemcpyAsync(recv_lo, hub->ptr[4 * (rank - 1) + 1], n * sizeof(double), cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess && err.empty() && recv_hi && rank < hub->n - 1 && hub->ptr[4 * (rank + 1) + 0])
      e = cudaMemcpyAsync(recv_hi, hub->ptr[4 * (rank + 1) + 0], n * sizeof(double), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess && err.empty()) err = cuda_err("cudaMemcpyAsync", e);
    std::string e2 = sync(st);
    if (err.empty()) err = e2;
    hub->barrier();   // the sources stay untouched until every rank has copied
    return err;
  }
  std::string shift_up(const double* send, double* recv, size_t n, cudaStream_t st) override {
    std::string err = sync(st);
    hub->ptr[4 * rank + 2] = send;
    hub->barrier();
    if (err.empty() && rank > 0) {
      cudaError_t e = cudaMemcpyAsync(recv, hub->ptr[4 * (rank - 1) + 2], n * sizeof(double), cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) err = cuda_err("cudaMemcpyAsync", e);
    }
    std::string e2 = sync(st);
    if (err.empty()) err = e2;
    hub->barrier();
    return err;
  }
  std::string allreduce_sum(double* dev, int n, cudaStream_t st) override {
    if (n > 64) return "loopback allreduce: at most 64 values";
    double h[64];
    cudaError_t e = cudaMemcpyAsync(h, dev, n * sizeof(double), cudaMemcpyDeviceToHost, st);
    std::string err = (e == cudaSuccess) ? sync(st) : cuda_err("cudaMemcpyAsync", e);
    for (int i = 0; i < n; ++i) hub->val[64 * rank + i] = h[i];
    hub->barrier();
    for (int i = 0; i < n; ++i) {   // rank order: every rank gets bitwise the same sum
      double s = 0.0;
      for (int q = 0; q < hub->n; ++q) s += hub->val[64 * q + i];
      h[i] = s;
    }
    hub->barrier();
    if (err.empty()) {
      e = cudaMemcpyAsync(dev, h, n * sizeof(double), cudaMemcpyHostToDevice, st);
      err = (e == cudaSuccess) ? sync(st) : cuda_err("cudaMemcpyAsync", e);
    }
    return err;
  }
  void exclusive_begin() override { hub->excl.lock(); }
  std::string exclusive_end(cudaStream_t st) override {
    std::string err = sync(st);
    hub->excl.unlock();
    return err;
  }
  std::string allgather(const double* send, double* recv, size_t n, cudaStream_t st) override {
    std::string err = sync(st);
    hub->ptr[4 * rank + 3] = send;
    hub->barrier();
    for (int q = 0; q < hub->n && err.empty(); ++q) {
      cudaError_t e = cudaMemcpyAsync(recv + (size_t)q * n, hub->ptr[4 * q + 3], n * sizeof(double),
                                      cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) err = cuda_err("cudaMemcpyAsync", e);
    }
    std::string e2 = sync(st);
    if (err.empty()) err = e2;
    hub->barrier();
    return err;
  }
};
}  // namespace

std::string make_transport(int rank, int nranks, const void* nccl_id, void* loopback, Transport** out) {
  *out = nullptr;
  // one rank without a transport: plain one-GPU path.  One rank WITH an nccl_id builds a
  // communicator of size 1 -- the whole z-slab machinery (allgathered coarse RHS, allreduced
  // norms, NCCL calls inside the captured graph) runs with no neighbours (tests on one GPU).
  if (nranks == 1 && !nccl_id && !loopback) return "";
  if ((nccl_id != nullptr) == (loopback != nullptr)) return "nranks > 1 needs exactly one of nccl_id / loopback";
  if (loopback) {
    LoopHub* hub = static_cast<LoopHub*>(loopback);
    if (hub->n != nranks) return "loopback hub was created for a different nranks";
    LoopTransport* t = new LoopTransport();
    t->hub = hub;
    t->rank = rank;
    *out = t;
    return "";
  }
  if (!nccl().err.empty()) return nccl().err;
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, sizeof(id));
  NcclTransport* t = new NcclTransport();
  t->rank = rank;
  t->nranks = nranks;
  ncclResult_t r = nccl().CommInitRank(&t->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    t->comm = nullptr;
    delete t;
    return nccl_err("ncclCommInitRank", r);
  }
  *out = t;
  return "";
}

std::string nccl_unique_id(void* out128) {
  if (!nccl().err.empty()) return nccl().err;
  ncclUniqueId id;
  ncclResult_t r = nccl().GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_err("ncclGetUniqueId", r);
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, sizeof(id));
  return "";
}

void* loopback_create(int nranks) { return nranks >= 1 ? new LoopHub(nranks) : nullptr; }
void loopback_destroy(void* hub) { delete static_cast<LoopHub*>(hub); }

}  // namespace pmg
