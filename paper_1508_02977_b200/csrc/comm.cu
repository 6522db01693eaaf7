// Exchange backends of the multi-GPU solve (comm.hpp).
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "comm.hpp"
#include "ffb_internal.cuh"

namespace ffb {

// ------------------------------------------------------------------------------ NCCL
namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// libnccl.so.2 at run time: a process that already loaded NCCL (torch) shares that copy
const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("/usr/lib/x86_64-linux-gnu/libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [&](auto& f, const char* n) { f = reinterpret_cast<std::decay_t<decltype(f)>>(dlsym(h, n)); };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.Send, "ncclSend");
    sym(api.Recv, "ncclRecv");
    sym(api.Broadcast, "ncclBroadcast");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.GetErrorString, "ncclGetErrorString");
    if (api.GetUniqueId && api.CommInitRank && api.AllReduce && api.Send && api.Recv &&
        api.Broadcast && api.GroupStart && api.GroupEnd)
      api.h = h;
  });
  if (!api.h) fail("schwarz.comm: libnccl.so.2 not found (multi-GPU needs NCCL)");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  const NcclApi& a = nccl();
  fail(std::string("schwarz.comm: ") + what + ": " +
       (a.GetErrorString ? a.GetErrorString(r) : std::to_string(static_cast<int>(r))));
}

struct NcclComm final : Comm {
  ncclComm_t comm = nullptr;
  const char* kind() const override { return "nccl"; }
  ~NcclComm() override {
    if (comm && nccl().CommDestroy) nccl().CommDestroy(comm);
  }
  void allreduce_sum(const double* send, double* recv, size_t n, cudaStream_t st) override {
    nccl_check(nccl().AllReduce(send, recv, n, ncclFloat64, ncclSum, comm, st), "ncclAllReduce");
  }
  void exchange(const Xfer* x, int nx, cudaStream_t st) override {
    const NcclApi& a = nccl();
    nccl_check(a.GroupStart(), "ncclGroupStart");
    for (int k = 0; k < nx; ++k) {
      if (x[k].n == 0) continue;
      if (x[k].send)
        nccl_check(a.Send(x[k].ptr, x[k].n, ncclFloat64, x[k].peer, comm, st), "ncclSend");
      else
        nccl_check(a.Recv(x[k].ptr, x[k].n, ncclFloat64, x[k].peer, comm, st), "ncclRecv");
    }
    nccl_check(a.GroupEnd(), "ncclGroupEnd");
  }
  void allgather_rows(double* buf, const size_t* off, const size_t* cnt,
                      cudaStream_t st) override {
    const NcclApi& a = nccl();
    nccl_check(a.GroupStart(), "ncclGroupStart");
    for (int q = 0; q < world; ++q)
      if (cnt[q])
        nccl_check(a.Broadcast(buf + off[q], buf + off[q], cnt[q], ncclFloat64, q, comm, st),
                   "ncclBroadcast");
    nccl_check(a.GroupEnd(), "ncclGroupEnd");
  }
};

}  // namespace

void nccl_unique_id(unsigned char* id128) {
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id128, &id, sizeof id);
}

std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const unsigned char* id128) {
  auto c = std::make_unique<NcclComm>();
  c->rank = rank;
  c->world = world;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  nccl_check(nccl().CommInitRank(&c->comm, world, id, rank), "ncclCommInitRank");
  return c;
}

// ------------------------------------------------------------------------ in-process hub
struct LocalHub {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<double*> post;
  std::vector<std::vector<Xfer>> xf;
  explicit LocalHub(int w) : world(w), post(w, nullptr), xf(w) {}
  // a rank that failed never arrives: the others give up after a generous timeout instead
  // of waiting forever
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g; })) {
      fail("schwarz.comm: a rank of the in-process communicator did not arrive (failed?)");
    }
  }
};

LocalHub* local_hub_create(int world) {
  if (world < 1) fail("schwarz.comm: world must be >= 1");
  return new LocalHub(world);
}
void local_hub_destroy(LocalHub* h) { delete h; }

namespace {

__global__ void k_sum_ranks(const double* __restrict__ stage, int world, size_t n,
                            double* __restrict__ out) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    double s = stage[i];
    for (int q = 1; q < world; ++q) s += stage[q * n + i];
    out[i] = s;
  }
}

struct LocalComm final : Comm {
  LocalHub* hub = nullptr;
  double* stage = nullptr;
  size_t stage_n = 0;
  const char* kind() const override { return "local"; }
  ~LocalComm() override {
    if (stage) cudaFree(stage);
  }
  void allreduce_sum(const double* send, double* recv, size_t n, cudaStream_t st) override {
    FFB_CUDA(cudaStreamSynchronize(st));
    if (stage_n < n * world) {
      if (stage) cudaFree(stage);
      FFB_CUDA(cudaMalloc(&stage, n * world * sizeof(double)));
      stage_n = n * world;
    }
    hub->post[rank] = const_cast<double*>(send);
    hub->barrier();
    // Copies go on the rank's own stream and are waited for before the second rendezvous: a
    // device-to-device cudaMemcpy does not block the host and runs on the legacy stream, which
    // the contexts' non-blocking streams are not ordered after — the peer could overwrite its
    // buffer, or this rank's next kernel read the destination, before the copy had landed (a
    // rare glitch of one CG scalar or halo: seen as a 1e-8 difference once in ~20 suite runs).
    for (int q = 0; q < world; ++q)
      FFB_CUDA(cudaMemcpyAsync(stage + q * n, hub->post[q], n * sizeof(double), cudaMemcpyDefault, st));
    FFB_CUDA(cudaStreamSynchronize(st));
    hub->barrier();  // every rank holds every buffer: now they may be overwritten
    k_sum_ranks<<<64, 256, 0, st>>>(stage, world, n, recv);
    FFB_LAUNCHED();
    FFB_CUDA(cudaStreamSynchronize(st));
  }
  void exchange(const Xfer* x, int nx, cudaStream_t st) override {
    FFB_CUDA(cudaStreamSynchronize(st));
    hub->xf[rank].assign(x, x + nx);
    hub->barrier();
    for (int k = 0; k < nx; ++k) {
      if (x[k].send || x[k].n == 0) continue;
      bool found = false;
      for (const Xfer& t : hub->xf[x[k].peer])
        if (t.send && t.peer == rank && t.n == x[k].n) {
          FFB_CUDA(cudaMemcpyAsync(x[k].ptr, t.ptr, t.n * sizeof(double), cudaMemcpyDefault, st));
          found = true;
          break;
        }
      if (!found) fail("schwarz.comm: unmatched halo receive");
    }
    FFB_CUDA(cudaStreamSynchronize(st));  // received before the senders may reuse their buffers
    hub->barrier();
  }
  void allgather_rows(double* buf, const size_t* off, const size_t* cnt,
                      cudaStream_t st) override {
    FFB_CUDA(cudaStreamSynchronize(st));
    hub->post[rank] = buf;
    hub->barrier();
    for (int q = 0; q < world; ++q)
      if (q != rank && cnt[q])
        FFB_CUDA(cudaMemcpyAsync(buf + off[q], hub->post[q] + off[q], cnt[q] * sizeof(double),
                                 cudaMemcpyDefault, st));
    FFB_CUDA(cudaStreamSynchronize(st));
    hub->barrier();
  }
};

}  // namespace

std::unique_ptr<Comm> make_local_comm(LocalHub* hub, int rank) {
  if (!hub || rank < 0 || rank >= hub->world) fail("schwarz.comm: bad local hub rank");
  auto c = std::make_unique<LocalComm>();
  c->hub = hub;
  c->rank = rank;
  c->world = hub->world;
  return c;
}

}  // namespace ffb
