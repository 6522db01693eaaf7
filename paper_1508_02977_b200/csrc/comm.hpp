// The exchange layer of the multi-GPU solve (one rank per GPU, row bands of subdomains;
// SURVEY.md §8e): three primitives, all enqueued on the solver's stream.
//   allreduce_sum  — the CG reduction units (every unit is non-zero on one rank only, so the
//                    sum is exact and the scalars are identical on every rank);
//   exchange       — paired sends/receives with the neighbouring ranks (halo rows);
//   allgather_rows — every rank's owned rows of a vector to every rank, in place.
// Backends: NCCL (ncclSend/ncclRecv over NVLink P2P, ncclAllReduce, grouped ncclBroadcast;
// libnccl.so.2 is opened at run time, so single-GPU use never needs it) and an in-process
// hub that lets N contexts on host threads — possibly on ONE device — run the same protocol
// for testing (host rendezvous + device copies; no kernel ever waits on another).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <memory>

namespace ffb {

struct Xfer {
  int peer;      // rank
  int send;      // 1 send, 0 receive
  double* ptr;   // device
  size_t n;      // doubles
};

struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() = default;
  virtual const char* kind() const = 0;
  // recv = sum over ranks of send (out of place: send keeps this rank's own entries)
  virtual void allreduce_sum(const double* send, double* recv, size_t n, cudaStream_t st) = 0;
  virtual void exchange(const Xfer* x, int nx, cudaStream_t st) = 0;
  // buf holds the full vector on every rank; rank q's rows are [off[q], off[q] + cnt[q])
  virtual void allgather_rows(double* buf, const size_t* off, const size_t* cnt,
                              cudaStream_t st) = 0;
};

// NCCL: id is the 128-byte ncclUniqueId made by nccl_unique_id on one rank and shared by the
// caller (torch.distributed, MPI, a file ...)
std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const unsigned char* id);
void nccl_unique_id(unsigned char* id128);

struct LocalHub;
LocalHub* local_hub_create(int world);
void local_hub_destroy(LocalHub* h);
std::unique_ptr<Comm> make_local_comm(LocalHub* hub, int rank);

}  // namespace ffb
