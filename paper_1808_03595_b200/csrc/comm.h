// Rank-to-rank transports of the z-slab decomposition (comm.cpp).  Internal; not part of the C ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstring>
#include <string>

namespace pmg {

// same fields and meaning as pmg_slab (include/pmg.h)
struct SlabPlan {
  int z0, z1, zb, nplanes, own_lo, own_hi, lower, upper;
};
int slab_plan(int k3, int nranks, int rank, SlabPlan* out);

// Every call returns "" on success, else an error message.  Device pointers; work is ordered on st.
struct Transport {
  virtual ~Transport() {}
  virtual bool graph_safe() const = 0;   // may the calls be captured into a CUDA graph?
  // send send_lo (n doubles) to rank-1 and receive rank-1's send_hi into recv_lo; likewise with
  // rank+1 (send_hi -> its recv_lo); NULL pointers skip a direction
  virtual std::string halo(const double* send_lo, double* recv_lo, const double* send_hi, double* recv_hi, size_t n,
                           cudaStream_t st) = 0;
  // send `send` to rank+1 and receive rank-1's into `recv` (one-directional shift)
  virtual std::string shift_up(const double* send, double* recv, size_t n, cudaStream_t st) = 0;
  virtual std::string allreduce_sum(double* dev, int n, cudaStream_t st) = 0;
  // recv[q n + i] = send_q[i] for every rank q
  virtual std::string allgather(const double* send, double* recv, size_t n, cudaStream_t st) = 0;
  // bracket a grid-synchronising (cooperative) kernel: loopback ranks share one GPU, so their
  // cooperative launches run one at a time (a partially resident cooperative grid would spin)
  virtual void exclusive_begin() {}
  virtual std::string exclusive_end(cudaStream_t) { return ""; }
};

// nranks == 1 -> *out = nullptr (no communication)
std::string make_transport(int rank, int nranks, const void* nccl_id, void* loopback, Transport** out);
std::string nccl_unique_id(void* out128);
void* loopback_create(int nranks);
void loopback_destroy(void* hub);

}  // namespace pmg
