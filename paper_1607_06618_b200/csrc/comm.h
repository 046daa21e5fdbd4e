// comm.h — step (c) transport: NCCL over NVLink/NVSwitch (one process per
// GPU), or an in-process loopback group (P virtual ranks sharing one GPU; a
// test seam for the shard/partition logic, never a CPU fallback).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include <string>

namespace gerbil {

class Comm {
 public:
  virtual ~Comm() {}
  int rank = 0, world = 1;
  std::string err;
  // d_recv receives world * bytes (rank-major). Blocking w.r.t. the host.
  virtual bool allgather(const void* d_send, void* d_recv, size_t bytes, cudaStream_t s) = 0;
  // Byte-granular all-to-allv; offsets/sizes indexed by peer. Blocking.
  virtual bool alltoallv(const void* d_send, const size_t* send_off, const size_t* send_bytes,
                         void* d_recv, const size_t* recv_off, const size_t* recv_bytes,
                         cudaStream_t s) = 0;
  // Several all-to-allv exchanges issued as ONE grouped send/recv (NCCL group): buffer b of
  // every peer p is sent from send[b] + send_off[b][p] (send_bytes[b][p] bytes) and received
  // at recv[b] + recv_off[b][p]. Blocking; NCCL errors and a stalled peer (timeout) fail it.
  struct Xfer {
    const void* send;
    const size_t *send_off, *send_bytes;
    void* recv;
    const size_t *recv_off, *recv_bytes;
  };
  virtual bool alltoallv_multi(const Xfer* x, int n, cudaStream_t s) = 0;
};

// backend 0 = NCCL (dlopen'ed libnccl.so.2), 1 = loopback. id: 128 bytes.
Comm* make_comm(int backend, const void* id, int rank, int world, std::string& err);
bool nccl_get_unique_id(void* out128, std::string& err);

}  // namespace gerbil
