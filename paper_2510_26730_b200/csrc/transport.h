// transport.h — the collectives of the expert-parallel decode step
// (engine.cu ep_step_on): an all-gather of every rank's routing block and an
// all-to-all of expert outputs, both enqueued on the engine's compute stream.
//
//   NcclTransport      one process per GPU: NCCL 2.x (resolved at run time
//                      from the libnccl.so.2 already mapped by torch, else the
//                      system one) over NVLink / NVSwitch;
//   CallbackTransport  a host callback (ef_collective_cb) — the multi-process
//                      CPU-transport tests run G ranks on one GPU through it
//                      (gloo), where NCCL refuses two ranks on one device;
//   LocalTransport     G = 1: device copies.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <memory>
#include <string>

#include "../../include/expertflow.h"

namespace ef {

struct Transport {
  virtual ~Transport() = default;
  // recv[g * bytes ...] = rank g's send[0 .. bytes)
  virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) = 0;
  // recv[g * chunk ...] = rank g's send[me * chunk ...]
  virtual void alltoall(const void* send, void* recv, size_t chunk, cudaStream_t st) = 0;
  virtual const char* name() const = 0;
};

std::unique_ptr<Transport> make_local_transport();
std::unique_ptr<Transport> make_nccl_transport(int world, int rank, const void* unique_id128);
std::unique_ptr<Transport> make_callback_transport(ef_collective_cb cb, void* user);
// 128-byte NCCL unique id (rank 0 creates it, the others receive it)
void nccl_unique_id(void* out128);

}  // namespace ef
