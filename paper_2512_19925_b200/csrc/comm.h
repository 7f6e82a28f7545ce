// Collectives of the multi-GPU driver behind one interface.
//
// The driver needs five exchanges per step: the census-closure snapshot
// all-reduce at every window-update barrier, the step-end all-reduce of the
// tally slab and counters, the replay-decision max, the all-gather of the rank
// census weights that plans the global comb, and the grouped point-to-point
// rebalance of the combed particles.  Two backends implement them:
//
//   NcclComm      one process per GPU, NCCL over NVLink/NVSwitch (production);
//   LoopbackComm  W ranks as W host threads of ONE process on one device,
//                 sharing one CUDA stream, exchanging through host staging
//                 buffers with a host barrier per collective.  It exists so the
//                 real driver_step shard / snapshot / all-reduce / rebalance
//                 code runs (and is tested) on a single GPU.  The ranks share
//                 the stream so their persistent transport grids never co-reside
//                 (a partially resident persistent grid must not wait for its
//                 own non-resident blocks behind another rank's grid).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "hwwg.h"

namespace hwwg {

enum class DType { kF64, kU64, kU32 };
enum class RedOp { kSum, kMax };

inline size_t dtype_bytes(DType t) { return t == DType::kU32 ? 4 : 8; }

class Comm {
 public:
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int world() const = 0;
  // recv may alias send (in place)
  virtual void all_reduce(const void* send, void* recv, size_t count, DType t, RedOp op,
                          cudaStream_t s) = 0;
  // recv holds world * count elements, rank-major
  virtual void all_gather(const void* send, void* recv, size_t count, DType t,
                          cudaStream_t s) = 0;
  // point-to-point inside a group; matched per (sender, receiver) pair in call order
  virtual void group_start() = 0;
  virtual void send(const void* buf, size_t count, DType t, int peer, cudaStream_t s) = 0;
  virtual void recv(void* buf, size_t count, DType t, int peer, cudaStream_t s) = 0;
  virtual void group_end(cudaStream_t s) = 0;
  // the stream the driver must use (loopback: the hub's shared stream), or nullptr
  virtual cudaStream_t shared_stream() const { return nullptr; }
};

Comm* make_nccl_comm(const uint8_t id[128], int rank, int world);
Comm* make_loopback_comm(hwwg_loopback* hub, int rank);
int loopback_world(const hwwg_loopback* hub);

}  // namespace hwwg
