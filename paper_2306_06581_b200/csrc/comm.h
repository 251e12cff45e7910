// comm.h -- collectives of the sharded solve (comm.cu): one rank's view.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

struct spk_ctx;

namespace spk {
enum class CommType { Bytes, F64, I64 };
}

// The C ABI's opaque spk_comm: rank `rank` of `world`, bound to a context
// (its device and stream). Every collective is issued on the given stream.
struct spk_comm {
  int world = 1, rank = 0;
  spk_ctx* ctx = nullptr;
  virtual ~spk_comm() = default;
  // In place: buf holds `world` blocks of chunk_bytes; this rank's block is filled.
  virtual void all_gather(void* buf, size_t chunk_bytes, cudaStream_t s) = 0;
  // send: blocks for ranks 0..W-1 back to back (send_bytes[p] each); recv:
  // blocks from ranks 0..W-1 back to back (recv_bytes[p] each).
  virtual void all_to_all_v(const void* send, const int64_t* send_bytes, void* recv, const int64_t* recv_bytes,
                            cudaStream_t s) = 0;
  // Element-wise sum over ranks (8-byte elements, F64 or I64), in place.
  virtual void all_reduce_sum(void* buf, size_t count, spk::CommType t, cudaStream_t s) = 0;
  // Stream-ordered without host synchronisation (may be captured in a CUDA graph).
  virtual bool capturable() const = 0;
};

namespace spk {
using Comm = ::spk_comm;
}
