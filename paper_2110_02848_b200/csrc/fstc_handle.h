// fstc_handle.h -- host-side definition of the opaque fst handle.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <vector>

#include "../../include/fstc.h"

namespace fstc {

// Stream-ordered device allocation released with cudaFreeAsync on the owning stream.
struct DeviceBuffer {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaStream_t stream = nullptr;
  ~DeviceBuffer() {
    if (ptr) cudaFreeAsync(ptr, stream);
  }
};
using BufferPtr = std::shared_ptr<DeviceBuffer>;

// Allocates `bytes` (rounded up to 256 B) on `s`'s pool; returns nullptr-holding ptr on failure.
fst_status alloc_buffer(size_t bytes, cudaStream_t s, BufferPtr* out);

enum ViewId { kOutByOlabel = 0, kInByOlabel = 1, kOutByIlabel = 2, kInByIlabel = 3 };

struct View {
  int32_t* off = nullptr;    // [V+1]
  int32_t* key = nullptr;    // [E]
  int32_t* other = nullptr;  // [E]
  int32_t* carry = nullptr;  // [E]
  float* w = nullptr;        // [E]
  int32_t* arc = nullptr;    // [E] original arc index
};

}  // namespace fstc

struct fst {
  bool composed = false;
  int32_t V = 0;
  int64_t E = 0;
  cudaStream_t stream = nullptr;
  // the CSR (device)
  int64_t* row_ptr = nullptr;
  int32_t* ilabel = nullptr;
  int32_t* olabel = nullptr;
  int32_t* dst = nullptr;
  float* weight = nullptr;
  uint8_t* is_start = nullptr;
  uint8_t* is_accept = nullptr;
  int32_t* pair_a = nullptr;
  int32_t* pair_b = nullptr;
  // label-sorted views (built by fst_create, lazily for composed handles)
  bool has_views = false;
  fstc::View views[4];
  int32_t* start_list = nullptr;
  int32_t* accept_list = nullptr;
  int32_t n_start = 0, n_accept = 0;
  fst_compose_stats stats{};
  std::vector<int64_t> level_sizes[2];  // frontier size per BFS level, stage 1 / stage 2
  std::vector<fstc::BufferPtr> buffers;  // owned (or shared with a batch) device memory
};
