// memory.cu -- device buffers for handles and compose workspaces.
//
// Small buffers use the stream-ordered pool (cudaMallocAsync / cudaFreeAsync).  Large buffers
// (composed graphs are tens of GB at configs[3]) are recycled through a small cache: a freed large
// buffer is kept with an event recorded on its stream and handed to the next request of a similar
// size (best fit, at most 25% + 64 MiB larger), after making the requesting stream wait on that
// event.  This keeps repeated compositions from re-mapping tens of GB of physical memory per call.
#include <mutex>
#include <vector>

#include "fstc_handle.h"
#include "fstc_internal.cuh"

namespace fstc {

namespace {
constexpr size_t kCacheMin = size_t(32) << 20;
struct Cached {
  void* ptr;
  size_t bytes;
  cudaEvent_t ready;
};
std::mutex g_mu;
std::vector<Cached> g_cache;
size_t g_cached_bytes = 0;

void drop_all_locked() {
  for (auto& c : g_cache) {
    cudaEventSynchronize(c.ready);
    cudaEventDestroy(c.ready);
    cudaFree(c.ptr);
  }
  g_cache.clear();
  g_cached_bytes = 0;
}

size_t cache_limit() {
  static size_t lim = 0;
  if (!lim) {
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    lim = tot / 3;
  }
  return lim;
}
}  // namespace

void release_buffer(void* ptr, size_t bytes, cudaStream_t s) {
  if (bytes >= kCacheMin) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_cached_bytes + bytes <= cache_limit()) {
      cudaEvent_t ev;
      if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess) {
        cudaEventRecord(ev, s);
        g_cache.push_back({ptr, bytes, ev});
        g_cached_bytes += bytes;
        return;
      }
    }
  }
  cudaFreeAsync(ptr, s);
}

fst_status alloc_buffer(size_t bytes, cudaStream_t s, BufferPtr* out) {
  auto b = std::make_shared<DeviceBuffer>();
  bytes = (bytes + 255) & ~size_t(255);
  if (bytes == 0) bytes = 256;
  if (bytes >= kCacheMin) {
    std::lock_guard<std::mutex> lk(g_mu);
    int best = -1;
    for (int i = 0; i < (int)g_cache.size(); ++i) {
      const size_t cb = g_cache[i].bytes;
      if (cb >= bytes && cb <= bytes + bytes / 4 + (size_t(64) << 20) && (best < 0 || cb < g_cache[best].bytes))
        best = i;
    }
    if (best >= 0) {
      Cached c = g_cache[best];
      g_cache.erase(g_cache.begin() + best);
      g_cached_bytes -= c.bytes;
      cudaStreamWaitEvent(s, c.ready, 0);
      cudaEventDestroy(c.ready);
      b->ptr = c.ptr;
      b->bytes = c.bytes;
      b->stream = s;
      *out = std::move(b);
      return FST_OK;
    }
  }
  cudaError_t e = cudaMallocAsync(&b->ptr, bytes, s);
  if (e == cudaErrorMemoryAllocation) {  // give cached memory back and retry once
    cudaGetLastError();
    {
      std::lock_guard<std::mutex> lk(g_mu);
      drop_all_locked();
    }
    e = cudaMallocAsync(&b->ptr, bytes, s);
  }
  if (e != cudaSuccess) {
    b->ptr = nullptr;
    cudaGetLastError();
    set_error(e == cudaErrorMemoryAllocation ? FST_E_OOM : FST_E_CUDA, "cudaMallocAsync(%zu) failed: %s", bytes,
              cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? FST_E_OOM : FST_E_CUDA;
  }
  b->bytes = bytes;
  b->stream = s;
  *out = std::move(b);
  return FST_OK;
}

}  // namespace fstc
