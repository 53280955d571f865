// scan.cu -- device-wide exclusive scan (reduce -> scan tile sums -> down-sweep), int64 output.
#include "fstc_internal.cuh"
#include "scan.cuh"

namespace fstc {

namespace {
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;  // 4096

template <typename T>
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const T* __restrict__ in, int64_t n,
                                                              int64_t* __restrict__ tile_sum) {
  __shared__ int64_t sh[kScanThreads / 32 + 1];
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = base + (int64_t)k * kScanThreads + threadIdx.x;  // coalesced
    if (i < n) s += (int64_t)in[i];
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < kScanThreads / 32; ++w) t += sh[w];
    tile_sum[blockIdx.x] = t;
  }
}

// single CTA: exclusive scan of m tile sums in place, total to tile_sum[m]
__global__ void __launch_bounds__(1024) k_scan_tiles(int64_t* __restrict__ tile_sum, int64_t m) {
  __shared__ int64_t sh[1024 / 32 + 1];
  int64_t carry = 0;
  for (int64_t b = 0; b < m; b += blockDim.x) {
    int64_t i = b + threadIdx.x;
    int64_t v = i < m ? tile_sum[i] : 0;
    int64_t tot;
    int64_t ex = block_excl_scan(v, sh, &tot);
    if (i < m) tile_sum[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) tile_sum[m] = carry;
}

template <typename T>
__global__ void __launch_bounds__(kScanThreads) k_scan_down(const T* __restrict__ in, int64_t n,
                                                            const int64_t* __restrict__ tile_sum,
                                                            int64_t* __restrict__ out) {
  __shared__ int64_t sh[kScanThreads / 32 + 1];
  // blocked arrangement: thread t owns items [t*16, t*16+16) of the tile
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t v[kScanItems];
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = base + k;
    v[k] = i < n ? (int64_t)in[i] : 0;
    s += v[k];
  }
  int64_t tot;
  int64_t ex = block_excl_scan(s, sh, &tot) + tile_sum[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = base + k;
    if (i < n) out[i] = ex;
    ex += v[k];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = tile_sum[gridDim.x];
}

template <typename T>
fst_status scan_impl(const T* in, int64_t n, int64_t* out, int64_t* tmp, cudaStream_t s) {
  if (n == 0) {
    FSTC_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(int64_t), s));
    return FST_OK;
  }
  int64_t m = (n + kScanTile - 1) / kScanTile;
  k_scan_reduce<T><<<(unsigned)m, kScanThreads, 0, s>>>(in, n, tmp);
  FSTC_LAUNCH_CHECK();
  k_scan_tiles<<<1, 1024, 0, s>>>(tmp, m);
  FSTC_LAUNCH_CHECK();
  k_scan_down<T><<<(unsigned)m, kScanThreads, 0, s>>>(in, n, tmp, out);
  FSTC_LAUNCH_CHECK();
  return FST_OK;
}
}  // namespace

int64_t scan_tmp_elems(int64_t n) { return (n + kScanTile - 1) / kScanTile + 1; }

fst_status exclusive_scan_i32(const int32_t* in, int64_t n, int64_t* out, int64_t* tmp, cudaStream_t s) {
  return scan_impl<int32_t>(in, n, out, tmp, s);
}
fst_status exclusive_scan_u64(const unsigned long long* in, int64_t n, int64_t* out, int64_t* tmp,
                              cudaStream_t s) {
  return scan_impl<unsigned long long>(in, n, out, tmp, s);
}

}  // namespace fstc
