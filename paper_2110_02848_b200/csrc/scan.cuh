// scan.cuh -- CUB-free warp / block / device exclusive scans ("row_ptr =
// exclusive_scan(c) in int64"; "The offset ... is known at this point").
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fstc.h"

namespace fstc {

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += u;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

// Block-wide exclusive scan of one value per thread.  `sh` needs blockDim/32 + 1 slots.
// Returns the exclusive prefix; *total receives the block sum (all threads).
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* sh, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) sh[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T s = lane < nw ? sh[lane] : T(0);
    T si = warp_incl_scan(s);
    if (lane < nw) sh[lane] = si - s;
    if (lane == nw - 1) sh[nw] = si;
  }
  __syncthreads();
  T res = inc - v + sh[warp];
  *total = sh[nw];
  __syncthreads();
  return res;
}

// Device-wide exclusive scan: out[i] = sum(in[0..i)), out[n] = total (int64).  `tmp` must hold
// scan_tmp_elems(n) int64.  Three launches (reduce, scan of tile sums, down-sweep).
int64_t scan_tmp_elems(int64_t n);
fst_status exclusive_scan_i32(const int32_t* in, int64_t n, int64_t* out, int64_t* tmp, cudaStream_t s);
fst_status exclusive_scan_u64(const unsigned long long* in, int64_t n, int64_t* out, int64_t* tmp,
                              cudaStream_t s);

}  // namespace fstc
