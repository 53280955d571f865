// forward.cu -- forward score over a graph in the log semiring (the paper's
// future-work consumer of the composed graph; log semiring PAPER.md:89-91).
//
// For an ACYCLIC graph: alpha(v) = logsumexp([0 if v is a start] + {alpha(u) + w(e) : e = u -> v}),
// total = logsumexp over accept states of alpha.  Level-synchronous Kahn traversal on the GPU:
// k_fwd_indeg counts in-arcs; a level kernel expands every state of the current frontier (one
// thread per state, its out-arcs in order), folds alpha(u) + w into alpha(v) with a float64
// compare-and-swap log-add, and decrements v's remaining in-degree -- the thread that takes it to
// zero appends v to the next frontier (its alpha is then final: every in-arc has been folded).
// States never expanded => the graph has a cycle => FST_E_INVALID_GRAPH.  alpha and the total are
// float64; the fold order of a state's in-arcs is not fixed (atomics), so results agree with an
// exact evaluation to float64 rounding.
#include <math.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

#include "fstc_handle.h"
#include "fstc_internal.cuh"

namespace fstc {

fst_status alloc_buffer(size_t bytes, cudaStream_t s, BufferPtr* out);
int sm_count();

namespace {

__device__ __forceinline__ double log_add(double a, double b) {
  if (a == -INFINITY) return b;
  if (b == -INFINITY) return a;
  const double m = fmax(a, b);
  return m + log1p(exp(-fabs(a - b)));
}

__device__ __forceinline__ void atomic_log_add(double* p, double x) {
  unsigned long long* q = (unsigned long long*)p;
  unsigned long long old = *q, assumed;
  do {
    assumed = old;
    const double cur = __longlong_as_double((long long)assumed);
    const double nv = log_add(cur, x);
    if (__double_as_longlong(nv) == (long long)assumed) return;
    old = atomicCAS(q, assumed, (unsigned long long)__double_as_longlong(nv));
  } while (assumed != old);
}

struct FwdCtx {
  int32_t V;
  const int64_t* row_ptr;
  const int32_t* dst;
  const float* w;
  double* alpha;
  int32_t* indeg;
  int32_t* list0;
  int32_t* list1;
  unsigned long long* cnt;  // ring of 3 frontier sizes + [3] = states expanded
};

__global__ void k_fwd_indeg(int64_t E, const int32_t* __restrict__ dst, int32_t* __restrict__ indeg) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&indeg[dst[e]], 1);
}

// alpha = 0 at start states, -inf elsewhere; states with no in-arcs form frontier 0
__global__ void k_fwd_init(FwdCtx f, const uint8_t* __restrict__ is_start) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < f.V; v += gridDim.x * blockDim.x) {
    f.alpha[v] = is_start[v] ? 0.0 : -INFINITY;
    if (f.indeg[v] == 0) f.list0[atomicAdd(&f.cnt[0], 1ull)] = v;
  }
}

__global__ void k_fwd_level(FwdCtx f, int level) {
  const unsigned long long n = *((volatile unsigned long long*)&f.cnt[level % 3]);
  const int32_t* cur = (level & 1) ? f.list1 : f.list0;
  int32_t* nxt = (level & 1) ? f.list0 : f.list1;
  unsigned long long* cn = &f.cnt[(level + 1) % 3];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    f.cnt[(level + 2) % 3] = 0;
    if (n) f.cnt[3] += n;
  }
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const int32_t u = cur[i];
    const double au = f.alpha[u];
    for (int64_t e = f.row_ptr[u]; e < f.row_ptr[u + 1]; ++e) {
      const int32_t v = f.dst[e];
      if (au != -INFINITY) atomic_log_add(&f.alpha[v], au + (double)f.w[e]);
      __threadfence();  // the fold is visible before v can be released to the next frontier
      if (atomicSub(&f.indeg[v], 1) == 1) nxt[atomicAdd(cn, 1ull)] = v;
    }
  }
}

// per-block (max, sum exp(x - max)) over the accept states, combined on the host in float64
__global__ void k_fwd_total(int32_t V, const uint8_t* __restrict__ is_accept, const double* __restrict__ alpha,
                            double2* __restrict__ part) {
  __shared__ double sm[32], ss[32];
  double m = -INFINITY, sum = 0.0;
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
    if (!is_accept[v]) continue;
    const double a = alpha[v];
    if (a == -INFINITY) continue;
    if (a > m) {
      sum = sum * exp(m - a) + 1.0;
      m = a;
    } else {
      sum += exp(a - m);
    }
  }
  for (int d = 16; d > 0; d >>= 1) {
    const double m2 = __shfl_xor_sync(0xffffffffu, m, d), s2 = __shfl_xor_sync(0xffffffffu, sum, d);
    const double mm = fmax(m, m2);
    sum = (m == -INFINITY ? 0.0 : sum * exp(m - mm)) + (m2 == -INFINITY ? 0.0 : s2 * exp(m2 - mm));
    m = mm;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    sm[warp] = m;
    ss[warp] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double M = -INFINITY, S = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      if (sm[i] == -INFINITY) continue;
      const double mm = fmax(M, sm[i]);
      S = (M == -INFINITY ? 0.0 : S * exp(M - mm)) + ss[i] * exp(sm[i] - mm);
      M = mm;
    }
    part[blockIdx.x] = make_double2(M, S);
  }
}

inline unsigned nblk(int64_t n, int t, unsigned cap) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + t - 1) / t, cap));
}

}  // namespace

fst_status forward_score_impl(fst* h, cudaStream_t s, double* total, double* alpha_out) {
  if (!h || !total) {
    set_error(FST_E_INVALID_ARG, "fst_forward_score: NULL argument");
    return FST_E_INVALID_ARG;
  }
  const int32_t V = h->V;
  const int64_t E = h->E;
  *total = -INFINITY;
  if (V == 0) return FST_OK;
  const unsigned grid = (unsigned)(sm_count() * 8);
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
  const size_t o_alpha = alpha_out ? 0 : take(8 * (size_t)V), o_deg = take(4 * (size_t)V), o_l0 = take(4 * (size_t)V),
               o_l1 = take(4 * (size_t)V), o_cnt = take(8 * 4), o_part = take(sizeof(double2) * grid);
  BufferPtr wb;
  fst_status st = alloc_buffer(off, s, &wb);
  if (st) return st;
  char* base = (char*)wb->ptr;
  FwdCtx f;
  f.V = V;
  f.row_ptr = h->row_ptr;
  f.dst = h->dst;
  f.w = h->weight;
  f.alpha = alpha_out ? alpha_out : (double*)(base + o_alpha);
  f.indeg = (int32_t*)(base + o_deg);
  f.list0 = (int32_t*)(base + o_l0);
  f.list1 = (int32_t*)(base + o_l1);
  f.cnt = (unsigned long long*)(base + o_cnt);
  FSTC_CUDA_TRY(cudaMemsetAsync(f.indeg, 0, 4 * (size_t)V, s));
  FSTC_CUDA_TRY(cudaMemsetAsync(f.cnt, 0, 8 * 4, s));
  if (E > 0) {
    k_fwd_indeg<<<nblk(E, 256, grid * 4), 256, 0, s>>>(E, h->dst, f.indeg);
    FSTC_LAUNCH_CHECK();
  }
  k_fwd_init<<<nblk(V, 256, grid * 4), 256, 0, s>>>(f, h->is_start);
  FSTC_LAUNCH_CHECK();
  unsigned long long hc[4] = {0, 0, 0, 0};
  int level = 0, batch = 1;
  for (;;) {  // speculative batches of level launches between size checks (empty levels are no-ops)
    for (int k = 0; k < batch; ++k, ++level) {
      k_fwd_level<<<grid, 256, 0, s>>>(f, level);
      FSTC_LAUNCH_CHECK();
    }
    FSTC_CUDA_TRY(cudaMemcpyAsync(hc, f.cnt, sizeof(hc), cudaMemcpyDeviceToHost, s));
    FSTC_CUDA_TRY(cudaStreamSynchronize(s));
    if (hc[level % 3] == 0) break;
    batch = std::min(batch * 2, 16);
  }
  if ((int64_t)hc[3] != (int64_t)V) {
    set_error(FST_E_INVALID_GRAPH, "fst_forward_score: the graph has a cycle (%lld of %d states ordered)",
              (long long)hc[3], V);
    return FST_E_INVALID_GRAPH;
  }
  double2* part = (double2*)(base + o_part);
  k_fwd_total<<<grid, 256, 0, s>>>(V, h->is_accept, f.alpha, part);
  FSTC_LAUNCH_CHECK();
  std::vector<double2> hp(grid);
  FSTC_CUDA_TRY(cudaMemcpyAsync(hp.data(), part, sizeof(double2) * grid, cudaMemcpyDeviceToHost, s));
  FSTC_CUDA_TRY(cudaStreamSynchronize(s));
  double M = -INFINITY, S = 0.0;
  for (const double2& p : hp) {
    if (p.x == -INFINITY) continue;
    const double mm = std::max(M, p.x);
    S = (M == -INFINITY ? 0.0 : S * exp(M - mm)) + p.y * exp(p.x - mm);
    M = mm;
  }
  *total = M == -INFINITY ? -INFINITY : M + log(S);
  return FST_OK;
}

}  // namespace fstc
