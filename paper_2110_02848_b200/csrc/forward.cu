// forward.cu -- forward score over a graph in the log semiring (the paper's
// future-work consumer of the composed graph; log semiring PAPER.md:89-91).
//
// For an ACYCLIC graph: alpha(v) = logsumexp([0 if v is a start] + {alpha(u) + w(e) : e = u -> v}),
// total = logsumexp over accept states of alpha.  Level-synchronous Kahn traversal on the GPU with
// PULL folds (no contended atomics on alpha: a lexicon root pair has thousands of in-arcs):
//   1. in-degrees (atomicAdd per arc), their exclusive scan, and a transposed CSR (source, weight
//      per in-arc) scattered per source state;
//   2. per level, one warp per frontier state v: alpha(v) = logsumexp over v's in-arcs of
//      alpha(u) + w (all u are in earlier levels, so final) -- lanes stride the in-arcs with an
//      online (max, sum) pair, then a warp reduction; then the lanes walk v's out-arcs and decrement
//      the remaining in-degree of each successor: the lane that takes it to zero appends it to
//      the next frontier.
// States never reached by the traversal => the graph has a cycle => FST_E_INVALID_GRAPH.  Float64
// throughout; the in-arc order of the transposed CSR is not fixed (scatter atomics), so results
// agree with an exact evaluation to float64 rounding.
#include <math.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

#include "fstc_handle.h"
#include "fstc_internal.cuh"
#include "scan.cuh"

namespace fstc {

fst_status alloc_buffer(size_t bytes, cudaStream_t s, BufferPtr* out);
int sm_count();

namespace {

constexpr int kFwdChunk = 32;   // in-arcs per work item: hub states (thousands of in-arcs) are split
constexpr int kFwdOut = 64;     // states with more out-arcs are released by k_fwd_release ...
constexpr int kFwdPiece = 256;  // ... in pieces of this many out-arcs, spread over the grid

struct FwdCtx {
  int32_t V;
  const int64_t* row_ptr;
  const int32_t* dst;
  const float* w;
  double* alpha;
  int32_t* rem;             // remaining in-arcs not yet released
  int32_t* done;            // finished work items of a split state
  const int64_t* in_off;    // [V+1] transposed CSR
  const int32_t* in_src;    // [E]
  const float* in_w;        // [E]
  const uint8_t* is_start;
  int2* list0;              // work items (state, chunk); the chunks of a state are contiguous
  int2* list1;
  double2* part;            // per list slot: partial (max, sum) of a split state's chunk
  unsigned long long* cnt;  // ring of 3 frontier item counts, [3] = states expanded, [4..5] release pieces
  unsigned long long cap;   // list capacity (items)
  int2* rq;                 // release pieces (state, piece) of the level
  unsigned long long rcap;
};

__device__ __forceinline__ int fwd_chunks(const FwdCtx& f, int32_t v) {
  const int64_t n = f.in_off[v + 1] - f.in_off[v];
  return n <= kFwdChunk ? 1 : (int)((n + kFwdChunk - 1) / kFwdChunk);
}

// Warp-aggregated push (all lanes call it; lanes with push == false contribute nothing): one
// atomicAdd per warp on the list counter instead of one per state.
__device__ __forceinline__ void fwd_push(const FwdCtx& f, int2* list, unsigned long long* cn, bool push, int32_t v) {
  const int lane = threadIdx.x & 31;
  const int k = push ? fwd_chunks(f, v) : 0;
  const int incl = warp_incl_scan(k);
  const int tot = __shfl_sync(0xffffffffu, incl, 31);
  if (tot == 0) return;
  unsigned long long b = 0;
  if (lane == 31) b = atomicAdd(cn, (unsigned long long)tot);
  b = __shfl_sync(0xffffffffu, b, 31) + (unsigned long long)(incl - k);
  for (int c = 0; c < k; ++c)
    if (b + c < f.cap) list[b + c] = make_int2(v, c);
}

__device__ __forceinline__ void lse_merge(double& m, double& s, double m2, double s2) {
  const double mm = fmax(m, m2);
  s = (m == -INFINITY ? 0.0 : s * exp(m - mm)) + (m2 == -INFINITY ? 0.0 : s2 * exp(m2 - mm));
  m = mm;
}

__global__ void k_fwd_indeg(int64_t E, const int32_t* __restrict__ dst, int32_t* __restrict__ indeg) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&indeg[dst[e]], 1);
}

// transposed CSR: in-arc slots of v = [in_off[v], in_off[v+1]); one thread per source state
__global__ void k_fwd_scatter(FwdCtx f, int32_t* __restrict__ cursor, int32_t* __restrict__ in_src,
                              float* __restrict__ in_w) {
  for (int32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < f.V; u += gridDim.x * blockDim.x)
    for (int64_t e = f.row_ptr[u]; e < f.row_ptr[u + 1]; ++e) {
      const int32_t v = f.dst[e];
      const int64_t p = f.in_off[v] + atomicAdd(&cursor[v], 1);
      in_src[p] = u;
      in_w[p] = f.w[e];
    }
}

// states with no in-arcs form frontier 0
__global__ void k_fwd_init(FwdCtx f) {
  for (int32_t v0 = blockIdx.x * blockDim.x; v0 < f.V; v0 += gridDim.x * blockDim.x) {  // warp-uniform trip count
    const int32_t v = v0 + threadIdx.x;
    fwd_push(f, f.list0, &f.cnt[0], v < f.V && f.rem[v] == 0, v);
  }
}

// One thread per work item (v, chunk of <= kFwdChunk in-arcs): the chunk's alpha(u) + w folded into
// an online (max, sum); the thread that completes v (its only chunk, or the last of its chunks,
// which combines the published partials) writes alpha(v) and releases v's successors -- the one
// that takes a successor's remaining in-degree to zero pushes it (warp-aggregated).
__global__ void k_fwd_level(FwdCtx f, int level) {
  const unsigned long long n = min(*((volatile unsigned long long*)&f.cnt[level % 3]), f.cap);
  const int2* cur = (level & 1) ? f.list1 : f.list0;
  int2* nxt = (level & 1) ? f.list0 : f.list1;
  unsigned long long* cn = &f.cnt[(level + 1) % 3];
  if (blockIdx.x == 0 && threadIdx.x == 0) f.cnt[(level + 2) % 3] = 0;
  unsigned long long ndone = 0;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long i0 = (unsigned long long)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {  // warp-uniform
    const unsigned long long i = i0 + threadIdx.x;
    bool fin = false;
    int32_t v = 0;
    if (i < n) {
      const int2 it = cur[i];
      v = it.x;
      const int c = it.y;
      const int k = fwd_chunks(f, v);
      double m = (c == 0 && f.is_start[v]) ? 0.0 : -INFINITY, sum = m == 0.0 ? 1.0 : 0.0;
      const int64_t j0 = f.in_off[v] + (int64_t)c * kFwdChunk, j1 = min(f.in_off[v + 1], j0 + kFwdChunk);
#pragma unroll 4
      for (int64_t j = j0; j < j1; ++j) {
        const double x = f.alpha[f.in_src[j]] + (double)f.in_w[j];
        if (x == -INFINITY) continue;
        if (x > m) {
          sum = (m == -INFINITY ? 0.0 : sum * exp(m - x)) + 1.0;
          m = x;
        } else {
          sum += exp(x - m);
        }
      }
      fin = true;
      if (k > 1) {  // split state: publish the partial; the last chunk to finish combines them all
        f.part[i] = make_double2(m, sum);
        __threadfence();
        fin = atomicAdd(&f.done[v], 1) == k - 1;
        if (fin) {
          __threadfence();
          const unsigned long long b = i - (unsigned long long)c;  // slot of chunk 0
          m = -INFINITY;
          sum = 0.0;
          for (int q = 0; q < k; ++q) {
            const double2 pq = __ldcg(&f.part[b + q]);  // L2: written by other threads of this launch
            lse_merge(m, sum, pq.x, pq.y);
          }
        }
      }
      if (fin) {
        f.alpha[v] = m == -INFINITY ? -INFINITY : (sum == 1.0 ? m : m + log(sum));
        ++ndone;
      }
    }
    // release the successors (warp-uniform trip count for the aggregated pushes); hubs go to
    // k_fwd_release in pieces
    int64_t e0 = fin ? f.row_ptr[v] : 0, deg = fin ? f.row_ptr[v + 1] - e0 : 0;
    if (deg > kFwdOut) {
      const int np = (int)((deg + kFwdPiece - 1) / kFwdPiece);
      const unsigned long long b = atomicAdd(&f.cnt[4 + (level & 1)], (unsigned long long)np);
      for (int q = 0; q < np; ++q)
        if (b + q < f.rcap) f.rq[b + q] = make_int2(v, q);
      deg = 0;
    }
    const int64_t dmax = (int64_t)__reduce_max_sync(0xffffffffu, (unsigned)deg);
    for (int64_t q = 0; q < dmax; ++q) {
      const int32_t x = q < deg ? f.dst[e0 + q] : 0;
      fwd_push(f, nxt, cn, q < deg && atomicSub(&f.rem[x], 1) == 1, x);
    }
  }
  const unsigned long long nd = warp_sum(ndone);
  if ((threadIdx.x & 31) == 0 && nd) atomicAdd(&f.cnt[3], nd);  // states expanded (cycle check)
}

// Releases the out-arcs of the level's hub states, one thread per out-arc of each piece.
__global__ void k_fwd_release(FwdCtx f, int level) {
  const unsigned long long np = min(*((volatile unsigned long long*)&f.cnt[4 + (level & 1)]), f.rcap);
  int2* nxt = (level & 1) ? f.list0 : f.list1;
  unsigned long long* cn = &f.cnt[(level + 1) % 3];
  if (blockIdx.x == 0 && threadIdx.x == 0) f.cnt[4 + ((level + 1) & 1)] = 0;  // next level's pieces
  const unsigned long long tot = np * kFwdPiece, stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long t0 = (unsigned long long)blockIdx.x * blockDim.x; t0 < tot; t0 += stride) {  // warp-uniform
    const unsigned long long t = t0 + threadIdx.x;
    bool ok = false;
    int32_t x = 0;
    if (t < tot) {
      const int2 pc = f.rq[t / kFwdPiece];
      const int64_t e = f.row_ptr[pc.x] + (int64_t)pc.y * kFwdPiece + (int64_t)(t % kFwdPiece);
      if (e < f.row_ptr[pc.x + 1]) {
        x = f.dst[e];
        ok = atomicSub(&f.rem[x], 1) == 1;
      }
    }
    fwd_push(f, nxt, cn, ok, x);
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
  // work-item lists: at most sum over states of max(1, ceil(indeg / kFwdChunk)) <= V + E / kFwdChunk
  const unsigned long long cap = (unsigned long long)V + (unsigned long long)(E / kFwdChunk) + 1;
  const size_t o_alpha = alpha_out ? 0 : take(8 * (size_t)V), o_rem = take(4 * (size_t)V),
               o_cur = take(4 * (size_t)V), o_done = take(4 * (size_t)V), o_l0 = take(8 * (size_t)cap),
               o_l1 = take(8 * (size_t)cap), o_pt = take(16 * (size_t)cap), o_cnt = take(8 * 4),
               o_part = take(sizeof(double2) * grid), o_off = take(8 * ((size_t)V + 1)),
               o_tmp = take(8 * (size_t)scan_tmp_elems(V)), o_src = take(4 * (size_t)std::max<int64_t>(E, 1)),
               o_w = take(4 * (size_t)std::max<int64_t>(E, 1));
  const unsigned long long rcap = (unsigned long long)(E / kFwdPiece) + (unsigned long long)(E / kFwdOut) + 1;
  const size_t o_rq = take(8 * (size_t)rcap);
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
  f.rem = (int32_t*)(base + o_rem);
  int64_t* in_off = (int64_t*)(base + o_off);
  f.in_off = in_off;
  f.in_src = (int32_t*)(base + o_src);
  f.in_w = (float*)(base + o_w);
  f.is_start = h->is_start;
  f.list0 = (int2*)(base + o_l0);
  f.list1 = (int2*)(base + o_l1);
  f.part = (double2*)(base + o_pt);
  f.done = (int32_t*)(base + o_done);
  f.cap = cap;
  f.rq = (int2*)(base + o_rq);
  f.rcap = rcap;
  f.cnt = (unsigned long long*)(base + o_cnt);
  int32_t* cursor = (int32_t*)(base + o_cur);
  FSTC_CUDA_TRY(cudaMemsetAsync(f.rem, 0, 4 * (size_t)V, s));
  FSTC_CUDA_TRY(cudaMemsetAsync(cursor, 0, 4 * (size_t)V, s));
  FSTC_CUDA_TRY(cudaMemsetAsync(f.done, 0, 4 * (size_t)V, s));
  FSTC_CUDA_TRY(cudaMemsetAsync(f.cnt, 0, 8 * 8, s));
  if (E > 0) {
    k_fwd_indeg<<<nblk(E, 256, grid * 4), 256, 0, s>>>(E, h->dst, f.rem);
    FSTC_LAUNCH_CHECK();
  }
  st = exclusive_scan_i32(f.rem, V, in_off, (int64_t*)(base + o_tmp), s);
  if (st) return st;
  k_fwd_scatter<<<nblk(V, 256, grid * 4), 256, 0, s>>>(f, cursor, (int32_t*)(base + o_src), (float*)(base + o_w));
  FSTC_LAUNCH_CHECK();
  k_fwd_init<<<nblk(V, 256, grid * 4), 256, 0, s>>>(f);
  FSTC_LAUNCH_CHECK();
  unsigned long long hc[4] = {0, 0, 0, 0};
  int level = 0, batch = 1;
  for (;;) {  // speculative batches of level launches between size checks (empty levels are no-ops)
    for (int k = 0; k < batch; ++k, ++level) {
      k_fwd_level<<<grid, 256, 0, s>>>(f, level);
      FSTC_LAUNCH_CHECK();
      k_fwd_release<<<grid, 256, 0, s>>>(f, level);
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
