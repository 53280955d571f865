// wave.cu -- the WAVE path of a composition whose A is topologically numbered (every A arc has
// src < dst: lexicon o emissions trellises, DAG acceptors), DESIGN.md §6c.
//
// Alg. 1 computes two sets of the pair space, R (co-accessible: stage 1, the
// backward BFS from F_A x F_B) and V (accessible within R: stage 2, the forward BFS
// from S_A x S_B, Alg. 1 l.12-31), then the arcs between states of V.  The BFS order is not part of
// the result: R and V are sets and state ids are ranks by ascending key (reading R12).  When A's rows
// are in topological order, every move except M3 (A stays, B takes an eps-input arc) goes from row a
// to a row a' > a, so the sets are computed row by row instead of level by level:
//   stage 1, rows a = V_A-1 .. 0:  R(a, b) <=> (a, b) in F_A x F_B, or an M1 / M2 move from (a, b)
//                                  lands in R (rows > a: final), or an M3 move lands in R(a, .)
//                                  (the in-row fixed point: iterated over B's eps arcs);
//   stage 2, rows a = 0 .. V_A-1:  V(a, b) <=> (a, b) in R and [(a, b) in S_A x S_B, or an M1 / M2
//                                  predecessor is in V (rows < a), or an M3 predecessor is in V(a, .)].
// A trellis of T frames is T+1 dependent row steps instead of ~1.2 T frontier-synchronous levels of
// the whole batch (configs[4]: 585 levels of ~46 us each per stage), and every row step is a
// word-parallel PULL (one lane per column b, B's items in a word-tiled ELL, the A row's arcs as
// label -> slot masks in shared memory): no atomics on the pair space, whole words stored once.
//
// One composition is processed by one thread-block CLUSTER of G CTAs (persistent; compositions are
// taken in LPT order from a counter): CTA k owns the words [wpr k / G, wpr (k+1) / G) of every row.
// Per row step each CTA pulls its words into a per-CTA slice, a cluster barrier publishes the slices,
// every CTA gathers the whole row through distributed shared memory, runs the M3 fixed point on its
// copy (identical on all CTAs: the fixed point is unique), stores its own words, and keeps the row in
// shared memory as the "hot" row for the next step (a trellis row's arcs all lead to the previous /
// next row: its tests are shared-memory loads).  Rows other than the hot row are read from global
// memory through L2 (ld.global.cg: rows written by other SMs of the cluster earlier in the kernel).
//
// k_wave_count then writes pass-1 counts for the general emit: cnt8 (the kept-move
// count of every state of C, saturated at 255 = recount) and kept[block] (exact), fully parallel.
#include <cooperative_groups.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <atomic>
#include <vector>

#include "fstc_handle.h"
#include "fstc_internal.cuh"
#include "scan.cuh"
#include "wave.h"

namespace cg = cooperative_groups;

namespace fstc {
namespace {

constexpr int kWThreads = 1024;
constexpr int kWWarps = kWThreads / 32;
constexpr int kWHeavy = 32;    // B columns with more items (in a direction) are walked by the whole CTA
constexpr int kWSlots = 64;    // A arcs per row (label -> slot masks are 64-bit)
constexpr int kWLab = 256;     // label index = label + 2 (eps = 1); 255 = ELL padding (never set)
constexpr int kCThreads = 512; // count CTAs

struct WaveDir {  // B role, one direction (view by ilabel)
  const uint32_t* ell;
  const uint32_t* woff;
  const uint8_t* wmax;
  const uint32_t* hmask;
  const int4* heavy;
  int32_t nheavy;
  const int32_t* key;    // the view's arrays (heavy columns are walked there)
  const int32_t* other;
};

struct WaveComp {
  int64_t W, K;      // first word / block of the composition's pair space
  int64_t rowbase;   // first global row (count tasks)
  int32_t VA, VB, wpr, bpr;
  const int32_t* aoff[2];   // A role: [0] out-by-olabel (key = olabel, other = dst), [1] in-by-olabel (other = src)
  const int32_t* akey[2];
  const int32_t* aother[2];
  const uint8_t* startA;
  const uint8_t* accA;
  const uint8_t* startB;
  const uint8_t* accB;
  WaveDir bd[2];     // B role: [0] out-by-ilabel (stage 1, counts), [1] in-by-ilabel (stage 2)
  const int2* eps;   // B arcs with ilabel eps, (src, dst): the M3 moves
  int32_t neps;
};

struct WaveArgs {
  const WaveComp* comps;
  const int32_t* order;  // compositions by decreasing V_A (LPT)
  int32_t ncomp;
  int32_t wprmax;
  uint32_t* R;
  uint32_t* V;
  uint8_t* cnt8;
  unsigned long long* kept;
  int32_t* next;         // composition counter of the stage kernels
  int64_t nrows;         // rows of all compositions (count tasks)
};

__device__ __forceinline__ uint32_t bit_of(const uint32_t* row, int32_t col) { return (row[col >> 5] >> (col & 31)) & 1u; }

// ------------------------------------------------------------------------------ stage kernels
template <bool kS2>
__global__ void __launch_bounds__(kWThreads, 1) k_wave(WaveArgs wa) {
  cg::cluster_group cl = cg::this_cluster();
  const int G = (int)cl.num_blocks(), crank = (int)cl.block_rank();
  extern __shared__ __align__(16) unsigned char wsm[];
  unsigned long long* lm = (unsigned long long*)wsm;  // [kWLab] slots of the A row's arcs by label index
  int32_t* srow = (int32_t*)(lm + kWLab);              // [kWSlots] row at the other end of slot s
  int32_t* misc = srow + kWSlots;                      // [0] composition, [1] [2] heavy range
  const int wprmax = wa.wprmax, rng = (wprmax + G - 1) / G;
  uint32_t* rowbuf = (uint32_t*)(misc + 16);           // [2][wprmax] current / hot row (whole row)
  uint32_t* Rrow = rowbuf + 2 * wprmax;                // [wprmax] stage 2: R of the current row
  uint32_t* pullbuf = Rrow + (kS2 ? wprmax : 0);       // [2][rng] this CTA's pulled words (read by the cluster)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t* vis = kS2 ? wa.V : wa.R;
  constexpr int dir = kS2 ? 1 : 0;
  for (;;) {
    if (crank == 0 && tid == 0) misc[0] = atomicAdd(wa.next, 1);
    cl.sync();
    const int ci = *cl.map_shared_rank(misc, 0);
    cl.sync();  // everyone has read rank 0's slot before it can be rewritten
    if (ci >= wa.ncomp) break;
    const WaveComp& C = wa.comps[wa.order[ci]];
    const int wpr = C.wpr, VB = C.VB, VA = C.VA;
    const int64_t W = C.W;
    const int w0 = (int)((int64_t)wpr * crank / G), w1 = (int)((int64_t)wpr * (crank + 1) / G);
    const WaveDir D = C.bd[dir];
    const int32_t* __restrict__ aoff = C.aoff[dir];
    const int32_t* __restrict__ akey = C.akey[dir];
    const int32_t* __restrict__ aother = C.aother[dir];
    const uint8_t* __restrict__ seedA = kS2 ? C.startA : C.accA;
    const uint8_t* __restrict__ seedB = kS2 ? C.startB : C.accB;
    if (tid == 0) {  // heavy columns inside this CTA's words
      int lo = 0, hi = D.nheavy;
      while (lo < hi) { const int m = (lo + hi) >> 1; if (__ldg(&D.heavy[m]).x < w0 * 32) lo = m + 1; else hi = m; }
      misc[1] = lo;
      hi = D.nheavy;
      while (lo < hi) { const int m = (lo + hi) >> 1; if (__ldg(&D.heavy[m]).x < w1 * 32) lo = m + 1; else hi = m; }
      misc[2] = lo;
    }
    __syncthreads();
    const int h0 = misc[1], h1 = misc[2];
    int hot = -1, hp = 0;
    for (int step = 0; step < VA; ++step) {
      const int r = kS2 ? step : VA - 1 - step;
      const int cp = hp ^ 1;
      uint32_t* cur = rowbuf + cp * wprmax;
      const uint32_t* hrow = rowbuf + hp * wprmax;
      uint32_t* pb = pullbuf + cp * rng;
      const int64_t rowW = W + (int64_t)r * wpr;
      const int32_t e0 = __ldg(&aoff[r]), d = __ldg(&aoff[r + 1]) - e0;
      for (int i = tid; i < kWLab; i += kWThreads) lm[i] = 0ull;
      if (kS2)
        for (int i = tid; i < wpr; i += kWThreads) Rrow[i] = __ldcg(&wa.R[rowW + i]);
      __syncthreads();
      if (tid < d) {
        const int li = __ldg(&akey[e0 + tid]) + 2;
        srow[tid] = __ldg(&aother[e0 + tid]);
        if (li <= 254) atomicOr(&lm[li], 1ull << tid);
      }
      __syncthreads();
      const unsigned long long meps = lm[1];  // A arcs with olabel eps: M2 (B stays) and M1 eps:eps
      const bool rowseed = __ldg(&seedA[r]) != 0;
      auto test = [&](int32_t row, int32_t col) -> bool {
        if (row == hot) return bit_of(hrow, col);
        return (__ldcg(&vis[W + (int64_t)row * wpr + (col >> 5)]) >> (col & 31)) & 1u;
      };
      // ---- pull: one warp per word, one lane per column (light columns: items from the ELL)
      for (int w = w0 + warp; w < w1; w += kWWarps) {
        const int32_t col = w * 32 + lane;
        bool in = false;
        if (col < VB) {
          const bool allowed = kS2 ? ((Rrow[w] >> lane) & 1u) != 0u : true;
          if (allowed) {
            in = rowseed && __ldg(&seedB[col]) != 0;
            if (!in && d > 0) {
              for (unsigned long long m = meps; m && !in; m &= m - 1ull) in = test(srow[__ffsll((long long)m) - 1], col);
              const int jn = __ldg(&D.wmax[w]);
              const uint32_t* __restrict__ pe = D.ell + (size_t)__ldg(&D.woff[w]) * 32 + lane;
              for (int j = 0; j < jn && !in; ++j) {
                const uint32_t it = __ldg(pe + j * 32);
                const int32_t o = (int32_t)(it & 0xFFFFFFu);
                for (unsigned long long m = lm[it >> 24]; m && !in; m &= m - 1ull)
                  in = test(srow[__ffsll((long long)m) - 1], o);
              }
            }
          }
        }
        const uint32_t word = __ballot_sync(0xffffffffu, in);
        if (lane == 0) pb[w - w0] = word;
      }
      // ---- heavy columns of this CTA: the whole CTA walks the column's items
      if (h1 > h0 && d > 0) {
        __syncthreads();
        for (int h = h0; h < h1; ++h) {
          const int4 hv = __ldg(&D.heavy[h]);
          const int32_t col = hv.x;
          const bool seeded = rowseed && __ldg(&seedB[col]) != 0;
          const bool allowed = kS2 ? bit_of(Rrow, col) != 0u : true;
          if (seeded || !allowed) continue;  // uniform over the CTA
          bool found = false;
          if (tid < kWSlots && ((meps >> tid) & 1ull)) found = test(srow[tid], col);
          for (int e = (meps ? hv.y : hv.z) + tid; e < hv.w && !found; e += kWThreads) {
            const int li = __ldg(&D.key[e]) + 2;
            if (li > 254) continue;
            unsigned long long m = lm[li];
            if (!m) continue;
            const int32_t o = __ldg(&D.other[e]);
            for (; m && !found; m &= m - 1ull) found = test(srow[__ffsll((long long)m) - 1], o);
          }
          if (__syncthreads_or(found) && tid == 0) pb[(col >> 5) - w0] |= 1u << (col & 31);
        }
      }
      // ---- publish the slices, gather the whole row
      cl.sync();
      for (int k = 0; k < G; ++k) {
        const int kw0 = (int)((int64_t)wpr * k / G), kw1 = (int)((int64_t)wpr * (k + 1) / G);
        const uint32_t* src = k == crank ? pb : cl.map_shared_rank(pb, k);
        for (int i = tid; i < kw1 - kw0; i += kWThreads) cur[kw0 + i] = src[i];
      }
      __syncthreads();
      // ---- M3 fixed point of the row (B's eps-input arcs; A stays)
      if (C.neps > 0) {
        for (;;) {
          int changed = 0;
          for (int i = tid; i < C.neps; i += kWThreads) {
            const int2 a = __ldg(&C.eps[i]);  // B arc a.x -> a.y with ilabel eps
            if (kS2) {  // (r, a.x) in V  =>  (r, a.y) in V  if in R
              if (bit_of(cur, a.x) && !bit_of(cur, a.y) && bit_of(Rrow, a.y)) {
                atomicOr(&cur[a.y >> 5], 1u << (a.y & 31));
                changed = 1;
              }
            } else {    // (r, a.y) in R  =>  (r, a.x) in R
              if (bit_of(cur, a.y) && !bit_of(cur, a.x)) {
                atomicOr(&cur[a.x >> 5], 1u << (a.x & 31));
                changed = 1;
              }
            }
          }
          if (!__syncthreads_or(changed)) break;
        }
      }
      for (int i = w0 + tid; i < w1; i += kWThreads) vis[rowW + i] = cur[i];
      hot = r;
      hp = cp;
    }
  }
}

// ------------------------------------------------------------------------------ pass-1 counts
// Per state (a, b) of C: the number of moves into V (= into R for a state of V) -- M1 over A's
// out-arcs x B's out-items, M2 (A eps olabel, B stays), M3 (B eps ilabel, A stays) -- as cnt8
// (saturated at 255: the emit recounts those) and kept[block] (exact).  One CTA per row.
__global__ void __launch_bounds__(kCThreads) k_wave_count(WaveArgs wa) {
  __shared__ unsigned long long lm[kWLab];
  __shared__ int32_t srow[kWSlots];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarp = kCThreads / 32;
  const uint32_t* __restrict__ Vg = wa.V;
  for (int64_t t = blockIdx.x; t < wa.nrows; t += gridDim.x) {
    int lo = 0, hi = wa.ncomp - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (wa.comps[mid].rowbase <= t) lo = mid; else hi = mid - 1;
    }
    const WaveComp& C = wa.comps[lo];
    const int32_t r = (int32_t)(t - C.rowbase);
    const int wpr = C.wpr, bpr = C.bpr, VB = C.VB;
    const int64_t W = C.W, rowW = W + (int64_t)r * wpr;
    const WaveDir D = C.bd[0];
    const int32_t e0 = __ldg(&C.aoff[0][r]), d = __ldg(&C.aoff[0][r + 1]) - e0;
    __syncthreads();  // previous task's readers of lm / srow
    for (int i = tid; i < kWLab; i += kCThreads) lm[i] = 0ull;
    __syncthreads();
    if (tid < d) {
      const int li = __ldg(&C.akey[0][e0 + tid]) + 2;
      srow[tid] = __ldg(&C.aother[0][e0 + tid]);
      if (li <= 254) atomicOr(&lm[li], 1ull << tid);
    }
    __syncthreads();
    const unsigned long long meps = lm[1];
    auto inV = [&](int32_t row, int32_t col) -> int {
      return (int)((__ldg(&Vg[W + (int64_t)row * wpr + (col >> 5)]) >> (col & 31)) & 1u);
    };
    for (int blk = warp; blk < bpr; blk += nwarp) {
      const int wb = blk * 32, nw = min(32, wpr - wb);
      const uint32_t myw = lane < nw ? __ldg(&Vg[rowW + wb + lane]) : 0u;
      const uint32_t myh = lane < nw ? __ldg(&D.hmask[wb + lane]) : 0u;
      unsigned long long tot = 0;
      for (int i = 0; i < nw; ++i) {
        const uint32_t vw = __shfl_sync(0xffffffffu, myw, i) & ~__shfl_sync(0xffffffffu, myh, i);
        if (!vw) continue;
        const int w = wb + i;
        const int32_t col = w * 32 + lane;
        if ((vw >> lane) & 1u) {
          int cnt = 0;
          for (unsigned long long m = meps; m; m &= m - 1ull) cnt += inV(srow[__ffsll((long long)m) - 1], col);
          const int jn = __ldg(&D.wmax[w]);
          const uint32_t* __restrict__ pe = D.ell + (size_t)__ldg(&D.woff[w]) * 32 + lane;
          for (int j = 0; j < jn; ++j) {
            const uint32_t it = __ldg(pe + j * 32);
            const uint32_t li = it >> 24;
            const int32_t o = (int32_t)(it & 0xFFFFFFu);
            for (unsigned long long m = lm[li]; m; m &= m - 1ull) cnt += inV(srow[__ffsll((long long)m) - 1], o);
            if (li == 1u) cnt += inV(r, o);  // M3
          }
          wa.cnt8[(rowW + w) * 32 + lane] = (uint8_t)min(cnt, 255);
          tot += (unsigned long long)cnt;
        }
      }
      tot = warp_sum(tot);
      if (lane == 0) wa.kept[C.K + (int64_t)r * bpr + blk] = tot;
    }
    if (D.nheavy > 0) {
      __syncthreads();  // kept[] stores of the warps before the heavy credits
      for (int h = 0; h < D.nheavy; ++h) {
        const int4 hv = __ldg(&D.heavy[h]);
        const int32_t col = hv.x;
        if (col >= VB || !inV(r, col)) continue;  // uniform
        unsigned long long cnt = 0;
        if (tid < kWSlots && ((meps >> tid) & 1ull)) cnt += inV(srow[tid], col);
        for (int e = hv.y + tid; e < hv.w; e += kCThreads) {
          const int li = __ldg(&D.key[e]) + 2;
          if (li > 254) continue;
          const int32_t o = __ldg(&D.other[e]);
          for (unsigned long long m = lm[li]; m; m &= m - 1ull) cnt += inV(srow[__ffsll((long long)m) - 1], o);
          if (li == 1) cnt += inV(r, o);
        }
        cnt = warp_sum(cnt);
        __shared__ unsigned long long hsum;
        if (tid == 0) hsum = 0ull;
        __syncthreads();
        if (lane == 0 && cnt) atomicAdd(&hsum, cnt);
        __syncthreads();
        if (tid == 0) {
          wa.cnt8[(rowW + (col >> 5)) * 32 + (col & 31)] = (uint8_t)min(hsum, 255ull);
          atomicAdd(&wa.kept[C.K + (int64_t)r * bpr + (col >> 10)], hsum);
        }
        __syncthreads();
      }
    }
  }
}

__global__ void k_topo_check(int32_t V, const int32_t* __restrict__ off, const int32_t* __restrict__ other,
                             int32_t* bad) {
  const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  for (int32_t e = off[v]; e < off[v + 1]; ++e)
    if (other[e] <= v) {
      atomicOr(bad, 1);
      return;
    }
}

// ------------------------------------------------------------------------------ host
std::atomic<int>& wave_mode_ref() {
  static std::atomic<int> m{[] {
    const char* e = getenv("FSTC_WAVE");
    const int v = e ? atoi(e) : 1;
    return (v >= 0 && v <= 2) ? v : 1;
  }()};
  return m;
}

// Automatic mode: compositions of at most this many rows (the row steps of one composition are
// sequential; a deep A with few BFS levels is better served by the level kernels).
constexpr int32_t kWaveAutoRows = 4096;

fst_status topo_of(fst* A, cudaStream_t s, bool* out) {
  if (A->a_topo < 0) {
    const View& v = A->views[kOutByOlabel];
    BufferPtr tb;
    fst_status st = alloc_buffer(4, s, &tb);
    if (st) return st;
    FSTC_CUDA_TRY(cudaMemsetAsync(tb->ptr, 0, 4, s));
    if (A->V > 0 && A->E > 0) {
      k_topo_check<<<(A->V + 255) / 256, 256, 0, s>>>(A->V, v.off, v.other, (int32_t*)tb->ptr);
      FSTC_LAUNCH_CHECK();
    }
    int32_t bad = 0;
    FSTC_CUDA_TRY(cudaMemcpyAsync(&bad, tb->ptr, 4, cudaMemcpyDeviceToHost, s));
    FSTC_CUDA_TRY(cudaStreamSynchronize(s));
    A->a_topo = bad ? 0 : 1;
  }
  *out = A->a_topo == 1;
  return FST_OK;
}

// B role: the word-tiled ELL of both by-ilabel views (light columns), the heavy column lists and the
// eps arc list, built once per handle from host copies of the views (index construction only).
fst_status ensure_wave_ell(fst* B, cudaStream_t s) {
  if (B->wave_ell[0].ok && B->wave_ell[1].ok) return FST_OK;
  const int32_t V = B->V;
  const int wpr = (V + 31) / 32;
  for (int dir = 0; dir < 2; ++dir) {
    fst::WaveEll& T = B->wave_ell[dir];
    if (T.ok) continue;
    const View& v = B->views[dir == 0 ? kOutByIlabel : kInByIlabel];
    const int64_t E = B->E;
    std::vector<int32_t> off(V + 1), key(E), other(E);
    FSTC_CUDA_TRY(cudaMemcpyAsync(off.data(), v.off, sizeof(int32_t) * (V + 1), cudaMemcpyDeviceToHost, s));
    if (E) {
      FSTC_CUDA_TRY(cudaMemcpyAsync(key.data(), v.key, sizeof(int32_t) * E, cudaMemcpyDeviceToHost, s));
      FSTC_CUDA_TRY(cudaMemcpyAsync(other.data(), v.other, sizeof(int32_t) * E, cudaMemcpyDeviceToHost, s));
    }
    FSTC_CUDA_TRY(cudaStreamSynchronize(s));
    std::vector<uint32_t> woff(wpr + 1, 0), hmask(wpr, 0);
    std::vector<uint8_t> wmax(std::max(wpr, 1), 0);
    std::vector<int4> heavy;
    std::vector<int2> eps;
    for (int w = 0; w < wpr; ++w) {
      int m = 0;
      for (int l = 0; l < 32; ++l) {
        const int32_t b = w * 32 + l;
        if (b >= V) break;
        const int deg = off[b + 1] - off[b];
        if (deg > kWHeavy) {
          int32_t ne = off[b];
          while (ne < off[b + 1] && key[ne] < 0) ++ne;
          heavy.push_back(make_int4(b, off[b], ne, off[b + 1]));
          hmask[w] |= 1u << l;
        } else {
          m = std::max(m, deg);
        }
      }
      wmax[w] = (uint8_t)m;
      woff[w + 1] = woff[w] + (uint32_t)m;
    }
    std::vector<uint32_t> ell((size_t)woff[wpr] * 32 + 32, 0xFF000000u);
    for (int w = 0; w < wpr; ++w)
      for (int l = 0; l < 32; ++l) {
        const int32_t b = w * 32 + l;
        if (b >= V || ((hmask[w] >> l) & 1u)) continue;
        for (int32_t e = off[b]; e < off[b + 1]; ++e)
          ell[((size_t)woff[w] + (e - off[b])) * 32 + l] = ((uint32_t)(key[e] + 2) << 24) | (uint32_t)other[e];
      }
    if (dir == 0)
      for (int32_t b = 0; b < V; ++b)
        for (int32_t e = off[b]; e < off[b + 1] && key[e] < 0; ++e) eps.push_back(make_int2(b, other[e]));
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o += (bytes + 255) & ~size_t(255); return r; };
    const size_t o_ell = take(4 * ell.size()), o_woff = take(4 * woff.size()), o_wmax = take(wmax.size()),
                 o_hm = take(4 * std::max<size_t>(hmask.size(), 1)), o_h = take(16 * std::max<size_t>(heavy.size(), 1)),
                 o_e = take(8 * std::max<size_t>(eps.size(), 1));
    BufferPtr buf;
    fst_status st = alloc_buffer(o, s, &buf);
    if (st) return st;
    char* base = (char*)buf->ptr;
    T.ell = (uint32_t*)(base + o_ell);
    T.woff = (uint32_t*)(base + o_woff);
    T.wmax = (uint8_t*)(base + o_wmax);
    T.hmask = (uint32_t*)(base + o_hm);
    T.heavy = (int4*)(base + o_h);
    T.eps = (int2*)(base + o_e);
    T.nheavy = (int32_t)heavy.size();
    T.neps = (int32_t)eps.size();
    FSTC_CUDA_TRY(cudaMemcpyAsync(T.ell, ell.data(), 4 * ell.size(), cudaMemcpyHostToDevice, s));
    FSTC_CUDA_TRY(cudaMemcpyAsync(T.woff, woff.data(), 4 * woff.size(), cudaMemcpyHostToDevice, s));
    FSTC_CUDA_TRY(cudaMemcpyAsync(T.wmax, wmax.data(), wmax.size(), cudaMemcpyHostToDevice, s));
    if (!hmask.empty()) FSTC_CUDA_TRY(cudaMemcpyAsync(T.hmask, hmask.data(), 4 * hmask.size(), cudaMemcpyHostToDevice, s));
    if (!heavy.empty()) FSTC_CUDA_TRY(cudaMemcpyAsync(T.heavy, heavy.data(), 16 * heavy.size(), cudaMemcpyHostToDevice, s));
    if (!eps.empty()) FSTC_CUDA_TRY(cudaMemcpyAsync(T.eps, eps.data(), 8 * eps.size(), cudaMemcpyHostToDevice, s));
    FSTC_CUDA_TRY(cudaStreamSynchronize(s));
    T.buf = buf;
    T.ok = true;
  }
  return FST_OK;
}

size_t wave_smem(int wprmax, int G, bool s2) {
  const int rng = (wprmax + G - 1) / G;
  return 8 * kWLab + 4 * kWSlots + 4 * 16 + 4 * (size_t)(2 * wprmax + (s2 ? wprmax : 0) + 2 * rng);
}

template <bool kS2>
fst_status launch_wave(const WaveArgs& wa, int G, int nclusters, size_t smem, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(G * nclusters));
  cfg.blockDim = dim3(kWThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  FSTC_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_wave<kS2>, wa));
  count_launch();
  return FST_OK;
}

template <bool kS2>
int max_clusters(int G, size_t smem) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(G * 148));
  cfg.blockDim = dim3(kWThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k_wave<kS2>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

}  // namespace

void wave_mode_set(int mode) { wave_mode_ref().store((mode >= 0 && mode <= 2) ? mode : 1); }

struct WavePlan::Impl {
  BufferPtr buf;
  WaveArgs wa{};
  int G1 = 1, G2 = 1, nc1 = 0, nc2 = 0;
  size_t smem1 = 0, smem2 = 0;
};

WavePlan::WavePlan() : impl(new Impl) {}
WavePlan::~WavePlan() { delete impl; }

fst_status wave_plan(int32_t n, const fst_handle* a, const fst_handle* b, const int64_t* W, const int64_t* K,
                     cudaStream_t s, WavePlan* plan) {
  plan->ok = false;
  const int mode = wave_mode_ref().load();
  if (mode == 0 || n <= 0) return FST_OK;
  int32_t maxrows = 0, wprmax = 0;
  for (int i = 0; i < n; ++i) {
    fst* A = a[i];
    fst* B = b[i];
    if (A->views[kOutByOlabel].max_deg > kWSlots || A->views[kInByOlabel].max_deg > kWSlots) return FST_OK;
    if (B->max_ilabel > 252 || B->V >= (1 << 24)) return FST_OK;
    maxrows = std::max(maxrows, A->V);
    wprmax = std::max(wprmax, (B->V + 31) / 32);
  }
  if (mode == 1 && maxrows > kWaveAutoRows) return FST_OK;
  for (int i = 0; i < n; ++i) {
    bool topo = false;
    fst_status st = topo_of(a[i], s, &topo);
    if (st) return st;
    if (!topo) return FST_OK;
  }
  for (int i = 0; i < n; ++i) {
    fst_status st = ensure_wave_ell(b[i], s);
    if (st) return st;
  }
  // cluster size: the largest G in {8, 4, 2, 1} that keeps every composition on its own cluster
  // (all run concurrently) with >= 64 words per CTA; else G = 1
  static bool attr_done = false;
  size_t smem_max = wave_smem(wprmax, 1, true);
  if (smem_max > (size_t)227 * 1024) return FST_OK;  // rows too wide for the staged row copies
  if (!attr_done) {
    FSTC_CUDA_TRY(cudaFuncSetAttribute(k_wave<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    FSTC_CUDA_TRY(cudaFuncSetAttribute(k_wave<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr_done = true;
  }
  WavePlan::Impl& P = *plan->impl;
  P.G1 = P.G2 = 1;
  for (int G : {8, 4, 2}) {
    if (wprmax < 64 * G) continue;
    const int c = max_clusters<true>(G, wave_smem(wprmax, G, true));
    if (c >= n) {
      P.G1 = P.G2 = G;
      break;
    }
  }
  P.smem1 = wave_smem(wprmax, P.G1, false);
  P.smem2 = wave_smem(wprmax, P.G2, true);
  P.nc1 = max_clusters<false>(P.G1, P.smem1);
  P.nc2 = max_clusters<true>(P.G2, P.smem2);
  if (P.nc1 <= 0 || P.nc2 <= 0) return FST_OK;
  P.nc1 = std::min(P.nc1, n);
  P.nc2 = std::min(P.nc2, n);
  // per-composition descriptors
  std::vector<WaveComp> comps(n);
  std::vector<int32_t> order(n);
  int64_t rows = 0;
  for (int i = 0; i < n; ++i) {
    fst* A = a[i];
    fst* B = b[i];
    WaveComp& C = comps[i];
    memset(&C, 0, sizeof(C));
    C.W = W[i];
    C.K = K[i];
    C.rowbase = rows;
    rows += A->V;
    C.VA = A->V;
    C.VB = B->V;
    C.wpr = (B->V + 31) / 32;
    C.bpr = (C.wpr + kWordsPerBlock - 1) / kWordsPerBlock;
    for (int d = 0; d < 2; ++d) {
      const View& av = A->views[d == 0 ? kOutByOlabel : kInByOlabel];
      C.aoff[d] = av.off;
      C.akey[d] = av.key;
      C.aother[d] = av.other;
      const View& bv = B->views[d == 0 ? kOutByIlabel : kInByIlabel];
      const fst::WaveEll& T = B->wave_ell[d];
      C.bd[d] = WaveDir{T.ell, T.woff, T.wmax, T.hmask, T.heavy, T.nheavy, bv.key, bv.other};
    }
    C.startA = A->is_start;
    C.accA = A->is_accept;
    C.startB = B->is_start;
    C.accB = B->is_accept;
    C.eps = B->wave_ell[0].eps;
    C.neps = B->wave_ell[0].neps;
    order[i] = i;
  }
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return comps[x].VA > comps[y].VA; });
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o += (bytes + 255) & ~size_t(255); return r; };
  const size_t o_c = take(sizeof(WaveComp) * n), o_o = take(4 * n), o_n = take(8);
  fst_status st = alloc_buffer(o, s, &P.buf);
  if (st) return st;
  char* base = (char*)P.buf->ptr;
  FSTC_CUDA_TRY(cudaMemcpyAsync(base + o_c, comps.data(), sizeof(WaveComp) * n, cudaMemcpyHostToDevice, s));
  FSTC_CUDA_TRY(cudaMemcpyAsync(base + o_o, order.data(), 4 * n, cudaMemcpyHostToDevice, s));
  FSTC_CUDA_TRY(cudaStreamSynchronize(s));  // host vectors go out of scope
  P.wa.comps = (const WaveComp*)(base + o_c);
  P.wa.order = (const int32_t*)(base + o_o);
  P.wa.ncomp = n;
  P.wa.wprmax = wprmax;
  P.wa.next = (int32_t*)(base + o_n);
  P.wa.nrows = rows;
  plan->ok = true;
  plan->depth = maxrows;
  plan->cluster = P.G2;
  return FST_OK;
}

fst_status wave_stage(const WavePlan& plan, int stage, uint32_t* R, uint32_t* V, cudaStream_t s) {
  WavePlan::Impl& P = *plan.impl;
  P.wa.R = R;
  P.wa.V = V;
  FSTC_CUDA_TRY(cudaMemsetAsync(P.wa.next, 0, 4, s));
  return stage == 1 ? launch_wave<false>(P.wa, P.G1, P.nc1, P.smem1, s) : launch_wave<true>(P.wa, P.G2, P.nc2, P.smem2, s);
}

fst_status wave_count(const WavePlan& plan, uint32_t* V, uint8_t* cnt8, unsigned long long* kept, cudaStream_t s) {
  WavePlan::Impl& P = *plan.impl;
  P.wa.V = V;
  P.wa.cnt8 = cnt8;
  P.wa.kept = kept;
  const int64_t grid = std::min<int64_t>(std::max<int64_t>(P.wa.nrows, 1), (int64_t)sm_count() * 4);
  k_wave_count<<<(unsigned)grid, kCThreads, 0, s>>>(P.wa);
  FSTC_LAUNCH_CHECK();
  return FST_OK;
}

}  // namespace fstc
