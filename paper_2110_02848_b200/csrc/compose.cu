// compose.cu -- eager trimmed composition on the GPU (arXiv 2110.02848 §3.3).
//
// Two frontier-synchronous BFS stages over the pair space V_A x V_B, then one numbering pass and
// one emit pass:
//   stage 1  (Alg. 1 line 3): backward BFS from the accept pairs over
//            in-arc views; R = co-accessible pairs (bitmap).  "made parallel in the same way".
//   stage 2  (Alg. 1 lines 4-31): forward BFS from the start pairs in R over
//            out-arc views; a candidate is kept iff its destination is in R; new pairs are claimed
//            by an atomic test-and-set on the visited bitmap V (the V_A x V_B state table).  The
//            per-block count of kept moves is the paper's pass-1 count ("the number of new nodes
//            ... along with the number of ... output arcs").
//   number   vcount/kept per 1024-pair block -> exclusive scans -> state ids (= rank of the pair
//            in V, i.e. ascending key) and arc offsets ("The offset ... is known").
//   emit     re-enumerate the moves of every state of C, write each arc at a scan-derived slot
//            (pass 2; deterministic slots replace the paper's atomic cursors).
//
// Work decomposition (B200-first, not the paper's thread-per-arc-pair): a CTA owns one 1024-pair
// block (row u_a, 1024 consecutive u_b).  It compacts the block's frontier bits, then walks the
// B-side arcs of those states with one thread per arc ("item"), finding the matching A arcs of
// row u_a by binary search in the label-sorted A view.  Moves M1/M2/M3 of N1.
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "fstc_handle.h"
#include "fstc_internal.cuh"
#include "scan.cuh"

namespace fstc {

fst_status ensure_views(fst* h, cudaStream_t s);
fst_status alloc_buffer(size_t bytes, cudaStream_t s, BufferPtr* out);
bool profiling_enabled();

namespace {

constexpr int kThreads = 256;
constexpr int kStatesPerThread = kPairsPerBlock / kThreads;  // 4

struct Ctx {
  // device pointers of the workspace (passed by value to every kernel)
  uint32_t* R;
  uint32_t* V;
  uint32_t* F0;
  uint32_t* F1;
  uint32_t* flag0;
  uint32_t* flag1;
  int32_t* list0;
  int32_t* list1;
  LevelCtrl* ctrl;
  unsigned long long* kept;
  int32_t* vcount;
  uint16_t* wpre;
  int64_t* idbase;
  int64_t* arcbase;
  unsigned long long* hist;  // per-level discovered states
  unsigned long long* misc;  // [0] nonempty levels, [1] |R|, [2] emit consistency errors
  const CompDev* comps;
  const int64_t* seedbase;  // [ncomp+1] prefix of seed-pair counts
  int32_t ncomp;
  int64_t nwords, nblocks;
};

struct BlockInfo {
  int comp;
  int32_t ua;
  int32_t ub0;
  int32_t nwords;
  int64_t word0;
};

__device__ __forceinline__ BlockInfo decode_block(const Ctx& cx, int64_t blk) {
  BlockInfo bi;
  bi.comp = cx.ncomp == 1 ? 0 : find_comp(cx.comps, cx.ncomp, blk);
  const CompDev& C = cx.comps[bi.comp];
  int64_t local = blk - C.K;
  bi.ua = (int32_t)(local / C.bpr);
  int32_t j = (int32_t)(local - (int64_t)bi.ua * C.bpr);
  bi.ub0 = j * kPairsPerBlock;
  bi.nwords = min(kWordsPerBlock, C.wpr - j * kWordsPerBlock);
  bi.word0 = C.W + (int64_t)bi.ua * C.wpr + (int64_t)j * kWordsPerBlock;
  return bi;
}

__device__ __forceinline__ int32_t lower_bound_key(const int32_t* __restrict__ key, int32_t lo, int32_t hi,
                                                   int32_t x) {
  while (lo < hi) {
    int32_t mid = (lo + hi) >> 1;
    if (__ldg(&key[mid]) < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Frontier mark of a newly claimed pair: F_next bit, block flag, block list append.
__device__ __forceinline__ void push_frontier(const CompDev& C, int32_t va, int32_t vb, int64_t w, uint32_t bit,
                                              uint32_t* __restrict__ Fn, uint32_t* __restrict__ flagn,
                                              int32_t* __restrict__ listn, LevelCtrl* ctrln) {
  atomicOr(&Fn[w], bit);
  int64_t blk = C.K + (int64_t)va * C.bpr + (vb >> 10);
  if (*((volatile uint32_t*)&flagn[blk]) == 0 && atomicExch(&flagn[blk], 1u) == 0) {
    unsigned long long pos = atomicAdd(&ctrln->count, 1ull);
    listn[pos] = (int32_t)blk;
  }
}

// Visit a candidate pair: stage-2 filter (R), test-then-set claim on the visited bitmap.
template <bool kFilter>
__device__ __forceinline__ void visit(const CompDev& C, int32_t va, int32_t vb, uint32_t* __restrict__ vis,
                                      const uint32_t* __restrict__ R, uint32_t* __restrict__ Fn,
                                      uint32_t* __restrict__ flagn, int32_t* __restrict__ listn, LevelCtrl* ctrln,
                                      unsigned& kept, unsigned& nnew) {
  const int64_t w = C.W + (int64_t)va * C.wpr + (vb >> 5);
  const uint32_t bit = 1u << (vb & 31);
  if (kFilter) {
    if (!(__ldg(&R[w]) & bit)) return;
    ++kept;
  }
  if (*((volatile uint32_t*)&vis[w]) & bit) return;  // test before the atomic (bits only get set)
  uint32_t old = atomicOr(&vis[w], bit);
  if (old & bit) return;
  ++nnew;
  push_frontier(C, va, vb, w, bit, Fn, flagn, listn, ctrln);
}

// Shared per-block staging of the CTA: compacted states of one 1024-pair block and their item
// offsets.  Item 0 of a state is its "M2 item" (only in the emit pass, or when A's row has eps
// outputs); the following items are the B-side arcs of the state in view order.
struct BlockSmem {
  uint32_t words[kWordsPerBlock];
  int32_t wpre[kWordsPerBlock + 1];
  int32_t state[kPairsPerBlock];      // u_b of the i-th set bit
  int32_t scan[kPairsPerBlock + 1];   // item offsets
  int32_t a0, a1, aeps;               // A row [a0,a1), eps prefix [a0,aeps)
  unsigned long long red[kThreads / 32 + 1];
  int32_t red32[kThreads / 32 + 1];
};

// Compact the set bits of s.words into s.state (ascending u_b).
__device__ __forceinline__ void compact_bits(BlockSmem& s, int32_t ub0) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = warp; i < kWordsPerBlock; i += kThreads / 32) {
    uint32_t w = s.words[i];
    if ((w >> lane) & 1u) {
      int pos = s.wpre[i] + __popc(w & ((1u << lane) - 1u));
      s.state[pos] = ub0 + i * 32 + lane;
    }
  }
}

// Load the block's words of `bits` (optionally clearing them), prefix popcounts into s.
__device__ __forceinline__ void load_words(BlockSmem& s, uint32_t* bits, const BlockInfo& bi, bool clear) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    uint32_t w = 0;
    if (lane < bi.nwords) {
      w = bits[bi.word0 + lane];
      if (clear && w) bits[bi.word0 + lane] = 0u;
    }
    s.words[lane] = w;
    int pc = __popc(w);
    int inc = warp_incl_scan(pc);
    s.wpre[lane] = inc - pc;
    if (lane == 31) s.wpre[32] = inc;
  }
}

// Item offsets of the nst compacted states: items(state) = extra + deg_B(state).  Returns total.
__device__ __forceinline__ int32_t scan_items(BlockSmem& s, int nst, const int32_t* __restrict__ Boff, int extra) {
  int32_t c[kStatesPerThread];
  int32_t sum = 0;
#pragma unroll
  for (int k = 0; k < kStatesPerThread; ++k) {
    int i = threadIdx.x * kStatesPerThread + k;
    c[k] = 0;
    if (i < nst) {
      int32_t ub = s.state[i];
      c[k] = extra + __ldg(&Boff[ub + 1]) - __ldg(&Boff[ub]);
    }
    sum += c[k];
  }
  int32_t tot;
  int32_t ex = block_excl_scan(sum, s.red32, &tot);
#pragma unroll
  for (int k = 0; k < kStatesPerThread; ++k) {
    int i = threadIdx.x * kStatesPerThread + k;
    if (i < nst) s.scan[i] = ex;
    ex += c[k];
  }
  if (threadIdx.x == 0) s.scan[nst] = tot;
  __syncthreads();
  return tot;
}

__device__ __forceinline__ int item_state(const BlockSmem& s, int nst, int32_t item) {
  // last state i with scan[i] <= item
  int lo = 0, hi = nst - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (s.scan[mid] <= item) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Enumerate the moves of one item; f(va, vb, kind, ea, eb) with kind 1 = M1, 2 = M2, 3 = M3.
// ea / eb are view positions.  Order: M2 item -> A eps prefix; B item -> M1 matches then M3.
template <typename Fn>
__device__ __forceinline__ void for_item_moves(const ViewDev& Av, const ViewDev& Bv, const BlockSmem& s,
                                               int32_t ua, int32_t ub, int32_t k, int extra, Fn&& f) {
  if (k < extra) {  // M2 item
    for (int32_t ea = s.a0; ea < s.aeps; ++ea) f(__ldg(&Av.other[ea]), ub, 2, ea, -1);
    return;
  }
  const int32_t eb = __ldg(&Bv.off[ub]) + (k - extra);
  const int32_t lab = __ldg(&Bv.key[eb]);
  const int32_t ob = __ldg(&Bv.other[eb]);
  int32_t ea = lower_bound_key(Av.key, s.a0, s.a1, lab);
  for (; ea < s.a1 && __ldg(&Av.key[ea]) == lab; ++ea) f(__ldg(&Av.other[ea]), ob, 1, ea, eb);
  if (lab == FST_EPS) f(ua, ob, 3, -1, eb);
}

__device__ __forceinline__ void load_arow(BlockSmem& s, const ViewDev& Av, int32_t ua) {
  if (threadIdx.x == 0) {
    s.a0 = __ldg(&Av.off[ua]);
    s.a1 = __ldg(&Av.off[ua + 1]);
    s.aeps = lower_bound_key(Av.key, s.a0, s.a1, 0);
  }
}

// ------------------------------------------------------------------------------ seeds
template <bool kStage2>
__global__ void k_seed(Ctx cx) {
  const int64_t total = cx.seedbase[cx.ncomp];
  uint32_t* vis = kStage2 ? cx.V : cx.R;
  unsigned kept = 0, nnew = 0;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    int c = 0;
    {
      int lo = 0, hi = cx.ncomp - 1;
      while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (cx.seedbase[mid] <= g) lo = mid; else hi = mid - 1;
      }
      c = lo;
    }
    const CompDev& C = cx.comps[c];
    int64_t i = g - cx.seedbase[c];
    int32_t nb = kStage2 ? C.nStartB : C.nAccB;
    int32_t va = kStage2 ? C.startListA[i / nb] : C.accListA[i / nb];
    int32_t vb = kStage2 ? C.startListB[i % nb] : C.accListB[i % nb];
    visit<kStage2>(C, va, vb, vis, cx.R, cx.F0, cx.flag0, cx.list0, &cx.ctrl[0], kept, nnew);
  }
  nnew = warp_sum(nnew);
  if ((threadIdx.x & 31) == 0 && nnew) atomicAdd(&cx.ctrl[0].nnew, (unsigned long long)nnew);
}

// ------------------------------------------------------------------------------ one BFS level
template <bool kForward>
__global__ void __launch_bounds__(kThreads) k_expand(Ctx cx, int level) {
  __shared__ BlockSmem s;
  const int p = level & 1;
  LevelCtrl* ctrl_cur = &cx.ctrl[level % 3];
  LevelCtrl* ctrl_nxt = &cx.ctrl[(level + 1) % 3];
  uint32_t* Fc = p ? cx.F1 : cx.F0;
  uint32_t* Fn = p ? cx.F0 : cx.F1;
  uint32_t* flagc = p ? cx.flag1 : cx.flag0;
  uint32_t* flagn = p ? cx.flag0 : cx.flag1;
  const int32_t* listc = p ? cx.list1 : cx.list0;
  int32_t* listn = p ? cx.list0 : cx.list1;
  uint32_t* vis = kForward ? cx.V : cx.R;
  const unsigned long long nlist = *((volatile unsigned long long*)&ctrl_cur->count);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    LevelCtrl* z = &cx.ctrl[(level + 2) % 3];
    z->count = 0;
    z->nnew = 0;
    if (nlist) {
      cx.misc[0] += 1;
      if (level < kMaxLevelStats) cx.hist[level] = ctrl_cur->nnew;
    }
  }
  unsigned nnew = 0;
  for (unsigned long long e = blockIdx.x; e < nlist; e += gridDim.x) {
    const int64_t blk = listc[e];
    const BlockInfo bi = decode_block(cx, blk);
    const CompDev& C = cx.comps[bi.comp];
    const ViewDev& Av = kForward ? C.Af : C.Ab;
    const ViewDev& Bv = kForward ? C.Bf : C.Bb;
    load_words(s, Fc, bi, true);
    load_arow(s, Av, bi.ua);
    if (threadIdx.x == 0) flagc[blk] = 0u;
    __syncthreads();
    const int nst = s.wpre[32];
    const int extra = s.aeps > s.a0 ? 1 : 0;
    compact_bits(s, bi.ub0);
    __syncthreads();
    const int32_t total = scan_items(s, nst, Bv.off, extra);
    unsigned kept = 0;
    for (int32_t base = 0; base < total; base += kThreads) {
      const int32_t it = base + threadIdx.x;
      if (it < total) {
        const int st = item_state(s, nst, it);
        const int32_t ub = s.state[st];
        for_item_moves(Av, Bv, s, bi.ua, ub, it - s.scan[st], extra,
                       [&](int32_t va, int32_t vb, int, int32_t, int32_t) {
                         visit<kForward>(C, va, vb, vis, cx.R, Fn, flagn, listn, ctrl_nxt, kept, nnew);
                       });
      }
    }
    if (kForward) {  // pass-1 arc count of this block
      unsigned long long k = warp_sum((unsigned long long)kept);
      if ((threadIdx.x & 31) == 0) s.red[threadIdx.x >> 5] = k;
      __syncthreads();
      if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < kThreads / 32; ++w) t += s.red[w];
        cx.kept[blk] += t;
      }
    }
    __syncthreads();
  }
  nnew = warp_sum(nnew);
  if ((threadIdx.x & 31) == 0 && nnew) atomicAdd(&ctrl_nxt->nnew, (unsigned long long)nnew);
}

// ------------------------------------------------------------------------------ numbering
// One warp per block: vcount[blk] = popcount of V in the block; wpre[word] = exclusive prefix.
__global__ void k_block_counts(Ctx cx) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t blk = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); blk < cx.nblocks; blk += warps) {
    const BlockInfo bi = decode_block(cx, blk);
    uint32_t w = lane < bi.nwords ? cx.V[bi.word0 + lane] : 0u;
    int pc = __popc(w);
    int inc = warp_incl_scan(pc);
    if (lane < bi.nwords) cx.wpre[bi.word0 + lane] = (uint16_t)(inc - pc);
    if (lane == 31) cx.vcount[blk] = inc;
  }
}

__global__ void k_popcount(const uint32_t* __restrict__ bits, int64_t n, unsigned long long* out) {
  unsigned long long s = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += __popc(bits[i]);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

// per-composition totals: tot[2c] = idbase[K_c], tot[2c+1] = arcbase[K_c] (c = 0..ncomp, K_ncomp = nblocks)
__global__ void k_comp_bases(Ctx cx, int64_t* __restrict__ tot) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > cx.ncomp) return;
  int64_t K = c < cx.ncomp ? cx.comps[c].K : cx.nblocks;
  tot[2 * c] = cx.idbase[K];
  tot[2 * c + 1] = cx.arcbase[K];
}

__global__ void k_finish_rowptr(Ctx cx, const int64_t* __restrict__ tot) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cx.ncomp) return;
  const CompDev& C = cx.comps[c];
  int64_t nv = tot[2 * c + 2] - tot[2 * c];
  int64_t ne = tot[2 * c + 3] - tot[2 * c + 1];
  C.row_ptr[nv] = ne;
}

// ------------------------------------------------------------------------------ emit
// Writes the composed CSR: per state (pair_a, pair_b, flags, row_ptr), per arc (dst id, labels,
// weight).  Arc slots = block arc base + CTA running prefix (deterministic; no cursor atomics).
__global__ void __launch_bounds__(kThreads) k_emit(Ctx cx, const int64_t* __restrict__ tot) {
  __shared__ BlockSmem s;
  for (int64_t blk = blockIdx.x; blk < cx.nblocks; blk += gridDim.x) {
    if (cx.vcount[blk] == 0) continue;
    const BlockInfo bi = decode_block(cx, blk);
    const CompDev& C = cx.comps[bi.comp];
    const ViewDev& Av = C.Af;
    const ViewDev& Bv = C.Bf;
    const int64_t id_comp = tot[2 * bi.comp];
    const int64_t arc_comp = tot[2 * bi.comp + 1];
    load_words(s, cx.V, bi, false);
    load_arow(s, Av, bi.ua);
    __syncthreads();
    const int nst = s.wpre[32];
    compact_bits(s, bi.ub0);
    __syncthreads();
    const int32_t total = scan_items(s, nst, Bv.off, 1);
    const int64_t id0 = cx.idbase[blk] - id_comp;
    int64_t run = cx.arcbase[blk] - arc_comp;  // running arc slot of this CTA
    const int64_t run0 = run;
    const int32_t ua = bi.ua;
    auto kept_of = [&](int32_t va, int32_t vb) -> bool {
      const int64_t w = C.W + (int64_t)va * C.wpr + (vb >> 5);
      return (__ldg(&cx.V[w]) >> (vb & 31)) & 1u;
    };
    for (int32_t base = 0; base < total; base += kThreads) {
      const int32_t it = base + threadIdx.x;
      int st = 0;
      int32_t ub = 0, k = 0;
      unsigned cnt = 0;
      if (it < total) {
        st = item_state(s, nst, it);
        ub = s.state[st];
        k = it - s.scan[st];
        for_item_moves(Av, Bv, s, ua, ub, k, 1, [&](int32_t va, int32_t vb, int, int32_t, int32_t) {
          cnt += kept_of(va, vb);
        });
      }
      unsigned long long tot_chunk;
      unsigned long long ex = block_excl_scan((unsigned long long)cnt, s.red, &tot_chunk);
      if (it < total) {
        int64_t pos = run + (int64_t)ex;
        if (k == 0) {  // the state's first item: per-state outputs
          const int64_t id = id0 + st;
          C.row_ptr[id] = pos;
          C.pair_a[id] = ua;
          C.pair_b[id] = ub;
          C.is_start[id] = (uint8_t)(__ldg(&C.startA[ua]) & __ldg(&C.startB[ub]));
          C.is_accept[id] = (uint8_t)(__ldg(&C.accA[ua]) & __ldg(&C.accB[ub]));
        }
        for_item_moves(Av, Bv, s, ua, ub, k, 1, [&](int32_t va, int32_t vb, int kind, int32_t ea, int32_t eb) {
          const int64_t w = C.W + (int64_t)va * C.wpr + (vb >> 5);
          const uint32_t word = __ldg(&cx.V[w]);
          if (!((word >> (vb & 31)) & 1u)) return;
          const int64_t vblk = C.K + (int64_t)va * C.bpr + (vb >> 10);
          const int64_t did = __ldg(&cx.idbase[vblk]) - id_comp + __ldg(&cx.wpre[w]) +
                              __popc(word & ((1u << (vb & 31)) - 1u));
          int32_t il, ol;
          float wt;
          if (kind == 1) {
            il = __ldg(&Av.carry[ea]);
            ol = __ldg(&Bv.carry[eb]);
            wt = __fadd_rn(__ldg(&Av.w[ea]), __ldg(&Bv.w[eb]));  // one IEEE binary32 add, RN-even
          } else if (kind == 2) {
            il = __ldg(&Av.carry[ea]);
            ol = FST_EPS;
            wt = __ldg(&Av.w[ea]);  // bit copy
          } else {
            il = FST_EPS;
            ol = __ldg(&Bv.carry[eb]);
            wt = __ldg(&Bv.w[eb]);
          }
          C.dst[pos] = (int32_t)did;
          C.ilabel[pos] = il;
          C.olabel[pos] = ol;
          C.weight[pos] = wt;
          ++pos;
        });
      }
      run += (int64_t)tot_chunk;
    }
    if (threadIdx.x == 0 && (unsigned long long)(run - run0) != cx.kept[blk]) atomicAdd(&cx.misc[2], 1ull);
    __syncthreads();
  }
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

int g_grid_expand = 0, g_grid_emit = 0;

void init_grids() {
  if (g_grid_expand) return;
  int sms = sm_count();
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_expand<true>, kThreads, 0);
  g_grid_expand = sms * std::max(occ, 1);
  occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_emit, kThreads, 0);
  g_grid_emit = sms * std::max(occ, 1);
}

struct EventTimer {
  bool on;
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s;
  EventTimer(bool on_, cudaStream_t s_) : on(on_), s(s_) {
    if (on) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, s);
    }
  }
  float stop() {
    if (!on) return 0.f;
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms;
  }
};

// Runs one BFS stage (level loop); returns the number of non-empty levels.
template <bool kForward>
fst_status run_stage(const Ctx& cx, cudaStream_t s, unsigned long long* h_pinned, int64_t* expand_launches,
                     std::vector<int64_t>* sizes) {
  int level = 0;
  int batch = 1;
  for (;;) {
    for (int k = 0; k < batch; ++k, ++level) {
      k_expand<kForward><<<g_grid_expand, kThreads, 0, s>>>(cx, level);
      FSTC_LAUNCH_CHECK();
      ++*expand_launches;
    }
    FSTC_CUDA_TRY(cudaMemcpyAsync(h_pinned, &cx.ctrl[level % 3].count, sizeof(unsigned long long),
                                  cudaMemcpyDeviceToHost, s));
    FSTC_CUDA_TRY(cudaStreamSynchronize(s));
    if (*h_pinned == 0) break;
    batch = std::min(batch * 2, 8);  // speculative level batches: empty levels are no-op launches
  }
  unsigned long long nl = 0;
  FSTC_CUDA_TRY(cudaMemcpyAsync(h_pinned, cx.misc, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  FSTC_CUDA_TRY(cudaStreamSynchronize(s));
  nl = *h_pinned;
  if (sizes) {
    int n = (int)std::min<unsigned long long>(nl, kMaxLevelStats);
    std::vector<unsigned long long> tmp(n);
    if (n) {
      FSTC_CUDA_TRY(cudaMemcpyAsync(tmp.data(), cx.hist, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost, s));
      FSTC_CUDA_TRY(cudaStreamSynchronize(s));
    }
    sizes->assign(tmp.begin(), tmp.end());
  }
  return FST_OK;
}

}  // namespace

// Pinned host scratch (one per thread).
static unsigned long long* pinned_scratch() {
  static thread_local unsigned long long* p = nullptr;
  if (!p) {
    if (cudaMallocHost(&p, 64 * sizeof(unsigned long long)) != cudaSuccess) p = nullptr;
  }
  return p;
}

std::vector<int64_t>& level_sizes_slot(fst* h, int stage);

fst_status compose_impl(int32_t n, const fst_handle* a, const fst_handle* b, cudaStream_t s, fst_handle* c) {
  EventTimer t_total(profiling_enabled(), s);
  for (int i = 0; i < n; ++i) c[i] = nullptr;
  for (int i = 0; i < n; ++i) {
    if (!a[i] || !b[i]) {
      set_error(FST_E_INVALID_ARG, "fst_compose: NULL handle at %d", i);
      return FST_E_INVALID_ARG;
    }
    fst_status st = ensure_views(a[i], s);
    if (st) return st;
    st = ensure_views(b[i], s);
    if (st) return st;
  }
  init_grids();
  const int64_t launches0 = fst_launch_count();
  // ---- layout of the concatenated pair space
  std::vector<CompDev> comps(n);
  std::vector<int64_t> seed1(n + 1, 0), seed2(n + 1, 0);
  int64_t W = 0, K = 0, pairs = 0;
  for (int i = 0; i < n; ++i) {
    const fst* A = a[i];
    const fst* B = b[i];
    CompDev& C = comps[i];
    memset(&C, 0, sizeof(C));
    auto vd = [](const View& v) { return ViewDev{v.off, v.key, v.other, v.carry, v.w}; };
    C.Af = vd(A->views[kOutByOlabel]);
    C.Ab = vd(A->views[kInByOlabel]);
    C.Bf = vd(B->views[kOutByIlabel]);
    C.Bb = vd(B->views[kInByIlabel]);
    C.startA = A->is_start; C.startB = B->is_start; C.accA = A->is_accept; C.accB = B->is_accept;
    C.startListA = A->start_list; C.startListB = B->start_list;
    C.accListA = A->accept_list; C.accListB = B->accept_list;
    C.nStartA = A->n_start; C.nStartB = B->n_start; C.nAccA = A->n_accept; C.nAccB = B->n_accept;
    C.VA = A->V;
    C.VB = B->V;
    C.wpr = (B->V + 31) / 32;
    C.bpr = (C.wpr + kWordsPerBlock - 1) / kWordsPerBlock;
    C.W = W;
    C.K = K;
    W += (int64_t)C.VA * C.wpr;
    K += (int64_t)C.VA * C.bpr;
    pairs += (int64_t)C.VA * C.VB;
    seed1[i + 1] = seed1[i] + (int64_t)C.nAccA * C.nAccB;
    seed2[i + 1] = seed2[i] + (int64_t)C.nStartA * C.nStartB;
  }
  const int64_t nwords = W, nblocks = K;
  if (nblocks >= INT32_MAX) {
    set_error(FST_E_CAPACITY, "pair space too large (%lld blocks)", (long long)nblocks);
    return FST_E_CAPACITY;
  }
  // ---- workspace
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
  const size_t oR = take(4 * nwords), oV = take(4 * nwords), oF0 = take(4 * nwords), oF1 = take(4 * nwords);
  const size_t ofl0 = take(4 * nblocks), ofl1 = take(4 * nblocks);
  const size_t ol0 = take(4 * nblocks), ol1 = take(4 * nblocks);
  const size_t octrl = take(sizeof(LevelCtrl) * 3);
  const size_t okept = take(8 * nblocks), ovc = take(4 * nblocks), owpre = take(2 * nwords);
  const size_t oid = take(8 * (nblocks + 1)), oarc = take(8 * (nblocks + 1));
  const size_t otmp = take(8 * scan_tmp_elems(nblocks));
  const size_t ohist = take(8 * kMaxLevelStats), omisc = take(8 * 8);
  const size_t ocomps = take(sizeof(CompDev) * n), oseed1 = take(8 * (n + 1)), oseed2 = take(8 * (n + 1));
  const size_t otot = take(8 * 2 * (n + 1));
  BufferPtr wb;
  fst_status st = alloc_buffer(off, s, &wb);
  if (st) {
    if (st == FST_E_OOM) set_error(FST_E_CAPACITY, "pair space workspace (%zu bytes) does not fit", off);
    return st == FST_E_OOM ? FST_E_CAPACITY : st;
  }
  char* base = (char*)wb->ptr;
  Ctx cx;
  cx.R = (uint32_t*)(base + oR);
  cx.V = (uint32_t*)(base + oV);
  cx.F0 = (uint32_t*)(base + oF0);
  cx.F1 = (uint32_t*)(base + oF1);
  cx.flag0 = (uint32_t*)(base + ofl0);
  cx.flag1 = (uint32_t*)(base + ofl1);
  cx.list0 = (int32_t*)(base + ol0);
  cx.list1 = (int32_t*)(base + ol1);
  cx.ctrl = (LevelCtrl*)(base + octrl);
  cx.kept = (unsigned long long*)(base + okept);
  cx.vcount = (int32_t*)(base + ovc);
  cx.wpre = (uint16_t*)(base + owpre);
  cx.idbase = (int64_t*)(base + oid);
  cx.arcbase = (int64_t*)(base + oarc);
  cx.hist = (unsigned long long*)(base + ohist);
  cx.misc = (unsigned long long*)(base + omisc);
  CompDev* d_comps = (CompDev*)(base + ocomps);
  cx.comps = d_comps;
  cx.ncomp = n;
  cx.nwords = nwords;
  cx.nblocks = nblocks;
  int64_t* d_seed1 = (int64_t*)(base + oseed1);
  int64_t* d_seed2 = (int64_t*)(base + oseed2);
  int64_t* d_tot = (int64_t*)(base + otot);
  int64_t* d_tmp = (int64_t*)(base + otmp);
  unsigned long long* hp = pinned_scratch();
  if (!hp) {
    set_error(FST_E_CUDA, "cudaMallocHost failed");
    return FST_E_CUDA;
  }

  // zero: R, V, F0, F1, flags (contiguous), ctrl, kept, misc
  FSTC_CUDA_TRY(cudaMemsetAsync(base + oR, 0, ol0 - oR, s));
  FSTC_CUDA_TRY(cudaMemsetAsync(base + octrl, 0, sizeof(LevelCtrl) * 3, s));
  FSTC_CUDA_TRY(cudaMemsetAsync(base + okept, 0, 8 * nblocks, s));
  FSTC_CUDA_TRY(cudaMemsetAsync(base + omisc, 0, 64, s));
  FSTC_CUDA_TRY(cudaMemcpyAsync(d_comps, comps.data(), sizeof(CompDev) * n, cudaMemcpyHostToDevice, s));
  FSTC_CUDA_TRY(cudaMemcpyAsync(d_seed1, seed1.data(), 8 * (n + 1), cudaMemcpyHostToDevice, s));
  FSTC_CUDA_TRY(cudaMemcpyAsync(d_seed2, seed2.data(), 8 * (n + 1), cudaMemcpyHostToDevice, s));

  fst_compose_stats stats{};
  stats.pair_space = pairs;
  stats.num_coaccessible = -1;
  int64_t expand_launches = 0;
  std::vector<int64_t> sizes1, sizes2;
  const bool prof = profiling_enabled();

  // ---- stage 1: co-accessible set R (backward BFS from accept pairs)
  {
    EventTimer t(prof, s);
    cx.seedbase = d_seed1;
    if (seed1[n] > 0) {
      k_seed<false><<<nblk(seed1[n], 256), 256, 0, s>>>(cx);
      FSTC_LAUNCH_CHECK();
      st = run_stage<false>(cx, s, hp, &expand_launches, &sizes1);
      if (st) return st;
    }
    stats.levels_stage1 = (int32_t)sizes1.size();
    stats.ms_stage1 = t.stop();
  }
  // ---- stage 2: accessible states restricted to R (forward BFS from start pairs)
  FSTC_CUDA_TRY(cudaMemsetAsync(base + octrl, 0, sizeof(LevelCtrl) * 3, s));
  FSTC_CUDA_TRY(cudaMemsetAsync(base + omisc, 0, 8, s));
  {
    EventTimer t(prof, s);
    cx.seedbase = d_seed2;
    if (seed2[n] > 0 && seed1[n] > 0) {
      k_seed<true><<<nblk(seed2[n], 256), 256, 0, s>>>(cx);
      FSTC_LAUNCH_CHECK();
      st = run_stage<true>(cx, s, hp, &expand_launches, &sizes2);
      if (st) return st;
    }
    stats.levels_stage2 = (int32_t)sizes2.size();
    stats.ms_stage2 = t.stop();
  }
  // ---- numbering: per-block state counts, word prefixes, scans, per-composition totals
  std::vector<int64_t> tot(2 * (n + 1));
  {
    EventTimer t(prof, s);
    k_block_counts<<<nblk(nblocks * 32, 256), 256, 0, s>>>(cx);
    FSTC_LAUNCH_CHECK();
    st = exclusive_scan_i32(cx.vcount, nblocks, cx.idbase, d_tmp, s);
    if (st) return st;
    st = exclusive_scan_u64(cx.kept, nblocks, cx.arcbase, d_tmp, s);
    if (st) return st;
    k_comp_bases<<<nblk(n + 1, 128), 128, 0, s>>>(cx, d_tot);
    FSTC_LAUNCH_CHECK();
    if (prof) {
      k_popcount<<<sm_count() * 4, 256, 0, s>>>(cx.R, nwords, cx.misc + 1);
      FSTC_LAUNCH_CHECK();
    }
    FSTC_CUDA_TRY(cudaMemcpyAsync(tot.data(), d_tot, 8 * 2 * (n + 1), cudaMemcpyDeviceToHost, s));
    if (prof) FSTC_CUDA_TRY(cudaMemcpyAsync(hp + 1, cx.misc + 1, 8, cudaMemcpyDeviceToHost, s));
    FSTC_CUDA_TRY(cudaStreamSynchronize(s));
    if (prof) stats.num_coaccessible = (int64_t)hp[1];
    // ---- output allocation (one buffer per composition)
    std::vector<fst*> outs(n, nullptr);
    auto cleanup = [&]() {
      for (auto* h : outs) delete h;
    };
    for (int i = 0; i < n; ++i) {
      const int64_t nv = tot[2 * i + 2] - tot[2 * i], ne = tot[2 * i + 3] - tot[2 * i + 1];
      if (nv >= INT32_MAX) {
        cleanup();
        set_error(FST_E_CAPACITY, "composition %d has %lld states (>= 2^31)", i, (long long)nv);
        return FST_E_CAPACITY;
      }
      size_t ob = 0;
      auto tk = [&](size_t bytes) { size_t o = ob; ob += (bytes + 255) & ~size_t(255); return o; };
      const size_t o_rp = tk(8 * (nv + 1)), o_il = tk(4 * ne), o_ol = tk(4 * ne), o_d = tk(4 * ne),
                   o_w = tk(4 * ne), o_st = tk(nv), o_ac = tk(nv), o_pa = tk(4 * nv), o_pb = tk(4 * nv);
      BufferPtr obuf;
      st = alloc_buffer(ob, s, &obuf);
      if (st) {
        cleanup();
        return st;
      }
      fst* h = new fst();
      outs[i] = h;
      h->composed = true;
      h->V = (int32_t)nv;
      h->E = ne;
      h->stream = s;
      char* pb = (char*)obuf->ptr;
      h->row_ptr = (int64_t*)(pb + o_rp);
      h->ilabel = (int32_t*)(pb + o_il);
      h->olabel = (int32_t*)(pb + o_ol);
      h->dst = (int32_t*)(pb + o_d);
      h->weight = (float*)(pb + o_w);
      h->is_start = (uint8_t*)(pb + o_st);
      h->is_accept = (uint8_t*)(pb + o_ac);
      h->pair_a = (int32_t*)(pb + o_pa);
      h->pair_b = (int32_t*)(pb + o_pb);
      h->buffers.push_back(obuf);
      CompDev& C = comps[i];
      C.row_ptr = h->row_ptr;
      C.ilabel = h->ilabel;
      C.olabel = h->olabel;
      C.dst = h->dst;
      C.weight = h->weight;
      C.is_start = h->is_start;
      C.is_accept = h->is_accept;
      C.pair_a = h->pair_a;
      C.pair_b = h->pair_b;
    }
    FSTC_CUDA_TRY(cudaMemcpyAsync(d_comps, comps.data(), sizeof(CompDev) * n, cudaMemcpyHostToDevice, s));
    stats.ms_number = t.stop();
    // ---- emit
    {
      EventTimer te(prof, s);
      k_emit<<<g_grid_emit, kThreads, 0, s>>>(cx, d_tot);
      FSTC_LAUNCH_CHECK();
      k_finish_rowptr<<<nblk(n, 128), 128, 0, s>>>(cx, d_tot);
      FSTC_LAUNCH_CHECK();
      FSTC_CUDA_TRY(cudaMemcpyAsync(hp + 2, cx.misc + 2, 8, cudaMemcpyDeviceToHost, s));
      cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) {
        cleanup();
        set_error(FST_E_CUDA, "compose: %s", cudaGetErrorString(e));
        return FST_E_CUDA;
      }
      stats.ms_emit = te.stop();
      if (hp[2] != 0) {
        cleanup();
        set_error(FST_E_INTERNAL, "emit/count mismatch in %llu blocks", hp[2]);
        return FST_E_INTERNAL;
      }
    }
    wb.reset();
    stats.ms_total = t_total.stop();
    stats.launches = fst_launch_count() - launches0;
    stats.expand_launches = expand_launches;
    stats.emit_launches = 1;
    for (int i = 0; i < n; ++i) {
      outs[i]->stats = stats;
      level_sizes_slot(outs[i], 1) = sizes1;
      level_sizes_slot(outs[i], 2) = sizes2;
      c[i] = outs[i];
    }
  }
  return FST_OK;
}

}  // namespace fstc
