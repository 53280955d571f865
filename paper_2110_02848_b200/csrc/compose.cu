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
// Work decomposition (B200-first, not the paper's thread-per-arc-pair): one CTA task is a CHUNK =
// a run of 1024-pair blocks of one pair-space row u_a.  All moves out of row u_a land in the few
// destination rows {dst(e_a)} U {u_a}; the CTA stages the A row (label mask table) and those
// destination rows' bitmaps / rank tables in shared memory, then streams the B-side "items" (one
// sentinel + the out-arcs of every state, contiguous in B's view) of the chunk.  Candidates are
// tested and claimed in shared memory and merged into the global bitmaps one 32-bit word at a
// time.  Sparse chunks and rows whose staging does not fit fall back to compacted per-state work
// with global test-and-set.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <vector>

#include "fstc_handle.h"
#include "fstc_internal.cuh"
#include "scan.cuh"
#include "wave.h"

namespace fstc {

fst_status ensure_views(fst* h, cudaStream_t s);
fst_status alloc_buffer(size_t bytes, cudaStream_t s, BufferPtr* out);
bool profiling_enabled();

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kAMax = 64;           // A-row arcs staged in shared memory
constexpr int kSlotMax = 32;        // destination rows staged in shared memory
constexpr int kChunkMaxBlocks = 32; // blocks per chunk (<= 1024 words)
constexpr int kDynSmem = 88 * 1024; // staging area (destination rows)
constexpr int kSimpleMoves = 4;    // warps whose items have <= this many moves skip the expansion
constexpr int kHeavy = 64;         // states with more B arcs are walked cooperatively by the CTA
constexpr int kWCap = 160;         // per-warp output window of the fast emit (arcs), at most
constexpr int kWCapMin = 64;       // ... and at least (smaller when the staged rows take the space)
constexpr int kOwnerCap = 384;     // per-warp arc-slot owner table of the BFS walk (end of dynamic smem)
constexpr int kOwnerBytes = kWarps * kOwnerCap;

constexpr int kCompQ = 64;

struct Ctx {
  uint32_t* R;
  uint32_t* V;
  uint32_t* F0;
  uint32_t* F1;
  uint32_t* flag0;  // per chunk
  uint32_t* flag1;
  int32_t* list0;   // active chunk lists
  int32_t* list1;
  LevelCtrl* ctrl;
  unsigned long long* kept;  // per block
  int32_t* vcount;           // per block
  uint16_t* wpre;            // per word
  int64_t* idbase;           // per block (+1)
  int64_t* arcbase;          // per block (+1)
  unsigned long long* hist;  // per-level frontier sizes
  unsigned long long* misc;  // [0] nonempty levels, [1] |R|, [2] emit consistency errors, [3] staged tasks
  uint8_t* cnt8;             // per pair: out-degree in C recorded by the stage-2 fast path (255 = recount)
  uint32_t* warc;            // tile path: per word, arcs of its states (k_tile_count), then the exclusive
                             // prefix inside the word's block (k_block_counts); aliases cnt8's memory
  uint32_t* OUT;             // sharded mode: claims for pairs in rows owned by other shards
  const CompDev* comps;
  const int64_t* seedbase;
  int32_t ncomp;
  int64_t nwords, nblocks, nchunks;
  int32_t* level_dev;  // graph-driven level loop: the true level number (hist index), advanced by block 0
  // first chunk of every composition (batches of <= kCompQ): kernel-parameter copy, so a task's
  // composition is found in the constant bank instead of by dependent global loads every level
  int64_t compQ[kCompQ];
  int64_t ptotal;   // pairs over all compositions (pull decision of stage 1)
  int32_t pull_ok;  // stage 1 may run bottom-up (pull) levels (unsharded compositions only)
  int32_t pull_num; // pull threshold: frontier * pull_num >= unvisited * 4
};

struct Chunk {
  int comp;
  int32_t ua;
  int32_t b0, b1;   // blocks [b0, b1) of the row
  int64_t rowW;     // global word index of (ua, 0)
};

__device__ __forceinline__ int find_comp_q(const CompDev* __restrict__ comps, int ncomp, int64_t q) {
  int lo = 0, hi = ncomp - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (comps[mid].Q <= q) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ Chunk decode_chunk(const Ctx& cx, int64_t q) {
  Chunk ch;
  if (cx.ncomp == 1) {
    ch.comp = 0;
  } else if (cx.ncomp <= kCompQ) {
    int lo = 0, hi = cx.ncomp - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (cx.compQ[mid] <= q) lo = mid; else hi = mid - 1;
    }
    ch.comp = lo;
  } else {
    ch.comp = find_comp_q(cx.comps, cx.ncomp, q);
  }
  const CompDev& C = cx.comps[ch.comp];
  int64_t local = q - C.Q;
  ch.ua = (int32_t)(local / C.cpr);
  int32_t j = (int32_t)(local - (int64_t)ch.ua * C.cpr);
  ch.b0 = j * C.CB;
  ch.b1 = min(ch.b0 + C.CB, C.bpr);
  ch.rowW = C.W + (int64_t)ch.ua * C.wpr;
  return ch;
}

__device__ __forceinline__ int64_t chunk_of(const CompDev& C, int32_t row, int32_t col) {
  return C.Q + (int64_t)row * C.cpr + ((col >> 10) / C.CB);
}

__device__ __forceinline__ int32_t lower_bound_g(const int32_t* __restrict__ key, int32_t lo, int32_t hi, int32_t x) {
  while (lo < hi) {
    int32_t mid = (lo + hi) >> 1;
    if (__ldg(&key[mid]) < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int32_t lower_bound_s(const int32_t* key, int32_t lo, int32_t hi, int32_t x) {
  while (lo < hi) {
    int32_t mid = (lo + hi) >> 1;
    if (key[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Mark a newly claimed pair in the next frontier: bits, chunk flag and list append.
__device__ __forceinline__ void push_bits(const CompDev& C, int32_t row, int32_t col, int64_t gw, uint32_t bits,
                                          uint32_t* __restrict__ Fn, uint32_t* __restrict__ flagn,
                                          int32_t* __restrict__ listn, LevelCtrl* ctrln) {
  atomicOr(&Fn[gw], bits);
  const int64_t q = chunk_of(C, row, col);
  if (*((volatile uint32_t*)&flagn[q]) == 0 && atomicExch(&flagn[q], 1u) == 0) {
    unsigned long long pos = atomicAdd(&ctrln->count, 1ull);
    listn[pos] = (int32_t)q;
  }
}

// ------------------------------------------------------------------------------ shared state
struct TaskSmem {
  uint32_t fw[kChunkMaxBlocks * 32];  // source bits of the chunk (frontier or V)
  int32_t a_key[kAMax];
  int32_t a_other[kAMax];
  int32_t a_slot[kAMax];
  int32_t a_carry[kAMax];
  float a_w[kAMax];
  unsigned long long labmask[64];     // labmask[l+1] = A-row positions with olabel l (l < 63)
  uint32_t labmask32[64];             // the same for rows of <= 32 arcs
  int32_t mask32;
  int32_t slot_row[kSlotMax];
  int32_t a0, a1, deg, aeps, m, arow_smem, dst_staged, small;
  unsigned long long repmask;         // stage_arow: A arcs that open a new destination-row slot
  int32_t state[kPairsPerBlock];      // compacted source states of a sparse block (ascending u_b)
  int32_t scan[kPairsPerBlock + 1];   // their item offsets
  int32_t bwpre[33];
  int32_t wtot[kWarps + 1];
  int32_t red32[kWarps + 1];
  unsigned long long keptb;
  // label-major path: A-row label groups and their B segment ranges
  int32_t G;                              // groups (0 = label-major path unavailable for this row)
  int32_t g_label[kAMax + 1];
  unsigned long long g_mask[kAMax + 1];   // A-row positions with the group's olabel
  int32_t g_s0[kAMax + 1], g_s1[kAMax + 1];
  int32_t g_lo[kAMax + 1];                // per block: first segment of the group in the block
  int32_t g_pre[kAMax + 2];               // per block: item prefix over groups
  int32_t cur[kPairsPerBlock + 1];        // emit: per-state arc cursor / count
  int32_t nheavy;
  int32_t segnext;
  unsigned long long keptc[kChunkMaxBlocks];  // per-block kept counts of the chunk (stage 2)
};

// Label groups of the staged A row, matched against B's label-major index (thread 0).
__device__ void build_groups(TaskSmem& s, const ViewDev& Bv) {
  if (threadIdx.x != 0) return;
  s.G = 0;
  if (!s.arow_smem) return;
  const int nlab = Bv.nlab;
  const bool b_has_eps = nlab > 0 && __ldg(&Bv.lab_val[0]) == FST_EPS;
  int G = 0;
  int k = 0;
  if (b_has_eps && !(s.deg > 0 && s.a_key[0] == FST_EPS)) {  // eps group for M3 even without A eps arcs
    s.g_label[G] = FST_EPS;
    s.g_mask[G] = 0ull;
    ++G;
  }
  while (k < s.deg) {
    const int32_t lab = s.a_key[k];
    unsigned long long m = 0ull;
    while (k < s.deg && s.a_key[k] == lab) m |= 1ull << k++;
    s.g_label[G] = lab;
    s.g_mask[G] = m;
    ++G;
  }
  int out = 0;
  for (int g = 0; g < G; ++g) {  // keep groups whose label occurs in B
    const int32_t lab = s.g_label[g];
    int lo = 0, hi = nlab;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (__ldg(&Bv.lab_val[mid]) < lab) lo = mid + 1; else hi = mid;
    }
    if (lo < nlab && __ldg(&Bv.lab_val[lo]) == lab) {
      s.g_label[out] = lab;
      s.g_mask[out] = s.g_mask[g];
      s.g_s0[out] = __ldg(&Bv.lab_seg[lo]);
      s.g_s1[out] = __ldg(&Bv.lab_seg[lo + 1]);
      ++out;
    }
  }
  s.G = out > 0 ? out : -1;  // -1: label-major possible but nothing matches
}

// Segment ranges of every group for states [ub0, ub1); returns the total item count.
__device__ __forceinline__ int block_groups(TaskSmem& s, const ViewDev& Bv, int32_t ub0, int32_t ub1) {
  if ((int)threadIdx.x < s.G) {
    const int g = threadIdx.x;
    int lo = s.g_s0[g], hi = s.g_s1[g];
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (__ldg(&Bv.seg_node[mid]) < ub0) lo = mid + 1; else hi = mid;
    }
    int lo2 = lo, hi2 = s.g_s1[g];
    while (lo2 < hi2) {
      int mid = (lo2 + hi2) >> 1;
      if (__ldg(&Bv.seg_node[mid]) < ub1) lo2 = mid + 1; else hi2 = mid;
    }
    s.g_lo[g] = lo;
    s.g_pre[g + 1] = lo2 - lo;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    s.g_pre[0] = 0;
    for (int g = 0; g < s.G; ++g) s.g_pre[g + 1] += s.g_pre[g];
  }
  __syncthreads();
  return s.G > 0 ? s.g_pre[s.G] : 0;
}

__device__ __forceinline__ int item_group(const TaskSmem& s, int i) {
  int g = 0;
  while (g + 1 < s.G && s.g_pre[g + 1] <= i) ++g;
  return g;
}

__device__ __forceinline__ bool rep_is(unsigned long long rm, int t) { return (rm >> t) & 1ull; }

// Stage the A row u_a of view Av: arcs (label-sorted), label masks, destination-row slots.
// dst_words = shared words needed per destination row; staging succeeds iff m * dst_words fits.
__device__ void stage_arow(TaskSmem& s, const CompDev& C, const ViewDev& Av, int32_t ua, int dst_words,
                           int cap_words = kDynSmem / 4) {
  if (threadIdx.x == 0) {
    s.a0 = __ldg(&Av.off[ua]);
    s.a1 = __ldg(&Av.off[ua + 1]);
    s.deg = s.a1 - s.a0;
    s.arow_smem = s.deg <= kAMax;
    s.small = s.arow_smem && C.smallA;
    s.aeps = 0;
    s.repmask = 0ull;
  }
  __syncthreads();
  if (s.arow_smem) {
    for (int k = threadIdx.x; k < s.deg; k += kThreads) {
      s.a_key[k] = __ldg(&Av.key[s.a0 + k]);
      s.a_other[k] = __ldg(&Av.other[s.a0 + k]);
      s.a_carry[k] = __ldg(&Av.carry[s.a0 + k]);
      s.a_w[k] = __ldg(&Av.w[s.a0 + k]);
    }
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (s.arow_smem) {  // (all in parallel, threads < 64) label masks, eps count, slot-opening arcs
    const int deg = s.deg;
    if (t < 64) {
      unsigned long long lm = 0ull;
      if (s.small)
        for (int k = 0; k < deg; ++k) lm |= (unsigned long long)(s.a_key[k] + 1 == t) << k;
      s.labmask[t] = lm;
      s.labmask32[t] = (uint32_t)lm;
      if (t < deg) {
        if (s.a_key[t] < 0 && (t + 1 == deg || s.a_key[t + 1] >= 0)) s.aeps = t + 1;  // eps arcs sort first
        const int r = s.a_other[t];
        bool first = r != ua;
        for (int j = 0; j < t && first; ++j) first = s.a_other[j] != r;
        if (first) atomicOr(&s.repmask, 1ull << t);
      }
    }
  } else if (t == 0) {
    s.aeps = lower_bound_g(Av.key, s.a0, s.a1, 0) - s.a0;
    s.m = 0;
    s.dst_staged = 0;
  }
  __syncthreads();
  if (s.arow_smem) {
    // destination-row slots: slot 0 = u_a (M3 moves), then the distinct rows in order of first arc
    const unsigned long long rm = s.repmask;
    const int m = 1 + __popcll(rm);
    const bool ok = m <= kSlotMax;
    if (t < s.deg) {
      const int r = s.a_other[t];
      int slot = 0;
      if (r != ua) {
        int rep = 0;
        while (s.a_other[rep] != r) ++rep;
        slot = 1 + __popcll(rm & ((1ull << rep) - 1ull));
      }
      s.a_slot[t] = slot;
      if (slot > 0 && rep_is(rm, t) && slot < kSlotMax) s.slot_row[slot] = r;
    }
    if (t == 0) {
      s.slot_row[0] = ua;
      s.m = ok ? m : kSlotMax;
      s.mask32 = s.deg <= 32;
      s.dst_staged = ok && (int64_t)m * dst_words <= cap_words;
      if (!ok) s.small = 0;  // slots incomplete: the fast paths need a slot for every A arc
    }
  }
  __syncthreads();
}

// One B-side item (a state's sentinel, or one of its B arcs) and its matching A arcs.
struct Item {
  unsigned long long mask;  // s.small: A-row positions of the matches
  int32_t lo;               // otherwise: first matching A-row position
  int32_t n;                // moves of the item (M2 | M1 [+ M3])
  int32_t col;              // B-side destination: other end of the arc, u_b for the sentinel
  int32_t it, ub;           // item index, source state
  int32_t kind;             // 1 = arc (M1, then M3 if eps), 2 = sentinel (M2)
  int32_t m3;
};

__device__ __forceinline__ Item make_item(const TaskSmem& s, const ViewDev& Av, int32_t it, int32_t ub, int2 kd,
                                          bool valid) {
  Item x;
  x.mask = 0ull;
  x.lo = 0;
  x.n = 0;
  x.col = kd.y;
  x.it = it;
  x.ub = ub;
  x.kind = 1;
  x.m3 = 0;
  if (!valid) return x;
  if (kd.x == kSentinel) {  // M2: A arcs with olabel eps, B stays
    x.kind = 2;
    x.col = ub;
    if (s.small) {
      x.mask = s.labmask[0];
      x.n = __popcll(x.mask);
    } else {
      x.n = s.aeps;
    }
    return x;
  }
  const int32_t lab = kd.x;
  if (s.small) {
    x.mask = (lab + 1 < 64) ? s.labmask[lab + 1] : 0ull;
    x.n = __popcll(x.mask);
  } else if (s.arow_smem) {
    x.lo = lower_bound_s(s.a_key, 0, s.deg, lab);
    x.n = lower_bound_s(s.a_key, x.lo, s.deg, lab + 1) - x.lo;
  } else {
    const int32_t lo = lower_bound_g(Av.key, s.a0, s.a1, lab);
    x.lo = lo - s.a0;
    x.n = lower_bound_g(Av.key, lo, s.a1, lab + 1) - lo;
  }
  x.m3 = lab == FST_EPS;
  x.n += x.m3;
  return x;
}

// A candidate move: destination (row, col) (slot = staged destination-row index or -1), kind
// 1 = M1, 2 = M2, 3 = M3, k = A-row position (-1 for M3), eb = B view position (-1 for M2).
struct Cand {
  int32_t slot, row, col, kind, k, eb;
};

__device__ __forceinline__ int kth_bit(unsigned long long m, int k) {
  for (int i = 0; i < k; ++i) m &= m - 1;
  return __ffsll((long long)m) - 1;
}

// The k-th move (0 <= k < x.n) of item x: M1/M2 matches in A-row order, then M3.
__device__ __forceinline__ Cand item_move(const TaskSmem& s, const ViewDev& Av, int32_t ua, const Item& x, int k) {
  Cand cd;
  cd.col = x.col;
  cd.eb = x.kind == 1 ? x.it - x.ub - 1 : -1;
  if (k < x.n - x.m3) {
    const int a = s.small ? kth_bit(x.mask, k) : x.lo + k;
    cd.kind = x.kind;
    cd.k = a;
    if (s.arow_smem) {
      cd.slot = s.a_slot[a];
      cd.row = s.a_other[a];
    } else {
      cd.slot = -1;
      cd.row = __ldg(&Av.other[s.a0 + a]);
    }
  } else {
    cd.kind = 3;
    cd.k = -1;
    cd.slot = 0;
    cd.row = ua;
  }
  return cd;
}

// Warp-cooperative expansion of the 32 lanes' items into rounds of (up to) 32 candidates, in item
// order then match order.  f(active, cand, round) is called by ALL lanes every round (so it may use
// warp ballots).  This keeps the candidate work convergent whatever the per-item match counts.
template <typename F>
__device__ __forceinline__ void warp_expand(const TaskSmem& s, const ViewDev& Av, int32_t ua, const Item& x, F&& f) {
  const int lane = threadIdx.x & 31;
  const int incl = warp_incl_scan(x.n);
  const int start = incl - x.n;
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  for (int r = 0; r < total; r += 32) {
    const int c = r + lane;
    int j = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
      const int sj = __shfl_sync(0xffffffffu, start, j + step);
      if (sj <= c) j += step;
    }
    const int rank = c - __shfl_sync(0xffffffffu, start, j);
    const unsigned mlo = __shfl_sync(0xffffffffu, (unsigned)x.mask, j);
    const unsigned mhi = __shfl_sync(0xffffffffu, (unsigned)(x.mask >> 32), j);
    const int lo = __shfl_sync(0xffffffffu, x.lo, j);
    const int n = __shfl_sync(0xffffffffu, x.n, j);
    const int m3 = __shfl_sync(0xffffffffu, x.m3, j);
    const int col = __shfl_sync(0xffffffffu, x.col, j);
    const int kind = __shfl_sync(0xffffffffu, x.kind, j);
    const int it = __shfl_sync(0xffffffffu, x.it, j);
    const int ub = __shfl_sync(0xffffffffu, x.ub, j);
    const bool act = c < total;
    Cand cd;
    cd.col = col;
    cd.eb = kind == 1 ? it - ub - 1 : -1;
    if (act && rank < n - m3) {
      const int k = s.small ? kth_bit(((unsigned long long)mhi << 32) | mlo, rank) : lo + rank;
      cd.kind = kind == 2 ? 2 : 1;
      cd.k = k;
      if (s.arow_smem) {
        cd.slot = s.a_slot[k];
        cd.row = s.a_other[k];
      } else {
        cd.slot = -1;
        cd.row = __ldg(&Av.other[s.a0 + k]);
      }
    } else {
      cd.kind = 3;
      cd.k = -1;
      cd.slot = 0;
      cd.row = ua;
    }
    f(act, cd, r);
  }
}

// Source bits of the chunk -> s.fw (optionally consuming them).  Returns the popcount (all threads).
__device__ __forceinline__ int load_chunk_bits(TaskSmem& s, uint32_t* bits, const CompDev& C, const Chunk& ch,
                                               bool consume) {
  const int w0 = ch.b0 * 32, w1 = min(ch.b1 * 32, C.wpr);
  int cnt = 0;
  for (int w = w0 + threadIdx.x; w < w1; w += kThreads) {
    uint32_t x = bits[ch.rowW + w];
    if (consume && x) bits[ch.rowW + w] = 0u;
    s.fw[w - w0] = x;
    cnt += __popc(x);
  }
  cnt = warp_sum(cnt);
  if ((threadIdx.x & 31) == 0) s.red32[threadIdx.x >> 5] = cnt;
  __syncthreads();
  int tot = 0;
  for (int i = 0; i < kWarps; ++i) tot += s.red32[i];
  __syncthreads();
  return tot;
}

// Number of source bits of block `blk` in s.fw (all threads; one barrier).
__device__ __forceinline__ int block_popc(TaskSmem& s, const CompDev& C, const Chunk& ch, int32_t blk) {
  const int lw0 = (blk - ch.b0) * 32;
  const int nw = min(32, C.wpr - blk * 32);
  if (threadIdx.x < 32) {
    const int pc = threadIdx.x < nw ? __popc(s.fw[lw0 + threadIdx.x]) : 0;
    const int t = warp_sum(pc);
    if (threadIdx.x == 0) s.red32[kWarps] = t;
  }
  __syncthreads();
  const int t = s.red32[kWarps];
  __syncthreads();
  return t;
}

__device__ __forceinline__ bool src_bit(const TaskSmem& s, int lw0, int32_t ub0, int32_t ub) {
  return (s.fw[lw0 + ((ub - ub0) >> 5)] >> (ub & 31)) & 1u;
}

// Walk the items of block `blk` whose source state bit is set in s.fw.  Dense blocks stream the
// contiguous item range of B's view; sparse blocks compact their states first.  g(valid, it, ub, kd)
// is called by every thread in every round (uniform trip count; g may __syncthreads).
template <typename G>
__device__ __forceinline__ void for_block_items(TaskSmem& s, const ViewDev& Bv, const CompDev& C, const Chunk& ch,
                                                int32_t blk, G&& g) {
  const int lw0 = (blk - ch.b0) * 32;
  const int nw = min(32, C.wpr - blk * 32);
  const int32_t ub0 = blk * kPairsPerBlock;
  const int32_t ub1 = min(ub0 + kPairsPerBlock, C.VB);
  if (threadIdx.x < 32) {
    uint32_t w = threadIdx.x < nw ? s.fw[lw0 + threadIdx.x] : 0u;
    int pc = __popc(w);
    int inc = warp_incl_scan(pc);
    s.bwpre[threadIdx.x] = inc - pc;
    if (threadIdx.x == 31) s.bwpre[32] = inc;
  }
  __syncthreads();
  const int nst = s.bwpre[32];
  if (nst == 0) return;
  if (nst * 4 >= (ub1 - ub0)) {  // dense: stream every item of the block (next round prefetched)
    const int32_t i0 = __ldg(&Bv.off[ub0]) + ub0;
    const int32_t i1 = __ldg(&Bv.off[ub1]) + ub1;
    int32_t it = i0 + threadIdx.x;
    int2 kd = make_int2(0, 0);
    int32_t ub = ub0;
    if (it < i1) {
      kd = __ldg(&Bv.ikd[it]);
      ub = __ldg(&Bv.isrc[it]);
    }
    for (int32_t base = i0; base < i1; base += kThreads) {
      const int32_t nit = it + kThreads;
      int2 nkd = make_int2(0, 0);
      int32_t nub = ub0;
      if (nit < i1) {
        nkd = __ldg(&Bv.ikd[nit]);
        nub = __ldg(&Bv.isrc[nit]);
      }
      const bool valid = it < i1 && ((s.fw[lw0 + ((ub - ub0) >> 5)] >> (ub & 31)) & 1u);
      g(valid, it, ub, kd);
      it = nit;
      kd = nkd;
      ub = nub;
    }
  } else {  // sparse: compact the states, scan their item counts (1 sentinel + deg_B)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = warp; i < nw; i += kWarps) {
      uint32_t w = s.fw[lw0 + i];
      if ((w >> lane) & 1u) s.state[s.bwpre[i] + __popc(w & ((1u << lane) - 1u))] = ub0 + i * 32 + lane;
    }
    __syncthreads();
    int32_t c0 = 0, c1 = 0;
    const int i0s = threadIdx.x * 2;
    if (i0s < nst) { int32_t ub = s.state[i0s]; c0 = 1 + __ldg(&Bv.off[ub + 1]) - __ldg(&Bv.off[ub]); }
    if (i0s + 1 < nst) { int32_t ub = s.state[i0s + 1]; c1 = 1 + __ldg(&Bv.off[ub + 1]) - __ldg(&Bv.off[ub]); }
    int32_t tot;
    int32_t ex = block_excl_scan(c0 + c1, s.red32, &tot);
    if (i0s < nst) s.scan[i0s] = ex;
    if (i0s + 1 < nst) s.scan[i0s + 1] = ex + c0;
    if (threadIdx.x == 0) s.scan[nst] = tot;
    __syncthreads();
    for (int32_t base = 0; base < tot; base += kThreads) {
      const int32_t li = base + threadIdx.x;
      const bool valid = li < tot;
      int2 kd = make_int2(0, 0);
      int32_t ub = ub0, it = 0;
      if (valid) {
        int lo = 0, hi = nst - 1;
        while (lo < hi) {
          int mid = (lo + hi + 1) >> 1;
          if (s.scan[mid] <= li) lo = mid; else hi = mid - 1;
        }
        ub = s.state[lo];
        it = __ldg(&Bv.off[ub]) + ub + (li - s.scan[lo]);
        kd = __ldg(&Bv.ikd[it]);
      }
      g(valid, it, ub, kd);
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------------------------ fast paths
// Lean per-state walkers for the common case: A row staged with label masks (olabels < 63, <= 64
// arcs) and the destination rows staged in shared memory.  One thread walks one state's B arcs
// (packed (label, other) items); states with more than kHeavy arcs are walked by the whole CTA.

// f(slot, col, kind, a, eb) for every move of state ub (M2, then per B arc: M1 matches, M3).
template <bool kM32, typename F>
__device__ __forceinline__ void fast_arc(const TaskSmem& s, int2 x, int32_t eb, F&& f) {
  if (kM32) {
    uint32_t m = (unsigned)(x.x + 1) < 64u ? s.labmask32[x.x + 1] : 0u;
    while (m) {
      const int a = __ffs(m) - 1;
      m &= m - 1;
      f(s.a_slot[a], x.y, 1, a, eb);
    }
  } else {
    unsigned long long m = (unsigned)(x.x + 1) < 64u ? s.labmask[x.x + 1] : 0ull;
    while (m) {
      const int a = __ffsll((long long)m) - 1;
      m &= m - 1;
      f(s.a_slot[a], x.y, 1, a, eb);
    }
  }
  if (x.x == FST_EPS) f(0, x.y, 3, -1, eb);
}

template <bool kM32, typename F>
__device__ __forceinline__ void fast_state(const TaskSmem& s, const int2* __restrict__ ikd, int32_t ub, int32_t e,
                                           int32_t e1, F&& f) {
  for (int a = 0; a < s.aeps; ++a) f(s.a_slot[a], ub, 2, a, -1);
  // items e .. e1-1 are the arcs (view positions e - ub - 1)
  for (; e + 2 <= e1; e += 2) {
    const int2 x0 = __ldg(&ikd[e]), x1 = __ldg(&ikd[e + 1]);
    fast_arc<kM32>(s, x0, e - ub - 1, f);
    fast_arc<kM32>(s, x1, e - ub, f);
  }
  if (e < e1) fast_arc<kM32>(s, __ldg(&ikd[e]), e - ub - 1, f);
}

// Same walk over the 16-byte items (label, other, carry, weight bits):
// g(slot, col, kind, a, carry, wbits, it) with it = the item index (-1 for M2 moves)
template <bool kM32, typename G>
__device__ __forceinline__ void fast_state4(const TaskSmem& s, const int4* __restrict__ ikcw, int32_t ub, int32_t e,
                                            int32_t e1, G&& g) {
  for (int a = 0; a < s.aeps; ++a) g(s.a_slot[a], ub, 2, a, 0, 0, -1);
  auto one = [&](const int4 x, int32_t it) {
    if (kM32) {
      uint32_t m = (unsigned)(x.x + 1) < 64u ? s.labmask32[x.x + 1] : 0u;
      while (m) {
        const int a = __ffs(m) - 1;
        m &= m - 1;
        g(s.a_slot[a], x.y, 1, a, x.z, x.w, it);
      }
    } else {
      unsigned long long m = (unsigned)(x.x + 1) < 64u ? s.labmask[x.x + 1] : 0ull;
      while (m) {
        const int a = __ffsll((long long)m) - 1;
        m &= m - 1;
        g(s.a_slot[a], x.y, 1, a, x.z, x.w, it);
      }
    }
    if (x.x == FST_EPS) g(0, x.y, 3, -1, x.z, x.w, it);
  };
  for (; e + 2 <= e1; e += 2) {
    const int4 x0 = __ldg(&ikcw[e]), x1 = __ldg(&ikcw[e + 1]);
    one(x0, e);
    one(x1, e + 1);
  }
  if (e < e1) one(__ldg(&ikcw[e]), e);
}

// Fast emit of one dense block (staged rows, label masks, no heavy state): per-thread state walks,
// block scan of per-state counts, then per-warp windows of wcap slots staged in shared memory and
// stored coalesced.  Returns the block's arc count.
template <bool kM32, bool kProv, typename Rank, typename StateOut>
__device__ __forceinline__ int emit_block_fast(TaskSmem& s, const ViewDev& Bv, const CompDev& C, int32_t ub0,
                                               int32_t ub1, int lw0, int wpr, const int2* VR, int4* wb4, int wcap,
                                               const uint8_t* __restrict__ cnt8row, int64_t run, Rank&& rank_of,
                                               StateOut&& state_out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int2* __restrict__ ikd = Bv.ikd;
  const int4* __restrict__ ikcw = Bv.ikcw;
  const int32_t* __restrict__ boff = Bv.off;
  const int nub = ub1 - ub0;
  auto present = [&](int slot, int32_t col) -> bool {
    return ((uint32_t)VR[slot * wpr + (col >> 5)].x >> (col & 31)) & 1u;
  };
  // count: states 2t, 2t+1 of thread t; heavy states (> kHeavy arcs) are counted by the whole CTA
  if (threadIdx.x == 0) s.nheavy = 0;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int i = 2 * threadIdx.x + j;
    int c = 0;
    if (i < nub && ((s.fw[lw0 + (i >> 5)] >> (i & 31)) & 1u)) {
      const int32_t ub = ub0 + i;
      const int32_t e = __ldg(&boff[ub]) + ub + 1, e1 = __ldg(&boff[ub + 1]) + ub + 1;
      if (e1 - e > kHeavy) {
        s.state[atomicAdd(&s.nheavy, 1)] = i;
      } else {
        c = cnt8row[ub];  // out-degree in C recorded by the stage-2 fast path (never 255 for <= kHeavy arcs
        if (c == 255)     // unless the count saturated: then count here)
          fast_state<kM32>(s, ikd, ub, e, e1, [&](int slot, int32_t col, int, int, int32_t) { c += present(slot, col); }),
              c -= 255;
      }
    }
    s.cur[i] = c;
  }
  __syncthreads();
  const int nheavy = s.nheavy;
  for (int h = 0; h < nheavy; ++h) {
    const int i = s.state[h];
    const int32_t ub = ub0 + i;
    const int32_t e0 = __ldg(&boff[ub]) + ub + 1, e1 = __ldg(&boff[ub + 1]) + ub + 1;
    int c = 0;
    if (threadIdx.x == 0)
      for (int a = 0; a < s.aeps; ++a) c += present(s.a_slot[a], ub);
    for (int32_t e = e0 + threadIdx.x; e < e1; e += kThreads)
      fast_arc<kM32>(s, __ldg(&ikd[e]), e - ub - 1, [&](int slot, int32_t col, int, int, int32_t) { c += present(slot, col); });
    c = warp_sum(c);
    if (lane == 0 && c) atomicAdd(&s.cur[i], c);
    __syncthreads();
  }
  const int c0 = s.cur[2 * threadIdx.x], c1 = s.cur[2 * threadIdx.x + 1];
  __syncthreads();
  int btot;
  const int ex = block_excl_scan(c0 + c1, s.red32, &btot);
  s.cur[2 * threadIdx.x] = ex;
  s.cur[2 * threadIdx.x + 1] = ex + c0;
  if (threadIdx.x == 0) s.cur[kPairsPerBlock] = btot;
  __syncthreads();
  int32_t* __restrict__ od = C.dst;
  int32_t* __restrict__ oi = C.ilabel;
  int32_t* __restrict__ oo = C.olabel;
  float* __restrict__ ow = C.weight;
  // provenance of the record at slot pos: A arc (A-row position a) unless M3, B arc (view position
  // eb) unless M2, as input arc indices (FST_COMPOSE_PROVENANCE)
  auto prov = [&](int64_t pos, int kind, int a, int32_t eb) {
    __stcs(&C.arc_a[pos], kind != 3 ? __ldg(&C.Af.arc[s.a0 + a]) : -1);
    __stcs(&C.arc_b[pos], kind != 2 ? __ldg(&Bv.arc[eb]) : -1);
  };
  auto fill = [&](int kind, int a, int32_t carry, int32_t wbits, int32_t& il, int32_t& ol, float& wt) {
    if (kind == 1) {
      il = s.a_carry[a];
      ol = carry;
      wt = __fadd_rn(s.a_w[a], __int_as_float(wbits));  // one binary32 add, RN-even
    } else if (kind == 2) {
      il = s.a_carry[a];
      ol = FST_EPS;
      wt = s.a_w[a];  // bit copy
    } else {
      il = FST_EPS;
      ol = carry;
      wt = __int_as_float(wbits);  // bit copy
    }
  };
  for (int r = 0; r < 2; ++r) {
    const int first = warp * 64 + r * 32;
    const int i = first + lane;
    const int32_t ub = ub0 + i;
    const bool has = i < nub && ((s.fw[lw0 + (i >> 5)] >> (i & 31)) & 1u);
    const int q0 = s.cur[first], q1 = s.cur[first + 32];
    const int my0 = s.cur[i], my1 = s.cur[i + 1];
    if (has) state_out(ub, run + my0);
    const int32_t e = has ? __ldg(&boff[ub]) + ub + 1 : 0, e1 = has ? __ldg(&boff[ub + 1]) + ub + 1 : 0;
    const bool walk = has && e1 - e <= kHeavy;  // heavy states are written by the whole CTA below
    for (int win = q0; win < q1; win += wcap) {
      const bool mine = walk && my1 > win && my0 < win + wcap;
      if (!__any_sync(0xffffffffu, mine)) continue;  // window entirely inside a heavy state's range
      if (mine) {
        int p = my0;
        fast_state4<kM32>(s, ikcw, ub, e, e1, [&](int slot, int32_t col, int kind, int a, int32_t carry, int32_t wbits,
                                                 int32_t it) {
          bool pr;
          const int32_t did = rank_of(slot, col, pr);
          if (!pr) return;
          const int t = p - win;
          ++p;
          if ((unsigned)t >= (unsigned)wcap) return;
          int32_t il, ol;
          float wt;
          fill(kind, a, carry, wbits, il, ol, wt);
          wb4[t] = make_int4(did, il, ol, __float_as_int(wt));
          if (kProv) prov(run + win + t, kind, a, it - ub - 1);
        });
      }
      __syncwarp();
      const int n = min(wcap, q1 - win);
      for (int t = lane; t < n; t += 32) {  // slots of heavy states get overwritten below
        const int64_t pos = run + win + t;
        const int4 v = wb4[t];
        __stcs(&od[pos], v.x);
        __stcs(&oi[pos], v.y);
        __stcs(&oo[pos], v.z);
        __stcs(&ow[pos], __int_as_float(v.w));
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int h = 0; h < nheavy; ++h) {  // heavy states: M2 (thread 0), then rounds of kThreads arcs
    const int i = s.state[h];
    const int32_t ub = ub0 + i;
    const int32_t e0 = __ldg(&boff[ub]) + ub + 1, e1 = __ldg(&boff[ub + 1]) + ub + 1;
    int64_t p0 = run + s.cur[i];
    auto put = [&](int slot, int32_t col, int kind, int a, int32_t carry, int32_t wbits, int64_t pos, int32_t eb) {
      bool pr;
      const int32_t did = rank_of(slot, col, pr);
      int32_t il, ol;
      float wt;
      fill(kind, a, carry, wbits, il, ol, wt);
      __stcs(&od[pos], did);
      __stcs(&oi[pos], il);
      __stcs(&oo[pos], ol);
      __stcs(&ow[pos], wt);
      if (kProv) prov(pos, kind, a, eb);
    };
    int m2 = 0;
    for (int a = 0; a < s.aeps; ++a) m2 += present(s.a_slot[a], ub);
    if (threadIdx.x == 0) {
      int64_t q = p0;
      for (int a = 0; a < s.aeps; ++a)
        if (present(s.a_slot[a], ub)) put(s.a_slot[a], ub, 2, a, 0, 0, q++, -1);
    }
    p0 += m2;
    for (int32_t eb = e0; eb < e1; eb += kThreads) {
      const int32_t e = eb + threadIdx.x;
      int4 x = make_int4(0, 0, 0, 0);
      int c = 0;
      if (e < e1) {
        x = __ldg(&ikcw[e]);
        fast_arc<kM32>(s, make_int2(x.x, x.y), 0, [&](int slot, int32_t col, int, int, int32_t) { c += present(slot, col); });
      }
      int tchunk;
      const int exh = block_excl_scan(c, s.red32, &tchunk);
      if (c) {
        int64_t q = p0 + exh;
        fast_arc<kM32>(s, make_int2(x.x, x.y), 0, [&](int slot, int32_t col, int kind, int a, int32_t) {
          if (present(slot, col)) put(slot, col, kind, a, x.z, x.w, q++, e - ub - 1);
        });
      }
      p0 += tchunk;
    }
  }
  return btot;
}


// ceil(2^32 / d) for 2 <= d < 64: floor(c / d) = __umulhi(c, kRecip32[d]) exactly for every batch
// slot c < 32 d + 32 (checked exhaustively for d <= 62)
__constant__ unsigned kRecip32[64] = {0u, 0u, 2147483648u, 1431655766u, 1073741824u, 858993460u, 715827883u, 613566757u, 536870912u, 477218589u, 429496730u, 390451573u, 357913942u, 330382100u, 306783379u, 286331154u, 268435456u, 252645136u, 238609295u, 226050911u, 214748365u, 204522253u, 195225787u, 186737709u, 178956971u, 171798692u, 165191050u, 159072863u, 153391690u, 148102321u, 143165577u, 138547333u, 134217728u, 130150525u, 126322568u, 122713352u, 119304648u, 116080198u, 113025456u, 110127367u, 107374183u, 104755300u, 102261127u, 99882961u, 97612894u, 95443718u, 93368855u, 91382283u, 89478486u, 87652394u, 85899346u, 84215046u, 82595525u, 81037119u, 79536432u, 78090315u, 76695845u, 75350304u, 74051161u, 72796056u, 71582789u, 70409300u, 69273667u, 68174085u};

// Whole-chunk BFS walk (fast path): one thread per source state of the chunk, no per-block barriers.
// kStaged: candidates claimed in the staged NEW bits; else test-and-set on the global bitmaps.
// Per-block kept counts (stage 2) are accumulated warp-aggregated in s.keptc[].
template <bool kStage2, bool kStaged, bool kM32, typename Glob>
__device__ __forceinline__ void bfs_chunk_fast(TaskSmem& s, const ViewDev& Bv, int32_t cub0, int32_t cub1, int nst,
                                               int wpr, const uint32_t* Rs, const uint32_t* VS, uint32_t* NW,
                                               uint8_t* __restrict__ cnt8row, Glob&& glob) {
  const int2* __restrict__ ikd = Bv.ikd;
  const int32_t* __restrict__ off = Bv.off;
  extern __shared__ uint32_t dyn_bfs[];
  uint8_t* dynsm = (uint8_t*)dyn_bfs;
  unsigned kept = 0;
  auto cand = [&](int slot, int32_t col, int, int, int32_t) {
    if (kStaged) {
      const int idx = slot * wpr + (col >> 5);
      const uint32_t bit = 1u << (col & 31);
      if (kStage2) {  // (R word, NEW word) pairs: one 64-bit shared load per candidate
        const uint2 rn = reinterpret_cast<const uint2*>(Rs)[idx];
        if (!(rn.x & bit)) return;
        ++kept;
        if (rn.y & bit) return;  // NEW starts as the visited snapshot
        atomicOr(&NW[2 * idx], bit);
        return;
      }
      if (NW[idx] & bit) return;  // NW starts as the visited snapshot
      atomicOr(&NW[idx], bit);
    } else {
      kept += glob(slot, col);
    }
  };
  if (threadIdx.x == 0) {
    s.nheavy = 0;
    s.segnext = 0;
  }
  if (threadIdx.x < kChunkMaxBlocks) s.keptc[threadIdx.x] = 0ull;
  __syncthreads();
  // Each warp owns 32-word (1024-pair) segments of the chunk: it selects the segment's frontier states
  // 32 at a time (warp scan over the words' popcounts + in-word select, no shared memory, no CTA
  // barrier) and spreads the 32 states' B arcs over its lanes in rounds of 32 (uniform, coalesced
  // packed-item loads).  States with more than kHeavy arcs are deferred to the whole CTA.
  const int lane = threadIdx.x & 31;
  const int nw = (cub1 - cub0 + 31) >> 5;
  constexpr int kSegWords = 8;  // 256-pair segments, handed out dynamically (load balance)
  // stage 2: per-warp kept-move counters of the batch's 32 states, indexed by owner lane (the
  // compacted-state scratch s.state is unused on this path)
  int32_t* cntw = s.state + (threadIdx.x >> 5) * 32;
  if (kStage2) cntw[lane] = 0;
  __syncwarp();
  for (;;) {
    int seg = 0;
    if (lane == 0) seg = atomicAdd(&s.segnext, 1);
    seg = __shfl_sync(0xffffffffu, seg, 0);
    if (seg * kSegWords >= nw) break;
    const int wi = seg * kSegWords + lane;
    const uint32_t word = (lane < kSegWords && wi < nw) ? s.fw[wi] : 0u;
    const int pc = __popc(word);
    const int winc = warp_incl_scan(pc);
    const int wex = winc - pc;
    const int stot = __shfl_sync(0xffffffffu, winc, 31);
    unsigned long long segkept = 0;
    for (int b0 = 0; b0 < stot; b0 += 32) {
      const int k = b0 + lane;
      int j = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1)
        if (__shfl_sync(0xffffffffu, wex, j + step) <= k) j += step;
      uint32_t wj = __shfl_sync(0xffffffffu, word, j);
      int r = k - __shfl_sync(0xffffffffu, wex, j);
      int32_t ub = 0, e = 0, deg = 0;
      if (k < stot) {
        int pos = 0;  // r-th set bit of wj (binary search on popcounts)
#pragma unroll
        for (int h = 16; h > 0; h >>= 1) {
          const int c = __popc(wj & ((1u << h) - 1u));
          if (r >= c) {
            r -= c;
            pos += h;
            wj >>= h;
          }
        }
        ub = cub0 + (seg * kSegWords + j) * 32 + pos;
        e = __ldg(&off[ub]) + ub + 1;
        deg = __ldg(&off[ub + 1]) + ub + 1 - e;
        kept = 0;
        for (int a = 0; a < s.aeps; ++a) cand(s.a_slot[a], ub, 2, a, -1);  // M2 moves of the state
        segkept += kept;
        if (deg > kHeavy) {
          const int hh = atomicAdd(&s.nheavy, 1);
          if (hh < kPairsPerBlock) {
            s.cur[hh] = ub;
            deg = 0;
          }
        }
      }
      int own_cnt = kept;  // stage 2: kept moves (= out-degree in C) of my own state
      const bool heavy_own = k < stot && deg == 0 && __ldg(&off[ub + 1]) - __ldg(&off[ub]) > kHeavy;
      if (__reduce_max_sync(0xffffffffu, (unsigned)deg) <= 2u) {
        // low-degree batch (e.g. a lexicon trie): every lane walks its own state's <= 2 arcs
        const int2 x0 = deg > 0 ? __ldg(&ikd[e]) : make_int2(0, 0);
        const int2 x1 = deg > 1 ? __ldg(&ikd[e + 1]) : make_int2(0, 0);
        kept = 0;
        if (deg > 0) fast_arc<kM32>(s, x0, e - ub - 1, cand);
        if (deg > 1) fast_arc<kM32>(s, x1, e - ub, cand);
        segkept += kept;
        if (kStage2 && k < stot) cnt8row[ub] = (uint8_t)(heavy_own ? 255 : min(own_cnt + (int)kept, 255));
        continue;
      }
      const int incl = warp_incl_scan(deg);
      const int start = incl - deg;
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      kept = 0;
      // arc slot -> owner lane: a per-warp byte table when the batch is small enough, else a
      // binary search over the lanes' start offsets
      // (uniform degree d <= 62 over the batch's states, e.g. random graphs: owner = floor(c / d) as
      // the high word of c * ceil(2^32 / d), exact for the slots c < 32 d + 32 <= 2016 of a batch)
      const unsigned dmax = __reduce_max_sync(0xffffffffu, (unsigned)deg);
      const unsigned dmin = __reduce_min_sync(0xffffffffu, k < stot ? (unsigned)deg : dmax);
      // (dmax >= 2: kRecip32[d] = ceil(2^32 / d) does not fit 32 bits for d = 1; batches with d <= 2
      // take the low-degree branch above anyway, this keeps the lookup valid on its own)
      const bool uni = dmax == dmin && dmax >= 2u && dmax <= 62u;
      const unsigned uinv = uni ? kRecip32[dmax] : 0u;
      uint8_t* own = dynsm + (kDynSmem - kOwnerBytes) + (threadIdx.x >> 5) * kOwnerCap;
      const bool tbl = !uni && total <= kOwnerCap;
      if (tbl)
        for (int p = start; p < incl; ++p) own[p] = (uint8_t)lane;
      __syncwarp();
      auto owner_of = [&](int c) -> int {
        if (uni) return c < total ? (int)__umulhi((unsigned)c, uinv) : 0;
        if (tbl) return c < total ? own[c] : 0;
        int jj = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1)
          if (__shfl_sync(0xffffffffu, start, jj + step) <= c) jj += step;
        return jj;
      };
      int jn = owner_of(lane);
      int32_t en = __shfl_sync(0xffffffffu, e, jn) + (lane - __shfl_sync(0xffffffffu, start, jn));
      int32_t un = __shfl_sync(0xffffffffu, ub, jn);
      int2 xn = lane < total ? __ldg(&ikd[en]) : make_int2(0, 0);
      for (int rr = 0; rr < total; rr += 32) {
        const int c = rr + lane;
        const int32_t ej = en, uj = un;
        const int jc = jn;  // owner lane of this round's item
        const int2 xc = xn;
        if (rr + 32 < total) {  // prefetch the next round's item
          const int cn = c + 32;
          jn = owner_of(cn);
          en = __shfl_sync(0xffffffffu, e, jn) + (cn - __shfl_sync(0xffffffffu, start, jn));
          un = __shfl_sync(0xffffffffu, ub, jn);
          if (cn < total) xn = __ldg(&ikd[en]);
        }
        const unsigned k0 = kept;
        if (c < total) fast_arc<kM32>(s, xc, ej - uj - 1, cand);
        if (kStage2 && kept != k0) atomicAdd(&cntw[jc], (int)(kept - k0));  // credit the owner state
      }
      segkept += kept;
      __syncwarp();
      if (kStage2) {
        if (k < stot) cnt8row[ub] = (uint8_t)(heavy_own ? 255 : min(own_cnt + cntw[lane], 255));
        cntw[lane] = 0;
        __syncwarp();
      }
    }
    if (kStage2) {  // the segment lies inside one 1024-pair block
      const unsigned long long t = warp_sum(segkept);
      if (lane == 0 && t) atomicAdd(&s.keptc[seg / (32 / kSegWords)], t);
    }
  }
  __syncthreads();
  const int nh = min(s.nheavy, kPairsPerBlock);
  for (int h = 0; h < nh; ++h) {
    const int32_t ub = s.cur[h];
    const int32_t e0 = __ldg(&off[ub]) + ub + 1, e1 = __ldg(&off[ub + 1]) + ub + 1;
    kept = 0;
    // 4 coalesced item loads in flight per thread (a lexicon root has ~10^4 arcs: 20 dependent
    // rounds of 512 would sit on the level's critical path)
    constexpr int kHU = 4;
    for (int32_t e = e0 + threadIdx.x; e < e1; e += kHU * kThreads) {
      int2 x[kHU];
#pragma unroll
      for (int u = 0; u < kHU; ++u) x[u] = e + u * kThreads < e1 ? __ldg(&ikd[e + u * kThreads]) : make_int2(0, 0);
#pragma unroll
      for (int u = 0; u < kHU; ++u)
        if (e + u * kThreads < e1) fast_arc<kM32>(s, x[u], e + u * kThreads - ub - 1, cand);
    }
    if (kStage2) {
      const unsigned long long k = warp_sum((unsigned long long)kept);
      if ((threadIdx.x & 31) == 0 && k) atomicAdd(&s.keptc[(ub - cub0) >> 10], k);
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------------------------ seeds
template <bool kStage2>
__global__ void k_seed(Ctx cx) {
  const int64_t total = cx.seedbase[cx.ncomp];
  uint32_t* vis = kStage2 ? cx.V : cx.R;
  unsigned nnew = 0;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = cx.ncomp - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (cx.seedbase[mid] <= g) lo = mid; else hi = mid - 1;
    }
    const CompDev& C = cx.comps[lo];
    int64_t i = g - cx.seedbase[lo];
    int32_t nb = kStage2 ? C.nStartB : C.nAccB;
    int32_t va = kStage2 ? C.startListA[i / nb] : C.accListA[i / nb];
    int32_t vb = kStage2 ? C.startListB[i % nb] : C.accListB[i % nb];
    if (!owned(C, va, vb)) continue;  // sharded: another shard seeds it
    const int64_t gw = C.W + (int64_t)va * C.wpr + (vb >> 5);
    const uint32_t bit = 1u << (vb & 31);
    if (kStage2 && !(cx.R[gw] & bit)) continue;
    if (atomicOr(&vis[gw], bit) & bit) continue;
    ++nnew;
    push_bits(C, va, vb, gw, bit, cx.F0, cx.flag0, cx.list0, &cx.ctrl[0]);
  }
  nnew = warp_sum(nnew);
  if ((threadIdx.x & 31) == 0 && nnew) atomicAdd(&cx.ctrl[0].nnew, (unsigned long long)nnew);
}

// ------------------------------------------------------------------------------ bottom-up level (stage 1)
// Direction-optimising BFS (pull): once the frontier is at least as large as the set of pairs not yet
// in R, a level costs less as "every unvisited pair looks for ONE forward move into R" than as "every
// frontier pair enumerates all its predecessors".  R is a set, so a pair may be claimed as soon as
// any successor is in R (at most one level early): the final R is the same set (Alg. 1 line 3).  A
// CTA owns row u_a of a chunk: it consumes the chunk's frontier words (pull does not read them), stages
// the R words of the destination rows {dst(e_a)} U {u_a} of A's OUT-view, walks the chunk's unvisited
// pairs (one lane per pair, early exit) over B's out-items, and ORs the new bits into its own row of R
// and into the next frontier -- no other task writes that row during a pull level.
// pull iff frontier * pull_num >= unvisited * 4 AND frontier >= pairs / 16 (the level scans every
// chunk of the pair space, so the frontier must be a sizable share of it: never on trellis levels)

__device__ __forceinline__ void level_pull(const Ctx& cx, TaskSmem& s, uint32_t* dyn, uint32_t* Fc, uint32_t* Fn,
                                           uint32_t* flagc, uint32_t* flagn, int32_t* listn, LevelCtrl* ctrl_nxt,
                                           unsigned& nnew) {
  const int lane = threadIdx.x & 31;
  for (int64_t q = blockIdx.x; q < cx.nchunks; q += gridDim.x) {
    const Chunk ch = decode_chunk(cx, q);
    const CompDev& C = cx.comps[ch.comp];
    const ViewDev& Av = C.Af;
    const ViewDev& Bv = C.Bf;
    const int wpr = C.wpr;
    if (threadIdx.x == 0) flagc[q] = 0u;
    // unvisited pairs of the chunk -> s.fw; the chunk's frontier words are consumed
    const int w0 = ch.b0 * 32, w1 = min(ch.b1 * 32, wpr);
    int cnt = 0;
    for (int w = w0 + threadIdx.x; w < w1; w += kThreads) {
      const int64_t gw = ch.rowW + w;
      if (Fc[gw]) Fc[gw] = 0u;
      uint32_t x = ~cx.R[gw];
      if (w == wpr - 1 && (C.VB & 31)) x &= (1u << (C.VB & 31)) - 1u;  // columns beyond V_B
      s.fw[w - w0] = x;
      cnt += __popc(x);
    }
    cnt = warp_sum(cnt);
    if (lane == 0) s.red32[threadIdx.x >> 5] = cnt;
    __syncthreads();
    int tot = 0;
    for (int i = 0; i < kWarps; ++i) tot += s.red32[i];
    __syncthreads();
    if (tot == 0) continue;
    const int nwc = w1 - w0;
    uint32_t* NEWW = dyn + ((kDynSmem / 4) - kChunkMaxBlocks * 32);  // claimed bits of the chunk
    stage_arow(s, C, Av, ch.ua, wpr, (kDynSmem / 4) - kChunkMaxBlocks * 32);
    const bool staged = s.dst_staged;
    uint32_t* RS = dyn;  // R words of the destination rows (slot-major)
    for (int i = threadIdx.x; i < nwc; i += kThreads) NEWW[i] = 0u;
    if (staged) {
      const int n = s.m * wpr;
      for (int i = threadIdx.x; i < n; i += kThreads) {
        const int r = i / wpr, w = i - r * wpr;
        RS[i] = cx.R[C.W + (int64_t)s.slot_row[r] * wpr + w];
      }
    }
    __syncthreads();
    const bool fastp = staged && s.small;
    auto in_r = [&](const Cand& c) -> bool {
      const uint32_t bit = 1u << (c.col & 31);
      if (staged && c.slot >= 0) return RS[c.slot * wpr + (c.col >> 5)] & bit;
      return __ldg(&cx.R[C.W + (int64_t)c.row * wpr + (c.col >> 5)]) & bit;
    };
    // warps take 8-word segments; lanes take the segment's unvisited pairs 32 at a time
    if (threadIdx.x == 0) s.segnext = 0;
    __syncthreads();
    constexpr int kSegWords = 8;
    for (;;) {
      int seg = 0;
      if (lane == 0) seg = atomicAdd(&s.segnext, 1);
      seg = __shfl_sync(0xffffffffu, seg, 0);
      if (seg * kSegWords >= nwc) break;
      const int wi = seg * kSegWords + lane;
      const uint32_t word = (lane < kSegWords && wi < nwc) ? s.fw[wi] : 0u;
      const int pc = __popc(word);
      const int winc = warp_incl_scan(pc);
      const int wex = winc - pc;
      const int stot = __shfl_sync(0xffffffffu, winc, 31);
      for (int b0 = 0; b0 < stot; b0 += 32) {
        const int k = b0 + lane;
        int j = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1)
          if (__shfl_sync(0xffffffffu, wex, j + step) <= k) j += step;
        uint32_t wj = __shfl_sync(0xffffffffu, word, j);
        int r = k - __shfl_sync(0xffffffffu, wex, j);
        if (k >= stot) continue;
        int pos = 0;
#pragma unroll
        for (int h = 16; h > 0; h >>= 1) {
          const int c = __popc(wj & ((1u << h) - 1u));
          if (r >= c) {
            r -= c;
            pos += h;
            wj >>= h;
          }
        }
        const int lw = seg * kSegWords + j;  // chunk-local word
        const int32_t ub = (w0 + lw) * 32 + pos;
        // forward moves of (u_a, ub): the sentinel item (M2) then its B arcs (M1, M3), early exit
        // (the sentinel carries only M2 moves: skipped when the A row has no eps outputs)
        bool hit = false;
        if (fastp) {  // label-mask rows with staged destination rows: direct bit tests
          const uint32_t ubit = 1u << (ub & 31);
          for (int a = 0; a < s.aeps && !hit; ++a) hit = RS[s.a_slot[a] * wpr + (ub >> 5)] & ubit;  // M2
          const int32_t i0 = __ldg(&Bv.off[ub]) + ub + 1, i1 = __ldg(&Bv.off[ub + 1]) + ub + 1;
          int2 kn = i0 < i1 ? __ldg(&Bv.ikd[i0]) : make_int2(0, 0);
          for (int32_t it = i0; it < i1 && !hit; ++it) {
            const int2 kd = kn;
            if (it + 1 < i1) kn = __ldg(&Bv.ikd[it + 1]);  // next item in flight while this one is tested
            const int cw = kd.y >> 5;
            const uint32_t cbit = 1u << (kd.y & 31);
            unsigned long long m = (unsigned)(kd.x + 1) < 64u ? s.labmask[kd.x + 1] : 0ull;
            while (m && !hit) {  // M1
              const int a = __ffsll((long long)m) - 1;
              m &= m - 1;
              hit = RS[s.a_slot[a] * wpr + cw] & cbit;
            }
            if (kd.x == FST_EPS && !hit) hit = RS[cw] & cbit;  // M3: slot 0 = u_a
          }
        } else {
          // (the sentinel carries only M2 moves: skipped when the A row has no eps outputs)
          const int32_t i0 = __ldg(&Bv.off[ub]) + ub + (s.aeps == 0 ? 1 : 0), i1 = __ldg(&Bv.off[ub + 1]) + ub + 1;
          int2 kn = i0 < i1 ? __ldg(&Bv.ikd[i0]) : make_int2(0, 0);
          for (int32_t it = i0; it < i1 && !hit; ++it) {
            const int2 kd = kn;
            if (it + 1 < i1) kn = __ldg(&Bv.ikd[it + 1]);
            const Item x = make_item(s, Av, it, ub, kd, true);
            for (int m = 0; m < x.n && !hit; ++m) hit = in_r(item_move(s, Av, ch.ua, x, m));
          }
        }
        if (hit) atomicOr(&NEWW[lw], 1u << pos);
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nwc; i += kThreads) {  // own row: plain OR into R, then the frontier
      const uint32_t nb = NEWW[i];
      if (!nb) continue;
      const int64_t gw = ch.rowW + w0 + i;
      cx.R[gw] |= nb;
      nnew += __popc(nb);
      push_bits(C, ch.ua, (w0 + i) * 32, gw, nb, Fn, flagn, listn, ctrl_nxt);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------ one BFS level
// kStage2 = false: backward BFS over in-views, visited set R.
// kStage2 = true : forward BFS over out-views, filter R, visited set V, per-block kept counts.
template <bool kStage2>
__global__ void __launch_bounds__(kThreads, 2) k_level(Ctx cx, int level) {
  __shared__ TaskSmem s;
  extern __shared__ uint32_t dyn[];
  const int p = level & 1;
  LevelCtrl* ctrl_cur = &cx.ctrl[level % 3];
  LevelCtrl* ctrl_nxt = &cx.ctrl[(level + 1) % 3];
  uint32_t* Fc = p ? cx.F1 : cx.F0;
  uint32_t* Fn = p ? cx.F0 : cx.F1;
  uint32_t* flagc = p ? cx.flag1 : cx.flag0;
  uint32_t* flagn = p ? cx.flag0 : cx.flag1;
  const int32_t* listc = p ? cx.list1 : cx.list0;
  int32_t* listn = p ? cx.list0 : cx.list1;
  uint32_t* vis = kStage2 ? cx.V : cx.R;
  const unsigned long long nlist = *((volatile unsigned long long*)&ctrl_cur->count);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    LevelCtrl* z = &cx.ctrl[(level + 2) % 3];
    z->count = 0;
    z->nnew = 0;
    int hl = level;  // graph-driven loop: `level` is only right modulo 6 (ring phase); the true level
    if (cx.level_dev) {  // number lives in device memory and is advanced here
      hl = *cx.level_dev;
      *cx.level_dev = hl + 1;
    }
    if (nlist) {
      cx.misc[0] += 1;
      if (hl < kMaxLevelStats) cx.hist[hl] = ctrl_cur->nnew;
    }
    ctrl_nxt->pad[0] = ctrl_cur->pad[0] + ctrl_cur->nnew;  // pairs visited through this level's frontier
  }
  unsigned nnew = 0;
  if (!kStage2 && cx.pull_ok && nlist) {  // uniform decision: inputs fixed before this launch
    const unsigned long long nf = ctrl_cur->nnew;
    const unsigned long long visited = ctrl_cur->pad[0] + nf;
    const unsigned long long unvisited = (unsigned long long)cx.ptotal > visited ? cx.ptotal - visited : 0ull;
    if (nf * (unsigned long long)cx.pull_num >= unvisited * 4ull && nf * 16ull >= (unsigned long long)cx.ptotal) {
      level_pull(cx, s, dyn, Fc, Fn, flagc, flagn, listn, ctrl_nxt, nnew);
      nnew = warp_sum(nnew);
      if ((threadIdx.x & 31) == 0 && nnew) atomicAdd(&ctrl_nxt->nnew, (unsigned long long)nnew);
      return;
    }
  }
  // narrow levels (fewer active chunks than CTAs, e.g. a trellis A with one row per level): split
  // every chunk into `split` block ranges so the whole grid works on the level
  const unsigned split = nlist == 0 ? 1u : (unsigned)max(1ull, min((unsigned long long)kChunkMaxBlocks, gridDim.x / nlist));
  for (unsigned long long e = blockIdx.x; e < nlist * split; e += gridDim.x) {
    const int64_t q = listc[e / split];
    Chunk ch = decode_chunk(cx, q);
    if (split > 1) {
      const int sub = (int)(e % split), per = (ch.b1 - ch.b0 + (int)split - 1) / (int)split;
      ch.b0 += sub * per;
      ch.b1 = min(ch.b1, ch.b0 + per);
      if (ch.b0 >= ch.b1) continue;
    }
    const CompDev& C = cx.comps[ch.comp];
    const ViewDev& Av = kStage2 ? C.Af : C.Ab;
    const ViewDev& Bv = kStage2 ? C.Bf : C.Bb;
    if (threadIdx.x == 0) flagc[q] = 0u;
    const int nst = load_chunk_bits(s, Fc, C, ch, true);
    if (nst == 0) continue;
    const int wpr = C.wpr;
    const int per_word = kStage2 ? 3 : 2;  // R, V-snapshot, NEW  |  R-snapshot, NEW
    stage_arow(s, C, Av, ch.ua, per_word * wpr, (kDynSmem - kOwnerBytes) / 4);
    // stage destination rows only when the chunk has enough work to amortise the staging traffic
    const bool staged = s.dst_staged && (int64_t)nst * 16 >= (int64_t)s.m * wpr;
    // stage 2: (R, NEW) word pairs interleaved, then the V snapshot; stage 1: R snapshot, then NEW.
    // NEW word of pair-word i: NW[kNS * i].
    constexpr int kNS = kStage2 ? 2 : 1;
    uint32_t* Rs = dyn;
    uint32_t* VS = kStage2 ? dyn + 2 * s.m * wpr : dyn;
    uint32_t* NW = kStage2 ? dyn + 1 : VS + s.m * wpr;
    if (staged) {
      const int n = s.m * wpr;
      for (int i0 = threadIdx.x; i0 < n; i0 += 4 * kThreads) {  // 4 independent loads in flight per thread
        uint32_t v[4], rv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * kThreads;
          v[u] = rv[u] = 0u;
          if (i < n) {
            const int r = i / wpr, w = i - r * wpr;
            const int64_t gw = C.W + (int64_t)s.slot_row[r] * wpr + w;
            v[u] = kStage2 ? cx.V[gw] : cx.R[gw];
            if (kStage2) rv[u] = __ldg(&cx.R[gw]);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * kThreads;
          if (i < n) {
            if (kStage2) Rs[2 * i] = rv[u];
            VS[i] = v[u];
            NW[kNS * i] = v[u];  // claims accumulate on top of the snapshot
          }
        }
      }
      __syncthreads();
    }
    unsigned kept = 0;
    auto sink = [&](bool act, const Cand& c, int) {
      if (!act) return;
      const uint32_t bit = 1u << (c.col & 31);
      if (staged) {
        const int i = c.slot * wpr + (c.col >> 5);
        if (kStage2) {
          if (!(Rs[2 * i] & bit)) return;
          ++kept;
        }
        if (NW[kNS * i] & bit) return;  // NEW starts as the visited snapshot
        atomicOr(&NW[kNS * i], bit);
      } else {
        const int64_t gw = C.W + (int64_t)c.row * wpr + (c.col >> 5);
        if (kStage2) {
          if (!(__ldg(&cx.R[gw]) & bit)) return;
          ++kept;
        }
        if (!owned(C, c.row, c.col)) {  // sharded: the owner claims it after the exchange
          atomicOr(&cx.OUT[gw], bit);
          return;
        }
        if (vis[gw] & bit) return;  // test before the atomic (bits only get set)
        if (atomicOr(&vis[gw], bit) & bit) return;
        ++nnew;
        push_bits(C, c.row, c.col, gw, bit, Fn, flagn, listn, ctrl_nxt);
      }
    };
    if (s.small) {  // fast path: compacted source states, one thread per state
      const int32_t cub0 = ch.b0 * kPairsPerBlock, cub1 = min(ch.b1 * kPairsPerBlock, C.VB);
      uint8_t* cnt8row = cx.cnt8 + ch.rowW * 32;
      auto glob = [&](int slot, int32_t col) -> unsigned {
        const int32_t row = s.slot_row[slot];
        const int64_t gw = C.W + (int64_t)row * wpr + (col >> 5);
        const uint32_t bit = 1u << (col & 31);
        unsigned k = 0;
        if (kStage2) {
          if (!(__ldg(&cx.R[gw]) & bit)) return 0u;
          k = 1;
        }
        if (!owned(C, row, col)) {  // sharded: the owner claims it after the exchange
          atomicOr(&cx.OUT[gw], bit);
          return k;
        }
        if (vis[gw] & bit) return k;
        if (atomicOr(&vis[gw], bit) & bit) return k;
        ++nnew;
        push_bits(C, row, col, gw, bit, Fn, flagn, listn, ctrl_nxt);
        return k;
      };
      if (staged) {
        if (s.mask32) bfs_chunk_fast<kStage2, true, true>(s, Bv, cub0, cub1, nst, wpr, Rs, VS, NW, cnt8row, glob);
        else bfs_chunk_fast<kStage2, true, false>(s, Bv, cub0, cub1, nst, wpr, Rs, VS, NW, cnt8row, glob);
      } else {
        if (s.mask32) bfs_chunk_fast<kStage2, false, true>(s, Bv, cub0, cub1, nst, wpr, Rs, VS, NW, cnt8row, glob);
        else bfs_chunk_fast<kStage2, false, false>(s, Bv, cub0, cub1, nst, wpr, Rs, VS, NW, cnt8row, glob);
      }
      if (kStage2 && (int)threadIdx.x < ch.b1 - ch.b0 && s.keptc[threadIdx.x])
        cx.kept[C.K + (int64_t)ch.ua * C.bpr + ch.b0 + threadIdx.x] += s.keptc[threadIdx.x];
    }
    if (!s.small) {
      build_groups(s, Bv);
      __syncthreads();
    }
    for (int32_t blk = s.small ? ch.b1 : ch.b0; blk < ch.b1; ++blk) {
      kept = 0;
      const int32_t ub0 = blk * kPairsPerBlock, ub1 = min(ub0 + kPairsPerBlock, C.VB);
      const int lw0 = (blk - ch.b0) * 32;
      const int nb = block_popc(s, C, ch, blk);
      if (nb == 0) continue;
      if (s.G != 0 && nb * 4 >= ub1 - ub0) {
        // dense block, label-major: only B arcs whose label occurs in the A row
        const int total = block_groups(s, Bv, ub0, ub1);
        if (s.aeps > 0) {  // M2 moves of every source state
          for (int32_t ub = ub0 + threadIdx.x; ub < ub1; ub += kThreads)
            if (src_bit(s, lw0, ub0, ub))
              for (int a = 0; a < s.aeps; ++a) sink(true, Cand{s.a_slot[a], s.a_other[a], ub, 2, a, -1}, 0);
        }
        for (int i = threadIdx.x; i < total; i += kThreads) {
          const int g = item_group(s, i);
          const int32_t sid = s.g_lo[g] + (i - s.g_pre[g]);
          const int32_t ub = __ldg(&Bv.seg_node[sid]);
          if (!src_bit(s, lw0, ub0, ub)) continue;
          const int32_t e0 = __ldg(&Bv.seg_beg[sid]), e1 = __ldg(&Bv.seg_beg[sid + 1]);
          const unsigned long long gm = s.g_mask[g];
          const bool eps = s.g_label[g] == FST_EPS;
          for (int32_t j = e0; j < e1; ++j) {
            const int32_t ob = __ldg(&Bv.lm_other[j]);
            for (unsigned long long m = gm; m; m &= m - 1) {
              const int a = __ffsll((long long)m) - 1;
              sink(true, Cand{s.a_slot[a], s.a_other[a], ob, 1, a, -1}, 0);
            }
            if (eps) sink(true, Cand{0, ch.ua, ob, 3, -1, -1}, 0);
          }
        }
        __syncthreads();
      } else
      for_block_items(s, Bv, C, ch, blk, [&](bool valid, int32_t it, int32_t ub, int2 kd) {
        const Item x = make_item(s, Av, it, ub, kd, valid);
        const int maxn = __reduce_max_sync(0xffffffffu, (unsigned)x.n);
        if (maxn <= kSimpleMoves) {  // few moves per item: every lane walks its own
          for (int k = 0; k < maxn; ++k)
            if (k < x.n) sink(true, item_move(s, Av, ch.ua, x, k), 0);
        } else {
          warp_expand(s, Av, ch.ua, x, sink);
        }
      });
      if (kStage2) {  // pass-1 arc count of this block
        if (threadIdx.x == 0) s.keptb = 0ull;
        __syncthreads();
        unsigned long long k = warp_sum((unsigned long long)kept);
        if ((threadIdx.x & 31) == 0 && k) atomicAdd(&s.keptb, k);
        __syncthreads();
        if (threadIdx.x == 0 && s.keptb) cx.kept[C.K + (int64_t)ch.ua * C.bpr + blk] += s.keptb;
        __syncthreads();
      }
    }
    if (staged) {  // merge the claimed bits into the global visited / frontier bitmaps
      __syncthreads();
      const int m = s.m;
      for (int i = threadIdx.x; i < m * wpr; i += kThreads) {
        const uint32_t nb = NW[kNS * i] & ~VS[i];
        if (!nb) continue;
        const int r = i / wpr, w = i - r * wpr;
        const int32_t row = s.slot_row[r];
        const int64_t gw = C.W + (int64_t)row * wpr + w;
        if (!owned(C, row, w * 32)) {  // sharded: the owner claims it after the exchange
          atomicOr(&cx.OUT[gw], nb);
          continue;
        }
        const uint32_t win = nb & ~atomicOr(&vis[gw], nb);
        if (win) {
          nnew += __popc(win);
          push_bits(C, row, w * 32, gw, win, Fn, flagn, listn, ctrl_nxt);
        }
      }
      if (threadIdx.x == 0) atomicAdd(&cx.misc[3], 1ull);
    }
    __syncthreads();
  }
  nnew = warp_sum(nnew);
  if ((threadIdx.x & 31) == 0 && nnew) atomicAdd(&ctrl_nxt->nnew, (unsigned long long)nnew);
}

// ------------------------------------------------------------------------------ sharded exchange
// Owner-side claim of the pairs other shards found in this shard's blocks during level `level` (their
// OUT bits): new bits become visited and join the next frontier exactly like local claims.  `in` is
// either the sender's whole OUT bitmap (in-process shards) or a PACKED slice: this rank's blocks in
// order (block id rank, rank + world, ...), 32 words each.  Single composition (ncomp == 1).
template <bool kStage2>
__global__ void k_apply_remote(Ctx cx, const uint32_t* __restrict__ in, int packed, int level) {
  const int p = level & 1;
  LevelCtrl* ctrl_nxt = &cx.ctrl[(level + 1) % 3];
  uint32_t* Fn = p ? cx.F0 : cx.F1;
  uint32_t* flagn = p ? cx.flag0 : cx.flag1;
  int32_t* listn = p ? cx.list0 : cx.list1;
  uint32_t* vis = kStage2 ? cx.V : cx.R;
  const CompDev& C = cx.comps[0];
  const int me = C.sh_rank;
  const int64_t mine = owner_nblocks(C, me);
  unsigned nnew = 0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < mine * 32; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t blk = owner_block(C, me, t >> 5);
    const int32_t row = (int32_t)(blk / C.bpr), j = (int32_t)(blk - (int64_t)row * C.bpr);
    const int w = j * 32 + (int)(t & 31);
    if (w >= C.wpr) continue;
    const int64_t gw = C.W + (int64_t)row * C.wpr + w;
    const uint32_t nbits = packed ? in[t] : in[gw];
    if (!nbits) continue;
    const uint32_t win = nbits & ~atomicOr(&vis[gw], nbits);
    if (!win) continue;
    nnew += __popc(win);
    push_bits(C, row, w * 32, gw, win, Fn, flagn, listn, ctrl_nxt);
  }
  nnew = warp_sum(nnew);
  if ((threadIdx.x & 31) == 0 && nnew) atomicAdd(&ctrl_nxt->nnew, (unsigned long long)nnew);
}

// Packs rank q's blocks of a bitmap (block id q, q + world, ...; 32 words each, zero-padded) into dst.
__global__ void k_pack_owner(const CompDev* __restrict__ comp, const uint32_t* __restrict__ bits, int q,
                             uint32_t* __restrict__ dst) {
  const CompDev& C = comp[0];
  const int64_t n = owner_nblocks(C, q);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n * 32; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t blk = owner_block(C, q, t >> 5);
    const int32_t row = (int32_t)(blk / C.bpr), j = (int32_t)(blk - (int64_t)row * C.bpr);
    const int w = j * 32 + (int)(t & 31);
    dst[t] = w < C.wpr ? bits[C.W + (int64_t)row * C.wpr + w] : 0u;
  }
}

// In-process shards: dst gets, for every word, the copy of its block's owner (replication of R / V).
struct ShardPtrs {
  const uint32_t* p[16];
};
__global__ void k_gather_owned(const CompDev* __restrict__ comp, ShardPtrs src, uint32_t* __restrict__ dst) {
  const CompDev& C = comp[0];
  const int64_t n = (int64_t)C.VA * C.wpr;
  for (int64_t gw = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gw < n; gw += (int64_t)gridDim.x * blockDim.x) {
    const int32_t row = (int32_t)(gw / C.wpr), w = (int32_t)(gw - (int64_t)row * C.wpr);
    const int q = blk_owner(C, (int64_t)row * C.bpr + (w >> 5));
    if (src.p[q] != dst) dst[gw] = src.p[q][gw];
  }
}
struct ShardPtrs64 {
  const unsigned long long* p[16];
};
__global__ void k_gather_owned_blocks(const CompDev* __restrict__ comp, ShardPtrs64 src,
                                      unsigned long long* __restrict__ dst) {
  const CompDev& C = comp[0];
  const int64_t nblocks = (int64_t)C.VA * C.bpr;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nblocks; b += (int64_t)gridDim.x * blockDim.x) {
    const int q = blk_owner(C, b);
    if (src.p[q] != dst) dst[b] = src.p[q][b];
  }
}

// NCCL replication of a bitmap: every rank keeps only the words of its own blocks, then an all-reduce
// (sum of disjoint bits = OR) gives every rank the whole bitmap.
__global__ void k_mask_unowned(const CompDev* __restrict__ comp, uint32_t* __restrict__ bits) {
  const CompDev& C = comp[0];
  const int64_t n = (int64_t)C.VA * C.wpr;
  for (int64_t gw = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gw < n; gw += (int64_t)gridDim.x * blockDim.x) {
    const int32_t row = (int32_t)(gw / C.wpr), w = (int32_t)(gw - (int64_t)row * C.wpr);
    if (!owned(C, row, w * 32) && bits[gw]) bits[gw] = 0u;
  }
}

// Owner-major numbering of a sharded composition: per-block values in the order (owner, block id)
// -- rank q's blocks q, q + G, ... are positions [start_q, start_q + n_q) -- so every shard's states
// and arcs are one contiguous range of ids / slots (the shards concatenate into the whole CSR).
__device__ __forceinline__ int64_t om_pos(int64_t blk, int64_t nb, int G) {  // block-interleaved mode
  if (G <= 1) return blk;  // (rows mode passes G = 1: owner-major order is block order)
  const int64_t q = blk % G, base = nb / G, rem = nb % G;
  return q * base + min(q, rem) + blk / G;
}
template <typename T>
__global__ void k_om_gather(const T* __restrict__ in, int64_t nb, int G, T* __restrict__ out) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x)
    out[om_pos(b, nb, G)] = in[b];
}
__global__ void k_om_scatter(const int64_t* __restrict__ scanned, int64_t nb, int G, int64_t* __restrict__ out) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= nb; b += (int64_t)gridDim.x * blockDim.x)
    out[b] = b < nb ? scanned[om_pos(b, nb, G)] : scanned[nb];
}

__global__ void k_shift_i64(int64_t* __restrict__ a, int64_t n, int64_t d) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] -= d;
}

// ------------------------------------------------------------------------------ numbering
// One warp per block: vcount[blk] = popcount of V in the block; wpre[word] = exclusive prefix.
__global__ void k_block_counts(Ctx cx) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t blk = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); blk < cx.nblocks; blk += warps) {
    int c = cx.ncomp == 1 ? 0 : find_comp(cx.comps, cx.ncomp, blk);
    const CompDev& C = cx.comps[c];
    const int64_t local = blk - C.K;
    const int32_t ua = (int32_t)(local / C.bpr);
    const int32_t j = (int32_t)(local - (int64_t)ua * C.bpr);
    const int nw = min(32, C.wpr - j * 32);
    const int64_t w0 = C.W + (int64_t)ua * C.wpr + (int64_t)j * 32;
    uint32_t w = lane < nw ? cx.V[w0 + lane] : 0u;
    int pc = __popc(w);
    int inc = warp_incl_scan(pc);
    if (lane < nw) cx.wpre[w0 + lane] = (uint16_t)(inc - pc);
    if (lane == 31) cx.vcount[blk] = inc;
    if (cx.warc) {  // tile path: arc offset of each word inside its block
      const uint32_t a = lane < nw ? cx.warc[w0 + lane] : 0u;
      const uint32_t ai = warp_incl_scan(a);
      if (lane < nw) cx.warc[w0 + lane] = ai - a;
    }
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
// weight).  Per round of kThreads items: phase 1 counts each warp's kept moves, a CTA prefix over
// the warp totals gives every warp its slot base, phase 2 re-expands and writes the kept moves at
// consecutive slots (warp ballots; coalesced streaming stores).  Slots = block arc base + running
// prefix in (state, item, match) order: deterministic, no cursor atomics.
__global__ void __launch_bounds__(kThreads, 2) k_emit(Ctx cx, const int64_t* __restrict__ tot) {
  __shared__ TaskSmem s;
  extern __shared__ uint32_t dyn[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t q = blockIdx.x; q < cx.nchunks; q += gridDim.x) {
    const Chunk ch = decode_chunk(cx, q);
    const CompDev& C = cx.comps[ch.comp];
    const int64_t kb0 = C.K + (int64_t)ch.ua * C.bpr;  // global block index of (ua, block 0)
    if (!owned(C, ch.ua, ch.b0 * kPairsPerBlock)) continue;  // sharded (one block per chunk): another shard emits it
    if (C.sh_world > 1 ? cx.vcount[kb0 + ch.b0] == 0 : cx.idbase[kb0 + ch.b1] == cx.idbase[kb0 + ch.b0])
      continue;  // no states in the chunk
    const ViewDev& Av = C.Af;
    const ViewDev& Bv = C.Bf;
    const int64_t id_comp = tot[2 * ch.comp];
    const int64_t arc_comp = tot[2 * ch.comp + 1];
    const int wpr = C.wpr;
    load_chunk_bits(s, cx.V, C, ch, false);
    stage_arow(s, C, Av, ch.ua, 2 * wpr);
    const bool staged = s.dst_staged;
    int2* VR = (int2*)dyn;  // per staged word: (V word, rank of its first pair)
    if (staged) {
      for (int i = threadIdx.x; i < s.m * wpr; i += kThreads) {
        const int r = i / wpr, w = i - r * wpr;
        const int32_t row = s.slot_row[r];
        const int64_t gw = C.W + (int64_t)row * wpr + w;
        const int64_t blk = C.K + (int64_t)row * C.bpr + (w >> 5);
        VR[i] = make_int2((int32_t)__ldg(&cx.V[gw]),
                          (int32_t)(__ldg(&cx.idbase[blk]) - id_comp + __ldg(&cx.wpre[gw])));
      }
      __syncthreads();
    }
    // state id of pair (row, col) inside its composition; present = the pair is a state of C
    auto rank_of = [&](int slot, int32_t row, int32_t col, bool& present) -> int32_t {
      const uint32_t bit = 1u << (col & 31);
      const uint32_t lowmask = bit - 1u;
      if (staged) {
        const int2 vr = VR[slot * wpr + (col >> 5)];
        present = (uint32_t)vr.x & bit;
        return vr.y + __popc((uint32_t)vr.x & lowmask);
      }
      const int64_t gw = C.W + (int64_t)row * wpr + (col >> 5);
      const uint32_t w = __ldg(&cx.V[gw]);
      present = w & bit;
      if (!present) return 0;
      const int64_t blk = C.K + (int64_t)row * C.bpr + (col >> 10);
      return (int32_t)(__ldg(&cx.idbase[blk]) - id_comp + __ldg(&cx.wpre[gw]) + __popc(w & lowmask));
    };
    const int32_t ua = ch.ua;
    const uint8_t stA = __ldg(&C.startA[ua]), acA = __ldg(&C.accA[ua]);
    int32_t* const xa = C.arc_a;
    int32_t* const xb = C.arc_b;
    auto emit_arc = [&](const Cand& c, int64_t pos) {
      bool pr;
      const int32_t did = rank_of(c.slot, c.row, c.col, pr);
      int32_t il, ol;
      float wt;
      if (c.kind == 1) {
        const int2 b = __ldg(&Bv.cw[c.eb]);
        il = __ldg(&Av.carry[s.a0 + c.k]);
        ol = b.x;
        wt = __fadd_rn(__ldg(&Av.w[s.a0 + c.k]), __int_as_float(b.y));  // one binary32 add, RN-even
      } else if (c.kind == 2) {
        il = __ldg(&Av.carry[s.a0 + c.k]);
        ol = FST_EPS;
        wt = __ldg(&Av.w[s.a0 + c.k]);  // bit copy
      } else {
        const int2 b = __ldg(&Bv.cw[c.eb]);
        il = FST_EPS;
        ol = b.x;
        wt = __int_as_float(b.y);  // bit copy
      }
      __stcs(&C.dst[pos], did);
      __stcs(&C.ilabel[pos], il);
      __stcs(&C.olabel[pos], ol);
      __stcs(&C.weight[pos], wt);
      if (xa) {  // provenance: input arc indices (FST_COMPOSE_PROVENANCE)
        __stcs(&xa[pos], c.kind != 3 ? __ldg(&Av.arc[s.a0 + c.k]) : -1);
        __stcs(&xb[pos], c.kind != 2 ? __ldg(&Bv.arc[c.eb]) : -1);
      }
    };
    // output window per warp: what the staged (V word, rank) rows leave of the dynamic shared memory
    const int vr_words = (2 * s.m * wpr + 3) & ~3;
    const int wcap = min(kWCap, ((kDynSmem / 4 - vr_words) / (kWarps * 4)) & ~31);
    const bool fastE = staged && s.small && wcap >= kWCapMin;
    if (!fastE) {
      build_groups(s, Bv);
      __syncthreads();
    }
    for (int32_t blk = ch.b0; blk < ch.b1; ++blk) {
      const int64_t gblk = kb0 + blk;
      if (cx.vcount[gblk] == 0) continue;
      int64_t run = cx.arcbase[gblk] - arc_comp;
      const int64_t run0 = run;
      const int32_t ub0 = blk * kPairsPerBlock, ub1 = min(ub0 + kPairsPerBlock, C.VB);
      const int lw0 = (blk - ch.b0) * 32;
      if (fastE) {
        int4* wb = (int4*)(dyn + vr_words) + warp * wcap;
        auto rk = [&](int slot, int32_t col, bool& pr) -> int32_t { return rank_of(slot, 0, col, pr); };
        auto so = [&](int32_t ub, int64_t at) {
          bool pr;
          const int32_t id = rank_of(0, ua, ub, pr);
          __stcs((long long*)&C.row_ptr[id], (long long)at);
          __stcs(&C.pair_a[id], ua);
          __stcs(&C.pair_b[id], ub);
          C.is_start[id] = (uint8_t)(stA & __ldg(&C.startB[ub]));
          C.is_accept[id] = (uint8_t)(acA & __ldg(&C.accB[ub]));
        };
        const uint8_t* cnt8row = cx.cnt8 + ch.rowW * 32;
        const int btot =
            C.arc_a ? (s.mask32 ? emit_block_fast<true, true>(s, Bv, C, ub0, ub1, lw0, wpr, VR, wb, wcap, cnt8row, run, rk, so)
                                : emit_block_fast<false, true>(s, Bv, C, ub0, ub1, lw0, wpr, VR, wb, wcap, cnt8row, run, rk, so))
                    : (s.mask32 ? emit_block_fast<true, false>(s, Bv, C, ub0, ub1, lw0, wpr, VR, wb, wcap, cnt8row, run, rk, so)
                                : emit_block_fast<false, false>(s, Bv, C, ub0, ub1, lw0, wpr, VR, wb, wcap, cnt8row, run, rk, so));
        if (threadIdx.x == 0 && (unsigned long long)btot != cx.kept[gblk]) atomicAdd(&cx.misc[2], 1ull);
        run += btot;
        __syncthreads();
      } else if (s.G != 0 && cx.vcount[gblk] * 4 >= ub1 - ub0) {
        // dense block, label-major.  count: per-state kept moves (M2 first, then the groups)
        const int total = block_groups(s, Bv, ub0, ub1);
        for (int i = threadIdx.x; i < kPairsPerBlock; i += kThreads) {
          const int32_t ub = ub0 + i;
          int c = 0;
          if (ub < ub1 && src_bit(s, lw0, ub0, ub)) {
            for (int a = 0; a < s.aeps; ++a) {
              bool pr;
              rank_of(s.a_slot[a], s.a_other[a], ub, pr);
              c += pr;
            }
          }
          s.cur[i] = c;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < total; i += kThreads) {
          const int g = item_group(s, i);
          const int32_t sid = s.g_lo[g] + (i - s.g_pre[g]);
          const int32_t ub = __ldg(&Bv.seg_node[sid]);
          if (!src_bit(s, lw0, ub0, ub)) continue;
          const int32_t e0 = __ldg(&Bv.seg_beg[sid]), e1 = __ldg(&Bv.seg_beg[sid + 1]);
          const unsigned long long gm = s.g_mask[g];
          const bool eps = s.g_label[g] == FST_EPS;
          int c = 0;
          for (int32_t j = e0; j < e1; ++j) {
            const int32_t ob = __ldg(&Bv.lm_other[j]);
            for (unsigned long long m = gm; m; m &= m - 1) {
              const int a = __ffsll((long long)m) - 1;
              bool pr;
              rank_of(s.a_slot[a], s.a_other[a], ob, pr);
              c += pr;
            }
            if (eps) {
              bool pr;
              rank_of(0, ua, ob, pr);
              c += pr;
            }
          }
          if (c) atomicAdd(&s.cur[ub - ub0], c);
        }
        __syncthreads();
        // exclusive scan of the per-state counts -> state start offsets
        const int i0 = 2 * threadIdx.x;
        const int c0 = s.cur[i0], c1 = s.cur[i0 + 1];
        int btot;
        const int ex = block_excl_scan(c0 + c1, s.red32, &btot);
        if (threadIdx.x == 0 && (unsigned long long)btot != cx.kept[gblk]) atomicAdd(&cx.misc[2], 1ull);
        // per-state outputs and M2 arcs; cursors
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int i = i0 + j;
          const int32_t ub = ub0 + i;
          int64_t pos = run + ex + (j ? c0 : 0);
          if (ub < ub1 && src_bit(s, lw0, ub0, ub)) {
            bool pr;
            const int32_t id = rank_of(0, ua, ub, pr);
            __stcs((long long*)&C.row_ptr[id], (long long)pos);
            __stcs(&C.pair_a[id], ua);
            __stcs(&C.pair_b[id], ub);
            C.is_start[id] = (uint8_t)(stA & __ldg(&C.startB[ub]));
            C.is_accept[id] = (uint8_t)(acA & __ldg(&C.accB[ub]));
            for (int a = 0; a < s.aeps; ++a) {
              const Cand c{s.a_slot[a], s.a_other[a], ub, 2, a, -1};
              bool p2;
              rank_of(c.slot, c.row, c.col, p2);
              if (p2) emit_arc(c, pos++);
            }
          }
          s.cur[i] = (int32_t)(pos - run);
        }
        __syncthreads();
        // groups in label order; a state has at most one segment per group, so its cursor is
        // owned by one thread per group pass
        for (int g = 0; g < s.G; ++g) {
          const int n = s.g_pre[g + 1] - s.g_pre[g];
          const unsigned long long gm = s.g_mask[g];
          const bool eps = s.g_label[g] == FST_EPS;
          for (int i = threadIdx.x; i < n; i += kThreads) {
            const int32_t sid = s.g_lo[g] + i;
            const int32_t ub = __ldg(&Bv.seg_node[sid]);
            if (!src_bit(s, lw0, ub0, ub)) continue;
            const int32_t e0 = __ldg(&Bv.seg_beg[sid]), e1 = __ldg(&Bv.seg_beg[sid + 1]);
            int64_t pos = run + s.cur[ub - ub0];
            for (int32_t j = e0; j < e1; ++j) {
              const int32_t ob = __ldg(&Bv.lm_other[j]);
              const int32_t eb = __ldg(&Bv.lm_pos[j]);
              for (unsigned long long m = gm; m; m &= m - 1) {
                const int a = __ffsll((long long)m) - 1;
                const Cand c{s.a_slot[a], s.a_other[a], ob, 1, a, eb};
                bool pr;
                rank_of(c.slot, c.row, c.col, pr);
                if (pr) emit_arc(c, pos++);
              }
              if (eps) {
                const Cand c{0, ua, ob, 3, -1, eb};
                bool pr;
                rank_of(0, ua, ob, pr);
                if (pr) emit_arc(c, pos++);
              }
            }
            s.cur[ub - ub0] = (int32_t)(pos - run);
          }
          __syncthreads();
        }
        run += btot;
      } else
      for_block_items(s, Bv, C, ch, blk, [&](bool valid, int32_t it, int32_t ub, int2 kd) {
        const Item x = make_item(s, Av, it, ub, kd, valid);
        const int maxn = __reduce_max_sync(0xffffffffu, (unsigned)x.n);
        const bool simple = maxn <= kSimpleMoves;
        // phase 1: kept moves of this lane (simple) / of this warp (expanded)
        unsigned lk = 0, keptbits = 0;
        if (simple) {
          for (int k = 0; k < maxn; ++k) {
            if (k < x.n) {
              const Cand c = item_move(s, Av, ua, x, k);
              bool pr;
              rank_of(c.slot, c.row, c.col, pr);
              if (pr) {
                keptbits |= 1u << k;
                ++lk;
              }
            }
          }
        } else {
          warp_expand(s, Av, ua, x, [&](bool act, const Cand& c, int) {
            bool pr = false;
            if (act) rank_of(c.slot, c.row, c.col, pr);
            if (lane == 0) lk += __popc(__ballot_sync(0xffffffffu, pr));
            else __ballot_sync(0xffffffffu, pr);
          });
        }
        const unsigned linc = warp_incl_scan(lk);  // simple: lane prefix; expanded: lane 0 holds the total
        const unsigned wk = simple ? __shfl_sync(0xffffffffu, linc, 31) : __shfl_sync(0xffffffffu, lk, 0);
        if (lane == 0) s.wtot[warp] = (int32_t)wk;
        __syncthreads();
        int64_t wbase, rtot;
        {
          const int32_t t = lane < kWarps ? s.wtot[lane] : 0;
          const int32_t inc = warp_incl_scan(t);
          wbase = run + __shfl_sync(0xffffffffu, inc - t, warp);
          rtot = __shfl_sync(0xffffffffu, inc, kWarps - 1);
        }
        // phase 2: write
        const bool sent = valid && x.kind == 2;
        int64_t spos = -1;
        if (simple) {
          int64_t pos = wbase + (linc - lk);
          spos = pos;
          for (int k = 0; k < maxn; ++k)
            if ((keptbits >> k) & 1u) emit_arc(item_move(s, Av, ua, x, k), pos++);
        } else {
          const int start = warp_incl_scan(x.n) - x.n;
          unsigned before = 0;
          warp_expand(s, Av, ua, x, [&](bool act, const Cand& c, int r) {
            bool pr = false;
            if (act) rank_of(c.slot, c.row, c.col, pr);
            const unsigned bal = __ballot_sync(0xffffffffu, pr);
            if (sent && start >= r && start < r + 32) spos = wbase + before + __popc(bal & ((1u << (start - r)) - 1u));
            if (pr) emit_arc(c, wbase + before + __popc(bal & ((1u << lane) - 1u)));
            before += __popc(bal);
          });
          if (sent && spos < 0) spos = wbase + before;
        }
        if (sent) {  // per-state outputs of a state of C
          bool pr;
          const int32_t id = rank_of(0, ua, ub, pr);
          __stcs((long long*)&C.row_ptr[id], (long long)spos);
          __stcs(&C.pair_a[id], ua);
          __stcs(&C.pair_b[id], ub);
          C.is_start[id] = (uint8_t)(stA & __ldg(&C.startB[ub]));
          C.is_accept[id] = (uint8_t)(acA & __ldg(&C.accB[ub]));
        }
        run += rtot;
        __syncthreads();
      });
      if (threadIdx.x == 0 && (unsigned long long)(run - run0) != cx.kept[gblk]) atomicAdd(&cx.misc[2], 1ull);
      __syncthreads();
    }
    __syncthreads();
  }
}

#include "tile.cuh"

inline unsigned nblk(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

int g_grid = 0;

fst_status init_kernels() {
  if (g_grid) return FST_OK;
  FSTC_CUDA_TRY(cudaFuncSetAttribute(k_level<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmem));
  FSTC_CUDA_TRY(cudaFuncSetAttribute(k_level<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmem));
  FSTC_CUDA_TRY(cudaFuncSetAttribute(k_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmem));
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_level<true>, kThreads, kDynSmem);
  int occ2 = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_emit, kThreads, kDynSmem);
  g_grid = sm_count() * std::max(1, std::min(occ, occ2));
  return FST_OK;
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

// Body tail of the graph-driven level loop: advance the device level counter and keep looping
// while the next level has active chunks (CUDA graph while-node, set from the device).
__global__ void k_level_advance(Ctx cx, const int32_t* level_dev, cudaGraphConditionalHandle h) {
  const int32_t l = *level_dev;  // the next level to run
  const bool more = *((volatile unsigned long long*)&cx.ctrl[l % 3].count) != 0ull;
  cudaGraphSetConditional(h, more ? 1u : 0u);
}

int32_t* level_scratch() {
  static thread_local int32_t* p = nullptr;
  if (!p && cudaMalloc(&p, 256) != cudaSuccess) p = nullptr;
  return p;
}

// A per-thread side stream with the priority of `s`.
cudaStream_t side_stream(cudaStream_t s) {
  static thread_local cudaStream_t ss[2] = {nullptr, nullptr};
  int pr = 0, lo = 0, hi = 0;
  cudaStreamGetPriority(s, &pr);
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  const int k = (pr < lo) ? 1 : 0;  // numerically lower = higher priority
  if (!ss[k] && cudaStreamCreateWithPriority(&ss[k], cudaStreamNonBlocking, k ? hi : lo) != cudaSuccess) ss[k] = nullptr;
  return ss[k];
}

cudaStream_t capture_stream() {
  static thread_local cudaStream_t cs = nullptr;
  if (!cs && cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) cs = nullptr;
  return cs;
}

// Levels [level, ...) of a deep BFS in ONE graph launch: a while-node whose body is 6 k_level
// launches (one period of the frontier / control-block rings: the captured level arguments are
// right modulo 6) + the advance kernel that tests the next level's list, so there is no host round
// trip per level batch (lexicon trellises run hundreds of levels).  Up to 5 trailing levels are
// no-op launches, as in the host loop's speculative batches.
template <bool kStage2>
fst_status run_levels_graph(const Ctx& cx, cudaStream_t s, int* level, int64_t* level_launches) {
  int32_t* d_level = level_scratch();
  cudaStream_t cs = capture_stream();
  if (!d_level || !cs) {
    set_error(FST_E_CUDA, "level loop: scratch allocation failed");
    return FST_E_CUDA;
  }
  const int32_t l0 = *level;
  FSTC_CUDA_TRY(cudaMemcpyAsync(d_level, &l0, sizeof(int32_t), cudaMemcpyHostToDevice, s));
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  FSTC_CUDA_TRY(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  cudaGraphNodeParams cp = {};
  cudaGraphNode_t node;
  cudaGraph_t body;
  cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  if (e == cudaSuccess) {
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    e = cudaGraphAddNode(&node, g, nullptr, 0, &cp);
  }
  if (e == cudaSuccess) {
    body = cp.conditional.phGraph_out[0];
    e = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
    if (e == cudaSuccess) {
      Ctx cg = cx;
      cg.level_dev = d_level;
      for (int j = 0; j < 6; ++j) k_level<kStage2><<<g_grid, kThreads, kDynSmem, cs>>>(cg, l0 + j);
      k_level_advance<<<1, 1, 0, cs>>>(cx, d_level, h);
      e = cudaStreamEndCapture(cs, &body);
    }
  }
  if (e == cudaSuccess) e = cudaGraphInstantiate(&ge, g, 0);
  if (e == cudaSuccess) e = cudaGraphLaunch(ge, s);
  int32_t lend = l0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&lend, d_level, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (ge) cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    set_error(FST_E_CUDA, "graph level loop: %s", cudaGetErrorString(e));
    return FST_E_CUDA;
  }
  count_launch((int64_t)(lend - l0) * 7 / 6);
  *level_launches += lend - l0;
  *level = lend;
  return FST_OK;
}

// FSTC_NO_PULL=1 disables the bottom-up stage-1 levels (A/B and debugging).
bool pull_enabled() {
  static const bool on = [] {
    const char* e = getenv("FSTC_NO_PULL");
    return !(e && e[0] == '1');
  }();
  return on;
}

// FSTC_PULL_NUM=k (A/B tuning): pull when frontier * k >= unvisited * 4 (default 8: configs[3] stage 1
// 36.4 -> 29.5 ms; 4: 30.3, 16: 29.4 but D=4 +12%).
int32_t pull_num() {
  static const int32_t v = [] {
    const char* e = getenv("FSTC_PULL_NUM");
    const int k = e ? atoi(e) : 8;
    return k > 0 ? k : 8;
  }();
  return v;
}

// FSTC_NO_GRAPH_LOOP=1 keeps every level on the host loop (ncu cannot profile kernels inside a graph
// with conditional nodes).
bool graph_loop_enabled() {
  static const bool on = [] {
    const char* e = getenv("FSTC_NO_GRAPH_LOOP");
    return !(e && e[0] == '1');
  }();
  return on;
}

// Runs one BFS stage (level loop); fills the per-level frontier sizes.  The first levels run as
// host-driven speculative batches; a BFS still going after kHostLevels levels continues in one
// graph launch (run_levels_graph).
// FSTC_HOST_LEVELS=n: levels run host-driven before the graph loop takes over (default 64).
int host_levels() {
  static const int v = [] {
    const char* e = getenv("FSTC_HOST_LEVELS");
    const int k = e ? atoi(e) : 64;
    return k >= 0 ? k : 64;
  }();
  return v;
}
template <bool kStage2>
fst_status run_stage(const Ctx& cx, cudaStream_t s, unsigned long long* h_pinned, int64_t* level_launches,
                     std::vector<int64_t>* sizes) {
  int level = 0;
  int batch = 1;
  for (;;) {
    for (int k = 0; k < batch; ++k, ++level) {
      k_level<kStage2><<<g_grid, kThreads, kDynSmem, s>>>(cx, level);
      FSTC_LAUNCH_CHECK();
      ++*level_launches;
    }
    FSTC_CUDA_TRY(cudaMemcpyAsync(h_pinned, &cx.ctrl[level % 3].count, sizeof(unsigned long long),
                                  cudaMemcpyDeviceToHost, s));
    FSTC_CUDA_TRY(cudaStreamSynchronize(s));
    if (*h_pinned == 0) break;
    if (level >= host_levels() && graph_loop_enabled()) {  // deep BFS: the rest in one graph launch
      fst_status st = run_levels_graph<kStage2>(cx, s, &level, level_launches);
      if (st) return st;
      break;
    }
    batch = std::min(batch * 2, 32);  // speculative level batches: empty levels are no-op launches
  }
  FSTC_CUDA_TRY(cudaMemcpyAsync(h_pinned, cx.misc, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  FSTC_CUDA_TRY(cudaStreamSynchronize(s));
  const unsigned long long nl = *h_pinned;
  const int n = (int)std::min<unsigned long long>(nl, kMaxLevelStats);
  std::vector<unsigned long long> tmp(n);
  if (n) {
    FSTC_CUDA_TRY(cudaMemcpyAsync(tmp.data(), cx.hist, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost, s));
    FSTC_CUDA_TRY(cudaStreamSynchronize(s));
  }
  sizes->assign(tmp.begin(), tmp.end());
  return FST_OK;
}

unsigned long long* pinned_scratch() {
  static thread_local unsigned long long* p = nullptr;
  if (!p && cudaMallocHost(&p, 64 * sizeof(unsigned long long)) != cudaSuccess) p = nullptr;
  return p;
}

// ------------------------------------------------------------------------------ tile path (host)
std::atomic<int>& tile_mode_ref() {
  static std::atomic<int> m{[] {
    const char* e = getenv("FSTC_TILE");
    const int v = e ? atoi(e) : 1;
    return (v >= 0 && v <= 4) ? v : 1;
  }()};
  return m;
}

constexpr int64_t kTileMinPairs = 1ll << 23;

// FSTC_SPARSE_PUSH=0: the tile path's push levels run on k_level instead of k_sparse_push (A/B).
bool sparse_push_enabled() {
  static const bool on = [] {
    const char* e = getenv("FSTC_SPARSE_PUSH");
    return !(e && e[0] == '0');
  }();
  return on;
}

// FSTC_TILE_PUSH=1: the tile path's push levels run on k_tile_push instead of k_level (opt-in: measured
// 13.0 ms vs 9.9 ms over the 34 push levels of configs[3] -- the per-tile RT builds cost more than the
// word-parallel tests save at these frontier sizes).
bool tile_push_enabled() {
  static const bool on = [] {
    const char* e = getenv("FSTC_TILE_PUSH");
    return e && e[0] == '1';
  }();
  return on;
}

// FSTC_TILE_PULL_K=k: a level runs bottom-up when frontier * k >= the stage's pair set (stage 1: the
// pair space, stage 2: R).  A bottom-up round costs about one sweep whatever its frontier, a push level
// grows with its frontier.  Default 512 (configs[3] with the sparse push levels: K = 128 / 256 / 512 /
// 1024 -> 38.8 / 37.7 / 36.9 / 37.5 ms per composition).
int64_t tile_pull_k() {
  static const int64_t v = [] {
    const char* e = getenv("FSTC_TILE_PULL_K");
    const long long k = e ? atoll(e) : 512;
    return (int64_t)(k > 0 ? k : 512);
  }();
  return v;
}
// FSTC_TILE_PULL_KEXIT=k: after a bottom-up round, the next level stays bottom-up only while the
// round's claims * k >= the stage's pairs (default = FSTC_TILE_PULL_K).
int64_t tile_pull_kexit() {
  static const int64_t v = [] {
    const char* e = getenv("FSTC_TILE_PULL_KEXIT");
    const long long k = e ? atoll(e) : 0;
    return (int64_t)(k > 0 ? k : tile_pull_k());
  }();
  return v;
}

int smem_optin() {
  static int v = 0;
  if (!v) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (v <= 0) v = 227 * 1024;
  }
  return v;
}

// B role: ELL of view `which` (0 = out-by-ilabel, with (carry, weight); 1 = in-by-ilabel), cached in
// the handle.
fst_status ensure_tile_ell(fst* B, int which, cudaStream_t s) {
  fst::TileEll& T = B->tile_ell[which];
  if (T.ok) return FST_OK;
  const View& v = B->views[which == 0 ? kOutByIlabel : kInByIlabel];
  const int32_t V = B->V;
  const int wd = v.max_deg + 1;
  const int wpr = (V + 31) / 32;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
  const size_t o_ell = take(4ull * wd * wpr * 32), o_cw = which == 0 ? take(8ull * wd * wpr * 32) : 0;
  const size_t o_wmax = take(wpr), o_flag = take(4);
  BufferPtr buf;
  fst_status st = alloc_buffer(off, s, &buf);
  if (st) return st;
  char* base = (char*)buf->ptr;
  T.ell = (uint32_t*)(base + o_ell);
  T.cw = which == 0 ? (int2*)(base + o_cw) : nullptr;
  T.wmax = (uint8_t*)(base + o_wmax);
  int32_t* d_flag = (int32_t*)(base + o_flag);
  FSTC_CUDA_TRY(cudaMemsetAsync(d_flag, 0, 4, s));
  k_build_ell<<<nblk((int64_t)wpr * 32, 256), 256, 0, s>>>(V, v.off, v.key, v.other, which == 0 ? v.cw : nullptr, wd,
                                                           T.ell, T.cw, T.wmax, d_flag);
  FSTC_LAUNCH_CHECK();
  int32_t flag = 0;
  FSTC_CUDA_TRY(cudaMemcpyAsync(&flag, d_flag, 4, cudaMemcpyDeviceToHost, s));
  FSTC_CUDA_TRY(cudaStreamSynchronize(s));
  T.has_eps = flag != 0;
  T.wd = wd;
  T.buf = buf;
  T.ok = true;
  return FST_OK;
}

// A role: tile row starts for view `which` (0 = out-by-olabel, 1 = in-by-olabel): consecutive rows,
// at most kTRows rows and `slot_cap` slots (arcs + self slot; 8 per row in byte mode) per tile, and
// (slots + rows) <= vr_cap when vr_cap > 0 (the emit's staged rank rows).  Greedy; cached.
fst_status tile_rows(fst* A, int which, int self, int slot_cap, int vr_cap, int bytemode, cudaStream_t s,
                     const int32_t** d, int32_t* ntiles) {
  const int64_t key = (int64_t)which | ((int64_t)self << 1) | ((int64_t)bytemode << 2) | ((int64_t)slot_cap << 3) |
                      ((int64_t)vr_cap << 16);
  for (const auto& tr : A->tile_rows)
    if (tr.key == key) {
      *d = tr.d;
      *ntiles = tr.n;
      return FST_OK;
    }
  std::vector<int32_t>& hoff = A->tile_hoff[which];
  const int32_t V = A->V;
  if ((int32_t)hoff.size() != V + 1) {
    hoff.resize(V + 1);
    const View& v = A->views[which == 0 ? kOutByOlabel : kInByOlabel];
    FSTC_CUDA_TRY(cudaMemcpyAsync(hoff.data(), v.off, sizeof(int32_t) * (V + 1), cudaMemcpyDeviceToHost, s));
    FSTC_CUDA_TRY(cudaStreamSynchronize(s));
  }
  std::vector<int32_t> tr{0};
  int slots = 0, rows = 0;
  for (int32_t r = 0; r < V; ++r) {
    const int n = bytemode ? 8 : hoff[r + 1] - hoff[r] + self;
    if (rows > 0 && (slots + n > slot_cap || rows + 1 > kTRows || (vr_cap > 0 && slots + n > vr_cap))) {
      tr.push_back(r);
      slots = rows = 0;
    }
    slots += n;
    ++rows;
  }
  tr.push_back(V);
  fst::TileRows out;
  out.key = key;
  out.n = (int32_t)tr.size() - 1;
  out.h = tr;
  fst_status st = alloc_buffer(sizeof(int32_t) * tr.size(), s, &out.buf);
  if (st) return st;
  out.d = (int32_t*)out.buf->ptr;
  FSTC_CUDA_TRY(cudaMemcpyAsync(out.d, tr.data(), sizeof(int32_t) * tr.size(), cudaMemcpyHostToDevice, s));
  FSTC_CUDA_TRY(cudaStreamSynchronize(s));
  A->tile_rows.push_back(out);
  *d = out.d;
  *ntiles = out.n;
  return FST_OK;
}

size_t tile_emit_smem(int vr_rows, int wpr, int wd) {
  (void)wd;
  const size_t vr = (size_t)vr_rows * wpr;
  return (size_t)wpr * 128 + 4 * vr + 4 * ((vr + 1) / 2) + (size_t)kEWarps * kECap * 4;
}

// Everything the tile kernels need for one composition; ok = false if the inputs do not fit.
struct TilePlan {
  bool ok = false;
  TileArgs s1, s2, cnt, emit;
  int vr_rows = 0;
  size_t smem_pull = 0, smem_count = 0, smem_emit = 0, smem_push = 0;
  int max_li = 255;  // largest label index (label + 2) of the matched tapes
  int grid_pull1 = 0, grid_pull2 = 0, grid_count = 0, grid_emit = 0;
};

fst_status tile_plan(fst* A, fst* B, int64_t pairs, bool want_prov, cudaStream_t s, TilePlan* P) {
  P->ok = false;
  const int mode = tile_mode_ref().load();
  if (mode == 0 || want_prov) return FST_OK;
  if (mode == 1 && pairs < kTileMinPairs) return FST_OK;
  if (A->V < 1 || B->V < 1 || B->V > 65535) return FST_OK;
  if (A->max_olabel > 252 || B->max_ilabel > 252) return FST_OK;
  if (B->views[kOutByIlabel].max_deg + 1 > 32 || B->views[kInByIlabel].max_deg + 1 > 32) return FST_OK;
  const int degA_out = A->views[kOutByOlabel].max_deg, degA_in = A->views[kInByOlabel].max_deg;
  if (degA_out + 1 > kESlots || degA_in + 1 > kPSlots) return FST_OK;
  const int wpr = (B->V + 31) / 32, bpr = (wpr + kWordsPerBlock - 1) / kWordsPerBlock;
  const int smem_cap = smem_optin() - 4096;  // static shared memory of the kernels stays below 4 KB
  const size_t smem_pull = (size_t)wpr * 256, smem_count = smem_pull + 8ull * kTRows * bpr;
  const size_t smem_push = smem_pull + 4ull * kTRows * wpr;
  if (smem_push > (size_t)(smem_optin() - 4096)) return FST_OK;
  if (smem_count > (size_t)smem_cap) return FST_OK;
  if ((bpr + 0) > 64) return FST_OK;  // the bottom-up rounds track <= 64 chunks per row
  const int wd_out = B->views[kOutByIlabel].max_deg + 1;
  // emit: staged rank rows fill what RT and the per-warp code buffers leave
  const size_t per_warp = (size_t)kEWarps * kECap * 4 + (size_t)wpr * 128;
  if ((size_t)smem_cap <= per_warp || B->V > 65535) return FST_OK;
  int vr_rows = (int)std::min<size_t>(kESlots, ((size_t)smem_cap - per_warp) / ((size_t)wpr * 6 + 2));  // slot rows
  while (vr_rows > 0 && tile_emit_smem(vr_rows, wpr, wd_out) > (size_t)smem_cap) --vr_rows;
  if (vr_rows < degA_out + 1) return FST_OK;  // one row with its self slot must fit
  fst_status st = ensure_tile_ell(B, 0, s);
  if (!st) st = ensure_tile_ell(B, 1, s);
  if (st) return st;
  const int self = B->tile_ell[0].has_eps ? 1 : 0;  // same flag for both views (B ilabels)
  auto side = [&](int which_a, int which_b) {
    const View& v = A->views[which_a == 0 ? kOutByOlabel : kInByOlabel];
    const fst::TileEll& T = B->tile_ell[which_b];
    return TileSide{v.off, v.key, v.other, v.carry, v.w, T.ell, T.cw, T.wmax, T.wd};
  };
  const int byte1 = degA_out + self <= 8 ? 1 : 0, byte2 = degA_in + self <= 8 ? 1 : 0;
  const int32_t* d;
  int32_t nt;
  st = tile_rows(A, 0, self, kPSlots, 0, byte1, s, &d, &nt);
  if (st) return st;
  P->s1 = TileArgs{side(0, 0), d, nt, self, byte1, 8, 0, nt};
  P->cnt = P->s1;
  st = tile_rows(A, 1, self, kPSlots, 0, byte2, s, &d, &nt);
  if (st) return st;
  P->s2 = TileArgs{side(1, 1), d, nt, self, byte2, 8, 0, nt};
  st = tile_rows(A, 0, self, kESlots, vr_rows, 0, s, &d, &nt);
  if (st) return st;
  P->emit = TileArgs{side(0, 0), d, nt, self, 0, 8, 0, nt};
  P->vr_rows = vr_rows;
  P->max_li = std::max(A->max_olabel, B->max_ilabel) + 2;
  P->smem_pull = smem_pull;
  P->smem_push = smem_push;
  P->smem_count = smem_count;
  P->smem_emit = tile_emit_smem(vr_rows, wpr, wd_out);
  static bool attrs = false;
  if (!attrs) {
    const void* fs[] = {(const void*)k_tile_push<false, 8>, (const void*)k_tile_push<false, 16>,
                        (const void*)k_tile_push<true, 8>,  (const void*)k_tile_push<true, 16>,
                        (const void*)k_tile_pull<false, 8, kTP1Threads>, (const void*)k_tile_pull<false, 16, kTP1Threads>,
                        (const void*)k_tile_pull<true, 8, kTP2Threads>,  (const void*)k_tile_pull<true, 16, kTP2Threads>,
                        (const void*)k_tile_count<false, 8>, (const void*)k_tile_count<false, 16>,
                        (const void*)k_tile_count<true, 8>,  (const void*)k_tile_count<true, 16>,
                        (const void*)k_tile_emit<8>,        (const void*)k_tile_emit<16>};
    for (const void* f : fs) FSTC_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap));
    attrs = true;
  }
  P->s1.kj = B->tile_ell[0].wd - 1 <= 8 ? 8 : 16;
  P->cnt.kj = P->s1.kj;
  P->emit.kj = P->s1.kj;
  P->s2.kj = B->tile_ell[1].wd - 1 <= 8 ? 8 : 16;
  // one CTA per SM (the staged tables take the shared memory), never more CTAs than tiles
  P->grid_pull1 = std::max(1, std::min(P->s1.ntiles, sm_count()));
  P->grid_pull2 = std::max(1, std::min(P->s2.ntiles, sm_count()));
  P->grid_count = std::max(1, std::min(P->cnt.ntiles, sm_count()));
  // the emit: one CTA per tile (tiles are handed out as CTAs retire: configs[3] 12.1 -> 11.9 ms against
  // the persistent one-CTA-per-SM grid; the rounds and the counts showed no difference)
  P->grid_emit = std::max(1, P->emit.ntiles);
  P->ok = true;
  return FST_OK;
}

template <bool kStage2>
void launch_tile_pull(const TileArgs& ta, int grid, size_t smem, cudaStream_t s, const Ctx& cx, int level) {
  constexpr int nt = kStage2 ? kTP2Threads : kTP1Threads;
  if (ta.kj == 8) k_tile_pull<kStage2, 8, nt><<<grid, nt, smem, s>>>(cx, ta, level);
  else k_tile_pull<kStage2, 16, nt><<<grid, nt, smem, s>>>(cx, ta, level);
}
// push level in tile form: stage 1 walks the reversed moves (in-view tiles: TilePlan::s2), stage 2 the
// forward moves (out-view tiles: TilePlan::s1)
template <bool kStage2>
void launch_tile_push(const TileArgs& ta, int grid, size_t smem, cudaStream_t s, const Ctx& cx, int level) {
  if (ta.kj == 8) k_tile_push<kStage2, 8><<<grid, kTThreads, smem, s>>>(cx, ta, level);
  else k_tile_push<kStage2, 16><<<grid, kTThreads, smem, s>>>(cx, ta, level);
}
void launch_tile_count(const TileArgs& ta, int grid, size_t smem, cudaStream_t s, const Ctx& cx) {
  if (ta.bytemode) {
    if (ta.kj == 8) k_tile_count<true, 8><<<grid, kTThreads, smem, s>>>(cx, ta);
    else k_tile_count<true, 16><<<grid, kTThreads, smem, s>>>(cx, ta);
  } else {
    if (ta.kj == 8) k_tile_count<false, 8><<<grid, kTThreads, smem, s>>>(cx, ta);
    else k_tile_count<false, 16><<<grid, kTThreads, smem, s>>>(cx, ta);
  }
}
void launch_tile_emit(const TileArgs& ta, int grid, size_t smem, cudaStream_t s, const Ctx& cx, const CompDev& C,
                      const int64_t* tot, int vr_rows) {
  const EmitIO io{C.row_ptr, C.dst,    C.ilabel, C.olabel, C.weight, C.pair_a, C.pair_b,
                  C.is_start, C.is_accept, C.startA, C.accA,  C.startB, C.accB};
  if (ta.kj == 8) k_tile_emit<8><<<grid, kEThreads, smem, s>>>(cx, ta, io, tot, vr_rows);
  else k_tile_emit<16><<<grid, kEThreads, smem, s>>>(cx, ta, io, tot, vr_rows);
}

// One BFS stage with per-level direction choice: push levels are k_level; a level whose frontier is a
// sizable share of the stage's pairs (frontier * k >= total) runs bottom-up on the tile kernels.
template <bool kStage2>
fst_status run_stage_tile(const Ctx& cx, const TilePlan& tp, int64_t total, cudaStream_t s, unsigned long long* hp,
                          int64_t* level_launches, std::vector<int64_t>* sizes, int* npull) {
  const int64_t K = tile_pull_k(), Kexit = tile_pull_kexit();
  const bool all_pull = tile_mode_ref().load() == 3;  // test mode: every level bottom-up
  bool pulled = false;                                 // the previous level was a bottom-up round
  const TileArgs& ta = kStage2 ? tp.s2 : tp.s1;       // bottom-up rounds: in-view tiles for stage 2
  const TileArgs& tb = kStage2 ? tp.s1 : tp.s2;       // push levels: the opposite direction
  const int grid_pull = kStage2 ? tp.grid_pull2 : tp.grid_pull1, grid_push = kStage2 ? tp.grid_pull1 : tp.grid_pull2;
  const bool tile_push = tile_push_enabled() || tile_mode_ref().load() == 4;
  const bool sparse_push_ok = sparse_push_enabled() && tp.max_li < kSPLab;
  int level = 0;
  for (;;) {
    FSTC_CUDA_TRY(cudaMemcpyAsync(hp, &cx.ctrl[level % 3], sizeof(LevelCtrl), cudaMemcpyDeviceToHost, s));
    FSTC_CUDA_TRY(cudaStreamSynchronize(s));
    const unsigned long long cnt = hp[0], nf = hp[1], pad0 = hp[2];
    if (cnt == 0) break;
    const int64_t visited = (int64_t)(pad0 + nf);
    const int64_t unvisited = total > visited ? total - visited : 0;
    (void)unvisited;
    const bool pull = all_pull || (int64_t)nf * (pulled ? Kexit : K) >= total;
    pulled = pull;
    if (pull) {
      launch_tile_pull<kStage2>(ta, grid_pull, tp.smem_pull, s, cx, level);
      FSTC_LAUNCH_CHECK();
      ++*npull;
    } else if (tile_push) {
      launch_tile_push<kStage2>(tb, grid_push, tp.smem_push, s, cx, level);
      FSTC_LAUNCH_CHECK();
      k_push_finish<<<sm_count() * 8, 256, 0, s>>>(cx, level);
      FSTC_LAUNCH_CHECK();
    } else if (sparse_push_ok) {
      k_sparse_push<kStage2><<<sm_count() * kSPGrid, 256, 0, s>>>(cx, tb, level);
      FSTC_LAUNCH_CHECK();
      k_push_finish<<<sm_count() * 8, 256, 0, s>>>(cx, level);
      FSTC_LAUNCH_CHECK();
    } else {
      k_level<kStage2><<<g_grid, kThreads, kDynSmem, s>>>(cx, level);
      FSTC_LAUNCH_CHECK();
    }
    ++*level_launches;
    ++level;
  }
  FSTC_CUDA_TRY(cudaMemcpyAsync(hp, cx.misc, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  FSTC_CUDA_TRY(cudaStreamSynchronize(s));
  const int n = (int)std::min<unsigned long long>(hp[0], kMaxLevelStats);
  std::vector<unsigned long long> tmp(n);
  if (n) {
    FSTC_CUDA_TRY(cudaMemcpyAsync(tmp.data(), cx.hist, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost, s));
    FSTC_CUDA_TRY(cudaStreamSynchronize(s));
  }
  sizes->assign(tmp.begin(), tmp.end());
  return FST_OK;
}

}  // namespace

void tile_mode_set(int mode) { tile_mode_ref().store((mode >= 0 && mode <= 4) ? mode : 1); }

std::vector<int64_t>& level_sizes_slot(fst* h, int stage);

fst_status compose_run(int32_t n, const fst_handle* a, const fst_handle* b, cudaStream_t s, fst_handle* c,
                       uint32_t flags) {
  const bool want_prov = flags & FST_COMPOSE_PROVENANCE;
  const bool prof = profiling_enabled();
  EventTimer t_total(prof, s);
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
  fst_status st = init_kernels();
  if (st) return st;
  const int64_t launches0 = fst_launch_count();
  // ---- layout of the concatenated pair space
  int64_t total_rows = 0;
  for (int i = 0; i < n; ++i) total_rows += a[i]->V;
  const int64_t target_tasks = 8ll * g_grid;
  std::vector<CompDev> comps(n);
  std::vector<int64_t> seed1(n + 1, 0), seed2(n + 1, 0);
  int64_t W = 0, K = 0, Q = 0, pairs = 0;
  for (int i = 0; i < n; ++i) {
    const fst* A = a[i];
    const fst* B = b[i];
    CompDev& C = comps[i];
    memset(&C, 0, sizeof(C));
    auto vd = [](const View& v) { return ViewDev{v.off, v.key, v.other, v.carry, v.w, v.cw, v.ikd, v.isrc, v.ikcw, v.lm_other, v.lm_pos, v.seg_node, v.seg_beg, v.lab_val, v.lab_seg, v.nlab, v.arc}; };
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
    // chunks: enough CTA tasks to fill the GPU, at most kChunkMaxBlocks blocks each
    int64_t want = total_rows > 0 ? (target_tasks + total_rows - 1) / total_rows : 1;
    int32_t cpr = (int32_t)std::max<int64_t>(1, std::min<int64_t>(want, C.bpr));
    cpr = std::max<int32_t>(cpr, (C.bpr + kChunkMaxBlocks - 1) / kChunkMaxBlocks);
    C.CB = std::max<int32_t>(1, (C.bpr + cpr - 1) / cpr);
    C.cpr = std::max<int32_t>(1, (C.bpr + C.CB - 1) / C.CB);
    C.smallA = A->max_olabel < 63;
    C.sh_world = 1;
    C.sh_rank = 0;
    C.W = W;
    C.K = K;
    C.Q = Q;
    W += (int64_t)C.VA * C.wpr;
    K += (int64_t)C.VA * C.bpr;
    Q += (int64_t)C.VA * C.cpr;
    pairs += (int64_t)C.VA * C.VB;
    seed1[i + 1] = seed1[i] + (int64_t)C.nAccA * C.nAccB;
    seed2[i + 1] = seed2[i] + (int64_t)C.nStartA * C.nStartB;
  }
  const int64_t nwords = W, nblocks = K, nchunks = Q;
  // compositions whose A is topologically numbered (trellises): row-by-row stages (wave.cu); a
  // forced tile mode (>= 2) keeps single compositions on the tile path
  WavePlan wp;
  if (n > 1 || tile_mode_ref().load() < 2) {
    std::vector<int64_t> Wv(n), Kv(n);
    for (int i = 0; i < n; ++i) Wv[i] = comps[i].W, Kv[i] = comps[i].K;
    st = wave_plan(n, a, b, Wv.data(), Kv.data(), s, &wp);
    if (st) return st;
  }
  TilePlan tp;
  if (n == 1 && !wp.ok) {  // single large compositions: bottom-up levels, count and emit on the tile kernels
    st = tile_plan(a[0], b[0], pairs, want_prov, s, &tp);
    if (st) return st;
  }
  if (nblocks >= INT32_MAX || nchunks >= INT32_MAX) {
    set_error(FST_E_CAPACITY, "pair space too large (%lld blocks)", (long long)nblocks);
    return FST_E_CAPACITY;
  }
  // ---- workspace
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
  const size_t oR = take(4 * nwords), oV = take(4 * nwords), oF0 = take(4 * nwords), oF1 = take(4 * nwords);
  const size_t ofl0 = take(4 * nchunks), ofl1 = take(4 * nchunks);
  const size_t ol0 = take(4 * nchunks), ol1 = take(4 * nchunks);
  const size_t octrl = take(sizeof(LevelCtrl) * 3);
  const size_t okept = take(8 * nblocks), ovc = take(4 * nblocks), owpre = take(2 * nwords);
  const size_t oid = take(8 * (nblocks + 1)), oarc = take(8 * (nblocks + 1));
  const size_t otmp = take(8 * scan_tmp_elems(nblocks));
  const size_t ohist = take(8 * kMaxLevelStats), omisc = take(8 * 8);
  const size_t ocomps = take(sizeof(CompDev) * n), oseed1 = take(8 * (n + 1)), oseed2 = take(8 * (n + 1));
  const size_t otot = take(8 * 2 * (n + 1));
  const size_t ocnt8 = take(32 * nwords);
  BufferPtr wb;
  st = alloc_buffer(off, s, &wb);
  if (st) {
    if (st == FST_E_OOM) set_error(FST_E_CAPACITY, "pair space workspace (%zu bytes) does not fit", off);
    return st == FST_E_OOM ? FST_E_CAPACITY : st;
  }
  char* base = (char*)wb->ptr;
  Ctx cx{};
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
  cx.cnt8 = (uint8_t*)(base + ocnt8);
  cx.warc = nullptr;  // set after stage 2 when the tile path runs (the push levels use cnt8 until then)
  CompDev* d_comps = (CompDev*)(base + ocomps);
  cx.comps = d_comps;
  cx.ncomp = n;
  for (int i = 0; i < n && i < kCompQ; ++i) cx.compQ[i] = comps[i].Q;
  cx.ptotal = pairs;
  cx.pull_ok = (pull_enabled() && n == 1 && !tp.ok) ? 1 : 0;  // batches are many narrow problems (trellises)
  cx.pull_num = pull_num();
  cx.nwords = nwords;
  cx.nblocks = nblocks;
  cx.nchunks = nchunks;
  cx.seedbase = nullptr;
  cx.OUT = nullptr;
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
  int64_t level_launches = 0;
  std::vector<int64_t> sizes1, sizes2;

  // ---- stage 1: co-accessible set R (backward BFS from accept pairs)
  {
    EventTimer t(prof, s);
    cx.seedbase = d_seed1;
    if (wp.ok) {
      if (seed1[n] > 0) {
        st = wave_stage(wp, 1, cx.R, cx.V, s);
        if (st) return st;
      }
    } else if (seed1[n] > 0) {
      k_seed<false><<<nblk(seed1[n], 256), 256, 0, s>>>(cx);
      FSTC_LAUNCH_CHECK();
      st = tp.ok ? run_stage_tile<false>(cx, tp, pairs, s, hp, &level_launches, &sizes1, &stats.pull_levels)
                 : run_stage<false>(cx, s, hp, &level_launches, &sizes1);
      if (st) return st;
    }
    stats.levels_stage1 = wp.ok ? wp.depth : (int32_t)sizes1.size();
    stats.ms_stage1 = t.stop();
  }
  // ---- stage 2: accessible states restricted to R (forward BFS from start pairs)
  FSTC_CUDA_TRY(cudaMemsetAsync(base + octrl, 0, sizeof(LevelCtrl) * 3, s));
  FSTC_CUDA_TRY(cudaMemsetAsync(base + omisc, 0, 8, s));
  {
    EventTimer t(prof, s);
    cx.seedbase = d_seed2;
    if (wp.ok) {
      if (seed2[n] > 0 && seed1[n] > 0) {
        // the pass-1 counts need only R: they run on a side stream concurrently with stage 2 (on the SMs
        // its clusters leave idle); the block sums over V join after stage 2
        cudaStream_t s2 = side_stream(s);
        if (!s2) {
          set_error(FST_E_CUDA, "side stream creation failed");
          return FST_E_CUDA;
        }
        cudaEvent_t e1 = nullptr, e2 = nullptr;
        FSTC_CUDA_TRY(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
        FSTC_CUDA_TRY(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
        FSTC_CUDA_TRY(cudaEventRecord(e1, s));
        st = wave_stage(wp, 2, cx.R, cx.V, s);  // first: its clusters take their SMs before the counts
        if (st) return st;
        FSTC_CUDA_TRY(cudaStreamWaitEvent(s2, e1, 0));
        {
          EventTimer tc(prof, s2);
          st = wave_count(wp, cx.R, cx.cnt8, s2);
          if (st) return st;
          FSTC_CUDA_TRY(cudaEventRecord(e2, s2));
          stats.ms_count = tc.stop();
        }
        FSTC_CUDA_TRY(cudaStreamWaitEvent(s, e2, 0));
        cudaEventDestroy(e1);
        cudaEventDestroy(e2);
        st = wave_kept(wp, cx.V, cx.kept, s);
        if (st) return st;
      }
    } else if (seed2[n] > 0 && seed1[n] > 0) {
      k_seed<true><<<nblk(seed2[n], 256), 256, 0, s>>>(cx);
      FSTC_LAUNCH_CHECK();
      if (tp.ok) {
        k_popcount<<<sm_count() * 4, 256, 0, s>>>(cx.R, nwords, cx.misc + 1);  // |R|: stage 2's unvisited set
        FSTC_LAUNCH_CHECK();
        FSTC_CUDA_TRY(cudaMemcpyAsync(hp + 8, cx.misc + 1, 8, cudaMemcpyDeviceToHost, s));
        FSTC_CUDA_TRY(cudaStreamSynchronize(s));
        stats.num_coaccessible = (int64_t)hp[8];
        st = run_stage_tile<true>(cx, tp, (int64_t)hp[8], s, hp, &level_launches, &sizes2, &stats.pull_levels);
      } else {
        st = run_stage<true>(cx, s, hp, &level_launches, &sizes2);
      }
      if (st) return st;
    }
    if (tp.ok) {  // pass-1 counts of every block (the bottom-up levels do not count)
      EventTimer tc(prof, s);
      cx.warc = (uint32_t*)cx.cnt8;
      launch_tile_count(tp.cnt, tp.grid_count, tp.smem_count, s, cx);
      FSTC_LAUNCH_CHECK();
      stats.ms_count = tc.stop();
    }
    stats.levels_stage2 = wp.ok ? wp.depth : (int32_t)sizes2.size();
    stats.ms_stage2 = t.stop();
  }
  // ---- numbering: per-block state counts, word prefixes, scans, per-composition totals
  std::vector<int64_t> tot(2 * (n + 1));
  std::vector<fst*> outs(n, nullptr);
  auto cleanup = [&]() {
    for (auto*& h : outs) {
      delete h;
      h = nullptr;
    }
  };
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
    if (prof && !tp.ok) {
      k_popcount<<<sm_count() * 4, 256, 0, s>>>(cx.R, nwords, cx.misc + 1);
      FSTC_LAUNCH_CHECK();
    }
    FSTC_CUDA_TRY(cudaMemcpyAsync(tot.data(), d_tot, 8 * 2 * (n + 1), cudaMemcpyDeviceToHost, s));
    FSTC_CUDA_TRY(cudaMemcpyAsync(hp + 1, cx.misc + 1, 8, cudaMemcpyDeviceToHost, s));
    FSTC_CUDA_TRY(cudaStreamSynchronize(s));
    if (prof || tp.ok) stats.num_coaccessible = (int64_t)hp[1];
    stats.ms_number = t.stop();
  }
  // ---- output allocation (one buffer per composition)
  {
    EventTimer t(prof, s);
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
      const size_t o_xa = want_prov ? tk(4 * ne) : 0, o_xb = want_prov ? tk(4 * ne) : 0;
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
      if (want_prov) {
        h->arc_a = (int32_t*)(pb + o_xa);
        h->arc_b = (int32_t*)(pb + o_xb);
      }
      h->src_arcs_a = a[i]->E;
      h->src_arcs_b = b[i]->E;
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
      C.arc_a = h->arc_a;
      C.arc_b = h->arc_b;
    }
    FSTC_CUDA_TRY(cudaMemcpyAsync(d_comps, comps.data(), sizeof(CompDev) * n, cudaMemcpyHostToDevice, s));
    stats.ms_alloc = t.stop();
  }
  // ---- emit
  {
    EventTimer te(prof, s);
    if (tp.ok) {
      launch_tile_emit(tp.emit, tp.grid_emit, tp.smem_emit, s, cx, comps[0], d_tot, tp.vr_rows);
      FSTC_LAUNCH_CHECK();
    } else if (wp.ok && wp.emit_ok && !want_prov && [&] {  // the wave emit indexes a composition's arcs with 32 bits
                 for (int i = 0; i < n; ++i)
                   if (tot[2 * i + 3] - tot[2 * i + 1] >= INT32_MAX) return false;
                 return true;
               }()) {
      st = wave_emit(wp, d_comps, d_tot, cx.idbase, cx.arcbase, cx.wpre, cx.V, (int32_t*)(cx.misc + 2), s);
      if (st) {
        cleanup();
        return st;
      }
    } else {
      k_emit<<<g_grid, kThreads, kDynSmem, s>>>(cx, d_tot);
      FSTC_LAUNCH_CHECK();
    }
    stats.ms_emit = te.stop();
    k_finish_rowptr<<<nblk(n, 128), 128, 0, s>>>(cx, d_tot);
    FSTC_LAUNCH_CHECK();
    FSTC_CUDA_TRY(cudaMemcpyAsync(hp + 2, cx.misc + 2, 16, cudaMemcpyDeviceToHost, s));
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      cleanup();
      set_error(FST_E_CUDA, "compose: %s", cudaGetErrorString(e));
      return FST_E_CUDA;
    }
    if (hp[2] != 0) {
      cleanup();
      set_error(FST_E_INTERNAL, "emit/count mismatch in %llu blocks", hp[2]);
      return FST_E_INTERNAL;
    }
    stats.staged_tasks = wp.ok ? wp.cluster : (int64_t)hp[3];
  }
  wb.reset();
  stats.ms_total = t_total.stop();
  stats.launches = fst_launch_count() - launches0;
  stats.expand_launches = level_launches;
  stats.emit_launches = 1;
  stats.tile_path = tp.ok ? 1 : (wp.ok ? 2 : 0);
  for (int i = 0; i < n; ++i) {
    outs[i]->stats = stats;
    level_sizes_slot(outs[i], 1) = sizes1;
    level_sizes_slot(outs[i], 2) = sizes2;
    c[i] = outs[i];
  }
  return FST_OK;
}


fst_status compose_impl(int32_t n, const fst_handle* a, const fst_handle* b, cudaStream_t s, fst_handle* c,
                        uint32_t flags) {
  return compose_run(n, a, b, s, c, flags);
}
}  // namespace fstc

namespace fstc {
// ------------------------------------------------------------------------------ gradient scatter
// dL/dw_a[i] += sum of dL/dw_c over the arcs of C with arc_a == i (w_c = w_a + w_b, or a copy), and
// the same for B.  One thread per composed arc, float atomics.
__global__ void k_grad_scatter(int64_t E, const int32_t* __restrict__ arc_a, const int32_t* __restrict__ arc_b,
                               const float* __restrict__ g, float* __restrict__ ga, float* __restrict__ gb) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < E; k += (int64_t)gridDim.x * blockDim.x) {
    const float x = __ldg(&g[k]);
    const int32_t i = __ldg(&arc_a[k]), j = __ldg(&arc_b[k]);
    if (ga && i >= 0) atomicAdd(&ga[i], x);
    if (gb && j >= 0) atomicAdd(&gb[j], x);
  }
}

fst_status grad_scatter_impl(fst* c, const float* grad_c, float* grad_a, int64_t n_a, float* grad_b, int64_t n_b,
                             cudaStream_t s) {
  if (!c || !c->composed || !c->arc_a) {
    set_error(FST_E_INVALID_ARG, "fst_grad_scatter: handle was not composed with FST_COMPOSE_PROVENANCE");
    return FST_E_INVALID_ARG;
  }
  if ((c->E > 0 && !grad_c) || (grad_a && n_a < c->src_arcs_a) || (grad_b && n_b < c->src_arcs_b)) {
    set_error(FST_E_INVALID_ARG, "fst_grad_scatter: NULL grad_c or gradient buffer shorter than the input's arcs");
    return FST_E_INVALID_ARG;
  }
  if (c->E == 0 || (!grad_a && !grad_b)) return FST_OK;
  const unsigned grid = (unsigned)std::min<int64_t>((c->E + 255) / 256, 148 * 16);
  k_grad_scatter<<<grid, 256, 0, s>>>(c->E, c->arc_a, c->arc_b, grad_c, grad_a, grad_b);
  FSTC_LAUNCH_CHECK();
  // the scatter reads c's arc_a / arc_b asynchronously on s: fst_free(c) makes the release of c's
  // buffers wait for it (the buffers are released stream-ordered on the stream that allocated them)
  if (s != c->stream) {
    cudaEvent_t ev;
    FSTC_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    FSTC_CUDA_TRY(cudaEventRecord(ev, s));
    c->use_events.push_back(ev);
  }
  return FST_OK;
}
}  // namespace fstc

// =============================================================================================
// Sharded single composition: the pair-space rows (states of A) are split into
// `world` contiguous ranges, one per shard.  Every BFS level each shard expands the frontier of its
// own rows; claims that land in rows of another shard go to its OUT bitmap, are delivered to the
// owner (all-to-all of row slices) and claimed there by k_apply_remote.  After each stage the owned
// slices of R (stage 1) and V + the per-block arc counts (stage 2) are replicated (NCCL: all-reduce
// sum of disjoint bits == OR), so numbering is global and the emit of each shard's rows is local,
// with global state ids.  The shards' outputs concatenated in rank order are the unsharded result.
// Transports: NCCL (one process per GPU; fst_compose_sharded) or all shards in this process on one
// device (fst_compose_sharded_local, the same kernels and slices moved by device copies).
#include <dlfcn.h>

#include "nccl_dl.h"

namespace fstc {

const NcclApi* nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = (int (*)(ncclUniqueId*))dlsym(h, "ncclGetUniqueId");
      api.CommInitRank = (int (*)(ncclComm_t*, int, ncclUniqueId, int))dlsym(h, "ncclCommInitRank");
      api.CommDestroy = (int (*)(ncclComm_t))dlsym(h, "ncclCommDestroy");
      api.AllReduce = (int (*)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t))dlsym(h, "ncclAllReduce");
      api.Send = (int (*)(const void*, size_t, int, int, ncclComm_t, cudaStream_t))dlsym(h, "ncclSend");
      api.Recv = (int (*)(void*, size_t, int, int, ncclComm_t, cudaStream_t))dlsym(h, "ncclRecv");
      api.GroupStart = (int (*)())dlsym(h, "ncclGroupStart");
      api.GroupEnd = (int (*)())dlsym(h, "ncclGroupEnd");
      api.GetErrorString = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
      api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.Send && api.Recv &&
               api.GroupStart && api.GroupEnd;
    }
  }
  if (!api.ok) {
    set_error(FST_E_NCCL, "NCCL (libnccl.so.2) is not available in this process");
    return nullptr;
  }
  return &api;
}

#define FSTC_NCCL_TRY(expr)                                                                      \
  do {                                                                                           \
    int _r = (expr);                                                                             \
    if (_r != 0) {                                                                               \
      set_error(FST_E_NCCL, "%s failed: %s", #expr, nc->GetErrorString ? nc->GetErrorString(_r) : "?"); \
      return FST_E_NCCL;                                                                         \
    }                                                                                            \
  } while (0)

namespace {

struct Shard {
  int rank = 0;
  BufferPtr wb;
  Ctx cx{};
  CompDev comp{};
  CompDev* d_comp = nullptr;
  int64_t *d_seed1 = nullptr, *d_seed2 = nullptr, *d_tot = nullptr, *d_tmp = nullptr;
  uint32_t* recv = nullptr;  // NCCL: one packed slice per peer (received claims in this rank's blocks)
  uint32_t* send = nullptr;  // NCCL: one packed slice per peer (claims in the peer's blocks)
  int64_t *om_vals = nullptr, *om_ids = nullptr, *om_arcs = nullptr;  // owner-major numbering scratch
  unsigned long long* d_cnt = nullptr;
  char* base = nullptr;
  size_t zero_lo = 0, zero_hi = 0, o_ctrl = 0, o_kept = 0, o_misc = 0;
  std::vector<int64_t> sizes1, sizes2;
  fst* out = nullptr;
};

}  // namespace

fst_status compose_sharded_impl(fst* A, fst* B, int world, fst_comm* comm, cudaStream_t s, fst_handle* c) {
  const bool local = comm == nullptr;
  const NcclApi* nc = nullptr;
  if (!local) {
    nc = nccl_api();
    if (!nc) return FST_E_NCCL;
    world = comm->world;
  }
  if (world < 1) {
    set_error(FST_E_INVALID_ARG, "sharded compose: world must be >= 1");
    return FST_E_INVALID_ARG;
  }
  fst_status st = ensure_views(A, s);
  if (st) return st;
  st = ensure_views(B, s);
  if (st) return st;
  st = init_kernels();
  if (st) return st;
  const bool prof = profiling_enabled();
  EventTimer t_total(prof, s);
  const int64_t launches0 = fst_launch_count();
  // ---- layout (one composition), chunks sized for the shard's share of rows
  CompDev C0;
  memset(&C0, 0, sizeof(C0));
  auto vd = [](const View& v) {
    return ViewDev{v.off, v.key, v.other, v.carry, v.w, v.cw, v.ikd, v.isrc, v.ikcw,
                   v.lm_other, v.lm_pos, v.seg_node, v.seg_beg, v.lab_val, v.lab_seg, v.nlab, v.arc};
  };
  C0.Af = vd(A->views[kOutByOlabel]);
  C0.Ab = vd(A->views[kInByOlabel]);
  C0.Bf = vd(B->views[kOutByIlabel]);
  C0.Bb = vd(B->views[kInByIlabel]);
  C0.startA = A->is_start; C0.startB = B->is_start; C0.accA = A->is_accept; C0.accB = B->is_accept;
  C0.startListA = A->start_list; C0.startListB = B->start_list;
  C0.accListA = A->accept_list; C0.accListB = B->accept_list;
  C0.nStartA = A->n_start; C0.nStartB = B->n_start; C0.nAccA = A->n_accept; C0.nAccB = B->n_accept;
  C0.VA = A->V;
  C0.VB = B->V;
  C0.wpr = (B->V + 31) / 32;
  C0.bpr = (C0.wpr + kWordsPerBlock - 1) / kWordsPerBlock;
  C0.sh_world = world;
  // compositions that fit the tile path are sharded by contiguous row ranges (each rank's tiles are its
  // own; ids stay in key order); the others by interleaved blocks (trellis rows spread over all ranks)
  TilePlan tp;
  st = tile_plan(A, B, (int64_t)A->V * B->V, false, s, &tp);
  if (st) return st;
  C0.sh_rows = tp.ok ? 1 : 0;
  if (C0.sh_rows) {  // chunks as in the unsharded call, for the rows of one rank
    const int64_t rows = std::max<int64_t>(1, C0.VA / world);
    int64_t want = (8ll * g_grid + rows - 1) / rows;
    int32_t cpr = (int32_t)std::max<int64_t>(1, std::min<int64_t>(want, C0.bpr));
    cpr = std::max<int32_t>(cpr, (C0.bpr + kChunkMaxBlocks - 1) / kChunkMaxBlocks);
    C0.CB = std::max<int32_t>(1, (C0.bpr + cpr - 1) / cpr);
    C0.cpr = std::max<int32_t>(1, (C0.bpr + C0.CB - 1) / C0.CB);
  } else {  // one block per chunk: a chunk then has a single owner
    C0.CB = 1;
    C0.cpr = C0.bpr;
  }
  C0.smallA = A->max_olabel < 63;
  const int64_t nwords = (int64_t)C0.VA * C0.wpr, nblocks = (int64_t)C0.VA * C0.bpr,
                nchunks = (int64_t)C0.VA * C0.cpr;
  if (nblocks >= INT32_MAX || nchunks >= INT32_MAX) {
    set_error(FST_E_CAPACITY, "pair space too large (%lld blocks)", (long long)nblocks);
    return FST_E_CAPACITY;
  }
  const int64_t seed1 = (int64_t)C0.nAccA * C0.nAccB, seed2 = (int64_t)C0.nStartA * C0.nStartB;
  if (world > 16) {
    set_error(FST_E_INVALID_ARG, "sharded compose: at most 16 shards");
    return FST_E_INVALID_ARG;
  }
  // blocks of rank q (owner_block / owner_nblocks); owner-major positions [om_start(q), +om_n(q))
  auto om_n = [&](int q) { return owner_nblocks(C0, q); };
  auto om_start = [&](int q) {
    int64_t st0 = 0;
    for (int r = 0; r < q; ++r) st0 += om_n(r);
    return st0;
  };
  const int omG = C0.sh_rows ? 1 : world;  // owner-major order == block order in rows mode
  int64_t slot = 0;  // packed words per peer
  for (int q = 0; q < world; ++q) slot = std::max<int64_t>(slot, om_n(q) * 32);
  unsigned long long* hp = pinned_scratch();
  if (!hp) {
    set_error(FST_E_CUDA, "cudaMallocHost failed");
    return FST_E_CUDA;
  }
  // ---- shards hosted by this process
  std::vector<Shard> sh(local ? world : 1);
  for (size_t i = 0; i < sh.size(); ++i) {
    Shard& S = sh[i];
    S.rank = local ? (int)i : comm->rank;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
    const size_t oR = take(4 * nwords), oV = take(4 * nwords), oF0 = take(4 * nwords), oF1 = take(4 * nwords);
    const size_t ofl0 = take(4 * nchunks), ofl1 = take(4 * nchunks);
    const size_t oOUT = take(4 * nwords);
    const size_t ol0 = take(4 * nchunks), ol1 = take(4 * nchunks);
    const size_t octrl = take(sizeof(LevelCtrl) * 3);
    const size_t okept = take(8 * nblocks), ovc = take(4 * nblocks), owpre = take(2 * nwords);
    const size_t oid = take(8 * (nblocks + 1)), oarc = take(8 * (nblocks + 1));
    const size_t otmp = take(8 * scan_tmp_elems(nblocks));
    const size_t ohist = take(8 * kMaxLevelStats), omisc = take(8 * 8);
    const size_t ocomps = take(sizeof(CompDev)), oseed1 = take(16), oseed2 = take(16), otot = take(8 * 4);
    const size_t ocnt8 = take(32 * nwords), ocnt = take(8);
    const size_t orecv = take(local ? 4 : 4 * (size_t)world * slot), osend = take(local ? 4 * (size_t)slot : 4 * (size_t)world * slot);
    const size_t oomv = take(8 * (nblocks + 1)), oomi = take(8 * (nblocks + 1)), oomk = take(8 * (nblocks + 1));
    st = alloc_buffer(off, s, &S.wb);
    if (st) return st == FST_E_OOM ? FST_E_CAPACITY : st;
    char* base = (char*)S.wb->ptr;
    S.base = base;
    Ctx& cx = S.cx;
    cx.R = (uint32_t*)(base + oR);
    cx.V = (uint32_t*)(base + oV);
    cx.F0 = (uint32_t*)(base + oF0);
    cx.F1 = (uint32_t*)(base + oF1);
    cx.flag0 = (uint32_t*)(base + ofl0);
    cx.flag1 = (uint32_t*)(base + ofl1);
    cx.OUT = (uint32_t*)(base + oOUT);
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
    cx.cnt8 = (uint8_t*)(base + ocnt8);
    S.d_comp = (CompDev*)(base + ocomps);
    cx.comps = S.d_comp;
    cx.ncomp = 1;
    cx.nwords = nwords;
    cx.nblocks = nblocks;
    cx.nchunks = nchunks;
    S.d_seed1 = (int64_t*)(base + oseed1);
    S.d_seed2 = (int64_t*)(base + oseed2);
    S.d_tot = (int64_t*)(base + otot);
    S.d_tmp = (int64_t*)(base + otmp);
    S.d_cnt = (unsigned long long*)(base + ocnt);
    S.recv = (uint32_t*)(base + orecv);
    S.send = (uint32_t*)(base + osend);
    S.om_vals = (int64_t*)(base + oomv);
    S.om_ids = (int64_t*)(base + oomi);
    S.om_arcs = (int64_t*)(base + oomk);
    S.zero_lo = oR;
    S.zero_hi = ol0;
    S.o_ctrl = octrl;
    S.o_kept = okept;
    S.o_misc = omisc;
    S.comp = C0;
    S.comp.sh_rank = S.rank;
    S.comp.sh_r0 = sh_row0(C0, S.rank);
    S.comp.sh_r1 = sh_row0(C0, S.rank + 1);
    FSTC_CUDA_TRY(cudaMemsetAsync(base + oR, 0, ol0 - oR, s));  // bitmaps, flags, OUT
    FSTC_CUDA_TRY(cudaMemsetAsync(base + octrl, 0, sizeof(LevelCtrl) * 3, s));
    FSTC_CUDA_TRY(cudaMemsetAsync(base + okept, 0, 8 * nblocks, s));
    FSTC_CUDA_TRY(cudaMemsetAsync(base + omisc, 0, 64, s));
    FSTC_CUDA_TRY(cudaMemcpyAsync(S.d_comp, &S.comp, sizeof(CompDev), cudaMemcpyHostToDevice, s));
    int64_t sd1[2] = {0, seed1}, sd2[2] = {0, seed2};
    FSTC_CUDA_TRY(cudaMemcpyAsync(S.d_seed1, sd1, 16, cudaMemcpyHostToDevice, s));
    FSTC_CUDA_TRY(cudaMemcpyAsync(S.d_seed2, sd2, 16, cudaMemcpyHostToDevice, s));
  }
  const unsigned agrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nblk(slot, 256), 8 * sm_count()));
  // replicate a bitmap (uint32 words over the whole pair space): every shard gets the owners' blocks
  auto replicate_bits = [&](uint32_t* Shard::*dummy, bool isR) -> fst_status {
    (void)dummy;
    if (local) {
      if (world > 1) {
        ShardPtrs src{};
        for (auto& Sq : sh) src.p[Sq.rank] = isR ? Sq.cx.R : Sq.cx.V;
        for (auto& Sr : sh) {
          k_gather_owned<<<nblk(nwords, 256) < 8u * sm_count() ? nblk(nwords, 256) : 8u * sm_count(), 256, 0, s>>>(
              Sr.d_comp, src, isR ? Sr.cx.R : Sr.cx.V);
          FSTC_LAUNCH_CHECK();
        }
      }
    } else if (world > 1) {
      uint32_t* p = isR ? sh[0].cx.R : sh[0].cx.V;
      k_mask_unowned<<<8 * sm_count(), 256, 0, s>>>(sh[0].d_comp, p);  // others' (stale) copies out
      FSTC_LAUNCH_CHECK();
      FSTC_NCCL_TRY(nc->AllReduce(p, p, (size_t)nwords, kNcclUint32, kNcclSum, comm->comm, s));
    }
    return FST_OK;
  };
  // tile ranges of every shard: the tiles over its rows
  auto tile_range = [&](const TileArgs& ta0, const fst* Ah, int which, const Shard& S) {
    TileArgs ta = ta0;
    if (world > 1) {
      const std::vector<int32_t>* tr = nullptr;
      for (const auto& r : Ah->tile_rows)
        if (r.d == ta0.trow) tr = &r.h;
      const int32_t lo = sh_row0(C0, S.rank), hi = sh_row0(C0, S.rank + 1);
      int t0 = 0, t1 = 0;
      if (tr && hi > lo) {
        t0 = (int)(std::upper_bound(tr->begin(), tr->end(), lo) - tr->begin()) - 1;
        t1 = (int)(std::lower_bound(tr->begin(), tr->end(), hi) - tr->begin());
      }
      ta.t0 = std::max(0, t0);
      ta.t1 = std::min(ta0.ntiles, std::max(ta.t0, t1));
    }
    (void)which;
    return ta;
  };
  const int64_t K_pull = tile_pull_k();
  fst_compose_stats stats{};
  stats.pair_space = (int64_t)C0.VA * C0.VB;
  stats.num_coaccessible = -1;
  int64_t level_launches = 0;
  // ---- one stage: seeds, then levels with an exchange after each
  auto run_stage_sharded = [&](bool stage2) -> fst_status {
    for (auto& S : sh) {
      S.cx.seedbase = stage2 ? S.d_seed2 : S.d_seed1;
      FSTC_CUDA_TRY(cudaMemsetAsync(S.base + S.o_ctrl, 0, sizeof(LevelCtrl) * 3, s));
      FSTC_CUDA_TRY(cudaMemsetAsync(S.base + S.o_misc, 0, 8, s));
      const int64_t ns = stage2 ? seed2 : seed1;
      if (ns > 0) {
        if (stage2) k_seed<true><<<nblk(ns, 256), 256, 0, s>>>(S.cx);
        else k_seed<false><<<nblk(ns, 256), 256, 0, s>>>(S.cx);
        FSTC_LAUNCH_CHECK();
      }
    }
    if ((stage2 ? seed2 : seed1) == 0 || (stage2 && seed1 == 0)) return FST_OK;
    // pairs of the stage (direction choice on the tile path): the pair space, then |R|
    int64_t stage_total = (int64_t)C0.VA * C0.VB;
    if (stage2 && tp.ok) {
      FSTC_CUDA_TRY(cudaMemsetAsync(sh[0].cx.misc + 1, 0, 8, s));
      k_popcount<<<sm_count() * 4, 256, 0, s>>>(sh[0].cx.R, nwords, sh[0].cx.misc + 1);  // R is replicated
      FSTC_LAUNCH_CHECK();
      FSTC_CUDA_TRY(cudaMemcpyAsync(hp + 8, sh[0].cx.misc + 1, 8, cudaMemcpyDeviceToHost, s));
      FSTC_CUDA_TRY(cudaStreamSynchronize(s));
      stage_total = (int64_t)hp[8];
    }
    unsigned long long nf_global = stage2 ? seed2 : seed1;  // (an upper bound for level 0)
    bool replicated = false;  // vis complete on every shard (after a bottom-up round)
    for (int level = 0;; ++level) {
      const bool pull = tp.ok && (int64_t)nf_global * K_pull >= stage_total;
      if (pull) {
        if (!replicated) {  // a round tests against the whole visited set
          st = replicate_bits(nullptr, !stage2);
          if (st) return st;
        }
        for (auto& S : sh) {
          const TileArgs ta = tile_range(stage2 ? tp.s2 : tp.s1, A, stage2 ? 1 : 0, S);
          if (stage2) launch_tile_pull<true>(ta, tp.grid_pull2, tp.smem_pull, s, S.cx, level);
          else launch_tile_pull<false>(ta, tp.grid_pull1, tp.smem_pull, s, S.cx, level);
          FSTC_LAUNCH_CHECK();
          ++level_launches;
          ++stats.pull_levels;
        }
        // the round's claims (own rows only) -> every shard
        st = replicate_bits(nullptr, !stage2);
        if (st) return st;
        replicated = true;
      } else {
      for (auto& S : sh) {
        if (stage2) k_level<true><<<g_grid, kThreads, kDynSmem, s>>>(S.cx, level);
        else k_level<false><<<g_grid, kThreads, kDynSmem, s>>>(S.cx, level);
        FSTC_LAUNCH_CHECK();
        ++level_launches;
      }
      replicated = false;
      // deliver the claims in other shards' blocks to their owners, who claim them: in-process shards
      // read each other's OUT bitmaps; NCCL ranks pack the OUT words of every peer's blocks into one
      // slice per peer and exchange them (grouped send / recv = all-to-all)
      if (local) {  // the same packed slices as the NCCL path; the "transport" is the shared device
        for (auto& Sr : sh)
          for (auto& Sq : sh) {
            if (&Sr == &Sq) continue;
            k_pack_owner<<<agrid, 256, 0, s>>>(Sq.d_comp, Sq.cx.OUT, Sr.rank, Sq.send);
            FSTC_LAUNCH_CHECK();
            if (stage2) k_apply_remote<true><<<agrid, 256, 0, s>>>(Sr.cx, Sq.send, 1, level);
            else k_apply_remote<false><<<agrid, 256, 0, s>>>(Sr.cx, Sq.send, 1, level);
            FSTC_LAUNCH_CHECK();
          }
      } else if (world > 1) {
        Shard& S = sh[0];
        for (int q = 0; q < world; ++q) {
          if (q == S.rank) continue;
          k_pack_owner<<<agrid, 256, 0, s>>>(S.d_comp, S.cx.OUT, q, S.send + (size_t)q * slot);
          FSTC_LAUNCH_CHECK();
        }
        FSTC_NCCL_TRY(nc->GroupStart());
        for (int q = 0; q < world; ++q) {
          if (q == S.rank) continue;
          FSTC_NCCL_TRY(nc->Send(S.send + (size_t)q * slot, (size_t)(om_n(q) * 32), kNcclUint32, q, comm->comm, s));
          FSTC_NCCL_TRY(nc->Recv(S.recv + (size_t)q * slot, (size_t)(om_n(S.rank) * 32), kNcclUint32, q, comm->comm, s));
        }
        FSTC_NCCL_TRY(nc->GroupEnd());
        for (int q = 0; q < world; ++q) {
          if (q == S.rank) continue;
          if (stage2) k_apply_remote<true><<<agrid, 256, 0, s>>>(S.cx, S.recv + (size_t)q * slot, 1, level);
          else k_apply_remote<false><<<agrid, 256, 0, s>>>(S.cx, S.recv + (size_t)q * slot, 1, level);
          FSTC_LAUNCH_CHECK();
        }
      }
      for (auto& S : sh) FSTC_CUDA_TRY(cudaMemsetAsync(S.cx.OUT, 0, 4 * nwords, s));
      }  // push level
      // global size of the next frontier: (active chunks, pairs), summed over the ranks
      unsigned long long total = 0, nfn = 0;
      if (local) {
        for (auto& S : sh) {
          FSTC_CUDA_TRY(cudaMemcpyAsync(hp, &S.cx.ctrl[(level + 1) % 3].count, 16, cudaMemcpyDeviceToHost, s));
          FSTC_CUDA_TRY(cudaStreamSynchronize(s));
          total += hp[0];
          nfn += hp[1];
        }
      } else {
        Shard& S = sh[0];
        FSTC_CUDA_TRY(cudaMemcpyAsync(S.d_cnt, &S.cx.ctrl[(level + 1) % 3].count, 16, cudaMemcpyDeviceToDevice, s));
        FSTC_NCCL_TRY(nc->AllReduce(S.d_cnt, S.d_cnt, 2, kNcclUint64, kNcclSum, comm->comm, s));
        FSTC_CUDA_TRY(cudaMemcpyAsync(hp, S.d_cnt, 16, cudaMemcpyDeviceToHost, s));
        FSTC_CUDA_TRY(cudaStreamSynchronize(s));
        total = hp[0];
        nfn = hp[1];
      }
      nf_global = nfn;
      if (total == 0) {
        for (auto& S : sh) {  // per-level frontier sizes of this shard
          FSTC_CUDA_TRY(cudaMemcpyAsync(hp, S.cx.misc, 8, cudaMemcpyDeviceToHost, s));
          FSTC_CUDA_TRY(cudaStreamSynchronize(s));
          const int n = (int)std::min<unsigned long long>(*hp, kMaxLevelStats);
          std::vector<unsigned long long> tmp(n);
          if (n) {
            FSTC_CUDA_TRY(cudaMemcpyAsync(tmp.data(), S.cx.hist, 8 * n, cudaMemcpyDeviceToHost, s));
            FSTC_CUDA_TRY(cudaStreamSynchronize(s));
          }
          (stage2 ? S.sizes2 : S.sizes1).assign(tmp.begin(), tmp.end());
        }
        break;
      }
    }
    return FST_OK;
  };
  {
    EventTimer t(prof, s);
    st = run_stage_sharded(false);
    if (st) return st;
    st = replicate_bits(nullptr, true);
    if (st) return st;
    stats.ms_stage1 = t.stop();
  }
  {
    EventTimer t(prof, s);
    st = run_stage_sharded(true);
    if (st) return st;
    st = replicate_bits(nullptr, false);
    if (st) return st;
    if (tp.ok) {  // pass-1 counts of the own rows (the bottom-up rounds do not count)
      for (auto& S : sh) {
        S.cx.warc = (uint32_t*)S.cx.cnt8;
        launch_tile_count(tile_range(tp.cnt, A, 0, S), tp.grid_count, tp.smem_count, s, S.cx);
        FSTC_LAUNCH_CHECK();
      }
    }
    // per-block arc counts of the owners' blocks
    if (local) {
      if (world > 1) {
        ShardPtrs64 src{};
        for (auto& Sq : sh) src.p[Sq.rank] = Sq.cx.kept;
        for (auto& Sr : sh) {
          k_gather_owned_blocks<<<nblk(nblocks, 256), 256, 0, s>>>(Sr.d_comp, src, Sr.cx.kept);
          FSTC_LAUNCH_CHECK();
        }
      }
    } else {
      FSTC_NCCL_TRY(nc->AllReduce(sh[0].cx.kept, sh[0].cx.kept, (size_t)nblocks, kNcclUint64, kNcclSum, comm->comm, s));
    }
    stats.ms_stage2 = t.stop();
    stats.levels_stage1 = (int32_t)sh[0].sizes1.size();
    stats.levels_stage2 = (int32_t)sh[0].sizes2.size();
  }
  // ---- numbering (identical on every shard) and per-shard outputs
  std::vector<fst*> outs(sh.size(), nullptr);
  auto cleanup = [&]() {
    for (auto*& h : outs) {
      delete h;
      h = nullptr;
    }
  };
  int64_t total_states = 0, total_arcs = 0;
  for (size_t i = 0; i < sh.size(); ++i) {
    Shard& S = sh[i];
    k_block_counts<<<nblk(nblocks * 32, 256), 256, 0, s>>>(S.cx);
    FSTC_LAUNCH_CHECK();
    // owner-major numbering: scan the per-block counts in (owner, block id) order, then give every
    // block its base (rank q's states / arcs are then the contiguous ranges starting at om_start(q))
    const unsigned gb = nblk(nblocks + 1, 256);
    k_om_gather<int32_t><<<gb, 256, 0, s>>>(S.cx.vcount, nblocks, omG, (int32_t*)S.om_vals);
    FSTC_LAUNCH_CHECK();
    st = exclusive_scan_i32((const int32_t*)S.om_vals, nblocks, S.om_ids, S.d_tmp, s);
    if (st) return st;
    k_om_scatter<<<gb, 256, 0, s>>>(S.om_ids, nblocks, omG, S.cx.idbase);
    FSTC_LAUNCH_CHECK();
    k_om_gather<unsigned long long><<<gb, 256, 0, s>>>(S.cx.kept, nblocks, omG, (unsigned long long*)S.om_vals);
    FSTC_LAUNCH_CHECK();
    st = exclusive_scan_u64((const unsigned long long*)S.om_vals, nblocks, S.om_arcs, S.d_tmp, s);
    if (st) return st;
    k_om_scatter<<<gb, 256, 0, s>>>(S.om_arcs, nblocks, omG, S.cx.arcbase);
    FSTC_LAUNCH_CHECK();
    int64_t hb[6];
    const int64_t p0 = om_start(S.rank), p1 = p0 + om_n(S.rank);
    FSTC_CUDA_TRY(cudaMemcpyAsync(&hb[0], S.om_ids + p0, 8, cudaMemcpyDeviceToHost, s));
    FSTC_CUDA_TRY(cudaMemcpyAsync(&hb[1], S.om_ids + p1, 8, cudaMemcpyDeviceToHost, s));
    FSTC_CUDA_TRY(cudaMemcpyAsync(&hb[2], S.om_arcs + p0, 8, cudaMemcpyDeviceToHost, s));
    FSTC_CUDA_TRY(cudaMemcpyAsync(&hb[3], S.om_arcs + p1, 8, cudaMemcpyDeviceToHost, s));
    FSTC_CUDA_TRY(cudaMemcpyAsync(&hb[4], S.om_ids + nblocks, 8, cudaMemcpyDeviceToHost, s));
    FSTC_CUDA_TRY(cudaMemcpyAsync(&hb[5], S.om_arcs + nblocks, 8, cudaMemcpyDeviceToHost, s));
    FSTC_CUDA_TRY(cudaStreamSynchronize(s));
    total_states = hb[4];
    total_arcs = hb[5];
    const int64_t nv = hb[1] - hb[0], ne = hb[3] - hb[2];
    if (total_states >= INT32_MAX) {
      cleanup();
      set_error(FST_E_CAPACITY, "composition has %lld states (>= 2^31)", (long long)total_states);
      return FST_E_CAPACITY;
    }
    size_t ob = 0;
    auto tk = [&](size_t bytes) { size_t o = ob; ob += (bytes + 255) & ~size_t(255); return o; };
    const size_t o_rp = tk(8 * (nv + 1)), o_il = tk(4 * ne), o_ol = tk(4 * ne), o_d = tk(4 * ne), o_w = tk(4 * ne),
                 o_st = tk(nv), o_ac = tk(nv), o_pa = tk(4 * nv), o_pb = tk(4 * nv);
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
    h->shard_rank = S.rank;
    h->shard_world = world;
    h->shard_state_offset = hb[0];
    h->shard_arc_offset = hb[2];
    // outputs biased so that global state ids / arc slots index the shard's buffers
    const int64_t ida = hb[0], arca = hb[2];
    S.comp.row_ptr = h->row_ptr - ida;
    S.comp.ilabel = h->ilabel - arca;
    S.comp.olabel = h->olabel - arca;
    S.comp.dst = h->dst - arca;
    S.comp.weight = h->weight - arca;
    S.comp.is_start = h->is_start - ida;
    S.comp.is_accept = h->is_accept - ida;
    S.comp.pair_a = h->pair_a - ida;
    S.comp.pair_b = h->pair_b - ida;
    FSTC_CUDA_TRY(cudaMemcpyAsync(S.d_comp, &S.comp, sizeof(CompDev), cudaMemcpyHostToDevice, s));
    int64_t tot[4] = {0, 0, hb[4], hb[5]};
    FSTC_CUDA_TRY(cudaMemcpyAsync(S.d_tot, tot, sizeof(tot), cudaMemcpyHostToDevice, s));
    {
      EventTimer te(prof, s);
      if (tp.ok) launch_tile_emit(tile_range(tp.emit, A, 0, S), tp.grid_emit, tp.smem_emit, s, S.cx, S.comp, S.d_tot,
                                  tp.vr_rows);
      else k_emit<<<g_grid, kThreads, kDynSmem, s>>>(S.cx, S.d_tot);
      FSTC_LAUNCH_CHECK();
      stats.ms_emit += te.stop();
    }
    if (nv > 0) {  // shard-local row_ptr
      k_shift_i64<<<nblk(nv, 256), 256, 0, s>>>(h->row_ptr, nv, arca);
      FSTC_LAUNCH_CHECK();
    }
    FSTC_CUDA_TRY(cudaMemcpyAsync(h->row_ptr + nv, &ne, 8, cudaMemcpyHostToDevice, s));
    FSTC_CUDA_TRY(cudaMemcpyAsync(hp + 2, S.cx.misc + 2, 8, cudaMemcpyDeviceToHost, s));
    FSTC_CUDA_TRY(cudaStreamSynchronize(s));
    if (hp[2] != 0) {
      cleanup();
      set_error(FST_E_INTERNAL, "sharded emit/count mismatch in %llu blocks", hp[2]);
      return FST_E_INTERNAL;
    }
  }
  for (auto& S : sh) S.wb.reset();
  stats.ms_total = t_total.stop();
  stats.launches = fst_launch_count() - launches0;
  stats.expand_launches = level_launches;
  stats.emit_launches = (int64_t)sh.size();
  stats.tile_path = tp.ok ? 1 : 0;
  for (size_t i = 0; i < sh.size(); ++i) {
    outs[i]->stats = stats;
    outs[i]->shard_total_states = total_states;
    outs[i]->shard_total_arcs = total_arcs;
    level_sizes_slot(outs[i], 1) = sh[i].sizes1;
    level_sizes_slot(outs[i], 2) = sh[i].sizes2;
    c[i] = outs[i];
  }
  return FST_OK;
}

}  // namespace fstc
