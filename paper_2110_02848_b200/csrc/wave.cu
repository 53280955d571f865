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
#include <cuda_pipeline.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <functional>
#include <atomic>
#include <vector>

#include "fstc_handle.h"
#include "fstc_internal.cuh"
#include "scan.cuh"
#include "wave.h"

namespace cg = cooperative_groups;

namespace fstc {
namespace {

#ifndef FSTC_WAVE_THREADS  // (build experiments: FSTC_BUILD_DEFS="FSTC_WAVE_THREADS=n" python build.py)
#define FSTC_WAVE_THREADS 512
#endif
constexpr int kWThreads = FSTC_WAVE_THREADS;
constexpr int kWWarps = kWThreads / 32;
#ifndef FSTC_WAVE_WPI
#define FSTC_WAVE_WPI 4
#endif
constexpr int kWpi = FSTC_WAVE_WPI;  // words per warp iteration of the trellis pull
constexpr int kWHeavy = 32;    // B columns with more items (in a direction) are walked by the whole CTA
constexpr int kWSlots = 64;    // A arcs per row (label -> slot masks are 64-bit)
constexpr int kWLab = 256;     // label index = label + 2 (eps = 1); 255 = ELL padding (never set)
#ifndef FSTC_WC_THREADS
#define FSTC_WC_THREADS 256
#endif
#ifndef FSTC_WC_MINB
#define FSTC_WC_MINB 4
#endif
constexpr int kCThreads = FSTC_WC_THREADS; // count CTAs
constexpr int kEpsHub = 64;    // eps in-arcs that make a column an M3 hub (source set kept as a bitmap)
constexpr int kEpsHubMax = 16;

struct WaveDir {  // B role, one direction (view by ilabel)
  const uint32_t* ell;   // light columns' non-eps items by word: [(woff[w] + j) * 32 + lane]
  const uint32_t* woff;
  const uint8_t* wmax;
  const uint32_t* eell;  // light columns' eps items, same layout
  const uint32_t* ewoff;
  const uint8_t* ewmax;
  const uint32_t* hmask;
  const int4* heavy;
  int32_t nheavy;
  const uint32_t* hitems; // items of the heavy columns, packed like the ELL (heavy[h].y/.z/.w index them)
  uint32_t blab[8];       // label indices of the light non-eps items
  // [0] (out-view) only, for the emit: (B olabel, weight bits) parallel to ell / eell / hitems, and the
  // heavy columns before each word (heavy index of a column = hbefore[w] + popc(hmask[w] below it))
  const int2* ellcw;
  const int2* eellcw;
  const int2* hcw;
  const uint32_t* hbefore;
  const uint32_t* wo;   // [wpr] woff << 8 | wmax  (the emit: one load per word)
  const uint32_t* ewo;  // [wpr] ewoff << 8 | ewmax
};

struct WaveComp {
  int64_t W, K;      // first word / block of the composition's pair space
  int64_t rowbase;   // first global row (count tasks)
  int64_t hcnt_base; // first entry of the composition's exact heavy-state counts ([row][heavy])
  int32_t VA, VB, wpr, bpr;
  const int32_t* aoff[2];   // A role: [0] out-by-olabel (key = olabel, other = dst), [1] in-by-olabel (other = src)
  const int32_t* akey[2];
  const int32_t* aother[2];
  const uint8_t* startA;
  const uint8_t* accA;
  const uint8_t* startB;
  const uint8_t* accB;
  WaveDir bd[2];     // B role: [0] out-by-ilabel (stage 1, counts), [1] in-by-ilabel (stage 2)
  const int2* eps;   // B arcs with ilabel eps, (src, dst), whose dst is not a hub: the M3 moves
  int32_t neps;
  int32_t nhub;      // hub targets: columns with >= kEpsHub eps in-arcs
  const int32_t* hub_col;
  const uint32_t* hub_src;  // [nhub][wpr] bitmap of each hub's eps sources
  // relevance masks of the M3 passes ([wpr] each): [0] stage 1 arc phase (dsts of non-hub eps arcs),
  // [1] stage 1 hub phase ([0] + hub columns), [2] stage 2 hub phase (eps sources of hubs), [3] stage 2
  // arc phase ([2] + sources of non-hub eps arcs)
  const uint32_t* rel[4];
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
  uint32_t cache_words;  // shared-memory words for the ELL cache of a stage CTA
  long long* probe;      // FSTC_WAVE_PROBE=1: per-cluster cycle counts of the row-step phases (else null)
  int64_t nrows;         // rows of all compositions (count tasks)
  int32_t* hcnt;         // exact kept-move counts of heavy states (the emit's arc offsets)
  // emit inputs (numbering of compose.cu: per-block id / arc bases, per-word popcount prefixes)
  const int64_t* idbase;
  const int64_t* arcbase;
  const uint16_t* wpre;
  int32_t* err;          // emit: heavy-state queue overflow (reported as an internal error)
};

__device__ __forceinline__ uint32_t bit_of(const uint32_t* row, int32_t col) { return (row[col >> 5] >> (col & 31)) & 1u; }
// shared-memory load at a 32-bit shared-window address, for data that does not change while it is read
// (not volatile: the compiler may schedule it freely)
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

// ------------------------------------------------------------------------------ stage kernels
template <bool kS2>
__global__ void __launch_bounds__(kWThreads, 1) k_wave(WaveArgs wa) {
  cg::cluster_group cl = cg::this_cluster();
  const int G = (int)cl.num_blocks(), crank = (int)cl.block_rank();
  extern __shared__ __align__(16) unsigned char wsm[];
  unsigned long long* lm = (unsigned long long*)wsm;  // [kWLab] slots of the A row's arcs by label index
  int32_t* srow = (int32_t*)(lm + kWLab);              // [kWSlots] row at the other end of slot s
  int32_t* misc = srow + kWSlots;                      // [32]: [0] composition, [1] [2] heavy range, [3] cached,
                                                       //       [4..4+G] word ranges of the cluster's CTAs
  uint32_t* lp = (uint32_t*)(misc + 32);               // [8] label indices present in the A row
  const int wprmax = wa.wprmax, rng = (wprmax + G - 1) / G;
  uint32_t* rowbuf = lp + kWLab / 32;                  // [2][wprmax] current / hot row (whole row)
  uint32_t* Rbuf = rowbuf + 2 * wprmax;                // stage 2: [2][wprmax] R of the current / next row
  uint32_t* pullbuf = Rbuf + (kS2 ? 2 * wprmax : 0);   // [2][rng] this CTA's pulled words (read by the cluster)
  uint32_t* wo = pullbuf + 2 * rng;                    // [rng] per word of this CTA: ELL row (relative) << 8 | rows
  uint32_t* cache = wo + rng;                          // this CTA's ELL rows, then its heavy columns' items
  struct ClosurePtrs {
    const uint32_t *S, *Ma, *Mh;
    const int2* E;
    const int32_t* H;
  };
  __shared__ ClosurePtrs cp_;  // the M3 pass's tables (shared or global memory)
  __shared__ uint32_t* peer_row[2][8];  // [buffer][rank]: the cluster CTAs' row buffers (DSMEM)
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
    if (tid == 0) {  // heavy columns inside this CTA's words; cache decision
      int lo = 0, hi = D.nheavy;
      while (lo < hi) { const int m = (lo + hi) >> 1; if (__ldg(&D.heavy[m]).x < w0 * 32) lo = m + 1; else hi = m; }
      const int hl = lo;
      hi = D.nheavy;
      while (lo < hi) { const int m = (lo + hi) >> 1; if (__ldg(&D.heavy[m]).x < w1 * 32) lo = m + 1; else hi = m; }
      misc[1] = hl;
      misc[2] = lo;
      const int64_t nell = (int64_t)(__ldg(&D.woff[w1]) - __ldg(&D.woff[w0])) * 32;
      const int64_t nh = lo > hl ? (int64_t)__ldg(&D.heavy[lo - 1]).w - __ldg(&D.heavy[hl]).y : 0;
      misc[3] = nell + nh <= (int64_t)wa.cache_words ? 1 : 0;
    }
    if (tid <= G) misc[4 + tid] = (int)((int64_t)wpr * tid / G);
    if (tid < 2 * G) peer_row[tid / G][tid % G] = cl.map_shared_rank(rowbuf + (tid / G) * wprmax, tid % G);
    __syncthreads();
    const int h0 = misc[1], h1 = misc[2];
    const bool cached = misc[3] != 0;
    const uint32_t er0 = __ldg(&D.woff[w0]);
    const uint32_t nell = (__ldg(&D.woff[w1]) - er0) * 32u;
    const int32_t hb0 = h1 > h0 ? __ldg(&D.heavy[h0]).y : 0;
    for (int w = w0 + tid; w < w1; w += kWThreads) wo[w - w0] = ((__ldg(&D.woff[w]) - er0) << 8) | __ldg(&D.wmax[w]);
    if (cached) {
      for (uint32_t i = tid; i < nell; i += kWThreads) cache[i] = __ldg(&D.ell[(size_t)er0 * 32 + i]);
      const int32_t nh = h1 > h0 ? __ldg(&D.heavy[h1 - 1]).w - hb0 : 0;
      for (int32_t i = tid; i < nh; i += kWThreads) cache[nell + i] = __ldg(&D.hitems[hb0 + i]);
    }
    // the M3 pass's tables (hub source bitmaps, this stage's two relevance masks, hub columns, the other
    // eps arcs) in shared memory after the ELL cache when they fit (they are read every row step)
    const int neps = C.neps, nhub = C.nhub;
    // (the table pointers live in shared memory: registers are the stage kernels' scarce resource)
    if (tid == 0) {
      cp_.S = C.hub_src;
      cp_.Ma = C.rel[kS2 ? 3 : 0];
      cp_.Mh = C.rel[kS2 ? 2 : 1];
      cp_.E = C.eps;
      cp_.H = C.hub_col;
    }
    {
      const uint32_t used = cached ? nell + (uint32_t)(h1 > h0 ? __ldg(&D.heavy[h1 - 1]).w - hb0 : 0) : 0u;
      const uint64_t need = (uint64_t)nhub * wpr + 2ull * wpr + 2ull * neps + (uint64_t)nhub + 1;  // (+1: alignment)
      if ((neps > 0 || nhub > 0) && used + need <= wa.cache_words) {
        uint32_t* q = cache + used;
        const uint32_t* gMa = C.rel[kS2 ? 3 : 0];
        const uint32_t* gMh = C.rel[kS2 ? 2 : 1];
        for (int i = tid; i < nhub * wpr; i += kWThreads) q[i] = __ldg(&C.hub_src[i]);
        for (int i = tid; i < wpr; i += kWThreads) {
          q[nhub * wpr + i] = __ldg(&gMa[i]);
          q[nhub * wpr + wpr + i] = __ldg(&gMh[i]);
        }
        uint32_t* qa = q + nhub * wpr + 2 * wpr;
        if ((uintptr_t)qa & 7u) ++qa;  // int2 alignment
        int2* qe = (int2*)qa;
        for (int i = tid; i < neps; i += kWThreads) qe[i] = __ldg(&C.eps[i]);
        int32_t* qh = (int32_t*)(qe + neps);
        for (int i = tid; i < nhub; i += kWThreads) qh[i] = __ldg(&C.hub_col[i]);
        __syncthreads();  // (thread 0's global pointers written above are replaced)
        if (tid == 0) {
          cp_.S = q;
          cp_.Ma = q + nhub * wpr;
          cp_.Mh = q + nhub * wpr + wpr;
          cp_.E = qe;
          cp_.H = qh;
        }
      }
    }
    // heavy columns' items: shared memory when cached, else global (generic pointer)
    const uint32_t* hitp = cached ? cache + nell - hb0 : D.hitems;
    // the first row's A arcs and (stage 2) R row are loaded ahead, like every next row's
    int r = kS2 ? 0 : VA - 1;
    int32_t ne0 = 0, nd = 0, nkey = 0, noth = 0;
    if (VA > 0) {
      ne0 = __ldg(&aoff[r]);
      nd = __ldg(&aoff[r + 1]) - ne0;
      if (tid < nd) {
        nkey = __ldg(&akey[ne0 + tid]);
        noth = __ldg(&aother[ne0 + tid]);
      }
      if (kS2) {
        const int64_t rw = W + (int64_t)r * wpr;
        for (int i = tid; i < wpr; i += kWThreads) __pipeline_memcpy_async(&Rbuf[i], &wa.R[rw + i], 4);
        __pipeline_commit();
      }
    }
    for (int i = tid; i < kWLab; i += kWThreads) lm[i] = 0ull;
    if (tid < kWLab / 32) lp[tid] = 0u;
    __syncthreads();
#ifdef FSTC_WAVE_PROBE_BUILD  // per-phase cycle counts (a build with -DFSTC_WAVE_PROBE_BUILD + FSTC_WAVE_PROBE=1)
    long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, pt = clock64();
    const bool probing = wa.probe != nullptr && tid == 0 && crank == 0;
    auto probe = [&](int k) {
      if (probing) {
        const long long x = clock64();
        pc[k] += x - pt;
        pt = x;
      }
    };
#else
    auto probe = [](int) {};
#endif
    int hot = -1, hp = 0, rb = 0;
    for (int step = 0; step < VA; ++step) {
      r = kS2 ? step : VA - 1 - step;
      const int cp = hp ^ 1;
      uint32_t* cur = rowbuf + cp * wprmax;
      const uint32_t* hrow = rowbuf + hp * wprmax;
      const uint32_t* Rrow = Rbuf + rb * wprmax;
      const int64_t rowW = W + (int64_t)r * wpr;
      const int32_t d = nd;
      const int32_t mykey = nkey, myoth = noth;
      if (kS2) __pipeline_wait_prior(0);  // (lm / lp were cleared after the previous step's pull)
      bool slot_hot = true;
      if (tid < d) {
        const int li = mykey + 2;
        srow[tid] = myoth;
        slot_hot = myoth == hot;
        if (li <= 254) {
          atomicOr(&lm[li], 1ull << tid);
          atomicOr(&lp[li >> 5], 1u << (li & 31));
        }
      }
      // uniform row: every A arc of the row leads to the hot row (a trellis) -- a move exists iff the
      // item's label occurs in the row and the target column is set in the hot row
      const bool uni = __syncthreads_and(slot_hot) != 0;
      probe(0);
      const unsigned long long meps = lm[1];  // A arcs with olabel eps: M2 (B stays) and M1 eps:eps
      const bool rowseed = __ldg(&seedA[r]) != 0;
      auto test = [&](int32_t row, int32_t col) -> bool {
        if (row == hot) return bit_of(hrow, col);
        return (__ldcg(&vis[W + (int64_t)row * wpr + (col >> 5)]) >> (col & 31)) & 1u;
      };
      // ---- pull: one warp per word, one lane per column (light columns: items from the ELL)
      auto pull = [&](const uint32_t* __restrict__ ellb, bool smem_items) {
        if (uni && !rowseed) {  // trellis rows: label present in the row AND target set in the hot row
          bool full = true;     // the row has every label of the light items: no label test
#pragma unroll
          for (int k = 0; k < kWLab / 32; ++k) full &= (lp[k] & D.blab[k]) == D.blab[k];
          if (full && meps == 0ull && smem_items) {
            // the common trellis case on 32-bit shared-window addresses computed once (generic pointers
            // cost a window-base computation per access); wo, the item cache and the hot row are not
            // written during the pull
            const uint32_t wo_s = (uint32_t)__cvta_generic_to_shared(wo) - 4u * (uint32_t)w0;
            const uint32_t it_s = (uint32_t)__cvta_generic_to_shared(ellb) + 4u * (uint32_t)lane;
            const uint32_t hr_s = (uint32_t)__cvta_generic_to_shared(hrow);
            // kWpi words per warp iteration: their item -> hot-row load chains are in flight together
            for (int wb = w0 + warp; wb < w1; wb += kWpi * kWWarps) {
              uint32_t x[kWpi], in[kWpi];
              int jm = 0;
#pragma unroll
              for (int u = 0; u < kWpi; ++u) {
                const int w = wb + u * kWWarps;
                x[u] = w < w1 ? lds32(wo_s + 4u * (uint32_t)w) : 0u;
                in[u] = 0u;
                jm = max(jm, (int)(x[u] & 255u));
              }
#pragma unroll 1
              for (int j = 0; j < jm; ++j) {
                uint32_t it[kWpi];
#pragma unroll
                for (int u = 0; u < kWpi; ++u)  // padding (label index 255) never matches
                  it[u] = j < (int)(x[u] & 255u) ? lds32(it_s + ((x[u] >> 8) << 7) + 128u * (uint32_t)j) : 0xFF000000u;
#pragma unroll
                for (int u = 0; u < kWpi; ++u)
                  in[u] |= (it[u] < 0xFF000000u ? lds32(hr_s + (((it[u] & 0xFFFFFFu) >> 5) << 2)) : 0u) >> (it[u] & 31u);
              }
#pragma unroll
              for (int u = 0; u < kWpi; ++u) {
                const int w = wb + u * kWWarps;
                if (w >= w1) break;  // (warp-uniform)
                uint32_t word = __ballot_sync(0xffffffffu, (in[u] & 1u) != 0u);
                if (kS2) word &= Rrow[w];
                if (lane < G) peer_row[cp][lane][w] = word;  // into every cluster CTA's copy of the row
              }
            }
            return;
          }
          for (int w = w0 + warp; w < w1; w += kWWarps) {
            const uint32_t x = wo[w - w0];
            const uint32_t* pe = ellb + (size_t)(x >> 8) * 32 + lane;
            uint32_t in = 0u;
            if (meps != 0ull) {  // M2 (B stays) and M1 eps:eps, all into the hot row
              in = hrow[w] >> lane;
              const uint32_t* ep = D.eell + (size_t)__ldg(&D.ewoff[w]) * 32 + lane;
              for (int j = __ldg(&D.ewmax[w]); j > 0; --j, ep += 32) {
                const uint32_t it = __ldg(ep);  // padding (label index 255) never matches
                in |= (it < 0xFF000000u ? hrow[(it & 0xFFFFFFu) >> 5] : 0u) >> (it & 31u);
              }
            }
            if (full) {
#pragma unroll 1
              for (int j = (int)(x & 255u); j > 0; --j, pe += 32) {
                const uint32_t it = *pe;  // padding (label index 255) never matches
                in |= (it < 0xFF000000u ? hrow[(it & 0xFFFFFFu) >> 5] : 0u) >> (it & 31u);
              }
            } else {
#pragma unroll 1
              for (int j = (int)(x & 255u); j > 0; --j, pe += 32) {
                const uint32_t it = *pe;
                const uint32_t li = it >> 24;
                in |= (lp[li >> 5] >> (li & 31u)) & (hrow[(it & 0xFFFFFFu) >> 5] >> (it & 31u));
              }
            }
            uint32_t word = __ballot_sync(0xffffffffu, (in & 1u) != 0u);
            if (kS2) word &= Rrow[w];
            if (lane < G) peer_row[cp][lane][w] = word;
          }
          return;
        }
        for (int w = w0 + warp; w < w1; w += kWWarps) {
          const int32_t col = w * 32 + lane;
          bool in = false;
          if (col < VB) {
            const bool allowed = kS2 ? ((Rrow[w] >> lane) & 1u) != 0u : true;
            if (allowed) {
              in = rowseed && __ldg(&seedB[col]) != 0;
              if (!in && d > 0) {
                const uint32_t x = wo[w - w0];
                const int jn = (int)(x & 255u);
                const uint32_t* pe = ellb + (size_t)(x >> 8) * 32 + lane;
                for (unsigned long long m = meps; m && !in; m &= m - 1ull) in = test(srow[__ffsll((long long)m) - 1], col);
                if (meps != 0ull) {  // M1 eps:eps
                  const uint32_t* ep = D.eell + (size_t)__ldg(&D.ewoff[w]) * 32 + lane;
                  for (int j = __ldg(&D.ewmax[w]); j > 0 && !in; --j, ep += 32) {
                    const uint32_t it = __ldg(ep);
                    if ((it >> 24) != 1u) continue;
                    for (unsigned long long m = meps; m && !in; m &= m - 1ull)
                      in = test(srow[__ffsll((long long)m) - 1], (int32_t)(it & 0xFFFFFFu));
                  }
                }
                for (int j = 0; j < jn && !in; ++j) {
                  const uint32_t it = pe[j * 32];
                  const int32_t o = (int32_t)(it & 0xFFFFFFu);
                  for (unsigned long long m = lm[it >> 24]; m && !in; m &= m - 1ull)
                    in = test(srow[__ffsll((long long)m) - 1], o);
                }
              }
            }
          }
          const uint32_t word = __ballot_sync(0xffffffffu, in);
          if (lane < G) peer_row[cp][lane][w] = word;
        }
      };
      if (d > 0 || rowseed) {
        if (cached) pull(cache, true);
        else pull(D.ell + (size_t)er0 * 32, false);
      } else {  // no A arcs and no seeds: the row is empty before the M3 pass
        for (int i = tid; i < (w1 - w0) * G; i += kWThreads) peer_row[cp][i % G][w0 + i / G] = 0u;
      }
      // ---- heavy columns of this CTA: the whole CTA walks the column's items
      probe(1);
      if (h1 > h0 && d > 0) {
        __syncthreads();
        for (int h = h0; h < h1; ++h) {
          const int4 hv = __ldg(&D.heavy[h]);
          const int32_t col = hv.x;
          const bool seeded = rowseed && __ldg(&seedB[col]) != 0;
          const bool allowed = kS2 ? bit_of(Rrow, col) != 0u : true;
          const int eb = meps ? hv.y : hv.z;
          if (seeded || !allowed || (eb >= hv.w && !meps)) continue;  // uniform over the CTA
          bool found = false;
          if (tid < kWSlots && ((meps >> tid) & 1ull)) found = test(srow[tid], col);
          for (int e = eb + tid; e < hv.w && !found; e += kWThreads) {
            const uint32_t it = hitp[e];
            const uint32_t li = it >> 24;
            const int32_t o = (int32_t)(it & 0xFFFFFFu);
            if (uni) {
              found = ((lp[li >> 5] >> (li & 31)) & 1u) && bit_of(hrow, o);
            } else {
              for (unsigned long long m = lm[li]; m && !found; m &= m - 1ull) found = test(srow[__ffsll((long long)m) - 1], o);
            }
          }
          if (__syncthreads_or(found) && tid < G) atomicOr(&peer_row[cp][tid][col >> 5], 1u << (col & 31));
        }
      }
      // ---- the cluster barrier publishes the row (pushed into every CTA's copy during the pull)
      // loads for the next row (used next step): its A arcs and, stage 2, its R row -- issued here so that
      // their latency overlaps the cluster barrier and the gather
      if (step + 1 < VA) {
        const int rn = kS2 ? r + 1 : r - 1;
        ne0 = __ldg(&aoff[rn]);
        nd = __ldg(&aoff[rn + 1]) - ne0;
        if (tid < nd) {
          nkey = __ldg(&akey[ne0 + tid]);
          noth = __ldg(&aother[ne0 + tid]);
        }
        if (kS2) {
          const int64_t rw = W + (int64_t)rn * wpr;
          uint32_t* dstR = Rbuf + (rb ^ 1) * wprmax;
          for (int i = tid; i < wpr; i += kWThreads) __pipeline_memcpy_async(&dstR[i], &wa.R[rw + i], 4);
          __pipeline_commit();
        }
      }
      probe(2);
      cl.sync();
      probe(3);
      for (int i = tid; i < kWLab; i += kWThreads) lm[i] = 0ull;  // for the next row (the pulls are done)
      if (tid < kWLab / 32) lp[tid] = 0u;
      // (every CTA pushed its words into all the cluster's copies of the row: the barrier completes them)
      __syncthreads();
      probe(4);
      // ---- M3 fixed point of the row (B's eps-input arcs; A stays).  Hub targets (many eps sources,
      // kept as a bitmap) are word-parallel, the other eps arcs one thread each.  Pass order: stage 2
      // hubs then arcs, stage 1 arcs then hubs; another pass runs only when a new bit could feed a unit
      // already processed in this pass (the relevance masks of DESIGN.md §6c), so lexicon closures take
      // one pass.
      if (neps > 0 || nhub > 0) {
        for (;;) {
          int changed = 0;
          auto arcs = [&]() {
            for (int i = tid; i < neps; i += kWThreads) {
              const int2 a = cp_.E[i];  // B arc a.x -> a.y with ilabel eps
              if (kS2) {  // (r, a.x) in V  =>  (r, a.y) in V  if in R
                if (bit_of(cur, a.x) && !bit_of(cur, a.y) && bit_of(Rrow, a.y)) {
                  atomicOr(&cur[a.y >> 5], 1u << (a.y & 31));
                  if (bit_of(cp_.Ma, a.y)) changed = 1;
                }
              } else {    // (r, a.y) in R  =>  (r, a.x) in R
                if (bit_of(cur, a.y) && !bit_of(cur, a.x)) {
                  atomicOr(&cur[a.x >> 5], 1u << (a.x & 31));
                  if (bit_of(cp_.Ma, a.x)) changed = 1;
                }
              }
            }
          };
          auto hubs = [&]() {
            for (int h = 0; h < nhub; ++h) {
              if (h > 0 || !kS2) __syncthreads();  // (stage 2 starts with the hubs, right after a barrier)
              const int32_t t = cp_.H[h];
              const uint32_t* S = cp_.S + (size_t)h * wpr;
              if (kS2) {  // V(r, t) if some eps source of t is in V (and (r, t) in R)
                if (bit_of(cur, t) || !bit_of(Rrow, t)) continue;  // uniform
                int any = 0;
                for (int i = tid; i < wpr; i += kWThreads) any |= (cur[i] & S[i]) != 0u;
                if (__syncthreads_or(any) && tid == 0) {
                  cur[t >> 5] |= 1u << (t & 31);
                  if (bit_of(cp_.Mh, t)) changed = 1;
                }
              } else {    // R(r, t)  =>  every eps source of t is in R
                if (!bit_of(cur, t)) continue;  // uniform
                for (int i = tid; i < wpr; i += kWThreads) {
                  const uint32_t x = cur[i], y = x | S[i];
                  if (y != x) {
                    cur[i] = y;
                    if ((y & ~x) & cp_.Mh[i]) changed = 1;
                  }
                }
              }
            }
          };
          if (kS2) {
            hubs();
            __syncthreads();
            arcs();
          } else {
            arcs();
            hubs();
          }
          if (!__syncthreads_or(changed)) break;
        }
      }
      probe(5);
      for (int i = w0 + tid; i < w1; i += kWThreads) vis[rowW + i] = cur[i];
      probe(6);
      hot = r;
      hp = cp;
      rb ^= 1;
    }
#ifdef FSTC_WAVE_PROBE_BUILD
    if (probing) {
      const int cid = blockIdx.x / G;
      for (int k = 0; k < 7; ++k) wa.probe[cid * 8 + k] += pc[k];
      wa.probe[cid * 8 + 7] += VA;
    }
#endif
  }
}

// ------------------------------------------------------------------------------ pass-1 counts
// Per pair (a, b) of R: the number of moves into R -- M1 over A's out-arcs x B's out-items, M2 (A eps
// olabel, B stays), M3 (B eps ilabel, A stays) -- as cnt8 (saturated at 255: the general emit recounts
// those) and, for heavy states, exactly (hcnt).  For a state of V the moves into R are its moves into V
// (the target is accessible), i.e. its out-degree in C; the kernel needs only R, so it runs on a second
// stream CONCURRENTLY with stage 2 (on the SMs the stage-2 clusters leave idle), and k_wave_kept sums
// the counts over V.  One CTA per row.
__global__ void __launch_bounds__(kCThreads, FSTC_WC_MINB) k_wave_count(WaveArgs wa) {
  __shared__ unsigned long long lm[kWLab];
  __shared__ uint32_t lc[kWLab];  // uniform rows: popc(lm[li]) (moves per matching item)
  __shared__ int32_t srow[kWSlots];
  __shared__ unsigned long long hsum;
  extern __shared__ uint32_t csm[];  // [wprmax] V of the row's single destination row, [wprmax] V of the row
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarp = kCThreads / 32;
  const uint32_t* __restrict__ Vg = wa.R;  // counts against R (see above)
  uint32_t* Vd = csm;
  uint32_t* Vr = csm + wa.wprmax;
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
    __syncthreads();  // previous task's readers of the shared tables
    for (int i = tid; i < kWLab; i += kCThreads) lm[i] = 0ull;
    const int32_t dr0 = d > 0 ? __ldg(&C.aother[0][e0]) : r;
    __syncthreads();
    bool same = true;
    if (tid < d) {
      const int li = __ldg(&C.akey[0][e0 + tid]) + 2;
      const int32_t o = __ldg(&C.aother[0][e0 + tid]);
      srow[tid] = o;
      same = o == dr0;
      if (li <= 254) atomicOr(&lm[li], 1ull << tid);
    }
    // uniform row: every A arc leads to the same row dr0; its V row and this row's are staged
    const bool uni = __syncthreads_and(same) != 0;
    if (uni) {
      for (int i = tid; i < kWLab; i += kCThreads) lc[i] = (uint32_t)__popcll(lm[i]);
      for (int i = tid; i < wpr; i += kCThreads) {
        Vd[i] = __ldg(&Vg[W + (int64_t)dr0 * wpr + i]);
        Vr[i] = __ldg(&Vg[rowW + i]);
      }
      __syncthreads();
    }
    const unsigned long long meps = lm[1];
    auto inV = [&](int32_t row, int32_t col) -> int {
      return (int)((__ldg(&Vg[W + (int64_t)row * wpr + (col >> 5)]) >> (col & 31)) & 1u);
    };
    const bool line = uni && meps == 0ull;  // trellis rows: straight-line words (<= 1 item of each kind)
    for (int blk = warp; blk < bpr; blk += nwarp) {
      const int wb = blk * 32, nw = min(32, wpr - wb);
      const uint32_t myw = lane < nw ? __ldg(&Vg[rowW + wb + lane]) : 0u;
      const uint32_t myh = lane < nw ? __ldg(&D.hmask[wb + lane]) : 0u;
      const uint32_t myx = lane < nw ? __ldg(&D.wo[wb + lane]) : 0u;
      const uint32_t mye = lane < nw ? __ldg(&D.ewo[wb + lane]) : 0u;
      unsigned long long tot = 0;
      for (int i = 0; i < nw; ++i) {
        const uint32_t vw = __shfl_sync(0xffffffffu, myw, i) & ~__shfl_sync(0xffffffffu, myh, i);
        if (!vw) continue;
        const int w = wb + i;
        const int32_t col = w * 32 + lane;
        const uint32_t xn = __shfl_sync(0xffffffffu, myx, i), xe = __shfl_sync(0xffffffffu, mye, i);
        if (line && (xn & 255u) <= 1u && (xe & 255u) <= 1u) {
          const uint32_t itn = (xn & 255u) ? __ldg(D.ell + (size_t)(xn >> 8) * 32 + lane) : 0xFF000000u;
          const uint32_t ite = (xe & 255u) ? __ldg(D.eell + (size_t)(xe >> 8) * 32 + lane) : 0xFF000000u;
          const int32_t on = (int32_t)(itn & 0xFFFFFFu), oe = (int32_t)(ite & 0xFFFFFFu);
          const int cnt = (int)(lc[itn >> 24] * bit_of(Vd, on)) + ((ite >> 24) == 1u ? (int)bit_of(Vr, oe) : 0);
          wa.cnt8[(rowW + w) * 32 + lane] = ((vw >> lane) & 1u) ? (uint8_t)cnt : (uint8_t)0;
          continue;
        }
        if ((vw >> lane) & 1u) {
          int cnt = 0;
          const int jn = __ldg(&D.wmax[w]), ejn = __ldg(&D.ewmax[w]);
          const uint32_t* __restrict__ pe = D.ell + (size_t)__ldg(&D.woff[w]) * 32 + lane;
          const uint32_t* __restrict__ ep = D.eell + (size_t)__ldg(&D.ewoff[w]) * 32 + lane;
          if (uni) {
            const int ne = (int)__popcll(meps);
            cnt = ne * (int)bit_of(Vd, col);  // M2
            for (int j = 0; j < ejn; ++j) {   // eps items: M1 eps:eps into the destination row, M3 into this row
              const uint32_t it = __ldg(ep + j * 32);
              if ((it >> 24) != 1u) continue;
              const int32_t o = (int32_t)(it & 0xFFFFFFu);
              cnt += ne * (int)bit_of(Vd, o) + (int)bit_of(Vr, o);
            }
            for (int j = 0; j < jn; ++j) {
              const uint32_t it = __ldg(pe + j * 32);
              cnt += (int)(lc[it >> 24] * bit_of(Vd, (int32_t)(it & 0xFFFFFFu)));
            }
          } else {
            for (unsigned long long m = meps; m; m &= m - 1ull) cnt += inV(srow[__ffsll((long long)m) - 1], col);
            for (int j = 0; j < ejn; ++j) {
              const uint32_t it = __ldg(ep + j * 32);
              if ((it >> 24) != 1u) continue;
              const int32_t o = (int32_t)(it & 0xFFFFFFu);
              for (unsigned long long m = meps; m; m &= m - 1ull) cnt += inV(srow[__ffsll((long long)m) - 1], o);
              cnt += inV(r, o);  // M3
            }
            for (int j = 0; j < jn; ++j) {
              const uint32_t it = __ldg(pe + j * 32);
              const int32_t o = (int32_t)(it & 0xFFFFFFu);
              for (unsigned long long m = lm[it >> 24]; m; m &= m - 1ull) cnt += inV(srow[__ffsll((long long)m) - 1], o);
            }
          }
          wa.cnt8[(rowW + w) * 32 + lane] = (uint8_t)min(cnt, 255);
          tot += (unsigned long long)cnt;
        }
      }
      (void)tot;
    }
    if (D.nheavy > 0) {
      for (int h = 0; h < D.nheavy; ++h) {
        const int4 hv = __ldg(&D.heavy[h]);
        const int32_t col = hv.x;
        if (col >= VB || !inV(r, col)) continue;  // uniform
        unsigned long long cnt = 0;
        if (tid < kWSlots && ((meps >> tid) & 1ull)) cnt += inV(srow[tid], col);
        for (int e = hv.y + tid; e < hv.w; e += kCThreads) {
          const uint32_t it = __ldg(&D.hitems[e]);
          const int li = (int)(it >> 24);
          const int32_t o = (int32_t)(it & 0xFFFFFFu);
          for (unsigned long long m = lm[li]; m; m &= m - 1ull) cnt += inV(srow[__ffsll((long long)m) - 1], o);
          if (li == 1) cnt += inV(r, o);
        }
        cnt = warp_sum(cnt);
        if (tid == 0) hsum = 0ull;
        __syncthreads();
        if (lane == 0 && cnt) atomicAdd(&hsum, cnt);
        __syncthreads();
        if (tid == 0) {
          wa.cnt8[(rowW + (col >> 5)) * 32 + (col & 31)] = (uint8_t)min(hsum, 255ull);
          wa.hcnt[C.hcnt_base + (int64_t)r * D.nheavy + h] = (int32_t)hsum;
        }
        __syncthreads();
      }
    }
  }
}

// ------------------------------------------------------------------------------ pass-1 block sums
// kept[block] = sum of the out-degrees in C of the block's states (cnt8 of k_wave_count, exact counts of
// heavy states from hcnt), OVERWRITTEN for every block.  One warp per block.
__global__ void __launch_bounds__(256) k_wave_kept(WaveArgs wa, int64_t nblocks) {
  const int lane = threadIdx.x & 31;
  const int64_t nw_all = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < nblocks; g += nw_all) {
    int lo = 0, hi = wa.ncomp - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (wa.comps[mid].K <= g) lo = mid; else hi = mid - 1;
    }
    const WaveComp& C = wa.comps[lo];
    const int64_t local = g - C.K;
    const int32_t r = (int32_t)(local / C.bpr), j = (int32_t)(local - (int64_t)r * C.bpr);
    const int w = j * 32 + lane;  // one lane per word
    const int64_t rowW = C.W + (int64_t)r * C.wpr;
    const WaveDir& D = C.bd[0];
    unsigned long long tot = 0;
    if (w < C.wpr) {
      const uint32_t hm = __ldg(&D.hmask[w]);
      uint32_t vw = __ldg(&wa.V[rowW + w]);
      if (vw & hm) {  // heavy states of V: exact counts
        const int64_t hb = C.hcnt_base + (int64_t)r * D.nheavy + __ldg(&D.hbefore[w]);
        for (uint32_t m = vw & hm; m; m &= m - 1u)
          tot += (unsigned long long)__ldg(&wa.hcnt[hb + __popc(hm & ((1u << (__ffs(m) - 1)) - 1u))]);
        vw &= ~hm;
      }
      if (vw) {
        const uint4* q = (const uint4*)(wa.cnt8 + (rowW + w) * 32);
        const uint4 c0 = __ldg(q), c1 = __ldg(q + 1);
        const uint32_t cw[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t sel = (vw >> (4 * k)) & 15u;
          if (!sel) continue;
          const uint32_t x = cw[k];
          tot += ((sel & 1u) ? (x & 255u) : 0u) + ((sel & 2u) ? ((x >> 8) & 255u) : 0u) +
                 ((sel & 4u) ? ((x >> 16) & 255u) : 0u) + ((sel & 8u) ? (x >> 24) : 0u);
        }
      }
    }
    tot = warp_sum(tot);
    if (lane == 0) wa.kept[g] = tot;
  }
}

// ------------------------------------------------------------------------------ pass 2: emit
// Writes the composed CSR of every state of C: one CTA per row, one warp per 1024-pair
// block at a time, one lane per column.  A state's arcs are its moves in the general emit's order (M2 in
// A-slot order, then per B item in view order: M1 in slot order, M3 for an eps item), at consecutive
// slots from the block's arc base (exclusive scans: deterministic, no cursor atomics), so the arrays
// equal the level path's.  Rank of a pair = the block's id base + the word's popcount prefix + the
// popcount below it; the row itself and (uniform rows) its single destination row are staged as (V word,
// rank) pairs.  Heavy states (> kWHeavy B arcs) take their exact count from k_wave_count and are written
// by the whole CTA.
#ifndef FSTC_WEM_THREADS
#define FSTC_WEM_THREADS 256
#endif
#ifndef FSTC_WEM_MINB
#define FSTC_WEM_MINB 2
#endif
constexpr int kEmThreads = FSTC_WEM_THREADS;
constexpr int kEmHeavyQ = 256;
__global__ void __launch_bounds__(kEmThreads, FSTC_WEM_MINB) k_wave_emit(WaveArgs wa, const CompDev* __restrict__ cd,
                                                          const int64_t* __restrict__ tot) {
  __shared__ unsigned long long lm[kWLab];
  __shared__ uint32_t lc[kWLab];
  __shared__ int32_t srow[kWSlots], scar[kWSlots];
  __shared__ float sw[kWSlots];
  __shared__ int32_t hq_n, red[kEmThreads / 32 + 1];
  __shared__ int32_t hq_col[kEmHeavyQ], hq_h[kEmHeavyQ];
  __shared__ long long hq_pos[kEmHeavyQ], hq_id[kEmHeavyQ];
  // the task's pointers, in shared memory: held there (global stores cannot alias them) instead of being
  // re-read from the composition descriptors after every store
  struct EmitPtrs {
    int64_t* row_ptr;
    int32_t *dst, *ilabel, *olabel, *pair_a, *pair_b;
    float* weight;
    uint8_t *is_start, *is_accept;
    const uint32_t *ell, *eell, *wo, *ewo, *hmask, *hbefore;
    const int2 *ellcw, *eellcw;
    const int32_t* hcnt;
  };
  __shared__ EmitPtrs P;
  extern __shared__ int2 esm[];  // [wprmax] own row, [wprmax] destination row: (V word, rank of its first pair),
                                 // [wprmax] per-word item metadata (wo, ewo, hmask, hbefore) of B
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarp = kEmThreads / 32;
  const uint32_t* __restrict__ Vg = wa.V;
  int2* Vr = esm;
  int2* Vd = esm + wa.wprmax;
  uint4* wmeta = (uint4*)(esm + 2 * wa.wprmax);
  const uint32_t* wtag = nullptr;  // B whose metadata wmeta holds
  for (int64_t t = blockIdx.x; t < wa.nrows; t += gridDim.x) {
    int ci = 0, hi = wa.ncomp - 1;
    while (ci < hi) {
      const int mid = (ci + hi + 1) >> 1;
      if (wa.comps[mid].rowbase <= t) ci = mid; else hi = mid - 1;
    }
    const WaveComp& C = wa.comps[ci];
    const CompDev& O = cd[ci];
    const int32_t r = (int32_t)(t - C.rowbase);
    const int wpr = C.wpr, bpr = C.bpr;
    const int64_t W = C.W, K = C.K, rowW = W + (int64_t)r * wpr;
    const int64_t id_comp = tot[2 * ci], arc_comp = tot[2 * ci + 1];
    if (__ldg(&wa.idbase[K + (int64_t)r * bpr + bpr]) == __ldg(&wa.idbase[K + (int64_t)r * bpr])) continue;  // no states
    const WaveDir& D = C.bd[0];
    const int32_t e0 = __ldg(&C.aoff[0][r]), d = __ldg(&C.aoff[0][r + 1]) - e0;
    const int32_t dr0 = d > 0 ? __ldg(&C.aother[0][e0]) : r;
    __syncthreads();  // previous task's readers of the shared tables
    for (int i = tid; i < kWLab; i += kEmThreads) lm[i] = 0ull;
    if (tid == 0) {
      hq_n = 0;
      P.row_ptr = O.row_ptr;
      P.dst = O.dst;
      P.ilabel = O.ilabel;
      P.olabel = O.olabel;
      P.pair_a = O.pair_a;
      P.pair_b = O.pair_b;
      P.weight = O.weight;
      P.is_start = O.is_start;
      P.is_accept = O.is_accept;
      P.ell = D.ell;
      P.eell = D.eell;
      P.wo = D.wo;
      P.ewo = D.ewo;
      P.hmask = D.hmask;
      P.hbefore = D.hbefore;
      P.ellcw = D.ellcw;
      P.eellcw = D.eellcw;
      P.hcnt = wa.hcnt + C.hcnt_base + (int64_t)r * D.nheavy;
    }
    __syncthreads();
    bool same = true;
    if (tid < d) {
      const int li = __ldg(&C.akey[0][e0 + tid]) + 2;
      const int32_t o = __ldg(&C.aother[0][e0 + tid]);
      srow[tid] = o;
      scar[tid] = __ldg(&O.Af.carry[e0 + tid]);
      sw[tid] = __ldg(&O.Af.w[e0 + tid]);
      same = o == dr0;
      if (li <= 254) atomicOr(&lm[li], 1ull << tid);
    }
    const bool uni = __syncthreads_and(same) != 0 && dr0 != r;
    for (int i = tid; i < kWLab; i += kEmThreads) lc[i] = (uint32_t)__popcll(lm[i]);
    for (int i = tid; i < wpr; i += kEmThreads) {
      const int64_t bk = K + (int64_t)r * bpr + (i >> 5);
      Vr[i] = make_int2((int32_t)__ldg(&Vg[rowW + i]), (int32_t)(__ldg(&wa.idbase[bk]) - id_comp + __ldg(&wa.wpre[rowW + i])));
      if (uni) {
        const int64_t dW = W + (int64_t)dr0 * wpr;
        const int64_t dk = K + (int64_t)dr0 * bpr + (i >> 5);
        Vd[i] = make_int2((int32_t)__ldg(&Vg[dW + i]), (int32_t)(__ldg(&wa.idbase[dk]) - id_comp + __ldg(&wa.wpre[dW + i])));
      }
    }
    __syncthreads();
    const unsigned long long meps = lm[1];
    const uint8_t stA = __ldg(&C.startA[r]), acA = __ldg(&C.accA[r]);
    // (present, rank) of pair (row, col)
    auto look = [&](int32_t row, int32_t col, int32_t& rank) -> bool {
      const uint32_t lowm = (1u << (col & 31)) - 1u;
      if (row == r || (uni && row == dr0)) {
        const int2 v = (row == r ? Vr : Vd)[col >> 5];
        rank = v.y + __popc((uint32_t)v.x & lowm);
        return ((uint32_t)v.x >> (col & 31)) & 1u;
      }
      const int64_t gw = W + (int64_t)row * wpr + (col >> 5);
      const uint32_t v = __ldg(&Vg[gw]);
      if (!((v >> (col & 31)) & 1u)) return false;
      rank = (int32_t)(__ldg(&wa.idbase[K + (int64_t)row * bpr + (col >> 10)]) - id_comp + __ldg(&wa.wpre[gw]) + __popc(v & lowm));
      return true;
    };
    auto put = [&](int64_t pos, int32_t dst, int32_t il, int32_t ol, float w) {
      __stcs(&P.dst[pos], dst);
      __stcs(&P.ilabel[pos], il);
      __stcs(&P.olabel[pos], ol);
      __stcs(&P.weight[pos], w);
    };
    const uint8_t* __restrict__ startB = C.startB;
    const uint8_t* __restrict__ accB = C.accB;
    auto state_out = [&](int64_t id, int32_t col, int64_t pos) {
      __stcs((long long*)&P.row_ptr[id], (long long)pos);
      __stcs(&P.pair_a[id], r);
      __stcs(&P.pair_b[id], col);
      P.is_start[id] = stA ? __ldg(&startB[col]) : (uint8_t)0;
      P.is_accept[id] = acA ? __ldg(&accB[col]) : (uint8_t)0;
    };
    auto heavy_push = [&](int32_t col, int hidx, int64_t pos) {
      const int q = atomicAdd(&hq_n, 1);
      if (q < kEmHeavyQ) {
        hq_col[q] = col;
        hq_h[q] = hidx;
        hq_pos[q] = pos;
      }
    };
    // trellis rows (every A arc to one row dr0, no eps-output A arcs): M1 = label in the row and target in
    // V(dr0); M3 = eps item with target in V(r)
    const bool fast = uni && meps == 0ull;
    if (fast && wtag != P.wo) {  // per-word item metadata of B (same for every row of a composition)
      __syncthreads();
      for (int w = tid; w < wpr; w += kEmThreads)
        wmeta[w] = make_uint4(__ldg(&P.wo[w]), __ldg(&P.ewo[w]), __ldg(&P.hmask[w]), __ldg(&P.hbefore[w]));
      __syncthreads();
      wtag = P.wo;
    }
    for (int blk = fast ? warp : bpr; blk < bpr; blk += nwarp) {
      int64_t arc = __ldg(&wa.arcbase[K + (int64_t)r * bpr + blk]) - arc_comp;
      uint32_t arc32 = (uint32_t)arc;  // the straight-line words: 32-bit slots (composition arcs < 2^31)
      const int wb = blk * 32, nw = min(32, wpr - wb);
      // software pipeline: the first items (and their (olabel, weight)) of words w + 2, w + 3 are loaded
      // while words w, w + 1 are processed
      uint32_t pn[2], pe0[2];
      int2 pbn[2], pbe[2];
      auto prefetch = [&](int i) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint4 m = i + u < nw ? wmeta[wb + i + u] : make_uint4(0u, 0u, 0u, 0u);
          pn[u] = (m.x & 255u) ? __ldg(P.ell + (size_t)(m.x >> 8) * 32 + lane) : 0xFF000000u;
          pe0[u] = (m.y & 255u) ? __ldg(P.eell + (size_t)(m.y >> 8) * 32 + lane) : 0xFF000000u;
          pbn[u] = (m.x & 255u) ? __ldg(P.ellcw + (size_t)(m.x >> 8) * 32 + lane) : make_int2(0, 0);
          pbe[u] = (m.y & 255u) ? __ldg(P.eellcw + (size_t)(m.y >> 8) * 32 + lane) : make_int2(0, 0);
        }
      };
      // one word, any shape (straight-line or general); advances arc / arc32
      auto one_word = [&](int w, uint32_t n0it, uint32_t e0it, int2 n0bw, int2 e0bw) {
        const int2 vv = Vr[w];
        const uint32_t vw = (uint32_t)vv.x;
        if (!vw) return;
        const int32_t col = w * 32 + lane;
        const uint4 mt = wmeta[w];
        const uint32_t xn = mt.x, xe = mt.y, hm = mt.z;
        const bool has = (vw >> lane) & 1u, heavy = (hm >> lane) & 1u;
        const uint32_t* __restrict__ pe = P.ell + (size_t)(xn >> 8) * 32 + lane;
        const uint32_t* __restrict__ ep = P.eell + (size_t)(xe >> 8) * 32 + lane;
        const int jn = (int)(xn & 255u), ejn = (int)(xe & 255u);
        if (jn <= 1 && ejn <= 1 && !hm) {  // straight-line: at most one eps item (M3) and one item (M1)
          const int32_t oe = (int32_t)(e0it & 0xFFFFFFu), on = (int32_t)(n0it & 0xFFFFFFu);
          const int2 ve = Vr[oe >> 5], vn = Vd[on >> 5];
          const bool he = has && e0it < 0xFF000000u && (((uint32_t)ve.x >> (oe & 31)) & 1u);
          const unsigned long long mn = lm[n0it >> 24];
          const bool hn = has && mn != 0ull && (((uint32_t)vn.x >> (on & 31)) & 1u);
          const int cnt = (int)he + (hn ? (int)lc[n0it >> 24] : 0);
          const int inc = warp_incl_scan(cnt);
          if (has) {
            uint32_t pos = arc32 + (uint32_t)(inc - cnt);
            const uint32_t id = (uint32_t)vv.y + __popc(vw & ((1u << lane) - 1u));
            __stcs((long long*)(P.row_ptr + id), (long long)pos);
            __stcs(P.pair_a + id, r);
            __stcs(P.pair_b + id, col);
            P.is_start[id] = stA ? __ldg(&startB[col]) : (uint8_t)0;
            P.is_accept[id] = acA ? __ldg(&accB[col]) : (uint8_t)0;
            if (he) {
              __stcs(P.dst + pos, ve.y + __popc((uint32_t)ve.x & ((1u << (oe & 31)) - 1u)));
              __stcs(P.ilabel + pos, FST_EPS);
              __stcs(P.olabel + pos, e0bw.x);
              __stcs(P.weight + pos, __int_as_float(e0bw.y));
              ++pos;
            }
            if (hn) {
              const int32_t rk = vn.y + __popc((uint32_t)vn.x & ((1u << (on & 31)) - 1u));
              for (unsigned long long m = mn; m; m &= m - 1ull, ++pos) {
                const int a = __ffsll((long long)m) - 1;
                __stcs(P.dst + pos, rk);
                __stcs(P.ilabel + pos, scar[a]);
                __stcs(P.olabel + pos, n0bw.x);
                __stcs(P.weight + pos, __fadd_rn(sw[a], __int_as_float(n0bw.y)));
              }
            }
          }
          const uint32_t t = (uint32_t)__shfl_sync(0xffffffffu, inc, 31);
          arc32 += t;
          arc += t;
          return;
        }
        int cnt = 0;
        if (has) {
          if (heavy) {
            cnt = __ldg(&P.hcnt[(int)mt.w + __popc(hm & ((1u << lane) - 1u))]);
          } else {
#pragma unroll 1
            for (int j = 0; j < ejn; ++j) {
              const uint32_t it = j == 0 ? e0it : __ldg(ep + j * 32);
              const int32_t o = (int32_t)(it & 0xFFFFFFu);
              if (it < 0xFF000000u) cnt += (int)((((uint32_t)Vr[o >> 5].x) >> (o & 31)) & 1u);
            }
#pragma unroll 1
            for (int j = 0; j < jn; ++j) {
              const uint32_t it = j == 0 ? n0it : __ldg(pe + j * 32);
              const int32_t o = (int32_t)(it & 0xFFFFFFu);
              cnt += (int)(lc[it >> 24] * ((((uint32_t)Vd[o >> 5].x) >> (o & 31)) & 1u));
            }
          }
        }
        const int inc = warp_incl_scan(cnt);
        const int wtot = __shfl_sync(0xffffffffu, inc, 31);
        if (has) {
          int64_t pos = arc + inc - cnt;
          state_out(vv.y + __popc(vw & ((1u << lane) - 1u)), col, pos);
          if (heavy) {
            heavy_push(col, (int)mt.w + __popc(hm & ((1u << lane) - 1u)), pos);
          } else if (cnt) {
#pragma unroll 1
            for (int j = 0; j < ejn; ++j) {  // M3
              const uint32_t it = j == 0 ? e0it : __ldg(ep + j * 32);
              if (it >= 0xFF000000u) continue;
              const int32_t o = (int32_t)(it & 0xFFFFFFu);
              const int2 v = Vr[o >> 5];
              if (!(((uint32_t)v.x >> (o & 31)) & 1u)) continue;
              const int2 bw = j == 0 ? e0bw : __ldg(&P.eellcw[(size_t)(xe >> 8) * 32 + lane + j * 32]);
              put(pos++, v.y + __popc((uint32_t)v.x & ((1u << (o & 31)) - 1u)), FST_EPS, bw.x, __int_as_float(bw.y));
            }
#pragma unroll 1
            for (int j = 0; j < jn; ++j) {  // M1
              const uint32_t it = j == 0 ? n0it : __ldg(pe + j * 32);
              unsigned long long m = lm[it >> 24];
              if (!m) continue;
              const int32_t o = (int32_t)(it & 0xFFFFFFu);
              const int2 v = Vd[o >> 5];
              if (!(((uint32_t)v.x >> (o & 31)) & 1u)) continue;
              const int32_t rk = v.y + __popc((uint32_t)v.x & ((1u << (o & 31)) - 1u));
              const int2 bw = j == 0 ? n0bw : __ldg(&P.ellcw[(size_t)(xn >> 8) * 32 + lane + j * 32]);
              for (; m; m &= m - 1ull) {
                const int a = __ffsll((long long)m) - 1;
                put(pos++, rk, scar[a], bw.x, __fadd_rn(sw[a], __int_as_float(bw.y)));
              }
            }
          }
        }
        arc += wtot;
        arc32 += (uint32_t)wtot;
      };
      // straight-line word (at most one eps item (M3) and one item (M1) per column): its moves
      struct SL {
        bool he, hn;
        int2 ve, vn;
        unsigned long long mn;
        int cnt;
      };
      auto sl_count = [&](int2 vv, uint32_t n0it, uint32_t e0it) -> SL {
        SL q;
        const bool has = ((uint32_t)vv.x >> lane) & 1u;
        const int32_t oe = (int32_t)(e0it & 0xFFFFFFu), on = (int32_t)(n0it & 0xFFFFFFu);
        q.ve = Vr[oe >> 5];
        q.vn = Vd[on >> 5];
        q.he = has && e0it < 0xFF000000u && (((uint32_t)q.ve.x >> (oe & 31)) & 1u);
        q.mn = lm[n0it >> 24];
        q.hn = has && q.mn != 0ull && (((uint32_t)q.vn.x >> (on & 31)) & 1u);
        q.cnt = (int)q.he + (q.hn ? (int)lc[n0it >> 24] : 0);
        return q;
      };
      auto sl_store = [&](int w, int2 vv, const SL& q, uint32_t pos, uint32_t n0it, uint32_t e0it, int2 n0bw, int2 e0bw) {
        const uint32_t vw = (uint32_t)vv.x;
        const int32_t col = w * 32 + lane;
        const uint32_t id = (uint32_t)vv.y + __popc(vw & ((1u << lane) - 1u));
        __stcs((long long*)(P.row_ptr + id), (long long)pos);
        __stcs(P.pair_a + id, r);
        __stcs(P.pair_b + id, col);
        P.is_start[id] = stA ? __ldg(&startB[col]) : (uint8_t)0;
        P.is_accept[id] = acA ? __ldg(&accB[col]) : (uint8_t)0;
        if (q.he) {
          const int32_t oe = (int32_t)(e0it & 0xFFFFFFu);
          __stcs(P.dst + pos, q.ve.y + __popc((uint32_t)q.ve.x & ((1u << (oe & 31)) - 1u)));
          __stcs(P.ilabel + pos, FST_EPS);
          __stcs(P.olabel + pos, e0bw.x);
          __stcs(P.weight + pos, __int_as_float(e0bw.y));
          ++pos;
        }
        if (q.hn) {
          const int32_t on = (int32_t)(n0it & 0xFFFFFFu);
          const int32_t rk = q.vn.y + __popc((uint32_t)q.vn.x & ((1u << (on & 31)) - 1u));
          for (unsigned long long m = q.mn; m; m &= m - 1ull, ++pos) {
            const int a = __ffsll((long long)m) - 1;
            __stcs(P.dst + pos, rk);
            __stcs(P.ilabel + pos, scar[a]);
            __stcs(P.olabel + pos, n0bw.x);
            __stcs(P.weight + pos, __fadd_rn(sw[a], __int_as_float(n0bw.y)));
          }
        }
      };
      prefetch(0);
      for (int i = 0; i < nw; i += 2) {
        const int w = wb + i;
        const bool twoB = i + 1 < nw;
        const uint32_t nA = pn[0], nB = pn[1], eA = pe0[0], eB = pe0[1];
        const int2 bnA = pbn[0], bnB = pbn[1], beA = pbe[0], beB = pbe[1];
        if (i + 2 < nw) prefetch(i + 2);
        const uint4 mA = wmeta[w], mB = twoB ? wmeta[w + 1] : make_uint4(0u, 0u, 0u, 0u);
        const bool sA = (mA.x & 255u) <= 1u && (mA.y & 255u) <= 1u && !mA.z;
        const bool sB = (mB.x & 255u) <= 1u && (mB.y & 255u) <= 1u && !mB.z;
        if (sA && sB) {  // two straight-line words: one warp scan of both counts (16-bit halves)
          const int2 vA = Vr[w], vB = twoB ? Vr[w + 1] : make_int2(0, 0);
          if (!(vA.x | vB.x)) continue;
          const SL qA = sl_count(vA, nA, eA), qB = sl_count(vB, nB, eB);
          const uint32_t pk = (uint32_t)qA.cnt | ((uint32_t)qB.cnt << 16);  // (sums < 32 * 65: no carry)
          const uint32_t inc = warp_incl_scan(pk);
          const uint32_t tt = __shfl_sync(0xffffffffu, inc, 31);
          const uint32_t tA = tt & 0xFFFFu, tB = tt >> 16;
          if (((uint32_t)vA.x >> lane) & 1u) sl_store(w, vA, qA, arc32 + (inc & 0xFFFFu) - (uint32_t)qA.cnt, nA, eA, bnA, beA);
          if (((uint32_t)vB.x >> lane) & 1u) sl_store(w + 1, vB, qB, arc32 + tA + (inc >> 16) - (uint32_t)qB.cnt, nB, eB, bnB, beB);
          arc32 += tA + tB;
          arc += tA + tB;
          continue;
        }
        one_word(w, nA, eA, bnA, beA);
        if (twoB) one_word(w + 1, nB, eB, bnB, beB);
      }
    }
    for (int blk = fast ? bpr : warp; blk < bpr; blk += nwarp) {
      int64_t arc = __ldg(&wa.arcbase[K + (int64_t)r * bpr + blk]) - arc_comp;
      const int wb = blk * 32, nw = min(32, wpr - wb);
      for (int i = 0; i < nw; ++i) {
        const int w = wb + i;
        const int2 vv = Vr[w];
        const uint32_t vw = (uint32_t)vv.x;
        if (!vw) continue;
        const int32_t col = w * 32 + lane;
        const bool has = (vw >> lane) & 1u;
        const uint32_t hm = __ldg(&D.hmask[w]);
        const bool heavy = (hm >> lane) & 1u;
        const uint32_t* __restrict__ pe = D.ell + (size_t)__ldg(&D.woff[w]) * 32 + lane;
        const uint32_t* __restrict__ ep = D.eell + (size_t)__ldg(&D.ewoff[w]) * 32 + lane;
        const int jn = __ldg(&D.wmax[w]), ejn = __ldg(&D.ewmax[w]);
        int cnt = 0, hidx = 0, rk;
        if (has) {
          if (heavy) {
            hidx = (int)__ldg(&D.hbefore[w]) + __popc(hm & ((1u << lane) - 1u));
            cnt = __ldg(&wa.hcnt[C.hcnt_base + (int64_t)r * D.nheavy + hidx]);
          } else {
            for (unsigned long long m = meps; m; m &= m - 1ull) cnt += look(srow[__ffsll((long long)m) - 1], col, rk);
            for (int j = 0; j < ejn; ++j) {
              const uint32_t it = __ldg(ep + j * 32);
              if ((it >> 24) != 1u) continue;
              const int32_t o = (int32_t)(it & 0xFFFFFFu);
              for (unsigned long long m = meps; m; m &= m - 1ull) cnt += look(srow[__ffsll((long long)m) - 1], o, rk);
              cnt += look(r, o, rk);
            }
            for (int j = 0; j < jn; ++j) {
              const uint32_t it = __ldg(pe + j * 32);
              const int32_t o = (int32_t)(it & 0xFFFFFFu);
              if (uni) {
                cnt += (int)lc[it >> 24] * (int)look(dr0, o, rk);
              } else {
                for (unsigned long long m = lm[it >> 24]; m; m &= m - 1ull) cnt += look(srow[__ffsll((long long)m) - 1], o, rk);
              }
            }
          }
        }
        const int inc = warp_incl_scan(cnt);
        const int wtot = __shfl_sync(0xffffffffu, inc, 31);
        if (has) {
          int64_t pos = arc + inc - cnt;
          state_out(vv.y + __popc(vw & ((1u << lane) - 1u)), col, pos);
          if (heavy) {
            heavy_push(col, hidx, pos);
          } else {
            for (unsigned long long m = meps; m; m &= m - 1ull) {  // M2: B stays
              const int a = __ffsll((long long)m) - 1;
              if (look(srow[a], col, rk)) put(pos++, rk, scar[a], FST_EPS, sw[a]);
            }
            for (int j = 0; j < ejn; ++j) {  // eps items: M1 eps:eps, then M3
              const uint32_t it = __ldg(ep + j * 32);
              if ((it >> 24) != 1u) continue;
              const int32_t o = (int32_t)(it & 0xFFFFFFu);
              const int2 bw = __ldg(&D.eellcw[(ep - D.eell) + j * 32]);
              for (unsigned long long m = meps; m; m &= m - 1ull) {
                const int a = __ffsll((long long)m) - 1;
                if (look(srow[a], o, rk)) put(pos++, rk, scar[a], bw.x, __fadd_rn(sw[a], __int_as_float(bw.y)));
              }
              if (look(r, o, rk)) put(pos++, rk, FST_EPS, bw.x, __int_as_float(bw.y));
            }
            for (int j = 0; j < jn; ++j) {
              const uint32_t it = __ldg(pe + j * 32);
              const uint32_t li = it >> 24;
              const int32_t o = (int32_t)(it & 0xFFFFFFu);
              unsigned long long m = lm[li];
              if (!m) continue;
              if (uni && !look(dr0, o, rk)) continue;
              const int2 bw = __ldg(&D.ellcw[(pe - D.ell) + j * 32]);
              for (; m; m &= m - 1ull) {
                const int a = __ffsll((long long)m) - 1;
                if (uni || look(srow[a], o, rk)) put(pos++, rk, scar[a], bw.x, __fadd_rn(sw[a], __int_as_float(bw.y)));
              }
            }
          }
        }
        arc += wtot;
      }
    }
    __syncthreads();
    // heavy states: M2 (thread 0); the items split into one contiguous run per warp: each warp counts
    // its run's moves, a scan over the warps gives every run its first slot, then each warp writes its run
    // in rounds of 32 items (warp scans) -- item order = view order
    const int nq = min(hq_n, kEmHeavyQ);
    for (int q = 0; q < nq; ++q) {
      const int32_t col = hq_col[q];
      const int4 hv = __ldg(&D.heavy[hq_h[q]]);
      const int per = (hv.w - hv.y + nwarp - 1) / nwarp;
      const int c0 = hv.y + warp * per, c1 = min(hv.w, c0 + per);
      auto moves = [&](uint32_t it) -> int {
        const uint32_t li = it >> 24;
        const int32_t o = (int32_t)(it & 0xFFFFFFu);
        int c = 0, rk;
        if (it >= 0xFF000000u) return 0;
        if (fast) return (int)(lc[li] * ((((uint32_t)Vd[o >> 5].x) >> (o & 31)) & 1u)) +
                         (li == 1u ? (int)((((uint32_t)Vr[o >> 5].x) >> (o & 31)) & 1u) : 0);
        for (unsigned long long m = lm[li]; m; m &= m - 1ull) c += look(srow[__ffsll((long long)m) - 1], o, rk);
        if (li == 1u) c += look(r, o, rk);
        return c;
      };
      int wc = 0;
      for (int e = c0 + lane; e < c1; e += 32) wc += moves(__ldg(&D.hitems[e]));
      wc = warp_sum(wc);
      if (lane == 0) red[warp] = wc;
      if (tid == 0) {
        int64_t pos = hq_pos[q];
        int rk;
        for (unsigned long long m = meps; m; m &= m - 1ull) {
          const int a = __ffsll((long long)m) - 1;
          if (look(srow[a], col, rk)) put(pos++, rk, scar[a], FST_EPS, sw[a]);
        }
        hq_id[q] = pos;
      }
      __syncthreads();
      int64_t pos = hq_id[q];
      for (int k = 0; k < warp; ++k) pos += red[k];
      for (int e0i = c0; e0i < c1; e0i += 32) {
        const int e = e0i + lane;
        const uint32_t it = e < c1 ? __ldg(&D.hitems[e]) : 0xFF000000u;
        const int c = moves(it);
        const int inc = warp_incl_scan(c);
        if (c) {
          int64_t p = pos + inc - c;
          int rk;
          const uint32_t li = it >> 24;
          const int32_t o = (int32_t)(it & 0xFFFFFFu);
          const int2 bw = __ldg(&D.hcw[e]);
          for (unsigned long long m = lm[li]; m; m &= m - 1ull) {
            const int a = __ffsll((long long)m) - 1;
            if (look(srow[a], o, rk)) put(p++, rk, scar[a], bw.x, __fadd_rn(sw[a], __int_as_float(bw.y)));
          }
          if (li == 1u && look(r, o, rk)) put(p++, rk, FST_EPS, bw.x, __int_as_float(bw.y));
        }
        pos += __shfl_sync(0xffffffffu, inc, 31);
      }
      __syncthreads();
    }
    if (hq_n > kEmHeavyQ && tid == 0) atomicAdd(wa.err, 1);
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
    std::vector<int2> cw(dir == 0 ? E : 0);
    FSTC_CUDA_TRY(cudaMemcpyAsync(off.data(), v.off, sizeof(int32_t) * (V + 1), cudaMemcpyDeviceToHost, s));
    if (E) {
      FSTC_CUDA_TRY(cudaMemcpyAsync(key.data(), v.key, sizeof(int32_t) * E, cudaMemcpyDeviceToHost, s));
      FSTC_CUDA_TRY(cudaMemcpyAsync(other.data(), v.other, sizeof(int32_t) * E, cudaMemcpyDeviceToHost, s));
      if (dir == 0) FSTC_CUDA_TRY(cudaMemcpyAsync(cw.data(), v.cw, sizeof(int2) * E, cudaMemcpyDeviceToHost, s));
    }
    FSTC_CUDA_TRY(cudaStreamSynchronize(s));
    // light columns: non-eps items (label index >= 2) in `ell`, eps items in `eell` (needed only when an A
    // row has eps-output arcs: M1 eps:eps; M3 goes through the eps arc list / hubs)
    std::vector<uint32_t> woff(wpr + 1, 0), ewoff(wpr + 1, 0), hmask(wpr, 0), blab(8, 0u);
    std::vector<uint8_t> wmax(std::max(wpr, 1), 0), ewmax(std::max(wpr, 1), 0);
    std::vector<int4> heavy;
    std::vector<uint32_t> hitems, hbefore(wpr + 1, 0);
    std::vector<int2> hcw;
    std::vector<int2> eps;
    std::vector<uint32_t> rel;
    for (int w = 0; w < wpr; ++w) {
      hbefore[w] = (uint32_t)heavy.size();
      int m = 0, me = 0;
      for (int l = 0; l < 32; ++l) {
        const int32_t b = w * 32 + l;
        if (b >= V) break;
        const int deg = off[b + 1] - off[b];
        if (deg > kWHeavy) {
          const int32_t h0 = (int32_t)hitems.size();
          int32_t ne = h0;
          for (int32_t e = off[b]; e < off[b + 1]; ++e) {
            hitems.push_back(((uint32_t)(key[e] + 2) << 24) | (uint32_t)other[e]);
            if (dir == 0) hcw.push_back(cw[e]);
            if (key[e] < 0) ++ne;
          }
          heavy.push_back(make_int4(b, h0, ne, (int32_t)hitems.size()));
          hmask[w] |= 1u << l;
        } else {
          int ne = 0;
          for (int32_t e = off[b]; e < off[b + 1]; ++e) ne += key[e] < 0;
          m = std::max(m, deg - ne);
          me = std::max(me, ne);
        }
      }
      wmax[w] = (uint8_t)m;
      ewmax[w] = (uint8_t)me;
      woff[w + 1] = woff[w] + (uint32_t)m;
      ewoff[w + 1] = ewoff[w] + (uint32_t)me;
    }
    std::vector<uint32_t> ell((size_t)woff[wpr] * 32 + 32, 0xFF000000u), eell((size_t)ewoff[wpr] * 32 + 32, 0xFF000000u);
    std::vector<int2> ellcw(dir == 0 ? ell.size() : 0), eellcw(dir == 0 ? eell.size() : 0);
    for (int w = 0; w < wpr; ++w)
      for (int l = 0; l < 32; ++l) {
        const int32_t b = w * 32 + l;
        if (b >= V || ((hmask[w] >> l) & 1u)) continue;
        int j = 0, je = 0;
        for (int32_t e = off[b]; e < off[b + 1]; ++e) {
          const uint32_t li = (uint32_t)(key[e] + 2);
          const uint32_t it = (li << 24) | (uint32_t)other[e];
          if (key[e] < 0) {
            const size_t q = ((size_t)ewoff[w] + je++) * 32 + l;
            eell[q] = it;
            if (dir == 0) eellcw[q] = cw[e];
          } else {
            const size_t q = ((size_t)woff[w] + j++) * 32 + l;
            ell[q] = it;
            if (dir == 0) ellcw[q] = cw[e];
            blab[li >> 5] |= 1u << (li & 31);
          }
        }
      }
    for (int k = 0; k < 8; ++k) T.blab[k] = blab[k];
    std::vector<int32_t> hub_col;
    std::vector<uint32_t> hub_src;
    if (dir == 0) {
      std::vector<int32_t> nin(V, 0), hub_of(V, -1);
      for (int32_t b = 0; b < V; ++b)
        for (int32_t e = off[b]; e < off[b + 1] && key[e] < 0; ++e) ++nin[other[e]];
      for (int32_t t = 0; t < V && (int)hub_col.size() < kEpsHubMax; ++t)
        if (nin[t] >= kEpsHub) {
          hub_of[t] = (int32_t)hub_col.size();
          hub_col.push_back(t);
        }
      hub_src.assign(hub_col.size() * (size_t)wpr, 0u);
      for (int32_t b = 0; b < V; ++b)
        for (int32_t e = off[b]; e < off[b + 1] && key[e] < 0; ++e) {
          const int32_t t = other[e];
          if (hub_of[t] >= 0) hub_src[(size_t)hub_of[t] * wpr + (b >> 5)] |= 1u << (b & 31);
          else eps.push_back(make_int2(b, t));
        }
      rel.assign(4 * (size_t)wpr, 0u);
      auto setb = [&](int k, int32_t c) { rel[(size_t)k * wpr + (c >> 5)] |= 1u << (c & 31); };
      for (const int2& a : eps) {
        setb(0, a.y);
        setb(1, a.y);
        setb(3, a.x);
      }
      for (int32_t t : hub_col) setb(1, t);
      for (size_t i = 0; i < hub_src.size(); ++i) {
        rel[2 * (size_t)wpr + i % wpr] |= hub_src[i];
        rel[3 * (size_t)wpr + i % wpr] |= hub_src[i];
      }
    }
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o += (bytes + 255) & ~size_t(255); return r; };
    const size_t o_eell = take(4 * eell.size()), o_ewoff = take(4 * ewoff.size()), o_ewmax = take(ewmax.size());
    std::vector<uint32_t> wo(wpr + 1, 0), ewo(wpr + 1, 0);
    for (int w = 0; w < wpr; ++w) {
      wo[w] = (woff[w] << 8) | wmax[w];
      ewo[w] = (ewoff[w] << 8) | ewmax[w];
    }
    if (woff[wpr] >= (1u << 24) || ewoff[wpr] >= (1u << 24)) {
      set_error(FST_E_CAPACITY, "wave ELL too large");
      return FST_E_CAPACITY;
    }
    const size_t o_wo = take(4 * wo.size()), o_ewo = take(4 * ewo.size());
    const size_t o_ellcw = take(8 * std::max<size_t>(ellcw.size(), 1)), o_eellcw = take(8 * std::max<size_t>(eellcw.size(), 1)),
                 o_hcw = take(8 * std::max<size_t>(hcw.size(), 1)), o_hb = take(4 * hbefore.size());
    const size_t o_ell = take(4 * ell.size()), o_woff = take(4 * woff.size()), o_wmax = take(wmax.size()),
                 o_hm = take(4 * std::max<size_t>(hmask.size(), 1)), o_h = take(16 * std::max<size_t>(heavy.size(), 1)),
                 o_e = take(8 * std::max<size_t>(eps.size(), 1)), o_hc = take(4 * std::max<size_t>(hub_col.size(), 1)),
                 o_hs = take(4 * std::max<size_t>(hub_src.size(), 1)), o_hi = take(4 * std::max<size_t>(hitems.size(), 1)),
                 o_rel = take(4 * std::max<size_t>(rel.size(), 1));
    BufferPtr buf;
    fst_status st = alloc_buffer(o, s, &buf);
    if (st) return st;
    char* base = (char*)buf->ptr;
    T.wo = (uint32_t*)(base + o_wo);
    T.ewo = (uint32_t*)(base + o_ewo);
    FSTC_CUDA_TRY(cudaMemcpyAsync(T.wo, wo.data(), 4 * wo.size(), cudaMemcpyHostToDevice, s));
    FSTC_CUDA_TRY(cudaMemcpyAsync(T.ewo, ewo.data(), 4 * ewo.size(), cudaMemcpyHostToDevice, s));
    T.ellcw = (int2*)(base + o_ellcw);
    T.eellcw = (int2*)(base + o_eellcw);
    T.hcw = (int2*)(base + o_hcw);
    T.hbefore = (uint32_t*)(base + o_hb);
    if (!ellcw.empty()) FSTC_CUDA_TRY(cudaMemcpyAsync(T.ellcw, ellcw.data(), 8 * ellcw.size(), cudaMemcpyHostToDevice, s));
    if (!eellcw.empty()) FSTC_CUDA_TRY(cudaMemcpyAsync(T.eellcw, eellcw.data(), 8 * eellcw.size(), cudaMemcpyHostToDevice, s));
    if (!hcw.empty()) FSTC_CUDA_TRY(cudaMemcpyAsync(T.hcw, hcw.data(), 8 * hcw.size(), cudaMemcpyHostToDevice, s));
    FSTC_CUDA_TRY(cudaMemcpyAsync(T.hbefore, hbefore.data(), 4 * hbefore.size(), cudaMemcpyHostToDevice, s));
    T.eell = (uint32_t*)(base + o_eell);
    T.ewoff = (uint32_t*)(base + o_ewoff);
    T.ewmax = (uint8_t*)(base + o_ewmax);
    T.ell = (uint32_t*)(base + o_ell);
    T.woff = (uint32_t*)(base + o_woff);
    T.wmax = (uint8_t*)(base + o_wmax);
    T.hmask = (uint32_t*)(base + o_hm);
    T.heavy = (int4*)(base + o_h);
    T.eps = (int2*)(base + o_e);
    T.hub_col = (int32_t*)(base + o_hc);
    T.hub_src = (uint32_t*)(base + o_hs);
    T.nhub = (int32_t)hub_col.size();
    T.hitems = (uint32_t*)(base + o_hi);
    T.rel = (uint32_t*)(base + o_rel);
    T.nheavy = (int32_t)heavy.size();
    T.neps = (int32_t)eps.size();
    FSTC_CUDA_TRY(cudaMemcpyAsync(T.ell, ell.data(), 4 * ell.size(), cudaMemcpyHostToDevice, s));
    FSTC_CUDA_TRY(cudaMemcpyAsync(T.eell, eell.data(), 4 * eell.size(), cudaMemcpyHostToDevice, s));
    FSTC_CUDA_TRY(cudaMemcpyAsync(T.ewoff, ewoff.data(), 4 * ewoff.size(), cudaMemcpyHostToDevice, s));
    FSTC_CUDA_TRY(cudaMemcpyAsync(T.ewmax, ewmax.data(), ewmax.size(), cudaMemcpyHostToDevice, s));
    FSTC_CUDA_TRY(cudaMemcpyAsync(T.woff, woff.data(), 4 * woff.size(), cudaMemcpyHostToDevice, s));
    FSTC_CUDA_TRY(cudaMemcpyAsync(T.wmax, wmax.data(), wmax.size(), cudaMemcpyHostToDevice, s));
    if (!hmask.empty()) FSTC_CUDA_TRY(cudaMemcpyAsync(T.hmask, hmask.data(), 4 * hmask.size(), cudaMemcpyHostToDevice, s));
    if (!heavy.empty()) FSTC_CUDA_TRY(cudaMemcpyAsync(T.heavy, heavy.data(), 16 * heavy.size(), cudaMemcpyHostToDevice, s));
    if (!eps.empty()) FSTC_CUDA_TRY(cudaMemcpyAsync(T.eps, eps.data(), 8 * eps.size(), cudaMemcpyHostToDevice, s));
    if (!hitems.empty()) FSTC_CUDA_TRY(cudaMemcpyAsync(T.hitems, hitems.data(), 4 * hitems.size(), cudaMemcpyHostToDevice, s));
    if (!rel.empty()) FSTC_CUDA_TRY(cudaMemcpyAsync(T.rel, rel.data(), 4 * rel.size(), cudaMemcpyHostToDevice, s));
    if (!hub_col.empty()) {
      FSTC_CUDA_TRY(cudaMemcpyAsync(T.hub_col, hub_col.data(), 4 * hub_col.size(), cudaMemcpyHostToDevice, s));
      FSTC_CUDA_TRY(cudaMemcpyAsync(T.hub_src, hub_src.data(), 4 * hub_src.size(), cudaMemcpyHostToDevice, s));
    }
    FSTC_CUDA_TRY(cudaStreamSynchronize(s));
    T.buf = buf;
    T.ok = true;
  }
  return FST_OK;
}

constexpr size_t kWSmem = 225 * 1024;  // dynamic shared memory of a stage CTA (one CTA per SM; + static)

// shared memory of a stage CTA without the ELL cache (the cache takes the rest of kWSmem)
size_t wave_smem(int wprmax, int G, bool s2) {
  const int rng = (wprmax + G - 1) / G;
  return 8 * kWLab + 4 * kWSlots + 4 * 32 + 4 * (kWLab / 32) + 4 * (size_t)(2 * wprmax + (s2 ? 2 * wprmax : 0) + 3 * rng);
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
  uint32_t cw1 = 0, cw2 = 0;
  int64_t nblocks = 0;
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
  static std::atomic<bool> attr_done{false};
  if (wave_smem(wprmax, 1, true) + 1024 > kWSmem) return FST_OK;  // rows too wide for the staged row copies
  if (!attr_done) {
    FSTC_CUDA_TRY(cudaFuncSetAttribute(k_wave<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWSmem));
    FSTC_CUDA_TRY(cudaFuncSetAttribute(k_wave<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWSmem));
    attr_done = true;
  }
  WavePlan::Impl& P = *plan->impl;
  // cluster size: LPT makespan (in rows, compositions taken longest first by the next free cluster)
  // times the per-row cost of a G-CTA cluster (its words per CTA + a fixed per-row overhead)
  std::vector<int32_t> rows_desc(n);
  for (int i = 0; i < n; ++i) rows_desc[i] = a[i]->V;
  std::sort(rows_desc.begin(), rows_desc.end(), std::greater<int32_t>());
  P.G1 = P.G2 = 1;
  double best = -1.0;
  for (int G : {8, 4, 2, 1}) {
    if (G > 1 && wprmax < 32 * G) continue;
    const int c = max_clusters<true>(G, kWSmem);
    if (c <= 0) continue;
    std::vector<int64_t> load(std::min(c, n), 0);
    for (int32_t rws : rows_desc) *std::min_element(load.begin(), load.end()) += rws;
    // per-row cost: words per CTA + a cluster overhead growing with G (barrier, DSMEM gather); fitted to
    // configs[4] (G = 1 / 2 / 4 / 8: 30 / 14 / 10 / 11 us per row step)
    const double cost = (double)*std::max_element(load.begin(), load.end()) * ((double)wprmax / G + 128.0 * G);
    if (best < 0 || cost < best) {
      best = cost;
      P.G1 = P.G2 = G;
    }
  }
  if (const char* e = getenv("FSTC_WAVE_G")) {  // A/B: a fixed cluster size
    const int g = atoi(e);
    if (g == 1 || g == 2 || g == 4 || g == 8) P.G1 = P.G2 = g;
  }
  P.smem1 = P.smem2 = kWSmem;
  P.cw1 = (uint32_t)((kWSmem - wave_smem(wprmax, P.G1, false)) / 4);
  P.cw2 = (uint32_t)((kWSmem - wave_smem(wprmax, P.G2, true)) / 4);
  P.nc1 = max_clusters<false>(P.G1, P.smem1);
  P.nc2 = max_clusters<true>(P.G2, P.smem2);
  if (P.nc1 <= 0 || P.nc2 <= 0) return FST_OK;
  P.nc1 = std::min(P.nc1, n);
  P.nc2 = std::min(P.nc2, n);
  // per-composition descriptors
  std::vector<WaveComp> comps(n);
  std::vector<int32_t> order(n);
  int64_t rows = 0, hrows = 0;
  for (int i = 0; i < n; ++i) {
    fst* A = a[i];
    fst* B = b[i];
    WaveComp& C = comps[i];
    memset(&C, 0, sizeof(C));
    C.W = W[i];
    C.K = K[i];
    C.rowbase = rows;
    C.hcnt_base = hrows;
    hrows += (int64_t)A->V * B->wave_ell[0].nheavy;
    rows += A->V;
    C.VA = A->V;
    C.VB = B->V;
    C.wpr = (B->V + 31) / 32;
    C.bpr = (C.wpr + kWordsPerBlock - 1) / kWordsPerBlock;
    P.nblocks = std::max<int64_t>(P.nblocks, C.K + (int64_t)C.VA * C.bpr);
    for (int d = 0; d < 2; ++d) {
      const View& av = A->views[d == 0 ? kOutByOlabel : kInByOlabel];
      C.aoff[d] = av.off;
      C.akey[d] = av.key;
      C.aother[d] = av.other;
      const View& bv = B->views[d == 0 ? kOutByIlabel : kInByIlabel];
      const fst::WaveEll& T = B->wave_ell[d];
      C.bd[d] = WaveDir{T.ell, T.woff, T.wmax, T.eell, T.ewoff, T.ewmax, T.hmask, T.heavy, T.nheavy, T.hitems, {},
                        T.ellcw, T.eellcw, T.hcw, T.hbefore, T.wo, T.ewo};
      for (int k = 0; k < 8; ++k) C.bd[d].blab[k] = T.blab[k];
      (void)bv;
    }
    C.startA = A->is_start;
    C.accA = A->is_accept;
    C.startB = B->is_start;
    C.accB = B->is_accept;
    C.eps = B->wave_ell[0].eps;
    C.neps = B->wave_ell[0].neps;
    C.nhub = B->wave_ell[0].nhub;
    C.hub_col = B->wave_ell[0].hub_col;
    C.hub_src = B->wave_ell[0].hub_src;
    for (int k = 0; k < 4; ++k) C.rel[k] = B->wave_ell[0].rel + (size_t)k * C.wpr;
    order[i] = i;
  }
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return comps[x].VA > comps[y].VA; });
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o += (bytes + 255) & ~size_t(255); return r; };
  const size_t o_c = take(sizeof(WaveComp) * n), o_o = take(4 * n), o_n = take(8), o_h = take(4 * std::max<int64_t>(hrows, 1));
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
  P.wa.hcnt = (int32_t*)(base + o_h);
  P.wa.nrows = rows;
  plan->ok = true;
  {  // the wave emit stages 32 bytes per word of the widest row: wider rows take the general emit
    static const size_t emit_limit = [] {
      int dev = 0, optin = 0;
      cudaFuncAttributes fa{};
      if (cudaGetDevice(&dev) != cudaSuccess ||
          cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess ||
          cudaFuncGetAttributes(&fa, k_wave_emit) != cudaSuccess)
        return (size_t)0;
      return (size_t)optin > fa.sharedSizeBytes ? (size_t)optin - fa.sharedSizeBytes : (size_t)0;
    }();
    plan->emit_ok = 32ull * (size_t)wprmax <= emit_limit;
  }
  plan->depth = maxrows;
  plan->cluster = P.G2;
  return FST_OK;
}

fst_status wave_stage(const WavePlan& plan, int stage, uint32_t* R, uint32_t* V, cudaStream_t s) {
  WavePlan::Impl& P = *plan.impl;
  P.wa.R = R;
  P.wa.V = V;
  FSTC_CUDA_TRY(cudaMemsetAsync(P.wa.next, 0, 4, s));
  static const bool nocache = [] {  // FSTC_WAVE_CACHE=0: items from global memory (tests / A-B)
    const char* e = getenv("FSTC_WAVE_CACHE");
    return e && e[0] == '0';
  }();
  P.wa.cache_words = nocache ? 0u : (stage == 1 ? P.cw1 : P.cw2);
  static const bool probe_on = [] {
    const char* e = getenv("FSTC_WAVE_PROBE");
    return e && e[0] == '1';
  }();
  static long long* d_probe = nullptr;
  const int ncl = stage == 1 ? P.nc1 : P.nc2;
  if (probe_on && !d_probe) FSTC_CUDA_TRY(cudaMalloc(&d_probe, 8 * 8 * 1024));
  if (probe_on) FSTC_CUDA_TRY(cudaMemsetAsync(d_probe, 0, 8 * 8 * 1024, s));
  P.wa.probe = probe_on ? d_probe : nullptr;
  if (probe_on) {
    fst_status st = stage == 1 ? launch_wave<false>(P.wa, P.G1, P.nc1, P.smem1, s) : launch_wave<true>(P.wa, P.G2, P.nc2, P.smem2, s);
    if (st) return st;
    std::vector<long long> h(8 * 1024);
    FSTC_CUDA_TRY(cudaMemcpyAsync(h.data(), d_probe, 8 * 8 * ncl, cudaMemcpyDeviceToHost, s));
    FSTC_CUDA_TRY(cudaStreamSynchronize(s));
    int best = 0;
    for (int c = 0; c < ncl; ++c)
      if (h[c * 8 + 7] > h[best * 8 + 7]) best = c;
    const double rows = (double)std::max(1ll, h[best * 8 + 7]);
    fprintf(stderr, "wave probe stage %d cluster %d rows %.0f cycles/row: setup %.0f pull %.0f heavy %.0f csync %.0f gather %.0f closure %.0f store %.0f\n",
            stage, best, rows, h[best * 8 + 0] / rows, h[best * 8 + 1] / rows, h[best * 8 + 2] / rows, h[best * 8 + 3] / rows,
            h[best * 8 + 4] / rows, h[best * 8 + 5] / rows, h[best * 8 + 6] / rows);
    P.wa.probe = nullptr;
    return FST_OK;
  }
  return stage == 1 ? launch_wave<false>(P.wa, P.G1, P.nc1, P.smem1, s) : launch_wave<true>(P.wa, P.G2, P.nc2, P.smem2, s);
}

fst_status wave_count(const WavePlan& plan, uint32_t* R, uint8_t* cnt8, cudaStream_t s) {
  WavePlan::Impl& P = *plan.impl;
  P.wa.R = R;
  P.wa.cnt8 = cnt8;
  const size_t smem = 8ull * P.wa.wprmax;
  static std::atomic<size_t> smem_set{0};
  if (smem > smem_set) {  // (dynamic + static may pass the 48 KB default below that size)
    FSTC_CUDA_TRY(cudaFuncSetAttribute(k_wave_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    smem_set = smem;
  }
  // one CTA per row (not persistent): CTAs retire quickly, so a higher-priority stream (the longer
  // half of a split batch) gets SMs as soon as it needs them
  const int64_t grid = std::min<int64_t>(std::max<int64_t>(P.wa.nrows, 1), (int64_t)INT32_MAX);
  k_wave_count<<<(unsigned)grid, kCThreads, smem, s>>>(P.wa);
  FSTC_LAUNCH_CHECK();
  return FST_OK;
}

fst_status wave_kept(const WavePlan& plan, uint32_t* V, unsigned long long* kept, cudaStream_t s) {
  WavePlan::Impl& P = *plan.impl;
  P.wa.V = V;
  P.wa.kept = kept;
  const int64_t warps = std::max<int64_t>(P.nblocks, 1);
  const int64_t grid = std::min<int64_t>((warps + 7) / 8, (int64_t)sm_count() * 16);
  k_wave_kept<<<(unsigned)grid, 256, 0, s>>>(P.wa, P.nblocks);
  FSTC_LAUNCH_CHECK();
  return FST_OK;
}

fst_status wave_emit(const WavePlan& plan, const CompDev* d_comps, const int64_t* d_tot, const int64_t* idbase,
                     const int64_t* arcbase, const uint16_t* wpre, uint32_t* V, int32_t* err, cudaStream_t s) {
  WavePlan::Impl& P = *plan.impl;
  P.wa.V = V;
  P.wa.idbase = idbase;
  P.wa.arcbase = arcbase;
  P.wa.wpre = wpre;
  P.wa.err = err;
  const size_t smem = 32ull * P.wa.wprmax;
  static std::atomic<size_t> smem_set{0};
  if (smem > smem_set) {  // (dynamic + static may pass the 48 KB default below that size)
    FSTC_CUDA_TRY(cudaFuncSetAttribute(k_wave_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    smem_set = smem;
  }
  // one CTA per row (not persistent): CTAs retire quickly, so a higher-priority stream (the longer
  // half of a split batch) gets SMs as soon as it needs them
  const int64_t grid = std::min<int64_t>(std::max<int64_t>(P.wa.nrows, 1), (int64_t)INT32_MAX);
  k_wave_emit<<<(unsigned)grid, kEmThreads, smem, s>>>(P.wa, d_comps, d_tot);
  FSTC_LAUNCH_CHECK();
  return FST_OK;
}

}  // namespace fstc
